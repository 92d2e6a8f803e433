"""Template warping and image-grid finite differences (drop-in for ngfreg.warp).

Each operator is one sm_100a kernel reproducing the reference's operation
order (warp.py:26-184 of the reference), so results are bit-identical.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device as dev
from ._lib import check, dtype_code, lib, ngf_grid
from .geometry import Grid3, Image3, VectorField3

__all__ = ["WarpResult", "image_gradient", "image_gradient_apply_transpose", "warp_image",
           "warp_jacobian_apply_transpose"]


@dataclass
class WarpResult:
    warped: Image3
    inside_mask: object


def warp_image(template: Image3, yhat: VectorField3, workers: int = 1) -> WarpResult:
    """Trilinear T(yhat), Dirichlet zero outside the cell-centre hull (warp.py:64-90)."""
    np_out = not dev.is_tensor(yhat.field)
    yd = dev.to_device(yhat.field)
    Td = dev.to_device(template.values, dev.np_dtype(yd.dtype))
    n = yhat.grid.num_points
    W = dev.empty(yhat.grid.shape, yd.dtype)
    mask = dev.torch().empty(yhat.grid.shape, dtype=dev.torch().uint8, device="cuda")
    check(lib().ngf_warp(ctypes.byref(ngf_grid(template.grid)), dtype_code(yd.dtype), dev.ptr(Td),
                         dev.ptr(yd), n, dev.ptr(W), dev.ptr(mask), dev.stream()), "ngf_warp")
    if np_out:
        return WarpResult(Image3(yhat.grid, dev.to_host(W)), dev.to_host(mask).astype(bool))
    return WarpResult(Image3(yhat.grid, W), mask.bool())


def warp_jacobian_apply_transpose(template: Image3, yhat: VectorField3, w, workers: int = 1):
    """Per voxel w * grad of the trilinear interpolant / h, zero outside (warp.py:93-127)."""
    np_out = not dev.is_tensor(yhat.field)
    yd = dev.to_device(yhat.field)
    dt = dev.np_dtype(yd.dtype)
    Td = dev.to_device(template.values, dt)
    wd = dev.to_device(w, dt)
    out = dev.empty((3,) + yhat.grid.shape, yd.dtype)
    check(lib().ngf_warp_jt(ctypes.byref(ngf_grid(template.grid)), dtype_code(yd.dtype),
                            dev.ptr(Td), dev.ptr(yd), dev.ptr(wd), yhat.grid.num_points,
                            dev.ptr(out), dev.stream()), "ngf_warp_jt")
    return VectorField3(yhat.grid, dev.to_host(out) if np_out else out)


def image_gradient(img: Image3, workers: int = 1) -> VectorField3:
    """Central differences inside, one-sided at faces (warp.py:130-152)."""
    np_out = not dev.is_tensor(img.values)
    v = dev.to_device(img.values)
    out = dev.empty((3,) + img.grid.shape, v.dtype)
    check(lib().ngf_gradient(ctypes.byref(ngf_grid(img.grid)), dtype_code(v.dtype), dev.ptr(v),
                             dev.ptr(out), dev.stream()), "ngf_gradient")
    return VectorField3(img.grid, dev.to_host(out) if np_out else out)


def image_gradient_apply_transpose(w: VectorField3, grid: Grid3):
    """Exact G^T (warp.py:159-184)."""
    np_out = not dev.is_tensor(w.field)
    wd = dev.to_device(w.field)
    out = dev.empty(grid.shape, wd.dtype)
    check(lib().ngf_gradient_t(ctypes.byref(ngf_grid(grid)), dtype_code(wd.dtype), dev.ptr(wd),
                               dev.ptr(out), dev.stream()), "ngf_gradient_t")
    return dev.to_host(out) if np_out else out
