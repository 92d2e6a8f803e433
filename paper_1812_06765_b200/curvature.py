"""Curvature regulariser S = (vol/2) sum_c ||L u_c||^2 on the displacement
(drop-in for ngfreg.curvature; reference curvature.py:1-81).

L is the 7-point Laplacian with zero rows at the faces (linear extrapolation),
so affine maps are in its null space; grad S = vol L^T L u.  Kernels follow
the reference operation order, including the pairwise f32/f64 sum of S.
"""

from __future__ import annotations

import ctypes

from . import _device as dev
from ._lib import check, dtype_code, lib, ngf_grid
from .geometry import DeformationField, Grid3

__all__ = ["apply_laplacian", "apply_laplacian_transpose", "curvature_gradient", "curvature_value"]


def _one(fn, u, grid: Grid3, name: str):
    np_out = not dev.is_tensor(u)
    ud = dev.to_device(u)
    out = dev.empty(grid.shape, ud.dtype)
    check(fn(ctypes.byref(ngf_grid(grid)), dtype_code(ud.dtype), dev.ptr(ud), dev.ptr(out),
             dev.stream()), name)
    return dev.to_host(out) if np_out else out


def apply_laplacian(u, grid: Grid3):
    """curvature.py:48-53 (one scalar component)."""
    return _one(lib().ngf_laplacian, u, grid, "ngf_laplacian")


def apply_laplacian_transpose(w, grid: Grid3):
    """curvature.py:56-60."""
    return _one(lib().ngf_laplacian_t, w, grid, "ngf_laplacian_t")


def _curv(y: DeformationField, want_value: bool, want_grad: bool):
    yd = dev.to_device(y.field)
    S = dev.zeros((1,), "float64") if want_value else None
    grad = dev.empty((3,) + y.grid.shape, yd.dtype) if want_grad else None
    check(lib().ngf_curvature(ctypes.byref(ngf_grid(y.grid)), dtype_code(yd.dtype), dev.ptr(yd),
                              dev.ptr(S), dev.ptr(grad), dev.stream()), "ngf_curvature")
    return S, grad


def curvature_value(y: DeformationField) -> float:
    """S (curvature.py:63-71)."""
    S, _ = _curv(y, True, False)
    return float(S.item())


def curvature_gradient(y: DeformationField):
    """vol L^T L u per component (curvature.py:74-81)."""
    _, g = _curv(y, False, True)
    return g if dev.is_tensor(y.field) else dev.to_host(g)
