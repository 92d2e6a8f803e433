"""Grid conversion P / P^T between deformation and image grids (drop-in for ngfreg.transfer).

The index maps and gather plans are computed by libngfb200's host code in IEEE
f64 (bit-exact with transfer.py:54-110); P and P^T run as sm_100a kernels that
reproduce the reference operation order (transfer.py:117-192).  The three reference
P^T variants run as their own kernels (transfer.py:173-256): "gather" and "redblack"
bit-identical to the reference, "scatter" with float atomics (equal up to
reassociation, as the reference's lock-based scatter, pkg/README.md:33-39).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device as dev
from ._lib import GridError, check, dtype_code, lib, ngf_grid
from .geometry import DeformationField, Grid3, VectorField3

__all__ = ["AxisPlan", "GatherPlan", "PT_VARIANTS", "apply_P", "apply_Pt", "apply_Pt_gather",
           "apply_Pt_redblack", "apply_Pt_scatter_atomic", "axis_transfer", "build_gather_plan",
           "check_compatible", "dense_P_oracle"]

PT_VARIANTS = ("gather", "scatter", "redblack")


def check_compatible(def_grid: Grid3, image_grid: Grid3) -> None:
    """transfer.py:42-51 (host check, raises GridError like the reference)."""
    if not def_grid.same_extent(image_grid):
        raise GridError(f"deformation grid extent {def_grid.extent} (min {def_grid.domain_min}) "
                        f"does not match image grid extent {image_grid.extent} "
                        f"(min {image_grid.domain_min})")
    if any(mi < md for mi, md in zip(image_grid.dims, def_grid.dims)):
        raise GridError(f"image grid dims {image_grid.dims} must be >= deformation grid dims "
                        f"{def_grid.dims}")


@dataclass(frozen=True)
class AxisPlan:
    start: np.ndarray
    counts: np.ndarray
    weights: np.ndarray


class _Plan:
    """Owns one ngf_plan_t (host f64 maps + device copies)."""

    def __init__(self, def_grid: Grid3, image_grid: Grid3, prolong: bool = False):
        self.def_grid, self.image_grid = def_grid, image_grid
        h = ctypes.c_void_p()
        fn = lib().ngf_plan_create_prolong if prolong else lib().ngf_plan_create
        check(fn(ctypes.byref(ngf_grid(def_grid)), ctypes.byref(ngf_grid(image_grid)),
                 ctypes.byref(h)), "ngf_plan_create")
        self.handle = h

    def axis(self, a: int):
        ni, nd = self.image_grid.dims[a], self.def_grid.dims[a]
        width = ctypes.c_int32()
        check(lib().ngf_plan_axis(self.handle, a, None, None, None, None, None,
                                  ctypes.byref(width)), "ngf_plan_axis")
        i0 = np.empty(ni, np.int32)
        w1 = np.empty(ni, np.float64)
        st = np.empty(nd, np.int32)
        cnt = np.empty(nd, np.int32)
        w = np.empty((nd, width.value), np.float64)
        check(lib().ngf_plan_axis(self.handle, a, i0.ctypes.data, w1.ctypes.data, st.ctypes.data,
                                  cnt.ctypes.data, w.ctypes.data, ctypes.byref(width)),
              "ngf_plan_axis")
        return i0.astype(np.intp), w1, st.astype(np.intp), cnt.astype(np.intp), w

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib().ngf_plan_destroy(h)
            except Exception:
                pass
            self.handle = None


class GatherPlan:
    """Per-axis transposed interpolation plan (transfer.py:66-110)."""

    def __init__(self, def_grid: Grid3, image_grid: Grid3, _plan: _Plan | None = None):
        self.def_grid = def_grid
        self.image_grid = image_grid
        self._plan = _plan or _Plan(def_grid, image_grid)
        self._axes = None

    @property
    def handle(self):
        return self._plan.handle

    @property
    def axes(self):
        if self._axes is None:
            out = []
            for a in range(3):
                _, _, st, cnt, w = self._plan.axis(a)
                out.append(AxisPlan(start=st, counts=cnt, weights=w))
            self._axes = tuple(out)
        return self._axes


def build_gather_plan(def_grid: Grid3, image_grid: Grid3) -> GatherPlan:
    check_compatible(def_grid, image_grid)
    return GatherPlan(def_grid, image_grid)


def axis_transfer(image_grid: Grid3, def_grid: Grid3, axis: int):
    """(i0, w1) of transfer.py:54-63, computed by the library's host f64 code."""
    if not def_grid.same_extent(image_grid):
        raise GridError("grids must cover the same world domain")
    i0, w1, _, _, _ = _Plan(def_grid, image_grid, prolong=True).axis(axis)
    return i0, w1


_axis_transfer = axis_transfer


def _field_io(field):
    """(device tensor, was_numpy)"""
    return dev.to_device(field), not dev.is_tensor(field)


def _ret(grid, t, numpy_out, cls=VectorField3):
    return cls(grid, dev.to_host(t) if numpy_out else t)


def apply_P(y: DeformationField, image_grid: Grid3, workers: int = 1, plan: GatherPlan | None = None):
    """yhat = P y (transfer.py:129-148); bit-exact, numpy in -> numpy out."""
    check_compatible(y.grid, image_grid)
    plan = plan or GatherPlan(y.grid, image_grid)
    yd, np_out = _field_io(y.field)
    out = dev.empty((3,) + image_grid.shape, yd.dtype)
    check(lib().ngf_apply_P(plan.handle, dtype_code(yd.dtype), dev.ptr(yd), dev.ptr(out),
                            dev.stream()), "ngf_apply_P")
    return _ret(image_grid, out, np_out)


def apply_Pt_gather(r: VectorField3, plan: GatherPlan, workers: int = 1):
    """Deterministic gather P^T (transfer.py:173-192)."""
    if r.grid != plan.image_grid:
        raise GridError("input field grid does not match the plan's image grid")
    rd, np_out = _field_io(r.field)
    out = dev.empty((3,) + plan.def_grid.shape, rd.dtype)
    check(lib().ngf_apply_Pt(plan.handle, dtype_code(rd.dtype), dev.ptr(rd), dev.ptr(out),
                             dev.stream()), "ngf_apply_Pt")
    return _ret(plan.def_grid, out, np_out)


def _apply_Pt_variant(r: VectorField3, plan: GatherPlan, variant: int, name: str):
    rd, np_out = _field_io(r.field)
    out = dev.empty((3,) + plan.def_grid.shape, rd.dtype)
    check(lib().ngf_apply_Pt_variant(plan.handle, dtype_code(rd.dtype), variant, dev.ptr(rd),
                                     dev.ptr(out), dev.stream()), name)
    return _ret(plan.def_grid, out, np_out)


def apply_Pt_scatter_atomic(r: VectorField3, def_grid: Grid3, workers: int = 1):
    """P^T by scattering the x/y-reduced image slices onto their two def planes with
    float atomics (transfer.py:199-222): equal to the gather up to floating-point
    reassociation, like the reference's lock-based scatter."""
    check_compatible(def_grid, r.grid)
    return _apply_Pt_variant(r, GatherPlan(def_grid, r.grid), 1, "ngf_apply_Pt_variant(scatter)")


def apply_Pt_redblack(r: VectorField3, def_grid: Grid3, workers: int = 1):
    """P^T with slices grouped by target def plane, even then odd groups
    (transfer.py:225-256); bit-identical to the reference's red-black."""
    check_compatible(def_grid, r.grid)
    return _apply_Pt_variant(r, GatherPlan(def_grid, r.grid), 2, "ngf_apply_Pt_variant(redblack)")


def apply_Pt(r: VectorField3, plan: GatherPlan, variant: str = "gather", workers: int = 1):
    """Dispatcher (transfer.py:259-266)."""
    if variant == "gather":
        return apply_Pt_gather(r, plan, workers)
    if variant == "scatter":
        check_compatible(plan.def_grid, r.grid)
        return _apply_Pt_variant(r, plan, 1, "ngf_apply_Pt_variant(scatter)")
    if variant == "redblack":
        check_compatible(plan.def_grid, r.grid)
        return _apply_Pt_variant(r, plan, 2, "ngf_apply_Pt_variant(redblack)")
    raise ValueError(f"unknown P^T variant {variant!r}, expected one of {PT_VARIANTS}")


def dense_P_oracle(def_grid: Grid3, image_grid: Grid3) -> np.ndarray:
    """Explicit (m_image, m_def) matrix of one component of P (transfer.py:269-287); test-only,
    built from the library's f64 index maps."""
    check_compatible(def_grid, image_grid)
    if image_grid.num_points > 512 or def_grid.num_points > 512:
        raise ValueError("dense_P_oracle is limited to grids of at most 8^3 points")
    mats = []
    for a in range(3):
        i0, w1 = axis_transfer(image_grid, def_grid, a)
        ni, nd = image_grid.dims[a], def_grid.dims[a]
        A = np.zeros((ni, nd))
        rows = np.arange(ni)
        np.add.at(A, (rows, i0), 1.0 - w1)
        np.add.at(A, (rows, np.minimum(i0 + 1, nd - 1)), w1)
        mats.append(A)
    return np.kron(mats[2], np.kron(mats[1], mats[0]))
