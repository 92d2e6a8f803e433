"""Joint level objective J(y) = D_NGF + alpha * S_curvature (drop-in for ngfreg.objective).

The flat variable is the component-major ravel of the (3, nz, ny, nx) field
(reference objective.py:1-6).  One evaluation is one call into libngfb200:
the fused sm_100a pipeline (mode 0, default) or the bit-exact reference-order
pipeline (mode 1, `exact=True`).  `__call__` keeps the reference contract
(numpy in, (float, numpy) out, inf + zeros on a non-finite trial point);
`eval_device` is the device-resident path the L-BFGS driver uses.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device as dev
from ._lib import check, dtype_code, lib, ngf_grid
from .geometry import DeformationField, Grid3, Image3
from .ngf import NgfParams, ReferenceTerms
from .transfer import PT_VARIANTS, GatherPlan

__all__ = ["LevelObjective", "DeviceLevel"]


class DeviceLevel:
    """Owns one ngf_level_t: template, reference terms, fused workspace."""

    def __init__(self, image_grid: Grid3, def_grid: Grid3, T_dev, params: NgfParams, alpha: float,
                 R_dev=None, gR_dev=None, nR_dev=None):
        self.image_grid, self.def_grid = image_grid, def_grid
        self.dtype = T_dev.dtype
        self.T = T_dev  # kept alive: the level reads it on every evaluation
        self.alpha = float(alpha)
        h = ctypes.c_void_p()
        ig, dg = ngf_grid(image_grid), ngf_grid(def_grid)
        code = dtype_code(self.dtype)
        if R_dev is not None:
            rc = lib().ngf_level_create(ctypes.byref(ig), ctypes.byref(dg), code, dev.ptr(T_dev),
                                        dev.ptr(R_dev), float(params.tau), float(params.rho),
                                        self.alpha, dev.stream(), ctypes.byref(h))
        else:
            rc = lib().ngf_level_create_terms(ctypes.byref(ig), ctypes.byref(dg), code,
                                              dev.ptr(T_dev), dev.ptr(gR_dev), dev.ptr(nR_dev),
                                              float(params.tau), float(params.rho), self.alpha,
                                              dev.stream(), ctypes.byref(h))
        check(rc, "ngf_level_create")
        self.handle = h
        self.n = 3 * def_grid.num_points
        self.scalars = dev.zeros((3,), "float64")

    def eval(self, y_dev, grad_dev, scalars_dev=None, exact: bool = False):
        """Launch one evaluation (no host sync); scalars_dev <- (J, D, S)."""
        sc = self.scalars if scalars_dev is None else scalars_dev
        check(lib().ngf_level_eval(self.handle, dev.ptr(y_dev), dev.ptr(grad_dev), dev.ptr(sc),
                                   1 if exact else 0, dev.stream()), "ngf_level_eval")
        return sc

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib().ngf_level_destroy(h)
            except Exception:
                pass
            self.handle = None


@dataclass
class LevelObjective:
    """Callable objective for one multilevel level; records the last D/S split
    (objective.py:22-60)."""

    template: Image3
    ref: ReferenceTerms
    plan: GatherPlan
    params: NgfParams
    alpha: float
    pt_variant: str = "gather"
    workers: int = 1
    last_D: float = 0.0
    last_S: float = 0.0
    exact: bool = False
    evals: int = 0
    _level: DeviceLevel | None = field(default=None, repr=False)
    _R_dev: object = field(default=None, repr=False)
    _sc_host: np.ndarray = field(default_factory=lambda: np.zeros(3), repr=False)

    def __post_init__(self):
        if self.pt_variant not in PT_VARIANTS:
            raise ValueError(f"unknown P^T variant {self.pt_variant!r}, expected one of {PT_VARIANTS}")

    @classmethod
    def from_device(cls, T_dev, R_dev, plan: GatherPlan, params: NgfParams, alpha: float,
                    exact: bool = False, pt_variant: str = "gather"):
        """Device-resident construction used by `register`: reference terms are
        computed on the device from R (ngf.py:60-67) inside the level."""
        obj = cls(template=Image3(plan.image_grid, T_dev), ref=None, plan=plan, params=params,
                  alpha=alpha, pt_variant=pt_variant, exact=exact)
        obj._level = DeviceLevel(plan.image_grid, plan.def_grid, T_dev, params, alpha, R_dev=R_dev)
        obj._set_variant()
        return obj

    def _set_variant(self):
        # the exact path runs the requested P^T variant; the fused march always uses its
        # deterministic tile gather (the reference's default, ngf.py:121)
        check(lib().ngf_level_set_pt_variant(self._level.handle, PT_VARIANTS.index(self.pt_variant)),
              "ngf_level_set_pt_variant")

    @property
    def def_grid(self) -> Grid3:
        return self.plan.def_grid

    @property
    def level(self) -> DeviceLevel:
        if self._level is None:
            T = dev.to_device(self.template.values)
            dt = dev.np_dtype(T.dtype)
            gR = dev.to_device(self.ref.grad.field, dt)
            nR = dev.to_device(self.ref.norm, dt)
            self._level = DeviceLevel(self.plan.image_grid, self.plan.def_grid, T, self.params,
                                      self.alpha, gR_dev=gR, nR_dev=nR)
            self._set_variant()
        return self._level

    def field_from_flat(self, x) -> DeformationField:
        return DeformationField(self.def_grid, x.reshape((3,) + self.def_grid.shape))

    def eval_device(self, x_dev, grad_dev, scalars_dev=None):
        """One evaluation on device buffers, no host sync; returns the (J, D, S) tensor."""
        self.evals += 1
        return self.level.eval(x_dev, grad_dev, scalars_dev, exact=self.exact)

    def evaluate(self, y: DeformationField):
        """Returns (J, D, S, flat gradient) like objective.py:43-52."""
        np_out = not dev.is_tensor(y.field)
        x = dev.to_device(y.field).reshape(-1)
        g = dev.empty(x.shape, x.dtype)
        sc = self.eval_device(x, g).cpu().numpy()
        J, D, S = float(sc[0]), float(sc[1]), float(sc[2])
        return J, D, S, (dev.to_host(g) if np_out else g)

    def _host_call(self, x: np.ndarray):
        """numpy in / out through ngf_level_eval_host: the library stages x through
        page-locked memory with its copy threads (overlapping the upload DMA), evaluates,
        and downloads the gradient; one stream sync."""
        t = dev.torch()
        lvl = self.level
        ndt = dev.np_dtype(lvl.dtype)
        x = np.ascontiguousarray(x.reshape(-1), dtype=ndt)
        if x.size != lvl.n:
            raise ValueError(f"x has {x.size} values, the level's deformation has {lvl.n}")
        # the gradient lands in a fresh page-locked buffer from torch's caching host
        # allocator (a direct DMA) and is returned without a host copy; the caller owns it
        # (the reference returns a new array per call), and it is recycled once released
        g_out = t.empty(lvl.n, dtype=lvl.dtype, pin_memory=True)
        sc = self._sc_host
        check(lib().ngf_level_eval_host(lvl.handle, x.ctypes.data, g_out.data_ptr(),
                                        sc.ctypes.data, 1 if self.exact else 0, dev.stream()),
              "ngf_level_eval_host")
        self.evals += 1
        return float(sc[0]), float(sc[1]), float(sc[2]), g_out.numpy()

    def __call__(self, x):
        if dev.is_tensor(x):
            J, D, S, g = self.evaluate(self.field_from_flat(x))
        else:
            # non-finite trial points are detected on the device (J = inf), so the host
            # does not re-scan x (objective.py:55-57 semantics are kept below)
            J, D, S, g = self._host_call(np.asarray(x))
        if not np.isfinite(J):
            # overflowed line-search trial point; force a backtrack (objective.py:55-57)
            return float("inf"), (np.zeros_like(g) if not dev.is_tensor(g) else g.zero_())
        self.last_D, self.last_S = D, S
        return J, g
