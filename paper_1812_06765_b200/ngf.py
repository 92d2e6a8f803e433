"""Normalized-gradient-fields distance and its matrix-free gradient (drop-in for ngfreg.ngf).

    D = (hbar/2) sum_i (1 - r_i^2),  r_i = (<gT_i, gR_i> + tau rho) / (||gT_i||_tau ||gR_i||_rho)

The functions here chain the bit-exact standalone kernels (reference order,
ngf.py:60-134), including numpy's pairwise summation for D.  The fused
performance path is `LevelObjective` (objective.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _device as dev
from ._lib import check, dtype_code, lib, ngf_grid
from .geometry import DeformationField, Grid3, Image3, VectorField3
from .transfer import GatherPlan, apply_P, apply_Pt
from .warp import WarpResult, image_gradient_apply_transpose, warp_image, warp_jacobian_apply_transpose

__all__ = ["NgfParams", "ReferenceTerms", "distance_and_gradient", "ngf_gradient_wrt_yhat",
           "ngf_value", "precompute_reference_terms"]


@dataclass(frozen=True)
class NgfParams:
    """Edge parameters tau (template) and rho (reference) (ngf.py:40-49)."""

    tau: float = 10.0
    rho: float = 10.0

    def __post_init__(self):
        if not (self.tau > 0 and self.rho > 0):
            raise ValueError(f"tau and rho must be > 0, got tau={self.tau}, rho={self.rho}")


@dataclass
class ReferenceTerms:
    """grad R and ||grad R||_rho per voxel (ngf.py:52-57); device tensors or numpy."""

    grad: VectorField3
    norm: object


def precompute_reference_terms(R: Image3, params: NgfParams, workers: int = 1) -> ReferenceTerms:
    np_out = not dev.is_tensor(R.values)
    Rd = dev.to_device(R.values)
    gR = dev.empty((3,) + R.grid.shape, Rd.dtype)
    nR = dev.empty(R.grid.shape, Rd.dtype)
    check(lib().ngf_ref_terms(ctypes.byref(ngf_grid(R.grid)), dtype_code(Rd.dtype), dev.ptr(Rd),
                              float(params.rho), dev.ptr(gR), dev.ptr(nR), dev.stream()),
          "ngf_ref_terms")
    if np_out:
        return ReferenceTerms(VectorField3(R.grid, dev.to_host(gR)), dev.to_host(nR))
    return ReferenceTerms(VectorField3(R.grid, gR), nR)


def _terms_and_q(W, ref: ReferenceTerms, params: NgfParams, grid: Grid3, want_q: bool):
    Wd = dev.to_device(W)
    dt = dev.np_dtype(Wd.dtype)
    gR = dev.to_device(ref.grad.field, dt)
    nR = dev.to_device(ref.norm, dt)
    terms = dev.empty(grid.shape, Wd.dtype)
    q = dev.empty((3,) + grid.shape, Wd.dtype) if want_q else None
    check(lib().ngf_ngf_terms(ctypes.byref(ngf_grid(grid)), dtype_code(Wd.dtype), dev.ptr(Wd),
                              dev.ptr(gR), dev.ptr(nR), float(params.tau), float(params.rho),
                              dev.ptr(terms), dev.ptr(q), dev.stream()), "ngf_ngf_terms")
    return terms, q


def _pairwise_sum(x) -> float:
    out = dev.zeros((1,), "float64")
    check(lib().ngf_pairwise_sum(dtype_code(x.dtype), dev.ptr(x), x.numel(), dev.ptr(out),
                                 dev.stream()), "ngf_pairwise_sum")
    return float(out.item())


def ngf_value(warped: WarpResult, ref: ReferenceTerms, params: NgfParams, h_bar: float,
              workers: int = 1) -> float:
    """D with the reference's pairwise f32/f64 sum and rounding (ngf.py:83-90)."""
    grid = warped.warped.grid
    terms, _ = _terms_and_q(warped.warped.values, ref, params, grid, False)
    s = _pairwise_sum(terms)
    dt = dev.np_dtype(terms.dtype)
    return float(dt(h_bar / 2) * dt(s))


def ngf_gradient_wrt_yhat(warped: WarpResult, ref: ReferenceTerms, template: Image3,
                          yhat: VectorField3, params: NgfParams, h_bar: float,
                          workers: int = 1) -> VectorField3:
    """q, s = G^T q, then the warp Jacobian transpose (ngf.py:93-114)."""
    grid = yhat.grid
    if abs(h_bar - grid.cell_volume) > 0:
        raise ValueError("h_bar must be the image cell volume")
    _, q = _terms_and_q(warped.warped.values, ref, params, grid, True)
    s = image_gradient_apply_transpose(VectorField3(grid, q), grid)
    out = warp_jacobian_apply_transpose(template, VectorField3(grid, dev.to_device(yhat.field)), s)
    if not dev.is_tensor(yhat.field):
        return VectorField3(grid, dev.to_host(out.field))
    return out


def distance_and_gradient(y: DeformationField, ref: ReferenceTerms, template: Image3,
                          plan: GatherPlan, params: NgfParams, pt_variant: str = "gather",
                          workers: int = 1):
    """(D, grad_y D): P, warp, D, q, G^T, J^T, P^T (ngf.py:117-134), bit-exact."""
    np_out = not dev.is_tensor(y.field)
    image_grid = plan.image_grid
    yd = DeformationField(y.grid, dev.to_device(y.field))
    yhat = apply_P(yd, image_grid, plan=plan)
    Tdev = Image3(template.grid, dev.to_device(template.values, dev.np_dtype(yd.field.dtype)))
    warped = warp_image(Tdev, yhat)
    h_bar = image_grid.cell_volume
    D = ngf_value(warped, ref, params, h_bar)
    ghat = ngf_gradient_wrt_yhat(warped, ref, Tdev, yhat, params, h_bar)
    grad = apply_Pt(ghat, plan, pt_variant)
    if np_out:
        grad = VectorField3(grad.grid, dev.to_host(grad.field))
    return D, grad
