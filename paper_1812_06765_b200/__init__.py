"""B200-native (sm_100a) NGF + curvature deformable registration hot path of arXiv 1812.06765.

Drop-in for the reference package `ngfreg`: same names, argument meaning and
error behaviour for the registration entry point (`register`), the level
objective callable (`LevelObjective`), the L-BFGS driver (`lbfgs_minimize`) and
the operators on the path (P / P^T, warp, NGF, curvature, pyramid,
prolongation).  Host code is Python; every volume operation is a hand-written
CUDA kernel in libngfb200.so called through a ctypes C-ABI (include/ngf_b200.h).
There is no CPU fallback.
"""

from ._lib import GridError
from .curvature import apply_laplacian, apply_laplacian_transpose, curvature_gradient, curvature_value
from .geometry import (DeformationField, Grid3, Image3, VectorField3, identity_field_array,
                       make_identity, precision_dtype)
from .lbfgs import (IterationRecord, LbfgsConfig, OptimizeTrace, StoppingRules, lbfgs_minimize,
                    two_loop_direction)
from .multilevel import (LevelReport, MultilevelConfig, RegistrationReport, build_pyramid,
                         deformation_grid_for, downsample_image, num_auto_levels, prolong_deformation,
                         register, warp_with_field)
from .ngf import (NgfParams, ReferenceTerms, distance_and_gradient, ngf_gradient_wrt_yhat, ngf_value,
                  precompute_reference_terms)
from .objective import DeviceLevel, LevelObjective
from .synthetic import (analytic_intensity, ct_pair, gaussian_bump_mapping, make_registration_pair,
                        make_volume, probe_lattice, smooth_random_field, smooth_random_volume)
from .transfer import (GatherPlan, apply_P, apply_Pt, apply_Pt_gather, apply_Pt_redblack,
                       apply_Pt_scatter_atomic, build_gather_plan, dense_P_oracle)
from .warp import (WarpResult, image_gradient, image_gradient_apply_transpose, warp_image,
                   warp_jacobian_apply_transpose)

__version__ = "0.1.0"

__all__ = [
    "DeformationField", "DeviceLevel", "GatherPlan", "Grid3", "GridError", "Image3",
    "IterationRecord", "LbfgsConfig", "LevelObjective", "LevelReport", "MultilevelConfig",
    "NgfParams", "OptimizeTrace", "ReferenceTerms", "RegistrationReport", "StoppingRules",
    "VectorField3", "WarpResult", "analytic_intensity", "apply_P", "apply_Pt", "apply_Pt_gather",
    "apply_Pt_redblack", "apply_Pt_scatter_atomic", "apply_laplacian", "apply_laplacian_transpose",
    "build_gather_plan", "build_pyramid", "ct_pair", "curvature_gradient", "curvature_value",
    "deformation_grid_for", "dense_P_oracle", "distance_and_gradient", "downsample_image",
    "gaussian_bump_mapping", "identity_field_array", "image_gradient",
    "image_gradient_apply_transpose", "lbfgs_minimize", "make_identity", "make_registration_pair",
    "make_volume", "ngf_gradient_wrt_yhat", "ngf_value", "num_auto_levels", "precision_dtype",
    "precompute_reference_terms", "probe_lattice", "prolong_deformation", "register",
    "smooth_random_field", "smooth_random_volume", "two_loop_direction", "warp_image",
    "warp_jacobian_apply_transpose", "warp_with_field",
]
