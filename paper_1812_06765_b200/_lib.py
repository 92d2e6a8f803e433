"""ctypes binding of libngfb200.so (include/ngf_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_1812_06765_b200/csrc`).  There is no fallback: if the library
is missing every device entry point raises, naming the build command.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libngfb200.so")

NGF_F32, NGF_F64 = 0, 1
NGF_EARG, NGF_EGRID, NGF_ENOMEM, NGF_ESTATE = -1, -2, -3, -4


class GridError(ValueError):
    """Invalid grid definition or mismatched grids (reference geometry.py:20-21)."""


class NgfGrid(ctypes.Structure):
    _fields_ = [("dims", ctypes.c_int64 * 3), ("spacing", ctypes.c_double * 3),
                ("origin", ctypes.c_double * 3)]


_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_d = ctypes.c_double
_pg = ctypes.POINTER(NgfGrid)
_pd = ctypes.POINTER(ctypes.c_double)

_PROTOS = {
    "ngf_version": (_i, []),
    "ngf_launch_count": (_i64, []),
    "ngf_error_string": (ctypes.c_char_p, [_i]),
    "ngf_plan_create": (_i, [_pg, _pg, ctypes.POINTER(_vp)]),
    "ngf_plan_create_prolong": (_i, [_pg, _pg, ctypes.POINTER(_vp)]),
    "ngf_plan_destroy": (None, [_vp]),
    "ngf_plan_axis": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(ctypes.c_int32)]),
    "ngf_apply_P": (_i, [_vp, _i, _vp, _vp, _vp]),
    "ngf_apply_Pt": (_i, [_vp, _i, _vp, _vp, _vp]),
    "ngf_apply_Pt_variant": (_i, [_vp, _i, _i, _vp, _vp, _vp]),
    "ngf_sample_field": (_i, [_vp, _i, _vp, _vp, ctypes.c_int64, _vp, _vp]),
    "ngf_lbfgs_run_level": (_i, [_vp, _i, _i, _vp, ctypes.c_int64, _vp, _vp, _vp, _vp, _i, _vp]),
    "ngf_warp": (_i, [_pg, _i, _vp, _vp, _i64, _vp, _vp, _vp]),
    "ngf_warp_jt": (_i, [_pg, _i, _vp, _vp, _vp, _i64, _vp, _vp]),
    "ngf_gradient": (_i, [_pg, _i, _vp, _vp, _vp]),
    "ngf_gradient_t": (_i, [_pg, _i, _vp, _vp, _vp]),
    "ngf_ref_terms": (_i, [_pg, _i, _vp, _d, _vp, _vp, _vp]),
    "ngf_ngf_terms": (_i, [_pg, _i, _vp, _vp, _vp, _d, _d, _vp, _vp, _vp]),
    "ngf_pairwise_sum": (_i, [_i, _vp, _i64, _vp, _vp]),
    "ngf_laplacian": (_i, [_pg, _i, _vp, _vp, _vp]),
    "ngf_laplacian_t": (_i, [_pg, _i, _vp, _vp, _vp]),
    "ngf_curvature": (_i, [_pg, _i, _vp, _vp, _vp, _vp]),
    "ngf_downsample": (_i, [_pg, _i, _vp, _vp, _vp]),
    "ngf_prolong": (_i, [_vp, _i, _vp, _vp, _vp]),
    "ngf_level_create": (_i, [_pg, _pg, _i, _vp, _vp, _d, _d, _d, _vp, ctypes.POINTER(_vp)]),
    "ngf_level_create_terms": (_i, [_pg, _pg, _i, _vp, _vp, _vp, _d, _d, _d, _vp,
                                    ctypes.POINTER(_vp)]),
    "ngf_level_create_zslab": (_i, [_pg, _pg, _i, _vp, _vp, _d, _d, _d, _i64, _i64, _vp, ctypes.POINTER(_vp)]),
    "ngf_level_destroy": (None, [_vp]),
    "ngf_level_eval": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "ngf_level_eval_host": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "ngf_lbfgs_set_graph": (_i, [_i]),
    "ngf_lbfgs_graph_runs": (_i64, []),
    "ngf_host_upload": (_i, [_vp, _vp, ctypes.c_size_t, _vp]),
    "ngf_host_download": (_i, [_vp, _vp, ctypes.c_size_t, _vp]),
    "ngf_host_is_pinned": (_i, [_vp]),
    "ngf_level_ref_terms": (_vp, [_vp]),
    "ngf_level_set_timing": (_i, [_vp, _i]),
    "ngf_level_set_pt_variant": (_i, [_vp, _i]),
    "ngf_level_kernel_ms": (_i, [_vp, ctypes.POINTER(ctypes.c_float)]),
    "ngf_level_info": (_i, [_vp, ctypes.POINTER(ctypes.c_int64)]),
    "ngf_level_variant": (_i, [_vp]),
    "ngf_level_set_host_pipeline": (_i, [_vp, _i]),
    "ngf_level_set_zrange": (_i, [_vp, _i64, _i64]),
    "ngf_level_add_curvature": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "ngf_vec_dot": (_i, [_i, _vp, _vp, _i64, _vp, _vp]),
    "ngf_vec_stats": (_i, [_i, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "ngf_vec_axpy_step": (_i, [_i, _vp, _d, _vp, _vp, _i64, _vp]),
    "ngf_vec_sub": (_i, [_i, _vp, _vp, _vp, _i64, _vp]),
    "ngf_lbfgs_pair": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "ngf_lbfgs_two_loop": (_i, [_i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _pd, _d, _i, _vp, _vp,
                                _i64, _vp, _vp]),
}

EXPORTED = tuple(_PROTOS)

_lib = None


def load(path: str = LIB_PATH):
    """Load libngfb200.so (no GPU needed) and attach the prototypes."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_1812_06765_b200/csrc` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return _lib if _lib is not None else load()


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = lib().ngf_error_string(rc).decode()
    if rc == NGF_EGRID:
        raise GridError(f"{what}: {msg}")
    if rc == NGF_EARG:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: libngfb200 error {rc} ({msg})")


def ngf_grid(g) -> NgfGrid:
    """ctypes grid from anything with dims/spacing/origin."""
    s = NgfGrid()
    for a in range(3):
        s.dims[a] = int(g.dims[a])
        s.spacing[a] = float(g.spacing[a])
        s.origin[a] = float(g.origin[a])
    return s


def dtype_code(dtype) -> int:
    dt = np.dtype(dtype) if not hasattr(dtype, "is_floating_point") else None
    if dt is None:  # torch dtype
        import torch
        if dtype == torch.float32:
            return NGF_F32
        if dtype == torch.float64:
            return NGF_F64
        raise ValueError(f"unsupported dtype {dtype}")
    if dt == np.float32:
        return NGF_F32
    if dt == np.float64:
        return NGF_F64
    raise ValueError(f"unsupported dtype {dt}")


def launch_count() -> int:
    return int(lib().ngf_launch_count())
