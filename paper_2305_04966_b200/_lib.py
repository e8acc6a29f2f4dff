"""ctypes loader for libnacc.so (include/nacc.h) and libnacc_harness.so.

Argument marshalling only.  There is no fallback: if the library is missing
the import of any op raises, and ops refuse non-CUDA tensors.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# NACC_DEBUG=1 loads the precondition-checking build (libnacc_debug.so, csrc/debug.cu)
LIB_PATH = os.path.join(_PKG, "libnacc_debug.so" if os.environ.get("NACC_DEBUG") == "1" else "libnacc.so")
HARNESS_PATH = os.path.join(_PKG, "libnacc_harness.so")

NACC_OK = 0
NACC_ERR_INVALID_ARGUMENT = 1
NACC_ERR_INSUFFICIENT_CAPACITY = 2
NACC_ERR_CUDA = 3
NACC_ERR_UNSUPPORTED = 4
_NAMES = {0: "NACC_OK", 1: "NACC_ERR_INVALID_ARGUMENT", 2: "NACC_ERR_INSUFFICIENT_CAPACITY",
          3: "NACC_ERR_CUDA", 4: "NACC_ERR_UNSUPPORTED"}


class NaccError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_NAMES.get(status, status)}: {msg}")
        self.status = status


class Grid(C.Structure):
    _fields_ = [("levels", C.c_int32), ("res", C.c_int32), ("roi", C.c_float * 6)]


class March(C.Structure):
    _fields_ = [("near_plane", C.c_float), ("far_plane", C.c_float), ("step", C.c_float),
                ("max_step", C.c_float), ("cone_angle", C.c_float), ("stratified", C.c_int32),
                ("seed", C.c_uint64)]


P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
SZ = C.c_size_t
D = C.c_double
F = C.c_float
U64 = C.c_uint64
GP = C.POINTER(Grid)
MP = C.POINTER(March)

# name -> (restype, argtypes); mirrors include/nacc.h
SIGNATURES = {
    "nacc_last_error": (C.c_char_p, []),
    "nacc_abi_version": (C.c_int, []),
    "nacc_launch_count": (C.c_uint64, []),
    "nacc_grid_bits_bytes": (SZ, [GP]),
    "nacc_grid_prepare": (C.c_int, [GP, P, P]),
    "nacc_sampling_occgrid_workspace_bytes": (SZ, [GP, MP, I64]),
    "nacc_sampling_occgrid": (C.c_int, [GP, P, MP, P, P, P, P, I64, P, P, P, P, I64, P, P, P, SZ, P]),
    "nacc_sampling_occgrid_fill": (C.c_int, [GP, P, MP, P, P, P, P, I64, P, P, P, P, P, SZ, P]),
    "nacc_filter_workspace_bytes": (SZ, [I64]),
    "nacc_filter_early_stop": (C.c_int, [P, I64, P, P, P, I64, D, P, P, P, P, I64, P, P, SZ, P]),
    "nacc_render_weights_fwd": (C.c_int, [P, I64, P, P, P, I64, D, P, P, P, P]),
    "nacc_render_weights_fwd_flat": (C.c_int, [P, P, I64, P, P, P, I64, D, P, P, P, P]),
    "nacc_render_weights_bwd_flat_workspace_bytes": (C.c_size_t, [I64]),
    "nacc_render_weights_bwd_flat": (C.c_int, [P, P, I64, P, P, P, I64, D, P, P, P, P, C.c_size_t, P]),
    "nacc_render_weights_bwd": (C.c_int, [P, I64, P, P, P, I64, D, P, P, P, P]),
    "nacc_render_weights_alpha_fwd": (C.c_int, [P, I64, P, I64, D, P, P, P]),
    "nacc_render_weights_alpha_fwd_flat": (C.c_int, [P, P, I64, P, I64, D, P, P, P]),
    "nacc_render_weights_alpha_bwd_workspace_bytes": (SZ, [I64]),
    "nacc_render_weights_alpha_bwd": (C.c_int, [P, I64, P, I64, D, P, P, P, P, SZ, P]),
    "nacc_render_weights_alpha_bwd_flat": (C.c_int, [P, P, I64, P, I64, D, P, P, P, P, SZ, P]),
    "nacc_accumulate_along_rays": (C.c_int, [P, I64, P, P, I32, I64, P, P]),
    "nacc_accumulate_along_rays_bwd": (C.c_int, [P, I64, P, P, I32, I64, P, P, P, P]),
    "nacc_accumulate_along_rays_flat": (C.c_int, [P, P, I64, P, P, I32, I64, P, P]),
    "nacc_accumulate_along_rays_bwd_flat": (C.c_int, [P, I64, P, P, I32, I64, P, P, P, P]),
    "nacc_render_fwd": (C.c_int, [P, P, I64, P, P, P, P, I64, D, P, P, P, P, P]),
    "nacc_render_bwd": (C.c_int, [P, P, I64, P, P, P, P, I64, D, P, P, P, P, P, P, P, SZ, P]),
    "nacc_render_bwd_workspace_bytes": (SZ, [I64]),
    "nacc_importance_sample": (C.c_int, [I64, I32, P, P, P, C.c_int, D, D, I32, I32, U64, P, P, P]),
    "nacc_importance_sample_ranged": (C.c_int, [I64, I32, P, P, P, C.c_int, P, P, I32, I32, U64, P, P, P]),
    "nacc_pdf_loss": (C.c_int, [I64, I32, P, P, I32, P, P, D, P, P]),
    "nacc_pdf_loss_bwd": (C.c_int, [I64, I32, P, P, I32, P, P, D, P, P, P]),
    "nacc_occgrid_ray_bounds": (C.c_int, [GP, P, MP, P, P, P, P, I64, P, P, P, P, SZ, P]),
    "nacc_occgrid_times": (C.c_int, [GP, U64, I64, I32, I64, I64, P, P]),
    "nacc_max_merge": (C.c_int, [P, P, I64, P]),
    "nacc_occgrid_points": (C.c_int, [GP, U64, I64, I32, I64, I64, P, P]),
    "nacc_occgrid_workspace_bytes": (SZ, [GP]),
    "nacc_occgrid_update": (C.c_int, [GP, P, P, C.c_int, F, F, C.c_int, P, P, P, SZ, P]),
}

HARNESS_SIGNATURES = {
    "naccx_field_at_samples": (C.c_int, [P, I32, F, F, I32, P, P, P, P, P, I64, P, P, P, P]),
    "naccx_sigma_at_samples": (C.c_int, [P, I32, F, F, I32, P, P, P, P, P, I64, P, P, P]),
    "naccx_field_at_points": (C.c_int, [P, I32, F, F, I32, P, I64, F, P, P]),
    "naccx_mse_grad": (C.c_int, [P, P, I64, P, P]),
    "naccx_tex_create": (C.c_int, [P, I32, C.POINTER(C.c_uint64), P]),
    "naccx_tex_destroy": (None, [C.c_uint64]),
    "naccx_tex_at_samples": (C.c_int, [C.c_uint64, F, F, I32, P, P, P, P, P, I64, P, P, P, P]),
    "naccx_launch_count": (C.c_uint64, []),
}

_lib = None
_hlib = None


def _load(path, sigs, what):
    if not os.path.exists(path):
        raise RuntimeError(
            f"{what} is not built ({path} missing). Run `python -c \"import __graft_entry__ as g; g.build()\"`. "
            "There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    global _lib
    if _lib is None:
        _lib = _load(LIB_PATH, SIGNATURES, "libnacc.so")
    return _lib


def harness():
    global _hlib
    if _hlib is None:
        _hlib = _load(HARNESS_PATH, HARNESS_SIGNATURES, "libnacc_harness.so")
    return _hlib


def check(status: int, where: str = "") -> None:
    if status != NACC_OK:
        msg = lib().nacc_last_error().decode(errors="replace") if _lib is not None else ""
        raise NaccError(status, f"{where}: {msg}")
