"""ctypes binding of the C ABI in ``include/pdf_abi.h`` (libpdfb200.so).

This is the binding a maintainer of the reference would add (see
INTEGRATION.md).  There is no CPU fallback: if the shared library is missing
or fails to load, importing the GPU path raises immediately.
"""
from __future__ import annotations

import ctypes as ct
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PDF_LIB_PATH") or os.path.join(_HERE, "libpdfb200.so")   # override: A/B measurements only
# (an override library must still export every symbol: a missing one raises below)

ABI_VERSION = 1
PDF_ENOCONV = -4
PDF_EGEOMETRY = -5
PDF_F64, PDF_F32 = 0, 1

ERR_POLE = 1
ERR_NONFINITE_STATE = 2
ERR_NONFINITE_DATA = 4
ERR_NONFINITE_BOUND = 8
ERR_NONFINITE_TV = 16
ERR_NONFINITE_BRIDGE = 32
ERR_NONFINITE_GRAD = 64
ERR_NONFINITE_PARAM = 128

# every symbol include/pdf_abi.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "pdf_last_error", "pdf_abi_version", "pdf_workspace_bytes", "pdf_ctx_create", "pdf_ctx_destroy",
    "pdf_net_dims", "pdf_loss_grad", "pdf_loss_value", "pdf_net_setup", "pdf_net_forward",
    "pdf_grad_loss", "pdf_adam_step", "pdf_set_norms", "pdf_train", "pdf_apply_gd", "pdf_gs_forward", "pdf_gs_adjoint",
    "pdf_expand", "pdf_truncate", "pdf_apply_cco", "pdf_get_error", "pdf_profile_train", "pdf_fp64_probe",
    "pdf_timeline_reset", "pdf_timeline_read", "pdf_ctx_paths",
    "pdf_net_setup_sharded", "pdf_shard_buffer_sizes", "pdf_shard_step_a", "pdf_shard_step_b", "pdf_shard_step_c",
    "pdf_relative_error", "pdf_count_components", "pdf_solver_workspace_bytes", "pdf_solve_total_field",
    "pdf_bessel", "pdf_build_greens", "pdf_incident_fields", "pdf_shard_step_c_part", "pdf_net_offsets",
    "pdf_adam_step_dev", "pdf_shard_step_c_scatter", "pdf_adam_gather", "pdf_chi_to_r", "pdf_default_eps_reg",
    "pdf_pixel_ls", "pdf_cie_fields", "pdf_masked_residual", "pdf_regularizers", "pdf_box_mean", "pdf_guided_filter",
    "pdf_cco_image", "pdf_net_features", "pdf_net_layer_fwd", "pdf_net_layer_bwd", "pdf_bias_tanh",
    "pdf_shard_tp_a", "pdf_shard_tp_c",
)
PHASES = ("fwd_l1", "fwd_l2", "fwd_l3", "view_fwd", "pixel", "view_bwd", "finalize", "bwd_l3", "bwd_l2", "bwd_l1")


class PdfDesc(ct.Structure):
    _fields_ = [
        ("abi_version", ct.c_int32), ("dtype", ct.c_int32), ("S", ct.c_int32), ("n", ct.c_int32),
        ("m1", ct.c_int32), ("m2", ct.c_int32), ("R", ct.c_int32), ("mf", ct.c_int32),
        ("joint", ct.c_int32), ("freeze_r", ct.c_int32),
        ("beta", ct.c_double), ("lambda1", ct.c_double), ("lambda2", ct.c_double),
        ("lambda3", ct.c_double), ("tau_b", ct.c_double),
        ("lr", ct.c_double), ("adam_b1", ct.c_double), ("adam_b2", ct.c_double),
        ("adam_eps", ct.c_double),
        ("e_inc", ct.c_void_p), ("e_inc_scene_stride", ct.c_int64), ("gd_kernel_hat", ct.c_void_p),
        ("gs_matrix", ct.c_void_p), ("data", ct.c_void_p), ("mask", ct.c_void_p),
        ("r_fixed", ct.c_void_p), ("c_inc", ct.POINTER(ct.c_double)),
        ("c_sca", ct.POINTER(ct.c_double)), ("k_iters_max", ct.c_int32),
    ]


_lib = None


def lib():
    """Load libpdfb200.so once; raise loudly if it is absent or stale."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2602_13805_b200.build` "
                          "(there is no CPU fallback)")
    import torch  # noqa: F401  -- load torch's CUDA runtime first so both share one context
    L = ct.CDLL(LIB_PATH)
    vp, i32, i64, dp = ct.c_void_p, ct.c_int32, ct.c_int64, ct.POINTER(ct.c_double)
    sig = {
        "pdf_last_error": (ct.c_char_p, []),
        "pdf_abi_version": (ct.c_int, []),
        "pdf_workspace_bytes": (ct.c_size_t, [ct.POINTER(PdfDesc)]),
        "pdf_ctx_create": (ct.c_int, [ct.POINTER(PdfDesc), vp, ct.c_size_t, vp, ct.POINTER(vp)]),
        "pdf_ctx_destroy": (ct.c_int, [vp]),
        "pdf_net_dims": (ct.c_int, [vp, ct.POINTER(i32), ct.POINTER(i32), ct.POINTER(i32), ct.POINTER(i64)]),
        "pdf_loss_grad": (ct.c_int, [vp, vp, vp, vp, vp]),
        "pdf_loss_value": (ct.c_int, [vp, vp, vp, vp, vp]),
        "pdf_net_setup": (ct.c_int, [vp, vp, vp]),
        "pdf_net_forward": (ct.c_int, [vp, vp, vp, vp]),
        "pdf_grad_loss": (ct.c_int, [vp, vp, vp, vp, vp]),
        "pdf_adam_step": (ct.c_int, [vp, vp, vp, vp, vp, i64, i32, vp]),
        "pdf_set_norms": (ct.c_int, [vp, dp, dp, vp]),
        "pdf_train": (ct.c_int, [vp, vp, vp, vp, i32, i32, vp, i32, vp]),
        "pdf_apply_gd": (ct.c_int, [vp, vp, vp, i32, i32, vp]),
        "pdf_gs_forward": (ct.c_int, [vp, vp, vp, i32, vp]),
        "pdf_gs_adjoint": (ct.c_int, [vp, vp, vp, i32, vp]),
        "pdf_expand": (ct.c_int, [vp, vp, vp, i32, vp]),
        "pdf_truncate": (ct.c_int, [vp, vp, vp, i32, vp]),
        "pdf_apply_cco": (ct.c_int, [vp, vp, vp, i32, ct.c_double, ct.c_double, ct.c_double, i32,
                                     ct.c_double, vp]),
        "pdf_get_error": (ct.c_int, [vp, ct.POINTER(i32), vp]),
        "pdf_profile_train": (ct.c_int, [vp, vp, vp, vp, i32, i32, ct.POINTER(ct.c_float), vp]),
        "pdf_fp64_probe": (ct.c_int, [dp, vp]),
        "pdf_timeline_reset": (ct.c_int, [vp, i32, vp]),
        "pdf_ctx_paths": (ct.c_int, [vp, ct.POINTER(i32)]),
        "pdf_timeline_read": (ct.c_int, [ct.POINTER(ct.c_uint64), vp]),
        "pdf_net_setup_sharded": (ct.c_int, [vp, vp, i32, i32, vp]),
        "pdf_shard_buffer_sizes": (ct.c_int, [vp, ct.POINTER(i64), ct.POINTER(i64)]),
        "pdf_shard_step_a": (ct.c_int, [vp, vp, vp, vp]),
        "pdf_shard_step_b": (ct.c_int, [vp, vp, vp, vp, vp]),
        "pdf_shard_step_c": (ct.c_int, [vp, vp, vp, vp, vp, vp]),
        "pdf_solver_workspace_bytes": (ct.c_size_t, [vp, i32]),
        "pdf_shard_step_c_part": (ct.c_int, [vp, vp, vp, vp, i32, vp, vp]),
        "pdf_net_offsets": (ct.c_int, [vp, ct.POINTER(i64)]),
        "pdf_adam_step_dev": (ct.c_int, [vp, vp, vp, vp, vp, i64, vp, vp]),
        "pdf_shard_step_c_scatter": (ct.c_int, [vp, vp, vp, vp, i32, i32, i64, i32, vp, vp]),
        "pdf_adam_gather": (ct.c_int, [vp, vp, vp, vp, vp, i32, i32, i64, vp, vp]),
        "pdf_bessel": (ct.c_int, [i32, vp, vp, vp, i64, vp]),
        "pdf_build_greens": (ct.c_int, [ct.c_double, ct.c_double, i32, i32, vp, vp, vp, i32, vp, vp, vp, dp, vp]),
        "pdf_incident_fields": (ct.c_int, [i32, ct.c_double, i32, i32, vp, vp, vp, i32, vp, vp]),
        "pdf_solve_total_field": (ct.c_int, [vp, vp, vp, i64, vp, i32, i32, ct.c_double, i32, vp, ct.c_size_t, vp,
                                             ct.POINTER(i32), vp]),
        "pdf_relative_error": (ct.c_int, [vp, vp, i32, i64, i32, ct.c_double, vp, vp]),
        "pdf_count_components": (ct.c_int, [vp, i32, i32, i32, i32, ct.c_double, ct.c_double, vp, vp, vp]),
        "pdf_chi_to_r": (ct.c_int, [vp, vp, i64, ct.c_double, ct.c_double, i32, vp, vp]),
        "pdf_default_eps_reg": (ct.c_int, [vp, i32, i64, vp, vp]),
        "pdf_pixel_ls": (ct.c_int, [vp, vp, i32, i64, vp, vp, vp, vp, vp, vp]),
        "pdf_cie_fields": (ct.c_int, [vp, vp, vp, i64, vp, ct.c_double, ct.c_double, i32, i64, vp, vp, vp, vp]),
        "pdf_masked_residual": (ct.c_int, [vp, vp, vp, vp, i64, vp]),
        "pdf_regularizers": (ct.c_int, [vp, i32, i32, i32, ct.c_double, ct.c_double, ct.c_double, ct.c_double,
                                        ct.c_double, vp, vp, vp, vp, vp, vp]),
        "pdf_box_mean": (ct.c_int, [vp, vp, i32, i32, i32, i32, vp]),
        "pdf_guided_filter": (ct.c_int, [vp, vp, vp, i32, i32, i32, ct.c_double, i32, vp, vp]),
        "pdf_net_features": (ct.c_int, [vp, vp, vp, vp]),
        "pdf_net_layer_fwd": (ct.c_int, [vp, vp, i32, i32, vp, i64, i64, vp, i32, vp]),
        "pdf_net_layer_bwd": (ct.c_int, [vp, vp, vp, i32, i32, vp, i64, i64, vp, vp, vp]),
        "pdf_bias_tanh": (ct.c_int, [vp, vp, i64, i32, vp]),
        "pdf_shard_tp_a": (ct.c_int, [vp, vp, i32, i32, i32, vp, vp]),
        "pdf_shard_tp_c": (ct.c_int, [vp, vp, vp, i32, i32, i32, vp, vp]),
        "pdf_cco_image": (ct.c_int, [vp, vp, i32, i32, i32, ct.c_double, ct.c_double, ct.c_double, i32, ct.c_double,
                                     vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)      # AttributeError names the missing symbol
        f.restype = res
        f.argtypes = args
    if L.pdf_abi_version() != ABI_VERSION:
        raise ImportError("libpdfb200.so ABI version mismatch; rebuild")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().pdf_last_error().decode(errors="replace")
        raise RuntimeError(f"pdf ABI call failed ({rc}): {msg}")
