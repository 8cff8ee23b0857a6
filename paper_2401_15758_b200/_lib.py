"""Loader for the in-tree CUDA library ``_build/libsdv_cuda.so`` (C-ABI in include/sdv.h).

There is no CPU fallback: if the library is missing or cannot be loaded the
import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libsdv_cuda.so")

SDV_OK = 0
SDV_EINVAL = -22
SDV_ENUMERIC = -34
SDV_ECUDA = -5

D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)
I32 = C.POINTER(C.c_int)


class ProblemDesc(C.Structure):
    _fields_ = [("model", C.c_int), ("n", C.c_int), ("nu", C.c_double), ("dt", C.c_double), ("n_t", C.c_int),
                ("steps_per_interval", C.c_int), ("prior_sigma", C.c_double), ("prior_length", C.c_double),
                ("block_group", C.c_int), ("prior_kind", C.c_int), ("prior_alpha", C.c_double),
                ("prior_beta", C.c_double), ("ny", C.c_int), ("reynolds", C.c_double), ("rossby", C.c_double)]


class GNConfigC(C.Structure):
    _fields_ = [("mode", C.c_int), ("method", C.c_int), ("rank", C.c_int), ("rank2", C.c_int), ("growth", C.c_int),
                ("max_rank", C.c_int), ("eps_sketch", C.c_double), ("eps_reuse", C.c_double),
                ("seed", C.c_uint64), ("grad_tol", C.c_double), ("pcg_tol", C.c_double),
                ("max_gn_iters", C.c_int), ("pcg_max_iter", C.c_int)]


class SdvError(RuntimeError):
    pass


class SdvCudaError(SdvError):
    pass


_lib = None


def lib():
    """Load the CUDA library (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsdv_cuda.so not built ({LIB_PATH}); run __graft_entry__.build() — "
                          "there is no CPU fallback for the product path")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "sdv_last_error": (C.c_char_p, []),
        "sdv_version": (C.c_char_p, []),
        "sdv_device_init": (C.c_int, [C.c_int]),
        "sdv_launch_count": (C.c_ulonglong, []),
        "sdv_path_counts": (C.c_int, [C.POINTER(C.c_uint64), C.c_int]),
        "sdv_path_name": (C.c_char_p, [C.c_int]),
        "sdv_problem_create": (C.c_int, [C.POINTER(ProblemDesc), C.c_int64, I64, D, D, D, C.POINTER(vp)]),
        "sdv_problem_destroy": (None, [vp]),
        "sdv_problem_dims": (C.c_int, [vp, I64]),
        "sdv_forward": (C.c_int, [vp, D, C.c_int, D]),
        "sdv_linearize": (C.c_int, [vp, D, C.POINTER(vp)]),
        "sdv_linearize_dev": (C.c_int, [vp, vp, C.POINTER(vp)]),
        "sdv_linearize_ex": (C.c_int, [vp, D, C.c_int, C.c_int, C.POINTER(vp)]),
        "sdv_linearize_ex_dev": (C.c_int, [vp, vp, C.c_int, C.c_int, C.POINTER(vp)]),
        "sdv_traj_info": (C.c_int, [vp, C.POINTER(C.c_int64)]),
        "sdv_sub_blocks": (C.c_int, [vp, C.c_int, C.POINTER(C.c_int)]),
        "sdv_traj_destroy": (None, [vp]),
        "sdv_traj_state_at": (C.c_int, [vp, C.c_int, D]),
        "sdv_tlm_range": (C.c_int, [vp, C.c_int, C.c_int, D, C.c_int, D]),
        "sdv_adj_range": (C.c_int, [vp, C.c_int, C.c_int, D, C.c_int, D]),
        "sdv_prior_sqrt_block": (C.c_int, [vp, D, C.c_int, D]),
        "sdv_misfit_apply_block": (C.c_int, [vp, D, C.c_int, D]),
        "sdv_misfit_adjoint_block": (C.c_int, [vp, D, C.c_int, D]),
        "sdv_gram_apply_block": (C.c_int, [vp, D, C.c_int, D]),
        "sdv_misfit_apply_block_dev": (C.c_int, [vp, vp, C.c_int, vp]),
        "sdv_misfit_adjoint_block_dev": (C.c_int, [vp, vp, C.c_int, vp]),
        "sdv_gram_apply_block_dev": (C.c_int, [vp, vp, C.c_int, vp]),
        "sdv_evaluate": (C.c_int, [vp, D, D, D, D, D]),
        "sdv_woodbury_apply": (C.c_int, [vp, C.c_int64, D, D, D, C.c_int, D]),
        "sdv_thin_qr": (C.c_int, [vp, C.c_int64, C.c_int64, D, D, D, I32]),
        "sdv_thin_qr_dev": (C.c_int, [vp, C.c_int64, C.c_int64, vp, D, I32]),
        "sdv_evd_from_tall_dev": (C.c_int, [vp, C.c_int64, C.c_int64, vp, C.c_double, C.c_int, vp, D]),
        "sdv_nystrom_assemble_dev": (C.c_int, [vp, C.c_int64, C.c_int64, vp, vp, vp, D]),
        "sdv_sketch": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_uint64, D, D, I64]),
        "sdv_lanczos_sketch": (C.c_int, [vp, C.c_int, D, D, D, I64]),
        "sdv_pcg_solve": (C.c_int, [vp, D, C.c_int64, D, D, C.c_double, C.c_int, D, I32]),
        "sdv_sketch_adaptive": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                          D, D, I64, D, C.c_int]),
        "sdv_cond_estimate": (C.c_int, [vp, C.c_int64, D, D, C.c_uint64, D]),
        "sdv_gn_solve": (C.c_int, [vp, C.POINTER(GNConfigC), D, D, C.c_int, I32, D, D, C.c_int]),
        "sdv_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        "sdv_gaussian_matrix": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, D]),
        "sdv_dev_alloc": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
        "sdv_dev_free": (C.c_int, [vp]),
        "sdv_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
        "sdv_host_free": (C.c_int, [vp]),
        "sdv_memcpy_htod": (C.c_int, [vp, vp, C.c_size_t]),
        "sdv_memcpy_dtoh": (C.c_int, [vp, vp, C.c_size_t]),
        "sdv_synchronize": (C.c_int, [vp]),
        "sdv_event_create": (C.c_int, [C.POINTER(vp)]),
        "sdv_event_destroy": (C.c_int, [vp]),
        "sdv_event_record": (C.c_int, [vp, vp]),
        "sdv_event_elapsed_ms": (C.c_int, [vp, vp, C.POINTER(C.c_float)]),
        "sdv_probe_stage_kernels": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
        "sdv_probe_adj_stage_kernels": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc):
    """Map C-ABI status codes onto the reference's exception types."""
    if rc == SDV_OK:
        return rc
    msg = lib().sdv_last_error().decode()
    if rc == SDV_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == SDV_ECUDA:
        raise SdvCudaError(msg)
    raise SdvError(msg)  # std::runtime_error
