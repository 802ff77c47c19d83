"""ctypes binding of libbastion.so (the C ABI in include/bastion.h).

The library is the product path: if it is missing, or no CUDA device is
present, every compute entry point raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("BASTION_LIB", PKG / "libbastion.so"))

BST_OK, BST_EINVAL, BST_ECUDA, BST_ECAP = 0, -1, -2, -3
POLICY_ADAPTIVE, POLICY_FIXED, POLICY_BEAM = 0, 1, 2
ALGO_AUTO, ALGO_SORT, ALGO_HEAP = 0, 1, 2
STOP_NAMES = {0: "first-decrease", 1: "frontier-exhausted", 2: "budget-cap"}


class Curve(C.Structure):
    """bst_curve_t — LatencyCurve coefficients (cost_model.py:287-303)."""

    _fields_ = [("flops_lin", C.c_int64), ("flops_quad", C.c_int64), ("bytes_const", C.c_int64),
                ("bytes_lin", C.c_int64), ("bytes_quad", C.c_int64), ("inv_peak", C.c_double),
                ("inv_bw", C.c_double), ("slope", C.c_double), ("intercept", C.c_double), ("ratio", C.c_double),
                ("flops_const", C.c_int64)]


class Plan(C.Structure):
    _fields_ = [("policy", C.c_int32), ("n_max", C.c_int32), ("width", C.c_int32), ("depth", C.c_int32),
                ("algo", C.c_int32), ("_pad", C.c_int32), ("curve", Curve), ("fixed_cost", C.c_double),
                ("l_ar", C.c_double), ("state", C.c_void_p), ("c_idx", C.c_int32), ("_pad2", C.c_int32),
                ("d_flops_lin", C.c_int64), ("d_bytes_const", C.c_int64), ("d_bytes_lin", C.c_int64),
                ("a_offset", C.c_double)]


class Tree(C.Structure):
    _fields_ = [("parent", C.c_void_p), ("depth", C.c_void_p), ("token", C.c_void_p), ("rank", C.c_void_p),
                ("rho", C.c_void_p), ("trace", C.c_void_p), ("meta", C.c_void_p), ("surrogate", C.c_void_p),
                ("anc_mask", C.c_void_p), ("mask_words", C.c_int32), ("_pad", C.c_int32),
                ("child_start", C.c_void_p), ("child_list", C.c_void_p)]


class GemmSched(C.Structure):
    """bst_gemm_sched_t — stream-K schedule of one GEMM shape."""

    _fields_ = [("n_out", C.c_int32), ("k", C.c_int32), ("m", C.c_int32), ("bn", C.c_int32),
                ("n_mt", C.c_int32), ("n_kb", C.c_int32), ("grid", C.c_int32), ("s_max", C.c_int32),
                ("units", C.c_int64), ("tmem_cols", C.c_int32), ("stages", C.c_int32),
                ("partial_floats", C.c_int64), ("pair", C.c_int32), ("reserved", C.c_int32),
                ("cta2", C.c_int32), ("pad_", C.c_int32)]


class Prefetch(C.Structure):
    """bst_prefetch_t — up to two weight ranges to stream into L2 during the next K3/K5 launch."""

    _fields_ = [("ptr", C.c_void_p * 2), ("bytes", C.c_uint64 * 2)]


_P, _I, _I64, _SZ, _D = C.c_void_p, C.c_int, C.c_int64, C.c_size_t, C.c_double
SIGNATURES = {
    "bst_abi_version": (C.c_int, []),
    "bst_last_error": (C.c_char_p, []),
    "bst_curve_latency": (_D, [C.POINTER(Curve), _I64]),
    "bst_topk_workspace": (_SZ, [_I, _I, _I]),
    "bst_topk_logits": (_I, [_P, _I, _I, _I, _I64, _I, _P, _P, _P, _P, _SZ, _P]),
    "bst_topk_probs": (_I, [_P, _I, _I, _I, _P, _P, _P, _SZ, _P]),
    "bst_topk_gemm_partial": (_I, [_P, C.POINTER(GemmSched), _I, _I, _I, _P, _P, _P, _SZ, _P]),
    "bst_expand_workspace": (_SZ, [_I, _I, _I]),
    "bst_expand": (_I, [_P, _P, _I, _I, C.POINTER(Plan), _I, C.POINTER(Tree), _P, _SZ, _P]),
    "bst_linearize_mask": (_I, [_P, _I, _I, _I, _P, _P]),
    "bst_ancestor_mask": (_I, [_P, _I, _I, _P, _P]),
    "bst_gemm_schedule": (_I, [_I, _I, _I, _I, C.POINTER(GemmSched)]),
    "bst_gemm": (_I, [_P, _P, _I64, C.POINTER(GemmSched), _P, _SZ, _P]),
    "bst_gemm_reduce": (_I, [_P, C.POINTER(GemmSched), _P, _P, _I64, _P]),
    "bst_gemm_argmax": (_I, [_P, C.POINTER(GemmSched), _P, _P, _P]),
    "bst_gemm_argmax_keys": (_I, [_P, C.POINTER(GemmSched), _P, _I, _P]),
    "bst_gemm_sample": (_I, [_P, C.POINTER(GemmSched), _P, _P, _P, _P, _I, C.c_float, C.c_uint64, _P]),
    "bst_argmax_from_keys": (_I, [_P, _I, _P, _P]),
    "bst_expand_dev": (_I, [_P, _P, _I, _I, _P, _I, _I, _I, C.POINTER(Tree), _P, _SZ, _P]),
    "bst_expand_dev_batch": (_I, [_P, _P, _I64, _I, _I, _P, _I, _I, _I, _P, _I, _P, _SZ, _P]),
    "bst_attention": (_I, [_P, _I64, _P, _I64, _P, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _P, _I, _I, _P, _I, _I,
                           _P, _SZ, _P]),
    "bst_attention_batch": (_I, [_P, _I64, _P, _I64, _P, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _I, _P, _I, _I, _I,
                                 _P, _I, _I, _P, _SZ, _P]),
    "bst_attention_workspace": (_SZ, [_I, _I, _I]),
    "bst_attention_keymajor": (_I, [_P, _I64, _P, _I64, _P, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _P, _I, _I, _P,
                                    _I, _I, _P, _SZ, _P]),
    "bst_embed_rmsnorm": (_I, [_P, _I, _P, _I, _P, C.c_float, _P, _P, _I64, _P]),
    "bst_residual_dense": (_I, [_P, _I, _I64, _P, _I, _I, _P, C.c_float, _P, _I64, _P, _I64, _P]),
    "bst_residual_rmsnorm": (_I, [_P, _P, _P, _I, _I, _P, C.c_float, _P, _I64, _P, _I64, _P]),
    "bst_qkv_rope": (_I, [_P, C.POINTER(GemmSched), _I, _I, _I, _P, _P, C.c_float, _P, _P, _P, _P, _P, _I64, _P, _I64,
                          _P, _I, _P, _I, _P]),
    "bst_qkv_rope_batch": (_I, [_P, C.POINTER(GemmSched), _I, _I, _I, _P, _P, C.c_float, _P, _P, _P, _P, _P, _I64,
                                _P, _I64, _P, _I, _P, _I, _I, _I, _I, _I, _P, _P]),
    "bst_swiglu": (_I, [_P, C.POINTER(GemmSched), _I, _I, _P, _I64, _P]),
    "bst_gather_rows": (_I, [_P, _I64, _P, _P, _I, _I, _P, _I64, _P, _P]),
    "bst_attention_ragged": (_I, [_P, _I64, _P, _I64, _P, _I, _I, _I, _P, _I, _I, _I, _I, _I, _P, _P, _I, _I, _P, _I,
                                  _I, _I, _P, _I, _I, _P, _SZ, _P]),
    "bst_ragged_rows": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bst_ragged_unpack": (_I, [_P, _P, _P, _I, _I, _P, _P]),
    "bst_batch_plan": (_I, [_P, _P, _P, _P, _I, _I, _I, _P]),
    "bst_struct_size": (_I, [_I]),
    "bst_verify_rows": (_I, [_P, _P, _P, _P, _I, _P, _P, _P, _P]),
    "bst_drafter_rows": (_I, [_P, _I, _I, _I, _P, _P, _P, _P, _P]),
    "bst_drafter_rows_batch": (_I, [_P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "bst_commit_state": (_I, [_P, _P, _P, _I, _P, _I, _P, _P, _P, _P, _I, _P]),
    "bst_set_prefetch": (_I, [C.POINTER(Prefetch)]),
    "bst_accept": (_I, [_P, _P, _P, _P, _I, _P, _P, _P, _P]),
    "bst_kv_compact": (_I, [_P, _I, _I, _I, _I, _I64, _P, _P, _P, _P, _I, _P]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libbastion.so once; raise loudly if it is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"libbastion.so not built at {LIB_PATH}; run __graft_entry__.build()")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == BST_OK:
        return
    msg = (lib().bst_last_error() or b"").decode(errors="replace")
    if rc == BST_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"bastion error {rc}: {msg}")


# kernels launched by one call of each C-ABI entry point (for the bench's gpu_launches claim)
KERNELS_PER_CALL = {
    "bst_topk_logits": 2, "bst_topk_gemm_partial": 2, "bst_topk_probs": 2, "bst_expand": 1, "bst_expand_dev": 1, "bst_expand_dev_batch": 1, "bst_linearize_mask": 1,
    "bst_ancestor_mask": 1, "bst_accept": 1, "bst_kv_compact": 1, "bst_gemm": 1, "bst_gemm_reduce": 1,
    "bst_gemm_argmax": 2, "bst_attention": 1, "bst_attention_keymajor": 1, "bst_attention_batch": 1, "bst_embed_rmsnorm": 1, "bst_residual_rmsnorm": 1, "bst_residual_dense": 1, "bst_qkv_rope": 1,
    "bst_swiglu": 1, "bst_gather_rows": 1, "bst_verify_rows": 1, "bst_drafter_rows": 1, "bst_commit_state": 1,
    "bst_qkv_rope_batch": 1, "bst_drafter_rows_batch": 1, "bst_attention_ragged": 1, "bst_ragged_rows": 1,
    "bst_ragged_unpack": 1, "bst_batch_plan": 1, "bst_gemm_argmax_keys": 2, "bst_argmax_from_keys": 1, "bst_gemm_sample": 2,
}
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    check(getattr(lib(), name)(*args))
    launch_count += KERNELS_PER_CALL.get(name, 0)
    if name in ("bst_attention", "bst_attention_keymajor") and args[20] != 1:  # split-KV combine kernel (n_splits arg may resolve > 1)
        launch_count += 1
