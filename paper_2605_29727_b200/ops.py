"""Python handles for the model-side kernels (K3/K4/K5) of libbastion.so.

Each op takes device tensors and launches on the current torch stream; there
is no eager/torch fallback — a missing library or device raises.
"""

from __future__ import annotations

import ctypes as C
from functools import lru_cache

import torch

from . import _lib
from .device import stream_ptr


@lru_cache(maxsize=None)
def gemm_schedule(n_out: int, k: int, m: int, grid: int = 0) -> _lib.GemmSched:
    s = _lib.GemmSched()
    _lib.call("bst_gemm_schedule", n_out, k, m, grid, C.byref(s))
    return s


class PartialOut:
    """fp32 stream-K partial slots of one GEMM launch (consumed by fused epilogues)."""

    def __init__(self, sched: _lib.GemmSched, buf: torch.Tensor):
        self.sched, self.buf = sched, buf


def gemm_partial(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None, grid: int = 0) -> PartialOut:
    """X[m,K] (bf16, row stride ld) . W[n_out,K]^T -> fp32 partial slots."""
    m, k = x.shape
    n_out = w.shape[0]
    assert w.shape[1] == k and x.dtype == torch.bfloat16 and w.dtype == torch.bfloat16
    assert x.stride(1) == 1 and w.is_contiguous()
    s = gemm_schedule(n_out, k, m, grid)
    if out is None or out.numel() < s.partial_floats:
        out = torch.empty(s.partial_floats, dtype=torch.float32, device=x.device)
    _lib.call("bst_gemm", w.data_ptr(), x.data_ptr(), x.stride(0), C.byref(s), out.data_ptr(), out.numel() * 4,
              stream_ptr())
    return PartialOut(s, out)


def gemm_reduce(p: PartialOut, dtype=torch.float32) -> torch.Tensor:
    s = p.sched
    y = torch.empty((s.m, s.n_out), dtype=dtype, device=p.buf.device)
    f32 = y.data_ptr() if dtype == torch.float32 else None
    b16 = y.data_ptr() if dtype == torch.bfloat16 else None
    _lib.call("bst_gemm_reduce", p.buf.data_ptr(), C.byref(s), f32, b16, s.n_out, stream_ptr())
    return y


def linear(x: torch.Tensor, w: torch.Tensor, dtype=torch.float32) -> torch.Tensor:
    """Convenience: Y = X W^T through the tcgen05 kernel (tests / non-fused callers)."""
    return gemm_reduce(gemm_partial(x, w), dtype)


def gemm_argmax(p: PartialOut, out: torch.Tensor | None = None, scratch: torch.Tensor | None = None) -> torch.Tensor:
    s = p.sched
    out = out if out is not None else torch.empty(s.m, dtype=torch.int32, device=p.buf.device)
    scratch = scratch if scratch is not None else torch.empty(s.m, dtype=torch.int64, device=p.buf.device)
    _lib.call("bst_gemm_argmax", p.buf.data_ptr(), C.byref(s), scratch.data_ptr(), out.data_ptr(), stream_ptr())
    return out
