"""Python handles for the model-side kernels (K3/K4/K5) of libbastion.so.

Each op takes device tensors and launches on the current torch stream; there
is no eager/torch fallback — a missing library or device raises.
"""

from __future__ import annotations

import ctypes as C
import os
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


def gemm_reduce_into(p: PartialOut, y: torch.Tensor) -> torch.Tensor:
    """Dense Y[m, n_out] (fp32 or bf16, row stride y.stride(0)) from the partial slots."""
    s = p.sched
    assert y.dtype in (torch.float32, torch.bfloat16) and y.stride(1) == 1
    assert y.shape[0] >= s.m and y.shape[1] >= s.n_out
    f32 = y.data_ptr() if y.dtype == torch.float32 else None
    b16 = y.data_ptr() if y.dtype == torch.bfloat16 else None
    _lib.call("bst_gemm_reduce", p.buf.data_ptr(), C.byref(s), f32, b16, y.stride(0), stream_ptr())
    return y


def gemm_argmax_keys(p: PartialOut, keys: torch.Tensor, vocab_offset: int) -> torch.Tensor:
    """Signed int64 packed (value, global index) argmax keys of a vocab-parallel LM-head shard."""
    assert keys.dtype == torch.int64 and keys.numel() >= p.sched.m
    _lib.call("bst_gemm_argmax_keys", p.buf.data_ptr(), C.byref(p.sched), keys.data_ptr(), int(vocab_offset),
              stream_ptr())
    return keys


def argmax_from_keys(keys: torch.Tensor, m: int, out: torch.Tensor) -> torch.Tensor:
    assert keys.dtype == torch.int64 and out.dtype == torch.int32
    _lib.call("bst_argmax_from_keys", keys.data_ptr(), int(m), out.data_ptr(), stream_ptr())
    return out


def gemm_sample(p: PartialOut, pos: torch.Tensor, state: torch.Tensor | None, temperature: float, seed: int,
                out: torch.Tensor, scratch: torch.Tensor) -> torch.Tensor:
    """Per-row temperature sample (Gumbel-max keyed by (seed, c + pos[row], vocab index))."""
    s = p.sched
    _lib.call("bst_gemm_sample", p.buf.data_ptr(), C.byref(s), scratch.data_ptr(), out.data_ptr(), pos.data_ptr(),
              None if state is None else state.data_ptr(), 0, float(temperature), int(seed) & ((1 << 64) - 1),
              stream_ptr())
    return out


def gemm_argmax(p: PartialOut, out: torch.Tensor | None = None, scratch: torch.Tensor | None = None) -> torch.Tensor:
    s = p.sched
    out = out if out is not None else torch.empty(s.m, dtype=torch.int32, device=p.buf.device)
    scratch = scratch if scratch is not None else torch.empty(s.m, dtype=torch.int64, device=p.buf.device)
    _lib.call("bst_gemm_argmax", p.buf.data_ptr(), C.byref(s), scratch.data_ptr(), out.data_ptr(), stream_ptr())
    return out


def _p(t):
    return None if t is None else t.data_ptr()


def attention(q, out, kv, n_layers, n_pages, layer, page_table, n_q, n_kv, s, c, keys_after_c, max_keys, state,
              mode, anc=None, mask_words=0, ws=None, n_splits=0, keymajor=False):
    """K3 launch; q/out [s][n_q*128] bf16 (token stride = row stride).  keymajor: the
    key-major kernel (bst_attention_keymajor, measurements/tests); the engine never sets it."""
    _lib.call("bst_attention_keymajor" if keymajor else "bst_attention", q.data_ptr(), q.stride(0), out.data_ptr(), out.stride(0), kv.data_ptr(), n_layers,
              n_pages, layer, page_table.data_ptr(), n_q, n_kv, s, c, keys_after_c, max_keys, _p(state), 0, mode,
              _p(anc), mask_words, n_splits, _p(ws), 0 if ws is None else ws.numel() * 4, stream_ptr())


def attention_batch(q, out, kv, n_layers, n_pages, layer, page_table, req_pages, n_q, n_kv, n_req, s, keys_after_c,
                    max_keys, state, req_state, mode, anc=None, mask_words=0, ws=None, n_splits=0):
    """Batched K3: n_req requests of s rows each (request r: rows [r*s, r*s+s), pages
    page_table[r*req_pages:], c = state[r*req_state], mask rows anc[(r*s + i)*mask_words:])."""
    _lib.call("bst_attention_batch", q.data_ptr(), q.stride(0), out.data_ptr(), out.stride(0), kv.data_ptr(),
              n_layers, n_pages, layer, page_table.data_ptr(), req_pages, n_q, n_kv, n_req, s, keys_after_c,
              max_keys, _p(state), req_state, 0, mode, _p(anc), mask_words, n_splits, _p(ws),
              0 if ws is None else ws.numel() * 4, stream_ptr())


def embed_rmsnorm(tokens, rows, emb, w, eps, resid, x):
    _lib.call("bst_embed_rmsnorm", tokens.data_ptr(), rows, emb.data_ptr(), emb.shape[1], w.data_ptr(),
              C.c_float(eps), resid.data_ptr(), x.data_ptr(), x.stride(0), stream_ptr())


def residual_rmsnorm(p: PartialOut | None, resid, rows, h, w, eps, x=None, feat=None):
    sched = C.byref(p.sched) if p is not None else None
    _lib.call("bst_residual_rmsnorm", None if p is None else p.buf.data_ptr(), sched, _p(resid), rows, h,
              w.data_ptr(), C.c_float(eps), _p(x), 0 if x is None else x.stride(0), _p(feat),
              0 if feat is None else feat.stride(0), stream_ptr())


def residual_dense(y, resid, rows, w, eps, x, feat=None) -> None:
    """resid += y (dense fp32 / bf16 [rows, h], e.g. an all-reduced row-parallel output; None:
    normalise only); x = RMSNorm(resid) * w (bf16); feat = bf16(resid)."""
    yb = y is not None and y.dtype == torch.bfloat16
    _lib.call("bst_residual_dense", _p(y), int(yb), 0 if y is None else y.stride(0), resid.data_ptr(), rows,
              resid.shape[1], w.data_ptr(), C.c_float(eps), x.data_ptr(), x.stride(0), _p(feat),
              0 if feat is None else feat.stride(0), stream_ptr())


def gemm_qkv_rope(x, w, out, n_q, n_kv, q_norm, k_norm, eps, inv_freq, pos, slot, qrow, q_out, kv,
                  layer_off, page_table, page_size, state, req=(0, 1, 0, 0), row_req=None) -> None:
    """q/k/v projection (K4) then q/k RMSNorm + RoPE + q and paged-KV stores (K5 qkv_rope)
    of the m = x.shape[0] rows.  (A variant fusing the epilogue into the GEMM's stream-K
    tile fixup was measured slower: it raised the GEMM to 168 registers, which blocks the
    PDL co-residency of the epilogue kernels, and serialised one head x all rows per CTA.)"""
    p = gemm_partial(x, w, out=out)
    qkv_rope_batch(p, x.shape[0], n_q, n_kv, q_norm, k_norm, eps, inv_freq, pos, slot, qrow, q_out, kv, layer_off,
                   page_table, page_size, state, *req, row_req=row_req)


def qkv_rope(p: PartialOut, rows, n_q, n_kv, q_norm, k_norm, eps, inv_freq, pos, slot, qrow, q_out, kv, layer_off,
             page_table, page_size, state):
    _lib.call("bst_qkv_rope", p.buf.data_ptr(), C.byref(p.sched), rows, n_q, n_kv, q_norm.data_ptr(),
              k_norm.data_ptr(), C.c_float(eps), inv_freq.data_ptr(), pos.data_ptr(), slot.data_ptr(), _p(qrow),
              q_out.data_ptr(), q_out.stride(0), kv.data_ptr(), layer_off, page_table.data_ptr(), page_size,
              _p(state), 0, stream_ptr())


def qkv_rope_batch(p: PartialOut, rows, n_q, n_kv, q_norm, k_norm, eps, inv_freq, pos, slot, qrow, q_out, kv,
                   layer_off, page_table, page_size, state, req_rows, req_span, req_state, req_slots, row_req=None):
    _lib.call("bst_qkv_rope_batch", p.buf.data_ptr(), C.byref(p.sched), rows, n_q, n_kv, q_norm.data_ptr(),
              k_norm.data_ptr(), C.c_float(eps), inv_freq.data_ptr(), pos.data_ptr(), slot.data_ptr(), _p(qrow),
              q_out.data_ptr(), q_out.stride(0), kv.data_ptr(), layer_off, page_table.data_ptr(), page_size,
              _p(state), 0, req_rows, req_span, req_state, req_slots, _p(row_req), stream_ptr())


def swiglu(p: PartialOut, rows, ffn, act):
    _lib.call("bst_swiglu", p.buf.data_ptr(), C.byref(p.sched), rows, ffn, act.data_ptr(), act.stride(0),
              stream_ptr())


def gather_rows(src, idx, count, max_rows, dst, row_base=None):
    """dst[r] = src[row_base + idx[r]] for r < count (row_base: a device int32, default 0)."""
    _lib.call("bst_gather_rows", src.data_ptr(), src.stride(0), idx.data_ptr(), _p(count), max_rows, src.shape[1],
              dst.data_ptr(), dst.stride(0), _p(row_base), stream_ptr())


def attention_ragged(q, out, kv, n_layers, n_pages, layer, page_table, req_pages, n_q, n_kv, n_req, s_max, row_off,
                     row_cnt, keys_after_c, max_keys, state, req_state, mode, anc, mask_words, ws=None, n_splits=0):
    """Ragged batched K3: request r's rows are q/out rows [row_off[r], row_off[r] + row_cnt[r])."""
    _lib.call("bst_attention_ragged", q.data_ptr(), q.stride(0), out.data_ptr(), out.stride(0), kv.data_ptr(),
              n_layers, n_pages, layer, page_table.data_ptr(), req_pages, n_q, n_kv, n_req, s_max, row_off.data_ptr(),
              row_cnt.data_ptr(), keys_after_c, max_keys, state.data_ptr(), req_state, 0, mode, _p(anc), mask_words,
              n_splits, _p(ws), 0 if ws is None else ws.numel() * 4, stream_ptr())


def ragged_rows(trees_dev, state, n_req, s_max, rows_cap, row_off, row_cnt, total, tokens, pos, slot, row_req):
    _lib.call("bst_ragged_rows", trees_dev.data_ptr(), state.data_ptr(), state.stride(0), n_req, s_max, rows_cap,
              row_off.data_ptr(), row_cnt.data_ptr(), total.data_ptr(), tokens.data_ptr(), pos.data_ptr(),
              slot.data_ptr(), row_req.data_ptr(), stream_ptr())


def ragged_unpack(src, row_off, row_cnt, n_req, s_max, dst):
    _lib.call("bst_ragged_unpack", src.data_ptr(), row_off.data_ptr(), row_cnt.data_ptr(), n_req, s_max,
              dst.data_ptr(), stream_ptr())


def batch_plan(base, out, trees_dev, state, n_req, first):
    _lib.call("bst_batch_plan", base.data_ptr(), out.data_ptr(), trees_dev.data_ptr(), state.data_ptr(),
              state.stride(0), n_req, int(first), stream_ptr())


def kv_compact(kv, n_layers, n_kv, page_size, layer_stride, page_table, state, path, meta, max_path):
    _lib.call("bst_kv_compact", kv.data_ptr(), n_layers, n_kv, 128, page_size, layer_stride, page_table.data_ptr(),
              state.data_ptr(), path.data_ptr(), meta.data_ptr(), max_path, stream_ptr())


def verify_rows(state, tree_token, tree_depth, meta, rows, tokens, pos, slot):
    _lib.call("bst_verify_rows", state.data_ptr(), tree_token.data_ptr(), tree_depth.data_ptr(), meta.data_ptr(),
              rows, tokens.data_ptr(), pos.data_ptr(), slot.data_ptr(), stream_ptr())


def drafter_rows(state, gamma, mask_token, ctx_rows, tokens, pos, slot, qrow):
    _lib.call("bst_drafter_rows", state.data_ptr(), gamma, mask_token, ctx_rows, tokens.data_ptr(), pos.data_ptr(),
              slot.data_ptr(), qrow.data_ptr(), stream_ptr())


def drafter_rows_batch(state, req_state, n_req, gamma, mask_token, ctx_rows, tokens, pos, slot, qrow):
    _lib.call("bst_drafter_rows_batch", state.data_ptr(), req_state, n_req, gamma, mask_token, ctx_rows,
              tokens.data_ptr(), pos.data_ptr(), slot.data_ptr(), qrow.data_ptr(), stream_ptr())


def commit_state(state, accept_meta, committed, max_path, out_tokens, tree_meta=None, surrogate=None, log_i32=None,
                 log_f64=None):
    cap = 0 if log_i32 is None else log_i32.numel() // 8
    _lib.call("bst_commit_state", state.data_ptr(), accept_meta.data_ptr(), committed.data_ptr(), max_path,
              out_tokens.data_ptr(), out_tokens.numel(), _p(tree_meta), _p(surrogate), _p(log_i32), _p(log_f64), cap,
              stream_ptr())


def set_prefetch(*ranges) -> None:
    """L2 prefetch hint for the next K3/K5 launch: up to two (tensor, max_bytes) ranges."""
    pf = _lib.Prefetch()
    for i, r in enumerate(ranges[:2]):
        if r is None or r[0] is None:
            continue
        t, nbytes = r
        n = min(int(nbytes), t.numel() * t.element_size()) & ~15
        pf.ptr[i] = t.data_ptr()
        pf.bytes[i] = n
    _lib.call("bst_set_prefetch", C.byref(pf))
