"""Target verify forward and DFlash-style drafter forward over the C-ABI kernels.

Every launch goes to the current torch stream and reads its per-cycle scalars
(context length c, pending drafter rows, bonus token) from the device-resident
decode ``state`` — so both forwards can be captured once in a CUDA graph and
replayed every cycle without a host round trip.

Per target layer (s rows):
  qkv  = K4(x)                     -> K5 qkv_rope: q/k norm, RoPE(c+depth), KV append at c+row
  attn = K3(q, paged KV, ancestor bitmask)
  o    = K4(attn)                  -> K5 residual += o; x = RMSNorm
  gu   = K4(x)                     -> K5 SwiGLU
  dn   = K4(act)                   -> K5 residual += dn; x = RMSNorm(next); tap features
LM head: K4 -> per-row argmax (numpy tie-break) or fp32 logits.
"""

from __future__ import annotations

import math

import torch

from .. import ops
from .config import DrafterConfig, ModelConfig
from .weights import DrafterWeights, TargetWeights, rope_inv_freq

import os

PAGE = 64
MODE_TREE, MODE_CAUSAL, MODE_FULL = 0, 1, 2
# profiling only: skip kernel families to measure their in-graph cost (results become garbage)
_ABLATE = set(filter(None, os.environ.get("BST_ABLATE", "").split(",")))
# L2 weight prefetch during DRAM-idle kernels: off by default (measured no gain: the small
# GEMMs are bound by per-SM TMA issue + DRAM burst latency, not by DRAM bytes); BST_PREFETCH=1
# (BST_PREFETCH=o,gate_up,down,qkv selects single sites for measurement)
_PF_ENV = os.environ.get("BST_PREFETCH", "0")
_PREFETCH = {"o", "gate_up", "down", "qkv"} if _PF_ENV == "1" else set(filter(None, _PF_ENV.split(","))) - {"0"}
MB = 1 << 20


def _pf(site: str, *ranges) -> None:
    if site in _PREFETCH:
        ops.set_prefetch(*ranges)
SKIP_SLOT = -(2**31)


class PagedKV:
    """[layer][page][K|V][n_kv][64][128] bf16, zero-initialised (masked slots stay finite)."""

    def __init__(self, n_layers: int, n_kv: int, max_slots: int, dev) -> None:
        self.n_layers, self.n_kv = n_layers, n_kv
        self.n_pages = (max_slots + PAGE - 1) // PAGE
        self.layer_stride = self.n_pages * 2 * n_kv * PAGE * 128
        self.buf = torch.zeros(n_layers * self.layer_stride, dtype=torch.bfloat16, device=dev)
        self.page_table = torch.arange(self.n_pages, dtype=torch.int32, device=dev)

    @property
    def max_slots(self) -> int:
        return self.n_pages * PAGE


def _n_sm(dev) -> int:
    return torch.cuda.get_device_properties(dev).multi_processor_count if torch.cuda.is_available() else 148


def _attn_ws_floats(cfg: ModelConfig, max_rows: int, pages: int, n_sm: int = 148) -> int:
    """Split partials of the largest K3 launch: the default split count is n_sm / (n_kv x
    row blocks) (bst_attention); twice that bounds the key-major kernel's cluster plans."""
    g = cfg.n_q // cfg.n_kv
    best = 0
    for s in range(1, max_rows + 1):
        rb = math.ceil(g * s / 128)
        splits = max(1, 2 * n_sm // (cfg.n_kv * rb))
        splits = min(splits, pages)
        pps = math.ceil(pages / splits)
        splits = math.ceil(pages / pps)
        if splits > 1:
            best = max(best, splits * s * cfg.n_q * 130)
    # two alternating banks of partials + the 4 KiB split-counter head (zero-initialised, kept zero by K3)
    return 2 * best + 1024


def _row_cap(n_out: int, k: int) -> int:
    """Most rows one K4 launch of this weight shape takes: 512 on the CTA-pair kernel
    (even weight-tile counts), else 256."""
    try:
        ops.gemm_schedule(n_out, k, 512)
        return 512
    except ValueError:
        return 256


def _gemm_rows(n: int, k: int, rows: int) -> int:
    """Largest row count <= rows one K4 launch of this shape takes."""
    return min(rows, _row_cap(n, k))


def row_chunks(n: int, cap: int) -> list[tuple[int, int]]:
    """Balanced row ranges of at most `cap` rows covering [0, n) (verify trees > 512 rows)."""
    nch = -(-n // cap)
    base = -(-n // nch)
    return [(r0, min(n, r0 + base)) for r0 in range(0, n, base)]


def _max_partial(shapes, max_rows: int) -> int:
    """Partial-slot floats of the largest launch any row chunk <= max_rows needs."""
    best = 0
    for n, k in shapes:
        cap = _gemm_rows(n, k, max_rows)
        for m in sorted({cap, *range(16, cap + 1, 16)}):
            best = max(best, ops.gemm_schedule(n, k, m).partial_floats)
    return best


class TargetModel:
    def __init__(self, cfg: ModelConfig, w: TargetWeights, max_slots: int, max_rows: int, feat_layers, dev) -> None:
        self.cfg, self.w, self.dev, self.max_rows = cfg, w, dev, max_rows
        self.kv = PagedKV(cfg.L, cfg.n_kv, max_slots, dev)
        self.inv_freq = rope_inv_freq(cfg, dev)
        self.feat_layers = tuple(feat_layers)
        R, h = max_rows, cfg.h
        f32, bf = dict(dtype=torch.float32, device=dev), dict(dtype=torch.bfloat16, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self.resid = torch.empty(R, h, **f32)
        self.x = torch.empty(R, h, **bf)
        self.q = torch.empty(R, cfg.h_q, **bf)
        self.attn = torch.empty(R, cfg.h_q, **bf)
        self.act = torch.empty(R, cfg.h_ffn, **bf)
        self.feat = torch.empty(R, max(1, len(self.feat_layers)) * h, **bf)
        self.tokens = torch.zeros(R, **i32)
        self.pos = torch.zeros(R, **i32)
        self.slot = torch.zeros(R, **i32)
        self.argmax = torch.zeros(R, **i32)
        self.amx_scratch = torch.zeros(R, dtype=torch.int64, device=dev)
        shapes = [(cfg.qkv_out, h), (h, cfg.h_q), (2 * cfg.h_ffn, h), (h, cfg.h_ffn), (cfg.V, h)]
        self.partial = torch.empty(_max_partial(shapes, R), **f32)
        self.attn_ws = torch.zeros(_attn_ws_floats(cfg, R, self.kv.n_pages, _n_sm(dev)), **f32)
        self.attn_splits = 0  # K3 split count (0: automatic); parity tests pin it
        self.logits = None
        self.temperature, self.sample_seed = 0.0, 0  # head "sample": Gumbel-max at T keyed by (seed, c + pos)

    def _chunks(self, n: int) -> dict:
        cfg, h = self.cfg, self.cfg.h
        cap_qkv = _row_cap(cfg.qkv_out, h)
        cap_mlp = min(_row_cap(h, cfg.h_q), _row_cap(2 * cfg.h_ffn, h), _row_cap(h, cfg.h_ffn))
        return {"qkv": row_chunks(n, cap_qkv), "mlp": row_chunks(n, cap_mlp)}

    def forward(self, rows: int, state: torch.Tensor, mode: int, keys_after_c: int, anc=None, mask_words: int = 0,
                head: str | None = "argmax", c_host: int = 0, pt: torch.Tensor | None = None,
                batch: tuple[int, int, int] | None = None, ragged: tuple | None = None) -> None:
        """Run `rows` query rows (tokens/pos/slot buffers already filled, relative to c = state[0]).

        pt: page-table view (a request's page range in a shared pool; default the whole table).
        batch = (n_req, S, req_pages): rows are n_req requests of S rows each; request r's
        state is state[r] (8 words), its pages pt[r*req_pages:], its mask rows anc[r*S:].
        ragged = (n_req, S, req_pages, row_req, row_off, row_cnt): packed rows of variable
        per-request counts (device arrays from bst_ragged_rows); masks keep the S stride."""
        cfg, w, kv = self.cfg, self.w, self.kv
        n, eps = rows, cfg.eps
        if head == "sample" and (batch is not None or ragged is not None):
            # bst_gemm_sample keys every row by one state's context c
            raise ValueError("sampled verification is per request: the batched head supports argmax only")
        pt = kv.page_table if pt is None else pt
        x, resid = self.x[:n], self.resid[:n]
        ops.embed_rmsnorm(self.tokens, n, w.emb, w.layers[0].in_norm, eps, resid, x)
        # trees wider than one K4 launch (> 256/512 rows, N_max up to 1024) run every GEMM and
        # its row-local epilogue in balanced row chunks; K3 always takes every row at once
        ck = self._chunks(n)
        for li, lw in enumerate(w.layers):
            nxt_l = w.layers[li + 1] if li + 1 < cfg.L else None
            for r0, r1 in ck["qkv"]:
                if "rope" in _ABLATE:
                    ops.gemm_partial(x[r0:r1], lw.qkv, out=self.partial)
                    continue
                req, row_req = (0, 1, 0, 0), None
                if batch is not None:
                    req = (batch[1], batch[0] * batch[1], state.stride(0), batch[2] * PAGE)
                elif ragged is not None:
                    req, row_req = (0, 1, state.stride(0), ragged[2] * PAGE), ragged[3][r0:]
                ops.gemm_qkv_rope(x[r0:r1], lw.qkv, self.partial, cfg.n_q, cfg.n_kv, lw.q_norm, lw.k_norm,
                                  eps, self.inv_freq, self.pos[r0:], self.slot[r0:], None, self.q[r0:], kv.buf,
                                  li * kv.layer_stride, pt, PAGE, state, req, row_req)
            if "attn" not in _ABLATE:
                _pf("o", (lw.o, lw.o.numel() * 2), (lw.gate_up, 32 * MB) if "gate_up" in _PREFETCH else None)
                if ragged is not None:
                    nr, S, rp, _, off, cnt = ragged
                    ops.attention_ragged(self.q[:n], self.attn[:n], kv.buf, cfg.L, kv.n_pages, li, pt, rp, cfg.n_q,
                                         cfg.n_kv, nr, S, off, cnt, S, rp * PAGE, state, state.stride(0), mode, anc,
                                         mask_words, self.attn_ws, n_splits=self.attn_splits)
                elif batch is None:
                    ops.attention(self.q[:n], self.attn[:n], kv.buf, cfg.L, kv.n_pages, li, pt, cfg.n_q,
                                  cfg.n_kv, n, c_host, keys_after_c, kv.max_slots, state, mode, anc, mask_words,
                                  self.attn_ws, n_splits=self.attn_splits)
                else:
                    nr, S, rp = batch
                    ops.attention_batch(self.q[:n], self.attn[:n], kv.buf, cfg.L, kv.n_pages, li, pt, rp, cfg.n_q,
                                        cfg.n_kv, nr, S, keys_after_c, rp * PAGE, state, state.stride(0), mode, anc,
                                        mask_words, self.attn_ws, n_splits=self.attn_splits)
            nxt = w.layers[li + 1].in_norm if li + 1 < cfg.L else w.final_norm
            j = self.feat_layers.index(li) if li in self.feat_layers else -1
            for r0, r1 in ck["mlp"]:
                m = r1 - r0
                p = ops.gemm_partial(self.attn[r0:r1], lw.o, out=self.partial)
                if "resid" not in _ABLATE:
                    _pf("gate_up", (lw.gate_up[lw.gate_up.shape[0] // 8:], 24 * MB))
                    ops.residual_rmsnorm(p, resid[r0:r1], m, cfg.h, lw.post_norm, eps, x=x[r0:r1])
                p = ops.gemm_partial(x[r0:r1], lw.gate_up, out=self.partial)
                if "swiglu" not in _ABLATE:
                    _pf("down", (lw.down, 16 * MB))
                    ops.swiglu(p, m, cfg.h_ffn, self.act[r0:r1])
                p = ops.gemm_partial(self.act[r0:r1], lw.down, out=self.partial)
                feat = self.feat[r0:r1, j * cfg.h:(j + 1) * cfg.h] if j >= 0 else None
                if "resid" not in _ABLATE:
                    _pf("qkv", (nxt_l.qkv, nxt_l.qkv.numel() * 2) if nxt_l is not None else (w.lm_head, 48 * MB))
                    ops.residual_rmsnorm(p, resid[r0:r1], m, cfg.h, nxt, eps, x=x[r0:r1], feat=feat)
        # LM head in row chunks the K4 schedule accepts (odd vocab tile counts: <= 256 rows)
        hr = _gemm_rows(w.lm_head.shape[0], cfg.h, n)
        logits = []
        for r0 in range(0, n, hr):
            r1 = min(n, r0 + hr)
            if head == "argmax":
                p = ops.gemm_partial(x[r0:r1], w.lm_head, out=self.partial)
                ops.gemm_argmax(p, out=self.argmax[r0:r1], scratch=self.amx_scratch[r0:])
            elif head == "sample":
                p = ops.gemm_partial(x[r0:r1], w.lm_head, out=self.partial)
                ops.gemm_sample(p, self.pos[r0:], state, self.temperature, self.sample_seed, out=self.argmax[r0:r1],
                                scratch=self.amx_scratch[r0:])
            elif head == "logits":
                p = ops.gemm_partial(x[r0:r1], w.lm_head, out=self.partial)
                logits.append(ops.gemm_reduce(p))
        if head == "logits":
            self.logits = logits[0] if len(logits) == 1 else torch.cat(logits)


class DrafterModel:
    """Block drafter: gamma+1 query rows ([bonus] + gamma masks) + gamma+1 context rows."""

    def __init__(self, cfg: ModelConfig, dcfg: DrafterConfig, w: DrafterWeights, target: TargetWeights,
                 max_slots: int, n_feat: int, dev, prefill_rows: int = 256, n_req_max: int = 1) -> None:
        self.cfg, self.dcfg, self.w, self.tw, self.dev = cfg, dcfg, w, target, dev
        self.kv = PagedKV(dcfg.layers, cfg.n_kv, max_slots, dev)
        self.inv_freq = rope_inv_freq(cfg, dev)
        self.B = dcfg.gamma + 1
        self.CR = dcfg.gamma + 1
        self.n_req_max = n_req_max
        self.mask_token = dcfg.mask_token if dcfg.mask_token >= 0 else cfg.V - 1
        R = max((self.B + self.CR) * n_req_max, prefill_rows)
        QB = self.B * n_req_max
        h = cfg.h
        f32, bf = dict(dtype=torch.float32, device=dev), dict(dtype=torch.bfloat16, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self.resid = torch.empty(QB, h, **f32)
        self.X = torch.zeros(R, h, **bf)
        self.q = torch.empty(QB, cfg.h_q, **bf)
        self.attn = torch.empty(QB, cfg.h_q, **bf)
        self.act = torch.empty(QB, cfg.h_ffn, **bf)
        self.feat_in = torch.zeros(max(self.CR * n_req_max, prefill_rows), n_feat * h, **bf)
        self.tokens = torch.zeros(R, **i32)
        self.pos = torch.zeros(R, **i32)
        self.slot = torch.zeros(R, **i32)
        self.qrow = torch.zeros(R, **i32)
        shapes = [(cfg.qkv_out, h), (h, cfg.h_q), (2 * cfg.h_ffn, h), (h, cfg.h_ffn), (cfg.V, h), (h, n_feat * h)]
        self.partial = torch.empty(_max_partial(shapes, min(R, 256)), **f32)  # every GEMM call has <= 256 rows
        self.attn_ws = torch.zeros(_attn_ws_floats(cfg, QB, self.kv.n_pages, _n_sm(dev)), **f32)
        self.attn_splits = 0
        self.logits = torch.empty(dcfg.gamma, cfg.V, **f32)
        self.logits_b = torch.empty(QB, cfg.V, **f32) if n_req_max > 1 else None

    def _ctx_rows(self, n: int, x_ctx: torch.Tensor, state: torch.Tensor, feat: torch.Tensor | None = None) -> None:
        """fc + hidden_norm of n feature rows -> x_ctx (context inputs of every drafter layer)."""
        cfg = self.cfg
        p = ops.gemm_partial(self.feat_in[:n] if feat is None else feat[:n], self.w.fc, out=self.partial)
        ops.residual_rmsnorm(p, None, n, cfg.h, self.w.hidden_norm, cfg.eps, x=x_ctx)

    def prefill_ctx(self, n: int, state: torch.Tensor, pt: torch.Tensor | None = None) -> None:
        """Write context K/V for n prompt rows (features in feat_in[:n], pos/slot = 0..n-1 relative to c)."""
        cfg = self.cfg
        pt = self.kv.page_table if pt is None else pt
        x = self.X[:n]
        self._ctx_rows(n, x, state)
        self.qrow[:n].fill_(-1)
        for li, lw in enumerate(self.w.layers):
            ops.gemm_qkv_rope(x, lw.qkv, self.partial, cfg.n_q, cfg.n_kv, lw.q_norm, lw.k_norm,
                              cfg.eps, self.inv_freq, self.pos, self.slot, self.qrow, self.q, self.kv.buf,
                              li * self.kv.layer_stride, pt, PAGE, state)

    def forward(self, state: torch.Tensor, reduce: bool = True):
        """Draft one block: returns logits [gamma, V] fp32 for future positions c+1..c+gamma
        (reduce=False: the LM head's ``ops.PartialOut`` for K1 to read directly)."""
        cfg, w, B, CR = self.cfg, self.w, self.B, self.CR
        eps, M = cfg.eps, B + CR
        ops.drafter_rows(state, self.dcfg.gamma, self.mask_token, CR, self.tokens, self.pos, self.slot, self.qrow)
        self._ctx_rows(CR, self.X[B:M], state)
        xb, resid = self.X[:B], self.resid[:B]
        ops.embed_rmsnorm(self.tokens, B, self.tw.emb, w.layers[0].in_norm, eps, resid, xb)
        for li, lw in enumerate(w.layers):
            ops.gemm_qkv_rope(self.X[:M], lw.qkv, self.partial, cfg.n_q, cfg.n_kv, lw.q_norm,
                              lw.k_norm, eps, self.inv_freq, self.pos, self.slot, self.qrow, self.q, self.kv.buf,
                              li * self.kv.layer_stride, self.kv.page_table, PAGE, state)
            ops.attention(self.q[:B], self.attn[:B], self.kv.buf, self.dcfg.layers, self.kv.n_pages, li,
                          self.kv.page_table, cfg.n_q, cfg.n_kv, B, 0, B, self.kv.max_slots, state, MODE_FULL, None, 0,
                          self.attn_ws, n_splits=self.attn_splits)
            p = ops.gemm_partial(self.attn[:B], lw.o, out=self.partial)
            ops.residual_rmsnorm(p, resid, B, cfg.h, lw.post_norm, eps, x=xb)
            p = ops.gemm_partial(xb, lw.gate_up, out=self.partial)
            ops.swiglu(p, B, cfg.h_ffn, self.act[:B])
            p = ops.gemm_partial(self.act[:B], lw.down, out=self.partial)
            nxt = w.layers[li + 1].in_norm if li + 1 < len(w.layers) else w.final_norm
            ops.residual_rmsnorm(p, resid, B, cfg.h, nxt, eps, x=xb)
        p = ops.gemm_partial(self.X[1:B], self.tw.lm_head, out=self.partial)
        if not reduce:
            return p
        _reduce_into(p, self.logits)
        return self.logits

    def forward_batch(self, state: torch.Tensor, n: int, pt: torch.Tensor, req_pages: int,
                      feat: torch.Tensor | None = None) -> torch.Tensor:
        """Draft one block for n requests at once (state[r] = request r's 8 state words,
        pages pt[r*req_pages:], context features feat_in[r*CR:(r+1)*CR]).

        Rows: the n*(gamma+1) block rows first (request-major), then the n*CR context rows.
        Returns fp32 logits [n*(gamma+1), V]; request r's draft rows are 1..gamma of its block."""
        cfg, w, B, CR = self.cfg, self.w, self.B, self.CR
        eps = cfg.eps
        QB, M = n * B, n * (B + CR)
        rs = state.stride(0)
        ops.drafter_rows_batch(state, rs, n, self.dcfg.gamma, self.mask_token, CR, self.tokens, self.pos, self.slot,
                               self.qrow)
        self._ctx_rows(n * CR, self.X[QB:M], state, feat)
        xb, resid = self.X[:QB], self.resid[:QB]
        ops.embed_rmsnorm(self.tokens, QB, self.tw.emb, w.layers[0].in_norm, eps, resid, xb)
        for li, lw in enumerate(w.layers):
            # block rows, then context rows: two GEMMs of <= 256 rows each (the K4 row limit), so
            # a chunk of up to 256 / (gamma + 1) requests shares every drafter weight pass
            for lo, hi in ((0, QB), (QB, M)):
                ops.gemm_qkv_rope(self.X[lo:hi], lw.qkv, self.partial, cfg.n_q, cfg.n_kv, lw.q_norm,
                                  lw.k_norm, eps, self.inv_freq, self.pos[lo:], self.slot[lo:], self.qrow[lo:],
                                  self.q, self.kv.buf, li * self.kv.layer_stride, pt, PAGE, state,
                                  (B, QB, rs, req_pages * PAGE))
            ops.attention_batch(self.q[:QB], self.attn[:QB], self.kv.buf, self.dcfg.layers, self.kv.n_pages, li, pt,
                                req_pages, cfg.n_q, cfg.n_kv, n, B, B, req_pages * PAGE, state, rs, MODE_FULL, None,
                                0, self.attn_ws, n_splits=self.attn_splits)
            p = ops.gemm_partial(self.attn[:QB], lw.o, out=self.partial)
            ops.residual_rmsnorm(p, resid, QB, cfg.h, lw.post_norm, eps, x=xb)
            p = ops.gemm_partial(xb, lw.gate_up, out=self.partial)
            ops.swiglu(p, QB, cfg.h_ffn, self.act[:QB])
            p = ops.gemm_partial(self.act[:QB], lw.down, out=self.partial)
            nxt = w.layers[li + 1].in_norm if li + 1 < len(w.layers) else w.final_norm
            ops.residual_rmsnorm(p, resid, QB, cfg.h, nxt, eps, x=xb)
        p = ops.gemm_partial(xb, self.tw.lm_head, out=self.partial)
        _reduce_into(p, self.logits_b[:QB])
        return self.logits_b[:QB]


DRAFT_PREFILL_ROWS = 256  # drafter context rows per prefill launch (its GEMM partials hold 256 rows)


def drafter_prefill(d: "DrafterModel", feat: torch.Tensor, n: int, state: torch.Tensor, start: int,
                    pt: torch.Tensor | None = None) -> None:
    """Drafter context K/V for prompt rows [start, start + n) from the target's feature rows
    feat[:n], in launches of <= DRAFT_PREFILL_ROWS rows; state[0] (c) is set to each piece's
    first absolute position (the rows' slots are relative to c)."""
    for d0 in range(0, n, DRAFT_PREFILL_ROWS):
        dn = min(DRAFT_PREFILL_ROWS, n - d0)
        if d0:
            state[0:1].fill_(start + d0)
        d.feat_in[:dn].copy_(feat[d0:d0 + dn])
        ar = torch.arange(dn, dtype=torch.int32, device=feat.device)
        d.pos[:dn].copy_(ar)
        d.slot[:dn].copy_(ar)
        d.prefill_ctx(dn, state, pt=pt)


def _reduce_into(p: ops.PartialOut, y: torch.Tensor) -> None:
    import ctypes as C

    from .. import _lib
    from ..device import stream_ptr
    _lib.call("bst_gemm_reduce", p.buf.data_ptr(), C.byref(p.sched), y.data_ptr(), None, y.stride(0), stream_ptr())
