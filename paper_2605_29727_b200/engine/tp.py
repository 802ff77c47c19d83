"""Tensor-parallel target verify — BASELINE config 5 (Qwen3-32B shape, TP=8, NCCL
all-reduce over NVLink, tree verify + accept).  SURVEY §8e.

Rank r of a tp-way group holds
  * q/k/v (column-parallel): query heads [r n_q/tp, (r+1) n_q/tp) and KV heads
    [r n_kv/tp, ...), so attention and the paged KV cache are head-local;
  * o_proj, down_proj (row-parallel): the matching input columns; their outputs are
    partial sums of the residual stream, all-reduced (SUM, bf16 by default: half the
    NVLink bytes of fp32, ``set_allreduce_dtype``) before the residual update + RMSNorm;
  * gate/up (column-parallel): FFN columns [r h_ffn/tp, ...) of gate and of up;
  * the LM head (vocab-parallel): vocabulary rows [r V/tp, ...); the per-row argmax
    is reduced as one signed 64-bit key (order-preserving fp32 bits | ~global index,
    bst_gemm_argmax_keys) with a MAX all-reduce, which keeps np.argmax's lowest-index
    tie-break (verify_sim.py:107-109) bit-exactly across shards.
Embedding, norms and the decode bookkeeping (tree, accept walk, KV compaction of the
local heads, committed stream) are replicated: every rank computes the same tree from
the same lattice, so no broadcast is needed.

The collective points are exposed by ``forward_steps`` (a generator yielding
``(op, tensor)``), so the same code runs under NCCL (``dist_collective``) and in a
single-process lock-step simulation of tp shards (``run_lockstep``, the parity test).
Residual protocol at each row-parallel output: every rank reduces its partial output
y_r into a dense bf16 (or fp32) buffer (bst_gemm_reduce), the SUM all-reduce leaves
sum_r y_r on every rank, and bst_residual_dense adds it to the replicated fp32
residual and writes RMSNorm(residual) for the next column-parallel GEMM.  NCCL picks
NVLS (in-switch reduction) for this all-reduce on NVSwitch systems when available.
"""

from __future__ import annotations

from dataclasses import replace

import torch

from .. import ops
from .config import ModelConfig
from .forward import PAGE, TargetModel
from .weights import LayerWeights, TargetWeights, _normal, _ones

TP_ROWS = 256  # verify rows per TP step (config 5 budgets N in {16, 64, 256}: trees <= 255 nodes)


def local_config(cfg: ModelConfig, tp: int) -> ModelConfig:
    """Per-rank shapes of a tp-way shard (heads, FFN columns and vocabulary split evenly)."""
    if tp < 1 or cfg.n_q % tp or cfg.n_kv % tp or cfg.h_ffn % tp or cfg.V % tp:
        raise ValueError(f"{cfg.name} does not split {tp} ways (n_q, n_kv, h_ffn and V must divide)")
    return replace(cfg, name=f"{cfg.name}/tp{tp}", n_q=cfg.n_q // tp, n_kv=cfg.n_kv // tp, h_ffn=cfg.h_ffn // tp,
                   V=cfg.V // tp)


def shard_layer(lw: LayerWeights, cfg: ModelConfig, tp: int, rank: int) -> LayerWeights:
    d, hq, hkv, f = cfg.d, cfg.h_q // tp, cfg.h_kv // tp, cfg.h_ffn // tp
    q = lw.qkv[rank * hq:(rank + 1) * hq]
    k = lw.qkv[cfg.h_q + rank * hkv:cfg.h_q + (rank + 1) * hkv]
    v = lw.qkv[cfg.h_q + cfg.h_kv + rank * hkv:cfg.h_q + cfg.h_kv + (rank + 1) * hkv]
    gate = lw.gate_up[rank * f:(rank + 1) * f]
    up = lw.gate_up[cfg.h_ffn + rank * f:cfg.h_ffn + (rank + 1) * f]
    del d
    return LayerWeights(in_norm=lw.in_norm, qkv=torch.cat([q, k, v]).contiguous(), q_norm=lw.q_norm,
                        k_norm=lw.k_norm, o=lw.o[:, rank * hq:(rank + 1) * hq].contiguous(), post_norm=lw.post_norm,
                        gate_up=torch.cat([gate, up]).contiguous(),
                        down=lw.down[:, rank * f:(rank + 1) * f].contiguous())


def shard_weights(full: TargetWeights, cfg: ModelConfig, tp: int, rank: int) -> TargetWeights:
    """Rank `rank`'s slice of full target weights (parity tests)."""
    local_config(cfg, tp)
    vl = cfg.V // tp
    return TargetWeights(emb=full.emb, layers=[shard_layer(lw, cfg, tp, rank) for lw in full.layers],
                         final_norm=full.final_norm, lm_head=full.lm_head[rank * vl:(rank + 1) * vl].contiguous())


def random_shard(cfg: ModelConfig, tp: int, rank: int, seed: int, dev) -> TargetWeights:
    """Random-init weights of one shard only (the 32B bench: no rank builds the full model)."""
    lc = local_config(cfg, tp)
    g = torch.Generator(device=dev).manual_seed(seed * 1009 + rank)
    layers = [LayerWeights(in_norm=_ones(cfg.h, dev), qkv=_normal((lc.qkv_out, cfg.h), g, dev),
                           q_norm=_ones(cfg.d, dev), k_norm=_ones(cfg.d, dev), o=_normal((cfg.h, lc.h_q), g, dev),
                           post_norm=_ones(cfg.h, dev), gate_up=_normal((2 * lc.h_ffn, cfg.h), g, dev),
                           down=_normal((cfg.h, lc.h_ffn), g, dev)) for _ in range(cfg.L)]
    eg = torch.Generator(device=dev).manual_seed(seed * 1009 + 997)  # embedding replicated: same on every rank
    return TargetWeights(emb=_normal((cfg.V, cfg.h), eg, dev), layers=layers, final_norm=_ones(cfg.h, dev),
                         lm_head=_normal((lc.V, cfg.h), g, dev))


class TPTargetModel(TargetModel):
    """One rank of the tensor-parallel target (heads / FFN / vocabulary shards)."""

    def __init__(self, cfg: ModelConfig, tp: int, rank: int, w: TargetWeights, max_slots: int, max_rows: int,
                 dev) -> None:
        if not 0 <= rank < tp:
            raise ValueError("rank out of range")
        self.full_cfg, self.tp, self.rank = cfg, tp, rank
        super().__init__(local_config(cfg, tp), w, max_slots, max_rows, (), dev)
        self.keys = torch.zeros(max_rows, dtype=torch.int64, device=dev)
        self.y_ar = torch.zeros(max_rows, cfg.h, dtype=torch.bfloat16, device=dev)  # all-reduce payload

    def set_allreduce_dtype(self, dtype: torch.dtype) -> None:
        """bf16 (default) or fp32 payload of the row-parallel output all-reduce."""
        if dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("all-reduce dtype must be bf16 or fp32")
        self.y_ar = torch.zeros(self.y_ar.shape, dtype=dtype, device=self.dev)

    def _row_parallel_out(self, p: ops.PartialOut, n: int, norm_w: torch.Tensor):
        """Row-parallel output: dense y_r, SUM all-reduce (yielded), residual += sum, RMSNorm."""
        cfg = self.cfg
        y = self.y_ar[:n]
        ops.gemm_reduce_into(p, y)
        yield "sum", y
        ops.residual_dense(y, self.resid[:n], n, norm_w, cfg.eps, self.x[:n])

    def forward_steps(self, rows: int, state: torch.Tensor, mode: int, keys_after_c: int, anc=None,
                      mask_words: int = 0, head: str | None = "argmax", c_host: int = 0):
        """The verify forward of this shard; yields (op, tensor) at every collective."""
        cfg, w, kv = self.cfg, self.w, self.kv
        n, eps = rows, cfg.eps
        pt = kv.page_table
        x, resid = self.x[:n], self.resid[:n]
        ops.embed_rmsnorm(self.tokens, n, w.emb, w.layers[0].in_norm, eps, resid, x)
        for li, lw in enumerate(w.layers):
            ops.gemm_qkv_rope(x, lw.qkv, self.partial, cfg.n_q, cfg.n_kv, lw.q_norm, lw.k_norm, eps,
                              self.inv_freq, self.pos, self.slot, None, self.q, kv.buf, li * kv.layer_stride, pt,
                              PAGE, state)
            ops.attention(self.q[:n], self.attn[:n], kv.buf, cfg.L, kv.n_pages, li, pt, cfg.n_q, cfg.n_kv, n,
                          c_host, keys_after_c, kv.max_slots, state, mode, anc, mask_words, self.attn_ws,
                          n_splits=self.attn_splits)
            p = ops.gemm_partial(self.attn[:n], lw.o, out=self.partial)
            yield from self._row_parallel_out(p, n, lw.post_norm)
            p = ops.gemm_partial(x, lw.gate_up, out=self.partial)
            ops.swiglu(p, n, cfg.h_ffn, self.act[:n])
            p = ops.gemm_partial(self.act[:n], lw.down, out=self.partial)
            nxt = w.layers[li + 1].in_norm if li + 1 < cfg.L else w.final_norm
            yield from self._row_parallel_out(p, n, nxt)
        if head == "argmax":
            p = ops.gemm_partial(x, w.lm_head, out=self.partial)
            ops.gemm_argmax_keys(p, self.keys[:n], self.rank * cfg.V)
            yield "max", self.keys[:n]
            ops.argmax_from_keys(self.keys, n, self.argmax)

    def forward(self, rows: int, state: torch.Tensor, mode: int, keys_after_c: int, anc=None, mask_words: int = 0,
                head: str | None = "argmax", c_host: int = 0, pt=None, batch=None, collective=None) -> None:
        if pt is not None or batch is not None:
            raise ValueError("the tensor-parallel target serves one request per group")
        coll = collective or dist_collective
        for op, t in self.forward_steps(rows, state, mode, keys_after_c, anc, mask_words, head, c_host):
            coll(op, t)


def dist_collective(op: str, t: torch.Tensor) -> None:
    """NCCL all-reduce over the tensor-parallel group (the default process group)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return
    dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)


def run_lockstep(models: list[TPTargetModel], streams: list, *args, **kw) -> None:
    """Single-process simulation of a tp group: run every shard's forward_steps in lock
    step and reduce at each collective (SUM / MAX over the shard tensors), on one GPU."""
    gens = [m.forward_steps(*args, **kw) for m in models]
    while True:
        items = []
        for g, st in zip(gens, streams):
            with torch.cuda.stream(st):
                items.append(next(g, None))
        if all(it is None for it in items):
            return
        if any(it is None for it in items):
            raise RuntimeError("shards disagree on the collective sequence")
        for st in streams:
            st.synchronize()
        op = items[0][0]
        ts = [it[1] for it in items]
        acc = ts[0].clone()
        for t in ts[1:]:
            acc = acc + t if op == "sum" else torch.maximum(acc, t)
        for t in ts:
            t.copy_(acc)
        torch.cuda.synchronize()


def pack_argmax_key(value: float, global_index: int) -> int:
    """Host restatement of the shard key (bst_gemm_argmax_keys): order-preserving fp32
    bits in the high word, 0xFFFFFFFF - index in the low word, top bit flipped into the
    signed int64 order.  max() over shards' keys decodes to np.argmax of the full row."""
    import struct
    b = struct.unpack("<I", struct.pack("<f", value))[0]
    b = (~b & 0xFFFFFFFF) if b & 0x80000000 else (b | 0x80000000)
    u = (b << 32) | (0xFFFFFFFF - global_index)
    f = u ^ (1 << 63)  # uint64 with the top bit flipped, read as int64
    return f - (1 << 64) if f >> 63 else f


def unpack_argmax_key(key: int) -> int:
    return 0xFFFFFFFF - (key & 0xFFFFFFFF)


class TPVerifier:
    """Config 5 engine: one request per tensor-parallel group, tree verify + accept.

    Every rank runs the same replicated bookkeeping (K2 tree from the same lattice,
    verify rows, the K6 accept walk, KV compaction of its local heads, the committed
    stream); only the target forward is sharded.  The lattice is a fixed seeded one
    (config 5 measures verify + accept at fixed budgets, BASELINE.json configs[4])."""

    def __init__(self, cfg: ModelConfig, tp: int, rank: int, max_ctx: int, seed: int = 0,
                 weights: TargetWeights | None = None, n_cap: int = 255, gamma: int = 16, top_k: int = 8,
                 device=None) -> None:
        from ..draft_tree import DeviceTree
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dev, self.cfg, self.tp, self.rank = dev, cfg, tp, rank
        if not 1 <= n_cap <= TP_ROWS - 1:
            raise ValueError(f"TP engine n_cap must be in [1, {TP_ROWS - 1}], got {n_cap}")
        self.gamma, self.top_k, self.n_cap = gamma, top_k, n_cap
        self.max_ctx = max_ctx
        w = weights if weights is not None else random_shard(cfg, tp, rank, seed, dev)
        self.target = TPTargetModel(cfg, tp, rank, w, max_ctx + TP_ROWS + PAGE, TP_ROWS, dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self.state = torch.zeros(8, **i32)
        self.tree = DeviceTree(self.n_cap, dev)
        self.path = torch.zeros(gamma + 1, **i32)
        self.committed = torch.zeros(gamma + 1, **i32)
        self.acc_meta = torch.zeros(4, **i32)
        self.out_tokens = torch.zeros(max_ctx + TP_ROWS, **i32)
        self.stream = torch.cuda.Stream(dev)
        self.graphs: dict[int, torch.cuda.CUDAGraph] = {}
        self.n_nodes = 0

    def reset(self, prompt) -> None:
        """Prefill prompt[:-1] causally (chunks of TP_ROWS); prompt[-1] is the pending root."""
        from .forward import MODE_CAUSAL
        prompt = [int(t) for t in prompt]
        P = len(prompt)
        if not 1 <= P <= self.max_ctx:
            raise ValueError("prompt length must be in [1, max_ctx]")
        t = self.target
        with torch.cuda.stream(self.stream):
            for start in range(0, P - 1, TP_ROWS):
                n = min(TP_ROWS, P - 1 - start)
                self.state.copy_(torch.tensor([start, 0, prompt[-1], 0, 0, 0, 0, 0], dtype=torch.int32))
                t.tokens[:n].copy_(torch.tensor(prompt[start:start + n], dtype=torch.int32))
                ar = torch.arange(n, dtype=torch.int32, device=self.dev)
                t.pos[:n].copy_(ar)
                t.slot[:n].copy_(ar)
                t.forward(n, self.state, MODE_CAUSAL, keys_after_c=n, head=None, c_host=start)
            self.state.copy_(torch.tensor([P - 1, 0, prompt[-1], 0, 0, 0, 0, 0], dtype=torch.int32))
        self.stream.synchronize()

    def set_tree(self, n_nodes: int, seed: int = 0) -> int:
        """K2 (fixed budget, best-first) on a seeded lattice: the same tree on every rank."""
        import numpy as np

        from .. import _lib
        from ..draft_tree import expand_device
        rng = np.random.default_rng(seed)
        tok = np.stack([rng.choice(self.cfg.V, self.top_k, replace=False) for _ in range(self.gamma)]).astype(np.int32)
        raw = np.sort(rng.dirichlet(np.full(self.top_k, 0.6), self.gamma), axis=1)[:, ::-1] * 0.95
        plan = _lib.Plan(policy=_lib.POLICY_FIXED, n_max=int(n_nodes))
        with torch.cuda.stream(self.stream):
            expand_device(torch.from_numpy(tok).to(self.dev), torch.from_numpy(raw.copy()).to(self.dev), plan,
                          self.n_cap, out=self.tree)
        self.stream.synchronize()
        self.n_nodes = int(self.tree.meta[0].item())
        return self.n_nodes

    def _verify_body(self, rows: int) -> None:
        from ..verify_sim import accept_device
        from .forward import MODE_TREE
        t, tr, cfg = self.target, self.tree, self.target.cfg
        ops.verify_rows(self.state, tr.token, tr.depth, tr.meta, rows, t.tokens, t.pos, t.slot)
        t.forward(rows, self.state, MODE_TREE, keys_after_c=rows, anc=tr.anc_mask, mask_words=tr.mask_words,
                  head="argmax")
        accept_device(tr.token, tr.child_start, tr.child_list, t.argmax, self.gamma + 1, self.path, self.committed,
                      self.acc_meta)
        kv = t.kv
        ops.kv_compact(kv.buf, cfg.L, cfg.n_kv, PAGE, kv.layer_stride, kv.page_table, self.state, self.path,
                       self.acc_meta, self.gamma + 1)
        ops.commit_state(self.state, self.acc_meta, self.committed, self.gamma + 1, self.out_tokens)

    def step(self, graph: bool = True) -> None:
        """One verify + accept + compact + commit on the current tree (asynchronous)."""
        from .decode import BUCKET
        rows = min(TP_ROWS, ((self.n_nodes + 1 + BUCKET - 1) // BUCKET) * BUCKET)
        if not graph:
            with torch.cuda.stream(self.stream):
                self._verify_body(rows)
            return
        g = self.graphs.get(rows)
        if g is None:
            saved = self.state.clone()
            with torch.cuda.stream(self.stream):
                self._verify_body(rows)  # warm-up (attributes, tensor maps, communicators)
            self.stream.synchronize()
            self.state.copy_(saved)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self._verify_body(rows)
            self.stream.synchronize()
            self.state.copy_(saved)
            self.graphs[rows] = g
        with torch.cuda.stream(self.stream):
            g.replay()
