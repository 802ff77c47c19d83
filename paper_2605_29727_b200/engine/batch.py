"""BatchEngine — many independent decode streams on one GPU (BASELINE config 3).

SURVEY §8(e): requests share nothing, so a GPU batches its shard of
requests: their draft blocks and their trees are concatenated along the row
dimension of the K4 GEMMs (weights are streamed once per row chunk instead of
once per request) and K3 runs over every request of a chunk in one launch
(``bst_attention_batch``: per-request context length, page range and ancestor
mask).  Each request keeps its own device state, lattice, tree, accept walk, KV
compaction and committed stream — the per-request controllers stay independent.

Layout
  * one paged KV pool per model; request r owns pages [r*P, (r+1)*P) of the
    identity page table (P = pages per request);
  * verify rows: request r's tree occupies rows [r*S, r*S+S) of its chunk
    (S = N+1 for a fixed budget N; fixed-N trees always have N nodes here);
  * draft rows: a chunk's n*(gamma+1) block rows, then its n*(gamma+1) context rows.

A whole cycle (draft all chunks -> K1 -> K2 per request -> verify all chunks ->
accept/compact/gather/commit per request) is one CUDA graph with no host sync:
fixed budgets make every shape static.  Batching changes only how rows are
grouped into launches, so the token streams equal running each request alone
through ``B200Engine`` — bit for bit while every GEMM launch runs on the same K4
kernel; verify chunks above 256 rows run on the CTA-pair kernel, whose stream-K
split points differ, so there the fp32 sums agree to rounding and a stream can
differ only at a near-tie argmax (tests/test_gpu_batch.py).
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np
import torch

from .. import _lib, ops
from ..device import graph_kernel_nodes
from ..draft_tree import DeviceTree, expand_device_plan_batch, tree_structs_device
from ..lattice import topk_logits_into
from ..verify_sim import accept_device
from .config import QWEN3_8B, DrafterConfig, ModelConfig, default_feat_layers
from .decode import PREFILL_ROWS, ST_BONUS, ST_C, ST_COMMITTED, ST_CYCLE

MAX_ROWS = 256  # rows per request tree (fixed budgets <= 255) and per batched draft chunk
from .forward import _gemm_rows

# rows per batched verify launch (K4 CTA-pair kernel takes up to 512); BST_VERIFY_ROWS: measurement
VERIFY_ROWS = min(512, int(os.environ.get("BST_VERIFY_ROWS", "512")))
from .forward import MODE_CAUSAL, MODE_TREE, PAGE, DrafterModel, TargetModel, drafter_prefill
from .weights import DrafterWeights, TargetWeights


class BatchEngine:
    def __init__(self, cfg: ModelConfig = QWEN3_8B, dcfg: DrafterConfig | None = None, n_req: int = 8,
                 n_fixed: int = 64, max_ctx: int = 4096, seed: int = 0, top_k: int = 8, device=None,
                 max_cycles: int = 1024):
        if not torch.cuda.is_available():
            raise RuntimeError("BatchEngine needs a CUDA device; there is no CPU fallback")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        torch.cuda.set_device(dev)
        dcfg = dcfg or DrafterConfig()
        feat = dcfg.feat_layers or default_feat_layers(cfg.L)
        self.dcfg = DrafterConfig(layers=dcfg.layers, gamma=dcfg.gamma, feat_layers=feat, mask_token=dcfg.mask_token,
                                  logit_scale=dcfg.logit_scale)
        self.cfg, self.n_req, self.top_k = cfg, n_req, top_k
        self.gamma = self.dcfg.gamma
        self.N = n_fixed
        self.S = n_fixed + 1
        if self.S > MAX_ROWS:
            raise ValueError(f"fixed budget must be <= {MAX_ROWS - 1}")
        G1 = self.gamma + 1
        self.G1 = G1
        # verify chunks of up to 512 rows when every layer GEMM takes them (CTA-pair kernel):
        # the weights stream once per chunk, so wider chunks stream them fewer times
        layer_shapes = [(cfg.qkv_out, cfg.h), (cfg.h, cfg.h_q), (2 * cfg.h_ffn, cfg.h), (cfg.h, cfg.h_ffn)]
        vrows = VERIFY_ROWS if all(_gemm_rows(n_, k_, VERIFY_ROWS) == VERIFY_ROWS for n_, k_ in layer_shapes) \
            else MAX_ROWS
        self.chunk_v = max(1, vrows // self.S)             # requests per verify chunk
        # keep the chunk's batched attention grid (n_kv x row blocks x requests, one split)
        # to one wave of CTAs when that costs at most ~15% more weight passes
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        wave = max(1, n_sm // (cfg.n_kv * math.ceil(cfg.n_q // cfg.n_kv * self.S / 128)))
        if wave < self.chunk_v and math.ceil(n_req / wave) <= 1.15 * math.ceil(n_req / self.chunk_v):
            self.chunk_v = wave
        self.chunk_d = max(1, MAX_ROWS // G1)              # requests per draft chunk (block rows <= 256)
        self.max_ctx = max_ctx
        self.req_pages = math.ceil((max_ctx + MAX_ROWS + PAGE) / PAGE)
        slots = n_req * self.req_pages * PAGE
        self.tw = TargetWeights.random(cfg, seed, dev)
        self.dw = DrafterWeights.random(cfg, self.dcfg, len(feat), seed, dev)
        self.rows_cap = n_req * self.S  # ragged verify: every request's tree packed in one forward
        self.target = TargetModel(cfg, self.tw, slots, max(MAX_ROWS, self.chunk_v * self.S, self.rows_cap), feat, dev)
        self.drafter = DrafterModel(cfg, self.dcfg, self.dw, self.tw, slots, len(feat), dev, n_req_max=self.chunk_d)
        i32 = dict(dtype=torch.int32, device=dev)
        self.state = torch.zeros(n_req, 8, **i32)
        self.out_tokens = torch.zeros(n_req, max_ctx + MAX_ROWS, **i32)
        self.lat_tok = torch.zeros(n_req * G1, top_k, **i32)
        self.lat_prob = torch.zeros(n_req * G1, top_k, dtype=torch.float64, device=dev)
        self.trees = [DeviceTree(self.S - 1, dev) for _ in range(n_req)]
        self.mask_words = self.trees[0].mask_words
        self.anc = torch.zeros(n_req, self.S * self.mask_words, **i32)  # contiguous ancestor masks (batched K3)
        for r, tr in enumerate(self.trees):
            tr.anc_mask = self.anc[r]
        self.trees_dev = tree_structs_device(self.trees, dev)  # K2 writes every request's tree in one launch
        n_feat = len(feat) * cfg.h
        self.feat = torch.zeros(n_req * G1, n_feat, dtype=torch.bfloat16, device=dev)  # drafter context features
        self.path = torch.zeros(n_req, G1, **i32)
        self.committed = torch.zeros(n_req, G1, **i32)
        self.acc_meta = torch.zeros(n_req, 4, **i32)
        self.log_i32 = torch.zeros(n_req, max_cycles * 8, **i32)
        self.log_f64 = torch.zeros(n_req, max_cycles, dtype=torch.float64, device=dev)
        self.plan_dev = torch.zeros(n_req, C.sizeof(_lib.Plan), dtype=torch.uint8, device=dev)
        self.plan_base = torch.zeros_like(self.plan_dev)  # adaptive: per-request plans before the batch shift
        self.row_off = torch.zeros(n_req, **i32)
        self.row_cnt = torch.zeros(n_req, **i32)
        self.row_total = torch.zeros(1, **i32)
        self.row_req = torch.zeros(self.rows_cap, **i32)
        self.argmax_u = torch.zeros(n_req * self.S, **i32)  # per-request [S] argmax for the K6 walk
        self.total_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.graph_d = None
        self.graphs_v: dict[int, torch.cuda.CUDAGraph] = {}
        self.policy = _lib.POLICY_FIXED
        self.set_policy("fixed")
        self.stream = torch.cuda.Stream(dev)
        self.graph = None
        self.graph_kernels = 0
        self.graph_nodes: dict[int, int] = {}
        self.last_rows = 0
        self.use_graphs = True
        self._c_bound = 0
        torch.cuda.synchronize()

    def set_policy(self, kind: str, estimator=None, latencies=None) -> None:
        """Per-request K2 plans: fixed-N (N = n_fixed), or adaptive Algorithm 1 with N_max = n_fixed
        and a batch-aware verify cost (each request reads its own context from its state row).

        Adaptive (the reference controller is batch-1): the
        requests' trees are verified together in one ragged pass (rows packed, no padding),
        whose cost is the weights once plus every request's rows.  Before each cycle
        ``bst_batch_plan`` shifts request r's curve by the other requests' flops and bytes
        at their last tree sizes and scores S_hat with the batch's surrogate (a_offset), so
        each request's K2 is Algorithm 1 against the batch it is verified in — the best
        response for the batch's tokens per pass; with one request it is run_cycle exactly."""
        if kind == "fixed":
            plans = [_lib.Plan(policy=_lib.POLICY_FIXED, n_max=self.N) for _ in range(self.n_req)]
            self.policy = _lib.POLICY_FIXED
        elif kind == "adaptive":
            if estimator is None or latencies is None:
                raise ValueError("adaptive policy needs an estimator and cycle latencies")
            curve = estimator.curve(0).device_struct()
            p = estimator.params
            plans = [_lib.Plan(policy=_lib.POLICY_ADAPTIVE, n_max=self.N, curve=curve,
                               fixed_cost=latencies.t_draft + latencies.t_aux, l_ar=latencies.l_ar,
                               state=self.state[r].data_ptr(), c_idx=ST_C, d_flops_lin=4 * p.L * p.h_q,
                               d_bytes_const=p.bp * p.L * 2 * p.h_kv, d_bytes_lin=p.bp * p.L * 2 * p.n_q)
                     for r in range(self.n_req)]
            self.policy = _lib.POLICY_ADAPTIVE
        else:
            raise ValueError(f"unsupported batch policy {kind!r}")
        raw = b"".join(bytes(pl) for pl in plans)
        self.plan_dev.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8).view(self.n_req, -1))
        self.plan_base.copy_(self.plan_dev)
        if kind == "adaptive":
            with torch.cuda.stream(self.stream):
                ops.batch_plan(self.plan_base, self.plan_dev, self.trees_dev, self.state, self.n_req, first=True)
            self.stream.synchronize()
        self.graph = self.graph_d = None  # the policy is a launch parameter of K2
        self.graphs_v = {}

    def set_attention_splits(self, n: int) -> None:
        """Pin the K3 split count of both models (0 = automatic); parity tests use 1."""
        self.target.attn_splits = n
        self.drafter.attn_splits = n

    def _pt(self, r0: int) -> torch.Tensor:
        return self.target.kv.page_table[r0 * self.req_pages:]

    def _dpt(self, r0: int) -> torch.Tensor:
        return self.drafter.kv.page_table[r0 * self.req_pages:]

    # ------------------------------------------------------------------ setup
    def reset(self, prompts) -> None:
        """Prefill every request's prompt[:-1] into its page range; prompt[-1] becomes its pending root."""
        if len(prompts) != self.n_req:
            raise ValueError(f"need {self.n_req} prompts, got {len(prompts)}")
        t, d = self.target, self.drafter
        with torch.cuda.stream(self.stream):
            for r, prompt in enumerate(prompts):
                prompt = [int(x) for x in prompt]
                if not prompt or len(prompt) > self.max_ctx:
                    raise ValueError("prompt must hold 1..max_ctx tokens")
                P = len(prompt)
                st = self.state[r]
                for start in range(0, P - 1, PREFILL_ROWS):
                    n = min(PREFILL_ROWS, P - 1 - start)
                    st.copy_(torch.tensor([start, 0, prompt[-1], 0, 0, 0, 0, 0], dtype=torch.int32))
                    t.tokens[:n].copy_(torch.tensor(prompt[start:start + n], dtype=torch.int32))
                    ar = torch.arange(n, dtype=torch.int32, device=self.dev)
                    t.pos[:n].copy_(ar)
                    t.slot[:n].copy_(ar)
                    t.forward(n, st, MODE_CAUSAL, keys_after_c=n, head=None, c_host=start, pt=self._pt(r))
                    drafter_prefill(d, t.feat, n, st, start, pt=self._dpt(r))
                st.copy_(torch.tensor([P - 1, 0, prompt[-1], 0, 0, 0, 0, 0], dtype=torch.int32))
        self.stream.synchronize()
        self._c_bound = int(self.contexts().max())
        if self.policy == _lib.POLICY_ADAPTIVE:  # first plans against the new contexts
            with torch.cuda.stream(self.stream):
                ops.batch_plan(self.plan_base, self.plan_dev, self.trees_dev, self.state, self.n_req, first=True)
            self.stream.synchronize()

    # ------------------------------------------------------------------ cycle
    def _draft_phase(self) -> None:
        """Draft every request (chunks of chunk_d), K1 over all block rows, K2 per request."""
        G1, rp, n_req = self.G1, self.req_pages, self.n_req
        d = self.drafter
        for r0 in range(0, n_req, self.chunk_d):
            n = min(self.chunk_d, n_req - r0)
            logits = d.forward_batch(self.state[r0:r0 + n], n, self._dpt(r0), rp,
                                     feat=self.feat[r0 * G1:(r0 + n) * G1])
            topk_logits_into(logits, self.top_k, self.lat_tok[r0 * G1:(r0 + n) * G1],
                             self.lat_prob[r0 * G1:(r0 + n) * G1], None)
        # block row 0 of each request is the bonus position: request r's lattice is rows r*G1+1 ..
        expand_device_plan_batch(self.lat_tok[1:], self.lat_prob[1:], G1 * self.top_k, self.gamma, self.plan_dev,
                                 self.policy, self.N, self.trees, self.trees_dev)

    def _accept_commit(self, r: int, argmax: torch.Tensor, feat_rows: torch.Tensor, row_base=None) -> None:
        """K6 walk, KV compaction, drafter feature gather and state update of request r."""
        t, tr, G1 = self.target, self.trees[r], self.G1
        accept_device(tr.token, tr.child_start, tr.child_list, argmax, G1, self.path[r], self.committed[r],
                      self.acc_meta[r])
        kv = t.kv
        ops.kv_compact(kv.buf, self.cfg.L, self.cfg.n_kv, PAGE, kv.layer_stride, self._pt(r), self.state[r],
                       self.path[r], self.acc_meta[r], G1)
        ops.gather_rows(feat_rows, self.path[r], self.acc_meta[r], G1, self.feat[r * G1:(r + 1) * G1], row_base)
        ops.commit_state(self.state[r], self.acc_meta[r], self.committed[r], G1, self.out_tokens[r], tr.meta,
                         tr.surrogate, self.log_i32[r], self.log_f64[r])

    def _cycle_body(self) -> None:
        """Fixed budget: one static-shape cycle (every tree has N nodes)."""
        S, rp, n_req = self.S, self.req_pages, self.n_req
        t = self.target
        self._draft_phase()
        # phase 2: verify every request (chunks of chunk_v), then accept / compact / gather / commit
        for r0 in range(0, n_req, self.chunk_v):
            n = min(self.chunk_v, n_req - r0)
            for i in range(n):
                tr = self.trees[r0 + i]
                ops.verify_rows(self.state[r0 + i], tr.token, tr.depth, tr.meta, S, t.tokens[i * S:],
                                t.pos[i * S:], t.slot[i * S:])
            t.forward(n * S, self.state[r0:r0 + n], MODE_TREE, keys_after_c=S, anc=self.anc[r0:r0 + n],
                      mask_words=self.mask_words, head="argmax", pt=self._pt(r0), batch=(n, S, rp))
            for i in range(n):
                self._accept_commit(r0 + i, t.argmax[i * S:(i + 1) * S], t.feat[i * S:(i + 1) * S])

    # ------------------------------------------------ adaptive: ragged verify
    def _draft_ragged(self) -> None:
        """Draft + K2 (batch-aware plans), then the packed verify row layout of this cycle."""
        t = self.target
        self._draft_phase()
        ops.ragged_rows(self.trees_dev, self.state, self.n_req, self.S, self.rows_cap, self.row_off, self.row_cnt,
                        self.row_total, t.tokens, t.pos, t.slot, self.row_req)

    def _verify_ragged(self, rows: int) -> None:
        """One target pass over the packed trees of every request (rows = the 64-row bucket of
        the total), per-request accept / compaction / commit, next cycle's batch-aware plans."""
        t, S, n = self.target, self.S, self.n_req
        t.forward(rows, self.state, MODE_TREE, keys_after_c=S, anc=self.anc, mask_words=self.mask_words,
                  head="argmax", pt=self._pt(0),
                  ragged=(n, S, self.req_pages, self.row_req, self.row_off, self.row_cnt))
        ops.ragged_unpack(t.argmax, self.row_off, self.row_cnt, n, S, self.argmax_u)
        for r in range(n):
            self._accept_commit(r, self.argmax_u[r * S:(r + 1) * S], t.feat, self.row_off[r:r + 1])
        ops.batch_plan(self.plan_base, self.plan_dev, self.trees_dev, self.state, n, first=False)

    def _cycle_adaptive(self) -> int:
        """Graph D (draft + K2 + row layout) -> one host read of the packed row total ->
        graph V of its 64-row bucket.  Returns the total verified rows."""
        st = self.stream
        if not self.use_graphs:
            with torch.cuda.stream(st):
                self._draft_ragged()
        else:
            if self.graph_d is None:
                self.graph_d = self._capture_fn(self._draft_ragged)
            with torch.cuda.stream(st):
                self.graph_d.replay()
        with torch.cuda.stream(st):
            self.total_host.copy_(self.row_total, non_blocking=True)
        st.synchronize()
        total = int(self.total_host[0])
        rows = min(self.rows_cap, -(-total // 64) * 64)
        if not self.use_graphs:
            with torch.cuda.stream(st):
                self._verify_ragged(rows)
            return total
        g = self.graphs_v.get(rows)
        if g is None:
            g = self.graphs_v[rows] = self._capture_fn(lambda: self._verify_ragged(rows))
        with torch.cuda.stream(st):
            g.replay()
        return total

    def precapture(self, max_rows: int | None = None) -> int:
        """Adaptive policy: capture the verify graph of every 64-row bucket up to max_rows
        (default rows_cap) and the draft graph now, so no capture lands inside a timed
        loop.  The decode state is restored by each capture.  Returns the graph count."""
        if self.policy != _lib.POLICY_ADAPTIVE or not self.use_graphs:
            return 0
        top = min(self.rows_cap, max_rows or self.rows_cap)
        if self.graph_d is None:
            self.graph_d = self._capture_fn(self._draft_ragged)
        for rows in range(64, -(-top // 64) * 64 + 1, 64):
            rows = min(rows, self.rows_cap)
            if rows not in self.graphs_v:
                self.graphs_v[rows] = self._capture_fn(lambda r=rows: self._verify_ragged(r))
        return len(self.graphs_v)

    def _capture(self) -> torch.cuda.CUDAGraph:
        g = self._capture_fn(self._cycle_body)
        self.graph_kernels = self.graph_nodes[id(g)]
        return g

    def _capture_fn(self, fn) -> torch.cuda.CUDAGraph:
        # warm-up run outside the graph (workspaces, tensor maps, kernel attributes), then
        # capture; every mutable decode buffer is restored so the capture changes nothing
        keep = [self.state, self.plan_dev, self.out_tokens, self.log_i32, self.log_f64, self.feat]
        saved = [x.clone() for x in keep]
        with torch.cuda.stream(self.stream):
            fn()
        self.stream.synchronize()
        for x, y in zip(keep, saved):
            x.copy_(y)
        g = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.graph(g, stream=self.stream):
            fn()
        self.graph_nodes[id(g)] = graph_kernel_nodes(g)
        g.instantiate()
        self.stream.synchronize()
        for x, y in zip(keep, saved):
            x.copy_(y)
        torch.cuda.synchronize()
        return g

    def cycle(self) -> None:
        """One draft -> expand -> verify -> accept cycle for every request (asynchronous).

        A host-side bound on every request's context (each cycle commits at most gamma+1
        tokens) keeps the verify rows inside each request's page range: a request never
        writes KV into the next request's pages; raises when the bound is hit."""
        if self._c_bound + self.S > self.req_pages * PAGE or self._c_bound + self.S > self.max_ctx + MAX_ROWS:
            self._c_bound = int(self.contexts().max())  # tighten with the true contexts (one sync)
            if self._c_bound + self.S > self.max_ctx + MAX_ROWS:
                raise RuntimeError(f"KV cache full: a request's context {self._c_bound} + {self.S} verify rows "
                                   f"exceeds max_ctx={self.max_ctx}")
        self._c_bound += self.G1
        if self.policy == _lib.POLICY_ADAPTIVE:
            self.last_rows = self._cycle_adaptive()
            return
        if not self.use_graphs:
            with torch.cuda.stream(self.stream):
                self._cycle_body()
            return
        if self.graph is None:
            self.graph = self._capture()
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def committed_counts(self) -> np.ndarray:
        self.stream.synchronize()
        return self.state[:, ST_COMMITTED].cpu().numpy()

    def run(self, max_new_tokens: int, check_every: int = 8) -> np.ndarray:
        """Cycle until every request has committed >= max_new_tokens tokens; returns the counts."""
        while True:
            for _ in range(check_every):
                self.cycle()
            counts = self.committed_counts()
            if counts.min() >= max_new_tokens:
                return counts

    def tokens(self, r: int) -> list[int]:
        self.stream.synchronize()
        n = int(self.state[r, ST_COMMITTED].item())
        return self.out_tokens[r, :n].cpu().tolist()

    def contexts(self) -> np.ndarray:
        self.stream.synchronize()
        return self.state[:, ST_C].cpu().numpy()

    def cycles(self) -> np.ndarray:
        self.stream.synchronize()
        return self.state[:, ST_CYCLE].cpu().numpy()

    def roots(self) -> np.ndarray:
        self.stream.synchronize()
        return self.state[:, ST_BONUS].cpu().numpy()
