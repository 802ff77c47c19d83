"""B200Engine — the on-device draft -> expand -> verify -> accept loop.

One decode cycle (the reference's ``decode_full`` body, verify_sim.py:437-460):

  [graph D]  drafter forward (K3/K4/K5) -> K1 top-K lattice -> K2 expand
             (adaptive Algorithm 1 with the latency curve at the device-side
             context c, or fixed-N best-first)
  [host]     read the tree size N* (the only host sync of the cycle)
  [graph V_b] verify rows -> target forward on s = N*+1 rows padded to the
             bucket b (K4/K5/K3 with the ancestor bitmask) -> LM-head argmax
             -> K6 accept walk -> KV compaction -> drafter feature gather ->
             state update (c += accepted_len, pending bonus) + per-cycle log

Both graphs read every per-cycle scalar from the device ``state`` vector, so
they are captured once (V per 16-row bucket) and replayed.  CUDA events
around the two graphs give T_draft/T_verify; the verify time feeds the
estimator's online EMA (``VerifyLatencyEstimator.observe``, K7).

The engine also implements the reference plugin protocol
(``drafter_marginals`` / ``next_token`` / ``tree_argmax``) and the decode fast
path (``engine_decode``) the façade's ``decode`` dispatches to.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from .. import _lib, ops
from ..controller import STOP_BUDGET_CAP
from ..cost_model import CycleLatencies, VerifyLatencyEstimator
from ..device import graph_kernel_nodes
from ..draft_tree import DeviceTree, expand_device_plan
from ..lattice import MarginalBlock, topk_logits_into, topk_partial_into
from .config import QWEN3_8B, DrafterConfig, ModelConfig, default_feat_layers
from .forward import _ABLATE, MODE_CAUSAL, MODE_TREE, PAGE, DrafterModel, TargetModel, drafter_prefill
from .weights import DrafterWeights, TargetWeights

ST_C, ST_NNEW, ST_BONUS, ST_COMMITTED, ST_CYCLE = 0, 1, 2, 3, 4
MAX_TREE = 1024      # reference default n_max (sp/harness.py:62, fixed grid up to 1024 at :49)
BUCKET = 16          # verify rows are padded to 16-row buckets up to 256 rows ...
WIDE_BUCKET = 64     # ... and to 64-row buckets above (one captured verify graph per bucket)
MAX_ROWS = 1088      # verify rows of the largest tree (1025) rounded up to its bucket
PREFILL_ROWS = 512   # causal prefill chunk (one CTA-pair GEMM launch per weight: the weights stream once per 512 rows)


@dataclass
class CycleStats:
    tree_size: int
    n_expanded: int
    stop: int
    accepted_len: int
    context: int
    bonus: int
    surrogate: float
    t_draft: float
    t_verify: float


class B200Engine:
    """Qwen3-shape target + DFlash-style drafter, random-init bf16, one request per engine."""

    def __init__(self, cfg: ModelConfig = QWEN3_8B, dcfg: DrafterConfig | None = None, max_ctx: int = 4096,
                 seed: int = 0, n_cap: int = MAX_TREE, top_k: int = 8, device=None, max_cycles: int = 4096):
        if not torch.cuda.is_available():
            raise RuntimeError("B200Engine needs a CUDA device; there is no CPU fallback")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        torch.cuda.set_device(self.dev)
        self.cfg = cfg
        dcfg = dcfg or DrafterConfig()
        feat = dcfg.feat_layers or default_feat_layers(cfg.L)
        self.dcfg = DrafterConfig(layers=dcfg.layers, gamma=dcfg.gamma, feat_layers=feat, mask_token=dcfg.mask_token,
                                  logit_scale=dcfg.logit_scale)
        self.gamma, self.top_k = self.dcfg.gamma, top_k
        if not 1 <= n_cap <= MAX_TREE:
            raise ValueError(f"n_cap must be in [1, {MAX_TREE}], got {n_cap}")
        self.n_cap = n_cap
        self.max_rows = self._bucket(n_cap)
        self.max_ctx = max_ctx
        slots = max_ctx + self.max_rows + PAGE
        self.tw = TargetWeights.random(cfg, seed, self.dev)
        self.dw = DrafterWeights.random(cfg, self.dcfg, len(feat), seed, self.dev)
        self.target = TargetModel(cfg, self.tw, slots, max(self.max_rows, PREFILL_ROWS), feat, self.dev)
        self.drafter = DrafterModel(cfg, self.dcfg, self.dw, self.tw, slots, len(feat), self.dev)
        i32 = dict(dtype=torch.int32, device=self.dev)
        self.state = torch.zeros(8, **i32)
        self.out_tokens = torch.zeros(max_ctx + self.max_rows, **i32)
        self.lat_tok = torch.zeros(self.gamma, top_k, **i32)
        self.lat_prob = torch.zeros(self.gamma, top_k, dtype=torch.float64, device=self.dev)
        self.probs_full = None  # fp64 [gamma, V] when export is on
        self.tree = DeviceTree(self.n_cap, self.dev)
        self.path = torch.zeros(self.gamma + 1, **i32)
        self.committed = torch.zeros(self.gamma + 1, **i32)
        self.acc_meta = torch.zeros(4, **i32)
        self.log_i32 = torch.zeros(max_cycles * 8, **i32)
        self.log_f64 = torch.zeros(max_cycles, dtype=torch.float64, device=self.dev)
        self.plan_dev = torch.zeros(C.sizeof(_lib.Plan), dtype=torch.uint8, device=self.dev)
        self.plan_host = torch.zeros(C.sizeof(_lib.Plan), dtype=torch.uint8).pin_memory()
        self.meta_host = torch.zeros(16, dtype=torch.int32).pin_memory()
        self.stream = torch.cuda.Stream(self.dev)
        self.graph_d = None
        self.graphs_d: dict[tuple, torch.cuda.CUDAGraph] = {}
        self.graphs_v: dict[int, torch.cuda.CUDAGraph] = {}
        self.graph_ar = None
        self.policy = (_lib.POLICY_FIXED, 64)
        self.prompt_len = 0
        self.use_graphs = True
        self.export = False  # debug: keep fp64 drafter rows + verify argmax per cycle (parity tests)
        self.exported: list[dict] = []
        self.draft_override = None
        self.graph_kernels: dict[int, int] = {}
        torch.cuda.synchronize()

    # ------------------------------------------------------------------ setup
    def reset(self, prompt) -> None:
        """Prefill prompt[:-1] (causal, chunks of 256) and make prompt[-1] the pending root."""
        prompt = [int(t) for t in prompt]
        if not prompt:
            raise ValueError("prompt must contain at least one token")
        P = len(prompt)
        if P > self.max_ctx:
            raise ValueError("prompt longer than max_ctx")
        self.prompt_len = P
        with torch.cuda.stream(self.stream):
            t, d = self.target, self.drafter
            for start in range(0, P - 1, PREFILL_ROWS):
                n = min(PREFILL_ROWS, P - 1 - start)
                self.state.copy_(torch.tensor([start, 0, prompt[-1], 0, 0, 0, 0, 0], dtype=torch.int32))
                t.tokens[:n].copy_(torch.tensor(prompt[start:start + n], dtype=torch.int32))
                ar = torch.arange(n, dtype=torch.int32, device=self.dev)
                t.pos[:n].copy_(ar)
                t.slot[:n].copy_(ar)
                t.forward(n, self.state, MODE_CAUSAL, keys_after_c=n, head=None, c_host=start)
                drafter_prefill(d, t.feat, n, self.state, start)
            self.state.copy_(torch.tensor([P - 1, 0, prompt[-1], 0, 0, 0, 0, 0], dtype=torch.int32))
        self.stream.synchronize()
        self.exported = []
        self._pending = None
        self._c_host = P - 1

    def set_policy(self, kind: str, n: int = 0, estimator: VerifyLatencyEstimator | None = None,
                   latencies: CycleLatencies | None = None, n_max: int | None = None) -> None:
        """Adaptive (Algorithm 1 on the device) or fixed-N best-first."""
        cfg = self.cfg
        if kind == "fixed":
            if not 1 <= n <= self.n_cap:
                raise ValueError(f"fixed budget must be in [1, {self.n_cap}]")
            self.policy = (_lib.POLICY_FIXED, n)
            plan = _lib.Plan(policy=_lib.POLICY_FIXED, n_max=n)
        elif kind == "adaptive":
            if estimator is None or latencies is None:
                raise ValueError("adaptive policy needs an estimator and cycle latencies")
            n_max = self.n_cap if n_max is None else int(n_max)
            if not 1 <= n_max <= self.n_cap:
                # never clamp: a smaller budget cap changes trees and stop reasons
                raise ValueError(f"n_max {n_max} outside [1, {self.n_cap}] (engine n_cap; build with n_cap >= n_max)")
            curve = estimator.curve(0).device_struct()
            p = estimator.params
            plan = _lib.Plan(policy=_lib.POLICY_ADAPTIVE, n_max=n_max, curve=curve,
                             fixed_cost=latencies.t_draft + latencies.t_aux, l_ar=latencies.l_ar,
                             state=self.state.data_ptr(), c_idx=ST_C, d_flops_lin=4 * p.L * p.h_q,
                             d_bytes_const=p.bp * p.L * 2 * p.h_kv, d_bytes_lin=p.bp * p.L * 2 * p.n_q)
            self.policy = (_lib.POLICY_ADAPTIVE, n_max)
        else:
            raise ValueError(f"unsupported engine policy {kind!r} (beam/greedy run through the façade)")
        raw = bytes(plan)
        self.plan_host.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
        with torch.cuda.stream(self.stream):
            self.plan_dev.copy_(self.plan_host, non_blocking=True)
        self.graph_d = self.graphs_d.get(self.policy)  # policy/n_max are launch parameters of K2

    def refresh_plan(self, estimator: VerifyLatencyEstimator, latencies: CycleLatencies) -> None:
        """Re-upload the adaptive plan (e.g. after an EMA update) — one small H2D copy, no recapture."""
        self.set_policy("adaptive", estimator=estimator, latencies=latencies, n_max=self.policy[1])

    # --------------------------------------------------------------- phases
    def _draft_body(self) -> None:
        if self.draft_override is not None:  # test hook: externally supplied drafter logits [gamma, V]
            logits = self.draft_override(self)
        elif self.probs_full is None:  # hot path: K1 reads the LM head's partial slots (no reduce pass)
            p = self.drafter.forward(self.state, reduce=False)
            if "k1" not in _ABLATE:
                topk_partial_into(p, self.gamma, self.top_k, self.lat_tok, self.lat_prob)
            logits = None
        else:
            logits = self.drafter.forward(self.state)
        if logits is not None and "k1" not in _ABLATE:
            topk_logits_into(logits, self.top_k, self.lat_tok, self.lat_prob, self.probs_full)
        if "k2" not in _ABLATE:
            expand_device_plan(self.lat_tok, self.lat_prob, self.plan_dev, self.policy[0], self.policy[1], self.tree)

    def _head(self) -> str:
        return "sample" if self.target.temperature > 0.0 else "argmax"

    def _verify_forward(self, rows: int) -> None:
        t, tr = self.target, self.tree
        ops.verify_rows(self.state, tr.token, tr.depth, tr.meta, rows, t.tokens, t.pos, t.slot)
        t.forward(rows, self.state, MODE_TREE, keys_after_c=rows, anc=tr.anc_mask, mask_words=tr.mask_words,
                  head=self._head())

    def _verify_body(self, rows: int) -> None:
        self._verify_forward(rows)
        from ..verify_sim import accept_device
        t, tr = self.target, self.tree
        accept_device(tr.token, tr.child_start, tr.child_list, t.argmax, self.gamma + 1, self.path, self.committed,
                      self.acc_meta)
        self._commit_tail()

    def _commit_tail(self) -> None:
        """KV compaction of the accepted path, drafter feature gather, state update."""
        t, d, tr = self.target, self.drafter, self.tree
        kv = t.kv
        ops.kv_compact(kv.buf, self.cfg.L, self.cfg.n_kv, PAGE, kv.layer_stride, kv.page_table, self.state, self.path,
                       self.acc_meta, self.gamma + 1)
        ops.gather_rows(t.feat, self.path, self.acc_meta, d.CR, d.feat_in)
        ops.commit_state(self.state, self.acc_meta, self.committed, self.gamma + 1, self.out_tokens, tr.meta,
                         tr.surrogate, self.log_i32, self.log_f64)

    def _bucket(self, n_nodes: int) -> int:
        """Verify rows of an n-node tree: padded to its row bucket, never past the engine's
        n_cap + 1 rows (the ancestor mask and tree buffers hold n_cap + 1 rows)."""
        rows = n_nodes + 1
        b = BUCKET if rows <= 256 else WIDE_BUCKET
        return min(((rows + b - 1) // b) * b, self.n_cap + 1)

    def _capture(self, fn) -> torch.cuda.CUDAGraph:
        # warm-up run outside the graph (kernel attributes, tensor maps, workspaces), then capture
        saved = self.state.clone()
        with torch.cuda.stream(self.stream):
            fn()
        self.stream.synchronize()
        self.state.copy_(saved)
        g = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.graph(g, stream=self.stream):
            fn()
        self.graph_kernels[id(g)] = graph_kernel_nodes(g)  # exact launches per replay
        g.instantiate()
        self.stream.synchronize()
        self.state.copy_(saved)
        torch.cuda.synchronize()
        return g

    def _run_draft(self) -> None:
        if not self.use_graphs or self.export or self.draft_override is not None:
            with torch.cuda.stream(self.stream):
                self._draft_body()
            return
        if self.graph_d is None:
            self.graph_d = self.graphs_d[self.policy] = self._capture(self._draft_body)
        with torch.cuda.stream(self.stream):
            self.graph_d.replay()

    def precapture(self, max_rows: int | None = None) -> int:
        """Capture the verify graph of every row bucket up to ``max_rows`` (default: the
        engine's capacity) now, so no capture lands inside a timed decode loop (a bucket
        first seen mid-run otherwise pays its eager warm-up run + capture + instantiate in
        that cycle).  KV slots at and beyond c written by the warm-up runs are overwritten
        by the next real verify; the decode state is restored.  Returns the graph count."""
        if not self.use_graphs:
            return 0
        top = self.max_rows if max_rows is None else min(self._bucket(max_rows - 1), self.max_rows)
        self._check_room(self._c_host, top)
        for n in range(self.n_cap + 1):
            b = self._bucket(n)
            if b > top:
                break
            if b not in self.graphs_v:
                self.graphs_v[b] = self._capture(lambda rows=b: self._verify_body(rows))
        return len(self.graphs_v)

    def _run_verify(self, rows: int) -> None:
        if not self.use_graphs or self.export:
            with torch.cuda.stream(self.stream):
                self._verify_body(rows)
            return
        g = self.graphs_v.get(rows)
        if g is None:
            g = self.graphs_v[rows] = self._capture(lambda: self._verify_body(rows))
        with torch.cuda.stream(self.stream):
            g.replay()

    # --------------------------------------------------------------- decode
    def draft(self, events=None) -> tuple[int, int]:
        """Phase 1 (graph D) + the cycle's single host sync.

        Returns (tree size N*, tokens committed before this cycle)."""
        st = self.stream
        if events:
            events[0].record(st)
        if self.export:
            self.probs_full = torch.empty(self.gamma, self.cfg.V, dtype=torch.float64, device=self.dev)
        self._run_draft()
        if events:
            events[1].record(st)
        with torch.cuda.stream(st):
            self.meta_host[:8].copy_(self.tree.meta, non_blocking=True)
            self.meta_host[8:].copy_(self.state, non_blocking=True)
        st.synchronize()
        self._c_host = int(self.meta_host[8 + ST_C])
        return int(self.meta_host[0]), int(self.meta_host[8 + ST_COMMITTED])

    def _check_room(self, c: int, rows: int) -> None:
        """The verify rows' KV slots c .. c+rows-1 must lie inside this engine's page range
        (the K5 KV store does not bound-check)."""
        if c + rows > self.target.kv.max_slots or c + rows > self.drafter.kv.max_slots:
            raise RuntimeError(f"KV cache full: context {c} + {rows} verify rows exceeds max_ctx={self.max_ctx}")

    def verify(self, n_nodes: int, events=None) -> None:
        """Phase 2 (graph V_bucket): verify, accept, compact, commit — asynchronous."""
        self._check_room(self._c_host, self._bucket(n_nodes))
        if self.export:
            self._export_pre(n_nodes)
        self._run_verify(self._bucket(n_nodes))
        if events:
            events[2].record(self.stream)
        if self.export:
            self._export_post(n_nodes)

    def cycle(self, events=None) -> int:
        """One draft->expand->verify->accept cycle; returns the tree size N*."""
        n_nodes, _ = self.draft(events)
        self.verify(n_nodes, events)
        return n_nodes

    def _export_pre(self, n: int) -> None:
        tr = self.tree
        self.exported.append(dict(
            probs=self.probs_full.cpu().numpy(), tok=self.lat_tok.cpu().numpy(), prob=self.lat_prob.cpu().numpy(),
            parent=tr.parent[: n + 1].cpu().numpy(), depth=tr.depth[: n + 1].cpu().numpy(),
            token=tr.token[: n + 1].cpu().numpy(), rho=tr.rho[: n + 1].cpu().numpy(),
            meta=tr.meta.cpu().numpy(), trace=tr.trace[: int(tr.meta[1].item())].cpu().numpy(),
            surrogate=float(tr.surrogate.item()), c=int(self.state[ST_C].item())))

    def _export_post(self, n: int) -> None:
        self.stream.synchronize()
        e = self.exported[-1]
        e["argmax"] = self.target.argmax[: n + 1].cpu().numpy()
        e["path"] = self.path[: int(self.acc_meta[0].item())].cpu().numpy()
        e["bonus"] = int(self.acc_meta[1].item())

    def run(self, max_new_tokens: int, timing: bool = True) -> tuple[list[CycleStats], list[int]]:
        """Decode until >= max_new_tokens tokens are committed (the reference loop condition)."""
        stats_t: list = []
        while True:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if timing else None
            n_nodes, committed = self.draft(ev)  # committed count is read at the cycle's one sync
            if committed >= max_new_tokens:
                break  # the speculative draft of a cycle that will not run is discarded
            self.verify(n_nodes, ev)
            stats_t.append(ev)
        self.stream.synchronize()
        return self.read_log(stats_t), self.tokens()

    def read_log(self, events=None) -> list[CycleStats]:
        self.stream.synchronize()
        ncyc = int(self.state[ST_CYCLE].item())
        li = self.log_i32[: ncyc * 8].view(ncyc, 8).cpu().numpy()
        lf = self.log_f64[:ncyc].cpu().numpy()
        out = []
        for i in range(ncyc):
            td = tv = float("nan")
            if events and i < len(events) and events[i]:
                e = events[i]
                td = e[0].elapsed_time(e[1]) * 1e-3
                tv = e[1].elapsed_time(e[2]) * 1e-3
            out.append(CycleStats(int(li[i, 0]), int(li[i, 1]), int(li[i, 2]), int(li[i, 3]), int(li[i, 4]),
                                  int(li[i, 5]), float(lf[i]), td, tv))
        return out

    def tokens(self) -> list[int]:
        self.stream.synchronize()  # the last verify graph runs asynchronously on the engine stream
        n = int(self.state[ST_COMMITTED].item())
        return self.out_tokens[:n].cpu().tolist()

    # ------------------------------------------------------- AR reference
    def ar_step_body(self) -> None:
        """One autoregressive target step on the pending root (s = 1)."""
        t = self.target
        t.tokens[:1].copy_(self.state[ST_BONUS:ST_BONUS + 1])
        t.pos[:1].zero_()
        t.slot[:1].zero_()
        t.forward(1, self.state, MODE_CAUSAL, keys_after_c=1, head=self._head())
        # commit: c += 1, root <- argmax (or the T > 0 sample)
        self.state[ST_C:ST_C + 1].add_(1)
        self.state[ST_BONUS:ST_BONUS + 1].copy_(t.argmax[:1])

    def ar_decode(self, n_tokens: int) -> list[int]:
        self._check_room(int(self.state[ST_C].item()), n_tokens)
        out = []
        with torch.cuda.stream(self.stream):
            for _ in range(n_tokens):
                self.ar_step_body()
                out.append(self.target.argmax[:1].clone())
        self.stream.synchronize()
        return [int(x.item()) for x in out]

    def measure_ar_step(self, iters: int = 10) -> float:
        """CUDA-event latency of one AR target step (the l_ar of Algorithm 1)."""
        saved = self.state.clone()
        if self.graph_ar is None:
            self.graph_ar = self._capture(self.ar_step_body)
        ts = []
        for _ in range(iters + 3):
            self.state.copy_(saved)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            with torch.cuda.stream(self.stream):
                self.graph_ar.replay()
            b.record(self.stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        self.state.copy_(saved)
        torch.cuda.synchronize()
        return float(np.median(ts[3:]))

    # --------------------------------------------------- plugin protocol
    def engine_decode(self, sim_cfg, policy, estimator: VerifyLatencyEstimator):
        """Fast path of the façade's ``decode`` (verify_sim.py:464): the loop runs on the device.

        The context of every cycle is the engine's KV length c (= prompt_len - 1 +
        committed), the reference's ``context_len + len(prefix)`` under the
        alignment contract (SURVEY §8a′); the SimConfig's latencies drive
        Algorithm 1.  Every measured verify time is fed to ``estimator.observe``
        (K7, §5.2); EMA variants re-plan the next cycle from the updated bias.
        """
        from ..verify_sim import CycleRecord
        lat = sim_cfg.controller.latencies
        adaptive = policy.kind == "adaptive"
        if adaptive:
            self.set_policy("adaptive", estimator=estimator, latencies=lat, n_max=sim_cfg.controller.n_max)
        elif policy.kind == "fixed":
            self.set_policy("fixed", n=policy.n)
        else:
            raise ValueError("engine fast path supports adaptive and fixed-N policies")
        if sim_cfg.top_k != self.top_k:
            raise ValueError(f"engine was built with top_k={self.top_k}")
        ema = estimator.variant in ("ema", "ema_calib")
        self.set_temperature(sim_cfg.temperature, self.target.sample_seed)
        self._sync(self.tokens())
        events: list = []
        pending = None  # (index, s, events) of the previous cycle, observed at this cycle's sync
        cyc0 = int(self.state[ST_CYCLE].item())
        while True:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            n_nodes, committed = self.draft(ev)
            if pending is not None:
                s, c, pev = pending
                estimator.observe(s, c, pev[1].elapsed_time(pev[2]) * 1e-3)
                if ema and adaptive:
                    self.refresh_plan(estimator, lat)
            if committed >= sim_cfg.run_length:
                break
            c = int(self.meta_host[8 + ST_C])
            self.verify(n_nodes, ev)
            events.append(ev)
            pending = (n_nodes + 1, c, ev)
        if pending is not None and ema:
            self.stream.synchronize()
        stats = self.read_log(events=[None] * cyc0 + events)[cyc0:]
        records = []
        for st in stats:
            t_verify = estimator.estimate_for_budget(st.tree_size, st.context)
            cyc = lat.t_draft + t_verify + lat.t_aux
            records.append(CycleRecord(tree_size=st.tree_size, accepted_len=st.accepted_len, surrogate=st.surrogate,
                                       t_draft=lat.t_draft, t_verify=t_verify, t_aux=lat.t_aux, l_ar=lat.l_ar,
                                       cycle_speedup=st.accepted_len * lat.l_ar / cyc))
        return records, tuple(self.tokens())

    def drafter_marginals(self, prefix) -> MarginalBlock:
        """fp64 drafter rows for the engine's current state (prefix must be its committed stream,
        possibly extended by the acceptance of the last verified tree / the last next_token)."""
        self._sync(prefix)
        self.probs_full = torch.empty(self.gamma, self.cfg.V, dtype=torch.float64, device=self.dev)
        with torch.cuda.stream(self.stream):
            logits = self.drafter.forward(self.state)
            topk_logits_into(logits, self.top_k, self.lat_tok, self.lat_prob, self.probs_full)
        self.stream.synchronize()
        return MarginalBlock(gamma=self.gamma, vocab_size=self.cfg.V, probs=self.probs_full.cpu().numpy())

    def _check_prefix(self, prefix) -> None:
        if tuple(prefix) != tuple(self.tokens()):
            raise ValueError("engine plugin: prefix does not match the engine's committed stream")

    # ----------------------------- reference plugin protocol, general façade loop
    def set_temperature(self, temperature: float, seed: int = 0) -> None:
        """Verify / AR head: T = 0 greedy argmax (np.argmax tie-break), T > 0 Gumbel-max samples
        keyed by (seed, absolute position) (bst_gemm_sample), so a tree decode reproduces the
        sampled AR decode token for token (exact-match sampled verification,
        verify_sim.py:111-126).  Changing it drops the captured verify / AR graphs."""
        if temperature < 0.0:
            raise ValueError("temperature must be >= 0")
        t = self.target
        if (float(temperature), int(seed)) != (t.temperature, t.sample_seed):
            t.temperature, t.sample_seed = float(temperature), int(seed)
            self.graphs_v.clear()
            self.graph_ar = None

    def _sync(self, prefix) -> None:
        """Bring the device state to ``prefix``: the committed stream, or it extended by the
        acceptance of the last tree verified through ``tree_argmax`` / ``tree_sample`` (the
        same K6 walk on the same target tokens) or by the last ``next_token`` result."""
        prefix = tuple(int(x) for x in prefix)
        pend, self._pending = getattr(self, "_pending", None), None
        if prefix == tuple(self.tokens()):
            return
        from ..verify_sim import accept_device
        with torch.cuda.stream(self.stream):
            if pend == "tree":
                t, tr = self.target, self.tree
                accept_device(tr.token, tr.child_start, tr.child_list, t.argmax, self.gamma + 1, self.path,
                              self.committed, self.acc_meta)
                self._commit_tail()
            elif isinstance(pend, tuple) and pend[0] == "ar":
                self.path[:1].zero_()
                self.committed[:1].fill_(pend[1])
                self.acc_meta[:2].copy_(torch.tensor([1, pend[1]], dtype=torch.int32))
                self._commit_tail()
        self.stream.synchronize()
        if prefix != tuple(self.tokens()):
            raise ValueError("engine plugin: prefix does not continue the engine's committed stream")

    def _tree_verify(self, tree, prefix) -> torch.Tensor:
        from ..verify_sim import _device_children
        self._sync(prefix)
        n = len(tree.nodes) - 1
        if n > self.n_cap:
            raise ValueError(f"tree of {n} nodes exceeds the engine's capacity {self.n_cap}")
        tr, t = self.tree, self.target
        parents = [-1] + [x.parent for x in tree.nodes[1:]]
        with torch.cuda.stream(self.stream):
            tok, start, kids = _device_children(tree)
            tr.token[: n + 1].copy_(tok[: n + 1])
            tr.child_start[: n + 2].copy_(start[: n + 2])
            tr.child_list[: max(n, 1)].copy_(kids[: max(n, 1)])
            tr.parent[: n + 1].copy_(torch.tensor(parents, dtype=torch.int32))
            tr.depth[: n + 1].copy_(torch.tensor([x.depth for x in tree.nodes], dtype=torch.int32))
            tr.meta.zero_()
            tr.meta[0] = n
            self._check_room(int(self.state[ST_C].item()), self._bucket(n))
            _lib.call("bst_ancestor_mask", tr.parent.data_ptr(), n + 1, tr.mask_words, tr.anc_mask.data_ptr(),
                      self.stream.cuda_stream)
            self._verify_forward(self._bucket(n))
        self.stream.synchronize()
        self._pending = "tree"
        return t.argmax[: n + 1]

    def tree_argmax(self, tree, prefix) -> torch.Tensor:
        """Greedy target token after every tree node (int32 device tensor, one batched verify)."""
        self.set_temperature(0.0, self.target.sample_seed)
        return self._tree_verify(tree, prefix)

    def tree_sample(self, tree, prefix, temperature: float) -> torch.Tensor:
        """Temperature-T target sample after every tree node (exact-match sampled verification)."""
        self.set_temperature(temperature, self.target.sample_seed)
        return self._tree_verify(tree, prefix)

    def next_token(self, prefix, temperature: float) -> int:
        """One target step after ``prefix`` (greedy at T = 0, else the keyed sample)."""
        self.set_temperature(temperature, self.target.sample_seed)
        self._sync(prefix)
        self._check_room(int(self.state[ST_C].item()), 1)
        t = self.target
        with torch.cuda.stream(self.stream):
            t.tokens[:1].copy_(self.state[ST_BONUS:ST_BONUS + 1])
            t.pos[:1].zero_()
            t.slot[:1].zero_()
            t.forward(1, self.state, MODE_CAUSAL, keys_after_c=1, head=self._head())
        self.stream.synchronize()
        tok = int(t.argmax[0].item())
        self._pending = ("ar", tok)
        return tok

    def __repr__(self) -> str:  # pragma: no cover
        return f"B200Engine({self.cfg.name}, gamma={self.gamma}, top_k={self.top_k}, n_cap={self.n_cap})"


def default_stop_name(stop: int) -> str:
    return _lib.STOP_NAMES.get(stop, STOP_BUDGET_CAP)
