"""CPU ORACLE — test infrastructure only, never the product path.

A numpy / pure-Python restatement of the reference ``specplan`` hot path
(arxiv/paper_2605_29727, package at ``/root/reference/pkg/src/specplan``; ``sp/``
below).  It works on flat arrays (the same layout the CUDA kernels emit) instead
of the reference's frozen dataclasses, so a GPU result can be diffed field by
field.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg
and ``--impl reference``) may import this module, and there only as the checker
or the timed CPU baseline.

Parity pinning: every function here is checked against golden vectors produced
by the real reference in this container (``tests/golden/make_golden.py``) and
against the SPEC known-answer tests (``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np

STOP_FIRST_DECREASE = 0  # "first-decrease"      sp/controller.py:19
STOP_FRONTIER_EXHAUSTED = 1  # "frontier-exhausted"  sp/controller.py:20
STOP_BUDGET_CAP = 2  # "budget-cap"          sp/controller.py:21
STOP_NAMES = ("first-decrease", "frontier-exhausted", "budget-cap")


# ---------------------------------------------------------------------------
# a2: top-K lattice                                   sp/lattice.py:128-142
# ---------------------------------------------------------------------------
def topk_rows(probs: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Per row: the k largest probabilities, ties by ascending token id.

    Follows ``top_k_truncate`` (sp/lattice.py:128-142): ``np.lexsort`` with the
    token id as the secondary key and ``-prob`` as the primary key.
    Returns ``tok int32[gamma,k]`` and ``prob float64[gamma,k]``.
    """
    probs = np.asarray(probs, dtype=np.float64)
    gamma, vocab = probs.shape
    if not 1 <= k <= vocab:
        raise ValueError(f"k must be in [1, {vocab}], got {k}")
    ids = np.arange(vocab)
    tok = np.empty((gamma, k), dtype=np.int32)
    val = np.empty((gamma, k), dtype=np.float64)
    for r in range(gamma):
        order = np.lexsort((ids, -probs[r]))[:k]
        tok[r] = order
        val[r] = probs[r][order]
    return tok, val


def softmax_rows_f64(logits: np.ndarray) -> np.ndarray:
    """fp64 softmax of fp32/bf16 logits, the drafter-plugin side of a1.

    Not part of the reference (which receives probabilities from its plugin);
    used by the CPU baseline to turn logits into a MarginalBlock.
    """
    x = np.asarray(logits, dtype=np.float64)
    x = x - x.max(axis=1, keepdims=True)
    w = np.exp(x)
    return w / w.sum(axis=1, keepdims=True)


# ---------------------------------------------------------------------------
# Trees as flat arrays (node 0 = root).  DraftTree  sp/draft_tree.py:37-66
# ---------------------------------------------------------------------------
@dataclass
class FlatTree:
    parent: np.ndarray  # int32[n+1], root -1
    depth: np.ndarray  # int32[n+1]
    token: np.ndarray  # int32[n+1], root -1
    rank: np.ndarray  # int32[n+1] lattice rank of the node's token, root -1
    rho: np.ndarray  # float64[n+1], root 1.0
    surrogate: float

    @property
    def size(self) -> int:
        return len(self.parent) - 1


def _flat(rows: list[tuple[int, int, int, int, float]], surrogate: float) -> FlatTree:
    parent = np.array([-1] + [r[0] for r in rows], dtype=np.int32)
    depth = np.array([0] + [r[1] for r in rows], dtype=np.int32)
    token = np.array([-1] + [r[2] for r in rows], dtype=np.int32)
    rank = np.array([-1] + [r[3] for r in rows], dtype=np.int32)
    rho = np.array([1.0] + [r[4] for r in rows], dtype=np.float64)
    return FlatTree(parent, depth, token, rank, rho, surrogate)


# ---------------------------------------------------------------------------
# a3/a4: lazy best-first order                     sp/draft_tree.py:69-135
# ---------------------------------------------------------------------------
def best_first_stream(tok: np.ndarray, prob: np.ndarray):
    """Yield (parent, depth, token, rank, rho) in best-first pop order.

    Heap key (-rho, depth, token, parent, rank) as in ExpansionFrontier
    (sp/draft_tree.py:79-94); on each pop the rank-0 child of the new node
    (sp/draft_tree.py:96-104) and the next sibling of the popped entry
    (sp/draft_tree.py:106-115) are pushed when their path score is > 0.
    """
    gamma, k = tok.shape
    t = [[int(x) for x in row] for row in tok]
    p = [[float(x) for x in row] for row in prob]
    heap: list[tuple[float, int, int, int, int]] = []
    if k > 0 and p[0][0] > 0.0:
        heapq.heappush(heap, (-p[0][0], 1, t[0][0], 0, 0))
    score = [1.0]
    while heap:
        neg, d, token, par, r = heapq.heappop(heap)
        rho = -neg
        node = len(score)
        score.append(rho)
        if d < gamma:  # rank-0 child of the node just added
            c_rho = rho * p[d][0]
            if c_rho > 0.0:
                heapq.heappush(heap, (-c_rho, d + 1, t[d][0], node, 0))
        if r + 1 < k:  # next sibling of the popped entry
            s_rho = score[par] * p[d - 1][r + 1]
            if s_rho > 0.0:
                heapq.heappush(heap, (-s_rho, d, t[d - 1][r + 1], par, r + 1))
        yield par, d, token, r, rho


def _require_nonempty(prob: np.ndarray) -> None:
    # sp/draft_tree.py:304-307
    if prob.shape[1] == 0 or not prob[0, 0] > 0.0:
        raise ValueError("lattice has no positive-probability candidates at position 1")


def best_first(tok: np.ndarray, prob: np.ndarray, n_max: int) -> FlatTree:
    """``best_first_expand`` (sp/draft_tree.py:138-155): first min(n_max, reachable) nodes."""
    if n_max < 1:
        raise ValueError(f"n_max must be >= 1, got {n_max}")
    _require_nonempty(prob)
    rows = []
    acc = 1.0
    for row in best_first_stream(tok, prob):
        rows.append(row)
        acc += row[4]
        if len(rows) >= n_max:
            break
    return _flat(rows, acc)


def beam(tok: np.ndarray, prob: np.ndarray, width: int, depth: int) -> FlatTree:
    """``beam_expand`` (sp/draft_tree.py:158-189): level-wise top-``width`` by (-rho, token, parent)."""
    gamma, k = tok.shape
    if width < 1:
        raise ValueError(f"width must be >= 1, got {width}")
    if not 1 <= depth <= gamma:
        raise ValueError(f"depth must be in [1, {gamma}], got {depth}")
    _require_nonempty(prob)
    rows: list[tuple[int, int, int, int, float]] = []
    acc = 1.0
    alive = [(0, 1.0)]  # (node id, rho)
    for level in range(1, depth + 1):
        cand = []
        for pid, prho in alive:
            for r in range(k):
                v = prho * float(prob[level - 1, r])
                if v > 0.0:
                    cand.append((-v, int(tok[level - 1, r]), pid, r, v))
        if not cand:
            break
        cand.sort(key=lambda c: (c[0], c[1], c[2]))
        alive = []
        for _, token, pid, r, v in cand[:width]:
            rows.append((pid, level, token, r, v))
            acc += v
            alive.append((len(rows), v))
    return _flat(rows, acc)


# ---------------------------------------------------------------------------
# a8/a9: cost model                                    sp/cost_model.py:113-309
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Dims:
    """CostModelParams (sp/cost_model.py:26-57)."""

    L: int
    h: int
    n_q: int
    n_kv: int
    d: int
    h_ffn: int
    V: int
    bp: int
    peak_flops: float
    bandwidth: float

    @property
    def h_q(self) -> int:
        return self.n_q * self.d

    @property
    def h_kv(self) -> int:
        return self.n_kv * self.d


def flops(p: Dims, s: int, c: int) -> int:
    """Appendix-D FLOPs, sp/cost_model.py:118-123."""
    layer = 4 * s * p.h * p.h_q + 4 * s * p.h * p.h_kv + 4 * s * (c + s) * p.h_q + 6 * s * p.h * p.h_ffn
    return p.L * layer + 2 * s * p.h * p.V


def bytes_moved(p: Dims, s: int, c: int) -> int:
    """Appendix-D bytes (closed form), sp/cost_model.py:145-156."""
    layer = (
        2 * p.h * (p.h_q + p.h_kv)
        + 3 * p.h * p.h_ffn
        + 2 * p.h_kv * (c + 2 * s)
        + 4 * s * (p.h + p.h_q + p.h_ffn)
        + 2 * p.n_q * s * (c + s)
    )
    return p.bp * (2 * p.V * p.h + s * (p.h + p.V) + p.L * layer)


def bytes_by_category(p: Dims, s: int, c: int) -> tuple[int, int, int]:
    """(weights, kv cache, activations), sp/cost_model.py:126-142."""
    w = p.bp * (p.L * (2 * p.h * p.h_q + 2 * p.h * p.h_kv + 3 * p.h * p.h_ffn) + 2 * p.V * p.h)
    kv = p.bp * p.L * (2 * c * p.h_kv + 2 * s * p.h_kv)
    act_layer = 4 * s * p.h + 4 * s * p.h_q + 2 * s * p.h_kv + 4 * s * p.h_ffn + 2 * p.n_q * s * (c + s)
    act = p.bp * (p.L * act_layer + s * p.h + s * p.V)
    return w, kv, act


def roofline(p: Dims, s: int, c: int) -> float:
    """sp/cost_model.py:159-161 (true divisions, not reciprocal multiplies)."""
    return max(flops(p, s, c) / p.peak_flops, bytes_moved(p, s, c) / p.bandwidth)


def apply_variant(variant: str, raw: float, slope: float, intercept: float, ratio: float) -> float:
    """``_apply_variant`` (sp/cost_model.py:208-223) with the fit/bias unpacked."""
    if variant in ("static", "ema_calib"):
        raw = slope * raw + intercept
    if variant in ("ema", "ema_calib"):
        raw = ratio * raw
    return raw


@dataclass(frozen=True)
class Curve:
    """Exact-integer coefficients of ``LatencyCurve`` (sp/cost_model.py:287-303)."""

    flops_lin: int
    flops_quad: int
    bytes_const: int
    bytes_lin: int
    bytes_quad: int
    inv_peak: float
    inv_bw: float
    slope: float
    intercept: float
    ratio: float
    flops_const: int = 0  # batched verify: the other requests' flops (not in the reference)

    def latency(self, s: int) -> float:
        """sp/cost_model.py:305-309 — note the reciprocal multiply."""
        compute = (self.flops_const + (self.flops_lin + self.flops_quad * s) * s) * self.inv_peak
        memory = (self.bytes_const + (self.bytes_lin + self.bytes_quad * s) * s) * self.inv_bw
        raw = compute if compute > memory else memory
        return self.ratio * (self.slope * raw + self.intercept)


def curve_for(p: Dims, c: int, variant: str = "static", slope: float = 1.0,
              intercept: float = 0.0, ratio: float = 1.0) -> Curve:
    """Coefficients at fixed context ``c`` (sp/cost_model.py:287-303).

    ``slope/intercept`` only apply to static/ema_calib and ``ratio`` only to
    ema/ema_calib, exactly like the reference constructor.
    """
    h, hq, hkv, hf = p.h, p.h_q, p.h_kv, p.h_ffn
    s_, i_, r_ = 1.0, 0.0, 1.0
    if variant in ("static", "ema_calib"):
        s_, i_ = slope, intercept
    if variant in ("ema", "ema_calib"):
        r_ = ratio
    return Curve(
        flops_lin=p.L * (4 * h * hq + 4 * h * hkv + 4 * c * hq + 6 * h * hf) + 2 * h * p.V,
        flops_quad=4 * p.L * hq,
        bytes_const=p.bp * (2 * p.V * h + p.L * (2 * h * (hq + hkv) + 3 * h * hf + 2 * hkv * c)),
        bytes_lin=p.bp * (h + p.V + p.L * (4 * hkv + 4 * (h + hq + hf) + 2 * p.n_q * c)),
        bytes_quad=p.bp * p.L * 2 * p.n_q,
        inv_peak=1.0 / p.peak_flops,
        inv_bw=1.0 / p.bandwidth,
        slope=s_,
        intercept=i_,
        ratio=r_,
    )


def ema_step(ratio: float, alpha: float, predicted: float, observed: float) -> float:
    """``ema_update`` (sp/cost_model.py:184-189)."""
    if predicted <= 0.0 or observed <= 0.0:
        raise ValueError("predicted and observed must be > 0")
    return (1.0 - alpha) * ratio + alpha * (observed / predicted)


def ols_fit(pairs: list[tuple[float, float]]) -> tuple[float, float, float, float]:
    """``fit_static_calibration`` (sp/cost_model.py:164-181): biased cov / var."""
    if len(pairs) < 2:
        raise ValueError("need at least 2 (predicted, observed) pairs")
    x = np.array([a for a, _ in pairs], dtype=np.float64)
    y = np.array([b for _, b in pairs], dtype=np.float64)
    var = float(np.var(x))
    if var == 0.0:
        raise ValueError("all predicted values are equal; fit is underdetermined")
    slope = float(np.cov(x, y, bias=True)[0, 1] / var)
    icpt = float(y.mean() - slope * x.mean())
    before = float(np.sqrt(np.mean((y - x) ** 2)))
    after = float(np.sqrt(np.mean((y - (slope * x + icpt)) ** 2)))
    return slope, icpt, before, after


# ---------------------------------------------------------------------------
# a7: Algorithm 1                                       sp/controller.py:56-107
# ---------------------------------------------------------------------------
@dataclass
class Decision:
    tree: FlatTree
    budget: int
    trace: list[float]
    stop: int


def controller(tok: np.ndarray, prob: np.ndarray, n_max: int, curve: Curve,
               t_draft: float, t_aux: float, l_ar: float, a_offset: float = 0.0) -> Decision:
    """Expand best-first and stop at the first strict decrease of S_hat.

    Arithmetic order follows sp/controller.py:73-98: fixed = t_draft + t_aux;
    a_hat += rho; c_hat = fixed + curve.latency(n + 1); s_hat = a_hat * l_ar / c_hat.
    Equal S_hat keeps expanding without moving best_n.  ``a_offset`` (batched verify,
    not in the reference; 0 reproduces it exactly): s_hat = (a_hat + a_offset) * l_ar / c_hat.
    """
    if n_max < 1:
        raise ValueError(f"n_max must be >= 1, got {n_max}")
    fixed = t_draft + t_aux
    rows = []
    trace: list[float] = []
    a_hat, best_s, best_n, best_a = 1.0, float("-inf"), 0, 1.0
    stop = STOP_FRONTIER_EXHAUSTED
    for row in best_first_stream(tok, prob):
        rows.append(row)
        n = len(rows)
        a_hat += row[4]
        s_hat = (a_hat + a_offset) * l_ar / (fixed + curve.latency(n + 1))
        trace.append(s_hat)
        if s_hat > best_s:
            best_s, best_n, best_a = s_hat, n, a_hat
        elif s_hat < best_s:
            stop = STOP_FIRST_DECREASE
            break
        if n >= n_max:
            stop = STOP_BUDGET_CAP
            break
    return Decision(_flat(rows[:best_n], best_a), best_n, trace, stop)


def replay(gains: list[float], costs: list[float], l_ar: float) -> tuple[int, list[float], int]:
    """``replay_trace`` stopping rule (sp/controller.py:110-147), minus validation."""
    trace = []
    a_hat, best_s, best_n, stop = 1.0, float("-inf"), 0, STOP_BUDGET_CAP
    for i, g in enumerate(gains):
        a_hat += g
        s = a_hat * l_ar / costs[i]
        trace.append(s)
        if s > best_s:
            best_s, best_n = s, i + 1
        elif s < best_s:
            stop = STOP_FIRST_DECREASE
            break
    return best_n, trace, stop


# ---------------------------------------------------------------------------
# a11: linearize                                        sp/verify_sim.py:336-355
# ---------------------------------------------------------------------------
def ancestor_bits(parent: np.ndarray) -> np.ndarray:
    """bool[t, t]: row i marks i and every ancestor of i (tree-block part of the mask)."""
    t = len(parent)
    m = np.zeros((t, t), dtype=bool)
    for i in range(t):
        if parent[i] >= 0:
            m[i] = m[parent[i]]
        m[i, i] = True
    return m


def linear_mask(parent: np.ndarray, prefix_len: int) -> np.ndarray:
    """Full (prefix+t)^2 mask: prefix columns visible to every row, tree part ancestor-or-self.

    sp/verify_sim.py:345-352 — note the prefix rows are all-True over the prefix
    columns (not causal) and False over the tree columns.
    """
    t = len(parent)
    n = prefix_len + t
    m = np.zeros((n, n), dtype=bool)
    m[:, :prefix_len] = True
    m[prefix_len:, prefix_len:] = ancestor_bits(parent)
    return m


# ---------------------------------------------------------------------------
# a12/a13: acceptance walk + commit                 sp/verify_sim.py:358-405
# ---------------------------------------------------------------------------
def accept_walk(parent: np.ndarray, token: np.ndarray, choose) -> tuple[list[int], int]:
    """Descend from the root while the target's choice matches a child.

    ``choose(node_id, seq_tokens)`` returns the target's token after the path to
    ``node_id``.  Returns (path including root 0, bonus token).
    """
    kids: dict[int, dict[int, int]] = {}
    for i in range(1, len(parent)):
        kids.setdefault(int(parent[i]), {})[int(token[i])] = i
    path, seq, cur = [0], [], 0
    while True:
        t = int(choose(cur, seq))
        nxt = kids.get(cur, {}).get(t)
        if nxt is None:
            return path, t
        path.append(nxt)
        seq.append(t)
        cur = nxt


def accept_from_argmax(parent: np.ndarray, token: np.ndarray, argmax: np.ndarray) -> tuple[list[int], int]:
    """Same walk with a per-node greedy target table (the verify forward's argmax rows)."""
    return accept_walk(parent, token, lambda node, _seq: int(argmax[node]))


def committed_tokens(path: list[int], token: np.ndarray, bonus: int) -> list[int]:
    """``commit`` (sp/verify_sim.py:392-405): accepted draft tokens then the bonus."""
    return [int(token[i]) for i in path[1:]] + [int(bonus)]


def compaction_moves(path: list[int], c: int) -> list[tuple[int, int]]:
    """KV slot moves implied by commit: slot c+path[i] -> c+i (SURVEY §8a′)."""
    return [(c + p, c + i) for i, p in enumerate(path) if p != i]


# ---------------------------------------------------------------------------
# a14/a15: policy dispatch + decode loop          sp/verify_sim.py:408-461
# ---------------------------------------------------------------------------
def plan(tok, prob, policy: tuple, n_max: int, curve: Curve | None,
         t_draft: float, t_aux: float, l_ar: float) -> FlatTree:
    """``plan_tree`` (sp/verify_sim.py:408-423). policy = (kind, n, width, depth)."""
    kind = policy[0]
    if kind == "adaptive":
        return controller(tok, prob, n_max, curve, t_draft, t_aux, l_ar).tree
    if kind == "fixed":
        return best_first(tok, prob, policy[1])
    if kind == "greedy-chain":
        return beam(tok, prob, 1, tok.shape[0])
    if kind == "beam":
        return beam(tok, prob, policy[2], policy[3])
    raise ValueError(f"unknown policy kind {kind!r}")


def decode_loop(drafter, target, run_length: int, top_k: int, policy: tuple, n_max: int,
                dims: Dims, context_len: int, t_draft: float, t_aux: float, l_ar: float,
                variant: str = "static", slope: float = 1.0, intercept: float = 0.0,
                ratio: float = 1.0, temperature: float = 0.0):
    """``decode_full`` (sp/verify_sim.py:426-461) over array trees.

    ``drafter(prefix) -> probs[gamma,V]``; ``target(seq, T) -> int``.
    Returns (records, tokens) with records as dicts of the CycleRecord fields.
    """
    cache: list[int] = []
    records = []
    while len(cache) < run_length:
        prefix = tuple(cache)
        ctx = context_len + len(prefix)
        probs = drafter(prefix)
        tok, prob = topk_rows(probs, min(top_k, probs.shape[1]))
        curve = curve_for(dims, ctx, variant, slope, intercept, ratio)
        tree = plan(tok, prob, policy, n_max, curve, t_draft, t_aux, l_ar)
        path, bonus = accept_walk(tree.parent, tree.token,
                                  lambda _n, seq: target(list(prefix) + seq, temperature))
        cache += committed_tokens(path, tree.token, bonus)
        t_verify = apply_variant(variant, roofline(dims, tree.size + 1, ctx), slope, intercept, ratio)
        cyc = t_draft + t_verify + t_aux
        records.append(dict(tree_size=tree.size, accepted_len=len(path), surrogate=tree.surrogate,
                            t_draft=t_draft, t_verify=t_verify, t_aux=t_aux, l_ar=l_ar,
                            cycle_speedup=len(path) * l_ar / cyc))
    return records, tuple(cache)
