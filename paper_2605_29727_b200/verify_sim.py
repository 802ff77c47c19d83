"""Linearize / verify / commit and the multi-cycle decode loop.

API mirrors ``specplan.verify_sim`` (verify_sim.py:206-511).  Compute runs on
the device: ``linearize`` expands the K2 ancestor bitmask into the reference's
dense mask (``bst_linearize_mask``), ``verify_tree`` runs the K6 acceptance
walk (``bst_accept``) whenever the target can score the whole tree in one pass
(a plugin with ``tree_argmax`` — the B200 engine), and ``decode`` hands the
whole loop to the engine's on-device fast path when the plugin is an engine.

Plugin protocol (verify_sim.py:433,440,381): ``drafter_marginals(prefix) ->
MarginalBlock`` and ``next_token(prefix, temperature) -> int``.  A plain
Python plugin that only answers ``next_token`` one sequence at a time is
walked exactly like the reference does (the walk is the plugin's call order).
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _lib
from .controller import ControllerConfig, run_cycle
from .cost_model import VerifyLatencyEstimator
from .device import require_cuda, stream_ptr
from .draft_tree import DeviceTree, DraftTree, beam_expand, best_first_expand
from .lattice import CandidateLattice, MarginalBlock, top_k_truncate

CYCLE_CSV_COLUMNS = ("cycle", "policy", "N", "accepted_len", "surrogate", "t_draft", "t_verify", "t_aux",
                     "cum_tokens", "cum_time")


@dataclass(frozen=True)
class LinearizedTree:
    """Flattened tree + (prefix+t)^2 mask (verify_sim.py:206-221)."""

    tokens: tuple[int, ...]
    position_ids: tuple[int, ...]
    parents: tuple[int, ...]
    prefix_len: int
    mask: np.ndarray


@dataclass(frozen=True)
class AcceptanceRecord:
    accepted_path: tuple[int, ...]
    accepted_len: int
    bonus_token: int

    def __post_init__(self) -> None:
        if self.accepted_len != len(self.accepted_path):
            raise ValueError("accepted_len must count accepted draft tokens plus the bonus")


@dataclass(frozen=True)
class SimCache:
    tokens: tuple[int, ...] = ()

    def __len__(self) -> int:
        return len(self.tokens)


@dataclass(frozen=True)
class CycleRecord:
    """One decode cycle (verify_sim.py:247-262)."""

    tree_size: int
    accepted_len: int
    surrogate: float
    t_draft: float
    t_verify: float
    t_aux: float
    l_ar: float
    cycle_speedup: float

    @property
    def cycle_time(self) -> float:
        return self.t_draft + self.t_verify + self.t_aux


@dataclass(frozen=True)
class Policy:
    """adaptive | fixed-N | greedy-chain | beam-WxD (verify_sim.py:265-315)."""

    kind: str
    n: int = 0
    width: int = 0
    depth: int = 0

    @classmethod
    def adaptive(cls) -> "Policy":
        return cls(kind="adaptive")

    @classmethod
    def fixed(cls, n: int) -> "Policy":
        if n < 1:
            raise ValueError("fixed policy needs n >= 1")
        return cls(kind="fixed", n=n)

    @classmethod
    def greedy_chain(cls) -> "Policy":
        return cls(kind="greedy-chain")

    @classmethod
    def beam(cls, width: int, depth: int) -> "Policy":
        if width < 1 or depth < 1:
            raise ValueError("beam policy needs width >= 1 and depth >= 1")
        return cls(kind="beam", width=width, depth=depth)

    @property
    def label(self) -> str:
        return {"fixed": f"fixed-{self.n}", "beam": f"beam-{self.width}x{self.depth}"}.get(self.kind, self.kind)

    @classmethod
    def parse(cls, text: str) -> "Policy":
        text = text.strip()
        if text == "adaptive":
            return cls.adaptive()
        if text in ("greedy-chain", "greedy"):
            return cls.greedy_chain()
        if text.startswith("fixed-"):
            return cls.fixed(int(text.split("-", 1)[1]))
        if text.startswith("beam-"):
            w, _, d = text.split("-", 1)[1].partition("x")
            return cls.beam(int(w), int(d))
        raise ValueError(f"unknown policy {text!r}")


@dataclass(frozen=True)
class SimConfig:
    controller: ControllerConfig
    run_length: int
    top_k: int = 8
    temperature: float = 0.0

    def __post_init__(self) -> None:
        if self.run_length < 1:
            raise ValueError("run_length must be >= 1")
        if self.top_k < 1:
            raise ValueError("top_k must be >= 1")
        if self.temperature < 0.0:
            raise ValueError("temperature must be >= 0")


# --------------------------------------------------------------------- helpers
def _device_mask(tree: DraftTree) -> tuple[torch.Tensor, int]:
    """Ancestor bitmask rows 0..size on the device (from K2, or built for host trees)."""
    t = len(tree.nodes)
    dt = tree.device
    if dt is not None:
        return dt.anc_mask, dt.mask_words
    dev = require_cuda()
    parents = torch.tensor([-1] + [n.parent for n in tree.nodes[1:]], dtype=torch.int32, device=dev)
    words = (t + 31) // 32
    mask = torch.empty(t * words, dtype=torch.int32, device=dev)
    _lib.call("bst_ancestor_mask", parents.data_ptr(), t, words, mask.data_ptr(), stream_ptr())
    return mask, words


def _device_children(tree: DraftTree) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """(token, child_start, child_list) device arrays for the acceptance walk."""
    dt = tree.device
    if dt is not None:
        return dt.token, dt.child_start, dt.child_list
    dev = require_cuda()
    t = len(tree.nodes)
    kids: list[list[int]] = [[] for _ in range(t)]
    for n in tree.nodes[1:]:
        kids[n.parent].append(n.id)
    start = np.zeros(t + 1, dtype=np.int32)
    start[1:] = np.cumsum([len(k) for k in kids])
    flat = np.array([c for k in kids for c in k] or [0], dtype=np.int32)
    token = np.array([-1] + [n.token for n in tree.nodes[1:]], dtype=np.int32)
    return (torch.from_numpy(token).to(dev), torch.from_numpy(start).to(dev), torch.from_numpy(flat).to(dev))


def accept_device(token: torch.Tensor, child_start: torch.Tensor, child_list: torch.Tensor, argmax: torch.Tensor,
                  max_path: int, path: torch.Tensor | None = None, committed: torch.Tensor | None = None,
                  meta: torch.Tensor | None = None):
    """K6 walk on the device; returns (path, committed, meta) device tensors (asynchronous)."""
    dev = token.device
    path = path if path is not None else torch.empty(max_path, dtype=torch.int32, device=dev)
    committed = committed if committed is not None else torch.empty(max_path, dtype=torch.int32, device=dev)
    meta = meta if meta is not None else torch.empty(4, dtype=torch.int32, device=dev)
    _lib.call("bst_accept", token.data_ptr(), child_start.data_ptr(), child_list.data_ptr(), argmax.data_ptr(),
              max_path, path.data_ptr(), committed.data_ptr(), meta.data_ptr(), stream_ptr())
    return path, committed, meta


# ------------------------------------------------------------------- public API
def linearize(tree: DraftTree, prefix_len: int) -> LinearizedTree:
    """Expansion-order tokens/positions/parents + ancestor-only mask (verify_sim.py:336-355)."""
    if prefix_len < 0:
        raise ValueError("prefix_len must be >= 0")
    nodes = tree.nodes
    t = len(nodes)
    anc, words = _device_mask(tree)
    n = prefix_len + t
    dense = torch.empty((n, n), dtype=torch.uint8, device=anc.device)
    _lib.call("bst_linearize_mask", anc.data_ptr(), words, t, prefix_len, dense.data_ptr(), stream_ptr())
    return LinearizedTree(
        tokens=tuple(-1 if x.token is None else x.token for x in nodes),
        position_ids=tuple(x.depth for x in nodes),
        parents=tuple(-1 if x.parent is None else x.parent for x in nodes),
        prefix_len=prefix_len,
        mask=dense.cpu().numpy().astype(bool))


def verify_tree(lin: LinearizedTree, tree: DraftTree, target, temperature: float,
                prefix: Sequence[int] = ()) -> AcceptanceRecord:
    """Longest target-consistent root chain + bonus (verify_sim.py:358-389)."""
    if temperature < 0.0:
        raise ValueError("temperature must be >= 0")
    if len(lin.tokens) != len(tree.nodes):
        raise ValueError("linearization does not match the tree")
    batched = hasattr(target, "tree_argmax") if temperature == 0.0 else hasattr(target, "tree_sample")
    if batched:
        # one batched verify pass, int32[t] on device: the target's token after every node
        argmax = (target.tree_argmax(tree, tuple(prefix)) if temperature == 0.0
                  else target.tree_sample(tree, tuple(prefix), temperature))
        token, start, kids = _device_children(tree)
        max_path = tree.lattice.gamma + 1
        path, _, meta = accept_device(token, start, kids, argmax, max_path)
        m = meta.cpu().numpy()
        p = tuple(int(x) for x in path[: int(m[0])].cpu().numpy())
        return AcceptanceRecord(accepted_path=p, accepted_len=len(p), bonus_token=int(m[1]))
    children = tree.child_index()
    seq, path, cur = list(prefix), [0], 0
    while True:
        tok = target.next_token(seq, temperature)
        nxt = children[cur].get(tok)
        if nxt is None:
            return AcceptanceRecord(accepted_path=tuple(path), accepted_len=len(path), bonus_token=tok)
        path.append(nxt)
        seq.append(tok)
        cur = nxt


def commit(cache: SimCache, rec: AcceptanceRecord, tree: DraftTree) -> SimCache:
    """Append accepted draft tokens then the bonus (verify_sim.py:392-405)."""
    path = rec.accepted_path
    if not path or path[0] != 0:
        raise ValueError("accepted path must start at the root")
    out: list[int] = []
    for a, b in zip(path, path[1:]):
        if b >= len(tree.nodes):
            raise ValueError(f"accepted node {b} is not in the tree")
        node = tree.nodes[b]
        if node.parent != a:
            raise ValueError("accepted path is not a root-anchored chain in this tree")
        out.append(node.token)
    return SimCache(tokens=cache.tokens + tuple(out) + (rec.bonus_token,))


def plan_tree(lattice: CandidateLattice, policy: Policy, cfg: ControllerConfig,
              estimator: VerifyLatencyEstimator) -> DraftTree:
    """Policy dispatch (verify_sim.py:408-423)."""
    if policy.kind == "adaptive":
        return run_cycle(lattice, cfg, estimator).tree
    if policy.kind == "fixed":
        return best_first_expand(lattice, policy.n)
    if policy.kind == "greedy-chain":
        return beam_expand(lattice, width=1, depth=lattice.gamma)
    if policy.kind == "beam":
        return beam_expand(lattice, width=policy.width, depth=policy.depth)
    raise ValueError(f"unknown policy kind {policy.kind!r}")


def decode_full(pair, cfg: SimConfig, policy: Policy, estimator: VerifyLatencyEstimator):
    """Decode until run_length tokens are committed; returns (records, tokens) (verify_sim.py:426-461)."""
    rule = pair[1] if isinstance(pair, tuple) else pair
    if hasattr(rule, "engine_decode") and policy.kind in ("adaptive", "fixed"):
        return rule.engine_decode(cfg, policy, estimator)  # the whole loop on the device
    # any other policy (greedy chain, beam) runs the reference loop below; a GPU engine
    # still serves it through the plugin protocol (drafter_marginals / tree_argmax)
    lat = cfg.controller.latencies
    cache = SimCache()
    records: list[CycleRecord] = []
    while len(cache) < cfg.run_length:
        prefix = cache.tokens
        context = cfg.controller.context_len + len(prefix)
        block = rule.drafter_marginals(prefix)
        lattice = top_k_truncate(block, min(cfg.top_k, block.vocab_size))
        tree = plan_tree(lattice, policy, replace(cfg.controller, context_len=context), estimator)
        lin = linearize(tree, prefix_len=context)
        rec = verify_tree(lin, tree, rule, cfg.temperature, prefix)
        cache = commit(cache, rec, tree)
        t_verify = estimator.estimate_for_budget(tree.size, context)
        cyc = lat.t_draft + t_verify + lat.t_aux
        records.append(CycleRecord(tree_size=tree.size, accepted_len=rec.accepted_len, surrogate=tree.surrogate,
                                   t_draft=lat.t_draft, t_verify=t_verify, t_aux=lat.t_aux, l_ar=lat.l_ar,
                                   cycle_speedup=rec.accepted_len * lat.l_ar / cyc))
    return records, cache.tokens


def decode(pair, cfg: SimConfig, policy: Policy, estimator: VerifyLatencyEstimator) -> list[CycleRecord]:
    """Run decode cycles until cfg.run_length tokens are committed (verify_sim.py:464-479)."""
    return decode_full(pair, cfg, policy, estimator)[0]


def realized_speedup(records: Sequence[CycleRecord]) -> float:
    if not records:
        raise ValueError("realized_speedup needs at least one cycle record")
    return sum(r.accepted_len for r in records) * records[0].l_ar / sum(r.cycle_time for r in records)


def ar_decode(rule, length: int, temperature: float = 0.0) -> tuple[int, ...]:
    """One-token-per-step reference decode of a plugin (verify_sim.py:491-496)."""
    if hasattr(rule, "engine_ar_decode"):
        return rule.engine_ar_decode(length)
    seq: list[int] = []
    for _ in range(length):
        seq.append(rule.next_token(seq, temperature))
    return tuple(seq)


def cycle_csv_rows(records: Iterable[CycleRecord], policy_label: str) -> list[str]:
    rows, tok, tim = [], 0, 0.0
    for i, r in enumerate(records):
        tok += r.accepted_len
        tim += r.cycle_time
        rows.append(f"{i},{policy_label},{r.tree_size},{r.accepted_len},{r.surrogate!r},"
                    f"{r.t_draft!r},{r.t_verify!r},{r.t_aux!r},{tok},{tim!r}")
    return rows
