"""Prefix-closed draft trees built on the device (K2).

Types mirror ``specplan.draft_tree`` (draft_tree.py:26-66); the builders keep
the reference signatures and node order — best-first (draft_tree.py:138-155)
and beam (draft_tree.py:158-189) — but run ``bst_expand`` on one CTA.
:class:`DeviceTree` is the engine-side result: every array stays on the GPU,
including the ancestor bitmask the verify attention consumes and the children
CSR the acceptance walk uses.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .device import require_cuda, stream_ptr, workspace
from .lattice import CandidateLattice

SURROGATE_TOL = 1e-9


@dataclass(frozen=True, slots=True)
class TreeNode:
    id: int
    parent: int | None
    depth: int
    token: int | None
    path_score: float


@dataclass(frozen=True)
class DraftTree:
    """Immutable tree; nodes[0] is the root, order = expansion order (draft_tree.py:37-66)."""

    nodes: tuple[TreeNode, ...]
    lattice: CandidateLattice
    surrogate: float
    method: str
    device: "DeviceTree | None" = field(default=None, compare=False, repr=False)

    @property
    def size(self) -> int:
        return len(self.nodes) - 1

    def node_path(self, node_id: int) -> tuple[int, ...]:
        out = []
        n = self.nodes[node_id]
        while n.parent is not None:
            out.append(n.token)
            n = self.nodes[n.parent]
        return tuple(reversed(out))

    def child_index(self) -> dict[int, dict[int, int]]:
        idx: dict[int, dict[int, int]] = {n.id: {} for n in self.nodes}
        for n in self.nodes[1:]:
            idx[n.parent][n.token] = n.id
        return idx


class DeviceTree:
    """Device buffers of one bst_expand result (row 0 = root, capacity n_cap+1)."""

    def __init__(self, n_cap: int, device: torch.device | None = None, with_trace: bool = True) -> None:
        dev = device or require_cuda()
        self.n_cap = n_cap
        i32 = dict(dtype=torch.int32, device=dev)
        self.parent = torch.empty(n_cap + 1, **i32)
        self.depth = torch.empty(n_cap + 1, **i32)
        self.token = torch.empty(n_cap + 1, **i32)
        self.rank = torch.empty(n_cap + 1, **i32)
        self.rho = torch.empty(n_cap + 1, dtype=torch.float64, device=dev)
        self.trace = torch.empty(max(n_cap, 1), dtype=torch.float64, device=dev) if with_trace else None
        self.meta = torch.zeros(8, **i32)
        self.surrogate = torch.empty(1, dtype=torch.float64, device=dev)
        self.mask_words = (n_cap + 1 + 31) // 32
        self.anc_mask = torch.empty((n_cap + 1) * self.mask_words, dtype=torch.int32, device=dev)
        self.child_start = torch.empty(n_cap + 2, **i32)
        self.child_list = torch.empty(max(n_cap, 1), **i32)

    def struct(self) -> _lib.Tree:
        p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        return _lib.Tree(p(self.parent), p(self.depth), p(self.token), p(self.rank), p(self.rho), p(self.trace),
                         p(self.meta), p(self.surrogate), p(self.anc_mask), self.mask_words, 0,
                         p(self.child_start), p(self.child_list))


def expand_device(tok: torch.Tensor, prob: torch.Tensor, plan: _lib.Plan, n_cap: int,
                  out: DeviceTree | None = None) -> DeviceTree:
    """Launch K2 on a device lattice; asynchronous (read ``out.meta`` for n_nodes)."""
    gamma, k = tok.shape
    out = out or DeviceTree(n_cap, tok.device)
    need = _lib.lib().bst_expand_workspace(gamma, k, n_cap)
    ws = workspace("expand", need)
    st = out.struct()
    _lib.call("bst_expand", tok.data_ptr(), prob.data_ptr(), gamma, k, plan, n_cap, st, ws.data_ptr(), ws.numel(),
              stream_ptr())
    return out


def _require_nonempty(lattice: CandidateLattice) -> None:
    first = lattice.position_entries(1)
    if not first or first[0][1] <= 0.0:
        raise ValueError("lattice has no positive-probability candidates at position 1")


def tree_from_device(dt: DeviceTree, lattice: CandidateLattice, method: str) -> tuple[DraftTree, np.ndarray]:
    """Download a DeviceTree into the reference DraftTree type (compatibility path)."""
    meta = dt.meta.cpu().numpy()
    n = int(meta[0])
    parent = dt.parent[: n + 1].cpu().numpy()
    depth = dt.depth[: n + 1].cpu().numpy()
    token = dt.token[: n + 1].cpu().numpy()
    rho = dt.rho[: n + 1].cpu().numpy()
    nodes = [TreeNode(0, None, 0, None, 1.0)]
    nodes += [TreeNode(i, int(parent[i]), int(depth[i]), int(token[i]), float(rho[i])) for i in range(1, n + 1)]
    sur = float(dt.surrogate.cpu().item())
    return DraftTree(nodes=tuple(nodes), lattice=lattice, surrogate=sur, method=method, device=dt), meta


def best_first_expand(lattice: CandidateLattice, n_max: int) -> DraftTree:
    """Surrogate-optimal nested tree of min(n_max, reachable) nodes (draft_tree.py:138-155)."""
    if n_max < 1:
        raise ValueError(f"n_max must be >= 1, got {n_max}")
    _require_nonempty(lattice)
    tok, prob = lattice.device_arrays()
    plan = _lib.Plan(policy=_lib.POLICY_FIXED, n_max=n_max)
    dt = expand_device(tok, prob, plan, n_max)
    return tree_from_device(dt, lattice, "best_first")[0]


def beam_expand(lattice: CandidateLattice, width: int, depth: int) -> DraftTree:
    """Rigid width x depth beam baseline (draft_tree.py:158-189)."""
    if width < 1:
        raise ValueError(f"width must be >= 1, got {width}")
    if not 1 <= depth <= lattice.gamma:
        raise ValueError(f"depth must be in [1, {lattice.gamma}], got {depth}")
    _require_nonempty(lattice)
    tok, prob = lattice.device_arrays()
    plan = _lib.Plan(policy=_lib.POLICY_BEAM, width=width, depth=depth)
    dt = expand_device(tok, prob, plan, width * depth)
    return tree_from_device(dt, lattice, "beam")[0]


def surrogate_of(tree: DraftTree) -> float:
    """Fresh sum of path scores, root included (draft_tree.py:192-195)."""
    return math.fsum(n.path_score for n in tree.nodes)


def marginal_gains(tree: DraftTree) -> list[float]:
    if tree.method != "best_first":
        raise ValueError(f"marginal gains are defined for best-first trees, got {tree.method!r}")
    return [n.path_score for n in tree.nodes[1:]]


def build_tree(lattice: CandidateLattice, paths: Sequence[Sequence[int]]) -> DraftTree:
    """Tree from explicit token paths in insertion order (draft_tree.py:204-236; fixture utility)."""
    probs = lattice.source.probs
    nodes = [TreeNode(0, None, 0, None, 1.0)]
    seen: dict[tuple[int, ...], TreeNode] = {(): nodes[0]}
    for raw in paths:
        path = tuple(int(t) for t in raw)
        if not path:
            raise ValueError("paths must be non-empty (the root is implicit)")
        if path in seen:
            raise ValueError(f"duplicate path {path}")
        par = seen.get(path[:-1])
        if par is None:
            raise ValueError(f"path {path} arrives before its parent (tree must stay prefix-closed)")
        if len(path) > lattice.gamma:
            raise ValueError(f"path {path} exceeds block size {lattice.gamma}")
        tok = path[-1]
        if not 0 <= tok < lattice.source.vocab_size:
            raise ValueError(f"token {tok} outside the vocabulary")
        node = TreeNode(len(nodes), par.id, len(path), tok, par.path_score * float(probs[len(path) - 1][tok]))
        nodes.append(node)
        seen[path] = node
    return DraftTree(nodes=tuple(nodes), lattice=lattice, surrogate=math.fsum(n.path_score for n in nodes),
                     method="manual")


def expand_device_plan(tok: torch.Tensor, prob: torch.Tensor, plan_dev: torch.Tensor, policy: int, n_max: int,
                       out: DeviceTree) -> DeviceTree:
    """K2 with the plan read from device memory (re-plannable inside a captured graph)."""
    gamma, k = tok.shape
    need = _lib.lib().bst_expand_workspace(gamma, k, out.n_cap)
    ws = workspace("expand", need)
    st = out.struct()
    _lib.call("bst_expand_dev", tok.data_ptr(), prob.data_ptr(), gamma, k, plan_dev.data_ptr(), policy, n_max,
              out.n_cap, st, ws.data_ptr(), ws.numel(), stream_ptr())
    return out


def expand_device_plan_batch(tok: torch.Tensor, prob: torch.Tensor, lat_stride: int, gamma: int,
                             plan_dev: torch.Tensor, policy: int, n_max: int, trees: list[DeviceTree],
                             trees_dev: torch.Tensor) -> None:
    """K2 for every request in one launch: request r's lattice at row offset r * lat_stride / k,
    plan plan_dev[r], output trees[r] (trees_dev: their bst_tree_t structs on the device)."""
    k = tok.shape[-1]
    n_cap = trees[0].n_cap
    need = _lib.lib().bst_expand_workspace(gamma, k, n_cap) * len(trees)
    ws = workspace("expand_batch", need)
    _lib.call("bst_expand_dev_batch", tok.data_ptr(), prob.data_ptr(), int(lat_stride), gamma, k, plan_dev.data_ptr(),
              policy, n_max, n_cap, trees_dev.data_ptr(), len(trees), ws.data_ptr(), ws.numel(), stream_ptr())


def tree_structs_device(trees: list[DeviceTree], device) -> torch.Tensor:
    """Device array of the trees' bst_tree_t structs (for expand_device_plan_batch)."""
    import ctypes as _C
    structs = [t.struct() for t in trees]  # keep the ctypes objects alive while their bytes are read
    raw = b"".join(_C.string_at(_C.addressof(st), _C.sizeof(_lib.Tree)) for st in structs)
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)
