"""Drafter marginals and the top-K candidate lattice (K1 on the device).

Types mirror ``specplan.lattice`` (lattice.py:24-96); :func:`top_k_truncate`
keeps the reference signature and ordering (prob desc, token asc —
lattice.py:128-142) but runs ``bst_topk_probs`` on the GPU.  The engine path
uses :func:`lattice_from_logits`, which fuses the drafter softmax with the
selection (``bst_topk_logits``) and never leaves the device.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .device import require_cuda, stream_ptr, workspace

ROW_SUM_TOL = 1e-9


@dataclass(frozen=True)
class MarginalBlock:
    """gamma x V fp64 distributions; rows sum to 1 +/- 1e-9 (lattice.py:24-61)."""

    gamma: int
    vocab_size: int
    probs: np.ndarray

    def __post_init__(self) -> None:
        if self.gamma < 1:
            raise ValueError(f"gamma must be >= 1, got {self.gamma}")
        if self.vocab_size < 2:
            raise ValueError(f"vocab_size must be >= 2, got {self.vocab_size}")
        probs = np.asarray(self.probs, dtype=np.float64)
        if probs.shape != (self.gamma, self.vocab_size):
            raise ValueError(f"probs must have shape ({self.gamma}, {self.vocab_size}), got {probs.shape}")
        if np.any(probs < 0.0) or np.any(probs > 1.0):
            raise ValueError("probabilities must lie in [0, 1]")
        sums = probs.sum(axis=1)
        off = np.abs(sums - 1.0) > ROW_SUM_TOL
        if off.any():
            r = int(np.argmax(off))
            raise ValueError(f"row {r} sums to {sums[r]!r}, expected 1 +/- {ROW_SUM_TOL}")
        probs.setflags(write=False)
        object.__setattr__(self, "probs", probs)

    def row(self, position: int) -> np.ndarray:
        if not 1 <= position <= self.gamma:
            raise ValueError(f"position must be in [1, {self.gamma}], got {position}")
        return self.probs[position - 1]


@dataclass(frozen=True)
class CandidateLattice:
    """Per-position top-K (token, prob) entries (lattice.py:64-96).

    ``device`` optionally carries the same lattice as device tensors
    (tok int32[gamma,K], prob float64[gamma,K]) so K2 can consume it without a
    host round trip.
    """

    source: MarginalBlock
    top_k: int
    entries: tuple[tuple[tuple[int, float], ...], ...]
    device: tuple | None = field(default=None, compare=False, repr=False)

    @property
    def gamma(self) -> int:
        return self.source.gamma

    def position_entries(self, position: int) -> tuple[tuple[int, float], ...]:
        return self.entries[position - 1]

    def reachable_size(self) -> int:
        total, layer = 0, 1
        for pos in self.entries:
            layer *= sum(1 for _, p in pos if p > 0.0)
            total += layer
            if layer == 0:
                break
        return total

    def device_arrays(self) -> tuple[torch.Tensor, torch.Tensor]:
        """(tok int32[gamma,K], prob float64[gamma,K]) on the current CUDA device."""
        if self.device is not None:
            return self.device
        dev = require_cuda()
        tok = torch.tensor([[t for t, _ in row] for row in self.entries], dtype=torch.int32, device=dev)
        prob = torch.tensor([[p for _, p in row] for row in self.entries], dtype=torch.float64, device=dev)
        return tok, prob


@dataclass(frozen=True)
class SyntheticPairConfig:
    """Synthetic drafter/target knobs (lattice.py:99-125)."""

    gamma: int
    vocab_size: int
    alignment: float
    concentration: float
    seed: int

    def __post_init__(self) -> None:
        if self.gamma < 1:
            raise ValueError("gamma must be >= 1")
        if self.vocab_size < 2:
            raise ValueError("vocab_size must be >= 2")
        if not 0.0 <= self.alignment <= 1.0:
            raise ValueError(f"alignment must be in [0, 1], got {self.alignment}")
        if not self.concentration > 0.0:
            raise ValueError(f"concentration must be > 0, got {self.concentration}")


def _entries(tok: np.ndarray, prob: np.ndarray) -> tuple:
    return tuple(tuple((int(t), float(p)) for t, p in zip(tr, pr)) for tr, pr in zip(tok, prob))


def topk_device(probs: torch.Tensor, k: int) -> tuple[torch.Tensor, torch.Tensor]:
    """K1 on an fp64 device block: (tok int32[gamma,k], prob float64[gamma,k])."""
    gamma, vocab = probs.shape
    probs = probs.contiguous()
    tok = torch.empty((gamma, k), dtype=torch.int32, device=probs.device)
    prob = torch.empty((gamma, k), dtype=torch.float64, device=probs.device)
    need = _lib.lib().bst_topk_workspace(gamma, vocab, k)
    ws = workspace("topk", need)
    _lib.call("bst_topk_probs", probs.data_ptr(), gamma, vocab, k, tok.data_ptr(), prob.data_ptr(),
              ws.data_ptr(), ws.numel(), stream_ptr())
    return tok, prob


def top_k_truncate(block: MarginalBlock, k: int) -> CandidateLattice:
    """Keep each position's k most probable tokens (prob desc, token asc) — on the GPU."""
    if not 1 <= k <= block.vocab_size:
        raise ValueError(f"k must be in [1, {block.vocab_size}], got {k}")
    dev = require_cuda()
    probs = torch.from_numpy(np.array(block.probs, dtype=np.float64)).to(dev)
    tok, prob = topk_device(probs, k)
    return CandidateLattice(source=block, top_k=k, entries=_entries(tok.cpu().numpy(), prob.cpu().numpy()),
                            device=(tok, prob))


def lattice_from_logits(logits: torch.Tensor, k: int, full_probs: bool = False):
    """Fused K1: drafter logits [gamma, V] (fp32/bf16, device) -> (tok, prob[, probs_full]).

    probs_full (fp64 [gamma, V]) is the MarginalBlock a reference plugin would
    return; the lattice equals top_k_truncate of exactly those rows.
    """
    gamma, vocab = logits.shape
    if not 1 <= k <= vocab:
        raise ValueError(f"k must be in [1, {vocab}], got {k}")
    if logits.stride(1) != 1:
        logits = logits.contiguous()
    dtype = {torch.float32: 0, torch.bfloat16: 1}[logits.dtype]
    tok = torch.empty((gamma, k), dtype=torch.int32, device=logits.device)
    prob = torch.empty((gamma, k), dtype=torch.float64, device=logits.device)
    full = torch.empty((gamma, vocab), dtype=torch.float64, device=logits.device) if full_probs else None
    need = _lib.lib().bst_topk_workspace(gamma, vocab, k)
    ws = workspace("topk", need)
    _lib.call("bst_topk_logits", logits.data_ptr(), dtype, gamma, vocab, logits.stride(0), k, tok.data_ptr(),
              prob.data_ptr(), None if full is None else full.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
    return (tok, prob, full) if full_probs else (tok, prob)


def sample_continuation(block: MarginalBlock, rng: np.random.Generator) -> np.ndarray:
    """One length-gamma draw, row k sampled independently (lattice.py:145-150)."""
    return np.array([rng.choice(block.vocab_size, p=block.probs[i]) for i in range(block.gamma)], dtype=np.int64)


def block_to_text(block: MarginalBlock) -> str:
    out = io.StringIO()
    out.write(f"{block.gamma} {block.vocab_size}\n")
    for row in block.probs:
        out.write(" ".join(repr(float(x)) for x in row) + "\n")
    return out.getvalue()


def block_from_text(text: str) -> MarginalBlock:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise ValueError("empty block text")
    head = lines[0].split()
    if len(head) != 2:
        raise ValueError(f"bad header line: {lines[0]!r}")
    gamma, vocab = int(head[0]), int(head[1])
    if len(lines) != 1 + gamma:
        raise ValueError(f"expected {gamma} rows, found {len(lines) - 1}")
    return MarginalBlock(gamma=gamma, vocab_size=vocab,
                         probs=np.array([[float(x) for x in ln.split()] for ln in lines[1:]], dtype=np.float64))


def block_from_rows(rows: Sequence[Sequence[float]]) -> MarginalBlock:
    probs = np.asarray(rows, dtype=np.float64)
    if probs.ndim != 2:
        raise ValueError("rows must be a 2-D table")
    return MarginalBlock(gamma=probs.shape[0], vocab_size=probs.shape[1], probs=probs)


def topk_partial_into(p, gamma: int, k: int, tok: torch.Tensor, prob: torch.Tensor) -> None:
    """K1 on the drafter LM head's GEMM output (``ops.PartialOut``, rows 0..gamma-1) without a
    reduce pass: bit-identical to ``topk_logits_into`` on the reduced fp32 logits."""
    import ctypes as _C
    vocab = int(p.sched.n_out)
    need = _lib.lib().bst_topk_workspace(gamma, vocab, k)
    ws = workspace("topk", need)
    _lib.call("bst_topk_gemm_partial", p.buf.data_ptr(), _C.byref(p.sched), gamma, vocab, k, tok.data_ptr(),
              prob.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())


def topk_logits_into(logits: torch.Tensor, k: int, tok: torch.Tensor, prob: torch.Tensor,
                     full: torch.Tensor | None = None) -> None:
    """K1 into caller-owned buffers (graph-capturable; workspace must already be sized)."""
    gamma, vocab = logits.shape
    dtype = {torch.float32: 0, torch.bfloat16: 1}[logits.dtype]
    need = _lib.lib().bst_topk_workspace(gamma, vocab, k)
    ws = workspace("topk", need)
    _lib.call("bst_topk_logits", logits.data_ptr(), dtype, gamma, vocab, logits.stride(0), k, tok.data_ptr(),
              prob.data_ptr(), None if full is None else full.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
