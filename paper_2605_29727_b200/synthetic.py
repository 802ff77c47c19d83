"""The reference's synthetic drafter/target pair, kept for drop-in callers.

``TargetRule`` / ``generate_synthetic_pair`` (sp/verify_sim.py:56-205,
sp/lattice.py:153-165) are the reference's stand-in *model*: a seed-keyed
latent next-token distribution per committed sequence (greedy target = its
argmax) and a linked drafter whose row for a future position is that
distribution, with the true argmax occasionally demoted to a geometric lower
rank.  It is a plugin — a data source on the host — not part of the hot path:
every call a decode makes on it goes through the same GPU planning kernels as
the engine's rows.  The random streams must be bit-identical to the reference
for a caller's runs to reproduce, so the keying (blake2b-128 of
``"{seed}|{tag}|{extra}|"`` + the int64 prefix bytes -> Philox) and the draw
order follow the reference exactly; tests/test_synthetic.py pins the outputs
against tests/golden/synthetic.json made by the reference.
"""

from __future__ import annotations

import hashlib
from typing import Sequence

import numpy as np

from .lattice import MarginalBlock, SyntheticPairConfig

LOG_SPREAD = 1.25       # difficulty jitter (natural-log units) of the latent concentration
WINDOW = 32             # stream positions sharing one difficulty draw
DEMOTE_P = 0.5          # geometric rank of a demoted target token
DEFICIT_DRAWS = 512     # rows behind the mean confidence-deficit normaliser


def _philox(material: bytes) -> np.random.Generator:
    key = int.from_bytes(hashlib.blake2b(material, digest_size=16).digest(), "little")
    return np.random.Generator(np.random.Philox(key=key))


def _softmax_scores(rng: np.random.Generator, vocab: int, temperature: float) -> np.ndarray:
    z = rng.standard_normal(vocab) / max(temperature, 1e-12)
    w = np.exp(z - z.max())
    return w / w.sum()


def _concentration(rng: np.random.Generator, base: float) -> float:
    return base * float(np.exp(rng.uniform(-LOG_SPREAD, LOG_SPREAD)))


def mean_confidence_deficit(cfg: SyntheticPairConfig) -> float:
    """E[1 - max q] of the latent rows for this (vocab, concentration) — seed-free."""
    rng = _philox(f"deficit-calibration|{cfg.vocab_size}|{cfg.concentration!r}".encode())
    acc = []
    for _ in range(DEFICIT_DRAWS):
        temp = _concentration(rng, cfg.concentration)
        acc.append(1.0 - float(_softmax_scores(rng, cfg.vocab_size, temp).max()))
    return max(float(np.mean(acc)), 1e-9)


class TargetRule:
    """Deterministic synthetic target + its linked drafter (the reference plugin protocol:
    ``next_token(prefix, T)`` and ``drafter_marginals(prefix)``)."""

    def __init__(self, cfg: SyntheticPairConfig, mode: str = "greedy-aligned") -> None:
        if mode not in ("greedy-aligned", "sampled"):
            raise ValueError(f"mode must be 'greedy-aligned' or 'sampled', got {mode!r}")
        self.cfg, self.mode = cfg, mode
        self.seed, self.vocab_size, self.gamma, self.alignment = cfg.seed, cfg.vocab_size, cfg.gamma, cfg.alignment
        self._latent: dict[tuple, np.ndarray] = {}
        self._draft_rows: dict[tuple, np.ndarray] = {}
        self._drawn: dict[tuple, int] = {}
        self._deficit = mean_confidence_deficit(cfg)

    @classmethod
    def from_config(cls, cfg: SyntheticPairConfig) -> "TargetRule":
        return cls(cfg)

    def _stream(self, tag: str, prefix: tuple, extra: str = "") -> np.random.Generator:
        head = f"{self.seed}|{tag}|{extra}|".encode()
        return _philox(head + np.asarray(prefix, dtype=np.int64).tobytes())

    def target_distribution(self, prefix: Sequence[int]) -> np.ndarray:
        key = tuple(prefix)
        if key not in self._latent:
            temp = _concentration(self._stream("difficulty", (len(key) // WINDOW,)), self.cfg.concentration)
            d = _softmax_scores(self._stream("dist", key), self.vocab_size, temp)
            d.setflags(write=False)
            self._latent[key] = d
        return self._latent[key]

    def choice(self, prefix: Sequence[int]) -> int:
        return int(np.argmax(self.target_distribution(prefix)))

    def sample(self, prefix: Sequence[int], temperature: float) -> int:
        if temperature <= 0.0:
            return self.choice(prefix)
        key = (tuple(prefix), float(temperature))
        if key not in self._drawn:
            p = self.target_distribution(key[0]) ** (1.0 / temperature)
            p /= p.sum()
            rng = self._stream("sample", key[0], extra=repr(float(temperature)))
            self._drawn[key] = int(rng.choice(self.vocab_size, p=p))
        return self._drawn[key]

    def next_token(self, prefix: Sequence[int], temperature: float) -> int:
        return self.sample(prefix, temperature) if temperature > 0.0 else self.choice(prefix)

    def rollout(self, prefix: Sequence[int], length: int) -> tuple[int, ...]:
        seq, out = list(prefix), []
        for _ in range(length):
            out.append(self.choice(seq))
            seq.append(out[-1])
        return tuple(out)

    def drafter_row(self, prefix: Sequence[int]) -> np.ndarray:
        key = tuple(prefix)
        if key not in self._draft_rows:
            d = self.target_distribution(key)
            rng = self._stream("row", key)
            miss = min(1.0, (1.0 - self.alignment) * (1.0 - float(d.max())) / self._deficit)
            if rng.random() < miss:  # near-miss: swap the argmax with a geometric lower rank
                d = d.copy()
                order = np.argsort(-d, kind="stable")
                r = min(int(rng.geometric(DEMOTE_P)), self.vocab_size - 1)
                d[order[0]], d[order[r]] = d[order[r]], d[order[0]]
                d.setflags(write=False)
            self._draft_rows[key] = d
        return self._draft_rows[key]

    def drafter_marginals(self, prefix: Sequence[int]) -> MarginalBlock:
        key = tuple(prefix)
        cont = self.rollout(key, self.gamma)
        rows = np.stack([self.drafter_row(key + cont[:k]) for k in range(self.gamma)]).astype(np.float64)
        return MarginalBlock(gamma=self.gamma, vocab_size=self.vocab_size, probs=rows)


def generate_synthetic_pair(cfg: SyntheticPairConfig) -> tuple[MarginalBlock, TargetRule]:
    """(drafter block for the empty prefix, the rule) — sp/lattice.py:153-165."""
    rule = TargetRule.from_config(cfg)
    return rule.drafter_marginals(()), rule
