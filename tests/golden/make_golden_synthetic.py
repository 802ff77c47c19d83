"""Golden outputs of the reference's synthetic pair (TargetRule / generate_synthetic_pair).

    python tests/golden/make_golden_synthetic.py   # writes tests/golden/synthetic.json

Greedy choices and drafter blocks are also pinned by decode.json's recorded plugin
answers; this file adds temperature samples, rollouts, the empty-prefix block of
generate_synthetic_pair and the 'sampled' mode constructor."""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from codec import enc, save  # noqa: E402

REF = os.environ.get("BASTION_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import specplan as sp  # noqa: E402


def main() -> None:
    rng = np.random.default_rng(77)
    cases = []
    for gamma, V, align, conc, seed in ((16, 64, 0.8, 0.1, 1), (5, 300, 0.5, 0.7, 9), (8, 2, 1.0, 0.05, 4)):
        cfg = sp.SyntheticPairConfig(gamma=gamma, vocab_size=V, alignment=align, concentration=conc, seed=seed)
        block, rule = sp.generate_synthetic_pair(cfg)
        prefixes = [tuple(int(x) for x in rng.integers(0, V, n)) for n in (0, 1, 3, 31, 32, 70)]
        samples = [[list(p), T, rule.next_token(p, T)] for p in prefixes for T in (0.0, 0.5, 1.0, 1.7)]
        rollouts = [[list(p), list(rule.rollout(p, 12))] for p in prefixes[:3]]
        blocks = [[list(p), enc(rule.drafter_marginals(p).probs)] for p in prefixes[:4]]
        cases.append({"cfg": [gamma, V, align, conc, seed], "block0": enc(block.probs), "samples": samples,
                      "rollouts": rollouts, "blocks": blocks})
    save("synthetic", {"cases": cases})


if __name__ == "__main__":
    main()
