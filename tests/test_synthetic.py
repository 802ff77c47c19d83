"""The synthetic pair (TargetRule / generate_synthetic_pair, sp/verify_sim.py:56-205,
sp/lattice.py:153-165) reproduces the reference's random streams bit for bit: the
recorded plugin answers of tests/golden/decode.json and the samples / rollouts /
blocks of tests/golden/synthetic.json (both made by the real reference)."""

import numpy as np
import pytest
from codec import dec, load

import paper_2605_29727_b200 as P


def test_decode_golden_plugin_answers():
    for run in load("decode")["runs"]:
        cfg = P.SyntheticPairConfig(gamma=run["gamma"], vocab_size=run["V"], alignment=0.8, concentration=0.1,
                                    seed=run["seed"])
        rule = P.TargetRule.from_config(cfg)
        for prefix, blk in run["blocks"]:
            assert rule.drafter_marginals(prefix).probs.tobytes() == dec(blk).tobytes()
        for prefix, tok in run["choices"]:
            assert rule.next_token(prefix, 0.0) == tok
        assert list(P.ar_decode(P.TargetRule.from_config(cfg), len(run["ar_tokens"]))) == run["ar_tokens"]


def test_synthetic_golden():
    for case in load("synthetic")["cases"]:
        g, v, a, c, s = case["cfg"]
        block, rule = P.generate_synthetic_pair(P.SyntheticPairConfig(gamma=g, vocab_size=v, alignment=a,
                                                                      concentration=c, seed=s))
        assert block.probs.tobytes() == dec(case["block0"]).tobytes()
        for prefix, T, tok in case["samples"]:
            assert rule.next_token(prefix, T) == tok
        for prefix, roll in case["rollouts"]:
            assert list(rule.rollout(prefix, 12)) == roll
        for prefix, blk in case["blocks"]:
            assert np.array_equal(rule.drafter_marginals(prefix).probs, dec(blk))


def test_bad_mode_raises():
    cfg = P.SyntheticPairConfig(gamma=2, vocab_size=4, alignment=0.5, concentration=0.1, seed=0)
    with pytest.raises(ValueError):
        P.TargetRule(cfg, mode="other")
