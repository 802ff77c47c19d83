"""Config 1 on the CPU oracle alone (no GPU): the tiny target + block-16 drafter decoded
end to end by the oracle model through the reference plugin protocol and the oracle
decode loop (sp/verify_sim.py:426-461).  Greedy tree decode must reproduce the oracle
target's own autoregressive greedy decode — the property the GPU engine
is then held to against this oracle (tests/test_gpu_parity.py)."""

import numpy as np
import pytest
import torch

from oracle import specplan_port as O
from oracle.model_ref import RefModel, RefPlugin, causal_mask


@pytest.fixture(scope="module")
def tiny():
    from paper_2605_29727_b200.engine.config import TINY, DrafterConfig, default_feat_layers
    from paper_2605_29727_b200.engine.weights import DrafterWeights, TargetWeights, rope_inv_freq
    feat = default_feat_layers(TINY.L)
    dcfg = DrafterConfig(layers=1, gamma=16, feat_layers=feat, logit_scale=4.0)
    tw = TargetWeights.random(TINY, 0, "cpu")
    dw = DrafterWeights.random(TINY, dcfg, len(feat), 0, "cpu")
    return TINY, RefModel(TINY, tw, dw, feat, rope_inv_freq(TINY, "cpu"))


@pytest.mark.parametrize("n_fixed", [16, 32])
def test_config1_tree_decode_equals_oracle_ar(tiny, n_fixed):
    cfg, ref = tiny
    prompt = np.random.default_rng(0).integers(0, cfg.V - 1, 64).tolist()
    plugin = RefPlugin(ref, prompt, 16, cfg.V - 1, 8)
    dims = O.Dims(L=cfg.L, h=cfg.h, n_q=cfg.n_q, n_kv=cfg.n_kv, d=cfg.d, h_ffn=cfg.h_ffn, V=cfg.V, bp=2,
                  peak_flops=1e15, bandwidth=1e12)
    recs, toks = O.decode_loop(plugin.drafter_marginals, plugin.next_token, 24, 8, ("fixed", n_fixed, 0, 0), n_fixed,
                               dims, len(prompt) - 1, 0.0, 0.0, 1.0)
    assert all(r["tree_size"] == n_fixed for r in recs)
    seq = list(prompt)
    ar = []
    for _ in range(len(toks)):  # the oracle target's own AR greedy decode
        lg, _ = ref.target(seq, list(range(len(seq))), causal_mask(len(seq)))
        ar.append(int(torch.argmax(lg[-1])))
        seq.append(ar[-1])
    assert list(toks) == ar
    assert sum(r["accepted_len"] for r in recs) == len(toks)
