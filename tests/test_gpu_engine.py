"""End-to-end engine tests on the tiny config (C1): GPU forward vs the torch
oracle, planning bit-parity given the GPU-exported logits, and KV compaction
correctness through greedy-output preservation."""

import numpy as np
import pytest
import torch

from oracle import specplan_port as O
from engine_util import _decoy_drafter, _prompt, _replay_check

pytestmark = pytest.mark.gpu

GAMMA = 8


@pytest.fixture(scope="module")
def eng():
    from paper_2605_29727_b200.engine.config import TINY, DrafterConfig
    from paper_2605_29727_b200.engine.decode import B200Engine
    return B200Engine(TINY, DrafterConfig(layers=2, gamma=GAMMA, logit_scale=4.0), max_ctx=640, seed=0, n_cap=64)


@pytest.fixture(scope="module")
def ref(eng):
    from oracle.model_ref import RefModel
    return RefModel(eng.cfg, eng.tw, eng.dw, eng.target.feat_layers, eng.target.inv_freq)


def test_forward_matches_oracle(eng, ref):
    from oracle.model_ref import causal_mask, verify_mask
    prompt = _prompt(300, eng.cfg.V)  # > 256: exercises chunked prefill
    eng.reset(prompt)
    eng.export = True
    eng.set_policy("fixed", n=40)
    eng.cycle()
    eng.export = False
    ex = eng.exported[-1]
    c = len(prompt) - 1
    logits_p, feat = ref.target(prompt[:-1], list(range(c)), causal_mask(c))
    # drafter block vs oracle (probabilities, fp64 rows exported by K1)
    dl = ref.drafter(feat, c, prompt[-1], GAMMA, eng.cfg.V - 1).double()
    p_ref = torch.softmax(dl, -1).numpy()
    assert np.abs(ex["probs"] - p_ref).max() < 2e-2
    # verify logits/argmax vs oracle on the same tree
    parent, depth, token = ex["parent"], ex["depth"], ex["token"]
    anc = torch.from_numpy(O.ancestor_bits(parent))
    toks = prompt[:-1] + [prompt[-1]] + token[1:].tolist()
    pos = list(range(c)) + [c + int(d) for d in depth]
    lv, _ = ref.target(toks, pos, verify_mask(c, anc))
    lv = lv[c:]
    top2 = lv.topk(2, dim=-1).values
    clear = (top2[:, 0] - top2[:, 1]) > 1e-2
    am_ref = lv.argmax(-1).numpy()
    assert clear.float().mean() > 0.8
    assert (ex["argmax"][clear.numpy()] == am_ref[clear.numpy()]).all()


def test_planning_bit_parity_fixed(eng):
    eng.reset(_prompt(50, eng.cfg.V, seed=1))
    eng.export = True
    eng.set_policy("fixed", n=24)
    _, toks = eng.run(30)
    eng.export = False
    dims = O.Dims(L=2, h=256, n_q=4, n_kv=2, d=128, h_ffn=512, V=1024, bp=2, peak_flops=1e15, bandwidth=1e12)
    _replay_check(eng, eng.exported, toks, ("fixed", 24, 0, 0), dims)


def test_planning_bit_parity_adaptive(eng):
    from paper_2605_29727_b200 import CostModelParams, CycleLatencies, VerifyLatencyEstimator
    from paper_2605_29727_b200.engine.config import QWEN3_8B
    params = QWEN3_8B.cost_params(1649.1e12, 6457.7e9)  # plan with the 8B roofline on the tiny engine
    est = VerifyLatencyEstimator(params, variant="static")
    l_ar = est.estimate(1, 1000)
    lat = CycleLatencies(t_draft=3e-4, t_aux=2e-5, l_ar=l_ar)
    eng.reset(_prompt(60, eng.cfg.V, seed=2))
    eng.export = True
    eng.set_policy("adaptive", estimator=est, latencies=lat, n_max=64)
    _, toks = eng.run(30)
    eng.export = False
    dims = O.Dims(**{k: getattr(params, k) for k in ("L", "h", "n_q", "n_kv", "d", "h_ffn", "V", "bp")},
                  peak_flops=params.peak_flops, bandwidth=params.bandwidth)
    recs = _replay_check(eng, eng.exported, toks, ("adaptive", 0, 0, 0), dims, 3e-4, 2e-5, l_ar, 64)
    assert all(r["tree_size"] >= 1 for r in recs)
    for e in eng.exported:  # the device S_hat trace equals the oracle's
        c = e["c"]
        want = O.controller(e["tok"], e["prob"], 64, O.curve_for(dims, c), 3e-4, 2e-5, l_ar)
        assert np.array(want.trace).tobytes() == e["trace"].tobytes()
        assert want.budget == int(e["meta"][0])


@pytest.mark.parametrize("graphs", [False, True])
def test_kv_compaction_preserves_greedy_output(eng, graphs):
    """Greedy output preservation: tree decode with acceptance == target AR decode."""
    prompt = _prompt(70, eng.cfg.V, seed=3)
    eng.reset(prompt)
    ar = eng.ar_decode(80)
    eng.reset(prompt)
    eng.set_policy("fixed", n=48)
    eng.draft_override = _decoy_drafter(ar, GAMMA, eng.cfg.V, 0)
    eng.use_graphs = graphs
    try:
        stats, toks = eng.run(60)
    finally:
        eng.draft_override = None
        eng.use_graphs = True
    assert toks[:60] == ar[:60]
    accepted = [s.accepted_len for s in stats]
    assert max(accepted) > 3 and np.mean(accepted) > 2.0  # compaction really ran
    # non-contiguous paths happened (moves, not just identity)
    assert len(stats) < 40


def test_graph_and_eager_cycles_agree(eng):
    prompt = _prompt(40, eng.cfg.V, seed=4)
    eng.set_policy("fixed", n=32)
    out = []
    for graphs in (False, True):
        eng.use_graphs = graphs
        eng.reset(prompt)
        out.append(eng.run(20)[1])
    eng.use_graphs = True
    assert out[0] == out[1]


def test_sampled_tree_decode_preserves_ar_samples(eng):
    """T > 0 exact-match verification (verify_sim.py:111-126): with Gumbel noise keyed by
    (seed, absolute position), tree decode with compaction == the sampled AR decode."""
    prompt = _prompt(70, eng.cfg.V, seed=5)
    eng.set_temperature(0.8, 11)
    try:
        eng.reset(prompt)
        ar = eng.ar_decode(60)
        eng.reset(prompt)
        eng.set_policy("fixed", n=48)
        eng.draft_override = _decoy_drafter(ar, GAMMA, eng.cfg.V, 1)
        stats, toks = eng.run(45)
    finally:
        eng.draft_override = None
        eng.set_temperature(0.0, 0)
    assert toks[:45] == ar[:45]
    assert max(s.accepted_len for s in stats) > 3
    eng.reset(prompt)
    assert eng.ar_decode(60) != ar  # the sampling path really ran


class _Plugin:
    """The reference plugin protocol only (no engine_decode): forces the façade's general loop."""

    def __init__(self, e):
        self.e = e

    def drafter_marginals(self, prefix):
        return self.e.drafter_marginals(prefix)

    def tree_argmax(self, tree, prefix):
        return self.e.tree_argmax(tree, prefix)

    def tree_sample(self, tree, prefix, temperature):
        return self.e.tree_sample(tree, prefix, temperature)

    def next_token(self, prefix, temperature):
        return self.e.next_token(prefix, temperature)


@pytest.mark.parametrize("temperature", [0.0, 0.9])
def test_general_facade_loop_matches_engine_fast_path(eng, temperature):
    import paper_2605_29727_b200 as P
    prompt = _prompt(50, eng.cfg.V, seed=6)
    est = P.VerifyLatencyEstimator(eng.cfg.cost_params(1.6e15, 6.5e12))
    lat = P.CycleLatencies(t_draft=3e-4, t_aux=0.0, l_ar=1e-3)
    sim = P.SimConfig(controller=P.ControllerConfig(n_max=32, latencies=lat, variant="static",
                                                    context_len=len(prompt) - 1), run_length=40, top_k=eng.top_k,
                      temperature=temperature)
    eng.set_temperature(0.0, 3)
    try:
        eng.reset(prompt)
        rec_fast, tok_fast = P.decode_full(eng, sim, P.Policy.fixed(24), est)
        eng.reset(prompt)
        rec_gen, tok_gen = P.decode_full(_Plugin(eng), sim, P.Policy.fixed(24), est)
        assert tuple(tok_gen) == tuple(tok_fast)
        assert [r.accepted_len for r in rec_gen] == [r.accepted_len for r in rec_fast]
        assert [r.tree_size for r in rec_gen] == [r.tree_size for r in rec_fast]
        # the reference's AR baseline through next_token (lazy commit of each token)
        eng.reset(prompt)
        ar = P.ar_decode(_Plugin(eng), 12, temperature)
        eng.set_temperature(temperature, 3)
        eng.reset(prompt)
        assert list(ar) == eng.ar_decode(12)
    finally:
        eng.set_temperature(0.0, 0)


def test_beam_policy_runs_through_the_plugin_protocol(eng):
    """Policies the on-device loop does not implement (beam, greedy chain) run the façade's
    reference loop with the engine as plugin; the committed stream is the engine's own."""
    import paper_2605_29727_b200 as P
    prompt = _prompt(40, eng.cfg.V, seed=8)
    est = P.VerifyLatencyEstimator(eng.cfg.cost_params(1.6e15, 6.5e12))
    lat = P.CycleLatencies(t_draft=3e-4, t_aux=0.0, l_ar=1e-3)
    sim = P.SimConfig(controller=P.ControllerConfig(n_max=32, latencies=lat, variant="static",
                                                    context_len=len(prompt) - 1), run_length=20, top_k=eng.top_k)
    eng.set_temperature(0.0, 0)
    for pol in (P.Policy.beam(2, 4), P.Policy.greedy_chain()):
        eng.reset(prompt)
        recs, toks = P.decode_full(eng, sim, pol, est)
        assert len(toks) >= 20 and all(r.tree_size >= 1 for r in recs)
        assert tuple(eng.tokens())[: len(toks) - recs[-1].accepted_len] == tuple(toks)[: len(toks) - recs[-1].accepted_len]


def test_ema_observe_replans_every_cycle(eng):
    """K7 wiring (sp/cost_model.py:184-189,266-270): every measured verify time goes through
    ``observe``; the EMA ratio follows ``ema_update`` bit for bit, and each cycle's tree is
    Algorithm 1 at the ratio its plan was uploaded with (the previous cycle's observation
    is applied after the next draft: one cycle of lag, engine_decode)."""
    import paper_2605_29727_b200 as P
    from paper_2605_29727_b200.engine.config import QWEN3_8B
    params = QWEN3_8B.cost_params(1649.1e12, 6457.7e9)
    est = P.VerifyLatencyEstimator(params, variant="ema", bias=P.EmaBias(ratio_bias=1.0, alpha=0.1))
    l_ar = est.estimate(1, 1000)
    lat = P.CycleLatencies(t_draft=3e-4, t_aux=2e-5, l_ar=l_ar)
    prompt = _prompt(60, eng.cfg.V, seed=9)
    sim = P.SimConfig(controller=P.ControllerConfig(n_max=64, latencies=lat, variant="ema",
                                                    context_len=len(prompt) - 1), run_length=24, top_k=eng.top_k)
    plan_ratios, observed = [], []
    orig_set, orig_obs = eng.set_policy, est.observe

    def set_policy(kind, n=0, estimator=None, latencies=None, n_max=None):
        plan_ratios.append(estimator.bias.ratio_bias)
        return orig_set(kind, n=n, estimator=estimator, latencies=latencies, n_max=n_max)

    def observe(s, c, obs):
        before = est.bias.ratio_bias
        orig_obs(s, c, obs)
        observed.append((s, c, obs, before, est.bias.ratio_bias))
    eng.set_policy, est.observe = set_policy, observe
    eng.reset(prompt)
    eng.export = True
    try:
        records, toks = P.decode_full(eng, sim, P.Policy.adaptive(), est)
    finally:
        eng.export = False
        del eng.set_policy
    dims = O.Dims(**{k: getattr(params, k) for k in ("L", "h", "n_q", "n_kv", "d", "h_ffn", "V", "bp")},
                  peak_flops=params.peak_flops, bandwidth=params.bandwidth)
    assert len(observed) >= len(records) - 1 and len(records) >= 3
    for s, c, obs, before, after in observed:  # ema_update arithmetic, bit for bit
        assert after == O.ema_step(before, 0.1, O.roofline(dims, s, c), obs)
    assert len({r for r in plan_ratios}) > 1, "the plan never changed"
    for k, e in enumerate(eng.exported):
        ratio = plan_ratios[max(0, k - 1)]
        want = O.controller(e["tok"], e["prob"], 64, O.curve_for(dims, e["c"], "ema", ratio=ratio), 3e-4, 2e-5, l_ar)
        assert want.budget == int(e["meta"][0]), k
        assert np.array(want.trace).tobytes() == e["trace"].tobytes(), k
