"""Trees up to the reference's N_max = 1024 (sp/harness.py:49,62; controller.py:96-98).

Verify rows above one K4 launch (256/512 rows) run every GEMM + epilogue in row
chunks and K3 over all rows at once.  The on-device loop's exported fp64 rows and
verify argmax, replayed through the oracle decode loop, must reproduce the engine's
tokens, tree sizes and surrogates bit for bit — at fixed N = 512 and adaptive
N_max = 1024 with trees that exceed 255 nodes.
"""

import numpy as np
import pytest
import torch

from engine_util import _decoy_drafter, _prompt, _replay_check
from oracle import specplan_port as O

pytestmark = pytest.mark.gpu

GAMMA = 8


@pytest.fixture(scope="module")
def eng():
    from paper_2605_29727_b200.engine.config import TINY, DrafterConfig
    from paper_2605_29727_b200.engine.decode import B200Engine
    return B200Engine(TINY, DrafterConfig(layers=2, gamma=GAMMA, logit_scale=2.0), max_ctx=1024, seed=0, n_cap=1024)


def _flat_compute_params():
    """Qwen3-8B profile on a hypothetical machine with 1e6x the compute and 1e3x the
    bandwidth: with a 1 s fixed draft cost (T_DRAFT) the verify curve is flat, so
    Algorithm 1 expands to the budget cap N_max = 1024 (the regime the r1 clamp at 255
    broke)."""
    from paper_2605_29727_b200.engine.config import QWEN3_8B
    return QWEN3_8B.cost_params(1649.1e12 * 1e6, 6457.7e9 * 1e3)


T_DRAFT = 1.0


def _dims(params):
    return O.Dims(**{k: getattr(params, k) for k in ("L", "h", "n_q", "n_kv", "d", "h_ffn", "V", "bp")},
                  peak_flops=params.peak_flops, bandwidth=params.bandwidth)


def test_fixed_512_bit_parity(eng):
    eng.reset(_prompt(80, eng.cfg.V, seed=11))
    eng.export = True
    eng.set_policy("fixed", n=512)
    try:
        _, toks = eng.run(12)
    finally:
        eng.export = False
    assert all(int(e["meta"][0]) == 512 for e in eng.exported)
    params = _flat_compute_params()
    _replay_check(eng, eng.exported, toks, ("fixed", 512, 0, 0), _dims(params), n_max=512)


def test_adaptive_nmax_1024_bit_parity(eng):
    from paper_2605_29727_b200 import CycleLatencies, VerifyLatencyEstimator
    params = _flat_compute_params()
    est = VerifyLatencyEstimator(params, variant="static")
    l_ar = est.estimate(1, 100)
    lat = CycleLatencies(t_draft=T_DRAFT, t_aux=2e-5, l_ar=l_ar)
    eng.reset(_prompt(70, eng.cfg.V, seed=12))
    eng.export = True
    eng.set_policy("adaptive", estimator=est, latencies=lat, n_max=1024)
    try:
        _, toks = eng.run(12)
    finally:
        eng.export = False
    sizes = [int(e["meta"][0]) for e in eng.exported]
    assert max(sizes) > 255, sizes  # the wide-tree path really ran
    recs = _replay_check(eng, eng.exported, toks, ("adaptive", 0, 0, 0), _dims(params), T_DRAFT, 2e-5, l_ar, 1024)
    for e in eng.exported:  # device S_hat traces and stop reasons equal the oracle's
        want = O.controller(e["tok"], e["prob"], 1024, O.curve_for(_dims(params), e["c"]), T_DRAFT, 2e-5, l_ar)
        assert np.array(want.trace).tobytes() == e["trace"].tobytes()
        assert want.budget == int(e["meta"][0])
    assert len(recs) == len(eng.exported)


def test_decode_full_nmax_1024_through_facade(eng):
    """decode_full(engine, SimConfig(n_max=1024), adaptive) — the reference default budget
    cap — runs without clamping and matches the replay through the oracle loop."""
    import paper_2605_29727_b200 as P
    params = _flat_compute_params()
    est = P.VerifyLatencyEstimator(params, variant="static")
    lat = P.CycleLatencies(t_draft=T_DRAFT, t_aux=0.0, l_ar=est.estimate(1, 100))
    prompt = _prompt(60, eng.cfg.V, seed=13)
    sim = P.SimConfig(controller=P.ControllerConfig(n_max=1024, latencies=lat, variant="static",
                                                    context_len=len(prompt) - 1), run_length=10, top_k=eng.top_k)
    eng.reset(prompt)
    eng.export = True
    try:
        records, toks = P.decode_full(eng, sim, P.Policy.adaptive(), est)
    finally:
        eng.export = False
    assert max(r.tree_size for r in records) > 255
    replay = _replay_check(eng, eng.exported, toks, ("adaptive", 0, 0, 0), _dims(params), T_DRAFT, 0.0, lat.l_ar,
                           1024)
    assert [r.tree_size for r in records] == [r["tree_size"] for r in replay]
    assert [r.accepted_len for r in records] == [r["accepted_len"] for r in replay]
    assert [r.surrogate for r in records] == [r["surrogate"] for r in replay]


def test_wide_tree_compaction_preserves_greedy_output(eng):
    """Greedy-output preservation through 600-node trees: chunked verify GEMMs,
    K3 over 601 rows, non-contiguous accepted paths compacted in the KV cache."""
    prompt = _prompt(70, eng.cfg.V, seed=14)
    eng.reset(prompt)
    ar = eng.ar_decode(60)
    eng.reset(prompt)
    eng.set_policy("fixed", n=600)
    eng.draft_override = _decoy_drafter(ar, GAMMA, eng.cfg.V, 2)
    try:
        stats, toks = eng.run(40)
    finally:
        eng.draft_override = None
    assert toks[:40] == ar[:40]
    assert max(s.accepted_len for s in stats) > 3


def test_nmax_over_capacity_raises(eng):
    from paper_2605_29727_b200 import CycleLatencies, VerifyLatencyEstimator
    from paper_2605_29727_b200.engine.config import TINY, DrafterConfig
    from paper_2605_29727_b200.engine.decode import B200Engine
    est = VerifyLatencyEstimator(_flat_compute_params(), variant="static")
    lat = CycleLatencies(t_draft=3e-4, t_aux=0.0, l_ar=1e-3)
    small = B200Engine(TINY, DrafterConfig(layers=1, gamma=GAMMA), max_ctx=256, seed=0, n_cap=64)
    with pytest.raises(ValueError):
        small.set_policy("adaptive", estimator=est, latencies=lat, n_max=1024)
    with pytest.raises(ValueError):
        small.set_policy("fixed", n=65)
    with pytest.raises(ValueError):
        B200Engine(TINY, DrafterConfig(layers=1, gamma=GAMMA), max_ctx=256, n_cap=1025)
    del small
    torch.cuda.empty_cache()


def test_kv_cache_full_raises():
    """a cycle whose verify rows would pass the page range raises instead of
    writing KV out of bounds."""
    from paper_2605_29727_b200.engine.config import TINY, DrafterConfig
    from paper_2605_29727_b200.engine.decode import B200Engine
    e = B200Engine(TINY, DrafterConfig(layers=1, gamma=GAMMA), max_ctx=128, seed=0, n_cap=64)
    e.reset(_prompt(100, TINY.V, seed=15))
    e.set_policy("fixed", n=64)
    with pytest.raises(RuntimeError, match="KV cache full"):
        e.run(400)
