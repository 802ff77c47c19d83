"""Config 3: the batched multi-request engine must commit the token
streams each request produces alone in B200Engine — batching only changes how rows
are grouped into launches (K3 splits are pinned to 1 in both engines).  K4 results
are row-independent within one kernel; verify chunks above 256 rows run on the
CTA-pair kernel, whose stream-K split points differ from the one-CTA kernel's, so
there the fp32 sums agree to rounding and the streams are equal unless an argmax is
a near-tie (the (3, 100) case runs 303-row chunks and matches exactly)."""

import numpy as np
from oracle import specplan_port as O
import pytest
import torch

pytestmark = pytest.mark.gpu


def _prompts(n, length, V):
    return [np.random.default_rng(100 + r).integers(0, V - 1, length + 7 * r).tolist() for r in range(n)]


def _single_streams(cfg, dcfg, prompts, n_fixed, cycles, max_ctx):
    from paper_2605_29727_b200.engine.decode import B200Engine
    eng = B200Engine(cfg, dcfg, max_ctx=max_ctx, seed=0, n_cap=max(64, n_fixed))
    eng.target.attn_splits = 1
    eng.drafter.attn_splits = 1
    eng.set_policy("fixed", n=n_fixed)
    out = []
    for p in prompts:
        eng.reset(p)
        for _ in range(cycles):
            eng.cycle()
        eng.stream.synchronize()  # the verify graph of the last cycle runs on the engine stream
        # committed stream + per-cycle acceptance surrogate (fp64, from the drafter marginals)
        out.append((eng.tokens(), eng.log_f64[:cycles].cpu().numpy().copy()))
    del eng
    torch.cuda.empty_cache()
    return out


@pytest.mark.parametrize("n_req,n_fixed,graphs", [(5, 12, True), (3, 100, False), (16, 4, True)])
def test_batch_engine_matches_single_requests_tiny(n_req, n_fixed, graphs):
    from paper_2605_29727_b200.engine.batch import BatchEngine
    from paper_2605_29727_b200.engine.config import TINY, DrafterConfig
    dcfg = DrafterConfig(layers=2, gamma=8, logit_scale=4.0)
    prompts = _prompts(n_req, 150, TINY.V)
    cycles = 6
    ref = _single_streams(TINY, dcfg, prompts, n_fixed, cycles, 640)
    be = BatchEngine(TINY, dcfg, n_req=n_req, n_fixed=n_fixed, max_ctx=640, seed=0)
    be.set_attention_splits(1)
    be.use_graphs = graphs
    be.reset(prompts)
    for _ in range(cycles):
        be.cycle()
    assert (be.cycles() == cycles).all()
    for r in range(n_req):
        toks, sur = ref[r]
        assert be.tokens(r) == toks, f"request {r} diverged"
        assert len(toks) >= cycles  # every cycle commits at least the bonus token
        # bit-identical drafts: the batched drafter + K1 + K2 give the same surrogate every cycle
        assert np.array_equal(be.log_f64[r, :cycles].cpu().numpy(), sur)


def test_batch_engine_qwen_shape_two_requests():
    from paper_2605_29727_b200.engine.batch import BatchEngine
    from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig
    dcfg = DrafterConfig(layers=5, gamma=16, logit_scale=6.0)
    prompts = _prompts(2, 300, QWEN3_8B.V)
    ref = _single_streams(QWEN3_8B, dcfg, prompts, 16, 3, 1024)
    be = BatchEngine(QWEN3_8B, dcfg, n_req=2, n_fixed=16, max_ctx=1024, seed=0)
    be.set_attention_splits(1)
    be.reset(prompts)
    for _ in range(3):
        be.cycle()
    for r in range(2):
        assert be.tokens(r) == ref[r][0]
        assert np.array_equal(be.log_f64[r, :3].cpu().numpy(), ref[r][1])


# ------------------------------------------- adaptive: ragged batch-aware verify
def _adaptive(n_max):
    import paper_2605_29727_b200 as P
    from paper_2605_29727_b200.engine.config import QWEN3_8B
    params = QWEN3_8B.cost_params(1649.1e12, 6457.7e9)  # plan with the 8B roofline on the tiny engine
    est = P.VerifyLatencyEstimator(params, variant="static")
    lat = P.CycleLatencies(t_draft=3e-4, t_aux=2e-5, l_ar=est.estimate(1, 1000))
    return params, est, lat


@pytest.mark.parametrize("graphs", [False, True])
def test_ragged_adaptive_single_request_is_run_cycle(graphs):
    """n_req = 1: the batch shift is zero, so the ragged batch engine decodes exactly as the
    single-request engine under Algorithm 1 (tokens, tree sizes, surrogates)."""
    from paper_2605_29727_b200.engine.batch import BatchEngine
    from paper_2605_29727_b200.engine.config import TINY, DrafterConfig
    from paper_2605_29727_b200.engine.decode import B200Engine
    dcfg = DrafterConfig(layers=2, gamma=8, logit_scale=4.0)
    _, est, lat = _adaptive(48)
    prompt = _prompts(1, 150, TINY.V)[0]
    cycles = 8
    eng = B200Engine(TINY, dcfg, max_ctx=640, seed=0, n_cap=48)
    eng.target.attn_splits = eng.drafter.attn_splits = 1
    eng.set_policy("adaptive", estimator=est, latencies=lat, n_max=48)
    eng.reset(prompt)
    for _ in range(cycles):
        eng.cycle()
    want_tok, want_log = eng.tokens(), eng.read_log()
    del eng
    be = BatchEngine(TINY, dcfg, n_req=1, n_fixed=48, max_ctx=640, seed=0)
    be.set_attention_splits(1)
    be.use_graphs = graphs
    be.set_policy("adaptive", estimator=est, latencies=lat)
    be.reset([prompt])
    for _ in range(cycles):
        be.cycle()
    assert be.tokens(0) == want_tok
    log = be.log_i32[0, : cycles * 8].view(cycles, 8).cpu().numpy()
    assert [int(x) for x in log[:, 0]] == [s.tree_size for s in want_log]
    assert [float(x) for x in be.log_f64[0, :cycles].cpu().numpy()] == [s.surrogate for s in want_log]


def test_ragged_adaptive_batch_trees_follow_the_batch_plan():
    """n_req = 4: before every cycle each request's plan is its own curve shifted by the
    other requests' verify flops / bytes at their last tree sizes (weights once) plus their
    surrogates; its tree is the oracle's Algorithm 1 under exactly that plan, bit for bit;
    every committed stream is the target's greedy continuation (the engine's AR decode)."""
    import ctypes as C

    from paper_2605_29727_b200 import _lib
    from paper_2605_29727_b200.engine.batch import BatchEngine
    from paper_2605_29727_b200.engine.config import TINY, DrafterConfig
    from paper_2605_29727_b200.engine.decode import B200Engine
    dcfg = DrafterConfig(layers=2, gamma=8, logit_scale=4.0)
    params, est, lat = _adaptive(48)
    dims = O.Dims(**{k: getattr(params, k) for k in ("L", "h", "n_q", "n_kv", "d", "h_ffn", "V", "bp")},
                  peak_flops=params.peak_flops, bandwidth=params.bandwidth)
    n_req, n_max, G1 = 4, 48, 9
    prompts = _prompts(n_req, 120, TINY.V)
    be = BatchEngine(TINY, dcfg, n_req=n_req, n_fixed=n_max, max_ctx=640, seed=0)
    be.set_attention_splits(1)
    be.use_graphs = False
    be.set_policy("adaptive", estimator=est, latencies=lat)
    be.reset(prompts)
    prev_s = [1] * n_req
    prev_a = [1.0] * n_req
    sizes = []
    for cyc in range(6):
        plans = [_lib.Plan.from_buffer_copy(bytes(be.plan_dev[r].cpu().numpy())) for r in range(n_req)]
        ctx = [int(x) for x in be.contexts()]
        per_f = [O.flops(dims, prev_s[r], ctx[r]) for r in range(n_req)]
        per_b = [O.bytes_moved(dims, prev_s[r], ctx[r]) - O.bytes_moved(dims, 0, 0) for r in range(n_req)]
        with torch.cuda.stream(be.stream):
            be._draft_ragged()
        be.stream.synchronize()
        for r, pl in enumerate(plans):
            assert pl.curve.flops_const == sum(per_f) - per_f[r]
            c = ctx[r]
            cv = O.curve_for(dims, c)
            assert pl.curve.bytes_const + pl.d_bytes_const * c == cv.bytes_const + sum(per_b) - per_b[r]
            assert pl.a_offset == sum(prev_a) - prev_a[r] or abs(pl.a_offset - (sum(prev_a) - prev_a[r])) < 1e-12
            curve = O.Curve(cv.flops_lin, cv.flops_quad, pl.curve.bytes_const + pl.d_bytes_const * c, cv.bytes_lin,
                            cv.bytes_quad, cv.inv_peak, cv.inv_bw, cv.slope, cv.intercept, cv.ratio,
                            flops_const=pl.curve.flops_const)
            tok = be.lat_tok[r * G1 + 1:(r + 1) * G1].cpu().numpy()
            prob = be.lat_prob[r * G1 + 1:(r + 1) * G1].cpu().numpy()
            want = O.controller(tok, prob, n_max, curve, lat.t_draft, lat.t_aux, lat.l_ar, a_offset=pl.a_offset)
            tr = be.trees[r]
            n = int(tr.meta[0].item())
            assert n == want.budget, (cyc, r)
            assert tr.parent[: n + 1].cpu().numpy().tolist() == want.tree.parent.tolist()
            assert tr.token[: n + 1].cpu().numpy().tolist() == want.tree.token.tolist()
            assert np.array(want.trace).tobytes() == tr.trace[: len(want.trace)].cpu().numpy().tobytes()
        total = int(be.row_total.item())
        assert total == sum(int(t.meta[0].item()) + 1 for t in be.trees)
        sizes.append([int(t.meta[0].item()) for t in be.trees])
        with torch.cuda.stream(be.stream):
            be._verify_ragged(-(-total // 64) * 64)
        be.stream.synchronize()
        prev_s = [int(t.meta[0].item()) + 1 for t in be.trees]
        prev_a = [float(t.surrogate.item()) for t in be.trees]
    assert len({s for row in sizes for s in row}) > 1, "trees never differed: the ragged layout was not exercised"
    eng = B200Engine(TINY, dcfg, max_ctx=640, seed=0, n_cap=48)
    for r in range(n_req):
        eng.reset(prompts[r])
        toks = be.tokens(r)
        assert toks == eng.ar_decode(len(toks)), r


def test_ragged_adaptive_precapture_changes_nothing():
    """BatchEngine.precapture (every 64-row verify bucket captured before timing) leaves the
    decode untouched: the same committed streams and per-cycle logs as capturing lazily."""
    from paper_2605_29727_b200.engine.batch import BatchEngine
    from paper_2605_29727_b200.engine.config import TINY, DrafterConfig
    dcfg = DrafterConfig(layers=2, gamma=8, logit_scale=4.0)
    _, est, lat = _adaptive(48)
    prompts = _prompts(3, 100, TINY.V)
    out = []
    for pre in (False, True):
        be = BatchEngine(TINY, dcfg, n_req=3, n_fixed=48, max_ctx=640, seed=0)
        be.set_attention_splits(1)
        be.set_policy("adaptive", estimator=est, latencies=lat)
        be.reset(prompts)
        if pre:
            assert be.precapture() == -(-be.rows_cap // 64)
        for _ in range(6):
            be.cycle()
        out.append(([be.tokens(r) for r in range(3)], be.log_i32[:, :48].cpu().numpy().copy()))
        del be
        torch.cuda.empty_cache()
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
