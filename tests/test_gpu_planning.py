"""GPU parity of the planning kernels (K1 top-K, K2 expand, K6 accept, linearize)
against the reference golden vectors and the CPU oracle — bit-exact."""

import numpy as np
import pytest
import torch

from codec import dec, load, unhex
from oracle import specplan_port as O

pytestmark = pytest.mark.gpu

STOP = {"first-decrease": 0, "frontier-exhausted": 1, "budget-cap": 2}


@pytest.fixture(scope="module")
def P():
    import paper_2605_29727_b200 as P
    return P


@pytest.fixture(scope="module")
def lattice_cases():
    return load("lattice_trees")["cases"]


def _lat(P, case):
    probs = dec(case["probs"])
    block = P.MarginalBlock(gamma=probs.shape[0], vocab_size=probs.shape[1], probs=probs)
    tok, prob = dec(case["tok"]), dec(case["prob"])
    entries = tuple(tuple((int(t), float(p)) for t, p in zip(tr, pr)) for tr, pr in zip(tok, prob))
    return P.CandidateLattice(source=block, top_k=case["k"], entries=entries)


def _tree_equal(tree, want):
    parent = [-1 if n.parent is None else n.parent for n in tree.nodes]
    token = [-1 if n.token is None else n.token for n in tree.nodes]
    depth = [n.depth for n in tree.nodes]
    rho = np.array([n.path_score for n in tree.nodes])
    assert parent == dec(want["parent"]).tolist()
    assert depth == dec(want["depth"]).tolist()
    assert token == dec(want["token"]).tolist()
    assert rho.tobytes() == dec(want["rho"]).tobytes()


# ---------------------------------------------------------------- K1
def test_k1_top_k_truncate_golden(P, lattice_cases):
    for case in lattice_cases:
        probs = dec(case["probs"])
        block = P.MarginalBlock(gamma=probs.shape[0], vocab_size=probs.shape[1], probs=probs)
        lat = P.top_k_truncate(block, case["k"])
        tok = np.array([[t for t, _ in r] for r in lat.entries])
        prob = np.array([[p for _, p in r] for r in lat.entries])
        assert tok.tolist() == dec(case["tok"]).tolist(), case["name"]
        assert prob.tobytes() == dec(case["prob"]).tobytes(), case["name"]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("scale", [1.0, 6.0, 10.0])
def test_k1_logits_full_vocab_matches_oracle(P, dtype, scale):
    from paper_2605_29727_b200.lattice import lattice_from_logits
    g = torch.Generator(device="cuda").manual_seed(int(scale * 7))
    logits = (torch.randn(16, 151936, device="cuda", generator=g) * scale).to(dtype)
    tok, prob, full = lattice_from_logits(logits, 8, full_probs=True)
    full_h = full.cpu().numpy()
    # rows are valid MarginalBlock rows (sum 1 +/- 1e-9)
    P.MarginalBlock(gamma=16, vocab_size=151936, probs=full_h)
    otok, oprob = O.topk_rows(full_h, 8)  # reference ordering on the GPU-exported fp64 rows
    assert tok.cpu().numpy().tolist() == otok.tolist()
    assert prob.cpu().numpy().tobytes() == oprob.tobytes()
    # probabilities agree with a plain fp64 softmax of the same logits (1e-12 rel)
    ref = O.softmax_rows_f64(logits.float().cpu().numpy())
    np.testing.assert_allclose(full_h, ref, rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("vocab,scale", [(151936, 6.0), (151936, 30.0), (1024, 6.0)])
def test_k1_on_gemm_partials_equals_reduced_logits(P, vocab, scale):
    """bst_topk_gemm_partial (K1 reading the LM head's stream-K partial slots, the engine's
    draft path) is bit-identical to K1 on the reduced fp32 logits (the export path)."""
    from paper_2605_29727_b200 import ops
    from paper_2605_29727_b200.lattice import topk_logits_into, topk_partial_into
    g = torch.Generator(device="cuda").manual_seed(vocab + int(scale))
    w = (torch.randn(vocab, 4096, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    x = (torch.randn(16, 4096, device="cuda", generator=g) * scale).to(torch.bfloat16)
    part = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    p = ops.gemm_partial(x, w, out=part)
    logits = torch.empty(16, vocab, device="cuda")
    from paper_2605_29727_b200.engine.forward import _reduce_into
    _reduce_into(p, logits)
    tok_a = torch.empty(16, 8, dtype=torch.int32, device="cuda")
    prob_a = torch.empty(16, 8, dtype=torch.float64, device="cuda")
    tok_b, prob_b = torch.empty_like(tok_a), torch.empty_like(prob_a)
    topk_logits_into(logits, 8, tok_a, prob_a)
    topk_partial_into(p, 16, 8, tok_b, prob_b)
    torch.cuda.synchronize()
    assert torch.equal(tok_a, tok_b)
    assert prob_a.cpu().numpy().tobytes() == prob_b.cpu().numpy().tobytes()


def test_k1_bf16_ties_token_order(P):
    from paper_2605_29727_b200.lattice import lattice_from_logits
    # many exactly equal logits: order must be token ascending among ties
    logits = torch.zeros(4, 5000, device="cuda", dtype=torch.bfloat16)
    logits[:, 4000:4010] = 2.0
    logits[1, 17] = 2.0
    tok, _ = lattice_from_logits(logits, 8)
    assert tok[0].tolist() == list(range(4000, 4008))
    assert tok[1].tolist() == [17] + list(range(4000, 4007))


# ---------------------------------------------------------------- K2
def test_k2_best_first_golden(P, lattice_cases):
    n = 0
    for case in lattice_cases:
        if not case["best_first"]:
            continue
        lat = _lat(P, case)
        for bf in case["best_first"]:
            tree = P.best_first_expand(lat, bf["n_max"])
            _tree_equal(tree, bf["nodes"])
            assert tree.surrogate == unhex(bf["surrogate"])
            n += 1
    assert n > 100


def test_k2_beam_golden(P, lattice_cases):
    for case in lattice_cases:
        if not case["beam"]:
            continue
        lat = _lat(P, case)
        for bm in case["beam"]:
            if bm["width"] * lat.top_k > 8192:
                continue
            tree = P.beam_expand(lat, bm["width"], bm["depth"])
            _tree_equal(tree, bm["nodes"])
            assert tree.surrogate == unhex(bm["surrogate"])


def test_k2_run_cycle_golden(P, lattice_cases):
    g = load("controller")
    lats = {c["name"]: c for c in lattice_cases}
    prof = {k: P.CostModelParams(**{x: v[x] for x in ("L", "h", "n_q", "n_kv", "d", "h_ffn", "V", "bp")},
                                 peak_flops=unhex(v["peak_flops"]), bandwidth=unhex(v["bandwidth"]))
            for k, v in g["profiles"].items()}
    for run in g["runs"]:
        lat = _lat(P, lats[run["lattice"]])
        fit = P.CalibrationFit(unhex(run["slope"]), unhex(run["intercept"]), 0.0, 0.0) if run["slope"] else None
        bias = P.EmaBias(unhex(run["ratio"])) if run["ratio"] else None
        if run["variant"] == "static" and fit is not None and fit.slope == 1.0 and fit.intercept == 0.0:
            fit = None
        est = P.VerifyLatencyEstimator(prof[run["profile"]], variant=run["variant"], fit=fit, bias=bias)
        cfg = P.ControllerConfig(n_max=run["n_max"], latencies=P.CycleLatencies(
            unhex(run["t_draft"]), unhex(run["t_aux"]), unhex(run["l_ar"])), variant=run["variant"],
            context_len=run["c"])
        d = P.run_cycle(lat, cfg, est)
        assert d.budget == run["budget"], run
        assert d.stop_reason == run["stop"]
        assert np.array(d.s_hat_trace).tobytes() == dec(run["trace"]).tobytes()
        _tree_equal(d.tree, run["nodes"])
        assert d.tree.surrogate == unhex(run["surrogate"])


@pytest.mark.parametrize("algo", [1, 2])
@pytest.mark.parametrize("seed", range(6))
def test_k2_sort_and_heap_paths_match_oracle_full_shape(P, algo, seed):
    """gamma=16, K=8, bf16 drafter logits of V=151936 (heavy exact ties), N up to 1024."""
    from paper_2605_29727_b200 import _lib
    from paper_2605_29727_b200.draft_tree import expand_device
    from paper_2605_29727_b200.lattice import lattice_from_logits
    g = torch.Generator(device="cuda").manual_seed(100 + seed)
    scale = [3.0, 6.0, 8.0, 10.0, 1.0, 0.3][seed]
    logits = (torch.randn(16, 151936, device="cuda", generator=g) * scale).to(torch.bfloat16)
    tok, prob = lattice_from_logits(logits, 8)
    tok_h, prob_h = tok.cpu().numpy(), prob.cpu().numpy()
    for n_max in (64, 256, 1024):
        dt = expand_device(tok, prob, _lib.Plan(policy=_lib.POLICY_FIXED, n_max=n_max, algo=algo), n_max)
        want = O.best_first(tok_h, prob_h, n_max)
        n = int(dt.meta[0].item())
        assert n == want.size
        assert dt.parent[: n + 1].cpu().numpy().tolist() == want.parent.tolist()
        assert dt.token[: n + 1].cpu().numpy().tolist() == want.token.tolist()
        assert dt.depth[: n + 1].cpu().numpy().tolist() == want.depth.tolist()
        assert dt.rank[1: n + 1].cpu().numpy().tolist() == want.rank[1:].tolist()
        assert dt.rho[: n + 1].cpu().numpy().tobytes() == want.rho.tobytes()
        assert dt.surrogate.item() == want.surrogate
    # adaptive at Qwen3-8B / B200 shape
    dims = O.Dims(L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288, V=151936, bp=2, peak_flops=1649.1e12,
                  bandwidth=6457.7e9)
    for c in (2048, 32768):
        cv = O.curve_for(dims, c)
        l_ar = O.roofline(dims, 1, c)
        want = O.controller(tok_h, prob_h, 1024, cv, 3e-4, 0.0, l_ar)
        plan = _lib.Plan(policy=_lib.POLICY_ADAPTIVE, n_max=1024, algo=algo,
                         curve=_lib.Curve(cv.flops_lin, cv.flops_quad, cv.bytes_const, cv.bytes_lin, cv.bytes_quad,
                                          cv.inv_peak, cv.inv_bw, cv.slope, cv.intercept, cv.ratio),
                         fixed_cost=3e-4 + 0.0, l_ar=l_ar)
        dt = expand_device(tok, prob, plan, 1024)
        meta = dt.meta.cpu().numpy()
        assert int(meta[0]) == want.budget
        assert int(meta[2]) == want.stop
        assert dt.trace[: int(meta[1])].cpu().numpy().tobytes() == np.array(want.trace).tobytes()
        assert dt.surrogate.item() == want.tree.surrogate


@pytest.mark.parametrize("fixed_cost", [3e-4, 3e-3, 3e-2, 1.0, 1e3])
def test_k2_adaptive_stop_beyond_first_pass(P, fixed_cost):
    """Adaptive K2 plans the best 256 nodes first and enumerates up to n_max only when S_hat
    has not decreased by then; large fixed costs push the stop past 256 nodes (or to the
    budget cap), and the tree, trace and stop must still equal the oracle's Algorithm 1."""
    from paper_2605_29727_b200 import _lib
    from paper_2605_29727_b200.draft_tree import expand_device
    from paper_2605_29727_b200.lattice import lattice_from_logits
    g = torch.Generator(device="cuda").manual_seed(7)
    logits = torch.randn(16, 151936, device="cuda", generator=g) * 0.1
    for r in range(16):  # three dominant candidates per position: rho decays slowly, trees grow large
        logits[r, 1000 + 7 * r: 1003 + 7 * r] = torch.tensor([10.0, 9.9, 9.8], device="cuda")
    tok, prob = lattice_from_logits(logits, 8)
    tok_h, prob_h = tok.cpu().numpy(), prob.cpu().numpy()
    dims = O.Dims(L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288, V=151936, bp=2, peak_flops=1649.1e12,
                  bandwidth=6457.7e9)
    cv = O.curve_for(dims, 2048)
    l_ar = O.roofline(dims, 1, 2048)
    want = O.controller(tok_h, prob_h, 1024, cv, fixed_cost, 0.0, l_ar)
    plan = _lib.Plan(policy=_lib.POLICY_ADAPTIVE, n_max=1024,
                     curve=_lib.Curve(cv.flops_lin, cv.flops_quad, cv.bytes_const, cv.bytes_lin, cv.bytes_quad,
                                      cv.inv_peak, cv.inv_bw, cv.slope, cv.intercept, cv.ratio),
                     fixed_cost=fixed_cost, l_ar=l_ar)
    dt = expand_device(tok, prob, plan, 1024)
    meta = dt.meta.cpu().numpy()
    n = int(meta[0])
    assert n == want.budget
    assert int(meta[2]) == want.stop
    assert dt.trace[: int(meta[1])].cpu().numpy().tobytes() == np.array(want.trace).tobytes()
    assert dt.parent[: n + 1].cpu().numpy().tolist() == want.tree.parent.tolist()
    assert dt.token[: n + 1].cpu().numpy().tolist() == want.tree.token.tolist()
    assert dt.surrogate.item() == want.tree.surrogate
    _report_budget = (fixed_cost, n, int(meta[1]), int(meta[2]))
    print("adaptive budget", _report_budget)


def test_k2_ancestor_mask_and_csr(P):
    from paper_2605_29727_b200 import _lib
    from paper_2605_29727_b200.draft_tree import expand_device
    from paper_2605_29727_b200.lattice import lattice_from_logits
    logits = (torch.randn(16, 4096, device="cuda") * 5).to(torch.bfloat16)
    tok, prob = lattice_from_logits(logits, 8)
    dt = expand_device(tok, prob, _lib.Plan(policy=_lib.POLICY_FIXED, n_max=300), 300)
    n = int(dt.meta[0].item())
    parent = dt.parent[: n + 1].cpu().numpy()
    want = O.ancestor_bits(parent)
    words = dt.mask_words
    m = dt.anc_mask.view(-1)[: (n + 1) * words].cpu().numpy().view(np.uint32).reshape(n + 1, words)
    bits = np.unpackbits(m.view(np.uint8), bitorder="little").reshape(n + 1, words * 32)[:, : n + 1].astype(bool)
    np.testing.assert_array_equal(bits, want)
    cs = dt.child_start[: n + 2].cpu().numpy()
    cl = dt.child_list[:n].cpu().numpy()
    for i in range(n + 1):
        kids = sorted(cl[cs[i]: cs[i + 1]].tolist())
        assert kids == [j for j in range(1, n + 1) if parent[j] == i]


# ---------------------------------------------------------------- K6 + linearize
def test_linearize_golden(P, lattice_cases):
    for case in load("linearize")["cases"]:
        nodes = case["nodes"]
        parent, depth, token = dec(nodes["parent"]), dec(nodes["depth"]), dec(nodes["token"])
        rho = dec(nodes["rho"])
        tn = [P.TreeNode(0, None, 0, None, 1.0)] + [
            P.TreeNode(i, int(parent[i]), int(depth[i]), int(token[i]), float(rho[i])) for i in range(1, len(parent))]
        lat = _lat(P, lattice_cases[0])
        tree = P.DraftTree(nodes=tuple(tn), lattice=lat, surrogate=1.0, method="manual")
        lin = P.linearize(tree, case["prefix_len"])
        want = np.unpackbits(dec(case["mask"]), axis=1)[:, : case["mask_shape"][1]].astype(bool)
        np.testing.assert_array_equal(lin.mask, want)
        assert list(lin.position_ids) == case["position_ids"]
        assert list(lin.parents) == case["parents"]


def test_k6_accept_matches_oracle(P):
    from paper_2605_29727_b200 import _lib
    from paper_2605_29727_b200.draft_tree import expand_device
    from paper_2605_29727_b200.lattice import lattice_from_logits
    from paper_2605_29727_b200.verify_sim import accept_device
    rng = np.random.default_rng(0)
    for trial in range(20):
        logits = (torch.randn(16, 2048, device="cuda") * 6).to(torch.bfloat16)
        tok, prob = lattice_from_logits(logits, 8)
        dt = expand_device(tok, prob, _lib.Plan(policy=_lib.POLICY_FIXED, n_max=256), 256)
        n = int(dt.meta[0].item())
        parent = dt.parent[: n + 1].cpu().numpy()
        token = dt.token[: n + 1].cpu().numpy()
        # target argmax: follow a random root path for a random number of steps, then diverge
        am = rng.integers(0, 2048, n + 1).astype(np.int32)
        cur = 0
        for _ in range(int(rng.integers(0, 17))):
            kids = [j for j in range(1, n + 1) if parent[j] == cur]
            if not kids:
                break
            j = int(rng.choice(kids))
            am[cur] = token[j]
            cur = j
        path, committed, meta = accept_device(dt.token, dt.child_start, dt.child_list,
                                              torch.from_numpy(am).cuda(), 17)
        want_path, want_bonus = O.accept_from_argmax(parent, token, am)
        m = meta.cpu().numpy()
        assert int(m[0]) == len(want_path) and int(m[1]) == want_bonus
        assert path[: len(want_path)].cpu().numpy().tolist() == want_path
        assert committed[: len(want_path)].cpu().numpy().tolist() == O.committed_tokens(want_path, token, want_bonus)


class ReplayPlugin:
    """Replays the reference plugin answers recorded in tests/golden/decode.json."""

    def __init__(self, P, run):
        self.P = P
        self.blocks = {tuple(k): dec(v) for k, v in run["blocks"]}
        self.choices = {tuple(k): v for k, v in run["choices"]}

    def drafter_marginals(self, prefix):
        p = self.blocks[tuple(prefix)]
        return self.P.MarginalBlock(gamma=p.shape[0], vocab_size=p.shape[1], probs=p)

    def next_token(self, prefix, temperature):
        return self.choices[tuple(prefix)]


class ReplayTreePlugin(ReplayPlugin):
    """Same answers, but scored per tree (one 'verify pass') so the K6 device walk runs."""

    def tree_argmax(self, tree, prefix):
        am = []
        for node in tree.nodes:
            am.append(self.choices.get(tuple(prefix) + tree.node_path(node.id), -1))
        return torch.tensor(am, dtype=torch.int32, device="cuda")


def _target_rule(P, run):
    """The synthetic pair itself (paper_2605_29727_b200.TargetRule), not a replay."""
    return P.TargetRule.from_config(P.SyntheticPairConfig(gamma=run["gamma"], vocab_size=run["V"], alignment=0.8,
                                                          concentration=0.1, seed=run["seed"]))


@pytest.mark.parametrize("plugin_cls", [ReplayPlugin, ReplayTreePlugin, _target_rule])
def test_decode_loop_golden(P, plugin_cls):
    g = load("decode")
    prof = load("controller")["profiles"]["crossover"]
    params = P.CostModelParams(**{x: prof[x] for x in ("L", "h", "n_q", "n_kv", "d", "h_ffn", "V", "bp")},
                               peak_flops=unhex(prof["peak_flops"]), bandwidth=unhex(prof["bandwidth"]))
    for run in g["runs"]:
        plugin = plugin_cls(P, run)
        est = P.VerifyLatencyEstimator(params, variant="static")
        lat = P.CycleLatencies(unhex(run["t_draft"]), unhex(run["t_aux"]), unhex(run["l_ar"]))
        cfg = P.SimConfig(controller=P.ControllerConfig(n_max=run["n_max"], latencies=lat, variant="static",
                                                        context_len=run["context_len"]),
                          run_length=run["run_length"], top_k=run["top_k"])
        records, tokens = P.decode_full(plugin, cfg, P.Policy.parse(run["policy"]), est)
        assert list(tokens) == run["tokens"]
        got = [[r.tree_size, r.accepted_len] + [getattr(r, f).hex() for f in
               ("surrogate", "t_draft", "t_verify", "t_aux", "l_ar", "cycle_speedup")] for r in records]
        assert got == run["records"]
