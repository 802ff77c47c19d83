"""The SPEC.md known-answer tests driven through the device path:
K1 (`top_k_truncate` on a hand-built MarginalBlock) -> K2 (`best_first_expand`,
`beam_expand`, `run_cycle`) through the reference-named façade, with the SPEC's
2 x 2 lattice relabelled to tokens a=5, b=9, c=7, d=3 (SURVEY §4.2 last row:
the GPU-lattice parity seam).  Expected values are the SPEC's, cross-checked
against the CPU oracle on the same lattice."""

import numpy as np
import pytest

from oracle import specplan_port as O

pytestmark = pytest.mark.gpu

V = 10
A, B, C, D = 5, 9, 7, 3


@pytest.fixture(scope="module")
def P():
    import paper_2605_29727_b200 as P
    return P


def _block(P):
    # q1 = {a: .6, b: .3}, q2 = {c: .7, d: .2}; the remaining .1 spread evenly
    probs = np.full((2, V), 0.1 / (V - 2))
    probs[0, A], probs[0, B] = 0.6, 0.3
    probs[1, C], probs[1, D] = 0.7, 0.2
    return P.MarginalBlock(gamma=2, vocab_size=V, probs=probs)


def _nodes(tree):
    parent = [-1 if n.parent is None else n.parent for n in tree.nodes]
    token = [-1 if n.token is None else n.token for n in tree.nodes]
    return parent, token, np.array([n.path_score for n in tree.nodes[1:]])


def test_k1_spec_lattice_entries(P):
    lat = P.top_k_truncate(_block(P), 2)
    assert [[t for t, _ in row] for row in lat.entries] == [[A, B], [C, D]]
    assert [[p for _, p in row] for row in lat.entries] == [[0.6, 0.3], [0.7, 0.2]]


def test_k2_spec_best_first_order(P):
    # SPEC.md:133 / :160: a(.60), ac(.42), b(.30), bc(.21), ad(.12), bd(.06); gains non-increasing
    tree = P.best_first_expand(P.top_k_truncate(_block(P), 2), 10)
    parent, token, rho = _nodes(tree)
    assert parent == [-1, 0, 1, 0, 3, 1, 3]
    assert token == [-1, A, C, B, C, D, D]
    np.testing.assert_allclose(rho, [0.6, 0.42, 0.3, 0.21, 0.12, 0.06], rtol=0, atol=1e-15)
    assert np.all(np.diff(rho) <= 0)
    assert abs(tree.surrogate - 2.71) < 1e-12
    want = O.best_first(np.array([[A, B], [C, D]], dtype=np.int32), np.array([[0.6, 0.3], [0.7, 0.2]]), 10)
    assert parent == want.parent.tolist() and token == want.token.tolist()
    assert rho.tobytes() == want.rho[1:].tobytes() and tree.surrogate == want.surrogate


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_k2_spec_nested_prefixes(P, n):
    # best-first trees are nested: the n-node tree is the first n pops
    lat = P.top_k_truncate(_block(P), 2)
    full = _nodes(P.best_first_expand(lat, 10))
    part = _nodes(P.best_first_expand(lat, n))
    assert part[0] == full[0][: n + 1] and part[1] == full[1][: n + 1]


def test_k2_spec_beam(P):
    # beam w=2, d=2 -> {a, b, ac, bc}, A_hat = 2.53 (level order)
    tree = P.beam_expand(P.top_k_truncate(_block(P), 2), 2, 2)
    parent, token, _ = _nodes(tree)
    assert token == [-1, A, B, C, C] and parent == [-1, 0, 0, 1, 2]
    assert abs(tree.surrogate - 2.53) < 1e-12


def test_k2_spec_run_cycle_budget_cap(P):
    # run_cycle with n_max = 1 -> budget 1, stop "budget-cap", the node a
    params = P.CostModelParams(L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288, V=151936, bp=2,
                               peak_flops=1.6e15, bandwidth=6.5e12)
    est = P.VerifyLatencyEstimator(params, variant="static")
    cfg = P.ControllerConfig(n_max=1, latencies=P.CycleLatencies(5e-4, 0.0, 3e-3), variant="static",
                             context_len=2048)
    d = P.run_cycle(P.top_k_truncate(_block(P), 2), cfg, est)
    assert d.budget == 1 and d.stop_reason == "budget-cap"
    parent, token, rho = _nodes(d.tree)
    assert parent == [-1, 0] and token == [-1, A] and rho.tolist() == [0.6]


def test_k2_spec_controller_trace(P):
    # gains .6, .42, .3, .21, ... with C(N) = 1 + 0.15 N and L_AR = 1 stop at N = 3,
    # S_hat trace (1.3913, 1.5538, 1.6, 1.58125).  Device plan: fixed 0.85 + curve(N + 1) with
    # memory = 15 * s * 0.01 (integer bytes, reciprocal bandwidth as in sp/cost_model.py:305-309).
    from paper_2605_29727_b200 import _lib
    from paper_2605_29727_b200.draft_tree import expand_device

    lat = P.top_k_truncate(_block(P), 2)
    tok, prob = lat.device_arrays()
    plan = _lib.Plan(policy=_lib.POLICY_ADAPTIVE, n_max=16,
                     curve=_lib.Curve(0, 0, 0, 15, 0, 0.0, 0.01, 1.0, 0.0, 1.0), fixed_cost=0.85, l_ar=1.0)
    dt = expand_device(tok, prob, plan, 16)
    n, n_exp, stop = (int(x) for x in dt.meta[:3].cpu().tolist())
    assert n == 3 and _lib.STOP_NAMES[stop] == "first-decrease"
    trace = dt.trace[:n_exp].cpu().numpy()
    np.testing.assert_allclose(trace, [1.6 / 1.15, 2.02 / 1.3, 2.32 / 1.45, 2.53 / 1.6], rtol=1e-12)
    cv = O.Curve(0, 0, 0, 15, 0, 0.0, 0.01, 1.0, 0.0, 1.0)
    want = O.controller(lat.device_arrays()[0].cpu().numpy(), lat.device_arrays()[1].cpu().numpy(), 16, cv,
                        0.85, 0.0, 1.0)
    assert want.budget == 3 and trace.tobytes() == np.asarray(want.trace).tobytes()
    assert dt.parent[:4].cpu().tolist() == [-1, 0, 1, 0] and dt.token[:4].cpu().tolist() == [-1, A, C, B]


class _TableTarget:
    """Greedy target given as a per-node table: the token it predicts after each node."""

    def __init__(self, table):
        self.table = table

    def tree_argmax(self, tree, prefix):
        import torch
        return torch.tensor(self.table, dtype=torch.int32, device="cuda")


def _parent_walk_mask(parents, prefix_len):
    # independent restatement of the ancestor rule: row i sees the prefix,
    # then itself and its ancestors by walking parent pointers
    t = len(parents)
    m = np.zeros((prefix_len + t, prefix_len + t), dtype=bool)
    m[:prefix_len, :prefix_len] = True  # the prefix block is all-True (sp/verify_sim.py:346-352)
    for i in range(t):
        m[prefix_len + i, :prefix_len] = True
        j = i
        while j >= 0:
            m[prefix_len + i, prefix_len + j] = True
            j = parents[j]
    return m


@pytest.mark.parametrize("prefix_len", [0, 3])
def test_linearize_spec_six_node_mask(P, prefix_len):
    # the gamma = 2 / K = 2 six-node tree, mask cell by cell against a parent walk
    tree = P.best_first_expand(P.top_k_truncate(_block(P), 2), 6)
    lin = P.linearize(tree, prefix_len)
    assert lin.parents == (-1, 0, 1, 0, 3, 1, 3) and lin.position_ids == (0, 1, 2, 1, 2, 2, 2)
    want = _parent_walk_mask(list(lin.parents), prefix_len)
    blk = slice(prefix_len, None)
    assert np.array_equal(lin.mask[blk, blk], want[blk, blk])
    assert lin.mask[blk, :prefix_len].all()
    assert np.array_equal(lin.mask, want)


def test_linearize_spec_chain_and_siblings(P):
    # a depth-2 chain is causal over the tree block; depth-1 siblings see root + self
    lat = P.top_k_truncate(_block(P), 2)
    chain = P.beam_expand(lat, 1, 2)
    m = P.linearize(chain, 0).mask
    assert np.array_equal(m, np.tril(np.ones((3, 3), dtype=bool)))
    sib = P.beam_expand(lat, 2, 1)
    m = P.linearize(sib, 0).mask
    assert np.array_equal(m, np.array([[1, 0, 0], [1, 1, 0], [1, 0, 1]], dtype=bool))


def test_k6_spec_verify_and_commit(P):
    # a target preferring b then c on the six-node tree -> root -> b -> bc, accepted_len 3;
    # a first choice that is not a child of the root -> accepted_len 1 (bonus only)
    tree = P.best_first_expand(P.top_k_truncate(_block(P), 2), 6)
    lin = P.linearize(tree, 0)
    table = [0] * 7
    table[0], table[3], table[4] = B, C, 1
    rec = P.verify_tree(lin, tree, _TableTarget(table), 0.0)
    assert rec.accepted_path == (0, 3, 4) and rec.accepted_len == 3 and rec.bonus_token == 1
    parent = np.array(lin.parents)
    token = np.array(lin.tokens)
    wpath, wbonus = O.accept_from_argmax(parent, token, np.array(table))
    assert list(rec.accepted_path) == wpath and rec.bonus_token == wbonus
    cache = P.commit(P.SimCache(tokens=(42,)), rec, tree)
    assert tuple(cache.tokens) == (42, B, C, 1)
    miss = [8] + [0] * 6
    rec = P.verify_tree(lin, tree, _TableTarget(miss), 0.0)
    assert rec.accepted_path == (0,) and rec.accepted_len == 1 and rec.bonus_token == 8
    assert tuple(P.commit(P.SimCache(tokens=(42,)), rec, tree).tokens) == (42, 8)


class _AlignedPair:
    """alignment 1.0 with a one-hot drafter.  The greedy target emits
    f(position); the drafter's row j puts all mass on the target's token at j."""

    gamma, vocab = 6, 32

    def __init__(self, P):
        self.P = P

    @staticmethod
    def f(pos):
        return (pos * 7 + 3) % 31

    def drafter_marginals(self, prefix):
        p = np.zeros((self.gamma, self.vocab))
        for j in range(self.gamma):
            p[j, self.f(len(prefix) + j)] = 1.0
        return self.P.MarginalBlock(gamma=self.gamma, vocab_size=self.vocab, probs=p)

    def next_token(self, prefix, temperature):
        return self.f(len(prefix))


class _AlignedTreePair(_AlignedPair):
    def tree_argmax(self, tree, prefix):
        import torch
        am = [self.f(len(prefix) + len(tree.node_path(n.id))) for n in tree.nodes]
        return torch.tensor(am, dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("cls", [_AlignedPair, _AlignedTreePair])
@pytest.mark.parametrize("policy", ["adaptive", "fixed-16", "greedy-chain", "beam-2x6"])
def test_decode_spec_full_acceptance(P, cls, policy):
    # every cycle commits gamma + 1 tokens and the stream equals AR decoding
    pair = cls(P)
    params = P.CostModelParams(L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288, V=151936, bp=2,
                               peak_flops=1.6e15, bandwidth=6.5e12)
    est = P.VerifyLatencyEstimator(params, variant="static")
    lat = P.CycleLatencies(5e-4, 1e-4, 3e-3)
    cfg = P.SimConfig(controller=P.ControllerConfig(n_max=64, latencies=lat, variant="static", context_len=2048),
                      run_length=70, top_k=4)
    records, tokens = P.decode_full(pair, cfg, P.Policy.parse(policy), est)
    assert all(r.accepted_len == pair.gamma + 1 for r in records)
    assert list(tokens) == [pair.f(i) for i in range(len(tokens))] and len(tokens) >= 70
    assert len(records) == -(-70 // (pair.gamma + 1))


def _edge_blocks():
    rng = np.random.default_rng(7)
    out = []
    out.append(("v2_g1", np.array([[0.5, 0.5]])))                         # smallest shape, an exact tie
    out.append(("uniform", np.full((3, 16), 1 / 16)))                    # all ties: token-ascending
    z = np.zeros((4, 12))
    z[:, :3] = [0.5, 0.3, 0.2]                                            # zero-probability tail
    out.append(("zeros", z))
    oh = np.zeros((5, 8))
    oh[np.arange(5), rng.integers(0, 8, 5)] = 1.0                        # one-hot rows: a chain only
    out.append(("onehot", oh))
    q = np.round(rng.dirichlet(np.full(24, 0.3), size=6) * 64) + 1        # quantised: many rho ties
    out.append(("quantised", q / q.sum(1, keepdims=True)))
    return out


@pytest.mark.parametrize("name,probs", _edge_blocks(), ids=[n for n, _ in _edge_blocks()])
@pytest.mark.parametrize("k", [1, 2, 4])
def test_edge_lattices_match_oracle(P, name, probs, k):
    k = min(k, probs.shape[1])
    block = P.MarginalBlock(gamma=probs.shape[0], vocab_size=probs.shape[1], probs=probs)
    lat = P.top_k_truncate(block, k)
    otok, oprob = O.topk_rows(probs, k)
    assert [[t for t, _ in r] for r in lat.entries] == otok.tolist()
    assert np.array([[p for _, p in r] for r in lat.entries]).tobytes() == oprob.tobytes()
    for n in (1, 3, 50):
        parent, token, rho = _nodes(P.best_first_expand(lat, n))
        want = O.best_first(otok, oprob, n)
        assert parent == want.parent.tolist() and token == want.token.tolist()
        assert rho.tobytes() == want.rho[1:].tobytes()
    params = P.CostModelParams(L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288, V=151936, bp=2,
                               peak_flops=1.6e15, bandwidth=6.5e12)
    est = P.VerifyLatencyEstimator(params, variant="static")
    for n_max, fixed in ((64, 1e-4), (64, 1e-1)):   # cheap and expensive fixed cost: short / long trees
        cfg = P.ControllerConfig(n_max=n_max, latencies=P.CycleLatencies(fixed, 0.0, 3e-3), variant="static",
                                 context_len=2048)
        d = P.run_cycle(lat, cfg, est)
        want = O.controller(otok, oprob, n_max, O.curve_for(O.Dims(L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288,
                                                                   V=151936, bp=2, peak_flops=1.6e15,
                                                                   bandwidth=6.5e12), 2048), fixed, 0.0, 3e-3)
        assert d.budget == want.budget and np.array(d.s_hat_trace).tobytes() == np.asarray(want.trace).tobytes()
        assert d.stop_reason == O.STOP_NAMES[want.stop]
        parent, token, _ = _nodes(d.tree)
        assert parent == want.tree.parent.tolist() and token == want.tree.token.tolist()
