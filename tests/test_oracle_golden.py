"""Pin the CPU oracle (oracle/specplan_port.py) against the reference's golden vectors.

The fixtures under tests/golden/ were produced by the real reference
(tests/golden/make_golden.py); these tests need no GPU and no reference.
"""

import numpy as np
import pytest

from codec import dec, load, unhex
from oracle import specplan_port as O

STOP = {"first-decrease": O.STOP_FIRST_DECREASE, "frontier-exhausted": O.STOP_FRONTIER_EXHAUSTED,
        "budget-cap": O.STOP_BUDGET_CAP}


def _dims(d):
    return O.Dims(L=d["L"], h=d["h"], n_q=d["n_q"], n_kv=d["n_kv"], d=d["d"], h_ffn=d["h_ffn"], V=d["V"],
                  bp=d["bp"], peak_flops=unhex(d["peak_flops"]), bandwidth=unhex(d["bandwidth"]))


def _assert_tree(flat, want):
    np.testing.assert_array_equal(flat.parent, dec(want["parent"]))
    np.testing.assert_array_equal(flat.depth, dec(want["depth"]))
    np.testing.assert_array_equal(flat.token, dec(want["token"]))
    # bit-exact path scores
    assert flat.rho.tobytes() == dec(want["rho"]).tobytes()


@pytest.fixture(scope="module")
def lattice_cases():
    return load("lattice_trees")["cases"]


def test_topk_matches_reference(lattice_cases):
    for case in lattice_cases:
        tok, prob = O.topk_rows(dec(case["probs"]), case["k"])
        np.testing.assert_array_equal(tok, dec(case["tok"]), err_msg=case["name"])
        assert prob.tobytes() == dec(case["prob"]).tobytes(), case["name"]


def test_spec_topk_kats():
    # SPEC.md:55-57
    tok, prob = O.topk_rows(np.array([[0.5, 0.3, 0.2]]), 2)
    assert tok.tolist() == [[0, 1]] and prob.tolist() == [[0.5, 0.3]]
    tok, _ = O.topk_rows(np.array([[0.4, 0.4, 0.2]]), 1)
    assert tok.tolist() == [[0]]
    tok, _ = O.topk_rows(np.array([[0.1, 0.2, 0.3, 0.4], [0.25] * 4]), 2)
    assert tok.tolist() == [[3, 2], [0, 1]]
    with pytest.raises(ValueError):
        O.topk_rows(np.array([[0.5, 0.5]]), 3)


def test_best_first_matches_reference(lattice_cases):
    n = 0
    for case in lattice_cases:
        tok, prob = dec(case["tok"]), dec(case["prob"])
        for bf in case["best_first"]:
            flat = O.best_first(tok, prob, bf["n_max"])
            _assert_tree(flat, bf["nodes"])
            assert flat.surrogate == unhex(bf["surrogate"])
            n += 1
    assert n > 100


def test_spec_best_first_kat():
    # a(.60), ac(.42), b(.30), bc(.21), ad(.12), bd(.06)
    tok = np.array([[0, 1], [2, 3]], dtype=np.int32)
    prob = np.array([[0.6, 0.3], [0.7, 0.2]])
    t = O.best_first(tok, prob, 10)
    assert t.parent.tolist() == [-1, 0, 1, 0, 3, 1, 3]
    assert t.token.tolist() == [-1, 0, 2, 1, 2, 3, 3]
    np.testing.assert_allclose(t.rho[1:], [0.6, 0.42, 0.3, 0.21, 0.12, 0.06])
    assert abs(t.surrogate - 2.71) < 1e-12
    b = O.beam(tok, prob, 2, 2)
    assert abs(b.surrogate - 2.53) < 1e-12 and b.token.tolist() == [-1, 0, 1, 2, 2]


def test_beam_matches_reference(lattice_cases):
    for case in lattice_cases:
        tok, prob = dec(case["tok"]), dec(case["prob"])
        for bm in case["beam"]:
            flat = O.beam(tok, prob, bm["width"], bm["depth"])
            _assert_tree(flat, bm["nodes"])
            assert flat.surrogate == unhex(bm["surrogate"])


def test_controller_matches_reference(lattice_cases):
    g = load("controller")
    profiles = {k: _dims(v) for k, v in g["profiles"].items()}
    lat = {c["name"]: (dec(c["tok"]), dec(c["prob"])) for c in lattice_cases}
    assert len(g["runs"]) > 50
    for run in g["runs"]:
        tok, prob = lat[run["lattice"]]
        curve = O.curve_for(profiles[run["profile"]], run["c"], run["variant"],
                            unhex(run["slope"]) if run["slope"] else 1.0,
                            unhex(run["intercept"]) if run["intercept"] else 0.0,
                            unhex(run["ratio"]) if run["ratio"] else 1.0)
        d = O.controller(tok, prob, run["n_max"], curve, unhex(run["t_draft"]), unhex(run["t_aux"]),
                         unhex(run["l_ar"]))
        assert d.budget == run["budget"]
        assert d.stop == STOP[run["stop"]]
        assert np.array(d.trace).tobytes() == dec(run["trace"]).tobytes()
        _assert_tree(d.tree, run["nodes"])
        assert d.tree.surrogate == unhex(run["surrogate"])


def test_cost_model_matches_reference():
    g = load("cost_model")
    profiles = {k: _dims(v) for k, v in g["profiles"].items()}
    for row in g["rows"]:
        p, c, var = profiles[row["profile"]], row["c"], row["variant"]
        sl = unhex(row["slope"]) if row["slope"] else 1.0
        ic = unhex(row["intercept"]) if row["intercept"] else 0.0
        ra = unhex(row["ratio"]) if row["ratio"] else 1.0
        curve = O.curve_for(p, c, var, sl, ic, ra)
        for i, s in enumerate(row["s"]):
            assert curve.latency(s) == unhex(row["curve"][i])
            assert O.flops(p, s, c) == int(row["flops"][i])
            assert O.bytes_moved(p, s, c) == int(row["bytes"][i])
            w, kv, act = O.bytes_by_category(p, s, c)
            assert (w, kv, act) == (int(row["weights"][i]), int(row["kv"][i]), int(row["act"][i]))
            assert w + kv + act == O.bytes_moved(p, s, c)  # SPEC Table-6 decomposition
            assert O.roofline(p, s, c) == unhex(row["roofline"][i])
            assert O.apply_variant(var, O.roofline(p, s, c), sl, ic, ra) == unhex(row["estimate"][i])
    for r, a, pr, ob, want in g["ema"]:
        assert O.ema_step(unhex(r), unhex(a), unhex(pr), unhex(ob)) == unhex(want)
    for case in g["ols"]:
        pairs = [(unhex(a), unhex(b)) for a, b in case["pairs"]]
        assert list(O.ols_fit(pairs)) == [unhex(x) for x in case["fit"]]


def test_spec_cost_kats():
    # SPEC.md:293 flops toy = 3712; ema KAT SPEC.md:330
    p = O.Dims(L=1, h=8, n_q=2, n_kv=1, d=4, h_ffn=16, V=32, bp=2, peak_flops=1.0, bandwidth=1.0)
    assert O.flops(p, 2, 4) == 3712
    assert sum(O.bytes_by_category(p, 2, 4)) == O.bytes_moved(p, 2, 4)
    assert O.ema_step(1.0, 0.1, 1.0, 2.0) == pytest.approx(1.1)


def test_replay_matches_reference():
    for case in load("replay")["cases"]:
        budget, trace, stop = O.replay([unhex(x) for x in case["gains"]], [unhex(x) for x in case["costs"]],
                                       unhex(case["l_ar"]))
        assert budget == case["budget"] and stop == STOP[case["stop"]]
        assert trace == [unhex(x) for x in case["trace"]]


def test_linearize_matches_reference():
    for case in load("linearize")["cases"]:
        parent = dec(case["nodes"]["parent"])
        m = O.linear_mask(parent, case["prefix_len"])
        want = np.unpackbits(dec(case["mask"]), axis=1)[:, : case["mask_shape"][1]].astype(bool)
        np.testing.assert_array_equal(m, want)
        assert case["position_ids"] == dec(case["nodes"]["depth"]).tolist()
        assert case["parents"] == parent.tolist()


def test_decode_loop_matches_reference():
    g = load("decode")
    crossover = _dims(load("controller")["profiles"]["crossover"])
    for run in g["runs"]:
        blocks = {tuple(k): dec(v) for k, v in run["blocks"]}
        choices = {tuple(k): v for k, v in run["choices"]}
        pol = run["policy"]
        if pol == "adaptive":
            policy = ("adaptive", 0, 0, 0)
        elif pol.startswith("fixed-"):
            policy = ("fixed", int(pol[6:]), 0, 0)
        elif pol == "greedy-chain":
            policy = ("greedy-chain", 0, 0, 0)
        else:
            w, d = pol[5:].split("x")
            policy = ("beam", 0, int(w), int(d))
        records, tokens = O.decode_loop(
            lambda prefix: blocks[tuple(prefix)], lambda seq, T: choices[tuple(seq)],
            run["run_length"], run["top_k"], policy, run["n_max"], crossover, run["context_len"],
            unhex(run["t_draft"]), unhex(run["t_aux"]), unhex(run["l_ar"]))
        assert list(tokens) == run["tokens"]
        assert list(tokens) == run["ar_tokens"]  # criterion 8: greedy output preservation
        for rec, want in zip(records, run["records"]):
            got = [rec["tree_size"], rec["accepted_len"]] + [rec[k].hex() for k in
                   ("surrogate", "t_draft", "t_verify", "t_aux", "l_ar", "cycle_speedup")]
            assert got == want
        assert len(records) == len(run["records"])
