"""CPU-side checks of the C ABI: the library loads, exports every symbol
include/bastion.h declares, and its host-side curve arithmetic matches the
reference LatencyCurve bit for bit (no GPU needed)."""

import re
from pathlib import Path

from codec import load, unhex
from oracle import specplan_port as O

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "bastion.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(bst_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2605_29727_b200 import _lib
    lib = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 12
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.bst_abi_version() == 1


def test_ctypes_struct_layouts_match_the_library():
    import ctypes as C

    from paper_2605_29727_b200 import _lib
    for which, struct in enumerate((_lib.Curve, _lib.Plan, _lib.Tree, _lib.GemmSched)):
        assert _lib.lib().bst_struct_size(which) == C.sizeof(struct), struct.__name__


def test_host_curve_matches_reference_golden():
    from paper_2605_29727_b200 import _lib
    g = load("cost_model")
    for row in g["rows"]:
        d = g["profiles"][row["profile"]]
        dims = O.Dims(L=d["L"], h=d["h"], n_q=d["n_q"], n_kv=d["n_kv"], d=d["d"], h_ffn=d["h_ffn"], V=d["V"],
                      bp=d["bp"], peak_flops=unhex(d["peak_flops"]), bandwidth=unhex(d["bandwidth"]))
        cv = O.curve_for(dims, row["c"], row["variant"], unhex(row["slope"]) if row["slope"] else 1.0,
                         unhex(row["intercept"]) if row["intercept"] else 0.0,
                         unhex(row["ratio"]) if row["ratio"] else 1.0)
        st = _lib.Curve(cv.flops_lin, cv.flops_quad, cv.bytes_const, cv.bytes_lin, cv.bytes_quad, cv.inv_peak,
                        cv.inv_bw, cv.slope, cv.intercept, cv.ratio)
        for s, want in zip(row["s"], row["curve"]):
            assert _lib.lib().bst_curve_latency(st, s) == unhex(want)


def test_facade_exports_reference_api():
    import paper_2605_29727_b200 as P
    names = ["AcceptanceRecord", "CalibrationFit", "CandidateLattice", "ControllerConfig", "ControllerDecision",
             "CostModelParams", "CycleLatencies", "CycleRecord", "DraftTree", "EmaBias", "LatencyQuery",
             "MarginalBlock", "Policy", "SimCache", "SimConfig", "SyntheticPairConfig", "TreeNode",
             "VerifyLatencyEstimator", "ar_decode", "beam_expand", "best_first_expand", "build_tree", "bytes_moved",
             "commit", "decode", "ema_update", "estimate_verify_latency", "fit_static_calibration", "flops",
             "linearize", "marginal_gains", "realized_speedup", "roofline_latency", "run_cycle", "replay_trace",
             "sample_continuation", "surrogate_of", "top_k_truncate", "verify_tree"]
    for n in names:
        assert hasattr(P, n), n


def test_device_entry_points_fail_loudly_without_gpu():
    import numpy as np
    import pytest
    import torch
    import paper_2605_29727_b200 as P
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    block = P.MarginalBlock(gamma=1, vocab_size=3, probs=np.array([[0.5, 0.3, 0.2]]))
    with pytest.raises(RuntimeError, match="CUDA device"):
        P.top_k_truncate(block, 2)
    with pytest.raises(ValueError):  # argument errors keep the reference's ValueError
        P.top_k_truncate(block, 4)


def test_cost_model_facade_matches_golden():
    import paper_2605_29727_b200 as P
    g = load("cost_model")
    for row in g["rows"][:40]:
        d = g["profiles"][row["profile"]]
        p = P.CostModelParams(L=d["L"], h=d["h"], n_q=d["n_q"], n_kv=d["n_kv"], d=d["d"], h_ffn=d["h_ffn"],
                              V=d["V"], bp=d["bp"], peak_flops=unhex(d["peak_flops"]),
                              bandwidth=unhex(d["bandwidth"]))
        fit = P.CalibrationFit(unhex(row["slope"]), unhex(row["intercept"]), 0.0, 0.0) if row["slope"] else None
        bias = P.EmaBias(unhex(row["ratio"])) if row["ratio"] else None
        est = P.VerifyLatencyEstimator(p, variant=row["variant"], fit=fit, bias=bias)
        curve = est.curve(row["c"])
        for s, want, want_est in zip(row["s"], row["curve"], row["estimate"]):
            assert curve.latency(s) == unhex(want)
            assert est.estimate(s, row["c"]) == unhex(want_est)


def test_gemm_schedule_pair_mode_and_slot_cover():
    """Stream-K schedule (host side, explicit grid, no GPU): two weight tiles per unit
    above 128 token columns, and every CTA's unit range maps to a valid partial slot."""
    from paper_2605_29727_b200 import ops
    # (n_out, k, m, pair, cta2): CTA pairs for m > 128 on even tile counts (stream-K over 74
    # pairs), two-tile units on one CTA for odd wide outputs
    for n_out, k, m, pair, cta2 in [(24576, 4096, 256, 2, 1), (300, 4096, 256, 1, 0), (4096, 12288, 129, 2, 1),
                                    (151936, 4096, 129, 2, 0), (6144, 4096, 128, 1, 0), (151936, 4096, 64, 1, 0),
                                    (128, 4096, 256, 1, 0), (24576, 4096, 455, 2, 1)]:
        s = ops.gemm_schedule(n_out, k, m, 148)
        assert (s.pair, s.cta2) == (pair, cta2), (n_out, m, s.pair, s.cta2)
        assert s.grid == (74 if cta2 else min(148, s.units))
        n_st = -(-s.n_mt // s.pair)
        assert s.units == n_st * s.n_kb
        assert s.partial_floats == s.n_mt * s.s_max * s.bn * 128 and s.bn >= m
        assert s.tmem_cols <= 512 and s.stages >= 2
        # every CTA's first unit lies in a super-tile whose slot count covers it
        for c in range(s.grid):
            u0 = c * s.units // s.grid
            st = u0 // s.n_kb
            first = max(0, min(s.grid - 1, -(-((st * s.n_kb + 1) * s.grid) // s.units) - 1))
            assert 0 <= c - first < s.s_max


def test_gemm_schedule_rejects_wide_m_without_cta_pairs():
    """m > 256 rows run only on the CTA-pair kernel (two N chunks); odd tile counts raise."""
    import pytest
    from paper_2605_29727_b200 import ops
    with pytest.raises(ValueError):
        ops.gemm_schedule(151936, 4096, 300, 148)
    with pytest.raises(ValueError):
        ops.gemm_schedule(4096, 4096, 513, 148)
