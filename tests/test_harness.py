"""Run outputs + offline calibration vs the reference's own bytes (tests/golden/harness.json,
made by tests/golden/make_golden_harness.py from the real specplan package).

Per-cycle CSV (verify_sim.py:499-511), summary CSV (harness.py:263-319) and the
calibration report of ``calibrate(profile, trace)`` (harness.py:341-376) must be
byte-identical for the same records / trace."""

from pathlib import Path

from codec import load, unhex

from paper_2605_29727_b200 import harness as H
from paper_2605_29727_b200.verify_sim import CycleRecord

G = load("harness")


def _records(cell):
    return [CycleRecord(tree_size=r["tree_size"], accepted_len=r["accepted_len"], surrogate=unhex(r["surrogate"]),
                        t_draft=unhex(r["t_draft"]), t_verify=unhex(r["t_verify"]), t_aux=unhex(r["t_aux"]),
                        l_ar=unhex(r["l_ar"]), cycle_speedup=unhex(r["cycle_speedup"])) for r in cell["records"]]


def test_cycle_csv_bytes():
    for cell in G["cells"]:
        assert H.render_cycle_csv(_records(cell), cell["policy"]) == cell["csv"]


def test_summary_csv_bytes():
    l_ar = unhex(G["l_ar"])
    rows, order = [], []
    for cell in G["cells"]:
        if cell["policy"] not in order:
            order.append(cell["policy"])
    for pol in order:
        bodies = [c["csv"] for c in G["cells"] if c["policy"] == pol]
        rows.append(H.summarize(0, pol, bodies, l_ar))
    assert H.render_summary_csv(rows) == G["summary_csv"]


def test_parse_cycle_csv_rejects_wrong_columns():
    import pytest
    with pytest.raises(ValueError):
        H.parse_cycle_csv("a,b,c\n1,2,3\n")


def test_calibration_report_bytes(tmp_path: Path):
    prof = tmp_path / "crossover.txt"
    prof.write_text(G["profile"])
    trace = tmp_path / "trace.csv"
    trace.write_text(G["trace_csv"])
    assert H.calibrate(prof, trace).render() == G["calibration_report"]


def test_committed_b200_profile_and_calibration():
    """profiles/qwen3_8b_b200.txt is a 10-key reference profile; the committed engine trace
    recalibrates to the committed report (scripts/calibrate_b200.py wrote both)."""
    root = Path(__file__).resolve().parents[1] / "profiles"
    from paper_2605_29727_b200.cost_model import load_params
    p = load_params(root / "qwen3_8b_b200.txt")
    assert (p.L, p.h, p.n_q, p.n_kv, p.d, p.h_ffn, p.V, p.bp) == (36, 4096, 32, 8, 128, 12288, 151936, 2)
    trace = root / "r2_qwen3_8b_b200_trace.csv"
    report = root / "r2_qwen3_8b_b200_calibration.txt"
    if trace.exists() and report.exists():
        assert H.calibrate(root / "qwen3_8b_b200.txt", trace).render() == report.read_text()


def test_realized_speedup_spec_kats():
    # 1 token per cycle at cycle time l_ar -> 1.0; 5 tokens at 2 l_ar -> 2.5; empty -> error
    import pytest

    import paper_2605_29727_b200 as P

    def rec(acc, t):
        return P.CycleRecord(tree_size=1, accepted_len=acc, surrogate=1.0, t_draft=t / 2, t_verify=t / 2, t_aux=0.0,
                             l_ar=0.01, cycle_speedup=acc * 0.01 / t)

    assert P.realized_speedup([rec(1, 0.01)] * 4) == pytest.approx(1.0, rel=1e-15)
    assert P.realized_speedup([rec(5, 0.02)] * 3) == pytest.approx(2.5, rel=1e-15)
    with pytest.raises(ValueError):
        P.realized_speedup([])
