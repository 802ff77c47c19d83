"""Golden run outputs from the REAL reference (``specplan.harness`` / ``verify_sim``).

    python tests/golden/make_golden_harness.py    # writes tests/golden/harness.json

Inputs: synthetic-pair decode records of the reference (three trials x four
policies on the crossover profile, as ``specplan run`` produces them) and an
``s,c,observed_seconds`` trace.  Outputs: the reference's per-cycle CSV bodies,
its summary CSV, and its calibration report text — the byte strings our
``harness`` module must reproduce (tests/test_harness.py).
"""

from __future__ import annotations

import os
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from codec import fhex, save  # noqa: E402

REF = os.environ.get("BASTION_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import specplan as sp  # noqa: E402
from specplan import harness as sph  # noqa: E402
from specplan import verify_sim as spv  # noqa: E402

PROFILE = Path(REF).parent / "profiles" / "crossover.txt"


def record_fields(r) -> dict:
    return {"tree_size": r.tree_size, "accepted_len": r.accepted_len, "surrogate": fhex(r.surrogate),
            "t_draft": fhex(r.t_draft), "t_verify": fhex(r.t_verify), "t_aux": fhex(r.t_aux), "l_ar": fhex(r.l_ar),
            "cycle_speedup": fhex(r.cycle_speedup)}


def main() -> None:
    params = sp.cost_model.load_params(PROFILE)
    l_ar = sp.roofline_latency(params, sp.LatencyQuery(s=1, c=256))
    lat = sp.CycleLatencies(t_draft=1.25e-4, t_aux=1.2e-5, l_ar=l_ar)
    pair = sp.SyntheticPairConfig(gamma=16, vocab_size=64, alignment=0.8, concentration=0.1, seed=1)
    cells = []
    summary_rows = []
    for policy in (sp.Policy.adaptive(), sp.Policy.fixed(32), sp.Policy.greedy_chain(), sp.Policy.beam(4, 15)):
        bodies = []
        for trial in range(3):
            rule = sp.TargetRule.from_config(replace(pair, seed=sph.trial_rule_seed(0, pair, trial)))
            sim = sp.SimConfig(controller=sp.ControllerConfig(n_max=1024, latencies=lat, variant="static",
                                                              context_len=256), run_length=60, top_k=8)
            recs = sp.decode(rule, sim, policy, sp.VerifyLatencyEstimator(params, variant="static"))
            body = "\n".join([",".join(spv.CYCLE_CSV_COLUMNS)] + spv.cycle_csv_rows(recs, policy.label)) + "\n"
            bodies.append(body)
            cells.append({"policy": policy.label, "trial": trial, "records": [record_fields(r) for r in recs],
                          "csv": body})
        summary_rows.append(sph._summarize(0, policy.label, bodies, l_ar))
    summary = sph.render_summary_csv(summary_rows)
    # calibration: a noisy affine trace over (s, c) against the same profile
    rng = np.random.default_rng(5)
    trace = []
    for c in (64, 256, 1024):
        for s in (1, 9, 33, 65, 129, 257, 513, 1025):
            pred = sp.roofline_latency(params, sp.LatencyQuery(s=s, c=c))
            trace.append((s, c, 1.7 * pred + 2.5e-4 + float(rng.normal(0, 1e-5))))
    trace_text = "s,c,observed_seconds\n" + "".join(f"{s},{c},{o!r}\n" for s, c, o in trace)
    tmp = Path(__file__).resolve().parent / "_trace_tmp.csv"
    tmp.write_text(trace_text)
    try:
        report = sph.calibrate(PROFILE, tmp).render()
    finally:
        tmp.unlink()
    save("harness", {"profile": PROFILE.read_text(), "l_ar": fhex(l_ar), "cells": cells, "summary_csv": summary,
                     "trace_csv": trace_text, "calibration_report": report})


if __name__ == "__main__":
    main()
