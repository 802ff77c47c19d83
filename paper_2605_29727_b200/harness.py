"""Run outputs and the offline latency calibration (host side, no kernels).

Mirrors the parts of ``specplan.harness`` a decode deployment needs around the
hot path:

* per-cycle CSV text (``cycle_csv_rows`` in verify_sim, columns
  ``CYCLE_CSV_COLUMNS``, verify_sim.py:26-37,499-511) and its parser;
* the per-(pair, policy) summary over trials — mean / standard error of the
  realized speedup, accepted length and tree size (harness.py:263-319);
* ``calibrate(profile, trace)`` — roofline predictions for an
  ``s,c,observed_seconds`` trace, the OLS Static fit and its report
  (harness.py:341-376).  The engine writes such traces from CUDA-event verify
  timings (``VerifyLatencyEstimator.trace`` + ``cost_model.save_trace``); ``profiles/`` holds the B200 ones.

Every float is rendered with ``repr`` exactly as the reference does, so the
files are byte-identical to the reference's for the same records
(tests/test_harness.py against tests/golden/harness.json).
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

from .cost_model import (CalibrationFit, CostModelParams, fit_static_calibration, load_params, load_trace,
                         trace_predictions)
from .verify_sim import CYCLE_CSV_COLUMNS, CycleRecord, cycle_csv_rows

SUMMARY_COLUMNS = ("pair", "policy", "trials", "mean_speedup", "se_speedup", "mean_aal", "se_aal", "mean_budget",
                   "se_budget")


def render_cycle_csv(records: Iterable[CycleRecord], policy_label: str) -> str:
    """Header + one row per cycle: the body of one (pair, policy, trial) cell file."""
    return "\n".join((",".join(CYCLE_CSV_COLUMNS), *cycle_csv_rows(records, policy_label))) + "\n"


def parse_cycle_csv(body: str) -> list[dict[str, str]]:
    rows = list(csv.DictReader(io.StringIO(body)))
    header = tuple(body.split("\n", 1)[0].split(","))
    if header != CYCLE_CSV_COLUMNS:
        raise ValueError(f"raw CSV must have columns {','.join(CYCLE_CSV_COLUMNS)}")
    return rows


@dataclass(frozen=True)
class SummaryRow:
    """Aggregate of one (pair, policy) over its trials (harness.py:96-108)."""

    pair: int
    policy: str
    trials: int
    mean_speedup: float
    se_speedup: float
    mean_aal: float
    se_aal: float
    mean_budget: float
    se_budget: float


def _mean(xs: Sequence[float]) -> float:
    return float(np.mean(xs))  # numpy's pairwise sum: bit-identical to the reference's aggregation


def _std_err(xs: Sequence[float]) -> float:
    return 0.0 if len(xs) < 2 else float(np.std(xs, ddof=1) / np.sqrt(len(xs)))


def _cell_totals(body: str) -> tuple[int, float, int, float]:
    """(committed tokens, simulated seconds, cycles, mean tree size) of one cell CSV."""
    rows = parse_cycle_csv(body)
    if not rows:
        raise ValueError("cell CSV has no cycles")
    return (int(rows[-1]["cum_tokens"]), float(rows[-1]["cum_time"]), len(rows),
            _mean([int(r["N"]) for r in rows]))


def summarize(pair: int, policy_label: str, trial_csvs: Sequence[str], l_ar: float) -> SummaryRow:
    """Speedup = tokens * l_ar / time per trial; AAL = tokens / cycles; budget = mean N."""
    totals = [_cell_totals(b) for b in trial_csvs]
    speed = [tok * l_ar / secs for tok, secs, _, _ in totals]
    aal = [tok / cyc for tok, _, cyc, _ in totals]
    budget = [mb for _, _, _, mb in totals]
    return SummaryRow(pair, policy_label, len(totals), _mean(speed), _std_err(speed), _mean(aal), _std_err(aal),
                      _mean(budget), _std_err(budget))


def render_summary_csv(rows: Iterable[SummaryRow]) -> str:
    out = [",".join(SUMMARY_COLUMNS)]
    for r in rows:
        out.append(f"{r.pair},{r.policy},{r.trials},{r.mean_speedup!r},{r.se_speedup!r},{r.mean_aal!r},"
                   f"{r.se_aal!r},{r.mean_budget!r},{r.se_budget!r}")
    return "\n".join(out) + "\n"


@dataclass(frozen=True)
class CalibrationReport:
    fit: CalibrationFit
    n_points: int

    @property
    def reduction_pct(self) -> float:
        before, after = self.fit.rmse_before, self.fit.rmse_after
        return 0.0 if before == 0.0 else 100.0 * (1.0 - after / before)

    def render(self) -> str:
        f = self.fit
        keys = (("n_points", self.n_points), ("slope", f.slope), ("intercept", f.intercept),
                ("rmse_before", f.rmse_before), ("rmse_after", f.rmse_after), ("reduction_pct", self.reduction_pct))
        return "".join(f"{k} = {v}\n" if k == "n_points" else f"{k} = {v!r}\n" for k, v in keys)


def calibrate(profile_path: str | Path, trace_path: str | Path) -> CalibrationReport:
    """Static fit of a measured trace against the profile's roofline (the
    ``specplan calibrate`` path)."""
    params: CostModelParams = load_params(profile_path)
    pairs = trace_predictions(params, load_trace(trace_path))
    return CalibrationReport(fit=fit_static_calibration(pairs), n_points=len(pairs))
