"""CPU BASELINE infrastructure — never the product path.

Times the reference's own planning path (the unmodified ``specplan`` package
installed under ``baseline/_ref``) on the host, as BASELINE.md §5 prescribes:
the per-cycle fp64 drafter rows and verify-argmax tokens a decode produced are
replayed through a plugin into the reference ``decode_full``
(sp/verify_sim.py:426-461), so the reference does exactly its per-cycle work —
MarginalBlock validation, ``top_k_truncate``, ``run_cycle`` / ``best_first_expand``,
``linearize``, ``verify_tree``, ``commit`` — on the same inputs as the GPU.

When ``baseline/_ref`` is absent the oracle port (``specplan_port``) runs the
same loop instead (``kind: "port"``).  Only bench.py's CPU legs import this.
"""

from __future__ import annotations

import os
import platform
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "baseline" / "_ref"


def load_reference():
    """The installed reference package, or None (then callers use the oracle port)."""
    if not (REF_DIR / "specplan" / "__init__.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import specplan  # noqa: PLC0415
    return specplan


def host_info() -> dict:
    model = platform.processor() or ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    return {"cpu_model": model, "host_cores": os.cpu_count()}


class ReplayPlugin:
    """Reference plugin protocol over recorded cycles (sp/verify_sim.py:125-126,158-169).

    ``cycles[i]`` holds ``probs`` (fp64 [gamma, V] rows), ``parent``/``token`` (the tree
    the producer verified) and ``argmax`` (the target's token after every tree node).
    ``drafter_marginals`` builds the reference ``MarginalBlock`` (its validation is
    reference work and is timed); ``next_token`` walks the recorded tree.
    """

    def __init__(self, sp, cycles: list[dict]):
        self.sp = sp
        self.by_prefix: dict[tuple, dict] = {}
        committed: list[int] = []
        for e in cycles:
            self.by_prefix[tuple(committed)] = e
            e["_kids"] = {}
            for i in range(1, len(e["parent"])):
                e["_kids"].setdefault(int(e["parent"][i]), {})[int(e["token"][i])] = i
            committed = committed + [int(e["token"][i]) for i in e["path"][1:]] + [int(e["bonus"])]

    def drafter_marginals(self, prefix):
        e = self.by_prefix[tuple(prefix)]
        g, v = e["probs"].shape
        return self.sp.MarginalBlock(gamma=g, vocab_size=v, probs=e["probs"])

    def next_token(self, seq, temperature: float = 0.0) -> int:
        seq = tuple(seq)
        for k in range(len(seq), -1, -1):
            e = self.by_prefix.get(seq[:k])
            if e is None:
                continue
            node = 0
            for t in seq[k:]:
                node = e["_kids"][node][t]
            return int(e["argmax"][node])
        raise KeyError("prefix not recorded")


def synthetic_cycles(n_cycles: int, seed: int, gamma: int = 16, vocab: int = 151936, scale: float = 6.0,
                     top_k: int = 8, n_max: int = 1024) -> list[dict]:
    """Recorded-cycle stand-ins when no GPU run exists (the reference arm): bf16-valued
    N(0, scale^2) drafter logits -> fp64 rows; the target rejects every tree at the root
    (random-init target), so each cycle commits the bonus only.  The trees are the
    oracle port's best-first prefix, enough for the replay's next_token walk."""
    from oracle import specplan_port as O
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_cycles):
        lg = rng.standard_normal((gamma, vocab), dtype=np.float32) * scale
        lg = (lg.view(np.uint32) & 0xFFFF0000).view(np.float32)
        probs = O.softmax_rows_f64(lg)
        tok, prob = O.topk_rows(probs, top_k)
        tree = O.best_first(tok, prob, min(n_max, 64))
        am = np.full(tree.size + 1, -1, dtype=np.int64)
        bonus = int(rng.integers(0, vocab))
        while bonus in set(int(t) for t in tree.token[1:]):
            bonus = int(rng.integers(0, vocab))
        am[:] = bonus  # never a child token: rejected at the root, bonus committed
        out.append(dict(probs=probs, parent=tree.parent, token=tree.token, argmax=am, path=[0], bonus=bonus))
    return out


def reference_decode(cycles: list[dict], params: dict, latencies: dict, context_len: int, n_max: int,
                     policy: str = "adaptive", fit: tuple[float, float] | None = None, top_k: int = 8,
                     check: bool = True) -> dict:
    """Replay ``cycles`` through the reference decode loop; per-cycle perf_counter times.

    ``params``: CostModelParams fields; ``latencies``: t_draft/t_aux/l_ar; ``fit``: the
    Static calibration (slope, intercept) or None.  With ``check`` the reference's tree
    sizes must equal the recorded ones (the GPU's trees, bit-exact planning)."""
    sp = load_reference()
    if sp is None:
        return _port_decode(cycles, params, latencies, context_len, n_max, policy, fit, top_k, check)
    kind = "reference"
    plugin = ReplayPlugin(sp, cycles)
    est_fit = sp.CalibrationFit(slope=fit[0], intercept=fit[1], rmse_before=0.0, rmse_after=0.0) if fit else None
    est = sp.VerifyLatencyEstimator(sp.CostModelParams(**params), variant="static", fit=est_fit)
    lat = sp.CycleLatencies(**latencies)
    pol = sp.Policy.adaptive() if policy == "adaptive" else sp.Policy.fixed(int(policy.split("-")[1]))
    run_length = sum(len(e["path"]) for e in cycles)
    cfg = sp.SimConfig(controller=sp.ControllerConfig(n_max=n_max, latencies=lat, variant="static",
                                                      context_len=context_len), run_length=run_length, top_k=top_k)
    # time each cycle: wrap the plugin's first call per cycle (drafter_marginals) as a clock tick
    ticks: list[float] = []
    orig = plugin.drafter_marginals

    def ticking(prefix):
        ticks.append(time.perf_counter())
        return orig(prefix)
    plugin.drafter_marginals = ticking
    t0 = time.perf_counter()
    from specplan.verify_sim import decode_full  # noqa: PLC0415  (not re-exported by specplan/__init__.py)
    records, tokens = decode_full(plugin, cfg, pol, est)
    t1 = time.perf_counter()
    ticks.append(t1)
    per = [b - a for a, b in zip(ticks, ticks[1:])]
    if check:
        got = [r.tree_size for r in records]
        want = [len(e["parent"]) - 1 for e in cycles[: len(records)]]
        if got != want:
            raise AssertionError(f"reference trees differ from the recorded ones: {got[:8]} vs {want[:8]}")
    return {"kind": kind, "seconds": t1 - t0, "cycles": len(records), "tokens": len(tokens),
            "median_cycle_s": float(np.median(per)) if per else 0.0, "tree_sizes": [r.tree_size for r in records]}


def _port_decode(cycles, params, latencies, context_len, n_max, policy, fit, top_k, check) -> dict:
    """The same replay through the oracle port's decode loop (no baseline/_ref install)."""
    from oracle import specplan_port as O
    plugin = ReplayPlugin(None, cycles)
    dims = O.Dims(**{k: params[k] for k in ("L", "h", "n_q", "n_kv", "d", "h_ffn", "V", "bp")},
                  peak_flops=params["peak_flops"], bandwidth=params["bandwidth"])
    ticks: list[float] = []

    def drafter(prefix):
        ticks.append(time.perf_counter())
        probs = plugin.by_prefix[tuple(prefix)]["probs"]
        sums = probs.sum(axis=1)  # MarginalBlock validation (sp/lattice.py:47-53)
        if np.any(probs < 0) or np.any(probs > 1) or np.any(np.abs(sums - 1.0) > 1e-9):
            raise ValueError("invalid marginal block")
        return probs
    pol = ("adaptive", 0, 0, 0) if policy == "adaptive" else ("fixed", int(policy.split("-")[1]), 0, 0)
    slope, intercept = fit if fit else (1.0, 0.0)
    run_length = sum(len(e["path"]) for e in cycles)
    t0 = time.perf_counter()
    records, tokens = O.decode_loop(drafter, plugin.next_token, run_length, top_k, pol, n_max, dims, context_len,
                                    latencies["t_draft"], latencies["t_aux"], latencies["l_ar"], "static", slope,
                                    intercept)
    t1 = time.perf_counter()
    ticks.append(t1)
    per = [b - a for a, b in zip(ticks, ticks[1:])]
    if check:
        got = [r["tree_size"] for r in records]
        want = [len(e["parent"]) - 1 for e in cycles[: len(records)]]
        if got != want:
            raise AssertionError(f"port trees differ from the recorded ones: {got[:8]} vs {want[:8]}")
    return {"kind": "port", "seconds": t1 - t0, "cycles": len(records), "tokens": len(tokens),
            "median_cycle_s": float(np.median(per)) if per else 0.0, "tree_sizes": [r["tree_size"] for r in records]}


def _stream_worker(job) -> dict:
    seed, n_cycles, params, latencies, context_len, n_max = job
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    cycles = synthetic_cycles(n_cycles, seed, n_max=n_max)
    return reference_decode(cycles, params, latencies, context_len, n_max, policy="fixed-64", check=False)


def process_pool_streams(n_streams: int, n_cycles: int, params: dict, latencies: dict, context_len: int,
                         n_max: int, workers: int | None = None) -> dict:
    """Config 3's CPU leg: one reference decode stream per request, a process pool over the
    host cores (as the reference harness runs cells, sp/harness.py:249-252)."""
    import multiprocessing as mp
    workers = workers or min(n_streams, os.cpu_count() or 1)
    jobs = [(s, n_cycles, params, latencies, context_len, n_max) for s in range(n_streams)]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(workers) as pool:
        res = pool.map(_stream_worker, jobs)
    wall = time.perf_counter() - t0
    tokens = sum(r["tokens"] for r in res)
    busy = sum(r["seconds"] for r in res)
    return {"streams": n_streams, "workers": workers, "cycles_per_stream": n_cycles, "tokens": tokens,
            "wall_s": wall, "tokens_per_s_wall": tokens / wall,
            "tokens_per_s_decode": tokens / max(busy / workers, 1e-9), "kind": res[0]["kind"]}
