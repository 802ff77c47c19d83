"""BASELINE config 3: Qwen3-8B shape, 64 concurrent requests sharded data-parallel.

Each rank (one process per GPU, torchrun) takes a contiguous shard of the 64
requests (prompt seeds 0..63, 2048 uniform tokens each) and decodes
them together in one BatchEngine (fixed tree budget N, default 64): rows of all
its requests share every weight pass.  There is no collective on the data path;
the timing and token counts are reduced once at the end (max time, sum tokens).

tokens/s = sum of committed tokens / max over ranks of the device time of the
timed region (CUDA events on each rank's engine stream).
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2605_29727_b200.engine.batch import BatchEngine  # noqa: E402
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--requests", type=int, default=64)
ap.add_argument("--n", type=int, default=64, help="fixed tree budget")
ap.add_argument("--context", type=int, default=2048)
ap.add_argument("--tokens", type=int, default=64, help="new tokens per request in the timed region")
ap.add_argument("--warmup-cycles", type=int, default=3)
ap.add_argument("--policy", default="fixed", choices=["fixed", "adaptive"],
                help="adaptive: batch-aware Algorithm 1 per request with N_max = --n (ragged verify)")
a = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
per = a.requests // world
shard = list(range(rank * per, (rank + 1) * per if rank < world - 1 else a.requests))
cfg = QWEN3_8B
prompts = [np.random.default_rng(r).integers(0, cfg.V - 1, a.context + 1).tolist() for r in shard]
max_ctx = a.context + 1 + (a.warmup_cycles + a.tokens + 16) * 17 + 64
t0 = time.time()
be = BatchEngine(cfg, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), n_req=len(shard), n_fixed=a.n,
                 max_ctx=max_ctx, seed=0)
if a.policy == "adaptive":
    import paper_2605_29727_b200 as P
    pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    params = cfg.cost_params(pk.get("bf16_tflops", 1590.0) * 1e12, pk.get("hbm_gbs", 6650.0) * 1e9)
    est = P.VerifyLatencyEstimator(params, variant="static")  # uncalibrated roofline curve
    lat = P.CycleLatencies(t_draft=est.estimate(17, a.context), t_aux=0.0, l_ar=est.estimate(1, a.context))
    be.set_policy("adaptive", estimator=est, latencies=lat)
be.reset(prompts)
be.precapture()  # adaptive: capture every verify bucket before timing
for _ in range(a.warmup_cycles):
    be.cycle()
base = be.committed_counts().copy()
t_setup = time.time() - t0
if world > 1:
    dist.barrier()
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(be.stream)
cycles = 0
while True:
    for _ in range(8):
        be.cycle()
    cycles += 8
    counts = be.committed_counts()
    if (counts - base).min() >= a.tokens:
        break
ev1.record(be.stream)
ev1.synchronize()
t = ev0.elapsed_time(ev1) * 1e-3
tokens = int((counts - base).sum())
if world > 1:
    tt = torch.tensor([t, float(tokens), float(cycles)], device="cuda", dtype=torch.float64)
    mx = tt.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(tt, op=dist.ReduceOp.SUM)
    t, tokens = float(mx[0]), int(tt[1])
if rank == 0:
    print(json.dumps({
        "config": "config3", "requests": a.requests, "n_gpus": world, "requests_per_gpu": len(shard),
        "fixed_budget": a.n, "policy": a.policy, "context": a.context, "value": tokens / t, "unit": "tokens/s",
        "tokens": tokens, "seconds": t, "cycles": cycles, "ms_per_cycle": t / cycles * 1e3,
        "mean_accept_len": tokens / (cycles * a.requests), "graph_kernels_per_cycle": be.graph_kernels,
        "mean_rows_per_cycle": getattr(be, "last_rows", None) if a.policy == "adaptive" else a.requests * (a.n + 1),
        "setup_s": round(t_setup, 1), "scaling": "weak-per-request (64 requests sharded)",
        "data": "synthetic (random-init bf16 weights, uniform random prompts, seeds 0..63)"}), flush=True)
if world > 1:
    dist.destroy_process_group()
