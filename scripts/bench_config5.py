"""BASELINE config 5: Qwen3-32B-shape target, tensor-parallel verify + accept.

  torchrun --nproc-per-node 8 scripts/bench_config5.py          # TP = world size (NCCL all-reduce)
  python scripts/bench_config5.py --emulate-tp 8                # one rank's shard on 1 GPU, no collective
  python scripts/bench_config5.py --tp 1                        # the full 32B target on 1 GPU

Per fixed tree budget N (seeded lattice, same tree on every rank): W warm-up, K timed
verify steps (CUDA graph of verify rows -> sharded target forward -> accept -> KV
compaction -> commit), CUDA events on the engine stream, max over ranks.  Prints one JSON
line per budget: us/step, accepted tokens/s, and the per-rank HBM roofline fraction
(shard weights + local KV read once per step)."""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200.engine.config import MODELS  # noqa: E402
from paper_2605_29727_b200.engine.tp import TPVerifier, local_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen3-32b")
ap.add_argument("--context", type=int, default=2048)
ap.add_argument("--budgets", type=int, nargs="+", default=[16, 64, 255])
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--emulate-tp", type=int, default=0, help="run rank 0 of an N-way split alone (no collective)")
ap.add_argument("--tp", type=int, default=0)
args = ap.parse_args()

world, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
    int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
tp = args.emulate_tp or args.tp or world
cfg = MODELS[args.model]
lc = local_config(cfg, tp)
peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
eng = TPVerifier(cfg, tp, rank if not args.emulate_tp else 0, max_ctx=args.context + 17 * (args.steps + args.warmup + 8)
                 + 512, seed=0)
prompt = np.random.default_rng(7).integers(0, cfg.V - 1, args.context + 1).tolist()
w_bytes = sum(t.numel() * 2 for lw in eng.target.w.layers for t in (lw.qkv, lw.o, lw.gate_up, lw.down)) + \
    eng.target.w.lm_head.numel() * 2
for n in args.budgets:
    eng.reset(prompt)
    nn = eng.set_tree(n)
    for _ in range(args.warmup):
        eng.step()
    eng.stream.synchronize()
    c0 = int(eng.state[3].item())
    if dist:
        dist.barrier()
    ts = []
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    a0.record(eng.stream)
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        eng.step()
        e1.record(eng.stream)
        ts.append((e0, e1))
    a1.record(eng.stream)
    a1.synchronize()
    total = a0.elapsed_time(a1) * 1e-3
    if dist:
        t = torch.tensor([total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    tokens = int(eng.state[3].item()) - c0
    us = 1e6 * total / args.steps
    c = int(eng.state[0].item())
    kv_bytes = 2 * cfg.L * (c + nn + 1) * lc.n_kv * 128 * 2
    byts = w_bytes + kv_bytes
    if rank == 0:
        print(json.dumps({"config": "config5", "model": cfg.name, "tp": tp, "world": world,
                          "emulated": bool(args.emulate_tp), "context": args.context, "budget": n, "tree_size": nn,
                          "verify_us_per_step": round(us, 1),
                          "median_step_us": round(1e3 * statistics.median(x.elapsed_time(y) for x, y in ts), 1),
                          "tokens_per_s": tokens / total, "mean_accept_len": tokens / args.steps,
                          "per_rank_bytes": byts, "achieved_GBps": round(byts / (us * 1e-6) / 1e9, 1),
                          "roofline_frac": round(byts / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 3),
                          "collective": "none (emulated shard)" if args.emulate_tp else ("none" if world == 1
                          else "NCCL all_reduce fp32 residual x 2 per layer + int64 argmax MAX")}), flush=True)
if dist:
    dist.destroy_process_group()
