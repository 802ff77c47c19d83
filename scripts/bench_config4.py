"""BASELINE config 4: Qwen3-8B shape, 32K-token KV context, tree budget sweep 16..256.

Prefills a 32768-token synthetic prompt, then for each fixed budget N times
`cycles` decode cycles (CUDA events on the engine stream) and reports the verify
µs/step next to the fused-minimum roofline of the verify step (weights + KV +
activations) and the K3 attention share measured by ablation.
One JSON line per N.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--context", type=int, default=32768)
ap.add_argument("--budgets", default="16,32,64,128,255")
ap.add_argument("--cycles", type=int, default=8)
a = ap.parse_args()

peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
BW, PF = peaks["hbm_gbs"] * 1e9, peaks["bf16_tflops"] * 1e12
cfg = QWEN3_8B
eng = B200Engine(cfg, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), max_ctx=a.context + 2048, n_cap=255)
prompt = np.random.default_rng(0).integers(0, cfg.V - 1, a.context + 1).tolist()
eng.reset(prompt)
saved = eng.state.clone()
for n in [int(x) for x in a.budgets.split(",")]:
    eng.state.copy_(saved)
    eng.set_policy("fixed", n=n)
    eng.cycle()  # capture graphs
    eng.state.copy_(saved)
    tv, td, sizes = [], [], []
    for _ in range(a.cycles):
        eng.state.copy_(saved)  # keep c fixed at the prompt length
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        nn = eng.cycle(ev)
        ev[2].synchronize()
        td.append(ev[0].elapsed_time(ev[1]) * 1e3)
        tv.append(ev[1].elapsed_time(ev[2]) * 1e3)
        sizes.append(nn)
    s = eng._bucket(sizes[-1])
    c = a.context
    h, hq, hkv, hf, L, V = cfg.h, cfg.h_q, cfg.h_kv, cfg.h_ffn, cfg.L, cfg.V
    w_bytes = 2 * (L * (h * (hq + 2 * hkv) + hq * h + 3 * h * hf) + V * h)
    kv_bytes = 2 * L * (2 * (c + s) * hkv)
    act_bytes = 2 * (L * (4 * s * h + 4 * s * hq + 2 * s * hkv + 4 * s * hf) + s * h + s * V)
    flops = L * (4 * s * h * hq + 4 * s * h * hkv + 4 * s * (c + s) * hq + 6 * s * h * hf) + 2 * s * h * V
    roof_us = max((w_bytes + kv_bytes + act_bytes) / BW, flops / PF) * 1e6
    attn_bytes = 2 * L * (2 * (c + s) * hkv + 2 * s * hq)
    r = dict(config="config4", context=c, budget=n, tree_size=sizes[-1], verify_rows=s,
             verify_us=round(statistics.median(tv[1:]), 1), draft_us=round(statistics.median(td[1:]), 1),
             roofline_us=round(roof_us, 1), frac=round(roof_us / statistics.median(tv[1:]), 3),
             attn_kv_bytes_per_step=attn_bytes, weights_bytes=w_bytes)
    print(json.dumps(r), flush=True)
