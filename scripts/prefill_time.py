"""Prompt prefill time (engine.reset) at 256- vs 512-row chunks, Qwen3-8B shape, 2048 tokens."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200.engine import decode as D  # noqa: E402
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402

eng = D.B200Engine(QWEN3_8B, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), max_ctx=4096, n_cap=255)
prompt = np.random.default_rng(0).integers(0, QWEN3_8B.V - 1, 2049).tolist()
for rows in (256, 512, 256, 512):
    D.PREFILL_ROWS = rows
    eng.reset(prompt)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        eng.reset(prompt)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"prefill rows={rows} ms={1e3 * min(ts):.1f}", flush=True)
