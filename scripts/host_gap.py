"""Device idle time between the draft graph and the verify graph caused by the
cycle's host synchronisation (read N*, pick the verify bucket, launch)."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402

eng = B200Engine(QWEN3_8B, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), max_ctx=4096, n_cap=255)
eng.reset(np.random.default_rng(0).integers(0, QWEN3_8B.V - 1, 2049).tolist())
eng.set_policy("fixed", n=52)
for _ in range(3):
    eng.cycle()
gaps, cyc, nodes = [], [], []
for _ in range(20):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(eng.stream)
    n, _ = eng.draft()
    ev[1].record(eng.stream)  # stream is idle here: records "now"
    eng.verify(n)
    ev[2].record(eng.stream)
    ev[2].synchronize()
    nodes.append(n)
    cyc.append(ev[0].elapsed_time(ev[2]))
    gaps.append(ev[0].elapsed_time(ev[1]))
print("median cycle ms", statistics.median(cyc), "draft+sync ms", statistics.median(gaps), "N*", statistics.median(nodes))
