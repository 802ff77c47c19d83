"""Time the captured verify graph (fixed N) — run under different BST_ABLATE settings."""
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 31
ctx = int(os.environ.get("CTX", "2048"))  # prompt context (32768: config 4)
eng = B200Engine(QWEN3_8B, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), max_ctx=ctx + 2048, n_cap=255)
eng.reset(np.random.default_rng(0).integers(0, QWEN3_8B.V - 1, ctx + 1).tolist())
eng.set_policy("fixed", n=n)
nn, _ = eng.draft()
rows = eng._bucket(nn)
saved = eng.state.clone()
eng.verify(nn)  # capture
ts_v, ts_d = [], []
for _ in range(12):
    eng.state.copy_(saved)
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record(eng.stream)
    eng._run_draft()
    b.record(eng.stream)
    eng._run_verify(rows)
    c.record(eng.stream)
    c.synchronize()
    ts_d.append(a.elapsed_time(b))
    ts_v.append(b.elapsed_time(c))
print(f"ablate={os.environ.get('BST_ABLATE', '-'):14s} rows={rows} draft_ms={statistics.median(ts_d[2:]):.3f} "
      f"verify_ms={statistics.median(ts_v[2:]):.3f}")
if os.environ.get("AR"):
    print(f"ar_step_ms={1e3 * eng.measure_ar_step():.3f}")
