"""Split of one decode cycle: draft graph | host gap (sync, read N*, launch) | verify graph."""
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
eng.set_policy("fixed", n=int(sys.argv[1]) if len(sys.argv) > 1 else 60)
for _ in range(3):
    eng.cycle()
res = []
for _ in range(20):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(eng.stream)
    eng._run_draft()
    e[1].record(eng.stream)
    with torch.cuda.stream(eng.stream):
        eng.meta_host[:8].copy_(eng.tree.meta, non_blocking=True)
        eng.meta_host[8:].copy_(eng.state, non_blocking=True)
    eng.stream.synchronize()
    n = int(eng.meta_host[0])
    e[2].record(eng.stream)
    eng._run_verify(eng._bucket(n))
    e[3].record(eng.stream)
    e[3].synchronize()
    res.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])))
d, g, v = (statistics.median(x[i] for x in res) for i in range(3))
print(f"draft {d:.3f} ms  host gap {g:.3f} ms  verify {v:.3f} ms  cycle {d + g + v:.3f} ms")
