"""Run a few decode cycles of the config-2 engine for profiling (ncu launch list / full capture)."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_29727_b200 as P  # noqa: E402
from paper_2605_29727_b200.engine.config import MODELS, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen3-8b")
ap.add_argument("--context", type=int, default=2048)
ap.add_argument("--n", type=int, default=31, help="fixed tree budget")
ap.add_argument("--cycles", type=int, default=3)
ap.add_argument("--graphs", type=int, default=1)
ap.add_argument("--ar", type=int, default=0)
a = ap.parse_args()
cfg = MODELS[a.model]
eng = B200Engine(cfg, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), max_ctx=a.context + 2048, n_cap=255)
prompt = np.random.default_rng(0).integers(0, cfg.V - 1, a.context + 1).tolist()
eng.reset(prompt)
eng.use_graphs = bool(a.graphs)
eng.set_policy("fixed", n=a.n)
for _ in range(2):
    eng.cycle()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
if a.ar:
    eng.ar_decode(a.cycles)
else:
    for _ in range(a.cycles):
        eng.cycle()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", eng.tokens()[-4:])
