"""Launch-list profile of config 3 (batched requests): 2 warm cycles, then cudaProfilerStart
around 2 cycles (use with ncu --profile-from-start off)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200.engine.batch import BatchEngine  # noqa: E402
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402

n_req = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n_fixed = int(sys.argv[2]) if len(sys.argv) > 2 else 16
prompts = [np.random.default_rng(r).integers(0, QWEN3_8B.V - 1, 2049).tolist() for r in range(n_req)]
be = BatchEngine(QWEN3_8B, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), n_req=n_req, n_fixed=n_fixed,
                 max_ctx=2049 + 20 * 17 + 64, seed=0)
be.reset(prompts)
for _ in range(2):
    be.cycle()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(2):
    be.cycle()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
