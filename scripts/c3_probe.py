"""Config-3 leg step by step with timestamps (diagnoses a stall of bench.py's config-3 GPU leg)."""
import faulthandler
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
faulthandler.dump_traceback_later(int(sys.argv[1]) if len(sys.argv) > 1 else 240, exit=True)
import numpy as np
import torch

from paper_2605_29727_b200.engine.batch import BatchEngine
from paper_2605_29727_b200.engine.config import MODELS, DrafterConfig

T0 = time.time()


def log(m):
    print(f"[{time.time() - T0:7.1f}s] {m}", flush=True)


cfg = MODELS["qwen3-8b"]
n_req = int(sys.argv[2]) if len(sys.argv) > 2 else 64
prompts = [np.random.default_rng(r).integers(0, cfg.V - 1, 2049).tolist() for r in range(n_req)]
be = BatchEngine(cfg, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), n_req=n_req, n_fixed=64,
                 max_ctx=2048 + 17 * 16 + 64, seed=0)
log("engine built")
import os
be.use_graphs = os.environ.get("GRAPHS", "1") == "1"
if os.environ.get("SPLITS"):
    be.set_attention_splits(int(os.environ["SPLITS"]))
if os.environ.get("CHUNKV"):
    be.chunk_v = int(os.environ["CHUNKV"])
if os.environ.get("CHUNKD"):
    be.chunk_d = int(os.environ["CHUNKD"])
log(f"chunk_v={be.chunk_v} chunk_d={be.chunk_d}")
be.reset(prompts)
log("reset done")
for i in range(int(os.environ.get("CYCLES", "4"))):
    be.cycle()
    torch.cuda.synchronize()
    log(f"cycle {i}")
