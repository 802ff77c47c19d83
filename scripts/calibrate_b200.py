"""Engine-measured verify-latency trace -> offline Static calibration.

Runs the Qwen3-8B-shape engine on the B200 at fixed tree budgets N and contexts c,
records the CUDA-event verify time of each cycle as an ``s,c,observed_seconds`` row
(s = N+1, the reference's trace format, cost_model.py:346-361), writes the trace, and
fits it against profiles/qwen3_8b_b200.txt with ``harness.calibrate`` — the
``specplan calibrate --profile --trace`` path:

    python scripts/calibrate_b200.py   # -> profiles/r2_qwen3_8b_b200_{trace.csv,calibration.txt}
"""

import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2605_29727_b200.cost_model import save_trace  # noqa: E402
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402
from paper_2605_29727_b200.harness import calibrate  # noqa: E402

CONTEXTS = (512, 2048, 8192)
BUDGETS = (15, 31, 63, 127, 255, 511, 1023)
REPS = 3

out_dir = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles"
eng = B200Engine(QWEN3_8B, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), max_ctx=max(CONTEXTS) + 1024,
                 seed=0, n_cap=1024)
rows = []
for c in CONTEXTS:
    prompt = np.random.default_rng(c).integers(0, QWEN3_8B.V - 1, c + 1).tolist()
    for n in BUDGETS:
        eng.reset(prompt)
        eng.set_policy("fixed", n=n)
        obs = []
        for i in range(REPS + 1):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            nn, _ = eng.draft(ev)
            ctx = eng._c_host
            eng.verify(nn, ev)
            ev[2].synchronize()
            if i:  # the first cycle of a bucket captures its graph
                obs.append((nn + 1, ctx, ev[1].elapsed_time(ev[2]) * 1e-3))
        s, ctx, _ = obs[-1]
        rows.append((s, ctx, statistics.median(o[2] for o in obs)))
        print(f"c={ctx} s={s} verify={rows[-1][2] * 1e3:.3f} ms", flush=True)
trace = out_dir / "r2_qwen3_8b_b200_trace.csv"
save_trace(trace, rows)
report = calibrate(ROOT / "profiles" / "qwen3_8b_b200.txt", trace)
(out_dir / "r2_qwen3_8b_b200_calibration.txt").write_text(report.render())
print(report.render())
