"""K4 per-shape HBM rate in steady state: a CUDA graph of 36 back-to-back launches of one
verify shape over 36 distinct weight matrices (>> L2), as in the verify forward."""
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import ops  # noqa: E402

peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
shapes = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 24576, 4096), ("down", 4096, 12288)]
if os.environ.get("LM_HEAD"):
    shapes = [("lm_head", 151936, 4096)]
NW = int(os.environ.get("NW", "36"))
st = torch.cuda.Stream()
for m in [int(a) for a in (sys.argv[1:] or ["16", "64"])]:
    for name, n, k in shapes:
        ws = [(torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(NW)]
        x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        buf = ops.gemm_partial(x, ws[0]).buf

        def run():
            for w in ws:
                ops.gemm_partial(x, w, out=buf)
        with torch.cuda.stream(st):
            run()
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            run()
        ts = []
        for it in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            with torch.cuda.stream(st):
                g.replay()
            b.record(st)
            b.synchronize()
            if it >= 1:
                ts.append(a.elapsed_time(b) * 1e-3 / NW)
        t = statistics.median(ts)
        byts = n * k * 2 + m * k * 2
        print(json.dumps(dict(m=m, shape=name, n=n, k=k, us=round(t * 1e6, 2), GBps=round(byts / t / 1e9),
                              frac=round(byts / t / 1e9 / peak, 3))), flush=True)
        del ws, g
        torch.cuda.empty_cache()
