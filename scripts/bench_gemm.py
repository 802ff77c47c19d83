"""Microbench: K4 GEMM HBM streaming rate at verify shapes (L2 flushed between launches)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import ops  # noqa: E402

peak = 6457.7
shapes = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 24576, 4096), ("down", 4096, 12288),
          ("lm_head", 151936, 4096)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for m in [int(a) for a in (sys.argv[1:] or ["17"])]:
    for name, n, k in shapes:
        w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
        x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        buf = ops.gemm_partial(x, w).buf
        ts = []
        for it in range(12):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ops.gemm_partial(x, w, out=buf)
            b.record()
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(a.elapsed_time(b) * 1e-3)
        t = sorted(ts)[len(ts) // 2]
        byts = n * k * 2 + m * k * 2
        gbs = byts / t / 1e9
        s = ops.gemm_schedule(n, k, m)
        res.append(dict(name=name, m=m, n=n, k=k, us=round(t * 1e6, 2), GBps=round(gbs, 1), frac=round(gbs / peak, 3),
                        tflops=round(2 * m * n * k / t / 1e12, 1), grid=s.grid, s_max=s.s_max, stages=s.stages))
        print(json.dumps(res[-1]), flush=True)
        del w
