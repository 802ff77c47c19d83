import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import ops  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
m = 32
for name, n, k in [("qkv", 6144, 4096), ("o", 4096, 4096), ("down", 4096, 12288)]:
    w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    buf = ops.gemm_partial(x, w).buf
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            ops.gemm_partial(x, w, out=buf)
    for mode in ("cold", "warm"):
        ts = []
        for it in range(8):
            if mode == "cold":
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 100)  # us per launch
        print(name, mode, f"{statistics.median(ts[2:]):.2f} us/launch", f"{n * k * 2 / statistics.median(ts[2:]) / 1e3:.0f} GB/s")
