"""Cost of one K4 -> K5 kernel boundary in steady state: CUDA graphs of 36 o_proj-shaped
GEMMs (distinct weights, m rows) alone vs each followed by its residual+RMSNorm epilogue
(the verify forward's pattern).  (B - A) / 36 = epilogue + boundary cost per layer."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import ops  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n, k, L = 4096, 4096, 36
ws = [(torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(L)]
x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
resid = torch.randn(m, n, device="cuda")
nw = torch.ones(n, device="cuda", dtype=torch.bfloat16)
bufs = [ops.gemm_partial(x, ws[0]).buf for _ in range(2)]
st = torch.cuda.Stream()


def timed(fn):
    with torch.cuda.stream(st):
        fn()
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        fn()
    ts = []
    for it in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        with torch.cuda.stream(st):
            g.replay()
        b.record(st)
        b.synchronize()
        if it >= 2:
            ts.append(a.elapsed_time(b) * 1e3 / L)
    return statistics.median(ts)


def gemms():
    for i, w in enumerate(ws):
        ops.gemm_partial(x, w, out=bufs[i & 1])


def gemm_epi():
    for i, w in enumerate(ws):
        p = ops.gemm_partial(x, w, out=bufs[i & 1])
        ops.residual_rmsnorm(p, resid, m, n, nw, 1e-6, x=x)


def gemm_reduce():
    for i, w in enumerate(ws):
        p = ops.gemm_partial(x, w, out=bufs[i & 1])
        ops.residual_rmsnorm(p, resid, m, n, nw, 1e-6)


a = timed(gemms)
b = timed(gemm_epi)
c = timed(gemm_reduce)
print(json.dumps(dict(m=m, gemm_us=round(a, 2), gemm_plus_resid_norm_us=round(b, 2), gemm_plus_resid_only_us=round(c, 2),
                      boundary_us=round(b - a, 2))))
