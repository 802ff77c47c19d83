"""Timeline of GEMM -> residual+RMSNorm -> GEMM boundaries inside a CUDA graph (BST_TRACE=1
build: BST_TRACE=1 python -m paper_2605_29727_b200.build, then BASTION_LIB=<pkg>/libbastion_trace.so).
Per launch: first CTA entry, first/last dependency release (griddepcontrol.wait return), last
CTA end, in us relative to the first launch's entry."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
os.environ.setdefault("BASTION_LIB", str(ROOT / "paper_2605_29727_b200" / "libbastion_trace.so"))
sys.path.insert(0, str(ROOT))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2605_29727_b200 import _lib, ops  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n, k, L = 4096, 4096, 8
ws = [(torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(L)]
x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
resid = torch.randn(m, n, device="cuda")
nw = torch.ones(n, device="cuda", dtype=torch.bfloat16)
bufs = [ops.gemm_partial(x, ws[0]).buf for _ in range(2)]
st = torch.cuda.Stream()


def run():
    for i, w in enumerate(ws):
        p = ops.gemm_partial(x, w, out=bufs[i & 1])
        ops.residual_rmsnorm(p, resid, m, n, nw, 1e-6, x=x)


with torch.cuda.stream(st):
    run()
st.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    run()
lib = _lib.lib()
tr = torch.zeros(4096, 4, dtype=torch.int64, device="cuda")
for it in range(3):
    tr[:, 0] = -1  # atomicMin slots (as unsigned: max)
    tr[:, 2] = -1
    tr[:, 1] = 0
    tr[:, 3] = 0
    torch.cuda.synchronize()
    for f in ("bst_debug_bnd_trace_gemm", "bst_debug_bnd_trace_elem"):
        getattr(lib, f).argtypes = [C.c_void_p]
        getattr(lib, f)(tr.data_ptr())
    with torch.cuda.stream(st):
        g.replay()
    st.synchronize()
    for f in ("bst_debug_bnd_trace_gemm", "bst_debug_bnd_trace_elem"):
        getattr(lib, f)(None)
rows = [r for r in tr.cpu().tolist() if r[1] != 0]
rows.sort(key=lambda r: r[0])
t0 = rows[0][0]
print("kind   entry   dep_first  dep_last   end    | gap(prev end -> dep_first)")
prev_end = None
for i, (e, end, d0, d1) in enumerate(rows):
    kind = "gemm" if i % 2 == 0 else "norm"
    gap = f"{(d0 - prev_end) / 1e3:6.2f}" if prev_end else "     -"
    print(f"{kind}  {(e - t0) / 1e3:7.2f} {(d0 - t0) / 1e3:9.2f} {(d1 - t0) / 1e3:9.2f} {(end - t0) / 1e3:7.2f}   | {gap}")
    prev_end = end
