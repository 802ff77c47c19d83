import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import _lib, ops  # noqa: E402

n, k, m = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
lib = _lib.lib()
lib.bst_debug_gemm_trace.argtypes = [C.c_void_p, C.c_int]
w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
buf = ops.gemm_partial(x, w).buf
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cta in (0, 77, 147):
    tr = torch.zeros(64, dtype=torch.int64, device="cuda")
    lib.bst_debug_gemm_trace(tr.data_ptr(), cta)
    flush.zero_()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    ops.gemm_partial(x, w, out=buf)
    b.record()
    torch.cuda.synchronize()
    t = tr.cpu().tolist()
    t0 = t[0]
    f = lambda i: f"{(t[i] - t0) / 1000:.2f}" if t[i] else "-"
    fulls = [f(i) for i in range(8, 40) if t[i]]
    print(f"cta {cta}: total_event={a.elapsed_time(b) * 1000:.1f}us setup={f(1)} pre_w_issued={f(2)} dep_ok={f(3)} "
          f"epi0={f(4)} epi1={f(5)} end={f(7)}")
    print("   full seen:", " ".join(fulls))
lib.bst_debug_gemm_trace(None, 0)
