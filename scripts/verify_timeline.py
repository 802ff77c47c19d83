"""Kernel-boundary timeline of the captured verify graph (BST_TRACE=1 build, see
scripts/boundary_trace.py).  Per traced launch: first CTA entry, first/last release from
griddepcontrol.wait, last CTA end.  Per layer the traced kernels are qkv GEMM, qkv_rope,
attention, o GEMM, residual+norm, gate_up GEMM, SwiGLU, down GEMM, residual+norm."""
import ctypes as C
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
os.environ.setdefault("BASTION_LIB", str(ROOT / "paper_2605_29727_b200" / "libbastion_trace.so"))
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_29727_b200 import _lib  # noqa: E402
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 63
ctx = int(os.environ.get("CTX", "2048"))
eng = B200Engine(QWEN3_8B, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), max_ctx=ctx + 2048, n_cap=255)
eng.reset(np.random.default_rng(0).integers(0, QWEN3_8B.V - 1, ctx + 1).tolist())
eng.set_policy("fixed", n=n)
nn, _ = eng.draft()
rows = eng._bucket(nn)
saved = eng.state.clone()
lib = _lib.lib()
lib.bst_debug_bnd_reset()  # number the verify graph's launches from 1
eng.verify(nn)  # capture
fns = ["bst_debug_bnd_trace_gemm", "bst_debug_bnd_trace_elem", "bst_debug_bnd_trace_attn"]
for f in fns:
    getattr(lib, f).argtypes = [C.c_void_p]
tr = torch.zeros(4096, 8, dtype=torch.int64, device="cuda")
for it in range(3):
    eng.state.copy_(saved)
    tr.zero_()
    tr[:, 0] = -1
    tr[:, 2] = -1
    torch.cuda.synchronize()
    for f in fns:
        getattr(lib, f)(tr.data_ptr())
    eng._run_verify(rows)
    torch.cuda.synchronize()
    for f in fns:
        getattr(lib, f)(None)
recs = [r for r in tr.cpu().tolist() if r[1] != 0 and r[4] != 0]
recs.sort(key=lambda r: r[2])
names = {2: "norm", 3: "rope", 4: "swiglu", 5: "attn"}
gemm_names = {6144: "qkv", 4096: "o/down", 24576: "gate_up", 151936: "lm_head"}


def name(r):
    return gemm_names.get(r[4] - 1000000, f"gemm{r[4] - 1000000}") if r[4] >= 1000000 else names.get(r[4], "?")


print(f"rows={rows} traced launches={len(recs)}")
t0 = recs[0][0]
starts = [i for i, r in enumerate(recs) if name(r) == "qkv"]
L = starts[10]
print("layer 10 (us): kind  entry  dep_first  dep_last  end | wait(prev end -> dep_first)  run(dep_first -> end)")
for i in range(L, L + 9):
    e, end, d0, d1 = recs[i][:4]
    pend = recs[i - 1][1]
    print(f"  {name(recs[i]):8s} {(e - t0) / 1e3:8.2f} {(d0 - t0) / 1e3:8.2f} {(d1 - t0) / 1e3:8.2f} {(end - t0) / 1e3:8.2f}"
          f" | {(d0 - pend) / 1e3:5.2f} {(end - d0) / 1e3:6.2f}")
wait, run = {}, {}
for a0, a1 in zip(starts[1:-1], starts[2:]):
    for j, i in enumerate(range(a0, a1)):
        key = f"{j}:{name(recs[i])}"
        wait.setdefault(key, []).append((recs[i][2] - recs[i - 1][1]) / 1e3)
        run.setdefault(key, []).append((recs[i][1] - recs[i][2]) / 1e3)
span = (recs[starts[-1]][2] - recs[starts[1]][2]) / 1e3 / (len(starts) - 2)
print(f"per-layer span {span:.2f} us over {len(starts) - 2} layers; medians:")
for k in wait:
    print(f"  {k:10s} wait {statistics.median(wait[k]):5.2f}  run {statistics.median(run[k]):6.2f}")
