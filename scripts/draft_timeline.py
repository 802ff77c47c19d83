"""Kernel timeline of the captured draft graph (BST_TRACE=1 build; see verify_timeline.py).
Lists every traced launch (K4 GEMMs, K5 epilogues, K3 attention) in dependency order with
its wait (previous traced end -> release) and run (release -> last CTA end); untraced
kernels (K1 top-K, K2 expansion, row builders) show up as gaps."""
import ctypes as C
import os
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

ctx = int(os.environ.get("CTX", "2048"))
eng = B200Engine(QWEN3_8B, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), max_ctx=ctx + 2048, n_cap=255)
eng.reset(np.random.default_rng(0).integers(0, QWEN3_8B.V - 1, ctx + 1).tolist())
nn, _ = eng.draft()
eng.verify(nn)
saved = eng.state.clone()
lib = _lib.lib()
lib.bst_debug_bnd_reset()
eng.graph_d = None
eng.graphs_d = {}
eng._run_draft()  # recapture with fresh launch numbers
torch.cuda.synchronize()
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
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    eng._run_draft()
    b.record(eng.stream)
    torch.cuda.synchronize()
    for f in fns:
        getattr(lib, f)(None)
recs = [r for r in tr.cpu().tolist() if r[1] != 0 and r[4] != 0]
recs.sort(key=lambda r: r[2])
names = {2: "norm", 3: "rope", 4: "swiglu", 5: "attn"}


def name(r):
    return f"gemm n={r[4] - 1000000}" if r[4] >= 1000000 else names.get(r[4], "?")


print(f"draft graph {a.elapsed_time(b) * 1e3:.1f} us (event); traced launches {len(recs)}")
t0 = recs[0][2]
prev = None
for r in recs:
    e, end, d0, d1 = r[:4]
    w = f"{(d0 - prev) / 1e3:6.2f}" if prev else "     -"
    print(f"  {name(r):16s} release {(d0 - t0) / 1e3:8.2f}  wait {w}  run {(end - d0) / 1e3:6.2f}")
    prev = end
print(f"last traced end at {(recs[-1][1] - t0) / 1e3:.2f} us after the first release")
