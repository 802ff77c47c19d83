"""Phase trace of one key-major attention CTA (needs a BST_TRACE=1 build)."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import _lib, ops  # noqa: E402
from paper_2605_29727_b200.engine.forward import PagedKV  # noqa: E402

c, s = int(sys.argv[1]), int(sys.argv[2])
y = int(sys.argv[3]) if len(sys.argv) > 3 else 0
lib = _lib.lib()
tr = torch.zeros(32 * 8, dtype=torch.int64, device="cuda")
n_q, n_kv = 32, 8
kv = PagedKV(1, n_kv, c + 320, "cuda")
kv.buf.normal_(0, 1)
q = torch.randn(s, n_q * 128, device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
words = (s + 31) // 32
anc = torch.full((s, words), -1, dtype=torch.int32, device="cuda")
ws = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
run = lambda: ops.attention(q, out, kv.buf, 1, kv.n_pages, 0, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0,
                            anc.view(-1), words, ws)
run()
torch.cuda.synchronize()
import time
w = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
t_end = time.time() + 1.0
while time.time() < t_end:  # ramp the clocks up before tracing
    for _ in range(20):
        w @ w
    torch.cuda.synchronize()
lib.bst_debug_attn_trace.argtypes = [C.c_void_p]
lib.bst_debug_attn_trace_cta(y)
lib.bst_debug_attn_trace(tr.data_ptr())
for _ in range(3):
    tr.zero_()
    tr[28 * 8:29 * 8] = 1 << 62
    for _ in range(3):
        w @ w
    run()
    torch.cuda.synchronize()
t = tr.view(32, 8).cpu()
t0 = int(t[31, 1])
f = lambda v: f"{(int(v) - t0) / 1000:7.2f}" if int(v) else "   -   "
print("entry->depwait/staged/o_final/merge_start/sm_end/exit:", [f(t[31, k]) for k in (2, 3, 4, 5, 6, 0)])
print("all CTAs max: merge_start/end/arrive/spin_done:", [f(t[29, k]) for k in (1, 2, 3, 4)])
print("CTA entry min/max, exit min/max:", [f(t[28, 0]), f(t[29, 5]), f(t[28, 1]), f(t[29, 6])])
print("merge: copied/spun/loaded:", [f(t[30, k]) for k in (2, 3, 4)])
names = ["tmaK", "S:issue", "PV:issue", "sm:s_full", "sm:fast", "sm:p_wait", "sm:p_arrive", "sm:slow"]
for i in range(29):
    if any(int(t[i, k]) for k in range(8)):
        print(f"{i:2d}", " ".join(f"{n}={f(t[i, k])}" for k, n in enumerate(names)))
