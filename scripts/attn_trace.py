import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import _lib, ops  # noqa: E402
from paper_2605_29727_b200.engine.forward import PagedKV  # noqa: E402

c, s = int(sys.argv[1]), int(sys.argv[2])
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
lib.bst_debug_attn_trace.argtypes = [C.c_void_p]
lib.bst_debug_attn_trace(tr.data_ptr())
if len(sys.argv) > 3:
    lib.bst_debug_attn_trace_cta(int(sys.argv[3]))
run()
torch.cuda.synchronize()
t = tr.view(32, 8).cpu()
t0 = int(t[31, 1])  # kernel entry of the traced CTA
rel = lambda i, k: round((int(t[i, k]) - t0) / 1000, 2) if int(t[i, k]) else None
print("row31:", [rel(31, k) for k in range(8)], "row30:", [rel(30, k) for k in range(8)])
print("entry->depwait/q_ready/staged/exit:", [round((int(t[31, k]) - t0) / 1000, 2) for k in (2, 3, 5, 0)])
print("all CTAs max depwait/staged/end/arrive/spin_done:", [round((int(t[29, k]) - t0) / 1000, 2) for k in range(5)])
names = ["tma_issued", "mma:full", "mma:p_full", "sm:s_full", "sm:sm_done", "sm:o_done", "sm:p_arrive", "sm:max_local"]
for i in range(min(32, 30)):
    print(i, " ".join(f"{n}={(int(t[i, k]) - t0) / 1000:8.2f}" if int(t[i, k]) else f"{n}=   -    " for k, n in enumerate(names)))
