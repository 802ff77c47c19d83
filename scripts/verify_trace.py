"""Phase stamps (globaltimer) of attention CTA (0,0,0) + combine block 0 inside the
captured verify graph (the last layer's stamps survive).  Needs a BST_TRACE=1 build
(BASTION_LIB=<trace lib>)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import _lib  # noqa: E402
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 31
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
trace_y = int(sys.argv[3]) if len(sys.argv) > 3 else 0
eng = B200Engine(QWEN3_8B, DrafterConfig(layers=5, gamma=16, logit_scale=6.0), max_ctx=ctx + 2048, n_cap=255)
eng.reset(np.random.default_rng(0).integers(0, QWEN3_8B.V - 1, ctx + 1).tolist())
eng.set_policy("fixed", n=n)
saved = eng.state.clone()
eng.cycle()
lib = _lib.lib()
tr = torch.zeros(32 * 8, dtype=torch.int64, device="cuda")
lib.bst_debug_attn_trace.argtypes = [C.c_void_p]
lib.bst_debug_attn_trace(tr.data_ptr())
lib.bst_debug_attn_trace_cta(trace_y)
for _ in range(3):
    eng.state.copy_(saved)
    eng.cycle()
torch.cuda.synchronize()
t = tr.view(32, 8).cpu().numpy()
t0 = t[31, 0]
f = lambda v: f"{(v - t0) / 1000:7.2f}" if v else "   -   "
print("cta  entry/setup/depwait/q_ready/epi_start/epi_end:", " ".join(f(v) for v in t[31, :6]))
print("all CTAs max depwait/staged/end/arrive/spin_done:", " ".join(f(v) for v in t[29, :5]))
print("combine start/end:", " ".join(f(v) for v in t[30, :2]))
names = ["tma", "mma:S", "mma:PV", "s_full", "sm_done", "o_wait", "p_arrive", "s_read"]
for i in range(4):
    print(i, " ".join(f"{nm}={f(t[i, k])}" for k, nm in enumerate(names)))
