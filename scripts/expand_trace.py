import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import _lib  # noqa: E402
from paper_2605_29727_b200.draft_tree import DeviceTree, expand_device  # noqa: E402
from paper_2605_29727_b200.lattice import lattice_from_logits  # noqa: E402

lib = _lib.lib()
lib.bst_debug_expand_trace.argtypes = [C.c_void_p]
tr = torch.zeros(16, dtype=torch.int64, device="cuda")
logits = torch.randn(16, 151936, device="cuda") * 6  # fp32, as the engine's LM head
tok, prob = lattice_from_logits(logits, 8)
for n, cap in ((31, 255), (111, 1024), (255, 1024), (1024, 1024)):
    dt = DeviceTree(cap)
    expand_device(tok, prob, _lib.Plan(policy=_lib.POLICY_FIXED, n_max=n), cap, dt)
    torch.cuda.synchronize()
    lib.bst_debug_expand_trace(tr.data_ptr())
    expand_device(tok, prob, _lib.Plan(policy=_lib.POLICY_FIXED, n_max=n), cap, dt)
    torch.cuda.synchronize()
    lib.bst_debug_expand_trace(None)
    t = tr.cpu().tolist()
    names = ["dp", "enumerate", "sort", "ties", "output", "finish"]
    print(n, "cap", cap, "enum", int(dt.meta[4].item()), " ".join(f"{nm}={(t[i + 1] - t[i]) / 1000:.1f}us" for i, nm in enumerate(names)))
