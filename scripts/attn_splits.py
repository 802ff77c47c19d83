"""K3 time vs forced split count (c, s from argv)."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import ops  # noqa: E402
from paper_2605_29727_b200.engine.forward import PagedKV  # noqa: E402

c, s = int(sys.argv[1]), int(sys.argv[2])
n_q, n_kv = 32, 8
kv = PagedKV(1, n_kv, c + 320, "cuda")
kv.buf.normal_(0, 1)
q = torch.randn(s, n_q * 128, device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
words = (s + 31) // 32
anc = torch.full((s, words), -1, dtype=torch.int32, device="cuda")
ws = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
import os
from paper_2605_29727_b200 import _lib  # noqa: E402
_lib.lib().bst_debug_kt_ablate(int(os.environ.get("KT_ABLATE", "0")))
for sp in [int(x) for x in sys.argv[3:]]:
    ts = []
    for it in range(15):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ops.attention(q, out, kv.buf, 1, kv.n_pages, 0, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0,
                      anc.view(-1), words, ws, n_splits=sp)
        b.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    print(json.dumps({"ablate": os.environ.get("KT_ABLATE", "0"), "c": c, "s": s, "splits": sp, "us": round(statistics.median(ts), 2)}), flush=True)
