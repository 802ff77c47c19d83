"""One K3 launch at (c, s) for ncu."""
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
for _ in range(3):
    ops.attention(q, out, kv.buf, 1, kv.n_pages, 0, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0, anc.view(-1),
                  words, ws)
torch.cuda.synchronize()
