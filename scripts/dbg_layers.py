import sys, torch
sys.path.insert(0, '.')
from paper_2605_29727_b200 import ops
from paper_2605_29727_b200.engine.forward import PagedKV
c, L = int(sys.argv[1]), int(sys.argv[2])
n_q, n_kv, s = 32, 8, 17
kv = PagedKV(L, n_kv, c + 320, "cuda"); kv.buf.normal_(0, 1)
ws = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
q = torch.randn(s, n_q * 128, device="cuda").to(torch.bfloat16); out = torch.empty_like(q)
anc = torch.full((s, 1), -1, dtype=torch.int32, device="cuda")
for li in range(L):
    ops.attention(q, out, kv.buf, L, kv.n_pages, li, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0, anc.view(-1), 1, ws)
    torch.cuda.synchronize()
    print("ok layer", li, flush=True)
