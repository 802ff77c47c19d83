"""K3 per-layer time inside a CUDA graph of L back-to-back launches (one per layer, as in
the verify forward; every layer's KV is distinct, 36 x 134 MB at c=32K >> L2, no flush).
Prints per-launch time and the fraction of the per-layer HBM roofline."""
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import ops  # noqa: E402
from paper_2605_29727_b200.engine.forward import PagedKV  # noqa: E402

peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
BW, PF = peaks["hbm_gbs"] * 1e9, peaks["bf16_tflops"] * 1e12
c = int(sys.argv[1])
L = 36
n_q, n_kv = 32, 8
kv = PagedKV(L, n_kv, c + 320, "cuda")
kv.buf.normal_(0, 1)
ws = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
st = torch.cuda.Stream()
for s in [int(x) for x in sys.argv[2:]] or [17, 33, 65, 129, 257]:
    q = torch.randn(s, n_q * 128, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    words = (s + 31) // 32
    anc = torch.zeros(s, words, dtype=torch.int32, device="cuda")
    for i in range(s):
        anc[i, 0] |= 1
        anc[i, i // 32] |= (1 << (i % 32)) if (i % 32) != 31 else -(1 << 31)

    def run():
        for li in range(L):
            ops.attention(q, out, kv.buf, L, kv.n_pages, li, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0,
                          anc.view(-1), words, ws, n_splits=int(os.environ.get("SPLITS", "0")))
    with torch.cuda.stream(st):
        run()
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        run()
    ts = []
    for it in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        with torch.cuda.stream(st):
            g.replay()
        b.record(st)
        b.synchronize()
        if it >= 2:
            ts.append(a.elapsed_time(b) * 1e-3 / L)
    t = statistics.median(ts)
    byts = 2 * (2 * (c + s) * n_kv * 128 + 2 * s * n_q * 128) + s * words * 4
    flops = 4 * s * (c + s) * n_q * 128
    t_roof = max(byts / BW, flops / PF)
    print(json.dumps(dict(c=c, s=s, us_per_layer=round(t * 1e6, 2), GBps=round(byts / t / 1e9, 1),
                          roofline_us=round(t_roof * 1e6, 2), frac=round(t_roof / t, 3),
                          bound="hbm" if byts / BW >= flops / PF else "tensor")), flush=True)
