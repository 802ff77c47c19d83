"""K3 tree-verify attention vs its HBM roofline (config 4: c up to 32K, tree budget sweep).

bytes per layer (fused minimum) = bp * (2 (c+s) h_kv + 2 s h_q) + mask;
flops per layer = 4 s (c+s) h_q.  Timed with CUDA events over one launch (+combine),
median of 20, L2 flushed between launches (the KV of one layer at c=32K is 134 MB).
"""
import json
import math
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import ops  # noqa: E402
from paper_2605_29727_b200.engine.forward import PagedKV  # noqa: E402

peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
BW, PF = peaks["hbm_gbs"] * 1e9, peaks["bf16_tflops"] * 1e12
n_q, n_kv = 32, 8
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for c in [int(x) for x in (sys.argv[1:] or ["2048", "32768"])]:
    kv = PagedKV(1, n_kv, c + 320, "cuda")
    kv.buf.normal_(0, 1)
    for s in (17, 33, 65, 129, 257):
        q = torch.randn(s, n_q * 128, device="cuda").to(torch.bfloat16)
        out = torch.empty_like(q)
        words = (s + 31) // 32
        anc = torch.zeros(s, words, dtype=torch.int32, device="cuda")
        # chain-of-siblings tree: every row sees the root and itself
        for i in range(s):
            anc[i, 0] |= 1
            anc[i, i // 32] |= (1 << (i % 32)) if (i % 32) != 31 else -(1 << 31)
        ws = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
        ts = []
        for it in range(23):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ops.attention(q, out, kv.buf, 1, kv.n_pages, 0, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0,
                          anc.view(-1), words, ws)
            b.record()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b) * 1e-3)
        t = statistics.median(ts)
        byts = 2 * (2 * (c + s) * n_kv * 128 + 2 * s * n_q * 128) + s * words * 4
        flops = 4 * s * (c + s) * n_q * 128
        t_roof = max(byts / BW, flops / PF)
        r = dict(c=c, s=s, us=round(t * 1e6, 2), GBps=round(byts / t / 1e9, 1), tflops=round(flops / t / 1e12, 1),
                 roofline_us=round(t_roof * 1e6, 2), frac=round(t_roof / t, 3),
                 bound="hbm" if byts / BW >= flops / PF else "tensor")
        res.append(r)
        print(json.dumps(r), flush=True)
