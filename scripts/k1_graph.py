"""K1 (top-K lattice of the drafter logits, gamma x V) in steady state: CUDA graph of 20
back-to-back launches on distinct fp32 logit blocks (as the draft graph feeds it)."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200.lattice import topk_logits_into  # noqa: E402

gamma, V, k, N = 16, 151936, 8, 20
logits = [(torch.randn(gamma, V, device="cuda") * 6) for _ in range(N)]
tok = torch.empty(gamma, k, dtype=torch.int32, device="cuda")
prob = torch.empty(gamma, k, dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()


def run():
    for lg in logits:
        topk_logits_into(lg, k, tok, prob, None)


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
        ts.append(a.elapsed_time(b) * 1e3 / N)
print(json.dumps({"k1_us_per_launch": round(statistics.median(ts), 2), "gamma": gamma, "V": V, "k": k}))
