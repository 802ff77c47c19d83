"""Launch the K4 GEMM at verify shapes (for ncu --set full)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200 import ops  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 48
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n, k in [(6144, 4096), (4096, 4096), (24576, 4096), (4096, 12288), (151936, 4096)]:
    w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        flush.zero_()
        ops.gemm_partial(x, w)
    torch.cuda.synchronize()
