"""Greedy output preservation at the Qwen3-8B shape: tree decode
(drafter proposing the target's greedy tokens among decoys, so accepted paths are
non-contiguous and KV compaction really moves rows) vs the engine's autoregressive decode.
Reports the first position where they differ (bf16 numerics: tree rows and AR rows reduce
the same keys in different tile positions, so near-ties may flip).  argv: context tokens."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29727_b200.engine.config import QWEN3_8B, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
n_tok = int(sys.argv[2]) if len(sys.argv) > 2 else 64
n_prompts = int(sys.argv[3]) if len(sys.argv) > 3 else 6
G = 16
eng = B200Engine(QWEN3_8B, DrafterConfig(layers=5, gamma=G, logit_scale=6.0), max_ctx=ctx + 1024, seed=0, n_cap=255)
rng = np.random.default_rng(0)
ar: list = []
import os  # noqa: E402
if os.environ.get("ATTN_SPLITS"):  # pin the K3 split count for both paths (split-independence probe)
    eng.target.attn_splits = int(os.environ["ATTN_SPLITS"])


def decoy(e):
    k = int(e.state[3].item())
    lg = torch.zeros(G, QWEN3_8B.V, device="cuda")
    for j in range(G):
        lg[j, int(rng.integers(0, QWEN3_8B.V))] = 10.3
        if k + j < len(ar):
            lg[j, ar[k + j]] = 10.0
    return lg


firsts, accepts = [], []
for seed in range(n_prompts):
    prompt = np.random.default_rng(100 + seed).integers(0, QWEN3_8B.V - 1, ctx + 1).tolist()
    eng.reset(prompt)
    ar = eng.ar_decode(n_tok + G + 1)
    eng.reset(prompt)
    eng.set_policy("fixed", n=48)
    eng.draft_override = decoy
    stats, toks = eng.run(n_tok)
    eng.draft_override = None
    first = next((i for i in range(n_tok) if toks[i] != ar[i]), None)
    firsts.append(n_tok if first is None else first)
    k = next((i for i, s in enumerate(stats) if sum(x.accepted_len for x in stats[:i + 1]) > firsts[-1]), len(stats))
    accepts.append(float(np.mean([s.accepted_len for s in stats[:max(k, 1)]])))
print(json.dumps({"context": ctx, "tokens_per_prompt": n_tok, "prompts": n_prompts,
                  "equal_prefix_lengths": firsts, "identical_runs": sum(f == n_tok for f in firsts),
                  "mean_accept_len_before_divergence": accepts}))
