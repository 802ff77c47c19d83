"""Diagnostic: ragged batch engine (n_req=1, adaptive) vs the single-request engine, cycle by cycle."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_2605_29727_b200 as P  # noqa: E402
from paper_2605_29727_b200.engine.batch import BatchEngine  # noqa: E402
from paper_2605_29727_b200.engine.config import QWEN3_8B, TINY, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402

dcfg = DrafterConfig(layers=2, gamma=8, logit_scale=4.0)
params = QWEN3_8B.cost_params(1649.1e12, 6457.7e9)
est = P.VerifyLatencyEstimator(params, variant="static")
lat = P.CycleLatencies(t_draft=3e-4, t_aux=2e-5, l_ar=est.estimate(1, 1000))
prompt = np.random.default_rng(100).integers(0, TINY.V - 1, 150).tolist()
eng = B200Engine(TINY, dcfg, max_ctx=640, seed=0, n_cap=48)
eng.target.attn_splits = eng.drafter.attn_splits = 1
eng.set_policy("adaptive", estimator=est, latencies=lat, n_max=48)
eng.reset(prompt)
eng.use_graphs = False
be = BatchEngine(TINY, dcfg, n_req=1, n_fixed=48, max_ctx=640, seed=0)
be.set_attention_splits(1)
be.use_graphs = False
be.set_policy("adaptive", estimator=est, latencies=lat)
be.reset([prompt])
for cyc in range(8):
    n1, _ = eng.draft()
    with torch.cuda.stream(be.stream):
        be._draft_ragged()
    be.stream.synchronize()
    n2 = int(be.trees[0].meta[0].item())
    same_tree = n1 == n2 and torch.equal(eng.tree.token[:n1 + 1], be.trees[0].token[:n2 + 1])
    lat_same = torch.equal(eng.lat_prob, be.lat_prob[1:9])
    eng.verify(n1)
    eng.stream.synchronize()
    total = int(be.row_total.item())
    with torch.cuda.stream(be.stream):
        be._verify_ragged(-(-total // 64) * 64)
    be.stream.synchronize()
    a1 = eng.target.argmax[: n1 + 1].cpu().numpy()
    a2 = be.argmax_u[: n2 + 1].cpu().numpy()
    print(f"cyc {cyc}: n {n1} {n2} same_tree {same_tree} lattice_same {lat_same} total {total} "
          f"argmax_equal {np.array_equal(a1, a2) if n1 == n2 else None} acc {int(eng.acc_meta[0])} {int(be.acc_meta[0, 0])} "
          f"c {int(eng.state[0])} {int(be.state[0, 0])}")
    if n1 == n2 and not np.array_equal(a1, a2):
        d = np.nonzero(a1 != a2)[0]
        print("  argmax differs at rows", d[:10], a1[d[:10]], a2[d[:10]])
