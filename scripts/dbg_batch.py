import sys; sys.path.insert(0, '.')
import numpy as np, torch
sys.path.insert(0, 'tests')
from test_gpu_batch import _prompts
from paper_2605_29727_b200.engine.batch import BatchEngine
from paper_2605_29727_b200.engine.decode import B200Engine
from paper_2605_29727_b200.engine.config import TINY, DrafterConfig
dcfg = DrafterConfig(layers=2, gamma=8, logit_scale=4.0)
n_req, N = 16, 4
prompts = _prompts(n_req, 150, TINY.V)
refs = {}
for g in (True, False):
    eng = B200Engine(TINY, dcfg, max_ctx=640, seed=0, n_cap=64)
    eng.target.attn_splits = 1; eng.drafter.attn_splits = 1; eng.use_graphs = g
    eng.set_policy("fixed", n=N)
    out = []
    for p in prompts:
        eng.reset(p)
        for _ in range(6): eng.cycle()
        eng.stream.synchronize()
        out.append((eng.tokens(), eng.log_f64[:6].cpu().numpy().copy()))
    refs[g] = out
for graphs in (True, False):
    be = BatchEngine(TINY, dcfg, n_req=n_req, n_fixed=N, max_ctx=640, seed=0)
    be.set_attention_splits(1); be.use_graphs = graphs
    be.reset(prompts)
    for _ in range(6): be.cycle()
    be.stream.synchronize()
    for rg in (True, False):
        ref = refs[rg]
        bad = [(r, np.nonzero(be.log_f64[r, :6].cpu().numpy() != ref[r][1])[0].tolist()) for r in range(n_req)
               if not np.array_equal(be.log_f64[r, :6].cpu().numpy(), ref[r][1])]
        print("batch graphs", graphs, "vs single graphs", rg, "mismatch (r, cycles):", bad)
print("single graph vs eager:", [r for r in range(n_req) if not np.array_equal(refs[True][r][1], refs[False][r][1])])
