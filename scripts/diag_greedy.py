import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2605_29727_b200.engine.config import TINY, DrafterConfig  # noqa: E402
from paper_2605_29727_b200.engine.decode import B200Engine  # noqa: E402
from test_gpu_engine import GAMMA, _decoy_drafter, _prompt  # noqa: E402

eng = B200Engine(TINY, DrafterConfig(layers=2, gamma=GAMMA, logit_scale=4.0), max_ctx=640, seed=0, n_cap=64)
prompt = _prompt(70, eng.cfg.V, seed=3)
eng.reset(prompt)
ar = eng.ar_decode(80)
eng.reset(prompt)
eng.set_policy("fixed", n=48)
eng.draft_override = _decoy_drafter(ar, GAMMA, eng.cfg.V, 0)
eng.use_graphs = False
stats, toks = eng.run(60)
mism = [i for i in range(60) if toks[i] != ar[i]]
print("mismatch at", mism[:5], "accepted", [s.accepted_len for s in stats][:12])
