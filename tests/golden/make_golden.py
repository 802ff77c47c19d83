"""Generate golden vectors by running the REAL reference ``specplan`` package.

Run in the build container (the reference is not present on the GPU box):

    python tests/golden/make_golden.py            # BASTION_REF_PATH defaults to /root/reference/pkg/src

Every fixture stores the inputs and the reference's outputs bit-exactly
(floats as hex / raw float64 bytes), so the oracle port and the CUDA path can
both be pinned against them without the reference at run time.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from codec import enc, fhex, save  # noqa: E402

REF = os.environ.get("BASTION_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True

import specplan as sp  # noqa: E402
from specplan import cost_model as spc  # noqa: E402
from specplan import verify_sim as spv  # noqa: E402

QWEN3_8B = dict(L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288, V=151936, bp=2)
QWEN3_32B = dict(L=64, h=5120, n_q=64, n_kv=8, d=128, h_ffn=25600, V=151936, bp=2)
TOY = dict(L=2, h=64, n_q=4, n_kv=2, d=16, h_ffn=128, V=256, bp=2)
B200 = dict(peak_flops=1649.1e12, bandwidth=6457.7e9)
PROFILES = {
    "qwen3_8b_b200": sp.CostModelParams(**QWEN3_8B, **B200),
    "qwen3_32b_b200": sp.CostModelParams(**QWEN3_32B, **B200),
    "toy": sp.CostModelParams(**TOY, peak_flops=1e13, bandwidth=1e11),
    "toy_huge": sp.CostModelParams(**TOY, peak_flops=1e18, bandwidth=1e17),
    "crossover": spc.load_params(Path(REF).parent / "profiles" / "crossover.txt"),
    "memory_bound": spc.load_params(Path(REF).parent / "profiles" / "memory_bound.txt"),
    "compute_bound": spc.load_params(Path(REF).parent / "profiles" / "compute_bound.txt"),
}


def params_dict(p) -> dict:
    return {k: getattr(p, k) for k in ("L", "h", "n_q", "n_kv", "d", "h_ffn", "V", "bp")} | {
        "peak_flops": fhex(p.peak_flops), "bandwidth": fhex(p.bandwidth)}


def tree_rows(tree) -> dict:
    """Flat arrays (root row included) — parent/depth/token int32, rho float64."""
    ns = tree.nodes
    return {"parent": enc(np.array([-1 if n.parent is None else n.parent for n in ns], dtype=np.int32)),
            "depth": enc(np.array([n.depth for n in ns], dtype=np.int32)),
            "token": enc(np.array([-1 if n.token is None else n.token for n in ns], dtype=np.int32)),
            "rho": enc(np.array([n.path_score for n in ns], dtype=np.float64))}


def lattice_arrays(lat):
    tok = np.array([[t for t, _ in row] for row in lat.entries], dtype=np.int32)
    prob = np.array([[p for _, p in row] for row in lat.entries], dtype=np.float64)
    return tok, prob


# --------------------------------------------------------------------------- blocks
def bf16_round(x: np.ndarray) -> np.ndarray:
    b = np.asarray(x, dtype=np.float32).view(np.uint32)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return b.view(np.float32)


def softmax64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    x = x - x.max(axis=1, keepdims=True)
    w = np.exp(x)
    return w / w.sum(axis=1, keepdims=True)


def make_blocks(rng: np.random.Generator) -> list[tuple[str, np.ndarray]]:
    out = [
        ("spec_topk_1", np.array([[0.5, 0.3, 0.2]])),
        ("spec_topk_2", np.array([[0.4, 0.4, 0.2]])),
        ("spec_topk_3", np.array([[0.1, 0.2, 0.3, 0.4], [0.25, 0.25, 0.25, 0.25]])),
        ("spec_lattice_2x2", np.array([[0.6, 0.3, 0.1], [0.7, 0.2, 0.1]])),
        ("one_hot", np.eye(5)[[2, 0, 4, 1]]),
    ]
    for i in range(12):
        g, v = int(rng.integers(1, 7)), int(rng.integers(2, 13))
        out.append((f"dirichlet_{i}", rng.dirichlet(np.full(v, 0.7), size=g)))
    for i in range(8):  # integer-count rows: many exact ties and zeros
        g, v = int(rng.integers(2, 9)), int(rng.integers(4, 40))
        cnt = rng.integers(0, 4, size=(g, v)).astype(np.float64)
        cnt[:, 0] += 1.0
        out.append((f"ties_{i}", cnt / cnt.sum(axis=1, keepdims=True)))
    for i, scale in enumerate((1.0, 3.0, 6.0, 10.0)):  # bf16-quantized logits, drafter-like
        lg = bf16_round(rng.standard_normal((16, 512)) * scale)
        out.append((f"bf16_g16_v512_s{int(scale)}", softmax64(lg)))
    lg = bf16_round(rng.standard_normal((24, 64)) * 2.0)
    out.append(("bf16_g24_v64", softmax64(lg)))
    return out


# --------------------------------------------------------------------------- families
def gen_lattice_and_trees(rng):
    cases = []
    for name, probs in make_blocks(rng):
        block = sp.MarginalBlock(gamma=probs.shape[0], vocab_size=probs.shape[1], probs=probs)
        V = probs.shape[1]
        ks = sorted({1, min(2, V), min(3, V), min(8, V), V if V <= 16 else 16})
        for k in ks:
            lat = sp.top_k_truncate(block, k)
            tok, prob = lattice_arrays(lat)
            case = {"name": f"{name}_k{k}", "probs": enc(probs), "k": k,
                    "tok": enc(tok), "prob": enc(prob), "reachable": lat.reachable_size(),
                    "best_first": [], "beam": []}
            if prob[0, 0] > 0.0:
                for n in (1, 2, 3, 5, 17, 64, 300, 1100):
                    t = sp.best_first_expand(lat, n)
                    case["best_first"].append({"n_max": n, "nodes": tree_rows(t),
                                               "surrogate": fhex(t.surrogate)})
                g = block.gamma
                for w, d in {(1, g), (2, min(2, g)), (4, min(15, g)), (3, 1), (8, g), (64, min(4, g))}:
                    t = sp.beam_expand(lat, w, d)
                    case["beam"].append({"width": w, "depth": d, "nodes": tree_rows(t),
                                         "surrogate": fhex(t.surrogate)})
            cases.append(case)
    save("lattice_trees", {"cases": cases})
    return cases


def gen_controller(rng, lattice_cases):
    picks = [c for c in lattice_cases if c["name"].startswith(("bf16_", "dirichlet_1", "spec_lattice"))]
    runs = []
    fit = sp.CalibrationFit(slope=1.3, intercept=2e-4, rmse_before=0.0, rmse_after=0.0)
    bias = sp.EmaBias(ratio_bias=1.7, alpha=0.1)
    from codec import dec
    for case in picks:
        tok, prob = dec(case["tok"]), dec(case["prob"])
        if prob[0, 0] <= 0.0:
            continue
        lat = sp.CandidateLattice(
            source=sp.MarginalBlock(gamma=tok.shape[0], vocab_size=int(dec(case["probs"]).shape[1]),
                                    probs=dec(case["probs"])),
            top_k=case["k"],
            entries=tuple(tuple((int(t), float(p)) for t, p in zip(tr, pr)) for tr, pr in zip(tok, prob)))
        for pname in ("qwen3_8b_b200", "toy", "crossover", "toy_huge"):
            p = PROFILES[pname]
            for c in (0, 2048, 32768):
                for variant, f, b in (("static", None, None), ("static", fit, None),
                                      ("ema", None, bias), ("ema_calib", fit, bias)):
                    est = sp.VerifyLatencyEstimator(p, variant=variant, fit=f, bias=b)
                    l_ar = spc.roofline_latency(p, sp.LatencyQuery(s=1, c=c))
                    for t_draft, t_aux in ((0.0, 0.0), (3e-4, 1e-5)):
                        for n_max in (1, 16, 1024):
                            if rng.random() < 0.85:
                                continue
                            lat_ = sp.CycleLatencies(t_draft=t_draft, t_aux=t_aux, l_ar=l_ar)
                            cfg = sp.ControllerConfig(n_max=n_max, latencies=lat_, variant=variant,
                                                      context_len=c)
                            dcs = sp.run_cycle(lat, cfg, est)
                            runs.append({
                                "lattice": case["name"], "profile": pname, "c": c, "variant": variant,
                                "slope": fhex(est.fit.slope) if est.fit else None,
                                "intercept": fhex(est.fit.intercept) if est.fit else None,
                                "ratio": fhex(est.bias.ratio_bias) if est.bias else None,
                                "t_draft": fhex(t_draft), "t_aux": fhex(t_aux), "l_ar": fhex(l_ar),
                                "n_max": n_max, "budget": dcs.budget, "stop": dcs.stop_reason,
                                "trace": enc(np.array(dcs.s_hat_trace, dtype=np.float64)),
                                "nodes": tree_rows(dcs.tree), "surrogate": fhex(dcs.tree.surrogate)})
    save("controller", {"profiles": {k: params_dict(v) for k, v in PROFILES.items()}, "runs": runs})


def gen_cost(rng):
    fit = sp.CalibrationFit(slope=0.85, intercept=-1e-5, rmse_before=0.0, rmse_after=0.0)
    bias = sp.EmaBias(ratio_bias=0.93, alpha=0.25)
    rows = []
    for pname, p in PROFILES.items():
        for c in (0, 1, 255, 2048, 32768):
            for variant, f, b in (("static", None, None), ("static", fit, None), ("ema", None, bias),
                                  ("ema_calib", fit, bias)):
                est = sp.VerifyLatencyEstimator(p, variant=variant, fit=f, bias=b)
                curve = est.curve(c)
                ss = sorted({1, 2, 3, 17, 64, 65, 129, 257, 513, 1025} | set(rng.integers(1, 1026, 12).tolist()))
                rows.append({
                    "profile": pname, "c": c, "variant": variant,
                    "slope": fhex(est.fit.slope) if est.fit else None,
                    "intercept": fhex(est.fit.intercept) if est.fit else None,
                    "ratio": fhex(est.bias.ratio_bias) if est.bias else None,
                    "s": ss,
                    "curve": [fhex(curve.latency(s)) for s in ss],
                    "estimate": [fhex(est.estimate(s, c)) for s in ss],
                    "flops": [str(spc.flops(p, sp.LatencyQuery(s=s, c=c))) for s in ss],
                    "bytes": [str(spc.bytes_moved(p, sp.LatencyQuery(s=s, c=c))) for s in ss],
                    "weights": [str(spc.weights_bytes(p, sp.LatencyQuery(s=s, c=c))) for s in ss],
                    "kv": [str(spc.kv_cache_bytes(p, sp.LatencyQuery(s=s, c=c))) for s in ss],
                    "act": [str(spc.activation_bytes(p, sp.LatencyQuery(s=s, c=c))) for s in ss],
                    "roofline": [fhex(spc.roofline_latency(p, sp.LatencyQuery(s=s, c=c))) for s in ss],
                })
    # EMA + OLS
    ema = []
    for _ in range(40):
        b = sp.EmaBias(ratio_bias=float(rng.uniform(0.2, 3)), alpha=float(rng.uniform(0.01, 1.0)))
        pr, ob = float(rng.uniform(1e-4, 1e-2)), float(rng.uniform(1e-4, 1e-2))
        ema.append([fhex(b.ratio_bias), fhex(b.alpha), fhex(pr), fhex(ob), fhex(sp.ema_update(b, pr, ob).ratio_bias)])
    ols = []
    for _ in range(20):
        n = int(rng.integers(2, 30))
        pairs = [(float(x), float(2.0 * x + 1e-3 + rng.normal(0, 1e-4))) for x in rng.uniform(1e-3, 1e-2, n)]
        f = sp.fit_static_calibration(pairs)
        ols.append({"pairs": [[fhex(a), fhex(b)] for a, b in pairs],
                    "fit": [fhex(f.slope), fhex(f.intercept), fhex(f.rmse_before), fhex(f.rmse_after)]})
    save("cost_model", {"profiles": {k: params_dict(v) for k, v in PROFILES.items()}, "rows": rows,
                        "ema": ema, "ols": ols})


def gen_replay(rng):
    out = []
    for _ in range(200):
        n = int(rng.integers(1, 40))
        gains = list(np.sort(rng.random(n))[::-1])
        costs = list(1.0 + np.cumsum(np.cumsum(rng.random(n) * 0.2)))
        l_ar = float(rng.uniform(0.5, 2.0))
        d = sp.replay_trace(gains, costs, l_ar)
        out.append({"gains": [fhex(g) for g in gains], "costs": [fhex(c) for c in costs], "l_ar": fhex(l_ar),
                    "budget": d.budget, "stop": d.stop_reason, "trace": [fhex(x) for x in d.s_hat_trace]})
    # SPEC controller example and tie handling
    for gains, costs in (([0.60, 0.42, 0.30, 0.21, 0.12, 0.06], [1 + 0.15 * n for n in range(1, 7)]),
                         ([1, .5, .1], [2, 2.5, 4]), ([1, .5, .5], [2, 2.5, 2.5])):
        d = sp.replay_trace(gains, costs, 1.0)
        out.append({"gains": [fhex(g) for g in gains], "costs": [fhex(c) for c in costs], "l_ar": fhex(1.0),
                    "budget": d.budget, "stop": d.stop_reason, "trace": [fhex(x) for x in d.s_hat_trace]})
    save("replay", {"cases": out})


def gen_linearize(rng):
    from codec import dec
    cases = []
    lat_cases = __import__("codec").load("lattice_trees")["cases"]
    for case in lat_cases[:30]:
        if not case["best_first"]:
            continue
        probs = dec(case["probs"])
        block = sp.MarginalBlock(gamma=probs.shape[0], vocab_size=probs.shape[1], probs=probs)
        lat = sp.top_k_truncate(block, case["k"])
        tree = sp.best_first_expand(lat, int(rng.integers(1, 40)))
        for prefix_len in (0, 3):
            lin = sp.linearize(tree, prefix_len)
            cases.append({"nodes": tree_rows(tree), "prefix_len": prefix_len, "tokens": list(lin.tokens),
                          "position_ids": list(lin.position_ids), "parents": list(lin.parents),
                          "mask": enc(np.packbits(lin.mask, axis=1)), "mask_shape": list(lin.mask.shape)})
    save("linearize", {"cases": cases})


class RecordingRule:
    """Wraps a reference TargetRule and records every plugin answer (replay tables)."""

    def __init__(self, rule):
        self.rule = rule
        self.blocks: dict[tuple, np.ndarray] = {}
        self.choices: dict[tuple, int] = {}

    def drafter_marginals(self, prefix):
        b = self.rule.drafter_marginals(prefix)
        self.blocks[tuple(prefix)] = np.array(b.probs)
        return b

    def next_token(self, prefix, temperature):
        t = self.rule.next_token(prefix, temperature)
        self.choices[tuple(prefix)] = int(t)
        return t


def gen_decode():
    runs = []
    p = PROFILES["crossover"]
    for gamma, V, seed, run_length in ((16, 64, 3, 48), (6, 32, 11, 40), (16, 48, 7, 40)):
        for pol in ("adaptive", "fixed-16", "fixed-64", "greedy-chain", "beam-4x5"):
            pair_cfg = sp.SyntheticPairConfig(gamma=gamma, vocab_size=V, alignment=0.8, concentration=0.1,
                                              seed=seed)
            rec = RecordingRule(spv.TargetRule.from_config(pair_cfg))
            est = sp.VerifyLatencyEstimator(p, variant="static")
            context_len = 256
            l_ar = spc.roofline_latency(p, sp.LatencyQuery(s=1, c=context_len))
            lat = sp.CycleLatencies(t_draft=2e-4, t_aux=1e-5, l_ar=l_ar)
            cfg = sp.SimConfig(controller=sp.ControllerConfig(n_max=1024, latencies=lat, variant="static",
                                                              context_len=context_len),
                               run_length=run_length, top_k=8, temperature=0.0)
            policy = sp.Policy.parse(pol)
            records, tokens = spv.decode_full(rec, cfg, policy, est)
            ar = sp.ar_decode(spv.TargetRule.from_config(pair_cfg), len(tokens))
            runs.append({
                "gamma": gamma, "V": V, "seed": seed, "policy": pol, "run_length": run_length,
                "context_len": context_len, "profile": "crossover", "t_draft": fhex(2e-4), "t_aux": fhex(1e-5),
                "l_ar": fhex(l_ar), "n_max": 1024, "top_k": 8,
                "records": [[r.tree_size, r.accepted_len, fhex(r.surrogate), fhex(r.t_draft), fhex(r.t_verify),
                             fhex(r.t_aux), fhex(r.l_ar), fhex(r.cycle_speedup)] for r in records],
                "tokens": list(tokens), "ar_tokens": list(ar),
                "realized_speedup": fhex(sp.realized_speedup(records)),
                "blocks": [[list(k), enc(v)] for k, v in rec.blocks.items()],
                "choices": [[list(k), v] for k, v in rec.choices.items()],
            })
    save("decode", {"runs": runs})


def main() -> None:
    rng = np.random.default_rng(20260517)
    lattice_cases = gen_lattice_and_trees(rng)
    gen_controller(rng, lattice_cases)
    gen_cost(rng)
    gen_replay(rng)
    gen_linearize(rng)
    gen_decode()
    print("golden fixtures written to", Path(__file__).resolve().parent)


if __name__ == "__main__":
    main()
