"""Benchmark: BASTION tree-speculative decode on B200 (BASELINE.json config 2).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

A "step" is one decode cycle of the hot path: drafter forward -> K1 top-K
lattice -> K2 adaptive best-first expansion (Algorithm 1) -> tree-masked
target verify -> K6 greedy accept + KV compaction.  Workload (config 2):
Qwen3-8B-shape target + DFlash-style 5-layer drafter, random-init bf16,
batch 1, 2048-token synthetic prompt, gamma 16, K 8, adaptive budget.
N > 1 (torchrun): one independent request per rank, no collective on the data
path (weak scaling); time = max over ranks of the device-timed region.

Prints ONE JSON line (rank 0).  `--impl reference` times the reference's
planning path (the CPU oracle port of specplan) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode tokens/s + tree-verify µs/step (Qwen3-8B shape, greedy); mean accept len"
WORKLOAD = ("config2: Qwen3-8B-shape target + DFlash-style 5-layer block drafter, random-init bf16, batch 1 "
            "per GPU, 2048-token context, gamma 16, top-K 8, adaptive budget (Algorithm 1, N_max 1024)")


_T0 = time.time()


def _log(msg: str) -> None:
    """Phase progress on stderr (the JSON line stays alone on stdout)."""
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback"}


# --------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc = index, None

    def __enter__(self):
        # 50 ms sampling, and the timed region starts only once nvidia-smi has printed its
        # first sample: a short region (40 cycles ~ 0.2 s) still gets several samples
        self.first = ""
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        if self.proc:
            import select
            ready, _, _ = select.select([self.proc.stdout], [], [], 10.0)
            if ready:
                self.first = self.proc.stdout.readline()
        return self

    def __exit__(self, *a):
        self.out = self.first
        if self.proc:
            self.proc.terminate()
            try:
                rest, _ = self.proc.communicate(timeout=5)
                self.out += rest or ""
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in (self.out or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons)}


# ------------------------------------------------------------- CPU baseline
def cost_params_dict(peaks: dict) -> dict:
    return dict(L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288, V=151936, bp=2,
                peak_flops=peaks["bf16_tflops"] * 1e12, bandwidth=peaks["hbm_gbs"] * 1e9)


def _reference_stream(job) -> dict:
    """One independent decode stream of the reference planning path (one process, one thread)."""
    seed, warmup, steps, params, latencies, context, n_max = job
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    from oracle import ref_replay as R
    if warmup:
        R.reference_decode(R.synthetic_cycles(warmup, 1000 + seed, n_max=n_max), params, latencies, context, n_max,
                           check=False)
    return R.reference_decode(R.synthetic_cycles(steps, seed, n_max=n_max), params, latencies, context, n_max,
                              check=False)


def run_reference(args) -> None:
    """The reference's own CPU implementation of the path (the unmodified specplan package
    from baseline/_ref, else the oracle port) on the same workload as our arm: N GPUs decode
    N independent requests, so the reference decodes N independent streams, one process per
    stream (the reference harness parallelises runs as processes, sp/harness.py:249-252).
    Each cycle replays config-2-shaped drafter rows (16 x 151936 fp64 from bf16 logits)
    through specplan's decode_full: MarginalBlock validation, top_k_truncate, run_cycle
    (adaptive, N_max 1024, Qwen3-8B roofline at the measured B200 peaks), linearize,
    verify_tree, commit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp

    from oracle import ref_replay as R
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    streams = max(1, world)
    cores = max(1, min(streams, os.cpu_count() or 1))
    peaks = load_peaks()
    params = cost_params_dict(peaks)
    lat = dict(t_draft=8e-4, t_aux=0.0, l_ar=3.3e-3)  # our arm's measured draft / AR step (BENCH_r01)
    jobs = [(i, args.warmup, args.steps, params, lat, args.context, 1024) for i in range(streams)]
    if streams == 1:
        res = [_reference_stream(jobs[0])]
    else:
        with mp.get_context("spawn").Pool(cores) as pool:
            res = pool.map(_reference_stream, jobs)
    tokens = sum(r["tokens"] for r in res)
    seconds = max(r["seconds"] for r in res)  # streams run concurrently: the slowest one bounds the job
    value = tokens / seconds
    info = R.host_info()
    sample = (f"{streams} stream(s) on {cores} process(es) x {args.steps} cycles of the {res[0]['kind']} "
              f"planning path (specplan decode_full over config-2-shaped drafter rows: 16 x 151936 fp64 from bf16 "
              f"logits, c=2048, adaptive N_max 1024); one thread per stream; model forward not included (the "
              f"reference has none); median {1e3 * statistics.median(r['median_cycle_s'] for r in res):.0f} ms/cycle")
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "tokens/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * seconds / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": res[0]["kind"], "sample": sample,
                         **info},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# -------------------------------------------------------------------- ours
def attention_roofline(peaks: dict, c: int, s: int, layers: int = 36) -> dict:
    """K3 per-layer time in a CUDA graph of `layers` launches (distinct layers, PDL) at context c,
    s tree rows; roofline = SURVEY §8d K3 bytes bp*(2(c+s)h_kv + 2 s h_q) + mask vs measured HBM."""
    import torch

    from paper_2605_29727_b200 import ops
    from paper_2605_29727_b200.engine.forward import PagedKV
    n_q, n_kv = 32, 8
    kv = PagedKV(layers, n_kv, c + 320, "cuda")
    kv.buf.normal_(0, 1)
    q = torch.randn(s, n_q * 128, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    words = (s + 31) // 32
    anc = torch.zeros(s, words, dtype=torch.int32, device="cuda")
    for i in range(s):  # chain of siblings: every row sees the root and itself
        anc[i, 0] |= 1
        anc[i, i // 32] |= (1 << (i % 32)) if (i % 32) != 31 else -(1 << 31)
    ws = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()

    def run():
        for li in range(layers):
            ops.attention(q, out, kv.buf, layers, kv.n_pages, li, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0,
                          anc.view(-1), words, ws)
    with torch.cuda.stream(st):
        run()
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        run()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for it in range(6):
        with torch.cuda.stream(st):
            flush.fill_(it)  # 256 MB > L2: every replay reads its KV from HBM
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        with torch.cuda.stream(st):
            g.replay()
        b.record(st)
        b.synchronize()
        if it >= 1:
            ts.append(a.elapsed_time(b) * 1e-3 / layers)
    t = statistics.median(ts)
    byts = 2 * (2 * (c + s) * n_kv * 128 + 2 * s * n_q * 128) + s * words * 4
    achieved = byts / t / 1e9
    del kv, g, flush
    torch.cuda.empty_cache()
    pages = (c + s + 63) // 64
    kern = "attn_tc2_kernel (K3)" if pages // max(1, 148 // (n_kv * ((4 * s + 127) // 128))) >= 8 else "attn_tc_kernel (K3)"
    return {"bound": "hbm", "kernel": kern, "context": c, "tree_rows": s, "layer_us": t * 1e6,
            "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
            "algorithmic_bytes_per_launch": byts, "traffic": "DRAM read = algorithmic (profiles/attn_tc2_ncu_summary.txt)",
            "timing": "CUDA events around a graph of 36 launches over distinct layers, L2 flushed before each replay"}


def step_bytes(p: dict, s: int, c: int) -> int:
    """Fused-minimum bytes of one verify step: weights + KV + activations once,
    no materialised score matrix; the embedding table counts as the s rows gathered."""
    L, h, hq, hkv, hf, V, bp = p["L"], p["h"], p["n_q"] * p["d"], p["n_kv"] * p["d"], p["h_ffn"], p["V"], p["bp"]
    weights = bp * (L * (2 * h * hq + 2 * h * hkv + 3 * h * hf) + V * h + s * h)
    kv = bp * L * (2 * c * hkv + 2 * s * hkv)
    act = bp * L * (4 * s * h + 4 * s * hq + 2 * s * hkv + 4 * s * hf) + bp * s * (h + V)
    return weights + kv + act


def step_flops(p: dict, s: int, c: int) -> int:
    L, h, hq, hkv, hf, V = p["L"], p["h"], p["n_q"] * p["d"], p["n_kv"] * p["d"], p["h_ffn"], p["V"]
    return L * (4 * s * h * hq + 4 * s * h * hkv + 4 * s * (c + s) * hq + 6 * s * h * hf) + 2 * s * h * V


def draft_bytes(p: dict, layers: int, n_feat: int, c: int, gamma: int) -> int:
    """One drafter block: its layers' weights, fc, the shared LM head, its context KV."""
    h, hq, hkv, hf, V, bp = p["h"], p["n_q"] * p["d"], p["n_kv"] * p["d"], p["h_ffn"], p["V"], p["bp"]
    per_layer = 2 * h * hq + 2 * h * hkv + 3 * h * hf
    return bp * (layers * per_layer + n_feat * h * h + V * h + layers * 2 * (c + 2 * (gamma + 1)) * hkv)


def gemm_replay_roofline(eng, cfg, peaks: dict, s_med: int) -> dict:
    """K4: the step's 145 GEMMs (36 x qkv/o/gate_up/down + LM head) at m = s_med, replayed
    back to back in a graph; achieved = algorithmic bytes (weights + X rows) / time."""
    import torch

    from paper_2605_29727_b200 import ops
    t = eng.target
    seq = []
    for lw in eng.tw.layers:
        for w in (lw.qkv, lw.o, lw.gate_up, lw.down):
            seq.append((w, {cfg.h: t.x, cfg.h_q: t.attn, cfg.h_ffn: t.act}[w.shape[1]][:s_med]))
    seq.append((eng.tw.lm_head, t.x[:min(s_med, 256)]))

    def gemm_seq():
        for w, xin in seq:
            ops.gemm_partial(xin, w, out=t.partial)
    with torch.cuda.stream(eng.stream):
        gemm_seq()
    eng.stream.synchronize()
    gg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gg, stream=eng.stream):
        gemm_seq()
    reps = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        with torch.cuda.stream(eng.stream):
            gg.replay()
        b.record(eng.stream)
        b.synchronize()
        reps.append(a.elapsed_time(b) * 1e-3)
    g_time = statistics.median(reps[1:])
    g_bytes = sum(w.numel() * 2 + x.shape[0] * w.shape[1] * 2 for w, x in seq)
    achieved = g_bytes / g_time / 1e9
    # ncu --set full DRAM bytes per launch of the same 145-launch sequence, from the capture
    # (profiles/gemm_dram_bytes*.json) whose row count is nearest to this step's
    traffic, traffic_m = None, None
    for prof in sorted((ROOT / "profiles").glob("gemm_dram_bytes*.json")):
        d = json.loads(prof.read_text())
        if traffic_m is None or abs(d.get("m", 0) - s_med) < abs(traffic_m - s_med):
            traffic, traffic_m = d.get("dram_bytes_per_launch"), d.get("m")
    del gg
    return {"bound": "hbm", "kernel": "gemm_bf16_kernel (K4, tcgen05 weight streaming)", "achieved": achieved,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
            "peak_src": peaks["src"], "avg_launch_us": 1e6 * g_time / len(seq), "traffic_m": traffic_m,
            "algorithmic_bytes": f"bf16 weights + X rows per launch, 36x(qkv,o,gate_up,down)+lm_head at m={s_med}",
            "timing": "CUDA events around a graph of the step's 145 GEMM launches (back to back, PDL)"}


def run_config3(args, world: int, rank: int, local: int, cfg, peaks: dict, policy: str = "adaptive") -> dict | None:
    """BASELINE config 3 at N GPUs: 64 requests (prompt seeds 0..63) sharded contiguously,
    each rank decodes its shard batched in one BatchEngine, no collective on the data path;
    tokens/s = all committed tokens / max over ranks of the device time.  policy "adaptive":
    per-request Algorithm 1 with the batch-aware verify curve (N_max = --c3-budget, ragged
    verify), "fixed": every tree has N = --c3-budget nodes."""
    import numpy as np
    import torch

    import paper_2605_29727_b200 as P
    from paper_2605_29727_b200.dist import reduce_throughput, shard
    from paper_2605_29727_b200.engine.batch import BatchEngine
    from paper_2605_29727_b200.engine.config import DrafterConfig
    mine = list(shard(args.c3_requests, world, rank))
    prompts = [np.random.default_rng(r).integers(0, cfg.V - 1, args.context + 1).tolist() for r in mine]
    cycles = args.c3_cycles
    be = BatchEngine(cfg, DrafterConfig(layers=5, gamma=16, logit_scale=args.logit_scale), n_req=len(mine),
                     n_fixed=args.c3_budget, max_ctx=args.context + 17 * (cycles + 8) + 64, seed=0)
    if policy == "adaptive":
        params = cfg.cost_params(peaks["bf16_tflops"] * 1e12, peaks["hbm_gbs"] * 1e9)
        est = P.VerifyLatencyEstimator(params, variant="static")  # roofline curve (batch shift on device)
        lat = P.CycleLatencies(t_draft=est.estimate(17, args.context), t_aux=0.0, l_ar=est.estimate(1, args.context))
        be.set_policy("adaptive", estimator=est, latencies=lat)
    be.reset(prompts)
    be.precapture()  # adaptive: every 64-row verify bucket's graph before anything is timed
    for _ in range(3):
        be.cycle()
    base = be.committed_counts().copy()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(be.stream)
    rows = []
    for _ in range(cycles):
        be.cycle()
        rows.append(be.last_rows if policy == "adaptive" else len(mine) * (args.c3_budget + 1))
    e1.record(be.stream)
    e1.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    tokens = float((be.committed_counts() - base).sum())
    t_max, tok_all, value = reduce_throughput(t, tokens)
    desc = (f"adaptive (batch-aware Algorithm 1 per request, N_max={args.c3_budget}, ragged verify)"
            if policy == "adaptive" else f"fixed N={args.c3_budget}")
    out = {"workload": f"config3: {args.c3_requests} requests (Qwen3-8B shape, 2048-token prompts) sharded "
                       f"data-parallel over {world} GPU(s), batched per GPU, {desc}",
           "value": value, "unit": "tokens/s", "n_gpus": world, "requests_per_gpu": len(mine),
           "cycles": cycles, "ms_per_cycle": 1e3 * t_max / cycles, "scaling": "strong (64 requests in total)",
           "verify_rows_per_cycle_mean": statistics.mean(rows), "mean_accept_len": tok_all / (cycles * args.c3_requests)}
    if policy == "fixed":
        out["graph_kernels_per_cycle"] = be.graph_kernels
    del be
    torch.cuda.empty_cache()
    return out


def run_ours(args) -> None:
    import numpy as np
    import torch

    import paper_2605_29727_b200 as P
    from paper_2605_29727_b200 import _lib
    from paper_2605_29727_b200.dist import reduce_throughput
    from paper_2605_29727_b200.engine.config import MODELS, DrafterConfig
    from paper_2605_29727_b200.engine.decode import ST_COMMITTED, B200Engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BST_BENCH_DEVICE / BST_DIST_BACKEND=gloo: exercise the N > 1 code path with several ranks
    # on one GPU (the 1-GPU test pool); the driver's runs use one GPU per rank and NCCL
    local = int(os.environ.get("BST_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BST_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    peaks = load_peaks()
    cfg = MODELS[args.model]
    pdict = cost_params_dict(peaks)
    steps_total = args.warmup + args.steps + args.e2e_cycles + args.cpu_cycles + 64
    dcfg = DrafterConfig(layers=5, gamma=16, logit_scale=args.logit_scale)
    eng = B200Engine(cfg, dcfg, max_ctx=args.context + 17 * steps_total + 256, seed=rank, n_cap=1024, top_k=8)
    prompt = np.random.default_rng(1000 + rank).integers(0, cfg.V - 1, args.context + 1).tolist()
    eng.reset(prompt)
    params = cfg.cost_params(peaks["bf16_tflops"] * 1e12, peaks["hbm_gbs"] * 1e9)

    if args.profile:  # short run for ncu launch lists: fixed budget, graphs, no calibration/e2e/cpu legs
        eng.set_policy("fixed", n=args.profile_n)
        for _ in range(args.warmup):
            eng.cycle()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        for _ in range(args.steps):
            eng.cycle()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        return
    # every verify bucket's graph is captured before anything is timed (a bucket first seen
    # inside the timed loop would otherwise pay its capture in that cycle)
    _log('precapture verify graphs')
    n_graphs = eng.precapture()
    _log(f'{n_graphs} verify graphs')
    # ---- K7: measure l_ar / t_draft, static calibration of the verify roofline
    _log('K7')
    l_ar = eng.measure_ar_step()
    calib = []
    for n in (15, 47, 95, 159, 255, 511):
        eng.reset(prompt)
        eng.set_policy("fixed", n=n)
        obs = []
        for _ in range(4):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            nn, _ = eng.draft(ev)
            eng.verify(nn, ev)
            ev[2].synchronize()
            obs.append((nn + 1, ev[0].elapsed_time(ev[1]) * 1e-3, ev[1].elapsed_time(ev[2]) * 1e-3))
        s, td, tv = obs[-1][0], statistics.median(o[1] for o in obs[1:]), statistics.median(o[2] for o in obs[1:])
        calib.append((s, td, tv))
    t_draft = statistics.median(x[1] for x in calib)
    pairs = [(P.roofline_latency(params, P.LatencyQuery(s=s, c=args.context)), tv) for s, _, tv in calib]
    fit = P.fit_static_calibration(pairs)
    est = P.VerifyLatencyEstimator(params, variant="static", fit=fit)
    lat = P.CycleLatencies(t_draft=t_draft, t_aux=0.0, l_ar=l_ar)

    def set_policy():
        if args.policy == "adaptive":
            eng.set_policy("adaptive", estimator=est, latencies=lat, n_max=1024)
        else:
            eng.set_policy("fixed", n=int(args.policy.split("-")[1]))

    # ---- device-timed decode (inputs resident, graphs)
    _log('device-timed decode')
    eng.reset(prompt)
    set_policy()
    for _ in range(args.warmup):
        eng.cycle()
    eng.stream.synchronize()
    c0 = int(eng.state[ST_COMMITTED].item())
    cyc0 = int(eng.state[4].item())
    _lib.launch_count = 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per, buckets = [], []
    with ClockSampler(local) as clk:
        start.record(eng.stream)
        for _ in range(args.steps):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            n = eng.cycle(ev)
            per.append(ev)
            buckets.append(eng._bucket(n))
        end.record(eng.stream)
        end.synchronize()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed = start.elapsed_time(end) * 1e-3
    tokens = int(eng.state[ST_COMMITTED].item()) - c0
    stats = eng.read_log()[cyc0:cyc0 + args.steps]
    t_ver = [e[1].elapsed_time(e[2]) * 1e-3 for e in per]  # seconds
    t_dr = [e[0].elapsed_time(e[1]) * 1e-3 for e in per]
    elapsed, tokens_all, _ = reduce_throughput(elapsed, float(tokens))
    value = tokens_all / elapsed
    kd = eng.graph_kernels[id(eng.graph_d)]
    kv = {b: eng.graph_kernels[id(g)] for b, g in eng.graphs_v.items()}
    gpu_launches = sum(kd + kv[b] for b in buckets)  # exact: nodes of the graphs replayed in the timed region

    # ---- step-level and decode-level rooflines of the timed cycles
    _log('step-level and decode-level rooflines of the timed cycles')
    bw, pk = peaks["hbm_gbs"] * 1e9, peaks["bf16_tflops"] * 1e12
    v_roof = [max(step_bytes(pdict, st.tree_size + 1, st.context) / bw,
                  step_flops(pdict, st.tree_size + 1, st.context) / pk) for st in stats]
    d_roof = [draft_bytes(pdict, dcfg.layers, len(eng.target.feat_layers), st.context, 16) / bw for st in stats]
    v_bytes = [step_bytes(pdict, st.tree_size + 1, st.context) for st in stats]
    accepted = sum(st.accepted_len for st in stats)
    decode_roof = accepted / (sum(v_roof) + sum(d_roof))
    step_roof = {"bound": "hbm", "what": "whole verify step (target forward over the tree + LM-head argmax + "
                 "accept + KV compaction), CUDA events on the engine stream per timed cycle",
                 "algorithmic_bytes_per_step_mean": statistics.mean(v_bytes),
                 "achieved": statistics.mean(b / t for b, t in zip(v_bytes, t_ver)) / 1e9,
                 "peak": peaks["hbm_gbs"], "unit": "GB/s",
                 "frac": statistics.mean(r / t for r, t in zip(v_roof, t_ver)),
                 "verify_roof_us_mean": 1e6 * statistics.mean(v_roof), "verify_us_mean": 1e6 * statistics.mean(t_ver),
                 "draft_roof_us_mean": 1e6 * statistics.mean(d_roof), "draft_us_mean": 1e6 * statistics.mean(t_dr),
                 "bytes_formula": "SURVEY §8d fused minimum: weights (embedding as gathered rows) + KV(c+s) + "
                                  "activations, no score matrix; time roof = max(bytes/BW, flops/peak)"}

    # ---- cycles exported for the CPU reference replay (same inputs as the GPU)
    _log('cycles exported for the CPU reference replay')
    exported = []
    if rank == 0 and world == 1 and not args.no_cpu:
        eng.reset(prompt)
        set_policy()
        eng.export = True
        for _ in range(args.cpu_cycles):
            eng.cycle()
        eng.export = False
        exported = [dict(probs=e["probs"], parent=e["parent"], token=e["token"], argmax=e["argmax"],
                         path=e["path"].tolist(), bonus=e["bonus"]) for e in eng.exported]
        eng.exported = []

    # ---- e2e: the public API, same estimator as the timed region; prompt upload + prefill inside
    _log('e2e')
    sim = P.SimConfig(controller=P.ControllerConfig(n_max=1024, latencies=lat, variant="static",
                                                    context_len=args.context), run_length=args.e2e_cycles,
                      top_k=8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.reset(prompt)  # H2D of the prompt from host memory + causal prefill
    records, toks_e2e = P.decode_full(eng, sim, P.Policy.adaptive() if args.policy == "adaptive"
                                      else P.Policy.fixed(int(args.policy.split("-")[1])), est)
    torch.cuda.synchronize()
    e2e_time = time.perf_counter() - t0
    e2e_tokens = sum(r.accepted_len for r in records)
    e2e_val = reduce_throughput(e2e_time, float(e2e_tokens))[2]

    # ---- dominant kernel (K4) and K3 probes
    _log('dominant kernel')
    s_med = int(statistics.median(buckets))
    gemm = gemm_replay_roofline(eng, cfg, peaks, s_med)
    attn = attn2k = None
    if not args.no_attn:
        attn2k = attention_roofline(peaks, args.context, s_med)
        attn = attention_roofline(peaks, 32768, 17)

    # ---- CPU baseline (rank 0, N=1 only): the reference decode over the GPU's own cycles
    _log('CPU baseline')
    cpu = cpu3 = None
    if exported:
        from oracle import ref_replay as R
        latd = dict(t_draft=lat.t_draft, t_aux=lat.t_aux, l_ar=lat.l_ar)
        r = R.reference_decode(exported, pdict, latd, args.context, 1024, policy=args.policy,
                               fit=(fit.slope, fit.intercept), check=True)
        cpu = {"value": r["tokens"] / r["seconds"], "unit": "tokens/s", "cores": 1, "kind": r["kind"],
               "sample": f"{r['cycles']} decode cycles of this run's workload: the GPU's own fp64 drafter rows and "
                         f"verify argmax per cycle replayed through {'specplan' if r['kind'] == 'reference' else 'the oracle port'}"
                         f".decode_full (MarginalBlock validation, top_k_truncate, run_cycle, linearize, verify_tree, "
                         f"commit); trees identical to the GPU's (checked); no model forward (the reference has "
                         f"none); median {1e3 * r['median_cycle_s']:.0f} ms/cycle, 1 of {os.cpu_count()} host cores",
               "trees_match_gpu": True, **R.host_info()}
        del exported
        if not args.no_cpu3:
            _log("config 3 CPU process-pool leg")
            c3 = R.process_pool_streams(args.c3_requests, 2, pdict, latd, args.context, 1024)
            cpu3 = {"value": c3["tokens_per_s_wall"], "unit": "tokens/s", "cores": c3["workers"], "kind": c3["kind"],
                    "sample": f"config 3: {c3['streams']} reference decode streams x {c3['cycles_per_stream']} cycles, "
                              f"a process pool of {c3['workers']} workers (sp/harness.py:249-252), wall clock"}

    c3 = c3f = None
    if not args.no_config3:
        _log("config 3 GPU leg")
        del eng
        torch.cuda.empty_cache()
        c3 = run_config3(args, world, rank, local, cfg, peaks, "adaptive")
        c3f = run_config3(args, world, rank, local, cfg, peaks, "fixed")

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init bf16 weights, uniform random prompt tokens)",
        "config": {"workload": WORKLOAD, "context": args.context, "policy": args.policy, "gamma": 16, "top_k": 8,
                   "n_max": 1024, "drafter_logit_scale": args.logit_scale,
                   "l2": "inputs larger than L2: 16.4 GB of target weights + 1.9 GB drafter streamed per step"},
        "tree_verify_us_per_step": 1e6 * statistics.mean(t_ver), "draft_us_per_step": 1e6 * statistics.mean(t_dr),
        "mean_accept_len": statistics.mean(s.accepted_len for s in stats),
        "mean_tree_size": statistics.mean(s.tree_size for s in stats), "verify_rows_bucket_median": s_med,
        "l_ar_us": l_ar * 1e6, "ar_tokens_per_s_equiv": 1.0 / l_ar,
        "decode_roofline": {"tokens_per_s": decode_roof, "frac": value / decode_roof,
                            "what": "AAL / (T_draft_roof + T_verify_roof(N*, c)) over the timed cycles"},
        "calibration": {"slope": fit.slope, "intercept": fit.intercept, "rmse_before": fit.rmse_before,
                        "rmse_after": fit.rmse_after, "points": [[s, tv] for s, _, tv in calib]},
        "roofline": {**gemm, "step": step_roof},
        "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": 4 * len(prompt) // max(1, len(records)),
                "d2h_bytes_per_step": 64 + 4 * int(round(e2e_tokens / max(1, len(records)))),
                "api": "engine.reset(prompt) + paper_2605_29727_b200.decode_full(engine, SimConfig, policy, "
                       "VerifyLatencyEstimator(static, fit)) — prompt upload and prefill inside the timed region",
                "cycles": len(records), "mean_tree_size": statistics.mean(r.tree_size for r in records)},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
    }
    if attn2k:
        line["verify_attention_roofline_c2k"] = attn2k
    if attn:
        line["verify_attention_roofline"] = attn
    if cpu:
        line["cpu_baseline"] = cpu
    if cpu3:
        line["cpu_baseline_config3"] = cpu3
    if c3:
        line["config3"] = c3
    if c3f:
        line["config3_fixed"] = c3f
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="qwen3-8b")
    ap.add_argument("--context", type=int, default=2048)
    ap.add_argument("--policy", default="adaptive")
    ap.add_argument("--logit-scale", type=float, default=6.0)
    ap.add_argument("--e2e-cycles", type=int, default=256,
                    help="decode_full run_length of the e2e leg (the reference harness default, sp/harness.py:57)")
    ap.add_argument("--cpu-cycles", type=int, default=24)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu3", action="store_true", help="skip the config-3 process-pool CPU leg")
    ap.add_argument("--no-config3", action="store_true", help="skip the config-3 (64 requests sharded) GPU leg")
    ap.add_argument("--c3-requests", type=int, default=64)
    ap.add_argument("--c3-budget", type=int, default=64)
    ap.add_argument("--c3-cycles", type=int, default=8)
    ap.add_argument("--profile-n", type=int, default=63)
    ap.add_argument("--no-attn", action="store_true", help="skip the K3 roofline probe (c=32K, s=17)")
    ap.add_argument("--profile", action="store_true", help="only the cycle loop (for ncu --profile-from-start off)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
