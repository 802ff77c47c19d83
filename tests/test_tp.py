"""Tensor-parallel verify (config 5).

CPU (gloo, world_size 2): the vocab-parallel argmax protocol — each rank packs its
shard's per-row (max, global index) into one signed int64 key, a MAX all-reduce and
the decode give np.argmax of the full row with its lowest-index tie-break
(verify_sim.py:107-109); weight-shard index math.
GPU: the kernel keys equal the host packing; a 2-way TP target run in lock step on
one GPU (collectives reduced in-process) reproduces the unsharded target's argmax
on prefill and on a tree-verify step; the NCCL path (world_size 1) runs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _argmax_worker(rank, world, port, rows, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2605_29727_b200.engine.tp import pack_argmax_key, unpack_argmax_key
    dist.init_process_group("gloo", rank=rank, world_size=world)
    V = rows.shape[1]
    vl = V // world
    mine = rows[:, rank * vl:(rank + 1) * vl]
    keys = torch.tensor([max(pack_argmax_key(float(v), rank * vl + j) for j, v in enumerate(r)) for r in mine],
                        dtype=torch.int64)
    dist.all_reduce(keys, op=dist.ReduceOp.MAX)
    out[rank] = [unpack_argmax_key(int(k)) for k in keys]
    dist.destroy_process_group()


def test_vocab_parallel_argmax_gloo_two_ranks():
    rng = np.random.default_rng(5)
    rows = rng.standard_normal((12, 64)).astype(np.float32)
    rows[0, [3, 40]] = 9.0          # tie across shards -> lowest index
    rows[1, [33, 35]] = 7.0         # tie inside shard 1
    rows[2] = -np.abs(rows[2])      # all negative
    rows[3, 10] = rows[3, 50] = np.float32(-0.0)
    rows[3][rows[3] > 0] *= -1
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_argmax_worker, args=(2, _free_port(), rows, out), nprocs=2, join=True)
        got = dict(out)
    want = [int(np.argmax(r)) for r in rows]
    assert got[0] == want and got[1] == want


def test_local_config_and_shard_shapes():
    from paper_2605_29727_b200.engine.config import QWEN3_32B, TINY
    from paper_2605_29727_b200.engine.tp import local_config
    lc = local_config(QWEN3_32B, 8)
    assert (lc.n_q, lc.n_kv, lc.h_ffn, lc.V, lc.h) == (8, 1, 3200, 18992, 5120)
    assert local_config(TINY, 2).n_kv == 1
    with pytest.raises(ValueError):
        local_config(TINY, 3)


# ------------------------------------------------------------------ GPU
def _fill(m, tokens, pos, slot):
    n = len(tokens)
    m.tokens[:n].copy_(torch.tensor(tokens, dtype=torch.int32))
    m.pos[:n].copy_(torch.tensor(pos, dtype=torch.int32))
    m.slot[:n].copy_(torch.tensor(slot, dtype=torch.int32))


@pytest.mark.gpu
def test_argmax_keys_kernel_matches_host_packing():
    from paper_2605_29727_b200 import ops
    from paper_2605_29727_b200.engine.tp import pack_argmax_key
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(5, 256, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(640, 256, device="cuda", generator=g).to(torch.bfloat16)
    p = ops.gemm_partial(x, w)
    y = ops.gemm_reduce(p).cpu().numpy()
    keys = torch.zeros(5, dtype=torch.int64, device="cuda")
    ops.gemm_argmax_keys(p, keys, 1280)
    want = [max(pack_argmax_key(float(v), 1280 + j) for j, v in enumerate(r)) for r in y]
    assert keys.cpu().tolist() == want


@pytest.mark.gpu
@pytest.mark.parametrize("tp,ar_dtype", [(2, "bf16"), (2, "fp32")])
def test_tp_lockstep_matches_unsharded_target(tp, ar_dtype):
    """bf16 (default) and fp32 all-reduce payloads of the row-parallel outputs."""
    from oracle import specplan_port as O
    from paper_2605_29727_b200.engine.config import TINY
    from paper_2605_29727_b200.engine.forward import MODE_CAUSAL, MODE_TREE, TargetModel
    from paper_2605_29727_b200.engine.tp import TPTargetModel, run_lockstep, shard_weights
    from paper_2605_29727_b200.engine.weights import TargetWeights
    dev = torch.device("cuda")
    cfg = TINY
    full = TargetWeights.random(cfg, 3, dev)
    slots, R = 512, 64
    ref = TargetModel(cfg, full, slots, R, (), dev)
    shards = [TPTargetModel(cfg, tp, r, shard_weights(full, cfg, tp, r), slots, R, dev) for r in range(tp)]
    for sh in shards:
        sh.set_allreduce_dtype(torch.bfloat16 if ar_dtype == "bf16" else torch.float32)
    streams = [torch.cuda.Stream() for _ in range(tp)]
    rng = np.random.default_rng(0)
    P = 200
    prompt = rng.integers(0, cfg.V, P).tolist()
    state = torch.zeros(8, dtype=torch.int32, device=dev)
    # prefill in chunks of R rows (causal), argmax of every prompt row
    ref_am, tp_am = [], []
    for start in range(0, P, R):
        n = min(R, P - start)
        state[0] = start
        for m in [ref] + shards:
            _fill(m, prompt[start:start + n], list(range(n)), list(range(n)))
        torch.cuda.synchronize()
        ref.forward(n, state, MODE_CAUSAL, keys_after_c=n, head="logits", c_host=start)
        logits = ref.logits[:n].clone()
        ref.forward(n, state, MODE_CAUSAL, keys_after_c=n, head="argmax", c_host=start)
        run_lockstep(shards, streams, n, state, MODE_CAUSAL, n, head="argmax", c_host=start)
        torch.cuda.synchronize()
        ref_am.append(ref.argmax[:n].cpu().numpy())
        tp_am.append(shards[0].argmax[:n].cpu().numpy())
        top2 = torch.topk(logits, 2, dim=1).values
        clear = ((top2[:, 0] - top2[:, 1]) > 1e-2).cpu().numpy()
        assert np.array_equal(ref_am[-1][clear], tp_am[-1][clear])
        for sh in shards[1:]:
            assert np.array_equal(sh.argmax[:n].cpu().numpy(), tp_am[-1])
    # tree verify over the prefilled context (random tree, s = 17)
    s = 17
    parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, s)])
    depth = np.zeros(s, dtype=np.int64)
    for i in range(1, s):
        depth[i] = depth[parent[i]] + 1
    anc = O.ancestor_bits(parent)
    words = (s + 31) // 32
    pad = np.zeros((s, words * 32), dtype=bool)
    pad[:, :s] = anc
    packed = torch.from_numpy(np.packbits(pad, axis=1, bitorder="little").view(np.int32).copy()).cuda()
    toks = rng.integers(0, cfg.V, s).tolist()
    state[0] = P
    for m in [ref] + shards:
        _fill(m, toks, (P + depth).tolist(), list(range(P, P + s)))
    torch.cuda.synchronize()
    ref.forward(s, state, MODE_TREE, keys_after_c=s, anc=packed.view(-1), mask_words=words, head="logits", c_host=P)
    logits = ref.logits[:s].clone()
    ref.forward(s, state, MODE_TREE, keys_after_c=s, anc=packed.view(-1), mask_words=words, head="argmax", c_host=P)
    run_lockstep(shards, streams, s, state, MODE_TREE, s, anc=packed.view(-1), mask_words=words, head="argmax",
                 c_host=P)
    torch.cuda.synchronize()
    top2 = torch.topk(logits, 2, dim=1).values
    clear = ((top2[:, 0] - top2[:, 1]) > 1e-2).cpu().numpy()
    assert clear.sum() >= s // 2
    assert np.array_equal(ref.argmax[:s].cpu().numpy()[clear], shards[0].argmax[:s].cpu().numpy()[clear])


@pytest.mark.gpu
def test_tp_nccl_world_one_runs():
    import torch.distributed as dist
    from paper_2605_29727_b200.engine.config import TINY
    from paper_2605_29727_b200.engine.forward import MODE_CAUSAL, TargetModel
    from paper_2605_29727_b200.engine.tp import TPTargetModel, shard_weights
    from paper_2605_29727_b200.engine.weights import TargetWeights
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        dev = torch.device("cuda")
        full = TargetWeights.random(TINY, 4, dev)
        ref = TargetModel(TINY, full, 256, 32, (), dev)
        m = TPTargetModel(TINY, 1, 0, shard_weights(full, TINY, 1, 0), 256, 32, dev)
        state = torch.zeros(8, dtype=torch.int32, device=dev)
        toks = list(range(3, 35))
        for mm in (ref, m):
            _fill(mm, toks, list(range(32)), list(range(32)))
        ref.forward(32, state, MODE_CAUSAL, keys_after_c=32, head="argmax")
        m.forward(32, state, MODE_CAUSAL, keys_after_c=32, head="argmax")
        torch.cuda.synchronize()
        agree = (ref.argmax[:32] == m.argmax[:32]).float().mean().item()
        assert agree >= 0.9
    finally:
        dist.destroy_process_group()


def _tp_process_worker(rank, world, port, out_dir):
    """One TP rank as its own process on cuda:0 (the 1-GPU pool): the real
    TPTargetModel.forward with torch.distributed collectives (gloo over CUDA tensors)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2605_29727_b200.engine.config import TINY
    from paper_2605_29727_b200.engine.forward import MODE_CAUSAL
    from paper_2605_29727_b200.engine.tp import TPTargetModel, shard_weights
    from paper_2605_29727_b200.engine.weights import TargetWeights
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        full = TargetWeights.random(TINY, 5, dev)
        m = TPTargetModel(TINY, world, rank, shard_weights(full, TINY, world, rank), 256, 64, dev)
        state = torch.zeros(8, dtype=torch.int32, device=dev)
        toks = np.random.default_rng(9).integers(0, TINY.V, 48).tolist()
        _fill(m, toks, list(range(48)), list(range(48)))
        m.forward(48, state, MODE_CAUSAL, keys_after_c=48, head="argmax")
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"am{rank}.npy"), m.argmax[:48].cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_tp2_processes_match_unsharded_target(tmp_path):
    """TP = 2 as two processes with a real process group (row-parallel bf16 SUM and
    argmax-key MAX all-reduces through torch.distributed) reproduces the unsharded target's
    argmax on every clear row; both ranks agree."""
    import torch.multiprocessing as mp
    from paper_2605_29727_b200.engine.config import TINY
    from paper_2605_29727_b200.engine.forward import MODE_CAUSAL, TargetModel
    from paper_2605_29727_b200.engine.weights import TargetWeights
    mp.spawn(_tp_process_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    dev = torch.device("cuda", 0)
    full = TargetWeights.random(TINY, 5, dev)
    ref = TargetModel(TINY, full, 256, 64, (), dev)
    state = torch.zeros(8, dtype=torch.int32, device=dev)
    toks = np.random.default_rng(9).integers(0, TINY.V, 48).tolist()
    _fill(ref, toks, list(range(48)), list(range(48)))
    ref.forward(48, state, MODE_CAUSAL, keys_after_c=48, head="logits")
    logits = ref.logits[:48].clone()
    ref.forward(48, state, MODE_CAUSAL, keys_after_c=48, head="argmax")
    torch.cuda.synchronize()
    want = ref.argmax[:48].cpu().numpy()
    a0, a1 = (np.load(tmp_path / f"am{r}.npy") for r in range(2))
    assert np.array_equal(a0, a1)
    top2 = torch.topk(logits, 2, dim=1).values
    clear = ((top2[:, 0] - top2[:, 1]) > 1e-2).cpu().numpy()
    assert clear.sum() >= 24
    assert np.array_equal(want[clear], a0[clear])
