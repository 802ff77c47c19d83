"""N>1 path on CPU: world_size-2 gloo processes shard requests with no data-path
collective and reduce timing as max-over-ranks / sum-of-tokens (bench.py contract)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    from paper_2605_29727_b200.dist import reduce_throughput, shard, world as w
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ws, r, _ = w()
    mine = list(shard(64, ws, r))
    # each rank "decodes" its own requests independently; elapsed differs per rank
    elapsed = 1.0 + r
    tokens = float(len(mine) * 10)
    mx, total, tput = reduce_throughput(elapsed, tokens)
    out[r] = (mine[0], mine[-1], mx, total, tput)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_shard_and_reduce(world):
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][:2] == (0, 31) and res[1][:2] == (32, 63)
    for r in range(world):
        assert res[r][2] == 2.0 and res[r][3] == 640.0 and res[r][4] == 320.0


def test_shard_covers_all_requests():
    from paper_2605_29727_b200.dist import shard
    for n in (1, 7, 64, 65):
        for ws in (1, 2, 4, 8):
            got = [i for r in range(ws) for i in shard(n, ws, r)]
            assert got == list(range(n))


# ---------------------------------------------------------------- TP protocol over gloo
def _tp_worker(rank, world, port, out):
    """Each rank holds a vocabulary shard / a row-parallel weight shard; the collectives are
    the product's own dist_collective (NCCL on the GPU box, gloo here)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2605_29727_b200.engine.tp import dist_collective, pack_argmax_key, unpack_argmax_key
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    V, rows = 64, 6
    full = rng.standard_normal((rows, V)).astype(np.float32)
    full[0, [5, 40]] = 9.0          # cross-shard tie -> the lower global index (5)
    full[1, [33, 34]] = 9.0         # tie inside shard 1 -> 33
    full[2, :] = -1.0               # all equal (negative) -> 0
    full[3, 63] = np.float32(np.inf)
    lo, hi = rank * V // world, (rank + 1) * V // world
    keys = torch.tensor([max(pack_argmax_key(float(v), lo + j) for j, v in enumerate(r[lo:hi])) for r in full],
                        dtype=torch.int64)
    dist_collective("max", keys)
    am = [unpack_argmax_key(int(k)) for k in keys]
    # row-parallel output: y = x W^T with W split along its input columns, SUM all-reduce
    k_in, n_out = 96, 40
    x = torch.from_numpy(rng.standard_normal((rows, k_in)).astype(np.float32))
    w = torch.from_numpy(rng.standard_normal((n_out, k_in)).astype(np.float32))
    c0, c1 = rank * k_in // world, (rank + 1) * k_in // world
    y32 = x[:, c0:c1] @ w[:, c0:c1].t()
    y16 = y32.to(torch.bfloat16)
    dist_collective("sum", y32)
    dist_collective("sum", y16)
    out[rank] = (am, (y32 - x @ w.t()).abs().max().item(), (y16.float() - x @ w.t()).abs().max().item(),
                 float((x @ w.t()).abs().max()), full.argmax(1).tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_tp_argmax_keys_and_row_parallel_sum():
    """World-2 run of the tensor-parallel collective protocol: packed int64 argmax keys of
    vocabulary shards reduced with MAX decode to np.argmax of the full row (lowest index on
    cross-shard ties), and the SUM of row-parallel partial outputs (fp32 and bf16 payloads)
    equals the unsharded product."""
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_tp_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    am0, e32, e16, scale, want = res[0]
    assert res[1][0] == am0 == want
    assert am0[:4] == [5, 33, 0, 63]
    assert e32 <= 1e-5 * scale and e16 <= 2e-2 * scale


# ------------------------------------------------------------- DP decode over gloo
def _decode_request(req: int) -> tuple:
    """One independent decode stream: the reference's synthetic pair (our TargetRule, host
    plugin) through the oracle's decode loop (the CPU restatement of decode_full)."""
    from oracle import specplan_port as O
    from paper_2605_29727_b200.lattice import SyntheticPairConfig
    from paper_2605_29727_b200.synthetic import TargetRule
    rule = TargetRule(SyntheticPairConfig(gamma=4, vocab_size=64, alignment=0.7, concentration=3.0, seed=req))
    dims = O.Dims(L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288, V=151936, bp=2, peak_flops=1649.1e12,
                  bandwidth=6457.7e9)
    _, toks = O.decode_loop(lambda prefix: rule.drafter_marginals(prefix).probs, rule.next_token, 12, 4,
                            ("fixed", 8), 8, dims, 100, 1e-4, 0.0, 2e-3)
    return toks


def _dp_worker(rank, world, port, out):
    """Config-3 partitioning: each rank decodes its contiguous shard of the requests with
    no collective on the data path; the job's throughput is reduced with the bench's rule
    (max elapsed over ranks, sum of tokens); the streams are gathered only for the check."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2605_29727_b200.dist import reduce_throughput, shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    streams = {req: _decode_request(req) for req in shard(6, world, rank)}
    mx, total, _ = reduce_throughput(1.0 + rank, float(sum(len(v) for v in streams.values())))
    gathered = [None] * world
    dist.all_gather_object(gathered, streams)
    out[rank] = (gathered, total, mx)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_dp_shards_decode_like_one_process():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_dp_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    merged = {}
    for part in res[0][0]:
        merged.update(part)
    single = {r: _decode_request(r) for r in range(6)}
    assert sorted(merged) == list(range(6)) and merged == single
    assert res[0][1] == res[1][1] == float(sum(len(v) for v in single.values()))
    assert res[0][2] == res[1][2] == 2.0
