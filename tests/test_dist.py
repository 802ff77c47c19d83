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
