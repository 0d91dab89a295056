"""CPU (gloo, world_size 2) coverage of the multi-process host logic.

The data path of the one-process-per-GPU group needs GPUs; what is testable
here is everything around it: the rank-indexed handle exchange (ordered by
rank, never by arrival -- collective.cpp:46-50), the per-rank shard plan
(layers.cpp:23-46) tiling K exactly, and the strong-scaling bookkeeping bench.py
does (max over ranks).
"""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import time

    import torch
    import torch.distributed as dist

    import paper_2511_17826_b200 as tb
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    # arrival order deliberately reversed: rank 1 publishes first
    if rank == 0:
        time.sleep(0.3)
    blob = bytes([rank]) * tb.api.TBIK_IPC_HANDLE_BYTES
    got = tb.exchange_handles(blob, world, dist)
    ok_order = [b[0] for b in got] == list(range(world))
    cfg = tb.BlockConfig(64, 256, 128, 0)
    sp = tb.make_row_shard_plan(14336, cfg, world, 8)
    mine = sp.bounds[rank]
    allb = [None] * world
    dist.all_gather_object(allb, mine)
    tiles = allb[0][0] == 0 and allb[-1][1] == 14336 and all(allb[i][1] == allb[i + 1][0] for i in range(world - 1))
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, ok_order, tiles, float(t.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_handle_exchange_and_shards_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_order, tiles, mx in res:
        assert ok_order, f"rank {rank}: handles not rank-ordered"
        assert tiles, f"rank {rank}: shard plan does not tile K"
        assert mx == float(world)


def test_bad_handle_blob_rejected():
    import paper_2511_17826_b200 as tb

    class FakeDist:
        @staticmethod
        def all_gather_object(out, obj):
            out[0] = obj
            out[1] = b"short"

    with pytest.raises(tb.TbikError) as e:
        tb.exchange_handles(b"x" * tb.api.TBIK_IPC_HANDLE_BYTES, 2, FakeDist)
    assert e.value.code == tb.ErrorCode.CollectiveMismatch
