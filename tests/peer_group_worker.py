"""One rank of the two-process PeerGroup test (tests/test_gpu_collective.py).

Launched twice with RANK=0/1, WORLD_SIZE=2, MASTER_ADDR/PORT set.  torch.distributed
(gloo) only carries the 128-byte IPC handles; the data path is libtbik_b200's peer
memory + device flag barrier.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tb.set_schedule("group_fused", int(os.environ.get("TBIK_GROUP_FUSED", "1")))
    M, K, N = 64, 14336, 1024
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    x = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    w = torch.randn(K, N, generator=g, device="cuda").to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    kb, ke = tb.make_row_shard_plan(K, cfg, world, 8).bounds[rank]
    xs, ws = x[:, kb:ke].contiguous(), w[kb:ke].contiguous()
    E_big = (1 << 20) + 4  # > 1 MiB of f32: the reduce-scatter + push path
    Mo, No = 1024, 2048  # >= 8 MiB of f32 output: the overlapped GEMM / all-reduce chunk pipeline
    Mg, Ng, Kg = 2560, 2048, 12044  # ragged K: the last rank's shard is shorter (layers.cpp:42)
    grp = tb.PeerGroup(world, rank, torch.cuda.current_device(), max(M * N, E_big, Mo * No, Mg * Ng), dist)
    ys = []
    for it in range(5):  # several epochs: exercises both send-buffer slots
        for leaf in (tb.LEAF_TCGEN05, tb.LEAF_FMA):
            ys.append(grp.row_parallel_forward(xs, ws, K, cfg, 8, leaf).clone())
    torch.cuda.synchronize()
    for i in range(2, len(ys)):
        assert torch.equal(ys[i].view(torch.int32), ys[i % 2].view(torch.int32)), f"epoch {i} differs"
    # plain all-reduce of rank-dependent data: must equal the local Algorithm-2 result
    parts = [torch.full((3, 5), float(r + 1) * 1e8 if r % 2 == 0 else 1.0, device="cuda") for r in range(world)]
    red = grp.tree_all_reduce(parts[rank])
    local = tb.tree_all_reduce(tb.DeviceGroup(world), parts)
    torch.cuda.synchronize()
    assert torch.equal(red.view(torch.int32), local.view(torch.int32))
    # large payloads take the two-phase path; interleave with one-shot epochs and an
    # unaligned output view -- every result must equal the local Algorithm-2 result
    gb = torch.Generator(device="cuda")
    gb.manual_seed(99)
    big = [torch.randn(E_big, device="cuda", generator=gb) * (1e6 if r % 2 else 1.0) for r in range(world)]
    local_big = tb.tree_all_reduce(tb.DeviceGroup(world), big)
    for it in range(4):
        red_big = grp.tree_all_reduce(big[rank])
        small = grp.tree_all_reduce(parts[rank])
        buf = torch.empty(E_big + 1, device="cuda")
        odd = grp.tree_all_reduce(big[rank], out=buf[1:])
        torch.cuda.synchronize()
        assert torch.equal(red_big.view(torch.int32), local_big.view(torch.int32)), f"two-phase differs ({it})"
        assert torch.equal(odd.view(torch.int32), local_big.view(torch.int32)), f"unaligned out differs ({it})"
        assert torch.equal(small.view(torch.int32), local.view(torch.int32)), f"one-shot differs ({it})"
    # overlapped chunk pipeline (GEMM of chunk c+1 beside the all-reduce of chunk c)
    xo = torch.randn(Mo, K, generator=g, device="cuda").to(torch.bfloat16)
    wo = torch.randn(K, No, generator=g, device="cuda").to(torch.bfloat16)
    yo_ref = tb.tree_matmul(xo, wo, cfg, tb.LEAF_TCGEN05)
    for it in range(3):
        yo = grp.row_parallel_forward(xo[:, kb:ke].contiguous(), wo[kb:ke].contiguous(), K, cfg, 8, tb.LEAF_TCGEN05)
        torch.cuda.synchronize()
        assert torch.equal(yo.view(torch.int32), yo_ref.view(torch.int32)), f"overlapped forward differs ({it})"
    # ragged rows (M % 256 != 0): the fused GEMM -> all-reduce tile flags / halves
    xr = xo[:1000].contiguous()
    yr_ref = tb.tree_matmul(xr, wo, cfg, tb.LEAF_TCGEN05)
    for it in range(2):
        yr = grp.row_parallel_forward(xr[:, kb:ke].contiguous(), wo[kb:ke].contiguous(), K, cfg, 8, tb.LEAF_TCGEN05)
        torch.cuda.synchronize()
        assert torch.equal(yr.view(torch.int32), yr_ref.view(torch.int32)), f"ragged forward differs ({it})"
    # ragged K (the fused-vs-separate choice must not depend on the
    # rank's own K range, or the ranks take different paths and hang)
    xg = torch.randn(Mg, Kg, generator=g, device="cuda").to(torch.bfloat16)
    wg = torch.randn(Kg, Ng, generator=g, device="cuda").to(torch.bfloat16)
    gb_, ge_ = tb.make_row_shard_plan(Kg, cfg, world, 8).bounds[rank]
    yg_ref_g = tb.row_parallel_forward(xg, wg, tb.DeviceGroup(world), cfg, 8, tb.LEAF_TCGEN05)
    for it in range(2):
        yg = grp.row_parallel_forward(xg[:, gb_:ge_].contiguous(), wg[gb_:ge_].contiguous(), Kg, cfg, 8,
                                      tb.LEAF_TCGEN05)
        torch.cuda.synchronize()
        assert torch.equal(yg.view(torch.int32), yg_ref_g.view(torch.int32)), f"ragged-K forward differs ({it})"
    fused = grp.fused_count()
    if os.environ.get("TBIK_GROUP_FUSED", "1") != "0":
        assert fused == 7, f"fused GEMM + all-reduce kernel ran {fused} times, expected 7"
    else:
        assert fused == 0
    # host-buffer pipeline through the group: chunked epochs, same bits as the device call
    xh = x[:, kb:ke].contiguous().cpu().pin_memory()
    yh = grp.row_parallel_forward_hostio(xh, ws, K, cfg, 8, tb.LEAF_TCGEN05, chunk_rows=24)
    torch.cuda.synchronize()
    assert torch.equal(yh.view(torch.int32), ys[0].cpu().view(torch.int32)), "host-io group result differs"
    out = os.environ["TBIK_TEST_OUT"]
    np.save(out, ys[0].cpu().numpy())
    if rank == 0:
        ref = tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05)
        np.save(out + ".ref.npy", ref.cpu().numpy())
    dist.barrier()
    grp.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
