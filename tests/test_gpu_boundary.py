"""The rest of the drop-in boundary on the GPU:

* the single-process multi-device DeviceGroup (tbik_local_group_*): rank r's GEMM
  on its own device and stream, partials reduced over peer memory by rank 0's
  device.  On this one-GPU box every rank maps to cuda:0 -- the same code path
  (per-rank streams, events, peer pointers) with local memory;
* leaf_dot (matmul.hpp:48) == the oracle's leaf, bit for bit;
* silu (demo.hpp:56) within 1e-6 of libm;
* baseline_row/column_parallel_forward (layers.hpp:48-54): cuBLAS + the ring sum,
  non-invariant across TP (the reference's check_baseline_kernel_divergence) while
  the tree path is invariant;
* the cuBLAS + NCCL status-quo layer (tbik_baseline_cublas_nccl) with a one-rank
  communicator: equals cuBLAS alone.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import bits, to_dev

pytestmark = pytest.mark.gpu


def test_local_group_row_parallel(tb, cuda):
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    M, K, N = 300, 14336, 512
    x = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    w = torch.randn(K, N, generator=g, device="cuda").to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    ref = tb.row_parallel_forward(x, w, tb.DeviceGroup(1), cfg, 8, tb.LEAF_TCGEN05)
    for W in (2, 4, 8):
        lg = tb.LocalGroup([0] * W)
        sp = tb.make_row_shard_plan(K, cfg, W, 8)
        xs = [x[:, b:e].contiguous() for b, e in sp.bounds]
        ws = [w[b:e].contiguous() for b, e in sp.bounds]
        for leaf in (tb.LEAF_TCGEN05, tb.LEAF_FMA):
            y = lg.row_parallel_forward(xs, ws, K, cfg, 8, leaf)
            want = ref if leaf == tb.LEAF_TCGEN05 else tb.row_parallel_forward(x, w, tb.DeviceGroup(1), cfg, 8, leaf)
            torch.cuda.synchronize()
            assert torch.equal(y.view(torch.int32), want.view(torch.int32)), f"W={W} leaf={leaf}"
        lg.close()
    with pytest.raises(tb.TbikError) as e:
        tb.LocalGroup([0, 0, 0])
    assert e.value.code == tb.ErrorCode.BadWorldSize


def test_leaf_dot_matches_oracle_leaf(tb, cuda, orc):
    rng = np.random.default_rng(3)
    for n in (1, 7, 256, 1000):
        a = (rng.standard_normal(n) * np.exp2(rng.integers(-20, 20, n))).astype(np.float32)
        b = rng.standard_normal(n).astype(np.float32)
        want = np.float32(orc.lib.tbo_leaf_dot(a.ctypes.data_as(C.POINTER(C.c_float)), b.ctypes.data_as(C.POINTER(C.c_float)), n))
        got = tb.leaf_dot(to_dev(a), to_dev(b)).cpu().numpy()
        assert bits(got)[0] == bits(np.array([want], np.float32))[0], n


def test_silu(tb, cuda):
    x = torch.linspace(-30, 30, 4001, device="cuda").reshape(1, -1)
    y = tb.silu(x)
    xd = x.double()
    want = xd / (1 + torch.exp(-xd))
    rel = ((y.double() - want).abs() / want.abs().clamp_min(1e-30)).max().item()
    assert rel < 1e-6, rel
    yb = tb.silu(x.to(torch.bfloat16))
    assert torch.equal(yb, tb.silu(x.to(torch.bfloat16).float()))


def test_baseline_layers_diverge_tree_does_not(tb, cuda, orc):
    a = orc.random_normal(1, 1, 4, 4096, "f32")
    b = orc.random_normal(1, 2, 4096, 8, "f32")
    x, w = to_dev(a), to_dev(b)
    base, tree = set(), set()
    for tp in (1, 2, 4, 8):
        yb = tb.baseline_row_parallel_forward(x, w, tb.DeviceGroup(tp)).cpu().numpy()
        base.add(orc.fingerprint(yb))
        yt = tb.row_parallel_forward(x, w, tb.DeviceGroup(tp), tb.BlockConfig(32, 128, 64, 0), 8, tb.LEAF_FMA)
        tree.add(orc.fingerprint(yt.cpu().numpy()))
    assert len(base) >= 2 and len(tree) == 1
    c1 = tb.baseline_column_parallel_forward(x, w, tb.DeviceGroup(1))
    c4 = tb.baseline_column_parallel_forward(x, w, tb.DeviceGroup(4))
    assert torch.equal(c1, c4)
    with pytest.raises(tb.TbikError) as e:
        tb.baseline_row_parallel_forward(x[:, :4095], w[:4095], tb.DeviceGroup(2))
    assert e.value.code == tb.ErrorCode.ShardError


def test_cublas_nccl_baseline_single_rank(tb, cuda):
    lib = tb.lib
    uid = (C.c_char * 128)()
    tb.api.check(lib.tbik_nccl_unique_id(uid))
    comm = C.c_void_p()
    tb.api.check(lib.tbik_nccl_comm_create(1, 0, 0, uid, C.byref(comm)))
    g = torch.Generator(device="cuda")
    g.manual_seed(2)
    x = torch.randn(64, 1024, generator=g, device="cuda").to(torch.bfloat16)
    w = torch.randn(1024, 256, generator=g, device="cuda").to(torch.bfloat16)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for out_f32, dt in ((1, torch.float32), (0, torch.bfloat16)):
        y = torch.empty(64, 256, device="cuda", dtype=dt)
        tb.api.check(lib.tbik_baseline_cublas_nccl(comm, C.c_void_p(x.data_ptr()), 1, 1024, C.c_void_p(w.data_ptr()),
                                                   1, 256, C.c_void_p(y.data_ptr()), 64, 256, 1024, out_f32, s))
        torch.cuda.synchronize()
        ref = (x.float() @ w.float())
        assert (y.float() - ref).abs().max().item() < (1e-3 if out_f32 else 0.5)
    lib.tbik_nccl_comm_destroy(comm)
