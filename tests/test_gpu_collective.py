"""GPU parity for the fixed-order tree all-reduce.

* check_collective_symmetry (runner.cpp:129-170): the device all-reduce equals
  oracle tree_reduce element-wise and is rank-symmetric;
* the golden all-reduce fingerprints of the reference (collective.cpp:52-106);
* the one-process-per-GPU group (CUDA IPC + device flag barrier) with two real
  processes: on this single-GPU box both ranks share cuda:0, which exercises
  the whole IPC / epoch / flag protocol; on an NVLink box the same code maps
  peer memory of other GPUs.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT, bits, fp_hex, to_dev

pytestmark = pytest.mark.gpu


def test_all_reduce_golden(tb, cuda, orc, golden):
    for row in golden["all_reduce"]:
        W = row["W"]
        contrib = [orc.random_normal(9, 1000 * W + k, 1, 257, "f32") for k in range(W)]
        g = tb.DeviceGroup(W)
        out = tb.tree_all_reduce(g, [to_dev(c) for c in contrib]).cpu().numpy()
        assert orc.fingerprint(out) == fp_hex(row["tree_fingerprint"])
        ring = tb.ring_reduce_baseline(g, [to_dev(c) for c in contrib]).cpu().numpy()
        assert orc.fingerprint(ring) == fp_hex(row["ring_fingerprint"])


def test_collective_symmetry(tb, cuda, orc):
    for W in (1, 2, 4, 8):
        for seed in range(1, 9):
            contrib = np.stack([orc.random_normal(seed, r + 1000 * W, 1, 8, "f32")[0] for r in range(W)])
            per_rank = tb.tree_all_reduce_per_rank(tb.DeviceGroup(W), [to_dev(c[None, :]) for c in contrib])
            want = np.array([orc.tree_reduce(contrib[:, e]) for e in range(8)], np.float32)
            for out in per_rank:
                assert np.array_equal(bits(out.cpu().numpy()[0]), bits(want))


def test_all_reduce_large_and_unaligned(tb, cuda, orc):
    rng = np.random.default_rng(4)
    for W, n in ((8, 4096 * 64 + 3), (4, 1000001), (2, 5)):
        c = (rng.standard_normal((W, n)) * 10).astype(np.float32)
        want = orc.tree_all_reduce(c)
        xs = [to_dev(c[r][None, :]) for r in range(W)]
        got = tb.tree_all_reduce(tb.DeviceGroup(W), xs).cpu().numpy()[0]
        assert np.array_equal(bits(got), bits(want))
        # unaligned views (offset by one element) take the scalar path
        big = torch.from_numpy(np.concatenate([np.zeros((W, 1), np.float32), c], 1)).to(cuda)
        xs2 = [big[r, 1:][None, :] for r in range(W)]
        got2 = tb.tree_all_reduce(tb.DeviceGroup(W), xs2).cpu().numpy()[0]
        assert np.array_equal(bits(got2), bits(want))


def test_all_reduce_errors(tb, cuda):
    xs = [torch.zeros(1, 4, device=cuda) for _ in range(3)]
    with pytest.raises(tb.TbikError) as e:
        tb.tree_all_reduce(tb.DeviceGroup(4), xs)
    assert e.value.code == tb.ErrorCode.CollectiveMismatch
    with pytest.raises(tb.TbikError) as e:
        tb.tree_all_reduce(tb.DeviceGroup(2), [torch.zeros(1, 4, device=cuda), torch.zeros(1, 5, device=cuda)])
    assert e.value.code == tb.ErrorCode.CollectiveMismatch
    with pytest.raises(tb.TbikError) as e:
        tb.tree_all_reduce(tb.DeviceGroup(2), [torch.zeros(1, 4, device=cuda, dtype=torch.bfloat16)] * 2)
    assert e.value.code == tb.ErrorCode.CollectiveMismatch


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("world", [2, 4])
def test_peer_group_processes(tb, cuda, tmp_path, world, fused):
    """`world` ranks (processes sharing this GPU) run the IPC group end to end:
    row-parallel down_proj shards -> peer-visible buffers -> flag barriers -> tree
    all-reduce (one-shot and two-phase), the fused one-kernel GEMM + all-reduce or
    the overlapped chunk pipeline, and the
    host-buffer path.  Every rank must produce bit-identical outputs equal to the
    single-process TP=1 result."""
    worker = os.path.join(ROOT, "tests", "peer_group_worker.py")
    port = _free_port()
    # fused=1: large row-parallel outputs take the one-kernel GEMM + tile-flag tree
    # all-reduce (tbik_gemm_tc.cu AR variant); fused=0: the chunked two-stream overlap
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
               TBIK_GROUP_FUSED=fused)
    procs = []
    for r in range(world):
        e = dict(env, RANK=str(r), LOCAL_RANK="0", TBIK_TEST_OUT=str(tmp_path / f"rank{r}.npy"))
        procs.append(subprocess.Popen([sys.executable, worker], env=e, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=420)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
    ys = [np.load(tmp_path / f"rank{r}.npy") for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(bits(ys[0]), bits(ys[r])), f"rank {r} diverged"
    y0 = ys[0]
    ref = np.load(tmp_path / "rank0.npy.ref.npy")
    assert np.array_equal(bits(y0), bits(ref)), "group result != TP=1 result"
