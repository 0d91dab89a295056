"""The north-star claim at real TP: W ranks,
one process each, every rank holding only its weight shards and exchanging data
only through the PeerGroup collectives (row-parallel tree all-reduce, column
all-gather, cross-rank (m, s) merge).  Logits and log-probs must be bit-identical
to the single-process TP = 1 forward.  On this one-GPU box the W processes share
cuda:0 (the IPC / flag protocol is the same as across NVLink)."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, cases, timeout=900):
    worker = os.path.join(ROOT, "tests", "sharded_forward_worker.py")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE=str(world),
               TBIK_SHARD_CASES=cases)
    procs = [subprocess.Popen([sys.executable, worker], env=dict(env, RANK=str(r), LOCAL_RANK="0"),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=timeout)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-4000:]
    print(outs[0])
    assert "SHARDED OK" in outs[0]
    return outs[0]


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_llama_forward_bit_identical(tb, cuda, world):
    out = _run(world, "llama")
    assert "llama3.1-8b x2 B=2 S=160 bit-identical" in out


def test_sharded_qwen_batch_sweep_bit_identical(tb, cuda):
    out = _run(4, "qwen")
    assert "qwen3-32b x2 B=8 S=16 bit-identical" in out


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_c5_logsoftmax_bit_identical(tb, cuda, world):
    out = _run(world, "c5")
    assert "bit-identical" in out
