"""CPU suite for the C ABI boundary (no GPU needed).

* the library loads and exports every symbol include/tbik_b200.h declares;
* the host-only planner entry points equal the reference (golden table);
* compute entry points fail LOUDLY without a device (no CPU fallback);
* error codes mirror tbik::ErrorCode (errors.hpp:8-20) one to one.
"""
import ctypes as C

import numpy as np
import pytest


def test_exports_every_header_symbol(tb):
    names = tb.header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(tb.lib, n)]
    assert not missing, f"declared but not exported: {missing}"


def test_status_strings_mirror_error_codes(tb):
    expect = ["BadDimension", "ShapeMismatch", "BadMagic", "Truncated", "UnknownDtype",
              "PlanInfeasible", "ShardError", "BadWorldSize", "CollectiveMismatch", "BadArgument", "Io"]
    for i, name in enumerate(expect, 1):
        assert tb.lib.tbik_status_string(i).decode() == name
        assert tb.ErrorCode(i).name == name


def test_default_block_config(tb):
    # matmul.cpp:11-14
    assert tb.default_block_config(tb.BF16) == tb.BlockConfig(64, 256, 128, 0)
    assert tb.default_block_config(tb.F32) == tb.BlockConfig(32, 128, 64, 0)


def test_planner_matches_reference_golden(tb, golden):
    for row in golden["plans"]:
        cfg = tb.BlockConfig(64, row["block_k"], 128, row["k_first"])
        if row["status"] == 0:
            p = tb.plan_blocks(row["K"], cfg, row["c_max"])
            assert [p.tiles_total, p.k_first, p.leaves, p.depth] == row["plan"]
        else:
            with pytest.raises(tb.TbikError) as e:
                tb.plan_blocks(row["K"], cfg, row["c_max"])
            assert e.value.code == row["status"]


def test_row_shards_match_reference_golden(tb, golden):
    for row in golden["row_shards"]:
        cfg = tb.BlockConfig(64, row["block_k"], 128, 0)
        if row["status"] == 0:
            sp = tb.make_row_shard_plan(row["K"], cfg, row["tp"], row["c_max"])
            assert [list(b) for b in sp.bounds] == row["bounds"]
        else:
            with pytest.raises(tb.TbikError) as e:
                tb.make_row_shard_plan(row["K"], cfg, row["tp"], row["c_max"])
            assert e.value.code == row["status"]


def test_column_shards(tb):
    assert tb.make_column_shard_plan(4096, 8).bounds[3] == (1536, 2048)
    with pytest.raises(tb.TbikError) as e:
        tb.make_column_shard_plan(512, 3)  # SPEC: C=3 with N=512 -> shard error
    assert e.value.code == tb.ErrorCode.ShardError


def test_planner_random_vs_oracle(tb, orc):
    rng = np.random.default_rng(11)
    for _ in range(300):
        K = int(rng.integers(1, 40000))
        bk = int(rng.choice([1, 16, 64, 100, 128, 256]))
        cmax = int(rng.choice([1, 2, 4, 8, 16]))
        try:
            want = orc.plan_blocks(K, bk, 0, cmax)
        except Exception as e:  # noqa: BLE001
            with pytest.raises(tb.TbikError) as e2:
                tb.plan_blocks(K, tb.BlockConfig(64, bk, 128, 0), cmax)
            assert e2.value.code == e.code
            continue
        p = tb.plan_blocks(K, tb.BlockConfig(64, bk, 128, 0), cmax)
        assert (p.tiles_total, p.k_first, p.leaves, p.depth) == want


def test_device_group_world_size(tb):
    with pytest.raises(tb.TbikError) as e:
        tb.DeviceGroup(3)
    assert e.value.code == tb.ErrorCode.BadWorldSize
    assert tb.DeviceGroup(8).world_size() == 8


def test_no_cpu_fallback(tb):
    """Without an sm_100 GPU the compute path must refuse, never compute on the host."""
    if tb.device_available():
        pytest.skip("a device is visible")
    a = np.zeros((4, 64), np.uint16)
    cfg = tb.BlockConfig(64, 64, 128, 0).c()
    out = np.zeros((4, 64), np.float32)
    st = tb.lib.tbik_tree_matmul(a.ctypes.data, 1, 64, a.ctypes.data, 1, 64, out.ctypes.data, 64,
                                 4, 64, 64, C.byref(cfg), 0, None)
    assert st == tb.ErrorCode.NoDevice
    st = tb.lib.tbik_tree_rmsnorm(a.ctypes.data, 1, 64, out.ctypes.data, 1e-5, out.ctypes.data, 0, 64,
                                  4, 64, None)
    assert st == tb.ErrorCode.NoDevice


def test_argument_errors_are_synchronous(tb):
    cfg = tb.BlockConfig(64, 256, 128, 0).c()
    # block sizes < 1 -> BadArgument (matmul.cpp:150-152)
    bad = tb.BlockConfig(0, 256, 128, 0).c()
    buf = np.zeros(64, np.float32)
    st = tb.lib.tbik_tree_matmul(buf.ctypes.data, 0, 4, buf.ctypes.data, 0, 4, buf.ctypes.data, 4, 4, 4, 4,
                                 C.byref(bad), 0, None)
    assert st == tb.ErrorCode.BadArgument
    st = tb.lib.tbik_tree_matmul(buf.ctypes.data, 7, 4, buf.ctypes.data, 0, 4, buf.ctypes.data, 4, 4, 4, 4,
                                 C.byref(cfg), 0, None)
    assert st == tb.ErrorCode.UnknownDtype
    st = tb.lib.tbik_tree_matmul(buf.ctypes.data, 0, 4, buf.ctypes.data, 0, 4, buf.ctypes.data, 4, 0, 4, 4,
                                 C.byref(cfg), 0, None)
    assert st == tb.ErrorCode.BadDimension
