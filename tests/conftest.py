import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libtbik_ref.so not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def tb():
    import paper_2511_17826_b200 as tb
    return tb


@pytest.fixture(scope="session")
def cuda(tb):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    torch.cuda.set_device(0)
    assert tb.device_available(), "libtbik_b200 sees no sm_100 device"
    return torch.device("cuda:0")


def bits(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def to_dev(arr: np.ndarray, device="cuda:0"):
    """numpy bf16-bits (uint16) or f32 -> torch CUDA tensor of the same bits."""
    import torch
    if arr.dtype == np.uint16:
        return torch.from_numpy(arr.view(np.int16).copy()).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(arr, np.float32)).to(device)


def fp_hex(h: str) -> int:
    return int(h, 16)
