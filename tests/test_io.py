"""The reference's TBIK matrix file (matrix.hpp:86-87, matrix.cpp:185-284) through
tbik_matrix_write / tbik_matrix_read, cross-checked against the UNMODIFIED
reference library (oracle/_ref): byte-identical files both ways and the same
error codes for every malformed input.  Host only (no GPU needed)."""
import os
import struct

import numpy as np
import pytest
import torch


def _torch_from(arr):
    if arr.dtype == np.uint16:
        return torch.from_numpy(arr.view(np.int16).copy()).view(torch.bfloat16)
    return torch.from_numpy(arr.copy())


def _np_from(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


@pytest.mark.parametrize("dtype,rows,cols", [("f32", 3, 5), ("bf16", 4, 7), ("f32", 1, 1), ("bf16", 64, 1)])
def test_round_trip_and_reference_byte_identity(tb, ref, tmp_path, dtype, rows, cols):
    m = ref.random_normal(3, 1, max(rows, 1), cols, dtype)[:rows].copy()
    ours, theirs = tmp_path / "ours.tbik", tmp_path / "theirs.tbik"
    tb.matrix_write(str(ours), _torch_from(m))
    assert ref.matrix_write(str(theirs), m) == 0
    assert ours.read_bytes() == theirs.read_bytes(), "file bytes differ from the reference's matrix_write"
    back = _np_from(tb.matrix_read(str(theirs)))
    assert back.dtype == m.dtype and back.shape == m.shape
    assert np.array_equal(back.view(np.uint8), m.view(np.uint8))
    st, rback = ref.matrix_read(str(ours))
    assert st == 0 and np.array_equal(rback.view(np.uint8), m.view(np.uint8))


def _header(version=1, dtype=0, rows=2, cols=2):
    return b"TBIK" + struct.pack("<HHQQ", version, dtype, rows, cols)


@pytest.mark.parametrize("name,blob,code", [
    ("short_header", b"TBIK\x01\x00", "Truncated"),
    ("bad_magic", b"XBIK" + struct.pack("<HHQQ", 1, 0, 1, 1) + b"\0" * 4, "BadMagic"),
    ("bad_version", _header(version=2) + b"\0" * 16, "UnknownDtype"),
    ("bad_dtype", _header(dtype=7) + b"\0" * 16, "UnknownDtype"),
    ("short_payload", _header() + b"\0" * 15, "Truncated"),
    ("long_payload", _header() + b"\0" * 17, "Truncated"),
    ("zero_rows", _header(rows=0), "BadDimension"),
])
def test_malformed_files_same_errors_as_reference(tb, ref, tmp_path, name, blob, code):
    p = tmp_path / f"{name}.tbik"
    p.write_bytes(blob)
    with pytest.raises(tb.TbikError) as e:
        tb.matrix_read(str(p))
    assert e.value.code == getattr(tb.ErrorCode, code)
    st, _ = ref.matrix_read(str(p))
    assert st == int(getattr(tb.ErrorCode, code)), f"reference returned {st}"


def test_empty_matrix_rejected_like_reference(tb, ref, tmp_path):
    p = str(tmp_path / "e.tbik")
    with pytest.raises(tb.TbikError) as e:
        tb.matrix_write(p, torch.zeros(0, 3))
    assert e.value.code == tb.ErrorCode.BadDimension
    assert ref.matrix_write(p, np.zeros((0, 3), np.float32)) == int(tb.ErrorCode.BadDimension)


def test_io_errors(tb, ref, tmp_path):
    missing = str(tmp_path / "nope" / "x.tbik")
    with pytest.raises(tb.TbikError) as e:
        tb.matrix_read(missing)
    assert e.value.code == tb.ErrorCode.Io
    assert ref.matrix_read(missing)[0] == int(tb.ErrorCode.Io)
    with pytest.raises(tb.TbikError) as e:
        tb.matrix_write(missing, torch.zeros(2, 2))
    assert e.value.code == tb.ErrorCode.Io
    assert ref.matrix_write(missing, np.zeros((2, 2), np.float32)) == int(tb.ErrorCode.Io)


def test_golden_fixtures_readable(tb):
    """The committed TBIK-format golden case (tests/golden/tbik_io/, written by the
    reference library via oracle/gen_golden.py) loads with the expected shapes."""
    d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "tbik_io")
    a = tb.matrix_read(os.path.join(d, "a.tbik"))
    b = tb.matrix_read(os.path.join(d, "b.tbik"))
    c = tb.matrix_read(os.path.join(d, "c_tree.tbik"))
    assert a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16 and c.dtype == torch.float32
    assert a.shape[1] == b.shape[0] and c.shape == (a.shape[0], b.shape[1])
