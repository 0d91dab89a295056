"""CPU checks of the drop-in C++ boundary:

* include/tbik/<name>.hpp exists for every reference hot-path header and declares
  every function / class the reference header declares (parsed from
  /root/reference/proj/include/tbik/ when it is present -- this container);
* a caller written against the reference headers compiles against ours, and the
  C++ layer links (tests/cpp/tbik_verify, built by build());
* the exported C++ symbols of libtbik_b200 include the reference signatures the
  headers declare (mangled names of the reference's own declarations);
* schedule knobs: every documented name is accepted, an unknown one is
  BadArgument, and the library reads no environment variable.
"""
import os
import re
import subprocess

import pytest

from conftest import ROOT

REF_INC = "/root/reference/proj/include/tbik"
HOT = ["errors", "numerics", "rng", "matrix", "matmul", "collective", "layers"]


def _decls(text: str):
    text = re.sub(r"//[^\n]*", "", text)
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    funcs = set(re.findall(r"\b([a-z_][a-z0-9_]*)\s*\(", text))
    classes = set(re.findall(r"\b(?:class|struct|enum class)\s+(?:TBIK_CPP_API\s+)?([A-Z][A-Za-z0-9_]*)", text))
    return funcs, classes


@pytest.mark.parametrize("name", HOT + ["demo"])
def test_header_exists(name):
    assert os.path.exists(os.path.join(ROOT, "include", "tbik", f"{name}.hpp"))


@pytest.mark.parametrize("name", HOT)
def test_header_declares_reference_surface(name):
    ref = os.path.join(REF_INC, f"{name}.hpp")
    if not os.path.exists(ref):
        pytest.skip("/root/reference is not present")
    rf, rc = _decls(open(ref).read())
    of, oc = _decls(open(os.path.join(ROOT, "include", "tbik", f"{name}.hpp")).read())
    keywords = {"if", "for", "while", "return", "sizeof", "static_cast", "reinterpret_cast", "switch", "defined",
                "memcpy", "fma", "sqrt", "log", "sin", "cos"}
    missing_f = sorted((rf - keywords) - of)
    missing_c = sorted(rc - oc)
    assert not missing_f and not missing_c, f"{name}.hpp lacks {missing_f} {missing_c}"


def test_demo_header_hot_path_functions():
    text = open(os.path.join(ROOT, "include", "tbik", "demo.hpp")).read()
    assert re.search(r"Matrix\s+rmsnorm\(", text) and re.search(r"Matrix\s+silu\(", text)


def test_reference_signatures_exported(tb):
    """The mangled names a reference caller links against."""
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2511_17826_b200", "libtbik_b200.so")],
                         capture_output=True, text=True, check=True).stdout
    demangled = subprocess.run(["c++filt"], input=out, capture_output=True, text=True, check=True).stdout
    for sig in ["tbik::tree_matmul(tbik::Matrix const&, tbik::Matrix const&, tbik::BlockConfig const&)",
                "tbik::plan_blocks(long, tbik::BlockConfig const&, long)",
                "tbik::leaf_dot(float const*, float const*, long)",
                "tbik::log2_exact(long)", "tbik::is_power_of_two(long)",
                "tbik::DeviceGroup::DeviceGroup(int)",
                "tbik::row_parallel_forward(tbik::Matrix const&, tbik::Matrix const&, tbik::DeviceGroup const&, "
                "tbik::BlockConfig const&, long)",
                "tbik::column_parallel_forward(tbik::Matrix const&, tbik::Matrix const&, tbik::DeviceGroup const&, "
                "tbik::BlockConfig const&)",
                "tbik::baseline_row_parallel_forward(tbik::Matrix const&, tbik::Matrix const&, tbik::DeviceGroup const&)",
                "tbik::baseline_column_parallel_forward(tbik::Matrix const&, tbik::Matrix const&, "
                "tbik::DeviceGroup const&)",
                "tbik::tree_all_reduce(tbik::DeviceGroup const&, std::vector<tbik::Matrix, std::allocator<tbik::Matrix> > "
                "const&)",
                "tbik::make_row_shard_plan(long, tbik::BlockConfig const&, int, long)",
                "tbik::rmsnorm(tbik::Matrix const&, std::vector<float, std::allocator<float> > const&, float)",
                "tbik::silu(tbik::Matrix const&)",
                "tbik::bit_fingerprint(tbik::Matrix const&)",
                "tbik::matrix_random_normal(tbik::Rng&, long, long, tbik::Dtype, float, float)"]:
        assert sig in demangled, sig


def test_schedule_knobs(tb):
    for k in tb.api.SCHEDULE_KNOBS:
        tb.set_schedule(k, 1)
        tb.set_schedule(k, -1)
    with pytest.raises(tb.TbikError) as e:
        tb.set_schedule("no_such_knob", 1)
    assert e.value.code == tb.ErrorCode.BadArgument
    tb.set_schedule(None)


def test_library_reads_no_environment():
    """No getenv in the product sources (schedule choices go through tbik_set_schedule)."""
    csrc = os.path.join(ROOT, "paper_2511_17826_b200", "csrc")
    for f in os.listdir(csrc):
        if f.endswith((".cu", ".cuh", ".h")):
            assert "getenv" not in open(os.path.join(csrc, f)).read(), f
