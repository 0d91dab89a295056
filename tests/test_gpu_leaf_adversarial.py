"""Adversarial inputs for the tcgen05 leaf: the product
path's one numeric contract with the reference's leaf_dot (matmul.cpp:69-75).

Each leaf P_t (block_k = 256 products, 16 tcgen05 K=16 steps) is compared with the
exact dot product (math.fsum of the exactly representable f64 products: correctly
rounded, far below f32 resolution) under patterns that stress the tensor core's
internal accumulation INSIDE one K=16 step:

  cancel      [2^27, 1, -2^27, 1, ...] inside one K=16 step (exact in-leaf cancellation)
  spread      +-2^e, e uniform in [-60, 60], per product
  absorb      one 2^60 term, 255 unit terms
  zeros       all -0.0 (signed zeros), and +0 / -0 mixes
  tiny        products below 2^-126 (f32 subnormal range)
  subnormal   bf16 subnormal inputs (exponent field 0)
  extreme     inputs near the bf16 maximum against 2^-100 weights
  random      N(0,1) * 2^randint(-60, 60)

The stated bound is

  |P_tc - P_exact| <= (block_k / 8) u * sum_k |a_k b_k|  +  F,     u = 2^-24,

i.e. at most 2u of sum|ab| per tcgen05 K=16 step (one aligned, truncating
accumulation into the f32 accumulator per step; 32u at block_k = 256), where F =
sum of |a_k b_k| over products below 2^-126 (f32 subnormal results: the tensor
core may flush them) -- F = 0 for inputs and products in the normal range.  The
reference's own leaf (an n-long fma chain) carries the classical gamma_n ~ n u
bound; its measured worst case on the same data is printed next to the tcgen05 one.  Every full GEMM output
must still equal the oracle tree over the GPU's own leaves bit for bit (signed
zeros included: the tree's 0 + P canonicalises a -0 leaf, matmul.cpp:101-103).
"""
import math

import numpy as np
import pytest
import torch

from conftest import bits, to_dev

pytestmark = pytest.mark.gpu

K, N, BK = 512, 32, 256


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """f32 -> bf16 bits, round to nearest even (inputs here are bf16-exact or near)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def widen(b16: np.ndarray) -> np.ndarray:
    return (b16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def signs(rng, shape):
    return rng.choice([-1.0, 1.0], shape)


def cases(rng, rows=16):
    """pattern -> (A [rows x K], B [K x N]) as f32 values that are exact in bf16,
    every product and partial sum finite (overflow / NaN are outside the contract,
    SPEC.md:31)."""
    out = {}
    c = np.zeros((rows, K), np.float32)
    for s_ in range(0, K, 16):
        c[:, s_:s_ + 4] = [2.0 ** 27, 1.0, -2.0 ** 27, 1.0]
    c[1::2] = np.roll(c[1::2], 5, axis=1)  # odd rows: the cancelling pair straddles two K=16 steps
    out["cancel"] = (c, np.where(rng.random((K, N)) < 0.5, 1.0, np.exp2(rng.integers(-3, 4, (K, N)))))
    out["spread"] = (signs(rng, (rows, K)) * np.exp2(rng.integers(-60, 61, (rows, K))),
                     signs(rng, (K, N)) * np.exp2(rng.integers(-60, 61, (K, N))))
    ab = np.ones((rows, K))
    ab[:, ::BK] = 2.0 ** 60
    ab[rows // 2:, 7::BK] = -2.0 ** 60  # ... and cancelled again inside the same leaf
    out["absorb"] = (ab, signs(rng, (K, N)))
    z = np.where(rng.random((rows, K)) < 0.5, -0.0, 0.0)
    z[0] = -0.0
    out["signed_zero"] = (z, signs(rng, (K, N)))
    out["tiny_products"] = (signs(rng, (rows, K)) * np.exp2(rng.integers(-75, -55, (rows, K))),
                            signs(rng, (K, N)) * np.exp2(rng.integers(-75, -55, (K, N))))
    sub = (rng.integers(1, 128, (rows, K)).astype(np.uint32) | (rng.integers(0, 2, (rows, K)).astype(np.uint32) << 15))
    out["subnormal_inputs"] = ((sub << 16).view(np.float32),
                               signs(rng, (K, N)) * np.exp2(rng.integers(90, 110, (K, N))))
    out["extreme"] = (signs(rng, (rows, K)) * np.exp2(rng.integers(110, 119, (rows, K))),
                      signs(rng, (K, N)) * np.exp2(rng.integers(-110, -100, (K, N))))
    out["random"] = (rng.standard_normal((rows, K)) * np.exp2(rng.integers(-40, 41, (rows, K))),
                     rng.standard_normal((K, N)) * np.exp2(rng.integers(-40, 41, (K, N))))
    return {k: (a.astype(np.float32), b.astype(np.float32)) for k, (a, b) in out.items()}


def test_tcgen05_leaf_adversarial(tb, cuda, orc):
    rng = np.random.default_rng(2025)
    u = 2.0 ** -24
    cfg = tb.BlockConfig(64, BK, 128, 1)
    report = {}
    viol = []
    for name, (a, b) in cases(rng).items():
        a16, b16 = bf16_bits(a), bf16_bits(b)
        af, bf = widen(a16), widen(b16)
        da, db = to_dev(a16), to_dev(b16)
        leaves = tb.tree_matmul_leaves(da, db, cfg, tb.LEAF_TCGEN05).cpu().numpy()
        fleaves = tb.tree_matmul_leaves(da, db, cfg, tb.LEAF_FMA).cpu().numpy()
        worst_rel = worst_flush = worst_fma = 0.0
        for t in range(K // BK):
            sl = slice(t * BK, (t + 1) * BK)
            for i in range(a.shape[0]):
                prods = af[i, sl, None] * bf[sl, :]      # exact in f64 (8-bit x 8-bit mantissas)
                absdot = np.abs(prods).sum(0)
                small = (np.abs(prods) < 2.0 ** -126) | (np.abs(af[i, sl, None]) < 2.0 ** -126) | \
                        (np.abs(bf[sl, :]) < 2.0 ** -126)
                flushed = np.where(small, np.abs(prods), 0.0).sum(0)
                for j in range(N):
                    exact = math.fsum(prods[:, j])
                    err = abs(float(leaves[t, i, j]) - exact)
                    ferr = abs(float(fleaves[t, i, j]) - exact)
                    if flushed[j] == 0:
                        worst_rel = max(worst_rel, err / (u * absdot[j]) if absdot[j] > 0 else (0 if err == 0 else 1e30))
                        worst_fma = max(worst_fma, ferr / (u * absdot[j]) if absdot[j] > 0 else 0)
                    else:
                        worst_flush = max(worst_flush, err / flushed[j])
                    if err > (BK / 8) * u * absdot[j] + flushed[j]:
                        viol.append((name, t, i, j, float(leaves[t, i, j]), exact, absdot[j], flushed[j]))
        report[name] = (worst_rel, worst_flush, worst_fma)
        # the full GEMM == the oracle tree over the GPU's own leaves, bit for bit
        y = tb.tree_matmul(da, db, cfg, tb.LEAF_TCGEN05).cpu().numpy()
        want = orc.tree_over_leaves(leaves, 1)
        assert np.array_equal(bits(y), bits(want)), name
        if name == "signed_zero":  # a -0 leaf never leaks: 0 + P canonicalises it (matmul.cpp:101-103)
            assert np.all(bits(y) == 0), "a -0.0 output escaped the tree's canonicalisation"
            yf = tb.tree_matmul(da, db, cfg, tb.LEAF_FMA).cpu().numpy()
            assert np.array_equal(bits(yf), bits(y))
    print("leaf vs exact, worst |P - exact| / (u sum|ab|) over normal-range products: tcgen05 | fma chain"
          " (reference leaf_dot order); tcgen05 worst |P - exact| / (flushed sum) where products underflow:")
    for k, (r, f, fm) in report.items():
        print(f"  {k:18s} tcgen05 {r:8.3f} u   fma {fm:8.3f} u   flushed {f:6.3f}")
    assert not viol, f"{len(viol)} leaves outside the bound, e.g. {viol[:4]}"


@pytest.mark.parametrize("M", [1024, 4096])
def test_tp_invariance_at_bench_config(tb, cuda, M):
    """TP = 1/2/4/8 bit identity of the tensor-core path at the bench shape (Llama
    down_proj K = 14336, N = 4096, M = 1024 / 4096: the FULL pair-tile launch)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(M)
    x = torch.randn(M, 14336, generator=g, device="cuda").to(torch.bfloat16)
    w = torch.randn(14336, 4096, generator=g, device="cuda").to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    ref = tb.row_parallel_forward(x, w, tb.DeviceGroup(1), cfg, 8, tb.LEAF_TCGEN05)
    for tp in (2, 4, 8):
        y = tb.row_parallel_forward(x, w, tb.DeviceGroup(tp), cfg, 8, tb.LEAF_TCGEN05)
        assert torch.equal(ref.view(torch.int32), y.view(torch.int32)), f"M={M} tp={tp}"
    # batch invariance across the launch shapes: rows computed alone equal the full-M rows
    for r0, r1 in ((0, 1), (1000, 1017), (M - 300, M)):
        part = tb.tree_matmul(x[r0:r1].contiguous(), w, cfg, tb.LEAF_TCGEN05)
        assert torch.equal(part.view(torch.int32), ref[r0:r1].view(torch.int32)), (r0, r1)


@pytest.mark.parametrize("M", [1024, 4096])
def test_tree_over_gpu_leaves_at_bench_config(tb, cuda, orc, M):
    """The in-kernel tree (k_first = 7, 8 groups) == the oracle tree over the GPU's own
    leaves, bit for bit, at the bench shape (a 1024-column slice of N keeps the
    56 dumped leaves within host memory; the launch is still the FULL pair-tile one)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(7 + M)
    Nn = 1024
    x = torch.randn(M, 14336, generator=g, device="cuda").to(torch.bfloat16)
    w = torch.randn(14336, Nn, generator=g, device="cuda").to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    y = tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05).cpu().numpy()
    leaves = tb.tree_matmul_leaves(x, w, cfg, tb.LEAF_TCGEN05).cpu().numpy()
    want = orc.tree_over_leaves(leaves, tb.plan_blocks(14336, cfg, 1).k_first)
    assert np.array_equal(bits(y), bits(want)), f"mismatches: {(bits(y) != bits(want)).sum()}"
