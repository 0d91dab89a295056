"""GPU parity for the tree-ordered RMSNorm and vocab-sharded log-softmax / log-prob.

These semantics are NEW (the reference only has sequential rmsnorm,
demo.cpp:11-34, and an internal softmax_row, demo.cpp:84-97); the canonical
orders are restated in oracle/tbik_oracle.c and the GPU must match that
restatement bit for bit, be TP-invariant (vocab shards 1/2/4/8) and batch-
invariant, and stay close to the reference's sequential rmsnorm.
"""
import numpy as np
import pytest
import torch

from conftest import bits, to_dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,cols,dt", [(4, 4096, "bf16"), (3, 5120, "bf16"), (5, 96, "f32"),
                                          (2, 1000, "bf16"), (7, 4097, "f32")])
def test_tree_rmsnorm_bit_exact(tb, cuda, orc, rows, cols, dt):
    x = orc.random_normal(rows + cols, 1, rows, cols, dt)
    gamma = orc.random_normal(rows + cols, 2, 1, cols, "f32", 1.0, 0.02)[0]
    want = orc.tree_rmsnorm(x, gamma, 1e-5)
    got = tb.rmsnorm(to_dev(x), to_dev(gamma), 1e-5).cpu().numpy()
    assert np.array_equal(bits(got), bits(want))
    ref_seq = orc.rmsnorm_seq(x, gamma, 1e-5)
    assert np.max(np.abs(got - ref_seq) / (np.abs(ref_seq) + 1e-6)) < 1e-5


def test_tree_rmsnorm_bf16_out_and_batch_invariance(tb, cuda):
    torch.manual_seed(0)
    x = torch.randn(300, 4096, device=cuda).to(torch.bfloat16)
    g = torch.randn(4096, device=cuda) * 0.02 + 1
    full = tb.rmsnorm(x, g, 1e-5, out_dtype=torch.bfloat16)
    part = tb.rmsnorm(x[37:38].contiguous(), g, 1e-5, out_dtype=torch.bfloat16)
    assert torch.equal(full[37:38].view(torch.int16), part.view(torch.int16))
    f32 = tb.rmsnorm(x, g, 1e-5)
    # bf16 output = bf16_round of the f32 result (numerics.hpp:49-56)
    assert torch.equal(full.float(), f32.to(torch.bfloat16).float())


@pytest.mark.parametrize("rows,V,G", [(3, 1024, 8), (4, 151936, 8), (2, 128256, 8), (5, 4000, 16),
                                      (1, 64, 8)])
def test_tree_logsoftmax_bit_exact(tb, cuda, orc, rows, V, G):
    rng = np.random.default_rng(V + rows)
    x = (rng.standard_normal((rows, V)) * 3).astype(np.float32)
    targets = rng.integers(0, V, rows)
    lse_w, lp_w, tlp_w = orc.tree_logsoftmax(x, G, targets=targets, full=True)
    dx = to_dev(x)
    tg = torch.from_numpy(targets).to(cuda)
    for tp in (1, 2, 4, 8):
        lse, lp, tlp = tb.log_softmax(dx, G, tp, tg, full=True)
        assert np.array_equal(bits(lse.cpu().numpy()), bits(lse_w)), f"lse tp={tp}"
        assert np.array_equal(bits(lp.cpu().numpy()), bits(lp_w)), f"logprobs tp={tp}"
        assert np.array_equal(bits(tlp.cpu().numpy()), bits(tlp_w)), f"target logprob tp={tp}"
    ref = np.log(np.sum(np.exp(x.astype(np.float64) - x.max(1, keepdims=True)), 1)) + x.max(1)
    assert np.max(np.abs(lse_w - ref)) < 2e-5


def test_logsoftmax_masked_and_extreme(tb, cuda, orc):
    x = np.full((2, 512), -np.inf, np.float32)
    x[0, 7] = 3.0
    x[1, :] = np.linspace(-300, 80, 512, dtype=np.float32)
    lse_w, lp_w, _ = orc.tree_logsoftmax(x, 8, full=True)
    lse, lp, _ = tb.log_softmax(to_dev(x), 8, 1)
    assert np.array_equal(bits(lse.cpu().numpy()), bits(lse_w))
    assert lse[0].item() == 3.0


def test_logsoftmax_bad_groups(tb, cuda):
    x = torch.zeros(2, 1000, device=cuda)
    with pytest.raises(tb.TbikError) as e:
        tb.log_softmax(x, 6, 1)
    assert e.value.code == tb.ErrorCode.ShardError
    with pytest.raises(tb.TbikError) as e:
        tb.log_softmax(x, 8, 3)
    assert e.value.code == tb.ErrorCode.BadWorldSize


@pytest.mark.parametrize("cols,dt,out", [(5120, "bf16", "bf16"), (4096, "bf16", "f32"), (9000, "bf16", "bf16"),
                                         (100, "f32", "f32"), (1000, "f32", "bf16")])
def test_tree_rmsnorm_many_rows(tb, cuda, orc, cols, dt, out):
    """2049 rows (several waves of CTAs, odd count), rows beyond the register
    cache (9000 columns) and ragged rows: oracle bits, and the same bits for a
    slice of the batch (batch invariance)."""
    rows = 2049
    x = orc.random_normal(cols, 3, rows, cols, dt)
    gamma = orc.random_normal(cols, 4, 1, cols, "f32", 1.0, 0.02)[0]
    od = torch.bfloat16 if out == "bf16" else torch.float32
    dx = to_dev(x)
    got = tb.rmsnorm(dx, to_dev(gamma), 1e-5, out_dtype=od)
    want = orc.tree_rmsnorm(x, gamma, 1e-5)
    got_f = got.float().cpu().numpy()
    want_t = torch.from_numpy(want)
    want_f = (want_t.to(torch.bfloat16).float() if out == "bf16" else want_t).numpy()
    assert np.array_equal(bits(got_f), bits(want_f))
    few = tb.rmsnorm(dx[2040:].contiguous(), to_dev(gamma), 1e-5, out_dtype=od)
    assert torch.equal(got[2040:].view(torch.int16 if out == "bf16" else torch.int32),
                       few.view(torch.int16 if out == "bf16" else torch.int32))


def test_logsoftmax_wide_range_blocks(tb, cuda, orc):
    """Logit blocks whose spread exceeds the exp fast path's range (x - max < -86)
    mixed with narrow ones: both exp paths must give the oracle's bits."""
    rng = np.random.default_rng(5)
    V = 32768
    x = (rng.standard_normal((3, V)) * 2).astype(np.float32)
    x[0, ::97] -= 120.0
    x[1, ::1000] += 95.0
    x[2, 5::333] = -np.inf
    lse_w, lp_w, _ = orc.tree_logsoftmax(x, 8, full=True)
    for tp in (1, 8):
        lse, lp, _ = tb.log_softmax(to_dev(x), 8, tp, full=True)
        assert np.array_equal(bits(lse.cpu().numpy()), bits(lse_w)), f"lse tp={tp}"
        assert np.array_equal(bits(lp.cpu().numpy()), bits(lp_w)), f"logprobs tp={tp}"


# ---- F2: the lm_head epilogue emits the log-softmax's chunk states -------------------
@pytest.mark.parametrize("M,K,V,G", [(300, 512, 2 * 16032, 8), (1000, 1024, 4096, 8), (64, 512, 4096, 8),
                                     (300, 512, 8 * 250, 8), (257, 4096, 18992 * 2, 2)])
def test_lm_head_chunk_states_fused(tb, cuda, orc, M, K, V, G):
    """tree_matmul_logits: the (m, s) state of every 16-logit chunk, from the tcgen05
    epilogue (M > 128, V/G % 16 == 0) or the fallback pass (M = 64: skinny GEMM;
    V/G = 250: ragged chunks), equals the oracle's chunk states of the same logits
    bit for bit, and the log-softmax from them equals the log-softmax from the logits
    at every simulated TP."""
    g = torch.Generator(device=cuda).manual_seed(M + V)
    x = (torch.randn(M, K, generator=g, device=cuda) * 0.5).to(torch.bfloat16)
    w = (torch.randn(K, V, generator=g, device=cuda) * 0.2).to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    logits, chunks = tb.tree_matmul_logits(x, w, G, cfg)
    assert torch.equal(logits.view(torch.int32), tb.tree_matmul(x, w, cfg).view(torch.int32))
    m_w, s_w = orc.logsoftmax_chunk_states(logits.cpu().numpy(), G)
    c = chunks.cpu().numpy()
    assert np.array_equal(bits(c[..., 0]), bits(m_w)) and np.array_equal(bits(c[..., 1]), bits(s_w))
    targets = torch.randint(0, V, (M,), generator=g, device=cuda)
    for tp in (1, 2, G):
        a = tb.log_softmax(logits, G, tp, targets, full=True)
        b = tb.log_softmax(logits, G, tp, targets, full=True, chunks=chunks)
        lg, ck = tb.column_parallel_logits(x, w, tb.DeviceGroup(tp), G, cfg)
        d = tb.log_softmax(lg, G, tp, targets, full=True, chunks=ck)
        for u, v_ in zip(a, b):
            assert torch.equal(u.view(torch.int32), v_.view(torch.int32)), f"tp={tp}"
        for u, v_ in zip(a, d):
            assert torch.equal(u.view(torch.int32), v_.view(torch.int32)), f"column-parallel tp={tp}"
    lse_w, _, _ = orc.tree_logsoftmax(logits.cpu().numpy(), G, full=False)
    assert np.array_equal(bits(a[0].cpu().numpy()), bits(lse_w))


def test_chunk_states_masked_and_wide(tb, cuda, orc):
    """-inf logits (masked vocab), whole masked chunks, and chunks whose spread leaves
    the fast exp range: the chunk-state pass equals the oracle."""
    rng = np.random.default_rng(11)
    V, G = 8 * 1024, 8
    x = (rng.standard_normal((5, V)) * 3).astype(np.float32)
    x[0, ::7] = -np.inf
    x[1, 32:64] = -np.inf
    x[2, ::33] -= 150.0
    x[3, :] = 0.0
    x[3, 5] = -0.0
    dx = to_dev(x)
    ns = tb.chunk_states_per_row(V, G)
    ck = torch.empty(5, ns, 2, device=cuda)
    tb.api.check(tb.lib.tbik_logsoftmax_chunk_states(
        tb.api.C.c_void_p(dx.data_ptr()), V, 5, V, G, tb.api.C.c_void_p(ck.data_ptr()), ns, tb.api._stream()))
    m_w, s_w = orc.logsoftmax_chunk_states(x, G)
    c = ck.cpu().numpy()
    assert np.array_equal(bits(c[..., 0]), bits(m_w)) and np.array_equal(bits(c[..., 1]), bits(s_w))


def test_tree_rmsnorm_bf16_out_special_values(tb, cuda, orc):
    """bf16 output through the hardware RNE pair conversion: gamma drives results into
    overflow (inf), bf16-subnormal and tie-to-even territory and through NaN; every
    element equals bf16_round of the f32 result (RNE, canonical NaN 0x7FC0,
    numerics.hpp:49-56) and the f32 path stays bit-exact with the oracle."""
    rows, cols = 3, 4096
    x = orc.random_normal(11, 1, rows, cols, "bf16")
    gamma = np.ones(cols, dtype=np.float32)
    gamma[0::7] = 3e38          # overflow -> +-inf
    gamma[1::7] = 1e-40         # f32-subnormal products -> bf16 subnormals / zeros
    gamma[2::7] = np.nan        # NaN results
    gamma[3::7] = 1.0 + 2.0 ** -8   # results near bf16 rounding ties
    gamma[4::7] = -2.5e-39
    want = orc.tree_rmsnorm(x, gamma, 1e-5)
    got32 = tb.rmsnorm(to_dev(x), to_dev(gamma), 1e-5).cpu().numpy()
    nan = np.isnan(want)  # f32 NaN payloads are outside parity; NaN-ness is not
    assert np.array_equal(np.isnan(got32), nan)
    assert np.array_equal(bits(got32)[~nan], bits(want)[~nan])
    got16 = tb.rmsnorm(to_dev(x), to_dev(gamma), 1e-5, out_dtype=torch.bfloat16).cpu().view(torch.int16).numpy()
    u = want.view(np.uint32).astype(np.uint64)  # bf16_round, vectorised (RNE, canonical NaN)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[np.isnan(want)] = 0x7FC0
    assert orc.bf16_round(float(want.flat[5])) == int(r.flat[5])  # the restatement agrees with the oracle's
    assert np.array_equal(got16, r.view(np.int16).reshape(got16.shape))
