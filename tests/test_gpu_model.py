"""GPU tests of the TBIK decoder forward (BASELINE configs[2]/[3]).

* each per-token kernel (SiLU*up, residual, RoPE, causal GQA attention) equals
  its oracle restatement bit for bit;
* the Llama-3.1-8B-shaped forward gives bit-identical logits AND log-probs at
  TP = 1/2/4/8 (the north-star claim), for both leaf kinds of the TBIK GEMM;
* batch invariance: a sequence's logits do not depend on what else is batched;
* the Qwen3-32B-shaped stack (q/k norm, block_k=128 down_proj) at TP=8 is
  batch- and TP-invariant together.
Layer counts are reduced for test time; every layer is identical in kind.
"""
import numpy as np
import pytest
import torch

from conftest import bits

pytestmark = pytest.mark.gpu


def u16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def test_silu_mul_and_residual_vs_oracle(tb, cuda, orc):
    import ctypes as C
    rng = np.random.default_rng(0)
    gu = (rng.standard_normal((37, 2 * 300)) * 4).astype(np.float32)
    dgu = torch.from_numpy(gu).to(cuda)
    out = torch.empty(37, 300, device=cuda, dtype=torch.bfloat16)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    tb.api.check(tb.lib.tbik_silu_mul(C.c_void_p(dgu.data_ptr()), 600, 37, 300, C.c_void_p(out.data_ptr()), 300, s))
    assert np.array_equal(u16(out), orc.silu_mul(gu, 300))
    h = torch.randn(37, 300, device=cuda).to(torch.bfloat16)
    f = torch.randn(37, 300, device=cuda)
    want = orc.residual_add(u16(h), f.cpu().numpy())
    tb.api.check(tb.lib.tbik_residual_add(C.c_void_p(h.data_ptr()), 300, C.c_void_p(f.data_ptr()), 300, 37, 300, s))
    assert np.array_equal(u16(h), want)


def test_rope_and_attention_vs_oracle(tb, cuda, orc):
    import ctypes as C

    from paper_2511_17826_b200 import model as mdl
    cfg = mdl.llama31_8b(1)
    cos, sin = mdl.rope_tables(cfg)
    B, S, nq, nkv, D = 2, 48, 4, 2, 128
    rng = np.random.default_rng(1)
    qkv = rng.standard_normal((B * S, (nq + 2 * nkv) * D)).astype(np.float32)
    pos = np.tile(np.arange(S, dtype=np.int32), B)
    dq = torch.from_numpy(qkv).to(cuda)
    dpos = torch.from_numpy(pos).to(cuda)
    dcos, dsin = torch.from_numpy(cos).to(cuda), torch.from_numpy(sin).to(cuda)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    q = torch.empty(B * S, nq * D, device=cuda, dtype=torch.bfloat16)
    k = torch.empty(B * S, nkv * D, device=cuda, dtype=torch.bfloat16)
    ld = qkv.shape[1]
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    tb.api.check(tb.lib.tbik_rope(vp(dq), ld, 0, nq, D, vp(dpos), vp(dcos), vp(dsin), vp(q), nq * D, B * S, s))
    tb.api.check(tb.lib.tbik_rope(vp(dq), ld, nq * D, nkv, D, vp(dpos), vp(dcos), vp(dsin), vp(k), nkv * D, B * S, s))
    assert np.array_equal(u16(q), orc.rope(qkv, 0, nq, D, pos, cos, sin))
    assert np.array_equal(u16(k), orc.rope(qkv, nq * D, nkv, D, pos, cos, sin))
    v = torch.from_numpy(qkv[:, (nq + nkv) * D:].copy()).to(cuda).to(torch.bfloat16)
    out = torch.empty(B * S, nq * D, device=cuda, dtype=torch.bfloat16)
    scale = 1.0 / np.sqrt(D)
    tb.api.check(tb.lib.tbik_attention_prefill(vp(q), nq * D, vp(k), nkv * D, vp(v), nkv * D, B, S, nq, nkv, D,
                                               scale, vp(out), nq * D, s))
    want = orc.attention_prefill(u16(q), u16(k), u16(v), B, S, nq, nkv, scale)
    assert np.array_equal(u16(out), want)
    # close to a float64 causal softmax attention on the same bf16 inputs
    qf = u16(q).astype(np.uint32) << 16
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.float().view(B, S, nq, D).transpose(1, 2), k.float().view(B, S, nkv, D).transpose(1, 2)
        .repeat_interleave(nq // nkv, 1), v.float().view(B, S, nkv, D).transpose(1, 2).repeat_interleave(nq // nkv, 1),
        is_causal=True).transpose(1, 2).reshape(B * S, nq * D)
    assert (out.float() - ref).abs().max().item() < 2e-2
    del qf


@pytest.fixture(scope="module")
def llama2(cuda):
    from paper_2511_17826_b200 import model as mdl
    cfg = mdl.llama31_8b(n_layers=2)
    w = mdl.random_weights(cfg, seed=1)
    return cfg, w


@pytest.mark.parametrize("leaf", ["tc", "fma"])
def test_llama_forward_bit_identical_across_tp(tb, cuda, llama2, leaf):
    from paper_2511_17826_b200 import model as mdl
    cfg, w = llama2
    dec = mdl.TbikDecoder(cfg, w, tb.LEAF_TCGEN05 if leaf == "tc" else tb.LEAF_FMA)
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    B, S = (2, 128) if leaf == "tc" else (1, 16)
    tokens = torch.randint(0, cfg.vocab, (B, S), device=cuda, generator=g)
    targets = torch.randint(0, cfg.vocab, (B * S,), device=cuda, generator=g)
    ref_logits = ref_lp = None
    for tp in (1, 2, 4, 8):
        logits = dec.forward(tokens, tp)
        lse, lp, tlp = dec.log_probs(logits, tp, targets)
        assert torch.isfinite(logits).all()
        if ref_logits is None:
            ref_logits, ref_lp, ref_tlp = logits, lp, tlp
            continue
        assert torch.equal(logits.view(torch.int32), ref_logits.view(torch.int32)), f"logits differ at tp={tp}"
        assert torch.equal(lp.view(torch.int32), ref_lp.view(torch.int32)), f"log-probs differ at tp={tp}"
        assert torch.equal(tlp.view(torch.int32), ref_tlp.view(torch.int32))


def test_llama_forward_batch_invariance(tb, cuda, llama2):
    from paper_2511_17826_b200 import model as mdl
    cfg, w = llama2
    dec = mdl.TbikDecoder(cfg, w)
    g = torch.Generator(device=cuda)
    g.manual_seed(6)
    tokens = torch.randint(0, cfg.vocab, (3, 64), device=cuda, generator=g)
    full = dec.forward(tokens, 2)
    for b in range(3):
        one = dec.forward(tokens[b:b + 1].contiguous(), 4)
        assert torch.equal(one.view(torch.int32), full[b * 64:(b + 1) * 64].view(torch.int32)), b


@pytest.mark.parametrize("rows,nq,nkv", [(300, 32, 8), (1, 8, 8), (77, 64, 8), (1024, 32, 8)])
def test_rope_qkv_equals_rope_and_cast(tb, cuda, rows, nq, nkv):
    """tbik_rope_qkv (RoPE of q and k + bf16 cast of v in one launch) == two
    tbik_rope calls and one tbik_cast_bf16, bit for bit."""
    import ctypes as C
    from paper_2511_17826_b200 import model as mdl
    from paper_2511_17826_b200._lib import lib
    cfg = mdl.llama31_8b(n_layers=1)
    cos, sin = (torch.from_numpy(t).to(cuda) for t in mdl.rope_tables(cfg))
    D = 128
    g = torch.Generator(device=cuda).manual_seed(rows)
    qkv = torch.randn(rows, (nq + 2 * nkv) * D, device=cuda, generator=g) * 3
    pos = torch.randint(0, cfg.max_pos, (rows,), device=cuda, generator=g, dtype=torch.int32)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    q = torch.empty(rows, nq * D, device=cuda, dtype=torch.bfloat16)
    k = torch.empty(rows, nkv * D, device=cuda, dtype=torch.bfloat16)
    v = torch.empty(rows, nkv * D, device=cuda, dtype=torch.bfloat16)
    assert lib.tbik_rope_qkv(vp(qkv), qkv.stride(0), nq, nkv, D, vp(pos), vp(cos), vp(sin), vp(q), vp(k), vp(v),
                             rows, st) == 0
    q2, k2, v2 = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ld = qkv.stride(0)
    assert lib.tbik_rope(vp(qkv), ld, 0, nq, D, vp(pos), vp(cos), vp(sin), vp(q2), nq * D, rows, st) == 0
    assert lib.tbik_rope(vp(qkv), ld, nq * D, nkv, D, vp(pos), vp(cos), vp(sin), vp(k2), nkv * D, rows, st) == 0
    assert lib.tbik_cast_bf16(C.c_void_p(qkv.data_ptr() + 4 * (nq + nkv) * D), ld, rows, nkv * D, vp(v2), nkv * D,
                              st) == 0
    for a_, b_ in ((q, q2), (k, k2), (v, v2)):
        assert torch.equal(a_.view(torch.int16), b_.view(torch.int16))


@pytest.mark.parametrize("B,S", [(2, 128), (2, 16)])
def test_llama_forward_pdl_on_off_same_bits(tb, cuda, llama2, B, S):
    """Programmatic dependent launch only moves kernel scheduling: the forward
    (prefill sizes on the pair-tile GEMMs, decode sizes on the skinny kernel, each
    GEMM following a kernel that triggered its dependents early) gives the same
    logits with the GEMMs launched with and without the attribute, eager and
    repeated back to back."""
    from paper_2511_17826_b200 import model as mdl
    cfg, w = llama2
    dec = mdl.TbikDecoder(cfg, w)
    g = torch.Generator(device=cuda)
    g.manual_seed(9)
    tokens = torch.randint(0, cfg.vocab, (B, S), device=cuda, generator=g)
    with tb.schedule(tc_pdl=0, sk_pdl=0):
        ref = dec.forward(tokens, 1).clone()
    for _ in range(3):
        with tb.schedule(tc_pdl=1, sk_pdl=1):
            got = dec.forward(tokens, 1)
        assert torch.equal(got.view(torch.int32), ref.view(torch.int32))


def test_llama_forward_graph_decode_size(tb, cuda, llama2):
    """A CUDA-graph capture of a decode-sized forward (2 x 16 tokens: every GEMM on
    the swap-AB skinny kernel, its K split in thread-block clusters) replays to
    the eager bits, at TP = 1 and 8."""
    from paper_2511_17826_b200 import model as mdl
    cfg, w = llama2
    dec = mdl.TbikDecoder(cfg, w)
    g = torch.Generator(device=cuda)
    g.manual_seed(8)
    tokens = torch.randint(0, cfg.vocab, (2, 16), device=cuda, generator=g)
    for tp in (1, 8):
        eager = dec.forward(tokens, tp).clone()
        graph, (logits, _lse, _lp) = dec.capture(tokens, tp)
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(logits.view(torch.int32), eager.view(torch.int32)), f"graph replay differs at tp={tp}"


def test_qwen3_stack_tp8_batch_sweep(tb, cuda):
    from paper_2511_17826_b200 import model as mdl
    cfg = mdl.qwen3_32b(n_layers=2)
    w = mdl.random_weights(cfg, seed=2)
    dec = mdl.TbikDecoder(cfg, w)
    g = torch.Generator(device=cuda)
    g.manual_seed(7)
    S = 32
    tokens = torch.randint(0, cfg.vocab, (8, S), device=cuda, generator=g)
    ref = dec.forward(tokens[:1].contiguous(), 1)          # batch 1, TP 1
    _, ref_lp, _ = dec.log_probs(ref, 1)
    for batch in (2, 8):
        out = dec.forward(tokens[:batch].contiguous(), 8)  # batch > 1, TP 8
        assert torch.equal(out[:S].view(torch.int32), ref.view(torch.int32)), f"batch {batch}"
        _, lp, _ = dec.log_probs(out, 8)
        assert torch.equal(lp[:S].view(torch.int32), ref_lp.view(torch.int32))
    del w
    torch.cuda.empty_cache()


@pytest.mark.parametrize("leaf", ["tc", "fma"])
@pytest.mark.parametrize("M", [64, 300, 2048])
def test_fused_silu_gate_up_equals_unfused(tb, cuda, leaf, M):
    """SiLU*up in the gate_up GEMM epilogue == column-parallel tree GEMM followed by
    tbik_silu_mul, bit for bit, for every simulated TP size (epilogue and fallback)."""
    import ctypes as C
    lf = tb.LEAF_TCGEN05 if leaf == "tc" else tb.LEAF_FMA
    K, inter = 4096, 1024
    g = torch.Generator(device=cuda).manual_seed(M)
    x = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(K, 2 * inter, device=cuda, generator=g) * 0.02).to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    gu = tb.column_parallel_forward(x, w, tb.DeviceGroup(1), cfg, lf)
    ref = torch.empty(M, inter, device=cuda, dtype=torch.bfloat16)
    tb.api.check(tb.lib.tbik_silu_mul(C.c_void_p(gu.data_ptr()), 2 * inter, M, inter, C.c_void_p(ref.data_ptr()),
                                      inter, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    w_il = tb.interleave_gate_up(w)
    for tp in (1, 2, 4, 8):
        act = tb.tree_matmul_silu_mul(x, w_il, tb.DeviceGroup(tp), cfg, lf)
        torch.cuda.synchronize()
        assert torch.equal(act.view(torch.int16), ref.view(torch.int16)), f"tp={tp}"


@pytest.mark.parametrize("form,S", [("mma_sync", 200), ("tcgen05", 200), ("tcgen05", 512), ("tcgen05", 37),
                                    ("tcgen05", 1000)])
def test_attention_tc_invariance_and_tolerance(tb, cuda, form, S):
    """Tensor-core flash attention (the mma.sync form and the tcgen05 form, knob
    attn_tc5): bit-identical across batch composition, head sharding and reruns;
    within tolerance of the exact two-pass kernel and of an f64 causal softmax."""
    with tb.schedule(attn_tc5=1 if form == "tcgen05" else 0):
        _attention_tc_checks(tb, cuda, S)


def _attention_tc_checks(tb, cuda, S):
    import ctypes as C
    B, nq, nkv, D = 3, 8, 2, 128
    g = torch.Generator(device=cuda).manual_seed(7)
    q = (torch.randn(B * S, nq * D, device=cuda, generator=g) * 2).to(torch.bfloat16)
    k = (torch.randn(B * S, nkv * D, device=cuda, generator=g) * 2).to(torch.bfloat16)
    v = torch.randn(B * S, nkv * D, device=cuda, generator=g).to(torch.bfloat16)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    scale = 1.0 / np.sqrt(D)

    def run(fn, qq, kk, vv, b, nqh, nkvh):
        o = torch.empty(b * S, nqh * D, device=cuda, dtype=torch.bfloat16)
        tb.api.check(fn(vp(qq), qq.stride(0), vp(kk), kk.stride(0), vp(vv), vv.stride(0), b, S, nqh, nkvh, D,
                        scale, vp(o), o.stride(0), s))
        return o

    fast = run(tb.lib.tbik_attention_prefill_tc, q, k, v, B, nq, nkv)
    again = run(tb.lib.tbik_attention_prefill_tc, q, k, v, B, nq, nkv)
    assert torch.equal(fast.view(torch.int16), again.view(torch.int16))
    # batch composition: sequence 1 alone
    one = run(tb.lib.tbik_attention_prefill_tc, q[S:2 * S].contiguous(), k[S:2 * S].contiguous(),
              v[S:2 * S].contiguous(), 1, nq, nkv)
    assert torch.equal(fast[S:2 * S].view(torch.int16), one.view(torch.int16))
    # head sharding (TP=2): q heads 4..7 with kv head 1
    shard = run(tb.lib.tbik_attention_prefill_tc, q[:, 4 * D:].contiguous(), k[:, D:].contiguous(),
                v[:, D:].contiguous(), B, nq // 2, nkv // 2)
    assert torch.equal(fast[:, 4 * D:].contiguous().view(torch.int16), shard.view(torch.int16))
    if S <= 512:  # the exact two-pass kernel's range
        exact = run(tb.lib.tbik_attention_prefill, q, k, v, B, nq, nkv)
        assert (fast.float() - exact.float()).abs().max().item() < 3e-2
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.double().view(B, S, nq, D).transpose(1, 2),
        k.double().view(B, S, nkv, D).transpose(1, 2).repeat_interleave(nq // nkv, 1),
        v.double().view(B, S, nkv, D).transpose(1, 2).repeat_interleave(nq // nkv, 1),
        is_causal=True).transpose(1, 2).reshape(B * S, nq * D)
    assert (fast.double() - ref).abs().max().item() < 3e-2
    assert (fast.double() - ref).abs().mean().item() < 2e-3


@pytest.mark.parametrize("rows,cols", [(37, 4096), (5, 5120), (3, 8192), (4, 9000), (2, 100)])
def test_residual_rmsnorm_fused_equals_two_kernels(tb, cuda, rows, cols):
    """tbik_residual_rmsnorm == tbik_residual_add then tbik_tree_rmsnorm, bit for bit
    (fused pass for 16-byte rows with cols % 8 == 0 and cols <= 8192, else the two
    kernels)."""
    import ctypes as C
    g = torch.Generator(device=cuda).manual_seed(cols)
    h0 = torch.randn(rows, cols, device=cuda, generator=g).to(torch.bfloat16)
    f = torch.randn(rows, cols, device=cuda, generator=g)
    gamma = torch.randn(cols, device=cuda, generator=g) * 0.1 + 1
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    h1 = h0.clone()
    y1 = torch.empty(rows, cols, device=cuda, dtype=torch.bfloat16)
    tb.api.check(tb.lib.tbik_residual_rmsnorm(vp(h1), cols, vp(f), cols, vp(gamma), 1e-5, vp(y1), cols, rows, cols, s))
    h2 = h0.clone()
    tb.api.check(tb.lib.tbik_residual_add(vp(h2), cols, vp(f), cols, rows, cols, s))
    y2 = tb.rmsnorm(h2, gamma, 1e-5, out_dtype=torch.bfloat16)
    assert torch.equal(h1.view(torch.int16), h2.view(torch.int16))
    assert torch.equal(y1.view(torch.int16), y2.view(torch.int16))


@pytest.mark.parametrize("M,inter", [(300, 1024), (1024, 1536), (2048, 1000)])
def test_fused_silu_gate_up_256x192_tiles(tb, cuda, M, inter):
    """The SiLU*up epilogue of the 256x192 pair-tile kernel (bf16 box staged in the dead
    tree-level slab, TMA store) == the 256x128 kernel's == tree GEMM + tbik_silu_mul."""
    K = 4096
    g = torch.Generator(device=cuda).manual_seed(M + inter)
    x = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(K, 2 * inter, device=cuda, generator=g) * 0.02).to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    w_il = tb.interleave_gate_up(w)
    with tb.schedule(tc_wide=0):
        ref = tb.tree_matmul_silu_mul(x, w_il, tb.DeviceGroup(1), cfg, tb.LEAF_TCGEN05)
    for tp in (1, 2):
        with tb.schedule(tc_wide=1):
            act = tb.tree_matmul_silu_mul(x, w_il, tb.DeviceGroup(tp), cfg, tb.LEAF_TCGEN05)
            kern = tb.last_kernel()
        torch.cuda.synchronize()
        # a rank's slice of a 1000-pair output is not 16-byte aligned: the 256x128
        # kernel's epilogue (direct stores) takes it
        aligned = (inter // tp) % 8 == 0
        assert kern == ("tc_w192_tree_gemm_kernel" if aligned else "tc_tree_gemm_kernel")
        assert torch.equal(act.view(torch.int16), ref.view(torch.int16)), f"tp={tp}"


@pytest.mark.parametrize("B,S,nq,nkv", [(4, 256, 32, 8), (1, 16, 8, 8), (2, 100, 16, 4), (1, 512, 8, 2), (3, 65, 8, 8)])
def test_attention_tc_single_v_buffer_same_bits(tb, cuda, B, S, nq, nkv):
    """The tensor-core attention with its V block single-buffered (knob attn_sv1,
    four CTAs per SM) == the double-buffered pipeline, bit for bit."""
    import ctypes as C
    from paper_2511_17826_b200._lib import lib
    D = 128
    g = torch.Generator(device=cuda).manual_seed(S * nq)
    q = torch.randn(B * S, nq * D, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(B * S, nkv * D, device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn(B * S, nkv * D, device=cuda, generator=g).to(torch.bfloat16)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    outs = []
    for sv1 in (0, 1):
        o = torch.empty(B * S, nq * D, device=cuda, dtype=torch.bfloat16)
        with tb.schedule(attn_sv1=sv1):
            assert lib.tbik_attention_prefill_tc(vp(q), nq * D, vp(k), nkv * D, vp(v), nkv * D, B, S, nq, nkv, D,
                                                 1.0 / D ** 0.5, vp(o), nq * D, st) == 0
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
