"""Full-size TBIK decoder prefill (BASELINE configs[2] / [3]) on one B200.

* builds random-init weights of the named architecture on the device,
* times the TBIK forward (TP=1 schedule) in tokens/s,
* checks logits AND log-probs bit-identical for simulated TP = 1/2/4/8,
* times a non-invariant forward of the same weights (cuBLAS bf16 GEMMs, PyTorch
  SDPA attention, torch RMSNorm/softmax) -- the end-to-end price of determinism.
Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from paper_2511_17826_b200 import model as mdl  # noqa: E402


def torch_forward(cfg, w, tokens):
    """Non-invariant status quo: bf16 cuBLAS GEMMs + SDPA + torch norms."""
    B, S = tokens.shape
    M = B * S
    H, D, nq, nkv, I = cfg.hidden, cfg.head_dim, cfg.n_heads, cfg.n_kv_heads, cfg.intermediate
    cos, sin = mdl.rope_tables(cfg)
    cos = torch.from_numpy(cos[:S]).cuda()
    sin = torch.from_numpy(sin[:S]).cuda()

    def rms(x, g):
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + cfg.rms_eps) * g).to(torch.bfloat16)

    def rope(x, heads):
        x = x.view(B, S, heads, D).float()
        c = torch.cat([cos, cos], -1)[None, :, None, :]
        s = torch.cat([sin, sin], -1)[None, :, None, :]
        rot = torch.cat([-x[..., D // 2:], x[..., :D // 2]], -1)
        return (x * c + rot * s).to(torch.bfloat16)

    h = w.embed[tokens.reshape(M)]
    for lw in w.layers:
        a = rms(h, lw.ln1)
        qkv = a @ lw.wqkv
        q = qkv[:, :nq * D]
        k = qkv[:, nq * D:(nq + nkv) * D]
        v = qkv[:, (nq + nkv) * D:]
        if cfg.qk_norm:
            q = rms(q.reshape(M * nq, D), lw.q_norm).view(M, nq * D)
            k = rms(k.reshape(M * nkv, D), lw.k_norm).view(M, nkv * D)
        q = rope(q, nq).transpose(1, 2)
        k = rope(k, nkv).transpose(1, 2)
        v = v.reshape(B, S, nkv, D).transpose(1, 2)
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        o = o.transpose(1, 2).reshape(M, nq * D)
        h = h + o @ lw.wo
        a = rms(h, lw.ln2)
        gu = a @ lw.wgu
        if getattr(w, "gate_up_interleaved", False):  # TbikDecoder keeps gate/up interleaved
            h = h + (torch.nn.functional.silu(gu[:, 0::2]) * gu[:, 1::2]) @ lw.wd
        else:
            h = h + (torch.nn.functional.silu(gu[:, :I]) * gu[:, I:]) @ lw.wd
    a = rms(h, w.ln_f)
    logits = (a @ w.lm_head).float()
    return torch.log_softmax(logits, -1)


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run(model="llama3.1-8b", layers=0, batch=4, seq=256, reps=3, tps=(1, 2, 4, 8)):
    cfg = mdl.llama31_8b() if model == "llama3.1-8b" else mdl.qwen3_32b()
    if layers:
        cfg.n_layers = layers
    t0 = time.time()
    w = mdl.random_weights(cfg, seed=3)
    torch.cuda.synchronize()
    t_w = time.time() - t0
    dec = mdl.TbikDecoder(cfg, w)
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    tokens = torch.randint(0, cfg.vocab, (batch, seq), device="cuda", generator=g)
    M = batch * seq

    def tbik_step():
        logits = dec.forward(tokens, 1)
        return dec.log_probs(logits, 1, full=True)

    ms = timeit(tbik_step, reps)
    graph, (g_logits, _, _) = dec.capture(tokens, 1, True)
    ms_graph = timeit(graph.replay, reps)
    eager_logits = dec.forward(tokens, 1)
    graph.replay()
    torch.cuda.synchronize()
    graph_same = bool(torch.equal(eager_logits.view(torch.int32), g_logits.view(torch.int32)))
    del graph, g_logits, eager_logits
    l0 = tb.launch_count()
    tbik_step()
    torch.cuda.synchronize()
    launches = tb.launch_count() - l0
    base_ms = timeit(lambda: torch_forward(cfg, w, tokens), reps)
    ref = None
    identical_logits = identical_lp = True
    for tp in tps:
        logits = dec.forward(tokens, tp)
        _, lp, _ = dec.log_probs(logits, tp)
        if ref is None:
            ref = (logits.clone(), lp.clone())
            continue
        identical_logits &= torch.equal(ref[0].view(torch.int32), logits.view(torch.int32))
        identical_lp &= torch.equal(ref[1].view(torch.int32), lp.view(torch.int32))
    lp_ref = torch_forward(cfg, w, tokens)
    diff = (ref[1] - lp_ref).abs()
    agree = (ref[1].argmax(-1) == lp_ref.argmax(-1)).float().mean().item()
    out = {
        "model": cfg.name, "layers": cfg.n_layers, "batch": batch, "seq": seq, "tokens": M,
        "data": "synthetic: random-init N(0, 0.02) bf16 weights, uniform random token ids",
        "tbik_ms": ms, "tbik_tokens_per_s": M / (ms * 1e-3),
        "tbik_graph_ms": ms_graph, "tbik_graph_tokens_per_s": M / (ms_graph * 1e-3),
        "graph_bit_identical_to_eager": graph_same,
        "noninvariant_ms": base_ms, "noninvariant_tokens_per_s": M / (base_ms * 1e-3),
        "noninvariant_path": "cuBLAS bf16 GEMMs + PyTorch SDPA + torch norms/softmax, same weights",
        "tbik_over_noninvariant": base_ms / ms,
        "tp_checked": list(tps), "logits_bit_identical": bool(identical_logits),
        "logprobs_bit_identical": bool(identical_lp),
        "logprob_diff_vs_noninvariant": {"max_abs": diff.max().item(), "mean_abs": diff.mean().item(),
                                         "argmax_agreement": agree},
        "weights_gen_s": t_w, "gpu_launches_per_forward": launches,
    }
    del dec, w
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3.1-8b", choices=["llama3.1-8b", "qwen3-32b"])
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--seq", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tps", default="1,2,4,8")
    args = ap.parse_args()
    print(json.dumps(run(args.model, args.layers, args.batch, args.seq, args.reps,
                         tuple(int(t) for t in args.tps.split(",")))))


if __name__ == "__main__":
    main()
