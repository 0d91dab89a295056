"""Full-size TBIK decoder prefill (BASELINE configs[2] / [3]) on one B200.

* builds random-init weights of the named architecture on the device,
* times the TBIK forward (TP=1 schedule) in tokens/s,
* checks logits AND log-probs bit-identical for simulated TP = 1/2/4/8,
* times a non-invariant forward of the same weights (cuBLAS bf16 GEMMs, PyTorch
  SDPA attention, torch.compile-fused norms / RoPE / SiLU*up, eager and as a CUDA
  graph) -- the end-to-end price of determinism.
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


class TorchForward:
    """Non-invariant status quo on the same weights: bf16 cuBLAS GEMMs, PyTorch SDPA
    (flash) attention, RMSNorm / RoPE / SiLU*up / residual fused by torch.compile
    (Inductor) per layer, the whole forward replayable as a CUDA graph.  gate/up are
    kept as a contiguous [gate | up] copy (TbikDecoder interleaves its own copy's
    columns for the fused SiLU*up epilogue), so no strided GEMM operand."""

    def __init__(self, cfg, w, compile_layers=True):
        self.cfg, self.w = cfg, w
        I = cfg.intermediate
        self.wgu = []
        for lw in w.layers:
            if getattr(w, "gate_up_interleaved", False):
                K = lw.wgu.shape[0]
                self.wgu.append(lw.wgu.view(K, I, 2).transpose(1, 2).reshape(K, 2 * I).contiguous())
            else:
                self.wgu.append(lw.wgu)
        cos, sin = mdl.rope_tables(cfg)
        self.cos = torch.from_numpy(cos).cuda()
        self.sin = torch.from_numpy(sin).cuda()
        self.compiled = False
        self.layer = self._layer
        self.head = self._head
        if compile_layers:
            try:
                self.layer = torch.compile(self._layer, dynamic=False)
                self.head = torch.compile(self._head, dynamic=False)
                self.compiled = True
            except Exception:  # noqa: BLE001 -- keep the eager baseline
                self.layer, self.head = self._layer, self._head

    def _rms(self, x, g):
        return torch.nn.functional.rms_norm(x.float(), (x.shape[-1],), g, self.cfg.rms_eps).to(torch.bfloat16)

    def _rope(self, x, heads, B, S):
        D = self.cfg.head_dim
        x = x.reshape(B, S, heads, D).float()
        c = torch.cat([self.cos[:S], self.cos[:S]], -1)[None, :, None, :]
        s = torch.cat([self.sin[:S], self.sin[:S]], -1)[None, :, None, :]
        rot = torch.cat([-x[..., D // 2:], x[..., :D // 2]], -1)
        return (x * c + rot * s).to(torch.bfloat16)

    def _layer(self, h, lw_ln1, wqkv, wo, lw_ln2, wgu, wd, qn, kn, B: int, S: int):
        cfg = self.cfg
        M = B * S
        D, nq, nkv, I = cfg.head_dim, cfg.n_heads, cfg.n_kv_heads, cfg.intermediate
        a = self._rms(h, lw_ln1)
        qkv = a @ wqkv
        q = qkv[:, :nq * D]
        k = qkv[:, nq * D:(nq + nkv) * D]
        v = qkv[:, (nq + nkv) * D:]
        if qn is not None:
            q = self._rms(q.reshape(M * nq, D), qn).view(M, nq * D)
            k = self._rms(k.reshape(M * nkv, D), kn).view(M, nkv * D)
        q = self._rope(q, nq, B, S).transpose(1, 2)
        k = self._rope(k, nkv, B, S).transpose(1, 2)
        v = v.reshape(B, S, nkv, D).transpose(1, 2)
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        h = h + o.transpose(1, 2).reshape(M, nq * D) @ wo
        gu = self._rms(h, lw_ln2) @ wgu
        return h + (torch.nn.functional.silu(gu[:, :I]) * gu[:, I:]) @ wd

    def _head(self, h, ln_f, lm_head):
        return torch.log_softmax((self._rms(h, ln_f) @ lm_head).float(), -1)

    def __call__(self, tokens):
        B, S = tokens.shape
        w = self.w
        h = w.embed[tokens.reshape(B * S)]
        for lw, wgu in zip(w.layers, self.wgu):
            h = self.layer(h, lw.ln1, lw.wqkv, lw.wo, lw.ln2, wgu, lw.wd, lw.q_norm, lw.k_norm, B, S)
        return self.head(h, w.ln_f, w.lm_head)

    def capture(self, tokens):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                self(tokens)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            out = self(tokens)
        return graph, out


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
    tf = TorchForward(cfg, w)
    t0 = time.time()
    lp_ref = tf(tokens)  # compiles (outside every timed region)
    torch.cuda.synchronize()
    compile_s = time.time() - t0
    base_ms = timeit(lambda: tf(tokens), reps)
    try:
        bgraph, _ = tf.capture(tokens)
        base_graph_ms = timeit(bgraph.replay, reps)
        del bgraph
    except Exception:  # noqa: BLE001
        base_graph_ms = None
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
    diff = (ref[1] - lp_ref).abs()
    agree = (ref[1].argmax(-1) == lp_ref.argmax(-1)).float().mean().item()
    out = {
        "model": cfg.name, "layers": cfg.n_layers, "batch": batch, "seq": seq, "tokens": M,
        "data": "synthetic: random-init N(0, 0.02) bf16 weights, uniform random token ids",
        "tbik_ms": ms, "tbik_tokens_per_s": M / (ms * 1e-3),
        "tbik_graph_ms": ms_graph, "tbik_graph_tokens_per_s": M / (ms_graph * 1e-3),
        "graph_bit_identical_to_eager": graph_same,
        "noninvariant_ms": base_ms, "noninvariant_tokens_per_s": M / (base_ms * 1e-3),
        "noninvariant_graph_ms": base_graph_ms,
        "noninvariant_graph_tokens_per_s": M / (base_graph_ms * 1e-3) if base_graph_ms else None,
        "noninvariant_path": ("cuBLAS bf16 GEMMs + PyTorch SDPA (flash) + " +
                              ("torch.compile-fused RMSNorm/RoPE/SiLU*up/residual" if tf.compiled else
                               "eager torch norms") + ", contiguous [gate|up], same weights"),
        "noninvariant_compile_s": compile_s,
        "tbik_over_noninvariant": base_ms / ms,
        "tbik_graph_over_noninvariant_graph": base_graph_ms / ms_graph if base_graph_ms else None,
        "tp_checked": list(tps), "logits_bit_identical": bool(identical_logits),
        "logprobs_bit_identical": bool(identical_lp),
        "logprob_diff_vs_noninvariant": {"max_abs": diff.max().item(), "mean_abs": diff.mean().item(),
                                         "argmax_agreement": agree},
        "weights_gen_s": t_w, "gpu_launches_per_forward": launches,
    }
    del dec, w, tf, lp_ref
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
