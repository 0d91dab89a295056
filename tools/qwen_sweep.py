"""BASELINE configs[3]: Qwen3-32B-shaped decoder stack, batch-size sweep at TP=8
(batch- and TP-invariance together) on one B200.

For every batch size B in the sweep the same first sequence is run inside a
batch of B sequences, at simulated TP=1 and TP=8; its logits and log-probs must
be bit-identical to the batch-1 / TP-1 result.  Tokens/s is the TP=1 prefill
throughput of the whole stack on this GPU (random-init N(0, 0.02) weights of
the named shapes, synthetic token ids).  Prints one JSON object.
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_17826_b200 import model as mdl  # noqa: E402


def run(layers=64, seq=16, batches=(1, 2, 4, 8, 16, 32, 64, 128, 256), reps=2):
    cfg = mdl.qwen3_32b(n_layers=layers)
    t0 = time.time()
    w = mdl.random_weights(cfg, seed=5)
    torch.cuda.synchronize()
    t_w = time.time() - t0
    dec = mdl.TbikDecoder(cfg, w)
    g = torch.Generator(device="cuda")
    g.manual_seed(17)
    tokens = torch.randint(0, cfg.vocab, (max(batches), seq), device="cuda", generator=g)
    ref = dec.forward(tokens[:1].contiguous(), 1)
    _, ref_lp, _ = dec.log_probs(ref, 1)
    ref_lp = ref_lp.clone()
    sweep = []
    for b in batches:
        tk = tokens[:b].contiguous()
        row = {"batch": b, "tokens": b * seq}
        for tp in (1, 8):
            out = dec.forward(tk, tp)
            _, lp, _ = dec.log_probs(out, tp)
            row[f"tp{tp}_logits_identical"] = bool(torch.equal(out[:seq].view(torch.int32), ref.view(torch.int32)))
            row[f"tp{tp}_logprobs_identical"] = bool(torch.equal(lp[:seq].view(torch.int32),
                                                                 ref_lp.view(torch.int32)))
            del out, lp
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            dec.log_probs(dec.forward(tk, 1), 1, full=False)
        e.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(e) / reps
        row["tp1_ms"] = ms
        row["tp1_tokens_per_s"] = b * seq / (ms * 1e-3)
        sweep.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    ok = all(r["tp1_logits_identical"] and r["tp8_logits_identical"] and r["tp1_logprobs_identical"]
             and r["tp8_logprobs_identical"] for r in sweep)
    return {"model": cfg.name, "layers": cfg.n_layers, "seq": seq, "weights_gen_s": t_w,
            "data": "synthetic: random-init N(0, 0.02) bf16 weights (Qwen3-32B shapes), uniform random token ids",
            "all_bit_identical": ok, "sweep": sweep}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=64)
    ap.add_argument("--seq", type=int, default=16)
    args = ap.parse_args()
    print(json.dumps(run(args.layers, args.seq)))
