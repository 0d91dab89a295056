"""One rank of the real tensor-parallel forward test (tests/test_gpu_sharded_forward.py).

Launched W times with RANK / WORLD_SIZE / MASTER_* set.  Each rank owns only its
shards of the weights (model.ShardedDecoder) and talks to the others through the
PeerGroup (CUDA IPC peer memory + device flags; gloo carries only the 128-byte
handles).  Rank 0 additionally runs the single-process TP = 1 forward on the full
weights and checks, bit for bit:

  llama   Llama-3.1-8B-shaped 2-layer forward, 2 x 160 tokens (ragged M = 320:
          fused GEMM + all-reduce row-parallel path): all-gathered logits, lse,
          all-gathered log-probs and target log-probs == TP = 1
  qwen    Qwen3-32B-shaped 2-layer stack, batch sweep 1 / 3 / 8 x 16 tokens
          (batch- and TP-invariance together)
  c5      tree log-softmax over vocab 151936 at 4096 tokens, vocab-sharded with
          the cross-rank (m, s) merge == tbik_tree_logsoftmax_local(tp = 1)
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from paper_2511_17826_b200 import model as mdl  # noqa: E402


def same(a, b) -> bool:
    return a.shape == b.shape and torch.equal(a.contiguous().view(torch.int32), b.contiguous().view(torch.int32))


def gather_targets(dec, tlp):
    """Each rank holds the target log-probs of the targets inside its vocab range
    (NaN elsewhere); exactly one rank holds each row's value."""
    allv = dec.gather(tlp[:, None].contiguous())  # [rows, W]
    ok = ~torch.isnan(allv)
    assert bool((ok.sum(1) == 1).all()), "each target must fall in exactly one vocab shard"
    return allv[ok]


def check_model(name, cfg, shapes, grp, rank, world, log):
    dec = mdl.ShardedDecoder(cfg, grp, seed=3)
    full = None
    if rank == 0:
        full = mdl.TbikDecoder(cfg, mdl.random_weights(cfg, seed=3))
    for B, S in shapes:
        g = torch.Generator(device="cuda")
        g.manual_seed(100 * B + S)
        tokens = torch.randint(0, cfg.vocab, (B, S), device="cuda", generator=g)
        targets = torch.randint(0, cfg.vocab, (B * S,), device="cuda", generator=g)
        logits_r = dec.forward(tokens)
        lse, lp_r, tlp_r = dec.log_probs(logits_r, targets=targets)
        logits = dec.gather(logits_r)
        lp = dec.gather(lp_r)
        tlp = gather_targets(dec, tlp_r)
        torch.cuda.synchronize()
        if rank == 0:
            ref_logits = full.forward(tokens, tp=1)
            ref_lse, ref_lp, ref_tlp = full.log_probs(ref_logits, tp=1, targets=targets)
            sim8 = full.forward(tokens, tp=world)  # simulated TP = W on one GPU, for good measure
            torch.cuda.synchronize()
            assert same(logits, ref_logits), f"{name} B={B} S={S}: logits differ from TP=1"
            assert same(sim8, ref_logits), f"{name} B={B} S={S}: simulated TP={world} differs"
            assert same(lse, ref_lse), f"{name} B={B} S={S}: lse differs"
            assert same(lp, ref_lp), f"{name} B={B} S={S}: log-probs differ"
            assert same(tlp, ref_tlp), f"{name} B={B} S={S}: target log-probs differ"
            log.append(f"{name} B={B} S={S} bit-identical (logits, lse, log-probs, target log-probs)")
    del dec, full
    torch.cuda.empty_cache()


def check_c5(grp, rank, world, log):
    rows, V, G = 4096, 151936, 8
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    logits = torch.randn(rows, V, device="cuda", generator=g) * 4.0
    vl = V // world
    shard = logits[:, rank * vl:(rank + 1) * vl].contiguous()
    targets = torch.randint(0, V, (rows,), device="cuda", generator=g)
    lse, lp_r, tlp_r = grp.log_softmax(shard, G // world, rank * vl, targets)
    lp = grp.all_gather(lp_r)
    allv = grp.all_gather(tlp_r[:, None].contiguous())
    tlp = allv[~torch.isnan(allv)]
    torch.cuda.synchronize()
    if rank == 0:
        ref_lse, ref_lp, ref_tlp = tb.log_softmax(logits, G, 1, targets)
        torch.cuda.synchronize()
        assert same(lse, ref_lse), "C5 lse differs from TP=1"
        assert same(lp, ref_lp), "C5 log-probs differ from TP=1"
        assert same(tlp, ref_tlp), "C5 target log-probs differ from TP=1"
        log.append(f"c5 rows={rows} V={V} W={world} bit-identical")


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    which = os.environ.get("TBIK_SHARD_CASES", "llama,qwen,c5").split(",")
    grp = tb.PeerGroup(world, rank, torch.cuda.current_device(), 8 << 20, dist)
    log = []
    if "llama" in which:
        check_model("llama3.1-8b x2", mdl.llama31_8b(2), [(2, 160), (1, 16)], grp, rank, world, log)
    if "qwen" in which:
        check_model("qwen3-32b x2", mdl.qwen3_32b(2), [(1, 16), (3, 16), (8, 16)], grp, rank, world, log)
    if "c5" in which:
        check_c5(grp, rank, world, log)
    fused = grp.fused_count()
    dist.barrier()
    grp.close()
    dist.destroy_process_group()
    if rank == 0:
        print("\n".join(log))
        print(f"fused GEMM+all-reduce calls on rank 0: {fused}")
        print("SHARDED OK")


if __name__ == "__main__":
    main()
