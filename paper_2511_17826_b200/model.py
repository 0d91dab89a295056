"""TBIK decoder forward: Llama-3.1-8B / Qwen3-32B-shaped prefill (SURVEY §8 F3,
BASELINE configs[2] and configs[3]).

The reference's toy model (demo.cpp:164-241: rmsnorm -> column-parallel gate/up
-> silu * up -> row-parallel down -> residual rounded through bf16 -> column-
parallel lm head -> softmax) is the structural template; this adds what a real
decoder needs -- GQA attention with RoPE (and Qwen3's per-head q/k RMSNorm) --
with every reduction in a fixed, shard-independent order:

  rmsnorm            tbik_tree_rmsnorm            replicated, per token
  qkv / gate_up / lm column_parallel_forward      per column: identical at any TP
  RoPE, attention    tbik_rope, tbik_attention_prefill   per token / (seq, head)
  o_proj, down_proj  row_parallel_forward         TBIK tree GEMM + tree all-reduce
  residual + norm    tbik_residual_rmsnorm        h = bf16(h + f)  (demo.cpp:216), then tree RMSNorm
  log-probs          tbik_tree_logsoftmax_local   vocab-sharded (m, s) tree

so logits and log-probs are bit-identical for TP = 1/2/4/8 and for any batch
composition.  TP ranks are simulated on one GPU (the reference's in-process
DeviceGroup); one process per GPU uses the same kernels through PeerGroup.
Weights are random-init (there is no checkpoint access); the shapes are the
public HF configs.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import api
from ._lib import check, lib


@dataclass
class DecoderConfig:
    name: str
    hidden: int
    intermediate: int
    n_heads: int
    n_kv_heads: int
    vocab: int
    n_layers: int
    head_dim: int = 128
    rms_eps: float = 1e-5
    rope_theta: float = 500000.0
    rope_llama3: Optional[dict] = None
    qk_norm: bool = False
    block_k: int = 256        # numerics-defining leaf width for every GEMM
    block_k_down: int = 256   # down_proj (Qwen3-32B needs 128: K=25600)
    c_max: int = 8
    vocab_groups: int = 8
    max_pos: int = 4096
    weight_std: float = 0.02


def llama31_8b(n_layers: int = 32) -> DecoderConfig:
    return DecoderConfig("llama3.1-8b", 4096, 14336, 32, 8, 128256, n_layers, rope_theta=500000.0,
                         rope_llama3=dict(factor=8.0, low_freq_factor=1.0, high_freq_factor=4.0,
                                          original_max_position_embeddings=8192))


def qwen3_32b(n_layers: int = 64) -> DecoderConfig:
    return DecoderConfig("qwen3-32b", 5120, 25600, 64, 8, 151936, n_layers, rms_eps=1e-6, rope_theta=1000000.0,
                         qk_norm=True, block_k_down=128)


def rope_tables(cfg: DecoderConfig):
    """cos/sin [max_pos, head_dim/2] f32, computed in float64 on the host (HF
    rotary embedding, with Llama-3 frequency scaling when configured)."""
    d = cfg.head_dim
    inv = 1.0 / (cfg.rope_theta ** (np.arange(0, d, 2, dtype=np.float64) / d))
    if cfg.rope_llama3:
        s = cfg.rope_llama3
        factor, lo, hi = s["factor"], s["low_freq_factor"], s["high_freq_factor"]
        orig = s["original_max_position_embeddings"]
        lo_wl, hi_wl = orig / lo, orig / hi
        wl = 2 * math.pi / inv
        scaled = np.where(wl > lo_wl, inv / factor, inv)
        smooth = (orig / wl - lo) / (hi - lo)
        smoothed = (1 - smooth) * scaled / factor + smooth * scaled
        medium = ~(wl < hi_wl) & ~(wl > lo_wl)
        inv = np.where(medium, smoothed, scaled)
    ang = np.arange(cfg.max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


@dataclass
class LayerWeights:
    ln1: object
    wqkv: object
    wo: object
    ln2: object
    wgu: object
    wd: object
    q_norm: object = None
    k_norm: object = None


@dataclass
class DecoderWeights:
    embed: object
    layers: List[LayerWeights] = field(default_factory=list)
    ln_f: object = None
    lm_head: object = None
    gate_up_interleaved: bool = False  # set by TbikDecoder (gate/up columns interleaved in place)


def _shard_cols(t, parts):
    """Concatenate column ranges [(b, e), ...] of a 2-D tensor (contiguous copy)."""
    import torch
    return torch.cat([t[:, b:e] for b, e in parts], dim=1).contiguous()


def random_weights(cfg: DecoderConfig, seed: int = 0, device="cuda", shard: Optional[tuple] = None) -> DecoderWeights:
    """Random-init weights of the named architecture, generated on the device
    from fixed per-tensor seeds (independent of TP and batch, like
    make_demo_weights, demo.cpp:123-162).

    shard = (W, r): keep only tensor-parallel rank r's part of every projection
    (each full tensor is generated from its own seed, sliced, and freed):
      wqkv    columns of rank r's q heads | k heads | v heads   (column-parallel)
      wo      rows [r, r+1) * nq*D/W  = make_row_shard_plan(nq*D)[r]  (row-parallel)
      wgu     gate_up pairs [r, r+1) * I/W, interleaved (column-parallel, SiLU*up fused)
      wd      rows [r, r+1) * I/W     = make_row_shard_plan(I)[r]     (row-parallel)
      lm_head columns [r, r+1) * V/W  = make_column_shard_plan(V)[r]
    embed and the norm gains are replicated.  The values are exactly the
    corresponding slices of shard=None's tensors."""
    import torch
    g = torch.Generator(device=device)
    counter = [seed * 1000003]

    def normal(shape, std, mean=0.0, dtype=torch.bfloat16):
        counter[0] += 1
        g.manual_seed(counter[0])
        t = torch.empty(shape, device=device, dtype=torch.float32)
        t.normal_(mean, std, generator=g)
        return t.to(dtype)

    H, I, D = cfg.hidden, cfg.intermediate, cfg.head_dim
    nq, nkv = cfg.n_heads, cfg.n_kv_heads
    W, r = shard if shard is not None else (1, 0)
    if nq % W or nkv % W or I % W or cfg.vocab % W:
        raise api.TbikError(api.ErrorCode.ShardError, f"{cfg.name}: heads / intermediate / vocab not divisible by {W}")
    qh, kh = nq // W, nkv // W
    qkv_parts = [(r * qh * D, (r + 1) * qh * D), (nq * D + r * kh * D, nq * D + (r + 1) * kh * D),
                 ((nq + nkv) * D + r * kh * D, (nq + nkv) * D + (r + 1) * kh * D)]

    def cut(t, kind):
        if W == 1:
            return t
        if kind == "qkv":
            return _shard_cols(t, qkv_parts)
        if kind == "rows":
            n = t.shape[0] // W
            return t[r * n:(r + 1) * n].contiguous()
        if kind == "cols":
            n = t.shape[1] // W
            return t[:, r * n:(r + 1) * n].contiguous()
        if kind == "gate_up":  # interleave the full tensor, then take rank r's pairs
            il = api.interleave_gate_up(t)
            n = il.shape[1] // W
            return il[:, r * n:(r + 1) * n].contiguous()
        raise ValueError(kind)

    w = DecoderWeights(embed=normal((cfg.vocab, H), 1.0))
    for _ in range(cfg.n_layers):
        lw = LayerWeights(
            ln1=normal((H,), 0.02, 1.0, torch.float32),
            wqkv=cut(normal((H, (nq + 2 * nkv) * D), cfg.weight_std), "qkv"),
            wo=cut(normal((nq * D, H), cfg.weight_std), "rows"),
            ln2=normal((H,), 0.02, 1.0, torch.float32),
            wgu=cut(normal((H, 2 * I), cfg.weight_std), "gate_up"),
            wd=cut(normal((I, H), cfg.weight_std), "rows"))
        if cfg.qk_norm:
            lw.q_norm = normal((D,), 0.02, 1.0, torch.float32)
            lw.k_norm = normal((D,), 0.02, 1.0, torch.float32)
        w.layers.append(lw)
    w.ln_f = normal((H,), 0.02, 1.0, torch.float32)
    w.lm_head = cut(normal((H, cfg.vocab), cfg.weight_std), "cols")
    w.gate_up_interleaved = W > 1
    return w


def _vp(t):
    return C.c_void_p(t.data_ptr())


class TbikDecoder:
    """Prefill forward of a TBIK decoder with `tp` simulated ranks."""

    def __init__(self, cfg: DecoderConfig, weights: DecoderWeights, leaf: int = api.LEAF_TCGEN05):
        import torch
        self.cfg, self.w, self.leaf = cfg, weights, leaf
        cos, sin = rope_tables(cfg)
        dev = weights.embed.device
        self.cos = torch.from_numpy(cos).to(dev)
        self.sin = torch.from_numpy(sin).to(dev)
        self.bcfg = api.BlockConfig(64, cfg.block_k, 128, 0)
        # gate_up weights are kept with gate/up columns interleaved so SiLU*up runs
        # in the GEMM epilogue (a column permutation: the per-column tree is unchanged)
        if not getattr(weights, "gate_up_interleaved", False):
            for lw in weights.layers:
                lw.wgu = api.interleave_gate_up(lw.wgu)
            weights.gate_up_interleaved = True
        self.bcfg_down = api.BlockConfig(64, cfg.block_k_down, 128, 0)

    # -- building blocks ------------------------------------------------------------
    # (simulated TP: the full weights, `tp` ranks on this GPU; ShardedDecoder
    # overrides these with one rank's shards and the PeerGroup collectives)
    def _heads(self):
        return self.cfg.n_heads, self.cfg.n_kv_heads

    def _col(self, x, w, tp):
        return api.column_parallel_forward(x, w, api.DeviceGroup(tp), self.bcfg, self.leaf)

    def _row(self, x, w, tp, cfg, k_global):
        return api.row_parallel_forward(x, w, api.DeviceGroup(tp), cfg, self.cfg.c_max, self.leaf)

    def _gate_up(self, x, w, tp):
        return api.tree_matmul_silu_mul(x, w, api.DeviceGroup(tp), self.bcfg, self.leaf)

    def _norm(self, x, gamma):
        import torch
        return api.rmsnorm(x, gamma, self.cfg.rms_eps, out_dtype=torch.bfloat16)

    def _residual_norm(self, h, f, gamma):
        """h = bf16(h + f) in place, returns tree_rmsnorm(h) (bf16) -- one fused pass."""
        import torch
        M, H = h.shape
        y = torch.empty(M, H, device=h.device, dtype=torch.bfloat16)
        check(lib.tbik_residual_rmsnorm(_vp(h), h.stride(0), _vp(f), f.stride(0), _vp(gamma), self.cfg.rms_eps,
                                        _vp(y), H, M, H, self._stream()))
        return y

    def _stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def _rope(self, src, ld, col0, heads, pos, rows):
        import torch
        D = self.cfg.head_dim
        out = torch.empty(rows, heads * D, device=src.device, dtype=torch.bfloat16)
        check(lib.tbik_rope(_vp(src), ld, col0, heads, D, _vp(pos), _vp(self.cos), _vp(self.sin), _vp(out),
                            heads * D, rows, self._stream()))
        return out

    def _qk_normed(self, qkv, col0, heads, gamma, rows):
        """Qwen3 q/k norm: per-head tree RMSNorm over head_dim (f32 out)."""
        D = self.cfg.head_dim
        blk = qkv[:, col0:col0 + heads * D].contiguous().view(rows * heads, D)
        return api.rmsnorm(blk, gamma, self.cfg.rms_eps).view(rows, heads * D)

    # -- forward ------------------------------------------------------------------------
    def forward(self, tokens, tp: int = 1):
        """tokens: int64 [B, S] on the device.  Returns f32 logits [B*S, vocab]
        (ShardedDecoder: this rank's vocab columns)."""
        import torch
        cfg, w = self.cfg, self.w
        B, S = tokens.shape
        M = B * S
        dev = tokens.device
        H, D, I = cfg.hidden, cfg.head_dim, cfg.intermediate
        nq, nkv = self._heads()  # this rank's heads (all of them with simulated TP)
        if S > cfg.max_pos:
            raise api.TbikError(api.ErrorCode.BadDimension, "sequence longer than the RoPE table")
        ids = tokens.reshape(M).contiguous()
        pos = torch.arange(S, device=dev, dtype=torch.int32).repeat(B).contiguous()
        h = torch.empty(M, H, device=dev, dtype=torch.bfloat16)
        check(lib.tbik_embedding(_vp(w.embed), cfg.vocab, H, _vp(ids), M, _vp(h), self._stream()))
        qcols = nq * D
        kcols = nkv * D
        scale = 1.0 / math.sqrt(D)
        a = self._norm(h, w.layers[0].ln1) if w.layers else None
        for li, lw in enumerate(w.layers):
            qkv = self._col(a, lw.wqkv, tp)                      # f32 [M, (nq + 2 nkv) D]
            ld = qkv.stride(0)
            if cfg.qk_norm:
                qn = self._qk_normed(qkv, 0, nq, lw.q_norm, M)
                kn = self._qk_normed(qkv, qcols, nkv, lw.k_norm, M)
                q = self._rope(qn, qcols, 0, nq, pos, M)
                k = self._rope(kn, kcols, 0, nkv, pos, M)
                v = torch.empty(M, kcols, device=dev, dtype=torch.bfloat16)
                check(lib.tbik_cast_bf16(C.c_void_p(qkv.data_ptr() + 4 * (qcols + kcols)), ld, M, kcols, _vp(v),
                                         kcols, self._stream()))
            else:
                # RoPE of q and k and the bf16 cast of v in one launch (same bits as
                # tbik_rope x 2 + tbik_cast_bf16)
                q = torch.empty(M, qcols, device=dev, dtype=torch.bfloat16)
                k = torch.empty(M, kcols, device=dev, dtype=torch.bfloat16)
                v = torch.empty(M, kcols, device=dev, dtype=torch.bfloat16)
                check(lib.tbik_rope_qkv(_vp(qkv), ld, nq, nkv, D, _vp(pos), _vp(self.cos), _vp(self.sin), _vp(q),
                                        _vp(k), _vp(v), M, self._stream()))
            attn = torch.empty(M, qcols, device=dev, dtype=torch.bfloat16)
            # tensor-core flash attention with the tcgen05 leaf, the exact order with the fma leaf
            attn_fn = lib.tbik_attention_prefill_tc if self.leaf == api.LEAF_TCGEN05 else lib.tbik_attention_prefill
            check(attn_fn(_vp(q), qcols, _vp(k), kcols, _vp(v), kcols, B, S, nq, nkv, D,
                          scale, _vp(attn), qcols, self._stream()))
            o = self._row(attn, lw.wo, tp, self.bcfg, cfg.n_heads * D)  # f32 [M, H], tree all-reduce
            a = self._residual_norm(h, o, lw.ln2)               # h = bf16(h + o); a = norm(h)
            act = self._gate_up(a, lw.wgu, tp)                  # bf16 [M, I / ranks]
            d = self._row(act, lw.wd, tp, self.bcfg_down, I)     # f32 [M, H]
            nxt = w.layers[li + 1].ln1 if li + 1 < len(w.layers) else w.ln_f
            a = self._residual_norm(h, d, nxt)                  # next layer's ln1 (or ln_f)
        if not w.layers:
            a = self._norm(h, w.ln_f)
        return self._head(a, tp)                                # f32 logits [M, vocab]

    # The lm_head's epilogue also emits the log-softmax's 16-column (m, s) chunk
    # states (F2); log_probs() of the same logits consumes them instead of
    # re-reading the logits.  Matched by identity + version of the logits tensor.
    def _head(self, a, tp):
        logits, chunks = api.column_parallel_logits(a, self.w.lm_head, api.DeviceGroup(tp), self.cfg.vocab_groups,
                                                    self.bcfg, self.leaf)
        self._chunk_cache = (logits, logits._version, chunks)
        return logits

    def _cached_chunks(self, logits):
        c = getattr(self, "_chunk_cache", None)
        if c is not None and c[0] is logits and c[1] == logits._version:
            return c[2]
        return None

    def log_probs(self, logits, tp: int = 1, targets=None, full: bool = True):
        """Vocab-sharded tree log-softmax over `tp` simulated vocab shards."""
        return api.log_softmax(logits, self.cfg.vocab_groups, tp, targets, full, chunks=self._cached_chunks(logits))

    # -- CUDA graphs -------------------------------------------------------------------
    def capture(self, tokens, tp: int = 1, full_logprobs: bool = True):
        """Capture one forward + log-softmax over the static token tensor `tokens`
        into a CUDA graph (no per-launch host cost on replay; bits unchanged).
        Returns (graph, (logits, lse, logprobs)); refill `tokens` in place and call
        graph.replay().  Two eager warm-up passes on the capture stream size that
        stream's library workspaces first, so nothing is allocated inside the
        capture; a later call on the same stream that grows a workspace (a larger
        shape) invalidates the graph."""
        import torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                logits = self.forward(tokens, tp)
                self.log_probs(logits, tp, full=full_logprobs)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        # capture on the warm-up stream: the library's scratch arenas are per stream
        with torch.cuda.graph(graph, stream=side):
            logits = self.forward(tokens, tp)
            lse, lp, _ = self.log_probs(logits, tp, full=full_logprobs)
        return graph, (logits, lse, lp)


class ShardedDecoder(TbikDecoder):
    """Rank r of a W-way tensor-parallel TBIK decoder, one process per GPU
    (the reference threads one DeviceGroup through ffn_block /
    greedy_generate, demo.cpp:164-241).  The rank owns only its shards
    (random_weights(shard=(W, r))):

      qkv, gate_up, lm_head  column-parallel: this rank's heads / pairs / vocab
                             columns, tree GEMM with the c_max = 1 plan (layers.cpp:48-72)
      o_proj, down_proj      PeerGroup.row_parallel_forward: the rank's leaf groups
                             (make_row_shard_plan) + the fixed-order tree all-reduce
                             over NVLink peer memory (one fused kernel when M > 128)
      attention              the rank's q heads with their kv heads (GQA), per
                             (sequence, head) -- independent of the head split
      norms, residual        replicated on every rank
      log-softmax            vocab-sharded (m, s) states, 8 bytes per row exchanged
                             (PeerGroup.log_softmax)

    so logits / log-probs equal the single-GPU TP = 1 forward bit for bit.
    Eager only: the group collectives carry host-side epoch counters that a
    CUDA graph would freeze."""

    def __init__(self, cfg: DecoderConfig, group, seed: int = 0, leaf: int = api.LEAF_TCGEN05, device="cuda",
                 weights: Optional[DecoderWeights] = None):
        self.group = group
        W, r = group.world, group.rank
        if weights is None:
            weights = random_weights(cfg, seed, device, shard=(W, r))
        super().__init__(cfg, weights, leaf)
        self.W, self.r = W, r
        self.v_local = cfg.vocab // W
        if cfg.vocab_groups % W:
            raise api.TbikError(api.ErrorCode.ShardError, f"vocab_groups {cfg.vocab_groups} not divisible by {W}")
        # the rank's K ranges must be the row shard plan's (leaf-group aligned)
        for k in (cfg.n_heads * cfg.head_dim, cfg.intermediate):
            bcfg = self.bcfg_down if k == cfg.intermediate else self.bcfg
            b, e = api.make_row_shard_plan(k, bcfg, W, cfg.c_max).bounds[r]
            if (b, e) != (r * k // W, (r + 1) * k // W):
                raise api.TbikError(api.ErrorCode.ShardError, f"row shard of K={k} is not the even split")

    def _heads(self):
        return self.cfg.n_heads // self.W, self.cfg.n_kv_heads // self.W

    def _col(self, x, w, tp):
        return api.tree_matmul(x, w, self.bcfg, self.leaf)

    def _row(self, x, w, tp, cfg, k_global):
        return self.group.row_parallel_forward(x, w, k_global, cfg, self.cfg.c_max, self.leaf)

    def _gate_up(self, x, w, tp):
        return api.tree_matmul_silu_mul(x, w, None, self.bcfg, self.leaf)

    def _head(self, a, tp):
        logits, chunks = api.tree_matmul_logits(a, self.w.lm_head, self.cfg.vocab_groups // self.W, self.bcfg,
                                                self.leaf)
        self._chunk_cache = (logits, logits._version, chunks)
        return logits

    def log_probs(self, logits, tp: int = 1, targets=None, full: bool = True):
        """(lse, this rank's log-prob columns, target log-probs of targets in this
        rank's vocab range -- NaN elsewhere)."""
        return self.group.log_softmax(logits, self.cfg.vocab_groups // self.W, self.r * self.v_local, targets, full,
                                      chunks=self._cached_chunks(logits))

    def gather(self, shard):
        """Rank-ordered column concatenation of a per-rank [rows x V/W] block."""
        return self.group.all_gather(shard)

    def capture(self, tokens, tp: int = 1, full_logprobs: bool = True):
        raise api.TbikError(api.ErrorCode.BadArgument, "ShardedDecoder runs eagerly (group epochs are host state)")
