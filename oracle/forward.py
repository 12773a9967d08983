"""CPU fp32 restatement of the preemptible prefill forward pass.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module, and only
as the checker or the timed CPU baseline -- never as part of the product path.

What it restates
----------------
The reference (FlowPrefill's ``prefillsim``) never computes tensors: its forward pass is the
operator timeline of ``build_timeline`` (prefillsim/cost_model.py:191-244) executed in virtual
time by the execution pool (prefillsim/engine.py:193-320). This module executes the same
timeline numerically, entry by entry, with the same semantics:

* the batch is the requests' tokens concatenated in order (cost_model.py:212-213);
* the stream is cut into ``chunk_size`` chunks, or one chunk when unchunked
  (cost_model.py:214-219);
* entries run chunk -> layer -> operator in ``DENSE_LAYER_OPS`` order
  ``qkv_proj, attn, o_proj, gate_up_proj, down_proj`` (cost_model.py:38-44, 224-242), or
  ``MOE_LAYER_OPS`` ``qkv_proj, attn, o_proj, gate, experts`` for MoE models
  (cost_model.py:46-52; pinned to HF ``Qwen3MoeForCausalLM``);
* linear operators act on all ``new_total`` tokens of the chunk (cost_model.py:225,236);
* attention is per request: each request's share of the chunk attends causally to its own
  prefix + share and never across the batch (cost_model.py:226-233;
  pkg/tests/test_cost_model.py:88-109);
* a cursor over entries supports stop/resume at any boundary; completed entries never rerun
  (engine.py:221-238, 279-291).

The layer math is standard Llama (RMSNorm, rotate-half RoPE, GQA softmax attention, SwiGLU),
i.e. the paper's Eq. (1)-(2). The reference does not specify it, so the
numeric oracle is **not pinned by the reference**; it is pinned instead against Hugging Face
``transformers.LlamaForCausalLM`` (an independent implementation) by the committed golden
vectors in tests/golden/ (see tests/golden/make_golden.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

OPS = ("qkv_proj", "attn", "o_proj", "gate_up_proj", "down_proj")
MOE_OPS = ("qkv_proj", "attn", "o_proj", "gate", "experts")  # cost_model.py:46-52


@dataclass(frozen=True)
class Shape:
    num_layers: int
    hidden: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float
    rms_eps: float = 1e-5
    qkv_bias: bool = False  # Qwen2.5: biases on q/k/v projections
    qk_norm: bool = False   # Qwen3: per-head RMSNorm of q and k before RoPE
    # MoE (Qwen3-MoE block; every layer sparse): the FFN becomes a router ("gate" entry:
    # softmax over experts, top-k, optional renormalisation) and the top-k SwiGLU experts
    # ("experts" entry: weighted sum added to the residual)
    n_experts: int = 0
    top_k: int = 0
    moe_ffn: int = 0
    norm_topk: bool = False
    router_std: float = 0.02

    @property
    def moe(self) -> bool:
        return self.n_experts > 0

    @property
    def ops(self) -> tuple:
        return MOE_OPS if self.moe else OPS

    @property
    def qdim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kvdim(self) -> int:
        return self.n_kv_heads * self.head_dim


SHAPES = {
    # BASELINE.json configs[0] / SURVEY 8(d) config 1
    "tiny": Shape(4, 512, 4, 2, 128, 1536, 8192, 1e4),
    # configs[1]: Llama-3-8B shape (public model card values)
    "llama3-8b": Shape(32, 4096, 32, 8, 128, 14336, 128256, 5e5),
    # small Qwen-style variants for parity tests (vocab not a multiple of 256 on purpose)
    "tiny-qwen3": Shape(2, 512, 4, 2, 128, 1536, 8000, 1e6, 1e-6, qk_norm=True),
    "tiny-qwen2": Shape(2, 512, 4, 2, 128, 1536, 8000, 1e6, 1e-6, qkv_bias=True),
    # tensor-parallel parity (config 4 family: Qwen2.5 QKV bias, GQA group 5 like Qwen2.5-32B;
    # TP=4 leaves 5 q heads / 1 kv head per rank and a padded 896-wide qkv shard)
    "tiny-qwen2-tp": Shape(4, 512, 20, 4, 128, 2048, 8000, 1e6, 1e-6, qkv_bias=True),
    # MoE parity (Qwen3-MoE block: q/k-norm, 16 experts, top-4, renormalised; the router scale
    # keeps the top-k margins far above bf16 rounding so routing is comparable exactly)
    "tiny-moe": Shape(2, 512, 4, 2, 128, 0, 8000, 1e6, 1e-6, qk_norm=True, n_experts=16,
                      top_k=4, moe_ffn=256, norm_topk=True, router_std=0.25),
}


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 value (ties to even), returned as fp32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 values that are exactly bf16 -> uint16 bit patterns (for the C ABI loader)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)


def make_weights(shape: Shape, seed: int, std: float = 0.02) -> dict:
    """Seeded random-init weights, bf16-exact fp32, canonical (HF Llama) layout."""
    rng = np.random.default_rng(seed)
    d, f = shape.hidden, shape.ffn

    def normal(*s):
        return bf16_round(rng.standard_normal(s, dtype=np.float32) * std)

    def gamma(n):
        return bf16_round(1.0 + 0.1 * rng.standard_normal(n, dtype=np.float32))

    w = {"embed": normal(shape.vocab, d)}
    for l in range(shape.num_layers):
        w[f"{l}.wq"] = normal(shape.qdim, d)
        w[f"{l}.wk"] = normal(shape.kvdim, d)
        w[f"{l}.wv"] = normal(shape.kvdim, d)
        w[f"{l}.wo"] = normal(d, shape.qdim)
        if shape.moe:
            E, I = shape.n_experts, shape.moe_ffn
            w[f"{l}.w_router"] = bf16_round(
                rng.standard_normal((E, d), dtype=np.float32) * shape.router_std)
            w[f"{l}.e_gate"] = normal(E, I, d)
            w[f"{l}.e_up"] = normal(E, I, d)
            w[f"{l}.e_down"] = normal(E, d, I)
        else:
            w[f"{l}.w_gate"] = normal(f, d)
            w[f"{l}.w_up"] = normal(f, d)
            w[f"{l}.w_down"] = normal(d, f)
        w[f"{l}.attn_norm"] = gamma(d)
        w[f"{l}.ffn_norm"] = gamma(d)
        if shape.qkv_bias:
            w[f"{l}.bq"] = normal(shape.qdim) * 10.0
            w[f"{l}.bk"] = normal(shape.kvdim) * 10.0
            w[f"{l}.bv"] = normal(shape.kvdim) * 10.0
        if shape.qk_norm:
            w[f"{l}.q_norm"] = gamma(shape.head_dim)
            w[f"{l}.k_norm"] = gamma(shape.head_dim)
    w["final_norm"] = gamma(d)
    w["lm_head"] = normal(shape.vocab, d)
    return w


def make_tokens(lens: Sequence[int], vocab: int, seed: int) -> list[np.ndarray]:
    """Token ids per request: default_rng(seed + i).integers(0, vocab, n)."""
    return [
        np.random.default_rng(seed + i).integers(0, vocab, n).astype(np.int32)
        for i, n in enumerate(lens)
    ]


# ----------------------------------------------------------------------------- layer math


def rmsnorm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    ms = np.mean(x.astype(np.float32) ** 2, axis=-1, keepdims=True)
    return (x / np.sqrt(ms + eps)).astype(np.float32) * g


def rope_tables(positions: np.ndarray, head_dim: int, theta: float):
    """cos/sin [n, head_dim/2] for rotate-half RoPE, computed in fp64."""
    j = np.arange(head_dim // 2, dtype=np.float64)
    inv = 1.0 / (theta ** (2.0 * j / head_dim))
    ang = positions.astype(np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def apply_rope(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """x [n, heads, hd]; pairs (j, j + hd/2) rotated (HF rotate_half convention)."""
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    c, s = cos[:, None, :], sin[:, None, :]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1).astype(np.float32)


def silu(x: np.ndarray) -> np.ndarray:
    return (x / (1.0 + np.exp(-x))).astype(np.float32)


def causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, q_pos0: int) -> np.ndarray:
    """q [s, Hq, hd], k/v [kv_len, Hkv, hd]; query i sits at position q_pos0 + i."""
    s, hq, hd = q.shape
    hkv = k.shape[1]
    rep = hq // hkv
    kr = np.repeat(k, rep, axis=1)  # [kv, Hq, hd]
    vr = np.repeat(v, rep, axis=1)
    scores = np.einsum("qhd,khd->hqk", q, kr, optimize=True) / math.sqrt(hd)
    qpos = q_pos0 + np.arange(s)[:, None]
    kpos = np.arange(k.shape[0])[None, :]
    scores = np.where(kpos <= qpos, scores, -np.inf)
    scores = scores - scores.max(axis=-1, keepdims=True)
    p = np.exp(scores)
    p /= p.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,khd->qhd", p, vr, optimize=True).astype(np.float32)


def moe_route(xn: np.ndarray, w_router: np.ndarray, top_k: int, norm_topk: bool):
    """Qwen3-MoE router: softmax over all experts (fp32), the top-k probabilities (ties to the
    lower expert index), renormalised to sum 1 when ``norm_topk``. Returns ids [n, k] in
    descending-probability order and their weights [n, k]."""
    logits = (xn @ w_router.T).astype(np.float32)
    z = logits - logits.max(axis=-1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(axis=-1, keepdims=True)
    order = np.lexsort((np.broadcast_to(np.arange(p.shape[1]), p.shape), -p), axis=-1)
    ids = order[:, :top_k]
    wts = np.take_along_axis(p, ids, axis=-1)
    if norm_topk:
        wts = wts / wts.sum(axis=-1, keepdims=True)
    return ids.astype(np.int64), wts.astype(np.float32)


def moe_experts(xn: np.ndarray, ids: np.ndarray, wts: np.ndarray, e_gate, e_up, e_down):
    """sum_j w_j * down_e(silu(gate_e(x)) * up_e(x)) over the token's top-k experts."""
    out = np.zeros_like(xn, dtype=np.float32)
    for e in np.unique(ids):
        tok, slot = np.nonzero(ids == e)
        x = xn[tok]
        y = (silu(x @ e_gate[e].T) * (x @ e_up[e].T)) @ e_down[e].T
        out[tok] += wts[tok, slot][:, None] * y
    return out


# ----------------------------------------------------------------------------- plan


@dataclass(frozen=True)
class Segment:
    req: int
    row0: int  # first row in the chunk
    share: int
    prefix: int


@dataclass(frozen=True)
class Chunk:
    start: int
    end: int
    segments: tuple[Segment, ...]
    last: tuple[tuple[int, int], ...]  # (request, row) of requests completing in this chunk

    @property
    def new_total(self) -> int:
        return self.end - self.start


def plan(per_request_tokens: Sequence[int], chunk_size: Optional[int]) -> list[Chunk]:
    """Chunk/segment decomposition of cost_model.py:212-233, with token-level rows."""
    if not per_request_tokens:
        raise ValueError("per_request_tokens must be non-empty")
    if any(t < 1 for t in per_request_tokens):
        raise ValueError("all token counts must be >= 1")
    if chunk_size is not None and chunk_size < 1:
        raise ValueError("chunk_size must be >= 1 when given")
    total = int(sum(per_request_tokens))
    starts = np.concatenate(([0], np.cumsum(per_request_tokens)))
    if chunk_size is None or chunk_size >= total:
        bounds = [(0, total)]
    else:
        bounds = [(lo, min(lo + chunk_size, total)) for lo in range(0, total, chunk_size)]
    chunks = []
    for s, e in bounds:
        segs, last = [], []
        for ri, n_r in enumerate(per_request_tokens):
            r0, r1 = int(starts[ri]), int(starts[ri + 1])
            share = min(e, r1) - max(s, r0)
            if share <= 0:
                continue
            prefix = min(max(s - r0, 0), n_r)
            segs.append(Segment(ri, max(s, r0) - s, share, prefix))
            if s <= r1 - 1 < e:
                last.append((ri, r1 - 1 - s))
        chunks.append(Chunk(s, e, tuple(segs), tuple(last)))
    return chunks


def quad_mass(chunk: Chunk) -> int:
    """The attention quadratic mass the reference charges this chunk (cost_model.py:226-233)."""
    return sum(g.share * (g.prefix + g.share) for g in chunk.segments)


# ----------------------------------------------------------------------------- executor


@dataclass
class OracleTask:
    """A batched prefill as a cursor over (chunk, layer, op) entries, like ExecutionTask."""

    shape: Shape
    weights: dict
    tokens: list  # per request int32 arrays
    chunk_size: Optional[int] = None
    cursor: int = 0
    chunks: list = field(default_factory=list)
    h: Optional[np.ndarray] = None
    q: Optional[np.ndarray] = None
    ao: Optional[np.ndarray] = None
    act: Optional[np.ndarray] = None
    k_cache: list = field(default_factory=list)  # [req][layer] -> [n_r, Hkv, hd]
    v_cache: list = field(default_factory=list)
    logits: Optional[np.ndarray] = None

    def __post_init__(self):
        lens = [len(t) for t in self.tokens]
        self.chunks = plan(lens, self.chunk_size)
        self.stream = np.concatenate(self.tokens).astype(np.int64)
        sh = self.shape
        self.k_cache = [
            [np.zeros((n, sh.n_kv_heads, sh.head_dim), np.float32) for _ in range(sh.num_layers)]
            for n in lens
        ]
        self.v_cache = [
            [np.zeros((n, sh.n_kv_heads, sh.head_dim), np.float32) for _ in range(sh.num_layers)]
            for n in lens
        ]
        self.logits = np.zeros((len(lens), sh.vocab), np.float32)

    def __len__(self) -> int:
        return len(self.chunks) * self.shape.num_layers * len(OPS)

    def entry(self, i: int) -> tuple[int, int, int]:
        per_chunk = self.shape.num_layers * len(OPS)
        return i // per_chunk, (i % per_chunk) // len(OPS), i % len(OPS)

    # MoE routing of the current chunk (the live state between the gate and experts entries)
    moe_ids: Optional[np.ndarray] = None
    moe_w: Optional[np.ndarray] = None
    xn: Optional[np.ndarray] = None

    def run(self, first: int, last: int) -> None:
        """Execute entries [first, last); first must equal the cursor (work conservation)."""
        if first != self.cursor:
            raise ValueError(f"entries must run in order: cursor {self.cursor}, asked {first}")
        for i in range(first, last):
            self._run_entry(i)
            self.cursor = i + 1

    def run_all(self) -> None:
        self.run(self.cursor, len(self))

    # -- one entry -----------------------------------------------------------------------
    def _positions(self, ch: Chunk) -> np.ndarray:
        pos = np.empty(ch.new_total, np.int64)
        for g in ch.segments:
            pos[g.row0 : g.row0 + g.share] = g.prefix + np.arange(g.share)
        return pos

    def _run_entry(self, i: int) -> None:
        sh, w = self.shape, self.weights
        ci, layer, op = self.entry(i)
        ch = self.chunks[ci]
        P = f"{layer}."
        if op == 0:  # qkv_proj: (embed) + rmsnorm + QKV GEMM + RoPE + KV write
            if layer == 0:
                self.h = w["embed"][self.stream[ch.start : ch.end]].astype(np.float32)
            xn = rmsnorm(self.h, w[P + "attn_norm"], sh.rms_eps)
            n = ch.new_total
            q, k, v = xn @ w[P + "wq"].T, xn @ w[P + "wk"].T, xn @ w[P + "wv"].T
            if sh.qkv_bias:
                q, k, v = q + w[P + "bq"], k + w[P + "bk"], v + w[P + "bv"]
            q = q.reshape(n, sh.n_heads, sh.head_dim)
            k = k.reshape(n, sh.n_kv_heads, sh.head_dim)
            v = v.reshape(n, sh.n_kv_heads, sh.head_dim)
            if sh.qk_norm:
                q = rmsnorm(q, w[P + "q_norm"], sh.rms_eps)
                k = rmsnorm(k, w[P + "k_norm"], sh.rms_eps)
            cos, sin = rope_tables(self._positions(ch), sh.head_dim, sh.rope_theta)
            self.q = apply_rope(q, cos, sin)
            k = apply_rope(k, cos, sin)
            for g in ch.segments:
                rows = slice(g.row0, g.row0 + g.share)
                self.k_cache[g.req][layer][g.prefix : g.prefix + g.share] = k[rows]
                self.v_cache[g.req][layer][g.prefix : g.prefix + g.share] = v[rows]
        elif op == 1:  # attn: per-request causal over own prefix + share
            ao = np.zeros((ch.new_total, sh.n_heads, sh.head_dim), np.float32)
            for g in ch.segments:
                kv_len = g.prefix + g.share
                ao[g.row0 : g.row0 + g.share] = causal_attention(
                    self.q[g.row0 : g.row0 + g.share],
                    self.k_cache[g.req][layer][:kv_len],
                    self.v_cache[g.req][layer][:kv_len],
                    g.prefix,
                )
            self.ao = ao.reshape(ch.new_total, sh.qdim)
        elif op == 2:  # o_proj + residual
            self.h = self.h + self.ao @ w[P + "wo"].T
        elif op == 3 and sh.moe:  # gate: rmsnorm + router softmax + top-k
            self.xn = rmsnorm(self.h, w[P + "ffn_norm"], sh.rms_eps)
            self.moe_ids, self.moe_w = moe_route(self.xn, w[P + "w_router"], sh.top_k,
                                                 sh.norm_topk)
        elif op == 3:  # rmsnorm + gate/up + SwiGLU
            xn = rmsnorm(self.h, w[P + "ffn_norm"], sh.rms_eps)
            self.act = silu(xn @ w[P + "w_gate"].T) * (xn @ w[P + "w_up"].T)
        else:  # down_proj / experts + residual (+ final norm and lm_head of completing requests)
            if sh.moe:
                self.h = self.h + moe_experts(self.xn, self.moe_ids, self.moe_w,
                                              w[P + "e_gate"], w[P + "e_up"], w[P + "e_down"])
            else:
                self.h = self.h + self.act @ w[P + "w_down"].T
            if layer == sh.num_layers - 1:
                for req, row in ch.last:
                    xf = rmsnorm(self.h[row : row + 1], w["final_norm"], sh.rms_eps)
                    self.logits[req] = (xf @ w["lm_head"].T)[0]


def forward_logits(shape: Shape, weights: dict, tokens: list, chunk_size=None) -> np.ndarray:
    t = OracleTask(shape, weights, tokens, chunk_size)
    t.run_all()
    return t.logits
