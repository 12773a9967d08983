"""Model shapes of the BASELINE configs (public model-card values; weights are random-init)."""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ModelShape:
    name: str
    num_layers: int
    hidden: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float
    rms_eps: float = 1e-5
    qkv_bias: bool = False  # Qwen2.5
    qk_norm: bool = False   # Qwen3
    # MoE (Qwen3-MoE: every layer's FFN is a router + top-k SwiGLU experts; ffn unused)
    n_experts: int = 0
    top_k: int = 0
    moe_ffn: int = 0
    norm_topk: bool = False

    @property
    def moe(self) -> bool:
        return self.n_experts > 0

    @property
    def qdim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kvdim(self) -> int:
        return self.n_kv_heads * self.head_dim

    def gemm_flops_per_token(self) -> float:
        """2 * (qkv + o + gate_up + down) weights, per token per layer."""
        d = self.hidden
        if self.moe:  # router + the top_k active experts
            ffn = self.n_experts * d + self.top_k * 3 * d * self.moe_ffn
        else:
            ffn = 3 * d * self.ffn
        w = d * (self.qdim + 2 * self.kvdim) + self.qdim * d + ffn
        return 2.0 * w

    def attn_flops(self, share: int, prefix: int) -> float:
        """Causal attention FLOPs of one request share with a prefix, per layer:
        QK^T and PV over the visible keys, 4 * qdim * sum_i (prefix + i)."""
        return 4.0 * self.qdim * (share * prefix + share * (share + 1) / 2.0)

    def kv_bytes_per_token(self) -> int:
        return self.num_layers * 2 * self.kvdim * 2


SHAPES = {
    "tiny": ModelShape("tiny", 4, 512, 4, 2, 128, 1536, 8192, 1e4),
    "llama3-8b": ModelShape("llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256, 5e5),
    # configs[2]: independent per-GPU instances
    "qwen3-8b": ModelShape("qwen3-8b", 36, 4096, 32, 8, 128, 12288, 151936, 1e6, 1e-6,
                           qk_norm=True),
    # configs[3]: tensor parallel
    "qwen2.5-32b": ModelShape("qwen2.5-32b", 64, 5120, 40, 8, 128, 27648, 152064, 1e6, 1e-6,
                              qkv_bias=True),
    # parity-test variants (match oracle.forward.SHAPES)
    "tiny-qwen3": ModelShape("tiny-qwen3", 2, 512, 4, 2, 128, 1536, 8000, 1e6, 1e-6,
                             qk_norm=True),
    "tiny-qwen2": ModelShape("tiny-qwen2", 2, 512, 4, 2, 128, 1536, 8000, 1e6, 1e-6,
                             qkv_bias=True),
    "tiny-qwen2-tp": ModelShape("tiny-qwen2-tp", 4, 512, 20, 4, 128, 2048, 8000, 1e6, 1e-6,
                                qkv_bias=True),
    # MoE: Qwen3-30B-A3B shape (128 experts, top-8, expert ffn 768)
    "qwen3-30b-a3b": ModelShape("qwen3-30b-a3b", 48, 2048, 32, 4, 128, 0, 151936, 1e6, 1e-6,
                                qk_norm=True, n_experts=128, top_k=8, moe_ffn=768,
                                norm_topk=True),
    "tiny-moe": ModelShape("tiny-moe", 2, 512, 4, 2, 128, 0, 8000, 1e6, 1e-6, qk_norm=True,
                           n_experts=16, top_k=4, moe_ffn=256, norm_topk=True),
}
