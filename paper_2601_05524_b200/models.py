"""Model-card shapes for the BASELINE.json configurations; weights are random-init
bf16 (N(0, init_std), norms = 1), a pure function of the seed."""
from __future__ import annotations

from ._capi import TransformerConfig

# name: (layers, hidden, ffn, heads, kv_heads, head_dim, vocab, tied, qk_norm, rope_theta)
PRESETS = {
    "qwen3-0.6b": (28, 1024, 3072, 16, 8, 128, 151936, 1, 1, 1e6),
    "qwen3-1.7b": (28, 2048, 6144, 16, 8, 128, 151936, 1, 1, 1e6),
    "qwen3-14b": (40, 5120, 17408, 40, 8, 128, 151936, 0, 1, 1e6),
    "qwen3-32b": (64, 5120, 25600, 64, 8, 128, 151936, 0, 1, 1e6),
    "llama-3.2-1b": (16, 2048, 8192, 32, 8, 64, 128256, 1, 0, 5e5),
    "llama-3.1-8b": (32, 4096, 14336, 32, 8, 128, 128256, 0, 0, 5e5),
    "llama-3.3-70b": (80, 8192, 28672, 64, 8, 128, 128256, 0, 0, 5e5),
    # small shapes for parity tests (same code paths, seconds to run)
    "tiny-qwen": (2, 256, 512, 4, 2, 64, 1024, 0, 1, 1e6),
    "tiny-qwen-draft": (1, 128, 384, 2, 1, 64, 1024, 1, 1, 1e6),
    "tiny-llama": (2, 256, 768, 4, 2, 64, 1000, 1, 0, 5e5),
}


def transformer_config(name: str, seed: int = 1, max_seq: int = 4096, tp_rank: int = 0,
                       tp_size: int = 1, init_std: float = 0.02, **override) -> TransformerConfig:
    L, h, f, nh, nkv, hd, V, tied, qkn, theta = PRESETS[name]
    d = dict(n_layers=L, hidden=h, ffn=f, n_heads=nh, n_kv_heads=nkv, head_dim=hd, vocab=V,
             tied_embeddings=tied, qk_norm=qkn, rope_theta=theta, rms_eps=1e-6, init_std=init_std,
             max_seq=max_seq, seed=seed, tp_rank=tp_rank, tp_size=tp_size)
    d.update(override)
    return TransformerConfig(**d)
