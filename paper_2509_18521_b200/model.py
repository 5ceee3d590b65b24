"""Decoder shapes, sampling settings and synthetic prompts for the B200 engine.

The reference has no model at all (its decode "engine" is the cost model
d0 + d1*b, src/april_sim/engine.py:167-171); these are the builder's shapes
from SURVEY.md §8d (public HF configs of the named checkpoints), with
random-init bf16 weights N(0, weight_std) generated on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .errors import ConfigError
from .rng import LANE_PROMPT, philox_key


@dataclass(frozen=True)
class ModelSpec:
    name: str
    n_layers: int
    d_model: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    qkv_bias: bool = False
    qk_norm: bool = False
    tied_embeddings: bool = True
    rope_theta: float = 1e6
    norm_eps: float = 1e-6

    def __post_init__(self):
        if self.n_q_heads % self.n_kv_heads:
            raise ConfigError("n_q_heads must be a multiple of n_kv_heads")
        if self.head_dim not in (64, 128):
            raise ConfigError("head_dim must be 64 or 128")
        if self.d_model % 64 or self.d_ff % 64:
            raise ConfigError("d_model and d_ff must be multiples of 64")

    def truncated(self, n_layers: int) -> "ModelSpec":
        return replace(self, name=f"{self.name}-L{n_layers}", n_layers=n_layers)

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * 2

    @property
    def weight_bytes(self) -> int:
        d, f, hq, hk, hd, v = self.d_model, self.d_ff, self.n_q_heads, self.n_kv_heads, self.head_dim, self.vocab
        per_layer = d * (hq + 2 * hk) * hd + hq * hd * d + 2 * d * f + f * d
        emb = v * d * (1 if self.tied_embeddings else 2)
        return 2 * (self.n_layers * per_layer + emb)


PRESETS = {
    # C1: tiny CPU-oracle decoder
    "tiny": ModelSpec("tiny", 2, 256, 4, 2, 64, 1024, 1024, rope_theta=1e4),
    # C2: Qwen2.5-1.5B shape
    "qwen2.5-1.5b": ModelSpec("qwen2.5-1.5b", 28, 1536, 12, 2, 128, 8960, 151936, qkv_bias=True),
    # C3/C4: Qwen3-4B shape
    "qwen3-4b": ModelSpec("qwen3-4b", 36, 2560, 32, 8, 128, 9728, 151936, qk_norm=True),
    # C5: DeepSeek-R1-Distill-Qwen-7B shape
    "r1-distill-7b": ModelSpec("r1-distill-7b", 28, 3584, 28, 4, 128, 18944, 152064, qkv_bias=True,
                               tied_embeddings=False, rope_theta=1e4),
}


@dataclass(frozen=True)
class SamplingConfig:
    """Fused-sampler settings.

    temperature=1, top_p=1, greedy=False reduces exactly to the reference's
    index-order inverse-CDF draw (policy.py:93-94).
    """

    temperature: float = 1.0
    top_p: float = 1.0
    greedy: bool = False
    eos_ids: tuple[int, ...] = ()

    def __post_init__(self):
        if not self.greedy and not self.temperature > 0:
            raise ConfigError(f"temperature must be > 0, got {self.temperature}")
        if not 0 < self.top_p <= 1:
            raise ConfigError(f"top_p must lie in (0, 1], got {self.top_p}")
        if len(self.eos_ids) > 8:
            raise ConfigError("at most 8 EOS ids")


def synthetic_prompt(seed: int, instance_id: int, length: int, vocab: int) -> np.ndarray:
    """Prompt ids uniform in [0, vocab-1) from Philox lane 4 keyed (seed, 4, iid, 0).

    id_j = floor(u_j * (vocab - 1)) with u_j the j-th draw of the stream
    (numpy-compatible Philox, same convention as the token streams).
    """
    k = philox_key(seed, LANE_PROMPT, instance_id, 0)
    gen = np.random.Generator(np.random.Philox(key=k))
    u = gen.random(length)
    return np.minimum(np.floor(u * (vocab - 1)), vocab - 2).astype(np.int32)
