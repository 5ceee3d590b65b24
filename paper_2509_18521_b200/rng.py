"""Host-side stream keys (src/april_sim/rng.py:33-77).

The per-sample Philox key is derived once on the host, when a sample is
created, and shipped to the device in its descriptor; the token stream
itself is generated on the GPU by the fused sampler (csrc/common.cuh
`philox_word`).  `Stream` remains for the host-side trace source
(workload.py), which the reference also draws on the host.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np
from scipy.special import ndtri

LANE_SAMPLE_LENGTH = 0
LANE_INSTANCE_SHARED = 1
LANE_POLICY_TOKENS = 2
LANE_HISTOGRAM = 3
LANE_PROMPT = 4  # synthetic prompt ids (this build only)

_EPS = 2.0 ** -53
_MASK64 = (1 << 64) - 1


def philox_key(global_seed: int, lane: int, instance_id: int, sample_index: int) -> int:
    digest = hashlib.blake2b(
        b"".join(int(v).to_bytes(8, "little", signed=True) for v in (global_seed, lane, instance_id, sample_index)),
        digest_size=16,
    ).digest()
    return int.from_bytes(digest, "little")


def key_words(key: int) -> tuple[int, int]:
    """(low, high) 64-bit words, the order the device Philox expects."""
    return key & _MASK64, key >> 64


@dataclass(frozen=True)
class Stream:
    global_seed: int
    lane: int
    instance_id: int
    sample_index: int = 0

    def key(self) -> int:
        return philox_key(self.global_seed, self.lane, self.instance_id, self.sample_index)

    def generator(self, position: int = 0) -> np.random.Generator:
        gen = np.random.Generator(np.random.Philox(key=self.key(), counter=[position >> 2, 0, 0, 0]))
        if position & 3:
            gen.random(position & 3)
        return gen

    def uniform(self, draw_index: int = 0) -> float:
        return min(max(float(self.generator(draw_index).random()), _EPS), 1.0 - _EPS)

    def uniforms(self, n: int, start: int = 0) -> np.ndarray:
        return np.clip(self.generator(start).random(n), _EPS, 1.0 - _EPS)

    def normal(self, draw_index: int = 0) -> float:
        return float(ndtri(self.uniform(draw_index)))
