"""Counter-based streams, restated without numpy's Generator (test oracle).

Reference: src/april_sim/rng.py:33-77.

* key = blake2b(digest_size=16) over the 8-byte little-endian signed
  encodings of (seed, lane, instance_id, sample_index)   (rng.py:42-47)
* word t of a stream = Philox4x64-10(counter=((t >> 2) + 1, 0, 0, 0),
  key=(key mod 2^64, key >> 64))[t & 3].  numpy's Philox increments the
  counter before producing the first block, hence the +1 (rng.py:50-55
  positions the generator at block t>>2 and discards t&3 words).
* draw u = (word >> 11) * 2^-53                          (numpy next_double)
* `Stream.uniform` clamps to [2^-53, 1-2^-53] (rng.py:71-74); the policy
  engine uses the raw draw (engine.py:276).
"""

from __future__ import annotations

import hashlib

import numpy as np

LANE_SAMPLE_LENGTH = 0
LANE_INSTANCE_SHARED = 1
LANE_POLICY_TOKENS = 2
LANE_HISTOGRAM = 3
LANE_PROMPT = 4  # build-specific: synthetic prompt ids (not used by the reference)

_M0 = 0xD2E7470EE14C6C93
_M1 = 0xCA5A826395121157
_W0 = 0x9E3779B97F4A7C15
_W1 = 0xBB67AE8584CAA73B
_U64 = (1 << 64) - 1
_INV53 = 2.0 ** -53


def stream_key(seed: int, lane: int, iid: int, sidx: int) -> int:
    """128-bit key; rng.py:42-47."""
    h = hashlib.blake2b(digest_size=16)
    h.update(b"".join(int(v).to_bytes(8, "little", signed=True) for v in (seed, lane, iid, sidx)))
    return int.from_bytes(h.digest(), "little")


def key_words(key: int) -> tuple[int, int]:
    return key & _U64, key >> 64


def philox_block(ctr0: int, k0: int, k1: int) -> tuple[int, int, int, int]:
    """Philox4x64-10 of counter (ctr0, 0, 0, 0)."""
    x0, x1, x2, x3 = ctr0 & _U64, 0, 0, 0
    for rnd in range(10):
        if rnd:
            k0 = (k0 + _W0) & _U64
            k1 = (k1 + _W1) & _U64
        a = _M0 * x0
        b = _M1 * x2
        x0, x1, x2, x3 = (b >> 64) ^ x1 ^ k0, b & _U64, (a >> 64) ^ x3 ^ k1, a & _U64
    return x0, x1, x2, x3


def word(key: int, t: int) -> int:
    k0, k1 = key_words(key)
    return philox_block((t >> 2) + 1, k0, k1)[t & 3]


def raw_uniform(key: int, t: int) -> float:
    """Unclamped draw t, as numpy Generator.random() yields it."""
    return (word(key, t) >> 11) * _INV53


def raw_uniforms(key: int, start: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    k0, k1 = key_words(key)
    cache_blk, cache = -1, None
    for i in range(n):
        t = start + i
        blk = t >> 2
        if blk != cache_blk:
            cache, cache_blk = philox_block(blk + 1, k0, k1), blk
        out[i] = (cache[t & 3] >> 11) * _INV53
    return out


def clamped_uniform(key: int, t: int) -> float:
    u = raw_uniform(key, t)
    return min(max(u, _INV53), 1.0 - _INV53)


class StreamCursor:
    """Sequential reader positioned at word `pos` (engine.py:265-269)."""

    __slots__ = ("k0", "k1", "pos", "_blk", "_words")

    def __init__(self, key: int, pos: int):
        self.k0, self.k1 = key_words(key)
        self.pos = pos
        self._blk = -1
        self._words = None

    def next_raw(self) -> float:
        blk = self.pos >> 2
        if blk != self._blk:
            self._words = philox_block(blk + 1, self.k0, self.k1)
            self._blk = blk
        w = self._words[self.pos & 3]
        self.pos += 1
        return (w >> 11) * _INV53
