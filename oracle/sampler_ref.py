"""CPU restatement of the fused sampler's row rule — TEST INFRASTRUCTURE ONLY.

Reference anchor: the toy policy's index-order inverse CDF (src/april_sim/policy.py:93-100;
`token_from_uniform` = #{i : cdf[i] <= u}, logp = log p[tok]) and the engine's use of the raw
draw (src/april_sim/engine.py:276).  Temperature and nucleus (top-p) truncation are not in the
reference (parity-unpinned by it); with temperature 1 and top_p 1 the rule reduces to the
reference's.  This restates the build's K1 arithmetic (csrc/sampler.cu `sample_row`):

* scaled mass p_j = 2^((z_j - max z) * k2) in float32, k2 = float32(1/T) * log2(e);
* nucleus: keep every token whose logit key >= k*, the largest key with
  mass{key >= k*} >= ceil(top_p * total) in fixed-point units floor(p_j * 2^40)
  (ties at the threshold are all kept);
* u * S_kept selects the first kept index whose running kept mass exceeds it;
* logp = float32((z_tok - max z) * (1/T)) - ln S_kept; greedy = argmax, lowest index.
"""

from __future__ import annotations

import math

import numpy as np

_LOG2E = np.float32(1.4426950408889634)
_SCALE = 1099511627776.0  # 2^40


def logit_keys(z: np.ndarray) -> np.ndarray:
    """Monotone uint32 key of float32 logits (larger logit <=> larger key)."""
    b = np.ascontiguousarray(z, dtype=np.float32).view(np.uint32)
    neg = (b & np.uint32(0x80000000)) != 0
    return np.where(neg, ~b, b | np.uint32(0x80000000)).astype(np.uint32)


def nucleus_threshold(z: np.ndarray, temperature: float, top_p: float) -> int:
    """k*: the largest logit key whose at-or-above fixed-point mass reaches ceil(top_p * total)."""
    z = np.asarray(z, dtype=np.float32)
    inv_t = np.float32(1.0) / np.float32(temperature)
    k2 = np.float32(inv_t * _LOG2E)
    m = np.float32(z.max())
    p = np.exp2(((z - m) * k2).astype(np.float32)).astype(np.float64)
    q = np.floor(p * _SCALE).astype(np.uint64)
    keys = logit_keys(z)
    tot = int(q.sum(dtype=np.uint64))
    target = max(1, math.ceil(float(top_p) * float(tot)))
    order = np.argsort(-keys.astype(np.int64), kind="stable")
    cum = 0
    for idx in order:
        cum += int(q[idx])
        if cum >= target:
            return int(keys[idx])
    return int(keys[order[-1]])


def sample_row(z: np.ndarray, temperature: float, greedy: bool, top_p: float, u: float) -> tuple[int, float]:
    z = np.asarray(z, dtype=np.float32)
    inv_t = np.float32(1.0) / np.float32(temperature) if temperature > 0 else np.float32(1.0)
    k2 = np.float32(inv_t * _LOG2E)
    m = np.float32(z.max())
    p = np.exp2(((z - m) * k2).astype(np.float32)).astype(np.float64)
    keep = np.ones(z.shape, dtype=bool)
    if not greedy and top_p < 1.0:
        keep = logit_keys(z) >= np.uint32(nucleus_threshold(z, temperature, top_p))
    pk = np.where(keep, p, 0.0)
    s = float(pk.sum())
    if greedy:
        tok = int(np.argmax(z))
    else:
        run = np.cumsum(pk)
        hit = np.nonzero(run > u * s)[0]
        tok = int(hit[0]) if hit.size else int(np.nonzero(keep)[0][-1])
    logp = float(np.float32((z[tok] - m) * inv_t)) - math.log(s)
    return tok, logp
