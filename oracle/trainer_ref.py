"""CPU restatement of the trainer-side clipped-ratio terms — TEST INFRASTRUCTURE ONLY.

Checker for K7 (`ab_clipped_ratio_terms`, csrc/advantage.cu).  Per token the importance ratio
r = exp(logp_now - logp_behaviour) and the clip rule of the reference's clipped-ratio gradient
(src/april_sim/policy.py:153-177: a token is clipped iff A > 0 and r > 1 + eps_high, or A < 0 and
r < 1 - eps; DAPO clip-higher eps_high = 0.28), and per response the surrogate
sum_t min(r A, clip(r, 1 - eps, 1 + eps_high) A) whose gradient that function takes.  GSPO's
sequence-level ratio exp(mean_t(logp_now - logp_behaviour)) is the paper's (parity-unpinned: the
reference has no GSPO code).
"""

from __future__ import annotations

import numpy as np


def clipped_ratio_terms(logp_now, logp_beh, advantages, eps_clip=0.2, eps_clip_high=0.28, sequence_level=False):
    lo, hi = 1.0 - eps_clip, 1.0 + eps_clip_high
    ratios, masks, surrogate = [], [], []
    for now, beh, a in zip(logp_now, logp_beh, np.asarray(advantages, dtype=float)):
        d = np.asarray(now, dtype=float) - np.asarray(beh, dtype=float)
        if sequence_level:
            r = np.array([np.exp(d.mean())]) if d.size else np.zeros(0)
        else:
            r = np.exp(d)
        clipped = ((a > 0) & (r > hi)) | ((a < 0) & (r < lo))  # policy.py:169-171
        ratios.append(r)
        masks.append(clipped)
        surrogate.append(float(np.sum(np.minimum(r * a, np.clip(r, lo, hi) * a))))
    return ratios, masks, surrogate
