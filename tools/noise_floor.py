"""Noise floor of the engine's numerics contract at full depth (CPU only).

The oracle (oracle/cpu_model.py) fixes WHERE activations are rounded to bf16, not the fp32 summation
order inside a projection; the GPU's tcgen05 GEMMs (and split-K reduce-adds) sum in a different
order, so a bf16 rounding occasionally lands on the other side, and the difference propagates
through the layers.  This tool measures how far two equally valid implementations of the same
contract drift apart: the oracle in fp32 vs the oracle summing in fp64 (same bf16 roundings), on
the same token sequence at the full-depth greedy test's shape.  Reported: argmax flips, their
margins, and max / mean |delta logp|, per position band.

  python tools/noise_floor.py --preset qwen2.5-1.5b --prompt 256 --gen 1600
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2509_18521_b200 as pb  # noqa: E402
from oracle.cpu_model import CpuDecoder, random_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="qwen2.5-1.5b")
    ap.add_argument("--prompt", type=int, default=256)
    ap.add_argument("--gen", type=int, default=1600)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    spec = pb.PRESETS[args.preset]
    w = random_weights(spec, seed=0)
    toks = [int(t) for t in pb.synthetic_prompt(13, 0, args.prompt + args.gen, spec.vocab)]
    prompt, gen = toks[: args.prompt], toks[args.prompt:]
    a = CpuDecoder(spec, w).score_all(prompt, gen)
    del_ = CpuDecoder(spec, w, compute_dtype=torch.float64)
    b = del_.score_all(prompt, gen)
    flips = a["argmax"] != b["argmax"]
    # margin of a flip under the fp64 form: how far from a tie the disagreement was
    dl = np.abs(a["logp"] - b["logp"])
    rep = {"preset": args.preset, "layers": spec.n_layers, "positions": len(gen), "flips": int(flips.sum()),
           "flip_frac": float(flips.mean()), "max_abs_dlogp": float(dl.max()), "mean_abs_dlogp": float(dl.mean()),
           "median_top2_margin": float(np.median(b["top2"])),
           "max_abs_dlogp_by_band": [float(dl[i:i + 400].max()) for i in range(0, len(gen), 400)]}
    print(json.dumps(rep))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
