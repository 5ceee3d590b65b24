"""Compare the scheduling decisions of a plain bench run with a --force-dp run (world-1 lockstep
wrapper): per timed step the generated tokens, iterations, carried-in tokens and buffer size must be
identical.  Usage: python tools/compare_forcedp.py plain.log dp.log"""
import json
import sys


def line(path):
    return json.loads([ln for ln in open(path) if ln.startswith("{")][-1])


a, b = line(sys.argv[1]), line(sys.argv[2])
pa, pb = a["april"]["per_step"], b["april"]["per_step"]
same = pa == pb
print(json.dumps({"identical_decisions": same, "plain": pa, "force_dp": pb,
                  "plain_tokens_per_s": a["value"], "force_dp_tokens_per_s": b["value"],
                  "plain_parallelism": a["config"]["parallelism"],
                  "force_dp_parallelism": b["config"]["parallelism"]}, indent=1))
sys.exit(0 if same else 1)
