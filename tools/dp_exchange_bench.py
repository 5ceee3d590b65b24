"""Per-iteration cost of the device-side data-parallel exchange (k_dp_exchange), one GPU.

`world` engines share cuda:0 in one process (one host thread each, as tests/test_dp_gpu.py) and
decode a long constant-length trace with no model, so an iteration is only admit + grow + finish
(+ the exchange when attached).  Reported: device µs per global iteration with the exchange
(world engines in lockstep) against the same engines run independently without it, and the
profiled average of the dp_exchange kernel itself (CUDA events in the iteration graph).

    python tools/dp_exchange_bench.py --world 2 --iters 20000
"""

import argparse
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2509_18521_b200 as pb  # noqa: E402
from paper_2509_18521_b200.dist import ThreadComm  # noqa: E402
from paper_2509_18521_b200.rollouts import RolloutSample  # noqa: E402


def run(world, iters, slots, attach):
    comms = ThreadComm.group(world)
    engs = [pb.LengthDrivenEngine(pb.EngineConfig(max_slots=slots, l_max=iters + 8)) for _ in range(world)]
    res = [None] * world

    def work(r):
        e = engs[r]
        if attach:
            e.dp_attach(comms[r])
        e.begin_step(1)
        for i in range(slots):
            s = RolloutSample(1000 * r + i, 0)
            s.target_length = iters
            e.submit(s)
        e.profile(True, 1)
        comms[r].allgather(None)
        c0 = e.clock
        evs = e.run_until_drained(1)
        c1 = e.clock
        k = {x["name"]: x for x in e.kernel_stats()}
        res[r] = {"seconds": c1 - c0, "iterations": e.last_run.iterations, "events": len(evs),
                  "dp_exchange_us": (1e3 * k["dp_exchange"]["ms"] / max(k["dp_exchange"]["launches"], 1)
                                     if "dp_exchange" in k else None)}

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in engs:
        e.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20000)
    ap.add_argument("--slots", type=int, default=64)
    a = ap.parse_args()
    run(a.world, 200, a.slots, True)  # warm-up (graphs, module load)
    base = run(1, a.iters, a.slots, False)[0]
    dp = run(a.world, a.iters, a.slots, True)
    per_it_base = 1e6 * base["seconds"] / base["iterations"]
    per_it_dp = 1e6 * max(r["seconds"] for r in dp) / dp[0]["iterations"]
    print(json.dumps({"world": a.world, "engines_per_gpu": a.world, "iterations": dp[0]["iterations"],
                      "us_per_iteration_single_engine": per_it_base,
                      "us_per_iteration_lockstep": per_it_dp,
                      "exchange_overhead_us_per_iteration": per_it_dp - per_it_base,
                      "dp_exchange_kernel_avg_us": [r["dp_exchange_us"] for r in dp],
                      "note": "model-off engines sharing one GPU: an iteration is admit + grow + finish "
                              "(+ exchange); on a multi-GPU box the peers are remote over NVLink"}, indent=1))


if __name__ == "__main__":
    main()
