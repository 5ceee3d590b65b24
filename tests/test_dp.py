"""Data-parallel path on CPU: world_size 2 over gloo.

Each rank runs the B200 build's replicated Scheduler over a DataParallelEngine
whose local engine is the CPU oracle engine (the per-rank GPU engine is not
available on a CPU box; the host logic under test — placement, lockstep
counter exchange, log gather/merge, remote mirrors, abort merge — is the same).
Rank 0's canonical step records must equal the composed k-engine oracle's
(oracle/sim_ref.py KEngineOracle, k = 2) bit for bit.
"""

import os
import socket
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, mode, steps, fused, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import canon
    import paper_2509_18521_b200 as pb
    from oracle import sim_ref
    from paper_2509_18521_b200.dist import DataParallelEngine, OracleLocal, TorchComm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = canon.CONFIGS[name]
        local = OracleLocal(sim_ref.OracleEngine(0.05, 0.002, cfg["slots"], cfg["l_max"]))
        eng = DataParallelEngine(local, TorchComm(), cfg["slots"])
        d = cfg["dist"]
        dist_obj = (pb.LengthDistribution.constant(int(d[1]), cfg["l_max"]) if d[0] == "constant"
                    else pb.LengthDistribution.lognormal(d[1], d[2], cfg["l_max"]))
        scfg = pb.SchedulerConfig(rollout_batch_size=cfg["n"], samples_per_prompt=cfg["g"],
                                  over_sampling_batch_size=cfg["n_prime"], mode=mode,
                                  trigger=cfg.get("trigger", "groups"))
        sched = pb.Scheduler(scfg, eng, pb.InstanceSource(group_size=cfg["g"]),
                             pb.LengthSampler(dist_obj, cfg["rho"], cfg["seed"]))
        sched._fused = fused
        sched.event_sink = []
        recs = []
        for k in range(steps):
            out = sched.run_step(k)
            evs = [[r["iteration_index"], *map(int, r["sample_id"].split(":")), r["tokens"], r["reason"]]
                   for r in sched.event_sink if r["reason"] != "aborted"]
            sched.event_sink.clear()
            recs.append(canon.step_record(sched, out, evs))
        if rank == 0:
            q.put(recs)
    finally:
        dist.destroy_process_group()


def _run_dp(name, mode, steps, fused):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, mode, steps, fused, q)) for r in range(2)]
    for p in procs:
        p.start()
    recs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return recs


def _k_oracle(name, mode, steps):
    import canon
    from oracle import sim_ref

    cfg = dict(canon.CONFIGS[name], mode=mode)
    eng, sch = sim_ref.make_k_oracle(cfg, 2)
    recs = []
    for k in range(steps):
        eng.event_log = []
        out = sch.run_step(k)
        recs.append(canon.step_record(sch, out, eng.event_log))
    return recs


@pytest.mark.parametrize("name,mode,steps,fused", [
    ("C1", "april", 8, True),
    ("E_samples", "april", 12, True),
    ("E_cap", "april", 10, False),
    ("C1", "baseline", 3, True),
])
def test_dp_world2_matches_k_engine_oracle(name, mode, steps, fused):
    import canon

    mine = _run_dp(name, mode, steps, fused)
    ref = _k_oracle(name, mode, steps)
    for a, b in zip(mine, ref):
        assert a == b, canon.first_diff(a, b)


def test_k_engine_oracle_k1_is_the_single_engine():
    import canon
    from oracle import sim_ref
    from oracle_runs import oracle_replay

    cfg = dict(canon.CONFIGS["C1"], mode="april")
    eng, sch = sim_ref.make_k_oracle(cfg, 1)
    recs = []
    for k in range(6):
        eng.event_log = []
        out = sch.run_step(k)
        recs.append(canon.step_record(sch, out, eng.event_log))
    assert recs == oracle_replay(canon.CONFIGS["C1"], "april", 6)


def _gather_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2509_18521_b200.dist import TorchComm, gather_responses
    from paper_2509_18521_b200.rollouts import RolloutSample

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batch = []
        for k in range(7):  # sample k is owned by rank k % world; the others hold payload-free mirrors
            s = RolloutSample(k, 0)
            for v in range(1 + k % 2):
                seg = s.open_segment(v, with_tokens=(k % world == rank))
                seg.token_count = 2 + k + v
                if seg.tokens is not None:
                    seg.tokens = [100 * k + 10 * v + j for j in range(seg.token_count)]
                    seg.behavior_logprobs = [-0.5 * j - k for j in range(seg.token_count)]
            batch.append(s)
        q.put((rank, gather_responses(TorchComm(), batch)))
    finally:
        dist.destroy_process_group()


def test_gather_responses_world2_gloo():
    """Finished-response gather (tokens + log-probs + lengths) over torch.distributed, in delivered order."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = []
    for k in range(7):
        toks, lps = [], []
        for v in range(1 + k % 2):
            n = 2 + k + v
            toks += [100 * k + 10 * v + j for j in range(n)]
            lps += [-0.5 * j - k for j in range(n)]
        want.append((toks, lps))
    assert got[0] == want and got[1] == want


@pytest.mark.parametrize("name,world", [("C1", 3), ("E_pool", 2)])
def test_dp_threads_match_k_engine_oracle(name, world):
    """The same host lockstep with in-process collectives (ThreadComm, one thread per rank): every
    rank's replicated scheduler produces the composed k-engine oracle's records."""
    import threading

    import canon
    import paper_2509_18521_b200 as pb
    from oracle import sim_ref
    from paper_2509_18521_b200.dist import DataParallelEngine, OracleLocal, ThreadComm

    cfg = canon.CONFIGS[name]
    steps = 6
    comms = ThreadComm.group(world, timeout=120)
    out, errors = [None] * world, []

    def work(r):
        try:
            local = OracleLocal(sim_ref.OracleEngine(0.05, 0.002, cfg["slots"], cfg["l_max"]))
            eng = DataParallelEngine(local, comms[r], cfg["slots"])
            d = cfg["dist"]
            dist_obj = pb.LengthDistribution.lognormal(d[1], d[2], cfg["l_max"])
            scfg = pb.SchedulerConfig(rollout_batch_size=cfg["n"], samples_per_prompt=cfg["g"],
                                      over_sampling_batch_size=cfg["n_prime"], mode="april")
            sched = pb.Scheduler(scfg, eng, pb.InstanceSource(group_size=cfg["g"]),
                                 pb.LengthSampler(dist_obj, cfg["rho"], cfg["seed"]))
            sched.event_sink = []
            recs = []
            for k in range(steps):
                o = sched.run_step(k)
                evs = [[x["iteration_index"], *map(int, x["sample_id"].split(":")), x["tokens"], x["reason"]]
                       for x in sched.event_sink if x["reason"] != "aborted"]
                sched.event_sink.clear()
                recs.append(canon.step_record(sched, o, evs))
            out[r] = recs
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)
            comms[r].abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    if errors:
        raise errors[0]
    ceng, csch = sim_ref.make_k_oracle(dict(cfg, mode="april"), world)
    for k in range(steps):
        ceng.event_log = []
        o = csch.run_step(k)
        ref = canon.step_record(csch, o, ceng.event_log)
        for r in range(world):
            assert out[r][k] == ref, (r, k, canon.first_diff(out[r][k], ref))
