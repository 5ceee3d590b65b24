"""Device-side data-parallel lockstep on the GPU.

`world` engines share cuda:0 inside one process, one host thread each (the ctypes calls release the
GIL, so the device loops run concurrently on separate streams).  Each engine is attached to the
others' exchange buffers (`Engine.dp_attach`, same-process pointers), so every decode iteration ends
with `k_dp_exchange`: the per-iteration counts cross over peer memory and the trigger / drain are
decided on the device — one `ab_engine_run` per scheduler call, exactly the multi-GPU code path
(`GpuLocal` + `DataParallelEngine`) minus CUDA IPC.  Rank 0's canonical step records must equal the
composed k-engine oracle's (oracle/sim_ref.py KEngineOracle) bit for bit; the finished-response gather
must hand every delivered sample's payload to every rank.  A second test runs the same path across two
processes (gloo for the host collectives, CUDA IPC for the exchange buffers).
"""

import os
import socket
import sys
import threading

import pytest

import canon
from product_runs import make_scheduler, step_events

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _k_oracle(name, mode, steps, world):
    from oracle import sim_ref

    cfg = dict(canon.CONFIGS[name], mode=mode)
    eng, sch = sim_ref.make_k_oracle(cfg, world)
    recs = []
    for k in range(steps):
        eng.event_log = []
        out = sch.run_step(k)
        recs.append(canon.step_record(sch, out, eng.event_log))
    return recs


def _engine(cfg, model=None, **kw):
    import paper_2509_18521_b200 as pb

    ecfg = pb.EngineConfig(max_slots=cfg["slots"], l_max=cfg["l_max"])
    return pb.LengthDrivenEngine(ecfg, global_seed=cfg.get("seed", 0), model=model, **kw)


def _run_threads(name, mode, steps, world, fused=True, model=None, gather=False, **kw):
    from paper_2509_18521_b200.dist import DataParallelEngine, GpuLocal, ThreadComm, gather_responses

    cfg = canon.CONFIGS[name]
    comms = ThreadComm.group(world)
    engines = [_engine(cfg, model, **kw) for _ in range(world)]  # created one by one (autotune timing)
    out = [None] * world
    errors = []

    def work(r):
        try:
            local = GpuLocal(engines[r]).attach(comms[r], timeout_ms=60_000)
            front = DataParallelEngine(local, comms[r], cfg["slots"])
            sched = make_scheduler(cfg, mode, fused=fused, engine=front)
            recs, gathered = [], []
            for k in range(steps):
                o = sched.run_step(k)
                recs.append(canon.step_record(sched, o, step_events(sched)))
                if gather:
                    samples = o.batch_samples()
                    got = gather_responses(comms[r], samples)
                    owned = {s.sample_id: (s.token_ids(), s.behavior_logprob_trace()) for s in samples
                             if s.segments and all(seg.tokens is not None for seg in s.segments)}
                    gathered.append(([s.sample_id for s in samples], got, owned))
            out[r] = (recs, gathered)
        except BaseException as exc:  # noqa: BLE001 - re-raised in the main thread
            errors.append((r, exc))
            comms[r].abort()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=900)
    for e in engines:
        e.close()
    if errors:
        raise errors[0][1]
    assert all(o is not None for o in out)
    return out


@pytest.mark.parametrize("name,mode,steps,world,fused", [
    ("C1", "april", 6, 2, True),
    ("C1", "april", 4, 4, True),
    ("E_samples", "april", 12, 2, True),
    ("E_cap", "april", 10, 2, False),   # decode_until_event: stop on the first global event
    ("E_pool", "april", 12, 3, True),
    ("C1", "baseline", 3, 2, True),
    ("C3", "april", 3, 2, True),
])
def test_device_lockstep_matches_k_engine_oracle(name, mode, steps, world, fused):
    out = _run_threads(name, mode, steps, world, fused=fused)
    ref = _k_oracle(name, mode, steps, world)
    for r in range(world):  # every rank's replicated scheduler sees the same global records
        for a, b in zip(out[r][0], ref):
            assert a == b, (r, canon.first_diff(a, b))


def test_device_lockstep_with_model_and_response_gather():
    """The tiny transformer decodes on both ranks (idle ranks sit iterations out with stop = 2);
    trace mode fixes the lengths, so the decisions must still equal the oracle's, and the gathered
    payload must equal each owner's token ids and behaviour log-probs."""
    import paper_2509_18521_b200 as pb

    out = _run_threads("C1", "april", 3, 2, model=pb.PRESETS["tiny"],
                       sampling=pb.SamplingConfig(temperature=0.8), prompt_len=32, kv_resume="reprefill", kv_pages=20000,
                       gather=True)
    ref = _k_oracle("C1", "april", 3, 2)
    for a, b in zip(out[0][0], ref):
        assert a == b, canon.first_diff(a, b)
    for k in range(3):
        ids0, got0, _ = out[0][1][k]
        ids1, got1, _ = out[1][1][k]
        assert ids0 == ids1 and got0 == got1
        owned = {**out[0][1][k][2], **out[1][1][k][2]}
        assert set(owned) == set(ids0)
        for sid, (tok, lp) in zip(ids0, got0):
            assert owned[sid] == (tok, lp)
            assert len(tok) == len(lp) > 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _proc_worker(rank, world, port, name, steps, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import canon as cn
    from paper_2509_18521_b200.dist import DataParallelEngine, GpuLocal, TorchComm
    from product_runs import make_scheduler as mk, step_events as se

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = cn.CONFIGS[name]
        comm = TorchComm()
        local = GpuLocal(_engine(cfg)).attach(comm, timeout_ms=30_000)  # CUDA IPC between the processes
        front = DataParallelEngine(local, comm, cfg["slots"])
        sched = mk(cfg, "april", engine=front)
        recs = []
        for k in range(steps):
            o = sched.run_step(k)
            recs.append(cn.step_record(sched, o, se(sched)))
        q.put((rank, recs))
    except BaseException as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_device_lockstep_across_processes_ipc():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_proc_worker, args=(r, 2, port, "C1", 3, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    ref = _k_oracle("C1", "april", 3, 2)
    for r in range(2):
        assert not isinstance(got[r], str), got[r]
        for a, b in zip(got[r], ref):
            assert a == b, canon.first_diff(a, b)


def test_device_lockstep_policy_mode_matches_k_engine_oracle():
    """Policy stop rules (the reference's toy PolicyDrivenEngine on the GPU: Philox draw, softmax,
    inverse CDF, STOP) under the device lockstep at world 2: no jump hints (the exchange's policy
    branch), token ids included in the comparison with the composed k-engine oracle."""
    import numpy as np

    import paper_2509_18521_b200 as pb
    from oracle import sim_ref
    from paper_2509_18521_b200.dist import DataParallelEngine, GpuLocal, ThreadComm

    t = canon.TOY
    z = np.array([0.4, -0.1, 0.2, 0.0, -0.6])
    steps, world = 10, 2
    # the composed oracle
    keng = sim_ref.KEngineOracle(world, t["d0"], t["d1"], t["slots"], t["l_max"], mode="policy", seed=t["seed"])
    ksch = sim_ref.OracleScheduler(t["n"], t["g"], t["n_prime"], keng, mode="april")
    ref, ref_tok = [], {}
    for k in range(steps):
        keng.event_log = []
        out = ksch.run_step(k, z)
        ref.append(canon.step_record(ksch, out, keng.event_log))
        ref_tok.update({(k, s.sample_id): s.token_ids() for s in out.batch_samples()})
    # the device lockstep
    comms = ThreadComm.group(world)
    ecfg = pb.EngineConfig(max_slots=t["slots"], l_max=t["l_max"])
    engines = [pb.PolicyDrivenEngine(ecfg, global_seed=t["seed"]) for _ in range(world)]
    for e in engines:
        e._create(z.size)  # the context-free engine is otherwise created at its first begin_step
    out_recs, errors = [None] * world, []

    def work(r):
        try:
            front = DataParallelEngine(GpuLocal(engines[r]).attach(comms[r]), comms[r], t["slots"])
            scfg = pb.SchedulerConfig(rollout_batch_size=t["n"], samples_per_prompt=t["g"],
                                      over_sampling_batch_size=t["n_prime"], mode="april")
            sched = pb.Scheduler(scfg, front, pb.InstanceSource(group_size=t["g"]), None)
            sched.event_sink = []
            recs, toks = [], {}
            for k in range(steps):
                o = sched.run_step(k, pb.PolicyParams(z, k))
                recs.append(canon.step_record(sched, o, step_events(sched)))
                # token ids of the delivered samples this rank generated (remote mirrors carry none)
                toks.update({(k, s.sample_id): s.token_ids() for s in o.batch_samples()
                             if s.segments and all(seg.tokens is not None for seg in s.segments)})
            out_recs[r] = (recs, toks)
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)
            comms[r].abort()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=600)
    for e in engines:
        e.close()
    if errors:
        raise errors[0]
    for r in range(world):
        for a, b in zip(out_recs[r][0], ref):
            assert a == b, (r, canon.first_diff(a, b))
    got = {**out_recs[0][1], **out_recs[1][1]}
    assert set(got) == set(ref_tok)
    assert all(got[k] == ref_tok[k] for k in ref_tok)
