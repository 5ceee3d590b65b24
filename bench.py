#!/usr/bin/env python
"""APRIL rollout benchmark on B200 (BASELINE.json metric).

Workload (SURVEY.md §8d, config C2 = BASELINE.json configs[1]):
  Qwen2.5-1.5B-shape random-init bf16 decoder, GRPO rollout, 64 prompts x n=8,
  over-provisioned to 128 groups (2x), max_len 4096, log-normal(6.6, 1.0)
  response lengths (rho 0.7) replayed as a length trace, 256-token synthetic
  prompts, temperature 0.8, S = 1024 decode slots, one B200.

A "step" is one RL rollout step of the scheduler: begin_step -> resume/open
groups -> (prefill) -> fused decode until N whole groups are complete ->
abort/park.  `value` is APRIL generated tokens/s with the step time measured
on the device clock (payload kept on the GPU); `e2e` runs the same steps
through the public API with the finished-response gather (token ids +
behaviour log-probs copied to host lists), synthetic rewards and the GPU
advantage kernel, timed by the host wall clock.  The synchronous baseline
(no over-provisioning, no recycling) runs on the same engine code, same
trace, afterwards.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rollout tokens/s & RL-step rollout time, APRIL vs sync, long-tail lengths, 1–8 B200"

WORKLOADS = {
    "C2": dict(model="qwen2.5-1.5b", n=64, g=8, n_prime=128, slots=1024, l_max=4096, mu=6.6, sigma=1.0, rho=0.7,
               prompt=256, temperature=0.8, adv="mean_std_baseline", page=64, nondet_gemm=True),
    # BASELINE.json configs[2] per engine: Qwen3-4B shape, DAPO, partial-rollout recycling, S = 64 (the
    # per-GPU slot count of the 8-GPU run); `--workload C3` (not the default line)
    "C3": dict(model="qwen3-4b", n=32, g=8, n_prime=64, slots=64, l_max=16384, mu=7.5, sigma=1.0, rho=0.7,
               prompt=256, temperature=0.8, adv="dapo", page=64, nondet_gemm=True),
    # BASELINE.json configs[3] per engine: Qwen3-4B shape, GSPO, heavy long tail (L_max 16384),
    # over-provision sweep N'/N in {1.5, 2, 3} via --over-provision (S = 64 per GPU; the rest queues)
    "C4": dict(model="qwen3-4b", n=32, g=8, n_prime=64, slots=64, l_max=16384, mu=7.8, sigma=1.2, rho=0.7,
               prompt=256, temperature=0.8, adv="gspo", page=64, nondet_gemm=True),
    # BASELINE.json configs[4] per engine of 8: R1-Distill-Qwen-7B shape (untied lm_head, GQA 7:1,
    # QKV bias), GRPO, 256 prompts x 16 over 8 GPUs = 32 x 16 per engine, N' = 2N; S = 128 rows keeps
    # the worst-case KV (128 x 16,640 tokens x 57,344 B = 122 GB) resident next to 14.1 GB of weights
    "C5": dict(model="r1-distill-7b", n=32, g=16, n_prime=64, slots=128, l_max=16384, mu=7.5, sigma=1.0,
               rho=0.7, prompt=256, temperature=0.8, adv="mean_std_baseline", page=64, nondet_gemm=True),
    # small smoke workload (tiny decoder) for quick checks
    "C1": dict(model="tiny", n=8, g=4, n_prime=16, slots=64, l_max=1024, mu=5.5, sigma=1.0, rho=0.7, prompt=32,
               temperature=0.8, adv="mean_std_baseline", page=16),
}


ADV_NAME = {"mean_std_baseline": "GRPO", "dapo": "DAPO", "gspo": "GSPO", "mean_baseline": "REINFORCE"}


def workload(args):
    w = dict(WORKLOADS[args.workload])
    if args.over_provision:  # C4 sweep: N' = round(x * N)
        w["n_prime"] = int(round(args.over_provision * w["n"]))
    return w


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows)}


def build_engine(pb, w, device, seed, record=True, kv_resume="retain", kv_pages=0):
    spec = pb.PRESETS[w["model"]]
    eng = pb.LengthDrivenEngine(
        pb.EngineConfig(max_slots=w["slots"], l_max=w["l_max"]), global_seed=seed, model=spec,
        sampling=pb.SamplingConfig(temperature=w["temperature"]), prompt_len=w["prompt"], page_size=w["page"],
        device=device, record_payload=record, max_handles=max(4096, 4 * w["n_prime"] * w["g"]),
        max_groups=4 * w["n_prime"] + 64, nondeterministic_gemm=w.get("nondet_gemm", False), kv_resume=kv_resume,
        kv_pages=kv_pages)
    return spec, eng


def make_scheduler(pb, w, eng, mode, seed, world=1):
    # weak scaling: N, N' grow with the number of data-parallel engines (fixed work per GPU)
    n, n_prime = w["n"] * world, w["n_prime"] * world
    cfg = pb.SchedulerConfig(rollout_batch_size=n, samples_per_prompt=w["g"],
                             over_sampling_batch_size=n_prime if mode == "april" else n, mode=mode)
    dist = pb.LengthDistribution.lognormal(w["mu"], w["sigma"], w["l_max"])
    return pb.Scheduler(cfg, eng, pb.InstanceSource(group_size=w["g"]), pb.LengthSampler(dist, w["rho"], seed))


def learner_glue(pb, w, out, target_token=0, comm=None):
    """Synthetic GRPO glue (simulate.py:47-65): target-token-fraction rewards on the
    delivered token ids, then the K6 advantage kernel over contiguous groups.  Data-parallel:
    the finished responses (int32 token ids, fp64 behaviour log-probs, lengths) are gathered
    over NCCL (`dist.gather_responses`), so the trainer sees the whole batch in delivery order."""
    samples = out.batch_samples()
    if comm is not None:
        from paper_2509_18521_b200.dist import gather_responses

        toks_all = [t for t, _ in gather_responses(comm, samples)]
    else:
        toks_all = [s.token_ids() for s in samples]
    rewards = [sum(1 for t in toks if t % 4 == target_token) / len(toks) if toks else 0.0 for toks in toks_all]
    pb.batch_advantages(rewards, w["g"], w["adv"])
    return float(sum(rewards) / len(rewards)) if rewards else 0.0


def run_steps(pb, w, sched, eng, k0, n, timed_e2e=False, comm=None):
    recs = []
    for k in range(k0, k0 + n):
        h2d0 = eng.io_bytes()
        t0 = time.perf_counter()
        out = sched.run_step(k)
        reward = learner_glue(pb, w, out, comm=comm) if timed_e2e else 0.0
        t1 = time.perf_counter()
        h2d1 = eng.io_bytes()
        recs.append(dict(step=k, tokens=out.tokens_generated, wall=out.rollout_wall_time, host=t1 - t0,
                         iters=out.iterations, carried=out.carried_in_tokens,
                         h2d=h2d1[0] - h2d0[0], d2h=h2d1[1] - h2d0[1], buffer=out.buffer_size_after,
                         outcome=out, reward=reward))
    return recs


def cpu_baseline(w, budget_s=15.0):
    import torch

    import paper_2509_18521_b200 as pb
    from oracle.cpu_model import CpuDecoder, random_weights

    spec = pb.PRESETS[w["model"]]
    dec = CpuDecoder(spec, random_weights(spec, 0))
    batch, ctx = 64, 1024
    probe = dec.decode_batch_rate(batch, ctx, 1)
    iters = max(1, min(64, int(budget_s / max(probe["seconds"], 1e-3))))
    r = dec.decode_batch_rate(batch, ctx, iters)
    return {"value": r["tokens_per_s"], "unit": "tokens/s", "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"oracle/cpu_model.py fp32 {spec.name} full depth, {iters} decode iterations x batch {batch} "
                      f"at context {ctx} ({r['seconds']:.1f} s)"}


def _cpu_model_name():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _import_reference():
    """The unmodified reference, installed into baseline/_ref."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "april_sim")):
        return None
    sys.path.insert(0, ref)
    import april_sim

    return april_sim


def reference_timings(w, a, budget_s=6.0):
    """The reference's own CPU path on one core: (1) april_sim replaying the workload's length trace
    through its Scheduler + LengthDrivenEngine (scheduling, abort, recycle; the decode is its d0+d1*b
    cost model), wall seconds per APRIL step; (2) its PolicyDrivenEngine per-token path (Philox draw,
    softmax, inverse CDF, STOP) on the toy policy, tokens per wall second."""
    ecfg = a.EngineConfig(d0=0.05, d1=0.002, max_slots=w["slots"], l_max=w["l_max"])
    eng = a.LengthDrivenEngine(ecfg)
    scfg = a.SchedulerConfig(rollout_batch_size=w["n"], samples_per_prompt=w["g"],
                             over_sampling_batch_size=w["n_prime"], mode="april")
    sampler = a.LengthSampler(a.LengthDistribution.lognormal(w["mu"], w["sigma"], w["l_max"]), w["rho"], 0)
    sched = a.Scheduler(scfg, eng, a.InstanceSource(group_size=w["g"]), sampler)
    t0, k, toks = time.perf_counter(), 0, 0
    while time.perf_counter() - t0 < budget_s and k < 50:
        toks += sched.run_step(k).tokens_generated
        k += 1
    replay = {"steps": k, "seconds_per_step": (time.perf_counter() - t0) / k,
              "simulated_tokens_per_wall_s": toks / (time.perf_counter() - t0), "cores": 1}
    sim = a.build_simulation(a.toy_policy_config().with_overrides(**{"run.steps": 10_000}))
    t0, toks, k = time.perf_counter(), 0, 0
    while time.perf_counter() - t0 < budget_s:
        toks += sim.run_step().tokens_generated
        k += 1
    policy = {"steps": k, "tokens_per_s": toks / (time.perf_counter() - t0), "cores": 1,
              "note": "toy context-free policy (4 symbols + STOP), reference PolicyDrivenEngine + reinforce_update"}
    return {"april_sim_replay": replay, "april_sim_policy_engine": policy}


def reference_arm(args):
    """--impl reference: the reference's CPU path for this workload on the box's host cores.  The
    scheduling half of every step is the unmodified reference (april_sim from baseline/_ref: its
    Scheduler + LengthDrivenEngine replaying the same length trace, one core); the reference has no
    decoder, so the decode half is a bounded sample of the same model's decode iterations on the CPU
    (oracle/cpu_model.py, fp32, all host threads).  value = decoded tokens / wall time of the two."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch

    import paper_2509_18521_b200 as pb
    from oracle.cpu_model import CpuDecoder, random_weights

    a = _import_reference()
    w = workload(args)
    spec = pb.PRESETS[w["model"]]
    dec = CpuDecoder(spec, random_weights(spec, 0))
    batch, ctx = 64, 1024
    probe = dec.decode_batch_rate(batch, ctx, 1)
    iters = max(1, min(32, int(args.ref_step_s / max(probe["seconds"], 1e-3))))
    sched = None
    if a is not None:
        ecfg = a.EngineConfig(d0=0.05, d1=0.002, max_slots=w["slots"], l_max=w["l_max"])
        scfg = a.SchedulerConfig(rollout_batch_size=w["n"], samples_per_prompt=w["g"],
                                 over_sampling_batch_size=w["n_prime"], mode="april")
        sampler = a.LengthSampler(a.LengthDistribution.lognormal(w["mu"], w["sigma"], w["l_max"]), w["rho"], 0)
        sched = a.Scheduler(scfg, a.LengthDrivenEngine(ecfg), a.InstanceSource(group_size=w["g"]), sampler)
    rates, times = [], []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if sched is not None:
            sched.run_step(k)
        r = dec.decode_batch_rate(batch, ctx + 8 * k, iters, seed=k)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            rates.append(r["tokens"] / dt)
            times.append(dt)
    v = statistics.mean(rates)
    sched_src = "april_sim (baseline/_ref, unmodified reference)" if a is not None else "reference not installed"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "shape": spec.name, "prompts": w["n"],
                       "samples_per_prompt": w["g"], "over_provision": w["n_prime"] / w["n"],
                       "max_len": w["l_max"]},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": torch.get_num_threads(),
                             "kind": "reference" if a is not None else "port", "cpu": _cpu_model_name(),
                             "sample": f"per step: one APRIL scheduling step of {sched_src} replaying the "
                                       f"{args.workload} trace + {iters} fp32 decode iterations x batch {batch} of "
                                       f"the full-depth {spec.name} decoder (oracle/cpu_model.py; the reference "
                                       f"has no decoder) at context ~{ctx}"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if a is not None:
        line["reference_cpu_path"] = reference_timings(w, a)
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--sync-steps", type=int, default=5)
    ap.add_argument("--over-provision", type=float, default=None,
                    help="N'/N (over-sampling groups over rollout groups); the workload's default otherwise")
    ap.add_argument("--no-sync", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-every", type=int, default=8)
    ap.add_argument("--ref-step-s", type=float, default=12.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=None,
                    help="also write the reference's run outputs (steps.jsonl, summary.json, samples.csv per arm, "
                         "comparison.json) for the e2e APRIL steps and the sync steps into this directory")
    ap.add_argument("--kv-resume", default="reprefill", choices=["retain", "reprefill"],
                    help="paused partials: re-prefill prompt + carried tokens at resume (the cost APRIL pays when "
                         "weights change every step; inside the rollout wall time) or keep their KV resident")
    ap.add_argument("--force-dp", action="store_true", help="run the data-parallel engine even at N = 1 (tests)")
    ap.add_argument("--kv-pages", type=int, default=0, help="KV pool pages (0: all HBM left after a margin)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent engine replicas instead of the lockstep data-parallel engine")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks: AB_BENCH_DEVICE pins every rank to one GPU and AB_BENCH_BACKEND=gloo runs the host
    # collectives on the CPU (a world-2 smoke test of the multi-rank path on a one-GPU box; the
    # per-iteration exchange still runs on the device through CUDA IPC)
    local = int(os.environ.get("AB_BENCH_DEVICE", local))
    backend = os.environ.get("AB_BENCH_BACKEND", "nccl")
    dist = None
    if world > 1 or args.force_dp:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group(backend, rank=rank, world_size=world)
    import paper_2509_18521_b200 as pb

    w = workload(args)
    dp = (world > 1 and not args.replicas) or args.force_dp
    # data-parallel: one replicated scheduler (same seed everywhere) over lockstep engines;
    # replicas: independent prompt streams per rank
    seed = args.seed if dp else args.seed + rank
    hbm_peak, tf_peak, peak_kind = _peaks()

    spec, eng = build_engine(pb, w, local, seed, record=True, kv_resume=args.kv_resume, kv_pages=args.kv_pages)
    comm = None
    front = eng  # what the scheduler drives
    if dp:
        from paper_2509_18521_b200.dist import DataParallelEngine, GpuLocal, TorchComm

        comm = TorchComm(device=f"cuda:{local}" if backend == "nccl" else "cpu")
        # device lockstep: the per-iteration count exchange runs over NVLink peer memory inside
        # the captured iteration graph (no host round trip per iteration)
        front = DataParallelEngine(GpuLocal(eng).attach(comm), comm, w["slots"])
    sched = make_scheduler(pb, w, front, "april", seed, world if dp else 1)
    run_steps(pb, w, sched, eng, 0, args.warmup, timed_e2e=True, comm=comm)
    if dist:
        dist.barrier()
    eng.profile(True, args.profile_every)
    st0 = eng.stats()
    launches0 = st0.kernel_launches
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        # the same timed steps give `value` (device clock, begin_step -> park) and `e2e` (host wall
        # clock of the public-API call plus the finished-response gather, rewards and advantages)
        rec = run_steps(pb, w, sched, eng, args.warmup, args.steps, timed_e2e=True, comm=comm)
        t_dev = sum(r["wall"] for r in rec)
        if dist:
            import torch

            tt = torch.tensor([t_dev], device="cuda" if backend == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_dev = float(tt)
        t_host = time.perf_counter() - t0
    st1 = eng.stats()
    launches = st1.kernel_launches - launches0
    reprefill = {"mode": args.kv_resume,
                 "tokens_per_step": (st1.reprefill_tokens - st0.reprefill_tokens) / max(args.steps, 1),
                 "prompt_prefill_tokens_per_step": (st1.prefill_tokens - st0.prefill_tokens) / max(args.steps, 1),
                 "seconds_per_step": (st1.reprefill_seconds - st0.reprefill_seconds) / max(args.steps, 1)}
    kstats = {k["name"]: k for k in eng.kernel_stats()}
    eng.profile(False)
    tokens = sum(r["tokens"] for r in rec)
    rec_e2e = rec
    e2e_tps = sum(r["tokens"] for r in rec_e2e) / sum(r["host"] for r in rec_e2e)
    stats = eng.stats()
    eng.close()
    del eng, sched

    sync = None
    if not args.no_sync:
        _, eng_s = build_engine(pb, w, local, seed, record=True, kv_pages=args.kv_pages)
        front_s = eng_s
        if dp:
            front_s = DataParallelEngine(GpuLocal(eng_s).attach(comm), comm, w["slots"])
        sch_s = make_scheduler(pb, w, front_s, "baseline", seed, world if dp else 1)
        run_steps(pb, w, sch_s, eng_s, 0, 1, timed_e2e=True, comm=comm)  # warm-up (graphs, autotune cache)
        rs = run_steps(pb, w, sch_s, eng_s, 1, args.sync_steps, timed_e2e=True, comm=comm)
        sync = {"tokens_per_s": sum(r["tokens"] for r in rs) / sum(r["wall"] for r in rs),
                "ms_per_step": 1e3 * statistics.mean(r["wall"] for r in rs), "steps": len(rs),
                "iterations_per_step": statistics.mean(r["iters"] for r in rs)}
        eng_s.close()
        if args.out and rank == 0:
            write_outputs(pb, w, args, rec_e2e, rs, world)

    # DP: every rank's scheduler already counts the whole job's tokens; replicas: per rank
    total_tokens = tokens if dp else tokens * world
    value = total_tokens / t_dev if t_dev > 0 else 0.0
    att = kstats.get("attention")
    roof = None
    if att and att["ms"] > 0:
        ach = att["bytes"] / (att["ms"] * 1e-3) / 1e9
        traffic, tpoint = _ncu_traffic(args.workload)
        roof = {"kernel": "paged GQA decode attention (k_decode_attn + combine)", "bound": "hbm",
                "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "peak_kind": peak_kind, "traffic": traffic, "traffic_at": tpoint, "launches_timed": att["launches"],
                "avg_launch_us": 1e3 * att["ms"] / att["launches"],
                "avg_algorithmic_bytes_per_launch": att["bytes"] / max(att["launches"], 1)}
    kern = {}
    tot_ms = sum(k["ms"] for k in kstats.values()) or 1.0
    for name, k in sorted(kstats.items(), key=lambda kv: -kv[1]["ms"]):
        ms = k["ms"]
        kern[name] = {"share": ms / tot_ms, "avg_us": 1e3 * ms / max(k["launches"], 1),
                      "GB/s": k["bytes"] / (ms * 1e-3) / 1e9 if ms else None,
                      "TFLOP/s": k["flops"] / (ms * 1e-3) / 1e12 if ms and k["flops"] else None}
    ms_step = 1e3 * t_dev / max(len(rec), 1)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, Philox prompts, replayed "
                                                     "log-normal length trace)",
        "config": {"workload": f"{args.workload}: {spec.name}-shape {ADV_NAME[w['adv']]} APRIL rollout", "prompts": w["n"],
                   "samples_per_prompt": w["g"], "over_provision_groups": w["n_prime"], "max_len": w["l_max"],
                   "length_dist": f"lognormal({w['mu']}, {w['sigma']}), rho {w['rho']}",
                   "prompt_len": w["prompt"], "slots": w["slots"], "temperature": w["temperature"],
                   "gemm": ("fp32-residual split-K partials reduce-added by TMA (split summation order not fixed)"
                            if w.get("nondet_gemm") else "deterministic schedules"),
                   "parallelism": (f"dp{world} lockstep engines (per-iteration count exchange over NVLink peer memory in the "
                                    f"iteration graph, NCCL response gather)"
                                   if dp else f"dp{world} replicas"),
                   "l2": "inputs larger than L2 (weights + KV >> 126 MB)"},
        "april": {"tokens_per_s": value, "ms_per_step": ms_step, "steps": len(rec),
                  "iterations_per_step": statistics.mean(r["iters"] for r in rec),
                  "carried_in_tokens_per_step": statistics.mean(r["carried"] for r in rec),
                  "per_step": [{"step": r["step"], "tokens": r["tokens"], "iterations": r["iters"],
                                "carried_in": r["carried"], "buffer_after": r["buffer"]} for r in rec]},
        "kv_resume": reprefill,
        "sync": sync,
        "april_over_sync": ((value if dp else value / world) / sync["tokens_per_s"]) if sync else None,
        "roofline": roof, "kernels": kern,
        "e2e": {"value": e2e_tps * (1 if dp else world), "unit": "tokens/s",
                "h2d_bytes_per_step": int(statistics.mean(r["h2d"] for r in rec_e2e)),
                "d2h_bytes_per_step": int(statistics.mean(r["d2h"] for r in rec_e2e))},
        "clocks": clk.summary(), "gpu_launches": int(launches),
        "kv_pages": {"total": stats.kv_pages_total, "free_after": stats.kv_pages_free},
        "host_seconds_timed": t_host,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(w)
        except Exception as exc:  # the baseline is reported, not required
            line["cpu_baseline"] = {"value": None, "error": repr(exc)[:200]}
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def write_outputs(pb, w, args, rec_april, rec_sync, world):
    """The reference CLI's run outputs (cli.py:50-129) for the e2e APRIL steps and the sync steps."""
    from paper_2509_18521_b200 import report
    from paper_2509_18521_b200.metrics import build_step_report

    cfg = {"engine": {"backend": "b200", "slots": w["slots"], "max_len": w["l_max"], "model": w["model"],
                      "kv_resume": args.kv_resume},
           "run": {"seed": args.seed, "steps": args.steps, "gpus": world},
           "scheduler": {"rollout_batch_size": w["n"], "samples_per_prompt": w["g"],
                         "over_sampling_batch_size": w["n_prime"]},
           "train": {"advantage": w["adv"]},
           "workload": {"length_dist": "lognormal", "mu": w["mu"], "sigma": w["sigma"], "rho": w["rho"]}}
    summaries = {}
    for mode, recs in (("april", rec_april), ("baseline", rec_sync)):
        # GPU runs have no cost-model peak: idle fraction against the best step of the run
        peak = max(r["tokens"] / r["wall"] for r in recs if r["wall"] > 0)
        reps = [build_step_report(r["outcome"], peak, r["host"] - r["wall"], r["reward"]) for r in recs]
        man = [row for r in recs for row in report.manifest_rows(r["outcome"].step, r["outcome"].batch)]
        summaries[mode] = pb.summarize_run(reps, buffer_high_water=max(r["buffer"] for r in recs))
        report.write_run_outputs(os.path.join(args.out, f"{mode}-seed{args.seed}"), reps, summaries[mode],
                                 dict(cfg, scheduler=dict(cfg["scheduler"], mode=mode)), manifest=man)
    tp = {m: statistics.mean(r["tokens"] / r["wall"] for r in recs) for m, recs in (("april", rec_april),
                                                                                  ("baseline", rec_sync))}
    entry = {"seed": args.seed, "baseline": summaries["baseline"].to_json_dict(),
             "april": summaries["april"].to_json_dict(), "improvement": tp["april"] / tp["baseline"] - 1.0}
    report.write_comparison(args.out, [entry], cfg)


def _ncu_traffic(workload):
    """DRAM read+write bytes per launch of the attention kernel from the committed ncu capture
    (profiles/attention_dram_bytes.json, tools/ncu_attn_point.py) and the operating point it was
    taken at (the bench's average live batch and context for C2); other workloads -> null."""
    p = os.path.join(ROOT, "profiles", "attention_dram_bytes.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d.get("workload", "C2") != workload:
            return None, None
        return d.get("bytes_per_launch"), {"point": d.get("point"),
                                           "algorithmic_bytes_per_launch": d.get("algorithmic_bytes_per_launch"),
                                           "source": "profiles/attention_dram_bytes.json"}
    except Exception:
        return None, None


if __name__ == "__main__":
    sys.exit(main())
