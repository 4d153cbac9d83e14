"""Throughput bench of the batched LOB environment step (BASELINE.json metric:
LOB env-steps/sec at 1/2/4/8 B200, % of HBM roofline, CPU reference beside it).

A "step" is one environment step of every env (bench::RandomStepHarness,
bench/bench.hpp:53-70: random actions keyed (seed, BenchAction, env, step),
auto-reset).  The unit of the metric is the message-level LOB step — one MBO
message (agent or replay) through one env's book — counted exactly like the
reference's messages_processed (env.hpp:233, bench.hpp:133-154).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload E|B|C|D] [--no-extra]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)
  python bench.py --impl reference ...                    (the reference on the host cores)

One step = act_kernel + book_kernel + outcome_kernel.  The line
carries the default workload (E) and, unless --no-extra, config D (deep book)
under "workloads"; "roofline" is the dominant kernel's (book_kernel: its own
algorithmic bytes over its CUDA-event time on the launching stream), with the
whole-step figure, the kernel's share of the step, the matching ncu capture's
DRAM traffic and an issue-rate roofline beside it.  Small workloads (working
set < 4 x L2) get the L2 flushed between timed steps, outside the events.
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

METRIC = "LOB env-steps/sec (1/2/4/8 B200) and % HBM roofline vs CPU reference"
UNIT = "msg-steps/s"
# Algorithmic bytes per message-level step, SURVEY.md §8(d) / DESIGN.md
# ("Roofline"): book slots r+w, replay message read, env/agent state r+w,
# outputs; per config.
B_MSG = {"B": 171.4, "C": 169.1, "D": 1431.0, "E": 169.1}
HBM_FALLBACK = 6650.0


def workload(name: str):
    """BASELINE.json configs: unique-start synthetic stores
    (an episode every 100 messages), 64 steps x 100 msgs, capacity 100."""
    from paper_2511_02136_b200 import abi
    ex = abi.agent_spec(abi.EXECUTOR)
    mm = abi.agent_spec(abi.MARKET_MAKER)
    if name == "D":  # deep book: SURVEY §8d config D (trimmed store, 64 full episodes)
        cfg = abi.env_config([mm, ex], steps_per_episode=64, messages_per_step=100,
                             start_stride_steps=64, book_capacity=1000)
        synth = abi.synth_config(n_messages=80 * 6400, state_sample_every=6400, initial_mid=100000,
                                 band=2000, p_new_passive=0.46, p_new_cross=0.04, p_cancel=0.30,
                                 p_delete=0.16, p_execute=0.02, state_depth=1000)
        return 262144, cfg, synth, "D: 262144 envs, two-agent, deep book (capacity 1000, 2000 live orders)"
    n_envs, specs, label = {
        "B": (4096, [ex], "B: 4096 envs, single execution agent"),
        "C": (65536, [mm, ex], "C: 65536 envs, two-agent (market maker + execution)"),
        "E": (1 << 20, [mm, ex], "E: 1M (2^20) envs, two-agent, env-sharded over the GPUs"),
    }[name]
    cfg = abi.env_config(specs, steps_per_episode=64, messages_per_step=100, start_stride_steps=1)
    synth = abi.synth_config(n_messages=(n_envs + 64) * 100, state_sample_every=100)
    return n_envs, cfg, synth, label


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def cpu_reference_run(n_envs_cap: int, steps: int, warmup: int, name: str, workers: int = 0):
    """bench::run_throughput (bench.hpp:98-160) of the compiled reference
    (oracle/_ref) on this host's cores, same workload, bounded env count."""
    from oracle.oracle import Oracle, available, bench_run
    if not available("ref"):
        raise RuntimeError("oracle/_ref not built")
    o = Oracle("ref")
    n_envs, cfg, synth, label = workload(name)
    n = min(n_envs, n_envs_cap)
    from paper_2511_02136_b200 import abi
    if name == "D":
        from oracle.oracle import OStore
        full = o.synth(synth, 0)
        msgs = full.messages()[16 * 6400:]
        states = [(i - 16 * 6400, b, a) for i, b, a in full.states() if i >= 16 * 6400]
        store = o.store_from(msgs, states)
    else:
        small = abi.synth_config(n_messages=(n + 64) * 100, state_sample_every=100)
        store = o.synth(small, 0)   # the same stream's prefix: identical episodes 0..n
    workers = workers or os.cpu_count() or 1
    row = bench_run(o, store, cfg, n, steps, warmup, workers, 0, 100, 1)
    return row, workers, n, label


def reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    row, workers, n, label = cpu_reference_run(args.ref_envs, args.steps, args.warmup, args.workload)
    cfg = workload(args.workload)[1]
    v = row.messages_per_sec
    sample = (f"{n} envs x {args.steps} timed steps (+{args.warmup} warm-up) of workload "
              f"{args.workload}, bench::run_throughput with {workers} worker threads")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * row.wall_seconds / max(1, args.steps), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
           "config": {"workload": label, "n_envs_sample": n, "messages_per_step": cfg.messages_per_step,
                      "book_capacity": cfg.book_capacity},
           "env_steps_per_s": row.steps_per_sec,
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def load_profile(name: str) -> dict:
    """The committed ncu capture of this workload's book_kernel
    (profiles/ncu_summary.json, one entry per workload), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get("workloads", {}).get(name, {})
    except Exception:
        return {}


def host_store(name, synth, world, local, barrier):
    """The workload's synthetic store, generated once per node: local rank 0
    synthesises and saves it, the other ranks of the node load the file."""
    from paper_2511_02136_b200.env import HostStore
    t0 = time.time()
    if world == 1:
        hs = HostStore.synth(synth, 0)
    else:
        import torch
        import torch.distributed as dist
        # the file name carries local rank 0's pid (shared by a max all-reduce)
        pid = torch.tensor([os.getpid() if local == 0 else 0], dtype=torch.int64)
        dist.all_reduce(pid, op=dist.ReduceOp.MAX, group=barrier)
        path = f"/tmp/mlob_store_{name}_{synth.n_messages}_{int(pid.item())}.bin"
        if local == 0:
            hs = HostStore.synth(synth, 0)
            hs.save(path)
        dist.barrier(group=barrier)
        if local != 0:
            hs = HostStore.load(path)
        dist.barrier(group=barrier)
        if local == 0:
            os.unlink(path)
    if name == "D":
        hs.trim_front(16 * 6400)  # every remaining episode starts with a full 1000-level book
    return hs, time.time() - t0


# Algorithmic bytes per message of the book kernel alone: B_MSG less the
# agent state / action / observation / reward terms that act_kernel and
# outcome_kernel move (Σ_agents 128 + 4 + 4·obs_dim + 5 per
# env-step).
B_BOOK = {"B": (17275 - 177) / 100.78, "C": (17488 - 346) / 103.41, "D": (148492 - 346) / 103.77,
          "E": (17488 - 346) / 103.41}
ISSUE_PEAK = 148 * 4 * 1.965e9  # warp instructions / s at 100 % issue, 1,965 MHz


def measure(name, args, world, rank, local, dev, allreduce, barrier, cpu_group, with_e2e=True):
    """One workload: device-timed value with per-kernel events, roofline, e2e."""
    import numpy as np
    import torch

    from paper_2511_02136_b200 import abi
    from paper_2511_02136_b200.env import DeviceStore, MarketVecEnv

    n_total, cfg, synth, label = workload(name)
    if args.mps:
        cfg.messages_per_step = args.mps
        synth.n_messages = (n_total + 64) * args.mps
        synth.state_sample_every = args.mps
    if args.envs and name == args.workload:
        n_total = args.envs
        synth.n_messages = (n_total + 64) * cfg.messages_per_step
    per = n_total // world
    base = rank * per
    n_local = per if rank < world - 1 else n_total - base
    hs, gen_s = host_store(name, synth, world, local, cpu_group)
    store = DeviceStore(hs, dev)
    del hs
    venv = MarketVecEnv(store, cfg, seed=0, n_envs=n_local, n_envs_global=n_total,
                        env_index_base=base, device=dev)
    venv.reset_all()
    stream = torch.cuda.ExternalStream(venv.stream, device=torch.device("cuda", dev))
    # working set against the L2: book slots + replay store + per-env state
    props = torch.cuda.get_device_properties(dev)
    l2 = int(getattr(props, "L2_cache_size", 126 * 2 ** 20))
    spl = max(1, -(-int(cfg.book_capacity) // 32))
    spl = 1 << (spl - 1).bit_length()
    work = n_local * 2 * spl * 32 * 20 + store.n_messages * 32 + n_local * 1024
    flush = work < 4 * l2  # small workloads: flush the L2 between timed steps
    scrub = torch.empty(2 * l2 // 4 + 1, dtype=torch.int32, device=f"cuda:{dev}") if flush else None

    gstep = 0
    for _ in range(args.warmup):
        venv.step_random(0, gstep)
        gstep += 1
    venv.synchronize()
    m0 = venv.messages_processed()
    l0 = venv.launches
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps if flush else 2)]
    barrier()
    with ClockSampler(dev) as clocks:
        if flush:
            for i in range(args.steps):
                with torch.cuda.stream(stream):
                    scrub.fill_(i)
                evs[2 * i].record(stream)
                venv.step_random(0, gstep)
                evs[2 * i + 1].record(stream)
                gstep += 1
        else:
            evs[0].record(stream)
            for _ in range(args.steps):
                venv.step_random(0, gstep)
                gstep += 1
            evs[1].record(stream)
        evs[-1].synchronize()
    launches = venv.launches - l0
    venv.synchronize()
    ms = sum(evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(len(evs) // 2))
    m_timed = venv.messages_processed() - m0
    # per-kernel split from a profiled pass right after the timed steps (the
    # profiled step runs its kernels in one stream, in order, with events
    # between them; the timed steps may overlap a chunk's thread kernels with
    # another chunk's book_kernel)
    venv.profile(True)
    for _ in range(max(1, min(3, args.steps))):
        if flush:
            with torch.cuda.stream(stream):
                scrub.fill_(7)
        venv.step_random(0, gstep)
        gstep += 1
    venv.synchronize()
    kms, ksteps = venv.kernel_ms()
    venv.profile(False)
    msgs = m_timed
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    m = torch.tensor([msgs], dtype=torch.float64, device="cuda")
    kb = torch.tensor([kms[1]], dtype=torch.float64, device="cuda")
    allreduce(t, "max")
    allreduce(m)
    allreduce(kb, "max")
    ms_max, msgs_all = float(t.item()), float(m.item())
    value = msgs_all / (ms_max / 1e3)
    env_steps = n_total * args.steps / (ms_max / 1e3)

    # K4 + the all-reduce: episode statistics across ranks (the only collective)
    stats = torch.zeros(abi.STAT_WORDS * cfg.n_specs, dtype=torch.float64, device="cuda")
    venv.episode_stats_device(stats.data_ptr())
    venv.synchronize()
    allreduce(stats)

    out = {"value": value, "ms_per_step": ms_max / args.steps, "env_steps_per_s": env_steps,
           "launches": launches, "clocks": clocks.summary(),
           "episodes": float(stats[4].item()), "label": label, "n_total": n_total, "n_local": n_local,
           "cfg": cfg, "gen_s": gen_s, "flush": flush, "work": work, "l2": l2}
    # roofline of the dominant kernel (book_kernel): its algorithmic bytes per
    # launch over its own event-timed duration on the launching stream
    book_s = float(kb.item()) / 1e3 / max(1, ksteps)
    step_s = ms_max / 1e3 / args.steps
    per_launch_msgs = msgs_all / args.steps
    peak, peak_kind = peaks()
    prof = load_profile(name)
    bb = B_BOOK.get(name, 165.8)
    achieved = bb * (msgs / args.steps) / book_s / 1e9 if book_s > 0 else None
    inst = prof.get("inst_per_msg")
    out["roofline"] = {
        "bound": "hbm", "kernel": f"book_kernel<{spl}, false, {'true' if spl <= 4 and n_local >= 16384 else 'false'}>",
        "achieved": achieved, "peak": peak,
        "unit": "GB/s", "frac": achieved / peak if achieved else None,
        "traffic": prof["dram_bytes_per_msg"] * (msgs / args.steps) if "dram_bytes_per_msg" in prof else None,
        "bytes_per_msg": round(bb, 1), "peak_kind": peak_kind,
        "kernel_share_of_step": (kms[1] / sum(kms)) if sum(kms) > 0 else None,
        "kernel_ms": [round(x / max(1, ksteps), 4) for x in kms],
        "step": {"bytes_per_msg": B_MSG.get(name, 169.1),
                 "achieved": B_MSG.get(name, 169.1) * per_launch_msgs / step_s / world / 1e9,
                 "frac": B_MSG.get(name, 169.1) * per_launch_msgs / step_s / world / 1e9 / peak},
        # issue-rate bound: book_kernel warp instructions per message (ncu) x rate
        "issue": ({"inst_per_msg": inst, "achieved": inst * (msgs / args.steps) / book_s,
                   "peak": ISSUE_PEAK, "unit": "warp-inst/s",
                   "frac": inst * (msgs / args.steps) / book_s / ISSUE_PEAK}
                  if inst and book_s > 0 else None),
        "ncu_capture": prof.get("capture")}

    if with_e2e:
        # e2e through the public API with host buffers, every step: pinned actions
        # H2D, step, rewards + dones + per-type observations and reset flags D2H
        # (mlob_venv_step_io: one call; the copies overlap the chunked step)
        A = venv.n_agents
        rng = np.random.default_rng(1234)
        ar = np.array([abi.action_arity(cfg.specs[s]) for s in abi.flat_specs(cfg)])
        e_steps = max(3, min(args.steps, args.e2e_steps))
        acts_all = [torch.from_numpy((rng.integers(0, 1 << 30, size=(n_local, A)) % ar).astype(np.int32))
                    .pin_memory() for _ in range(e_steps + 1)]
        obs_bufs = [torch.empty((venv.n_streams(t), venv.obs_dim(t)), dtype=torch.float64).pin_memory()
                    for t in range(cfg.n_specs)]
        rew = torch.empty((n_local, A), dtype=torch.float64).pin_memory()
        dn = torch.empty((n_local, A), dtype=torch.uint8).pin_memory()
        rsb = [torch.empty(venv.n_streams(t), dtype=torch.uint8).pin_memory() for t in range(cfg.n_specs)]

        def e2e_step(a):
            venv.step_io(actions=a, rewards=rew, dones=dn, obs=obs_bufs, resets=rsb)

        e2e_step(acts_all[e_steps])  # warm-up (creates the copy streams)
        em0 = venv.messages_processed()
        barrier()
        w0 = time.perf_counter()
        for i in range(e_steps):
            e2e_step(acts_all[i])
        torch.cuda.synchronize()
        e_wall = torch.tensor([time.perf_counter() - w0], dtype=torch.float64, device="cuda")
        allreduce(e_wall, "max")
        e_m = torch.tensor([venv.messages_processed() - em0], dtype=torch.float64, device="cuda")
        allreduce(e_m)
        h2d = acts_all[0].numel() * 4
        d2h = rew.numel() * 8 + dn.numel() + sum(b.numel() * 8 for b in obs_bufs) + \
            sum(b.numel() for b in rsb)
        out["e2e"] = {"value": float(e_m.item()) / float(e_wall.item()), "unit": UNIT,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e_steps}
    del venv, store
    torch.cuda.empty_cache()
    return out


def gpu_arm(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # diagnostics only: MLOB_BENCH_BACKEND=gloo + MLOB_BENCH_DEVICE=0 run several
    # ranks on one GPU to exercise the multi-rank path (sharding, max-over-ranks
    # timing, stats all-reduce); real runs use one GPU per rank and NCCL.
    backend = os.environ.get("MLOB_BENCH_BACKEND", "nccl")
    dev = int(os.environ.get("MLOB_BENCH_DEVICE", local))
    torch.cuda.set_device(dev)
    cpu_group = None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
        cpu_group = dist.new_group(backend="gloo") if backend == "nccl" else None
    coll_dev = "cuda" if backend == "nccl" else "cpu"

    def allreduce(t, op=None):
        if world > 1:
            x = t.to(coll_dev)
            dist.all_reduce(x, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
            t.copy_(x)
        return t

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    r = measure(args.workload, args, world, rank, local, dev, allreduce, barrier, cpu_group)
    extra = {}
    if args.workload != "D" and not args.no_extra:
        # config D (deep book, BASELINE.json configs[3]) in the same driver-run line
        d = measure("D", args, world, rank, local, dev, allreduce, barrier, cpu_group,
                    with_e2e=True)
        extra["D"] = {k: d[k] for k in ("value", "ms_per_step", "env_steps_per_s", "roofline", "e2e",
                                        "launches", "clocks")}
        extra["D"]["workload"] = d["label"]
        extra["D"]["n_envs"] = d["n_total"]
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cfg = r["cfg"]
    l2 = ("inputs larger than L2" if not r["flush"] else "L2 flushed between timed steps") + \
        f" (working set {r['work'] / 2 ** 30:.2f} GiB per GPU vs L2 {r['l2'] / 2 ** 20:.0f} MiB)"
    out = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
           "config": {"workload": r["label"], "n_envs": r["n_total"], "envs_per_gpu": r["n_local"],
                      "agents_per_env": cfg.n_agents if hasattr(cfg, "n_agents") else None,
                      "messages_per_step": cfg.messages_per_step,
                      "steps_per_episode": cfg.steps_per_episode,
                      "book_capacity": cfg.book_capacity, "parallelism": f"env-shard x{world}",
                      "l2": l2, "store_messages": None, "store_gen_s": round(r["gen_s"], 2)},
           "env_steps_per_s": r["env_steps_per_s"],
           "roofline": r["roofline"],
           "gpu_launches": r["launches"],
           "clocks": r["clocks"],
           "episode_stats": {"episodes": r["episodes"]},
           "e2e": r["e2e"]}
    from paper_2511_02136_b200 import abi
    out["config"]["agents_per_env"] = sum(s.count for s in cfg.specs[:cfg.n_specs])
    out["config"]["store_messages"] = int(workload(args.workload)[2].n_messages)
    if extra:
        out["workloads"] = extra
    if world == 1 and not args.no_cpu:
        try:
            row, workers, n, _ = cpu_reference_run(args.ref_envs, args.cpu_steps, 2, args.workload)
            out["cpu_baseline"] = {"value": row.messages_per_sec, "unit": UNIT, "cores": workers,
                                   "kind": "reference",
                                   "sample": f"{n} envs x {args.cpu_steps} timed steps (+2 warm-up), "
                                             f"bench::run_throughput, {workers} threads, "
                                             f"wall {row.wall_seconds:.2f}s"}
            row1, _, n1, _ = cpu_reference_run(4096, 30, 2, args.workload, workers=1)
            out["cpu_baseline"]["per_core"] = {
                "value": row1.messages_per_sec, "unit": UNIT, "cores": 1,
                "sample": f"{n1} envs x 30 timed steps (+2 warm-up), bench::run_throughput, 1 thread, "
                          f"wall {row1.wall_seconds:.2f}s"}
        except Exception as e:  # reported, not fatal
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="E", choices=["B", "C", "D", "E"])
    p.add_argument("--envs", type=int, default=0, help="override the env count")
    p.add_argument("--mps", type=int, default=0, help="override messages per step (diagnostics)")
    p.add_argument("--ref-envs", type=int, default=65536)
    p.add_argument("--cpu-steps", type=int, default=300)
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the config-D entry of the line")
    args = p.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
