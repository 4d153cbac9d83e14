"""Rollout throughput: collect_rollout — GRU policy
forward (fp64, hidden 32), categorical sampling, env step, GAE — on the GPU
(mlob_venv_collect_rollout, batch in HBM) against the reference's own
collect_rollout (oracle/_ref, MarketVecEnv stepping on every host core; the
reference's policy forward is single-threaded) on the same config.  Prints
one JSON line: env-steps/s (one env-step = every agent of one env acting once)
and msg-steps/s."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_02136_b200 import abi  # noqa: E402
from paper_2511_02136_b200.env import DeviceStore, HostStore, MarketVecEnv  # noqa: E402


def config():
    A = abi
    return A.env_config([A.agent_spec(A.MARKET_MAKER), A.agent_spec(A.EXECUTOR)],
                        steps_per_episode=64, messages_per_step=100, start_stride_steps=1)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--envs", type=int, default=262144)
    p.add_argument("--T", type=int, default=64)
    p.add_argument("--hidden", type=int, default=32)
    p.add_argument("--ref-envs", type=int, default=16384)
    p.add_argument("--ref-T", type=int, default=64)
    args = p.parse_args()
    from oracle.oracle import Oracle, OVecEnv, available
    orc = Oracle("orc")  # network initialisation only (make_policy_net)
    cfg = config()
    dims = [(abi.observation_size(cfg.specs[t].obs_space, cfg.obs_depth), abi.action_arity(cfg.specs[t]))
            for t in range(cfg.n_specs)]
    nets = [orc.make_policy_net(d, args.hidden, a, 100 + t) for t, (d, a) in enumerate(dims)]
    hs = HostStore.synth(abi.synth_config(n_messages=(args.envs + 64) * 100, state_sample_every=100), 0)
    dev = DeviceStore(hs, 0)
    del hs
    v = MarketVecEnv(dev, cfg, seed=0, n_envs=args.envs)
    v.reset_all()
    v.set_nets(nets)
    v.collect_rollout(args.T, seed=1, update_index=1)  # warm-up
    v.synchronize()
    m0 = v.messages_processed()
    stream = torch.cuda.ExternalStream(v.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    v.collect_rollout(args.T, seed=1, update_index=2)
    e1.record(stream)
    e1.synchronize()
    dt = e0.elapsed_time(e1) / 1e3
    msgs = v.messages_processed() - m0
    out = {"metric": "rollout env-steps/s", "unit": "env-steps/s", "value": args.envs * args.T / dt,
           "msg_steps_per_s": msgs / dt, "seconds": dt,
           "config": {"n_envs": args.envs, "rollout_len": args.T, "hidden": args.hidden,
                      "agents_per_env": 2, "messages_per_step": 100, "book_capacity": 100}}
    if available("ref"):
        ref = Oracle("ref")
        rnets = [ref.make_policy_net(d, args.hidden, a, 100 + t) for t, (d, a) in enumerate(dims)]
        ost = ref.synth(abi.synth_config(n_messages=(args.ref_envs + 64) * 100, state_sample_every=100), 0)
        workers = os.cpu_count() or 1
        rv = OVecEnv(ref, ost, cfg, 0, args.ref_envs, workers=workers)
        rv.reset_all()
        rv.collect_rollout(rnets, 2, 0.99, 0.95, 1, 1)  # warm-up
        w0 = time.perf_counter()
        rv.collect_rollout(rnets, args.ref_T, 0.99, 0.95, 1, 2)
        rdt = time.perf_counter() - w0
        out["cpu_baseline"] = {"value": args.ref_envs * args.ref_T / rdt, "unit": "env-steps/s",
                               "cores": workers, "kind": "reference",
                               "sample": f"ippo::collect_rollout, {args.ref_envs} envs x {args.ref_T} steps, "
                                         f"MarketVecEnv on {workers} threads, wall {rdt:.2f}s"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
