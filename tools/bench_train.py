"""Training-iteration throughput (SURVEY §8(f) rows 2+4): one train_loop update
(rollout.hpp:127-145) = collect_rollout (T = 64) + ppo_update for each agent
type (PpoConfig defaults: 4 epochs x 4 minibatches), all on the device, against
the reference's train iteration (oracle/_ref: MarketVecEnv on every host core,
single-threaded policy / PPO code) on a smaller env count.  Prints one JSON
line: env-steps/s of the whole iteration (rollout + update)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02136_b200 import abi  # noqa: E402
from paper_2511_02136_b200.env import DeviceStore, HostStore, MarketVecEnv  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--envs", type=int, default=65536)
    p.add_argument("--T", type=int, default=64)
    p.add_argument("--hidden", type=int, default=32)
    p.add_argument("--ref-envs", type=int, default=1024)
    args = p.parse_args()
    from oracle.oracle import Oracle, OVecEnv, available
    orc = Oracle("orc")
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER), abi.agent_spec(abi.EXECUTOR)],
                         steps_per_episode=64, messages_per_step=100, start_stride_steps=1)
    dims = [(abi.observation_size(cfg.specs[t].obs_space, cfg.obs_depth), abi.action_arity(cfg.specs[t]))
            for t in range(cfg.n_specs)]
    nets = [orc.make_policy_net(d, args.hidden, a, 100 + t) for t, (d, a) in enumerate(dims)]
    pcfg = abi.ppo_config()
    hs = HostStore.synth(abi.synth_config(n_messages=(args.envs + 64) * 100, state_sample_every=100), 0)
    v = MarketVecEnv(DeviceStore(hs, 0), cfg, seed=0, n_envs=args.envs)
    del hs
    v.reset_all()
    v.set_nets(nets)

    def iteration(upd):
        v.collect_rollout(args.T, seed=1, update_index=upd)
        for t in range(cfg.n_specs):
            v.ppo_update(t, pcfg, seed=1, update_index=upd)
        v.synchronize()

    iteration(1)  # warm-up
    w0 = time.perf_counter()
    iteration(2)
    dt = time.perf_counter() - w0
    w1 = time.perf_counter()
    v.collect_rollout(args.T, seed=1, update_index=3)
    v.synchronize()
    roll = time.perf_counter() - w1
    out = {"metric": "train iteration env-steps/s", "unit": "env-steps/s", "value": args.envs * args.T / dt,
           "seconds_per_iteration": dt, "rollout_seconds": roll, "update_seconds": dt - roll,
           "config": {"n_envs": args.envs, "rollout_len": args.T, "hidden": args.hidden, "epochs": 4,
                      "minibatches": 4, "agents_per_env": 2}}
    if available("ref"):
        ref = Oracle("ref")
        rnets = [ref.make_policy_net(d, args.hidden, a, 100 + t) for t, (d, a) in enumerate(dims)]
        ost = ref.synth(abi.synth_config(n_messages=(args.ref_envs + 64) * 100, state_sample_every=100), 0)
        workers = os.cpu_count() or 1
        rv = OVecEnv(ref, ost, cfg, 0, args.ref_envs, workers=workers)
        rv.reset_all()
        w0 = time.perf_counter()
        rv.collect_rollout(rnets, args.T, 0.99, 0.95, 1, 1)
        r_roll = time.perf_counter() - w0
        for t in range(cfg.n_specs):
            rv.ppo_update(t, pcfg, 1, 1)
        rdt = time.perf_counter() - w0
        out["cpu_baseline"] = {"value": args.ref_envs * args.T / rdt, "unit": "env-steps/s", "cores": workers,
                               "kind": "reference",
                               "sample": f"collect_rollout + ppo_update x2, {args.ref_envs} envs x {args.T} steps, "
                                         f"wall {rdt:.2f}s (rollout {r_roll:.2f}s)"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
