"""Cross-play throughput: ippo::evaluate_matrix over a
5 x 5 grid of scripted policies (NoOp / TWAP / AvSt / Random) on the GPU
(mlob_evaluate_matrix, one env per cell x episode) against the reference's own
evaluate_matrix compiled from /root/reference (oracle/_ref, one host thread —
the reference driver is sequential), on the same store, config and grid.
Prints one JSON line.  Both sides are timed end to end through their public
call (store upload excluded; the GPU leg includes env creation, reset, the
steps and the result readback)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02136_b200 import abi  # noqa: E402
from paper_2511_02136_b200.env import DeviceStore, HostStore, evaluate_matrix  # noqa: E402


def grid():
    A = abi
    t0 = [A.policy(A.POLICY_NOOP), A.policy(A.POLICY_AVST), A.policy(A.POLICY_AVST, gamma_index=3),
          A.policy(A.POLICY_RANDOM), A.policy(A.POLICY_AVST, gamma_index=0)]
    t1 = [A.policy(A.POLICY_TWAP), A.policy(A.POLICY_TWAP, twap_mode=A.TWAP_PASSIVE),
          A.policy(A.POLICY_RANDOM), A.policy(A.POLICY_NOOP), A.policy(A.POLICY_TWAP)]
    return t0, t1


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--episodes", type=int, default=4096)
    p.add_argument("--ref-episodes", type=int, default=512)
    p.add_argument("--reps", type=int, default=3)
    args = p.parse_args()
    A = abi
    cfg = A.env_config([A.agent_spec(A.MARKET_MAKER, mm_space=A.AVST), A.agent_spec(A.EXECUTOR)],
                       steps_per_episode=64, messages_per_step=100, start_stride_steps=1)
    synth = A.synth_config(n_messages=(args.episodes + 64) * 100, state_sample_every=100)
    t0, t1 = grid()
    eps = list(range(args.episodes))
    hs = HostStore.synth(synth, 0)
    dev = DeviceStore(hs, 0)
    evaluate_matrix(dev, cfg, eps[:64], t0, t1, 3)  # warm-up (module load, first launches)
    best = None
    for _ in range(args.reps):
        w0 = time.perf_counter()
        cells = evaluate_matrix(dev, cfg, eps, t0, t1, 3)
        dt = time.perf_counter() - w0
        best = dt if best is None else min(best, dt)
    n_env_eps = len(t0) * len(t1) * args.episodes
    out = {"metric": "crossplay episodes/s", "unit": "episodes/s",
           "value": n_env_eps / best, "wall_s": best,
           "config": {"grid": f"{len(t0)}x{len(t1)}", "episodes_per_cell": args.episodes,
                      "steps_per_episode": 64, "messages_per_step": 100, "book_capacity": 100},
           "cells_sample": [{"pv0": c.per_type[0].pv_mean, "completion1": c.per_type[1].completion_mean}
                            for c in cells[:3]]}
    try:
        from oracle.oracle import Oracle, available
        if available("ref"):
            ref = Oracle("ref")
            ost = ref.synth(A.synth_config(n_messages=(args.ref_episodes + 64) * 100,
                                           state_sample_every=100), 0)
            w0 = time.perf_counter()
            rc = ref.evaluate(ost, cfg, eps[:args.ref_episodes], t0, t1, 3)
            dt = time.perf_counter() - w0
            n_ref = len(t0) * len(t1) * args.ref_episodes
            mine = evaluate_matrix(dev, cfg, eps[:args.ref_episodes], t0, t1, 3)
            out["cpu_baseline"] = {"value": n_ref / dt, "unit": "episodes/s", "cores": 1,
                                   "kind": "reference",
                                   "sample": f"ippo::evaluate_matrix, {len(t0)}x{len(t1)} grid x "
                                             f"{args.ref_episodes} episodes, wall {dt:.2f}s",
                                   "identical_cells": [bytes(x) for x in rc] == [bytes(x) for x in mine]}
    except Exception as e:  # reported, not fatal
        out["cpu_baseline"] = {"value": None, "sample": f"unavailable: {e}"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
