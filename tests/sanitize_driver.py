"""A few steps of the product for the checked-build test
(tests/test_checked_build.py): python tests/sanitize_driver.py
{register|smem} [library].  With a library path the run binds that build
(libmlob_checked.so: device-side bounds / invariant checks that trap) instead
of the product library; it prints a digest of every output so the checked
and product builds can be compared.  No torch: the C ABI only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import hashlib  # noqa: E402

from paper_2511_02136_b200 import abi  # noqa: E402
from paper_2511_02136_b200 import env as E  # noqa: E402
from paper_2511_02136_b200.env import DeviceStore, HostStore, MarketVecEnv  # noqa: E402

DEEP = {"initial_mid": 100000, "band": 2000, "p_new_passive": 0.46, "p_new_cross": 0.04,
        "p_cancel": 0.30, "p_delete": 0.16, "p_execute": 0.02, "state_depth": 200}


def main(kind: str) -> None:
    mm, ex = abi.agent_spec(abi.MARKET_MAKER, obs_space=abi.OBS_MM_FULL), abi.agent_spec(abi.EXECUTOR)
    if kind == "register":  # C = 100: register book, 4 rows per lane
        cfg = abi.env_config([mm, ex], steps_per_episode=4, messages_per_step=100, start_stride_steps=1)
        synth = abi.synth_config(n_messages=20000, state_sample_every=100)
        n = 40
    else:  # C = 300: shared-memory book (bulk-copy load/store), full side evictions
        cfg = abi.env_config([mm, ex], steps_per_episode=4, messages_per_step=100, start_stride_steps=32,
                             book_capacity=300)
        synth = abi.synth_config(**dict(DEEP, n_messages=40000, state_sample_every=3200))
        n = 12
    store = DeviceStore(HostStore.synth(synth, 0), 0)
    v = MarketVecEnv(store, cfg, seed=1, n_envs=n)
    v.reset_all()
    h = hashlib.sha256()
    for t in range(6):  # crosses an episode boundary: the auto-reset path runs
        v.step_random(0, t)
        h.update(v.rewards().tobytes())
        h.update(v.dones().tobytes())
        for k in range(cfg.n_specs):
            o, r = v.gather(k)
            h.update(o.tobytes())
            h.update(r.tobytes())
    for e in range(n):
        h.update(v.view(e).book(0).tobytes())
        h.update(v.view(e).book(1).tobytes())
    v.synchronize()
    st = v.allreduce_episode_stats(0)
    h.update(b"".join(bytes(x) for x in st))
    print("driver ok", kind, v.messages_processed(), h.hexdigest())


if __name__ == "__main__":
    if len(sys.argv) > 2:
        E.LIB_PATH = sys.argv[2]  # test harness only: bind the checked build
    main(sys.argv[1])
