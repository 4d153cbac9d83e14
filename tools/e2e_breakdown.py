"""Diagnostic: time the parts of one e2e step (set_actions, step, rewards, dones, gather)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_2511_02136_b200 import abi, env as E
from paper_2511_02136_b200.env import DeviceStore, HostStore, MarketVecEnv

n_total, cfg, synth, label = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "E")
hs = HostStore.synth(synth, 0)
store = DeviceStore(hs, 0)
del hs
venv = MarketVecEnv(store, cfg, seed=0, n_envs=n_total, n_envs_global=n_total, env_index_base=0, device=0)
venv.reset_all()
A = venv.n_agents
L = E.lib()
rng = np.random.default_rng(1234)
ar = np.array([abi.action_arity(cfg.specs[s]) for s in abi.flat_specs(cfg)])
acts = torch.from_numpy((rng.integers(0, 1 << 30, size=(n_total, A)) % ar).astype(np.int32)).pin_memory()
obs = [torch.empty((venv.n_streams(t), venv.obs_dim(t)), dtype=torch.float64).pin_memory() for t in range(cfg.n_specs)]
rew = torch.empty((n_total, A), dtype=torch.float64).pin_memory()
dn = torch.empty((n_total, A), dtype=torch.uint8).pin_memory()
rs = torch.empty(max(venv.n_streams(t) for t in range(cfg.n_specs)), dtype=torch.uint8).pin_memory()
parts = {"set_actions": lambda: L.mlob_venv_set_actions(venv.h, acts.data_ptr(), 0),
         "step": lambda: (venv.step(), venv.synchronize()),
         "rewards": lambda: L.mlob_venv_rewards(venv.h, rew.data_ptr()),
         "dones": lambda: L.mlob_venv_dones(venv.h, dn.data_ptr())}
for t in range(cfg.n_specs):
    parts[f"gather{t}_obs"] = (lambda t=t: L.mlob_venv_gather(venv.h, t, obs[t].data_ptr(), None))
    parts[f"gather{t}_resets"] = (lambda t=t: L.mlob_venv_gather(venv.h, t, None, rs.data_ptr()))
tot = {k: 0.0 for k in parts}
for it in range(8):
    for k, f in parts.items():
        torch.cuda.synchronize()
        t0 = time.perf_counter(); f(); torch.cuda.synchronize()
        if it >= 3: tot[k] += time.perf_counter() - t0
for k, v in tot.items():
    print(f"{k:16s} {v / 5 * 1e3:8.2f} ms")
print("obs bytes", sum(o.numel() * 8 for o in obs), "rew", rew.numel() * 8)
rsb = [torch.empty(venv.n_streams(t), dtype=torch.uint8).pin_memory() for t in range(cfg.n_specs)]
import os
for ch in ["1", "2", "4", "8", "16", ""]:
    if ch:
        os.environ["MLOB_IO_CHUNKS"] = ch
    else:
        os.environ.pop("MLOB_IO_CHUNKS", None)
    f = lambda: venv.step_io(actions=acts, rewards=rew, dones=dn, obs=obs, resets=rsb)  # noqa: E731
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        f()
    print(f"step_io chunks={ch or 'default'} {(time.perf_counter() - t0) / 5 * 1e3:8.2f} ms")
