"""Diagnostic: per-phase clock64 deltas of the step kernel (MLOB_PHASE_TIMING build)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MLOB_TIMING"] = "1"
from paper_2511_02136_b200 import abi, env as E
from bench import workload
mps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
WL = os.environ.get("WL", "C")
n, cfg, synth, _ = workload(WL)
if WL != "D":
    cfg.messages_per_step = mps; synth.n_messages = (n + 64) * mps; synth.state_sample_every = mps
hs = E.HostStore.synth(synth, 0)
if WL == "D":
    hs.trim_front(16 * 6400)
    n = int(os.environ.get("ENVS", "65536"))
dev = E.DeviceStore(hs, 0)
v = E.MarketVecEnv(dev, cfg, seed=0, n_envs=n)
v.reset_all()
L = E.lib(); L.mlob_venv_read_timing.argtypes = [C.c_void_p, C.c_void_p]
for s in range(8):
    v.step_random(0, s)
v.synchronize()
t = np.zeros((n, 16), dtype=np.int64)
E._check(L.mlob_venv_read_timing(v.h, t.ctypes.data))
names = ["hdr+agents load", "convert+shuffle", "book load", "msg loop", "rebuild", "snapshot", "store book", "outcomes", "store state"]
d = np.diff(t[:, :10], axis=1)
print(f"mps={mps}  total cycles/env-step (mean) {np.mean(t[:,9]-t[:,0]):.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:26s} mean {d[:, i].mean():9.0f}  p50 {np.median(d[:, i]):9.0f}")
# barrier share: within each block (consecutive warps), the barrier releases at
# about the latest pre-barrier stamp (clock64 is per SM, so comparable in-block)
W = int(os.environ.get("MLOB_WPB", "24"))
nb = n // W
pre = t[: nb * W, 7].reshape(nb, W)
rel = pre.max(axis=1, keepdims=True)
wait = (rel - pre).mean()
print(f"  barrier wait (est.)        mean {wait:9.0f}   outcomes after barrier {(t[:nb*W, 8] - np.repeat(rel, W, axis=1).reshape(-1)).mean():9.0f}")
