"""Compiled C++ callers of the product (tests/cpp, built by build() /
`make -C tests/cpp`): the reference's own collect_rollout / train_loop
templates (rollout.hpp:41-145) instantiated over the C++ drop-in
CudaMarketVecEnv (include/mlob/vec_env.hpp) against MarketVecEnv, and the
NCCL all-reduce of the episode statistics through the C ABI."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin")


def _run(name, *args):
    exe = os.path.join(BIN, name)
    assert os.path.exists(exe), f"{exe} missing: run `make -C tests/cpp` (needs /root/reference)"
    p = subprocess.run([exe, *map(str, args)], capture_output=True, text=True, timeout=900)
    print(p.stdout[-4000:], p.stderr[-2000:])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert "OK" in p.stdout
    return p.stdout


def test_cpp_binaries_link_the_product():
    """The compiled callers resolve libmlob.so from the tree (no GPU needed)."""
    for name in ("vec_env_rollout", "nccl_stats"):
        exe = os.path.join(BIN, name)
        if not os.path.exists(exe):
            pytest.skip("tests/cpp not built")
        out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
        assert "paper_2511_02136_b200/libmlob.so" in out, out


@pytest.mark.gpu
def test_reference_collect_rollout_and_train_loop_over_cuda_vec_env():
    _run("vec_env_rollout", 96)


@pytest.mark.gpu
def test_nccl_allreduce_episode_stats_from_cpp():
    _run("nccl_stats")
