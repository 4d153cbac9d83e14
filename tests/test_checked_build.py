"""The checked build (libmlob_checked.so = the product sources with
-DMLOB_CHECKS=1: device-side bounds and invariant assertions on the hand-off
buffers, book rows, fill log and the mbarrier waits, trapping on failure;
and -DMLOB_PREFIX_WALK=1: crossing orders walk each price level by a warp
prefix sum over the resting quantities, mlob_step.cuh walk_level_t)
runs a register-book and a shared-memory-book workload — act / book /
outcome / reset / stats kernels, TMA bulk copies, evictions, auto-reset —
without a trap, and produces outputs bit-identical to the product library.
This replaces compute-sanitizer, which is closed on the GPU pool."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2511_02136_b200")


def _run(kind, lib=None):
    cmd = [sys.executable, os.path.join(ROOT, "tests", "sanitize_driver.py"), kind] + ([lib] if lib else [])
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("driver ok")]
    assert line, p.stdout[-2000:]
    return line[0]


def test_checked_library_built():
    assert os.path.exists(os.path.join(LIBDIR, "libmlob_checked.so")), "make -C paper_2511_02136_b200"


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["register", "smem"])
def test_checked_build_matches_product(kind):
    checked = _run(kind, os.path.join(LIBDIR, "libmlob_checked.so"))
    product = _run(kind)
    assert checked == product
