"""compute-sanitizer is closed on the B200 pool, so out-of-bounds / invariant violations are
hunted with a library built with device asserts (-DLB_CHECKS: probe positions < m, table slots in
range, queue bounds, document offsets) running the collision-heavy parity cases."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_cases_under_device_asserts():
    from paper_2411_04257_b200 import build
    build.build(checked=True)
    env = dict(os.environ, LSHBLOOM_LIB=build.LIB_CHECKED)
    sel = ("dense or edge or sub_batch or shapes or single_document or malformed or many_chunks or both_minhash"
           " or partition")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel,
                          os.path.join(ROOT, "tests", "test_gpu_parity.py")],
                         env=env, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]


def test_blocked_cases_under_device_asserts():
    from paper_2411_04257_b200 import build
    build.build(checked=True)
    env = dict(os.environ, LSHBLOOM_LIB=build.LIB_CHECKED)
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", "dense or sub_batch",
                          os.path.join(ROOT, "tests", "test_gpu_blocked.py")],
                         env=env, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
