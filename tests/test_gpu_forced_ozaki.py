"""The GPU parity suites re-run with the INT8 tensor-core MTTKRP forced for
every view (CALS_MTTKRP=ozaki; the kernel choice is fixed per process, so in
a subprocess): golden vectors, oracle sweeps, line search, NNLS, refill,
sharded driver and edge cases must all hold on that path too, not only on
the shapes the heuristic sends to it."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SUITES = ["test_gpu_mttkrp.py", "test_gpu_driver.py", "test_gpu_nnls.py", "test_gpu_sharded.py",
          "test_gpu_edge.py"]


def test_suites_with_forced_int8_mttkrp():
    env = dict(os.environ, CALS_MTTKRP="ozaki")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        *[os.path.join(HERE, f) for f in SUITES]],
                       env=env, capture_output=True, text=True, timeout=1200, cwd=HERE)
    assert r.returncode == 0, (r.stdout[-4000:], r.stderr[-2000:])


def test_int8_envelope_without_range_guard():
    """The accuracy-envelope suite with the dynamic-range guard off: every
    view of the spiky / log-uniform / EEM-like data runs on INT8 and must
    still meet the MTTKRP (1e-12) and sweep (1e-9) bars."""
    env = dict(os.environ, CALS_OZ_RANGE_GUARD="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_gpu_ozaki_envelope.py")],
                       env=env, capture_output=True, text=True, timeout=1200, cwd=HERE)
    assert r.returncode == 0, (r.stdout[-4000:], r.stderr[-2000:])
