"""GPU parity of the Ozaki-sliced INT8 tensor-core MTTKRP (csrc/ozaki.cuh)
against the FP64 reference contraction, next to the DMMA kernel.

The kernel choice is fixed per process (CALS_MTTKRP), so each path runs in a
subprocess (tests/_ozaki_worker.py).  Bars: the reference's own MTTKRP
tolerance (test_mttkrp.py:64-78, 1e-12 relative Frobenius) on normal,
uniform, wide-dynamic-range (rows 2^-60..2^60) and zero-column inputs; the
bitwise position-independence / duplicate-column properties the fused
kernels guarantee (test_mttkrp.py:145-187); and the north_star factor bar
(1e-9 after 5 iterations) for a full CALS sweep with converged-slot refill.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(path):
    env = dict(os.environ, CALS_MTTKRP=path)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_ozaki_worker.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module", params=["ozaki", "dmma"])
def result(request):
    return request.param, _run(request.param)


def test_mttkrp_parity(result):
    path, out = result
    for c in out["cases"]:
        assert max(c["rel"]) <= 1e-12, (path, c)


def test_bitwise_properties(result):
    path, out = result
    assert out["position_independent"], path
    assert out["duplicates_equal"], path


def test_sweep_factors(result):
    path, out = result
    assert out["sweep_factor_rel"] <= 1e-9, (path, out["sweep_factor_rel"])
