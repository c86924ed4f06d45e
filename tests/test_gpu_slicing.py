"""The single-pass X-slicing kernel (csrc/ozaki.cu oz_slice_rows_tile_kernel)
must build exactly the slices, exponents and range census of the two-pass
kernel: fused INT8 MTTKRPs bitwise identical under CALS_OZ_ROWS_TILE=0 / 1
(views with m contiguous and with p contiguous, odd extents, rows spanning
2^+-60, a non-finite tensor that falls back to DMMA)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tile):
    env = dict(os.environ, CALS_MTTKRP="ozaki", CALS_OZ_ROWS_TILE=tile)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_slice_worker.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_single_pass_slicing_bitwise():
    assert _run("0") == _run("1")
