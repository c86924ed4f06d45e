"""The Lo-slice fusion of the split update (csrc/update2.cu slice_lo_columns:
solves write the Ozaki Lo slices of a later INT8 contraction with the slicing
kernels' arithmetic -- in the same iteration, whose contraction then skips
its slicing kernel, and carried into the next iteration's mode-0
contraction, sliced again only after the plan moved columns) must leave a
sweep bitwise identical (CALS_FUSE_LO=0 turns it off): a Y-tree cube and an
EEM-shaped converging refill sweep whose plans move columns.  The same two
sweeps pin the deferred split reduction (solve kernels summing split-K
partials) against split_reduce_kernel."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(fuse, **extra):
    env = dict(os.environ, CALS_FUSE_LO=fuse, **extra)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_fuse_worker.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_lo_fusion_bitwise():
    off, on = _run("0"), _run("1")
    assert off["eem_iters"] == on["eem_iters"]
    assert off["cube"] == on["cube"]
    assert off["eem"] == on["eem"]


@pytest.mark.parametrize("path", ["int8", "dmma"])
def test_deferred_split_reduce_bitwise(path):
    """Non-last modes hand their split-K partials to the solve kernel, which
    sums them in split order (CALS_DEFER_REDUCE=0 keeps split_reduce_kernel):
    the same bits on the INT8 and the DMMA contraction paths."""
    extra = {} if path == "int8" else {"CALS_MTTKRP": "dmma"}
    off = _run("1", CALS_DEFER_REDUCE="0", **extra)
    on = _run("1", CALS_DEFER_REDUCE="1", **extra)
    assert off == on
