"""Subprocess body for test_gpu_slicing.py (the X-slicing kernel is chosen
once per process, CALS_OZ_ROWS_TILE): SHA-256 digests of fused INT8 MTTKRPs
of every mode on shapes whose views slice with m contiguous and with p
contiguous, plus odd extents, a wide-range and a non-finite tensor."""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2010_04678_b200 as cals  # noqa: E402


def main():
    rng = np.random.default_rng(21)
    out = {}
    cases = [((200, 200, 200), 96, "normal"), ((150, 141, 133), 70, "normal"),
             ((250, 251, 21), 40, "normal"), ((160, 130, 150), 33, "range"),
             ((140, 136, 132), 20, "inf")]
    for dims, width, kind in cases:
        arr = rng.standard_normal(dims)
        if kind == "range":
            arr *= np.exp2(rng.integers(-60, 60, size=(dims[0], 1, 1)))
        if kind == "inf":
            arr[3, 4, 5] = np.inf
        fac = [np.asfortranarray(rng.standard_normal((d, width))) for d in dims]
        t = cals.DenseTensor.from_array(arr)
        ws = cals.MttkrpWorkspace(dims, width)
        h = hashlib.sha256()
        for n in range(3):
            h.update(np.ascontiguousarray(np.array(cals.mttkrp(t, fac, n, ws=ws))).tobytes())
        out[f"{dims}/{kind}"] = h.hexdigest()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
