"""Golden fixture for the SEQUENTIAL / PARALLEL failure semantics, from the
REAL reference.  TEST INFRASTRUCTURE ONLY (imports /root/reference/pkg/src;
run in the build container):

    python oracle/make_golden_seq.py

``run_fail_seq.npz``: the inputs of ``fail_inputs.npz`` (one instance with a
NaN planted in its last factor, one healthy) run through
``cals.run(mode=SEQUENTIAL)`` -- the failed instance comes back from
``_fit_or_fail`` (driver.py:148-160) with its starting factors, 0 iterations,
error nan -- and the healthy one as usual.  Also records that
``run_single_als`` raises ValueError for the failing instance and leaves the
starting model's status alone.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def main() -> None:
    sys.path.insert(0, REF)
    from cals.als import ConvergenceConfig, run_single_als
    from cals.driver import ExecutionMode, run
    from cals.model import Model
    from cals.tensor import DenseTensor

    f = np.load(os.path.join(GOLDEN, "fail_inputs.npz"))
    t = DenseTensor((4, 4, 3), f["data"])

    def models():
        good = Model(id="good", rank=2, factors=[f[f"good_f{n}"] for n in range(3)])
        bad = Model(id="bad", rank=2, factors=[f[f"good_f{n}"] for n in range(3)])
        for n in range(3):
            bad.factors[n][...] = f[f"bad_f{n}"]
        return bad, good

    d = {}
    cfg = ConvergenceConfig(tol=0.0, max_iterations=3)
    for mode in (ExecutionMode.SEQUENTIAL, ExecutionMode.PARALLEL):
        bad, good = models()
        with np.errstate(invalid="ignore"):
            out = run(t, [bad, good], cfg, mode=mode)
        key = mode.value
        d[f"{key}_order"] = np.array([m.id for m in out])
        d[f"{key}_status"] = np.array([m.status.value for m in out])
        d[f"{key}_iterations"] = np.array([m.iterations_done for m in out])
        d[f"{key}_error"] = np.array([m.error for m in out])
        d[f"{key}_fit"] = np.array([m.fit for m in out])
        d[f"{key}_input_status"] = np.array([bad.status.value, good.status.value])
        for m in out:
            for n, a in enumerate(m.factors):
                d[f"{key}_{m.id}_f{n}"] = a
    bad, _ = models()
    try:
        with np.errstate(invalid="ignore"):
            run_single_als(t, bad, cfg)
        raised = ""
    except Exception as exc:  # noqa: BLE001 -- record the type
        raised = type(exc).__name__
    d["single_raises"] = np.array(raised)
    d["single_input_status"] = np.array(bad.status.value)
    np.savez(os.path.join(GOLDEN, "run_fail_seq.npz"), **d)
    print({k: v for k, v in d.items() if "_f" not in k})


if __name__ == "__main__":
    main()
