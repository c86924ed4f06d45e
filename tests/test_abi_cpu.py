"""CPU-side checks of the boundary: the library loads and exports exactly the
symbols include/cals_b200.h declares; the product fails loudly without a GPU."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "cals_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(cals_\w+)\(", src, re.M)))


def test_header_matches_binding():
    from paper_2010_04678_b200 import _native

    assert _declared() == sorted(_native.exported_symbols())


def test_library_exports_every_symbol():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2010_04678_b200 import _native

    lib = _native.load(require_cuda=False)
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.cals_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    import paper_2010_04678_b200 as cals
    from paper_2010_04678_b200._native import NativeUnavailable

    t = cals.DenseTensor((3, 3, 3), np.ones(27))
    m = cals.Model.random((3, 3, 3), 2, 0, id="x")
    with pytest.raises(NativeUnavailable):
        cals.run(t, [m], cals.ConvergenceConfig(max_iterations=2))
    with pytest.raises(NativeUnavailable):
        cals.mttkrp(t, m.factors, 0)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2010_04678_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            assert "oracle" not in re.sub(r'"""[\s\S]*?"""|#.*', "", open(os.path.join(pkg, f)).read()), f
