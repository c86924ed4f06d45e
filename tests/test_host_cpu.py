"""Host-side API pieces that need no GPU: CALS1 files, run configuration,
multi-matrix bookkeeping, variant table, flop model, CLI validation paths.
Mirrors the reference's test_io / test_multimatrix / test_cli cases."""
import json

import numpy as np
import pytest
from click.testing import CliRunner

import paper_2010_04678_b200 as cals
from paper_2010_04678_b200 import io as cio
from paper_2010_04678_b200.cli import main as cli_main


def test_tensor_file_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(70)
    t = cals.DenseTensor((5, 4, 3), rng.standard_normal(60))
    cio.write_tensor(tmp_path / "t.cals", t)
    back = cio.read_tensor(tmp_path / "t.cals")
    assert back.dims == t.dims and np.array_equal(back.data, t.data)
    (tmp_path / "bad.cals").write_bytes(b"NOPE!")
    with pytest.raises(cio.TensorFileError):
        cio.read_tensor(tmp_path / "bad.cals")
    good = (tmp_path / "t.cals").read_bytes()
    (tmp_path / "trunc.cals").write_bytes(good[:-8])
    with pytest.raises(cio.TensorFileError, match="payload"):
        cio.read_tensor(tmp_path / "trunc.cals")
    (tmp_path / "long.cals").write_bytes(good + b"\0" * 8)
    with pytest.raises(cio.TensorFileError, match="payload"):
        cio.read_tensor(tmp_path / "long.cals")
    m = np.asfortranarray(rng.standard_normal((6, 3)))
    cio.write_matrix(tmp_path / "m.cals", m)
    assert np.array_equal(cio.read_matrix(tmp_path / "m.cals"), m)


def test_csv_import(tmp_path):
    p = tmp_path / "t.csv"
    p.write_text("# comment\n0,0,0,1.5\n1,2,0,-2\n\n")
    t = cio.read_tensor_csv(p, (2, 3, 1))
    assert t.as_ndarray()[0, 0, 0] == 1.5 and t.as_ndarray()[1, 2, 0] == -2.0
    p.write_text("5,0,0,1\n")
    with pytest.raises(cio.TensorFileError):
        cio.read_tensor_csv(p, (2, 3, 1))


def test_parse_ranks_and_runconfig():
    assert cio.parse_ranks("3") == [3]
    assert cio.parse_ranks("1..4") == [1, 2, 3, 4]
    assert cio.parse_ranks("2,5,5") == [2, 5, 5]
    for bad in ("0", "5..2", ""):
        with pytest.raises(ValueError):
            cio.parse_ranks(bad)
    cfg = cio.RunConfig(ranks=[1, 2], r_star=2)
    cfg.validate()
    assert cfg.to_dict()["ranks"] == [1, 2]
    for kw in ({"tol": 0.0}, {"r_star": 1}, {"mode": "x"}, {"per_rank": 0}, {"threads": 0},
               {"line_search_alpha": 0.5}):
        with pytest.raises(ValueError):
            cio.RunConfig(ranks=[1, 2], **kw).validate()


def test_multimatrix_semantics():
    def mk(rank, seed, i):
        return cals.Model.random((4, 3), rank, np.random.default_rng(seed), id=i)

    mms = cals.MultiMatrixSet((4, 3), capacity=10)
    assert mms.try_insert(mk(3, 0, "a")) and mms.try_insert(mk(4, 1, "b"))
    assert not mms.try_insert(mk(5, 2, "c"))
    assert mms.active_width == 7
    with pytest.raises(cals.CapacityError):
        mms.try_insert(mk(11, 3, "big"))
    with pytest.raises(ValueError):
        mms.try_insert(mk(2, 4, "a"))
    removed = mms.remove("a")
    assert [f.shape for f in removed] == [(4, 3), (3, 3)]
    assert not mms.per_mode[0].is_compact()
    with pytest.raises(ValueError):
        mms.per_mode[0].packed_view()
    assert mms.compress() == 2 and mms.per_mode[0].is_compact()
    with pytest.raises(KeyError):
        mms.remove("nope")


def test_variants_and_flops():
    V = cals.MttkrpVariant
    assert cals.select_variant((300, 300, 300), 1, 1000) is V.MIDDLE_MODE_SLICE_GEMM
    assert cals.select_variant((4, 4, 4, 4), 2, 2) is V.EXPLICIT_KRP_GEMM
    assert cals.mttkrp_flops((300, 300, 300), 1) == 54_000_000
    assert cals.mttkrp_flops((10, 10, 10), 0) == 0
    from paper_2010_04678_b200.mttkrp import validate_variant

    for bad in [(V.FIRST_MODE_GEMM, 3, 1), (V.LAST_MODE_GEMM, 3, 0),
                (V.MIDDLE_MODE_SLICE_GEMM, 4, 1)]:
        with pytest.raises(ValueError):
            validate_variant(*bad)


def test_model_and_tensor_validation():
    with pytest.raises(ValueError):
        cals.DenseTensor((4,), np.zeros(4))
    with pytest.raises(ValueError):
        cals.DenseTensor((2, 2), np.ones(4), sqnorm=5.0)
    t = cals.DenseTensor((2, 2), np.ones(4), sqnorm=4.0)
    with pytest.raises(ValueError):
        t.data[0] = 1.0
    with pytest.raises(ValueError):
        cals.Model(id="x", rank=0, factors=[])
    with pytest.raises(ValueError):
        cals.Model(id="x", rank=1, factors=[np.array([[np.nan]])])
    assert cals.unfold(cals.DenseTensor((2, 2, 2), np.arange(1.0, 9.0)), 0).tolist() == \
        [[1, 3, 5, 7], [2, 4, 6, 8]]
    assert cals.khatri_rao(np.array([[1.0], [2.0]]),
                           np.array([[3.0], [4.0], [5.0]])).ravel().tolist() == [3, 4, 5, 6, 8, 10]
    g = cals.gramian(np.random.default_rng(0).standard_normal((7, 4)))
    assert np.array_equal(g, g.T)


def test_fit_and_error_formulas():
    assert cals.fit_from_error(0.0, 4.0) == 1.0
    assert cals.fit_from_error(1.0, 4.0) == 0.5
    with pytest.raises(ValueError):
        cals.fit_from_error(1.0, 0.0)
    with pytest.raises(ValueError):
        cals.fit_from_error(-1.0, 1.0)


def test_cli_gen_and_validation(tmp_path):
    r = CliRunner()
    out = tmp_path / "t.cals"
    res = r.invoke(cli_main, ["gen", "--dims", "5,4,3", "--rank", "2", "--noise", "0.1",
                              "--out", str(out)])
    assert res.exit_code == 0, res.output
    assert np.array_equal(cio.read_tensor(out).data,
                          cio.generate_synthetic((5, 4, 3), 2, 0.1, 0).data)
    res = r.invoke(cli_main, ["gen", "--dims", "5", "--rank", "2", "--out", str(out)])
    assert res.exit_code == 2
    res = r.invoke(cli_main, ["decompose", "--tensor", str(out), "--ranks", "1..3",
                              "--r-star", "2", "--out", str(tmp_path / "r.json")])
    assert res.exit_code == 2
    err = json.loads(res.output.strip().splitlines()[-1])
    assert err["error"]["code"] == "config"
