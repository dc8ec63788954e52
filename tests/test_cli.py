"""CLI / Matrix Market / stencil families.

CPU: the reference CLI's problem generators reproduce the reference's own
arrays bitwise (tests/golden/small_systems.npz, made by running the
reference); ``acr export`` writes the same bytes as the reference's
``acr export`` (tests/golden/mmio_*, made by make_golden.py mmio); Matrix
Market round trips; argument errors exit 1 like the reference
(``cli.py:374-404``).  GPU: ``acr solve`` on the device, from a problem and
from an exported file."""

import filecmp
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_npz
from paper_1604_00617_b200 import cli, mmio
from paper_1604_00617_b200 import stencils as S

BANDS = ("D_sub", "D_diag", "D_sup", "E", "F", "rhs")


@pytest.mark.parametrize("name,build", [
    ("poisson16", lambda: S.poisson2d(S.Grid2D(16))),
    ("checker16", lambda: S.poisson2d(S.Grid2D(16), S.checkerboard_kappa())),
    ("helm16_k1", lambda: S.helmholtz2d(S.Grid2D(16), 1.0)),
    ("helm16_k2", lambda: S.helmholtz2d(S.Grid2D(16), 2.0)),
    ("conv16_a100", lambda: S.convdiff2d(S.Grid2D(16), 100.0)),
    ("helm63_k6pi", lambda: S.helmholtz2d(S.Grid2D(63), 6.0 * np.pi)),
    ("conv63_a1e4", lambda: S.convdiff2d(S.Grid2D(63), 1e4)),
    ("poisson128_e6", lambda: S.poisson2d(S.Grid2D(128))),
])
def test_stencils_bitwise_reference(small_golden, name, build):
    s = build()
    for a in BANDS:
        np.testing.assert_array_equal(getattr(s, a), small_golden[f"{name}/{a}"], err_msg=a)


@pytest.mark.parametrize("argv,stem", [
    (["--problem", "poisson", "--n", "6", "--kappa", "checkerboard:100:2"], "mmio_poisson6"),
    (["--problem", "convdiff", "--n", "5", "--alpha", "30"], "mmio_convdiff5"),
])
def test_export_bytes_match_reference(tmp_path, argv, stem):
    assert cli.main(["export", *argv, "--out", str(tmp_path / stem)]) == 0
    for ext in (".mtx", ".rhs.txt"):
        assert filecmp.cmp(tmp_path / (stem + ext), os.path.join(GOLDEN, stem + ext),
                           shallow=False), ext


def test_matrix_market_round_trip(tmp_path):
    s = S.convdiff2d(S.Grid2D(7), 50.0)
    p = tmp_path / "a.mtx"
    mmio.write_matrix_market(p, S.assemble_full(s), comment="x\ny")
    A = mmio.read_matrix_market(p)
    np.testing.assert_array_equal(A.toarray(), S.assemble_full(s).toarray())
    mmio.write_vector(tmp_path / "f.txt", s.rhs)
    f = mmio.read_vector(tmp_path / "f.txt")
    np.testing.assert_array_equal(f, s.rhs)
    t = mmio.coo_to_system(A, 7, f)
    for a in BANDS:
        np.testing.assert_array_equal(getattr(t, a), getattr(s, a), err_msg=a)


def test_coo_to_system_rejects_foreign_pattern():
    import scipy.sparse as sp
    A = sp.coo_matrix(np.ones((8, 8)))
    with pytest.raises(ValueError, match="outside the block tridiagonal pattern"):
        mmio.coo_to_system(A, 4, np.zeros(8))


def test_export_baseline_config_round_trip(tmp_path):
    from paper_1604_00617_b200 import problems as P
    assert cli.main(["export", "--config", "cfg1", "--out", str(tmp_path / "c1")]) == 0
    t = mmio.coo_to_system(mmio.read_matrix_market(tmp_path / "c1.mtx"), 64,
                           mmio.read_vector(tmp_path / "c1.rhs.txt"))
    s = P.make_config("cfg1")
    for a in BANDS:
        np.testing.assert_array_equal(getattr(t, a), getattr(s, a), err_msg=a)


@pytest.mark.parametrize("argv", [
    ["solve", "--problem", "helmholtz", "--n", "8"],                 # needs --k
    ["solve", "--problem", "poisson", "--n", "8", "--alpha", "1"],   # foreign parameter
    ["solve", "--problem", "poisson", "--n", "1"],
    ["solve", "--problem", "poisson", "--n", "8", "--eps", "0"],
    ["solve", "--problem", "poisson", "--n", "8", "--device", "cpu"],
    ["solve", "--problem", "poisson", "--n", "8", "--config", "cfg1"],
    ["solve", "--input", "x.mtx"],
    ["sweep", "--problem", "poisson", "--n", "8", "--axis", "eps", "--values", "1e-4,1e-8"],
    ["export", "--problem", "poisson", "--n", "8"],
    ["solve", "--problem", "poisson", "--n", "8", "--kappa", "wobbly:3"],
])
def test_configuration_errors_exit_1(argv):
    assert cli.main(argv) == 1


@pytest.mark.gpu
def test_cli_solve_on_device(tmp_path, small_golden):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "r.json"
    rc = cli.main(["solve", "--problem", "poisson", "--n", "16", "--leaf-size", "8",
                   "--eps", "1e-12", "--out", str(out)])
    assert rc == 0
    rep = json.loads(out.read_text())
    assert rep["config"]["device"] == "cuda"
    assert rep["report"]["residual"] <= 2 * float(small_golden["poisson16/residual"]) + 1e-15
    assert rep["report"]["storage_bytes"] == int(small_golden["poisson16/storage_bytes"])
    # the same system through Matrix Market export -> --input
    stem = tmp_path / "p16"
    assert cli.main(["export", "--problem", "poisson", "--n", "16", "--out", str(stem)]) == 0
    out2 = tmp_path / "r2.json"
    assert cli.main(["solve", "--input", str(stem) + ".mtx", "--rhs", str(stem) + ".rhs.txt",
                     "--block-dim", "16", "--leaf-size", "8", "--eps", "1e-12",
                     "--out", str(out2)]) == 0
    rep2 = json.loads(out2.read_text())
    assert rep2["report"]["residual"] == rep["report"]["residual"]
    assert rep2["report"]["per_level_ranks"] == rep["report"]["per_level_ranks"]
    # residual above the threshold -> exit 2 (reference cli.py:201)
    assert cli.main(["solve", "--problem", "poisson", "--n", "16", "--leaf-size", "8",
                     "--eps", "1e-2", "--threshold", "1e-12", "--out",
                     str(tmp_path / "r3.json")]) == 2


@pytest.mark.gpu
def test_cli_verify_and_sweep_on_device(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert cli.main(["verify", "--problem", "convdiff", "--n", "16", "--alpha", "100",
                     "--leaf-size", "8", "--eps", "1e-12"]) == 0
    out = tmp_path / "s.csv"
    assert cli.main(["sweep", "--problem", "poisson", "--n", "8", "--axis", "n",
                     "--values", "16,32", "--leaf-size", "8", "--out", str(out)]) == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0].split(",") == cli.CSV_COLUMNS and len(lines) == 3
    assert os.path.exists(str(tmp_path / "s_fit.json"))
