"""Command-line harness (paper_1908_00204_b200/cli.py), modelled on the
reference's tests/test_cli.py: checksums agree across paths and with the
reference's golden LU values, RunReport JSON/CSV schema, exit codes 1/2/3,
solve round trip.  Matrix files are written from the golden fixtures."""

import hashlib
import json

import numpy as np
import pytest

import paper_1908_00204_b200 as glu
import paper_1908_00204_b200.cli as cli

from conftest import load_golden


def _write_mtx(path, g, symmetric=False):
    n = int(g["n"])
    cp, ri, v = g["a_col_ptr"], g["a_row_idx"], g["a_values"]
    cols = np.repeat(np.arange(n), np.diff(cp))
    lines = [f"{r + 1} {c + 1} {float(x)!r}" for r, c, x in zip(ri, cols, v)]
    kind = "symmetric" if symmetric else "general"
    path.write_text(f"%%MatrixMarket matrix coordinate real {kind}\n% written by test_cli\n"
                    f"{n} {n} {len(lines)}\n" + "\n".join(lines) + "\n")
    return str(path)


@pytest.fixture
def conflict8(tmp_path):
    return _write_mtx(tmp_path / "conflict8.mtx", load_golden("conflict8"))


@pytest.fixture
def diag5(tmp_path):
    return _write_mtx(tmp_path / "diag5.mtx", load_golden("diag5"))


def checksum_of(out):
    for line in out.splitlines():
        if line.startswith("checksum "):
            return line.split()[1]
    raise AssertionError(f"no checksum line in {out!r}")


# ---- CPU: reader and usage errors (no factorization reached) ----

def test_matrix_market_roundtrip(conflict8):
    g = load_golden("conflict8")
    with open(conflict8) as fh:
        a = glu.to_csc(glu.load_matrix_market(fh))
    assert np.array_equal(a.col_ptr, g["a_col_ptr"])
    assert np.array_equal(a.row_idx, g["a_row_idx"])
    assert np.array_equal(a.values, g["a_values"])


def test_matrix_market_symmetric_and_integer(tmp_path):
    p = tmp_path / "s.mtx"
    p.write_text("%%MatrixMarket matrix coordinate integer symmetric\n3 3 3\n1 1 4\n3 1 2\n3 3 5\n")
    with open(p) as fh:
        a = glu.to_csc(glu.load_matrix_market(fh))
    assert np.array_equal(a.to_dense(), [[4, 0, 2], [0, 0, 0], [2, 0, 5]])


@pytest.mark.parametrize("text", [
    "not a matrix\n",
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n",
])
def test_matrix_market_rejects(tmp_path, text):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with open(p) as fh, pytest.raises(glu.MatrixFormatError):
        glu.load_matrix_market(fh)
    assert cli.main(["factor", str(p)]) == cli.EXIT_USAGE


def test_exit_usage_cases(tmp_path, conflict8, diag5, capsys):
    assert cli.main(["factor", str(tmp_path / "missing.mtx")]) == cli.EXIT_USAGE
    assert cli.main(["factor", conflict8, "--sequential", "left", "--parallel"]) == cli.EXIT_USAGE
    assert cli.main(["factor", conflict8, "--deps", "bogus"]) == cli.EXIT_USAGE
    assert cli.main(["factor", conflict8, "--deps", "upward", "--parallel"]) == cli.EXIT_USAGE
    assert cli.main(["factor", conflict8, "--precision", "half"]) == cli.EXIT_USAGE
    assert cli.main([]) == cli.EXIT_USAGE
    pr = tmp_path / "pr.txt"
    pr.write_text("1\n0\n2\n3\n4\n")
    assert cli.main(["factor", diag5, "--perm", str(pr), "--row-perm", str(pr),
                     "--col-perm", str(pr)]) == cli.EXIT_USAGE
    assert cli.main(["factor", diag5, "--row-perm", str(pr)]) == cli.EXIT_USAGE
    short = tmp_path / "short.txt"
    short.write_text("0\n1\n")
    assert cli.main(["factor", diag5, "--perm", str(short)]) == cli.EXIT_USAGE
    rhs = tmp_path / "b.txt"
    rhs.write_text("1\n2\n")
    assert cli.main(["solve", diag5, str(rhs)]) == cli.EXIT_USAGE
    assert "error:" in capsys.readouterr().err


def test_exit_hazard_with_detect_races(conflict8, capsys):
    # the hazard check is host analysis and fires before any device work
    code = cli.main(["factor", conflict8, "--deps", "upward", "--parallel",
                     "--allow-unsafe", "--detect-races"])
    assert code == cli.EXIT_HAZARD
    assert "hazard" in capsys.readouterr().err.lower()


# ---- GPU: the factorization and solve run on the B200 ----

@pytest.mark.gpu
def test_factor_default_parallel(conflict8, capsys):
    assert cli.main(["factor", conflict8, "--check-residual"]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "n=8 nz=19 nnz=19" in out
    assert "deps=relaxed levels=4" in out
    assert "modes: Stream=4" in out
    assert float(out.split("residual ")[1].split()[0]) <= 1e-12
    # the reference's golden LU values (contract A) hash to the same line
    golden = hashlib.sha256(load_golden("conflict8")["lu_a"].tobytes()).hexdigest()[:16]
    assert checksum_of(out) == golden == "cb2c3e22567ad657"


@pytest.mark.gpu
def test_factor_paths_agree_bitwise(conflict8, capsys):
    sums = []
    for flags in (["--sequential", "left"], ["--sequential", "right"],
                  ["--parallel", "--threads", "2"], ["--parallel", "--atomic"]):
        assert cli.main(["factor", conflict8] + flags) == cli.EXIT_OK
        sums.append(checksum_of(capsys.readouterr().out))
    assert set(sums) == {"cb2c3e22567ad657"}


@pytest.mark.gpu
def test_factor_stats_out(tmp_path, conflict8, capsys):
    path = tmp_path / "report.json"
    assert cli.main(["factor", conflict8, "--check-residual",
                     "--stats-out", str(path)]) == cli.EXIT_OK
    d = json.loads(path.read_text())
    assert (d["n"], d["nz"], d["nnz"], d["deps_method"], d["level_count"]) == (8, 19, 19,
                                                                               "relaxed", 4)
    assert set(d["times"]) == {"symbolic", "detection", "levelization", "numeric"}
    assert d["residual"] <= 1e-12
    assert d["mode_histogram"] == {"Stream": 4}
    path = tmp_path / "report.csv"
    assert cli.main(["factor", conflict8, "--stats-out", str(path)]) == cli.EXIT_OK
    header, row = path.read_text().strip().splitlines()
    assert header.split(",")[:6] == ["matrix", "n", "nz", "nnz", "deps_method", "level_count"]
    assert row.split(",")[1:4] == ["8", "19", "19"]
    assert cli.main(["factor", conflict8, "--stats-out", "report.txt"]) == cli.EXIT_USAGE
    capsys.readouterr()


@pytest.mark.gpu
def test_factor_with_perms(tmp_path, diag5, capsys):
    p = tmp_path / "perm.txt"
    p.write_text("4\n3\n2\n1\n0\n")
    assert cli.main(["factor", diag5, "--perm", str(p), "--check-residual"]) == cli.EXIT_OK
    assert "n=5" in capsys.readouterr().out
    assert cli.main(["factor", diag5, "--row-perm", str(p), "--col-perm", str(p)]) == cli.EXIT_OK
    capsys.readouterr()


@pytest.mark.gpu
def test_exit_pivot(tmp_path, capsys):
    m = tmp_path / "singular.mtx"
    m.write_text("%%MatrixMarket matrix coordinate real general\n"
                 "2 2 4\n1 1 1.0\n2 1 1.0\n1 2 1.0\n2 2 1.0\n")
    for flags in ([], ["--sequential", "left"], ["--sequential", "right"], ["--atomic"]):
        assert cli.main(["factor", str(m)] + flags) == cli.EXIT_PIVOT
        assert "pivot" in capsys.readouterr().err


@pytest.mark.gpu
def test_solve_roundtrip(tmp_path, capsys):
    m = tmp_path / "d5.mtx"
    m.write_text("%%MatrixMarket matrix coordinate real general\n5 5 5\n"
                 + "".join(f"{i} {i} {float(i + 1)}\n" for i in range(1, 6)))
    rhs, xs = tmp_path / "b.txt", tmp_path / "x.txt"
    rhs.write_text("2.0\n6.0\n12.0\n20.0\n30.0\n")
    assert cli.main(["solve", str(m), str(rhs), "--out", str(xs)]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert f"wrote {xs}" in out
    assert np.allclose(np.loadtxt(xs), [1.0, 2.0, 3.0, 4.0, 5.0])
    assert float(out.split("residual ")[1].split()[0]) <= 1e-12
