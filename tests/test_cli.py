"""CLI: the reference CLI's file formats, commands and
exit codes (tests/test_cli.py of the reference), checked against the output
files of the reference CLI itself (sha256 frozen in golden.json["cli"])."""
import csv
import hashlib
import struct

import numpy as np
import pytest

from paper_1310_0956_b200.cli import (EXIT_ARG_ERROR, FORMAT_VERSION, MAGIC, main, read_grid,
                                      write_grid, write_pgm)
from paper_1310_0956_b200.phantom import shepp_logan


def run(*argv):
    return main([str(a) for a in argv])


def file_sha(path):
    return hashlib.sha256(path.read_bytes()).hexdigest()


class TestGridFormat:
    def test_round_trip(self, tmp_path):
        p = tmp_path / "g.bin"
        v = np.linspace(-3, 7, 12)
        write_grid(p, v, 3, 4)
        data, rows, cols = read_grid(p)
        assert (rows, cols) == (3, 4)
        assert np.array_equal(data, v)

    def test_header_layout(self, tmp_path):
        p = tmp_path / "g.bin"
        write_grid(p, np.zeros(6), 2, 3)
        raw = p.read_bytes()
        assert raw[:4] == MAGIC and struct.unpack("<III", raw[4:16]) == (FORMAT_VERSION, 2, 3)
        assert len(raw) == 16 + 48

    @pytest.mark.parametrize("raw", [b"XXXX" + b"\0" * 12,
                                     MAGIC + struct.pack("<III", 99, 1, 1) + b"\0" * 8,
                                     MAGIC + struct.pack("<III", 1, 2, 3) + b"\0" * 40,
                                     b"WMG"])
    def test_bad_files_rejected(self, tmp_path, raw):
        p = tmp_path / "bad.bin"
        p.write_bytes(raw)
        with pytest.raises(Exception):
            read_grid(p)

    def test_size_mismatch_rejected(self, tmp_path):
        with pytest.raises(Exception):
            write_grid(tmp_path / "g.bin", np.zeros(5), 2, 3)

    def test_pgm(self, tmp_path):
        p = tmp_path / "i.pgm"
        write_pgm(p, np.arange(4.0), 2, 2)
        raw = p.read_bytes()
        assert raw.startswith(b"P5\n2 2\n255\n") and raw[-4:] == bytes([0, 85, 170, 255])


class TestHostCommands:
    def test_phantom_matches_reference_bytes(self, tmp_path, golden):
        meta, _ = golden
        out = tmp_path / "ph.bin"
        assert run("phantom", "--n", 16, "--out", out, "--pgm", tmp_path / "ph.pgm") == 0
        assert file_sha(out) == meta["cli"]["ph.bin"]
        data, rows, cols = read_grid(out)
        assert (rows, cols) == (16, 16) and np.array_equal(data, shepp_logan(16))
        man = (tmp_path / "ph.bin.manifest").read_text()
        assert "command=phantom" in man and "n=16" in man
        assert (tmp_path / "ph.pgm").read_bytes().startswith(b"P5\n16 16\n")

    def test_argument_errors(self, tmp_path):
        ph = tmp_path / "ph.bin"
        run("phantom", "--n", 8, "--out", ph)
        assert run("project", "--image", ph, "--angles", 4, "--detectors", 8, "--noise", 0.01,
                   "--out", tmp_path / "s.bin") == EXIT_ARG_ERROR
        assert run("project", "--image", tmp_path / "nope.bin", "--angles", 4,
                   "--detectors", 8, "--out", tmp_path / "s.bin") == EXIT_ARG_ERROR
        write_grid(tmp_path / "rect.bin", np.zeros(6), 2, 3)
        assert run("project", "--image", tmp_path / "rect.bin", "--angles", 4,
                   "--detectors", 8, "--out", tmp_path / "s.bin") == EXIT_ARG_ERROR
        sino = tmp_path / "sino.bin"
        write_grid(sino, np.zeros(32), 4, 8)
        base = ["reconstruct", "--sino", sino, "--n", 8, "--detectors", 8, "--iters", 3,
                "--out", tmp_path / "x.bin", "--log", tmp_path / "c.csv"]
        assert run(*base, "--angles", 5, "--solver", "sirt") == EXIT_ARG_ERROR
        assert run(*base, "--angles", 4, "--solver", "sirt", "--levels", 2) == EXIT_ARG_ERROR
        assert run("spectrum", "--n", 8, "--angles", 4, "--operator", "normal",
                   "--out", tmp_path / "sp.csv") == EXIT_ARG_ERROR


@pytest.fixture()
def problem(tmp_path):
    ph, sino = tmp_path / "ph.bin", tmp_path / "sino.bin"
    assert run("phantom", "--n", 16, "--out", ph) == 0
    assert run("project", "--image", ph, "--angles", 24, "--detectors", 24, "--out", sino) == 0
    return ph, sino, tmp_path


@pytest.mark.gpu
class TestGpuCommands:
    def test_project_bytes_match_reference(self, gpu, golden, problem):
        meta, _ = golden
        ph, sino, tmp = problem
        assert file_sha(sino) == meta["cli"]["sino.bin"]
        noisy = tmp / "noisy.bin"
        assert run("project", "--image", ph, "--angles", 24, "--detectors", 24, "--noise",
                   0.01, "--seed", 5, "--out", noisy) == 0
        assert file_sha(noisy) == meta["cli"]["sino_noisy.bin"]
        assert "seed=5" in (tmp / "noisy.bin.manifest").read_text()

    def test_sirt_reconstruction_bit_identical(self, gpu, golden, problem):
        meta, g = golden
        ph, sino, tmp = problem
        out, log = tmp / "x.bin", tmp / "conv.csv"
        assert run("reconstruct", "--sino", sino, "--n", 16, "--angles", 24, "--detectors", 24,
                   "--solver", "sirt", "--iters", 30, "--xexact", ph, "--out", out,
                   "--log", log) == 0
        assert file_sha(out) == meta["cli"]["x_sirt.bin"]
        with open(log) as fh:
            rows = list(csv.DictReader(fh))
        assert len(rows) == 31 and rows[0]["iter"] == "0" and rows[0]["rel_res"] == "1.0"
        # iterates are bit-identical; the logged norms use DET_SUM instead of
        # BLAS, so they agree to rounding (SURVEY s8(c) parity protocol)
        np.testing.assert_allclose([float(r["rel_res"]) for r in rows], g["cli_sirt_res"],
                                   rtol=1e-12)
        np.testing.assert_allclose([float(r["rel_err_l2"]) for r in rows], g["cli_sirt_err"],
                                   rtol=1e-12)
        # regularised run on the noisy sinogram
        noisy = tmp / "noisy.bin"
        run("project", "--image", ph, "--angles", 24, "--detectors", 24, "--noise", 0.01,
            "--seed", 5, "--out", noisy)
        out2 = tmp / "x2.bin"
        assert run("reconstruct", "--sino", noisy, "--n", 16, "--angles", 24, "--detectors",
                   24, "--solver", "sirt", "--iters", 20, "--lambda", 0.25, "--out", out2,
                   "--log", tmp / "c2.csv") == 0
        assert file_sha(out2) == meta["cli"]["x_sirt_noisy.bin"]

    def test_wmg_bicgstab_matches_reference(self, gpu, golden, problem):
        _, g = golden
        ph, sino, tmp = problem
        out, log = tmp / "x.bin", tmp / "conv.csv"
        assert run("reconstruct", "--sino", sino, "--n", 16, "--angles", 24, "--detectors", 24,
                   "--solver", "wmg-bicgstab", "--levels", 2, "--lambda", 1.0, "--iters", 30,
                   "--tol", 1e-10, "--xexact", ph, "--out", out, "--log", log) == 0
        x, _, _ = read_grid(out)
        np.testing.assert_allclose(x, g["cli_wmg_x"], rtol=1e-8, atol=1e-10)
        with open(log) as fh:
            res = [float(r["rel_res"]) for r in csv.DictReader(fh)]
        assert len(res) == len(g["cli_wmg_res"])
        np.testing.assert_allclose(res, g["cli_wmg_res"], rtol=1e-6, atol=1e-14)
        assert "status=converged" in (tmp / "x.bin.manifest").read_text()

    @pytest.mark.parametrize("solver", ["bicgstab", "tg-bicgstab", "cgls", "wmg-cgls", "gmres"])
    def test_other_solvers_reduce_error(self, gpu, problem, solver):
        ph, sino, tmp = problem
        out, log = tmp / f"{solver}.bin", tmp / f"{solver}.csv"
        extra = ["--levels", 2] if solver in ("wmg-cgls", "gmres") else []
        assert run("reconstruct", "--sino", sino, "--n", 16, "--angles", 24, "--detectors", 24,
                   "--solver", solver, "--iters", 15, "--lambda", 0.5, "--xexact", ph,
                   "--out", out, "--log", log, *extra) == 0
        with open(log) as fh:
            rows = list(csv.DictReader(fh))
        assert float(rows[-1]["rel_err_l2"]) < float(rows[0]["rel_err_l2"])

    def test_bench_table_runs(self, gpu, tmp_path):
        assert run("bench", "--table", "1", "--outdir", tmp_path, "--n", 32, "--angles", 48,
                   "--levels", 2, "--iters-scale", 0.05) == 0
        with open(tmp_path / "table1.csv") as fh:
            rows = list(csv.DictReader(fh))
        assert [r["solver"] for r in rows] == ["sirt", "bicgstab", "wmg-bicgstab"]
        assert (tmp_path / "table1.csv.manifest").exists()
