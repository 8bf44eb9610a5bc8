"""Freeze golden vectors from the REFERENCE implementation (run in the build
container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/*.npz`` + ``golden.json``.  Nothing at test time reads
/root/reference; the GPU box only sees these committed fixtures.

What is frozen (all from ``wmgtomo`` itself):
  projector   sha256 of the reference CSR (indptr/indices as int64, data),
              row/col sums, W x and W^T y on seeded vectors, for the test
              fixtures, configs 0/1 and exact angle subsets of config 3;
  solvers     sirt_solve trajectories (x and residual history), the normal
              operator, bicgstab_solve (plain and WMG-preconditioned) histories;
  multilevel  wtg_apply results (hybrid / multiplicative, 2 and 3 levels);
  joseph      the same hashes for build_projector(kernel="joseph") (f4);
  cli         sha256 of the reference CLI's output files (phantom, project
              with/without noise, SIRT reconstructions) and residual logs (f3).
"""
from __future__ import annotations

import hashlib
import zlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    import wmgtomo
    from wmgtomo.geometry import Geometry, build_geometry, build_projector
    from wmgtomo.multilevel import build_wmg_hierarchy, wmg_preconditioner, wtg_apply
    from wmgtomo.phantom import shepp_logan
    from wmgtomo.solvers import SolverConfig, bicgstab_solve, normal_operator, sirt_solve

    sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
    from paper_1310_0956_b200.phantom import random_ellipses

    meta = {"reference_version": wmgtomo.__version__, "projector": {}, "solvers": {}}
    arrays = {}

    meta["joseph"] = {}

    def proj_case(name, n, d, m, subset=None, keep_vectors=True, kernel="line"):
        g = build_geometry(n, d, m)
        if subset is not None:
            g = Geometry(n, d, len(subset), angles=g.angles[np.asarray(subset)])
        w = build_projector(g, kernel=kernel)
        seed = zlib.crc32(name.encode())
        rs = np.random.default_rng(seed)
        x = rs.standard_normal(n * n)
        y = rs.standard_normal(g.n_data)
        wx = w @ x
        wty = w.T @ y
        rows = np.asarray(w.sum(axis=1)).ravel()
        cols = np.asarray(w.sum(axis=0)).ravel()
        meta["projector" if kernel == "line" else "joseph"][name] = {
            "n": n, "d": d, "m": m, "subset": None if subset is None else list(map(int, subset)),
            "nnz": int(w.nnz), "seed": seed,
            "indptr": sha(w.indptr.astype(np.int64)), "indices": sha(w.indices.astype(np.int64)),
            "data": sha(w.data), "wx": sha(wx), "wty": sha(wty), "rows": sha(rows),
            "cols": sha(cols), "wx_norm": float(np.linalg.norm(wx)),
            "wty_norm": float(np.linalg.norm(wty)),
        }
        if keep_vectors:
            arrays[f"{name}_wx"] = wx
            arrays[f"{name}_wty"] = wty
        print("projector", name, w.nnz, flush=True)
        return g, w

    proj_case("tiny_vertical", 4, 4, 1)
    proj_case("tiny_two", 4, 4, 2)
    proj_case("diag8", 8, 11, 4)
    proj_case("miss12", 4, 12, 1)
    _, w16 = proj_case("w16", 16, 24, 24)
    proj_case("w40", 40, 40, 100)
    _, w0 = proj_case("cfg0", 64, 91, 90)
    proj_case("cfg1", 256, 363, 180, keep_vectors=False)
    proj_case("bench160", 160, 160, 400, keep_vectors=False)
    for n, d in ((512, 725), (1024, 1449), (2048, 2897), (4096, 5793)):
        sub = ([0, n // 8, n // 4 + 1, n // 2, 3 * n // 4 - 3, n - 1] if n <= 1024
               else [0, n // 4 + 1, n // 2, 3 * n // 4 - 3])
        proj_case(f"cfg3_{n}_sub", n, d, n, subset=sub, keep_vectors=False)

    # ---- Joseph kernel ------------------------------------
    for name, (n, d, m) in {"jos_tiny_vertical": (4, 4, 1), "jos_tiny_two": (4, 4, 2),
                            "jos_diag8": (8, 11, 4), "jos_miss12": (4, 12, 1),
                            "jos_odd15": (15, 21, 7), "jos_w16": (16, 24, 24),
                            "jos_cfg0": (64, 91, 90)}.items():
        proj_case(name, n, d, m, kernel="joseph")
    proj_case("jos_cfg1", 256, 363, 180, keep_vectors=False, kernel="joseph")
    proj_case("jos_bench160", 160, 160, 400, keep_vectors=False, kernel="joseph")

    # ---- CLI: output files of the reference CLI ----------
    import tempfile
    from wmgtomo import cli as rcli
    meta["cli"] = {}
    with tempfile.TemporaryDirectory() as td:
        def f(nm):
            return os.path.join(td, nm)

        def run(*argv):
            rc = rcli.main([str(a) for a in argv])
            assert rc == 0, argv

        def file_sha(nm):
            with open(f(nm), "rb") as fh:
                return hashlib.sha256(fh.read()).hexdigest()

        run("phantom", "--n", 16, "--out", f("ph.bin"))
        run("project", "--image", f("ph.bin"), "--angles", 24, "--detectors", 24,
            "--out", f("sino.bin"))
        run("project", "--image", f("ph.bin"), "--angles", 24, "--detectors", 24,
            "--noise", 0.01, "--seed", 5, "--out", f("sino_noisy.bin"))
        run("reconstruct", "--sino", f("sino.bin"), "--n", 16, "--angles", 24,
            "--detectors", 24, "--solver", "sirt", "--iters", 30, "--xexact", f("ph.bin"),
            "--out", f("x_sirt.bin"), "--log", f("sirt.csv"))
        run("reconstruct", "--sino", f("sino_noisy.bin"), "--n", 16, "--angles", 24,
            "--detectors", 24, "--solver", "sirt", "--iters", 20, "--lambda", 0.25,
            "--out", f("x_sirt_noisy.bin"), "--log", f("sirt_noisy.csv"))
        run("reconstruct", "--sino", f("sino.bin"), "--n", 16, "--angles", 24,
            "--detectors", 24, "--solver", "wmg-bicgstab", "--levels", 2, "--lambda", 1.0,
            "--iters", 30, "--tol", 1e-10, "--xexact", f("ph.bin"), "--out", f("x_wmg.bin"),
            "--log", f("wmg.csv"))
        for nm in ("ph.bin", "sino.bin", "sino_noisy.bin", "x_sirt.bin", "x_sirt_noisy.bin"):
            meta["cli"][nm] = file_sha(nm)
        import csv as _csv
        for nm in ("sirt.csv", "wmg.csv"):
            with open(f(nm)) as fh:
                rows = list(_csv.DictReader(fh))
            arrays[f"cli_{nm[:-4]}_res"] = np.array([float(r["rel_res"]) for r in rows])
            arrays[f"cli_{nm[:-4]}_err"] = np.array([float(r["rel_err_l2"]) for r in rows])
        xw = np.frombuffer(open(f("x_wmg.bin"), "rb").read()[16:], dtype="<f8")
        arrays["cli_wmg_x"] = xw.copy()
    print("cli done", flush=True)

    # ---- solvers -------------------------------------------------------
    ph16 = shepp_logan(16)
    x0c = random_ellipses(64, 10, seed=0)
    b0 = w0 @ x0c
    xs, rec = sirt_solve(w0, b0, None, SolverConfig(max_iterations=200), x_ex=x0c)
    arrays["sirt_cfg0_x"] = xs
    arrays["sirt_cfg0_res"] = np.array(rec.rel_residual)
    arrays["sirt_cfg0_err"] = np.array(rec.rel_err_l2)
    arrays["cfg0_phantom"] = x0c
    xs, rec = sirt_solve(w16, w16 @ ph16, None,
                         SolverConfig(max_iterations=60, regularization_lambda=0.5))
    arrays["sirt_w16_lam_x"] = xs
    arrays["sirt_w16_lam_res"] = np.array(rec.rel_residual)

    v = np.random.default_rng(1).standard_normal(256)
    arrays["normal_w16_v"] = v
    arrays["normal_w16_out"] = normal_operator(w16, 2.5)(v)

    f16 = w16.T @ (w16 @ ph16)
    op = normal_operator(w16, 1.0)
    xb, rec = bicgstab_solve(op, f16, cfg=SolverConfig(max_iterations=30))
    arrays["bicg_w16_x"] = xb
    arrays["bicg_w16_res"] = np.array(rec.rel_residual)
    for lv in (2, 3):
        h = build_wmg_hierarchy(w16, 16, 1.0, lv)
        rr = np.random.default_rng(20 + lv).standard_normal(256)
        arrays[f"wtg_w16_l{lv}_r"] = rr
        arrays[f"wtg_w16_l{lv}_hyb"] = wtg_apply(h.root, rr, multiplicative=False)
        arrays[f"wtg_w16_l{lv}_mul"] = wtg_apply(h.root, rr, multiplicative=True)
        xw, rec = bicgstab_solve(op, f16, precond=wmg_preconditioner(h),
                                 cfg=SolverConfig(max_iterations=20, residual_tolerance=1e-10))
        arrays[f"wmgbicg_w16_l{lv}_x"] = xw
        arrays[f"wmgbicg_w16_l{lv}_res"] = np.array(rec.rel_residual)
        meta["solvers"][f"wmgbicg_w16_l{lv}_status"] = rec.status
    from wmgtomo.multilevel import classical_tg_preconditioner
    for steps in ((0, 0), (1, 1), (2, 1)):
        tg = classical_tg_preconditioner(w16, 16, 1.0, smoother_steps=steps)
        rr = np.random.default_rng(40 + sum(steps)).standard_normal(256)
        arrays[f"tg_w16_{steps[0]}{steps[1]}_r"] = rr
        arrays[f"tg_w16_{steps[0]}{steps[1]}_z"] = tg(rr)
    tg = classical_tg_preconditioner(w16, 16, 1.0)
    xt, rec = bicgstab_solve(op, f16, precond=tg,
                             cfg=SolverConfig(max_iterations=200, residual_tolerance=1e-10))
    arrays["tgbicg_w16_res"] = np.array(rec.rel_residual)
    print("solvers done", flush=True)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
