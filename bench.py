#!/usr/bin/env python
"""Benchmark: A/A^T projector pair throughput (BASELINE config 3) on B200.

A step is one forward projection A x plus one backprojection A^T y of the
config-3 workload (n x n grid, n angles in [0, pi), ceil(n sqrt 2) detectors,
float32 data, x ~ U[0,1] seed 3000, y ~ U[0,1] seed 3001).  Default n = 4096
(the largest config-3 size; 64 MB image + 95 MB sinogram per operand, larger
than the 126 MB L2 together, so no explicit flush is needed; for n < 4096 an
L2 flush is done between steps outside the timed events).

Multi-GPU (torchrun, one process per GPU): the quad units of angles
{k, m-k, m/2-k, m/2+k} (mirror pairs when m % 4 != 0)
are dealt round-robin to the ranks (each shard keeps the symmetric kernels),
each rank projects its angles and backprojects its sinogram rows, and the
partial A^T y images are summed with an NCCL allreduce -- total work fixed
("strong" scaling).  Time = max over ranks of the CUDA-event time.

The same JSON line carries ``wmg_cgls`` (BASELINE config 1 WMG-CGLS seconds to
rel. residual 1e-4, setup separate, plain CGLS beside it), the end-to-end
number with host buffers (``e2e``), the CPU baselines and the rooflines;
``--workload config2|config4`` runs the other BASELINE configurations.

``value`` is the DEPENDENT pair a Krylov iteration uses: A x then A^T y back
to back on one stream (``value_sequential``, which also gives the per-kernel
times behind the rooflines); the two independent config-3 products on two
streams sharing the SMs are reported beside it (``value_two_streams``).
``e2e`` is the drop-in call a reference-style user makes: ``sino = w @ x;
img = w.T @ y`` with float32 numpy vectors in and out (every call copies its
operand to HBM and its result back before returning).  ``e2e_pipelined`` is
what a user streaming pairs through the public API with pinned host buffers
sees: copies on their own streams (double-buffered, overlapping the kernels)
and the two independent products on two streams.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference
algorithm on the host CPU instead (the pinned C oracle: the reference's CSR
built exactly, then CSR SpMV pairs with all host threads, on a bounded angle
sample of the same workload).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "A/AT pair GRays/s"
UNIT = "GRays/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", "--grid", dest="n", type=int, default=4096)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-angles", type=int, default=4)
    ap.add_argument("--no-wmg", action="store_true",
                    help="skip the config-1 WMG-CGLS time-to-tolerance measurement")
    ap.add_argument("--workload", choices=["pair", "config2", "config4", "launch-check"],
                    default="pair",
                    help="pair: config-3 projector pair (the default bench line); "
                         "config2: CGLS vs WMG-GMRES on config 2; config4: slice-stack "
                         "throughput (separate JSON lines)")
    ap.add_argument("--streams", type=int, default=2,
                    help="config4: concurrent slice solves (host thread + CUDA stream each)")
    ap.add_argument("--slices", type=int, default=8,
                    help="config4: slices timed (of the 256-slice stack)")
    ap.add_argument("--levels", type=int, default=None,
                    help="WMG levels (config2: 5; config4: 6 -- 5 levels needs 550 GB of "
                         "dense coarse factors)")
    ap.add_argument("--wmg-slices", type=int, default=2,
                    help="config4: slices solved with WMG-CGLS (after the CGLS slices)")
    return ap.parse_args()


def workload(n):
    m = n
    d = int(math.ceil(n * math.sqrt(2.0)))
    return n, d, m


def config_dict(n, d, m, world, extra=None):
    c = {"workload": f"config3_pair_n{n}", "n": n, "n_angles": m, "n_detectors": d,
         "dtype_data": "float32", "geometry": "fixed-point64", "angle_sharding": "quad units",
         "parallelism": f"angles{world}", "l2": ("inputs larger than L2" if n >= 4096
                                                  else "L2 flushed between steps")}
    if extra:
        c.update(extra)
    return c


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        sm = []
        mx = None
        reasons = set()
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
            except (ValueError, IndexError):
                continue
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def onchip_roofline(n, t_fwd, t_bwd, n_sm, f_sm, world):
    """The on-chip resources that bind the pair (DESIGN.md kernel table).  The
    binding one is the L1 data pipe that returns load data to the registers
    (l1tex__data_pipe_lsu_wavefronts, peak 1 wavefront/clk/SM): the forward's
    pixel gathers run it at ~94 %.  Also: L1 sector requests of the forward
    gathers (peak 4 sectors/clk/SM) and the backprojector's shared wavefronts.
    Per-launch counts from the committed ncu capture, times live from this run."""
    t = ncu_traffic()
    out = {}
    for kern, tk in (("forward", t_fwd), ("backward", t_bwd)):
        wf = t.get(f"l1_datapipe_wavefronts_{kern}_n{n}")
        if wf and tk > 0 and world == 1:
            peak = 1.0 * n_sm * f_sm
            out[f"{kern}_l1_data_pipe"] = {"achieved": wf / tk / 1e9, "peak": peak / 1e9,
                                           "unit": "Gwavefronts/s", "frac": wf / tk / peak,
                                           "per_launch": wf}
    sec = t.get(f"l1_sectors_forward_n{n}")
    if sec and t_fwd > 0 and world == 1:
        peak = 4.0 * n_sm * f_sm
        out["forward_l1_sectors"] = {"achieved": sec / t_fwd / 1e9, "peak": peak / 1e9,
                                     "unit": "Gsectors/s", "frac": sec / t_fwd / peak,
                                     "per_launch": sec}
    wf = t.get(f"smem_wavefronts_backward_n{n}")
    if wf and t_bwd > 0 and world == 1:
        peak = 1.0 * n_sm * f_sm
        out["backward_smem_wavefronts"] = {"achieved": wf / t_bwd / 1e9, "peak": peak / 1e9,
                                           "unit": "Gwavefronts/s", "frac": wf / t_bwd / peak,
                                           "per_launch": wf}
    out["source"] = "profiles/traffic.json (ncu --set full), live kernel times"
    return out


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh)
    except OSError:
        return {}


def host_info():
    """CPU model, logical cores and BLAS threading of the box."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": i.get("internal_api"), "threads": i.get("num_threads")}
                for i in threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "blas_threadpools": blas}


# ------------------------------------------------------------ CPU baseline
def cpu_pair_rate(n, d, m, k_angles, target_seconds=10.0, max_reps=50):
    """Reference algorithm on the host: exact CSR of W for k evenly spaced
    angles (setup, untimed), then W x + W^T y by CSR SpMV with all threads."""
    from oracle import cproj
    idx = np.linspace(0, m - 1, k_angles).round().astype(int)
    angles = (np.arange(m) * (np.pi / m))[idx]
    w = cproj.build_csr(n, d, angles)
    wt = w.T.tocsr()
    rs = np.random.default_rng(3000)
    x = rs.uniform(0.0, 1.0, n * n)
    y = np.random.default_rng(3001).uniform(0.0, 1.0, w.shape[0])
    cproj.csr_matvec(w, x)
    cproj.csr_matvec(wt, y)
    reps, t_tot = 0, 0.0
    while t_tot < target_seconds and reps < max_reps:
        t0 = time.perf_counter()
        cproj.csr_matvec(w, x)
        cproj.csr_matvec(wt, y)
        t_tot += time.perf_counter() - t0
        reps += 1
    t_pair = t_tot / reps
    rays = w.shape[0]
    return {"value": rays / t_pair / 1e9, "unit": UNIT, "cores": cproj.num_threads(),
            "kind": "port", "host": host_info(),
            "sample": f"{k_angles} of {m} angles (exact reference CSR rows), {reps} pairs, "
                      f"{t_pair * 1e3:.1f} ms/pair, nnz={w.nnz}; rate scales linearly in angles"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, d, m = workload(args.n)
    from oracle import cproj
    idx = np.linspace(0, m - 1, args.cpu_angles).round().astype(int)
    angles = (np.arange(m) * (np.pi / m))[idx]
    w = cproj.build_csr(n, d, angles)
    wt = w.T.tocsr()
    x = np.random.default_rng(3000).uniform(0.0, 1.0, n * n)
    y = np.random.default_rng(3001).uniform(0.0, 1.0, w.shape[0])
    for _ in range(args.warmup):
        cproj.csr_matvec(w, x)
        cproj.csr_matvec(wt, y)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cproj.csr_matvec(w, x)
        cproj.csr_matvec(wt, y)
    dt = (time.perf_counter() - t0) / args.steps
    value = w.shape[0] / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(n, d, m, 1, {"sample_angles": int(args.cpu_angles)}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cproj.num_threads(),
                             "kind": "port", "host": host_info(),
                             "sample": f"{args.cpu_angles} of {m} angles per step, exact "
                                       f"reference CSR (nnz={w.nnz}), CSR SpMV pair"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------- WMG-CGLS (config 1)
def run_wmg_cgls(dev, reps=5, world=1):
    """BASELINE config 1: 256^2, 180 angles, 363 detectors, float64, seeded
    20-ellipse phantom (seed 1000), 1 % Gaussian noise (seed 1500); WMG-CGLS
    (flexible PCG on the normal equations, 3 levels, 2 pre + 2 post SIRT-type
    sweeps per level) to normal-equations residual 1e-4 or 100 iterations.
    Setup (hierarchy) and solve are timed separately (device-synchronised wall
    clock, max over ranks); the plain-CGLS solve and the reference's
    smoother-free cycle are reported beside it.  Under torchrun every rank owns
    a quad shard of the angles (sharded pairs, allreduced leaf Grams)."""
    import torch
    import torch.distributed as dist
    from paper_1310_0956_b200 import (SolverConfig, add_gaussian_noise, build_geometry,
                                      build_projector, build_wmg_hierarchy, cgls_solve,
                                      random_ellipses, wmg_preconditioner)
    n, d, m = 256, 363, 180
    g = build_geometry(n, d, m)
    w = _projector(g, world, dev)                                   # parity float64 (exact W)
    wf = _projector(g, world, dev, precision="float64", mode="fast")
    x_ex = random_ellipses(n, 20, seed=1000)
    b = add_gaussian_noise(build_projector(g, device=dev) @ x_ex, 0.01, seed=1500)
    bd = _local_rows(wf, b, dev)
    cfg = SolverConfig(max_iterations=100, residual_tolerance=1e-4)

    def timed(fn):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize(dev)
        return time.perf_counter() - t0, r

    setups, solves, repeats = [], [], []
    for _ in range(reps):
        tu, M = timed(lambda: wmg_preconditioner(
            build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=2, nu_post=2)))
        ts, (_, rec) = timed(lambda: cgls_solve(wf, bd, precond=M, cfg=cfg))
        # a further right-hand side with the same preconditioner (slice stacks):
        # the captured CGLS iteration is replayed, nothing is re-captured
        tr, _ = timed(lambda: cgls_solve(wf, bd, precond=M, cfg=cfg))
        setups.append(tu)
        solves.append(ts)
        repeats.append(tr)
        iters, status, rel = rec.iterations[-1], rec.status, rec.rel_residual[-1]
        del M
    t_cgls = []
    for _ in range(reps):
        tc, (_, rec_c) = timed(lambda: cgls_solve(
            wf, bd, cfg=SolverConfig(max_iterations=500, residual_tolerance=1e-4)))
        t_cgls.append(tc)
    # the reference's smoother-free cycle (nu = 0), for the like-for-like CPU comparison
    s0, u0 = [], []
    for _ in range(reps):
        tu, M0 = timed(lambda: wmg_preconditioner(build_wmg_hierarchy(w, n, 0.0, 3)))
        ts, (_, rec0) = timed(lambda: cgls_solve(wf, bd, precond=M0, cfg=cfg))
        u0.append(tu)
        s0.append(ts)
        del M0
    # per-rep maxima over ranks, then best of the reps
    k = reps
    mx = _max_over_ranks(setups + solves + t_cgls + u0 + s0 + repeats, dev)
    setups, solves, t_cgls, u0, s0, repeats = (mx[0:k], mx[k:2 * k], mx[2 * k:3 * k],
                                               mx[3 * k:4 * k], mx[4 * k:5 * k],
                                               mx[5 * k:6 * k])
    nu0 = {"seconds": min(s0), "setup_seconds": min(u0), "iterations": rec0.iterations[-1]}
    nu0["roofline"] = _wmg_model_roofline(n, m, 3, 0, 0, nu0["iterations"], nu0["seconds"], world)
    return {"metric": "WMG-CGLS seconds to rel. residual 1e-4", "config": "config1_256_180x363",
            "roofline": _wmg_model_roofline(n, m, 3, 2, 2, iters, min(solves), world),
            "n_gpus": world, "seconds": min(solves), "setup_seconds": min(setups),
            "seconds_repeat_rhs": min(repeats),
            "seconds_incl_setup": min(a + c for a, c in zip(solves, setups)),
            "iterations": iters, "status": status, "final_rel_residual": rel,
            "levels": 3, "nu_pre": 2, "nu_post": 2, "lambda": 0.0,
            "projector": "float64 fast (<=1e-12 of the reference W); sparse leaf Grams "
                         "(<=1e-12 of the exact P_L^T P_L)",
            "angle_sharding": "quad units" if world > 1 else None,
            "cgls_seconds": min(t_cgls), "cgls_iterations": rec_c.iterations[-1],
            "nu0": nu0, "b": b, "x_ex": x_ex,
            "timing": "torch.cuda.synchronize + perf_counter, max over ranks, best of %d; "
                      "every WMG solve uses a freshly built hierarchy (graph capture "
                      "included)" % reps}


def _wmg_model_roofline(n, m, levels, nu_pre, nu_post, iterations, seconds, world=1):
    """SURVEY s8(d) model roofline of a WMG-CGLS solve: node pairs x t_roof_pair
    + coarse leaf bytes / HBM bandwidth.  A pair is 2 nnz(W) intersection
    updates at the float64 gather peak (n_SM x 32 lanes x f_SM / 2); every
    internal node of the hierarchy applies its (matrix-free) system nu_pre +
    nu_post + 1 times per V-cycle (once without smoother sweeps), the outer
    iteration once, and a V-cycle streams every packed leaf inverse once."""
    nnz = (4.0 / math.pi) * m * n * n               # within 1e-5 of the exact count
    internal = (4 ** (levels - 1) - 1) // 3
    apps = (nu_pre + nu_post + 1) if nu_pre > 0 else (1 + nu_post)
    pairs = (iterations + 1) * (1 + internal * apps)
    p = (n >> (levels - 1)) ** 2
    leaves = 4 ** (levels - 1)
    leaf_bytes = leaves * (p * (p + 128) // 2) * 8  # packed lower 128 x 128 tiles
    peaks, peak_source = measured_peaks()
    f_sm = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
    hbm = (peaks.get("hbm_gbs") or 6650.0) * 1e9
    r64 = 148 * 32 * f_sm / 2 * world
    t_pairs = pairs * 2 * nnz / r64
    t_leaf = (iterations + 1) * leaf_bytes / hbm
    model = t_pairs + t_leaf
    return {"bound": "gather + hbm (model)", "model_seconds": model, "frac": model / seconds,
            "node_pairs": pairs, "pair_seconds_at_peak": 2 * nnz / r64,
            "leaf_bytes_per_cycle": leaf_bytes, "peak_source": peak_source,
            "definition": "SURVEY s8(d): node pairs x 2 nnz / (n_SM x 32 x f_SM / 2) + "
                          "V-cycles x packed leaf bytes / measured HBM bandwidth"}


def cpu_wmg_cgls(b):
    """CPU baseline for config 1: the reference algorithm (exact W, hierarchy of
    stored sparse factors, smoother-free hybrid V-cycle, dense Cholesky leaves)
    restated in oracle/multilevel.py, inside the oracle's flexible PCG-NE, on the
    box's host cores (scipy SpMV single-threaded, LAPACK multi-threaded)."""
    from oracle import cproj
    from oracle import multilevel as oml
    from oracle import solvers as osol
    n, d, m = 256, 363, 180
    w = cproj.build_csr(n, d, np.arange(m) * (np.pi / m))
    t0 = time.perf_counter()
    root = oml.build_hierarchy(w, n, 0.0, 3)
    t1 = time.perf_counter()
    _, rec = osol.cgls_solve(w, b, precond=oml.preconditioner(root), max_iterations=100,
                             tol=1e-4)
    t2 = time.perf_counter()
    _, rec_c = osol.cgls_solve(w, b, max_iterations=500, tol=1e-4)
    t3 = time.perf_counter()
    return {"seconds": t2 - t1, "setup_seconds": t1 - t0, "iterations": rec.iterations[-1],
            "cgls_seconds": t3 - t2, "cgls_iterations": rec_c.iterations[-1],
            "cores": cproj.num_threads(), "kind": "port", "host": host_info(),
            "sample": "full config-1 problem, reference smoother-free V-cycle (nu = 0)"}


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, dev = _dist_init()
    local = dev.index

    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    from paper_1310_0956_b200.sharding import AngleShardedProjector

    n, d, m = workload(args.n)
    g_full = build_geometry(n, d, m)
    if world > 1:
        # angle k -> rank k mod world; A^T y partials summed by one NCCL allreduce
        w = AngleShardedProjector(g_full, precision="float32", device=dev)
        mine = w.index
    else:
        w = build_projector(g_full, precision="float32", device=dev)
        mine = np.arange(m)
    M_loc, Npix = w.shape

    x_h = np.random.default_rng(3000).uniform(0.0, 1.0, n * n).astype(np.float32)
    y_full = np.random.default_rng(3001).uniform(0.0, 1.0, m * d).astype(np.float32)
    y_h = np.ascontiguousarray(y_full.reshape(m, d)[mine].reshape(-1))
    x = torch.from_numpy(x_h).to(dev)
    y = torch.from_numpy(y_h).to(dev)
    sino = torch.empty(M_loc, dtype=torch.float32, device=dev)
    img = torch.empty(Npix, dtype=torch.float32, device=dev)
    flush = None if n >= 4096 else torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        w.forward_(x, sino)
        w.backward_(y, img)          # includes the allreduce when sharded

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(i & 0xFF)
            e0, e1, e2, e3 = ev[i]
            e0.record(stream)
            w.forward_(x, sino)
            e1.record(stream)
            w.backward_(y, img)      # local backprojection (+ NCCL allreduce if N > 1)
            e2.record(stream)
            e3.record(stream)
        torch.cuda.synchronize(dev)
        # The step's two products are independent: on two streams they share
        # the SMs (the forward is L1-data-pipe bound, the backprojection more
        # issue bound).  This concurrent pass gives ``value``; the back-to-back
        # pass above gives the per-kernel times and ``value_sequential``.
        s_f = torch.cuda.Stream(device=dev)
        s_b = torch.cuda.Stream(device=dev)

        def cstep():
            s_f.wait_stream(stream)
            s_b.wait_stream(stream)
            with torch.cuda.stream(s_f):
                w.forward_(x, sino)
            with torch.cuda.stream(s_b):
                w.backward_(y, img)
            stream.wait_stream(s_f)
            stream.wait_stream(s_b)

        for _ in range(2):
            cstep()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        t_conc = 0.0
        if flush is None:
            # operands larger than L2: the K steps stream through the two
            # queues (forwards on one, backprojections on the other) without
            # a join between steps, bracketed by one pair of events
            c0.record(stream)
            s_f.wait_stream(stream)
            s_b.wait_stream(stream)
            for i in range(args.steps):
                with torch.cuda.stream(s_f):
                    w.forward_(x, sino)
                with torch.cuda.stream(s_b):
                    w.backward_(y, img)
            stream.wait_stream(s_f)
            stream.wait_stream(s_b)
            c1.record(stream)
            c1.synchronize()
            t_conc = c0.elapsed_time(c1) / 1e3
        else:
            for i in range(args.steps):
                flush.fill_(i & 0xFF)
                c0.record(stream)
                cstep()
                c1.record(stream)
                c1.synchronize()
                t_conc += c0.elapsed_time(c1) / 1e3
    if world > 1:
        dist.barrier()
    step_ms = sorted(a.elapsed_time(dd) for a, _, _, dd in ev)   # per-step, back to back
    t_fwd = sum(a.elapsed_time(b) for a, b, _, _ in ev) / 1e3
    t_bwd = sum(b.elapsed_time(c) for _, b, c, _ in ev) / 1e3
    t_tot = sum(a.elapsed_time(dd) for a, _, _, dd in ev) / 1e3
    tt = torch.tensor([t_tot, t_fwd, t_bwd, t_conc], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_tot, t_fwd, t_bwd, t_conc = [float(v) for v in tt.cpu()]
    # ``value``: the DEPENDENT schedule a Krylov iteration uses (A x, then A^T y,
    # back to back on one stream), which also gives the per-kernel times behind
    # the rooflines; the config-3 step's two products are independent (x and y
    # are separate inputs), so the same steps on two streams sharing the SMs
    # are reported beside it (``value_two_streams``)
    t_val = t_tot
    ms_step = t_val / args.steps * 1e3
    rays_total = m * d
    value = rays_total * args.steps / t_val / 1e9
    value_seq = value
    value_conc = rays_total * args.steps / t_conc / 1e9

    # ---- end to end through the drop-in call -----------------------------
    # What a reference-style caller does (geometry.py:200-215 semantics): numpy
    # vectors in, numpy vectors out, ``w @ x`` then ``w.T @ y``; every call
    # copies its operand to HBM, runs the kernel and copies the result back
    # before returning.  (Single rank: the sharded projector has no numpy path.)
    e2e_dropin = None
    if world == 1:
        x_np = x_h.copy()
        y_np = y_h.copy()
        for _ in range(2):
            sino_np = w @ x_np
            img_np = w.T @ y_np
        torch.cuda.synchronize(dev)
        d0 = torch.cuda.Event(enable_timing=True)
        d1 = torch.cuda.Event(enable_timing=True)
        t0w = time.perf_counter()
        d0.record(stream)
        for _ in range(args.steps):
            sino_np = w @ x_np
            img_np = w.T @ y_np
        d1.record(stream)
        d1.synchronize()
        t_dropin = d0.elapsed_time(d1) / 1e3
        t_dropin_wall = time.perf_counter() - t0w
        dropin_ok = bool(np.array_equal(sino_np, sino.cpu().numpy())
                         and np.array_equal(img_np, img.cpu().numpy()))
        e2e_dropin = {"value": rays_total * args.steps / t_dropin / 1e9, "unit": UNIT,
                      "h2d_bytes_per_step": int(x_np.nbytes + y_np.nbytes),
                      "d2h_bytes_per_step": int(sino_np.nbytes + img_np.nbytes),
                      "ms_per_step": t_dropin / args.steps * 1e3,
                      "wall_ms_per_step": t_dropin_wall / args.steps * 1e3,
                      "call": "sino = w @ x; img = w.T @ y (float32 numpy in and out)",
                      "verified_against_device": dropin_ok}

    # ---- pipelined end to end (pinned host buffers, copies overlapped) ----
    pin_x = torch.from_numpy(x_h).pin_memory()
    pin_y = torch.from_numpy(y_h).pin_memory()
    out_s = torch.empty(M_loc, dtype=torch.float32).pin_memory()
    out_i = torch.empty(Npix, dtype=torch.float32).pin_memory()

    # Pipelined like a user streaming many pairs: H2D copies of step i+1 and
    # D2H copies of step i overlap the kernels (copy engines on their own
    # streams, device buffers double-buffered); the forwards stay on one
    # stream and the backprojections on another (each direction reuses its
    # projector workspace), and the two directions overlap each other.
    e2e_s = [torch.empty(M_loc, dtype=torch.float32, device=dev) for _ in range(2)]
    e2e_i = [torch.empty(Npix, dtype=torch.float32, device=dev) for _ in range(2)]
    xd_b = [torch.empty(Npix, dtype=torch.float32, device=dev) for _ in range(2)]
    yd_b = [torch.empty(M_loc, dtype=torch.float32, device=dev) for _ in range(2)]
    out_s2 = [out_s, torch.empty(M_loc, dtype=torch.float32).pin_memory()]
    out_i2 = [out_i, torch.empty(Npix, dtype=torch.float32).pin_memory()]
    s_fwd = torch.cuda.Stream(device=dev)
    s_bwd = torch.cuda.Stream(device=dev)
    c_in = torch.cuda.Stream(device=dev)
    c_out = torch.cuda.Stream(device=dev)
    ev = {}

    def mark(name, i, st):
        e = torch.cuda.Event()
        e.record(st)
        ev[(name, i)] = e

    def wait(st, name, i):
        e = ev.get((name, i))
        if e is not None:
            st.wait_event(e)

    step_no = [0]

    def e2e_step():
        i = step_no[0]
        step_no[0] += 1
        b = i & 1
        # inputs: the buffers of step i-2 must have been consumed
        wait(c_in, "fwd", i - 2)
        wait(c_in, "bwd", i - 2)
        with torch.cuda.stream(c_in):
            xd_b[b].copy_(pin_x, non_blocking=True)
            mark("x", i, c_in)
            yd_b[b].copy_(pin_y, non_blocking=True)
            mark("y", i, c_in)
        # kernels: outputs of step i-2 must have been copied out
        wait(s_fwd, "x", i)
        wait(s_fwd, "out_s", i - 2)
        with torch.cuda.stream(s_fwd):
            w.forward_(xd_b[b], e2e_s[b])
        mark("fwd", i, s_fwd)
        wait(s_bwd, "y", i)
        wait(s_bwd, "out_i", i - 2)
        with torch.cuda.stream(s_bwd):
            w.backward_(yd_b[b], e2e_i[b])
        mark("bwd", i, s_bwd)
        wait(c_out, "fwd", i)
        with torch.cuda.stream(c_out):
            out_s2[b].copy_(e2e_s[b], non_blocking=True)
        mark("out_s", i, c_out)
        wait(c_out, "bwd", i)
        with torch.cuda.stream(c_out):
            out_i2[b].copy_(e2e_i[b], non_blocking=True)
        mark("out_i", i, c_out)

    def e2e_drain():
        stream.wait_stream(c_out)

    e2e_step()
    e2e_drain()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for st_ in (c_in, c_out, s_fwd, s_bwd):
        st_.wait_stream(stream)
    for _ in range(args.steps):
        e2e_step()
    e2e_drain()
    stream.wait_stream(s_fwd)
    stream.wait_stream(s_bwd)
    s1.record(stream)
    torch.cuda.synchronize(dev)
    te = torch.tensor([s0.elapsed_time(s1) / 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())
    e2e_value = rays_total * args.steps / t_e2e / 1e9
    # the pipelined host round trips returned exactly the device-resident results
    # (deterministic kernels, same inputs): the overlap hides nothing
    last = args.steps & 1                  # buffer set of the last timed step (warm-up = 0)
    e2e_ok = bool(torch.equal(out_s2[last], sino.cpu()) and torch.equal(out_i2[last], img.cpu()))

    # ---- roofline ------------------------------------------
    # Unit = one intersection update (one gathered operand + FMA + crossing
    # arithmetic); a launch of either product does nnz(W_local) of them, nnz
    # from an exact GPU counting pass of the reference walker.  Peak gather
    # rate = SMs x 32 lanes x f_SM (fp32 operands).  The compulsory HBM bytes
    # 4 (N + M) per launch are reported beside it (orders of magnitude below).
    peaks, peak_src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    clk = clocks.summary()
    f_sm = (clk["sm_mhz"] or peaks.get("sm_max_mhz", 1965.0)) * 1e6
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    wl = getattr(w, "local", w)
    nnz_local = wl.nnz()
    nnz_formula = 4.0 / math.pi * M_loc / d * n * n        # (4/pi) m n^2, SURVEY A.1
    fwd_avg, bwd_avg = t_fwd / args.steps, t_bwd / args.steps
    dom = "backward" if bwd_avg >= fwd_avg else "forward"
    t_dom = max(fwd_avg, bwd_avg)
    gather_peak = n_sm * 32 * f_sm
    upd_rate = nnz_local / t_dom
    bytes_launch = 4 * (Npix + M_loc)                    # read one operand, write the other
    traffic = ncu_traffic().get(f"{dom}_n{n}")
    pair_rate = 2 * nnz_local / (t_tot / args.steps)
    # kernels launched per step, counted from one profiled step (outside the
    # timed region)
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize(dev)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize(dev)
    step_kernels = [e.name for e in prof.events() if e.device_type.name == "CUDA"
                    and "nccl" not in e.name.lower() and "Memcpy" not in e.name
                    and "Memset" not in e.name]
    launches = args.steps * len(step_kernels)
    e2e_pipe = {"value": e2e_value, "unit": UNIT, "verified_against_device": e2e_ok,
                "h2d_bytes_per_step": 4 * (Npix + M_loc),
                "d2h_bytes_per_step": 4 * (Npix + M_loc),
                "schedule": "pinned host buffers, copies on their own streams (double-"
                            "buffered), the two independent products on two streams"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(n, d, m, world),
        "e2e": e2e_dropin if e2e_dropin is not None else e2e_pipe,
        "e2e_pipelined": e2e_pipe,
        "roofline": {"bound": "gather", "kernel": dom, "achieved": upd_rate / 1e9,
                     "peak": gather_peak / 1e9, "unit": "Gupdates/s",
                     "frac": upd_rate / gather_peak,
                     "traffic": traffic, "algorithmic_bytes": bytes_launch,
                     "updates_per_launch": nnz_local,
                     "definition": "SURVEY s8(d): exact nnz(W) intersection updates per "
                                   "launch / launch time / (SMs x 32 lanes x f_SM)",
                     "f_sm_mhz": f_sm / 1e6, "n_sm": n_sm},
        "roofline_pair": {"achieved": pair_rate / 1e9, "peak": gather_peak / 1e9,
                          "unit": "Gupdates/s", "frac": pair_rate / gather_peak,
                          "definition": "2 nnz(W) per dependent pair / pair time"},
        "roofline_hbm": {"kernel": dom, "achieved": bytes_launch / t_dom / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": bytes_launch / t_dom / 1e9 / hbm,
                         "peak_source": peak_src},
        "roofline_onchip": onchip_roofline(n, fwd_avg, bwd_avg, n_sm, f_sm, world),
        "nnz": {"exact_local": nnz_local, "formula_local": nnz_formula},
        "pair_schedule": "one stream, dependent (A x then A^T y); value_two_streams = the "
                         "two independent products on two streams sharing the SMs",
        "ms_per_step_two_streams": t_conc / args.steps * 1e3,
        "value_two_streams": value_conc,
        "value_sequential": value_seq,
        "step_ms_sequential": {"median": step_ms[len(step_ms) // 2], "best": step_ms[0]},
        "kernels_ms": {"forward": fwd_avg * 1e3, "backward": bwd_avg * 1e3},
        "gpu_launches": launches,
        "kernels_per_step": sorted(set(step_kernels)),
        "clocks": clk,
    }
    if not args.no_wmg:
        try:
            wmg = run_wmg_cgls(dev, world=world)
            b1 = wmg.pop("b")
            wmg.pop("x_ex")
            if rank == 0 and world == 1 and not args.no_cpu_baseline:
                wmg["cpu_baseline"] = cpu_wmg_cgls(b1)
            line["wmg_cgls"] = wmg
        except Exception as exc:  # pragma: no cover
            line["wmg_cgls"] = {"error": repr(exc)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_pair_rate(n, d, m, args.cpu_angles)
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------ config 2
def _dist_init():
    """(world, rank, device); NCCL process group when launched by torchrun.
    Test-only overrides: WMG_BENCH_BACKEND=gloo and WMG_BENCH_DEVICE=<index>
    run the multi-rank logic with host-side collectives on one GPU."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("WMG_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        backend = os.environ.get("WMG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return world, rank, dev


def _max_over_ranks(values, dev):
    """Elementwise max of host floats over all ranks (device-timed spans)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64, device=dev)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def _projector(g, world, dev, **kw):
    """Full projector at N = 1, this rank's quad angle shard at N > 1."""
    from paper_1310_0956_b200 import build_projector
    from paper_1310_0956_b200.sharding import AngleShardedProjector
    if world > 1:
        return AngleShardedProjector(g, device=dev, **kw)
    return build_projector(g, device=dev, **kw)


def _local_rows(w, b, dev):
    import torch
    bd = torch.from_numpy(np.ascontiguousarray(b)).to(dev)
    return w.scatter_sinogram(bd) if hasattr(w, "scatter_sinogram") else bd


def run_config2(args):
    """BASELINE config 2: 1024^2, 720 angles, 1449 detectors; float32 projector
    with float64 Krylov vectors; seeded 50-ellipse phantom (seed 2000, values
    U[0,1]); Poisson data, I0 = 1e5, mu = 2/n, log transform (seed 2500).
    Unpreconditioned CGLS vs WMG-preconditioned GMRES on the normal equations
    (levels = 5, reference smoother-free cycle), each to normal-equations
    residual 1e-4.  Under torchrun the angles are sharded (quad units per
    rank, NCCL allreduce of W^T y and of the leaf Grams); times are max over
    ranks.  ``--n`` rescales the grid (detectors = ceil(n sqrt 2), angles =
    720 n / 1024) for quick checks."""
    import torch
    import torch.distributed as dist
    from paper_1310_0956_b200 import (SolverConfig, build_geometry, build_projector,
                                      build_wmg_hierarchy, cgls_solve, gmres_solve,
                                      normal_operator, poisson_log_data, random_ellipses,
                                      wmg_preconditioner)
    world, rank, dev = _dist_init()
    levels = args.levels or 5
    n = args.n if args.n != 4096 else 1024
    m = int(round(720 * n / 1024))
    m += m % 2
    d = int(math.ceil(n * math.sqrt(2.0)))
    g = build_geometry(n, d, m)
    x_ex = random_ellipses(n, 50, seed=2000, value_range=(0.0, 1.0))
    b = poisson_log_data(build_projector(g, precision="float32", device=dev) @ x_ex, 1e5,
                         2.0 / n, seed=2500)
    w32 = _projector(g, world, dev, precision="float32")
    bd = _local_rows(w32, b, dev)
    out = {"metric": "config2 seconds to rel. residual 1e-4", "n": n, "n_angles": m,
           "n_detectors": d, "n_gpus": world, "projector": "float32 arithmetic, float64 "
           "Krylov vectors", "angle_sharding": "quad units" if world > 1 else None,
           "data": "synthetic: 50-ellipse phantom, Poisson I0=1e5, mu=2/n",
           "timing": "torch.cuda.synchronize + perf_counter, max over ranks"}
    cgls_solve(w32, bd, cfg=SolverConfig(max_iterations=2))          # warm-up
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    _, rec = cgls_solve(w32, bd, x_ex=x_ex,
                        cfg=SolverConfig(max_iterations=3000, residual_tolerance=1e-4))
    torch.cuda.synchronize(dev)
    t_cgls = time.perf_counter() - t0
    out["cgls"] = {"iterations": rec.iterations[-1], "status": rec.status,
                   "rel_err_l2": rec.rel_err_l2[-1]}
    op = normal_operator(w32, 0.0)
    f = w32.T @ bd
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    # leaf Grams from the exact line weights (sparse kernel, per-rank angles)
    wexact = _projector(g, world, dev)
    h = build_wmg_hierarchy(wexact, n, 0.0, levels, node_mode="fast32")
    M = wmg_preconditioner(h)
    torch.cuda.synchronize(dev)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, rec = gmres_solve(op, f, precond=M, x_ex=x_ex, restart=100,
                         cfg=SolverConfig(max_iterations=300, residual_tolerance=1e-4))
    torch.cuda.synchronize(dev)
    t_gm = time.perf_counter() - t0
    t_cgls, t_setup, t_gm = _max_over_ranks([t_cgls, t_setup, t_gm], dev)
    out["cgls"]["seconds"] = t_cgls
    out["wmg_gmres"] = {"seconds": t_gm, "setup_seconds": t_setup,
                        "iterations": rec.iterations[-1], "status": rec.status,
                        "rel_err_l2": rec.rel_err_l2[-1], "levels": levels,
                        "leaves": 4 ** (levels - 1),
                        "leaf_dim": (n >> (levels - 1)) ** 2}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------ config 4
def run_config4(args):
    """BASELINE config 4 (slice-stack throughput): independent 2048^2 slices,
    1024 angles, 2897 detectors, float32 projector / float64 Krylov; slice k has
    its own 30-ellipse phantom (seed 4000 + k) and 0.5 % Gaussian noise (seed
    4500 + k).  Slices are dealt to ranks (k -> k mod N, no collective); each
    slice is solved to normal-equations residual 1e-4.  WMG with 5 levels is
    not runnable as specified (256 coarse blocks of 16384^2 = 550 GB of dense
    factors), so the solver here is CGLS; value = slices / second over the
    timed slices (max over ranks)."""
    import torch
    import torch.distributed as dist
    from paper_1310_0956_b200 import (SolverConfig, add_gaussian_noise, build_geometry,
                                      build_projector, cgls_solve, random_ellipses)
    world, rank, dev = _dist_init()
    n = args.n if args.n != 4096 else 2048
    m = int(round(1024 * n / 2048))
    m += m % 2
    d = int(math.ceil(n * math.sqrt(2.0)))
    g = build_geometry(n, d, m)
    w = build_projector(g, precision="float32", device=dev)
    mine = [k for k in range(args.slices) if k % world == rank]
    data = []
    for k in mine:
        x_ex = random_ellipses(n, 30, seed=4000 + k)
        b = add_gaussian_noise(w @ x_ex, 0.005, seed=4500 + k)
        data.append(torch.from_numpy(b).to(dev))
    cfg = SolverConfig(max_iterations=2000, residual_tolerance=1e-4)
    # Independent slices run as S concurrent solves, one host thread and one CUDA
    # stream each, every solve with its own projector instance (own workspace and
    # captured iteration graph): one slice's forward overlaps another's
    # backprojection, as the pair's two products do in the config-3 bench.
    S = max(1, min(args.streams, len(data)))
    ws_ = [w] + [build_projector(g, precision="float32", device=dev) for _ in range(S - 1)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(S)]
    if S > 1:                       # concurrent solves: the forward's throughput dispatch
        for wi in ws_:
            wi.prefer_concurrent(True)
    for i in range(S):                                                  # warm-up / capture
        with torch.cuda.stream(streams[i]):
            cgls_solve(ws_[i], data[i], cfg=SolverConfig(max_iterations=3))
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    iters = [0] * len(data)
    errors = []

    def worker(i):
        try:
            torch.cuda.set_device(dev)
            with torch.cuda.stream(streams[i]):
                for k in range(i, len(data), S):
                    _, rec = cgls_solve(ws_[i], data[k], cfg=cfg)
                    iters[k] = rec.iterations[-1]
            streams[i].synchronize()
        except Exception as exc:          # pragma: no cover - surfaced below
            errors.append(exc)

    import threading
    t0 = time.perf_counter()
    threads = [threading.Thread(target=worker, args=(i,)) for i in range(S)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    torch.cuda.synchronize(dev)
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    t = float(dt.item())
    # ---- WMG-CGLS on the same slices: the hierarchy (leaf Grams + inverses)
    # is built once per geometry and shared by every slice; 5 levels would need
    # 256 dense 16384^2 coarse factors (550 GB fp64, 275 GB packed), so the
    # documented variant uses 6 levels: 1024 leaves of 4096^2, 69 GB packed.
    levels = args.levels or 6
    wmg = None
    if args.wmg_slices > 0:
        from paper_1310_0956_b200 import build_wmg_hierarchy, wmg_preconditioner
        wex = build_projector(g, device=dev)                 # exact weights for the Grams
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        h = build_wmg_hierarchy(wex, n, 0.0, levels, nu_pre=2, nu_post=2, node_mode="fast32")
        M = wmg_preconditioner(h)
        torch.cuda.synchronize(dev)
        t_setup = time.perf_counter() - t0
        del wex
        wslices = [k for k in range(args.wmg_slices) if k % world == rank]
        witers, wtimes = [], []
        for k in wslices:
            bk = data[mine.index(k)] if k in mine else torch.from_numpy(add_gaussian_noise(
                w @ random_ellipses(n, 30, seed=4000 + k), 0.005, seed=4500 + k)).to(dev)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            _, rec = cgls_solve(w, bk, precond=M, cfg=SolverConfig(max_iterations=200,
                                                                   residual_tolerance=1e-4))
            torch.cuda.synchronize(dev)
            wtimes.append(time.perf_counter() - t0)
            witers.append(rec.iterations[-1])
        tw = sum(wtimes)
        tw, t_setup = _max_over_ranks([tw, t_setup], dev)
        wmg = {"solver": "WMG-CGLS (flexible PCG-NE), %d levels, nu = 2+2, fp32 node "
                         "systems, packed leaf inverses" % levels,
               "slices_timed": args.wmg_slices, "seconds": tw,
               "slices_per_s": args.wmg_slices / tw if tw > 0 else None,
               "setup_seconds_once": t_setup, "iterations_rank0": witers,
               "seconds_per_slice_rank0": wtimes,
               "leaves": 4 ** (levels - 1), "leaf_dim": (n >> (levels - 1)) ** 2,
               "deviation": "levels = %d instead of 5: 5 levels -> 256 dense 16384^2 "
                            "coarse factors, 550 GB fp64 (275 GB packed) > 180 GB HBM"
                            % levels}
    if rank == 0:
        print(json.dumps({
            "metric": "config4 slices/s", "value": args.slices / t, "unit": "slices/s",
            "n_gpus": world, "slices_timed": args.slices, "seconds": t, "n": n,
            "n_angles": m, "n_detectors": d, "solver": "CGLS to rel. residual 1e-4",
            "iterations_rank0": iters, "scaling": "weak (slices dealt round-robin)",
            "concurrent_solves": S, "wmg_cgls": wmg,
            "data": "synthetic: 30-ellipse phantoms, 0.5 % Gaussian noise"}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _relaunch_under_torchrun(args):
    """``--gpus N`` (N > 1) without torchrun: re-run this command as N ranks,
    one process per GPU (torch.distributed.run, NCCL, rendezvous on
    127.0.0.1); rank 0 prints the JSON line.  Returns the launcher's exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")       # NCCL init lines show the rank count
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    print(f"[bench] --gpus {args.gpus}: launching {args.gpus} ranks: {' '.join(cmd)}",
          file=sys.stderr, flush=True)
    return subprocess.run(cmd, env=env).returncode


def _check_world(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return world


def run_launch_check(args):
    """``--workload launch-check``: rendezvous only (CPU-testable with
    WMG_BENCH_BACKEND=gloo): every rank joins the process group, rank 0 prints
    the world size the bench would time."""
    import torch.distributed as dist
    world = _check_world(args)
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group(os.environ.get("WMG_BENCH_BACKEND", "nccl"))
        ranks = [None] * world
        dist.all_gather_object(ranks, rank)
        dist.destroy_process_group()
    else:
        ranks = [0]
    if rank == 0:
        print(json.dumps({"workload": "launch-check", "n_gpus": world, "ranks": ranks}),
              flush=True)
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch_under_torchrun(args)
    _check_world(args)
    if args.workload == "launch-check":
        return run_launch_check(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "config2":
        return run_config2(args)
    if args.workload == "config4":
        return run_config4(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
