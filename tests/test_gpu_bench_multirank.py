"""bench.py's multi-rank path (torchrun, angle shards, max-over-ranks timing,
sharded WMG) exercised with two gloo ranks on the box's one GPU (host-side
collectives: no kernel waits on another rank).  The NCCL path differs only in
the process-group backend."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(args, timeout=600):
    env = dict(os.environ, WMG_BENCH_BACKEND="gloo", WMG_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py"] + args
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 prints one line
    return json.loads(lines[0])


def test_bench_pair_and_wmg_two_ranks(gpu):
    d = _torchrun(["--gpus", "2", "--steps", "2", "--warmup", "3", "--grid", "512",
                   "--no-cpu-baseline"])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["angle_sharding"] == "quad units"
    w = d["wmg_cgls"]
    assert w["n_gpus"] == 2 and w["status"] == "converged" and w["iterations"] == 15


def test_bench_config2_two_ranks(gpu):
    d = _torchrun(["--gpus", "2", "--workload", "config2", "--grid", "256", "--levels", "3"])
    assert d["n_gpus"] == 2 and d["cgls"]["status"] == "converged"
    assert d["wmg_gmres"]["status"] == "converged"
