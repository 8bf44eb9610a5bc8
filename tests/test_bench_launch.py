"""``bench.py --gpus N`` really runs N ranks (CPU, gloo): without an external
torchrun the bench re-launches itself under torch.distributed.run with N
processes (rendezvous on 127.0.0.1), and a WORLD_SIZE that disagrees with
--gpus is refused."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ, WMG_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=300)


def test_gpus_two_relaunches_two_ranks():
    r = _run(["--gpus", "2", "--workload", "launch-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and sorted(d["ranks"]) == [0, 1]
    assert "torch.distributed.run" in r.stderr


def test_world_size_mismatch_is_refused():
    r = _run(["--gpus", "4", "--workload", "launch-check"],
             {"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in (r.stderr + r.stdout)
