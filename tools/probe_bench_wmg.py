"""Run bench.run_wmg_cgls twice in one process (timing sanity check)."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda", 0)
for k in range(2):
    r = bench.run_wmg_cgls(dev)
    print(k, {kk: r[kk] for kk in ("seconds", "setup_seconds", "cgls_seconds", "iterations")},
          r["nu0"], flush=True)
