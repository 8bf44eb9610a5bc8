"""Leaf-Gram assembly: sparse (wmg_leaf_gram) vs dense (parity P_L + DGEMM)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402
from paper_1310_0956_b200.multilevel import _assemble_leaf_grams, _leaf_paths  # noqa: E402


def wall(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0, r


out = {}
for name, (n, d, m, levels, nleaf) in {"cfg1": (256, 363, 180, 3, None),
                                       "cfg2": (1024, 1449, 720, 5, 4)}.items():
    w = build_projector(build_geometry(n, d, m))
    paths = _leaf_paths(levels)
    if nleaf:
        paths = paths[:nleaf]
    _assemble_leaf_grams(w, n, 0.0, levels, paths=paths[:1], method="sparse")   # warm-up
    ts, (_, gs) = wall(lambda: _assemble_leaf_grams(w, n, 0.0, levels, paths=paths,
                                                    method="sparse"))
    td, (_, gd) = wall(lambda: _assemble_leaf_grams(w, n, 0.0, levels, paths=paths,
                                                    method="dense"))
    err = ((gs - gd).abs().amax(dim=(1, 2)) / gd.abs().amax(dim=(1, 2))).max().item()
    out[name] = {"leaves": len(paths), "sparse_s": ts, "dense_s": td,
                 "sparse_per_leaf_ms": ts / len(paths) * 1e3, "max_rel_err": err}
    del gs, gd
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
