"""Restatement of the reference WMG hierarchy and V-cycle on the CPU --
TEST INFRASTRUCTURE ONLY (checker and timed CPU baseline).

Follows /root/reference/pkg/src/wmgtomo/multilevel.py:
  haar_scaling_1d / haar_wavelet_1d / build_intergrid_set  (:36-79)
  node factors P_child = P R_band^T with the 1e-15 drop     (:123-148, sparse_kernels.py:30-39)
  leaf Gram P^T P + lam I, lower Cholesky                    (:125-130, sparse_kernels.py:53-65)
  wtg_apply hybrid / multiplicative                          (:175-198)
  + the SIRT-type node smoother of the WMG-CGLS configurations (BASELINE
    configs 1/2/4 "2+2 SIRT sweeps per level"; NOT defined by the reference,
    whose only sweep is the TG smoother at :241-242 -- SURVEY.md s8 a16
    option (ii)), restating paper_1310_0956_b200/multilevel.py's definition:
      C_p = 1 / (2^-k * block sums of W's column sums)   (zero -> 0)
      omega_p = 0.95 / lambda_max(C_p A_p), 10 power iterations from the fixed
                start vector v_i = 1 + ((7919 i) mod 1013) / 1013, DET_SUM
                norms / dots (oracle/solvers.py)
      node solve: nu_pre sweeps z += omega_p C_p (r - A_p z) from z = 0, the
                wavelet two-grid correction of the residual, nu_post sweeps.
Leaf factors are kept Fortran-ordered so cho_solve does not copy them (the
reference's C-ordered factors make each solve ~20x slower; the
arithmetic is identical).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse as sp

BANDS = ("LL", "LH", "HL", "HH")
DROP = 1e-15


def intergrid(n):
    h = n // 2
    rows = np.repeat(np.arange(h), 2)
    cols = np.arange(n)
    s = sp.csr_matrix((np.full(n, 1.0 / np.sqrt(2.0)), (rows, cols)), shape=(h, n))
    j = sp.csr_matrix((np.tile([1.0, -1.0], h) / np.sqrt(2.0), (rows, cols)), shape=(h, n))
    return {"LL": sp.kron(s, s, format="csr"), "LH": sp.kron(j, s, format="csr"),
            "HL": sp.kron(s, j, format="csr"), "HH": sp.kron(j, j, format="csr")}


def _spgemm(a, b):
    c = (a.tocsr() @ b.tocsr()).tocsr()
    if c.nnz:
        c.data[np.abs(c.data) < DROP] = 0.0
        c.eliminate_zeros()
    return c


class Node:
    def __init__(self, p, side, level, levels, lam, path):
        self.side, self.path, self.lam = side, path, lam
        self.depth = level - 1
        self.children = {}
        self.c = None
        self.omega = 0.0
        self.nu_pre = self.nu_post = 0
        if level == levels:
            gram = (p.T @ p).toarray()
            if lam != 0:
                gram[np.diag_indices_from(gram)] += lam
            self.lower = np.asfortranarray(scipy.linalg.cholesky(gram, lower=True))
            self.p = None
            return
        self.lower = None
        self.p = p
        self.pt = p.T.tocsr()
        self.grids = intergrid(side)
        for b in BANDS:
            child = _spgemm(p, self.grids[b].T)
            self.children[b] = Node(child, side // 2, level + 1, levels, lam,
                                    f"{path}/{b}" if path else b)

    def apply_system(self, v):
        out = self.pt @ (self.p @ v)
        if self.lam != 0:
            out = out + self.lam * v
        return out


def start_vector(dim):
    i = np.arange(dim, dtype=np.int64)
    return 1.0 + ((i * 7919) % 1013).astype(np.float64) / 1013.0


def _nodes(node):
    yield node
    for b in BANDS:
        if b in node.children:
            yield from _nodes(node.children[b])


def setup_smoothers(root, w, n, nu_pre, nu_post, power_iterations=10):
    from .solvers import det_dot, det_sq
    colsum = w.T @ np.ones(w.shape[0])            # bitwise the reference's W^T 1
    for nd in _nodes(root):
        if nd.lower is not None:
            continue
        k = nd.depth
        B = 1 << k
        blk = colsum.reshape(n // B, B, n // B, B).sum(axis=(1, 3)).reshape(-1)
        blk = blk * (0.5 ** k)
        with np.errstate(divide="ignore"):
            nd.c = np.where(blk > 0, 1.0 / blk, 0.0)
        v = start_vector(nd.side * nd.side)
        lam = None
        for _ in range(power_iterations):
            v = v / np.sqrt(det_sq(v))
            out = nd.apply_system(v) * nd.c
            lam = det_dot(v, out)
            v = out
        nd.omega = 0.95 / lam if lam > 0 else 0.0
        nd.nu_pre, nd.nu_post = nu_pre, nu_post


def build_hierarchy(w, n, lam, levels, nu_pre=0, nu_post=0):
    root = Node(w.tocsr(), n, 1, levels, lam, "")
    if nu_pre or nu_post:
        setup_smoothers(root, w, n, nu_pre, nu_post)
    return root


def _solve(node, r, mult):
    if node.lower is not None:
        return scipy.linalg.cho_solve((node.lower, True), r, check_finite=False)
    if node.nu_pre == 0 and node.nu_post == 0:
        return wtg_apply(node, r, mult)
    z = np.zeros_like(r)
    for _ in range(node.nu_pre):
        z = z + node.omega * (node.c * (r - node.apply_system(z)))
    if node.nu_pre:
        e = wtg_apply(node, r - node.apply_system(z), mult)
        z = z + e
    else:
        z = wtg_apply(node, r, mult)
    for _ in range(node.nu_post):
        z = z + node.omega * (node.c * (r - node.apply_system(z)))
    return z


def wtg_apply(node, r, multiplicative=False):
    g = node.grids
    e = g["LL"].T @ _solve(node.children["LL"], g["LL"] @ r, multiplicative)
    r_work = r - node.apply_system(e)
    for band in ("LH", "HL", "HH"):
        e = e + g[band].T @ _solve(node.children[band], g[band] @ r_work, multiplicative)
        if multiplicative and band != "HH":
            r_work = r - node.apply_system(e)
    return e


def preconditioner(root, multiplicative=False):
    # the root is an internal node: with nu = 0 this is exactly wtg_apply(root, v)
    return lambda v: _solve(root, np.asarray(v, dtype=np.float64), multiplicative)
