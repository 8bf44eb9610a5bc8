"""Restatement of the reference WMG hierarchy and V-cycle on the CPU --
TEST INFRASTRUCTURE ONLY (checker and timed CPU baseline).

Follows /root/reference/pkg/src/wmgtomo/multilevel.py:
  haar_scaling_1d / haar_wavelet_1d / build_intergrid_set  (:36-79)
  node factors P_child = P R_band^T with the 1e-15 drop     (:123-148, sparse_kernels.py:30-39)
  leaf Gram P^T P + lam I, lower Cholesky                    (:125-130, sparse_kernels.py:53-65)
  wtg_apply hybrid / multiplicative                          (:175-198)
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
        self.children = {}
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


def build_hierarchy(w, n, lam, levels):
    return Node(w.tocsr(), n, 1, levels, lam, "")


def _solve(node, r, mult):
    if node.lower is not None:
        return scipy.linalg.cho_solve((node.lower, True), r, check_finite=False)
    return wtg_apply(node, r, mult)


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
    return lambda v: wtg_apply(root, np.asarray(v, dtype=np.float64), multiplicative)
