"""Numpy restatements of the solver layer -- TEST INFRASTRUCTURE ONLY.

Each function follows the reference algorithm line for line where one exists
(/root/reference/pkg/src/wmgtomo/solvers.py) and uses the deterministic DET_SUM
reduction (same chunking and fixed tree as csrc/vecops.cu) for every dot and
norm, so the GPU solvers can be checked against it bit for bit:

  sirt_solve      <- solvers.py:95-137 (update order identical; norms DET)
  normal_operator <- solvers.py:140-156
  bicgstab_solve  <- solvers.py:159-243 (dots DET)
  cgls_solve      <- new, the definition in
                     paper_1310_0956_b200/solvers.py:cgls_solve
  gmres_solve     <- new, same definition as the GPU version
"""
from __future__ import annotations

import numpy as np

BREAKDOWN_REL_TOL = 1e-14


# ------------------------------------------------------------------ DET_SUM
def det_sum(v) -> float:
    """Chunked deterministic sum (csrc/vecops.cu): 1024-element chunks, lane l
    sums v[c*1024 + k*32 + l] over k sequentially, then the tree
    s[l] += s[l+off] for off = 16..1; repeat on the chunk sums."""
    v = np.asarray(v, dtype=np.float64).ravel()
    if v.size == 0:
        return 0.0
    while True:
        C = -(-v.size // 1024)
        pad = np.zeros(C * 1024)
        pad[: v.size] = v
        X = pad.reshape(C, 32, 32)
        s = X[:, 0, :].copy()
        for k in range(1, 32):
            s = s + X[:, k, :]
        off = 16
        while off >= 1:
            s = s[:, :off] + s[:, off:2 * off]
            off //= 2
        v = s[:, 0]
        if C == 1:
            return float(v[0])


def det_dot(a, b) -> float:
    return det_sum(np.asarray(a) * np.asarray(b))


def det_sq(a) -> float:
    a = np.asarray(a)
    return det_sum(a * a)


def det_norm(a) -> float:
    return float(np.sqrt(det_sq(a)))


# ---------------------------------------------------------------- records
class Record:
    def __init__(self):
        self.iterations, self.rel_residual = [], []
        self.rel_err_l2, self.rel_err_linf = [], []
        self.status = "max-iterations"

    def log(self, k, rel, e2, einf):
        self.iterations.append(int(k))
        self.rel_residual.append(float(rel))
        self.rel_err_l2.append(e2)
        self.rel_err_linf.append(einf)


class _Err:
    def __init__(self, x_ex):
        self.x_ex = None if x_ex is None else np.asarray(x_ex, dtype=np.float64)
        if self.x_ex is not None:
            self.n2 = float(np.sqrt(det_sq(self.x_ex)))
            self.ninf = float(np.abs(self.x_ex).max())

    def __call__(self, x):
        if self.x_ex is None:
            return None, None
        e = x - self.x_ex
        return float(np.sqrt(det_sq(e)) / self.n2), float(np.abs(e).max() / self.ninf)


# ------------------------------------------------------------------- SIRT
def sirt_scaling(w):
    from . import cproj
    rows = cproj.row_sums(w)
    cols = w.T @ np.ones(w.shape[0])
    with np.errstate(divide="ignore"):
        r = np.where(rows > 0, 1.0 / rows, 0.0)
        c = np.where(cols > 0, 1.0 / cols, 0.0)
    return c, r


def sirt_solve(w, b, x0, max_iterations, tol=0.0, lam=0.0, x_ex=None):
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros(w.shape[1]) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    c, r = sirt_scaling(w)
    wt = w.T.tocsr()
    err = _Err(x_ex)
    rec = Record()
    res = b - w @ x
    n0 = det_norm(res)
    rec.log(0, 1.0, *err(x))
    if n0 == 0.0:
        rec.status = "converged"
        return x, rec
    for k in range(1, max_iterations + 1):
        update = c * (wt @ (r * res))
        if lam > 0:
            update -= lam * (c * x)
        x += update
        res = b - w @ x
        rel = det_norm(res) / n0
        rec.log(k, rel, *err(x))
        if tol > 0 and rel < tol:
            rec.status = "converged"
            return x, rec
    return x, rec


def normal_operator(w, lam):
    wt = w.T.tocsr()

    def op(v):
        out = wt @ (w @ v)
        if lam != 0:
            out = out + lam * v
        return out
    return op


# --------------------------------------------------------------- BiCGStab
def bicgstab_solve(op, f, precond=None, x0=None, max_iterations=100, tol=0.0, x_ex=None):
    f = np.asarray(f, dtype=np.float64)
    x = np.zeros_like(f) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    minv = (lambda v: v) if precond is None else precond
    err = _Err(x_ex)
    rec = Record()
    r = f - op(x)
    n0 = det_norm(r)
    rec.log(0, 1.0, *err(x))
    if n0 == 0.0:
        rec.status = "converged"
        return x, rec
    r_hat = r.copy()
    r_hat_norm = n0
    rho_prev = alpha = omega = 1.0
    v = p = np.zeros_like(r)
    r_norm = n0
    for k in range(1, max_iterations + 1):
        rho = det_dot(r_hat, r)
        if abs(rho) <= BREAKDOWN_REL_TOL * r_hat_norm * r_norm:
            rec.status = "breakdown"
            return x, rec
        if k == 1:
            p = r.copy()
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            p = r + beta * (p - omega * v)
        p_hat = minv(p)
        v = op(p_hat)
        denom = det_dot(r_hat, v)
        if abs(denom) <= BREAKDOWN_REL_TOL * r_hat_norm * float(np.sqrt(det_sq(v))):
            rec.status = "breakdown"
            return x, rec
        alpha = rho / denom
        s = r - alpha * v
        s_hat = minv(s)
        t = op(s_hat)
        tt = det_sq(t)
        if tt < BREAKDOWN_REL_TOL ** 2 * n0 ** 2:
            x = x + alpha * p_hat
            r = s
            rec.log(k, det_norm(r) / n0, *err(x))
            rec.status = "converged"
            return x, rec
        omega = det_dot(t, s) / tt
        x = x + alpha * p_hat + omega * s_hat
        r = s - omega * t
        rho_prev = rho
        r_norm = det_norm(r)
        rel = r_norm / n0
        rec.log(k, rel, *err(x))
        if tol > 0 and rel < tol:
            rec.status = "converged"
            return x, rec
        if abs(omega) < BREAKDOWN_REL_TOL:
            rec.status = "breakdown"
            return x, rec
    return x, rec


# ------------------------------------------------------------------- CGLS
def cgls_solve(w, b, precond=None, x0=None, max_iterations=100, tol=0.0, lam=0.0, x_ex=None):
    b = np.asarray(b, dtype=np.float64)
    wt = w.T.tocsr()
    x = np.zeros(w.shape[1]) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    err = _Err(x_ex)
    rec = Record()
    r = b - w @ x
    s = wt @ r
    if lam != 0:
        s = s - lam * x
    if precond is None:
        z = s
        gamma = det_sq(s)
        s0 = float(np.sqrt(gamma))
    else:
        z = precond(s)
        s0 = det_norm(s)
        gamma = det_dot(z, s)
    p = z.copy()
    rec.log(0, 1.0, *err(x))
    if s0 == 0.0:
        rec.status = "converged"
        return x, rec
    for k in range(1, max_iterations + 1):
        q = w @ p
        delta = det_sq(q) + lam * det_sq(p) if lam != 0 else det_sq(q)
        if delta <= 0.0 or not np.isfinite(delta):
            rec.status = "breakdown"
            return x, rec
        alpha = gamma / delta
        x = x + alpha * p
        r = r - alpha * q
        s_old = s
        s = wt @ r
        if lam != 0:
            s = s - lam * x
        if precond is None:
            gnew = det_sq(s)
            snorm = float(np.sqrt(gnew))
        else:
            z = precond(s)
            snorm = det_norm(s)
            gnew = det_dot(z, s)
            pr = det_sum(z * (s - s_old))
        rel = snorm / s0
        rec.log(k, rel, *err(x))
        if tol > 0 and rel < tol:
            rec.status = "converged"
            return x, rec
        if precond is None:
            beta = gnew / gamma
            gamma = gnew
            p = 1.0 * s + beta * p
        else:
            beta = pr / gamma
            gamma = gnew
            p = 1.0 * z + beta * p
        if gamma == 0.0:
            rec.status = "converged"
            return x, rec
    return x, rec


# ------------------------------------------------------------------ GMRES
def gmres_solve(op, f, precond=None, x0=None, max_iterations=100, tol=0.0, x_ex=None,
                restart=100):
    f = np.asarray(f, dtype=np.float64)
    n = f.size
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    minv = (lambda v: v) if precond is None else precond
    err = _Err(x_ex)
    rec = Record()
    m = int(restart)
    r = f - op(x)
    beta = det_norm(r)
    n0 = beta
    rec.log(0, 1.0, *err(x))
    if n0 == 0.0:
        rec.status = "converged"
        return x, rec
    k = 0
    while True:
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        V[0] = (1.0 / beta) * r
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        stop = None
        for j in range(m):
            k += 1
            zj = minv(V[j])
            Z[j] = zj
            wv = np.array(op(zj), dtype=np.float64, copy=True)
            hcol = np.zeros(j + 2)
            for _ in range(2):
                hh = np.array([det_dot(V[i], wv) for i in range(j + 1)])
                for i in range(j + 1):
                    wv = wv - hh[i] * V[i]
                hcol[: j + 1] += hh
            hn = det_norm(wv)
            hcol[j + 1] = hn
            for i in range(j):
                a_, b_ = hcol[i], hcol[i + 1]
                hcol[i] = cs[i] * a_ + sn[i] * b_
                hcol[i + 1] = -sn[i] * a_ + cs[i] * b_
            den = np.hypot(hcol[j], hcol[j + 1])
            cs[j] = hcol[j] / den if den else 1.0
            sn[j] = hcol[j + 1] / den if den else 0.0
            hcol[j] = den
            hcol[j + 1] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            H[: j + 2, j] = hcol
            rel = abs(g[j + 1]) / n0
            happy = hn == 0.0
            if not happy:
                V[j + 1] = (1.0 / hn) * wv
            last = k >= max_iterations or happy or (tol > 0 and rel < tol)
            if err.x_ex is not None or last or j == m - 1:
                jd = j + 1
                y = np.linalg.solve(np.triu(H[:jd, :jd]), g[:jd])
                xk = x.copy()
                basis = V if precond is None else Z
                for i in range(jd):
                    xk = xk + y[i] * basis[i]
                rec.log(k, rel, *err(xk))
                if last or j == m - 1:
                    x = xk
                    if happy or (tol > 0 and rel < tol):
                        stop = "converged"
                    elif k >= max_iterations:
                        stop = "max-iterations"
                    break
            else:
                rec.log(k, rel, None, None)
        if stop is not None:
            rec.status = stop
            return x, rec
        r = f - op(x)
        beta = det_norm(r)
        if beta == 0.0:
            rec.status = "converged"
            return x, rec
