"""Numpy restatement of the reference IRL eigensolver (TEST INFRASTRUCTURE ONLY).

Algorithm of /root/reference/pkg/src/irlnqs/krylov.py: Lanczos with full
reorthogonalisation applied twice (kry:87-116), tridiagonal eigensolve by
LAPACK (kry:151-162), implicit shifted-QR restart (kry:165-256) and the k = 1
IRL driver (kry:268-345), restated as a small state machine.  Used to check
the device driver's Ritz value, matvec count and direction, and as the CPU
baseline's solver.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.linalg import eigh_tridiagonal

TOL_BREAK = 1e-12  # kry:19


class Counted:
    """kry:74-84: product counter with the float cast and the finiteness guard."""

    def __init__(self, fn):
        self.fn = fn
        self.n = 0

    def __call__(self, v):
        self.n += 1
        out = np.asarray(self.fn(v), dtype=float)
        if not np.isfinite(out).all():
            raise ValueError("matvec returned non-finite values")
        return out


def tri_eig(alpha, beta):
    """kry:151-162."""
    if len(alpha) == 1:
        return np.array([alpha[0]]), np.ones((1, 1))
    try:
        return eigh_tridiagonal(np.asarray(alpha, float), np.asarray(beta, float))
    except np.linalg.LinAlgError:
        t = np.diag(alpha) + np.diag(beta, 1) + np.diag(beta, -1)
        return np.linalg.eigh(t)


def grow(apply, rows, alpha, beta, m, reorth=True):
    """kry:87-116. rows/alpha/beta are extended in place; returns (f, breakdown)."""
    big = max([abs(x) for x in alpha] + [abs(x) for x in beta] + [0.0])
    while len(alpha) < m:
        q = rows[-1]
        r = apply(q)
        a = float(q @ r)
        alpha.append(a)
        r = r - a * q
        if len(rows) > 1:
            r = r - beta[-1] * rows[-2]
        if reorth:
            basis = np.array(rows)
            r = r - basis.T @ (basis @ r)
            r = r - basis.T @ (basis @ r)
        nrm = float(np.linalg.norm(r))
        big = max(big, abs(a), nrm)
        if len(alpha) == m:
            return r, False
        if nrm <= TOL_BREAK * max(1.0, big):
            return r, True
        beta.append(nrm)
        rows.append(r / nrm)
    return np.zeros_like(rows[0]), False


def qr_sweeps(alpha, beta, shifts):
    """kry:165-190 applied for every shift: returns (T', Q) with T' = Q^T T Q."""
    m = len(alpha)
    t = np.diag(np.asarray(alpha, float))
    if m > 1:
        t = t + np.diag(beta, 1) + np.diag(beta, -1)
    q = np.eye(m)
    for mu in shifts:
        x, z = t[0, 0] - mu, t[1, 0]
        for k in range(m - 1):
            r = math.hypot(x, z)
            c, s = (1.0, 0.0) if r == 0.0 else (x / r, z / r)
            for mat, cols in ((t, False), (t, True), (q, True)):
                a0 = (mat[:, k] if cols else mat[k, :]).copy()
                a1 = (mat[:, k + 1] if cols else mat[k + 1, :]).copy()
                if cols:
                    mat[:, k], mat[:, k + 1] = c * a0 + s * a1, -s * a0 + c * a1
                else:
                    mat[k, :], mat[k + 1, :] = c * a0 + s * a1, -s * a0 + c * a1
            if k < m - 2:
                x, z = t[k + 1, k], t[k + 2, k]
    return t, q


def restart(rows, alpha, beta, f, shifts, k):
    """kry:193-256 (without the collision warning): compact to order k.
    Returns (kept rows (k x n), v_next or None, alpha_k, beta_{k-1}, beta_k)."""
    m = len(alpha)
    ritz, _ = tri_eig(alpha, beta)
    spread = float(ritz[-1] - ritz[0]) or 1.0
    shifts = np.array(shifts, float)
    kept = np.array([r for r in ritz if np.min(np.abs(shifts - r)) > 0])
    for i in range(len(shifts)):
        if kept.size and np.min(np.abs(kept - shifts[i])) < 1e-14 * spread:
            shifts[i] += 1e-12 * spread
    t, q = qr_sweeps(alpha, beta, shifts)
    rot = q.T @ np.array(rows)
    f_new = rot[k] * t[k, k - 1] + f * q[m - 1, k - 1]
    bk = float(np.linalg.norm(f_new))
    a_new = np.diag(t)[:k].copy()
    b_new = np.diag(t, -1)[: k - 1].copy()
    keep = rot[:k].copy()
    nxt = f_new / bk if bk > 0 else None
    sgn = 1.0
    for i in range(k - 1):
        if b_new[i] < 0:
            sgn = -sgn
        b_new[i] = abs(b_new[i])
        keep[i + 1] *= sgn
    if sgn < 0 and nxt is not None:
        nxt = -nxt
    return keep, nxt, a_new, b_new, bk


def lowest(rows, alpha, beta):
    """kry:259-265."""
    vals, vecs = tri_eig(alpha, beta)
    u = vecs[:, 0]
    y = np.array(rows).T @ u
    return float(vals[0]), y / np.linalg.norm(y), float(abs(u[-1]))


def irl(matvec, dim, m=20, tol=1e-12, max_restarts=300, seed=0):
    """kry:268-345 -> dict(value, vector, residual, converged, n_matvec, n_restarts)."""
    if dim < 1:
        raise ValueError("problem dimension must be positive")
    apply = Counted(matvec)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(dim)
    rows = [x / np.linalg.norm(x)]
    alpha, beta = [], []
    me = min(m, dim)
    f, broke = grow(apply, rows, alpha, beta, me)
    best = None
    for it in range(max_restarts + 1):
        lam, y, ul = lowest(rows, alpha, beta)
        fn = float(np.linalg.norm(f))
        cheap = 0.0 if broke else fn * ul
        if cheap <= tol or broke or it == max_restarts:
            res = float(np.linalg.norm(apply(y) - lam * y))
            cand = dict(value=lam, vector=y, residual=res, converged=res <= tol, n_matvec=apply.n, n_restarts=it)
            if best is None or res < best["residual"]:
                best = cand
            if cand["converged"] or it == max_restarts:
                return cand if cand["converged"] else best
            if broke:
                z = y + 1e-8 * rng.standard_normal(dim)
                rows, alpha, beta = [z / np.linalg.norm(z)], [], []
                f, broke = grow(apply, rows, alpha, beta, me)
                continue
        vals, _ = tri_eig(alpha, beta)
        keep, nxt, a_new, _, bk = restart(rows, alpha, beta, f, vals[1:], 1)
        rows, alpha, beta = [keep[0]], [float(a_new[0])], []
        if nxt is None:
            broke = True
            f = np.zeros(dim)
            continue
        rows.append(nxt)
        beta.append(bk)
        f, broke = grow(apply, rows, alpha, beta, me)
    return best
