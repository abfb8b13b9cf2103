"""Bordered IRL-SR operator and update direction (TEST INFRASTRUCTURE ONLY).

Restates /root/reference/pkg/src/irlnqs/optimizer.py:138-165 for a synthetic
batch (no Hamiltonian partners, so the heff_offdiag term is zero), plus the
real embedding of the complex-parameter (Hermitian) problem of SURVEY §8(c).
"""

from __future__ import annotations

import numpy as np

from . import estimators as est
from . import krylov


def batch_seed(seed: int, step: int) -> int:
    """opt:100-101."""
    return (seed * 1_000_003 + step) % 2**31


def real_problem(w, e, o, n_samples):
    """(matvec, dim, gradient, mean) for real theta (opt:134-148)."""
    mean, _, _ = est.energy(w, e, n_samples)
    grad = est.gradient(w, e, o, mean)
    half = 0.5 * grad
    p = o.shape[1]

    def matvec(u):
        out = np.empty(p + 1)
        out[0] = half @ u[1:]
        out[1:] = u[0] * half + est.heff(w, e, o, mean, u[1:])
        return out

    return matvec, p + 1, grad, mean


def embedded_problem(w, e, o, n_samples):
    """Complex theta via the real embedding [O, iO]:
    heff on Re(e), gradient on the complex e; dim 2P + 1."""
    mean, _, _ = est.energy(w, e, n_samples)
    emb = np.concatenate([o, 1j * o], axis=1)
    grad = est.gradient(w, e, emb, mean)
    half = 0.5 * grad
    q = emb.shape[1]
    e_re = e.real

    def matvec(u):
        out = np.empty(q + 1)
        out[0] = half @ u[1:]
        out[1:] = u[0] * half + est.heff(w, e_re, emb, mean, u[1:])
        return out

    return matvec, q + 1, grad, mean


def direction(vec, grad):
    """opt:160-165."""
    c0 = vec[0]
    d = vec[1:]
    if abs(c0) > 1e-12:
        return d / c0
    return -d if float(grad @ d) > 0 else d


def solve(matvec, dim, grad, m, tol=1e-12, max_restarts=3, seed=0):
    pair = krylov.irl(matvec, dim, m=m, tol=tol, max_restarts=max_restarts, seed=seed)
    return pair, direction(pair["vector"], grad)


def structured_problem(sp, e, n_samples):
    """(matvec, dim, gradient, mean) of opt:134-148 at full size from the
    structured products of oracle/structured.py (real theta), or of the real
    embedding for complex theta, dim 2P + 1."""
    w = sp.w
    mean, _, _ = est.energy(w, e, n_samples)
    g = sp.colsum(w * (e - mean))  # sum w (e - E) conj(O) (= est:162 expanded form)
    coeff = w * (e - mean).real
    p = sp.p
    if np.iscomplexobj(g):
        grad = 2.0 * np.concatenate([g.real, g.imag])
        half = 0.5 * grad

        def matvec(u):
            out = np.empty(2 * p + 1)
            out[0] = half @ u[1:]
            hv = sp.product(coeff, u[1 : p + 1] + 1j * u[p + 1 :])
            out[1:] = u[0] * half + np.concatenate([hv.real, hv.imag])
            return out

        return matvec, 2 * p + 1, grad, mean
    grad = 2.0 * g.real
    half = 0.5 * grad

    def matvec(u):
        out = np.empty(p + 1)
        out[0] = half @ u[1:]
        out[1:] = u[0] * half + sp.product(coeff, u[1:])
        return out

    return matvec, p + 1, grad, mean
