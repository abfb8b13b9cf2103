"""Numpy RBM / shallow-MLP rows and log psi (TEST INFRASTRUCTURE ONLY).

The reference has no RBM/MLP; these rows follow BASELINE.json's
north star and SURVEY §8(a) A2 and are pinned by central finite differences
of ``log_psi`` (step 1e-6, the T/test_ansatz.py:67-81 pattern) and, for the
MLP, by the reference's phase-head gradient (ans:278-288, see make_golden.py).
Inputs are 0/1 occupations.
"""

from __future__ import annotations

import numpy as np


def rbm_split(theta, n, h):
    return theta[:n], theta[n : n + h], theta[n + h :].reshape(h, n)


def mlp_split(theta, n, h):
    w = theta[: h * n].reshape(h, n)
    b = theta[h * n : h * n + h]
    u = theta[h * n + h : h * n + 2 * h]
    c = theta[h * n + 2 * h]
    return w, b, u, c


def rbm_hidden(theta, x, n, h):
    _, b, w = rbm_split(theta, n, h)
    return np.tanh(b + x.astype(float) @ w.T)


def mlp_hidden(theta, x, n, h):
    w, b, u, _ = mlp_split(theta, n, h)
    t = np.tanh(b + x.astype(float) @ w.T)
    return t, u * (1.0 - t * t)


def rbm_rows(theta, x, n, h):
    """[x (n), tanh theta (h), (tanh theta_j x_i)_{j,i} (h n)]."""
    xf = x.astype(float)
    t = rbm_hidden(theta, x, n, h)
    outer = (t[:, :, None] * xf[:, None, :]).reshape(len(x), h * n)
    return np.concatenate([xf.astype(t.dtype), t, outer], axis=1)


def mlp_rows(theta, x, n, h):
    """[(g_j x_k)_{j,k} (h n), g (h), t (h), 1]."""
    xf = x.astype(float)
    t, g = mlp_hidden(theta, x, n, h)
    outer = (g[:, :, None] * xf[:, None, :]).reshape(len(x), h * n)
    return np.concatenate([outer, g, t, np.ones((len(x), 1))], axis=1)


def rbm_log_psi(theta, x, n, h):
    a, b, w = rbm_split(theta, n, h)
    xf = x.astype(float)
    return xf @ a + np.sum(np.log(np.cosh(b + xf @ w.T)), axis=-1)


def mlp_log_psi(theta, x, n, h):
    w, b, u, c = mlp_split(theta, n, h)
    return np.tanh(b + x.astype(float) @ w.T) @ u + c


def fd_rows(log_psi, theta, x, step=1e-6, holomorphic=False):
    """Central finite differences of log psi for every parameter (small cases)."""
    p = len(theta)
    out = np.zeros((len(x), p), dtype=complex if holomorphic else float)
    for k in range(p):
        tp = theta.copy()
        tm = theta.copy()
        tp[k] += step
        tm[k] -= step
        out[:, k] = (log_psi(tp, x) - log_psi(tm, x)) / (2 * step)
    return out
