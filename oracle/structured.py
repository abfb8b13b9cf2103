"""Full-size CPU products for the shallow NQS (TEST INFRASTRUCTURE ONLY).

The reference product (est:171-186, restated row by row in
``oracle/estimators.py``) needs the N x P matrix O, which is 61.5 GB (cfg4) or
110 GB (cfg5) at BASELINE sizes.  Its big block is an outer product (RBM:
``T_n (x) x_n``; MLP: ``g_n (x) x_n``, ``oracle/nqs.py``), so the same centred
products follow exactly from N x h and N x n matrices:

    O v        = x.v_a + T.v_b + sum_j T_nj (V_W x_n)_j            (RBM)
               = sum_j g_nj (V_W x_n)_j + g.v_b + t.v_u + v_c      (MLP)
    conj(O)^T y  blocks = X^T y, conj(T)^T y, (conj(T) * y)^T X     (RBM)

with ``Obar = w @ O`` formed the same way and the centring applied as
``O_c v = O v - Obar.v`` and ``O_c^H y = conj(O)^T y - conj(Obar) sum(y)``.
This is a restatement of est:166-186 in a different association order (numpy
BLAS GEMMs), not a copy of the device algorithm; ``tests/test_oracle_golden.py``
pins it to the row-based restatement on subsets.
"""

from __future__ import annotations

import numpy as np

from . import nqs


class RBMProducts:
    """Centred products of an RBM batch (real or complex theta)."""

    def __init__(self, theta, x, n, h, w):
        self.n, self.h = n, h
        self.a, self.b, self.W = nqs.rbm_split(np.asarray(theta), n, h)
        self.x = np.asarray(x).astype(float)
        self.t = np.tanh(self.b + self.x @ self.W.T)  # N x h
        self.w = np.asarray(w, dtype=float)
        self.obar = self.colsum(self.w, conj=False)

    @property
    def p(self):
        return self.n + self.h + self.h * self.n

    def colsum(self, y, conj=True):
        """sum_n y_n conj(O_n) (conj=True) or sum_n y_n O_n."""
        t = self.t.conj() if conj else self.t
        xa = self.x.T @ y
        tb = t.T @ y
        tw = (t * y[:, None]).T @ self.x  # h x n
        return np.concatenate([xa.astype(tb.dtype), tb, tw.reshape(-1)])

    def apply_o(self, v):
        va, vb, vw = v[: self.n], v[self.n : self.n + self.h], v[self.n + self.h :].reshape(self.h, self.n)
        return self.x @ va + np.sum(self.t * (vb + self.x @ vw.T), axis=1)

    def product(self, coeff, v):
        """O_c^H (coeff * (O_c v)) for the centred rows."""
        oc_v = self.apply_o(v) - self.obar @ v
        y = coeff * oc_v
        return self.colsum(y) - self.obar.conj() * np.sum(y)


class MLPProducts:
    """Centred products of a shallow-MLP batch, layout [W (h x n), b, u, c]."""

    def __init__(self, theta, x, n, h, w):
        self.n, self.h = n, h
        self.W, self.b, self.u, self.c = nqs.mlp_split(np.asarray(theta, dtype=float), n, h)
        self.x = np.asarray(x).astype(float)
        self.t = np.tanh(self.b + self.x @ self.W.T)
        self.g = self.u * (1.0 - self.t * self.t)
        self.w = np.asarray(w, dtype=float)
        self.obar = self.colsum(self.w)

    @property
    def p(self):
        return self.h * self.n + 2 * self.h + 1

    def colsum(self, y):
        gw = (self.g * y[:, None]).T @ self.x  # h x n
        return np.concatenate([gw.reshape(-1), self.g.T @ y, self.t.T @ y, [np.sum(y)]])

    def apply_o(self, v):
        hn = self.h * self.n
        vw = v[:hn].reshape(self.h, self.n)
        vb, vu, vc = v[hn : hn + self.h], v[hn + self.h : hn + 2 * self.h], v[hn + 2 * self.h]
        return np.sum(self.g * (self.x @ vw.T + vb), axis=1) + self.t @ vu + vc

    def product(self, coeff, v):
        oc_v = self.apply_o(v) - self.obar @ v
        y = coeff * oc_v
        return self.colsum(y) - self.obar * np.sum(y)
