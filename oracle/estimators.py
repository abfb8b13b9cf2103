"""Numpy restatement of the reference estimators (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/irlnqs/estimators.py operation by operation,
including the per-call centring copy (est:166-168) — so that, timed, it is a
faithful CPU baseline of the reference's own arithmetic.
"""

from __future__ import annotations

import numpy as np


def energy(w: np.ndarray, e: np.ndarray, n_samples: int):
    """est:146-153 -> (mean, variance, std_error)."""
    mean = complex(np.sum(w * e)).real
    variance = float(np.sum(w * np.abs(e - mean) ** 2))
    std = 0.0 if n_samples == 0 else float(np.sqrt(variance / n_samples))
    return mean, variance, std


def gradient(w, e, o, mean):
    """est:156-163: F = 2 Re((w e) @ conj(O) - E (w @ conj(O))) — the expanded form."""
    oc = o.conj()
    return 2.0 * ((w * e) @ oc - mean * (w @ oc)).real


def centred(w, e, o, mean):
    """est:166-168: materialised O - w@O copy and e - E."""
    return o - w @ o, e - mean


def heff(w, e, o, mean, v):
    """est:171-186 (real v): Re((w e_c (O_c v)) @ conj(O_c))."""
    o_c, e_c = centred(w, e, o, mean)
    proj = o_c @ v
    return ((w * e_c * proj) @ o_c.conj()).real


def qgt(w, o, v):
    """S v through the reference heff with e_loc = 1, E = 0."""
    return heff(w, np.ones_like(w), o, 0.0, v)


def heff_hermitian(w, e, o, mean, v):
    """Hermitian complex-parameter product O_c^H (w Re(e_c) (O_c v))."""
    o_c, e_c = centred(w, e, o, mean)
    return (w * e_c.real * (o_c @ v)) @ o_c.conj()


def heff_chunked(w, e, o_rows, mean, v, obar, chunk=4096, coeff=None):
    """Same product for N x P beyond host RAM: rows produced chunk by chunk by
    ``o_rows(lo, hi)``; obar precomputed.  coeff overrides w (e - E)."""
    n = len(w)
    out = None
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        oc = o_rows(lo, hi) - obar
        c = (w[lo:hi] * (e[lo:hi] - mean)) if coeff is None else coeff[lo:hi]
        part = (c * (oc @ v)) @ oc.conj()
        out = part if out is None else out + part
    return out


def dense_heff(w, e, o, mean):
    """est:319-332 (symmetrised, real part)."""
    o_c, e_c = centred(w, e, o, mean)
    mat = ((o_c.conj().T * (w * e_c)) @ o_c).real
    return (mat + mat.T) / 2


def dense_qgt(w, o):
    """est:335-344."""
    o_c = o - w @ o
    mat = ((o_c.conj().T * w) @ o_c).real
    return (mat + mat.T) / 2


def heff_offdiag(w, o, dist_index, indptr, partner_row, coeff, partner_o, v):
    """est:254-294 (real v): two-configuration completion, restated operation by operation.

    q = (O - Obar) v, q_part = (O_part - Obar) v; corr per distinct config by
    a segment sum (est:283-290); out = Re((w corr) @ conj(O_c)).
    """
    o_bar = w @ o
    q_batch = (o - o_bar) @ v
    q_part = (partner_o - o_bar) @ v if len(partner_o) else np.zeros(0)
    n_dist = len(indptr) - 1
    q_dist = np.zeros(n_dist, dtype=complex)
    q_dist[dist_index] = q_batch
    seg = np.repeat(np.arange(n_dist), np.diff(indptr))
    corr_dist = np.zeros(n_dist, dtype=complex)
    if len(seg):
        np.add.at(corr_dist, seg, coeff * (q_part[partner_row] - q_dist[seg]))
    corr = corr_dist[dist_index]
    o_c = o - o_bar
    return ((w * corr) @ o_c.conj()).real


def heff_offdiag_hermitian(w, o, dist_index, indptr, partner_row, coeff, partner_o, v):
    """Complex-parameter completion: the reference's est:254-294 on the real
    embedding [O, iO] equals [Re z, Im z] with
    z = sum_n w_n corr_n conj(O_c,n), q = O_c v for complex v."""
    o_bar = w @ o
    q_batch = (o - o_bar) @ v
    q_part = (partner_o - o_bar) @ v if len(partner_o) else np.zeros(0, dtype=complex)
    n_dist = len(indptr) - 1
    q_dist = np.zeros(n_dist, dtype=complex)
    q_dist[dist_index] = q_batch
    seg = np.repeat(np.arange(n_dist), np.diff(indptr))
    corr_dist = np.zeros(n_dist, dtype=complex)
    if len(seg):
        np.add.at(corr_dist, seg, coeff * (q_part[partner_row] - q_dist[seg]))
    corr = corr_dist[dist_index]
    return (w * corr) @ (o - o_bar).conj()
