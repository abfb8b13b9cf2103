"""The reference's own NQS on the device.

``irlnqs.ansatz`` (``ans``) is an autoregressive network with exact particle-
number masking: psi(n) = sqrt(p(n)) exp(i phi(n)), p a product of masked
conditionals of one shared tanh layer over the +-1 prefix and a position
one-hot, phi a linear-plus-tanh phase head (``ans:1-14``).  The reference
evaluates it one configuration and one position at a time in Python.  Here the
same network runs as one warp per configuration (``csrc/autoreg.cuh``):

* :func:`log_amplitude_batch` — ``log_amplitude`` (``ans:229-247``);
* :func:`log_derivative_batch` — ``log_derivative`` (``ans:249-290``): complex O
  rows straight into the padded device layout of :class:`SampleBatch`;
* :func:`sample` — ``sample`` (``ans:215-236``), bit-identical: the host spawns
  the same per-sample numpy PCG64 streams and the kernel replays them;
* :func:`local_energies`, :func:`build_batch`, :func:`build_connected_cache` —
  ``local_energy`` (``ham:290-302``), ``est.build_batch`` (``est:79-133``) and
  ``est.build_connected_cache`` (``est:221-251``) for this ansatz, so the
  reference's whole outer step (``opt:118-195``) runs on the device with the
  reference's own model (:func:`optimizer.outer_step`).

``Architecture``, ``AnsatzParameters`` and ``init_parameters`` keep the
reference's names, layout and seeded initialisation (``ans:26-128``); the
reference's own parameter objects are accepted as they are (same fields).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .estimators import KIND_COMPLEX_RAW, ConnectedCache, SampleBatch, _device, partner_rows_in_batch


@dataclass(frozen=True)
class Architecture:
    """ans:26-38."""

    n_orbitals: int
    hidden: int

    @property
    def param_count(self) -> int:
        m, h = self.n_orbitals, self.hidden
        return h * (2 * m) + h + 2 * h + 2 + h * m + h + h + m + 1


@dataclass(frozen=True)
class AnsatzParameters:
    """ans:41-53."""

    architecture: Architecture
    theta: np.ndarray

    def __post_init__(self):
        if np.shape(self.theta) != (self.architecture.param_count,):
            raise ValueError(f"theta has length {np.shape(self.theta)}, architecture needs "
                             f"{self.architecture.param_count}")


@dataclass(frozen=True)
class LogAmplitude:
    """ans:56-64."""

    log_prob_half: float
    phase: float

    @property
    def value(self) -> complex:
        return complex(self.log_prob_half, self.phase)


def init_parameters(arch: Architecture, seed: int = 111) -> AnsatzParameters:
    """ans:118-128: seeded uniform [-1/sqrt(fan_in), 1/sqrt(fan_in)] for the
    amplitude head and the phase hidden layer, zeros for up, w_lin, c."""
    rng = np.random.default_rng(seed)
    m, h = arch.n_orbitals, arch.hidden
    w1 = rng.uniform(-1, 1, (h, 2 * m)) / np.sqrt(2 * m)
    b1 = rng.uniform(-1, 1, h) / np.sqrt(2 * m)
    w2 = rng.uniform(-1, 1, (2, h)) / np.sqrt(h)
    b2 = rng.uniform(-1, 1, 2) / np.sqrt(h)
    wp = rng.uniform(-1, 1, (h, m)) / np.sqrt(m)
    bp = rng.uniform(-1, 1, h) / np.sqrt(m)
    theta = np.concatenate([w1.ravel(), b1, w2.ravel(), b2, wp.ravel(), bp, np.zeros(h), np.zeros(m), np.zeros(1)])
    return AnsatzParameters(arch, theta)


def is_autoregressive(params) -> bool:
    arch = getattr(params, "architecture", None)
    return hasattr(arch, "n_orbitals") and hasattr(arch, "hidden") and not hasattr(arch, "n_visible") \
        and not hasattr(arch, "n_in")


def _theta(params, dev) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(np.asarray(params.theta, dtype=np.float64)), device=dev)


def _bits(xbits, dev) -> torch.Tensor:
    if isinstance(xbits, torch.Tensor):
        return xbits.to(device=dev, dtype=torch.int64).contiguous()
    if isinstance(xbits, (list, tuple)) and xbits and hasattr(xbits[0], "bits"):
        xbits = [x.bits for x in xbits]  # reference OccupationVectors
    return torch.as_tensor(np.asarray(xbits, dtype=np.uint64).view(np.int64), device=dev)


def _check_error(err: torch.Tensor, what: str) -> None:
    code = int(err.item())
    if code == 1:
        raise ValueError("configuration outside the sector has zero amplitude")  # ans:256-257
    if code == 2:
        raise RuntimeError(f"infeasible prefix reached in {what}; masking invariant broken")  # ans:150-151


def log_amplitude_batch(params, sector, xbits, device=None) -> torch.Tensor:
    """ln psi = ln p / 2 + i phi for every configuration (complex128 device (N,));
    ``-inf`` real part outside the sector (ans:236-238)."""
    dev = _device(device)
    xb = _bits(xbits, dev)
    arch = params.architecture
    out = torch.empty(int(xb.shape[0]), dtype=torch.complex128, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("irl_ar_logamp", _lib.ptr(xb), int(xb.shape[0]), arch.n_orbitals, arch.hidden, sector.n_up,
              sector.n_down, _lib.ptr(_theta(params, dev)), _lib.ptr(out), _lib.ptr(err), _lib.stream_handle(dev))
    return out


def log_amplitude(params, x, sector) -> LogAmplitude:
    v = complex(log_amplitude_batch(params, sector, [int(getattr(x, "bits", x))])[0].item())
    return LogAmplitude(v.real, v.imag)


def log_derivative_batch(params, sector, xbits, *, ld: int | None = None, out: torch.Tensor | None = None,
                         device=None) -> torch.Tensor:
    """O rows (ans:249-290) as a complex128 device tensor (N, ld), padding zero."""
    dev = _device(device)
    xb = _bits(xbits, dev)
    arch = params.architecture
    p = arch.param_count
    if ld is None:
        ld = _lib.padded_ld(p, True)
    n = int(xb.shape[0])
    o = out if out is not None else torch.empty((n, ld), dtype=torch.complex128, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("irl_ar_rows", _lib.ptr(xb), n, arch.n_orbitals, arch.hidden, sector.n_up, sector.n_down,
              _lib.ptr(_theta(params, dev)), _lib.ptr(o), int(o.shape[1]), _lib.ptr(err), _lib.stream_handle(dev))
    _check_error(err, "log_derivative")
    return o


def log_derivative(params, x, sector) -> np.ndarray:
    """Single configuration (ans:249 signature): complex (P,)."""
    o = log_derivative_batch(params, sector, [int(getattr(x, "bits", x))])
    return o[0, : params.architecture.param_count].cpu().numpy()


def sample(params, sector, count: int, seed: int, device=None) -> np.ndarray:
    """Exact ancestral sampling (ans:215-236), bit-identical to the reference:
    per-sample PCG64 streams from ``SeedSequence(seed).spawn(count)``.
    Returns uint64 bitmasks (host)."""
    if count < 0:
        raise ValueError("count must be nonnegative")
    dev = _device(device)
    arch = params.architecture
    states = np.empty((count, 4), dtype=np.uint64)
    m64 = (1 << 64) - 1
    for k, stream in enumerate(np.random.SeedSequence(seed).spawn(count)):
        st = np.random.default_rng(stream).bit_generator.state["state"]
        states[k] = (st["state"] >> 64, st["state"] & m64, st["inc"] >> 64, st["inc"] & m64)
    if count == 0:
        return np.zeros(0, dtype=np.uint64)
    rs = torch.as_tensor(states.view(np.int64), device=dev)
    out = torch.empty(count, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("irl_ar_sample", _lib.ptr(rs), count, arch.n_orbitals, arch.hidden, sector.n_up, sector.n_down,
              _lib.ptr(_theta(params, dev)), _lib.ptr(out), _lib.ptr(err), _lib.stream_handle(dev))
    _check_error(err, "sample")
    return out.cpu().numpy().view(np.uint64)


def _ints(integrals, dev):
    if hasattr(integrals, "device_arrays"):
        return integrals.device_arrays(dev)
    return (torch.as_tensor(np.ascontiguousarray(integrals.h, dtype=np.float64), device=dev),
            torch.as_tensor(np.ascontiguousarray(integrals.g, dtype=np.float64), device=dev))


def hamiltonian_partners(integrals, xbits, *, drop_tolerance: float = 1e-14, device=None):
    """Ansatz-free enumeration (ham:238-287): diagonal elements and the CSR of
    kept partners with their elements, on the device."""
    dev = _device(device)
    xb = _bits(xbits, dev)
    n = int(xb.shape[0])
    h1, g2 = _ints(integrals, dev)
    diag = torch.empty(n, dtype=torch.float64, device=dev)
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    st = _lib.stream_handle(dev)
    _lib.call("irl_ham_diagonal_and_count", _lib.ptr(xb), n, integrals.n_spatial, float(integrals.e_core),
              _lib.ptr(h1), _lib.ptr(g2), float(drop_tolerance), _lib.ptr(diag), _lib.ptr(counts), st)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=indptr[1:])
    nnz = int(indptr[-1])
    pbits = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
    elem = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    _lib.call("irl_ham_partners_fill", _lib.ptr(xb), n, integrals.n_spatial, float(integrals.e_core), _lib.ptr(h1),
              _lib.ptr(g2), float(drop_tolerance), _lib.ptr(indptr), _lib.ptr(pbits), _lib.ptr(elem), st)
    return diag, indptr, pbits[:nnz], elem[:nnz]


def _partner_logamp(params, sector, xb: torch.Tensor, lp_x: torch.Tensor, pbits: torch.Tensor) -> torch.Tensor:
    """ln psi of the partners: looked up among the configurations already
    evaluated (every partner in exact mode: the batch is the whole sector),
    the network run only on the rest."""
    dev = xb.device
    if pbits.numel() == 0:
        return lp_x[:0]
    xh = xb.cpu().numpy().view(np.uint64)
    uniq, first = np.unique(xh, return_index=True)
    keys = torch.as_tensor(uniq.view(np.int64), device=dev)
    idx = torch.empty(pbits.numel(), dtype=torch.int64, device=dev)
    _lib.call("irl_sorted_lookup", _lib.ptr(keys), keys.numel(), _lib.ptr(pbits), pbits.numel(), _lib.ptr(idx),
              _lib.stream_handle(dev))
    lp_keys = lp_x[torch.as_tensor(first, device=dev)]
    found = idx >= 0
    lp_y = lp_keys[idx.clamp_min(0)]
    if not bool(found.all()):
        miss = ~found
        lp_y[miss] = log_amplitude_batch(params, sector, pbits[miss], device=dev)
    return lp_y


def local_energies(params, integrals, sector, xbits, device=None) -> torch.Tensor:
    """E_loc (ham:290-302) for this ansatz: diag + sum element psi(y)/psi(x), complex (N,)."""
    dev = _device(device)
    xb = _bits(xbits, dev)
    diag, indptr, pbits, elem = hamiltonian_partners(integrals, xb, device=dev)
    lp_x = log_amplitude_batch(params, sector, xb, device=dev)
    if not bool(torch.isfinite(lp_x.real).all()):
        raise ValueError("log-amplitude is not finite at the reference configuration")  # ham:295-296
    lp_y = _partner_logamp(params, sector, xb, lp_x, pbits)
    out = torch.empty(int(xb.shape[0]), dtype=torch.complex128, device=dev)
    _lib.call("irl_eloc_combine", _lib.ptr(indptr), _lib.ptr(elem), _lib.ptr(lp_y) if pbits.numel() else None,
              _lib.ptr(lp_x), _lib.ptr(diag), int(xb.shape[0]), _lib.ptr(out), _lib.stream_handle(dev))
    return out


def build_batch(params, integrals, sector, n_samples: int = 0, seed: int = 0, enumeration_cap: int = 10**6,
                device=None) -> SampleBatch:
    """est.build_batch (est:79-133) with this ansatz: exact enumeration with
    |psi|^2 weights, or n_samples exact samples (weights 1/n).  E_loc and O rows
    on the device (duplicate configurations get bit-identical rows, as the
    reference's per-distinct cache gives identical values)."""
    from .hamiltonian import enumerate_sector

    dev = _device(device)
    if n_samples == 0:
        bits = enumerate_sector(sector, cap=enumeration_cap)
    else:
        bits = sample(params, sector, n_samples, seed, device=dev)
    xb = _bits(bits, dev)
    e = local_energies(params, integrals, sector, xb, device=dev)
    if n_samples == 0:
        lp = log_amplitude_batch(params, sector, xb, device=dev)
        w = torch.exp(2.0 * lp.real)
        w = w / w.sum()
    else:
        w = torch.full((len(bits),), 1.0 / n_samples, dtype=torch.float64, device=dev)
    arch = params.architecture
    p = arch.param_count
    o = log_derivative_batch(params, sector, xb, device=dev)
    batch = SampleBatch(None, w, e, o, n_samples, kind=KIND_COMPLEX_RAW, param_count=p, device=dev)
    batch.xbits = np.asarray(bits, dtype=np.uint64)
    batch.sector = sector
    return batch


def build_connected_cache(params, integrals, sector, batch: SampleBatch) -> ConnectedCache:
    """est.build_connected_cache (est:221-251) with this ansatz on the device."""
    bits = getattr(batch, "xbits", None)
    if bits is None:
        raise ValueError("batch has no sample bitmasks (build it with autoregressive.build_batch)")
    dev = batch.device
    uniq, dist_index = np.unique(np.asarray(bits, dtype=np.uint64), return_inverse=True)
    _, indptr, pbits, elem = hamiltonian_partners(integrals, uniq, device=dev)
    ub = _bits(uniq, dev)
    lp_x = log_amplitude_batch(params, sector, ub, device=dev)
    nnz = pbits.numel()
    lp_y = _partner_logamp(params, sector, ub, lp_x, pbits)
    seg = torch.repeat_interleave(torch.arange(len(uniq), device=dev), indptr[1:] - indptr[:-1])
    coeff = elem.to(torch.complex128) * torch.exp(lp_y - lp_x[seg])
    keep = torch.isfinite(lp_y.real)  # est:246-247 skips zero-amplitude partners
    if nnz and not bool(keep.all()):
        counts = torch.bincount(seg[keep], minlength=len(uniq))
        indptr = torch.zeros(len(uniq) + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts, 0, out=indptr[1:])
        pbits, coeff = pbits[keep], coeff[keep]
    reps = np.full(len(uniq), -1, dtype=np.int64)
    order = np.arange(len(bits))[::-1]
    reps[dist_index.reshape(-1)[order]] = order
    rows = partner_rows_in_batch(uniq, reps, pbits) if pbits.numel() else None
    if rows is not None:
        return ConnectedCache(dist_index.reshape(-1), indptr, rows, coeff, None, batch=batch)
    pb = pbits.cpu().numpy().view(np.uint64)
    pu, pinv = np.unique(pb, return_inverse=True) if len(pb) else (pb, np.zeros(0, dtype=np.int64))
    po = log_derivative_batch(params, sector, pu, ld=batch.ld, device=dev) if len(pu) else \
        torch.zeros((0, batch.ld), dtype=torch.complex128, device=dev)
    return ConnectedCache(dist_index.reshape(-1), indptr, pinv.reshape(-1), coeff, po, batch=batch)
