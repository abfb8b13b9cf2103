"""Molecular Hamiltonians and local energies on the device.

The step before the hot path: ``irlnqs.hamiltonian`` (``ham``) parses FCIDUMP
integrals and evaluates ``E_loc(x) = sum_y <x|H|y> psi(y)/psi(x)`` over the
spin-conserving singles and doubles of every sample (``ham:238-302``), one
Python call per configuration.  Here:

* :class:`MolecularIntegrals`, :func:`parse_fcidump` — the same data model and
  Molpro FCIDUMP conventions (``ham:36-171``: 1-based indices, (0 0 0 0) core
  energy, (i j 0 0) one-electron, 8-fold symmetric (ij|kl)); host-side parsing;
* :class:`Sector`, :func:`enumerate_sector` — fixed (M, N_up, N_down) sectors in
  ascending bitmask order (``hilbert.py:54-124``), as uint64 arrays;
* :func:`local_energies` — E_loc for a batch of samples in one kernel
  (``k_local_energy``: Slater-Condon elements with the fermionic sign of
  ``classify_excitation``, amplitude ratios from incremental hidden-unit
  updates of the shallow NQS);
* :func:`connected_partners` — the kept off-diagonal partners, their elements
  and coefficients ``<x|H|y> psi(y)/psi(x)`` as a CSR (two kernel passes);
* :func:`build_batch` / :func:`build_connected_cache` — the reference
  signatures ``est.build_batch(params, integrals, sector, n_samples=0)``
  (exact mode: the whole sector, weights ``|psi|^2``) and
  ``est.build_connected_cache(params, integrals, sector, batch)``
  (``est:79-133``, ``est:221-251``) for the RBM / MLP ansatz.

Samples are bitmasks over ``M = 2 n_spatial <= 64`` spin-orbitals in the
reference's blocked layout (spin up first); the ansatz input ``x_i`` is the
occupation of spin-orbital ``i``.
"""

from __future__ import annotations

import re
from dataclasses import dataclass
from itertools import combinations
from math import comb

import numpy as np
import torch

from . import _lib
from .ansatz import AnsatzParameters, _theta_device, fill_o_rows, log_amplitude_batch
from .estimators import KIND_HERMITIAN, KIND_REAL, ConnectedCache, SampleBatch, _device, partner_rows_in_batch

DROP_TOLERANCE = 1e-14  # ham:24
MAX_ORBITALS = 64  # hilbert.py:14


class FcidumpError(Exception):
    """Malformed FCIDUMP content (ham:29-30)."""


@dataclass(frozen=True)
class Sector:
    """Fixed particle-number sector (hilbert.py:54-88)."""

    n_orbitals: int
    n_up: int
    n_down: int

    def __post_init__(self):
        if self.n_orbitals % 2 or self.n_orbitals > MAX_ORBITALS:
            raise ValueError(f"need an even spin-orbital count <= {MAX_ORBITALS}, got {self.n_orbitals}")
        half = self.n_orbitals // 2
        if not (0 <= self.n_up <= half and 0 <= self.n_down <= half):
            raise ValueError("electron counts out of range")

    @property
    def size(self) -> int:
        half = self.n_orbitals // 2
        return comb(half, self.n_up) * comb(half, self.n_down)


@dataclass(frozen=True)
class MolecularIntegrals:
    """Core energy, h (n, n) and chemists' g (n, n, n, n) (ham:36-63)."""

    n_spatial: int
    n_electrons: int
    ms2: int
    e_core: float
    h: np.ndarray
    g: np.ndarray

    @property
    def n_spin_orbitals(self) -> int:
        return 2 * self.n_spatial

    def sector(self) -> Sector:
        n_up = (self.n_electrons + self.ms2) // 2
        return Sector(self.n_spin_orbitals, n_up, self.n_electrons - n_up)

    def device_arrays(self, device) -> tuple[torch.Tensor, torch.Tensor]:
        """(h, g) uploaded once per device (contiguous float64)."""
        key = f"_dev_{torch.device(device)}"
        hit = self.__dict__.get(key)
        if hit is None:
            hit = (torch.as_tensor(np.ascontiguousarray(self.h, dtype=np.float64), device=device),
                   torch.as_tensor(np.ascontiguousarray(self.g, dtype=np.float64), device=device))
            object.__setattr__(self, key, hit)
        return hit


_PERMS = ((0, 1, 2, 3), (1, 0, 2, 3), (0, 1, 3, 2), (1, 0, 3, 2), (2, 3, 0, 1), (3, 2, 0, 1), (2, 3, 1, 0),
          (3, 2, 1, 0))


def parse_fcidump(text) -> MolecularIntegrals:
    """Molpro FCIDUMP text -> integrals (the conventions of ham:94-171).

    Header namelist up to ``&END`` or ``/`` with NORB, NELEC (MS2 default 0);
    body lines ``value i j k l``.  Conflicting duplicates raise.
    """
    if not isinstance(text, str):
        text = "".join(text)
    m = re.search(r"&END|/", text, flags=re.IGNORECASE)
    if m is None:
        raise FcidumpError("missing &END (or '/') after the namelist header")
    header, body = text[: m.start()], text[m.end():]
    fields = {k.upper(): v for k, v in re.findall(r"([A-Za-z0-9_]+)\s*=\s*([-\d]+)", header)}
    try:
        ns = int(fields["NORB"])
        ne = int(fields["NELEC"])
    except (KeyError, ValueError) as exc:
        raise FcidumpError(f"malformed FCIDUMP header: {exc}") from exc
    ms2 = int(fields.get("MS2", "0"))
    if ns < 1:
        raise FcidumpError(f"NORB must be positive, got {ns}")
    e_core, seen = 0.0, False
    h = np.zeros((ns, ns))
    g = np.zeros((ns,) * 4)
    tol = 1e-12
    for lineno, raw in enumerate(body.splitlines(), 1):
        parts = raw.split()
        if not parts:
            continue
        if len(parts) != 5:
            raise FcidumpError(f"body line {lineno}: expected 'value i j k l'")
        try:
            val = float(parts[0].replace("D", "E").replace("d", "e"))
            idx = [int(p) for p in parts[1:]]
        except ValueError as exc:
            raise FcidumpError(f"body line {lineno}: {exc}") from exc
        if any(i < 0 or i > ns for i in idx):
            raise FcidumpError(f"body line {lineno}: index out of range 0..{ns}")
        i, j, k, l = idx
        if i == j == k == l == 0:
            if seen and abs(e_core - val) > tol:
                raise FcidumpError(f"body line {lineno}: conflicting core energy")
            e_core, seen = val, True
        elif k == 0 and l == 0:
            if i == 0 or j == 0:
                raise FcidumpError(f"body line {lineno}: bad one-electron indices")
            old = h[i - 1, j - 1]
            if old != 0.0 and abs(old - val) > tol:
                raise FcidumpError(f"body line {lineno}: conflicting h[{i},{j}]")
            h[i - 1, j - 1] = h[j - 1, i - 1] = val
        elif 0 in idx:
            raise FcidumpError(f"body line {lineno}: bad two-electron indices")
        else:
            q = (i - 1, j - 1, k - 1, l - 1)
            for perm in _PERMS:
                key = tuple(q[t] for t in perm)
                old = g[key]
                if old != 0.0 and abs(old - val) > tol:
                    raise FcidumpError(f"body line {lineno}: conflicting duplicate integral")
                g[key] = val
    return MolecularIntegrals(ns, ne, ms2, e_core, h, g)


def enumerate_sector(sector: Sector, cap: int = 10**6) -> np.ndarray:
    """All configurations of a sector as ascending uint64 bitmasks (hilbert.py:100-123)."""
    if sector.size > cap:
        raise ValueError(f"sector has {sector.size} configurations, above the cap of {cap}")
    half = sector.n_orbitals // 2
    ups = np.array([sum(1 << i for i in c) for c in combinations(range(half), sector.n_up)], dtype=np.uint64)
    dns = np.array([sum(1 << (half + i) for i in c) for c in combinations(range(half), sector.n_down)],
                   dtype=np.uint64)
    return np.sort((ups[:, None] | dns[None, :]).reshape(-1))


def bits_to_occupations(bits, n_orbitals: int) -> np.ndarray:
    """uint64 bitmasks -> (N, M) uint8 occupations (the ansatz input)."""
    b = np.asarray(bits, dtype=np.uint64).reshape(-1, 1)
    return ((b >> np.arange(n_orbitals, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.uint8)


def occupations_to_bits(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    return (x << np.arange(x.shape[1], dtype=np.uint64)[None, :]).sum(axis=1, dtype=np.uint64)


def _check(params: AnsatzParameters, integrals: MolecularIntegrals):
    arch = params.architecture
    if arch.n_inputs != integrals.n_spin_orbitals:
        raise ValueError(f"ansatz has {arch.n_inputs} inputs, the Hamiltonian {integrals.n_spin_orbitals} "
                         "spin-orbitals")
    return arch


def _ham_call(fn: str, params, integrals, xb: torch.Tensor, drop: float, *tail):
    arch = _check(params, integrals)
    dev = xb.device
    h1, g2 = integrals.device_arrays(dev)
    theta = _theta_device(params, dev)
    cplx = int(bool(arch.complex_params))
    nbytes = int(_lib.lib().irl_ham_workspace_bytes(integrals.n_spatial, arch.hidden, cplx))
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
    _lib.call(fn, int(arch.model), cplx, _lib.ptr(xb), int(xb.shape[0]), integrals.n_spatial,
              float(integrals.e_core), _lib.ptr(h1), _lib.ptr(g2), float(drop), arch.hidden, _lib.ptr(theta),
              *tail, _lib.ptr(ws), ws.numel(), _lib.stream_handle(dev))


def _bits_device(xbits, dev) -> torch.Tensor:
    if isinstance(xbits, torch.Tensor):
        return xbits.to(device=dev, dtype=torch.int64).contiguous()
    return torch.as_tensor(np.asarray(xbits, dtype=np.uint64).view(np.int64), device=dev)


def local_energies(params: AnsatzParameters, integrals: MolecularIntegrals, xbits, *,
                   drop_tolerance: float = DROP_TOLERANCE, device=None) -> torch.Tensor:
    """E_loc for every sample bitmask (``local_energy``, ham:290-302), device (N,)."""
    dev = _device(device)
    xb = _bits_device(xbits, dev)
    cplx = bool(params.architecture.complex_params)
    out = torch.empty(int(xb.shape[0]), dtype=torch.complex128 if cplx else torch.float64, device=dev)
    _ham_call("irl_ham_local_energy", params, integrals, xb, drop_tolerance, _lib.ptr(out))
    return out


def connected_partners(params: AnsatzParameters, integrals: MolecularIntegrals, xbits, *,
                       drop_tolerance: float = DROP_TOLERANCE, device=None):
    """Kept off-diagonal partners of every sample (``connected_configurations``
    minus the diagonal entry, ham:238-287) as a CSR on the device:
    (indptr (N+1,), partner bits (nnz,) int64 view of uint64, elements (nnz,),
    coefficients element * psi(y)/psi(x) (nnz,), complex for complex theta).
    Partners are in enumeration order (singles up, singles down, same-spin
    doubles, opposite-spin doubles), not the reference's ascending-bitmask
    order; sums over them agree to rounding."""
    dev = _device(device)
    xb = _bits_device(xbits, dev)
    n = int(xb.shape[0])
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    _ham_call("irl_ham_connected_count", params, integrals, xb, drop_tolerance, _lib.ptr(counts))
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=indptr[1:])
    nnz = int(indptr[-1])
    cplx = bool(params.architecture.complex_params)
    pbits = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
    elem = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    coeff = torch.empty(max(nnz, 1), dtype=torch.complex128 if cplx else torch.float64, device=dev)
    _ham_call("irl_ham_connected_fill", params, integrals, xb, drop_tolerance, _lib.ptr(indptr), _lib.ptr(pbits),
              _lib.ptr(elem), _lib.ptr(coeff))
    return indptr, pbits[:nnz], elem[:nnz], coeff[:nnz]


def build_batch(params: AnsatzParameters, integrals: MolecularIntegrals, sector: Sector, n_samples: int = 0,
                seed: int = 0, *, configs=None, device=None, enumeration_cap: int = 10**6,
                mode: str = "stored") -> SampleBatch:
    """``est.build_batch`` (est:79-133) for the shallow NQS on the device.

    Exact mode (``n_samples == 0``): the whole sector, weights ``|psi|^2``
    normalised.  Stochastic mode needs the samples as ``configs`` (bitmasks):
    the RBM / MLP have no exact ancestral sampler (the reference's sampler
    belongs to its autoregressive ansatz, ans:215-236); weights are 1/n.
    E_loc comes from :func:`local_energies`, O from the row kernel; the batch
    keeps its sample bitmasks as ``batch.xbits``.
    """
    arch = _check(params, integrals)
    dev = _device(device)
    if n_samples == 0:
        bits = enumerate_sector(sector, cap=enumeration_cap)
    else:
        if configs is None:
            raise NotImplementedError("stochastic RBM/MLP batches need their samples (configs=bitmasks)")
        bits = np.asarray(configs, dtype=np.uint64)
        if bits.shape != (n_samples,):
            raise ValueError("configs must hold n_samples bitmasks")
    x = bits_to_occupations(bits, arch.n_inputs)
    xb = _bits_device(bits, dev)
    e_loc = local_energies(params, integrals, xb, device=dev)
    if n_samples == 0:
        lp = log_amplitude_batch(params, x, device=dev)
        lr = lp.real if torch.is_complex(lp) else lp
        w = torch.exp(2.0 * (lr - lr.max()))
        w = w / w.sum()
        # est:50-51 wants sum w = 1 within 1e-12: renormalise once more on the host sum
        w = w / float(w.sum())
    else:
        w = torch.full((len(bits),), 1.0 / n_samples, dtype=torch.float64, device=dev)
    if mode == "otf":  # O regenerated inside every product (ansatz.build_batch_otf)
        from .ansatz import build_batch_otf

        batch = build_batch_otf(params, x, e_loc, weights=w, n_samples=n_samples, device=dev)
        batch.xbits = bits
        return batch
    if mode != "stored":
        raise ValueError(f"unknown build mode {mode!r}")
    kind = KIND_HERMITIAN if arch.complex_params else KIND_REAL
    p = arch.param_count
    ld = _lib.padded_ld(p, arch.complex_params)
    odt = torch.complex128 if arch.complex_params else torch.float64
    o = torch.empty((len(bits), ld), dtype=odt, device=dev)
    batch = SampleBatch(None, w, e_loc, o, n_samples, kind=kind, param_count=p, device=dev)
    _, mean = batch._energy_pass(None)
    obar = torch.empty(ld, dtype=odt, device=dev)
    g = torch.empty(ld, dtype=odt, device=dev)
    xt = torch.as_tensor(x, device=dev)
    fill_o_rows(params, xt, o, batch.weights, batch.gradient_coefficients(mean), obar, g)
    batch._set_colstats(mean, obar, g)
    batch.xbits = bits
    return batch


def build_connected_cache(params: AnsatzParameters, integrals: MolecularIntegrals, sector: Sector,
                          batch: SampleBatch) -> ConnectedCache:
    """``est.build_connected_cache`` (est:221-251): distinct configurations of
    the batch, their kept partners and coefficients element * psi(y)/psi(x)
    (device enumeration), and the partner O rows: the batch's own rows when
    every partner is a batch configuration (exact mode), else the row kernel on
    the distinct partners (the reference's o_row table, est:236-242)."""
    bits = getattr(batch, "xbits", None)
    if bits is None:
        raise ValueError("batch has no sample bitmasks (build it with hamiltonian.build_batch)")
    dev = batch.device
    bits = np.asarray(bits, dtype=np.uint64)
    uniq, dist_index = np.unique(bits, return_inverse=True)
    dist_index = dist_index.reshape(-1)
    indptr, pbits, elem, coeff = connected_partners(params, integrals, uniq, device=dev)
    reps = np.full(len(uniq), -1, dtype=np.int64)
    order = np.arange(len(bits))[::-1]
    reps[dist_index[order]] = order
    rows = partner_rows_in_batch(uniq, reps, pbits) if pbits.numel() else None
    if rows is not None:
        cache = ConnectedCache(dist_index, indptr, rows, coeff, None, batch=batch)
    else:
        arch = params.architecture
        pb = pbits.cpu().numpy().view(np.uint64)
        pu, pinv = np.unique(pb, return_inverse=True)
        cdt = torch.complex128 if arch.complex_params else torch.float64
        po = torch.zeros((len(pu), batch.ld), dtype=cdt, device=dev)
        if len(pu):
            xt = torch.as_tensor(bits_to_occupations(pu, arch.n_inputs), device=dev)
            m = len(pu)
            w = torch.full((m,), 1.0 / m, dtype=torch.float64, device=dev)
            scratch = [torch.empty(batch.ld, dtype=cdt, device=dev) for _ in range(2)]
            fill_o_rows(params, xt, po, w, torch.zeros(m, dtype=cdt, device=dev), scratch[0], scratch[1])
        cache = ConnectedCache(dist_index, indptr, pinv.reshape(-1), coeff, po, batch=batch)
    cache.elements = elem
    return cache
