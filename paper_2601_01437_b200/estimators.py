"""Device-resident VMC estimators: the drop-in for ``irlnqs.estimators``.

Mirrors the reference entry points on the hot path:

* :class:`SampleBatch` — ``estimators.py:30-61`` (same constructor and
  validation: shapes, ``w >= 0``, ``sum w = 1 +- 1e-12``; frozen fields as
  the reference's frozen dataclass), but the caches live in HBM: the kernels
  stream ``o_padded``, an N x ld row-major device tensor with a padded leading
  dimension (``irl_padded_ld``, padding columns zero); ``o_matrix`` is its
  (N, P) view, so ``o_matrix.shape[1] == param_count`` as in ``est:55-57``.
* :func:`estimate_energy`   — ``estimators.py:146-153``  (k_energy)
* :func:`energy_gradient`   — ``estimators.py:156-163``  (fused column stats)
* :func:`heff_matvec`       — ``estimators.py:171-186``  (single-pass fused MVP)
* :func:`qgt_matvec`        — matrix-free form of ``dense_qgt`` (``:335-344``)
* :class:`ConnectedCache`, :func:`heff_offdiag_matvec` — ``estimators.py:189-294``
  (two-configuration completion); :func:`connected_heff_matvec`
  applies both terms of the optimizer's operator (``optimizer.py:144-147``)
* :func:`dense_heff`, :func:`dense_qgt`, :class:`DensePCapError` — ``:319-344``

Three parameter/O conventions are supported:

* ``real``         real theta, real O (RBM/MLP f64 configs);
* ``complex_raw``  real theta, complex O and E_loc — the reference's own
  autoregressive ansatz; products are ``Re(O_c^H (w e_c (O_c v)))`` with real v,
  exactly ``est.heff_matvec``;
* ``hermitian``    complex theta, holomorphic complex O (cfg4): products are
  the Hermitian ``O_c^H (w Re(e_c) (O_c v))`` on complex v.

The arithmetic runs only in the sm_100a kernels of ``libirlsr.so``; torch is
used for device memory and streams.  Without the library or a GPU every call
raises :class:`~paper_2601_01437_b200._lib.NativeUnavailable`.
"""

from __future__ import annotations

import os
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

DEFAULT_DENSE_P_CAP = 200  # est:22
IMAG_RESIDUAL_WARN = 1e-8  # est:23

KIND_REAL = "real"
KIND_COMPLEX_RAW = "complex_raw"
KIND_HERMITIAN = "hermitian"


class DensePCapError(Exception):
    """Parameter count too large for the dense p x p oracles (est:26-27)."""


@dataclass(frozen=True)
class EnergyEstimate:
    """est:64-68."""

    mean: float
    variance: float
    std_error: float


def _device(dev=None) -> torch.device:
    if dev is not None:
        return torch.device(dev)
    if not torch.cuda.is_available():
        raise _lib.NativeUnavailable("no CUDA device: the IRL-SR hot path runs only on sm_100a")
    return torch.device("cuda", torch.cuda.current_device())


def _as_tensor(x, dtype, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype)
    return torch.as_tensor(np.asarray(x), dtype=dtype, device=device)


class SampleBatch:
    """Configurations with weights and device-resident E_loc / O caches (est:30-61).

    ``o_matrix`` may be a host array (N, P) — it is uploaded once into the
    padded device layout — or an already padded device tensor (N, ld).
    ``kind`` selects the parameter convention (see module docstring); by
    default real O -> ``real`` and complex O -> ``complex_raw``.
    """

    def __init__(self, configs, weights, e_loc, o_matrix, n_samples: int = 0, *, kind: str | None = None,
                 param_count: int | None = None, device=None):
        if device is None and isinstance(o_matrix, torch.Tensor) and o_matrix.is_cuda:
            device = o_matrix.device
        dev = _device(device)
        is_complex = torch.is_complex(o_matrix) if isinstance(o_matrix, torch.Tensor) else np.iscomplexobj(o_matrix)
        if kind is None:
            kind = KIND_COMPLEX_RAW if is_complex else KIND_REAL
        if kind not in (KIND_REAL, KIND_COMPLEX_RAW, KIND_HERMITIAN):
            raise ValueError(f"unknown batch kind {kind!r}")
        if kind == KIND_REAL and is_complex:
            raise ValueError("complex o_matrix needs kind 'complex_raw' or 'hermitian'")
        n = len(configs) if configs is not None else int(np.shape(weights)[0])
        if o_matrix.shape[0] != n:
            raise ValueError("o_matrix rows do not match the config list")
        p = int(param_count) if param_count is not None else int(o_matrix.shape[1])
        ld = _lib.padded_ld(p, kind != KIND_REAL)
        self._init_common(weights, e_loc, n, n_samples, kind, p, ld, dev)
        cdt = torch.complex128 if kind != KIND_REAL else torch.float64
        if isinstance(o_matrix, torch.Tensor) and o_matrix.is_cuda and o_matrix.shape[1] == ld:
            o = o_matrix if o_matrix.dtype == cdt else o_matrix.to(cdt)
            if not o.is_contiguous():
                raise ValueError("device o_matrix must be contiguous")
        else:
            if o_matrix.shape[1] != p:
                raise ValueError("o_matrix width does not match param_count")
            o = torch.zeros((n, ld), dtype=cdt, device=dev)
            o[:, :p] = _as_tensor(o_matrix, cdt, dev)
        self.configs = tuple(configs) if configs is not None else None
        self.o_padded = o
        self._seal()

    # est:30 is a frozen dataclass: its fields cannot be rebound after
    # construction (dataclasses.FrozenInstanceError).  The device caches below
    # are private and keep being filled lazily.
    _FROZEN = ("configs", "weights", "e_loc", "o_matrix", "o_padded", "n_samples", "kind", "otf")

    def _seal(self) -> None:
        object.__setattr__(self, "_sealed", True)

    def __setattr__(self, name, value):
        if name in SampleBatch._FROZEN and self.__dict__.get("_sealed"):
            import dataclasses

            raise dataclasses.FrozenInstanceError(f"cannot assign to field {name!r}")
        object.__setattr__(self, name, value)

    @property
    def o_matrix(self) -> torch.Tensor:
        """The (N, P) log-derivative matrix (est:33): a view of the padded device buffer."""
        return self.o_padded[:, : self._p]

    def _init_common(self, weights, e_loc, n, n_samples, kind, p, ld, dev) -> None:
        """Weights / E_loc validation of est:44-53 and the device caches."""
        cdt = torch.complex128 if kind != KIND_REAL else torch.float64
        w = _as_tensor(weights, torch.float64, dev).contiguous()
        e_is_c = torch.is_complex(e_loc) if isinstance(e_loc, torch.Tensor) else np.iscomplexobj(e_loc)
        if kind == KIND_REAL and e_is_c:
            raise ValueError("complex e_loc needs a complex batch kind")
        e = _as_tensor(e_loc, cdt, dev).contiguous()
        if tuple(w.shape) != (n,) or tuple(e.shape) != (n,):
            raise ValueError("cache shapes do not match the config list")
        # est:50-51 validation (one host sync, once per batch)
        wmin = float(w.min()) if n else 0.0
        wsum = float(w.sum()) if n else 0.0
        if wmin < 0 or abs(wsum - 1.0) > 1e-12:  # an empty batch fails here, as in the reference
            raise ValueError("weights must be nonnegative and sum to 1")
        self.configs = None
        self.weights = w
        self.e_loc = e
        self.n_samples = int(n_samples)
        self.kind = kind
        self._p = p
        self.ld = ld
        self.device = dev
        self._coeff: dict = {}
        self._gcoeff: dict = {}
        self._colstats: dict = {}
        self._ws: dict = {}  # stream handle -> product workspace
        self._stats_e: float | None = None

    # -- reference properties (est:55-61)
    @property
    def param_count(self) -> int:
        return self._p

    @property
    def exact(self) -> bool:
        return self.n_samples == 0

    @property
    def n_rows(self) -> int:
        return int(self.weights.shape[0])

    @property
    def is_complex(self) -> bool:
        return self.kind != KIND_REAL

    # -- internals
    def _stream(self) -> int:
        return _lib.stream_handle(self.device)

    def mvp_workspace(self) -> torch.Tensor:
        """Product workspace of the current stream: products on one batch issued
        on two streams must not share partials (one buffer per stream handle)."""
        key = self._stream()
        ws = self._ws.get(key)
        if ws is None:
            if self.otf is not None:
                fn = "irl_otf_workspace_bytes_c128" if self.is_complex else "irl_otf_workspace_bytes"
                nbytes = int(getattr(_lib.lib(), fn)(self.n_rows, self.otf["n_in"], self.otf["hidden"]))
            else:
                nbytes = int(_lib.lib().irl_mvp_workspace_bytes(self.n_rows, self.ld, int(self.is_complex)))
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def mvp2_workspace(self) -> torch.Tensor:
        """Workspace of the two-output product (``irl_mvp2_*``) on the current stream."""
        key = ("mvp2", self._stream())
        ws = self._ws.get(key)
        if ws is None:
            nbytes = int(_lib.lib().irl_mvp2_workspace_bytes(self.n_rows, self.ld, int(self.is_complex)))
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def coefficients(self, mean: float) -> torch.Tensor:
        """Product coefficient c_n = w_n (e_n - E): est:166-168, est:186
        (Hermitian batches: w_n Re(e_n - E))."""
        key = float(mean)
        if key not in self._coeff:
            self._energy_pass(key)
        return self._coeff[key]

    def gradient_coefficients(self, mean: float) -> torch.Tensor:
        """Gradient coefficient w_n (e_n - E) with the full complex e (est:162)."""
        key = float(mean)
        if key not in self._gcoeff:
            self._energy_pass(key)
        return self._gcoeff[key]

    def _energy_pass(self, mean: float | None):
        """Run k_energy; caches both coefficient vectors; returns (stats3 host array, E)."""
        n = self.n_rows
        stats = torch.empty(3, dtype=torch.float64, device=self.device)
        gcoeff = torch.empty(n, dtype=self.e_loc.dtype, device=self.device)
        if self.is_complex:
            _lib.call("irl_energy_c128", _lib.ptr(self.weights), _lib.ptr(self.e_loc), n, 0,
                      _lib.ptr(stats), _lib.ptr(gcoeff), self._stream())
        else:
            _lib.call("irl_energy_f64", _lib.ptr(self.weights), _lib.ptr(self.e_loc), n,
                      _lib.ptr(stats), _lib.ptr(gcoeff), self._stream())
        coeff = gcoeff
        if self.kind == KIND_HERMITIAN:
            coeff = torch.empty_like(gcoeff)
            _lib.call("irl_energy_c128", _lib.ptr(self.weights), _lib.ptr(self.e_loc), n, 1,
                      _lib.ptr(stats), _lib.ptr(coeff), self._stream())
        host = stats.cpu().numpy()
        own = float(host[0])
        self._coeff[own] = coeff
        self._gcoeff[own] = gcoeff
        self._stats_e = own
        if mean is not None and float(mean) != own:
            # another energy reference (e.g. E = 0 for the S trick of SURVEY §8(c)):
            # c = w (e - mean), formed on device
            d = self.e_loc - float(mean)
            g = (self.weights * d).contiguous()
            self._gcoeff[float(mean)] = g
            if self.kind == KIND_HERMITIAN:
                d = torch.complex(d.real, torch.zeros_like(d.real))
                self._coeff[float(mean)] = (self.weights * d).contiguous()
            else:
                self._coeff[float(mean)] = g
        return host, own

    def colstats(self, mean: float):
        """(obar, g) with obar = w @ O and g = c @ conj(O), c = w (e - mean)."""
        key = float(mean)
        hit = self._colstats.get(key)
        if hit is not None:
            return hit
        c = self.gradient_coefficients(key)
        n = self.n_rows
        if self.otf is not None:
            return self._otf_colstats(key, c)
        obar = torch.empty(self.ld, dtype=self.o_padded.dtype, device=self.device)
        g = torch.empty(self.ld, dtype=self.o_padded.dtype, device=self.device)
        nbytes = int(_lib.lib().irl_colstats_workspace_bytes(n, self.ld, int(self.is_complex)))
        ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        fn = "irl_colstats_c128" if self.is_complex else "irl_colstats_f64"
        _lib.call(fn, _lib.ptr(self.o_padded), n, self.ld, _lib.ptr(self.weights), _lib.ptr(c),
                  _lib.ptr(obar), _lib.ptr(g), _lib.ptr(ws), ws.numel(), self._stream())
        self._colstats[key] = (obar, g)
        return obar, g

    # ---- on-the-fly (K6) MLP batches: O is never stored
    otf = None  # dict(xbits, t, g, n_in, hidden) for on-the-fly batches

    def _otf_colstats(self, key: float, c: torch.Tensor):
        o = self.otf
        n = self.n_rows
        dt = torch.complex128 if self.is_complex else torch.float64
        obar = torch.empty(self.ld, dtype=dt, device=self.device)
        g = torch.empty(self.ld, dtype=dt, device=self.device)
        ws = self.mvp_workspace()
        if self.is_complex:
            _lib.call("irl_otf_colstats_rbm_c128", _lib.ptr(o["xbits"]), _lib.ptr(o["t"]), n, o["n_in"],
                      o["hidden"], self.ld, _lib.ptr(self.weights), _lib.ptr(c), _lib.ptr(obar), _lib.ptr(g),
                      _lib.ptr(ws), ws.numel(), self._stream())
        elif o["model"] == _lib.MODEL_RBM:
            _lib.call("irl_otf_colstats_rbm_f64", _lib.ptr(o["xbits"]), _lib.ptr(o["t"]), n, o["n_in"], o["hidden"],
                      self.ld, _lib.ptr(self.weights), _lib.ptr(c), _lib.ptr(obar), _lib.ptr(g), _lib.ptr(ws),
                      ws.numel(), self._stream())
        else:
            _lib.call("irl_otf_colstats_mlp_f64", _lib.ptr(o["xbits"]), _lib.ptr(o["t"]), _lib.ptr(o["g"]), n,
                      o["n_in"], o["hidden"], self.ld, _lib.ptr(self.weights), _lib.ptr(c), _lib.ptr(obar),
                      _lib.ptr(g), _lib.ptr(ws), ws.numel(), self._stream())
        self._colstats[key] = (obar, g)
        return obar, g

    def _set_colstats(self, mean: float, obar: torch.Tensor, g: torch.Tensor) -> None:
        self._colstats[float(mean)] = (obar, g)

    def obar(self) -> torch.Tensor:
        if self._colstats:
            return next(iter(self._colstats.values()))[0]
        if self._stats_e is None:
            self._energy_pass(None)
        return self.colstats(self._stats_e)[0]


def _check_imag(value: complex, what: str) -> float:
    """est:136-143."""
    if abs(value.imag) > IMAG_RESIDUAL_WARN * max(1.0, abs(value.real)):
        warnings.warn(
            f"{what} has imaginary residual {value.imag:.3e}; expected a real-symmetric problem",
            stacklevel=3,
        )
    return value.real


def estimate_energy(batch: SampleBatch) -> EnergyEstimate:
    """est:146-153: E = Re sum w e, variance = sum w |e - E|^2, std error."""
    if batch.n_rows == 0:
        raise ValueError("empty batch")
    host, _ = batch._energy_pass(None)
    mean = _check_imag(complex(host[0], host[1]), "energy mean")
    variance = float(host[2])
    std_error = 0.0 if batch.exact else float(np.sqrt(variance / batch.n_samples))
    return EnergyEstimate(mean=mean, variance=variance, std_error=std_error)


def energy_gradient(batch: SampleBatch, energy: EnergyEstimate) -> torch.Tensor:
    """est:156-163: F = 2 Re( (w e) @ conj(O) - E (w @ conj(O)) ), device tensor (P,).

    Computed as 2 Re sum w (e - E) conj(O) (same value, no
    cancellation).  Hermitian batches return the complex 2 g, whose real and
    imaginary parts are the reference's real-embedding gradient halves.
    """
    if batch.n_rows == 0:
        raise ValueError("empty batch")
    _, g = batch.colstats(energy.mean)
    g = g[: batch.param_count]
    if batch.kind == KIND_HERMITIAN:
        return 2.0 * g
    return 2.0 * (g.real if batch.is_complex else g)


_OTF_FORM_G = os.environ.get("IRL_OTF_FORM_G", "1")


def _otf_form_g(o: dict) -> bool:
    """On-the-fly MLP product: form G = u (1 - t^2) inside the GEMM kernels
    (irl_otf_mvp_mlp_u_f64) instead of reading the stored g."""
    return o.get("u") is not None and _OTF_FORM_G != "0"


def _apply(batch: SampleBatch, coeff: torch.Tensor | None, v: torch.Tensor, out: torch.Tensor, *,
           mode: int = _lib.MVP_AUTO, half_f=None, u0=None, out0=None, cache: "ConnectedCache | None" = None) -> None:
    """Raw device product on padded vectors; no validation (driver fast path).

    real/complex_raw: v, out, half_f are real padded vectors (ld,) (views OK).
    hermitian: v, out, half_f are (re, im) tuples of real padded vectors.
    With ``cache`` the two-configuration completion (est:254-294) is added in
    the same launch sequence; ``coeff=None`` then gives the completion alone.
    """
    obar = batch.obar()
    stream = batch._stream()
    n = batch.n_rows
    if cache is not None:
        _apply_connected(batch, cache, coeff, obar, v, out, mode, half_f, u0, out0, stream)
        return
    ws = batch.mvp_workspace()
    if batch.otf is not None:
        o = batch.otf
        if batch.kind == KIND_HERMITIAN:
            (v_re, v_im), (o_re, o_im) = v, out
            h_re, h_im = half_f if half_f is not None else (None, None)
            _lib.call("irl_otf_mvp_rbm_c128", _lib.ptr(o["xbits"]), _lib.ptr(o["t"]), n, o["n_in"], o["hidden"],
                      batch.ld, _lib.ptr(obar), _lib.ptr(coeff), _lib.ptr(v_re), _lib.ptr(v_im), _lib.ptr(o_re),
                      _lib.ptr(o_im), _lib.ptr(h_re), _lib.ptr(h_im), _lib.ptr(u0), _lib.ptr(out0), _lib.ptr(ws),
                      ws.numel(), stream)
            return
        if o["model"] == _lib.MODEL_RBM:
            _lib.call("irl_otf_mvp_rbm_f64", _lib.ptr(o["xbits"]), _lib.ptr(o["t"]), n, o["n_in"], o["hidden"],
                      batch.ld, _lib.ptr(obar), _lib.ptr(coeff), _lib.ptr(v), _lib.ptr(out), _lib.ptr(half_f),
                      _lib.ptr(u0), _lib.ptr(out0), _lib.ptr(ws), ws.numel(), stream)
            return
        if _otf_form_g(o):
            fn, gv = "irl_otf_mvp_mlp_u_f64", o["u"]
        else:
            fn, gv = "irl_otf_mvp_mlp_f64", o["g"]
        _lib.call(fn, _lib.ptr(o["xbits"]), _lib.ptr(o["t"]), _lib.ptr(gv), n, o["n_in"],
                  o["hidden"], batch.ld, _lib.ptr(obar), _lib.ptr(coeff), _lib.ptr(v), _lib.ptr(out),
                  _lib.ptr(half_f), _lib.ptr(u0), _lib.ptr(out0), _lib.ptr(ws), ws.numel(), stream)
        return
    if not batch.is_complex:
        _lib.call("irl_mvp_f64", _lib.ptr(batch.o_padded), n, batch.param_count, batch.ld, _lib.ptr(obar),
                  _lib.ptr(coeff), _lib.ptr(v), _lib.ptr(out), _lib.ptr(half_f), _lib.ptr(u0), _lib.ptr(out0),
                  int(mode), _lib.ptr(ws), ws.numel(), stream)
        return
    if batch.kind == KIND_HERMITIAN:
        v_re, v_im = v
        o_re, o_im = out
        h_re, h_im = half_f if half_f is not None else (None, None)
    else:
        v_re, v_im, o_re, o_im = v, None, out, None
        h_re, h_im = half_f, None
    _lib.call("irl_mvp_c128", _lib.ptr(batch.o_padded), n, batch.param_count, batch.ld, _lib.ptr(obar),
              _lib.ptr(coeff), _lib.ptr(v_re), _lib.ptr(v_im), _lib.ptr(o_re), _lib.ptr(o_im), _lib.ptr(h_re),
              _lib.ptr(h_im), _lib.ptr(u0), _lib.ptr(out0), int(mode), _lib.ptr(ws), ws.numel(), stream)


def _apply2(batch: SampleBatch, coeff_a: torch.Tensor, coeff_b: torch.Tensor, v, out_a, out_b, *, half_f=None,
            u0=None, out0=None) -> None:
    """Two raw device products for the same padded ``v`` (``irl_mvp2_*``):
    ``out_a`` with ``coeff_a`` and the optional bordered terms, ``out_b`` with
    ``coeff_b``.  Stored batches whose rows take the fused single-pass path
    stream O once for both; every other batch runs two ``_apply`` calls."""
    if batch.otf is not None:
        _apply(batch, coeff_a, v, out_a, half_f=half_f, u0=u0, out0=out0)
        _apply(batch, coeff_b, v, out_b)
        return
    obar = batch.obar()
    stream = batch._stream()
    ws = batch.mvp2_workspace()
    n = batch.n_rows
    if not batch.is_complex:
        _lib.call("irl_mvp2_f64", _lib.ptr(batch.o_padded), n, batch.param_count, batch.ld, _lib.ptr(obar),
                  _lib.ptr(coeff_a), _lib.ptr(coeff_b), _lib.ptr(v), _lib.ptr(out_a), _lib.ptr(out_b),
                  _lib.ptr(half_f), _lib.ptr(u0), _lib.ptr(out0), _lib.ptr(ws), ws.numel(), stream)
        return
    if batch.kind == KIND_HERMITIAN:
        v_re, v_im = v
        a_re, a_im = out_a
        b_re, b_im = out_b
        h_re, h_im = half_f if half_f is not None else (None, None)
    else:
        v_re, v_im, a_re, a_im, b_re, b_im = v, None, out_a, None, out_b, None
        h_re, h_im = half_f, None
    _lib.call("irl_mvp2_c128", _lib.ptr(batch.o_padded), n, batch.param_count, batch.ld, _lib.ptr(obar),
              _lib.ptr(coeff_a), _lib.ptr(coeff_b), _lib.ptr(v_re), _lib.ptr(v_im), _lib.ptr(a_re), _lib.ptr(a_im),
              _lib.ptr(b_re), _lib.ptr(b_im), _lib.ptr(h_re), _lib.ptr(h_im), _lib.ptr(u0), _lib.ptr(out0),
              _lib.ptr(ws), ws.numel(), stream)


def _apply_connected(batch, cache, coeff, obar, v, out, mode, half_f, u0, out0, stream) -> None:
    cache._check_batch(batch)
    ws = cache.workspace(batch)
    n = batch.n_rows
    tail = (_lib.ptr(batch.weights), _lib.ptr(coeff), _lib.ptr(cache.dist_index), _lib.ptr(cache.indptr),
            _lib.ptr(cache.partner_row), _lib.ptr(cache.coeff))
    if batch.otf is not None:
        # on-the-fly batch: partner dots from the stored partner rows, or (in-batch
        # partners) from the product's own centred dots
        o = batch.otf
        po = _lib.ptr(cache.partner_o)
        pr = cache.partner_otf or {}
        regen = (_lib.ptr(pr.get("xbits")), _lib.ptr(pr.get("t")), _lib.ptr(pr.get("g")))
        if batch.kind == KIND_HERMITIAN:
            (v_re, v_im), (o_re, o_im) = v, out
            h_re, h_im = half_f if half_f is not None else (None, None)
            _lib.call("irl_otf_connected_mvp_rbm_c128", _lib.ptr(o["xbits"]), _lib.ptr(o["t"]), n, o["n_in"],
                      o["hidden"], batch.ld, _lib.ptr(obar), *tail, po, cache.n_partner, _lib.ptr(v_re),
                      _lib.ptr(v_im), _lib.ptr(o_re), _lib.ptr(o_im), _lib.ptr(h_re), _lib.ptr(h_im), _lib.ptr(u0),
                      _lib.ptr(out0), _lib.ptr(ws), ws.numel(), stream)
        elif o["model"] == _lib.MODEL_RBM:
            _lib.call("irl_otf_connected_mvp_rbm_f64", _lib.ptr(o["xbits"]), _lib.ptr(o["t"]), n, o["n_in"],
                      o["hidden"], batch.ld, _lib.ptr(obar), *tail, po, *regen, cache.n_partner, _lib.ptr(v),
                      _lib.ptr(out),
                      _lib.ptr(half_f), _lib.ptr(u0), _lib.ptr(out0), _lib.ptr(ws), ws.numel(), stream)
        else:
            _lib.call("irl_otf_connected_mvp_mlp_f64", _lib.ptr(o["xbits"]), _lib.ptr(o["t"]), _lib.ptr(o["g"]), n,
                      o["n_in"], o["hidden"], batch.ld, _lib.ptr(obar), *tail, po, *regen, cache.n_partner,
                      _lib.ptr(v),
                      _lib.ptr(out), _lib.ptr(half_f), _lib.ptr(u0), _lib.ptr(out0), _lib.ptr(ws), ws.numel(),
                      stream)
        return
    po = batch.o_padded if cache.in_batch else cache.partner_o
    common = (_lib.ptr(batch.o_padded), n, batch.param_count, batch.ld, _lib.ptr(obar), *tail, _lib.ptr(po),
              cache.n_partner)
    if not batch.is_complex:
        _lib.call("irl_connected_mvp_f64", *common, _lib.ptr(v), _lib.ptr(out), _lib.ptr(half_f), _lib.ptr(u0),
                  _lib.ptr(out0), int(mode), _lib.ptr(ws), ws.numel(), stream)
        return
    if batch.kind == KIND_HERMITIAN:
        (v_re, v_im), (o_re, o_im) = v, out
        h_re, h_im = half_f if half_f is not None else (None, None)
    else:
        v_re, v_im, o_re, o_im = v, None, out, None
        h_re, h_im = half_f, None
    _lib.call("irl_connected_mvp_c128", *common, _lib.ptr(v_re), _lib.ptr(v_im), _lib.ptr(o_re), _lib.ptr(o_im),
              _lib.ptr(h_re), _lib.ptr(h_im), _lib.ptr(u0), _lib.ptr(out0), int(mode), _lib.ptr(ws), ws.numel(),
              stream)


def _staging(batch: SampleBatch, shape) -> torch.Tensor:
    """Zero-padded device input buffer reused across calls on one stream.

    Only the first P entries of a row are ever written, so the padding stays
    zero; reuse is safe because every use is ordered on the same stream.
    """
    key = (_lib.stream_handle(batch.device), tuple(shape))
    st = batch.__dict__.setdefault("_stage", {})
    buf = st.get(key)
    if buf is None:
        buf = torch.zeros(shape, dtype=torch.float64, device=batch.device)
        st[key] = buf
    return buf


_E2E_GRAPHS = os.environ.get("IRL_E2E_GRAPH", "1") != "0"


def _host_product_graph(batch: SampleBatch, coeff, v: torch.Tensor, mode: int, cache) -> torch.Tensor:
    """Host vector in -> host vector out as ONE CUDA graph replay: the H2D copy
    from a pinned staging vector, the product's launches and the D2H copy are
    captured once per (batch, coefficient, mode, cache, stream); a call copies
    v into the staging vector, replays, synchronises and returns a fresh copy."""
    import gc

    dev = batch.device
    p, ld = batch.param_count, batch.ld
    key = (_lib.stream_handle(dev), id(coeff), int(mode), id(cache) if cache is not None else None)
    graphs = batch.__dict__.setdefault("_e2e_graphs", {})
    hit = graphs.get(key)
    if hit is None:
        vin = torch.zeros(ld, dtype=torch.float64, device=dev)
        vout = torch.empty(ld, dtype=torch.float64, device=dev)
        hin = torch.zeros(p, dtype=torch.float64, pin_memory=True)
        hout = torch.empty(p, dtype=torch.float64, pin_memory=True)

        def body():
            vin[:p].copy_(hin, non_blocking=True)
            _apply(batch, coeff, vin, vout, mode=mode, cache=cache)
            hout.copy_(vout[:p], non_blocking=True)

        body()  # eager once: plans, workspaces
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        gc.collect()
        was = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                body()
        finally:
            if was:
                gc.enable()
        # the graph reads and writes these buffers on every replay: they must live
        # as long as the graph (a freed vin / vout would be handed to other
        # tensors by the caching allocator and overwritten by later replays)
        hit = (g, hin, hout, coeff, cache, vin, vout, body)
        graphs[key] = hit
    g, hin, hout = hit[0], hit[1], hit[2]
    hin.copy_(v if v.dtype == torch.float64 else v.to(torch.float64))
    g.replay()
    torch.cuda.current_stream(dev).synchronize()
    return hout.clone()


def _product(batch: SampleBatch, coeff: torch.Tensor | None, v, mode: int, cache: "ConnectedCache | None" = None):
    p = batch.param_count
    as_numpy = not isinstance(v, torch.Tensor)
    on_host = (not as_numpy) and not v.is_cuda
    if as_numpy or on_host:
        v_arr = np.asarray(v) if as_numpy else v.detach().numpy()
        shape = v_arr.shape
        finite = bool(np.isfinite(v_arr).all()) if shape == (p,) else True
    else:
        shape = tuple(v.shape)
        finite = bool(torch.isfinite(v).all()) if shape == (p,) else True
    if shape != (p,):  # est:178-181
        raise ValueError(f"vector length {shape} does not match p={p}")
    if not finite:  # est:182-183
        raise ValueError("non-finite input vector")
    dev = batch.device
    ld = batch.ld
    # host tensors (pinned for async copies) in -> host tensor out: the e2e path
    if batch.kind == KIND_HERMITIAN:
        vt = _as_tensor(v, torch.complex128, dev) if not on_host else v.to(torch.complex128).to(dev, non_blocking=True)
        vin = _staging(batch, (2, ld))
        vin[0, :p] = vt.real
        vin[1, :p] = vt.imag
        vout = _staging(batch, (3, ld))[1:] if on_host else torch.empty((2, ld), dtype=torch.float64, device=dev)
        _apply(batch, coeff, (vin[0], vin[1]), (vout[0], vout[1]), mode=mode, cache=cache)
        res = torch.complex(vout[0, :p], vout[1, :p])
    else:
        if (not as_numpy) and torch.is_complex(v):
            raise ValueError("complex vector needs a hermitian batch")
        if on_host and _E2E_GRAPHS:
            return _host_product_graph(batch, coeff, v, mode, cache)
        vin = _staging(batch, (ld,))
        if on_host:
            vin[:p].copy_(v if v.dtype == torch.float64 else v.to(torch.float64), non_blocking=True)
        else:
            vin[:p] = _as_tensor(v, torch.float64, dev)
        vout = _staging(batch, (1, ld))[0] if on_host else torch.empty(ld, dtype=torch.float64, device=dev)
        _apply(batch, coeff, vin, vout, mode=mode, cache=cache)
        res = vout[:p]
    if on_host:
        dst = torch.empty(res.shape, dtype=res.dtype, pin_memory=v.is_pinned())
        dst.copy_(res, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return dst
    return res.cpu().numpy() if as_numpy else res


def heff_matvec(batch: SampleBatch, energy: EnergyEstimate, v, *, mode: int = _lib.MVP_AUTO):
    """est:171-186: H_eff v = O_c^H (w e_c (O_c v)) without forming O_c or H_eff.

    numpy in -> numpy out (reference behaviour); torch in -> torch out.
    """
    return _product(batch, batch.coefficients(energy.mean), v, mode)


def _qgt_coeff(batch: SampleBatch) -> torch.Tensor:
    """Coefficient w of S v (cached: the complex kinds need it as c128)."""
    if not batch.is_complex:
        return batch.weights
    c = batch.__dict__.get("_wc")
    if c is None:
        c = batch.weights.to(torch.complex128)
        batch._wc = c
    return c


def qgt_matvec(batch: SampleBatch, v, *, mode: int = _lib.MVP_AUTO):
    """S v = O_c^H (w (O_c v)) — matrix-free ``dense_qgt`` (est:335-344)."""
    return _product(batch, _qgt_coeff(batch), v, mode)


def heff_qgt_matvec(batch: SampleBatch, energy: EnergyEstimate, v):
    """(H_eff v, S v) for one v -- est:171-186 with both coefficient vectors
    (w e_c and w) over a single read of the stored O where the rows take the
    fused single-pass path (``irl_mvp2_*``); the GEVP form H_eff c = lambda S c
    (PAPER Eq. 11; dense oracles est:319-344) applies both to every iterate.

    numpy in -> numpy pair out; torch (device) in -> torch pair out.
    """
    p = batch.param_count
    as_numpy = not isinstance(v, torch.Tensor)
    shape = np.asarray(v).shape if as_numpy else tuple(v.shape)
    if shape != (p,):  # est:178-181
        raise ValueError(f"vector length {shape} does not match p={p}")
    dev, ld = batch.device, batch.ld
    ch, cs = batch.coefficients(energy.mean), _qgt_coeff(batch)
    if batch.kind == KIND_HERMITIAN:
        vt = _as_tensor(v, torch.complex128, dev)
        if not bool(torch.isfinite(torch.view_as_real(vt)).all()):  # est:182-183
            raise ValueError("non-finite input vector")
        vin = _staging(batch, (2, ld))
        vin[0, :p] = vt.real
        vin[1, :p] = vt.imag
        out = torch.empty((4, ld), dtype=torch.float64, device=dev)
        _apply2(batch, ch, cs, (vin[0], vin[1]), (out[0], out[1]), (out[2], out[3]))
        hv, sv = torch.complex(out[0, :p], out[1, :p]), torch.complex(out[2, :p], out[3, :p])
    else:
        if (not as_numpy) and torch.is_complex(v):
            raise ValueError("complex vector needs a hermitian batch")
        vt = _as_tensor(v, torch.float64, dev)
        if not bool(torch.isfinite(vt).all()):
            raise ValueError("non-finite input vector")
        vin = _staging(batch, (ld,))
        vin[:p] = vt
        out = torch.empty((2, ld), dtype=torch.float64, device=dev)
        _apply2(batch, ch, cs, vin, out[0], out[1])
        hv, sv = out[0, :p], out[1, :p]
    if as_numpy:
        return hv.cpu().numpy(), sv.cpu().numpy()
    return hv, sv


class ConnectedCache:
    """Device-resident off-diagonal couplings of a batch (est:189-218).

    Same fields as the reference dataclass: batch row n maps to distinct
    configuration ``dist_index[n]``; the partners of distinct configuration k
    are the CSR slice ``indptr[k]:indptr[k+1]`` of ``partner_row`` / ``coeff``;
    ``coeff`` holds <x|H|y> psi(y)/psi(x) and ``partner_row`` indexes rows of
    ``partner_o``.  Arrays may be numpy (uploaded once) or device tensors;
    ``partner_o`` may be host (M, P) or an already padded device tensor
    (M, ld).  Real batches keep ``Re(coeff)``: with real O the reference's
    ``Re((w corr) @ conj(O_c))`` only sees the real part.  Indices are checked
    once here (the reference indexes without checks; an out-of-range index
    would raise IndexError there).
    """

    def __init__(self, dist_index, indptr, partner_row, coeff, partner_o, *, batch: SampleBatch,
                 partner_otf: dict | None = None):
        dev = batch.device
        kind_c = batch.is_complex
        cdt = torch.complex128 if kind_c else torch.float64

        def idx(a):  # int64 device tensor; validation runs where the data lives
            if isinstance(a, torch.Tensor):
                return a.to(device=dev, dtype=torch.int64).contiguous()
            return torch.as_tensor(np.asarray(a, dtype=np.int64), device=dev)

        di, ip, pr = idx(dist_index), idx(indptr), idx(partner_row)
        n = batch.n_rows
        if tuple(di.shape) != (n,):
            raise ValueError("dist_index must have one entry per batch row")
        if ip.dim() != 1 or ip.numel() < 1 or int(ip[0]) != 0 or (ip.numel() > 1 and bool((ip[1:] < ip[:-1]).any())):
            raise ValueError("indptr must start at 0 and be non-decreasing")
        n_dist = ip.numel() - 1
        if n and (int(di.min()) < 0 or int(di.max()) >= n_dist):
            raise IndexError("dist_index out of range")
        nnz = int(ip[-1])
        if tuple(pr.shape) != (nnz,):
            raise ValueError("partner_row length must equal indptr[-1]")
        ld, p = batch.ld, batch.param_count
        if partner_otf is not None:
            # partners regenerated on the fly (real models): packed inputs + hidden activations
            if batch.otf is None or batch.is_complex:
                raise ValueError("regenerated partners need a real on-the-fly batch")
            po = None
        elif partner_o is None or partner_o is batch.o_padded or _same_view(partner_o, batch):
            po = None  # partners are batch rows (exact mode): partner_row indexes the batch
        elif isinstance(partner_o, torch.Tensor) and partner_o.is_cuda and partner_o.ndim == 2 \
                and partner_o.shape[1] == ld and partner_o.dtype == cdt:
            po = partner_o.contiguous()
        else:
            src = partner_o
            if not isinstance(src, torch.Tensor):
                src = np.asarray(src)
                if not kind_c and np.iscomplexobj(src):
                    imax = float(np.max(np.abs(src.imag))) if src.size else 0.0
                    if imax > 0.0:
                        raise ValueError("complex partner_o needs a complex batch kind")
                    src = src.real
            m = int(src.shape[0]) if src.ndim == 2 else 0
            if m and src.shape[1] != p:
                raise ValueError("partner_o width does not match param_count")
            po = torch.zeros((max(m, 0), ld), dtype=cdt, device=dev)
            if m:
                po[:, :p] = _as_tensor(src, cdt, dev)
        if partner_otf is not None:
            m = int(partner_otf["t"].shape[0])
        else:
            m = n if po is None else int(po.shape[0])
        if nnz and (int(pr.min()) < 0 or int(pr.max()) >= m):
            raise IndexError("partner_row out of range")
        if isinstance(coeff, torch.Tensor):
            c = coeff.detach().to(dev)
        else:
            c = torch.as_tensor(np.asarray(coeff), device=dev)
        if tuple(c.shape) != (nnz,):
            raise ValueError("coeff length must equal indptr[-1]")
        if not kind_c and torch.is_complex(c):
            c = c.real
        self.dist_index = di
        self.indptr = ip
        self.partner_row = pr
        self.coeff = c.to(cdt).contiguous()
        self.partner_o = po
        self.partner_otf = partner_otf
        self.n_partner = m
        self.n_dist = n_dist
        self._batch_id = id(batch)
        self._ws: dict = {}  # stream handle -> workspace

    @classmethod
    def from_reference(cls, cache, batch: SampleBatch) -> "ConnectedCache":
        """Upload a reference ``irlnqs.estimators.ConnectedCache`` (or any object with its fields)."""
        return cls(cache.dist_index, cache.indptr, cache.partner_row, cache.coeff, cache.partner_o, batch=batch)

    def _check_batch(self, batch: SampleBatch) -> None:
        if self._batch_id != id(batch):
            raise ValueError("connected cache was built for another batch")

    @property
    def in_batch(self) -> bool:
        """Partners are the batch's own rows (no separate partner O)."""
        return self.partner_o is None and self.partner_otf is None

    def workspace(self, batch: SampleBatch) -> torch.Tensor:
        """Per-stream workspace (see SampleBatch.mvp_workspace)."""
        key = batch._stream()
        ws = self._ws.get(key)
        if ws is None:
            if batch.otf is not None:
                o = batch.otf
                nbytes = int(_lib.lib().irl_otf_connected_workspace_bytes(
                    int(o["model"]), batch.n_rows, 0 if self.in_batch else self.n_partner, o["n_in"], o["hidden"],
                    batch.ld, int(batch.is_complex)))
            else:
                nbytes = int(_lib.lib().irl_connected_workspace_bytes(batch.n_rows, self.n_partner, batch.ld,
                                                                       int(batch.is_complex)))
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=batch.device)
            self._ws[key] = ws
        return ws


def _same_view(partner_o, batch: SampleBatch) -> bool:
    """``partner_o`` is the batch's own (N, P) ``o_matrix`` view."""
    if not isinstance(partner_o, torch.Tensor) or batch.otf is not None:
        return False
    o = batch.o_padded
    return (partner_o.is_cuda and partner_o.data_ptr() == o.data_ptr() and tuple(partner_o.shape) ==
            (batch.n_rows, batch.param_count) and partner_o.stride() == o.stride())


def partner_rows_in_batch(uniq_bits: np.ndarray, reps: np.ndarray, partner_bits: torch.Tensor):
    """Batch O rows of partner configurations, when every partner is a batch row.

    ``uniq_bits``: the batch's distinct configurations (ascending uint64),
    ``reps``: a batch row of each; ``partner_bits``: device int64 view of the
    partners' uint64 bitmasks.  Returns the batch row of every partner (device
    int64), or None when some partner is not in the batch.  In exact mode the
    batch is the whole sector, which every connected partner lies in, so the
    cache points into the batch's own O (the reference's o_row table,
    est:236-242, without a second copy of the rows).
    """
    dev = partner_bits.device
    keys = torch.as_tensor(np.ascontiguousarray(uniq_bits, dtype=np.uint64).view(np.int64), device=dev)
    out = torch.empty(partner_bits.numel(), dtype=torch.int64, device=dev)
    _lib.call("irl_sorted_lookup", _lib.ptr(keys), keys.numel(), _lib.ptr(partner_bits), partner_bits.numel(),
              _lib.ptr(out), _lib.stream_handle(dev))
    if out.numel() and bool((out < 0).any()):
        return None
    return torch.as_tensor(np.asarray(reps, dtype=np.int64), device=dev)[out]


def heff_offdiag_matvec(batch: SampleBatch, cache: ConnectedCache, v, *, mode: int = _lib.MVP_AUTO):
    """est:254-294: two-configuration completion of the H_eff product.

    ``Re(((w corr) @ conj(O_c)))`` with ``corr_n = sum_y coeff (q(y) - q(x_n))``,
    ``q = (O - Obar) v``; one partner dot pass, a per-row CSR kernel and one
    streaming pass over the batch O (``irl_connected_mvp_*`` with no diagonal
    coefficient).  Hermitian batches return the complex product of the
    reference's real embedding.
    """
    return _product(batch, None, v, mode, cache=cache)


def connected_heff_matvec(batch: SampleBatch, energy: EnergyEstimate, cache: ConnectedCache, v, *,
                          mode: int = _lib.MVP_AUTO):
    """``heff_matvec + heff_offdiag_matvec`` (the optimizer's operator, opt:144-147) in one product."""
    return _product(batch, batch.coefficients(energy.mean), v, mode, cache=cache)


def _dense_from_products(batch: SampleBatch, coeff: torch.Tensor, cap: int) -> np.ndarray:
    p = batch.param_count
    if p > cap:
        raise DensePCapError(f"p={p} above the dense cap of {cap}")
    cols = []
    for k in range(p):
        e_k = np.zeros(p, dtype=complex if batch.kind == KIND_HERMITIAN else float)
        e_k[k] = 1.0
        cols.append(_product(batch, coeff, e_k, _lib.MVP_AUTO))
    mat = np.stack(cols, axis=1)
    if batch.kind != KIND_HERMITIAN:
        mat = mat.real
        asym = float(np.max(np.abs(mat - mat.T))) if p else 0.0
        if asym > IMAG_RESIDUAL_WARN:
            warnings.warn(f"dense H_eff asymmetric by {asym:.3e}", stacklevel=3)
        return (mat + mat.T) / 2
    return (mat + mat.conj().T) / 2


def dense_heff(batch: SampleBatch, energy: EnergyEstimate, cap: int = DEFAULT_DENSE_P_CAP) -> np.ndarray:
    """est:319-332, assembled column by column from the device product."""
    return _dense_from_products(batch, batch.coefficients(energy.mean), cap)


def dense_qgt(batch: SampleBatch, cap: int = DEFAULT_DENSE_P_CAP) -> np.ndarray:
    """est:335-344, assembled column by column from the device product."""
    coeff = batch.weights if not batch.is_complex else batch.weights.to(torch.complex128)
    return _dense_from_products(batch, coeff, cap)
