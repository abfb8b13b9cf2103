"""Shallow NQS ansaetze (RBM, one-hidden-layer MLP) with batched device O-rows.

The reference's only ansatz is autoregressive (``ansatz.py:1-14``); BASELINE
names RBM and shallow-MLP NQS, so this module keeps the reference's *NQS
seam* — ``Architecture.param_count`` (``ans:26-38``), ``AnsatzParameters``
(``ans:41-53``), ``log_derivative(params, x, sector)`` (``ans:249-290``) — and
adds the batched form the hot path needs, ``log_derivative_batch`` and
``build_batch`` (the role of ``estimators.build_batch``, ``est:79-133``, with
synthetic E_loc instead of a Hamiltonian), ``log_amplitude_batch`` (``ans:200``)
and ``build_connected_cache`` (``est:221-251``, partners given as input).

Encodings: inputs are 0/1 occupations (``sigma_i = x_i``), not
the reference's +-1 encodings (``ans:156-162``, ``ans:243-246``).

Rows (layouts SURVEY Appendix A):

* RBM  theta = [a (n), b (h), W (h x n)],  theta_j = b_j + sum_i W_ji x_i,
  O = [x (n), tanh theta (h), (tanh theta_j x_i)_{j,i} (h n)]   (holomorphic
  in complex theta: cfg4);
* MLP  theta = [W (h x n_in), b (h), u (h), c],  t = tanh(W x + b),
  g = u (1 - t^2),  O = [(g_j x_k)_{j,k} (h n_in), g (h), t (h), 1]
  — the reference phase-head gradient (``ans:278-288``) without ``w_lin``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .estimators import KIND_HERMITIAN, KIND_REAL, ConnectedCache, SampleBatch, _as_tensor, _device


@dataclass(frozen=True)
class RBMArchitecture:
    n_visible: int
    hidden: int
    complex_params: bool = False

    @property
    def param_count(self) -> int:
        n, h = self.n_visible, self.hidden
        return n + h + h * n

    @property
    def model(self) -> int:
        return _lib.MODEL_RBM

    @property
    def n_inputs(self) -> int:
        return self.n_visible


@dataclass(frozen=True)
class MLPArchitecture:
    n_in: int
    hidden: int
    complex_params: bool = False

    def __post_init__(self):
        if self.complex_params:
            raise ValueError("the shallow MLP NQS has real parameters")

    @property
    def param_count(self) -> int:
        return self.hidden * self.n_in + 2 * self.hidden + 1

    @property
    def model(self) -> int:
        return _lib.MODEL_MLP

    @property
    def n_inputs(self) -> int:
        return self.n_in


Architecture = RBMArchitecture | MLPArchitecture


@dataclass(frozen=True)
class AnsatzParameters:
    """Flat parameter vector for an architecture (ans:41-53)."""

    architecture: RBMArchitecture | MLPArchitecture
    theta: np.ndarray

    def __post_init__(self):
        want = (self.architecture.param_count,)
        if tuple(np.shape(self.theta)) != want:
            raise ValueError(
                f"theta has length {np.shape(self.theta)}, architecture needs {self.architecture.param_count}"
            )
        if self.architecture.complex_params != np.iscomplexobj(self.theta):
            raise ValueError("theta dtype does not match architecture.complex_params")
        if isinstance(self.theta, np.ndarray):
            self.theta.setflags(write=False)


def _theta_device(params: AnsatzParameters, dev) -> torch.Tensor:
    arch = params.architecture
    if arch.complex_params:
        t = torch.as_tensor(np.array(params.theta, dtype=np.complex128), device=dev)
        return torch.view_as_real(t).reshape(-1).contiguous()  # interleaved (re, im)
    return torch.as_tensor(np.array(params.theta, dtype=np.float64), device=dev)


def _x_device(x, n_inputs: int, dev) -> torch.Tensor:
    xt = _as_tensor(x, torch.uint8, dev).contiguous()
    if xt.dim() != 2 or xt.shape[1] != n_inputs:
        raise ValueError(f"x must be (N, {n_inputs}) 0/1 occupations")
    return xt


AUTO_OTF_MIN_BYTES = 256 << 20


def otf_supported(arch) -> bool:
    """On-the-fly kernels: n_inputs <= 100 packed bits per row; real models need
    an even hidden width (16-byte tile rows)."""
    return arch.n_inputs <= 100 and (bool(arch.complex_params) or arch.hidden % 2 == 0)


def build_batch(params: AnsatzParameters, x, e_loc, weights=None, n_samples: int | None = None,
                device=None, mode: str = "stored") -> SampleBatch:
    """Device SampleBatch with O built by the fused row kernel (K1/K2).

    One launch sequence: k_energy (E, c = w (e - E)) -> hidden layer on FP64
    tensor cores -> k_orows (O rows; column statistics fused or from the DMMA
    GEMM) -> finisher.  ``weights`` defaults to 1/N (stochastic mode, est:99-100).

    ``mode``: "stored" materialises O in HBM; "otf" keeps only the hidden
    activations and regenerates O inside every product (see
    :func:`build_batch_otf`); "auto" picks "otf" whenever the model supports it
    and the stored O would exceed ``AUTO_OTF_MIN_BYTES`` (measured on B200: the
    DMMA regeneration beats streaming O from HBM 3.4x on cfg2, 3.6x on cfg3,
    13x on cfg4, 12x on cfg5, while a small L2-resident O such as cfg1 streams
    faster), and "stored" otherwise.
    """
    arch = params.architecture
    if mode not in ("stored", "otf", "auto"):
        raise ValueError(f"unknown build mode {mode!r}")
    if mode == "auto" and otf_supported(arch):
        n_rows = int(np.shape(x)[0]) if not isinstance(x, torch.Tensor) else int(x.shape[0])
        o_bytes = n_rows * arch.param_count * (16 if arch.complex_params else 8)
        if o_bytes >= AUTO_OTF_MIN_BYTES:
            mode = "otf"
    if mode == "otf":
        return build_batch_otf(params, x, e_loc, weights=weights, n_samples=n_samples, device=device)
    dev = _device(device)
    xt = _x_device(x, arch.n_inputs, dev)
    n = int(xt.shape[0])
    if n < 1:
        raise ValueError("empty batch")
    if weights is None:
        weights = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
        if n_samples is None:
            n_samples = n
    kind = KIND_HERMITIAN if arch.complex_params else KIND_REAL
    p = arch.param_count
    ld = _lib.padded_ld(p, arch.complex_params)
    odt = torch.complex128 if arch.complex_params else torch.float64
    o = torch.empty((n, ld), dtype=odt, device=dev)
    batch = SampleBatch(None, weights, e_loc, o, n_samples or 0, kind=kind, param_count=p, device=dev)
    _, mean = batch._energy_pass(None)
    obar = torch.empty(ld, dtype=odt, device=dev)
    g = torch.empty(ld, dtype=odt, device=dev)
    fill_o_rows(params, xt, o, batch.weights, batch.gradient_coefficients(mean), obar, g)
    batch._set_colstats(mean, obar, g)
    return batch


def fill_o_rows(params: AnsatzParameters, xt: torch.Tensor, o: torch.Tensor, w: torch.Tensor,
                coeff: torch.Tensor, obar: torch.Tensor, g: torch.Tensor) -> None:
    """Launch the O-row kernel into preallocated device buffers."""
    arch = params.architecture
    dev = o.device
    n = int(xt.shape[0])
    ld = int(o.shape[1])
    theta = _theta_device(params, dev)
    lib = _lib.lib()
    nbytes = int(lib.irl_obuild_workspace_bytes(arch.model, n, arch.n_inputs, arch.hidden, ld,
                                                int(arch.complex_params)))
    if nbytes == 0:
        raise _lib.NativeError("irl_obuild_workspace_bytes", -1, lib.irl_last_error().decode())
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    if arch.model == _lib.MODEL_RBM:
        fn = "irl_obuild_rbm_c128" if arch.complex_params else "irl_obuild_rbm_f64"
    else:
        fn = "irl_obuild_mlp_f64"
    _lib.call(fn, _lib.ptr(xt), n, arch.n_inputs, arch.hidden, _lib.ptr(theta), _lib.ptr(o), ld, _lib.ptr(w),
              _lib.ptr(coeff), _lib.ptr(obar), _lib.ptr(g), _lib.ptr(ws), nbytes, _lib.stream_handle(dev))


def log_derivative_batch(params: AnsatzParameters, x, device=None) -> torch.Tensor:
    """O = d log psi / d theta for every row of x: device tensor (N, P) view of
    the padded (N, ld) row-major buffer (weights 1/N for the fused stats)."""
    dev = _device(device)
    arch = params.architecture
    xt = _x_device(x, arch.n_inputs, dev)
    n = int(xt.shape[0])
    ld = _lib.padded_ld(arch.param_count, arch.complex_params)
    odt = torch.complex128 if arch.complex_params else torch.float64
    o = torch.empty((n, ld), dtype=odt, device=dev)
    w = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    coeff = torch.zeros(n, dtype=odt, device=dev)
    obar = torch.empty(ld, dtype=odt, device=dev)
    g = torch.empty(ld, dtype=odt, device=dev)
    fill_o_rows(params, xt, o, w, coeff, obar, g)
    return o[:, : arch.param_count]


def log_derivative(params: AnsatzParameters, x, sector=None) -> np.ndarray:
    """Single-sample O(x) (ans:249-290 signature); ``sector`` is accepted for
    API parity and unused (RBM/MLP have no particle-number mask)."""
    xa = np.asarray(x, dtype=np.uint8).reshape(1, -1)
    return log_derivative_batch(params, xa)[0].cpu().numpy()


def hidden_activations(params: AnsatzParameters, x, device=None):
    """(t, g) hidden-layer activations on device (g is None for the RBM)."""
    dev = _device(device)
    arch = params.architecture
    xt = _x_device(x, arch.n_inputs, dev)
    n = int(xt.shape[0])
    theta = _theta_device(params, dev)
    st = _lib.stream_handle(dev)
    if arch.model == _lib.MODEL_RBM:
        if arch.complex_params:
            t = torch.empty((n, arch.hidden), dtype=torch.complex128, device=dev)
            _lib.call("irl_hidden_rbm_c128", _lib.ptr(xt), n, arch.n_visible, arch.hidden, _lib.ptr(theta),
                      _lib.ptr(t), st)
        else:
            t = torch.empty((n, arch.hidden), dtype=torch.float64, device=dev)
            _lib.call("irl_hidden_rbm_f64", _lib.ptr(xt), n, arch.n_visible, arch.hidden, _lib.ptr(theta),
                      _lib.ptr(t), st)
        return t, None
    t = torch.empty((n, arch.hidden), dtype=torch.float64, device=dev)
    g = torch.empty((n, arch.hidden), dtype=torch.float64, device=dev)
    _lib.call("irl_hidden_mlp_f64", _lib.ptr(xt), n, arch.n_in, arch.hidden, _lib.ptr(theta), _lib.ptr(t),
              _lib.ptr(g), st)
    return t, g


def build_batch_otf(params: AnsatzParameters, x, e_loc, weights=None, n_samples: int | None = None,
                    device=None) -> SampleBatch:
    """Batch in on-the-fly mode (K6, SURVEY §2 mvp_onthefly_{mlp,rbm}): O is never stored.

    O's big block is an outer product (MLP: g (x) x, RBM: t (x) x), so every
    product is regenerated from the bit-packed inputs and the hidden
    activations t (, g) with FP64 tensor-core GEMMs.  Real parameters only.
    Same SampleBatch interface (estimate_energy, energy_gradient, heff_matvec,
    qgt_matvec, solve_step) as a stored-O batch.
    """
    arch = params.architecture
    cplx = bool(arch.complex_params)
    if cplx and arch.model != _lib.MODEL_RBM:
        raise ValueError("complex parameters are an RBM feature")
    dev = _device(device)
    xt = _x_device(x, arch.n_inputs, dev)
    n = int(xt.shape[0])
    if n < 1:
        raise ValueError("empty batch")
    if weights is None:
        weights = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
        if n_samples is None:
            n_samples = n
    p = arch.param_count
    ld = _lib.padded_ld(p, cplx)
    odt = torch.complex128 if cplx else torch.float64
    # a zero-width placeholder keeps SampleBatch's validation; O is not stored
    placeholder = torch.empty((n, ld), dtype=odt, device="meta")
    batch = SampleBatch.__new__(SampleBatch)
    SampleBatch._init_common(batch, weights, e_loc, n, n_samples or 0, KIND_HERMITIAN if cplx else KIND_REAL, p, ld,
                             dev)
    batch.o_padded = placeholder
    xbits = torch.empty((n, 2), dtype=torch.int64, device=dev)
    t = torch.empty((n, arch.hidden), dtype=odt, device=dev)
    theta = _theta_device(params, dev)
    if cplx:
        g = None
        _lib.call("irl_otf_prepare_rbm_c128", _lib.ptr(xt), n, arch.n_visible, arch.hidden, _lib.ptr(theta),
                  _lib.ptr(xbits), _lib.ptr(t), _lib.stream_handle(dev))
    elif arch.model == _lib.MODEL_RBM:
        g = None
        _lib.call("irl_otf_prepare_rbm_f64", _lib.ptr(xt), n, arch.n_visible, arch.hidden, _lib.ptr(theta),
                  _lib.ptr(xbits), _lib.ptr(t), _lib.stream_handle(dev))
    else:
        g = torch.empty((n, arch.hidden), dtype=torch.float64, device=dev)
        _lib.call("irl_otf_prepare_mlp_f64", _lib.ptr(xt), n, arch.n_in, arch.hidden, _lib.ptr(theta),
                  _lib.ptr(xbits), _lib.ptr(t), _lib.ptr(g), _lib.stream_handle(dev))
    batch.otf = {"xbits": xbits, "t": t, "g": g, "n_in": arch.n_inputs, "hidden": arch.hidden, "model": arch.model}
    if g is not None:
        # MLP output weights u (theta layout [W, b, u, c], ans:67-83): the product
        # can form G = u (1 - t^2) from t instead of reading g
        off = arch.hidden * arch.n_in + arch.hidden
        batch.otf["u"] = theta[off:off + arch.hidden].contiguous()
    batch._seal()
    return batch


def log_amplitude_batch(params: AnsatzParameters, x, device=None) -> torch.Tensor:
    """log psi for every row of x (role of ``ans.log_amplitude``, ans:200-247):
    RBM ``a.x + sum_j log cosh(b_j + W_j.x)`` (complex for complex theta), MLP
    ``u.tanh(W x + b) + c``.  Device tensor (N,), float64 or complex128."""
    dev = _device(device)
    arch = params.architecture
    xt = _x_device(x, arch.n_inputs, dev)
    n = int(xt.shape[0])
    cplx = bool(arch.complex_params)
    out = torch.empty(n, dtype=torch.complex128 if cplx else torch.float64, device=dev)
    if n == 0:
        return out
    theta = _theta_device(params, dev)
    nbytes = int(_lib.lib().irl_logamp_workspace_bytes(n, arch.hidden, int(cplx)))
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
    if arch.model == _lib.MODEL_RBM:
        fn = "irl_logamp_rbm_c128" if cplx else "irl_logamp_rbm_f64"
    else:
        fn = "irl_logamp_mlp_f64"
    _lib.call(fn, _lib.ptr(xt), n, arch.n_inputs, arch.hidden, _lib.ptr(theta), _lib.ptr(out), _lib.ptr(ws),
              ws.numel(), _lib.stream_handle(dev))
    return out


def log_amplitude(params: AnsatzParameters, x, sector=None):
    """Single-sample log psi (ans:200 signature; ``sector`` unused)."""
    xa = np.asarray(x, dtype=np.uint8).reshape(1, -1)
    v = log_amplitude_batch(params, xa)[0].item()
    return complex(v)


def build_connected_cache(params: AnsatzParameters, batch: SampleBatch, x, partners, elements, indptr,
                          dist_index=None, device=None) -> ConnectedCache:
    """``est.build_connected_cache`` (est:221-251) for the shallow NQS.

    The Hamiltonian side (which partners, and their <x|H|y>) is an input here:
    ``partners`` (nnz, n) holds the connected configurations of distinct
    configuration k in the CSR slice ``indptr[k]:indptr[k+1]``, with
    ``elements`` their matrix elements; ``dist_index`` maps batch rows to
    distinct configurations (default: every row distinct).  On device: log psi
    of the representatives and of the distinct partners (``k_logamp``),
    coefficients ``element * exp(log psi(y) - log psi(x))`` (est:246-248) and
    the partner O rows (the K1/K2 row kernel), deduplicated as the reference's
    ``o_row`` table is (est:236-242).
    """
    dev = _device(device) if device is not None else batch.device
    arch = params.architecture
    xa = np.asarray(x.cpu() if isinstance(x, torch.Tensor) else x, dtype=np.uint8)
    pa = np.asarray(partners.cpu() if isinstance(partners, torch.Tensor) else partners, dtype=np.uint8)
    ip = np.asarray(indptr, dtype=np.int64)
    n = xa.shape[0]
    if n != batch.n_rows:
        raise ValueError("x rows do not match the batch")
    di = np.arange(n, dtype=np.int64) if dist_index is None else np.asarray(dist_index, dtype=np.int64)
    n_dist = len(ip) - 1
    if di.shape != (n,) or (n and (di.min() < 0 or di.max() >= n_dist)):
        raise ValueError("dist_index does not match indptr")
    nnz = int(ip[-1])
    if pa.shape[0] != nnz or np.shape(elements) != (nnz,):
        raise ValueError("partners / elements must have indptr[-1] rows")
    # representative batch row of each distinct configuration (first occurrence, est:228-233)
    reps = np.full(n_dist, -1, dtype=np.int64)
    order = np.arange(n)[::-1]
    reps[di[order]] = order
    if np.any(reps < 0):
        raise ValueError("a distinct configuration has no batch row")
    if nnz:
        uniq, inv = np.unique(pa, axis=0, return_inverse=True)
        inv = inv.reshape(-1)
    else:
        uniq, inv = np.zeros((0, arch.n_inputs), dtype=np.uint8), np.zeros(0, dtype=np.int64)
    m = uniq.shape[0]
    cplx = bool(arch.complex_params)
    odt = torch.complex128 if cplx else torch.float64
    regen = batch.otf is not None and not cplx and m > 0
    po = torch.zeros((0 if regen else m, batch.ld), dtype=odt, device=dev)
    partner_otf = None
    if regen:
        # on-the-fly batch: the partner dots are regenerated from the partners'
        # packed inputs and hidden activations (no partner O stored)
        ut = _x_device(uniq, arch.n_inputs, dev)
        pxb = torch.empty((m, 2), dtype=torch.int64, device=dev)
        pt = torch.empty((m, arch.hidden), dtype=torch.float64, device=dev)
        theta_d = _theta_device(params, dev)
        if arch.model == _lib.MODEL_RBM:
            pg = None
            _lib.call("irl_otf_prepare_rbm_f64", _lib.ptr(ut), m, arch.n_visible, arch.hidden, _lib.ptr(theta_d),
                      _lib.ptr(pxb), _lib.ptr(pt), _lib.stream_handle(dev))
        else:
            pg = torch.empty((m, arch.hidden), dtype=torch.float64, device=dev)
            _lib.call("irl_otf_prepare_mlp_f64", _lib.ptr(ut), m, arch.n_in, arch.hidden, _lib.ptr(theta_d),
                      _lib.ptr(pxb), _lib.ptr(pt), _lib.ptr(pg), _lib.stream_handle(dev))
        partner_otf = {"xbits": pxb, "t": pt, "g": pg}
        lp = log_amplitude_batch(params, uniq, device=dev)
    elif m:
        ut = _x_device(uniq, arch.n_inputs, dev)
        w = torch.full((m,), 1.0 / m, dtype=torch.float64, device=dev)
        scratch = [torch.empty(batch.ld, dtype=odt, device=dev) for _ in range(2)]
        fill_o_rows(params, ut, po, w, torch.zeros(m, dtype=odt, device=dev), scratch[0], scratch[1])
        lp = log_amplitude_batch(params, ut, device=dev)
    lx = log_amplitude_batch(params, xa[reps], device=dev)
    if nnz:
        seg = torch.as_tensor(np.repeat(np.arange(n_dist), np.diff(ip)), device=dev)
        ratio = torch.exp(lp[torch.as_tensor(inv, device=dev)].to(torch.complex128) - lx[seg].to(torch.complex128))
        coeff = torch.as_tensor(np.asarray(elements), dtype=torch.complex128, device=dev) * ratio
    else:
        coeff = torch.zeros(0, dtype=torch.complex128, device=dev)
    return ConnectedCache(di, ip, inv, coeff, po, batch=batch, partner_otf=partner_otf)
