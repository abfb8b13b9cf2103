"""IRL-SR outer-step core: bordered operator, IRL solve, update direction.

The data-parallel part of ``irlnqs.optimizer.outer_step`` (``opt:130-165``):

* the bordered (p+1) closure of ``opt:140-148``
      A([u0; u]) = [ (F/2).u ; u0 F/2 + H_eff u ]
  — here ONE fused device launch (+ finisher) per product: the F/2 row and
  column are folded into the streaming kernel's prologue and epilogue;
  ``heff_offdiag_matvec`` (``opt:146``) is added when a
  :class:`~.estimators.ConnectedCache` is given (``connected=``): one partner
  dot pass and a per-row CSR kernel before the same streaming product; it is
  absent for synthetic E_loc;
* ``krylov.irl_smallest`` on it with the reference's seed rule
  ``_batch_seed`` (``opt:100-101``);
* the direction ``d = c[1:]/c0`` (``opt:160-165``).

With a molecular Hamiltonian (:mod:`.hamiltonian`) the whole reference
outer step runs on the device: :func:`outer_step` (``opt:118-195``: exact
batch, connected cache, the solve, the line search over ``config.line_search``
with the steepest-descent fallback) and :func:`energy_at` (``opt:104-115``).
Adam and the run loop (``opt:198-269``) are out of scope.

Complex-parameter (Hermitian, cfg4) batches use the reference's real
embedding ``[u0, Re c, Im c]`` (dimension 2P+1), so the driver,
start vector and matvec count are those of ``kry.irl_smallest`` on the
embedded operator.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _lib, krylov
from .estimators import (
    KIND_HERMITIAN,
    ConnectedCache,
    EnergyEstimate,
    SampleBatch,
    _apply,
    _apply2,
    _qgt_coeff,
    energy_gradient,
    estimate_energy,
)


DEFAULT_LINE_SEARCH_GRID = tuple(2.0**k for k in range(-6, 2))  # opt:29


@dataclass(frozen=True)
class OptimizerConfig:
    """``opt:41-57`` minus Adam (defaults identical)."""

    method: str = "irl"  # irl | sl | gevp
    m: int = 20
    tol: float = 1e-12
    max_restarts: int = 300
    sl_budget: int = 100
    seed: int = 111
    max_outer_steps: int = 50
    convergence_eps: float = 1e-10
    line_search: tuple = DEFAULT_LINE_SEARCH_GRID
    n_samples: int = 0  # 0 = exact enumeration
    gevp_tol: float = 1e-12  # method "gevp": relative residual of A c = lambda B c
    gevp_max_iter: int = 2000
    # method "gevp": S -> S + eps I with eps = gevp_shift * mean(diag S) (the SR diagonal
    # shift): the BASELINE batches have an exactly singular S (fixed particle number
    # makes the visible columns, and x_i t_j against t_j, linearly dependent)
    gevp_shift: float = 1e-3
    gevp_precond: bool = False  # Jacobi (inverse diag S~) preconditioning of the LOBPCG residuals

    def __post_init__(self):
        if self.method not in ("irl", "sl", "gevp"):
            raise ValueError(f"unknown method {self.method!r}")


def _batch_seed(config: OptimizerConfig, step: int) -> int:
    """opt:100-101."""
    return (config.seed * 1_000_003 + step) % 2**31


class BorderedLayout:
    """Physical device layout of the bordered vector.

    real / complex_raw : logical [u0, u (P)]            -> [u0, 0, u, 0-pad]  length 2 + ld
    hermitian          : logical [u0, Re c (P), Im c (P)] -> [u0, 0, Re c, pad, Im c, pad]  length 2 + 2 ld
    The zero slot after u0 keeps the P-part 16-byte aligned for the kernels.
    """

    def __init__(self, batch: SampleBatch):
        self.p = batch.param_count
        self.ld = batch.ld
        self.hermitian = batch.kind == KIND_HERMITIAN
        self.device = batch.device
        self.dim = 1 + (2 * self.p if self.hermitian else self.p)
        self.length = 2 + (2 * self.ld if self.hermitian else self.ld)
        idx = [0] + list(range(2, 2 + self.p))
        if self.hermitian:
            idx += list(range(2 + self.ld, 2 + self.ld + self.p))
        self.index = torch.as_tensor(np.array(idx, dtype=np.int64), device=self.device)

    def scatter(self, x: np.ndarray) -> torch.Tensor:
        out = torch.zeros(self.length, dtype=torch.float64, device=self.device)
        out[self.index] = torch.as_tensor(np.asarray(x, dtype=np.float64), device=self.device)
        return out

    def gather(self, v: torch.Tensor) -> torch.Tensor:
        return v[self.index]

    def parts(self, v: torch.Tensor):
        """(u0 view (1,), u-part views) for the kernel ABI."""
        u0 = v[0:1]
        if self.hermitian:
            return u0, (v[2 : 2 + self.ld], v[2 + self.ld : 2 + 2 * self.ld])
        return u0, v[2 : 2 + self.ld]


class BorderedOperator:
    """opt:140-148 on the device: one fused streaming launch per product."""

    def __init__(self, batch: SampleBatch, energy: EnergyEstimate, gradient: torch.Tensor | None = None,
                 mode: int = _lib.MVP_AUTO, use_graph: bool = True, connected: ConnectedCache | None = None):
        self.batch = batch
        self.connected = connected
        self.energy = energy
        self.layout = BorderedLayout(batch)
        self.mode = mode
        self.coeff = batch.coefficients(energy.mean)
        if gradient is None:
            gradient = energy_gradient(batch, energy)
        self.gradient = gradient
        ld, p = batch.ld, batch.param_count
        if self.layout.hermitian:
            half = torch.zeros((2, ld), dtype=torch.float64, device=batch.device)
            half[0, :p] = 0.5 * gradient.real
            half[1, :p] = 0.5 * gradient.imag
            self.half_f = (half[0], half[1])
            self._half = half
        else:
            half = torch.zeros(ld, dtype=torch.float64, device=batch.device)
            half[:p] = 0.5 * gradient
            self.half_f = half
        self.count = 0
        self.use_graph = use_graph
        self._sweepers: dict = {}

    supports_out = True

    def sweeper(self, length: int, m: int):
        """Persistent graph-captured Lanczos sweeper bound to this operator."""
        key = (length, m)
        sw = self._sweepers.get(key)
        if sw is None:
            sw = krylov._GraphSweeper(lambda v, w: self(v, out=w), length, m, self.batch.device,
                                      use_graph=self.use_graph)
            self._sweepers[key] = sw
        return sw

    shift = 0.0  # absolute diagonal shift of S in the metric (set by solve_step's GEVP form)

    def metric(self, u: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """The bordered metric S~ [u0; u] = [u0; (S + shift) u] of the GEVP form:
        the normalised state is orthogonal to the centred derivatives, so S~ = diag(1, S)."""
        if out is None:
            out = torch.zeros(self.layout.length, dtype=torch.float64, device=u.device)
        u0, uin = self.layout.parts(u)
        out0, uout = self.layout.parts(out)
        _apply(self.batch, _qgt_coeff(self.batch), uin, uout, mode=self.mode)
        if self.shift:
            if self.layout.hermitian:
                uout[0].add_(uin[0], alpha=self.shift)
                uout[1].add_(uin[1], alpha=self.shift)
            else:
                uout.add_(uin, alpha=self.shift)
        out0.copy_(u0)
        self.count += 1
        return out

    def both(self, u: torch.Tensor):
        """(H~ u, S~ u) of the GEVP form in one launch sequence: where the rows
        take the fused single-pass path, O is read once for both products
        (``irl_mvp2_*``); counts as two products."""
        if self.connected is not None or self.mode != _lib.MVP_AUTO:
            return self(u), self.metric(u)
        lay = self.layout
        ha = torch.zeros(lay.length, dtype=torch.float64, device=u.device)
        sb = torch.zeros(lay.length, dtype=torch.float64, device=u.device)
        u0, uin = lay.parts(u)
        a0, aout = lay.parts(ha)
        b0, bout = lay.parts(sb)
        _apply2(self.batch, self.coeff, _qgt_coeff(self.batch), uin, aout, bout, half_f=self.half_f, u0=u0, out0=a0)
        if self.shift:
            if lay.hermitian:
                bout[0].add_(uin[0], alpha=self.shift)
                bout[1].add_(uin[1], alpha=self.shift)
            else:
                bout.add_(uin, alpha=self.shift)
        b0.copy_(u0)
        self.count += 2
        return ha, sb

    def metric_diagonal(self) -> torch.Tensor | None:
        """diag(S~) = [1, S_ii] in the physical layout: S_ii = sum_n w_n |O_ni - Obar_i|^2
        (est:335-344's diagonal), from the stored O in row chunks; None for an
        on-the-fly batch (no stored rows to square)."""
        b = self.batch
        if b.otf is not None:
            return None
        lay = self.layout
        obar = b.obar()
        diag = torch.zeros(b.ld, dtype=torch.float64, device=b.device)
        w = b.weights
        step = max(1, (256 << 20) // (b.ld * b.o_padded.element_size()))
        for r0 in range(0, b.n_rows, step):
            oc = b.o_padded[r0 : r0 + step] - obar
            diag += (w[r0 : r0 + step, None] * (oc.real ** 2 + oc.imag ** 2 if oc.is_complex() else oc * oc)).sum(0)
        out = torch.ones(lay.length, dtype=torch.float64, device=b.device)
        _, parts = lay.parts(out)
        if lay.hermitian:
            parts[0].copy_(diag)
            parts[1].copy_(diag)
        else:
            parts.copy_(diag)
        return out

    def __call__(self, u: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.zeros(self.layout.length, dtype=torch.float64, device=u.device)
        u0, uin = self.layout.parts(u)
        out0, uout = self.layout.parts(out)
        _apply(self.batch, self.coeff, uin, uout, mode=self.mode, half_f=self.half_f, u0=u0, out0=out0,
               cache=self.connected)
        self.count += 1
        return out


@dataclass(frozen=True)
class StepResult:
    direction: torch.Tensor  # (P,) device; complex for hermitian batches
    lambda_min: float
    n_matvec: int
    converged: bool
    pair: krylov.RitzPair
    energy: EnergyEstimate


def direction_from_vector(vec: torch.Tensor, gradient: torch.Tensor, p: int, hermitian: bool) -> torch.Tensor:
    """opt:160-165: d = c[1:] / c0, or the descent-oriented c[1:] when c0 ~ 0."""
    c0 = float(vec[0])
    if hermitian:
        d = torch.complex(vec[1 : 1 + p], vec[1 + p : 1 + 2 * p])
        slope = float((gradient.real * d.real + gradient.imag * d.imag).sum())
    else:
        d = vec[1:]
        slope = None
    if abs(c0) > 1e-12:
        return d / c0
    if slope is None:
        slope = float(gradient @ d)
    return -d if slope > 0 else d


def solve_step(batch: SampleBatch, config: OptimizerConfig = OptimizerConfig(), step: int = 0, *,
               energy: EnergyEstimate | None = None, mode: int = _lib.MVP_AUTO, seed: int | None = None,
               use_graph: bool = True, connected: ConnectedCache | None = None) -> StepResult:
    """The IRL-SR hot path of one outer step (opt:134-165) on a device batch.

    ``connected`` adds ``heff_offdiag_matvec`` to the operator as ``opt:146`` does.
    """
    if energy is None:
        energy = estimate_energy(batch)
    # the operator (and its captured Lanczos graphs) is cached on the batch
    ops = batch.__dict__.setdefault("_bordered_ops", {})
    key = (float(energy.mean), int(mode), use_graph, id(connected) if connected is not None else None)
    op = ops.get(key)
    if op is None:
        op = BorderedOperator(batch, energy, energy_gradient(batch, energy), mode=mode, use_graph=use_graph,
                              connected=connected)
        ops[key] = op
    gradient = op.gradient
    s = _batch_seed(config, step) if seed is None else seed
    lay = op.layout
    if config.method == "irl":
        pair = krylov.irl_smallest(op, lay.dim, m=config.m, tol=config.tol, max_restarts=config.max_restarts,
                                   seed=s, device=batch.device, layout=lay)
    elif config.method == "gevp":
        if connected is not None:
            raise ValueError("the GEVP form takes the batch operator without the connected completion")
        d = op.__dict__.get("_metric_diag")
        if d is None:
            d = op.metric_diagonal()
            op._metric_diag = d
        if d is not None:
            p_idx = lay.index[1:]  # the logical P-part (padding slots excluded)
            op.shift = float(config.gevp_shift) * float(d[p_idx].mean())
            dd = d.clone()
            dd[p_idx] += op.shift
            # Jacobi preconditioner: the inverse diagonal of S~ (padding slots stay 0); without
            # it, a 0/1 mask keeps the search space out of S~'s exact null coordinates
            inv = torch.where(dd > 0, 1.0 / dd.clamp_min(1e-300), torch.zeros_like(dd))
            if not config.gevp_precond:
                inv = (inv > 0).to(inv.dtype)
            precond = lambda r: r * inv  # noqa: E731
        else:  # on-the-fly batch: no stored rows for diag(S); relative shift against tr(S)/P from the products
            op.shift = 0.0
            precond = None
        pair = krylov.lobpcg_smallest(op, op.metric, lay.dim, tol=config.gevp_tol, max_iter=config.gevp_max_iter,
                                      seed=s, device=batch.device, layout=lay, precond=precond, apply_ab=op.both)
    else:
        pair = krylov.sl_smallest(op, lay.dim, budget=config.sl_budget, seed=s, device=batch.device, layout=lay)
    d = direction_from_vector(pair.vector, gradient, batch.param_count, lay.hermitian)
    return StepResult(direction=d, lambda_min=float(pair.value), n_matvec=pair.n_matvec,
                      converged=pair.converged, pair=pair, energy=energy)


def energy_at(params, integrals, sector, config: OptimizerConfig = OptimizerConfig(), step: int = 0) -> float:
    """opt:104-115: the batch energy at ``params``.

    Only log psi (weights) and the local energies are needed -- no O rows.
    The reference's own autoregressive ansatz also runs stochastic batches
    (exact samples, seed ``_batch_seed(config, step)``); the RBM / MLP run in
    exact-enumeration mode.
    """
    from . import ansatz as A, autoregressive as AR, hamiltonian as H

    dev = torch.device("cuda", torch.cuda.current_device())
    if AR.is_autoregressive(params):
        if config.n_samples == 0:
            bits = H.enumerate_sector(sector)
        else:
            bits = AR.sample(params, sector, config.n_samples, _batch_seed(config, step), device=dev)
        e = AR.local_energies(params, integrals, sector, bits, device=dev)
        if config.n_samples == 0:
            lp = AR.log_amplitude_batch(params, sector, bits, device=dev)
            w = torch.exp(2.0 * lp.real)
        else:
            w = torch.ones(len(bits), dtype=torch.float64, device=dev)
        w = w / w.sum()
        return float((w.to(e.dtype) * e).sum().real)
    if config.n_samples != 0:
        raise NotImplementedError("stochastic RBM/MLP energies need a sampler (exact mode only)")
    bits = H.enumerate_sector(sector)
    xb = torch.as_tensor(bits.view(np.int64), device=dev)
    e = H.local_energies(params, integrals, xb, device=dev)
    lp = A.log_amplitude_batch(params, H.bits_to_occupations(bits, params.architecture.n_inputs), device=dev)
    lr = lp.real if torch.is_complex(lp) else lp
    w = torch.exp(2.0 * (lr - lr.max()))
    w = w / w.sum()
    val = (w.to(e.dtype) * e).sum()
    return float(val.real if torch.is_complex(val) else val)


class _OuterStepFields(NamedTuple):
    params: object
    lambda_min: float
    step_scale: float
    matvecs: int
    converged: bool


class OuterStep(_OuterStepFields):
    """The reference's 5-tuple ``(new params, lambda_min, step scale, matvec
    count, converged)`` (``opt:118-124``), so callers unpack it exactly as
    ``run_optimization`` does (``opt:257``); the named fields read the same
    values.  Two extra attributes (not tuple members): ``energy``, the batch
    energy the step was solved on, and ``best_energy``, the line-search energy
    at the accepted scale (= ``energy`` when no scale was accepted)."""

    def __new__(cls, params, lambda_min, step_scale, matvecs, converged, *, energy=float("nan"),
                best_energy=float("nan")):
        self = super().__new__(cls, params, lambda_min, step_scale, matvecs, converged)
        object.__setattr__(self, "energy", float(energy))
        object.__setattr__(self, "best_energy", float(best_energy))
        return self

    def __setattr__(self, name, value):
        raise AttributeError("OuterStep is immutable")


def outer_step(params, integrals, sector, config: OptimizerConfig = OptimizerConfig(), step: int = 0, *,
               mode: int = _lib.MVP_AUTO, use_graph: bool | None = None) -> OuterStep:
    """opt:118-195 on the device: the reference's own autoregressive ansatz
    (exact or stochastic batches) or the shallow RBM / MLP (exact mode).

    Batch (E_loc, |psi|^2 weights, O rows), energy, gradient, connected cache,
    the bordered IRL / SL solve with ``heff_matvec + heff_offdiag_matvec``,
    the direction ``c[1:]/c0``, then the line search over ``config.line_search``
    by exact energy re-evaluation, falling back to the normalised steepest
    descent ``-F/|F|`` when no scale lowers the energy (opt:167-190).
    """
    from . import ansatz as A, autoregressive as AR, hamiltonian as H

    if AR.is_autoregressive(params):
        # the reference's own model: exact or stochastic batches (opt:134-137)
        batch = AR.build_batch(params, integrals, sector, n_samples=config.n_samples,
                               seed=_batch_seed(config, step))
        energy = estimate_energy(batch)  # warns on an imaginary residual, as est:136-143
        cache = AR.build_connected_cache(params, integrals, sector, batch)
        make = lambda th: AR.AnsatzParameters(params.architecture, th)  # noqa: E731
    else:
        if config.n_samples != 0:
            raise NotImplementedError("stochastic RBM/MLP batches need a sampler (exact mode only)")
        batch = H.build_batch(params, integrals, sector)
        energy = estimate_energy(batch)
        cache = H.build_connected_cache(params, integrals, sector, batch)
        make = lambda th: A.AnsatzParameters(params.architecture, th)  # noqa: E731
    if use_graph is None:
        # every outer step builds a new batch: capturing a sweep that runs once
        # costs more than it saves (syn6 70-160 -> 11-17 ms, syn10 280 -> 153 ms
        # eager); capturing recurring restart orders only ("lazy") did not help
        # the long stochastic restart sequences either (670-930 vs 730 ms)
        use_graph = {"1": True, "lazy": "lazy"}.get(os.environ.get("IRL_OUTER_GRAPH", ""), False)
    res = solve_step(batch, config, step, energy=energy, mode=mode, connected=cache, use_graph=use_graph)
    grad = energy_gradient(batch, energy).detach().cpu().numpy()
    d0 = res.direction.detach().cpu().numpy()
    theta = np.asarray(params.theta)

    def line_search(d, best):
        best_scale, best_energy = best
        best_d = d
        for scale in config.line_search:
            cand = make(theta + scale * d)
            e_new = energy_at(cand, integrals, sector, config, step)
            if np.isfinite(e_new) and e_new < best_energy:
                best_energy, best_scale, best_d = e_new, scale, d
        return best_scale, best_energy, best_d

    best_scale, best_energy, best_d = line_search(d0, (0.0, energy.mean))
    if best_scale == 0.0:
        norm = float(np.linalg.norm(grad))
        if norm > 0.0:
            best_scale, best_energy, best_d = line_search(-grad / norm, (0.0, energy.mean))
    new = params
    if best_scale > 0.0:
        new = make(theta + best_scale * best_d)
    return OuterStep(new, res.lambda_min, best_scale, res.n_matvec, res.converged, energy=energy.mean,
                     best_energy=best_energy)
