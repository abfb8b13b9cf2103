"""Seeded synthetic workloads of BASELINE.json.

No public dataset stands behind these configurations: BASELINE.json fully
specifies them, and every config draws its inputs from
``np.random.SeedSequence(111 + i)`` (i = config number 1..5; 111 is the
paper's seed, ``PAPER.md:56`` / ``opt:53``), spawned into three independent
streams in the fixed order bitstrings, theta blocks, E_loc.  Independent
streams make a row subset (the first ``n_rows`` rows) identical across
sizes, which the parity tests rely on.  The Lanczos start vector is drawn by
``irl_smallest`` from ``default_rng(lanczos_seed)`` with
``lanczos_seed = 111 + i``.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class SyntheticConfig:
    index: int
    model: str  # "rbm" | "mlp"
    n_inputs: int
    hidden: int
    n_rows: int
    n_ones: int
    complex_params: bool
    theta_std: tuple  # rbm: (sigma,) ; mlp: (std_W_b, std_u_c)
    e_mean: float
    e_std: float
    e_imag_std: float
    m: int
    max_restarts: int = 3

    @property
    def param_count(self) -> int:
        n, h = self.n_inputs, self.hidden
        return n + h + h * n if self.model == "rbm" else h * n + 2 * h + 1

    @property
    def lanczos_seed(self) -> int:
        return 111 + self.index

    @property
    def name(self) -> str:
        kind = "c128" if self.complex_params else "f64"
        return f"cfg{self.index}-{self.model}-{kind}-{self.n_rows}x{self.param_count}"

    def with_rows(self, n_rows: int) -> "SyntheticConfig":
        return replace(self, n_rows=int(n_rows))


CONFIGS = {
    1: SyntheticConfig(1, "rbm", 20, 40, 8192, 10, False, (0.01,), -75.0, 0.01, 0.0, 20),
    2: SyntheticConfig(2, "rbm", 40, 160, 65536, 20, False, (0.01,), -150.0, 0.02, 0.0, 30),
    3: SyntheticConfig(3, "mlp", 20, 512, 131072, 18, False, (np.sqrt(1 / 20), np.sqrt(1 / 512)), -195.6, 0.05,
                       0.0, 30),
    4: SyntheticConfig(4, "rbm", 60, 480, 131072, 30, True, (0.005,), -230.0, 0.05, 0.01, 30),
    5: SyntheticConfig(5, "mlp", 100, 2048, 65536, 50, False, (np.sqrt(1 / 100), np.sqrt(1 / 2048)), -400.0, 0.1,
                       0.0, 40),
}


@dataclass(frozen=True)
class SyntheticInputs:
    config: SyntheticConfig
    x: np.ndarray  # (N, n) uint8 0/1, exactly n_ones ones per row
    theta: np.ndarray  # (P,) float64 or complex128
    e_loc: np.ndarray  # (N,) float64 or complex128


def make_inputs(cfg: SyntheticConfig) -> SyntheticInputs:
    rng_x, rng_t, rng_e = (np.random.default_rng(s) for s in np.random.SeedSequence(111 + cfg.index).spawn(3))
    n, h, N = cfg.n_inputs, cfg.hidden, cfg.n_rows
    occ = np.argsort(rng_x.random((N, n)), axis=1)[:, : cfg.n_ones]
    x = np.zeros((N, n), dtype=np.uint8)
    x[np.arange(N)[:, None], occ] = 1
    if cfg.model == "rbm":
        (s,) = cfg.theta_std
        if cfg.complex_params:
            theta = rng_t.normal(0.0, s, cfg.param_count) + 1j * rng_t.normal(0.0, s, cfg.param_count)
        else:
            theta = np.concatenate([rng_t.normal(0.0, s, n), rng_t.normal(0.0, s, h), rng_t.normal(0.0, s, h * n)])
    else:
        s_in, s_out = cfg.theta_std
        theta = np.concatenate([
            rng_t.normal(0.0, s_in, h * n),  # W (h x n_in)
            rng_t.normal(0.0, s_in, h),      # b
            rng_t.normal(0.0, s_out, h),     # u
            rng_t.normal(0.0, s_out, 1),     # c
        ])
    e = rng_e.normal(cfg.e_mean, cfg.e_std, N)
    if cfg.complex_params:
        e = e + 1j * rng_e.normal(0.0, cfg.e_imag_std, N)
    return SyntheticInputs(cfg, x, theta, e)


def connected_partners(x: np.ndarray, per_row: int, seed: int, element_std: float = 0.05):
    """Seeded synthetic stand-in for ``connected_configurations`` (ham:238-287).

    For every row of ``x`` (treated as distinct: dist_index = arange(N)), draw
    ``per_row`` spin-conserving-free single excitations (one occupied orbital
    emptied, one empty orbital filled: the partner keeps the particle number,
    like the reference's singles) with off-diagonal elements N(0, element_std^2).
    No Hamiltonian stands behind them; they exercise the completion's data path
    at BASELINE shapes.  Returns (partners (N*per_row, n) uint8, elements,
    indptr (N+1,), dist_index (N,)).
    """
    rng = np.random.default_rng(seed)
    N, n = x.shape
    occ = np.argsort(-x.astype(np.int8) + rng.random((N, n)) * 0.5, axis=1)  # occupied first, shuffled
    k = int(x[0].sum())
    holes = occ[:, :k][np.arange(N)[:, None], rng.integers(0, k, (N, per_row))]
    parts = occ[:, k:][np.arange(N)[:, None], rng.integers(0, n - k, (N, per_row))]
    partners = np.repeat(x, per_row, axis=0).reshape(N, per_row, n).copy()
    ri = np.arange(N)[:, None]
    ci = np.arange(per_row)[None, :]
    partners[ri, ci, holes] = 0
    partners[ri, ci, parts] = 1
    elements = rng.normal(0.0, element_std, N * per_row)
    indptr = np.arange(0, N * per_row + 1, per_row, dtype=np.int64)
    return partners.reshape(N * per_row, n), elements, indptr, np.arange(N, dtype=np.int64)


def molecule_fcidump(seed, ns, n_elec, ms2=0, scale=0.3):
    """Seeded synthetic FCIDUMP text with 8-fold symmetric integrals (one line per
    unique quadruple; diagonal h around -1, core energy around 0.5).  No molecule
    stands behind it: it feeds the local-energy path at chosen sizes."""
    rng = np.random.default_rng(seed)
    lines = [f"&FCI NORB={ns},NELEC={n_elec},MS2={ms2},", " ORBSYM=" + ",".join(["1"] * ns) + ",", " ISYM=1,", "&END"]
    seen = set()
    for i in range(1, ns + 1):
        for j in range(1, i + 1):
            for k in range(1, ns + 1):
                for l in range(1, k + 1):
                    key = tuple(sorted([(i, j), (k, l)]))
                    if key in seen:
                        continue
                    seen.add(key)
                    lines.append(f"{rng.normal(0.0, scale):.16e} {i} {j} {k} {l}")
    for i in range(1, ns + 1):
        for j in range(1, i + 1):
            lines.append(f"{rng.normal(-1.0 if i == j else 0.0, scale):.16e} {i} {j} 0 0")
    lines.append(f"{rng.normal(0.5, 0.1):.16e} 0 0 0 0")
    return "\n".join(lines) + "\n"
