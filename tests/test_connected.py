"""Two-configuration completion: ``build_connected_cache`` /
``heff_offdiag_matvec`` (est:189-294) and the optimizer's full operator
(opt:140-148 with :146).

CPU tests pin the oracle restatement to the reference's own outputs
(tests/golden/{h2,rbm,hermitian}_connected.npz, made by oracle/make_golden.py
from /root/reference); GPU tests pin the sm_100a path (through the C-ABI) to
the same fixtures and to the oracle.  Tolerances as in test_gpu_parity.py.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import estimators as oest
from oracle import nqs

PROD_TOL = 1e-10
RITZ_TOL = 1e-10
DIR_TOL = 1e-8


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def host(t):
    return t.detach().cpu().numpy()


def h2_case(tag):
    g = golden("h2_connected")
    return {k[len(tag) + 1:]: v for k, v in g.items() if k.startswith(tag + "_")}, g


def cache_args(d):
    return d["dist_index"], d["indptr"], d["partner_row"], d["coeff"], d["partner_o"]


# ------------------------------------------------------------------- CPU --
@pytest.mark.parametrize("tag", ["exact", "stoch"])
def test_oracle_offdiag_matches_reference_h2(tag):
    d, _ = h2_case(tag)
    for v, off in zip(d["vs"], d["off"]):
        assert rel(oest.heff_offdiag(d["w"], d["o"], *cache_args(d), v), off) < 1e-13


def test_h2_fixture_is_pinned_by_the_sandwich_oracle():
    """T/test_estimators.py:170-181: heff + offdiag == <dpsi|(H - E)|dpsi> on exact weights."""
    d, _ = h2_case("exact")
    for v, full in zip(d["vs"], d["full"]):
        ref = d["sandwich"] @ v
        assert np.max(np.abs(full - ref)) < 1e-10 * max(1.0, np.max(np.abs(ref)))


def test_h2_stochastic_fixture_has_duplicates():
    d, _ = h2_case("stoch")
    assert len(np.unique(d["dist_index"])) < len(d["dist_index"])  # est:105-126 dedup exercised


def test_oracle_offdiag_matches_reference_rbm():
    g = golden("rbm_connected")
    assert rel(nqs.rbm_log_psi(g["theta"], g["x"], int(g["n"]), int(g["h"])), g["logpsi_x"]) < 1e-15
    for v, off in zip(g["vs"], g["off"]):
        assert rel(oest.heff_offdiag(g["w"], g["o"], *cache_args(g), v), off) < 1e-13


def test_oracle_offdiag_matches_reference_embedding():
    g = golden("hermitian_connected")
    P = g["o"].shape[1]
    for v, off in zip(g["vs"], g["off"]):
        z = oest.heff_offdiag_hermitian(g["w"], g["o"], *cache_args(g), v[:P] + 1j * v[P:])
        assert rel(np.concatenate([z.real, z.imag]), off) < 1e-13


def test_oracle_offdiag_linearity():
    """T/test_estimators.py:183-193."""
    d, _ = h2_case("exact")
    rng = np.random.default_rng(99)
    v1, v2 = rng.standard_normal((2, d["o"].shape[1]))
    f = lambda v: oest.heff_offdiag(d["w"], d["o"], *cache_args(d), v)  # noqa: E731
    assert np.max(np.abs(f(v1 + 0.5 * v2) - f(v1) - 0.5 * f(v2))) < 1e-12


def test_synthetic_partners_conserve_particles():
    from paper_2601_01437_b200 import synthetic

    inp = synthetic.make_inputs(synthetic.CONFIGS[2].with_rows(64))
    partners, elements, indptr, dist = synthetic.connected_partners(inp.x, 4, seed=5)
    assert partners.shape == (256, inp.x.shape[1]) and elements.shape == (256,)
    assert np.all(partners.sum(axis=1) == inp.config.n_ones)
    diff = np.abs(partners.astype(int) - np.repeat(inp.x, 4, axis=0).astype(int)).sum(axis=1)
    assert np.all(diff == 2)  # exactly one hole and one particle
    assert indptr[-1] == 256 and np.array_equal(dist, np.arange(64))


# ------------------------------------------------------------------- GPU --
@pytest.fixture(scope="module")
def pkg(cuda):
    from paper_2601_01437_b200 import _lib

    _lib.lib()
    import paper_2601_01437_b200 as p

    return p


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["exact", "stoch"])
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_h2_connected_golden(pkg, tag, mode):
    from paper_2601_01437_b200 import estimators as E

    d, _ = h2_case(tag)
    b = E.SampleBatch(None, d["w"], d["e"], d["o"], int(d["n_samples"]))
    with pytest.warns(UserWarning) if tag == "stoch" else _null():
        en = E.estimate_energy(b)
    cache = E.ConnectedCache(*cache_args(d), batch=b)
    for v, off, full in zip(d["vs"], d["off"], d["full"]):
        assert rel(E.heff_offdiag_matvec(b, cache, v, mode=mode), off) < PROD_TOL
        assert rel(E.connected_heff_matvec(b, en, cache, v, mode=mode), full) < PROD_TOL


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["exact", "stoch"])
def test_h2_connected_irl_golden(pkg, tag):
    """The reference optimizer's full operator (opt:140-148 incl. :146): same
    matvec count, Ritz value within 1e-10, direction within 1e-8."""
    import warnings

    from paper_2601_01437_b200 import estimators as E, optimizer as OPT

    d, g = h2_case(tag)
    b = E.SampleBatch(None, d["w"], d["e"], d["o"], int(d["n_samples"]))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        en = E.estimate_energy(b)
    cache = E.ConnectedCache(*cache_args(d), batch=b)
    res = OPT.solve_step(b, OPT.OptimizerConfig(m=int(g["m"]), max_restarts=3), energy=en, seed=int(g["seed"]),
                         connected=cache)
    assert res.n_matvec == int(d["n_matvec"])
    assert abs(res.lambda_min - float(d["lam"])) <= RITZ_TOL * abs(float(d["lam"]))
    assert rel(host(res.direction), d["direction"]) < DIR_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_rbm_connected_cache_build_and_products(pkg, mode):
    from paper_2601_01437_b200 import ansatz as A, estimators as E

    g = golden("rbm_connected")
    n, h = int(g["n"]), int(g["h"])
    arch = A.RBMArchitecture(n, h)
    params = A.AnsatzParameters(arch, g["theta"])
    N = len(g["w"])
    b = A.build_batch(params, g["x"], np.zeros(N), weights=g["w"], n_samples=N)
    lp = host(A.log_amplitude_batch(params, g["x"]))
    assert rel(lp, g["logpsi_x"]) < 1e-14
    cache = A.build_connected_cache(params, b, g["x"], g["partners"], g["elements"], g["indptr"],
                                    dist_index=g["dist_index"])
    assert np.array_equal(host(cache.partner_row), g["partner_row"])
    assert rel(host(cache.coeff), g["coeff"].real) < 1e-14
    assert np.max(np.abs(host(cache.partner_o[:, : arch.param_count]) - g["partner_o"])) < 1e-14
    for v, off in zip(g["vs"], g["off"]):
        assert rel(E.heff_offdiag_matvec(b, cache, v, mode=mode), off) < PROD_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_hermitian_connected_golden(pkg, mode):
    from paper_2601_01437_b200 import ansatz as A, estimators as E

    g = golden("hermitian_connected")
    n, h = int(g["n"]), int(g["h"])
    arch = A.RBMArchitecture(n, h, complex_params=True)
    params = A.AnsatzParameters(arch, g["theta"])
    N = len(g["w"])
    b = A.build_batch(params, g["x"], np.zeros(N, dtype=complex), weights=g["w"], n_samples=N)
    lp = host(A.log_amplitude_batch(params, g["partners"]))
    assert rel(lp, g["logpsi_p"]) < 1e-13
    cache = A.build_connected_cache(params, b, g["x"], g["partners"], g["elements"], g["indptr"],
                                    dist_index=g["dist_index"])
    assert rel(host(cache.coeff), g["coeff"]) < 1e-13
    P = arch.param_count
    for v, off in zip(g["vs"], g["off"]):
        z = E.heff_offdiag_matvec(b, cache, v[:P] + 1j * v[P:], mode=mode)
        assert rel(np.concatenate([z.real, z.imag]), off) < PROD_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("build", ["stored", "otf"])
@pytest.mark.parametrize("idx,rows", [(1, 8192), (2, 2048), (3, 512), (4, 128)])
def test_config_connected_vs_oracle(pkg, idx, rows, build):
    """BASELINE shapes (row subsets) with seeded synthetic partners: the device
    completion and the full connected product against the oracle."""
    from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic

    inp = synthetic.make_inputs(synthetic.CONFIGS[idx].with_rows(rows))
    c = inp.config
    arch = (A.RBMArchitecture(c.n_inputs, c.hidden, c.complex_params) if c.model == "rbm"
            else A.MLPArchitecture(c.n_inputs, c.hidden))
    params = A.AnsatzParameters(arch, inp.theta)
    b = A.build_batch(params, inp.x, inp.e_loc, mode=build)  # otf: O regenerated, partner rows stored
    partners, elements, indptr, dist = synthetic.connected_partners(inp.x, 4, seed=100 + idx)
    cache = A.build_connected_cache(params, b, inp.x, partners, elements, indptr, dist_index=dist)
    # oracle: rows and coefficients from the numpy restatement
    rows_fn = nqs.rbm_rows if c.model == "rbm" else nqs.mlp_rows
    lp_fn = nqs.rbm_log_psi if c.model == "rbm" else nqs.mlp_log_psi
    o = rows_fn(inp.theta, inp.x, c.n_inputs, c.hidden)
    uniq, inv = np.unique(partners, axis=0, return_inverse=True)
    po = rows_fn(inp.theta, uniq, c.n_inputs, c.hidden)
    seg = np.repeat(np.arange(len(indptr) - 1), np.diff(indptr))
    coeff = elements * np.exp(lp_fn(inp.theta, partners, c.n_inputs, c.hidden)
                              - lp_fn(inp.theta, inp.x, c.n_inputs, c.hidden)[seg])
    w = np.full(rows, 1.0 / rows)
    rng = np.random.default_rng(7)
    en = E.estimate_energy(b)
    mean, _, _ = oest.energy(w, inp.e_loc, rows)
    for _ in range(2):
        if c.complex_params:
            v = rng.standard_normal(c.param_count) + 1j * rng.standard_normal(c.param_count)
            ref = oest.heff_offdiag_hermitian(w, o, dist, indptr, inv.reshape(-1), coeff, po, v)
            ref_full = ref + oest.heff_hermitian(w, inp.e_loc, o, mean, v)
        else:
            v = rng.standard_normal(c.param_count)
            ref = oest.heff_offdiag(w, o, dist, indptr, inv.reshape(-1), coeff.real, po, v)
            ref_full = ref + oest.heff(w, inp.e_loc, o, mean, v)
        assert rel(E.heff_offdiag_matvec(b, cache, v), ref) < PROD_TOL
        assert rel(E.connected_heff_matvec(b, en, cache, v), ref_full) < PROD_TOL


@pytest.mark.gpu
def test_log_amplitude_mlp_vs_oracle(pkg):
    from paper_2601_01437_b200 import ansatz as A, synthetic

    inp = synthetic.make_inputs(synthetic.CONFIGS[5].with_rows(300))
    c = inp.config
    params = A.AnsatzParameters(A.MLPArchitecture(c.n_inputs, c.hidden), inp.theta)
    lp = host(A.log_amplitude_batch(params, inp.x))
    assert rel(lp, nqs.mlp_log_psi(inp.theta, inp.x, c.n_inputs, c.hidden)) < 1e-13


@pytest.mark.gpu
def test_connected_validation_and_empty_partners(pkg):
    from paper_2601_01437_b200 import estimators as E

    d, _ = h2_case("exact")
    b = E.SampleBatch(None, d["w"], d["e"], d["o"], 0)
    n = len(d["w"])
    P = d["o"].shape[1]
    # no partners at all: the completion is zero, the full product equals heff_matvec
    empty = E.ConnectedCache(np.arange(n), np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int64),
                             np.zeros(0, dtype=complex), np.zeros((0, P), dtype=complex), batch=b)
    v = np.random.default_rng(3).standard_normal(P)
    assert np.max(np.abs(E.heff_offdiag_matvec(b, empty, v))) == 0.0
    en = E.estimate_energy(b)
    assert rel(E.connected_heff_matvec(b, en, empty, v), E.heff_matvec(b, en, v)) < 1e-14
    with pytest.raises(IndexError):
        E.ConnectedCache(np.full(n, n + 5), np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int64),
                         np.zeros(0), np.zeros((0, P), dtype=complex), batch=b)
    with pytest.raises(ValueError):
        E.ConnectedCache(*cache_args(d)[:-1], d["partner_o"][:, :-1], batch=b)
    cache = E.ConnectedCache(*cache_args(d), batch=b)
    with pytest.raises(ValueError):
        E.heff_offdiag_matvec(b, cache, np.zeros(P + 1))
    with pytest.raises(ValueError):
        E.heff_offdiag_matvec(b, cache, np.full(P, np.nan))
    other = E.SampleBatch(None, d["w"], d["e"], d["o"], 0)
    with pytest.raises(ValueError):
        E.heff_offdiag_matvec(other, cache, v)
