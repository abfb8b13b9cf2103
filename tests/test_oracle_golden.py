"""Pin the CPU oracle (oracle/) against vectors recorded from the real reference.

Fixtures: tests/golden/*.npz, written by oracle/make_golden.py (which imports
/root/reference/pkg/src/irlnqs).  Tolerances follow the reference's own tests
(T/test_estimators.py:126-154, T/test_krylov.py:129-139).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import bordered, estimators as est, krylov, nqs


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def test_real_batch_statistics_and_products():
    g = golden("real_rbm")
    mean, var, std = est.energy(g["w"], g["e"], len(g["w"]))
    assert mean == pytest.approx(float(g["mean"]), abs=1e-13)
    assert var == pytest.approx(float(g["variance"]), rel=1e-12)
    assert std == pytest.approx(float(g["std_error"]), rel=1e-12)
    assert rel(est.gradient(g["w"], g["e"], g["o"], mean), g["grad"]) < 1e-12
    for v, hv, sv in zip(g["vs"], g["hv"], g["sv"]):
        assert rel(est.heff(g["w"], g["e"], g["o"], mean, v), hv) < 1e-13
        assert rel(est.qgt(g["w"], g["o"], v), sv) < 1e-13
    assert np.max(np.abs(est.dense_heff(g["w"], g["e"], g["o"], mean) - g["dense_heff"])) < 1e-13
    assert np.max(np.abs(est.dense_qgt(g["w"], g["o"]) - g["dense_qgt"])) < 1e-13


def test_real_rbm_rows_match_golden_o():
    g = golden("real_rbm")
    o = nqs.rbm_rows(g["theta"], g["x"], int(g["n"]), int(g["h"]))
    assert np.max(np.abs(o - g["o"])) < 1e-15


def test_real_bordered_irl_matches_reference():
    g = golden("real_rbm")
    mv, dim, grad, _ = bordered.real_problem(g["w"], g["e"], g["o"], len(g["w"]))
    pair, d = bordered.solve(mv, dim, grad, int(g["m"]), seed=int(g["seed"]))
    assert pair["n_matvec"] == int(g["n_matvec"])
    assert abs(pair["value"] - float(g["lam"])) <= 1e-10 * abs(float(g["lam"]))
    assert rel(d, g["direction"]) < 1e-8


def test_complex_raw_products():
    g = golden("complex_raw")
    mean, var, _ = est.energy(g["w"], g["e"], int(g["n_samples"]))
    assert mean == pytest.approx(float(g["mean"]), abs=1e-13)
    assert rel(est.gradient(g["w"], g["e"], g["o"], mean), g["grad"]) < 1e-12
    for v, hv in zip(g["vs"], g["hv"]):
        assert rel(est.heff(g["w"], g["e"], g["o"], mean, v), hv) < 1e-13
    mv, dim, grad, _ = bordered.real_problem(g["w"], g["e"], g["o"], int(g["n_samples"]))
    pair, d = bordered.solve(mv, dim, grad, int(g["m"]), seed=int(g["seed"]))
    assert pair["n_matvec"] == int(g["n_matvec"])
    assert abs(pair["value"] - float(g["lam"])) <= 1e-10 * abs(float(g["lam"]))
    assert rel(d, g["direction"]) < 1e-8


def test_hermitian_embedding():
    g = golden("hermitian_rbm")
    o = nqs.rbm_rows(g["theta"], g["x"], int(g["n"]), int(g["h"]))
    assert np.max(np.abs(o - g["o"])) < 1e-15
    P = o.shape[1]
    mean = float(g["mean"])
    for v, hv in zip(g["vs"], g["hv"]):
        c = v[:P] + 1j * v[P:]
        out = est.heff_hermitian(g["w"], g["e"], o, mean, c)
        assert rel(np.concatenate([out.real, out.imag]), hv) < 1e-12
    mv, dim, grad, _ = bordered.embedded_problem(g["w"], g["e"], o, len(g["w"]))
    assert rel(grad, g["grad"]) < 1e-12
    pair, d = bordered.solve(mv, dim, grad, int(g["m"]), seed=int(g["seed"]))
    assert pair["n_matvec"] == int(g["n_matvec"])
    assert abs(pair["value"] - float(g["lam"])) <= 1e-10 * abs(float(g["lam"]))
    assert rel(d, g["direction"]) < 1e-8


def test_h2_reference_data_path():
    g = golden("h2_exact")
    mean, _, _ = est.energy(g["w"], g["e"], 0)
    assert mean == pytest.approx(float(g["mean"]), abs=1e-14)
    assert rel(est.gradient(g["w"], g["e"], g["o"], mean), g["grad"]) < 1e-12
    for v, hv in zip(g["vs"], g["hv"]):
        assert rel(est.heff(g["w"], g["e"], g["o"], mean, v), hv) < 1e-13


def test_mlp_rows_equal_reference_phase_head():
    g = golden("mlp_phase_head")
    rows = nqs.mlp_rows(g["theta"], g["s"], int(g["n"]), int(g["h"]))
    assert np.max(np.abs(rows - g["rows"])) < 1e-15


@pytest.mark.parametrize("holo", [False, True])
def test_rbm_rows_match_finite_differences(holo):
    rng = np.random.default_rng(3)
    n, h = 5, 4
    x = (rng.random((6, n)) < 0.5).astype(np.uint8)
    p = n + h + h * n
    theta = rng.normal(0, 0.3, p) + (1j * rng.normal(0, 0.3, p) if holo else 0)
    fd = nqs.fd_rows(lambda t, xx: nqs.rbm_log_psi(t, xx, n, h), theta.astype(complex) if holo else theta, x,
                     holomorphic=holo)
    rows = nqs.rbm_rows(theta, x, n, h)
    assert np.max(np.abs(rows - fd)) / max(1.0, np.max(np.abs(rows))) < 1e-6


def test_mlp_rows_match_finite_differences():
    rng = np.random.default_rng(4)
    n, h = 6, 5
    x = (rng.random((5, n)) < 0.5).astype(np.uint8)
    theta = rng.normal(0, 0.5, h * n + 2 * h + 1)
    fd = nqs.fd_rows(lambda t, xx: nqs.mlp_log_psi(t, xx, n, h), theta, x)
    rows = nqs.mlp_rows(theta, x, n, h)
    assert np.max(np.abs(rows - fd)) / max(1.0, np.max(np.abs(rows))) < 1e-6


def test_krylov_restatement_matches_reference():
    g = golden("krylov")
    for i in range(int(g["count"])):
        mat = g[f"mat{i}"]
        pair = krylov.irl(lambda v: mat @ v, mat.shape[0], m=20, tol=1e-12, seed=i)
        norm = np.linalg.norm(mat, 2)
        # matvec counts are only reproducible away from the roundoff floor (tol = 1e-12 absolute)
        if int(g[f"n_restarts{i}"]) <= 6:
            assert pair["n_matvec"] == int(g[f"n_matvec{i}"])
        assert abs(pair["value"] - float(g[f"value{i}"])) < 1e-12 * norm
        assert pair["residual"] <= 1e-12 * max(1.0, norm)
        assert abs(abs(pair["vector"] @ g[f"vector{i}"]) - 1.0) < 1e-10


@pytest.mark.parametrize("idx,rows", [(1, 300), (2, 128), (3, 200), (4, 64), (5, 32)])
def test_structured_oracle_matches_rows(idx, rows):
    """oracle/structured.py (full-size CPU products from N x h / N x n factors)
    equals the row-based restatement of est:171-186 on a row subset."""
    from oracle import estimators as oest, nqs
    from oracle.structured import MLPProducts, RBMProducts
    from paper_2601_01437_b200 import synthetic as S

    cfg = S.CONFIGS[idx].with_rows(rows)
    inp = S.make_inputs(cfg)
    n, h = cfg.n_inputs, cfg.hidden
    w = np.full(rows, 1.0 / rows)
    mean = float(np.sum(w * inp.e_loc).real)
    rng = np.random.default_rng(idx)
    if cfg.model == "rbm":
        o = nqs.rbm_rows(inp.theta, inp.x, n, h)
        sp = RBMProducts(inp.theta, inp.x, n, h, w)
    else:
        o = nqs.mlp_rows(inp.theta, inp.x, n, h)
        sp = MLPProducts(inp.theta, inp.x, n, h, w)
    P = o.shape[1]
    assert sp.p == P
    assert np.linalg.norm(sp.obar - w @ o) <= 1e-13 * np.linalg.norm(w @ o)
    if cfg.complex_params:
        v = rng.standard_normal(P) + 1j * rng.standard_normal(P)
        ref = oest.heff_hermitian(w, inp.e_loc, o, mean, v)
        got = sp.product(w * (inp.e_loc - mean).real, v)
    else:
        v = rng.standard_normal(P)
        ref = oest.heff(w, inp.e_loc, o, mean, v)
        got = sp.product(w * (inp.e_loc - mean), v)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    ref_s = oest.qgt(w, o, v.real) if not cfg.complex_params else None
    if ref_s is not None:
        got_s = sp.product(w, v)
        assert np.linalg.norm(got_s - ref_s) <= 1e-12 * np.linalg.norm(ref_s)
