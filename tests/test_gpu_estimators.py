"""Device restatement of the reference's TestHeffMatvec / dense-operator cases
(T/test_estimators.py:126-154, :197-213) over every stored-O product path:
unit vectors pick out the dense columns, random vectors match the dense
operator, products are linear, dense H_eff is symmetric and the QGT is
positive semidefinite -- for H_eff v (est:171-186) and the matrix-free S v."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MODES = [1, 2, 3, 4]  # fused, two-pass, rows, wide (IRL_MVP_*)


@pytest.fixture(scope="module")
def E(cuda):
    from paper_2601_01437_b200 import estimators

    return estimators


@pytest.fixture(scope="module")
def setup(E):
    rng = np.random.default_rng(126)
    n, p = 1500, 37
    o = rng.normal(0.0, 0.6, (n, p)) + 0.2
    e = rng.normal(-2.0, 0.4, n)
    w = rng.random(n) + 0.1
    w /= w.sum()
    b = E.SampleBatch(None, w, e, o, 0)  # exact mode: arbitrary weights
    en = E.estimate_energy(b)
    return b, en, E.dense_heff(b, en), E.dense_qgt(b), p


@pytest.mark.parametrize("mode", MODES)
def test_unit_vectors_extract_dense_columns(E, setup, mode):
    """T/test_estimators.py:137-143: H e_i is column i of the dense H_eff (1e-12)."""
    b, en, dh, dq, p = setup
    scale_h, scale_q = np.max(np.abs(dh)), np.max(np.abs(dq))
    for i in (0, 1, p // 2, p - 1):
        ei = np.zeros(p)
        ei[i] = 1.0
        assert np.max(np.abs(np.asarray(E.heff_matvec(b, en, ei, mode=mode)) - dh[:, i])) <= 1e-12 * scale_h
        assert np.max(np.abs(np.asarray(E.qgt_matvec(b, ei, mode=mode)) - dq[:, i])) <= 1e-12 * scale_q


@pytest.mark.parametrize("mode", MODES)
def test_matches_dense_on_random_vectors(E, setup, mode):
    """T/test_estimators.py:126-135: matvec vs dense product, rel 1e-10."""
    b, en, dh, dq, p = setup
    rng = np.random.default_rng(mode)
    for _ in range(3):
        v = rng.standard_normal(p)
        ref = dh @ v
        got = np.asarray(E.heff_matvec(b, en, v, mode=mode))
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
        ref = dq @ v
        got = np.asarray(E.qgt_matvec(b, v, mode=mode))
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("mode", MODES)
def test_linearity(E, setup, mode):
    """T/test_estimators.py:145-154: H(a u + c v) = a H u + c H v (1e-12)."""
    b, en, _, _, p = setup
    rng = np.random.default_rng(145 + mode)
    u, v = rng.standard_normal(p), rng.standard_normal(p)
    a, c = 1.7, -0.3
    lhs = np.asarray(E.heff_matvec(b, en, a * u + c * v, mode=mode))
    rhs = a * np.asarray(E.heff_matvec(b, en, u, mode=mode)) + c * np.asarray(E.heff_matvec(b, en, v, mode=mode))
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * max(1.0, np.max(np.abs(rhs)))


def test_dense_heff_symmetric_and_qgt_psd(E, setup):
    """T/test_estimators.py:197-206."""
    _, _, dh, dq, _ = setup
    assert np.max(np.abs(dh - dh.T)) <= 1e-12 * np.max(np.abs(dh))
    assert np.max(np.abs(dq - dq.T)) <= 1e-12 * np.max(np.abs(dq))
    assert np.linalg.eigvalsh(dq)[0] >= -1e-12 * np.max(np.abs(dq))


def test_gradient_matches_direct_sum(E, setup):
    """est:156-163: F = 2 Re sum_n w_n (e_n - E) conj(O_n), uncentred O."""
    b, en, _, _, _ = setup
    o = b.o_matrix[:, : b.param_count].cpu().numpy()
    w = b.weights.cpu().numpy()
    e = b.e_loc.cpu().numpy()
    ref = 2.0 * ((w * (e - en.mean)) @ o)
    got = E.energy_gradient(b, en).cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
