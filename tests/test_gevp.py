"""GEVP form of the update, H~ c = lambda S~ c (Eq. 11; the
reference validates it only through its dense oracles at small p, SPEC.md:408,
est:319-344): the device LOBPCG solver (krylov.lobpcg_smallest) on the
bordered pencil against scipy.linalg.eigh of the dense oracle matrices."""

import numpy as np
import pytest
import scipy.linalg

from oracle import estimators as oest


def _pencil(rng, p, cond=1e3):
    a = rng.standard_normal((p, p))
    a = (a + a.T) / 2
    q, _ = np.linalg.qr(rng.standard_normal((p, p)))
    b = (q * np.geomspace(1.0, 1.0 / cond, p)) @ q.T
    return a, (b + b.T) / 2


@pytest.mark.parametrize("p,cond", [(1, 1.0), (7, 10.0), (60, 1e3), (200, 1e4)])
def test_lobpcg_matches_dense_eigh(p, cond):
    import torch
    from paper_2601_01437_b200 import krylov

    rng = np.random.default_rng(p)
    a, b = _pencil(rng, p, cond)
    ta, tb = torch.as_tensor(a), torch.as_tensor(b)
    pair = krylov.lobpcg_smallest(lambda v: ta @ v, lambda v: tb @ v, p, tol=1e-11, max_iter=20000, seed=3)
    lam, vec = scipy.linalg.eigh(a, b)
    assert pair.converged
    assert abs(pair.value - lam[0]) <= 1e-10 * max(1.0, abs(lam[0]))
    x = pair.vector.numpy()
    x = x * np.sign(x @ b @ vec[:, 0])
    assert np.linalg.norm(x - vec[:, 0]) <= 1e-6 * np.linalg.norm(vec[:, 0])


def test_lobpcg_rejects_bad_input():
    import torch
    from paper_2601_01437_b200 import krylov

    with pytest.raises(ValueError):
        krylov.lobpcg_smallest(lambda v: v, lambda v: v, 0)
    with pytest.raises(ValueError):
        krylov.lobpcg_smallest(lambda v: v * float("nan"), lambda v: v, 3)
    with pytest.raises(ValueError):  # indefinite metric
        krylov.lobpcg_smallest(lambda v: v, lambda v: -v, 3)


def _bordered_dense(w, e, o, mean):
    """[[0, (F/2)^T], [F/2, H_eff]] and diag(1, S) from the dense oracles."""
    h = oest.dense_heff(w, e, o, mean)
    s = oest.dense_qgt(w, o)
    g = 0.5 * oest.gradient(w, e, o, mean)
    p = len(g)
    a = np.zeros((p + 1, p + 1))
    a[0, 1:] = g
    a[1:, 0] = g
    a[1:, 1:] = h
    b = np.zeros((p + 1, p + 1))
    b[0, 0] = 1.0
    b[1:, 1:] = s
    return a, b


@pytest.mark.gpu
@pytest.mark.parametrize("n,p", [(400, 17), (3000, 150), (2311, 200)])
def test_gevp_solve_step_vs_dense_oracle(cuda, n, p):
    """optimizer.solve_step(method="gevp") on a device batch: lambda within
    1e-10 and the direction c[1:]/c0 within 1e-8 of scipy's dense eigh."""
    from paper_2601_01437_b200 import estimators as E, optimizer as OPT

    rng = np.random.default_rng(n + p)
    o = rng.standard_normal((n, p)) * 0.1
    e = -1.0 + 0.05 * rng.standard_normal(n) + 0.02 * (o @ rng.standard_normal(p))
    w = np.full(n, 1.0 / n)
    batch = E.SampleBatch([None] * n, w, e, o, n)
    res = OPT.solve_step(batch, OPT.OptimizerConfig(method="gevp", gevp_shift=0.0), seed=5)
    mean, _, _ = oest.energy(w, e, n)
    a, b = _bordered_dense(w, e, o, mean)
    lam, vec = scipy.linalg.eigh(a, b)
    c = vec[:, 0]
    d_ref = c[1:] / c[0]
    assert res.converged
    assert abs(res.lambda_min - lam[0]) <= 1e-10 * abs(lam[0])
    d = res.direction.cpu().numpy()
    assert np.linalg.norm(d - d_ref) <= 1e-8 * np.linalg.norm(d_ref)


@pytest.mark.gpu
def test_gevp_with_diagonal_shift_vs_dense_oracle(cuda):
    """With the SR diagonal shift (S + eps I, eps = shift * mean diag S) on a
    batch whose S is exactly singular (fixed particle number, like the BASELINE
    batches): the solve matches scipy's eigh(H~, diag(1, S + eps I))."""
    from oracle import nqs
    from paper_2601_01437_b200 import ansatz as A, estimators as E, optimizer as OPT, synthetic as S

    cfg = S.CONFIGS[1].with_rows(2048)
    inp = S.make_inputs(cfg)
    arch = A.RBMArchitecture(cfg.n_inputs, cfg.hidden)
    batch = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc)
    conf = OPT.OptimizerConfig(method="gevp", gevp_shift=1e-3, gevp_tol=1e-11, gevp_max_iter=5000)
    res = OPT.solve_step(batch, conf, seed=cfg.lanczos_seed)
    o = nqs.rbm_rows(inp.theta, inp.x, cfg.n_inputs, cfg.hidden)
    n = len(o)
    w = np.full(n, 1.0 / n)
    mean, _, _ = oest.energy(w, inp.e_loc, n)
    a, b = _bordered_dense(w, inp.e_loc, o, mean)
    eps = 1e-3 * float(np.mean(np.diag(b)[1:]))
    b[1:, 1:] += eps * np.eye(len(b) - 1)
    lam, vec = scipy.linalg.eigh(a, b)
    assert np.linalg.matrix_rank(oest.dense_qgt(w, o)) < o.shape[1]  # S itself is singular
    assert res.converged
    assert abs(res.lambda_min - lam[0]) <= 1e-8 * abs(lam[0])
    d_ref = vec[1:, 0] / vec[0, 0]
    assert np.linalg.norm(res.direction.cpu().numpy() - d_ref) <= 1e-6 * np.linalg.norm(d_ref)


def test_lobpcg_apply_ab_equals_separate_products():
    """lobpcg_smallest(apply_ab=...) takes (A v, B v) from one call (the device
    operator streams O once for the pair): same iterates, same answer and the
    same product count as two separate calls."""
    import torch
    from paper_2601_01437_b200 import krylov

    rng = np.random.default_rng(11)
    a, b = _pencil(rng, 40, 100.0)
    ta, tb = torch.as_tensor(a), torch.as_tensor(b)
    calls = [0]

    def both(v):
        calls[0] += 1
        return ta @ v, tb @ v

    one = krylov.lobpcg_smallest(lambda v: ta @ v, lambda v: tb @ v, 40, tol=1e-11, max_iter=5000, seed=2)
    two = krylov.lobpcg_smallest(lambda v: ta @ v, lambda v: tb @ v, 40, tol=1e-11, max_iter=5000, seed=2,
                                 apply_ab=both)
    assert two.converged and one.converged
    assert two.value == one.value and two.n_matvec == one.n_matvec == 2 * calls[0]
    assert torch.equal(two.vector, one.vector)


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,kind", [
    (3000, 1500, "real"),        # fused single-pass rows: one read of O for both products
    (2048, 11265, "real"),       # cfg3 width (2-CTA cluster plan): two products
    (1501, 430, "real"),         # narrow rows: two products (warp-per-row path)
    (2500, 700, "hermitian"),    # complex fused rows
    (1200, 300, "complex_raw"),
])
def test_heff_qgt_matvec_one_read(cuda, n, p, kind):
    """estimators.heff_qgt_matvec (irl_mvp2_*): H_eff v and S v for one v equal
    the separate heff_matvec / qgt_matvec products bit for bit (the same
    operations in the same order, one pass over O) and the oracle's est:171-186
    restatement within 1e-10."""
    import torch
    from paper_2601_01437_b200 import estimators as E

    rng = np.random.default_rng(n + p)
    o = rng.standard_normal((n, p)) * 0.1
    v = rng.standard_normal(p)
    e = -1.0 + 0.05 * rng.standard_normal(n)
    if kind != "real":
        o = o + 0.1j * rng.standard_normal((n, p))
        e = e + 0.01j * rng.standard_normal(n)
    if kind == "hermitian":
        v = v + 1j * rng.standard_normal(p)
    w = rng.random(n)
    w /= w.sum()
    batch = E.SampleBatch([None] * n, w, e, o, n, kind=kind)
    en = E.estimate_energy(batch)
    vt = torch.as_tensor(v, device="cuda")
    hv, sv = E.heff_qgt_matvec(batch, en, vt)
    assert torch.equal(hv, E.heff_matvec(batch, en, vt))
    assert torch.equal(sv, E.qgt_matvec(batch, vt))
    hn, sn = E.heff_qgt_matvec(batch, en, v)  # numpy in -> numpy out
    assert np.array_equal(hn, hv.cpu().numpy()) and np.array_equal(sn, sv.cpu().numpy())
    if kind == "real":
        mean, _, _ = oest.energy(w, e, n)
        ref_h = oest.heff(w, e, o, mean, v)
        ref_s = oest.qgt(w, o, v)
        assert np.linalg.norm(hn - ref_h) <= 1e-10 * np.linalg.norm(ref_h)
        assert np.linalg.norm(sn - ref_s) <= 1e-10 * np.linalg.norm(ref_s)
    with pytest.raises(ValueError):
        E.heff_qgt_matvec(batch, en, np.zeros(p + 1))


@pytest.mark.gpu
def test_gevp_fused_pair_solve(cuda):
    """solve_step(method="gevp") on rows wide enough for the one-read pair
    (p = 1200): lambda within 1e-9 of scipy's dense eigh of the oracle pencil."""
    from paper_2601_01437_b200 import estimators as E, optimizer as OPT

    n, p = 4000, 1200
    rng = np.random.default_rng(77)
    o = rng.standard_normal((n, p)) * 0.1
    e = -1.0 + 0.05 * rng.standard_normal(n) + 0.02 * (o @ rng.standard_normal(p))
    w = np.full(n, 1.0 / n)
    batch = E.SampleBatch([None] * n, w, e, o, n)
    res = OPT.solve_step(batch, OPT.OptimizerConfig(method="gevp", gevp_shift=0.0, gevp_tol=1e-11,
                                                    gevp_max_iter=6000), seed=5)
    mean, _, _ = oest.energy(w, e, n)
    a, b = _bordered_dense(w, e, o, mean)
    lam = scipy.linalg.eigh(a, b, eigvals_only=True, subset_by_index=[0, 0])
    assert res.converged
    assert abs(res.lambda_min - lam[0]) <= 1e-9 * abs(lam[0])
