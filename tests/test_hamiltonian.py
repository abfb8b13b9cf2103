"""Local energies from FCIDUMP integrals (hamiltonian.py:94-302).

CPU tests pin the oracle restatement (oracle/hamiltonian.py) and the host
parser / sector enumeration to the reference's own outputs
(tests/golden/hamiltonian.npz, made by oracle/make_golden.py from
/root/reference: a seeded synthetic FCIDUMP and H2's real one).  GPU tests pin
the k_local_energy kernels (through the C-ABI) to the same fixture, and the
H2 Hamiltonian assembled from the device enumeration to the FCI energy
-1.1372930376796802 (T/test_optimizer.py:16).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import hamiltonian as oham
from oracle import nqs

ELOC_TOL = 1e-10


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def host(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def g():
    return golden("hamiltonian")


def occ(bits, m):
    return ((np.asarray(bits, dtype=np.uint64)[:, None] >> np.arange(m, dtype=np.uint64)[None, :])
            & np.uint64(1)).astype(np.uint8)


def logpsi_fns(g):
    M = 2 * int(g["ns"])
    hr, hm = int(g["hidden_rbm"]), int(g["hidden_mlp"])
    one = lambda b: occ([b], M)  # noqa: E731
    return {
        "rbm": lambda b: nqs.rbm_log_psi(g["theta_rbm"], one(b), M, hr)[0],
        "rbmc": lambda b: nqs.rbm_log_psi(g["theta_rbmc"], one(b), M, hr)[0],
        "mlp": lambda b: nqs.mlp_log_psi(g["theta_mlp"], one(b), M, hm)[0],
    }


# ------------------------------------------------------------------- CPU --
def test_parser_matches_reference(g):
    from paper_2601_01437_b200 import hamiltonian as H

    ints = H.parse_fcidump(str(g["fcidump"]))
    assert ints.n_spatial == int(g["ns"]) and ints.e_core == float(g["e_core"])
    assert np.array_equal(ints.h, g["h"]) and np.array_equal(ints.g, g["g"])
    sec = ints.sector()
    assert (sec.n_up, sec.n_down) == (int(g["n_up"]), int(g["n_down"]))
    assert np.array_equal(H.enumerate_sector(sec), g["bits"])


def test_parser_errors():
    from paper_2601_01437_b200 import hamiltonian as H

    with pytest.raises(H.FcidumpError):
        H.parse_fcidump("&FCI NORB=2,NELEC=2,\n 1.0 1 1 1 1\n")  # no &END
    with pytest.raises(H.FcidumpError):
        H.parse_fcidump("&FCI NORB=2,NELEC=2,\n&END\n 1.0 3 1 1 1\n")  # index out of range
    with pytest.raises(H.FcidumpError):
        H.parse_fcidump("&FCI NORB=2,NELEC=2,\n&END\n 1.0 1 2 0 0\n 2.0 2 1 0 0\n")  # conflicting h


def test_oracle_connected_matches_reference(g):
    ns = int(g["ns"])
    ip = g["partner_indptr"]
    for k, x in enumerate(g["bits"][:40]):
        ent = oham.connected(float(g["e_core"]), g["h"], g["g"], int(x), ns)
        assert ent[0][1] == pytest.approx(float(g["diag"][k]), abs=1e-13)
        ys = np.array([y for y, _ in ent[1:]], dtype=np.uint64)
        els = np.array([e for _, e in ent[1:]])
        assert np.array_equal(ys, g["partner_bits"][ip[k]:ip[k + 1]])
        assert np.max(np.abs(els - g["partner_elem"][ip[k]:ip[k + 1]]), initial=0.0) < 1e-13


@pytest.mark.parametrize("name", ["rbm", "rbmc", "mlp"])
def test_oracle_local_energy_matches_reference(g, name):
    ns = int(g["ns"])
    lp = logpsi_fns(g)[name]
    got = np.array([oham.local_energy(lp, float(g["e_core"]), g["h"], g["g"], int(x), ns) for x in g["bits"][:30]])
    assert rel(got, g[f"eloc_{name}"][:30]) < 1e-13


def test_oracle_dense_and_h2_fci(g):
    ns = int(g["ns"])
    d = oham.dense_hamiltonian(float(g["e_core"]), g["h"], g["g"], [int(b) for b in g["bits"]], ns)
    assert np.max(np.abs(d - g["dense"])) < 1e-13
    h2 = oham.dense_hamiltonian(float(g["h2_e_core"]), g["h2_h"], g["h2_g"], [int(b) for b in g["h2_bits"]],
                                int(g["h2_ns"]))
    assert np.max(np.abs(h2 - g["h2_dense"])) < 1e-14
    assert abs(np.linalg.eigvalsh(h2)[0] - float(g["h2_fci"])) < 1e-10


# ------------------------------------------------------------------- GPU --
def device_params(g, name):
    from paper_2601_01437_b200 import ansatz as A

    M = 2 * int(g["ns"])
    if name == "mlp":
        return A.AnsatzParameters(A.MLPArchitecture(M, int(g["hidden_mlp"])), g["theta_mlp"])
    cplx = name == "rbmc"
    return A.AnsatzParameters(A.RBMArchitecture(M, int(g["hidden_rbm"]), complex_params=cplx),
                              g["theta_rbmc" if cplx else "theta_rbm"])


def device_integrals(g, prefix=""):
    from paper_2601_01437_b200 import hamiltonian as H

    ns = int(g[prefix + "ns"])
    n_up, n_dn = int(g[prefix + "n_up"]), int(g[prefix + "n_down"])
    return H.MolecularIntegrals(ns, n_up + n_dn, n_up - n_dn, float(g[prefix + "e_core"]), g[prefix + "h"],
                                g[prefix + "g"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rbm", "rbmc", "mlp"])
def test_device_local_energy_golden(cuda, g, name):
    from paper_2601_01437_b200 import hamiltonian as H

    ints = device_integrals(g)
    e = host(H.local_energies(device_params(g, name), ints, g["bits"]))
    ref = g[f"eloc_{name}"]
    if name != "rbmc":
        ref = ref.real
    assert np.max(np.abs(e - ref) / np.maximum(1.0, np.abs(ref))) < ELOC_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rbm", "rbmc", "mlp"])
def test_device_connected_partners_golden(cuda, g, name):
    from paper_2601_01437_b200 import hamiltonian as H

    ints = device_integrals(g)
    params = device_params(g, name)
    indptr, pbits, elem, coeff = H.connected_partners(params, ints, g["bits"])
    ip, pb = host(indptr), host(pbits).view(np.uint64)
    el, cf = host(elem), host(coeff)
    assert np.array_equal(ip, g["partner_indptr"])  # same kept counts per sample
    lp = logpsi_fns(g)[name]
    gip = g["partner_indptr"]
    for k, x in enumerate(g["bits"]):
        order = np.argsort(pb[ip[k]:ip[k + 1]])  # device order is enumeration order
        assert np.array_equal(pb[ip[k]:ip[k + 1]][order], g["partner_bits"][gip[k]:gip[k + 1]])
        e_k = el[ip[k]:ip[k + 1]][order]
        assert np.max(np.abs(e_k - g["partner_elem"][gip[k]:gip[k + 1]]), initial=0.0) < 1e-13
        if k < 20:
            lx = complex(lp(int(x)))
            want = np.array([e * np.exp(complex(lp(int(y))) - lx) for y, e in zip(pb[ip[k]:ip[k + 1]], el[ip[k]:ip[k + 1]])])
            if name != "rbmc":
                want = want.real
            assert np.max(np.abs(cf[ip[k]:ip[k + 1]] - want), initial=0.0) < 1e-12


@pytest.mark.gpu
def test_device_h2_hamiltonian_fci_energy(cuda, g):
    """H2 (T/data/h2_sto3g.fcidump): the sector Hamiltonian assembled from the
    device enumeration (off-diagonal elements; diagonal = E_loc - sum of the
    partner coefficients) has the FCI ground-state energy."""
    from paper_2601_01437_b200 import ansatz as A, hamiltonian as H

    ints = device_integrals(g, "h2_")
    M = ints.n_spin_orbitals
    params = A.AnsatzParameters(A.RBMArchitecture(M, 3), np.random.default_rng(4).normal(0, 0.2, M + 3 + 3 * M))
    bits = g["h2_bits"]
    indptr, pbits, elem, coeff = H.connected_partners(params, ints, bits)
    eloc = host(H.local_energies(params, ints, bits))
    ip, pb, el, cf = host(indptr), host(pbits).view(np.uint64), host(elem), host(coeff)
    idx = {int(b): k for k, b in enumerate(bits)}
    mat = np.zeros((len(bits), len(bits)))
    for k in range(len(bits)):
        for e in range(ip[k], ip[k + 1]):
            mat[idx[int(pb[e])], k] = el[e]
        mat[k, k] = eloc[k] - cf[ip[k]:ip[k + 1]].sum()
    assert np.max(np.abs(mat - g["h2_dense"])) < 1e-12
    assert abs(np.linalg.eigvalsh(mat)[0] - float(g["h2_fci"])) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rbm", "mlp", "rbmc"])
def test_exact_batch_and_connected_step(cuda, g, name):
    """est.build_batch (exact mode) + est.build_connected_cache + the
    optimizer's full operator (opt:134-165) against the oracle."""
    import warnings

    from oracle import bordered as obord, estimators as oest
    from paper_2601_01437_b200 import estimators as E, hamiltonian as H, optimizer as OPT

    ints = device_integrals(g)
    params = device_params(g, name)
    b = H.build_batch(params, ints, ints.sector())
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        en = E.estimate_energy(b)
    M = 2 * int(g["ns"])
    lp = logpsi_fns(g)[name]
    bits = g["bits"]
    lpx = np.array([complex(lp(int(x))) for x in bits])
    w = np.exp(2 * (lpx.real - lpx.real.max()))
    w /= w.sum()
    e_ref = g[f"eloc_{name}"]
    assert abs(en.mean - float(np.sum(w * e_ref).real)) < 1e-10 * abs(en.mean)
    cache = H.build_connected_cache(params, ints, ints.sector(), b)
    # oracle rows, partner rows and coefficients
    x = occ(bits, M)
    if name == "mlp":
        o = nqs.mlp_rows(g["theta_mlp"], x, M, int(g["hidden_mlp"]))
        rows = lambda xx: nqs.mlp_rows(g["theta_mlp"], xx, M, int(g["hidden_mlp"]))  # noqa: E731
    else:
        th = g["theta_rbmc" if name == "rbmc" else "theta_rbm"]
        o = nqs.rbm_rows(th, x, M, int(g["hidden_rbm"]))
        rows = lambda xx: nqs.rbm_rows(th, xx, M, int(g["hidden_rbm"]))  # noqa: E731
    gip, gpb, gpe = g["partner_indptr"], g["partner_bits"], g["partner_elem"]
    uniq, inv = np.unique(gpb, return_inverse=True)
    po = rows(occ(uniq, M))
    seg = np.repeat(np.arange(len(bits)), np.diff(gip))
    coeff = gpe * np.exp(np.array([complex(lp(int(y))) for y in gpb]) - lpx[seg])
    rng = np.random.default_rng(3)
    P = o.shape[1]
    for _ in range(2):
        if name == "rbmc":
            v = rng.standard_normal(P) + 1j * rng.standard_normal(P)
            ref = oest.heff_offdiag_hermitian(w, o, np.arange(len(bits)), gip, inv.reshape(-1), coeff, po, v)
        else:
            v = rng.standard_normal(P)
            ref = oest.heff_offdiag(w, o, np.arange(len(bits)), gip, inv.reshape(-1), coeff.real, po, v)
        got = E.heff_offdiag_matvec(b, cache, v)
        assert rel(got, ref) < 1e-10
    if name == "rbmc":
        return
    res = OPT.solve_step(b, OPT.OptimizerConfig(m=20, max_restarts=3), energy=en, seed=9, connected=cache)
    mean = en.mean
    grad = oest.gradient(w, e_ref.real, o, mean)
    half = 0.5 * grad
    dist = np.arange(len(bits))

    def matvec(u):
        out = np.empty(P + 1)
        out[0] = half @ u[1:]
        out[1:] = (u[0] * half + oest.heff(w, e_ref.real, o, mean, u[1:])
                   + oest.heff_offdiag(w, o, dist, gip, inv.reshape(-1), coeff.real, po, u[1:]))
        return out

    pair, d = obord.solve(matvec, P + 1, grad, 20, max_restarts=3, seed=9)
    assert res.n_matvec == pair["n_matvec"]
    assert abs(res.lambda_min - pair["value"]) <= 1e-10 * abs(pair["value"])
    assert rel(host(res.direction), d) < 1e-8


@pytest.mark.gpu
def test_outer_step_golden(cuda, g):
    """The reference outer step (opt:118-195, assembled from reference
    primitives in oracle/make_golden.py::case_outer_step) on the device: same
    matvec count, Ritz value, direction, accepted line-search scale and energy."""
    from paper_2601_01437_b200 import ansatz as A, optimizer as OPT

    o = golden("outer_step")
    ints = device_integrals(g)
    M = ints.n_spin_orbitals
    params = A.AnsatzParameters(A.RBMArchitecture(M, int(o["hidden"])), o["theta"])
    cfg = OPT.OptimizerConfig()
    res = OPT.outer_step(params, ints, ints.sector(), cfg, int(o["step"]))
    assert abs(res.energy - float(o["energy"])) < 1e-10 * abs(float(o["energy"]))
    assert res.matvecs == int(o["n_matvec"])
    assert abs(res.lambda_min - float(o["lam"])) <= 1e-10 * abs(float(o["lam"]))
    assert res.step_scale == float(o["best_scale"])
    assert abs(res.best_energy - float(o["best_energy"])) < 1e-10 * abs(float(o["best_energy"]))
    assert rel(res.params.theta, o["theta_new"]) < 1e-8
    scan = [OPT.energy_at(A.AnsatzParameters(params.architecture, o["theta"] + s * o["direction"]), ints,
                          ints.sector()) for s in cfg.line_search]
    assert rel(scan, o["scan"][: len(scan)]) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rbm", "rbmc"])
def test_otf_batch_in_batch_partners(cuda, g, name):
    """Exact batch with O regenerated on the fly: the partners are batch rows, so
    the completion takes its partner dots from the product's own centred dots
    (no partner O at all); products and the solve match the stored-O batch."""
    from paper_2601_01437_b200 import estimators as E, hamiltonian as H, optimizer as OPT

    ints = device_integrals(g)
    params = device_params(g, name)
    bs = H.build_batch(params, ints, ints.sector())
    bo = H.build_batch(params, ints, ints.sector(), mode="otf")
    cs = H.build_connected_cache(params, ints, ints.sector(), bs)
    co = H.build_connected_cache(params, ints, ints.sector(), bo)
    assert co.in_batch and cs.in_batch
    ens, eno = E.estimate_energy(bs), E.estimate_energy(bo)
    P = bs.param_count
    rng = np.random.default_rng(5)
    for _ in range(2):
        v = rng.standard_normal(P) + (1j * rng.standard_normal(P) if name == "rbmc" else 0.0)
        a = E.heff_offdiag_matvec(bs, cs, v)
        b = E.heff_offdiag_matvec(bo, co, v)
        assert rel(b, a) < 1e-10
        a = E.connected_heff_matvec(bs, ens, cs, v)
        b = E.connected_heff_matvec(bo, eno, co, v)
        assert rel(b, a) < 1e-10
    conf = OPT.OptimizerConfig(m=20, max_restarts=3)
    rs = OPT.solve_step(bs, conf, energy=ens, seed=3, connected=cs)
    ro = OPT.solve_step(bo, conf, energy=eno, seed=3, connected=co)
    assert ro.n_matvec == rs.n_matvec
    assert abs(ro.lambda_min - rs.lambda_min) <= 1e-10 * abs(rs.lambda_min)


@pytest.mark.gpu
@pytest.mark.parametrize("ns,n_up,n_dn,hidden,seed", [
    (1, 1, 0, 2, 1),    # two spin-orbitals, one electron: no partners of one spin
    (3, 0, 2, 4, 2),    # empty spin-up channel
    (4, 4, 1, 2, 3),    # full spin-up channel: no up particles
    (5, 2, 3, 6, 4),
    (6, 3, 3, 4, 5),
])
def test_local_energy_sector_edges(cuda, ns, n_up, n_dn, hidden, seed):
    """Edge sectors (empty / full spin channels, a single orbital) of the
    device enumeration against the oracle restatement (ham:238-302): kept
    partner sets and elements, local energies for the real and complex RBM."""
    from paper_2601_01437_b200 import ansatz as A, hamiltonian as H, synthetic as S

    ints = H.parse_fcidump(S.molecule_fcidump(seed, ns, n_up + n_dn, ms2=n_up - n_dn))
    sec = ints.sector()
    assert (sec.n_up, sec.n_down) == (n_up, n_dn)
    bits = H.enumerate_sector(sec)
    M = 2 * ns
    rng = np.random.default_rng(seed)
    for cplx in (False, True):
        P = M + hidden + hidden * M
        theta = rng.normal(0, 0.3, P) + (1j * rng.normal(0, 0.3, P) if cplx else 0.0)
        params = A.AnsatzParameters(A.RBMArchitecture(M, hidden, complex_params=cplx), theta)
        e = host(H.local_energies(params, ints, bits))
        lp = lambda b: nqs.rbm_log_psi(theta, occ([b], M), M, hidden)[0]  # noqa: E731
        ref = np.array([oham.local_energy(lp, ints.e_core, ints.h, ints.g, int(b), ns) for b in bits])
        if not cplx:
            ref = ref.real
        assert np.max(np.abs(e - ref) / np.maximum(1.0, np.abs(ref))) < ELOC_TOL
        indptr, pbits, elem, _ = H.connected_partners(params, ints, bits)
        ip, pb, el = host(indptr), host(pbits).view(np.uint64), host(elem)
        for k, b in enumerate(bits):
            want = oham.connected(ints.e_core, ints.h, ints.g, int(b), ns)[1:]
            order = np.argsort(pb[ip[k]:ip[k + 1]])
            assert np.array_equal(pb[ip[k]:ip[k + 1]][order], np.array([y for y, _ in want], dtype=np.uint64))
            assert np.allclose(el[ip[k]:ip[k + 1]][order], [x for _, x in want], atol=1e-13, rtol=0)
