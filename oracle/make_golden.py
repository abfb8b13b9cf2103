"""Generate tests/golden/*.npz from the REAL reference package (this container only).

Run:  python oracle/make_golden.py
Imports irlnqs read-only from /root/reference/pkg/src (bytecode writing off)
and records its outputs on small seeded inputs.  The fixtures pin the
oracle restatement (tests/test_oracle_golden.py) and the device path
(tests/test_gpu_parity.py).  /root/reference is NOT needed at test time.
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import numpy as np  # noqa: E402

from irlnqs import ansatz as ans  # noqa: E402
from irlnqs import estimators as est  # noqa: E402
from irlnqs import krylov as kry  # noqa: E402
from irlnqs.hamiltonian import parse_fcidump  # noqa: E402
from irlnqs.hilbert import OccupationVector  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def placeholder_batch(w, e, o, n_samples):
    """SampleBatch with placeholder configs."""
    configs = (OccupationVector(0, 2),) * len(w)
    return est.SampleBatch(configs=configs, weights=w, e_loc=e, o_matrix=o, n_samples=n_samples)


def bordered(batch, energy, grad):
    """opt:140-148 minus the offdiag term (synthetic E_loc)."""
    p = batch.param_count
    half = 0.5 * grad

    def matvec(u):
        out = np.empty(p + 1)
        out[0] = half @ u[1:]
        out[1:] = u[0] * half + est.heff_matvec(batch, energy, u[1:])
        return out

    return matvec


def direction(vec, grad):
    c0 = vec[0]
    d = vec[1:]
    if abs(c0) > 1e-12:
        return d / c0
    return -d if float(grad @ d) > 0 else d


def rbm_rows_np(theta, x, n, h):
    xf = x.astype(float)
    a, b, w = theta[:n], theta[n : n + h], theta[n + h :].reshape(h, n)
    t = np.tanh(b + xf @ w.T)
    return np.concatenate([xf.astype(t.dtype), t, (t[:, :, None] * xf[:, None, :]).reshape(len(x), -1)], axis=1)


def case_real(seed=7, n=6, h=5, N=96, m=20):
    """Real RBM-shaped batch (P = n + h + h n = 41)."""
    rng = np.random.default_rng(seed)
    x = np.zeros((N, n), dtype=np.uint8)
    occ = np.argsort(rng.random((N, n)), axis=1)[:, : n // 2]
    x[np.arange(N)[:, None], occ] = 1
    theta = rng.normal(0, 0.3, n + h + h * n)
    e = rng.normal(-7.5, 0.4, N)
    w = np.full(N, 1.0 / N)
    o = rbm_rows_np(theta, x, n, h)
    batch = placeholder_batch(w, e, o, N)
    energy = est.estimate_energy(batch)
    grad = est.energy_gradient(batch, energy)
    vs = rng.standard_normal((4, o.shape[1]))
    hv = np.array([est.heff_matvec(batch, energy, v) for v in vs])
    sb = placeholder_batch(w, np.ones(N), o, N)
    sv = np.array([est.heff_matvec(sb, est.EnergyEstimate(0.0, 0.0, 0.0), v) for v in vs])
    pair = kry.irl_smallest(bordered(batch, energy, grad), o.shape[1] + 1, m=m, tol=1e-12, max_restarts=3, seed=seed)
    return dict(
        x=x, theta=theta, n=n, h=h, e=e, w=w, o=o, mean=energy.mean, variance=energy.variance,
        std_error=energy.std_error, grad=grad, vs=vs, hv=hv, sv=sv,
        dense_heff=est.dense_heff(batch, energy), dense_qgt=est.dense_qgt(batch),
        lam=pair.value, vec=pair.vector, residual=pair.residual, n_matvec=pair.n_matvec,
        n_restarts=pair.n_restarts, converged=pair.converged, direction=direction(pair.vector, grad),
        m=m, seed=seed,
    )


def case_complex_raw(seed=11, N=80, P=19, m=20):
    """Complex O and E_loc with real parameters: the reference's own convention."""
    rng = np.random.default_rng(seed)
    o = rng.normal(0.2, 0.5, (N, P)) + 1j * rng.normal(-0.1, 0.5, (N, P))
    e = rng.normal(-3.0, 0.2, N) + 1j * rng.normal(0.0, 0.05, N)
    w = rng.random(N) + 0.1
    w = w / w.sum()
    batch = placeholder_batch(w, e, o, N)
    energy = est.estimate_energy(batch)
    grad = est.energy_gradient(batch, energy)
    vs = rng.standard_normal((4, P))
    hv = np.array([est.heff_matvec(batch, energy, v) for v in vs])
    pair = kry.irl_smallest(bordered(batch, energy, grad), P + 1, m=m, tol=1e-12, max_restarts=3, seed=seed)
    return dict(o=o, e=e, w=w, mean=energy.mean, variance=energy.variance, std_error=energy.std_error, grad=grad,
                vs=vs, hv=hv, lam=pair.value, vec=pair.vector, n_matvec=pair.n_matvec, residual=pair.residual,
                direction=direction(pair.vector, grad), m=m, seed=seed, n_samples=N)


def case_hermitian(seed=13, n=4, h=3, N=72, m=20):
    """Complex-parameter RBM through the real embedding [O, iO]."""
    rng = np.random.default_rng(seed)
    x = np.zeros((N, n), dtype=np.uint8)
    occ = np.argsort(rng.random((N, n)), axis=1)[:, : n // 2]
    x[np.arange(N)[:, None], occ] = 1
    P = n + h + h * n
    theta = rng.normal(0, 0.2, P) + 1j * rng.normal(0, 0.2, P)
    e = rng.normal(-5.0, 0.3, N) + 1j * rng.normal(0.0, 0.1, N)
    w = np.full(N, 1.0 / N)
    o = rbm_rows_np(theta, x, n, h)
    emb = np.concatenate([o, 1j * o], axis=1)
    gbatch = placeholder_batch(w, e, emb, N)
    energy = est.estimate_energy(gbatch)
    grad = est.energy_gradient(gbatch, energy)
    hbatch = placeholder_batch(w, e.real.copy(), emb, N)
    vs = rng.standard_normal((3, 2 * P))
    hv = np.array([est.heff_matvec(hbatch, energy, v) for v in vs])
    pair = kry.irl_smallest(bordered(hbatch, energy, grad), 2 * P + 1, m=m, tol=1e-12, max_restarts=3, seed=seed)
    return dict(x=x, theta=theta, n=n, h=h, e=e, w=w, o=o, mean=energy.mean, grad=grad, vs=vs, hv=hv,
                lam=pair.value, vec=pair.vector, n_matvec=pair.n_matvec, residual=pair.residual,
                direction=direction(pair.vector, grad), m=m, seed=seed)


def case_h2():
    """The reference's own data path: H2 exact mode, autoregressive ansatz
    (T/test_estimators.py:20-28 setup, hidden 3, seed 9)."""
    with open(os.path.join(REF, "tests", "data", "h2_sto3g.fcidump")) as fh:
        integrals = parse_fcidump(fh.read())
    sector = integrals.sector()
    arch = ans.Architecture(sector.n_orbitals, 3)
    params = ans.init_parameters(arch, seed=9)
    rng = np.random.default_rng(41)
    theta = params.theta + 0.1 * rng.standard_normal(arch.param_count)  # generic complex state (:31-41)
    params = ans.AnsatzParameters(arch, theta)
    batch = est.build_batch(params, integrals, sector)
    energy = est.estimate_energy(batch)
    grad = est.energy_gradient(batch, energy)
    vs = np.random.default_rng(55).standard_normal((5, batch.param_count))
    hv = np.array([est.heff_matvec(batch, energy, v) for v in vs])
    return dict(o=np.array(batch.o_matrix), e=np.array(batch.e_loc), w=np.array(batch.weights),
                mean=energy.mean, variance=energy.variance, grad=grad, vs=vs, hv=hv,
                dense_heff=est.dense_heff(batch, energy), dense_qgt=est.dense_qgt(batch))


def case_mlp_phase_head(seed=17):
    """MLP rows == reference phase-head gradient (ans:278-288) minus w_lin."""
    arch = ans.Architecture(6, 5)
    rng = np.random.default_rng(seed)
    theta = ans.init_parameters(arch, seed=seed).theta + 0.3 * rng.standard_normal(arch.param_count)
    params = ans.AnsatzParameters(arch, theta)
    from irlnqs.hilbert import Sector, enumerate_sector

    sector = Sector(6, 2, 1)
    xs = enumerate_sector(sector)[:12]
    m, h = arch.n_orbitals, arch.hidden
    sizes = [h * 2 * m, h, 2 * h, 2, h * m, h, h, m, 1]
    off = np.cumsum([0] + sizes)
    rows = []
    s_list = []
    for x in xs:
        od = ans.log_derivative(params, x, sector).imag
        rows.append(np.concatenate([od[off[4] : off[5]], od[off[5] : off[6]], od[off[6] : off[7]], od[off[8] : off[9]]]))
        s_list.append([1.0 if x.occupied(j) else -1.0 for j in range(m)])
    mlp_theta = np.concatenate([theta[off[4] : off[5]], theta[off[5] : off[6]], theta[off[6] : off[7]], theta[off[8] : off[9]]])
    return dict(s=np.array(s_list), theta=mlp_theta, n=m, h=h, rows=np.array(rows))


def case_krylov(seed=100, count=4):
    """Reference irl_smallest / lanczos / implicit_restart on random symmetric matrices
    (the T/oracles.py:158-163 construction)."""
    from oracles import random_symmetric

    rng = np.random.default_rng(seed)
    out = {}
    for i in range(count):
        dim = int(rng.integers(60, 160))
        mat = random_symmetric(rng, dim, condition=10.0 ** rng.uniform(1, 3))
        pair = kry.irl_smallest(lambda v: mat @ v, dim, m=20, tol=1e-12, seed=i)
        v1 = rng.standard_normal(dim)
        v1 /= np.linalg.norm(v1)
        lz = kry.lanczos(lambda v: mat @ v, v1, 20)
        vals, _ = kry.tridiag_eigen(lz.tri)
        nb, nt = kry.implicit_restart(lz.basis, lz.tri, vals[1:], 1)
        nb5, nt5 = kry.implicit_restart(lz.basis, lz.tri, vals[5:], 5)
        out.update({
            f"mat{i}": mat, f"value{i}": pair.value, f"vector{i}": pair.vector, f"residual{i}": pair.residual,
            f"n_matvec{i}": pair.n_matvec, f"n_restarts{i}": pair.n_restarts, f"v1_{i}": v1,
            f"alpha{i}": lz.tri.alpha, f"beta{i}": lz.tri.beta, f"beta_last{i}": lz.tri.beta_last,
            f"restart_v{i}": nb.vectors, f"restart_next{i}": nb.next_vector, f"restart_alpha{i}": nt.alpha,
            f"restart_beta_last{i}": nt.beta_last, f"restart5_v{i}": nb5.vectors, f"restart5_alpha{i}": nt5.alpha,
            f"restart5_beta{i}": nt5.beta, f"restart5_beta_last{i}": nt5.beta_last,
        })
    out["count"] = count
    return out


def bordered_connected(batch, energy, grad, cache):
    """The reference optimizer's full operator, opt:140-148 WITH heff_offdiag_matvec (opt:146)."""
    p = batch.param_count
    half = 0.5 * grad

    def matvec(u):
        out = np.empty(p + 1)
        out[0] = half @ u[1:]
        out[1:] = u[0] * half + est.heff_matvec(batch, energy, u[1:]) + est.heff_offdiag_matvec(batch, cache, u[1:])
        return out

    return matvec


def _cache_arrays(cache):
    return dict(dist_index=np.array(cache.dist_index), indptr=np.array(cache.indptr),
                partner_row=np.array(cache.partner_row), coeff=np.array(cache.coeff),
                partner_o=np.array(cache.partner_o))


def case_h2_connected(m=20):
    """The reference's own connected completion (T/test_estimators.py:170-193):
    H2 generic complex state, exact batch and a stochastic batch with duplicate
    configurations (n_samples=64, seed=13, :71-80); both products, the sandwich
    oracle and the full optimizer operator's IRL solve (opt:134-165)."""
    from irlnqs.hamiltonian import build_dense_hamiltonian
    from irlnqs.hilbert import enumerate_sector

    with open(os.path.join(REF, "tests", "data", "h2_sto3g.fcidump")) as fh:
        integrals = parse_fcidump(fh.read())
    sector = integrals.sector()
    arch = ans.Architecture(sector.n_orbitals, 3)
    init = ans.init_parameters(arch, seed=9)
    rng = np.random.default_rng(41)
    params = ans.AnsatzParameters(arch, init.theta + 0.1 * rng.standard_normal(arch.param_count))
    out = {}
    for tag, kw in (("exact", {}), ("stoch", dict(n_samples=64, seed=13))):
        batch = est.build_batch(params, integrals, sector, **kw)
        energy = est.estimate_energy(batch)
        grad = est.energy_gradient(batch, energy)
        cache = est.build_connected_cache(params, integrals, sector, batch)
        vs = np.random.default_rng(88).standard_normal((6, batch.param_count))
        off = np.array([est.heff_offdiag_matvec(batch, cache, v) for v in vs])
        full = np.array([est.heff_matvec(batch, energy, v) + est.heff_offdiag_matvec(batch, cache, v) for v in vs])
        pair = kry.irl_smallest(bordered_connected(batch, energy, grad, cache), batch.param_count + 1, m=m,
                                tol=1e-12, max_restarts=3, seed=5)
        d = {"o": np.array(batch.o_matrix), "e": np.array(batch.e_loc), "w": np.array(batch.weights),
             "n_samples": batch.n_samples, "mean": energy.mean, "grad": grad, "vs": vs, "off": off, "full": full,
             "lam": pair.value, "vec": pair.vector, "n_matvec": pair.n_matvec,
             "direction": direction(pair.vector, grad), **_cache_arrays(cache)}
        if tag == "exact":
            hmat = build_dense_hamiltonian(integrals, sector)
            amps = np.array([np.exp(ans.log_amplitude(params, x, sector).value) for x in enumerate_sector(sector)])
            psi = amps / np.linalg.norm(amps)
            o_bar = batch.weights @ batch.o_matrix
            tangent = psi[:, None] * (batch.o_matrix - o_bar)
            d["sandwich"] = (tangent.conj().T @ (hmat - energy.mean * np.eye(len(psi))) @ tangent).real
        out.update({f"{tag}_{k}": v for k, v in d.items()})
    out["m"] = m
    out["seed"] = 5
    return out


def rbm_log_psi_np(theta, x, n, h):
    xf = x.astype(float)
    a, b, w = theta[:n], theta[n : n + h], theta[n + h :].reshape(h, n)
    return xf @ a + np.sum(np.log(np.cosh(b + xf @ w.T)), axis=-1)


def _rbm_partner_case(seed, n, h, N, per_row, complex_params):
    rng = np.random.default_rng(seed)
    x = np.zeros((N, n), dtype=np.uint8)
    occ = np.argsort(rng.random((N, n)), axis=1)[:, : n // 2]
    x[np.arange(N)[:, None], occ] = 1
    x[N // 2 :] = x[: N - N // 2]  # duplicate configurations (stochastic batches repeat samples)
    P = n + h + h * n
    theta = rng.normal(0, 0.2, P)
    if complex_params:
        theta = theta + 1j * rng.normal(0, 0.2, P)
    # distinct configurations, first-occurrence order (est:228-233)
    keys = [bytes(r) for r in x]
    first = {}
    for i, k in enumerate(keys):
        first.setdefault(k, len(first))
    dist_index = np.array([first[k] for k in keys])
    reps = np.array([keys.index(k) for k in first])
    # partners: random particle-conserving single excitations (the data shape of ham:260-264)
    partners, elements, indptr = [], [], [0]
    for r in reps:
        cnt = int(rng.integers(0, per_row + 1))
        for _ in range(cnt):
            y = x[r].copy()
            y[rng.choice(np.flatnonzero(y == 1))] = 0
            y[rng.choice(np.flatnonzero(x[r] == 0))] = 1
            partners.append(y)
            elements.append(rng.normal(0.0, 0.3))
        indptr.append(len(partners))
    partners = np.array(partners, dtype=np.uint8).reshape(-1, n)
    elements = np.array(elements)
    uniq, inv = np.unique(partners, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    seg = np.repeat(np.arange(len(reps)), np.diff(indptr))
    coeff = elements * np.exp(rbm_log_psi_np(theta, partners, n, h) - rbm_log_psi_np(theta, x[reps], n, h)[seg])
    o = rbm_rows_np(theta, x, n, h)
    po = rbm_rows_np(theta, uniq, n, h)
    w = rng.random(N) + 0.2
    w = w / w.sum()
    return dict(x=x, theta=theta, n=n, h=h, w=w, o=o, partners=partners, elements=elements, indptr=np.array(indptr),
                dist_index=dist_index, partner_row=inv, partner_o=po, uniq=uniq, coeff=coeff.astype(complex),
                logpsi_x=rbm_log_psi_np(theta, x, n, h), logpsi_p=rbm_log_psi_np(theta, partners, n, h))


def case_rbm_connected(seed=21, n=6, h=4, N=40, per_row=5):
    """Real RBM batch with a partner cache through the reference heff_offdiag_matvec (est:254-294)."""
    d = _rbm_partner_case(seed, n, h, N, per_row, False)
    batch = placeholder_batch(d["w"], np.zeros(N), d["o"].astype(complex), N)
    cache = est.ConnectedCache(d["dist_index"], d["indptr"], d["partner_row"], d["coeff"],
                               d["partner_o"].astype(complex))
    vs = np.random.default_rng(seed + 1).standard_normal((4, d["o"].shape[1]))
    d["vs"] = vs
    d["off"] = np.array([est.heff_offdiag_matvec(batch, cache, v) for v in vs])
    return d


def case_hermitian_connected(seed=23, n=6, h=4, N=40, per_row=5):
    """Complex-theta RBM completion through the real embedding [O, iO]."""
    d = _rbm_partner_case(seed, n, h, N, per_row, True)
    o, po = d["o"], d["partner_o"]
    batch = placeholder_batch(d["w"], np.zeros(N), np.concatenate([o, 1j * o], axis=1), N)
    cache = est.ConnectedCache(d["dist_index"], d["indptr"], d["partner_row"], d["coeff"],
                               np.concatenate([po, 1j * po], axis=1))
    vs = np.random.default_rng(seed + 1).standard_normal((4, 2 * o.shape[1]))
    d["vs"] = vs
    d["off"] = np.array([est.heff_offdiag_matvec(batch, cache, v) for v in vs])
    return d


def case_hamiltonian():
    """Local energies and connected configurations of the reference Hamiltonian
    path (ham:94-302) on a seeded synthetic FCIDUMP (5 spatial orbitals, 3 up +
    2 down) for the RBM (real, complex) and MLP log psi, plus H2 (its real
    FCIDUMP, T/data/h2_sto3g.fcidump)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from irlnqs.hamiltonian import build_dense_hamiltonian, connected_configurations, local_energy
    from irlnqs.hilbert import enumerate_sector
    from oracle import hamiltonian as oham
    from oracle import nqs

    text = oham.random_fcidump(31, 5, 5, ms2=1)
    ints = parse_fcidump(text)
    sector = ints.sector()
    configs = enumerate_sector(sector)
    bits = np.array([c.bits for c in configs], dtype=np.uint64)
    M = ints.n_spin_orbitals
    xocc = ((bits[:, None] >> np.arange(M, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.uint8)
    rng = np.random.default_rng(32)
    n, hr, hm = M, 6, 7
    th_rbm = rng.normal(0, 0.3, n + hr + hr * n)
    th_rbmc = rng.normal(0, 0.3, n + hr + hr * n) + 1j * rng.normal(0, 0.3, n + hr + hr * n)
    th_mlp = np.concatenate([rng.normal(0, np.sqrt(1 / n), hm * n + hm), rng.normal(0, np.sqrt(1 / hm), hm + 1)])
    occ_of = {int(b): xocc[k] for k, b in enumerate(bits)}

    def occ(x):
        b = x.bits
        return ((b >> np.arange(M)) & 1).astype(np.uint8)[None, :]

    lps = {
        "rbm": lambda x: nqs.rbm_log_psi(th_rbm, occ(x), n, hr)[0],
        "rbmc": lambda x: nqs.rbm_log_psi(th_rbmc, occ(x), n, hr)[0],
        "mlp": lambda x: nqs.mlp_log_psi(th_mlp, occ(x), n, hm)[0],
    }
    out = dict(fcidump=np.array(text), e_core=ints.e_core, h=ints.h, g=ints.g, ns=ints.n_spatial,
               n_up=sector.n_up, n_down=sector.n_down, bits=bits, theta_rbm=th_rbm, theta_rbmc=th_rbmc,
               theta_mlp=th_mlp, hidden_rbm=hr, hidden_mlp=hm,
               dense=build_dense_hamiltonian(ints, sector))
    for name, lp in lps.items():
        out[f"eloc_{name}"] = np.array([local_energy(lp, ints, x) for x in configs])
    pb, pe, ip = [], [], [0]
    for x in configs:
        ent = connected_configurations(ints, x)
        out.setdefault("diag", []).append(ent[0].element)
        pb += [e.config.bits for e in ent[1:]]
        pe += [e.element for e in ent[1:]]
        ip.append(len(pb))
    out["diag"] = np.array(out["diag"])
    out["partner_bits"] = np.array(pb, dtype=np.uint64)
    out["partner_elem"] = np.array(pe)
    out["partner_indptr"] = np.array(ip)
    # H2 from its own FCIDUMP
    with open(os.path.join(REF, "tests", "data", "h2_sto3g.fcidump")) as fh:
        h2 = parse_fcidump(fh.read())
    h2s = h2.sector()
    out["h2_e_core"] = h2.e_core
    out["h2_h"] = h2.h
    out["h2_g"] = h2.g
    out["h2_ns"] = h2.n_spatial
    out["h2_n_up"] = h2s.n_up
    out["h2_n_down"] = h2s.n_down
    out["h2_bits"] = np.array([c.bits for c in enumerate_sector(h2s)], dtype=np.uint64)
    out["h2_dense"] = build_dense_hamiltonian(h2, h2s)
    out["h2_fci"] = -1.1372930376796802  # T/test_optimizer.py:16
    return out


def case_outer_step(step=1):
    """The reference outer step (opt:118-195) assembled from reference
    primitives for the RBM on the synthetic FCIDUMP of case_hamiltonian:
    exact batch (local_energy, |psi|^2), est.energy_gradient, a ConnectedCache
    from connected_configurations (first-appearance o_row order, est:236-249),
    kry.irl_smallest on the full bordered operator with _batch_seed, the
    direction, and the line search by exact energy re-evaluation (opt:104-115)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from irlnqs.hamiltonian import connected_configurations, local_energy
    from irlnqs.hilbert import enumerate_sector
    from irlnqs.optimizer import OptimizerConfig, _batch_seed
    from oracle import hamiltonian as oham
    from oracle import nqs

    ints = parse_fcidump(oham.random_fcidump(31, 5, 5, ms2=1))
    sector = ints.sector()
    configs = enumerate_sector(sector)
    M, h = ints.n_spin_orbitals, 6
    theta = np.random.default_rng(33).normal(0, 0.3, M + h + h * M)

    def occ(b):
        return ((b >> np.arange(M)) & 1).astype(np.uint8)[None, :]

    def batch_at(th):
        lp = lambda x: nqs.rbm_log_psi(th, occ(x.bits), M, h)[0]  # noqa: E731
        lps = np.array([lp(x) for x in configs])
        w = np.exp(2 * (lps - lps.max()))
        w = w / w.sum()
        e = np.array([local_energy(lp, ints, x) for x in configs])
        xo = np.concatenate([occ(x.bits) for x in configs])
        o = rbm_rows_np(th, xo, M, h).astype(complex)
        return est.SampleBatch(configs=tuple(configs), weights=w, e_loc=e, o_matrix=o, n_samples=0), lp

    batch, lp = batch_at(theta)
    energy = est.estimate_energy(batch)
    grad = est.energy_gradient(batch, energy)
    o_rows, o_list, indptr, prow, coeff = {}, [], [0], [], []
    for x in configs:
        lx = lp(x)
        for ent in connected_configurations(ints, x)[1:]:
            b = ent.config.bits
            if b not in o_rows:
                o_rows[b] = len(o_list)
                o_list.append(rbm_rows_np(theta, occ(b), M, h)[0].astype(complex))
            prow.append(o_rows[b])
            coeff.append(ent.element * np.exp(lp(ent.config) - lx))
        indptr.append(len(prow))
    cache = est.ConnectedCache(np.arange(len(configs)), np.array(indptr), np.array(prow), np.array(coeff, dtype=complex),
                               np.array(o_list))
    config = OptimizerConfig()
    p = batch.param_count
    pair = kry.irl_smallest(bordered_connected(batch, energy, grad, cache), p + 1, m=config.m, tol=config.tol,
                            max_restarts=config.max_restarts, seed=_batch_seed(config, step))
    d = direction(pair.vector, grad)

    def energy_at(th):
        return est.estimate_energy(batch_at(th)[0]).mean

    scan = []

    def line_search(dd, best):
        best_scale, best_energy = best
        best_d = dd
        for scale in config.line_search:
            e_new = energy_at(theta + scale * dd)
            scan.append(e_new)
            if np.isfinite(e_new) and e_new < best_energy:
                best_energy, best_scale, best_d = e_new, scale, dd
        return best_scale, best_energy, best_d

    best_scale, best_energy, best_d = line_search(d, (0.0, energy.mean))
    if best_scale == 0.0:
        norm = float(np.linalg.norm(grad))
        if norm > 0.0:
            best_scale, best_energy, best_d = line_search(-grad / norm, (0.0, energy.mean))
    theta_new = theta + best_scale * best_d if best_scale > 0 else theta
    return dict(theta=theta, hidden=h, step=step, energy=energy.mean, grad=grad, lam=pair.value,
                n_matvec=pair.n_matvec, converged=pair.converged, direction=d, best_scale=best_scale,
                best_energy=best_energy, theta_new=theta_new, scan=np.array(scan))


def case_autoregressive():
    """The reference's own ansatz (ans:1-290) on H2 and on a seeded synthetic
    FCIDUMP (5 spatial orbitals, 3 up + 2 down): log amplitudes (in and out of
    the sector), log-derivative rows, exact samples, local energies, a
    stochastic build_batch, and the reference outer_step itself (opt:118-195)
    in exact and stochastic mode."""
    import warnings

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from irlnqs import optimizer as opt
    from irlnqs.hamiltonian import local_energy
    from irlnqs.hilbert import OccupationVector, enumerate_sector
    from paper_2601_01437_b200.synthetic import molecule_fcidump

    out = {}
    with open(os.path.join(REF, "tests", "data", "h2_sto3g.fcidump")) as fh:
        h2 = parse_fcidump(fh.read())
    syn = parse_fcidump(molecule_fcidump(31, 5, 5, ms2=1))
    for tag, ints, hidden, seed in (("h2", h2, 3, 9), ("syn", syn, 6, 5), ("wide", syn, 42, 7)):
        sector = ints.sector()
        arch = ans.Architecture(sector.n_orbitals, hidden)
        init = ans.init_parameters(arch, seed=seed)
        rng = np.random.default_rng(41)
        params = ans.AnsatzParameters(arch, init.theta + 0.1 * rng.standard_normal(arch.param_count))
        configs = enumerate_sector(sector)
        M = sector.n_orbitals
        bits = np.array([c.bits for c in configs], dtype=np.uint64)
        outside = np.array([3, (1 << M) - 1, 0], dtype=np.uint64)
        la = [ans.log_amplitude(params, OccupationVector(int(b), M), sector) for b in np.concatenate([bits, outside])]
        rows = np.array([ans.log_derivative(params, c, sector) for c in configs[:24]])
        samples = np.array([x.bits for x in ans.sample(params, sector, 64, seed=13)], dtype=np.uint64)
        lp = lambda x: ans.log_amplitude(params, x, sector).value  # noqa: E731
        eloc = np.array([local_energy(lp, ints, c) for c in configs[:40]])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            sb = est.build_batch(params, ints, sector, n_samples=64, seed=13)
        d = dict(theta=params.theta, hidden=hidden, n_up=sector.n_up, n_down=sector.n_down, M=M, bits=bits,
                 outside=outside, log_prob_half=np.array([a.log_prob_half for a in la]),
                 phase=np.array([a.phase for a in la]), rows=rows, samples=samples, eloc=eloc,
                 sb_e=np.array(sb.e_loc), sb_w=np.array(sb.weights), sb_o=np.array(sb.o_matrix),
                 sb_bits=np.array([x.bits for x in sb.configs], dtype=np.uint64),
                 e_core=ints.e_core, h=ints.h, g=ints.g, ns=ints.n_spatial)
        for mode, ns_ in ((("exact", 0),) if tag == "wide" else (("exact", 0), ("stoch", 64))):
            config = opt.OptimizerConfig(n_samples=ns_, max_restarts=300)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                new, lam, scale, matvecs, conv = opt.outer_step(params, ints, sector, config, 1)
            d.update({f"{mode}_theta_new": new.theta, f"{mode}_lam": lam, f"{mode}_scale": scale,
                      f"{mode}_matvecs": matvecs, f"{mode}_converged": conv})
        out.update({f"{tag}_{k}": v for k, v in d.items()})
    return out


def case_ar_edges():
    """The autoregressive ansatz on edge sectors (empty / full spin channels,
    ans:130-153 masking): log amplitudes, rows and exact samples."""
    from irlnqs.hilbert import Sector, enumerate_sector

    out = {}
    for tag, (m, nu, nd, hidden) in {"e1": (8, 0, 2, 5), "e2": (8, 4, 1, 5), "e3": (2, 1, 0, 3)}.items():
        sector = Sector(m, nu, nd)
        arch = ans.Architecture(m, hidden)
        rng = np.random.default_rng(len(tag) + m + nu)
        params = ans.AnsatzParameters(arch, ans.init_parameters(arch, seed=3).theta
                                      + 0.2 * rng.standard_normal(arch.param_count))
        configs = enumerate_sector(sector)
        la = [ans.log_amplitude(params, c, sector) for c in configs]
        out.update({f"{tag}_theta": params.theta, f"{tag}_shape": np.array([m, nu, nd, hidden]),
                    f"{tag}_bits": np.array([c.bits for c in configs], dtype=np.uint64),
                    f"{tag}_lp": np.array([a.log_prob_half for a in la]), f"{tag}_ph": np.array([a.phase for a in la]),
                    f"{tag}_rows": np.array([ans.log_derivative(params, c, sector) for c in configs]),
                    f"{tag}_samples": np.array([x.bits for x in ans.sample(params, sector, 32, seed=5)],
                                               dtype=np.uint64)})
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    only = set(sys.argv[1:])
    cases = {
        "real_rbm": case_real,
        "complex_raw": case_complex_raw,
        "hermitian_rbm": case_hermitian,
        "h2_exact": case_h2,
        "mlp_phase_head": case_mlp_phase_head,
        "krylov": case_krylov,
        "h2_connected": case_h2_connected,
        "rbm_connected": case_rbm_connected,
        "hermitian_connected": case_hermitian_connected,
        "hamiltonian": case_hamiltonian,
        "outer_step": case_outer_step,
        "autoregressive": case_autoregressive,
        "ar_edges": case_ar_edges,
    }
    for name, data in cases.items():
        if only and name not in only:
            continue
        data = data()
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
