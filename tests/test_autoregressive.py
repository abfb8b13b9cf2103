"""The reference's own autoregressive NQS on the device.

Golden vectors come from the reference itself (tests/golden/autoregressive.npz,
oracle/make_golden.py::case_autoregressive): log amplitudes in and out of the
sector (ans:229-247), log-derivative rows (ans:249-290), exact samples
(ans:215-236, bit for bit), local energies (ham:290-302), a stochastic
build_batch (est:79-133) and the reference's outer_step (opt:118-195) in exact
and stochastic mode, on H2 and on a seeded synthetic FCIDUMP.
"""

import numpy as np
import pytest

from conftest import golden

TAGS = ["h2", "syn", "wide"]  # wide: hidden 42 (two hidden units per lane, run_optimization's default)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def case(tag):
    g = golden("autoregressive")
    return {k[len(tag) + 1:]: v for k, v in g.items() if k.startswith(tag + "_")}


def objects(d):
    from paper_2601_01437_b200 import autoregressive as AR, hamiltonian as H

    M, h = int(d["M"]), int(d["hidden"])
    params = AR.AnsatzParameters(AR.Architecture(M, h), d["theta"])
    sector = H.Sector(M, int(d["n_up"]), int(d["n_down"]))
    n_up, n_dn = int(d["n_up"]), int(d["n_down"])
    ints = H.MolecularIntegrals(int(d["ns"]), n_up + n_dn, n_up - n_dn, float(d["e_core"]), d["h"], d["g"])
    return params, sector, ints


# ------------------------------------------------------------------- CPU --
@pytest.mark.parametrize("tag,seed", [("h2", 9), ("syn", 5), ("wide", 7)])
def test_init_parameters_matches_reference(tag, seed):
    from paper_2601_01437_b200 import autoregressive as AR

    d = case(tag)
    arch = AR.Architecture(int(d["M"]), int(d["hidden"]))
    theta = AR.init_parameters(arch, seed=seed).theta + 0.1 * np.random.default_rng(41).standard_normal(
        arch.param_count)
    assert np.array_equal(theta, d["theta"])


def test_pcg64_replay_matches_numpy():
    """The sampler's generator (csrc/autoreg.cuh Pcg64) restated on the host:
    step then XSL-RR, next_double = (x >> 11) 2^-53, as numpy's PCG64."""
    mult = 0x2360ED051FC65DA44385DF649FCCF645
    mask = (1 << 128) - 1
    for stream in np.random.SeedSequence(13).spawn(4):
        gen = np.random.default_rng(stream)
        st = gen.bit_generator.state["state"]
        state, inc = st["state"], st["inc"]
        want = gen.random(8)
        got = []
        for _ in range(8):
            state = (state * mult + inc) & mask
            x = (state >> 64) ^ (state & ((1 << 64) - 1))
            rot = state >> 122
            out = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
            got.append((out >> 11) * (1.0 / 9007199254740992.0))
        assert np.array_equal(np.array(got), want)


# ------------------------------------------------------------------- GPU --


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_log_amplitude_and_rows_golden(cuda, tag):
    from paper_2601_01437_b200 import autoregressive as AR

    d = case(tag)
    params, sector, _ = objects(d)
    allbits = np.concatenate([d["bits"], d["outside"]])
    lp = AR.log_amplitude_batch(params, sector, allbits).cpu().numpy()
    n_in = len(d["bits"])
    assert np.all(np.isneginf(lp.real[n_in:])) and np.all(lp.imag[n_in:] == 0.0)
    assert np.max(np.abs(lp.real[:n_in] - d["log_prob_half"][:n_in])) < 1e-12
    assert np.max(np.abs(lp.imag[:n_in] - d["phase"][:n_in])) < 1e-12
    rows = AR.log_derivative_batch(params, sector, d["bits"][:24]).cpu().numpy()
    P = params.architecture.param_count
    assert np.max(np.abs(rows[:, :P] - d["rows"])) < 1e-12
    assert np.all(rows[:, P:] == 0)
    with pytest.raises(ValueError):
        AR.log_derivative_batch(params, sector, d["outside"][:1])


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_samples_are_bit_identical(cuda, tag):
    from paper_2601_01437_b200 import autoregressive as AR

    d = case(tag)
    params, sector, _ = objects(d)
    assert np.array_equal(AR.sample(params, sector, 64, seed=13), d["samples"])


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_local_energies_and_stochastic_batch(cuda, tag):
    import warnings

    from paper_2601_01437_b200 import autoregressive as AR

    d = case(tag)
    params, sector, ints = objects(d)
    e = AR.local_energies(params, ints, sector, d["bits"][:40]).cpu().numpy()
    assert np.max(np.abs(e - d["eloc"]) / np.maximum(1.0, np.abs(d["eloc"]))) < 1e-10
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        b = AR.build_batch(params, ints, sector, n_samples=64, seed=13)
    assert np.array_equal(b.xbits, d["sb_bits"])
    P = params.architecture.param_count
    assert rel(b.e_loc.cpu().numpy(), d["sb_e"]) < 1e-10
    assert np.array_equal(b.weights.cpu().numpy(), d["sb_w"])
    assert np.max(np.abs(b.o_matrix[:, :P].cpu().numpy() - d["sb_o"])) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_reference_outer_step_exact(cuda, tag):
    """opt:118-195 with the reference's own model, exact enumeration."""
    import warnings

    from paper_2601_01437_b200 import optimizer as OPT

    d = case(tag)
    params, sector, ints = objects(d)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = OPT.outer_step(params, ints, sector, OPT.OptimizerConfig(), 1)
    assert res.matvecs == int(d["exact_matvecs"])
    assert abs(res.lambda_min - float(d["exact_lam"])) <= 1e-10 * abs(float(d["exact_lam"]))
    assert res.step_scale == float(d["exact_scale"])
    assert rel(res.params.theta, d["exact_theta_new"]) < 1e-8


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["h2", "syn"])
def test_reference_outer_step_stochastic(cuda, tag):
    """opt:118-195 with exact samples (n_samples=64): same samples, same batch;
    the long restart sequence (hundreds of restarts) is compared on the Ritz
    value and the accepted step."""
    import warnings

    from paper_2601_01437_b200 import optimizer as OPT

    d = case(tag)
    params, sector, ints = objects(d)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = OPT.outer_step(params, ints, sector, OPT.OptimizerConfig(n_samples=64), 1)
    assert abs(res.lambda_min - float(d["stoch_lam"])) <= 1e-8 * abs(float(d["stoch_lam"]))
    assert res.step_scale == float(d["stoch_scale"])
    assert rel(res.params.theta, d["stoch_theta_new"]) < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["e1", "e2", "e3"])
def test_edge_sectors_golden(cuda, tag):
    """Empty and full spin channels (the masking of ans:130-153): log
    amplitudes, rows and exact samples against the reference."""
    from paper_2601_01437_b200 import autoregressive as AR, hamiltonian as H

    g = golden("ar_edges")
    m, nu, nd, hidden = (int(v) for v in g[f"{tag}_shape"])
    params = AR.AnsatzParameters(AR.Architecture(m, hidden), g[f"{tag}_theta"])
    sector = H.Sector(m, nu, nd)
    lp = AR.log_amplitude_batch(params, sector, g[f"{tag}_bits"]).cpu().numpy()
    assert np.max(np.abs(lp.real - g[f"{tag}_lp"])) < 1e-12
    assert np.max(np.abs(lp.imag - g[f"{tag}_ph"])) < 1e-12
    rows = AR.log_derivative_batch(params, sector, g[f"{tag}_bits"]).cpu().numpy()
    assert np.max(np.abs(rows[:, : params.architecture.param_count] - g[f"{tag}_rows"])) < 1e-12
    assert np.array_equal(AR.sample(params, sector, 32, seed=5), g[f"{tag}_samples"])
