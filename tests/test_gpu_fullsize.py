"""Full BASELINE-size parity: the device products (stored O streamed from HBM,
and O regenerated on the fly) against the CPU restatement at the full N_s x P of
cfg2-cfg5 (oracle/structured.py, itself pinned to the row-based restatement of
est:171-186 in test_oracle_golden.py).  Tolerance: products rel-L2 <= 1e-10."""

import gc

import numpy as np
import pytest

from oracle.structured import MLPProducts, RBMProducts

pytestmark = pytest.mark.gpu

PROD_TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


@pytest.mark.parametrize("idx", [2, 3, 4, 5])
def test_full_size_products(cuda, idx):
    import torch
    from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S

    cfg = S.CONFIGS[idx]
    inp = S.make_inputs(cfg)
    n, h, N = cfg.n_inputs, cfg.hidden, cfg.n_rows
    arch = (A.RBMArchitecture(n, h, cfg.complex_params) if cfg.model == "rbm" else A.MLPArchitecture(n, h))
    params = A.AnsatzParameters(arch, inp.theta)
    w = np.full(N, 1.0 / N)
    oracle = (RBMProducts if cfg.model == "rbm" else MLPProducts)(inp.theta, inp.x, n, h, w)
    P = oracle.p
    rng = np.random.default_rng(100 + idx)
    v = rng.standard_normal(P) + (1j * rng.standard_normal(P) if cfg.complex_params else 0.0)
    results = {}
    for mode in ("stored", "otf"):
        b = A.build_batch(params, inp.x, inp.e_loc, mode=mode)
        assert (b.otf is not None) == (mode == "otf")
        en = E.estimate_energy(b)
        results[mode] = (en.mean, E.heff_matvec(b, en, v), E.qgt_matvec(b, v))
        del b
        gc.collect()
        torch.cuda.empty_cache()
    mean = results["stored"][0]
    assert results["otf"][0] == mean
    coeff = w * (inp.e_loc - mean)
    if cfg.complex_params:
        coeff = coeff.real  # Hermitian products use w Re(e - E)
    ref_h = oracle.product(coeff, v)
    ref_s = oracle.product(w, v)
    for mode, (_, hv, sv) in results.items():
        assert rel(hv, ref_h) < PROD_TOL, (idx, mode, "heff")
        assert rel(sv, ref_s) < PROD_TOL, (idx, mode, "S")
