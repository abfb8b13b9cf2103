"""The C-ABI library loads and exports every symbol include/irl_sr.h declares (no GPU needed)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2601_01437_b200 import _lib


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "irl_sr.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(irl_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.SIGNATURES)


def test_library_loads_and_exports_everything():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.irl_version() >= 100


@pytest.mark.parametrize(
    "p,cplx,ld",
    [(860, False, 864), (6600, False, 6624), (11265, False, 11296), (29340, True, 29344), (208897, False, 209024),
     (1, False, 32), (1, True, 16)],
)
def test_padded_ld(p, cplx, ld):
    assert _lib.padded_ld(p, cplx) == ld
    assert ld >= p and (ld * (16 if cplx else 8)) % 256 == 0


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_01437_b200 import estimators

    with pytest.raises(_lib.NativeUnavailable):
        estimators.SampleBatch(None, np.full(4, 0.25), np.zeros(4), np.zeros((4, 3)), 4)
    with pytest.raises(_lib.NativeUnavailable):
        _lib.lib()


def test_errors_without_device_are_codes_not_crashes():
    # argument validation happens before any CUDA call
    lib = _lib.load()
    rc = lib.irl_energy_f64(None, None, 0, None, None, None)
    assert rc == _lib.IRL_ERR_ARG
    assert b"bad energy" in lib.irl_last_error()


def test_otf_support_rule():
    """Which architectures the on-the-fly kernels take (ansatz.otf_supported)."""
    from paper_2601_01437_b200 import ansatz as A

    assert A.otf_supported(A.RBMArchitecture(40, 160))
    assert A.otf_supported(A.RBMArchitecture(60, 481, complex_params=True))
    assert not A.otf_supported(A.RBMArchitecture(40, 161))
    assert not A.otf_supported(A.MLPArchitecture(101, 64))
    assert A.otf_supported(A.MLPArchitecture(100, 2048))


def test_new_entry_points_validate_before_any_cuda_call():
    """Connected completion, local energies and the autoregressive ansatz
    return IRL_ERR_ARG for bad arguments without touching a device."""
    lib = _lib.load()
    # connected product: null batch pointers
    rc = lib.irl_connected_mvp_f64(None, 4, 3, 32, None, None, None, None, None, None, None, None, 0, None, None,
                                   None, None, None, 0, None, 0, None)
    assert rc == _lib.IRL_ERR_ARG
    # local energy: unknown model
    rc = lib.irl_ham_local_energy(7, 0, None, 1, 2, 0.0, None, None, 1e-14, 3, None, None, None, 0, None)
    assert rc == _lib.IRL_ERR_ARG
    # autoregressive ansatz: odd orbital count
    rc = lib.irl_ar_logamp(None, 1, 5, 3, 1, 1, None, None, None, None)
    assert rc == _lib.IRL_ERR_ARG
    assert b"autoregressive" in lib.irl_last_error()
    # sorted lookup: negative sizes
    assert lib.irl_sorted_lookup(None, -1, None, 0, None, None) == _lib.IRL_ERR_ARG
