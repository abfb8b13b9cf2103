"""ctypes binding of the in-tree C-ABI library ``libirlsr.so`` (include/irl_sr.h).

This is the reference-side binding a maintainer would add to ``irlnqs``
(INTEGRATION.md): plain pointers, sizes and a ``cudaStream_t``; no torch types
cross the boundary.  There is no CPU fallback: if the library or a CUDA device
is missing, every entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IRL_LIB_PATH") or os.path.join(_HERE, "libirlsr.so")  # override: A/B builds

IRL_OK = 0
IRL_ERR_ARG = 1
IRL_ERR_ALIGN = 2
IRL_ERR_WORKSPACE = 3
IRL_ERR_CUDA = 4
IRL_ERR_DEVICE = 5

MVP_AUTO = 0
MVP_FUSED = 1
MVP_TWO_PASS = 2
MVP_ROWS = 3
MVP_WIDE = 4

MODEL_RBM = 0
MODEL_MLP = 1

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_SZ = ctypes.c_size_t
_D = ctypes.c_double

# name -> (restype, argtypes); every symbol declared in include/irl_sr.h
SIGNATURES = {
    "irl_version": (_I, []),
    "irl_last_error": (ctypes.c_char_p, []),
    "irl_debug_wide_trace": (_SZ, [_P, _SZ]),
    "irl_padded_ld": (_I64, [_I64, _I]),
    "irl_energy_f64": (_I, [_P, _P, _I64, _P, _P, _P]),
    "irl_energy_c128": (_I, [_P, _P, _I64, _I, _P, _P, _P]),
    "irl_colstats_workspace_bytes": (_SZ, [_I64, _I64, _I]),
    "irl_colstats_f64": (_I, [_P, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_colstats_c128": (_I, [_P, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_obuild_workspace_bytes": (_SZ, [_I, _I64, _I, _I, _I64, _I]),
    "irl_obuild_rbm_f64": (_I, [_P, _I64, _I, _I, _P, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_obuild_rbm_c128": (_I, [_P, _I64, _I, _I, _P, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_obuild_mlp_f64": (_I, [_P, _I64, _I, _I, _P, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_hidden_rbm_f64": (_I, [_P, _I64, _I, _I, _P, _P, _P]),
    "irl_hidden_rbm_c128": (_I, [_P, _I64, _I, _I, _P, _P, _P]),
    "irl_hidden_mlp_f64": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P]),
    "irl_mvp_workspace_bytes": (_SZ, [_I64, _I64, _I]),
    "irl_mvp_f64": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _I, _P, _SZ, _P]),
    "irl_mvp_c128": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _SZ, _P]),
    "irl_mvp2_workspace_bytes": (_SZ, [_I64, _I64, _I]),
    "irl_mvp2_f64": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_mvp2_c128": (_I, [_P, _I64, _I64, _I64] + [_P] * 14 + [_SZ, _P]),
    "irl_mvp_plan": (_I, [_I64, _I64, _I, _I, _P, _P]),
    "irl_lanczos_step_small": (_I, [_P, _I64, _P, _I64, _I, _I, _P, _P]),
    "irl_lanczos_step_cluster": (_I, [_P, _I64, _P, _I64, _I, _I, _P, _P]),
    "irl_host_qr_sweeps": (_I, [_I, _P, _P, _P, _I]),
    "irl_otf_workspace_bytes": (_SZ, [_I64, _I, _I]),
    "irl_otf_prepare_mlp_f64": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P, _P]),
    "irl_otf_colstats_mlp_f64": (_I, [_P, _P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_otf_mvp_mlp_f64": (_I, [_P, _P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_otf_mvp_mlp_u_f64": (_I, [_P, _P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_otf_prepare_rbm_f64": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P]),
    "irl_otf_colstats_rbm_f64": (_I, [_P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_otf_mvp_rbm_f64": (_I, [_P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_otf_workspace_bytes_c128": (_SZ, [_I64, _I, _I]),
    "irl_otf_prepare_rbm_c128": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P]),
    "irl_otf_colstats_rbm_c128": (_I, [_P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_otf_mvp_rbm_c128": (_I, [_P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_connected_workspace_bytes": (_SZ, [_I64, _I64, _I64, _I]),
    "irl_connected_mvp_f64": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P,
                                   _I, _P, _SZ, _P]),
    "irl_connected_mvp_c128": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P,
                                    _P, _P, _P, _I, _P, _SZ, _P]),
    "irl_logamp_workspace_bytes": (_SZ, [_I64, _I, _I]),
    "irl_logamp_rbm_f64": (_I, [_P, _I64, _I, _I, _P, _P, _P, _SZ, _P]),
    "irl_logamp_rbm_c128": (_I, [_P, _I64, _I, _I, _P, _P, _P, _SZ, _P]),
    "irl_logamp_mlp_f64": (_I, [_P, _I64, _I, _I, _P, _P, _P, _SZ, _P]),
    "irl_ham_workspace_bytes": (_SZ, [_I, _I, _I]),
    "irl_ham_local_energy": (_I, [_I, _I, _P, _I64, _I, _D, _P, _P, _D, _I, _P, _P, _P, _SZ, _P]),
    "irl_ham_connected_count": (_I, [_I, _I, _P, _I64, _I, _D, _P, _P, _D, _I, _P, _P, _P, _SZ, _P]),
    "irl_ham_connected_fill": (_I, [_I, _I, _P, _I64, _I, _D, _P, _P, _D, _I, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_ar_logamp": (_I, [_P, _I64, _I, _I, _I, _I, _P, _P, _P, _P]),
    "irl_ar_rows": (_I, [_P, _I64, _I, _I, _I, _I, _P, _P, _I64, _P, _P]),
    "irl_ar_sample": (_I, [_P, _I64, _I, _I, _I, _I, _P, _P, _P, _P]),
    "irl_ham_diagonal_and_count": (_I, [_P, _I64, _I, _D, _P, _P, _D, _P, _P, _P]),
    "irl_ham_partners_fill": (_I, [_P, _I64, _I, _D, _P, _P, _D, _P, _P, _P, _P]),
    "irl_eloc_combine": (_I, [_P, _P, _P, _P, _P, _I64, _P, _P]),
    "irl_sorted_lookup": (_I, [_P, _I64, _P, _I64, _P, _P]),
    "irl_otf_connected_workspace_bytes": (_SZ, [_I, _I64, _I64, _I, _I, _I64, _I]),
    "irl_otf_connected_mvp_rbm_f64": (_I, [_P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                           _I64, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_otf_connected_mvp_mlp_f64": (_I, [_P, _P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                           _P, _I64, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "irl_otf_connected_mvp_rbm_c128": (_I, [_P, _P, _I64, _I, _I, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P,
                                            _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
}


class NativeUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is missing (no CPU fallback exists)."""


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, name: str, code: int, text: str):
        super().__init__(f"{name} failed with code {code}: {text}")
        self.code = code


_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the library and bind every declared symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `make` or __graft_entry__.build()"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("IRL_LIB_PATH") and not hasattr(lib, name):
                continue  # an older A/B build lacks newer entry points
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the IRL-SR hot path runs only on sm_100a")
    return load()


def check(name: str, code: int) -> None:
    if code != IRL_OK:
        text = load().irl_last_error().decode(errors="replace")
        raise NativeError(name, code, text)


def call(name: str, *args) -> None:
    check(name, getattr(lib(), name)(*args))


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes through as NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def padded_ld(p: int, is_complex: bool) -> int:
    return int(load().irl_padded_ld(int(p), 1 if is_complex else 0))


def mvp_plan(n: int, ld: int, is_complex: bool, mode: int = MVP_AUTO) -> dict:
    path = ctypes.c_int(0)
    geom = (ctypes.c_int * 7)()
    code = lib().irl_mvp_plan(int(n), int(ld), int(is_complex), int(mode), ctypes.byref(path), geom)
    check("irl_mvp_plan", code)
    keys = ("cluster", "units_per_slice", "threads", "rows_per_stage", "stages", "row_blocks", "units_per_thread")
    out = dict(zip(keys, list(geom)))
    out["path"] = {MVP_FUSED: "fused", MVP_TWO_PASS: "two_pass", MVP_ROWS: "rows", MVP_WIDE: "wide"}[path.value]
    return out
