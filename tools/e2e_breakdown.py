"""Where the end-to-end (pinned host vector -> product -> host) time goes on cfg2.

Times, per call, the public API (estimators.heff_matvec on a pinned host
tensor), the raw device product (_apply), and the host-side pieces of
_product in isolation.  Development tool; prints one JSON line.
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S  # noqa: E402


def timed(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = S.CONFIGS[idx]
    inp = S.make_inputs(cfg)
    arch = (A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm"
            else A.MLPArchitecture(cfg.n_inputs, cfg.hidden))
    params = A.AnsatzParameters(arch, inp.theta)
    b = A.build_batch(params, inp.x, inp.e_loc)
    en = E.estimate_energy(b)
    P, ld = b.param_count, b.ld
    vh = torch.randn(P, dtype=torch.float64).pin_memory()
    vd = torch.zeros(ld, dtype=torch.float64, device="cuda")
    vd[:P] = vh.cuda()
    od = torch.empty(ld, dtype=torch.float64, device="cuda")
    coeff = b.coefficients(en.mean)
    out = {
        "cfg": idx,
        "api_us": timed(lambda: E.heff_matvec(b, en, vh)),
        "apply_sync_us": timed(lambda: (E._apply(b, coeff, vd, od), torch.cuda.synchronize())),
        "apply_async_us": timed(lambda: E._apply(b, coeff, vd, od)),
        "isfinite_us": timed(lambda: bool(torch.isfinite(vh).all())),
        "zeros_h2d_us": timed(lambda: torch.zeros(ld, dtype=torch.float64, device="cuda")[:P].copy_(vh, non_blocking=True)),
        "d2h_pinned_us": timed(lambda: torch.empty(P, dtype=torch.float64, pin_memory=True).copy_(od[:P], non_blocking=True)),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
