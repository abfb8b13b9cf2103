"""Outer-step wall time with the reference's own autoregressive ansatz.

Runs ``optimizer.outer_step`` (opt:118-195: batch, energy, gradient,
connected cache, bordered IRL with heff + offdiag, direction, line search) on
the device for H2 (if its FCIDUMP is given) and for a seeded synthetic
molecule, exact enumeration and stochastic batches, and prints one JSON line
per case.  ``--reference`` times the reference's own ``outer_step`` on the
host instead (only where /root/reference exists: this build container).
"""

import argparse
import json
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

CASES = {
    # name: (ns, n_elec, ms2, hidden, n_samples); hidden 42 is run_optimization's default (opt:201)
    "syn6-exact": (6, 6, 0, 42, 0),        # 400 configurations
    "syn6-stoch": (6, 6, 0, 42, 1024),
    "syn10-exact": (10, 10, 0, 42, 0),     # 63504 configurations (device only)
}


def run_ours(name, steps):
    import torch

    from paper_2601_01437_b200 import autoregressive as AR, hamiltonian as H, optimizer as OPT, synthetic as S

    ns, ne, ms2, hidden, nsamp = CASES[name]
    ints = H.parse_fcidump(S.molecule_fcidump(51, ns, ne, ms2=ms2, scale=0.05))
    sector = ints.sector()
    params = AR.init_parameters(AR.Architecture(sector.n_orbitals, hidden), seed=111)
    cfg = OPT.OptimizerConfig(n_samples=nsamp)
    times, rec = [], []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        OPT.outer_step(params, ints, sector, cfg, 1)  # warm
        for step in range(1, steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = OPT.outer_step(params, ints, sector, cfg, step)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            rec.append((res.lambda_min, res.step_scale, res.matvecs))
            params = res.params
    return {"case": name, "impl": "ours", "sector_size": sector.size, "param_count": params.architecture.param_count,
            "n_samples": nsamp, "steps": steps, "outer_step_ms": [t * 1e3 for t in times],
            "median_ms": float(np.median(times) * 1e3), "lambda_scale_matvecs": rec}


def run_reference(name, steps):
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.dont_write_bytecode = True
    from irlnqs import ansatz as ans, optimizer as opt
    from irlnqs.hamiltonian import parse_fcidump

    from paper_2601_01437_b200 import synthetic as S

    ns, ne, ms2, hidden, nsamp = CASES[name]
    ints = parse_fcidump(S.molecule_fcidump(51, ns, ne, ms2=ms2, scale=0.05))
    sector = ints.sector()
    params = ans.init_parameters(ans.Architecture(sector.n_orbitals, hidden), seed=111)
    cfg = opt.OptimizerConfig(n_samples=nsamp)
    times, rec = [], []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for step in range(1, steps + 1):
            t0 = time.perf_counter()
            params, lam, scale, mv, _ = opt.outer_step(params, ints, sector, cfg, step)
            times.append(time.perf_counter() - t0)
            rec.append((lam, scale, mv))
    return {"case": name, "impl": "reference", "cores": len(os.sched_getaffinity(0)), "sector_size": sector.size,
            "n_samples": nsamp, "steps": steps, "outer_step_ms": [t * 1e3 for t in times],
            "median_ms": float(np.median(times) * 1e3), "lambda_scale_matvecs": rec}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--reference", action="store_true")
    args = ap.parse_args()
    for name in args.cases.split(","):
        fn = run_reference if args.reference else run_ours
        print(json.dumps(fn(name, args.steps)), flush=True)


if __name__ == "__main__":
    main()
