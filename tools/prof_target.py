#!/usr/bin/env python
"""Small fixed workload for ncu captures: build one config, run a few products."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--otf", type=int, default=0)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--rows", type=int, default=0)
args = ap.parse_args()
cfg = S.CONFIGS[args.config]
if args.rows:
    cfg = cfg.with_rows(args.rows)
inp = S.make_inputs(cfg)
arch = (A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm"
        else A.MLPArchitecture(cfg.n_inputs, cfg.hidden))
params = A.AnsatzParameters(arch, inp.theta)
b = A.build_batch_otf(params, inp.x, inp.e_loc) if args.otf else A.build_batch(params, inp.x, inp.e_loc)
en = E.estimate_energy(b)
c = b.coefficients(en.mean)
P, ld = b.param_count, b.ld
if b.kind == E.KIND_HERMITIAN:
    vin = torch.randn((2, ld), dtype=torch.float64, device="cuda")
    vin[:, P:] = 0
    vout = torch.empty_like(vin)
    vi, vo = (vin[0], vin[1]), (vout[0], vout[1])
else:
    vi = torch.randn(ld, dtype=torch.float64, device="cuda")
    vi[P:] = 0
    vo = torch.empty_like(vi)
for _ in range(args.reps):
    E._apply(b, c, vi, vo, mode=args.mode)
torch.cuda.synchronize()
print("ok", cfg.name, float(vo[:4].sum()))
