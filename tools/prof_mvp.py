"""One product on a BASELINE config through a chosen MVP path, for ncu captures (development tool)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--mode", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
cfg = S.CONFIGS[args.config]
inp = S.make_inputs(cfg)
arch = (A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm"
        else A.MLPArchitecture(cfg.n_inputs, cfg.hidden))
b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc, mode="stored")
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
E._apply(b, c, vi, vo, mode=args.mode)  # plans, attributes, first-touch
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.reps):
    E._apply(b, c, vi, vo, mode=args.mode)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
