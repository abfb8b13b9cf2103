"""One warm O-build (K1/K2 + statistics) on a BASELINE config, for ncu launch lists (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_01437_b200 import ansatz as A, synthetic as S  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = S.CONFIGS[idx]
inp = S.make_inputs(cfg)
arch = (A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm"
        else A.MLPArchitecture(cfg.n_inputs, cfg.hidden))
params = A.AnsatzParameters(arch, inp.theta)
b = A.build_batch(params, inp.x, inp.e_loc, mode="stored")
xt = A._x_device(inp.x, arch.n_inputs, b.device)
mean = b._stats_e
obar, g = b.colstats(mean)
gc = b.gradient_coefficients(mean)
for _ in range(2):
    A.fill_o_rows(params, xt, b.o_padded, b.weights, gc, obar, g)
torch.cuda.synchronize()
