#!/usr/bin/env python
"""Development tool: a few single-read wide products (IRL_MVP_WIDE) on a row
subset of a BASELINE config, for ncu.  usage: prof_wide.py <cfg> <rows> [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S  # noqa: E402

idx, rows = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = S.CONFIGS[idx].with_rows(rows)
inp = S.make_inputs(cfg)
arch = (A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm"
        else A.MLPArchitecture(cfg.n_inputs, cfg.hidden))
b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc, mode="stored")
en = E.estimate_energy(b)
rng = np.random.default_rng(1)
v = rng.standard_normal(arch.param_count) + (1j * rng.standard_normal(arch.param_count) if cfg.complex_params else 0)
v = torch.as_tensor(v, device="cuda")
for _ in range(reps):
    E.heff_matvec(b, en, v, mode=4)
torch.cuda.synchronize()
print("done")
