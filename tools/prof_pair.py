#!/usr/bin/env python
"""Development tool: a few one-read pair products (irl_mvp2_*) on a BASELINE
config, for ncu.  usage: prof_pair.py <cfg> [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S  # noqa: E402

idx = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = S.CONFIGS[idx]
inp = S.make_inputs(cfg)
arch = bench._arch(A, cfg)
b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc, mode="stored")
en = E.estimate_energy(b)
v = torch.randn(arch.param_count, dtype=torch.float64, device="cuda")
for _ in range(reps):
    E.heff_qgt_matvec(b, en, v)
    E.heff_matvec(b, en, v)
torch.cuda.synchronize()
print("done")
