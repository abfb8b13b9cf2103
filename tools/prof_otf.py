#!/usr/bin/env python
"""Development tool: a few on-the-fly products of a BASELINE config, for ncu.
usage: prof_otf.py <cfg> [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S  # noqa: E402

idx = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = S.CONFIGS[idx]
inp = S.make_inputs(cfg)
b = A.build_batch(A.AnsatzParameters(bench._arch(A, cfg), inp.theta), inp.x, inp.e_loc, mode="otf")
en = E.estimate_energy(b)
co = b.coefficients(en.mean)
b.obar()
apply = bench._vectors(torch, b, "cuda", 2, 5)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for k in range(reps):
    apply(k % 2, co, 0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
