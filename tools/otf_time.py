#!/usr/bin/env python
"""Development tool: device time of the on-the-fly product on BASELINE configs
(L2 write flush before every product).  usage: otf_time.py <cfgs>   (IRL_OTF_FORM_G=0/1 picks the MLP form)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S  # noqa: E402

l2buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for idx in [int(c) for c in sys.argv[1].split(",")]:
    cfg = S.CONFIGS[idx]
    inp = S.make_inputs(cfg)
    b = A.build_batch(A.AnsatzParameters(bench._arch(A, cfg), inp.theta), inp.x, inp.e_loc, mode="otf")
    en = E.estimate_energy(b)
    co = b.coefficients(en.mean)
    b.obar()
    apply = bench._vectors(torch, b, "cuda", 2, 5)
    ms = bench.graph_timed(torch, lambda: apply(0, co, 0), l2buf, k=10)
    print(f"cfg{idx} otf form_g={os.environ.get('IRL_OTF_FORM_G', '1')}: {ms:.4f} ms", flush=True)
    del b, apply
    torch.cuda.empty_cache()
