#!/usr/bin/env python
"""Development tool: device time of H_eff v + S v as two products against the
one-read pair (irl_mvp2_*) on BASELINE configs.  usage: pair_time.py <cfgs>"""
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
    arch = bench._arch(A, cfg)
    b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc, mode="stored")
    en = E.estimate_energy(b)
    ch, cs = b.coefficients(en.mean), E._qgt_coeff(b)
    b.obar()
    ld = b.ld
    herm = b.kind == E.KIND_HERMITIAN
    shape = (2, ld) if herm else (ld,)
    v = torch.zeros(shape, dtype=torch.float64, device="cuda")
    v[..., : b.param_count] = torch.randn(shape[:-1] + (b.param_count,), dtype=torch.float64, device="cuda")
    oa, ob = torch.empty_like(v), torch.empty_like(v)
    parts = (lambda t: (t[0], t[1])) if herm else (lambda t: t)

    def two():
        E._apply(b, ch, parts(v), parts(oa))
        E._apply(b, cs, parts(v), parts(ob))

    def pair():
        E._apply2(b, ch, cs, parts(v), parts(oa), parts(ob))

    t2 = bench.graph_timed(torch, two, l2buf, k=3)
    tp = bench.graph_timed(torch, pair, l2buf, k=3)
    print(f"cfg{idx}: two products {t2:.4f} ms, one-read pair {tp:.4f} ms ({t2 / tp:.2f}x)", flush=True)
    del b, v, oa, ob
    torch.cuda.empty_cache()
