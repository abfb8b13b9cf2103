#!/usr/bin/env python
"""Development tool: device time of the stored product on a chosen path
(MVP_MODE, default 0 = AUTO) on full BASELINE configs under several environment
settings, in one process (the launch reads its environment every time).
usage: mvp_time.py <cfgs, e.g. 2,3> <setting> [<setting> ...]   setting = "VAR=val,VAR=val" or "-" """
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

MODE = int(os.environ.get("MVP_MODE", "0"))
from paper_2601_01437_b200 import _lib, ansatz as A, estimators as E, synthetic as S  # noqa: E402

l2buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for idx in [int(c) for c in sys.argv[1].split(",")]:
    cfg = S.CONFIGS[idx]
    inp = S.make_inputs(cfg)
    arch = bench._arch(A, cfg)
    b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc, mode="stored")
    en = E.estimate_energy(b)
    co = b.coefficients(en.mean)
    b.obar()
    apply = bench._vectors(torch, b, "cuda", 2, 5)
    for setting in sys.argv[2:]:
        keys = []
        if setting != "-":
            for kv in setting.split(","):
                k, v = kv.split("=")
                os.environ[k] = v
                keys.append(k)
        try:
            plan = _lib.mvp_plan(b.n_rows, b.ld, b.is_complex, MODE)
            ms = bench.graph_timed(torch, lambda: apply(0, co, 0, mode=MODE), l2buf, k=3)
            print(f"cfg{idx} {setting:30s} {ms:8.3f} ms  {plan}", flush=True)
        except Exception as exc:  # noqa: BLE001
            print(f"cfg{idx} {setting:30s} error {str(exc)[:120]}", flush=True)
        for k in keys:
            del os.environ[k]
    del b, apply, co
    torch.cuda.empty_cache()
