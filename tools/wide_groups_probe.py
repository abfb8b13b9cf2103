#!/usr/bin/env python
"""Development probe: the wide product as NG concurrent cooperative launches of
148 / NG CTAs, each over a contiguous range of rows (IRL_WIDE_G), against the
single 148-CTA launch.  usage: wide_groups_probe.py <cfgs>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_01437_b200 import _lib, ansatz as A, estimators as E, synthetic as S  # noqa: E402

for idx in [int(c) for c in sys.argv[1].split(",")]:
    cfg = S.CONFIGS[idx]
    inp = S.make_inputs(cfg)
    arch = bench._arch(A, cfg)
    b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc, mode="stored")
    en = E.estimate_energy(b)
    co = b.coefficients(en.mean)
    obar = b.obar()
    n, p, ld = b.n_rows, b.param_count, b.ld
    cplx = b.is_complex
    rows = 2 if cplx else 1
    v = torch.zeros((rows, ld), dtype=torch.float64, device="cuda")
    v[:, :p] = torch.randn((rows, p), dtype=torch.float64, device="cuda")
    el = 16 if cplx else 8

    def launch(g, ng, out, ws, stream):
        r0, r1 = n * g // ng, n * (g + 1) // ng
        o_ptr = b.o_padded.data_ptr() + r0 * ld * el
        c_ptr = co.data_ptr() + r0 * el
        if cplx:
            _lib.call("irl_mvp_c128", o_ptr, r1 - r0, p, ld, _lib.ptr(obar), c_ptr, _lib.ptr(v[0]), _lib.ptr(v[1]),
                      _lib.ptr(out[0]), _lib.ptr(out[1]), None, None, None, None, 4, _lib.ptr(ws), ws.numel(), stream)
        else:
            _lib.call("irl_mvp_f64", o_ptr, r1 - r0, p, ld, _lib.ptr(obar), c_ptr, _lib.ptr(v[0]), _lib.ptr(out[0]),
                      None, None, None, 4, _lib.ptr(ws), ws.numel(), stream)

    for ng in (1, 2, 4):
        os.environ["IRL_WIDE_G"] = str(148 // ng)
        nbytes = int(_lib.lib().irl_mvp_workspace_bytes(n, ld, int(cplx)))
        wss = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(ng)]
        outs = [torch.empty((rows, ld), dtype=torch.float64, device="cuda") for _ in range(ng)]
        streams = [torch.cuda.Stream() for _ in range(ng)]
        times = []
        for rep in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            main = torch.cuda.current_stream()
            e0.record(main)
            for g in range(ng):
                streams[g].wait_stream(main)
                with torch.cuda.stream(streams[g]):
                    launch(g, ng, outs[g], wss[g], streams[g].cuda_stream)
            for g in range(ng):
                main.wait_stream(streams[g])
            e1.record(main)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        print(f"cfg{idx}: {ng} launch(es) of {148 // ng} CTAs: {min(times[1:]):.3f} ms (runs {[round(t, 3) for t in times]}), "
              f"plan {_lib.mvp_plan(n // ng, ld, cplx, 4)}", flush=True)
        del wss, outs
    del os.environ["IRL_WIDE_G"]
    del b, v
    torch.cuda.empty_cache()
