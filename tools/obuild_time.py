#!/usr/bin/env python
"""Development tool: warm O-build time (ansatz.fill_o_rows: hidden layer, row
writer, column statistics) per BASELINE config, CUDA events, median of 5.
usage: obuild_time.py <cfgs, e.g. 2,3,4,5>"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_01437_b200 import ansatz as A, synthetic as S  # noqa: E402

peak, _ = bench.measured_peak_gbs()
for idx in [int(c) for c in sys.argv[1].split(",")]:
    cfg = S.CONFIGS[idx]
    inp = S.make_inputs(cfg)
    arch = bench._arch(A, cfg)
    params = A.AnsatzParameters(arch, inp.theta)
    b = A.build_batch(params, inp.x, inp.e_loc, mode="stored")
    xt = A._x_device(inp.x, arch.n_inputs, "cuda")
    mean = b._stats_e
    obar, g = b.colstats(mean)
    gc = b.gradient_coefficients(mean)
    ts = []
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        A.fill_o_rows(params, xt, b.o_padded, b.weights, gc, obar, g)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts[1:])
    o_bytes = cfg.n_rows * cfg.param_count * (16 if cfg.complex_params else 8)
    print(f"cfg{idx}: O-build {ms:.3f} ms, {o_bytes / ms / 1e6:.0f} GB/s of O written = {o_bytes / ms / 1e6 / peak:.3f} of "
          f"the copy peak", flush=True)
    del b, xt, obar, g, gc
    torch.cuda.empty_cache()
