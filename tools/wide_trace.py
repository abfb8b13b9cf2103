#!/usr/bin/env python
"""Development tool: per-block timeline of the single-read wide product
(IRL_WIDE_TRACE=1).  Stamps (globaltimer ns) per CTA and block: 0 producer
issue, 1 consumer warp 0 dot done, 2 publish done, 3 counter complete seen,
4 y ready, 5 consumer warp 0 accumulate done.  Prints median intervals."""
import os
import sys

os.environ["IRL_WIDE_TRACE"] = os.environ.get("IRL_WIDE_TRACE", "1")  # stride: every k-th block
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_01437_b200 import _lib, ansatz as A, estimators as E, synthetic as S  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 5
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
cfg = S.CONFIGS[idx].with_rows(rows)
inp = S.make_inputs(cfg)
arch = (A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm"
        else A.MLPArchitecture(cfg.n_inputs, cfg.hidden))
b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc, mode="stored")
en = E.estimate_energy(b)
P = arch.param_count
v = torch.as_tensor(np.random.default_rng(1).standard_normal(P) + (1j * np.random.default_rng(2).standard_normal(P) if cfg.complex_params else 0), device="cuda")
for _ in range(3):
    E.heff_matvec(b, en, v, mode=4)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
E.heff_matvec(b, en, v, mode=4)
ev[1].record()
torch.cuda.synchronize()
print(f"cfg{idx} rows {rows}: product {ev[0].elapsed_time(ev[1]):.3f} ms, plan {_lib.mvp_plan(b.n_rows, b.ld, b.is_complex, 4)}")
G = 148
buf = np.zeros(G * 512 * 8, dtype=np.uint64)
n = _lib.lib().irl_debug_wide_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes)
t = buf.reshape(G, 512, 8).astype(np.int64)
nb = int((t[0, :, 0] > 0).sum())
t = t[:, :nb]
base = t[:, :, 0].min()
names = ["issue", "dot", "pub", "cnt", "y", "acc"]
print("blocks traced", nb)
for k in range(1, 6):
    d = t[:, :, k] - t[:, :, k - 1]
    print(f"{names[k-1]:>5} -> {names[k]:<5} median {np.median(d[:, 8:]):8.0f} ns  p90 {np.percentile(d[:, 8:], 90):8.0f}")
# block cadence at CTA 0 and the spread of publish times over CTAs
cad = np.diff(t[0, :, 0])
print("issue cadence CTA0 (per traced block) median", np.median(cad[8:]), "ns; over the trace", [int(x) for x in np.percentile(cad, [10, 50, 90, 99])], "ns; pub spread over CTAs (max-min) median",
      np.median((t[:, :, 2].max(0) - t[:, :, 2].min(0))[8:]), "ns")
for bb in (10, 11, 12, 100, 101):
    if bb < nb:
        print(bb, [(int(np.median(t[:, bb, k] - base))) for k in range(6)])
out = os.environ.get("WIDE_TRACE_OUT")
if out:
    np.save(out, t)
