"""Read-only HBM bandwidth on this GPU (development tool): torch's reduction
kernels over a 4 GiB f64 tensor (sum, and a vector norm), CUDA events, median
of 10 after warm-up.  The copy peak in MEASURED_PEAKS.json counts read+write
bytes of a copy; a pure read stream can go faster, and this is the ceiling the
single-read fused product is compared with in DESIGN.md."""
import json
import statistics

import torch

n = (4 << 30) // 8
x = torch.rand(n, dtype=torch.float64, device="cuda")
out = {}
for name, fn in (("sum", lambda: x.sum()), ("norm", lambda: torch.linalg.vector_norm(x))):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    med = statistics.median(ms)
    out[name] = {"ms": round(med, 4), "gbs": round(n * 8 / (med / 1e3) / 1e9, 1), "best_gbs": round(n * 8 / (min(ms) / 1e3) / 1e9, 1)}
print(json.dumps(out))
