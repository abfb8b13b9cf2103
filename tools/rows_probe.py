"""Product timing free of host launch overhead (development tool): CUDA graphs
of K x (flush + product) minus K x flush, for a write flush (dirty L2, the
bench rule) and a read-only flush (clean L2), and K x product warm (O
L2-resident when it fits).  Prints per-product microseconds."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S  # noqa: E402

cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 1
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
K = 20
cfg = S.CONFIGS[cfg_i]
inp = S.make_inputs(cfg)
arch = A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm" else A.MLPArchitecture(cfg.n_inputs, cfg.hidden)
b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc)
en = E.estimate_energy(b)
c = b.coefficients(en.mean)
vi = torch.randn(b.ld, dtype=torch.float64, device="cuda")
vi[b.param_count:] = 0
vo = torch.empty_like(vi)
buf = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
sink = torch.empty((), dtype=torch.float32, device="cuda")
wf = lambda: buf.add_(1.0)  # noqa: E731
rf = lambda: torch.sum(buf, dim=0, out=sink)  # noqa: E731
prod = lambda: E._apply(b, c, vi, vo, mode=mode)  # noqa: E731
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        wf(); rf(); prod()  # noqa: E702
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()


def graph(fns):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(K):
            for f in fns:
                f()
    return g


def t(g):
    ms = []
    for _ in range(7):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        z.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(z))
    return statistics.median(ms) * 1e3 / K


out = {"config": cfg.name, "env": {k: v for k, v in os.environ.items() if k.startswith("IRL_")}}
tw, tr, tp = t(graph([wf])), t(graph([rf])), t(graph([prod]))
out["write_flush_us"] = round(t(graph([wf, prod])) - tw, 2)
out["read_flush_us"] = round(t(graph([rf, prod])) - tr, 2)
out["warm_us"] = round(tp, 2)
out["flush_us"] = [round(tw, 1), round(tr, 1)]
print(json.dumps(out))
