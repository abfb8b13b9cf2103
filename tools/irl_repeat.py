"""Repeat one IRL solve N times: wall and device (CUDA event) time of each (development tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_01437_b200 import ansatz as A, estimators as E, optimizer as OPT, synthetic as S  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
mode = sys.argv[2] if len(sys.argv) > 2 else "stored"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
cfg = S.CONFIGS[idx]
inp = S.make_inputs(cfg)
arch = (A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm"
        else A.MLPArchitecture(cfg.n_inputs, cfg.hidden))
b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc, mode=mode)
en = E.estimate_energy(b)
conf = OPT.OptimizerConfig(m=cfg.m, max_restarts=cfg.max_restarts)
OPT.solve_step(b, conf, seed=cfg.lanczos_seed, energy=en)
torch.cuda.synchronize()
walls, devs = [], []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    r = OPT.solve_step(b, conf, seed=cfg.lanczos_seed, energy=en)
    e1.record()
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
    devs.append(e0.elapsed_time(e1))
print("wall ms", " ".join(f"{w:.2f}" for w in walls))
print("dev  ms", " ".join(f"{d:.2f}" for d in devs))
