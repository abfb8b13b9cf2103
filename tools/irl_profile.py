"""cProfile + CUDA timeline breakdown of one IRL solve (development tool)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_01437_b200 import ansatz as A, estimators as E, optimizer as OPT, synthetic as S  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = S.CONFIGS[idx]
inp = S.make_inputs(cfg)
arch = A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm" else A.MLPArchitecture(cfg.n_inputs, cfg.hidden)
b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc)
en = E.estimate_energy(b)
conf = OPT.OptimizerConfig(m=cfg.m, max_restarts=cfg.max_restarts)
OPT.solve_step(b, conf, seed=cfg.lanczos_seed, energy=en)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    r = OPT.solve_step(b, conf, seed=cfg.lanczos_seed, energy=en)
    torch.cuda.synchronize()
    print("solve ms", (time.perf_counter() - t0) * 1e3, r.n_matvec)
pr = cProfile.Profile()
pr.enable()
OPT.solve_step(b, conf, seed=cfg.lanczos_seed, energy=en)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
