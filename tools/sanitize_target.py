"""Small workload that launches every kernel once, for compute-sanitizer runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_01437_b200 import ansatz as A, estimators as E, optimizer as OPT, synthetic as S  # noqa: E402

for idx, rows in ((1, 300), (4, 96), (3, 200), (2, 130)):
    cfg = S.CONFIGS[idx].with_rows(rows)
    inp = S.make_inputs(cfg)
    arch = (A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm"
            else A.MLPArchitecture(cfg.n_inputs, cfg.hidden))
    params = A.AnsatzParameters(arch, inp.theta)
    b = A.build_batch(params, inp.x, inp.e_loc)
    en = E.estimate_energy(b)
    P = b.param_count
    rng = np.random.default_rng(0)
    v = rng.standard_normal(P) + (1j * rng.standard_normal(P) if cfg.complex_params else 0)
    for mode in (1, 2, 3):
        try:
            E.heff_matvec(b, en, v, mode=mode)
            E.qgt_matvec(b, v, mode=mode)
        except Exception as exc:  # noqa: BLE001
            print("mode", mode, "skipped:", str(exc)[:80])
    b._colstats.clear()
    E.energy_gradient(b, en)  # standalone colstats kernel
    OPT.solve_step(b, OPT.OptimizerConfig(m=8, max_restarts=1), seed=1, use_graph=False)
    if cfg.model == "mlp" or not cfg.complex_params:
        bo = A.build_batch_otf(params, inp.x, inp.e_loc)
        eo = E.estimate_energy(bo)
        E.heff_matvec(bo, eo, v)
        E.qgt_matvec(bo, v)
    torch.cuda.synchronize()
    print("ok", cfg.name)

# on-the-fly MLP with a tail hidden chunk (h = 130) and odd n_in: G formed from T
rng = np.random.default_rng(1)
n_in, hidden, rows = 37, 130, 257
x = np.zeros((rows, n_in), dtype=np.uint8)
occ = np.argsort(rng.random((rows, n_in)), axis=1)[:, : n_in // 2]
x[np.arange(rows)[:, None], occ] = 1
arch = A.MLPArchitecture(n_in, hidden)
theta = rng.normal(0, 0.1, arch.param_count)
bo = A.build_batch_otf(A.AnsatzParameters(arch, theta), x, rng.normal(-3, 0.1, rows))
eo = E.estimate_energy(bo)
E.heff_matvec(bo, eo, rng.standard_normal(arch.param_count))
torch.cuda.synchronize()
print("ok mlp tail")
