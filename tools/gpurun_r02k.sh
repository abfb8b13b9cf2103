mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gevp.py -q -m gpu > gpurun_out/gevp_tests.log 2>&1; echo "rc $?" >> gpurun_out/gevp_tests.log
timeout 900 python - > gpurun_out/gevp_cfg2.txt 2>&1 <<'PY'
import time, torch, bench
from paper_2601_01437_b200 import ansatz as A, estimators as E, optimizer as OPT, synthetic as S
for idx in (1, 2):
    cfg = S.CONFIGS[idx]; inp = S.make_inputs(cfg)
    b = A.build_batch(A.AnsatzParameters(bench._arch(A, cfg), inp.theta), inp.x, inp.e_loc, mode="stored")
    en = E.estimate_energy(b)
    for pc in (False, True):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = OPT.solve_step(b, OPT.OptimizerConfig(method="gevp", gevp_max_iter=4000, gevp_tol=1e-10, gevp_precond=pc), seed=cfg.lanczos_seed, energy=en)
        torch.cuda.synchronize()
        print(idx, "precond", pc, "wall ms", (time.perf_counter() - t0) * 1e3, "products", r.n_matvec, "lambda", r.lambda_min, "converged", r.converged, "res", r.pair.residual, flush=True)
PY
