import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S
import pynvml
pynvml.nvmlInit(); hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
idx = int(sys.argv[1]); mode = sys.argv[2]
cfg = S.CONFIGS[idx]; inp = S.make_inputs(cfg)
arch = A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm" else A.MLPArchitecture(cfg.n_inputs, cfg.hidden)
b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc, mode=mode)
en = E.estimate_energy(b); c = b.coefficients(en.mean)
P, ld = b.param_count, b.ld
vi = torch.randn(ld, dtype=torch.float64, device="cuda"); vi[P:] = 0; vo = torch.empty_like(vi)
for blk in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        E._apply(b, c, vi, vo)
    e1.record(); torch.cuda.synchronize()
    clk = pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
    reasons = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hnd)
    pw = pynvml.nvmlDeviceGetPowerUsage(hnd) / 1000
    print(f"blk {blk}: {e0.elapsed_time(e1)/50:.3f} ms/MVP  sm {clk} MHz  reasons 0x{reasons:x}  power {pw:.0f} W", flush=True)
