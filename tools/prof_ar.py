"""Autoregressive log amplitudes over a 63504-configuration sector, for ncu captures (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_01437_b200 import autoregressive as AR, hamiltonian as H  # noqa: E402

sector = H.Sector(20, 5, 5)
params = AR.init_parameters(AR.Architecture(20, 42), seed=111)
bits = H.enumerate_sector(sector)
for _ in range(2):
    AR.log_amplitude_batch(params, sector, bits)
    AR.log_derivative_batch(params, sector, bits[:8192])
torch.cuda.synchronize()
