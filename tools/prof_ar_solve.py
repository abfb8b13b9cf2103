"""Connected products of the reference ansatz's exact batch (syn10: 63504 configurations), for ncu launch lists."""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_01437_b200 import autoregressive as AR, estimators as E, hamiltonian as H, synthetic as S  # noqa: E402

warnings.simplefilter("ignore")
ints = H.parse_fcidump(S.molecule_fcidump(51, 10, 10, ms2=0, scale=0.05))
sector = ints.sector()
params = AR.init_parameters(AR.Architecture(sector.n_orbitals, 42), seed=111)
b = AR.build_batch(params, ints, sector)
c = AR.build_connected_cache(params, ints, sector, b)
en = E.estimate_energy(b)
v = np.random.default_rng(0).standard_normal(b.param_count)
for _ in range(3):
    E.connected_heff_matvec(b, en, c, v)
torch.cuda.synchronize()
