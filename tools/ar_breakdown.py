import sys, time, warnings, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2601_01437_b200 import autoregressive as AR, hamiltonian as H, optimizer as OPT, synthetic as S, estimators as E
ints = H.parse_fcidump(S.molecule_fcidump(51, 10, 10, ms2=0, scale=0.05))
sector = ints.sector()
params = AR.init_parameters(AR.Architecture(sector.n_orbitals, 42), seed=111)
warnings.simplefilter("ignore")
def t(f, *a, **k):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(*a, **k); torch.cuda.synchronize(); return r, (time.perf_counter()-t0)*1e3
out = {}
bits = H.enumerate_sector(sector)
_, out['enumerate'] = t(H.enumerate_sector, sector)
xb = torch.as_tensor(bits.view(np.int64), device='cuda')
for rep in range(2):
    (d, ip, pb, el), out['partners'] = t(AR.hamiltonian_partners, ints, xb)
    _, out['logamp_x'] = t(AR.log_amplitude_batch, params, sector, xb)
    _, out['logamp_partners'] = t(AR.log_amplitude_batch, params, sector, pb)
    _, out['local_energies'] = t(AR.local_energies, params, ints, sector, xb)
    _, out['rows'] = t(AR.log_derivative_batch, params, sector, xb)
    b, out['build_batch'] = t(AR.build_batch, params, ints, sector)
    c, out['cache'] = t(AR.build_connected_cache, params, ints, sector, b)
    en = E.estimate_energy(b)
    r, out['solve_step'] = t(OPT.solve_step, b, OPT.OptimizerConfig(), 1, energy=en, connected=c)
    _, out['energy_at'] = t(OPT.energy_at, params, ints, sector)
out['nnz'] = int(pb.numel())
print(json.dumps(out))
