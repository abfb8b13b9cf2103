import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch
from paper_2601_01437_b200 import ansatz as A, estimators as E, synthetic as S
from oracle import nqs, estimators as oest
cfg = S.CONFIGS[1].with_rows(8192)
inp = S.make_inputs(cfg)
arch = A.RBMArchitecture(cfg.n_inputs, cfg.hidden)
params = A.AnsatzParameters(arch, inp.theta)
otf = A.build_batch(params, inp.x, inp.e_loc, mode="otf")
eo = E.estimate_energy(otf)
o = nqs.rbm_rows(inp.theta, inp.x, cfg.n_inputs, cfg.hidden)
w = np.full(cfg.n_rows, 1/cfg.n_rows)
ref = oest.gradient(w, inp.e_loc, o, eo.mean)
got = E.energy_gradient(otf, eo).cpu().numpy()
n, h = cfg.n_inputs, cfg.hidden
for name, sl in (("a", slice(0,n)), ("b", slice(n,n+h)), ("W", slice(n+h, None))):
    d = got[sl]-ref[sl]; print(name, np.linalg.norm(d)/np.linalg.norm(ref[sl]))
Wd = (got[n+h:]-ref[n+h:]).reshape(h, n); Wr = ref[n+h:].reshape(h,n)
print("per j err", np.round(np.linalg.norm(Wd,axis=1)/np.linalg.norm(Wr,axis=1),3))
print("per i err", np.round(np.linalg.norm(Wd,axis=0)/np.linalg.norm(Wr,axis=0),3))
ob = otf.obar().cpu().numpy()[:o.shape[1]]; print("obar err", np.linalg.norm(ob - w@o)/np.linalg.norm(w@o))
t_ref = nqs.rbm_hidden(inp.theta, inp.x, n, h)
t_got = otf.otf["t"].cpu().numpy()
print("T err", np.abs(t_got - t_ref).max())
xb = otf.otf["xbits"].cpu().numpy().view(np.uint64)
bits = np.array([[(int(xb[r, k // 64]) >> (k % 64)) & 1 for k in range(n)] for r in range(5)])
print("bits ok", np.array_equal(bits, inp.x[:5]))
