import sys, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch
from paper_2601_01437_b200 import _lib, estimators as E
from oracle import estimators as oest
rng = np.random.default_rng(0)
for (n, p, cplx) in [(300, 20000, False), (257, 9001, True), (1000, 33000, False)]:
    o = rng.normal(0, 1, (n, p)) + (1j * rng.normal(0, 1, (n, p)) if cplx else 0)
    e = rng.normal(-1, 0.1, n) + (1j * rng.normal(0, 0.01, n) if cplx else 0)
    w = np.full(n, 1.0 / n)
    b = E.SampleBatch(None, w, e, o, n, kind="hermitian" if cplx else None)
    en = E.estimate_energy(b)
    v = rng.standard_normal(p) + (1j * rng.standard_normal(p) if cplx else 0)
    print(n, p, cplx, _lib.mvp_plan(n, b.ld, cplx, 4), flush=True)
    out = E.heff_matvec(b, en, v, mode=4)
    ref = E.heff_matvec(b, en, v, mode=2)
    print("  rel vs two-pass", np.linalg.norm(out - ref) / np.linalg.norm(ref), flush=True)
