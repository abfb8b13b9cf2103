"""Interleaving check (development tool): products on several batches of
different shapes and kinds in turn, each compared with the oracle."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2601_01437_b200 import estimators as E  # noqa: E402
from oracle import estimators as oest  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def random_batch(rng, n, p, cplx=False):
    o = rng.normal(0.1, 0.7, (n, p))
    e = rng.normal(-3.0, 0.3, n)
    if cplx:
        o = o + 1j * rng.normal(0, 0.5, (n, p))
        e = e + 1j * rng.normal(0, 0.05, n)
    w = np.ones(n)
    return o, e, w / w.sum()


rng = np.random.default_rng(11)
skip_real = len(sys.argv) > 1 and sys.argv[1] == "herm_only"
skip = set(sys.argv[2:]) if len(sys.argv) > 2 else set()
shapes = [(700, 13, False), (4099, 260, False), (333, 21, True), (1500, 37, False)]
bs = []
for n, p, c in shapes:
    o, e, w = random_batch(rng, n, p, c)
    b = E.SampleBatch(None, w, e, o, n, kind="hermitian") if c else E.SampleBatch(None, w, e, o, n)
    en = E.estimate_energy(b)
    bs.append((b, en, o, e, w, p, c))
for b, en, o, e, w, p, c in bs * 3:
    if c:
        v = rng.standard_normal(p) + 1j * rng.standard_normal(p)
        ref = oest.heff_hermitian(w, e, o, en.mean, v)
        got = E.heff_matvec(b, en, torch.as_tensor(v, device="cuda")).cpu().numpy()
        again = E.heff_matvec(b, en, torch.as_tensor(v).pin_memory()).numpy()
        print("herm", rel(got, ref), rel(again, ref), "mean", en.mean, "oracle mean", float(np.real(np.sum(w * e))))
        continue
    if skip_real:
        continue
    v = rng.standard_normal(p)
    ref = oest.heff(w, e, o, en.mean, v)
    big = torch.zeros(2 * p, dtype=torch.float64, device="cuda")
    big[::2] = torch.as_tensor(v, device="cuda")
    if "strided" not in skip:
        print(b.n_rows, "real strided", rel(E.heff_matvec(b, en, big[::2]).cpu().numpy(), ref))
    if "pinned" not in skip:
        print(b.n_rows, "real pinned", rel(E.heff_matvec(b, en, torch.as_tensor(v).pin_memory()).numpy(), ref))
    if "f32" not in skip:
        print(b.n_rows, "real f32", rel(np.asarray(E.heff_matvec(b, en, v.astype(np.float32))), oest.heff(w, e, o, en.mean, v.astype(np.float32).astype(np.float64))))
