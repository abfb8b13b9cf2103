"""Local-energy throughput on a synthetic molecule of BASELINE cfg2's size.

cfg2's RBM (n_visible = 40 spin-orbitals, hidden = 160) on a seeded synthetic
FCIDUMP with 20 spatial orbitals and 20 electrons (10 up + 10 down); samples
are random sector configurations.  Prints one JSON line: device E_loc and
connected-partner (count + fill) times, samples/s, partner evaluations/s, and
the oracle's E_loc per sample on a few samples (the reference's per-sample
Python path, ham:290-302) timed on this host.  Development / bench tool.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def sector_samples(rng, ns, n_up, n_dn, count):
    up = np.argsort(rng.random((count, ns)), axis=1)[:, :n_up]
    dn = np.argsort(rng.random((count, ns)), axis=1)[:, :n_dn] + ns
    bits = np.zeros(count, dtype=np.uint64)
    for cols in (up, dn):
        for c in cols.T:
            bits |= np.uint64(1) << c.astype(np.uint64)
    return bits


_CPU = {}  # state of the CPU baseline workers (set before the pool forks)


def _cpu_eloc(chunk):
    """The oracle's per-sample local energy (the reference's algorithm,
    ham:290-302) on a chunk of samples; runs in a forked worker process."""
    from oracle import hamiltonian as oham
    from oracle import nqs

    st = _CPU
    M, hidden, theta, ints, ns = st["M"], st["hidden"], st["theta"], st["ints"], st["ns"]

    def lp(b):
        x = ((np.uint64(b) >> np.arange(M, dtype=np.uint64)) & np.uint64(1)).astype(np.uint8)[None, :]
        return nqs.rbm_log_psi(theta, x, M, hidden)[0]

    return [oham.local_energy(lp, ints.e_core, ints.h, ints.g, int(b), ns) for b in chunk]


def run(n_samples=8192, cpu_samples=2, ns=20, n_elec=20, hidden=160, seed=7, with_cpu=True):
    from paper_2601_01437_b200 import ansatz as A, hamiltonian as H, synthetic as S

    ints = H.parse_fcidump(S.molecule_fcidump(seed, ns, n_elec, scale=0.05))
    sec = ints.sector()
    rng = np.random.default_rng(seed + 1)
    M = 2 * ns
    theta = rng.normal(0, 0.01, M + hidden + hidden * M)
    params = A.AnsatzParameters(A.RBMArchitecture(M, hidden), theta)
    bits = sector_samples(rng, ns, sec.n_up, sec.n_down, n_samples)
    xb = torch.as_tensor(bits.view(np.int64), device="cuda")
    H.local_energies(params, ints, xb[:64])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eloc = H.local_energies(params, ints, xb)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t0 = time.perf_counter()
    indptr, pbits, elem, coeff = H.connected_partners(params, ints, xb)
    torch.cuda.synchronize()
    cache_ms = (time.perf_counter() - t0) * 1e3
    nnz = int(indptr[-1])
    out = {"workload": f"synthetic FCIDUMP ns={ns} nelec={n_elec}, RBM n={M} h={hidden} (cfg2 shape)",
           "n_samples": n_samples, "eloc_ms": ms, "samples_per_s": n_samples / (ms / 1e3),
           "partners_kept": nnz, "partners_per_sample": nnz / n_samples,
           "partner_evals_per_s": nnz / (ms / 1e3), "connected_csr_ms": cache_ms}
    if with_cpu:
        import multiprocessing as mp

        cores = len(os.sched_getaffinity(0))
        _CPU.update(M=M, hidden=hidden, theta=theta, ints=ints, ns=ns)
        e_dev = eloc.cpu().numpy()
        sample = bits[:cpu_samples]
        chunks = [sample[i::cores] for i in range(cores) if len(sample[i::cores])]
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(len(chunks)) as pool:  # workers never touch CUDA
            parts = pool.map(_cpu_eloc, chunks)
        cpu_s = time.perf_counter() - t0
        ref = np.zeros(len(sample), dtype=complex)
        for i, part in enumerate(parts):
            ref[i::cores][: len(part)] = part
        out["cpu_baseline"] = {"value": len(sample) / cpu_s, "unit": "samples/s", "cores": len(chunks),
                               "kind": "port",
                               "sample": (f"oracle local_energy (reference algorithm, ham:290-302) on {len(sample)} "
                                          f"samples, one process per core ({len(chunks)} cores)")}
        out["parity_max_rel"] = float(np.max(np.abs(ref.real - e_dev[: len(sample)])
                                             / np.maximum(1.0, np.abs(e_dev[: len(sample)]))))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--cpu-samples", type=int, default=2)
    ap.add_argument("--hidden", type=int, default=160)
    args = ap.parse_args()
    print(json.dumps(run(args.n, args.cpu_samples, hidden=args.hidden)))


if __name__ == "__main__":
    main()
