#!/usr/bin/env python
"""Per-config performance sweep (one JSON line per config) — development tool.

For each BASELINE config: O-build time (warm), fused / two-pass MVP time and
GB/s (one O read per fused product, two per two-pass; device time per product
after an L2 write flush, from CUDA-graph replays), IRL solve wall time.
"""

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2601_01437_b200 import _lib, ansatz as A, estimators as E, optimizer as OPT, synthetic as S  # noqa: E402


def timed(fn, reps):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def flush_l2(buf):
    buf.add_(1.0)


def graph_timed(fn, l2buf, k=10, reps=5):
    """Per-call device time of fn() after a write flush of L2, free of host
    launch overhead: CUDA graphs of k x (flush, fn) and k x flush, replayed
    under events; the difference over k.  (Event-timing one eager call after a
    flush measures the Python/ctypes launch path when the product is short,
    e.g. cfg1: 25.6 us eager vs 17.5 us on the device.)"""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()

    def build(with_fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(k):
                flush_l2(l2buf)
                if with_fn:
                    fn()
        return g

    def run(g):
        out = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b))
        return statistics.median(out)

    g_both, g_flush = build(True), build(False)
    t = (run(g_both) - run(g_flush)) / k
    del g_both, g_flush
    return t


def _peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 8000.0 * 0.8


PEAK = _peak()
DMMA_PEAK_TFLOPS = 37.0  # measured FP64 tensor (DMMA) peak on this B200 pool, tools/fp64_peak.cu


def cpu_leg(cfg, budget_bytes: float = 1.5e9):
    """The reference's arithmetic (oracle port of est.heff_matvec, with its
    per-call centring copy) on a row sample sized to ~1.5 GB of O, extrapolated
    linearly in N_s ("extrapolated" when not the full N)."""
    sys.path.insert(0, ROOT)
    import bench

    b = 16 if cfg.complex_params else 8
    width = cfg.param_count * (2 if cfg.complex_params else 1)
    n_sub = int(max(256, min(cfg.n_rows, budget_bytes // (width * b))))
    sec = bench.cpu_reference_sample(cfg, n_sub, reps=3)
    full = sec * cfg.n_rows / n_sub
    return {"mvp_s": 1.0 / full, "cores": bench.cpu_cores(), "kind": "port", "rows_timed": n_sub,
            "extrapolated_x": cfg.n_rows / n_sub}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--irl", type=int, default=1)
    ap.add_argument("--otf", type=int, default=0, help="MLP configs in on-the-fly mode (O not stored)")
    ap.add_argument("--cpu", type=int, default=0, help="also time the CPU oracle port on a row sample (same run)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    l2buf = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    for idx in [int(c) for c in args.configs.split(",")]:
        cfg = S.CONFIGS[idx]
        if args.rows:
            cfg = cfg.with_rows(args.rows)
        t0 = time.perf_counter()
        inp = S.make_inputs(cfg)
        gen_s = time.perf_counter() - t0
        arch = (A.RBMArchitecture(cfg.n_inputs, cfg.hidden, cfg.complex_params) if cfg.model == "rbm"
                else A.MLPArchitecture(cfg.n_inputs, cfg.hidden))
        params = A.AnsatzParameters(arch, inp.theta)
        if args.otf:
            t0 = time.perf_counter()
            batch = A.build_batch_otf(params, inp.x, inp.e_loc)
            en = E.estimate_energy(batch)
            batch.obar()
            torch.cuda.synchronize()
            prep = (time.perf_counter() - t0) * 1e3
            P, ld = batch.param_count, batch.ld
            coeff = batch.coefficients(en.mean)
            shape = (2, ld) if cfg.complex_params else (ld,)
            vin = torch.randn(shape, dtype=torch.float64, device=dev)
            vin[..., P:] = 0
            vout = torch.empty(shape, dtype=torch.float64, device=dev)
            vi, vo = ((vin[0], vin[1]), (vout[0], vout[1])) if cfg.complex_params else (vin, vout)
            E._apply(batch, coeff, vi, vo)
            torch.cuda.synchronize()
            ms = timed(lambda: E._apply(batch, coeff, vi, vo), args.reps)
            med = statistics.median(ms)
            # useful DMMA flops: dot (n_in k-steps) + acc (n_in + 1 columns) per real hidden column
            cols = cfg.hidden * (2 if cfg.complex_params else 1)
            flops = 2.0 * batch.n_rows * cols * (2 * cfg.n_inputs + 1)
            tf = flops / (med / 1e3) / 1e12
            out = {"config": cfg.name + "-otf", "prepare_ms": prep, "otf": {"ms": med, "mvp_s": 1e3 / med,
                   "tflops": tf, "frac_dmma_measured": tf / DMMA_PEAK_TFLOPS}}
            if args.cpu:
                out["cpu_baseline"] = cpu_leg(cfg)
            if args.irl:
                conf = OPT.OptimizerConfig(m=cfg.m, max_restarts=cfg.max_restarts)
                OPT.solve_step(batch, conf, seed=cfg.lanczos_seed, energy=en)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = OPT.solve_step(batch, conf, seed=cfg.lanczos_seed, energy=en)
                torch.cuda.synchronize()
                out["irl"] = {"wall_ms": (time.perf_counter() - t0) * 1e3, "n_matvec": res.n_matvec,
                              "lambda": res.lambda_min, "converged": res.converged}
            print(json.dumps(out), flush=True)
            del batch
            torch.cuda.empty_cache()
            continue
        batch = A.build_batch(params, inp.x, inp.e_loc)
        torch.cuda.synchronize()
        # warm O-build time: refill the same buffers
        xt = A._x_device(inp.x, arch.n_inputs, dev)
        mean = batch._stats_e
        obar, g = batch.colstats(mean)
        gc = batch.gradient_coefficients(mean)
        ob = timed(lambda: A.fill_o_rows(params, xt, batch.o_padded, batch.weights, gc, obar, g), 3)
        en = E.estimate_energy(batch)
        N, P, ld = batch.n_rows, batch.param_count, batch.ld
        b_el = 16 if batch.is_complex else 8
        herm = batch.kind == E.KIND_HERMITIAN
        coeff = batch.coefficients(en.mean)
        if herm:
            vin = torch.randn((2, ld), dtype=torch.float64, device=dev)
            vin[:, P:] = 0
            vout = torch.empty((2, ld), dtype=torch.float64, device=dev)
            vi, vo = (vin[0], vin[1]), (vout[0], vout[1])
        else:
            vin = torch.randn(ld, dtype=torch.float64, device=dev)
            vin[P:] = 0
            vout = torch.empty(ld, dtype=torch.float64, device=dev)
            vi, vo = vin, vout
        out = {"config": cfg.name, "gen_s": gen_s, "obuild_ms": min(ob),
               "obuild_gbs": N * P * b_el / (min(ob) / 1e3) / 1e9}
        for mode, name, passes in ((1, "fused", 1), (2, "two_pass", 2), (3, "rows", 1), (4, "wide", 1)):
            try:
                plan = _lib.mvp_plan(N, ld, batch.is_complex, mode)
                E._apply(batch, coeff, vi, vo, mode=mode)
                torch.cuda.synchronize()
            except Exception as exc:  # noqa: BLE001
                out[name] = {"error": str(exc)[:200]}
                continue
            med = graph_timed(lambda: E._apply(batch, coeff, vi, vo, mode=mode), l2buf,
                              k=10 if N * ld < 1e9 else 3)
            out[name] = {"ms": med, "mvp_s": 1e3 / med, "gbs_one_read": N * P * b_el / (med / 1e3) / 1e9,
                         "gbs_traffic": passes * N * ld * b_el / (med / 1e3) / 1e9, "plan": plan}
        if args.irl:
            conf = OPT.OptimizerConfig(m=cfg.m, max_restarts=cfg.max_restarts)
            OPT.solve_step(batch, conf, seed=cfg.lanczos_seed, energy=en)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = OPT.solve_step(batch, conf, seed=cfg.lanczos_seed, energy=en)
            torch.cuda.synchronize()
            out["irl"] = {"wall_ms": (time.perf_counter() - t0) * 1e3, "n_matvec": res.n_matvec,
                          "lambda": res.lambda_min, "converged": res.converged}
        # roofline fractions of the AUTO path against the measured copy peak and the 8 TB/s spec
        auto = {"fused": "fused", "two_pass": "two_pass", "rows": "rows", "wide": "wide"}[
            _lib.mvp_plan(N, ld, batch.is_complex, 0)["path"]]
        if "ms" in out.get(auto, {}):
            ms = out[auto]["ms"]
            one, two = N * P * b_el / (ms / 1e3) / 1e9, 2 * N * P * b_el / (ms / 1e3) / 1e9
            out["roofline"] = {"auto_path": auto, "mvp_s": 1e3 / ms, "gbs_one_read": one, "gbs_two_pass": two,
                               "frac_measured_one_read": one / PEAK, "frac_measured_two_pass": two / PEAK,
                               "frac_spec_two_pass": two / 8000.0, "peak_measured_gbs": PEAK}
        if args.cpu:
            out["cpu_baseline"] = cpu_leg(cfg)
        print(json.dumps(out), flush=True)
        del batch, inp, xt, obar, g, gc, coeff
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
