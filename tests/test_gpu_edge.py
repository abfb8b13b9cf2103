"""Edge cases on the device path (reference behaviour: T/test_estimators.py:156-166,
:208-213; est:44-53, est:147-148, est:178-183): ragged and tiny shapes, exact-mode
weights, error paths, determinism, ABI status codes."""

import ctypes

import numpy as np
import pytest

from oracle import estimators as oest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def E(cuda):
    from paper_2601_01437_b200 import estimators

    return estimators


def random_batch(rng, n, p, cplx=False, exact=False):
    o = rng.normal(0.1, 0.7, (n, p))
    e = rng.normal(-3.0, 0.3, n)
    if cplx:
        o = o + 1j * rng.normal(0, 0.5, (n, p))
        e = e + 1j * rng.normal(0, 0.05, n)
    w = rng.random(n) + 0.05 if exact else np.ones(n)
    return o, e, w / w.sum()


@pytest.mark.parametrize("n,p", [(1, 1), (1, 17), (3, 2), (37, 5), (1237, 17), (4099, 33), (513, 1031), (700, 999)])
@pytest.mark.parametrize("mode", [1, 2, 3])
def test_ragged_shapes_real(E, n, p, mode):
    rng = np.random.default_rng(n * 1000 + p)
    o, e, w = random_batch(rng, n, p, exact=True)
    b = E.SampleBatch(None, w, e, o, 0)
    en = E.estimate_energy(b)
    mean, var, _ = oest.energy(w, e, 0)
    assert en.mean == pytest.approx(mean, abs=1e-12) and en.std_error == 0.0
    assert rel(E.energy_gradient(b, en).cpu().numpy(), oest.gradient(w, e, o, mean)) < 1e-9
    if mode == 3 and b.ld // 2 > 512:
        pytest.skip("rows path covers rows of at most 512 16-byte units")
    for _ in range(2):
        v = rng.standard_normal(p)
        assert rel(E.heff_matvec(b, en, v, mode=mode), oest.heff(w, e, o, mean, v)) < 1e-10
        assert rel(E.qgt_matvec(b, v, mode=mode), oest.qgt(w, o, v)) < 1e-10


@pytest.mark.parametrize("n,p", [(1, 3), (301, 7), (2050, 129)])
def test_ragged_shapes_complex_raw(E, n, p):
    rng = np.random.default_rng(n + p)
    o, e, w = random_batch(rng, n, p, cplx=True, exact=True)
    b = E.SampleBatch(None, w, e, o, 0)
    with pytest.warns(UserWarning):
        en = E.estimate_energy(b)
    mean, _, _ = oest.energy(w, e, 0)
    v = rng.standard_normal(p)
    for mode in (1, 2, 3, 4):
        assert rel(E.heff_matvec(b, en, v, mode=mode), oest.heff(w, e, o, mean, v)) < 1e-10


def test_validation_errors(E):
    rng = np.random.default_rng(0)
    o, e, w = random_batch(rng, 10, 4)
    with pytest.raises(ValueError):  # est:50-51
        E.SampleBatch(None, w * 2, e, o, 10)
    with pytest.raises(ValueError):
        E.SampleBatch(None, -w, e, o, 10)
    with pytest.raises(ValueError):  # empty batch: weights cannot sum to one
        E.SampleBatch(None, np.zeros(0), np.zeros(0), np.zeros((0, 4)), 0)
    with pytest.raises(ValueError):
        E.SampleBatch(None, w, e[:5], o, 10)
    b = E.SampleBatch(None, w, e, o, 10)
    en = E.estimate_energy(b)
    with pytest.raises(ValueError):  # est:178-181
        E.heff_matvec(b, en, np.zeros(5))
    bad = np.zeros(4)
    bad[1] = np.inf
    with pytest.raises(ValueError):  # est:182-183
        E.heff_matvec(b, en, bad)
    with pytest.raises(E.DensePCapError):  # est:324-325
        E.dense_heff(b, en, cap=3)


def test_host_tensor_inputs_and_outputs(E):
    import torch

    rng = np.random.default_rng(1)
    o, e, w = random_batch(rng, 333, 21)
    b = E.SampleBatch(None, w, e, o, 333)
    en = E.estimate_energy(b)
    v = rng.standard_normal(21)
    ref = oest.heff(w, e, o, en.mean, v)
    for t in (torch.as_tensor(v), torch.as_tensor(v).pin_memory()):
        out = E.heff_matvec(b, en, t)
        assert isinstance(out, torch.Tensor) and not out.is_cuda
        assert rel(out.numpy(), ref) < 1e-10
    out = E.heff_matvec(b, en, torch.as_tensor(v, device="cuda"))
    assert out.is_cuda and rel(out.cpu().numpy(), ref) < 1e-10


@pytest.mark.parametrize("mode", [1, 2, 3, 4])
def test_bitwise_determinism(E, mode):
    import torch

    rng = np.random.default_rng(2)
    o, e, w = random_batch(rng, 5000, 300, cplx=True)
    b = E.SampleBatch(None, w, e, o, 5000, kind="hermitian")
    en = E.estimate_energy(b)
    v = torch.as_tensor(rng.standard_normal(300) + 1j * rng.standard_normal(300), device="cuda")
    first = E.heff_matvec(b, en, v, mode=mode)
    for _ in range(3):
        assert torch.equal(first, E.heff_matvec(b, en, v, mode=mode))


def test_abi_status_codes(cuda):
    import torch

    from paper_2601_01437_b200 import _lib

    lib = _lib.lib()
    n, p = 64, 10
    ld = _lib.padded_ld(p, False)
    o = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    v = torch.zeros(ld, dtype=torch.float64, device="cuda")
    c = torch.zeros(n, dtype=torch.float64, device="cuda")
    ws_bytes = int(lib.irl_mvp_workspace_bytes(n, ld, 0))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    st = _lib.stream_handle()
    ok = lib.irl_mvp_f64(o.data_ptr(), n, p, ld, v.data_ptr(), c.data_ptr(), v.data_ptr(), v.data_ptr(), None, None,
                         None, 0, ws.data_ptr(), ws_bytes, st)
    assert ok == _lib.IRL_OK
    assert lib.irl_mvp_f64(o.data_ptr(), n, p, ld + 16, None, c.data_ptr(), v.data_ptr(), v.data_ptr(), None, None,
                           None, 0, ws.data_ptr(), ws_bytes, st) == _lib.IRL_ERR_ALIGN
    assert lib.irl_mvp_f64(o.data_ptr(), n, p, ld, None, c.data_ptr(), v.data_ptr(), v.data_ptr(), None, None, None,
                           0, ws.data_ptr(), 16, st) == _lib.IRL_ERR_WORKSPACE
    assert lib.irl_mvp_f64(o.data_ptr() + 8, n, p, ld, None, c.data_ptr(), v.data_ptr(), v.data_ptr(), None, None,
                           None, 0, ws.data_ptr(), ws_bytes, st) == _lib.IRL_ERR_ALIGN
    assert lib.irl_mvp_f64(None, n, p, ld, None, c.data_ptr(), v.data_ptr(), v.data_ptr(), None, None, None, 0,
                           ws.data_ptr(), ws_bytes, st) == _lib.IRL_ERR_ARG
    assert lib.irl_mvp_f64(o.data_ptr(), n, p, ld, None, c.data_ptr(), v.data_ptr(), v.data_ptr(), None, None, None,
                           7, ws.data_ptr(), ws_bytes, st) == _lib.IRL_ERR_ARG
    assert b"bad mvp mode" in lib.irl_last_error()
    torch.cuda.synchronize()


@pytest.mark.parametrize("stage", [True, False])
@pytest.mark.parametrize("L,j", [(866, 0), (866, 19), (6658, 7), (11282, 29), (60000, 39)])
def test_lanczos_step_kernels(cuda, L, j, stage, monkeypatch):
    """Fused Lanczos steps (single CTA, one cluster) == the BLAS-1/2 sequence
    of kry:96-116 (alpha, three-term update, two reorthogonalisation passes,
    beta, normalised next vector)."""
    import torch
    from paper_2601_01437_b200 import _lib

    if not stage:  # the global-memory cluster step instead of the shared-memory staged one
        monkeypatch.setenv("IRL_LANCZOS_NOSTAGE", "1")
    m = 41
    gen = torch.Generator(device="cuda").manual_seed(L + j)
    q, _ = torch.linalg.qr(torch.randn(L, j + 1, dtype=torch.float64, device="cuda", generator=gen))
    V0 = torch.zeros((m + 1, L), dtype=torch.float64, device="cuda")
    V0[: j + 1] = q.t()
    W0 = torch.randn(L, dtype=torch.float64, device="cuda", generator=gen)
    ab0 = torch.zeros((2, m), dtype=torch.float64, device="cuda")
    if j > 0:
        ab0[1, j - 1] = 0.37
    # reference sequence (the driver's torch branch)
    V, W, A = V0.clone(), W0.clone(), ab0.clone()
    v = V[j]
    a = torch.dot(v, W)
    W -= a * v
    if j > 0:
        W -= A[1, j - 1] * V[j - 1]
    vm = V[: j + 1]
    for _ in range(2):
        W -= vm.t() @ (vm @ W)
    b = torch.linalg.vector_norm(W)
    ref_v, ref_a, ref_b = (W / b), float(a), float(b)
    kernels = ["irl_lanczos_step_cluster"] + (["irl_lanczos_step_small"] if L <= 4096 else [])
    lib = _lib.lib()
    for name in kernels:
        V, W, A = V0.clone(), W0.clone(), ab0.clone()
        _lib.check(name, getattr(lib, name)(V.data_ptr(), L, W.data_ptr(), L, j, m, A.data_ptr(),
                                            _lib.stream_handle()))
        torch.cuda.synchronize()
        assert abs(float(A[0, j]) - ref_a) <= 1e-12 * max(1.0, abs(ref_a)), name
        assert abs(float(A[1, j]) - ref_b) <= 1e-12 * ref_b, name
        assert rel(V[j + 1].cpu().numpy(), ref_v.cpu().numpy()) < 1e-12, name
        # rows 0..j untouched
        assert torch.equal(V[: j + 1], V0[: j + 1]), name


def test_interleaved_batches_and_strided_inputs(E):
    """Plans, workspaces and captured host-path graphs are per batch / shape:
    alternating products on batches of different shapes and kinds stay exact;
    strided, float32 and host inputs are accepted like numpy's matmul would."""
    import torch

    rng = np.random.default_rng(11)
    shapes = [(700, 13, False), (4099, 260, False), (333, 21, True), (1500, 37, False)]
    batches = []
    for n, p, cplx in shapes:
        o, e, w = random_batch(rng, n, p, cplx=cplx)
        b = E.SampleBatch(None, w, e, o, n, kind="hermitian") if cplx else E.SampleBatch(None, w, e, o, n)
        if cplx:
            with pytest.warns(UserWarning):
                en = E.estimate_energy(b)
        else:
            en = E.estimate_energy(b)
        batches.append((b, en, o, e, w, p, cplx))
    for rep in range(3):
        for b, en, o, e, w, p, cplx in batches:
            if cplx:
                v = rng.standard_normal(p) + 1j * rng.standard_normal(p)
                ref = oest.heff_hermitian(w, e, o, en.mean, v)
                got = E.heff_matvec(b, en, torch.as_tensor(v, device="cuda"))
                again = E.heff_matvec(b, en, torch.as_tensor(v).pin_memory())
                assert rel(got.cpu().numpy(), again.numpy()) < 1e-14
                assert rel(got.cpu().numpy(), ref) < 1e-10
                continue
            v = rng.standard_normal(p)
            ref = oest.heff(w, e, o, en.mean, v)
            big = torch.zeros(2 * p, dtype=torch.float64, device="cuda")
            big[::2] = torch.as_tensor(v, device="cuda")
            strided = big[::2]  # non-contiguous device view
            assert rel(E.heff_matvec(b, en, strided).cpu().numpy(), ref) < 1e-10
            assert rel(E.heff_matvec(b, en, torch.as_tensor(v).pin_memory()).numpy(), ref) < 1e-10
            v32 = v.astype(np.float32)
            ref32 = oest.heff(w, e, o, en.mean, v32.astype(np.float64))
            assert rel(np.asarray(E.heff_matvec(b, en, v32)), ref32) < 1e-10


def test_interleaved_solves_are_bitwise_stable(E):
    """IRL solves and products on several batches (stored and on-the-fly, RBM
    and MLP, host and device vectors) in turn give bit-identical results to
    each batch's first, isolated call: no cached plan, workspace, staging
    buffer or captured graph leaks between batches."""
    import torch

    from paper_2601_01437_b200 import ansatz as A, optimizer as OPT

    rng = np.random.default_rng(5)

    def bits(n, k, rows):
        x = np.zeros((rows, n), dtype=np.uint8)
        occ = np.argsort(rng.random((rows, n)), axis=1)[:, :k]
        x[np.arange(rows)[:, None], occ] = 1
        return x

    specs = [("rbm", 12, 24, 900, "stored"), ("mlp", 10, 64, 1300, "otf"), ("rbm", 16, 40, 2100, "otf"),
             ("mlp", 14, 30, 700, "stored")]
    cases = []
    for model, n, h, rows, mode in specs:
        arch = A.RBMArchitecture(n, h) if model == "rbm" else A.MLPArchitecture(n, h)
        theta = rng.normal(0, 0.05, arch.param_count)
        x = bits(n, n // 2, rows)
        e = rng.normal(-5.0, 0.1, rows)
        b = A.build_batch(A.AnsatzParameters(arch, theta), x, e, mode=mode)
        en = E.estimate_energy(b)
        v = rng.standard_normal(arch.param_count)
        cases.append((b, en, v))
    conf = OPT.OptimizerConfig(m=12, max_restarts=2)
    first = []
    for b, en, v in cases:
        r = OPT.solve_step(b, conf, seed=1, energy=en)
        first.append((E.heff_matvec(b, en, torch.as_tensor(v).pin_memory()).clone(),
                      E.qgt_matvec(b, torch.as_tensor(v, device="cuda")).cpu(), r.lambda_min,
                      r.direction.cpu().clone()))
    for _ in range(2):
        for (b, en, v), (h0, s0, lam0, d0) in zip(cases[::-1], first[::-1]):
            r = OPT.solve_step(b, conf, seed=1, energy=en)
            assert r.lambda_min == lam0 and torch.equal(r.direction.cpu(), d0)
            assert torch.equal(E.heff_matvec(b, en, torch.as_tensor(v).pin_memory()), h0)
            assert torch.equal(E.qgt_matvec(b, torch.as_tensor(v, device="cuda")).cpu(), s0)


@pytest.mark.parametrize("kind", ["real", "complex_raw", "hermitian", "otf_rbm", "otf_mlp", "otf_herm"])
def test_workspace_and_output_canaries(E, kind):
    """Kernels stay inside the caller's buffers (the ABI's ownership rule): the
    workspace is handed over at exactly *_workspace_bytes() with a guard region
    behind it, outputs are views followed by guard words; every product path
    must leave the guards untouched.  (compute-sanitizer is not available on the
    GPU pool; this is the bounds check of our own.)"""
    import torch

    from paper_2601_01437_b200 import _lib, ansatz as A

    rng = np.random.default_rng(len(kind))
    guard = 1 << 20
    if kind.startswith("otf"):
        n_in, hidden, rows = (37, 130, 517) if kind == "otf_mlp" else (12, 72, 611)
        x = np.zeros((rows, n_in), dtype=np.uint8)
        occ = np.argsort(rng.random((rows, n_in)), axis=1)[:, : n_in // 2]
        x[np.arange(rows)[:, None], occ] = 1
        arch = (A.MLPArchitecture(n_in, hidden) if kind == "otf_mlp"
                else A.RBMArchitecture(n_in, hidden, kind == "otf_herm"))
        theta = rng.normal(0, 0.05, arch.param_count)
        if kind == "otf_herm":
            theta = theta + 1j * rng.normal(0, 0.05, arch.param_count)
        b = A.build_batch_otf(A.AnsatzParameters(arch, theta), x, rng.normal(-3, 0.1, rows))
        modes = [0]
    else:
        o, e, w = random_batch(rng, 2311, 301, cplx=kind != "real")
        b = (E.SampleBatch(None, w, e, o, 2311, kind="hermitian") if kind == "hermitian"
             else E.SampleBatch(None, w, e, o, 2311))
        modes = [1, 2, 3, 4]
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        en = E.estimate_energy(b)
    nbytes = b.mvp_workspace().numel()
    big = torch.full((nbytes + guard,), 0xA5, dtype=torch.uint8, device="cuda")
    b._ws[b._stream()] = big[:nbytes]  # this stream's workspace, exactly sized
    ld, p = b.ld, b.param_count
    herm = b.kind == E.KIND_HERMITIAN
    rows_v = 2 if herm else 1
    vin = torch.zeros((rows_v, ld), dtype=torch.float64, device="cuda")
    vin[:, :p] = torch.as_tensor(rng.standard_normal((rows_v, p)), device="cuda")
    outbuf = torch.full((rows_v, ld + 64), 7.25, dtype=torch.float64, device="cuda")
    coeff = b.coefficients(en.mean)
    for mode in modes:
        if mode == 3 and ld // (1 if b.is_complex else 2) > 512:
            continue
        if herm:
            E._apply(b, coeff, (vin[0], vin[1]), (outbuf[0, :ld], outbuf[1, :ld]), mode=mode)
        else:
            E._apply(b, coeff, vin[0], outbuf[0, :ld], mode=mode)
        torch.cuda.synchronize()
        assert bool((big[nbytes:] == 0xA5).all()), f"workspace overrun, mode {mode}"
        assert bool((outbuf[:, ld:] == 7.25).all()), f"output overrun, mode {mode}"


@pytest.mark.parametrize("model,n_in,hidden,rows,cplx", [("rbm", 12, 24, 1001, False), ("mlp", 37, 130, 517, False),
                                                          ("rbm", 10, 30, 333, True), ("mlp", 100, 512, 70, False)])
def test_obuild_output_canaries(E, model, n_in, hidden, rows, cplx):
    """The O-row writers (column tiles and row sweeps) and their fused
    statistics write exactly N x ld of O and ld entries of Obar / F."""
    import torch

    from paper_2601_01437_b200 import _lib, ansatz as A

    rng = np.random.default_rng(rows)
    x = np.zeros((rows, n_in), dtype=np.uint8)
    occ = np.argsort(rng.random((rows, n_in)), axis=1)[:, : n_in // 2]
    x[np.arange(rows)[:, None], occ] = 1
    arch = A.MLPArchitecture(n_in, hidden) if model == "mlp" else A.RBMArchitecture(n_in, hidden, cplx)
    theta = rng.normal(0, 0.05, arch.param_count) + (1j * rng.normal(0, 0.05, arch.param_count) if cplx else 0)
    params = A.AnsatzParameters(arch, theta)
    ref = A.build_batch(params, x, rng.normal(-3, 0.1, rows))
    ld = ref.ld
    odt = torch.complex128 if cplx else torch.float64
    guard = 4096
    mark = complex(7.25, -3.5) if cplx else 7.25
    obig = torch.full((rows * ld + guard,), mark, dtype=odt, device="cuda")
    sbig = torch.full((2, ld + guard), mark, dtype=odt, device="cuda")
    o = obig[: rows * ld].view(rows, ld)
    xt = A._x_device(x, n_in, torch.device("cuda"))
    A.fill_o_rows(params, xt, o, ref.weights, ref.gradient_coefficients(ref._stats_e), sbig[0, :ld], sbig[1, :ld])
    torch.cuda.synchronize()
    assert bool((obig[rows * ld:] == mark).all()), "O overrun"
    assert bool((sbig[:, ld:] == mark).all()), "statistics overrun"
    assert torch.equal(o[:, : ref.param_count], ref.o_matrix[:, : ref.param_count])


@pytest.mark.parametrize("mode", ["stored", "otf"])
def test_connected_workspace_canary(E, mode):
    """The connected completion (partner dots, per-row CSR, additive row term)
    stays inside its cache workspace."""
    import torch

    from paper_2601_01437_b200 import ansatz as A, synthetic as S

    cfg = S.CONFIGS[1].with_rows(777)
    inp = S.make_inputs(cfg)
    arch = A.RBMArchitecture(cfg.n_inputs, cfg.hidden)
    params = A.AnsatzParameters(arch, inp.theta)
    batch = A.build_batch(params, inp.x, inp.e_loc, mode=mode)
    en = E.estimate_energy(batch)
    partners, elements, indptr, dist = S.connected_partners(inp.x, 3, seed=9)
    cache = A.build_connected_cache(params, batch, inp.x, partners, elements, indptr, dist_index=dist)
    v = np.random.default_rng(4).standard_normal(arch.param_count)
    ref = np.asarray(E.connected_heff_matvec(batch, en, cache, v))
    nbytes = cache.workspace(batch).numel()
    guard = 1 << 20
    big = torch.full((nbytes + guard,), 0x5A, dtype=torch.uint8, device="cuda")
    cache._ws[batch._stream()] = big[:nbytes]  # this stream's workspace, exactly sized
    got = np.asarray(E.connected_heff_matvec(batch, en, cache, v))
    torch.cuda.synchronize()
    assert bool((big[nbytes:] == 0x5A).all()), "connected workspace overrun"
    assert np.array_equal(got, ref)


def test_wide_path_many_blocks_bitwise_stable(E):
    """The single-read wide path (IRL_MVP_WIDE) exchanges every row block's
    dots across its persistent grid through tagged records in a 64-slot ring
    (csrc/wide.cuh); with many blocks (ring wrap-around), repeated products must
    be bit-identical and match the two-pass product (a record read before its
    writer finished shows up as a small, varying error)."""
    import torch

    from paper_2601_01437_b200 import ansatz as A, synthetic as S

    cfg = S.CONFIGS[5].with_rows(1536)
    inp = S.make_inputs(cfg)
    arch = A.MLPArchitecture(cfg.n_inputs, cfg.hidden)
    b = A.build_batch(A.AnsatzParameters(arch, inp.theta), inp.x, inp.e_loc)
    en = E.estimate_energy(b)
    v = torch.as_tensor(np.random.default_rng(8).standard_normal(arch.param_count), device="cuda")
    first = E.heff_matvec(b, en, v, mode=4)
    two = E.heff_matvec(b, en, v, mode=2)
    assert rel(first.cpu().numpy(), two.cpu().numpy()) < 1e-12
    for _ in range(24):
        assert torch.equal(E.heff_matvec(b, en, v, mode=4), first)


def test_two_streams_two_batches(E):
    """Re-entrancy (include/irl_sr.h: every entry takes a stream, no global
    mutable state): products on two batches issued alternately on two CUDA
    streams without host synchronisation equal the serial results bit for bit."""
    import torch

    rng = np.random.default_rng(21)
    cases = []
    for n, p in ((3001, 157), (2048, 611)):
        o, e, w = random_batch(rng, n, p)
        b = E.SampleBatch(None, w, e, o, n)
        en = E.estimate_energy(b)
        vs = [torch.as_tensor(rng.standard_normal(p), device="cuda") for _ in range(4)]
        cases.append((b, en, vs))
    serial = [[E.heff_matvec(b, en, v).clone() for v in vs] for b, en, vs in cases]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [[None] * 4, [None] * 4]
    for k in range(4):
        for i, (b, en, vs) in enumerate(cases):
            with torch.cuda.stream(streams[i]):
                outs[i][k] = E.heff_matvec(b, en, vs[k])
    torch.cuda.synchronize()
    for i in range(2):
        for k in range(4):
            assert torch.equal(outs[i][k], serial[i][k])


@pytest.mark.gpu
def test_two_streams_one_batch(E):
    """Products on ONE batch issued alternately on two streams (each stream gets
    its own workspace and staging buffers) equal the serial results bit for bit,
    stored rows / fused / two-pass shapes alike."""
    import torch

    rng = np.random.default_rng(22)
    for n, p in ((3001, 157), (4096, 6600)):
        o, e, w = random_batch(rng, n, p)
        b = E.SampleBatch(None, w, e, o, n)
        en = E.estimate_energy(b)
        vs = [torch.as_tensor(rng.standard_normal(p), device="cuda") for _ in range(8)]
        serial = [E.heff_matvec(b, en, v).clone() if k % 2 == 0 else E.qgt_matvec(b, v).clone()
                  for k, v in enumerate(vs)]
        torch.cuda.synchronize()
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        outs = [None] * 8
        for k, v in enumerate(vs):
            with torch.cuda.stream(streams[k % 2]):
                outs[k] = E.heff_matvec(b, en, v) if k % 2 == 0 else E.qgt_matvec(b, v)
        torch.cuda.synchronize()
        for k in range(8):
            assert torch.equal(outs[k], serial[k]), (n, p, k)


@pytest.mark.parametrize("p", [20, 60, 90])
def test_rows_path_o_at_end_of_allocation(E, p):
    """Narrow rows (ld = 16-48 units, the warp-per-row kernel reads 128-unit
    row windows): with O placed so that its last row ends exactly at the end of
    a raw 2 MiB cudaMalloc block, the product reads nothing past O (a read past
    the mapping would fault) and matches the oracle."""
    import ctypes

    import torch

    from paper_2601_01437_b200 import _lib

    rt = ctypes.CDLL("libcudart.so.12")
    lib = _lib.lib()
    ld = _lib.padded_ld(p, False)
    n = 301
    nbytes = n * ld * 8
    block = 2 << 20
    assert nbytes < block
    base = ctypes.c_void_p()
    assert rt.cudaMalloc(ctypes.byref(base), ctypes.c_size_t(block)) == 0
    try:
        rng = np.random.default_rng(p)
        o, e, w = random_batch(rng, n, p)
        opad = np.zeros((n, ld))
        opad[:, :p] = o
        src = torch.as_tensor(opad, device="cuda")
        o_ptr = base.value + block - nbytes
        assert rt.cudaMemcpy(ctypes.c_void_p(o_ptr), ctypes.c_void_p(src.data_ptr()), ctypes.c_size_t(nbytes),
                             3) == 0  # device to device
        mean, _, _ = oest.energy(w, e, n)
        coeff = torch.as_tensor(w * (e - mean), device="cuda")
        obar = torch.zeros(ld, dtype=torch.float64, device="cuda")
        obar[:p] = torch.as_tensor(w @ o, device="cuda")
        v = rng.standard_normal(p)
        vd = torch.zeros(ld, dtype=torch.float64, device="cuda")
        vd[:p] = torch.as_tensor(v, device="cuda")
        out = torch.empty(ld, dtype=torch.float64, device="cuda")
        ws_bytes = int(lib.irl_mvp_workspace_bytes(n, ld, 0))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
        rc = lib.irl_mvp_f64(ctypes.c_void_p(o_ptr), n, p, ld, obar.data_ptr(), coeff.data_ptr(), vd.data_ptr(),
                             out.data_ptr(), None, None, None, 3, ws.data_ptr(), ws_bytes, _lib.stream_handle())
        assert rc == _lib.IRL_OK, lib.irl_last_error()
        torch.cuda.synchronize()
        assert rel(out[:p].cpu().numpy(), oest.heff(w, e, o, mean, v)) < 1e-10
    finally:
        torch.cuda.synchronize()
        rt.cudaFree(base)


@pytest.mark.parametrize("units,n,cplx", [
    (148 * 97, 211, False),    # 97 units per SM slice: 3 full lane-rows + 1 unit in the side buffer
    (148 * 120, 130, False),   # + 24 units: the widest side buffer
    (148 * 125, 130, False),   # + 29 units: all four lane-rows in TMEM (no side buffer)
    (148 * 97 + 5, 77, True),  # complex rows, uneven slices
    (148 * 177 - 3, 70, False),  # 6 lane-rows per lane (cfg5's instance), rows not a multiple of the block
])
def test_wide_path_lane_row_split(E, units, n, cplx):
    """The wide product parks a part's full lane-rows (32 units) in tensor
    memory and its partly filled last lane-row in a shared-memory side buffer
    (csrc/wide.cuh, SIDE instances): products over slice widths on both sides
    of the split match the oracle's est:171-186 restatement and the two-pass
    path, and repeat bit for bit."""
    import torch

    from paper_2601_01437_b200 import _lib

    rng = np.random.default_rng(units + n)
    p = units if cplx else 2 * units - 1
    o, e, w = random_batch(rng, n, p, cplx=cplx, exact=True)
    b = E.SampleBatch(None, w, e, o, 0, kind="hermitian" if cplx else None)
    en = E.estimate_energy(b)
    mean, _, _ = oest.energy(w, e, 0)
    assert _lib.mvp_plan(b.n_rows, b.ld, b.is_complex, 4)["path"] == "wide"
    v = rng.standard_normal(p) + (1j * rng.standard_normal(p) if cplx else 0)
    ref = oest.heff_hermitian(w, e, o, mean, v) if cplx else oest.heff(w, e, o, mean, v)
    vt = torch.as_tensor(v, device="cuda")
    first = E.heff_matvec(b, en, vt, mode=4)
    assert rel(first.cpu().numpy(), ref) < 1e-10
    assert rel(first.cpu().numpy(), E.heff_matvec(b, en, vt, mode=2).cpu().numpy()) < 1e-12
    for _ in range(5):
        assert torch.equal(E.heff_matvec(b, en, vt, mode=4), first)
