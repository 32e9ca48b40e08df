"""Parity at the benchmark's own workload (bench.py default = BASELINE configs[1] shape):
Hermite beam ne = 10^4 (n = 2e4), 8 shifts log-spaced in [10, 1e4], LS-SPAI on A's pattern,
the fixed 1000-iteration CG budget.  SURVEY.md 8(c) T2: fixed-k iterate parity (the
device's fixed reduction trees vs the reference's serial sums, measured noise ~1e-13 at
k = 1000), identical iteration counts / converged flags, no breakdown.  Every CG kernel
the bench can select is checked against the same oracle solves.
"""
import functools

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

NE, BUDGET = 10000, 1000
SHIFTS = [10.0 ** (1 + 3 * i / 7) for i in range(8)]


@functools.lru_cache(maxsize=1)
def _oracle_case():
    from oracle import Oracle
    orc = Oracle()
    M, D, K = orc.hermite_generate(NE)
    n = M.nrows
    b = np.zeros(n)
    b[n - 2] = 1.0
    ops, facs, sols = [], [], []
    for s in SHIFTS:
        A = orc.shifted_operator(M, D, K, s)
        P = orc.spai_ls(A, None, 0)
        r = orc.pcg_solve(A, [P], b, rtol=1e-10, maxit=BUDGET)
        ops.append(A)
        facs.append(P)
        sols.append(r)
    return (M, D, K), ops, facs, b, sols


@pytest.mark.parametrize("path", ["auto", "stream", "stream_flat", "banded"])
def test_bench_workload_iterate_parity(mg, path):
    (M, D, K), ops, facs, b, want = _oracle_case()
    ctx = mg.default_context()
    ctx.set_option("stream_tiles", 0 if path == "stream_flat" else 2)
    ctx.set_cg_path("stream" if path == "stream_flat" else path)
    try:
        # the bench's device pipeline: assembly + batched LS-SPAI + one batched solve
        dops = mg.shifted_operators(M, D, K, SHIFTS, ctx=ctx)
        dfac = mg.spai_ls_batched(dops, None, mg.PATTERN_A, ctx=ctx)
        for d, a in zip(dops, ops):
            np.testing.assert_array_equal(d.download().values, a.values)  # bitwise assembly
        for f, p in zip(dfac, facs):
            np.testing.assert_array_equal(f.matrix.download().values, p.values)  # bitwise LS-SPAI
        res = mg.cg_solve_batched(dops, [[f.matrix] for f in dfac], b, rtol=1e-10, maxit=BUDGET, ctx=ctx)
        if path == "auto":
            assert ctx.last_cg_path == "cluster"
        for r, w in zip(res, want):
            assert int(r.iterations[0]) == w["iterations"] == BUDGET
            assert bool(r.converged[0]) == w["converged"]
            assert rel(r.X[:, 0], w["solution"]) < 1e-8
    finally:
        ctx.set_cg_path("auto")
        ctx.set_option("stream_tiles", 1)


def test_config3_tile_plan_matches_contiguous_plan(mg):
    """BASELINE configs[3] shape (n = 1e6, m = 4, 16 shifts, P = I) through the streaming
    kernel: the slab x point tile plan (four tiles per block, the 16 points of a slab in flight
    together) against one contiguous row range per block, after 40 iterations.  Same arithmetic
    per element; only the dot-product trees differ, so the iterates agree to rounding noise."""
    ne, m, k = 500000, 4, 40
    shifts = [10.0 ** (1 + 3 * i / 15) for i in range(16)]
    ctx = mg.default_context()
    M, D, K = mg.model_hermite_device(ne, ctx=ctx)
    n = 2 * ne
    B = np.zeros((n, m))
    for c in range(m):
        B[2 * ((c + 1) * ne // m) - 2, c] = 1.0
    ops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
    ctx.set_cg_path("stream")
    try:
        ctx.set_option("stream_tiles", 0)
        ref = mg.cg_solve_batched(ops, [[] for _ in ops], B, rtol=1e-10, maxit=k, ctx=ctx)
        ctx.set_option("stream_tiles", 1)
        got = mg.cg_solve_batched(ops, [[] for _ in ops], B, rtol=1e-10, maxit=k, ctx=ctx)
    finally:
        ctx.set_cg_path("auto")
        ctx.set_option("stream_tiles", 1)
    for g, r in zip(got, ref):
        np.testing.assert_array_equal(g.iterations, r.iterations)
        assert rel(g.X, r.X) < 1e-10
        assert np.all(np.isfinite(g.X)) and np.max(np.abs(g.X)) > 0


@pytest.mark.parametrize("where", ["device", "host"])
def test_shifted_solve_one_call_matches_oracle(mg, where):
    """mgpu_shifted_solve (the bench's step: assembly + LS-SPAI + batched solve in one library
    call) on the configs[1] workload against the oracle's separate reference calls."""
    import torch
    (M, D, K), ops, facs, b, want = _oracle_case()
    ctx = mg.default_context()
    n, l = M.nrows, len(SHIFTS)
    if where == "device":
        dev = torch.device("cuda", 0)
        B_dev = torch.tensor(b[None, :], dtype=torch.float64, device=dev)
        X_dev = torch.empty((l, 1, n), dtype=torch.float64, device=dev)
        it, cv, st, bd, ph = mg.shifted_solve_device(M, D, K, SHIFTS, mg.PATTERN_A, B_dev, X_dev, rtol=1e-10,
                                                     maxit=BUDGET, ctx=ctx)
        X = X_dev.cpu().numpy()
        assert ph.shape == (3,) and np.all(ph >= 0)
    else:
        X = np.zeros((l, 1, n))
        status, it, cv, st, bd, ph = mg.shifted_solve_raw(ctx, M, D, K, SHIFTS, mg.PATTERN_A, 1, b.ctypes.data, 0,
                                                          1e-10, BUDGET, mg.mgpu.MGPU_HOST, X.ctypes.data, 0, 0)
        assert status == mg.mgpu.MGPU_OK
    assert np.all(st == 0)
    for p, w in enumerate(want):
        assert int(it[p]) == w["iterations"] == BUDGET
        assert bool(cv[p]) == w["converged"]
        assert rel(X[p, 0], w["solution"]) < 1e-8


def test_shifted_solve_reports_argument_errors(mg):
    M, D, K = mg.model_hermite(50)
    ctx = mg.default_context()
    X = np.zeros((1, 1, 100))
    b = np.ones(100)
    status, *_ = mg.shifted_solve_raw(ctx, M, D, K, [10.0], 7, 1, b.ctypes.data, 0, 1e-10, 10, mg.mgpu.MGPU_HOST,
                                      X.ctypes.data, 0, 0)
    assert status == mg.mgpu.MGPU_ERR_ARG


@pytest.mark.parametrize("ne,m,nshift,k", [(500000, 4, 2, 30), (5000000, 1, 1, 8)])
def test_full_size_iterates_match_oracle(mg, oracle, ne, m, nshift, k):
    """BASELINE configs[3] / configs[4] sizes (n = 1e6 with m = 4, n = 1e7) through the
    streaming kernel (P = I, as the bench runs them) against the oracle's block_solve after k
    iterations: same iteration count, iterates within 1e-8."""
    M, D, K = oracle.hermite_generate(ne)
    n = M.nrows
    B = np.zeros((n, m))
    for c in range(m):
        B[2 * ((c + 1) * ne // m) - 2, c] = 1.0
    shifts = [10.0 ** (1 + 3 * i / 15) for i in range(16)][:nshift]
    ctx = mg.default_context()
    res = mg.cg_solve_batched([oracle.shifted_operator(M, D, K, s) for s in shifts], [[] for _ in shifts], B,
                              rtol=1e-10, maxit=k, ctx=ctx)
    assert ctx.last_cg_path == "stream"
    for s, r in zip(shifts, res):
        want = oracle.block_solve(oracle.shifted_operator(M, D, K, s), [], B, rtol=1e-10, maxit=k)
        np.testing.assert_array_equal(r.iterations, want["iterations"])
        assert rel(r.X, want["X"]) < 1e-8


def test_shifted_solve_raises_the_spai_error(mg):
    """On the BASELINE beam at n = 5e5 the LS problems on A's pattern are rank-deficient
    (DESIGN.md 4): the one-call path raises the same NumericalError as spai_ls_batched and
    leaves the context usable."""
    import torch
    ctx = mg.default_context()
    M, D, K = mg.model_hermite_device(250000, ctx=ctx)
    n = 500000
    dev = torch.device("cuda", 0)
    B_dev = torch.zeros((1, n), dtype=torch.float64, device=dev)
    B_dev[0, n - 2] = 1.0
    X_dev = torch.empty((2, 1, n), dtype=torch.float64, device=dev)
    with pytest.raises(mg.NumericalError):
        mg.shifted_solve_device(M, D, K, [100.0, 1000.0], mg.PATTERN_A, B_dev, X_dev, maxit=5, ctx=ctx)
    ops = mg.shifted_operators(M, D, K, [100.0, 1000.0], ctx=ctx)
    with pytest.raises(mg.NumericalError):
        mg.spai_ls_batched(ops, None, mg.PATTERN_A, ctx=ctx)
    it, cv, st, bd, ph = mg.shifted_solve_device(M, D, K, [100.0], -1, B_dev, X_dev[:1], maxit=5, ctx=ctx)
    assert int(it[0]) == 5


@pytest.mark.parametrize("ne,m,pattern,nshift,k", [(500000, 4, 0x11, 2, 30), (5000000, 4, 0x10, 1, 8)])
def test_full_size_preconditioned_matches_oracle(mg, oracle, ne, m, pattern, nshift, k):
    """BASELINE configs[3] (n = 1e6, m = 4, column-equilibrated LS-SPAI on the A^2 pattern) and
    configs[4] (n = 1e7, m = 4, A pattern): the bench's one-call device path (assembly, batched
    LS-SPAI, streaming CG) against the oracle's separate calls after k iterations: factors
    bitwise, same iteration counts, iterates within 1e-8."""
    import torch
    M, D, K = oracle.hermite_generate(ne)
    n = M.nrows
    B = np.zeros((n, m))
    for c in range(m):
        B[2 * ((c + 1) * ne // m) - 2, c] = 1.0
    shifts = [10.0 ** (1 + 3 * i / 15) for i in range(16)][:: 16 // nshift][:nshift]
    ctx = mg.default_context()
    dev = torch.device("cuda", 0)
    B_dev = torch.tensor(B.T.copy(), dtype=torch.float64, device=dev)
    X_dev = torch.empty((nshift, m, n), dtype=torch.float64, device=dev)
    it, cv, st, bd, ph = mg.shifted_solve_device(M, D, K, shifts, pattern, B_dev, X_dev, rtol=1e-10, maxit=k,
                                                 ctx=ctx)
    assert ctx.last_cg_path == "stream"
    X = X_dev.cpu().numpy()
    dops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
    dfac = mg.spai_ls_batched(dops, None, pattern, ctx=ctx)
    for p, s in enumerate(shifts):
        A = oracle.shifted_operator(M, D, K, s)
        P = oracle.spai_ls(A, None, pattern)
        np.testing.assert_array_equal(dfac[p].matrix.download().values, P.values)
        want = oracle.block_solve(A, [P], B, rtol=1e-10, maxit=k)
        np.testing.assert_array_equal(it[p * m:(p + 1) * m], want["iterations"])
        assert rel(X[p].T, want["X"]) < 1e-8


@pytest.mark.parametrize("ne,m,l,pattern,k", [(6000, 4, 4, 0x11, 40), (50000, 1, 8, 0, 60), (200000, 4, 16, 0x11, 12)])
def test_stream_kernel_reruns_are_bitwise_identical(mg, ne, m, l, pattern, k):
    """The streaming kernel has no floating-point atomics and fixed reduction trees, and its warps
    run ahead of each other between the stage barriers (per-warp buffer release, double-buffered
    stage 0): a missing barrier would show up as run-to-run differences.  Five runs of the same
    solve (the last shape with the tile plan and several tiles per block), every output array
    compared bitwise."""
    ctx = mg.default_context()
    M, D, K = mg.model_hermite_device(ne, ctx=ctx)
    shifts = [10.0 ** (1 + 3 * i / (l - 1)) for i in range(l)]
    ops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
    chains = [[f.matrix] for f in mg.spai_ls_batched(ops, None, pattern, ctx=ctx)]
    n = 2 * ne
    B = np.zeros((n, m))
    for c in range(m):
        B[2 * ((c + 1) * ne // m) - 2, c] = 1.0
    ctx.set_cg_path("stream")
    ctx.set_option("stream_tiles", 2)
    try:
        runs = [mg.cg_solve_batched(ops, chains, B, rtol=1e-10, maxit=k, ctx=ctx) for _ in range(5)]
        assert ctx.last_cg_path == "stream"
    finally:
        ctx.set_cg_path("auto")
        ctx.set_option("stream_tiles", 1)
    for other in runs[1:]:
        for a, b in zip(runs[0], other):
            np.testing.assert_array_equal(a.X, b.X)
            np.testing.assert_array_equal(a.iterations, b.iterations)
    assert np.all(np.isfinite(runs[0][0].X)) and np.max(np.abs(runs[0][0].X)) > 0


@pytest.mark.parametrize("n,m,l", [(2001, 1, 3), (4999, 3, 2), (20011, 1, 3), (20011, 4, 3), (6007, 7, 2), (6007, 5, 2)])
def test_stream_kernel_ragged_shapes_match_oracle(mg, oracle, n, m, l):
    """Odd orders (chunks whose element counts are odd: the pair loops' half-empty last pair and the
    point blocks' 16-byte alignment), right-hand-side counts that are not the kernel's template
    width (3 and 5 take the per-column scalar loops, 7 the generic ones) and, at n = 20011 with 3
    shifts, the tile plan with three tiles per block: the reference chain model (T1, converges in a
    few iterations) through the streaming kernel against the oracle's block_solve."""
    M, D, K = oracle.chain_generate(n, consistent=True, stiffness_scale=1.0)
    shifts = [10.0, 31.0, 100.0][:l]
    ops = [oracle.shifted_operator(M, D, K, s) for s in shifts]
    facs = [oracle.spai_build(A, mode=1)[0] for A in ops]
    rng = np.random.default_rng(n + m)
    B = rng.standard_normal((n, m))
    B[:, 0] = 0.0
    B[n // 3, 0] = 1.0
    if m > 2:
        B[:, 2] = 0.0  # a zero column: converged in 0 iterations, zeros out (krylov.cpp:44-51)
    ctx = mg.default_context()
    ctx.set_cg_path("stream")
    ctx.set_option("stream_tiles", 2)
    try:
        got = mg.cg_solve_batched(ops, [[f] for f in facs], B, rtol=1e-10, ctx=ctx)
        assert ctx.last_cg_path == "stream"
    finally:
        ctx.set_cg_path("auto")
        ctx.set_option("stream_tiles", 1)
    for A, P, g in zip(ops, facs, got):
        want = oracle.block_solve(A, [P], B, rtol=1e-10)
        assert np.all(np.abs(g.iterations - want["iterations"]) <= 2), (g.iterations, want["iterations"])
        assert bool(np.all(g.converged)) == bool(want["all_converged"])
        assert rel(g.X, want["X"]) < 1e-8
        if m > 2:
            assert not g.X[:, 2].any() and int(g.iterations[2]) == 0
