"""K-cg parity: the persistent device CG against the oracle's pcg_solve / block_solve.

Bars (BASELINE.json north_star): solutions within 1e-8 relative, iteration
counts within +-2, identical converged flags, identical breakdown iteration.
T1 = reference chain model (converges); T2 = BASELINE Hermite beam at a fixed
iteration budget (rtol 1e-10 is unreachable in FP64 there).
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["auto", "cluster_v1", "stream", "stream_flat", "banded", "general"])
def cg_path(request, mg):
    """Every parity case runs through every CG kernel: cluster-resident (auto on these
    on-chip sizes), the streaming kernel (slab x point tile plan and one contiguous row range per block), the banded
    grid kernel and the general CSR kernel."""
    ctx = mg.default_context()
    if request.param == "stream_flat":
        ctx.set_option("stream_tiles", 0)
        ctx.set_cg_path("stream")
    else:
        if request.param == "stream":
            ctx.set_option("stream_tiles", 2)  # the tile plan wherever its shape allows, whatever the size
        ctx.set_cg_path(request.param)
    yield request.param
    ctx.set_cg_path("auto")
    ctx.set_option("stream_tiles", 1)


def test_path_selection(mg, oracle, cg_path):
    M, D, K = oracle.hermite_generate(300)
    A = oracle.shifted_operator(M, D, K, 100.0)
    P = oracle.spai_ls(A, None, 1)
    mg.pcg_solve(A, [P], np.ones(600), maxit=5)
    # A^2-pattern factor: 10 entries per row -> the shared-memory cluster kernel (v1); v2 packs <= 8
    assert mg.default_context().last_cg_path == {"auto": "cluster_v1", "cluster_v1": "cluster_v1", "stream": "stream",
                                                  "stream_flat": "stream", "banded": "banded",
                                                  "general": "general"}[cg_path]
    if cg_path == "auto":
        P1 = oracle.spai_ls(A, None, 0)
        mg.pcg_solve(A, [P1], np.ones(600), maxit=5)
        assert mg.default_context().last_cg_path == "cluster"
    # a wide operator (bandwidth > 64) always takes the general kernel
    from oracle import Csr
    rng = np.random.default_rng(9)
    W = np.eye(300) * 4.0
    for _ in range(40):
        i, j = rng.integers(0, 300, 2)
        if abs(i - j) > 70:
            W[i, j] = W[j, i] = 0.01
    want = oracle.pcg_solve(Csr.from_dense(W), [], np.ones(300))
    got = mg.pcg_solve(Csr.from_dense(W), [], np.ones(300))
    assert mg.default_context().last_cg_path == "general"
    assert rel(got["solution"], want["solution"]) < 1e-12


def _check(got, want, b=None, tol=1e-8, it_tol=2):
    assert abs(got["iterations"] - want["iterations"]) <= it_tol, (got["iterations"], want["iterations"])
    assert got["converged"] == want["converged"]
    assert rel(got["solution"], want["solution"]) < tol
    # the true residual b - A x is a cancellation; bound its difference by ||b||
    scale = np.max(np.abs(b)) if b is not None else np.max(np.abs(want["residual"]))
    assert np.max(np.abs(got["residual"] - want["residual"])) <= tol * max(scale, 1e-300)


@pytest.mark.parametrize("kscale,s", [(0.01, 0.025), (0.01, 1.0), (1.0, 10.0), (1.0, 100.0), (100.0, 100.0)])
def test_t1_pcg_with_mr_spai(mg, oracle, kscale, s):
    M, D, K = oracle.chain_generate(2000, consistent=True, stiffness_scale=kscale)
    A = oracle.shifted_operator(M, D, K, s)
    P, _ = oracle.spai_build(A, mode=1)
    b = np.zeros(2000)
    b[0] = 1.0
    want = oracle.pcg_solve(A, [P], b, rtol=1e-10)
    got = mg.pcg_solve(A, [P], b, rtol=1e-10, history_cap=64)
    _check(got, want, b)
    assert want["converged"]
    h = min(want["iterations"], got["iterations"])
    assert rel(got["relres_history"][:h], want["relres_history"][:h]) < 1e-6


def test_t1_plain_cg(mg, oracle):
    M, D, K = oracle.chain_generate(500, consistent=True, stiffness_scale=1.0)
    A = oracle.shifted_operator(M, D, K, 3.0)
    b = np.random.default_rng(3).standard_normal(500)
    _check(mg.pcg_solve(A, [], b, rtol=1e-10), oracle.pcg_solve(A, [], b, rtol=1e-10), b)


def test_t1_chain_of_two(mg, oracle):
    M, D, K = oracle.chain_generate(2000, consistent=True, stiffness_scale=1.0)
    A1 = oracle.shifted_operator(M, D, K, 10.0)
    A2 = oracle.shifted_operator(M, D, K, 12.5)
    P, _ = oracle.spai_build(A1, mode=1)
    Q, _ = oracle.spai_update(A1, A2, mode=1)
    b = np.zeros(2000)
    b[-1] = 1.0
    _check(mg.pcg_solve(A2, [Q, P], b), oracle.pcg_solve(A2, [Q, P], b), b)


def test_block_solve_zero_column_and_multi_rhs(mg, oracle):
    M, D, K = oracle.chain_generate(1500, consistent=True, stiffness_scale=1.0)
    A = oracle.shifted_operator(M, D, K, 5.0)
    P, _ = oracle.spai_build(A, mode=1)
    rng = np.random.default_rng(11)
    B = rng.standard_normal((1500, 4))
    B[:, 2] = 0.0
    want = oracle.block_solve(A, [P], B)
    got = mg.block_solve(A, [P], B)
    assert rel(got.X, want["X"]) < 1e-8
    np.testing.assert_array_equal(got.X[:, 2], 0.0)
    assert got.iterations[2] == 0 and got.converged[2]
    assert np.all(np.abs(got.iterations - want["iterations"]) <= 2)
    assert got.all_converged == want["all_converged"]


def test_multi_shift_batch(mg, oracle):
    """8 shifts x 2 rhs in one persistent kernel == 8 separate oracle block solves."""
    M, D, K = oracle.chain_generate(3000, consistent=True, stiffness_scale=1.0)
    shifts = [10.0 ** (1 + 3 * i / 7) for i in range(8)]
    ops = [oracle.shifted_operator(M, D, K, s) for s in shifts]
    Ps = [oracle.spai_build(A, mode=1)[0] for A in ops]
    B = np.zeros((3000, 2))
    B[0, 0] = 1.0
    B[1500, 1] = 1.0
    res = mg.cg_solve_batched(ops, [[P] for P in Ps], B, rtol=1e-10)
    for A, P, r in zip(ops, Ps, res):
        want = oracle.block_solve(A, [P], B)
        assert rel(r.X, want["X"]) < 1e-8
        assert np.all(np.abs(r.iterations - want["iterations"]) <= 2)


def test_many_shifts_split_launches(mg, oracle):
    """150 shifts x 1 rhs (more than one launch's 128 systems, and more points than a
    kernel's reduction table held before re-indexing) == per-shift oracle solves."""
    M, D, K = oracle.chain_generate(200, consistent=True, stiffness_scale=1.0)
    shifts = [10.0 ** (1 + 3 * i / 149) for i in range(150)]
    ops = [oracle.shifted_operator(M, D, K, s) for s in shifts]
    b = np.zeros(200)
    b[7] = 1.0
    res = mg.cg_solve_batched(ops, [[] for _ in ops], b, rtol=1e-10)
    for A, r in zip(ops, res):
        want = oracle.pcg_solve(A, [], b, rtol=1e-10)
        assert rel(r.X[:, 0], want["solution"]) < 1e-8
        assert abs(int(r.iterations[0]) - want["iterations"]) <= 2


def test_t2_hermite_fixed_k_iterates(mg, oracle):
    """BASELINE config 1 shape: n=2000, s=100, LS-SPAI (A pattern), fixed budget."""
    M, D, K = oracle.hermite_generate(1000)
    A = oracle.shifted_operator(M, D, K, 100.0)
    P = oracle.spai_ls(A, None, 0)
    b = np.zeros(2000)
    b[1998] = 1.0
    for k in (1, 10, 100):
        want = oracle.pcg_solve(A, [P], b, rtol=1e-10, maxit=k)
        got = mg.pcg_solve(A, [P], b, rtol=1e-10, maxit=k)
        assert got["iterations"] == want["iterations"] == k
        assert got["converged"] == want["converged"]
        assert rel(got["solution"], want["solution"]) < 1e-8


def test_breakdown_iteration_parity(mg, oracle):
    from oracle import Csr, OracleError
    A = Csr.from_dense(np.diag([1.0, -1.0, 2.0]))
    b = np.array([1.0, 1.0, 0.0])
    with pytest.raises(OracleError) as eo:
        oracle.pcg_solve(A, [], b)
    with pytest.raises(mg.BreakdownError) as eg:
        mg.pcg_solve(A, [], b)
    assert eg.value.iteration == eo.value.index == 0
    with pytest.raises(mg.BreakdownError) as eb:
        mg.block_solve(A, [], np.stack([np.array([1.0, 0.0, 0.0]), b], axis=1))
    assert "block_solve: column 1" in str(eb.value) and eb.value.iteration == 0


def test_maxit_zero_and_budget(mg, oracle):
    M, D, K = oracle.chain_generate(800, consistent=True, stiffness_scale=1.0)
    A = oracle.shifted_operator(M, D, K, 1.0)
    b = np.ones(800)
    for k in (0, 1, 2):
        _check(mg.pcg_solve(A, [], b, maxit=k), oracle.pcg_solve(A, [], b, maxit=k), b, it_tol=0)


def test_tight_rtol_restart_branch(mg, oracle):
    """rtol near the FP64 floor exercises the confirm / restart branch (krylov.cpp:77-103)."""
    M, D, K = oracle.chain_generate(1000, consistent=True, stiffness_scale=1.0)
    A = oracle.shifted_operator(M, D, K, 0.5)
    b = np.random.default_rng(5).standard_normal(1000)
    want = oracle.pcg_solve(A, [], b, rtol=1e-15, maxit=400)
    got = mg.pcg_solve(A, [], b, rtol=1e-15, maxit=400)
    assert got["converged"] == want["converged"]
    assert rel(got["solution"], want["solution"]) < 1e-8


def test_zero_rhs(mg, oracle):
    M, D, K = oracle.chain_generate(100)
    got = mg.pcg_solve(K, [], np.zeros(100))
    assert got["iterations"] == 0 and got["converged"]
    np.testing.assert_array_equal(got["solution"], 0.0)


@pytest.mark.parametrize("m", [2, 4])
def test_multi_rhs_restart_plain(mg, oracle, m):
    """P = I with m right-hand sides at an rtol near the FP64 floor: the true-residual confirm /
    restart branch per column (krylov.cpp:77-103).  On the stream kernel m = 2 runs the deferred
    x~ update (folded into phase A, the check pass adds the pending alpha d), m = 4 does not."""
    M, D, K = oracle.chain_generate(1200, consistent=True, stiffness_scale=1.0)
    A = oracle.shifted_operator(M, D, K, 0.5)
    B = np.random.default_rng(m).standard_normal((1200, m))
    want = oracle.block_solve(A, [], B, rtol=1e-15, maxit=400)
    got = mg.block_solve(A, [], B, rtol=1e-15, maxit=400)
    assert got.all_converged == want["all_converged"]
    assert rel(got.X, want["X"]) < 1e-8
    assert np.all(np.abs(np.asarray(got.iterations) - np.asarray(want["iterations"])) <= 2)


def test_mixed_structures_in_one_batch(mg, oracle):
    """Operators of different CSR structure in one batch (Hermite beam and chain model, same n):
    the streaming kernel shares ELL offsets only between structurally equal points (device
    pattern-equality flags), so every point must still match its own oracle solve."""
    Mh, Dh, Kh = oracle.hermite_generate(1000)
    Mc, Dc, Kc = oracle.chain_generate(2000, consistent=True, stiffness_scale=1.0)
    ops = [oracle.shifted_operator(Mh, Dh, Kh, 100.0), oracle.shifted_operator(Mc, Dc, Kc, 10.0),
           oracle.shifted_operator(Mh, Dh, Kh, 300.0), oracle.shifted_operator(Mc, Dc, Kc, 30.0)]
    Ps = [oracle.spai_ls(A, None, 0) for A in ops]
    b = np.zeros(2000)
    b[1998] = 1.0
    res = mg.cg_solve_batched(ops, [[P] for P in Ps], b, rtol=1e-10, maxit=120)
    for A, P, r in zip(ops, Ps, res):
        want = oracle.pcg_solve(A, [P], b, rtol=1e-10, maxit=120)
        assert int(r.iterations[0]) == want["iterations"]
        assert rel(r.X[:, 0], want["solution"]) < 1e-8
