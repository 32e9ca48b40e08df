"""The drop-in SolveBackend through its C entry points (include/mor_cuda.h): the call sequence of
the reference's own driver -- prepare(sys, points, outer), then solve(i, F) per point
(airga.cpp:108-181, 374-381) -- against the oracle's block_solve on the same operators and
factors.  Covers the speculative batched solve (solve(i, F) served from prepare), the on-demand
path (another rhs, a repeated request), and a system edited in place between prepares."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

NE, K_IT = 1000, 200
SHIFTS = [10.0, 100.0, 1000.0, 1e4]
PAT = 0x10  # LS-SPAI on A's pattern, column-equilibrated


def _F(n, m=2):
    F = np.zeros((n, m), order="F")
    F[n - 2, 0] = 1.0
    if m > 1:
        F[n // 2, 1] = 1.0
    return F


def _want(oracle, M, D, K, s, B):
    A = oracle.shifted_operator(M, D, K, s)
    P = oracle.spai_ls(A, None, PAT)
    return oracle.block_solve(A, [P], B, rtol=1e-10, maxit=K_IT)


@pytest.fixture
def plug(mg):
    from paper_1606_01216_b200.plugin import PluginBackend
    b = PluginBackend(solver="cg_spai", algorithm="ls", ls_pattern=PAT, maxit=K_IT)
    yield b
    b.close()


def test_prepare_then_solve_every_point(mg, oracle, plug):
    M, D, K = oracle.hermite_generate(NE)
    n = M.nrows
    F = _F(n)
    plug.set_system(M, D, K, F)
    secs = plug.prepare(SHIFTS, 1)
    assert secs.shape == (len(SHIFTS),) and np.all(secs >= 0)
    for i, s in enumerate(SHIFTS):
        X = np.zeros((n, 2), order="F")
        TR = np.zeros((n, 2), order="F")
        it, conv = plug.solve(i, F, X=X, TR=TR)
        want = _want(oracle, M, D, K, s, F)
        np.testing.assert_array_equal(it, want["iterations"])
        assert rel(X, want["X"]) < 1e-8
        assert rel(TR, want["true_residuals"]) < 1e-6


def test_other_rhs_and_repeated_request_solve_on_demand(mg, oracle, plug):
    M, D, K = oracle.hermite_generate(NE)
    n = M.nrows
    F = _F(n)
    plug.set_system(M, D, K, F)
    plug.prepare(SHIFTS, 1)
    X1 = np.zeros((n, 2), order="F")
    plug.solve(1, F, X=X1)  # from prepare's batched solve
    X2 = np.zeros((n, 2), order="F")
    plug.solve(1, F, X=X2)  # handed out already: solved again on demand
    assert rel(X2, X1) < 1e-10
    # other unit loads (a dense rhs on this cond ~1e13 beam amplifies the reduction-order noise of
    # any two CG implementations far past 1e-8 within 200 iterations; unit loads do not)
    G = np.zeros((n, 2), order="F")
    G[n // 4, 0] = 1.0
    G[3 * n // 4 + 1, 1] = 1.0
    XG = np.zeros((n, 2), order="F")
    it, _ = plug.solve(2, G, X=XG)
    want = _want(oracle, M, D, K, SHIFTS[2], G)
    np.testing.assert_array_equal(it, want["iterations"])
    assert rel(XG, want["X"]) < 1e-8


def test_system_edited_between_prepares(mg, oracle, plug):
    """The same SecondOrderSystem object with new K values: prepare must use them (the reference
    rebuilds shifted_operator(sys, s) on every prepare, airga.cpp:110-116)."""
    from oracle import Csr
    M, D, K = oracle.hermite_generate(NE)
    n = M.nrows
    F = _F(n)
    plug.set_system(M, D, K, F)
    plug.prepare(SHIFTS, 1)
    plug.solve(0, F)
    K2 = Csr(K.nrows, K.ncols, K.row_ptr.copy(), K.col_idx.copy(), K.values * 2.0)
    plug.set_system(M, D, K2, F)
    plug.prepare(SHIFTS, 2)
    X = np.zeros((n, 2), order="F")
    it, _ = plug.solve(0, F, X=X)
    want = _want(oracle, M, D, K2, SHIFTS[0], F)
    np.testing.assert_array_equal(it, want["iterations"])
    assert rel(X, want["X"]) < 1e-8


def test_spai_error_surfaces_from_prepare(mg, oracle):
    """The unscaled LS on A's pattern rank-flushes at n = 1e6 on this beam: prepare raises the
    NumericalError, as the C++ backend would."""
    from paper_1606_01216_b200.plugin import PluginBackend
    b = PluginBackend(solver="cg_spai", algorithm="ls", ls_pattern=0, maxit=5)
    M, D, K = oracle.hermite_generate(500000)
    b.set_system(M, D, K, _F(M.nrows, 1))
    with pytest.raises(mg.NumericalError, match="rank-deficient"):
        b.prepare([100.0], 1)
    b.close()


def test_multi_device_backend_shards_points(mg, oracle):
    """mor::MultiDeviceCgBackend: point i on devices[i % N], prepared concurrently.  With one GPU the
    two device slots are two contexts on cuda:0 (independent streams); results per point as the
    single-device backend's (oracle within 1e-8, same iteration counts)."""
    from paper_1606_01216_b200.plugin import PluginBackend
    b = PluginBackend(solver="cg_spai", algorithm="ls", ls_pattern=PAT, maxit=K_IT, devices=[0, 0])
    M, D, K = oracle.hermite_generate(NE)
    n = M.nrows
    F = _F(n)
    b.set_system(M, D, K, F)
    secs = b.prepare(SHIFTS, 1)
    assert secs.shape == (len(SHIFTS),)
    for i, s in enumerate(SHIFTS):
        X = np.zeros((n, 2), order="F")
        it, _ = b.solve(i, F, X=X)
        want = _want(oracle, M, D, K, s, F)
        np.testing.assert_array_equal(it, want["iterations"])
        assert rel(X, want["X"]) < 1e-8
    b.close()
