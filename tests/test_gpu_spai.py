"""SPAI parity: device MR-SPAI (reference Alg. 2/4, frozen and sequential) and LS-SPAI against the oracle.

Bar: SPAI entries within 1e-10 relative (BASELINE.json north_star), identical
sparsity pattern, per-column residuals within 1e-10, identical exception class
and column index.  SPEC.md known-answer tests included.
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def _csr_close(got, want, tol=1e-10):
    np.testing.assert_array_equal(got.row_ptr, want.row_ptr)
    np.testing.assert_array_equal(got.col_idx, want.col_idx)
    assert rel(got.values, want.values) <= tol


def _csr_equal(got, want):
    """LS-SPAI replays thin_qr's operation order: bitwise equal to the oracle."""
    np.testing.assert_array_equal(got.row_ptr, want.row_ptr)
    np.testing.assert_array_equal(got.col_idx, want.col_idx)
    np.testing.assert_array_equal(got.values, want.values)


# ------------------------------------------------------------------ MR-SPAI
@pytest.mark.parametrize("kscale,s", [(0.01, 1.0), (1.0, 1.0), (1.0, 10.0), (1.0, 100.0), (100.0, 10.0)])
def test_mr_build_t1(mg, oracle, kscale, s):
    M, D, K = oracle.chain_generate(2000, consistent=True, stiffness_scale=kscale)
    A = oracle.shifted_operator(M, D, K, s)
    want, wres = oracle.spai_build(A, mode=1)
    f = mg.spai_build(A, mode=mg.FROZEN)
    _csr_close(f.matrix.download(), want)
    assert rel(f.target_frob_residual, wres) < 1e-10


def test_mr_build_identity_mass(mg, oracle):
    M, D, K = oracle.chain_generate(1000, consistent=False)
    A = oracle.shifted_operator(M, D, K, 10.0)
    want, _ = oracle.spai_build(A, mode=1)
    _csr_close(mg.spai_build(A).matrix.download(), want)


def test_mr_update_t1(mg, oracle):
    M, D, K = oracle.chain_generate(2000, consistent=True, stiffness_scale=1.0)
    A1 = oracle.shifted_operator(M, D, K, 10.0)
    A2 = oracle.shifted_operator(M, D, K, 10.5)
    want, wres = oracle.spai_update(A1, A2, mode=1)
    f = mg.spai_update(A1, A2, mode=mg.FROZEN)
    _csr_close(f.matrix.download(), want)
    assert rel(f.target_frob_residual, wres) < 1e-10


def test_mr_update_identical_is_identity_bitwise(mg, oracle):
    """SPEC.md:256 / spai.hpp:57-60: K_new == K_old -> Q = I exactly, zero iterations."""
    M, D, K = oracle.chain_generate(500, consistent=True, stiffness_scale=1.0)
    A = oracle.shifted_operator(M, D, K, 10.0)
    Q = mg.spai_update(A, A).matrix.download()
    np.testing.assert_array_equal(Q.row_ptr, np.arange(501))
    np.testing.assert_array_equal(Q.col_idx, np.arange(500))
    np.testing.assert_array_equal(Q.values, 1.0)


def test_mr_update_scaled_identity(mg, oracle):
    from oracle import Csr
    I = Csr.from_dense(np.eye(6))
    Q = mg.spai_update(I, Csr.from_dense(2 * np.eye(6))).matrix.download()
    np.testing.assert_array_equal(Q.todense(), 0.5 * np.eye(6))


def test_mr_build_kats(mg, oracle):
    from oracle import Csr
    P = mg.spai_build(Csr.from_dense(np.eye(5))).matrix.download()  # K = I -> alpha = 1, P = I
    np.testing.assert_array_equal(P.todense(), np.eye(5))
    P = mg.spai_build(Csr.from_dense(np.diag([2.0, 4.0])), tol=1e-12).matrix.download()
    assert rel(P.todense(), np.diag([0.5, 0.25])) < 1e-12
    # random SPD 20x20: ||I - K P||_F <= tol sqrt(n)
    rng = np.random.default_rng(0)
    G = rng.standard_normal((20, 20))
    Kd = G @ G.T / 20 + np.eye(20)
    f = mg.spai_build(Csr.from_dense(Kd), tol=0.01, max_col_iters=500)
    Pd = f.matrix.download().todense()
    assert np.linalg.norm(np.eye(20) - Kd @ Pd) <= 0.01 * np.sqrt(20) + 1e-12
    want, _ = oracle.spai_build(Csr.from_dense(Kd), tol=0.01, max_col_iters=500, mode=1)
    assert rel(Pd, want.todense()) < 1e-10


def test_mr_stagnation_column_and_message(mg, oracle):
    """The BASELINE Hermite beam makes MR-SPAI stall at column 0."""
    from oracle import OracleError
    M, D, K = oracle.hermite_generate(1000)
    A = oracle.shifted_operator(M, D, K, 100.0)
    with pytest.raises(OracleError) as eo:
        oracle.spai_build(A, mode=1)
    with pytest.raises(mg.StagnationError) as eg:
        mg.spai_build(A, mode=mg.FROZEN)
    assert eg.value.column == eo.value.index == 0
    assert str(eg.value).split(" stalled")[0] == eo.value.msg.split(" stalled")[0]


# --------------------------------------------- frozen MR-SPAI beyond the 512-slot column window
def _banded(n, off, c=-0.5):
    """SPD, diagonally dominant: 4 on the diagonal, -1 at +-1, c at +-off (CSR built directly)."""
    from oracle import Csr
    rows, cols, vals = [], [], []
    for d, v in ((-off, c), (-1, -1.0), (0, 4.0), (1, -1.0), (off, c)):
        i = np.arange(max(0, -d), min(n, n - d))
        rows.append(i)
        cols.append(i + d)
        vals.append(np.full(i.shape, v))
    rows, cols, vals = (np.concatenate(x) for x in (rows, cols, vals))
    order = np.lexsort((cols, rows))
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return Csr(n, n, np.cumsum(rp).astype(np.int64), cols[order].astype(np.int32), vals[order].astype(np.float64))


@pytest.mark.parametrize("n,off,tol", [(3000, 40, 1e-2), (6000, 100, 1e-3)])
def test_mr_frozen_wide_columns(mg, oracle, n, off, tol):
    """Columns whose residual support outgrows 512 slots (about 800 and 3400 wide here) rerun on the
    2048- and 6144-slot windows: same factor as the reference."""
    K = _banded(n, off)
    want, wres = oracle.spai_build(K, tol=tol, mode=1)
    f = mg.spai_build(K, tol=tol, mode=mg.FROZEN)
    _csr_close(f.matrix.download(), want)
    assert rel(f.target_frob_residual, wres) < 1e-10


def test_mr_frozen_window_limit_is_reported(mg):
    """Beyond the widest window the build refuses (no fallback), naming the column."""
    K = _banded(40000, 3000)
    with pytest.raises(mg.UnsupportedError, match="outgrew the device window"):
        mg.spai_build(K, tol=1e-6, mode=mg.FROZEN)


# --------------------------------------------- MR-SPAI, sequential mode (the reference default)
@pytest.fixture(params=["dense", "sparse"])
def seq_kernel(request, mg):
    """Both device kernels of sequential mode: the dense-factor grid kernel (n <= 4096) and the
    sparse row-list chain (every size; forced here with the seq_sparse context option)."""
    ctx = mg.default_context()
    ctx.set_option("seq_sparse", 1 if request.param == "sparse" else 0)
    yield request.param
    ctx.set_option("seq_sparse", 0)


@pytest.mark.parametrize("n,kscale,s", [(300, 0.01, 1.0), (300, 1.0, 10.0), (300, 100.0, 10.0), (500, 1.0, 10.0),
                                        (2000, 1.0, 100.0)])
def test_mr_sequential_build_t1(mg, oracle, seq_kernel, n, kscale, s):
    """d = P r over the columns built so far (spai.cpp:138-158): heavy fill (200-700 nnz/column)."""
    M, D, K = oracle.chain_generate(n, consistent=True, stiffness_scale=kscale)
    A = oracle.shifted_operator(M, D, K, s)
    want, wres = oracle.spai_build(A, mode=0)
    f = mg.spai_build(A, mode=mg.SEQUENTIAL)
    _csr_close(f.matrix.download(), want)
    assert rel(f.target_frob_residual, wres) < 1e-10


def test_mr_sequential_update_t1(mg, oracle, seq_kernel):
    """s = 10 -> 10.5 at n = 100, sequential mode."""
    M, D, K = oracle.chain_generate(100, consistent=True, stiffness_scale=1.0)
    A1 = oracle.shifted_operator(M, D, K, 10.0)
    A2 = oracle.shifted_operator(M, D, K, 10.5)
    want, wres = oracle.spai_update(A1, A2, mode=0)
    f = mg.spai_update(A1, A2, mode=mg.SEQUENTIAL)
    _csr_close(f.matrix.download(), want)
    assert rel(f.target_frob_residual, wres) < 1e-10
    Q = mg.spai_update(A2, A2, mode=mg.SEQUENTIAL).matrix.download()  # K_new == K_old -> Q = I exactly
    np.testing.assert_array_equal(Q.todense(), np.eye(100))


def test_mr_sequential_kats(mg, seq_kernel):
    from oracle import Csr
    P = mg.spai_build(Csr.from_dense(np.eye(5)), mode=mg.SEQUENTIAL).matrix.download()
    np.testing.assert_array_equal(P.todense(), np.eye(5))
    P = mg.spai_build(Csr.from_dense(np.diag([2.0, 4.0])), tol=1e-12, mode=mg.SEQUENTIAL).matrix.download()
    assert rel(P.todense(), np.diag([0.5, 0.25])) < 1e-12


def test_mr_sequential_stagnation(mg, oracle, seq_kernel):
    from oracle import OracleError
    M, D, K = oracle.hermite_generate(1000)
    A = oracle.shifted_operator(M, D, K, 100.0)
    with pytest.raises(OracleError) as eo:
        oracle.spai_build(A, mode=0)
    with pytest.raises(mg.StagnationError) as eg:
        mg.spai_build(A, mode=mg.SEQUENTIAL)
    assert eg.value.column == eo.value.index
    assert str(eg.value).split(" stalled")[0] == eo.value.msg.split(" stalled")[0]


def test_mr_sequential_large_n(mg, oracle):
    """n = 2e4 (the sparse row-list factor; the earlier dense device layout stopped at 8192):
    ~660 nnz per column of fill, entries within 1e-10 of the oracle, same pattern and residuals,
    and the small-capacity retry path (a tiny problem whose first row-list capacity overflows)."""
    import time
    M, D, K = oracle.chain_generate(20000, consistent=True, stiffness_scale=1.0)
    A = oracle.shifted_operator(M, D, K, 10.0)
    t = time.perf_counter()
    f = mg.spai_build(A, mode=mg.SEQUENTIAL)
    dev_s = time.perf_counter() - t
    want, wres = oracle.spai_build(A, mode=0)
    got = f.matrix.download()
    assert got.nnz > 600 * 20000
    _csr_close(got, want)
    assert rel(f.target_frob_residual, wres) < 1e-10
    print(f"sequential MR n=2e4: device {dev_s:.2f} s, nnz {got.nnz}")


# ------------------------------------------------------------------ LS-SPAI
@pytest.mark.parametrize("pattern", [0, 1])
@pytest.mark.parametrize("s", [10.0, 100.0, 1e4])
def test_ls_build_hermite(mg, oracle, pattern, s):
    M, D, K = oracle.hermite_generate(1000)
    A = oracle.shifted_operator(M, D, K, s)
    want = oracle.spai_ls(A, None, pattern)
    got = mg.spai_ls(A, None, pattern).matrix.download()
    _csr_equal(got, want)


@pytest.mark.parametrize("pattern", [0, 1])
def test_ls_update_hermite(mg, oracle, pattern):
    M, D, K = oracle.hermite_generate(1000)
    A1 = oracle.shifted_operator(M, D, K, 100.0)
    A2 = oracle.shifted_operator(M, D, K, 150.0)
    want = oracle.spai_ls(A2, A1, pattern)
    got = mg.spai_ls(A2, A1, pattern).matrix.download()
    _csr_equal(got, want)


@pytest.mark.parametrize("pattern", [0x10, 0x11])
@pytest.mark.parametrize("s", [10.0, 1e4])
def test_ls_colscale_build_and_update_hermite(mg, oracle, pattern, s):
    """Column-equilibrated LS (pattern | MGPU_LS_COLSCALE): lane kernel (A pattern) and lane-group
    kernel (A^2 pattern), build and update, bitwise equal to the oracle restatement."""
    M, D, K = oracle.hermite_generate(1000)
    A = oracle.shifted_operator(M, D, K, s)
    _csr_equal(mg.spai_ls(A, None, pattern).matrix.download(), oracle.spai_ls(A, None, pattern))
    A2 = oracle.shifted_operator(M, D, K, 1.5 * s)
    _csr_equal(mg.spai_ls(A2, A, pattern).matrix.download(), oracle.spai_ls(A2, A, pattern))


@pytest.mark.parametrize("pattern", [0x10, 0x11])
def test_ls_colscale_full_size_batched(mg, oracle, pattern):
    """BASELINE configs[3] size (n = 1e6), where the unscaled LS rank-flushes: the batched
    column-equilibrated factors of 2 shifts are bitwise equal to the oracle's, every column."""
    M, D, K = oracle.hermite_generate(500000)
    shifts = [10.0, 1e4]
    ops = mg.shifted_operators(M, D, K, shifts)
    facs = mg.spai_ls_batched(ops, None, pattern)
    for s, f in zip(shifts, facs):
        _csr_equal(f.matrix.download(), oracle.spai_ls(oracle.shifted_operator(M, D, K, s), None, pattern))


def test_ls_colscale_zero_column(mg, oracle):
    """A zero column of S is rank deficiency in the equilibrated variant too (same column)."""
    from oracle import Csr, OracleError
    a = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 0.0], [0.0, 0.0, 3.0]])
    a[1, 1] = 1e-320  # stored, but squares to zero: ||S_c|| == 0
    A = Csr.from_dense(a)
    with pytest.raises(OracleError) as eo:
        oracle.spai_ls(A, None, 0x10)
    with pytest.raises(mg.NumericalError) as eg:
        mg.spai_ls(A, None, 0x10)
    assert eg.value.index == eo.value.index


def test_ls_chain_model_and_dense(mg, oracle):
    from oracle import Csr
    M, D, K = oracle.chain_generate(3000, consistent=True, stiffness_scale=1.0)
    A = oracle.shifted_operator(M, D, K, 3.0)
    _csr_close(mg.spai_ls(A, None, 1).matrix.download(), oracle.spai_ls(A, None, 1))
    rng = np.random.default_rng(1)
    G = rng.standard_normal((20, 20))
    Kd = Csr.from_dense(G @ G.T + 20 * np.eye(20))
    _csr_close(mg.spai_ls(Kd).matrix.download(), oracle.spai_ls(Kd, None, 0))


def test_ls_rank_deficiency(mg, oracle):
    from oracle import Csr, OracleError
    A = Csr.from_dense(np.array([[1.0, 2.0, 0.0], [1.0, 2.0, 0.0], [0.0, 0.0, 3.0]]))
    with pytest.raises(OracleError) as eo:
        oracle.spai_ls(A, None, 0)
    with pytest.raises(mg.NumericalError) as eg:
        mg.spai_ls(A)
    assert eg.value.index == eo.value.index == 0


@pytest.mark.parametrize("pattern", [0, 1])
def test_ls_batched_shared_pattern(mg, oracle, pattern):
    """8 shifted operators share one pattern: one launch, gathered factors, bitwise == oracle."""
    M, D, K = oracle.hermite_generate(500)
    shifts = [10.0 ** (1 + 3 * i / 7) for i in range(8)]
    ops = mg.shifted_operators(M, D, K, shifts)
    facs = mg.spai_ls_batched(ops, None, pattern)
    host = [oracle.shifted_operator(M, D, K, s) for s in shifts]
    for A, f in zip(host, facs):
        _csr_equal(f.matrix.download(), oracle.spai_ls(A, None, pattern))
    # batched update (K_old per point, same pattern) -- the AIRGA vertical update
    shifts2 = [s * 1.25 for s in shifts]
    ops2 = mg.shifted_operators(M, D, K, shifts2)
    upd = mg.spai_ls_batched(ops2, ops, pattern)
    for A_old, s2, f in zip(host, shifts2, upd):
        _csr_equal(f.matrix.download(), oracle.spai_ls(oracle.shifted_operator(M, D, K, s2), A_old, pattern))


def test_ls_batched_mixed_patterns(mg, oracle):
    """Operators with different patterns take the per-operator path."""
    Mh, Dh, Kh = oracle.hermite_generate(200)
    Mc, Dc, Kc = oracle.chain_generate(400, consistent=True, stiffness_scale=1.0)
    A1 = oracle.shifted_operator(Mh, Dh, Kh, 100.0)
    A2 = oracle.shifted_operator(Mc, Dc, Kc, 2.0)
    facs = mg.spai_ls_batched([A1, A2], None, 0)
    _csr_equal(facs[0].matrix.download(), oracle.spai_ls(A1, None, 0))
    _csr_equal(facs[1].matrix.download(), oracle.spai_ls(A2, None, 0))


def test_ls_batched_same_nnz_different_structure(mg, oracle):
    """Equal sizes and nnz but different column positions: the speculative shared-pattern path
    must detect the mismatch (device flag read with the LS status) and rerun per operator."""
    import numpy as np
    from oracle import Csr
    n = 300
    rng = np.random.default_rng(5)
    base = np.diag(np.full(n, 4.0)) + np.diag(np.full(n - 1, -1.0), 1) + np.diag(np.full(n - 1, -1.0), -1)
    a1 = base.copy()
    a2 = base.copy()
    # move one off-diagonal pair in a2 (same nnz, different structure), keep it symmetric
    a2[10, 11] = a2[11, 10] = 0.0
    a2[10, 12] = a2[12, 10] = -1.0
    a1 += np.diag(rng.uniform(0.0, 0.5, n))
    a2 += np.diag(rng.uniform(0.0, 0.5, n))
    A1, A2 = Csr.from_dense(a1), Csr.from_dense(a2)
    assert A1.nnz == A2.nnz
    facs = mg.spai_ls_batched([A1, A2, A1], None, 0)
    _csr_equal(facs[0].matrix.download(), oracle.spai_ls(A1, None, 0))
    _csr_equal(facs[1].matrix.download(), oracle.spai_ls(A2, None, 0))
    _csr_equal(facs[2].matrix.download(), oracle.spai_ls(A1, None, 0))


# ------------------------------------------------------------------ SpGEMM chain collapse
def test_spgemm_collapse(mg, oracle):
    M, D, K = oracle.hermite_generate(400)
    A1 = oracle.shifted_operator(M, D, K, 100.0)
    A2 = oracle.shifted_operator(M, D, K, 150.0)
    P = oracle.spai_ls(A1, None, 0)
    Q = oracle.spai_ls(A2, A1, 0)
    QP = mg.spgemm(Q, P).download()
    dense = Q.todense() @ P.todense()
    assert rel(QP.todense(), dense) < 1e-14
    v = np.random.default_rng(2).standard_normal(800)
    assert rel(mg.chain_apply([QP], v), oracle.chain_apply([Q, P], v)) < 1e-12


def test_spgemm_long_rows(mg):
    """No row-length cap: banded factors of bandwidth 40 give 161-entry product rows."""
    from oracle import Csr
    rng = np.random.default_rng(9)
    n, bw = 400, 40
    def banded():
        a = np.zeros((n, n))
        for i in range(n):
            lo, hi = max(0, i - bw), min(n, i + bw + 1)
            a[i, lo:hi] = rng.standard_normal(hi - lo)
        return a
    a, c = banded(), banded()
    AB = mg.spgemm(Csr.from_dense(a), Csr.from_dense(c)).download()
    assert np.max(np.diff(AB.row_ptr)) == 2 * 2 * bw + 1
    assert rel(AB.todense(), a @ c) < 1e-14


# ------------------------------------------------------------------ chain_quality
@pytest.mark.parametrize("z,samples,seed", [(0, 3, 42), (1, 8, 42), (2, 5, 7)])
def test_chain_quality_matches_reference(mg, oracle, ref, z, samples, seed):
    """spai.cpp:375-409: same probe stream (mt19937_64 + normal_distribution), device SpMM + sums."""
    M, D, K = oracle.chain_generate(1500, consistent=True, stiffness_scale=1.0)
    A1 = oracle.shifted_operator(M, D, K, 10.0)
    A2 = oracle.shifted_operator(M, D, K, 11.0)
    P, _ = oracle.spai_build(A1, mode=1)
    Q, _ = oracle.spai_update(A1, A2, mode=1)
    chain = [Q, P][2 - z:] if z else []
    want = ref.chain_quality(chain, A2, samples, seed)
    got = mg.chain_quality(chain, A2, samples, seed)
    assert abs(got - want) <= 1e-12 * abs(want)


def test_chain_quality_rejects_zero_samples(mg, oracle):
    M, D, K = oracle.chain_generate(50)
    with pytest.raises(mg.ArgumentError, match="samples must be >= 1"):
        mg.chain_quality([], K, 0)
