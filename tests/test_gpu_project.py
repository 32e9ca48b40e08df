"""Global Arnoldi + projection on the device against the reference.

thin_qr (dense.cpp:153-246), project_reduce (airga.cpp:485-500) and arnoldi_deflate
(airga.cpp:456-473).  The device replaces the reference's serial dot products by
fixed-order trees (thin_qr, deflate) and cuBLAS DGEMM (the dense products of the
projection), so the bar is 1e-12 relative (norm-wise); the rank decisions, flushed
columns and signs must be identical.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("rows,cols", [(3000, 40), (257, 256), (50, 1), (10000, 64)])
def test_thin_qr_matches_reference(mg, oracle, ref, rows, cols):
    rng = np.random.default_rng(rows + cols)
    A = np.asfortranarray(rng.standard_normal((rows, cols)))
    Qr, Rr, kr = ref.thin_qr(A)
    Qo, Ro, ko = oracle.thin_qr(A)
    Q, R, k = mg.thin_qr(A)
    assert k == kr == ko == cols
    assert _rel(Q, Qr) < 1e-12 and _rel(R, Rr) < 1e-12
    assert np.all(np.diag(R) >= 0)
    np.testing.assert_array_equal(np.tril(R, -1), 0.0)


def test_thin_qr_rank_deficient(mg, ref):
    """Duplicated and zero columns are flushed exactly like the reference (zero Q column, R_kk = 0)."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((500, 8))
    A[:, 3] = A[:, 1]
    A[:, 5] = 0.0
    A[:, 6] = 2.0 * A[:, 0] - A[:, 2]
    A = np.asfortranarray(A)
    Qr, Rr, kr = ref.thin_qr(A)
    Q, R, k = mg.thin_qr(A)
    assert k == kr == 5
    np.testing.assert_array_equal(np.diag(R) == 0.0, np.diag(Rr) == 0.0)
    for c in np.flatnonzero(np.diag(Rr) == 0.0):
        np.testing.assert_array_equal(Q[:, c], 0.0)
    assert _rel(Q, Qr) < 1e-12 and _rel(R, Rr) < 1e-12


def test_thin_qr_argument_errors(mg):
    with pytest.raises(mg.ArgumentError, match="nrows >= ncols"):
        mg.thin_qr(np.ones((3, 5)))


def _system(oracle, n):
    M, D, K = oracle.chain_generate(n, consistent=True, stiffness_scale=1.0)
    rng = np.random.default_rng(n)
    F = np.zeros((n, 2), order="F")
    F[0, 0] = 1.0
    F[n // 2, 1] = 1.0
    Cp = np.asfortranarray(rng.standard_normal((3, n)))
    Cv = np.asfortranarray(rng.standard_normal((3, n)))
    return M, D, K, F, Cp, Cv


@pytest.mark.parametrize("n,r", [(1500, 12), (4000, 64)])
def test_project_reduce_matches_reference(mg, oracle, ref, n, r):
    M, D, K, F, Cp, Cv = _system(oracle, n)
    V, _, _ = ref.thin_qr(np.asfortranarray(np.random.default_rng(1).standard_normal((n, r))))
    want = ref.project_reduce(M, D, K, V, F, Cp, Cv)
    got = mg.project_reduce(M, D, K, V, F, Cp, Cv)
    for key in ("Mh", "Dh", "Kh", "Fh", "Cph", "Cvh"):
        assert got[key].shape == want[key].shape
        assert _rel(got[key], want[key]) < 1e-12, key
    # no F / outputs: the r x r projections alone
    got2 = mg.project_reduce(M, D, K, V)
    assert _rel(got2["Kh"], want["Kh"]) < 1e-12


def test_arnoldi_deflate_matches_reference(mg, ref):
    rng = np.random.default_rng(3)
    n, m = 2000, 2
    blocks = []
    for _ in range(3):
        b = rng.standard_normal((n, m))
        blocks.append(np.asfortranarray(b / np.linalg.norm(b)))
    X = np.asfortranarray(rng.standard_normal((n, m)))
    Xr, gr = ref.arnoldi_deflate(X, blocks)
    Xg, gg = mg.arnoldi_deflate(X, blocks)
    assert _rel(Xg, Xr) < 1e-12
    assert _rel(gg, gr) < 1e-12
    # deflating against a block that spans X leaves (numerically) nothing
    Xs, g = mg.arnoldi_deflate(blocks[0] * 3.0, [blocks[0]])
    assert np.linalg.norm(Xs) < 1e-12 and abs(g[0] - 3.0) < 1e-12


def test_arnoldi_pipeline_end_to_end(mg, oracle, ref):
    """Zeroth moments -> deflation -> thin_qr -> project_reduce, as airga_run's projection step
    (airga.cpp:820-850), all on the device, against the same sequence on the reference."""
    n = 1200
    M, D, K, F, Cp, Cv = _system(oracle, n)
    shifts = [1.0, 10.0, 100.0]
    Xs = []
    for s in shifts:
        A = oracle.shifted_operator(M, D, K, s)
        Xs.append(np.column_stack([oracle.pcg_solve(A, [], F[:, c], rtol=1e-12)["solution"] for c in range(2)]))
    Vt = np.asfortranarray(np.hstack([x / np.linalg.norm(x) for x in Xs]))
    Qr, Rr, kr = ref.thin_qr(Vt)
    Q, R, k = mg.thin_qr(Vt)
    assert k == kr
    keep = np.flatnonzero(np.diag(Rr) > 0)
    want = ref.project_reduce(M, D, K, np.asfortranarray(Qr[:, keep]), F, Cp, Cv)
    got = mg.project_reduce(M, D, K, np.asfortranarray(Q[:, keep]), F, Cp, Cv)
    for key in ("Mh", "Dh", "Kh", "Fh"):
        assert _rel(got[key], want[key]) < 1e-10, key


def test_project_reduce_slabs_sum_to_global(mg, oracle, ref):
    """The row-slab kernel (what each rank runs in sharding.project_reduce_distributed): slab
    partials with halo-extended bases add up to the global projection."""
    from paper_1606_01216_b200 import sharding
    n, r = 3000, 10
    M, D, K, F, Cp, Cv = _system(oracle, n)
    V, _, _ = ref.thin_qr(np.asfortranarray(np.random.default_rng(2).standard_normal((n, r))))
    want = ref.project_reduce(M, D, K, V, F, Cp, Cv)
    h = max(sharding.bandwidth(x) for x in (M, D, K))
    total = None
    for rank in range(3):
        r0, r1 = sharding.row_range(n, rank, 3)
        lo, hi = max(0, r0 - h), min(n, r1 + h)
        part = mg.project_reduce_slab(sharding.row_slab(M, r0, r1), sharding.row_slab(D, r0, r1),
                                      sharding.row_slab(K, r0, r1), r0, lo, np.asfortranarray(V[lo:hi]),
                                      F[r0:r1], Cp[:, r0:r1], Cv[:, r0:r1])
        total = part if total is None else {k: total[k] + part[k] for k in total}
    for key in ("Mh", "Dh", "Kh", "Fh", "Cph", "Cvh"):
        assert _rel(total[key], want[key]) < 1e-12, key
    # the single-rank distributed call is the plain device projection
    single = sharding.project_reduce_distributed(M, D, K, V, 0, F, Cp, Cv)
    assert _rel(single["Kh"], want["Kh"]) < 1e-12
