"""Parity of the device sparse core with the oracle (bitwise where the arithmetic allows).

K-asm (system.cpp:64-68 / sparse.cpp:167-218): bitwise -- no FMA, same merge.
transpose (sparse.cpp:220-249): bitwise.  SpMV / chain_apply: bitwise with the
scalar kernel table (kernels_scalar.cpp:39-47).  trace / trace_inner: the
device reduction is a fixed tree, not the reference's serial sum -> 1e-14.
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

SHIFTS = [10.0 ** (1 + 3 * i / 7) for i in range(8)]


def _eq_csr(a, b):
    assert a.nrows == b.nrows
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.col_idx, b.col_idx)
    np.testing.assert_array_equal(a.values, b.values)


@pytest.mark.parametrize("model", ["hermite", "chain"])
def test_shifted_operators_bitwise(mg, oracle, model):
    if model == "hermite":
        M, D, K = oracle.hermite_generate(500)
    else:
        M, D, K = oracle.chain_generate(1000, consistent=True, stiffness_scale=1.0)
    ops = mg.shifted_operators(M, D, K, SHIFTS)
    for s, dA in zip(SHIFTS, ops):
        _eq_csr(dA.download(), oracle.shifted_operator(M, D, K, s))


def test_product_models_match_oracle(mg, oracle):
    for (pm, om) in [(mg.model_hermite(300), oracle.hermite_generate(300)),
                     (mg.model_chain(400, consistent=True), oracle.chain_generate(400, consistent=True))]:
        for a, b in zip(pm, om):
            _eq_csr(a, b)


def test_sp_add_scaled_exact_cancellation(mg, oracle):
    from oracle import Csr
    A = Csr.from_dense(np.array([[1.0, 2.0, 0.0], [0.0, 3.0, 4.0], [5.0, 0.0, 6.0]]))
    B = Csr.from_dense(np.array([[1.0, -1.0, 7.0], [0.0, 1.5, 0.0], [0.0, 0.0, -3.0]]))
    got = mg.sp_add_scaled(A, B, 1.0, 2.0).download()
    want = oracle.sp_add_scaled(A, B, 1.0, 2.0)  # (0,1): 2 - 2 = 0 dropped; (2,2): 6 - 6 = 0 dropped
    _eq_csr(got, want)
    assert want.nnz == 5


def test_transpose_bitwise(mg, oracle):
    rng = np.random.default_rng(7)
    a = rng.standard_normal((60, 45)) * (rng.random((60, 45)) < 0.1)
    from oracle import Csr
    A = Csr.from_dense(a)
    _eq_csr(mg.transpose(A).download(), oracle.transpose(A))


def test_traces(mg, oracle):
    M, D, K = oracle.hermite_generate(2000)
    A = oracle.shifted_operator(M, D, K, 100.0)
    B = oracle.shifted_operator(M, D, K, 105.0)
    assert rel(mg.trace(A), oracle.trace(A)) < 1e-12  # tree vs serial sum order
    assert rel(mg.trace_inner(A, B), oracle.trace_inner(A, B)) < 1e-12
    assert mg.trace_inner(A, B) == mg.trace_inner(B, A)  # spai_update's Q = I relies on this


def test_chain_apply_bitwise(mg, oracle):
    M, D, K = oracle.chain_generate(3000, consistent=True)
    A1 = oracle.shifted_operator(M, D, K, 2.0)
    A2 = oracle.shifted_operator(M, D, K, 3.0)
    v = np.random.default_rng(1).standard_normal(3000)
    np.testing.assert_array_equal(mg.chain_apply([A2, A1], v), oracle.chain_apply([A2, A1], v))
    np.testing.assert_array_equal(mg.chain_apply([], v), v)


def test_argument_errors(mg, oracle):
    M, D, K = oracle.chain_generate(50)
    M2, _, _ = oracle.chain_generate(60)
    with pytest.raises(mg.ArgumentError):
        mg.shifted_operators(M2, D, K, [1.0])
    with pytest.raises(mg.ArgumentError):
        mg.pcg_solve(K, [], np.ones(50), rtol=0.0)


@pytest.mark.parametrize("ne", [1, 2, 3, 1000, 250000])
def test_device_beam_generation_bitwise(mg, ne):
    """the Hermite cantilever assembled on the device == the host generator, bit for bit."""
    want = mg.model_hermite(ne)
    got = mg.model_hermite_device(ne)
    for g, w in zip(got, want):
        d = g.download()
        np.testing.assert_array_equal(d.row_ptr, w.row_ptr)
        np.testing.assert_array_equal(d.col_idx, w.col_idx)
        np.testing.assert_array_equal(d.values, w.values)


def test_binary_csr_sidecar_roundtrip(mg, tmp_path):
    """binary CSR written from / read into device memory, exact round trip."""
    M, D, K = mg.model_hermite(5000)
    dK = mg.DeviceCsr.upload(K)
    path = str(tmp_path / "K.mgcsr")
    dK.save(path)
    back = mg.DeviceCsr.load(path).download()
    np.testing.assert_array_equal(back.row_ptr, K.row_ptr)
    np.testing.assert_array_equal(back.col_idx, K.col_idx)
    np.testing.assert_array_equal(back.values, K.values)
    # a factor storing exact zeros is written in its download (reference) form
    P = mg.spai_ls(mg.shifted_operator(M, D, K, 100.0), None, 0)
    P.matrix.save(path)
    np.testing.assert_array_equal(mg.DeviceCsr.load(path).download().values, P.matrix.download().values)
    with open(path, "r+b") as f:
        f.truncate(40)
    with pytest.raises(mg.ArgumentError, match="truncated"):
        mg.DeviceCsr.load(path)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"not a csr file at all")
    with pytest.raises(mg.ArgumentError, match="not a binary CSR"):
        mg.DeviceCsr.load(str(bad))


def test_upload_many_round_trip_and_validation(mg):
    """DeviceCsr.upload_many (mgpu_csr_upload_batch): the same arrays back bit for bit, and an
    inconsistent CSR among the batch raises ArgumentError like a single upload."""
    import numpy as np
    M, D, K = mg.model_hermite(300)
    got = mg.DeviceCsr.upload_many([M, D, K])
    for g, w in zip(got, (M, D, K)):
        h = g.download()
        np.testing.assert_array_equal(h.row_ptr, w.row_ptr)
        np.testing.assert_array_equal(h.col_idx, w.col_idx)
        np.testing.assert_array_equal(h.values, w.values)
    bad = mg.SparseMatrix(M.nrows, M.ncols, M.row_ptr.copy(), M.col_idx.copy(), M.values.copy())
    bad.col_idx[5] = M.ncols + 3  # column out of range
    with pytest.raises(mg.ArgumentError):
        mg.DeviceCsr.upload_many([M, bad, K])
