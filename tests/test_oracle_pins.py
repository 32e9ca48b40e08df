"""CPU: the C restatement (oracle/oracle.c) pinned to the reference.

(1) against tests/golden/reference_golden.npz, produced by the UNMODIFIED
    reference library with its scalar kernel table (tests/golden/make_golden.py);
(2) against the SPEC.md known-answer tests for this path;
(3) live against oracle/_ref when it is built (this container).
Bitwise where the reference is deterministic and the restatement replays its
operation order, which is everywhere on this path.
"""
import os

import numpy as np
import pytest

from conftest import rel

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def _csr(prefix):
    from oracle import Csr
    rp = G[prefix + "_rp"]
    return Csr(len(rp) - 1, len(rp) - 1, rp, G[prefix + "_ci"], G[prefix + "_v"])


def _same(a, prefix):
    b = _csr(prefix)
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.col_idx, b.col_idx)
    np.testing.assert_array_equal(a.values, b.values)


def test_chain_model_and_assembly(oracle):
    M, D, K = oracle.chain_generate(200, alpha=0.1, beta=1e-5, stiffness_scale=1.0, consistent=True)
    _same(M, "chain_M"), _same(D, "chain_D"), _same(K, "chain_K")
    _same(oracle.shifted_operator(M, D, K, 3.0), "chain_A1")
    _same(oracle.shifted_operator(M, D, K, 3.5), "chain_A2")
    _same(oracle.transpose(_csr("chain_A1")), "chain_A1t")
    assert oracle.trace(_csr("chain_A1")) == G["chain_trace_A1"][0]
    assert oracle.trace_inner(_csr("chain_A1"), _csr("chain_A2")) == G["chain_trace_inner_A1A2"][0]
    np.testing.assert_array_equal(oracle.spmv(_csr("chain_A1"), G["chain_apply_v"]), G["chain_spmv_out"])


@pytest.mark.parametrize("mode,tag", [(1, "frozen"), (0, "seq")])
def test_mr_spai_build_update(oracle, mode, tag):
    A1, A2 = _csr("chain_A1"), _csr("chain_A2")
    P, res = oracle.spai_build(A1, mode=mode)
    _same(P, f"chain_P_{tag}")
    np.testing.assert_array_equal(res, G[f"chain_Pres_{tag}"])
    Q, qres = oracle.spai_update(A1, A2, mode=mode)
    _same(Q, f"chain_Q_{tag}")
    np.testing.assert_array_equal(qres, G[f"chain_Qres_{tag}"])


def test_chain_apply_and_pcg(oracle):
    P, Q, A2 = _csr("chain_P_frozen"), _csr("chain_Q_frozen"), _csr("chain_A2")
    np.testing.assert_array_equal(oracle.chain_apply([Q, P], G["chain_apply_v"]), G["chain_apply_out"])
    s = oracle.pcg_solve(A2, [Q, P], G["chain_b"], rtol=1e-10)
    np.testing.assert_array_equal(s["solution"], G["chain_pcg_x"])
    np.testing.assert_array_equal(s["residual"], G["chain_pcg_res"])
    np.testing.assert_array_equal(s["recurrence_residual"], G["chain_pcg_rec"])
    assert [s["iterations"], int(s["converged"])] == list(G["chain_pcg_it"])
    np.testing.assert_array_equal(s["relres_history"], G["chain_pcg_hist"])


def test_block_solve(oracle):
    bs = oracle.block_solve(_csr("chain_A1"), [_csr("chain_P_frozen")], G["chain_block_B"], rtol=1e-10)
    np.testing.assert_array_equal(bs["X"], G["chain_block_X"])
    np.testing.assert_array_equal(bs["iterations"], G["chain_block_it"])


def test_hermite_generator_matches_reference_assembly(oracle):
    M, D, K = oracle.hermite_generate(100)
    _same(M, "herm_M"), _same(D, "herm_D"), _same(K, "herm_K")
    _same(oracle.shifted_operator(M, D, K, 100.0), "herm_A1")
    assert K.nnz == 5 * 200 - 6  # interior (w, theta) couplings cancel exactly


@pytest.mark.parametrize("pat", [0, 1, 0x10, 0x11])
def test_ls_spai_against_reference_primitives(oracle, pat):
    A1, A2 = _csr("herm_A1"), _csr("herm_A2")
    _same(oracle.spai_ls(A1, None, pat), f"herm_LS{pat}")
    _same(oracle.spai_ls(A2, A1, pat), f"herm_LSU{pat}")


def test_hermite_pcg_and_mr_stagnation(oracle):
    from oracle import OracleError
    A1 = _csr("herm_A1")
    b = np.zeros(200)
    b[198] = 1.0
    s = oracle.pcg_solve(A1, [_csr("herm_LS0")], b, rtol=1e-10, maxit=60)
    np.testing.assert_array_equal(s["solution"], G["herm_pcg_x"])
    assert [s["iterations"], int(s["converged"])] == list(G["herm_pcg_it"])
    with pytest.raises(OracleError) as e:
        oracle.spai_build(A1, mode=1)
    assert [e.value.status, e.value.index] == list(G["herm_mr_err"])
    assert e.value.msg == str(G["herm_mr_msg"][0])


def test_thin_qr(oracle):
    Q, R, rank = oracle.thin_qr(G["qr_S"])
    np.testing.assert_array_equal(Q, G["qr_Q"])
    np.testing.assert_array_equal(R, G["qr_R"])
    assert rank == G["qr_rank"][0]


def test_breakdown(oracle):
    from oracle import Csr, OracleError
    with pytest.raises(OracleError) as e:
        oracle.pcg_solve(Csr.from_dense(np.diag([1.0, -1.0, 2.0])), [], np.array([1.0, 1.0, 0.0]))
    assert [e.value.status, e.value.index] == list(G["bd"])


# ------------------------------------------------------------------ SPEC.md KATs
def test_spec_kats_spai(oracle):
    from oracle import Csr
    P, res = oracle.spai_build(Csr.from_dense(np.eye(4)))  # K = I: alpha = 1, P = I, 0 iterations
    np.testing.assert_array_equal(P.todense(), np.eye(4))
    P, _ = oracle.spai_build(Csr.from_dense(np.diag([2.0, 4.0])), tol=1e-12)
    assert rel(P.todense(), np.diag([0.5, 0.25])) < 1e-12
    Q, _ = oracle.spai_update(Csr.from_dense(np.eye(3)), Csr.from_dense(2 * np.eye(3)))
    np.testing.assert_array_equal(Q.todense(), 0.5 * np.eye(3))
    A = _csr("chain_A1")
    Q, qres = oracle.spai_update(A, A)  # identical operands: Q = I bitwise
    np.testing.assert_array_equal(Q.todense(), np.eye(200))
    np.testing.assert_array_equal(qres, 0.0)


def test_spec_kats_krylov(oracle):
    from oracle import Csr
    I3 = Csr.from_dense(np.eye(3))
    s = oracle.pcg_solve(I3, [], np.array([1.0, 2.0, 3.0]))
    assert s["iterations"] == 1 and s["converged"]
    np.testing.assert_array_equal(s["solution"], [1.0, 2.0, 3.0])
    s = oracle.pcg_solve(I3, [], np.zeros(3))
    assert s["iterations"] == 0 and s["converged"]
    rng = np.random.default_rng(3)
    Gm = rng.standard_normal((10, 10))
    A = Gm @ Gm.T + 10 * np.eye(10)
    b = rng.standard_normal(10)
    s = oracle.pcg_solve(Csr.from_dense(A), [], b, rtol=1e-10)
    assert rel(s["solution"], np.linalg.solve(A, b)) < 10 * 1e-10 * np.linalg.cond(A)
    assert abs(s["solution"] @ s["residual"]) <= 1e-8 * np.linalg.norm(s["solution"]) * np.linalg.norm(b)
    np.testing.assert_array_equal(oracle.chain_apply([], b), b)  # empty chain = identity
    two, three = Csr.from_dense(2 * np.eye(10)), Csr.from_dense(3 * np.eye(10))
    np.testing.assert_array_equal(oracle.chain_apply([two, three], b), 6 * b)


def test_live_reference_matches_restatement(oracle, ref):
    """Only where oracle/_ref was built (this container): random chain cases."""
    for kscale, s in [(0.01, 1.0), (1.0, 10.0)]:
        M, D, K = ref.chain_generate(500, stiffness_scale=kscale, consistent=True)
        A = ref.shifted_operator(M, D, K, s)
        P, _ = ref.spai_build(A, mode=1)
        Po, _ = oracle.spai_build(A, mode=1)
        np.testing.assert_array_equal(P.values, Po.values)
        b = np.ones(500)
        np.testing.assert_array_equal(ref.pcg_solve(A, [P], b)["solution"], oracle.pcg_solve(A, [Po], b)["solution"])


def test_ls_colscale_avoids_the_global_rank_flush(oracle):
    """At n = 4e5 the reference thin_qr's global flush (sigma <= 1e-12 ||S||_F, dense.cpp:162-179)
    declares the A^2-pattern problems rank-deficient; the column-equilibrated variant (same
    least-squares minimiser) solves them.  Small n: both variants agree to rounding."""
    from oracle import OracleError
    M, D, K = oracle.hermite_generate(200000)
    A = oracle.shifted_operator(M, D, K, 100.0)
    with pytest.raises(OracleError):
        oracle.spai_ls(A, None, 1)
    P = oracle.spai_ls(A, None, 0x11)
    assert P.nnz == 10 * A.nrows - 24 and np.all(np.isfinite(P.values))
    M, D, K = oracle.hermite_generate(200)
    A = oracle.shifted_operator(M, D, K, 100.0)
    P0, P1 = oracle.spai_ls(A, None, 1), oracle.spai_ls(A, None, 0x11)
    assert np.array_equal(P0.col_idx, P1.col_idx)
    assert np.max(np.abs(P0.values - P1.values)) <= 1e-10 * np.max(np.abs(P0.values))
