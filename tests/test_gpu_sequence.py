"""BASELINE configs[2] at test size: the AIRGA-style outer sequence with the SPAI update chain.

Ten outer iterations of 8 shifts drawn from mt19937_64(42) (sharding.airga_shift_draws,
SURVEY.md 8(d)); LS-SPAI on A's pattern built at z = 1 and updated from z = 2 (CgBackend's
update mode, airga.cpp:127-156), so the chain reaches 10 factors (newest first,
spai.cpp:352-373).  The device backend mirror against the oracle restatement of the same
sequence: every factor bitwise, CG iterates at a fixed budget within 1e-8 (iterations equal),
for the update chain and for rebuild-from-scratch.
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

NE, OUTER, L, BUDGET = 1000, 10, 8, 150


@pytest.mark.parametrize("update,path", [(True, "auto"), (False, "auto"), (True, "stream"), (True, "banded"),
                                         (True, "general")])
def test_sequence_update_chain_matches_oracle(mg, oracle, update, path):
    from paper_1606_01216_b200.backend import CudaCgBackend, CudaCgConfig
    from paper_1606_01216_b200.sharding import airga_shift_draws
    draws = airga_shift_draws(OUTER, L)
    M, D, K = oracle.hermite_generate(NE)
    n = M.nrows
    b = np.zeros(n)
    b[n - 2] = 1.0
    be = CudaCgBackend(CudaCgConfig(solver="cg_spai_update" if update else "cg_spai", spai_algorithm="ls",
                                    update_start_iteration=2, maxit_override=BUDGET))
    be.ctx.set_cg_path(path)
    try:
        _run(oracle, be, draws, M, D, K, b, update)
    finally:
        be.ctx.set_cg_path("auto")


def _run(oracle, be, draws, M, D, K, b, update):
    prev, chains = [None] * L, [[] for _ in range(L)]
    for z, pts in enumerate(draws, start=1):
        recs = []
        be.prepare((M, D, K), pts, z, recs)
        assert [r.kind for r in recs] == ["update" if (update and z >= 2) else "base"] * L
        assert [r.chain_length for r in recs] == [z if update else 1] * L
        got = be.solve_all(b, raise_on_breakdown=False)
        for i, s in enumerate(pts):
            A = oracle.shifted_operator(M, D, K, s)
            f = oracle.spai_ls(A, prev[i], 0) if (update and z >= 2) else oracle.spai_ls(A, None, 0)
            chains[i] = [f] + chains[i] if (update and z >= 2) else [f]
            prev[i] = A
            np.testing.assert_array_equal(be.chains[i][0].matrix.download().values, f.values)
            want = oracle.pcg_solve(A, chains[i], b, rtol=1e-10, maxit=BUDGET)
            assert int(got[i].iterations[0]) == want["iterations"]
            assert bool(got[i].converged[0]) == want["converged"]
            assert rel(got[i].X[:, 0], want["solution"]) < 1e-8, (z, i)


@pytest.mark.parametrize("outer", [6])
def test_sequence_collapsed_chain_matches_chained_oracle(mg, oracle, outer):
    """North-star subsystem 2: with collapse the backend keeps ONE factor per point, P <- Q P by the
    device SpGEMM after every update; its CG iterates stay within 1e-8 of the oracle's solve with
    the whole chain [Q_z, ..., Q_2, P] applied factor by factor (chain_apply, spai.cpp:361-373), and
    the records report the logical chain length."""
    from paper_1606_01216_b200.backend import CudaCgBackend, CudaCgConfig
    from paper_1606_01216_b200.sharding import airga_shift_draws
    draws = airga_shift_draws(outer, L)
    M, D, K = oracle.hermite_generate(NE)
    n = M.nrows
    b = np.zeros(n)
    b[n - 2] = 1.0
    be = CudaCgBackend(CudaCgConfig(solver="cg_spai_update", spai_algorithm="ls", update_start_iteration=2,
                                    maxit_override=BUDGET, collapse=True))
    prev, chains = [None] * L, [[] for _ in range(L)]
    for z, pts in enumerate(draws, start=1):
        recs = []
        be.prepare((M, D, K), pts, z, recs)
        assert [r.chain_length for r in recs] == [z] * L
        assert all(len(c) == 1 for c in be.chains)
        got = be.solve_all(b, raise_on_breakdown=False)
        for i, s in enumerate(pts):
            A = oracle.shifted_operator(M, D, K, s)
            f = oracle.spai_ls(A, prev[i], 0) if z >= 2 else oracle.spai_ls(A, None, 0)
            chains[i] = [f] + chains[i] if z >= 2 else [f]
            prev[i] = A
            want = oracle.pcg_solve(A, chains[i], b, rtol=1e-10, maxit=BUDGET)
            assert int(got[i].iterations[0]) == want["iterations"]
            assert rel(got[i].X[:, 0], want["solution"]) < 1e-8, (z, i)
        if z >= 2:  # the collapsed factor is the product of the chain (dense check on one point)
            Pd = np.eye(n)
            for f in reversed(chains[0]):
                Pd = f.todense() @ Pd
            got0 = mg.mgpu._factor_mat(be.chains[0][0]).download().todense()
            assert np.max(np.abs(got0 - Pd)) <= 1e-12 * np.max(np.abs(Pd))
