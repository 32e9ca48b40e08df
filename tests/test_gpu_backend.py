"""The SolveBackend plugin (airga.hpp:133-147): device backends against the reference CgBackend.

(1) the C++ drop-in CudaCgBackend (paper_1606_01216_b200/host) linked with the
    unmodified reference library in one binary (tests/cpp/backend_parity.cpp);
(2) the Python mirror CudaCgBackend against the reference CgBackend through
    oracle/_ref (ref_backend_*), over an AIRGA-style sequence with the update chain.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, rel

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref", "backend_parity")


def test_cpp_dropin_backend_parity():
    if not os.path.exists(BIN):
        pytest.skip("backend_parity not built (needs the reference headers at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    res = json.loads(line)
    assert out.returncode == 0 and res["failures"] == 0, (res, out.stderr[-2000:])
    assert res["solves"] >= 20 and res["max_rel_x"] <= 1e-8 and res["max_iter_diff"] <= 2


@pytest.mark.parametrize("solver,mode,n", [("cg_spai_update", 1, 1500), ("cg_spai", 1, 1500), ("cg_plain", 1, 1500),
                                          ("cg_spai_update", 0, 400), ("cg_spai", 0, 400)])
def test_python_backend_sequence(mg, ref, solver, mode, n):
    """mode 1 = frozen, 0 = sequential (AirgaConfig's default)."""
    from paper_1606_01216_b200.backend import CudaCgBackend, CudaCgConfig
    M, D, K = ref.chain_generate(n, consistent=True, stiffness_scale=1.0)
    rb = ref.backend(solver, M, D, K, spai_mode=mode, update_start_iteration=2)
    gb = CudaCgBackend(CudaCgConfig(solver=solver, update_start_iteration=2, spai_mode=mode))
    F = np.zeros((n, 1))
    F[0, 0] = 1.0
    seq = [[1.0, 10.0, 100.0], [2.0, 12.0, 90.0], [3.0, 15.0, 80.0]]
    for z, pts in enumerate(seq, start=1):
        rr = rb.prepare(pts, z)
        gr = []
        gb.prepare((M, D, K), pts, z, gr)
        if solver != "cg_plain":
            assert [r["kind"] for r in rr] == [g.kind for g in gr]
            assert [r["chain_length"] for r in rr] == [g.chain_length for g in gr]
        batch = gb.solve_all(F)
        for i in range(len(pts)):
            want = rb.solve(i, F)
            got = gb.solve(i, F)
            assert rel(got.X, want["X"]) < 1e-8
            assert rel(batch[i].X, want["X"]) < 1e-8
            assert np.all(np.abs(got.iterations - want["iterations"]) <= 2)
            assert got.all_converged == want["all_converged"]
