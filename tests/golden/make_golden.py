"""Generates tests/golden/*.npz from the UNMODIFIED reference library (oracle/_ref).

Run in the build container (needs oracle/_ref/libmorref.so, i.e. /root/reference):
    make -C oracle ref && python tests/golden/make_golden.py
The reference runs with the SCALAR kernel table (MOR_KERNELS=scalar equivalent,
kernels_dispatch.cpp:633-641), the canonical oracle variant.
Every array written here is an output of a reference entry point; tests pin the
C restatement (oracle/oracle.c) to them bit for bit.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import OracleError, Reference  # noqa: E402


def csr(prefix, A):
    return {f"{prefix}_rp": A.row_ptr, f"{prefix}_ci": A.col_idx, f"{prefix}_v": A.values}


def hermite_triplets(ne, E=2.1e11, I=1e-8, rho=7800.0, area=1e-4, L=1.0):
    """BASELINE beam element loop; same coefficient arithmetic as the generators."""
    h = L / ne
    kc = (E * I) / (h * h * h)
    mc = (rho * area * h) / 420.0
    hh = h * h
    kcoef = [[12.0, 6.0 * h, -12.0, 6.0 * h], [6.0 * h, 4.0 * hh, -6.0 * h, 2.0 * hh],
             [-12.0, -6.0 * h, 12.0, -6.0 * h], [6.0 * h, 2.0 * hh, -6.0 * h, 4.0 * hh]]
    mcoef = [[156.0, 22.0 * h, 54.0, -13.0 * h], [22.0 * h, 4.0 * hh, 13.0 * h, -3.0 * hh],
             [54.0, 13.0 * h, 156.0, -22.0 * h], [-13.0 * h, -3.0 * hh, -22.0 * h, 4.0 * hh]]
    r, c, kv, mv = [], [], [], []
    for e in range(ne):
        dofs = [2 * e - 2, 2 * e - 1, 2 * e, 2 * e + 1]
        for a in range(4):
            for b in range(4):
                if dofs[a] < 0 or dofs[b] < 0:
                    continue
                r.append(dofs[a])
                c.append(dofs[b])
                kv.append(kc * kcoef[a][b])
                mv.append(mc * mcoef[a][b])
    return 2 * ne, np.array(r), np.array(c), np.array(kv), np.array(mv)


def main():
    ref = Reference()
    assert ref.force_kernels("scalar")
    out = {}
    # ---- reference chain model (model_io.cpp:18-87), consistent mass, stiffness 1
    M, D, K = ref.chain_generate(200, alpha=0.1, beta=1e-5, stiffness_scale=1.0, consistent=True)
    out.update(csr("chain_M", M) | csr("chain_D", D) | csr("chain_K", K))
    A1 = ref.shifted_operator(M, D, K, 3.0)
    A2 = ref.shifted_operator(M, D, K, 3.5)
    out.update(csr("chain_A1", A1) | csr("chain_A2", A2))
    out["chain_trace_A1"] = np.array([ref.trace(A1)])
    out["chain_trace_inner_A1A2"] = np.array([ref.trace_inner(A1, A2)])
    At = ref.transpose(A1)
    out.update(csr("chain_A1t", At))
    for mode, tag in ((1, "frozen"), (0, "seq")):
        P, res = ref.spai_build(A1, mode=mode)
        out.update(csr(f"chain_P_{tag}", P))
        out[f"chain_Pres_{tag}"] = res
        Q, qres = ref.spai_update(A1, A2, mode=mode)
        out.update(csr(f"chain_Q_{tag}", Q))
        out[f"chain_Qres_{tag}"] = qres
    P, _ = ref.spai_build(A1, mode=1)
    Q, _ = ref.spai_update(A1, A2, mode=1)
    b = np.zeros(200)
    b[0] = 1.0
    out["chain_b"] = b
    sol = ref.pcg_solve(A2, [Q, P], b, rtol=1e-10)
    out["chain_pcg_x"] = sol["solution"]
    out["chain_pcg_res"] = sol["residual"]
    out["chain_pcg_rec"] = sol["recurrence_residual"]
    out["chain_pcg_it"] = np.array([sol["iterations"], int(sol["converged"])])
    out["chain_pcg_hist"] = sol["relres_history"]
    v = np.linspace(-1.0, 1.0, 200)
    out["chain_apply_v"] = v
    out["chain_apply_out"] = ref.chain_apply([Q, P], v)
    out["chain_spmv_out"] = ref.spmv(A1, v)
    B = np.zeros((200, 3))
    B[0, 0] = 1.0
    B[:, 2] = np.cos(np.arange(200))
    bs = ref.block_solve(A1, [P], B, rtol=1e-10)
    out["chain_block_B"] = B
    out["chain_block_X"] = bs["X"]
    out["chain_block_it"] = bs["iterations"]
    # ---- Hermite beam (BASELINE), ne = 100: assembly through reference from_triplets
    n, r, c, kv, mv = hermite_triplets(100)
    Kh = ref.from_triplets(n, n, r, c, kv)
    Mh = ref.from_triplets(n, n, r, c, mv)
    Dh = ref.sp_add_scaled(Mh, Kh, 0.1, 1e-5)
    out.update(csr("herm_M", Mh) | csr("herm_D", Dh) | csr("herm_K", Kh))
    H1 = ref.shifted_operator(Mh, Dh, Kh, 100.0)
    H2 = ref.shifted_operator(Mh, Dh, Kh, 150.0)
    out.update(csr("herm_A1", H1) | csr("herm_A2", H2))
    # pattern | 0x10: the column-equilibrated LS variant (ref_shim.cpp ref_spai_ls, reference thin_qr)
    for pat in (0, 1, 0x10, 0x11):
        out.update(csr(f"herm_LS{pat}", ref.spai_ls(H1, None, pat)))
        out.update(csr(f"herm_LSU{pat}", ref.spai_ls(H2, H1, pat)))
    Pl = ref.spai_ls(H1, None, 0)
    bh = np.zeros(n)
    bh[n - 2] = 1.0
    sh = ref.pcg_solve(H1, [Pl], bh, rtol=1e-10, maxit=60)
    out["herm_pcg_x"] = sh["solution"]
    out["herm_pcg_it"] = np.array([sh["iterations"], int(sh["converged"])])
    try:
        ref.spai_build(H1, mode=1)
        out["herm_mr_err"] = np.array([-1])
    except OracleError as e:
        out["herm_mr_err"] = np.array([e.status, e.index])
        out["herm_mr_msg"] = np.array([e.msg])
    # ---- thin QR (dense.cpp:153-246)
    rng = np.random.default_rng(1234)
    S = rng.standard_normal((10, 5))
    S[:, 3] *= 1e-6
    Qm, R, rank = ref.thin_qr(S)
    out["qr_S"], out["qr_Q"], out["qr_R"], out["qr_rank"] = S, Qm, R, np.array([rank])
    # ---- breakdown (krylov.cpp:106-111) on an indefinite diagonal
    from oracle import Csr
    Ad = Csr.from_dense(np.diag([1.0, -1.0, 2.0]))
    try:
        ref.pcg_solve(Ad, [], np.array([1.0, 1.0, 0.0]))
        out["bd"] = np.array([-1, -1])
    except OracleError as e:
        out["bd"] = np.array([e.status, e.index])
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
