import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1606_01216_b200 as mg
from oracle import Oracle
o = Oracle()
ctx = mg.default_context()
for ne, pat, s, maxit in [(300, 1, 100.0, 8), (300, 0, 100.0, 8), (1000, 0, 100.0, 8), (5000, 0, 100.0, 8)]:
    M, D, K = o.hermite_generate(ne)
    A = o.shifted_operator(M, D, K, s)
    P = o.spai_ls(A, None, pat)
    b = np.ones(A.nrows)
    want = o.pcg_solve(A, [P], b, maxit=maxit)
    for path in ["banded", "stream"]:
        ctx.set_cg_path(path)
        try:
            got = mg.pcg_solve(A, [P], b, maxit=maxit, history_cap=maxit)
            print(ne, pat, path, ctx.last_cg_path, "hist", np.array2string(got["relres_history"][:6], precision=6),
                  "ref", np.array2string(want["relres_history"][:6], precision=6))
        except Exception as e:
            print(ne, pat, path, "ERR", e)
ctx.set_cg_path("auto")
