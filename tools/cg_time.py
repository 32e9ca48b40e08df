"""CG kernel time on a BASELINE shape: python tools/cg_time.py [iters] [ne] [m] [points] [pattern] [opt=val ...]
pattern: -1 none, 0 A, 1 A^2, 16/17 colscale.  Prints us per batched iteration and the algorithmic
HBM fraction (B_iter = 8 nnz(A) + 8 nnz(P) + 48 n m per point, MEASURED_PEAKS.json hbm_gbs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1606_01216_b200 as mg
args = [a for a in sys.argv[1:] if "=" not in a]
opts = [a.split("=") for a in sys.argv[1:] if "=" in a]
a = [int(x) for x in args] + [None] * 5
k, ne, m, l = a[0] or 200, a[1] or 500000, a[2] or 4, a[3] or 16
pat = 0x11 if a[4] is None else a[4]
ctx = mg.Context(0)
for kk, vv in opts:
    ctx.set_option(kk, int(vv))
M, D, K = mg.model_hermite_device(ne, ctx=ctx)
n = 2 * ne
shifts = [10.0 ** (1 + 3 * i / (l - 1)) for i in range(l)] if l > 1 else [100.0]
ops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
chains = [[f.matrix] for f in mg.spai_ls_batched(ops, None, pat, ctx=ctx)] if pat >= 0 else [[] for _ in ops]
B = np.zeros((n, m))
for c in range(m):
    B[2 * ((c + 1) * ne // m) - 2, c] = 1.0
mg.cg_solve_batched(ops, chains, B, maxit=5, ctx=ctx)
res = mg.cg_solve_batched(ops, chains, B, maxit=k, ctx=ctx)
ms, it = ctx.last_cg_timing()
bits = sum(8 * o.stored_nnz + 48 * n * m for o in ops) + sum(8 * c[0].stored_nnz for c in chains if c)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6548.2
us = 1e3 * ms / it
print(json.dumps({"path": ctx.last_cg_path, "iters": it, "us_per_iter": us, "bytes_per_iter": bits,
                  "alg_GBs": bits / us / 1e3, "frac": bits / us / 1e3 / peak, "X0": float(res[0].X[0, 0])}), flush=True)
