"""Per-phase clock64 breakdown of the streaming CG kernel (context option profile_phases; block 0,
thread 0).  Usage: python tools/stream_prof.py [iters] [ne] [m] [points] [ls]
(defaults: BASELINE configs[3] shape, 50 iterations; ls = pattern + 1 adds an LS-SPAI factor per point: 1 A, 2 A^2, 18 A^2 colscale)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1606_01216_b200 as mg
a = [int(x) for x in sys.argv[1:]] + [None] * 5
k, ne, m, l, ls = a[0] or 50, a[1] or 500000, a[2] or 4, a[3] or 16, a[4] or 0
ctx = mg.Context(0)
ctx.set_option("profile_phases", 1)
M, D, K = mg.model_hermite_device(ne, ctx=ctx)
shifts = [10.0 ** (1 + 3 * i / (l - 1)) for i in range(l)] if l > 1 else [100.0]
ops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
chains = [[f.matrix] for f in mg.spai_ls_batched(ops, None, ls - 1, ctx=ctx)] if ls else [[] for _ in ops]
B = np.zeros((2 * ne, m))
for c in range(m):
    B[2 * ((c + 1) * ne // m) - 2, c] = 1.0
ctx.set_cg_path("stream")
mg.cg_solve_batched(ops, chains, B, maxit=k, ctx=ctx)
t = ctx.last_cg_timing()
print("cg", t, "us/iter", 1e3 * t[0] / k)
del ops, chains, M, D, K
ctx.close()
