"""Per-phase clock64 breakdown of the streaming CG kernel on the BASELINE configs[3] shape
(MGPU_PROFILE_PHASES=1; block 0, thread 0).  Usage: python tools/stream_prof.py [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1606_01216_b200 as mg
k = int(sys.argv[1]) if len(sys.argv) > 1 else 50
ne, m = 500000, 4
ctx = mg.Context(0)
M, D, K = mg.model_hermite_device(ne, ctx=ctx)
shifts = [10.0 ** (1 + 3 * i / 15) for i in range(16)]
ops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
B = np.zeros((2 * ne, m))
for c in range(m):
    B[2 * ((c + 1) * ne // m) - 2, c] = 1.0
ctx.set_cg_path("stream")
mg.cg_solve_batched(ops, [[] for _ in ops], B, maxit=k, ctx=ctx)
t = ctx.last_cg_timing()
print("cg", t, "us/iter", 1e3 * t[0] / k if isinstance(t, tuple) else t)
del ops, M, D, K
ctx.close()
