"""A/B of cg_stream's work plans on one shape.  Usage: python tools/stream_exp.py [iters] [ne] [m] [points] [ls]
(defaults: BASELINE configs[3] with the column-equilibrated A^2 LS factor).  Prints us per iteration for
stream_tiles = 0 (one contiguous row range per block), 1 (tiles where they hold >= 16 chunks), 2 (tiles always).
(The traffic experiment quoted in DESIGN.md 5 -- every point streaming point 0's operator values -- was a
temporary switch in the kernel, removed after the measurement.)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1606_01216_b200 as mg
a = [int(x) for x in sys.argv[1:]] + [None] * 5
k, ne, m, l, ls = a[0] or 100, a[1] or 500000, a[2] or 4, a[3] or 16, a[4] if a[4] is not None else 18
ctx = mg.Context(0)
M, D, K = mg.model_hermite_device(ne, ctx=ctx)
shifts = [10.0 ** (1 + 3 * i / (l - 1)) for i in range(l)] if l > 1 else [100.0]
ops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
chains = [[f.matrix] for f in mg.spai_ls_batched(ops, None, ls - 1, ctx=ctx)] if ls else [[] for _ in ops]
B = np.zeros((2 * ne, m))
for c in range(m):
    B[2 * ((c + 1) * ne // m) - 2, c] = 1.0
ctx.set_cg_path("stream")
ref = None
for tiles in [0, 1, 0, 1, 2]:
    ctx.set_option("stream_tiles", tiles)
    res = mg.cg_solve_batched(ops, chains, B, maxit=k, ctx=ctx)
    t = ctx.last_cg_timing()
    X = np.stack([r.X for r in res])
    if ref is None:
        ref = X
    d = float(np.max(np.abs(X - ref)) / np.max(np.abs(ref)))
    print(f"tiles={tiles}: {1e3 * t[0] / k:9.2f} us/iter   max rel diff to first run {d:.3e}", flush=True)
