"""Chunk-height / ring-depth sweep of cg_stream on one shape (context options stream_chunk, stream_ring).
Usage: python tools/stream_chunk_sweep.py [iters] [ne] [m] [points] [ls]  (defaults: the configs[2] shape)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1606_01216_b200 as mg
a = [int(x) for x in sys.argv[1:]] + [None] * 5
k, ne, m, l, ls = a[0] or 1000, a[1] or 50000, a[2] or 1, a[3] or 8, a[4] if a[4] is not None else 1
ctx = mg.Context(0)
M, D, K = mg.model_hermite_device(ne, ctx=ctx)
shifts = [10.0 ** (1 + 3 * i / (l - 1)) for i in range(l)] if l > 1 else [100.0]
ops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
chains = [[f.matrix] for f in mg.spai_ls_batched(ops, None, ls - 1, ctx=ctx)] if ls else [[] for _ in ops]
B = np.zeros((2 * ne, m))
for c in range(m):
    B[2 * ((c + 1) * ne // m) - 2, c] = 1.0
ctx.set_cg_path("stream")
for ch, ring in [(0, 0)] + [(int(c), int(r)) for c, r in (x.split(":") for x in os.environ.get("SWEEP", "1024:2,768:3,512:3,512:4,384:4,256:4,256:3,320:2,192:3").split(","))]:
    ctx.set_option("stream_chunk", ch)
    if ch:
        ctx.set_option("stream_ring", ring)
    try:
        mg.cg_solve_batched(ops, chains, B, maxit=k, ctx=ctx)
        t = ctx.last_cg_timing()
        print(f"chunk={ch} ring={ring}: {1e3 * t[0] / k:9.2f} us/iter", flush=True)
    except Exception as e:  # a plan that does not fit falls back to the planner's; report errors only
        print(f"chunk={ch} ring={ring}: {type(e).__name__} {e}", flush=True)
