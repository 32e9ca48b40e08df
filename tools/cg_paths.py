"""Per-path CG kernel time (µs per batched iteration) on a Hermite workload (diagnostics; GPU box).

usage: python tools/cg_paths.py NE NSHIFTS M PATTERN(a|a2|none) BUDGET path[,path...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1606_01216_b200 as mg  # noqa: E402

ne, ns, m = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pat, budget = sys.argv[4], int(sys.argv[5])
paths = sys.argv[6].split(",")
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
ctx = mg.Context(0, stream=stream.cuda_stream)
M, D, K = mg.model_hermite(ne)
n = M.nrows
shifts = [10.0 ** (1 + 3 * i / max(ns - 1, 1)) for i in range(ns)]
dM, dD, dK = (mg.DeviceCsr.upload(x, ctx) for x in (M, D, K))
ops = mg.shifted_operators(dM, dD, dK, shifts, ctx=ctx)
if pat == "none":
    chains = [[] for _ in ops]
else:
    facs = mg.spai_ls_batched(ops, None, mg.PATTERN_A if pat == "a" else mg.PATTERN_A2, ctx=ctx)
    chains = [[f.matrix] for f in facs]
g = torch.Generator().manual_seed(7)
B_dev = torch.rand((m, n), dtype=torch.float64, generator=g).to(dev)
X = torch.empty((ns, m, n), dtype=torch.float64, device=dev)
R = torch.empty_like(X)
T = torch.empty_like(X)
for path in paths:
    ctx.set_cg_path(path)
    best = None
    for rep in range(3):
        mg.cg_solve_device(ops, chains, B_dev, X, R, T, maxit=budget, ctx=ctx)
        stream.synchronize()
        ms, loops = ctx.last_cg_timing()
        us = 1e3 * ms / max(loops, 1)
        best = us if best is None else min(best, us)
    print(f"ne={ne} shifts={ns} m={m} pattern={pat} path={path} ran={ctx.last_cg_path} "
          f"us_per_iter={best:.2f} loops={loops}", flush=True)
del ops, chains
if pat != "none":
    del facs
del dM, dD, dK
stream.synchronize()
ctx.close()
