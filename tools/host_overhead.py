"""Host-side cost of the bench step's API calls (configs[1]): each call timed with the device
idle before it (torch.cuda.synchronize), so the time is the host path plus its own device work.
cg_solve_device with maxit=1 isolates the solve's host planning from the CG loop."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cProfile, pstats
import numpy as np
import torch
import paper_1606_01216_b200 as mg
from paper_1606_01216_b200 import sharding

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
ctx = mg.Context(0, stream=stream.cuda_stream)
M, D, K = mg.model_hermite(10000)
n = M.nrows
shifts = sharding.log_shifts(8)
dM, dD, dK = (mg.DeviceCsr.upload(x, ctx) for x in (M, D, K))
B = np.zeros((n, 1)); B[n - 2, 0] = 1.0
B_dev = torch.tensor(B.T.copy(), dtype=torch.float64, device=dev).contiguous()
X_dev = torch.empty((8, 1, n), dtype=torch.float64, device=dev)
R_dev, T_dev = torch.empty_like(X_dev), torch.empty_like(X_dev)


def timed(label, fn, reps=20):
    out = None
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        ctx.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"{label:40s} median {1e6 * float(np.median(ts)):8.1f} us")
    return out

ops = timed("shifted_operators (8)", lambda: mg.shifted_operators(dM, dD, dK, shifts, ctx=ctx))
facs = timed("spai_ls_batched (8)", lambda: mg.spai_ls_batched(ops, None, 0, ctx=ctx))
chains = [[f.matrix] for f in facs]
timed("cg_solve_device maxit=1", lambda: mg.cg_solve_device(ops, chains, B_dev, X_dev, R_dev, T_dev, rtol=1e-10,
                                                             maxit=1, ctx=ctx))
timed("cg_solve_device maxit=0", lambda: mg.cg_solve_device(ops, chains, B_dev, X_dev, R_dev, T_dev, rtol=1e-10,
                                                             maxit=0, ctx=ctx))
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    mg.cg_solve_device(ops, chains, B_dev, X_dev, R_dev, T_dev, rtol=1e-10, maxit=1, ctx=ctx)
    ops2 = mg.shifted_operators(dM, dD, dK, shifts, ctx=ctx)
    f2 = mg.spai_ls_batched(ops2, None, 0, ctx=ctx)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
