import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1606_01216_b200 as mg
from paper_1606_01216_b200 import sharding
dev = torch.device("cuda", 0); stream = torch.cuda.Stream(device=dev)
ctx = mg.Context(0, stream=stream.cuda_stream)
M, D, K = mg.model_hermite(10000); n = M.nrows; shifts = sharding.log_shifts(8)
dM, dD, dK = (mg.DeviceCsr.upload(x, ctx) for x in (M, D, K))
B = np.zeros((n, 1)); B[n - 2, 0] = 1.0
B_dev = torch.tensor(B.T.copy(), dtype=torch.float64, device=dev).contiguous()
X_dev = torch.empty((8, 1, n), dtype=torch.float64, device=dev); R_dev, T_dev = torch.empty_like(X_dev), torch.empty_like(X_dev)
def mark(tr, what):
    if tr:
        print(f"[py   {time.monotonic_ns() / 1e3:10.1f} us] {what}", file=sys.stderr, flush=True)
def step(tr):
    t = time.perf_counter()
    ops = mg.shifted_operators(dM, dD, dK, shifts, ctx=ctx); t1 = time.perf_counter()
    mark(tr, "spai call")
    facs = mg.spai_ls_batched(ops, None, 0, ctx=ctx); t2 = time.perf_counter()
    mark(tr, "spai returned")
    ch = [[f.matrix] for f in facs]
    mark(tr, "before cg_solve_device")
    mg.cg_solve_device(ops, ch, B_dev, X_dev, R_dev, T_dev, rtol=1e-10, maxit=1000, ctx=ctx); t3 = time.perf_counter()
    if tr: print(f"py: asm {1e6*(t1-t):.0f} spai {1e6*(t2-t1):.0f} cg {1e6*(t3-t2):.0f} us", file=sys.stderr, flush=True)
for _ in range(3): step(False)
step(True)
