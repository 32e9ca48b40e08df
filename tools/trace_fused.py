"""Host trace of one fused configs[1] step (build libmgpu with -DMGPU_HOST_TRACE, then python tools/trace_fused.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_01216_b200 as mg
from paper_1606_01216_b200 import sharding
dev = torch.device("cuda", 0); stream = torch.cuda.Stream(device=dev)
ctx = mg.Context(0, stream=stream.cuda_stream)
M, D, K = mg.model_hermite(10000); n = M.nrows; shifts = sharding.log_shifts(8)
dM, dD, dK = (mg.DeviceCsr.upload(x, ctx) for x in (M, D, K))
B_dev = torch.zeros((1, n), dtype=torch.float64, device=dev); B_dev[0, n - 2] = 1.0
X_dev = torch.empty((8, 1, n), dtype=torch.float64, device=dev)
for k in range(4):
    if k == 3:
        print("---- traced step", file=sys.stderr, flush=True)
    mg.shifted_solve_device(dM, dD, dK, shifts, 0, B_dev, X_dev, rtol=1e-10, maxit=1000, ctx=ctx)
