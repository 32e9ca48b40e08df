"""GPU timeline of one configs[1] bench step (torch.profiler / CUPTI kernel and memcpy records):
every device activity with its start offset and duration, and the idle gaps between them."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
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


def step():
    ops = mg.shifted_operators(dM, dD, dK, shifts, ctx=ctx)
    facs = mg.spai_ls_batched(ops, None, 0, ctx=ctx)
    mg.cg_solve_device(ops, [[f.matrix] for f in facs], B_dev, X_dev, R_dev, T_dev, rtol=1e-10, maxit=1000, ctx=ctx)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
busy = 0.0
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = s - prev_end
    busy += d
    print(f"{s - t0:9.1f} us  +gap {gap:7.1f}  dur {d:9.1f}  {e.name[:70]}")
    prev_end = max(prev_end, e.time_range.end)
print(f"span {prev_end - t0:.1f} us, device busy {busy:.1f} us")
