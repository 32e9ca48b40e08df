"""GPU timeline of one configs[1] e2e step (host CSR upload, one-call solve, host outputs):
CUPTI kernel / memcpy records with the idle gaps between them."""
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
n, l, m = M.nrows, 8, 1
shifts = sharding.log_shifts(l)


def pinned(a, dtype):
    t = torch.empty(a.shape, dtype=dtype, pin_memory=True)
    t.numpy()[...] = a
    return t


host_sys = [mg.SparseMatrix(x.nrows, x.ncols, pinned(x.row_ptr, torch.int64).numpy(),
                            pinned(x.col_idx, torch.int32).numpy(), pinned(x.values, torch.float64).numpy())
            for x in (M, D, K)]
B = np.zeros((1, n)); B[0, n - 2] = 1.0
B_host = pinned(B, torch.float64)
X_host, R_host, T_host = (torch.empty((l, m, n), dtype=torch.float64, pin_memory=True) for _ in range(3))


def step():
    hM, hD, hK = mg.DeviceCsr.upload_many(host_sys, ctx)
    mg.shifted_solve_raw(ctx, hM, hD, hK, shifts, 0, m, B_host.data_ptr(), 0, 1e-10, 1000, mg.mgpu.MGPU_HOST,
                         X_host.data_ptr(), R_host.data_ptr(), T_host.data_ptr())


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    if d > 2.0 or s - prev_end > 10.0:
        print(f"{s - t0:9.1f} us  +gap {s - prev_end:7.1f}  dur {d:9.1f}  {e.name[:60]}")
    prev_end = max(prev_end, e.time_range.end)
print(f"span {prev_end - t0:.1f} us")
