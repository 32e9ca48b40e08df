"""Host/device time per API call of one bench step (diagnostics; run on the GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_01216_b200 as mg

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
ctx = mg.Context(0, stream=stream.cuda_stream)
ne = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
M, D, K = mg.model_hermite(ne)
n = M.nrows
shifts = [10.0 ** (1 + 3 * i / 7) for i in range(8)]
dM, dD, dK = (mg.DeviceCsr.upload(x, ctx) for x in (M, D, K))
B_dev = torch.zeros((1, n), dtype=torch.float64, device=dev); B_dev[0, n - 2] = 1
X = torch.empty((8, 1, n), dtype=torch.float64, device=dev); R = torch.empty_like(X); T = torch.empty_like(X)
for rep in range(4):
    t = [time.perf_counter()]
    ops = mg.shifted_operators(dM, dD, dK, shifts, ctx=ctx); stream.synchronize(); t.append(time.perf_counter())
    facs = mg.spai_ls_batched(ops, None, 0, ctx=ctx); stream.synchronize(); t.append(time.perf_counter())
    it = mg.cg_solve_device(ops, [[f.matrix] for f in facs], B_dev, X, R, T, maxit=1000, ctx=ctx); stream.synchronize(); t.append(time.perf_counter())
    del ops, facs; stream.synchronize(); t.append(time.perf_counter())
    cg_ms, loops = ctx.last_cg_timing()
    print("asm %.2f ms  spai %.2f ms  cg %.2f ms (kernel %.2f)  free %.2f ms" % tuple(
        [1e3 * (t[i + 1] - t[i]) for i in range(2)] + [1e3 * (t[3] - t[2]), cg_ms, 1e3 * (t[4] - t[3])]))
