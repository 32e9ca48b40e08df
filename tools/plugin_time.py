"""Stage times of the plugin (include/mor_cuda.h) step on BASELINE configs[3]: prepare, the per-point solves."""
import time, sys, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1606_01216_b200 as mg
from paper_1606_01216_b200.plugin import PluginBackend
ne, m, l = 500000, 4, 16
M, D, K = mg.model_hermite(ne)
n = 2 * ne
F = np.zeros((n, m), order="F")
for c in range(m):
    F[2 * ((c + 1) * ne // m) - 2, c] = 1.0
shifts = [10.0 ** (1 + 3 * i / 15) for i in range(16)]
pb = PluginBackend(solver="cg_spai", algorithm="ls", ls_pattern=0x11, maxit=1000)
pb.set_system(M, D, K, F)
X = torch.empty((l, m, n), dtype=torch.float64, pin_memory=True).numpy()
for rep in range(3):
    t0 = time.perf_counter(); pb.prepare(shifts, 1); t1 = time.perf_counter()
    ts = []
    for i in range(l):
        a = time.perf_counter(); pb.solve(i, F, X=X[i], REC=X[i], TR=X[i]); ts.append(time.perf_counter() - a)
    print(f"prepare {1e3*(t1-t0):.1f} ms, solves {1e3*sum(ts):.1f} ms (first {1e3*ts[0]:.1f})", flush=True)
ctx = mg.default_context()
dM, dD, dK = (mg.DeviceCsr.upload(x, ctx) for x in (M, D, K))
t0 = time.perf_counter(); hs = mg.DeviceCsr.upload_many([M, D, K], ctx); ctx.synchronize(); print("upload_many pageable ms", 1e3*(time.perf_counter()-t0))
