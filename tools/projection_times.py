"""Projection step time: thin_qr of the n x r basis block + project_reduce
(V^T M V, V^T D V, V^T K V, V^T F, Cp V, Cv V), device vs the unmodified reference on this
box.  Device times: host wall time around the synchronous C-ABI calls with the basis
already in host memory (the call stages it), median of 3.  Diagnostics for DESIGN.md.
"""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_01216_b200 as mg  # noqa: E402
from oracle import Oracle, Reference  # noqa: E402


def wall(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts)


def main():
    ref = Reference()
    orc = Oracle()
    ctx = mg.default_context()
    import ctypes as C
    import torch
    print("| n | r | device thin_qr (host arrays) | device thin_qr (device-resident) | reference thin_qr "
          "| device project_reduce | reference project_reduce |")
    print("|---|---|---|---|---|---|---|")
    for ne, r in ((50000, 16), (50000, 64), (500000, 16), (500000, 64)):
        M, D, K = orc.hermite_generate(ne)
        n = M.nrows
        rng = np.random.default_rng(r)
        Vt = np.asfortranarray(rng.standard_normal((n, r)))
        F = np.zeros((n, 1), order="F")
        F[n - 2, 0] = 1.0
        Cp = np.zeros((1, n), order="F")
        Cp[0, n - 2] = 1.0
        Cv = np.zeros((1, n), order="F")
        dM, dD, dK = (mg.DeviceCsr.upload(x, ctx) for x in (M, D, K))
        tq = wall(lambda: mg.thin_qr(Vt, ctx=ctx))
        # device-resident: the C ABI on device buffers (where = MGPU_DEVICE), no staging
        Ad = torch.tensor(np.asfortranarray(Vt).ravel(order="F"), device="cuda")
        Qd = torch.empty_like(Ad)
        Rd = torch.empty(r * r, dtype=torch.float64, device="cuda")
        rk = C.c_int64()

        def dev_qr():
            ctx.check(mg.lib().mgpu_thin_qr(ctx.handle, n, r, C.c_void_p(Ad.data_ptr()), 1e-12,
                                            C.c_void_p(Qd.data_ptr()), C.c_void_p(Rd.data_ptr()), C.byref(rk),
                                            mg.mgpu.MGPU_DEVICE))
        tqd = wall(dev_qr)
        tqr = wall(lambda: ref.thin_qr(Vt), reps=1)
        V, _, _ = mg.thin_qr(Vt, ctx=ctx)
        tp = wall(lambda: mg.project_reduce(dM, dD, dK, V, F, Cp, Cv, ctx=ctx))
        tpr = wall(lambda: ref.project_reduce(M, D, K, V, F, Cp, Cv), reps=1)
        print(f"| {n} | {r} | {tq * 1e3:.1f} ms | {tqd * 1e3:.1f} ms | {tqr * 1e3:.0f} ms | {tp * 1e3:.1f} ms "
              f"| {tpr * 1e3:.0f} ms |", flush=True)


if __name__ == "__main__":
    main()
