"""SPAI build time: device vs the unmodified reference (oracle/_ref) on this box's host cores.

Rows: MR-SPAI frozen mode (reference thread pool = nproc), MR-SPAI sequential mode (the
reference default, single-threaded by construction), LS-SPAI (A pattern; the reference's
thin_qr-based restatement, single-threaded).  Device times are host wall time around the
synchronous C-ABI call, median of 3 after a warm-up.  Diagnostics for DESIGN.md.
"""
import os
import statistics
import sys
import time

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
    ref.force_kernels("scalar")
    threads = os.cpu_count() or 1
    ctx = mg.default_context()
    rows = []
    # MR frozen on the reference chain model (converges)
    for n in (20000, 100000):
        M, D, K = ref.chain_generate(n, consistent=True, stiffness_scale=1.0)
        A = ref.shifted_operator(M, D, K, 10.0)
        dA = mg.DeviceCsr.upload(A, ctx)
        tg = wall(lambda: mg.spai_build(dA, mode=mg.FROZEN, ctx=ctx))
        tr = wall(lambda: ref.spai_build(A, mode=1, threads=threads), reps=1)
        rows.append(("MR frozen", n, tg, tr, f"{threads} threads"))
    # MR sequential (heavy fill)
    for n in (500, 2000):
        M, D, K = ref.chain_generate(n, consistent=True, stiffness_scale=1.0)
        A = ref.shifted_operator(M, D, K, 100.0)
        dA = mg.DeviceCsr.upload(A, ctx)
        tg = wall(lambda: mg.spai_build(dA, mode=mg.SEQUENTIAL, ctx=ctx), reps=1)
        tr = wall(lambda: ref.spai_build(A, mode=0, threads=1), reps=1)
        rows.append(("MR sequential", n, tg, tr, "1 thread"))
    # LS on the BASELINE beam (A pattern)
    for ne in (10000, 100000):
        M, D, K = Oracle().hermite_generate(ne)  # bitwise the host generator
        A = ref.shifted_operator(M, D, K, 100.0)
        dA = mg.DeviceCsr.upload(A, ctx)
        tg = wall(lambda: mg.spai_ls(dA, None, mg.PATTERN_A, ctx=ctx))
        tr = wall(lambda: ref.spai_ls(A, None, 0), reps=1)
        rows.append(("LS (A pattern)", 2 * ne, tg, tr, "1 thread"))
    print("| SPAI | n | device | reference | speed-up | reference threads |")
    print("|---|---|---|---|---|---|")
    for name, n, tg, tr, th in rows:
        print(f"| {name} | {n} | {tg * 1e3:.2f} ms | {tr * 1e3:.1f} ms | {tr / tg:.0f}x | {th} |")


if __name__ == "__main__":
    main()
