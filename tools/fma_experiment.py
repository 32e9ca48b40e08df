"""DESIGN.md 5 experiment: cg_cluster_v2 with DFMA in the SpMV / dot / axpy terms (the reference's AVX2
kernel table contracts them, kernels_avx2.cpp:34-35, 57, 88) against the default two-rounding terms
(the scalar table, bitwise).  BASELINE configs[1] (n = 2e4, 8 shifts, LS-SPAI on A's pattern), CG at
the 1000-iteration budget: us per batched iteration and the iterate drift from the oracle's
pcg_solve (scalar order) at k = 1000.
  make fma-exp && python tools/fma_experiment.py   (runs both libraries in subprocesses)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one():
    import numpy as np
    import paper_1606_01216_b200 as mg
    from oracle import Oracle
    orc = Oracle()
    M, D, K = orc.hermite_generate(10000)
    n = M.nrows
    b = np.zeros(n)
    b[n - 2] = 1.0
    shifts = [10.0 ** (1 + 3 * i / 7) for i in range(8)]
    ops = [orc.shifted_operator(M, D, K, s) for s in shifts]
    facs = [orc.spai_ls(A, None, 0) for A in ops]
    ctx = mg.default_context()
    mg.cg_solve_batched(ops, [[f] for f in facs], b, maxit=50, ctx=ctx)
    res = mg.cg_solve_batched(ops, [[f] for f in facs], b, maxit=1000, ctx=ctx)
    ms, it = ctx.last_cg_timing()
    drift = []
    for A, P, r in zip(ops, facs, res):
        w = orc.pcg_solve(A, [P], b, rtol=1e-10, maxit=1000)["solution"]
        drift.append(float(np.max(np.abs(r.X[:, 0] - w)) / np.max(np.abs(w))))
    print(json.dumps({"lib": os.environ.get("MGPU_LIB", "default"), "path": ctx.last_cg_path,
                      "us_per_iter": 1e3 * ms / it, "max_rel_drift_k1000": max(drift), "drift": drift}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one()
        sys.exit(0)
    out = {}
    for tag, lib in (("two_roundings", None), ("dfma", os.path.join(ROOT, "paper_1606_01216_b200", "lib", "exp",
                                                                     "libmgpu_fma.so"))):
        env = dict(os.environ)
        if lib:
            env["MGPU_LIB"] = lib
        p = subprocess.run([sys.executable, __file__, "--one"], capture_output=True, text=True, env=env)
        line = [l for l in p.stdout.splitlines() if l.startswith("{")]
        out[tag] = json.loads(line[-1]) if line else {"error": p.stderr[-1500:]}
        print(tag, json.dumps(out[tag]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "r02_fma_experiment.json"), "w") as f:
        json.dump(out, f, indent=1)
