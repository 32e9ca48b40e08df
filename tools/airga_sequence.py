"""BASELINE configs[2]: the AIRGA-style sequence, SPAI update against rebuild-from-scratch.

Hermite beam ne = 50,000 (n = 1e5); 10 outer iterations; in each, 8 shifts drawn
log-uniform in [10, 1e4] from mt19937_64(42) (sharding.airga_shift_draws),
sorted, update partners paired by index (airga.cpp:145).  Both arms run through the
SolveBackend mirror (backend.CudaCgBackend, airga.cpp:103-190) with LS-SPAI on A's pattern
(the reference's MR-SPAI stagnates at column 0 on this beam):

  update  -- solver cg_spai_update, update_start_iteration = 2: a fresh factor at z = 1,
             afterwards Q_z = LS update (K_new Q ~ K_old on A's pattern) pushed onto the
             chain, so the preconditioner at z is Q_z ... Q_2 P_1 (z factors);
  collapse-- the same updates, the chain collapsed into one factor after each (P <- Q P, device
             SpGEMM; north-star subsystem 2), so every CG iteration applies one wider factor;
  rebuild -- solver cg_spai: a fresh LS factor at every z (chain length 1).

Per outer iteration and arm: prepare time (device assembly of the 8 operators + the batched
SPAI build or update), CG kernel time at the fixed budget (rtol 1e-10 is unreachable in FP64
on this beam), the worst achieved true relative residual over the shifts, and the chain
length.  --ref-budget K also times the unmodified reference (oracle/_ref) on the same
sequence: shifted_operator, LS factor from reference primitives (ref_spai_ls, with K_old for
the update arm), pcg_solve with the whole chain, K CG iterations per shift, shifts on
concurrent host threads; its CG time is scaled to the device budget.

Usage: python tools/airga_sequence.py [--ne 50000] [--outer 10] [--budget 1000]
                                      [--ref-budget 20] [--out profiles/r01_airga_sequence.json]
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1606_01216_b200 as mg
from paper_1606_01216_b200.backend import CudaCgBackend, CudaCgConfig
from paper_1606_01216_b200.sharding import airga_shift_draws


def device_arm(update: bool, sysm, draws, b, budget, ctx, collapse=False):
    cfg = CudaCgConfig(solver="cg_spai_update" if update else "cg_spai", spai_algorithm="ls",
                       ls_pattern=mg.PATTERN_A, update_start_iteration=2, maxit_override=budget, collapse=collapse)
    be = CudaCgBackend(cfg, ctx=ctx)
    rows = []
    bn = np.linalg.norm(b)
    for z, pts in enumerate(draws, start=1):
        recs = []
        ctx.synchronize()
        t0 = time.perf_counter()
        be.prepare(sysm, pts, z, recs)
        ctx.synchronize()
        t1 = time.perf_counter()
        res = be.solve_all(b, raise_on_breakdown=False)
        t2 = time.perf_counter()
        cg_ms, loop_it = ctx.last_cg_timing()
        relres = [float(np.linalg.norm(r.true_residuals[:, 0]) / bn) for r in res]
        factor_nnz = sum(mg.mgpu._factor_mat(f).stored_nnz for f in be.chains[0]) if be.chains else 0
        rows.append({"outer": z, "shifts": pts, "kind": recs[0].kind, "chain_length": recs[0].chain_length,
                     "factors_applied": len(be.chains[0]) if be.chains else 0, "factor_nnz_point0": factor_nnz,
                     "prepare_ms": 1e3 * (t1 - t0), "spai_ms": 1e3 * sum(r.seconds for r in recs),
                     "solve_ms": 1e3 * (t2 - t1), "cg_kernel_ms": cg_ms, "cg_iterations": int(loop_it),
                     "cg_kernel": ctx.last_cg_path, "breakdowns": int(sum(int(r.status[0] != 0) for r in res)),
                     "max_true_relres": max(relres), "median_true_relres": float(np.median(relres))})
        print(json.dumps({"arm": ("collapse" if collapse else "update") if update else "rebuild",
                          **{k: v for k, v in rows[-1].items()
                                                                      if k != "shifts"}}), flush=True)
    return rows


def reference_arm(update: bool, ne, draws, b, ref_budget, budget, outers):
    from oracle import Oracle, Reference, reference_available
    lib = Reference() if reference_available() else Oracle()
    M, D, K = Oracle().hermite_generate(ne)
    threads = min(len(draws[0]), os.cpu_count() or 1)
    chains = [[] for _ in draws[0]]
    prev = [None] * len(draws[0])
    rows = []
    for z, pts in enumerate(draws, start=1):
        def one(i):
            t0 = time.perf_counter()
            A = lib.shifted_operator(M, D, K, pts[i])
            if update and z >= 2:
                chain = [lib.spai_ls(A, prev[i], 0)] + chains[i]
            else:
                chain = [lib.spai_ls(A, None, 0)]
            t1 = time.perf_counter()
            r = lib.pcg_solve(A, chain, b, rtol=1e-10, maxit=ref_budget, history_cap=1) if z in outers else None
            t2 = time.perf_counter()
            return A, chain, t1 - t0, t2 - t1, r

        with ThreadPoolExecutor(threads) as ex:
            t0 = time.perf_counter()
            out = list(ex.map(one, range(len(pts))))
            wall = time.perf_counter() - t0
        for i, (A, chain, _, _, _) in enumerate(out):
            prev[i], chains[i] = A, chain
        if z in outers:
            prep = max(o[2] for o in out)
            cg = max(o[3] for o in out)
            rows.append({"outer": z, "chain_length": len(chains[0]), "prepare_ms": 1e3 * prep,
                         "cg_ms_at_ref_budget": 1e3 * cg, "cg_ms_scaled_to_budget": 1e3 * cg * budget / ref_budget,
                         "wall_ms": 1e3 * wall, "threads": threads, "kind": lib.kind})
            print(json.dumps({"arm": ("update" if update else "rebuild") + "-reference", **rows[-1]}), flush=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ne", type=int, default=50000)
    ap.add_argument("--outer", type=int, default=10)
    ap.add_argument("--shifts", type=int, default=8)
    ap.add_argument("--budget", type=int, default=1000)
    ap.add_argument("--ref-budget", type=int, default=0, help="CG iterations per shift in the reference arm (0: skip)")
    ap.add_argument("--ref-outers", default="1,2,5,10")
    ap.add_argument("--out", default="")
    ap.add_argument("--cg-path", default="auto", help="auto | stream | banded | general (diagnostics)")
    ap.add_argument("--arms", default="update,collapse,rebuild")
    a = ap.parse_args()
    draws = airga_shift_draws(a.outer, a.shifts)
    ctx = mg.Context(0)
    ctx.set_cg_path(a.cg_path)
    M, D, K = mg.model_hermite_device(a.ne, ctx=ctx)
    n = 2 * a.ne
    b = np.zeros(n)
    b[n - 2] = 1.0
    # warm-up: build and update paths, several chain lengths (first-use module loading and memory
    # pool growth otherwise land in the first measured outer iterations)
    device_arm(True, (M, D, K), draws[:4], b, a.budget, ctx)
    result = {"workload": f"BASELINE configs[2]: Hermite ne={a.ne} (n={n}), {a.outer} outer iterations x "
                          f"{a.shifts} shifts log-uniform in [10,1e4] (mt19937_64 seed 42, sorted), LS-SPAI on the "
                          f"A pattern, update from z=2 vs rebuild, CG budget {a.budget}",
              "cg_path": a.cg_path}
    for arm in a.arms.split(","):
        result[arm] = device_arm(arm in ("update", "collapse"), (M, D, K), draws, b, a.budget, ctx,
                                 collapse=arm == "collapse")
    if a.ref_budget > 0:
        outers = {int(x) for x in a.ref_outers.split(",")}
        result["reference_update"] = reference_arm(True, a.ne, draws, b, a.ref_budget, a.budget, outers)
        result["reference_rebuild"] = reference_arm(False, a.ne, draws, b, a.ref_budget, a.budget, outers)
        result["reference_note"] = (f"reference CG timed at {a.ref_budget} iterations per shift and scaled to "
                                    f"{a.budget}; prepare = shifted_operator + ref_spai_ls per shift (max over the "
                                    f"concurrent shifts)")
    if a.out:
        with open(a.out, "w") as f:
            json.dump(result, f, indent=1)


if __name__ == "__main__":
    main()
