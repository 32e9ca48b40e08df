"""Per-phase clock64 breakdown of the cluster CG kernel (context option profile_phases)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1606_01216_b200 as mg
ctx = mg.Context(0)
ctx.set_option("profile_phases", 1)
M, D, K = mg.model_hermite(10000)
shifts = [10.0 ** (1 + 3 * i / 7) for i in range(8)]
ops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
facs = mg.spai_ls_batched(ops, None, 0, ctx=ctx)
b = np.zeros(M.nrows); b[-2] = 1
mg.cg_solve_batched(ops, [[f.matrix] for f in facs], b, maxit=1000, ctx=ctx)
print("cg ms", ctx.last_cg_timing(), ctx.last_cg_path)
del ops, facs
ctx.close()
