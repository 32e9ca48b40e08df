"""LS-SPAI batch timing and FP64 roofline (BASELINE configs): python tools/ls_bench.py [workload ...]
workloads: c1 (n=2e4, 8 shifts, A), c3 (n=1e6, 16 shifts, A^2 colscale), c4 (n=1e7, 8 shifts, A colscale).
Time = CUDA events around mgpu_spai_ls_batched on the context stream (median of 5 after 2 warm-ups).
Algorithmic FLOPs per column: 2|I||J|^2 - 2/3|J|^3 + 2|I||J| + |J|^2 with the Hermite
|I| x |J| = 10 x 5 (A pattern) / 14 x 10 (A^2) of the interior columns."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_01216_b200 as mg

W = {"c1": (10000, 8, 0), "c3": (500000, 16, 0x11), "c4": (5000000, 8, 0x10), "c2": (50000, 8, 0)}
peak = None
pf = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "fp64_peak.json")
if os.path.exists(pf):
    peak = json.load(open(pf)).get("dfma_tflops")
ctx = mg.Context(0, stream=torch.cuda.current_stream().cuda_stream)
for name in (sys.argv[1:] or ["c1", "c3"]):
    ne, l, pat = W[name]
    M, D, K = mg.model_hermite_device(ne, ctx=ctx)
    shifts = [10.0 ** (1 + 3 * i / (l - 1)) for i in range(l)]
    ops = mg.shifted_operators(M, D, K, shifts, ctx=ctx)
    ts = []
    for r in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f = mg.spai_ls_batched(ops, None, pat, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
        del f
    ms = statistics.median(ts)
    n = 2 * ne
    nj, ni = (10, 14) if pat & 1 else (5, 10)  # interior Hermite columns
    flop = 2 * ni * nj * nj - 2 / 3 * nj ** 3 + 2 * ni * nj + nj * nj
    tf = flop * n * l / (ms * 1e-3) / 1e12
    print(json.dumps({"workload": name, "n": n, "shifts": l, "pattern": hex(pat), "ms": ms, "columns_per_s": n * l / (ms * 1e-3),
                      "alg_flop_per_column": flop, "alg_tflops": tf, "fp64_peak_tflops": peak,
                      "frac": (tf / peak) if peak else None}), flush=True)
    del ops, M, D, K
