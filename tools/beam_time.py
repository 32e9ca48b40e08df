import sys, time
sys.path.insert(0, '.')
import torch
import paper_1606_01216_b200 as mg
ctx = mg.default_context()
for ne in (500000, 5000000):
    mg.model_hermite_device(1000)
    torch.cuda.synchronize()
    t = time.perf_counter(); M, D, K = mg.model_hermite_device(ne); torch.cuda.synchronize(); dt = time.perf_counter() - t
    t = time.perf_counter(); h = mg.model_hermite(ne); th = time.perf_counter() - t
    print(f"ne={ne} n={2*ne}: device {dt*1e3:.1f} ms, host generator {th*1e3:.0f} ms")
