"""NCCL data-plane check under torchrun (one process per GPU): shift-sharded columns ->
row slabs (mgpu_comm_columns_to_rows) -> distributed projection (mgpu_comm_project_reduce) must
equal the single-device mgpu_project_reduce of the whole basis.  Prints one JSON line on rank 0.
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/comm_check.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_1606_01216_b200 as mg
from paper_1606_01216_b200 import sharding

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ctx = mg.Context(local)
uid = [mg.Context.comm_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
ctx.comm_init(uid[0], world, rank)
ne, R = 20000, 24
M, D, K = mg.model_hermite(ne)
n = 2 * ne
rng = np.random.default_rng(7)
V, _ = np.linalg.qr(rng.standard_normal((n, R)))
F = rng.standard_normal((n, 2))
Cp = rng.standard_normal((3, n))
Cv = rng.standard_normal((3, n))
mine = sharding.shard(list(range(R)), rank, world)
X_local = torch.tensor(np.ascontiguousarray(V[:, mine].T), device=f"cuda:{local}")
out = sharding.project_reduce_nccl(ctx, M, D, K, X_local, mine, R, F, Cp, Cv)
want = mg.project_reduce(M, D, K, V, F, Cp, Cv, ctx=ctx)
err = max(float(np.max(np.abs(out[k] - want[k])) / max(np.max(np.abs(want[k])), 1e-300))
          for k in ("Mh", "Dh", "Kh", "Fh", "Cph", "Cvh"))
if rank == 0:
    print(json.dumps({"world": world, "n": n, "R": R, "max_rel": err}), flush=True)
ctx.comm_destroy()
dist.destroy_process_group()
