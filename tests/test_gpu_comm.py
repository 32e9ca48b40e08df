"""NCCL data plane in the C-ABI (mgpu_comm_*): single-rank communicator on this
GPU (the redistribution and the all-reduce degenerate to copies, so the device path is checked
against the single-device projection), and the 2-GPU launcher test for boxes with >= 2 GPUs."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm_ctx(mg):
    ctx = mg.Context(0)
    ctx.comm_init(mg.Context.comm_unique_id(), 1, 0)
    yield ctx
    ctx.comm_destroy()
    ctx.close()


def test_single_rank_columns_to_rows_and_projection(mg, comm_ctx):
    import torch
    from paper_1606_01216_b200 import sharding
    ctx = comm_ctx
    M, D, K = mg.model_hermite(3000)
    n, R = 6000, 10
    rng = np.random.default_rng(3)
    V, _ = np.linalg.qr(rng.standard_normal((n, R)))
    F = rng.standard_normal((n, 2))
    Cp = rng.standard_normal((2, n))
    Cv = rng.standard_normal((2, n))
    ids = [7, 2, 9, 0, 4, 1, 3, 5, 8, 6]  # columns held in a shuffled order
    X_local = torch.tensor(np.ascontiguousarray(V[:, ids].T), device="cuda:0")
    assert mg.csr_bandwidth(K, ctx) == 3
    Vext, ext0 = mg.comm_columns_to_rows(X_local, ids, R, 3, ctx)
    assert ext0 == 0 and tuple(Vext.shape) == (R, n)
    np.testing.assert_array_equal(Vext.cpu().numpy().T, V)
    out = sharding.project_reduce_nccl(ctx, M, D, K, X_local, ids, R, F, Cp, Cv)
    want = mg.project_reduce(M, D, K, V, F, Cp, Cv, ctx=ctx)
    for k in ("Mh", "Dh", "Kh", "Fh", "Cph", "Cvh"):
        np.testing.assert_array_equal(out[k], want[k])  # same slab kernel over the same rows


def test_single_rank_allreduce_and_rows(mg, comm_ctx):
    import torch
    t = torch.arange(10, dtype=torch.float64, device="cuda:0")
    mg.comm_allreduce_sum(t, comm_ctx)
    np.testing.assert_array_equal(t.cpu().numpy(), np.arange(10.0))
    assert comm_ctx.comm_rows(100, 3) == (0, 100, 0, 100)


def test_projection_rejects_a_short_halo(mg, comm_ctx):
    import torch
    M, D, K = mg.model_hermite(100)
    X = torch.zeros((2, 200), dtype=torch.float64, device="cuda:0")
    Vext, _ = mg.comm_columns_to_rows(X, [0, 1], 2, 1, comm_ctx)
    with pytest.raises(mg.ArgumentError, match="bandwidth"):
        mg.comm_project_reduce(M, D, K, 1, Vext, ctx=comm_ctx)


def test_two_gpu_launcher():
    """torchrun, 2 processes, 2 GPUs: shift-sharded columns -> NCCL row slabs -> distributed
    projection == the single-device projection (runs on boxes with >= 2 GPUs)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one process per GPU)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "tools", "comm_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert res["world"] == 2 and res["max_rel"] < 1e-12
