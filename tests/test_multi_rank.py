"""CPU, world_size 2 over gloo: the multi-GPU path's host logic (shift sharding, max-over-ranks
timing, solution gather) is exercised with the oracle standing in for each rank's device solve."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle import Oracle
    from paper_1606_01216_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    M, D, K = orc.chain_generate(300, consistent=True, stiffness_scale=1.0)
    shifts = sharding.log_shifts(6)
    mine = sharding.shard(list(range(len(shifts))), rank, world)
    blocks = []
    b = np.zeros(300)
    b[0] = 1.0
    for i in mine:
        A = orc.shifted_operator(M, D, K, shifts[i])
        P, _ = orc.spai_build(A, mode=1)
        blocks.append(orc.pcg_solve(A, [P], b)["solution"])
    full = sharding.gather_blocks(blocks, mine, len(shifts), dist)
    t = sharding.max_over_ranks([1.0 + rank, 5.0 - rank], dist)
    if rank == 0:
        q.put((mine, full, t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shift_sharding():
    from oracle import Oracle
    from paper_1606_01216_b200 import sharding
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    mine, full, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert mine == [0, 2, 4]
    assert t == [2.0, 5.0]
    orc = Oracle()
    M, D, K = orc.chain_generate(300, consistent=True, stiffness_scale=1.0)
    b = np.zeros(300)
    b[0] = 1.0
    for i, s in enumerate(sharding.log_shifts(6)):
        A = orc.shifted_operator(M, D, K, s)
        P, _ = orc.spai_build(A, mode=1)
        np.testing.assert_array_equal(full[i], orc.pcg_solve(A, [P], b)["solution"])


def test_shard_properties():
    from paper_1606_01216_b200 import sharding
    items = list(range(64))
    for world in (1, 2, 4, 8):
        parts = [sharding.shard(items, r, world) for r in range(world)]
        assert sorted(sum(parts, [])) == items
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
    s = sharding.log_shifts(8)
    assert s[0] == 10.0 and abs(s[-1] - 1e4) < 1e-9
    np.testing.assert_allclose(s, [10.0 ** (1 + 3 * i / 7) for i in range(8)], rtol=1e-15)
    with pytest.raises(ValueError):
        sharding.shard(items, 3, 2)


# ---------------------------------------------------------------- distributed projection (8e)
def _numpy_slab(Ms, Ds, Ks, row0, ext0, Vext, F, Cp, Cv):
    """CPU stand-in for mgpu.project_reduce_slab: the slab's partial V^T S V etc."""
    Vext = np.asarray(Vext)
    p = Ms.nrows
    Y = Vext[row0 - ext0:row0 - ext0 + p]
    out = {}
    for key, S in (("Mh", Ms), ("Dh", Ds), ("Kh", Ks)):
        dense = S.todense()[:, ext0:ext0 + Vext.shape[0]]
        assert np.all(S.todense()[:, :ext0] == 0) and np.all(S.todense()[:, ext0 + Vext.shape[0]:] == 0)
        out[key] = Y.T @ (dense @ Vext)
    out["Fh"] = Y.T @ F if F is not None else np.zeros((Vext.shape[1], 0))
    out["Cph"] = Cp @ Y if Cp is not None else np.zeros((0, Vext.shape[1]))
    out["Cvh"] = Cv @ Y if Cv is not None else np.zeros((0, Vext.shape[1]))
    return out


def _projection_case(n=600, r=6):
    from oracle import Oracle
    orc = Oracle()
    M, D, K = orc.chain_generate(n, consistent=True, stiffness_scale=1.0)
    rng = np.random.default_rng(11)
    V, _ = np.linalg.qr(rng.standard_normal((n, r)))
    F = rng.standard_normal((n, 2))
    Cp = rng.standard_normal((3, n))
    Cv = rng.standard_normal((3, n))
    return M, D, K, np.asfortranarray(V), F, Cp, Cv


def _proj_worker(rank, world, port, q, device_slab=False):
    import torch.distributed as dist

    from paper_1606_01216_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    M, D, K, V, F, Cp, Cv = _projection_case()
    n, r = V.shape
    mine = list(range(rank, r, world))  # shift-sharded solve columns
    V_slab = sharding.columns_to_rows(V[:, mine], mine, r, n, dist)
    r0, r1 = sharding.row_range(n, rank, world)
    assert np.array_equal(V_slab, V[r0:r1])
    # device_slab: each rank's partials from the sm_100a slab kernel (mgpu_project_reduce_slab on cuda:0,
    # both ranks share the one GPU; the gloo all-reduce sums host partials, no kernel waits on another rank)
    out = sharding.project_reduce_distributed(M, D, K, V_slab, r0, F, Cp, Cv, dist=dist,
                                              local=None if device_slab else _numpy_slab)
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("device_slab", [False, pytest.param(True, marks=pytest.mark.gpu)])
def test_two_rank_distributed_projection(device_slab):
    """Columns -> row slabs (all-to-all), halo rows, slab partials, all-reduce == global V^T S V."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_proj_worker, args=(r, 2, port, q, device_slab)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    M, D, K, V, F, Cp, Cv = _projection_case()
    for key, S in (("Mh", M), ("Dh", D), ("Kh", K)):
        want = V.T @ (S.todense() @ V)
        assert np.linalg.norm(out[key] - want) <= 1e-12 * np.linalg.norm(want)
    assert np.linalg.norm(out["Fh"] - V.T @ F) <= 1e-12 * np.linalg.norm(V.T @ F)
    assert np.linalg.norm(out["Cph"] - Cp @ V) <= 1e-12 * np.linalg.norm(Cp @ V)


def test_row_slab_and_halo_single_rank():
    from paper_1606_01216_b200 import sharding
    M, D, K, V, F, Cp, Cv = _projection_case(200, 3)
    assert sharding.bandwidth(K) == 1
    S = sharding.row_slab(K, 50, 120)
    np.testing.assert_array_equal(S.todense(), K.todense()[50:120])
    assert sharding.row_range(10, 1, 3) == (3, 6)
    ext, e0 = sharding.halo_rows(V, 0, 200, 1)
    assert e0 == 0 and np.array_equal(ext, V)
