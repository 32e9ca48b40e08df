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
