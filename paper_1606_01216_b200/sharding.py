"""Shift sharding across ranks: the l shifted systems are independent,
so rank r of N takes shifts r, r+N, ... and solves them with no collective on the
data path.  Only timing (max over ranks) and, optionally, the solution blocks
(all-gather, for a global Arnoldi block downstream) cross ranks."""
from __future__ import annotations

from typing import List, Sequence


def log_shifts(count: int, lo: float = 10.0, hi: float = 1e4) -> List[float]:
    """count real shifts log-spaced in [lo, hi] (BASELINE configs: 10^(1 + 3 i / (count - 1)))."""
    if count == 1:
        return [lo]
    a, b = __import__("math").log10(lo), __import__("math").log10(hi)
    return [10.0 ** (a + (b - a) * i / (count - 1)) for i in range(count)]


class Mt19937_64:
    """std::mt19937_64 (the C++ standard's 64-bit Mersenne twister; seeding per
    [rand.eng.mers]), so host-drawn shifts match a C++ driver seeded the same way."""

    _N, _M = 312, 156
    _MASK = (1 << 64) - 1

    def __init__(self, seed: int = 5489):
        mt = [0] * self._N
        mt[0] = seed & self._MASK
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & self._MASK
        self.mt, self.i = mt, self._N

    def __call__(self) -> int:
        mt, N, M = self.mt, self._N, self._M
        if self.i >= N:
            upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
            for k in range(N):
                x = (mt[k] & upper) | (mt[(k + 1) % N] & lower)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[k] = mt[(k + M) % N] ^ xa
            self.i = 0
        y = mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self._MASK


def airga_shift_draws(outer: int, count: int, seed: int = 42, lo_exp: float = 1.0, span: float = 3.0) -> List[List[float]]:
    """BASELINE configs[2]: per outer iteration, `count` shifts
    s = 10^(lo_exp + span u), u = (mt19937_64(seed)() >> 11) * 2^-53, one generator across
    the whole sequence, each draw sorted ascending (update partners pair by index,
    airga.cpp:145)."""
    g = Mt19937_64(seed)
    out = []
    for _ in range(outer):
        draw = [10.0 ** (lo_exp + span * ((g() >> 11) * 2.0 ** -53)) for _ in range(count)]
        out.append(sorted(draw))
    return out


def shard(items: Sequence, rank: int, world: int) -> list:
    """Round-robin shard of items for rank (disjoint, covering, balanced to +-1)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return list(items[rank::world])


def owner(index: int, world: int) -> int:
    return index % world


def max_over_ranks(values: Sequence[float], dist=None, device=None) -> List[float]:
    """Element-wise max over ranks (device-timed ms per rank -> job time)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in values]
    import torch
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def gather_blocks(local_blocks: Sequence, local_index: Sequence[int], total: int, dist=None):
    """All-gather per-shift solution blocks so every rank holds the full list (index order)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        out = [None] * total
        for i, b in zip(local_index, local_blocks):
            out[i] = b
        return out
    gathered = [None] * dist.get_world_size()
    dist.all_gather_object(gathered, list(zip(local_index, local_blocks)))
    out = [None] * total
    for part in gathered:
        for i, b in part:
            out[i] = b
    return out


# ---------------------------------------------------------------- distributed projection
# After the shift-sharded solves the Arnoldi basis is redistributed by ROWS: rank r keeps
# rows [r0, r1) of every basis column, computes its slab's partial V_slab^T (S V) with a
# halo of bandwidth rows from its neighbours, and one all-reduce sums the r x r partials
# (airga.cpp:485-500 split over row slabs).
def row_range(n: int, rank: int, world: int):
    """Balanced contiguous row slab [r0, r1) of rank."""
    return n * rank // world, n * (rank + 1) // world


def row_slab(A, r0: int, r1: int):
    """Rows [r0, r1) of a host CSR, global column indices kept (same type as A)."""
    import numpy as np
    b, e = int(A.row_ptr[r0]), int(A.row_ptr[r1])
    rp = (np.asarray(A.row_ptr[r0:r1 + 1], np.int64) - b).astype(np.int64)
    return type(A)(r1 - r0, A.ncols, rp, np.asarray(A.col_idx[b:e], np.int32).copy(),
                   np.asarray(A.values[b:e], np.float64).copy())


def bandwidth(A) -> int:
    """max |i - j| over stored entries of a host CSR."""
    import numpy as np
    if A.nnz == 0:
        return 0
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    return int(np.max(np.abs(rows - A.col_idx.astype(np.int64))))


def columns_to_rows(X_local, col_ids: Sequence[int], total_cols: int, n: int, dist=None):
    """All-to-all: every rank holds full-length columns col_ids of the basis (n x c_local);
    returns this rank's row slab of all total_cols columns, in global column order."""
    import numpy as np
    X_local = np.asarray(X_local, np.float64).reshape(n, -1)
    world = 1 if dist is None or not dist.is_initialized() else dist.get_world_size()
    rank = 0 if world == 1 else dist.get_rank()
    r0, r1 = row_range(n, rank, world)
    out = np.zeros((r1 - r0, total_cols), order="F")
    if world == 1:
        out[:, list(col_ids)] = X_local[r0:r1]
        return out
    if dist.get_backend() == "nccl":
        raise ValueError("columns_to_rows is the host (gloo) restatement; on NCCL use project_reduce_nccl, "
                         "which redistributes device buffers with mgpu_comm_columns_to_rows")
    # each destination d receives rows [r0_d, r1_d) of this rank's columns
    sends = [(list(col_ids), X_local[slice(*row_range(n, d, world))]) for d in range(world)]
    gathered = [None] * world
    dist.all_gather_object(gathered, sends)
    recv = [gathered[s][rank] for s in range(world)]
    for ids, block in recv:
        if len(ids):
            out[:, ids] = block
    return out


def halo_rows(V_slab, r0: int, n: int, h: int, dist=None):
    """Extend this rank's basis rows [r0, r1) by h rows on each side (clipped to [0, n)) with the
    neighbours' boundary rows; returns (Vext, ext0)."""
    import numpy as np
    V_slab = np.asarray(V_slab, np.float64)
    r1 = r0 + V_slab.shape[0]
    world = 1 if dist is None or not dist.is_initialized() else dist.get_world_size()
    lo, hi = max(0, r0 - h), min(n, r1 + h)
    if world == 1 or h == 0:
        if (lo, hi) != (r0, r1):
            raise ValueError("halo rows requested without neighbours")
        return np.asfortranarray(V_slab), r0
    k = min(h, V_slab.shape[0])
    mine = (r0, r1, V_slab[:k], V_slab[V_slab.shape[0] - k:])
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    ext = np.zeros((hi - lo, V_slab.shape[1]), order="F")
    ext[r0 - lo:r1 - lo] = V_slab
    for (a0, a1, first, last) in parts:
        for base, rows in ((a0, first), (a1 - len(last), last)):
            for t in range(len(rows)):
                g = base + t
                if lo <= g < hi and not (r0 <= g < r1):
                    ext[g - lo] = rows[t]
    return ext, lo


def project_reduce_distributed(M, D, K, V_slab, r0: int, F=None, Cp=None, Cv=None, dist=None, local=None,
                               device=None) -> dict:
    """airga.cpp:485-500 over a row-distributed basis: local slab partials (device:
    mgpu.project_reduce_slab) + one all-reduce.  `local` may stand in for the device product
    (CPU tests).  Returns replicated Mh, Dh, Kh, Fh, Cph, Cvh."""
    import numpy as np
    n = M.nrows
    V_slab = np.asarray(V_slab, np.float64)
    r1 = r0 + V_slab.shape[0]
    h = max(bandwidth(M), bandwidth(D), bandwidth(K))
    Vext, ext0 = halo_rows(V_slab, r0, n, h, dist)
    if local is None:
        from . import mgpu
        local = mgpu.project_reduce_slab
    part = local(row_slab(M, r0, r1), row_slab(D, r0, r1), row_slab(K, r0, r1), r0, ext0, Vext,
                 None if F is None else np.asarray(F)[r0:r1], None if Cp is None else np.asarray(Cp)[:, r0:r1],
                 None if Cv is None else np.asarray(Cv)[:, r0:r1])
    keys = ("Mh", "Dh", "Kh", "Fh", "Cph", "Cvh")
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return part
    import torch
    flat = np.concatenate([np.asarray(part[k]).ravel(order="F") for k in keys])
    t = torch.as_tensor(flat, device=device)
    dist.all_reduce(t)
    flat = t.cpu().numpy()
    out, o = {}, 0
    for k in keys:
        shape = np.asarray(part[k]).shape
        cnt = int(np.prod(shape))
        out[k] = flat[o:o + cnt].reshape(shape, order="F")
        o += cnt
    return out


def project_reduce_nccl(ctx, M, D, K, X_local, col_ids, R: int, F=None, Cp=None, Cv=None) -> dict:
    """airga.cpp:485-500 after the shift-sharded solves, entirely on the devices over NCCL: this rank's
    solution columns X_local (CUDA float64 tensor (c_local, n), global ids col_ids) become its row slab
    of the n x R block plus the operators' bandwidth halo (mgpu_comm_columns_to_rows: grouped
    ncclSend / ncclRecv), the slab partials run on the device and one ncclAllReduce sums them
    (mgpu_comm_project_reduce).  The context must hold a communicator (Context.comm_init).  M, D, K:
    the replicated operators (host CSR or DeviceCsr).  Returns the replicated reduced matrices."""
    from . import mgpu
    h = max(mgpu.csr_bandwidth(x, ctx) for x in (M, D, K))
    Vext, _ = mgpu.comm_columns_to_rows(X_local, col_ids, R, h, ctx)
    return mgpu.comm_project_reduce(M, D, K, h, Vext, F, Cp, Cv, ctx)

