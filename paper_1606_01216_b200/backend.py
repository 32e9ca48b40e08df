"""CudaCgBackend: the reference's SolveBackend plugin (airga.hpp:133-147) on the GPU.

Mirrors CgBackend (airga.cpp:103-190) method for method:
  prepare(sys, points, outer, records)   -- assemble the l shifted operators
                                            (one batched device call) and build
                                            or update the SPAI chain per point
  solve(point_index, rhs)                -- block_solve for one point
  provides_residuals()                   -- True
plus solve_all(rhs), which batches every point into one persistent CG kernel
(north star subsystem 4; the reference loops over points, airga.cpp:374-405).

Config fields are AirgaConfig's (airga.hpp:40-69) plus the GPU-only choices
spai_algorithm ("mr" = the reference's Alg. 2/4, "ls" = static-pattern
least squares) and ls_pattern (A or A^2).  spai_mode is the reference's
(sequential by default in AirgaConfig; the device sequential mode keeps the
built columns as sparse row lists, frozen mode is column-parallel).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence


from . import mgpu


@dataclass
class CudaCgConfig:
    solver: str = "cg_spai"  # cg_plain | cg_spai | cg_spai_update   (airga.hpp:42-48)
    spai_tol: float = 0.01
    spai_max_col_iters: int = 50
    spai_mode: int = mgpu.SEQUENTIAL  # AirgaConfig default (airga.hpp)
    cg_rtol: float = 1e-10
    cg_maxit_factor: int = 10
    update_start_iteration: int = 3
    spai_algorithm: str = "mr"  # "mr" | "ls"
    ls_pattern: int = mgpu.PATTERN_A
    maxit_override: Optional[int] = None  # fixed CG budget (benchmarks); None = factor * n
    # north-star subsystem 2: in update mode, collapse the chain after each update into one factor,
    # P <- Q P (device SpGEMM, the product chain_apply applies factor by factor, spai.cpp:361-373)
    collapse: bool = False


@dataclass
class PrecondRecord:  # airga.hpp:87-95
    outer: int
    point_index: int
    point: float
    seconds: float
    kind: str
    chain_length: int


class CudaCgBackend:
    def __init__(self, cfg: CudaCgConfig, ctx: Optional[mgpu.Context] = None):
        if cfg.solver not in ("cg_plain", "cg_spai", "cg_spai_update"):
            raise mgpu.ArgumentError(f"CudaCgBackend: unsupported solver {cfg.solver}")
        self.cfg = cfg
        self.ctx = ctx or mgpu.default_context()
        self.n = 0
        self.prev_ops: List[mgpu.DeviceCsr] = []
        self.chains: List[List[mgpu.SpaiFactor]] = []
        self.zlog: List[int] = []  # logical chain length (factors composed), as the reference counts it
        self._dev_sys = None

    def provides_residuals(self) -> bool:
        return True

    def _system(self, sys):
        M, D, K = sys
        if self._dev_sys is None or self._dev_sys[0] is not sys:
            self._dev_sys = (sys, [mgpu._dev(x, self.ctx) for x in (M, D, K)])
        return self._dev_sys[1]

    def _build(self, A) -> mgpu.SpaiFactor:
        c = self.cfg
        if c.spai_algorithm == "ls":
            return mgpu.spai_ls(A, None, c.ls_pattern, ctx=self.ctx)
        return mgpu.spai_build(A, c.spai_tol, c.spai_max_col_iters, c.spai_mode, ctx=self.ctx)

    def _update(self, K_old, K_new) -> mgpu.SpaiFactor:
        c = self.cfg
        if c.spai_algorithm == "ls":
            return mgpu.spai_ls(K_new, K_old, c.ls_pattern, ctx=self.ctx)
        return mgpu.spai_update(K_old, K_new, c.spai_tol, c.spai_max_col_iters, c.spai_mode, ctx=self.ctx)

    def prepare(self, sys, points: Sequence[float], outer: int, records: Optional[list] = None):
        """airga.cpp:108-164."""
        M, D, K = self._system(sys)
        self.n = M.nrows
        fresh = mgpu.shifted_operators(M, D, K, list(points), ctx=self.ctx)
        c = self.cfg
        if c.solver == "cg_plain":
            self.chains = [[] for _ in points]
        else:
            update_mode = (c.solver == "cg_spai_update" and outer >= c.update_start_iteration
                           and len(self.prev_ops) == len(points) and len(self.chains) == len(points))
            if not update_mode:
                self.chains = [[] for _ in points]
            if c.spai_algorithm == "ls":
                # every point's factor in one batched device call (the operators share one
                # pattern); each record carries an equal share of the batch time
                t0 = time.perf_counter()
                qs = mgpu.spai_ls_batched(fresh, self.prev_ops if update_mode else None, c.ls_pattern, ctx=self.ctx)
                self.ctx.synchronize()
                share = (time.perf_counter() - t0) / max(len(points), 1)
                if not update_mode:
                    self.zlog = [0] * len(points)
                for i, s in enumerate(points):
                    self._push(i, qs[i], update_mode)
                    if records is not None:
                        records.append(PrecondRecord(outer, i, float(s), share, "update" if update_mode else "base",
                                                     self.zlog[i]))
                self.prev_ops = fresh
                return
            if not update_mode:
                self.zlog = [0] * len(points)
            for i, s in enumerate(points):
                t0 = time.perf_counter()
                if update_mode:
                    q = self._update(self.prev_ops[i], fresh[i])
                    kind = "update"
                else:
                    q = self._build(fresh[i])
                    kind = "base"
                self.ctx.synchronize()
                self._push(i, q, update_mode)
                if records is not None:
                    records.append(PrecondRecord(outer, i, float(s), time.perf_counter() - t0, kind,
                                                 self.zlog[i]))
        self.prev_ops = fresh

    def _push(self, i: int, q, update_mode: bool):
        """push_newest (spai.cpp:352-359), or with collapse the product Q P of the new factor and the
        collapsed chain (one factor; the reference's chain_apply applies Q_z ... Q_2 P in that order)."""
        if self.cfg.collapse and update_mode and self.chains[i]:
            self.chains[i] = [mgpu.spgemm(q.matrix, mgpu._factor_mat(self.chains[i][0]), ctx=self.ctx)]
        else:
            self.chains[i].insert(0, q)
        self.zlog[i] += 1

    def _maxit(self) -> int:
        c = self.cfg
        return c.maxit_override if c.maxit_override is not None else c.cg_maxit_factor * self.n

    def solve(self, point_index: int, rhs) -> mgpu.BlockSolveResult:
        """airga.cpp:166-181."""
        A = self.prev_ops[point_index]
        chain = self.chains[point_index] if self.chains else []
        return mgpu.block_solve(A, chain, rhs, self.cfg.cg_rtol, self._maxit(), ctx=self.ctx)

    def solve_all(self, rhs, raise_on_breakdown: bool = True) -> List[mgpu.BlockSolveResult]:
        """Every point in one batched device solve (same rhs block, or one per point)."""
        chains = self.chains if self.chains else [[] for _ in self.prev_ops]
        return mgpu.cg_solve_batched(self.prev_ops, chains, rhs, self.cfg.cg_rtol, self._maxit(),
                                     raise_on_breakdown=raise_on_breakdown, ctx=self.ctx)
