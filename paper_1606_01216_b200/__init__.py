"""B200-native SPAI + shifted-system PCG (the AIRGA solve path of arXiv 1606.01216).

The compute path is libmgpu.so (hand-written sm_100a CUDA behind the C-ABI in
include/mgpu.h).  This package is the thin host mirror of the reference's
solver / preconditioner interface used by tests and the benchmark; the C++
drop-in for the reference itself is paper_1606_01216_b200/host/ (see
INTEGRATION.md).
"""
from .mgpu import (  # noqa: F401
    ArgumentError, BreakdownError, BlockSolveResult, Context, CudaError, DeviceCsr, MgpuError, NumericalError,
    SparseMatrix, SpaiFactor, StagnationError, UnsupportedError, block_solve, cg_solve_batched, cg_solve_device, cg_solve_raw, chain_apply, chain_quality, thin_qr, project_reduce, project_reduce_slab, arnoldi_deflate,
    default_context, lib, model_chain, model_hermite, model_hermite_device, pcg_solve, shifted_operator, shifted_operators, sp_add_scaled,
    spai_build, spai_ls, spai_ls_batched, spai_update, spgemm, trace, trace_inner, transpose,
    shifted_solve_raw, shifted_solve_device, csr_bandwidth, comm_allreduce_sum, comm_columns_to_rows, comm_project_reduce,
    FROZEN, SEQUENTIAL, PATTERN_A, PATTERN_A2, LS_COLSCALE,
)
from .backend import CudaCgBackend  # noqa: F401
