"""ctypes binding of libmgpu.so (include/mgpu.h) -- the C-ABI drop-in boundary.

Mirrors the reference's solver / preconditioner interface (proj/include/mor):
names, argument meaning and error behaviour follow spai.hpp, krylov.hpp,
sparse.hpp, system.hpp and airga.hpp.  There is no CPU fallback: if the CUDA
library is missing or no sm_100 device is present, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmgpu.so")
# diagnostics: A/B timing of an alternative build of the same library (never a fallback)
LIB_PATH = os.environ.get("MGPU_LIB", LIB_PATH)

MGPU_OK, MGPU_ERR_ARG, MGPU_ERR_STAGNATION, MGPU_ERR_BREAKDOWN = 0, 1, 2, 3
MGPU_ERR_NUMERICAL, MGPU_ERR_UNSUPPORTED, MGPU_ERR_CUDA, MGPU_ERR_NCCL = 4, 5, 6, 7
MGPU_HOST, MGPU_DEVICE = 0, 1
SEQUENTIAL, FROZEN = 0, 1
PATTERN_A, PATTERN_A2 = 0, 1
LS_COLSCALE = 0x10  # flag: column-equilibrated LS-SPAI (mgpu.h MGPU_LS_COLSCALE)

# Symbols include/mgpu.h declares; tests check the library exports all of them.
EXPORTED = [
    "mgpu_ctx_create", "mgpu_ctx_destroy", "mgpu_ctx_synchronize", "mgpu_last_error", "mgpu_status_string",
    "mgpu_launch_count", "mgpu_last_cg_timing", "mgpu_ctx_set_cg_path", "mgpu_last_cg_path", "mgpu_csr_upload", "mgpu_csr_upload_device", "mgpu_csr_info",
    "mgpu_csr_download", "mgpu_csr_device_view", "mgpu_csr_free", "mgpu_sp_add_scaled", "mgpu_shifted_operators",
    "mgpu_transpose", "mgpu_trace", "mgpu_trace_inner", "mgpu_spmv", "mgpu_chain_apply", "mgpu_chain_quality", "mgpu_spai_build",
    "mgpu_spai_update", "mgpu_spai_ls", "mgpu_spai_ls_batched", "mgpu_spgemm", "mgpu_cg_solve",
    "mgpu_model_chain", "mgpu_model_hermite", "mgpu_host_free", "mgpu_thin_qr", "mgpu_project_reduce", "mgpu_project_reduce_slab",
    "mgpu_arnoldi_deflate", "mgpu_model_hermite_device", "mgpu_csr_write", "mgpu_csr_read", "mgpu_shifted_solve",
    "mgpu_csr_upload_batch", "mgpu_ctx_set_option", "mgpu_ctx_get_option", "mgpu_phase_profile",
    "mgpu_buffer_alloc", "mgpu_buffer_free", "mgpu_memcpy_d2h", "mgpu_memcpy_h2d",
    "mgpu_comm_unique_id", "mgpu_comm_init", "mgpu_comm_destroy", "mgpu_comm_allreduce_sum", "mgpu_comm_rows",
    "mgpu_comm_columns_to_rows", "mgpu_comm_project_reduce", "mgpu_csr_bandwidth", "mgpu_host_pin", "mgpu_host_unpin",
]

# mgpu.h mgpu_option
OPTIONS = {"stream_chunk": 2, "stream_ring": 3, "stream_same_chb": 4,
           "cluster_cs": 5, "cluster_async": 6, "profile_phases": 7, "qr_unblocked": 8, "ls_group": 9,
           "stream_tiles": 10, "seq_sparse": 12}


# ---------------------------------------------------------------- errors
class MgpuError(RuntimeError):
    status = -1

    def __init__(self, msg: str, index: int = -1, rhs_column: int = -1, point: int = -1):
        super().__init__(msg)
        self.index, self.rhs_column, self.point = index, rhs_column, point


class ArgumentError(MgpuError, ValueError):  # errors.hpp:13-18
    status = MGPU_ERR_ARG


class StagnationError(MgpuError):  # errors.hpp:46-52
    status = MGPU_ERR_STAGNATION

    @property
    def column(self):
        return self.index


class BreakdownError(MgpuError):  # errors.hpp:38-44
    status = MGPU_ERR_BREAKDOWN

    @property
    def iteration(self):
        return self.index


class NumericalError(MgpuError):  # errors.hpp:54-59
    status = MGPU_ERR_NUMERICAL


class UnsupportedError(MgpuError):
    status = MGPU_ERR_UNSUPPORTED


class CudaError(MgpuError):
    status = MGPU_ERR_CUDA


_BY_STATUS = {c.status: c for c in (ArgumentError, StagnationError, BreakdownError, NumericalError,
                                     UnsupportedError, CudaError)}


# ---------------------------------------------------------------- library
class _HostCsr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int32)),
                ("values", C.POINTER(C.c_double))]


class _CgOut(C.Structure):
    _fields_ = [("X", C.c_void_p), ("recurrence", C.c_void_p), ("true_res", C.c_void_p),
                ("iterations", C.POINTER(C.c_int64)), ("converged", C.POINTER(C.c_int)),
                ("status", C.POINTER(C.c_int)), ("breakdown_iteration", C.POINTER(C.c_int64)),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int64)]


_lib = None


def lib():
    """Loads libmgpu.so; raises (never falls back) when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i64, dbl = C.c_void_p, C.c_int64, C.c_double
        L.mgpu_ctx_create.argtypes = [C.c_int, vp, C.POINTER(vp)]
        L.mgpu_ctx_destroy.argtypes = [vp]
        L.mgpu_ctx_synchronize.argtypes = [vp]
        L.mgpu_last_error.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.c_char_p, C.c_size_t]
        L.mgpu_status_string.restype = C.c_char_p
        L.mgpu_launch_count.argtypes = [vp]
        L.mgpu_launch_count.restype = i64
        L.mgpu_last_cg_timing.argtypes = [vp, C.POINTER(dbl), C.POINTER(i64)]
        L.mgpu_ctx_set_cg_path.argtypes = [vp, C.c_int]
        L.mgpu_ctx_set_option.argtypes = [vp, C.c_int, i64]
        L.mgpu_ctx_get_option.argtypes = [vp, C.c_int, C.POINTER(i64)]
        L.mgpu_phase_profile.argtypes = [vp, C.POINTER(C.c_longlong)]
        L.mgpu_last_cg_path.argtypes = [vp]
        L.mgpu_csr_upload.argtypes = [vp, i64, i64, i64, vp, vp, vp, C.POINTER(vp)]
        L.mgpu_csr_upload_device.argtypes = [vp, i64, i64, i64, vp, vp, vp, C.POINTER(vp)]
        L.mgpu_csr_upload_batch.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp, vp, vp]
        L.mgpu_csr_info.argtypes = [vp, vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
        L.mgpu_csr_download.argtypes = [vp, vp, vp, vp, vp]
        L.mgpu_csr_free.argtypes = [vp]
        L.mgpu_csr_device_view.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), vp, vp, vp]
        L.mgpu_sp_add_scaled.argtypes = [vp, vp, vp, dbl, dbl, C.POINTER(vp)]
        L.mgpu_shifted_operators.argtypes = [vp, vp, vp, vp, C.c_int, vp, vp]
        L.mgpu_transpose.argtypes = [vp, vp, C.POINTER(vp)]
        L.mgpu_trace.argtypes = [vp, vp, C.POINTER(dbl)]
        L.mgpu_trace_inner.argtypes = [vp, vp, vp, C.POINTER(dbl)]
        L.mgpu_spmv.argtypes = [vp, vp, vp, vp]
        L.mgpu_chain_apply.argtypes = [vp, C.c_int, vp, vp, vp, C.c_int]
        L.mgpu_chain_quality.argtypes = [vp, C.c_int, vp, vp, C.c_int64, C.c_uint64, C.POINTER(C.c_double)]
        L.mgpu_thin_qr.argtypes = [vp, i64, i64, vp, dbl, vp, vp, C.POINTER(C.c_int64), C.c_int]
        L.mgpu_project_reduce.argtypes = [vp, vp, vp, vp, i64, vp, i64, vp, i64, vp, vp] + [vp] * 6 + [C.c_int]
        L.mgpu_project_reduce_slab.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, vp, i64, vp, i64, vp, vp] + \
            [vp] * 6 + [C.c_int]
        L.mgpu_arnoldi_deflate.argtypes = [vp, i64, vp, C.c_int, vp, vp, C.c_int]
        L.mgpu_spai_build.argtypes = [vp, vp, dbl, i64, C.c_int, C.POINTER(vp), vp]
        L.mgpu_spai_update.argtypes = [vp, vp, vp, dbl, i64, C.c_int, C.POINTER(vp), vp]
        L.mgpu_spai_ls.argtypes = [vp, vp, vp, C.c_int, C.POINTER(vp)]
        L.mgpu_spai_ls_batched.argtypes = [vp, C.c_int, vp, vp, C.c_int, vp]
        L.mgpu_spgemm.argtypes = [vp, vp, vp, C.POINTER(vp)]
        L.mgpu_cg_solve.argtypes = [vp, C.c_int, vp, C.c_int, vp, i64, i64, vp, i64, dbl, i64, C.c_int,
                                    C.POINTER(_CgOut)]
        L.mgpu_shifted_solve.argtypes = [vp, vp, vp, vp, C.c_int, vp, C.c_int, vp, i64, i64, dbl, i64, C.c_int,
                                         C.POINTER(_CgOut), vp]
        L.mgpu_model_chain.argtypes = [i64, dbl, dbl, dbl, dbl, C.c_int] + [C.POINTER(_HostCsr)] * 3
        L.mgpu_model_hermite.argtypes = [i64] + [dbl] * 7 + [C.POINTER(_HostCsr)] * 3
        L.mgpu_csr_write.argtypes = [vp, vp, C.c_char_p]
        L.mgpu_csr_read.argtypes = [vp, C.c_char_p, C.POINTER(C.c_void_p)]
        L.mgpu_model_hermite_device.argtypes = [vp, i64] + [dbl] * 7 + [C.POINTER(C.c_void_p)] * 3
        L.mgpu_host_free.argtypes = [C.POINTER(_HostCsr)]
        L.mgpu_comm_unique_id.argtypes = [vp]
        L.mgpu_comm_init.argtypes = [vp, vp, C.c_int, C.c_int]
        L.mgpu_comm_destroy.argtypes = [vp]
        L.mgpu_comm_allreduce_sum.argtypes = [vp, vp, i64]
        L.mgpu_comm_rows.argtypes = [vp, i64, i64] + [C.POINTER(i64)] * 4
        L.mgpu_comm_columns_to_rows.argtypes = [vp, i64, i64, i64, vp, vp, i64, vp]
        L.mgpu_comm_project_reduce.argtypes = [vp, vp, vp, vp, i64, i64, vp, i64, vp, i64, vp, vp] + [vp] * 6 + \
            [C.c_int]
        L.mgpu_csr_bandwidth.argtypes = [vp, vp, C.POINTER(i64)]
        L.mgpu_buffer_alloc.argtypes = [vp, C.c_size_t, C.POINTER(vp)]
        L.mgpu_buffer_free.argtypes = [vp, vp]
        L.mgpu_memcpy_d2h.argtypes = [vp, vp, vp, C.c_size_t]
        L.mgpu_memcpy_h2d.argtypes = [vp, vp, vp, C.c_size_t]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- host CSR
@dataclass
class SparseMatrix:
    """Host CSR with the reference's invariants (sparse.hpp:12-46)."""

    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def todense(self) -> np.ndarray:
        out = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            out[i, self.col_idx[s:e]] = self.values[s:e]
        return out


def _from_host_struct(h: _HostCsr) -> SparseMatrix:
    n, nnz = h.nrows, h.nnz
    rp = np.ctypeslib.as_array(h.row_ptr, (n + 1,)).copy()
    ci = np.ctypeslib.as_array(h.col_idx, (max(nnz, 1),))[:nnz].copy()
    v = np.ctypeslib.as_array(h.values, (max(nnz, 1),))[:nnz].copy()
    lib().mgpu_host_free(C.byref(h))
    return SparseMatrix(n, h.ncols, rp, ci, v)


def model_hermite(ne: int, E=2.1e11, I=1e-8, rho=7800.0, area=1e-4, L=1.0, alpha=0.1, beta=1e-5):
    """BASELINE.json Hermite cantilever: returns (M, D, K) host CSR, n = 2 ne."""
    M, D, K = _HostCsr(), _HostCsr(), _HostCsr()
    st = lib().mgpu_model_hermite(ne, E, I, rho, area, L, alpha, beta, C.byref(M), C.byref(D), C.byref(K))
    if st != MGPU_OK:
        raise ArgumentError("hermite model: bad arguments")
    return _from_host_struct(M), _from_host_struct(D), _from_host_struct(K)


def model_hermite_device(ne: int, E=2.1e11, I=1e-8, rho=7800.0, area=1e-4, L=1.0, alpha=0.1, beta=1e-5, ctx=None):
    """The Hermite cantilever assembled on the device (same matrices as model_hermite, bit for bit):
    returns (M, D, K) as DeviceCsr."""
    ctx = ctx or default_context()
    hs = [C.c_void_p(), C.c_void_p(), C.c_void_p()]
    ctx.check(lib().mgpu_model_hermite_device(ctx.handle, ne, E, I, rho, area, L, alpha, beta,
                                              C.byref(hs[0]), C.byref(hs[1]), C.byref(hs[2])))
    return tuple(DeviceCsr(ctx, h, 2 * ne) for h in hs)


def model_chain(n: int, alpha=0.05, beta=0.05, stiffness_scale=0.01, mass_scale=1.0, consistent=False):
    """Reference chain model (model_io.cpp:18-87): returns (M, D, K)."""
    M, D, K = _HostCsr(), _HostCsr(), _HostCsr()
    st = lib().mgpu_model_chain(n, alpha, beta, stiffness_scale, mass_scale, 1 if consistent else 0, C.byref(M),
                                C.byref(D), C.byref(K))
    if st != MGPU_OK:
        raise ArgumentError("beam_generate: bad arguments")
    return _from_host_struct(M), _from_host_struct(D), _from_host_struct(K)


# ---------------------------------------------------------------- context
class Context:
    """One device + stream (mgpu_ctx)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        """stream: a cudaStream_t handle (e.g. torch.cuda.Stream().cuda_stream) or None (library-owned)."""
        self.handle = C.c_void_p()
        st = lib().mgpu_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(self.handle))
        if st != MGPU_OK:
            raise CudaError(f"mgpu_ctx_create(device={device}) failed: {lib().mgpu_status_string(st).decode()}")
        self.device = device

    def close(self):
        if self.handle:
            lib().mgpu_ctx_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st: int):
        if st == MGPU_OK:
            return
        idx, col, pt = C.c_int64(), C.c_int64(), C.c_int64()
        buf = C.create_string_buffer(1024)
        lib().mgpu_last_error(self.handle, C.byref(idx), C.byref(col), C.byref(pt), buf, 1024)
        cls = _BY_STATUS.get(st, MgpuError)
        raise cls(buf.value.decode(errors="replace"), idx.value, col.value, pt.value)

    def synchronize(self):
        self.check(lib().mgpu_ctx_synchronize(self.handle))

    @property
    def launches(self) -> int:
        return int(lib().mgpu_launch_count(self.handle))

    def set_cg_path(self, path: str):
        """'auto' (cluster / banded / general by shape), 'general' or 'banded' (grid kernel, no cluster)."""
        self.check(lib().mgpu_ctx_set_cg_path(self.handle,
                                              {"auto": 0, "general": 1, "banded": 2, "cluster_v1": 3,
                                               "stream": 4}[path]))

    # ---- NCCL data plane (mgpu_comm_*; one rank per context)
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        st = lib().mgpu_comm_unique_id(buf)
        if st != MGPU_OK:
            raise MgpuError("ncclGetUniqueId failed", -1, -1, -1)
        return buf.raw

    def comm_init(self, uid: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(bytes(uid), 128)
        self.check(lib().mgpu_comm_init(self.handle, buf, nranks, rank))

    def comm_destroy(self):
        self.check(lib().mgpu_comm_destroy(self.handle))

    def comm_rows(self, n: int, h: int):
        v = [C.c_int64() for _ in range(4)]
        self.check(lib().mgpu_comm_rows(self.handle, n, h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)  # row0, p, ext0, next

    def set_option(self, name: str, value: int):
        """mgpu_ctx_set_option (tuning / diagnostic switches; the library reads no environment)."""
        self.check(lib().mgpu_ctx_set_option(self.handle, OPTIONS[name], int(value)))

    def get_option(self, name: str) -> int:
        v = C.c_int64()
        self.check(lib().mgpu_ctx_get_option(self.handle, OPTIONS[name], C.byref(v)))
        return v.value

    def phase_profile(self):
        out = (C.c_longlong * 16)()
        self.check(lib().mgpu_phase_profile(self.handle, out))
        return list(out)

    @property
    def last_cg_path(self) -> str:
        return {0: "banded", 1: "general", 2: "cluster", 3: "cluster_v1", 4: "stream"}.get(
            lib().mgpu_last_cg_path(self.handle), "?")

    def last_cg_timing(self):
        ms, it = C.c_double(), C.c_int64()
        lib().mgpu_last_cg_timing(self.handle, C.byref(ms), C.byref(it))
        return ms.value, it.value


_default: dict = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


class DeviceCsr:
    """Device-resident CSR (mgpu_csr*), freed with the object."""

    def __init__(self, ctx: Context, handle: C.c_void_p, n: int):
        self.ctx, self.handle, self.nrows = ctx, handle, n

    @staticmethod
    def upload(A: SparseMatrix, ctx: Optional[Context] = None) -> "DeviceCsr":
        ctx = ctx or default_context()
        rp = np.ascontiguousarray(A.row_ptr, np.int64)
        ci = np.ascontiguousarray(A.col_idx, np.int32)
        v = np.ascontiguousarray(A.values, np.float64)
        h = C.c_void_p()
        ctx.check(lib().mgpu_csr_upload(ctx.handle, A.nrows, A.ncols, v.shape[0], _ptr(rp), _ptr(ci), _ptr(v),
                                        C.byref(h)))
        return DeviceCsr(ctx, h, A.nrows)

    @staticmethod
    def upload_many(mats: Sequence[SparseMatrix], ctx: Optional[Context] = None) -> list:
        """Several host CSR matrices in one call (mgpu_csr_upload_batch): the same validation as
        upload, one read-back for all of them."""
        ctx = ctx or default_context()
        arrs = [(np.ascontiguousarray(A.row_ptr, np.int64), np.ascontiguousarray(A.col_idx, np.int32),
                 np.ascontiguousarray(A.values, np.float64)) for A in mats]
        k = len(mats)
        nr = np.array([A.nrows for A in mats], np.int64)
        nc = np.array([A.ncols for A in mats], np.int64)
        nz = np.array([a[2].shape[0] for a in arrs], np.int64)
        ptrs = [(C.c_void_p * max(k, 1))(*[a[q].ctypes.data for a in arrs]) for q in range(3)]
        out = (C.c_void_p * max(k, 1))()
        ctx.check(lib().mgpu_csr_upload_batch(ctx.handle, k, _ptr(nr), _ptr(nc), _ptr(nz), ptrs[0], ptrs[1], ptrs[2],
                                              out))
        return [DeviceCsr(ctx, C.c_void_p(out[q]), mats[q].nrows) for q in range(k)]

    @property
    def stored_nnz(self) -> int:
        """Entries stored on the device (fixed-pattern factors may store exact zeros)."""
        n, nnz = C.c_int64(), C.c_int64()
        lib().mgpu_csr_device_view(self.handle, C.byref(n), C.byref(nnz), None, None, None)
        return nnz.value

    def download(self) -> SparseMatrix:
        n, nc, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        self.ctx.check(lib().mgpu_csr_info(self.ctx.handle, self.handle, C.byref(n), C.byref(nc), C.byref(nnz)))
        rp = np.zeros(n.value + 1, np.int64)
        ci = np.zeros(max(nnz.value, 1), np.int32)
        v = np.zeros(max(nnz.value, 1))
        self.ctx.check(lib().mgpu_csr_download(self.ctx.handle, self.handle, _ptr(rp), _ptr(ci), _ptr(v)))
        return SparseMatrix(n.value, nc.value, rp, ci[:nnz.value], v[:nnz.value])

    def save(self, path: str) -> None:
        """Binary CSR sidecar (mgpu_csr_write)."""
        self.ctx.check(lib().mgpu_csr_write(self.ctx.handle, self.handle, os.fsencode(path)))

    @staticmethod
    def load(path: str, ctx: Optional[Context] = None) -> "DeviceCsr":
        """Binary CSR sidecar straight into device memory (mgpu_csr_read)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        ctx.check(lib().mgpu_csr_read(ctx.handle, os.fsencode(path), C.byref(h)))
        n = C.c_int64()
        lib().mgpu_csr_device_view(h, C.byref(n), None, None, None, None)
        return DeviceCsr(ctx, h, n.value)

    def __del__(self):
        try:
            # a matrix outliving an explicitly closed context is left to process teardown
            # (its stream-ordered free would use the destroyed context)
            if self.handle and self.ctx.handle:
                lib().mgpu_csr_free(self.handle)
            self.handle = C.c_void_p()
        except Exception:
            pass


def _dev(A, ctx=None) -> DeviceCsr:
    return A if isinstance(A, DeviceCsr) else DeviceCsr.upload(A, ctx)


def _handles(mats) -> C.Array:
    arr = (C.c_void_p * max(len(mats), 1))()
    for i, m in enumerate(mats):
        arr[i] = m.handle
    return arr


# ---------------------------------------------------------------- core ops
def sp_add_scaled(A, B, a: float, b: float, ctx=None) -> DeviceCsr:
    """sparse.cpp:167-218."""
    ctx = ctx or default_context()
    dA, dB = _dev(A, ctx), _dev(B, ctx)
    h = C.c_void_p()
    ctx.check(lib().mgpu_sp_add_scaled(ctx.handle, dA.handle, dB.handle, a, b, C.byref(h)))
    return DeviceCsr(ctx, h, dA.nrows)


def shifted_operators(M, D, K, shifts: Sequence[float], ctx=None) -> list:
    """system.cpp:64-68 shifted_operator, batched over shifts (device)."""
    ctx = ctx or default_context()
    dM, dD, dK = _dev(M, ctx), _dev(D, ctx), _dev(K, ctx)
    s = np.ascontiguousarray(shifts, np.float64)
    out = (C.c_void_p * max(len(s), 1))()
    ctx.check(lib().mgpu_shifted_operators(ctx.handle, dM.handle, dD.handle, dK.handle, len(s), _ptr(s), out))
    return [DeviceCsr(ctx, C.c_void_p(out[i]), dM.nrows) for i in range(len(s))]


def shifted_operator(M, D, K, s: float, ctx=None) -> DeviceCsr:
    return shifted_operators(M, D, K, [s], ctx)[0]


def transpose(A, ctx=None) -> DeviceCsr:
    ctx = ctx or default_context()
    dA = _dev(A, ctx)
    h = C.c_void_p()
    ctx.check(lib().mgpu_transpose(ctx.handle, dA.handle, C.byref(h)))
    return DeviceCsr(ctx, h, dA.nrows)


def trace(A, ctx=None) -> float:
    ctx = ctx or default_context()
    dA = _dev(A, ctx)
    out = C.c_double()
    ctx.check(lib().mgpu_trace(ctx.handle, dA.handle, C.byref(out)))
    return out.value


def trace_inner(A, B, ctx=None) -> float:
    ctx = ctx or default_context()
    dA, dB = _dev(A, ctx), _dev(B, ctx)
    out = C.c_double()
    ctx.check(lib().mgpu_trace_inner(ctx.handle, dA.handle, dB.handle, C.byref(out)))
    return out.value


def chain_apply(chain: Sequence, v, ctx=None) -> np.ndarray:
    """spai.cpp:361-373; chain newest first; empty chain = identity."""
    ctx = ctx or default_context()
    v = np.ascontiguousarray(v, np.float64)
    if len(chain) == 0:
        return v.copy()
    dev = [_dev(f, ctx) for f in chain]
    out = np.zeros_like(v)
    ctx.check(lib().mgpu_chain_apply(ctx.handle, len(dev), _handles(dev), _ptr(v), _ptr(out), MGPU_HOST))
    return out


def chain_quality(chain: Sequence, K, samples: int, seed: int = 42, ctx=None) -> float:
    """spai.cpp:375-409: sqrt((n / samples) sum_k ||(I - K P) g_k||^2), the reference's probe
    stream (mt19937_64(seed), normal_distribution); chain newest first, may be empty."""
    ctx = ctx or default_context()
    dK = _dev(K, ctx)
    dev = [_dev(_factor_mat(f), ctx) for f in chain]
    out = C.c_double()
    ctx.check(lib().mgpu_chain_quality(ctx.handle, len(dev), _handles(dev) if dev else None, dK.handle,
                                       int(samples), int(seed), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- global Arnoldi + projection
def _fortran(a, rows=None):
    a = np.asfortranarray(np.asarray(a, np.float64))
    if a.ndim == 1:
        a = a.reshape(-1, 1, order="F")
    return a


def thin_qr(A, rank_tol: float = 1e-12, ctx=None):
    """dense.cpp:153-246 on the device: returns (Q, R, rank) like the reference's QrResult."""
    ctx = ctx or default_context()
    A = _fortran(A)
    rows, cols = A.shape
    Q = np.zeros((rows, cols), order="F")
    R = np.zeros((cols, cols), order="F")
    rank = C.c_int64()
    ctx.check(lib().mgpu_thin_qr(ctx.handle, rows, cols, _ptr(A), rank_tol, _ptr(Q), _ptr(R), C.byref(rank),
                                 MGPU_HOST))
    return Q, R, rank.value


def project_reduce(M, D, K, V, F=None, Cp=None, Cv=None, ctx=None) -> dict:
    """airga.cpp:485-500 on the device: Mh, Dh, Kh = V^T S V, Fh = V^T F, Cph / Cvh = C V."""
    ctx = ctx or default_context()
    dM, dD, dK = (_dev(x, ctx) for x in (M, D, K))
    V = _fortran(V)
    n, r = V.shape
    Fm = _fortran(F) if F is not None else np.zeros((n, 0), order="F")
    m = Fm.shape[1]
    q = 0 if Cp is None else _fortran(Cp).shape[0]
    Cpm = _fortran(Cp) if q else np.zeros((0, n), order="F")
    Cvm = _fortran(Cv) if q else np.zeros((0, n), order="F")
    out = {k: np.zeros(shape, order="F") for k, shape in
           (("Mh", (r, r)), ("Dh", (r, r)), ("Kh", (r, r)), ("Fh", (r, m)), ("Cph", (q, r)), ("Cvh", (q, r)))}
    ctx.check(lib().mgpu_project_reduce(ctx.handle, dM.handle, dD.handle, dK.handle, r, _ptr(V), m,
                                        _ptr(Fm) if m else None, q, _ptr(Cpm) if q else None,
                                        _ptr(Cvm) if q else None, _ptr(out["Mh"]), _ptr(out["Dh"]), _ptr(out["Kh"]),
                                        _ptr(out["Fh"]) if m else None, _ptr(out["Cph"]) if q else None,
                                        _ptr(out["Cvh"]) if q else None, MGPU_HOST))
    return out


def project_reduce_slab(M, D, K, row0: int, ext0: int, Vext, F=None, Cp=None, Cv=None, ctx=None) -> dict:
    """Partial projections of one row slab (mgpu_project_reduce_slab): M, D, K are the slab's rows with
    global column indices, Vext the basis rows [ext0, ext0 + len(Vext)), F / Cp / Cv the slab's parts."""
    ctx = ctx or default_context()
    dM, dD, dK = (_dev(x, ctx) for x in (M, D, K))
    V = _fortran(Vext)
    nx, r = V.shape
    p = dM.nrows
    Fm = _fortran(F) if F is not None else np.zeros((p, 0), order="F")
    m = Fm.shape[1]
    q = 0 if Cp is None else _fortran(Cp).shape[0]
    Cpm = _fortran(Cp) if q else np.zeros((0, p), order="F")
    Cvm = _fortran(Cv) if q else np.zeros((0, p), order="F")
    out = {k: np.zeros(shape, order="F") for k, shape in
           (("Mh", (r, r)), ("Dh", (r, r)), ("Kh", (r, r)), ("Fh", (r, m)), ("Cph", (q, r)), ("Cvh", (q, r)))}
    ctx.check(lib().mgpu_project_reduce_slab(ctx.handle, dM.handle, dD.handle, dK.handle, row0, ext0, nx, r, _ptr(V),
                                             m, _ptr(Fm) if m else None, q, _ptr(Cpm) if q else None,
                                             _ptr(Cvm) if q else None, _ptr(out["Mh"]), _ptr(out["Dh"]),
                                             _ptr(out["Kh"]), _ptr(out["Fh"]) if m else None,
                                             _ptr(out["Cph"]) if q else None, _ptr(out["Cvh"]) if q else None,
                                             MGPU_HOST))
    return out


def arnoldi_deflate(X, blocks: Sequence, ctx=None):
    """airga.cpp:456-473 on the device: returns (deflated X, gammas)."""
    ctx = ctx or default_context()
    X = _fortran(X).copy(order="F")
    bl = [_fortran(b) for b in blocks]
    for b in bl:
        if b.shape != X.shape:
            raise ArgumentError("arnoldi_deflate: block shape mismatch")
    ptrs = (C.c_void_p * max(len(bl), 1))(*[b.ctypes.data for b in bl])
    g = np.zeros(len(bl))
    ctx.check(lib().mgpu_arnoldi_deflate(ctx.handle, X.size, _ptr(X), len(bl), ptrs if bl else None,
                                         _ptr(g) if bl else None, MGPU_HOST))
    return X, g


# ---------------------------------------------------------------- SPAI
@dataclass
class SpaiFactor:
    """spai.hpp:18-29: device factor + per-column residuals + seconds."""

    matrix: DeviceCsr
    target_frob_residual: Optional[np.ndarray] = None
    build_seconds: float = 0.0
    kind: str = "base"


def spai_build(K, tol: float = 0.01, max_col_iters: int = 50, mode: int = FROZEN, ctx=None) -> SpaiFactor:
    """spai.cpp:314-331 (MR-SPAI)."""
    ctx = ctx or default_context()
    dK = _dev(K, ctx)
    res = np.zeros(dK.nrows)
    h = C.c_void_p()
    ctx.check(lib().mgpu_spai_build(ctx.handle, dK.handle, tol, max_col_iters, mode, C.byref(h), _ptr(res)))
    return SpaiFactor(DeviceCsr(ctx, h, dK.nrows), res, 0.0, "base")


def spai_update(K_old, K_new, tol: float = 0.01, max_col_iters: int = 50, mode: int = FROZEN,
                ctx=None) -> SpaiFactor:
    """spai.cpp:333-350 (MR-SPAI update)."""
    ctx = ctx or default_context()
    dO, dN = _dev(K_old, ctx), _dev(K_new, ctx)
    res = np.zeros(dN.nrows)
    h = C.c_void_p()
    ctx.check(lib().mgpu_spai_update(ctx.handle, dO.handle, dN.handle, tol, max_col_iters, mode, C.byref(h),
                                     _ptr(res)))
    return SpaiFactor(DeviceCsr(ctx, h, dN.nrows), res, 0.0, "update")


def spai_ls(A, K_old=None, pattern: int = PATTERN_A, ctx=None) -> SpaiFactor:
    """Static-pattern least-squares SPAI (north star subsystem 1)."""
    ctx = ctx or default_context()
    dA = _dev(A, ctx)
    dO = _dev(K_old, ctx) if K_old is not None else None
    h = C.c_void_p()
    ctx.check(lib().mgpu_spai_ls(ctx.handle, dA.handle, dO.handle if dO else None, pattern, C.byref(h)))
    return SpaiFactor(DeviceCsr(ctx, h, dA.nrows), None, 0.0, "base" if K_old is None else "update")


def spai_ls_batched(As: Sequence, K_olds: Optional[Sequence] = None, pattern: int = PATTERN_A, ctx=None) -> list:
    ctx = ctx or default_context()
    dA = [_dev(a, ctx) for a in As]
    dO = [_dev(k, ctx) for k in K_olds] if K_olds is not None else None
    out = (C.c_void_p * max(len(dA), 1))()
    ctx.check(lib().mgpu_spai_ls_batched(ctx.handle, len(dA), _handles(dA), _handles(dO) if dO else None, pattern,
                                         out))
    return [SpaiFactor(DeviceCsr(ctx, C.c_void_p(out[i]), dA[i].nrows)) for i in range(len(dA))]


def spgemm(A, B, ctx=None) -> DeviceCsr:
    ctx = ctx or default_context()
    dA, dB = _dev(A, ctx), _dev(B, ctx)
    h = C.c_void_p()
    ctx.check(lib().mgpu_spgemm(ctx.handle, dA.handle, dB.handle, C.byref(h)))
    return DeviceCsr(ctx, h, dA.nrows)


# ---------------------------------------------------------------- Krylov
@dataclass
class BlockSolveResult:
    """krylov.hpp:44-51 (per point when batched)."""

    X: np.ndarray
    recurrence_residuals: np.ndarray
    true_residuals: np.ndarray
    iterations: np.ndarray
    all_converged: bool
    converged: np.ndarray = field(default=None)
    status: np.ndarray = field(default=None)
    breakdown_iteration: np.ndarray = field(default=None)
    relres_history: Optional[np.ndarray] = None


def _factor_mat(f):
    return f.matrix if isinstance(f, SpaiFactor) else f


def cg_solve_raw(ctx: Context, dA: Sequence[DeviceCsr], flat_chain: Sequence[DeviceCsr], z: int, n: int, m: int,
                 B_ptr: int, ldb: int, rtol: float, maxit: int, where: int, X_ptr: int, REC_ptr: int, TR_ptr: int,
                 history_cap: int = 0):
    """Direct mgpu_cg_solve call: pointers are host (where=MGPU_HOST) or device (MGPU_DEVICE).
    Returns (status, iterations, converged, status_per_column, breakdown_iteration, history)."""
    l = len(dA)
    it = np.zeros(l * m, np.int64)
    cv = np.zeros(l * m, np.int32)
    st = np.zeros(l * m, np.int32)
    bd = np.zeros(l * m, np.int64)
    hist = np.zeros(max(l * m * history_cap, 1))
    out = _CgOut(X_ptr, REC_ptr, TR_ptr, it.ctypes.data_as(C.POINTER(C.c_int64)),
                 cv.ctypes.data_as(C.POINTER(C.c_int)), st.ctypes.data_as(C.POINTER(C.c_int)),
                 bd.ctypes.data_as(C.POINTER(C.c_int64)),
                 hist.ctypes.data_as(C.POINTER(C.c_double)) if history_cap > 0 else None, history_cap)
    status = lib().mgpu_cg_solve(ctx.handle, l, _handles(dA), z, _handles(flat_chain), n, m, C.c_void_p(B_ptr), ldb,
                                 rtol, maxit, where, C.byref(out))
    return status, it, cv, st, bd, (hist.reshape(l, m, history_cap) if history_cap > 0 else None)


def shifted_solve_raw(ctx: Context, M, D, K, shifts: Sequence[float], pattern: int, m: int, B_ptr: int, ldb: int,
                      rtol: float, maxit: int, where: int, X_ptr: int, REC_ptr: int, TR_ptr: int):
    """mgpu_shifted_solve: assembly of every shifted operator, LS-SPAI on `pattern` (-1: P = I)
    and the batched solve in one library call (CgBackend::prepare + solve of every point,
    airga.cpp:108-181).  Returns (status, iterations, converged, status_per_column,
    breakdown_iteration, phase_ms[assembly, spai, solve])."""
    dM, dD, dK = (_dev(x, ctx) for x in (M, D, K))
    sh = np.ascontiguousarray(shifts, np.float64)
    l = len(sh)
    it = np.zeros(l * m, np.int64)
    cv = np.zeros(l * m, np.int32)
    st = np.zeros(l * m, np.int32)
    bd = np.zeros(l * m, np.int64)
    ph = np.zeros(3)
    out = _CgOut(X_ptr, REC_ptr, TR_ptr, it.ctypes.data_as(C.POINTER(C.c_int64)),
                 cv.ctypes.data_as(C.POINTER(C.c_int)), st.ctypes.data_as(C.POINTER(C.c_int)),
                 bd.ctypes.data_as(C.POINTER(C.c_int64)), None, 0)
    status = lib().mgpu_shifted_solve(ctx.handle, dM.handle, dD.handle, dK.handle, l, _ptr(sh), pattern,
                                      C.c_void_p(B_ptr), m, ldb, rtol, maxit, where, C.byref(out), _ptr(ph))
    return status, it, cv, st, bd, ph


def shifted_solve_device(M, D, K, shifts: Sequence[float], pattern: int, B_dev, X_dev, REC_dev=None, TR_dev=None,
                         rtol: float = 1e-10, maxit: Optional[int] = None, ctx=None):
    """Device-resident shifted_solve: B_dev one (m, n) block shared by every point, X_dev /
    REC_dev / TR_dev torch CUDA float64 tensors [point][column][row].  Raises on every status
    but BREAKDOWN (reported per column).  Returns (iterations, converged, status, breakdown,
    phase_ms)."""
    ctx = ctx or default_context()
    n = _dev(M, ctx).nrows
    m = int(B_dev.shape[-2]) if B_dev.dim() >= 2 else 1
    maxit = 10 * n if maxit is None else maxit
    ptr = lambda t: t.data_ptr() if t is not None else 0
    status, it, cv, st, bd, ph = shifted_solve_raw(ctx, M, D, K, shifts, pattern, m, B_dev.data_ptr(), 0, rtol, maxit,
                                                   MGPU_DEVICE, ptr(X_dev), ptr(REC_dev), ptr(TR_dev))
    if status != MGPU_OK and status != MGPU_ERR_BREAKDOWN:
        ctx.check(status)
    return it, cv, st, bd, ph


def cg_solve_batched(As: Sequence, chains: Sequence[Sequence], B, rtol: float = 1e-10, maxit: Optional[int] = None,
                     history_cap: int = 0, raise_on_breakdown: bool = True, ctx=None, host_out=None):
    """Batched block_solve over points (mgpu_cg_solve), host buffers.
    B: (n,) / (n, m) shared by every point, or (l, n, m).  host_out: optional dict of
    preallocated (l, m, n) float64 arrays X / REC / TR (e.g. pinned memory)."""
    ctx = ctx or default_context()
    dA = [_dev(a, ctx) for a in As]
    l = len(dA)
    n = dA[0].nrows
    z = len(chains[0]) if chains else 0
    assert all(len(c) == z for c in chains), "uniform chain length per batch"
    flat = [_dev(_factor_mat(f), ctx) for c in chains for f in c]
    Bn = np.asarray(B, np.float64)
    if Bn.ndim == 1:
        Bn = Bn[:, None]
    if Bn.ndim == 2:
        m = Bn.shape[1]
        Bc = np.ascontiguousarray(Bn.T)  # [c][row]
        ldb = 0
    else:
        m = Bn.shape[2]
        Bc = np.ascontiguousarray(np.transpose(Bn, (0, 2, 1)))  # [p][c][row]
        ldb = n * m
    maxit = 10 * n if maxit is None else maxit
    if host_out is None:
        X, REC, TR = (np.zeros((l, m, n)) for _ in range(3))
    else:
        X, REC, TR = host_out["X"], host_out["REC"], host_out["TR"]
    status, it, cv, st, bd, hist = cg_solve_raw(ctx, dA, flat, z, n, m, Bc.ctypes.data, ldb, rtol, maxit, MGPU_HOST,
                                                X.ctypes.data, REC.ctypes.data, TR.ctypes.data, history_cap)
    if status != MGPU_OK and (raise_on_breakdown or status != MGPU_ERR_BREAKDOWN):
        ctx.check(status)
    results = []
    for p in range(l):
        sl = slice(p * m, (p + 1) * m)
        results.append(BlockSolveResult(X=X[p].T.copy(), recurrence_residuals=REC[p].T.copy(),
                                        true_residuals=TR[p].T.copy(), iterations=it[sl].copy(),
                                        all_converged=bool(cv[sl].all()), converged=cv[sl].astype(bool),
                                        status=st[sl].copy(), breakdown_iteration=bd[sl].copy(),
                                        relres_history=hist[p] if hist is not None else None))
    return results


def cg_solve_device(As: Sequence, chains: Sequence[Sequence], B_dev, X_dev, REC_dev=None, TR_dev=None,
                    rtol: float = 1e-10, maxit: Optional[int] = None, shared_rhs: bool = True, ctx=None):
    """Device-resident batched solve.  B_dev / X_dev / ...: torch CUDA float64 tensors laid out
    [point][column][row] (B_dev may be one (m, n) block shared by every point)."""
    ctx = ctx or default_context()
    dA = [_dev(a, ctx) for a in As]
    n = dA[0].nrows
    z = len(chains[0]) if chains else 0
    flat = [_dev(_factor_mat(f), ctx) for c in chains for f in c]
    m = int(B_dev.shape[-2]) if B_dev.dim() >= 2 else 1
    maxit = 10 * n if maxit is None else maxit
    ptr = lambda t: t.data_ptr() if t is not None else 0
    status, it, cv, st, bd, _ = cg_solve_raw(ctx, dA, flat, z, n, m, B_dev.data_ptr(), 0 if shared_rhs else n * m,
                                             rtol, maxit, MGPU_DEVICE, ptr(X_dev), ptr(REC_dev), ptr(TR_dev))
    if status != MGPU_OK and status != MGPU_ERR_BREAKDOWN:
        ctx.check(status)
    return it, cv, st, bd


def block_solve(A, chain: Sequence, B, rtol: float = 1e-10, maxit: Optional[int] = None, ctx=None):
    """krylov.cpp:141-174 with P = chain_apply(chain) (airga.cpp:166-181)."""
    return cg_solve_batched([A], [list(chain)], B, rtol, maxit, ctx=ctx)[0]


def pcg_solve(A, chain: Sequence, b, rtol: float = 1e-10, maxit: Optional[int] = None, history_cap: int = 0,
              ctx=None) -> dict:
    """krylov.cpp:28-139 for one rhs; returns the SolveReport fields."""
    try:
        r = cg_solve_batched([A], [list(chain)], np.asarray(b, np.float64)[:, None], rtol, maxit,
                             history_cap=history_cap, ctx=ctx)[0]
    except BreakdownError as e:  # pcg_solve reports without the block_solve column prefix
        msg = str(e).split(": ", 1)[1] if str(e).startswith("block_solve") else str(e)
        raise BreakdownError(msg, e.index, -1, -1) from None
    hist = None
    if history_cap > 0:
        hist = r.relres_history[0][:min(int(r.iterations[0]), history_cap)]
    return dict(solution=r.X[:, 0], residual=r.true_residuals[:, 0], recurrence_residual=r.recurrence_residuals[:, 0],
                iterations=int(r.iterations[0]), converged=bool(r.converged[0]), relres_history=hist)


# ---------------------------------------------------------------- NCCL data plane
def csr_bandwidth(A, ctx=None) -> int:
    ctx = ctx or default_context()
    v = C.c_int64()
    ctx.check(lib().mgpu_csr_bandwidth(ctx.handle, _dev(A, ctx).handle, C.byref(v)))
    return v.value


def comm_allreduce_sum(t, ctx=None):
    """In-place sum over the context's ranks of a CUDA float64 tensor."""
    ctx = ctx or default_context()
    ctx.check(lib().mgpu_comm_allreduce_sum(ctx.handle, t.data_ptr(), t.numel()))


def comm_columns_to_rows(X_local, col_ids, R: int, h: int, ctx=None):
    """Device redistribution (mgpu_comm_columns_to_rows).  X_local: CUDA float64 tensor of shape
    (c_local, n) (= n x c_local column-major), col_ids its global column ids.  Returns
    (Vext, ext0): Vext a CUDA tensor (R, next) = next x R column-major rows [ext0, ext0 + next)."""
    import torch
    ctx = ctx or default_context()
    c_local, n = (int(X_local.shape[0]), int(X_local.shape[1])) if X_local.dim() == 2 else (0, 0)
    row0, p, ext0, nx = ctx.comm_rows(n, h)
    Vext = torch.empty((R, nx), dtype=torch.float64, device=X_local.device)
    ids = np.ascontiguousarray(np.asarray(col_ids, np.int64))
    ctx.check(lib().mgpu_comm_columns_to_rows(ctx.handle, n, h, c_local, _ptr(ids) if c_local else None,
                                              X_local.data_ptr() if c_local else None, R, Vext.data_ptr()))
    return Vext, ext0


def comm_project_reduce(M, D, K, h: int, Vext, F=None, Cp=None, Cv=None, ctx=None) -> dict:
    """mgpu_comm_project_reduce: replicated device operators, this rank's extended slab (CUDA tensor
    (r, next)), host F (n x m) / Cp, Cv (q x n).  Every rank receives the reduced matrices."""
    ctx = ctx or default_context()
    dM, dD, dK = (_dev(x, ctx) for x in (M, D, K))
    n = dM.nrows
    r = int(Vext.shape[0])
    Fm = _fortran(F) if F is not None else np.zeros((n, 0), order="F")
    m = Fm.shape[1]
    q = 0 if Cp is None else _fortran(Cp).shape[0]
    Cpm = _fortran(Cp) if q else np.zeros((0, n), order="F")
    Cvm = _fortran(Cv) if q else np.zeros((0, n), order="F")
    out = {k: np.zeros(shape, order="F") for k, shape in
           (("Mh", (r, r)), ("Dh", (r, r)), ("Kh", (r, r)), ("Fh", (r, m)), ("Cph", (q, r)), ("Cvh", (q, r)))}
    ctx.check(lib().mgpu_comm_project_reduce(ctx.handle, dM.handle, dD.handle, dK.handle, h, r, Vext.data_ptr(), m,
                                             _ptr(Fm) if m else None, q, _ptr(Cpm) if q else None,
                                             _ptr(Cvm) if q else None, _ptr(out["Mh"]), _ptr(out["Dh"]),
                                             _ptr(out["Kh"]), _ptr(out["Fh"]) if m else None,
                                             _ptr(out["Cph"]) if q else None, _ptr(out["Cvh"]) if q else None,
                                             MGPU_HOST))
    return out

