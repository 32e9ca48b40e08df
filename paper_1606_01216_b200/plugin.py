"""ctypes binding of the drop-in SolveBackend's C entry points (include/mor_cuda.h, libmor_cuda.so).

This drives mor::CudaCgBackend -- the class the reference's make_backend returns
 -- the way the reference's own driver does: prepare(sys, points, outer), then
solve(i, rhs) per point (airga.cpp:108-181, 374-381).  bench.py's end-to-end leg and the plugin
tests use it.
"""
import ctypes as C
import os

import numpy as np

from . import mgpu as _mg

ROOT = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(ROOT, "lib", "libmor_cuda.so")
EXPORTED = ["mor_cuda_backend_create", "mor_cuda_backend_create_multi", "mor_cuda_backend_destroy", "mor_cuda_backend_set_system",
            "mor_cuda_backend_prepare", "mor_cuda_backend_solve"]
SOLVERS = {"cg_plain": 1, "cg_spai": 2, "cg_spai_update": 3}
_lib = None


def lib():
    global _lib
    if _lib is None:
        _mg.lib()  # libmgpu.so first (the plugin links it)
        if not os.path.exists(LIB_PATH):
            raise _mg.CudaError(f"{LIB_PATH} not built (make shim; it compiles against the reference headers)")
        # lazy binding: the LinearOperator adapters (cuda_backend.hpp SparseApply / ChainApply) call
        # the reference's host spmv / chain_apply, resolved only inside a reference process; the
        # backend itself never reaches them
        L = C.CDLL(LIB_PATH, mode=os.RTLD_LAZY)
        vp, i64, dp = C.c_void_p, C.c_int64, C.POINTER(C.c_double)
        L.mor_cuda_backend_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, i64, C.c_int,
                                              C.c_double, i64, i64, i64, C.c_int, C.POINTER(vp), C.c_char_p,
                                              C.c_size_t]
        L.mor_cuda_backend_create_multi.argtypes = [C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_double, i64,
                                                    C.c_int, C.c_double, i64, i64, i64, C.c_int, C.POINTER(vp),
                                                    C.c_char_p, C.c_size_t]
        L.mor_cuda_backend_destroy.argtypes = [vp]
        L.mor_cuda_backend_destroy.restype = None
        L.mor_cuda_backend_set_system.argtypes = [vp, i64] + [i64, vp, vp, vp] * 3 + [i64, vp, C.c_char_p,
                                                                                      C.c_size_t]
        L.mor_cuda_backend_prepare.argtypes = [vp, C.c_int, vp, i64, vp, C.c_char_p, C.c_size_t]
        L.mor_cuda_backend_solve.argtypes = [vp, i64, i64, vp, vp, vp, vp, vp, vp, C.c_char_p, C.c_size_t]
        _lib = L
    return _lib


def _raise(st, buf):
    if st != _mg.MGPU_OK:
        raise _mg._BY_STATUS.get(st, _mg.MgpuError)(buf.value.decode(errors="replace"), -1, -1, -1)


def _ptr(a):
    return a.ctypes.data if isinstance(a, np.ndarray) else int(a)


class PluginBackend:
    """mor::CudaCgBackend through include/mor_cuda.h."""

    def __init__(self, solver="cg_spai", algorithm="ls", ls_pattern=0, spai_tol=0.01, spai_max_col_iters=50,
                 spai_mode=1, cg_rtol=1e-10, cg_maxit_factor=10, maxit=0, update_start_iteration=3,
                 speculative=True, device=0, devices=None, collapse=False):
        """devices: several device ordinals -> mor::MultiDeviceCgBackend (point i on devices[i % N])."""
        self.h = C.c_void_p()
        buf = C.create_string_buffer(1024)
        devs = np.asarray(devices if devices is not None else [device], np.int32)
        st = lib().mor_cuda_backend_create_multi(len(devs), devs.ctypes.data, SOLVERS[solver],
                                                 1 if algorithm == "ls" else 0, ls_pattern, spai_tol,
                                                 spai_max_col_iters, spai_mode, cg_rtol, cg_maxit_factor, maxit,
                                                 update_start_iteration,
                                                 (1 if speculative else 0) | (2 if collapse else 0), C.byref(self.h),
                                                 buf, 1024)
        _raise(st, buf)
        self.n = 0

    def close(self):
        if self.h:
            lib().mor_cuda_backend_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_system(self, M, D, K, F):
        """M, D, K: objects with row_ptr / col_idx / values arrays (n x n); F: (n, m) float64."""
        F = np.asfortranarray(F, dtype=np.float64)
        self._keep = (M, D, K, F)
        n = M.nrows
        args = []
        for X in (M, D, K):
            args += [int(X.row_ptr[-1]), _ptr(X.row_ptr), _ptr(X.col_idx), _ptr(X.values)]
        buf = C.create_string_buffer(1024)
        st = lib().mor_cuda_backend_set_system(self.h, n, *args, F.shape[1], F.ctypes.data, buf, 1024)
        _raise(st, buf)
        self.n, self.m = n, F.shape[1]

    def prepare(self, points, outer):
        pts = np.ascontiguousarray(points, np.float64)
        secs = np.zeros(len(pts))
        buf = C.create_string_buffer(1024)
        st = lib().mor_cuda_backend_prepare(self.h, len(pts), pts.ctypes.data, outer, secs.ctypes.data, buf, 1024)
        _raise(st, buf)
        return secs

    def solve(self, i, rhs, X=None, REC=None, TR=None):
        """rhs: (n, m) Fortran-ordered float64 (or a raw pointer with self.m columns); outputs: optional
        preallocated n x m column-major buffers (numpy arrays or raw pointers, e.g. pinned memory).
        Returns (iterations, all_converged)."""
        if isinstance(rhs, np.ndarray):
            rhs = np.asfortranarray(rhs, dtype=np.float64)
            m = rhs.shape[1] if rhs.ndim == 2 else 1
        else:
            m = self.m
        it = np.zeros(m, np.int64)
        conv = C.c_int()
        buf = C.create_string_buffer(1024)
        p = lambda a: None if a is None else _ptr(a)
        st = lib().mor_cuda_backend_solve(self.h, i, m, _ptr(rhs), p(X), p(REC), p(TR), it.ctypes.data, C.byref(conv),
                                          buf, 1024)
        _raise(st, buf)
        return it, bool(conv.value)
