"""TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.

ctypes bindings for
  * ``liboracle.so``       -- oracle/oracle.c, the C restatement of the reference path;
  * ``_ref/libmorref.so``  -- the UNMODIFIED reference library compiled from
                              /root/reference/proj/src (oracle/Makefile) + ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  Both libraries expose the
same C signatures (``orc_*`` / ``ref_*``), so one binding class drives either.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmorref.so")

OK, ERR_ARG, ERR_STAGNATION, ERR_BREAKDOWN, ERR_NUMERICAL, ERR_UNSUPPORTED = 0, 1, 2, 3, 4, 5


@dataclass
class Csr:
    """Host CSR with the reference's conventions (sparse.hpp:12-22)."""

    nrows: int
    ncols: int
    row_ptr: np.ndarray  # int64
    col_idx: np.ndarray  # int32
    values: np.ndarray  # float64

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def todense(self) -> np.ndarray:
        out = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            out[i, self.col_idx[s:e]] = self.values[s:e]
        return out

    @staticmethod
    def from_dense(a: np.ndarray) -> "Csr":
        rows, cols = np.nonzero(a)
        rp = np.zeros(a.shape[0] + 1, np.int64)
        np.add.at(rp, rows + 1, 1)
        return Csr(a.shape[0], a.shape[1], np.cumsum(rp).astype(np.int64), cols.astype(np.int32),
                   a[rows, cols].astype(np.float64))


class _CCsr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int32)),
                ("values", C.POINTER(C.c_double))]


class _CErr(C.Structure):
    _fields_ = [("index", C.c_int64), ("msg", C.c_char * 512)]


class OracleError(RuntimeError):
    def __init__(self, status: int, index: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status, self.index, self.msg = status, index, msg


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


class _Lib:
    """Binding shared by the C restatement (prefix orc_) and the reference (ref_)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} is not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.kind = "reference" if prefix == "ref_" else "port"

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    # -- marshalling
    @staticmethod
    def _in(a: Csr) -> _CCsr:
        rp = np.ascontiguousarray(a.row_ptr, np.int64)
        ci = np.ascontiguousarray(a.col_idx, np.int32)
        v = np.ascontiguousarray(a.values, np.float64)
        c = _CCsr(a.nrows, a.ncols, v.shape[0], rp.ctypes.data_as(C.POINTER(C.c_int64)),
                  ci.ctypes.data_as(C.POINTER(C.c_int32)), v.ctypes.data_as(C.POINTER(C.c_double)))
        c._keep = (rp, ci, v)
        return c

    def _out(self, c: _CCsr) -> Csr:
        n, nnz = c.nrows, c.nnz
        rp = np.ctypeslib.as_array(c.row_ptr, (n + 1,)).copy()
        if nnz > 0:
            ci = np.ctypeslib.as_array(c.col_idx, (nnz,)).copy()
            v = np.ctypeslib.as_array(c.values, (nnz,)).copy()
        else:
            ci, v = np.zeros(0, np.int32), np.zeros(0)
        self._f("csr_free")(C.byref(c))
        return Csr(n, c.ncols, rp, ci, v)

    @staticmethod
    def _check(st: int, err: _CErr):
        if st != OK:
            raise OracleError(st, err.index, err.msg.decode(errors="replace"))

    def _chain(self, factors):
        z = len(factors)
        arr = (_CCsr * max(z, 1))()
        keep = []
        for i, f in enumerate(factors):
            c = self._in(f)
            keep.append(c)
            arr[i] = c
        return z, arr, keep

    # -- API
    def from_triplets(self, nrows, ncols, rows, cols, vals) -> Csr:
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        out, err = _CCsr(), _CErr()
        st = self._f("from_triplets")(C.c_int64(nrows), C.c_int64(ncols), C.c_int64(vals.shape[0]), _ip(rows),
                                      _ip(cols), _dp(vals), C.byref(out), C.byref(err))
        self._check(st, err)
        return self._out(out)

    def sp_add_scaled(self, A: Csr, B: Csr, a: float, b: float) -> Csr:
        out, err = _CCsr(), _CErr()
        st = self._f("sp_add_scaled")(C.byref(self._in(A)), C.byref(self._in(B)), C.c_double(a), C.c_double(b),
                                      C.byref(out), C.byref(err))
        self._check(st, err)
        return self._out(out)

    def shifted_operator(self, M: Csr, D: Csr, K: Csr, s: float) -> Csr:
        out, err = _CCsr(), _CErr()
        st = self._f("shifted_operator")(C.byref(self._in(M)), C.byref(self._in(D)), C.byref(self._in(K)),
                                         C.c_double(s), C.byref(out), C.byref(err))
        self._check(st, err)
        return self._out(out)

    def transpose(self, A: Csr) -> Csr:
        out, err = _CCsr(), _CErr()
        if self.prefix == "ref_":
            st = self._f("transpose")(C.byref(self._in(A)), C.byref(out), C.byref(err))
        else:
            st = self._f("transpose")(C.byref(self._in(A)), C.byref(out))
        self._check(st, err)
        return self._out(out)

    def trace(self, A: Csr) -> float:
        f = self._f("trace")
        f.restype = C.c_double
        return f(C.byref(self._in(A)))

    def trace_inner(self, A: Csr, B: Csr) -> float:
        f = self._f("trace_inner")
        f.restype = C.c_double
        return f(C.byref(self._in(A)), C.byref(self._in(B)))

    def spmv(self, A: Csr, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(A.nrows)
        if self.prefix == "ref_":
            err = _CErr()
            self._check(self._f("spmv")(C.byref(self._in(A)), _dp(x), _dp(y), C.byref(err)), err)
        else:
            self._f("spmv")(C.byref(self._in(A)), _dp(x), _dp(y))
        return y

    def chain_generate(self, n, alpha=0.05, beta=0.05, stiffness_scale=0.01, mass_scale=1.0, consistent=False):
        M, D, K, err = _CCsr(), _CCsr(), _CCsr(), _CErr()
        fn = self._f("beam_generate") if self.prefix == "ref_" else self._f("chain_generate")
        st = fn(C.c_int64(n), C.c_double(alpha), C.c_double(beta), C.c_double(stiffness_scale),
                C.c_double(mass_scale), C.c_int(1 if consistent else 0), C.byref(M), C.byref(D), C.byref(K),
                C.byref(err))
        self._check(st, err)
        return self._out(M), self._out(D), self._out(K)

    def spai_build(self, K: Csr, tol=0.01, max_col_iters=50, mode=1, threads=1):
        P, err = _CCsr(), _CErr()
        res = np.zeros(K.nrows)
        if self.prefix == "ref_":
            sec = C.c_double()
            st = self._f("spai_build")(C.byref(self._in(K)), C.c_double(tol), C.c_int64(max_col_iters), C.c_int(mode),
                                       C.c_int64(threads), C.byref(P), _dp(res), C.byref(sec), C.byref(err))
        else:
            st = self._f("spai_build")(C.byref(self._in(K)), C.c_double(tol), C.c_int64(max_col_iters), C.c_int(mode),
                                       C.byref(P), _dp(res), C.byref(err))
        self._check(st, err)
        return self._out(P), res

    def spai_update(self, K_old: Csr, K_new: Csr, tol=0.01, max_col_iters=50, mode=1, threads=1):
        Q, err = _CCsr(), _CErr()
        res = np.zeros(K_new.nrows)
        if self.prefix == "ref_":
            sec = C.c_double()
            st = self._f("spai_update")(C.byref(self._in(K_old)), C.byref(self._in(K_new)), C.c_double(tol),
                                        C.c_int64(max_col_iters), C.c_int(mode), C.c_int64(threads), C.byref(Q),
                                        _dp(res), C.byref(sec), C.byref(err))
        else:
            st = self._f("spai_update")(C.byref(self._in(K_old)), C.byref(self._in(K_new)), C.c_double(tol),
                                        C.c_int64(max_col_iters), C.c_int(mode), C.byref(Q), _dp(res), C.byref(err))
        self._check(st, err)
        return self._out(Q), res

    def spai_ls(self, A: Csr, K_old: Csr | None = None, pattern: int = 0) -> Csr:
        P, err = _CCsr(), _CErr()
        kold = C.byref(self._in(K_old)) if K_old is not None else None
        if self.prefix == "ref_":
            sec = C.c_double()
            st = self._f("spai_ls")(C.byref(self._in(A)), kold, C.c_int(pattern), C.byref(P), C.byref(sec),
                                    C.byref(err))
        else:
            st = self._f("spai_ls")(C.byref(self._in(A)), kold, C.c_int(pattern), C.byref(P), C.byref(err))
        self._check(st, err)
        return self._out(P)

    def thin_qr(self, A: np.ndarray, rank_tol=1e-12):
        rows, cols = A.shape
        a = np.asfortranarray(A, np.float64)
        Q = np.zeros((rows, cols), order="F")
        R = np.zeros((cols, cols), order="F")
        rank = C.c_int64()
        if self.prefix == "ref_":
            err = _CErr()
            st = self._f("thin_qr")(C.c_int64(rows), C.c_int64(cols), _dp(a), C.c_double(rank_tol), _dp(Q), _dp(R),
                                    C.byref(rank), C.byref(err))
            self._check(st, err)
        else:
            st = self._f("thin_qr")(C.c_int64(rows), C.c_int64(cols), _dp(a), C.c_double(rank_tol), _dp(Q), _dp(R),
                                    C.byref(rank))
            assert st == OK
        return Q, R, rank.value

    def project_reduce(self, M, D, K, V, F=None, Cp=None, Cv=None) -> dict:
        """airga.cpp:485-500 (reference only)."""
        V = np.asfortranarray(V, np.float64)
        n, r = V.shape
        Fm = np.asfortranarray(F, np.float64) if F is not None else np.zeros((n, 0), order="F")
        m = Fm.shape[1]
        q = 0 if Cp is None else np.asarray(Cp).shape[0]
        Cpm = np.asfortranarray(Cp, np.float64) if q else np.zeros((0, n), order="F")
        Cvm = np.asfortranarray(Cv, np.float64) if q else np.zeros((0, n), order="F")
        out = {k: np.zeros(shape, order="F") for k, shape in
               (("Mh", (r, r)), ("Dh", (r, r)), ("Kh", (r, r)), ("Fh", (r, m)), ("Cph", (q, r)), ("Cvh", (q, r)))}
        hM, hD, hK = self._in(M), self._in(D), self._in(K)
        err = _CErr()
        st = self._f("project_reduce")(C.byref(hM), C.byref(hD), C.byref(hK), C.c_int64(r), _dp(V), C.c_int64(m),
                                       _dp(Fm), C.c_int64(q), _dp(Cpm), _dp(Cvm), _dp(out["Mh"]), _dp(out["Dh"]),
                                       _dp(out["Kh"]), _dp(out["Fh"]), _dp(out["Cph"]), _dp(out["Cvh"]),
                                       C.byref(err))
        self._check(st, err)
        return out

    def arnoldi_deflate(self, X, blocks):
        """airga.cpp:456-473 (reference only): returns (deflated X, gammas)."""
        X = np.asfortranarray(X, np.float64).copy(order="F")
        rows, cols = X.shape if X.ndim == 2 else (X.shape[0], 1)
        bl = [np.asfortranarray(b, np.float64) for b in blocks]
        ptrs = (C.c_void_p * max(len(bl), 1))(*[b.ctypes.data for b in bl])
        g = np.zeros(max(len(bl), 1))
        err = _CErr()
        st = self._f("arnoldi_deflate")(C.c_int64(rows), C.c_int64(cols), _dp(X), C.c_int(len(bl)), ptrs, _dp(g),
                                        C.byref(err))
        self._check(st, err)
        return X, g[:len(bl)]

    def chain_quality(self, factors, K, samples: int, seed: int = 42) -> float:
        """spai.cpp:375-409 (reference only: its probes are libstdc++'s mt19937_64 / normal_distribution)."""
        if self.prefix != "ref_":
            raise NotImplementedError("chain_quality is checked against the reference itself")
        z, arr, keep = self._chain(factors)
        hK = self._in(K)
        f = self._f("chain_quality")
        f.restype = C.c_double
        return f(C.c_int(z), arr, C.byref(hK), C.c_int64(samples), C.c_uint64(seed))

    def chain_apply(self, factors, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros_like(v)
        z, arr, keep = self._chain(factors)
        if self.prefix == "ref_":
            err = _CErr()
            self._check(self._f("chain_apply")(C.c_int(z), arr, C.c_int64(v.shape[0]), _dp(v), _dp(out),
                                               C.byref(err)), err)
        else:
            self._f("chain_apply")(C.c_int(z), arr, C.c_int64(v.shape[0]), _dp(v), _dp(out))
        return out

    def pcg_solve(self, A: Csr, factors, b, rtol=1e-10, maxit=None, history_cap=None):
        n = A.nrows
        maxit = 10 * n if maxit is None else maxit
        b = np.ascontiguousarray(b, np.float64)
        x, res, rec = np.zeros(n), np.zeros(n), np.zeros(n)
        it, conv, hl = C.c_int64(), C.c_int(), C.c_int64()
        cap = min(maxit, 100000) if history_cap is None else history_cap
        hist = np.zeros(max(cap, 1))
        z, arr, keep = self._chain(factors)
        err = _CErr()
        st = self._f("pcg_solve")(C.byref(self._in(A)), C.c_int(z), arr, _dp(b), C.c_double(rtol), C.c_int64(maxit),
                                  _dp(x), _dp(res), _dp(rec), C.byref(it), C.byref(conv), _dp(hist),
                                  C.c_int64(cap), C.byref(hl), C.byref(err))
        self._check(st, err)
        return dict(solution=x, residual=res, recurrence_residual=rec, iterations=it.value,
                    converged=bool(conv.value), relres_history=hist[:min(hl.value, cap)])

    def block_solve(self, A: Csr, factors, B, rtol=1e-10, maxit=None):
        n = A.nrows
        B = np.asfortranarray(np.atleast_2d(np.asarray(B, np.float64).T).T)
        m = B.shape[1]
        maxit = 10 * n if maxit is None else maxit
        X, rec, tr = (np.zeros((n, m), order="F") for _ in range(3))
        iters = np.zeros(m, np.int64)
        allc = C.c_int()
        z, arr, keep = self._chain(factors)
        err = _CErr()
        st = self._f("block_solve")(C.byref(self._in(A)), C.c_int(z), arr, C.c_int64(m), _dp(B), C.c_double(rtol),
                                    C.c_int64(maxit), _dp(X), _dp(rec), _dp(tr), _ip(iters), C.byref(allc),
                                    C.byref(err))
        self._check(st, err)
        return dict(X=X, recurrence_residuals=rec, true_residuals=tr, iterations=iters,
                    all_converged=bool(allc.value))


class Oracle(_Lib):
    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path, "orc_")

    def hermite_generate(self, ne, E=2.1e11, I=1e-8, rho=7800.0, area=1e-4, L=1.0, alpha=0.1, beta=1e-5):
        M, D, K, err = _CCsr(), _CCsr(), _CCsr(), _CErr()
        st = self.lib.orc_hermite_generate(C.c_int64(ne), C.c_double(E), C.c_double(I), C.c_double(rho),
                                           C.c_double(area), C.c_double(L), C.c_double(alpha), C.c_double(beta),
                                           C.byref(M), C.byref(D), C.byref(K), C.byref(err))
        self._check(st, err)
        return self._out(M), self._out(D), self._out(K)

    def pattern_square(self, A: Csr) -> Csr:
        out = _CCsr()
        self.lib.orc_pattern_square(C.byref(self._in(A)), C.byref(out))
        return self._out(out)


class Reference(_Lib):
    """The unmodified reference library (oracle/_ref).  Available only where it was built."""

    def __init__(self, path: str = REF_SO):
        super().__init__(path, "ref_")

    def force_kernels(self, variant: str) -> bool:
        return bool(self.lib.ref_force_kernels(0 if variant == "scalar" else 1))

    def backend(self, solver: str, M: Csr, D: Csr, K: Csr, spai_tol=0.01, spai_max_col_iters=50, spai_mode=1,
                cg_rtol=1e-10, cg_maxit_factor=10, update_start_iteration=3):
        """The reference CgBackend through make_backend (airga.cpp:358-365)."""
        return _RefBackend(self, solver, M, D, K, spai_tol, spai_max_col_iters, spai_mode, cg_rtol, cg_maxit_factor,
                           update_start_iteration)


class _RefBackend:
    def __init__(self, ref, solver, M, D, K, spai_tol, spai_max_col_iters, spai_mode, cg_rtol, cg_maxit_factor,
                 update_start_iteration):
        self.ref, self.lib = ref, ref.lib
        self.lib.ref_backend_create.restype = C.c_void_p
        code = {"cg_plain": 1, "cg_spai": 2, "cg_spai_update": 3}[solver]
        self._keep = [ref._in(x) for x in (M, D, K)]
        self.h = C.c_void_p(self.lib.ref_backend_create(
            C.c_int(code), C.c_double(spai_tol), C.c_int64(spai_max_col_iters), C.c_int(spai_mode),
            C.c_double(cg_rtol), C.c_int64(cg_maxit_factor), C.c_int64(update_start_iteration),
            *[C.byref(c) for c in self._keep]))
        self.n = M.nrows

    def prepare(self, points, outer):
        pts = np.ascontiguousarray(points, np.float64)
        l = len(pts)
        sec, kind, chain = np.zeros(l), np.zeros(l, np.int32), np.zeros(l, np.int64)
        err = _CErr()
        st = self.lib.ref_backend_prepare(self.h, C.c_int64(l), _dp(pts), C.c_int64(outer), _dp(sec),
                                          kind.ctypes.data_as(C.POINTER(C.c_int)), _ip(chain), C.byref(err))
        self.ref._check(st, err)
        return [dict(kind="base" if k == 0 else "update", chain_length=int(c), seconds=float(t))
                for k, c, t in zip(kind, chain, sec)]

    def solve(self, i, B):
        B = np.asfortranarray(np.atleast_2d(np.asarray(B, np.float64).T).T)
        n, m = B.shape
        X, rec, tr = (np.zeros((n, m), order="F") for _ in range(3))
        it = np.zeros(m, np.int64)
        allc = C.c_int()
        err = _CErr()
        st = self.lib.ref_backend_solve(self.h, C.c_int64(i), C.c_int64(n), C.c_int64(m), _dp(B), _dp(X), _dp(rec),
                                        _dp(tr), _ip(it), C.byref(allc), C.byref(err))
        self.ref._check(st, err)
        return dict(X=X, recurrence_residuals=rec, true_residuals=tr, iterations=it, all_converged=bool(allc.value))

    def __del__(self):
        try:
            self.lib.ref_backend_destroy(self.h)
        except Exception:
            pass


def reference_available() -> bool:
    return os.path.exists(REF_SO)
