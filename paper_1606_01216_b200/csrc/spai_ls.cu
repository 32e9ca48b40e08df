// K-ls: static-pattern least-squares SPAI, one lane group per column (north
// star subsystem 1).  Not in the reference; its CPU definition is SURVEY.md 8(a')
// (oracle/oracle.c orc_spai_ls, pinned against reference thin_qr in
// oracle/ref_shim.cpp ref_spai_ls).
//
// Column j:  J = pattern row j (A's CSR pattern, or the symbolic A*A),
//            I = sorted union of the rows of A(:, J)      (from A^T rows),
//            S = A(I, J) gathered into shared memory (column-major, lane c = column c),
//            Householder thin QR of S in FP64 exactly as dense.cpp:153-246
//            (sign rule, rank flush, explicit Q, sign fix), y = Q^T e|_I,
//            back-substitution R m = y (acc = y_k - sum_t R_kt m_t, ascending t),
//            P(J, j) = m.
// Rank deficiency (sigma <= 1e-12 ||S||_F, dense.cpp:163-179, or |I| < |J|)
// raises NumericalError for the lowest such column.
//
// Output: P on a FIXED pattern (J-pattern transposed), exact zeros kept as
// storage (dropped on download), so the pattern is reusable across shifts.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <vector>

#include "internal.cuh"

namespace mgpu
{
mgpu_csr *transpose_csr(mgpu_ctx *ctx, const mgpu_csr *A);
mgpu_csr *transpose_perm(mgpu_ctx *ctx, const mgpu_csr *A, DBuf &perm);
void gather_dev(mgpu_ctx *ctx, int64_t nnz, const int64_t *perm, const double *src, double *dst);
void gather_batched(mgpu_ctx *ctx, int l, int64_t nnz, const int64_t *perm, const double *const *src,
                    double *const *dst);

namespace
{


// ---------------------------------------------------------------- A*A pattern
constexpr int kSqCap = 128;

__device__ int square_row(int64_t i, DCsr A, int32_t *buf)
{
  int cnt = 0;
  for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k)
  {
    const int32_t t = A.ci[k];
    for (int64_t q = A.rp[t]; q < A.rp[t + 1]; ++q)
    {
      const int32_t c = A.ci[q];
      bool seen = false;
      for (int u = 0; u < cnt; ++u)
        seen |= buf[u] == c;
      if (!seen)
      {
        if (cnt == kSqCap)
          return -1;
        buf[cnt++] = c;
      }
    }
  }
  for (int a = 1; a < cnt; ++a) // insertion sort (rows are short)
  {
    const int32_t v = buf[a];
    int b = a - 1;
    while (b >= 0 && buf[b] > v)
    {
      buf[b + 1] = buf[b];
      --b;
    }
    buf[b + 1] = v;
  }
  return cnt;
}

__global__ void square_count(int64_t n, DCsr A, int64_t *rp, int *overflow)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  int32_t buf[kSqCap];
  const int c = square_row(i, A, buf);
  if (c < 0)
    atomicOr(overflow, 1);
  rp[i + 1] = c < 0 ? 0 : c;
  if (i == 0)
    rp[0] = 0;
}

__global__ void square_fill(int64_t n, DCsr A, const int64_t *rp, int32_t *ci)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  int32_t buf[kSqCap];
  const int c = square_row(i, A, buf);
  for (int u = 0; u < c; ++u)
    ci[rp[i] + u] = buf[u];
}

// ---------------------------------------------------------------- LS columns
//
// One GROUP of G lanes per column j (G = 8, 16 or 32 = the |J| envelope, so a
// warp solves 32/G columns).  Lane c of the group owns column c of S and
// replays thin_qr (dense.cpp:153-246) with the scalar kernel table's
// in-order dot / axpy (kernels_scalar.cpp:13-29) for that column: the
// Householder vector of step k is broadcast through shared memory, every
// lane c > k applies it to its own column.  Q is formed column by column the
// same way, the sign fix is applied, y = Q^T e by in-order dots and
// R m = y is back-substituted by the group leader.  Same operations in the
// same order as the oracle -> bitwise equal results; the ill-conditioned
// update problems (cond(S) ~ 5e7 on the Hermite beam) need exactly that.
template <int G, int NI>
struct LsGroupSmem
{
  double dsc[G]; // column scales 1 / ||S_c|| (column-equilibrated variant)
  double W[G * (NI + 1)]; // S / Householder vectors, column-major, ld = NI + 1 (odd: bank spread)
  double Q[G * (NI + 1)]; // Q; before the QR: staged values of A^T row J_c (lane c)
  int32_t rows[G * NI];    // staged column indices of A^T row J_c (lane c)
  int cnt[G];
  double e[NI];
  double m[G];
  double diag[G];
  double tau[G];
  int32_t I[NI];
  int ni, nj, fail;
};

__device__ __forceinline__ double dot_serial(const double *x, const double *y, int len)
{
  double acc = 0.0;
  for (int i = 0; i < len; ++i)
    acc = __dadd_rn(acc, __dmul_rn(x[i], y[i]));
  return acc;
}

__device__ __forceinline__ void axpy_serial(int len, double a, const double *x, double *y)
{
  for (int i = 0; i < len; ++i)
    y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
}

// Error key: (column << 8) | status, atomicMin picks the lowest column.
__device__ __forceinline__ void report(unsigned long long *err, int64_t j, int status)
{
  atomicMin(err, (static_cast<unsigned long long>(j) << 8) | static_cast<unsigned long long>(status));
}

// Batched over l operators sharing one pattern: column g = p * n + j reads
// A_p through At (shared structure, values at At.v + p * at_stride), K_old_p
// likewise, and writes P_p^T values at out_vals + p * out_stride.
template <int G, int NI, bool CS>
__global__ void ls_columns(int64_t n, int l, DCsr pat, DCsr At, int64_t at_stride, DCsr Kot, int64_t ko_stride,
                           bool update, double *__restrict__ out_base, int64_t out_stride,
                           unsigned long long *__restrict__ err, int *__restrict__ overflow)
{
  extern __shared__ __align__(16) unsigned char ls_raw[];
  constexpr int kGroups = 32 / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G, c = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  auto &sm = reinterpret_cast<LsGroupSmem<G, NI> *>(ls_raw)[warp * kGroups + grp];
  const int64_t g = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp) * kGroups + grp;
  if (g >= static_cast<int64_t>(l) * n)
    return;
  const int p = static_cast<int>(g / n);
  const int64_t j = g - static_cast<int64_t>(p) * n;
  At.v += p * at_stride;
  if (update)
    Kot.v += p * ko_stride;
  double *out_vals = out_base + p * out_stride;
  const int64_t jb = pat.rp[j];
  const int nj = static_cast<int>(pat.rp[j + 1] - jb);
  if (nj == 0)
    return;
  if (nj > G)
  {
    if (c == 0)
      atomicOr(overflow, 1);
    return;
  }
  // ---- stage A^T row J_c (= column J_c of A) per lane: one dependent-load chain per lane
  if (c < nj)
  {
    const int32_t k = pat.ci[jb + c];
    const int64_t t0 = At.rp[k], t1 = At.rp[k + 1];
    const int len = static_cast<int>(t1 - t0);
    sm.cnt[c] = len;
    for (int u = 0; u < len && u < NI; ++u)
    {
      sm.rows[c * NI + u] = At.ci[t0 + u];
      sm.Q[c * (NI + 1) + u] = At.v[t0 + u];
    }
  }
  __syncwarp(gmask);
  // ---- I = sorted union of the rows of A(:, J)   (leader, insertion over the staged lists)
  if (c == 0)
  {
    int ni = 0;
    bool over = false;
    for (int q = 0; q < nj && !over; ++q)
    {
      if (sm.cnt[q] > NI)
      {
        over = true;
        break;
      }
      for (int u = 0; u < sm.cnt[q]; ++u)
      {
        const int32_t row = sm.rows[q * NI + u];
        int pos = ni;
        while (pos > 0 && sm.I[pos - 1] > row)
          --pos;
        if (pos > 0 && sm.I[pos - 1] == row)
          continue;
        if (ni == NI)
        {
          over = true;
          break;
        }
        for (int u2 = ni; u2 > pos; --u2)
          sm.I[u2] = sm.I[u2 - 1];
        sm.I[pos] = row;
        ++ni;
      }
    }
    sm.ni = ni;
    sm.nj = nj;
    sm.fail = over ? 2 : (ni < nj ? 1 : 0);
  }
  __syncwarp(gmask);
  if (sm.fail == 2)
  {
    if (c == 0)
      atomicOr(overflow, 1);
    return;
  }
  if (sm.fail == 1)
  {
    if (c == 0)
      report(err, g, MGPU_ERR_NUMERICAL);
    return;
  }
  const int ni = sm.ni;
  constexpr int LD = NI + 1;
  // ---- S = A(I, J): lane c fills column c from its staged row; e = rhs|_I
  if (c < nj)
  {
    double *col = sm.W + c * LD;
    for (int i = 0; i < ni; ++i)
      col[i] = 0.0;
    for (int u = 0; u < sm.cnt[c]; ++u)
    {
      const int32_t row = sm.rows[c * NI + u];
      int lo = 0, hi = ni;
      while (lo < hi)
      {
        const int mid = (lo + hi) >> 1;
        if (sm.I[mid] < row)
          lo = mid + 1;
        else
          hi = mid;
      }
      col[lo] = sm.Q[c * LD + u];
    }
  }
  if (c == 0)
  {
    for (int i = 0; i < ni; ++i)
      sm.e[i] = 0.0;
    if (update)
    {
      for (int64_t q = Kot.rp[j]; q < Kot.rp[j + 1]; ++q)
      {
        const int32_t row = Kot.ci[q];
        int lo = 0, hi = ni;
        while (lo < hi)
        {
          const int mid = (lo + hi) >> 1;
          if (sm.I[mid] < row)
            lo = mid + 1;
          else
            hi = mid;
        }
        if (lo < ni && sm.I[lo] == row)
          sm.e[lo] = Kot.v[q];
      }
    }
    else
    {
      for (int i = 0; i < ni; ++i)
        if (sm.I[i] == j)
          sm.e[i] = 1.0;
    }
  }
  __syncwarp(gmask);
  if (CS) // column equilibration: r_c = 1 / ||S_c|| (in-order dot), S_c *= r_c (oracle.c orc_spai_ls)
  {
    if (c < nj)
    {
      double *col = sm.W + c * LD;
      const double d = sqrt(dot_serial(col, col, ni));
      sm.dsc[c] = d == 0.0 ? 0.0 : 1.0 / d;
      if (d != 0.0)
        for (int i = 0; i < ni; ++i)
          col[i] = __dmul_rn(col[i], sm.dsc[c]);
    }
    __syncwarp(gmask);
    bool zero = false;
    for (int q = 0; q < nj; ++q)
      zero |= sm.dsc[q] == 0.0;
    if (zero)
    {
      if (c == 0)
        report(err, g, MGPU_ERR_NUMERICAL);
      return;
    }
  }
  // ---- thin_qr (dense.cpp:153-246)
  double tol = 0.0;
  if (c == 0)
  {
    double acc = 0.0; // frob_norm: dot over all values, column-major order (dense.cpp:32-36)
    for (int q = 0; q < nj; ++q)
      for (int i = 0; i < ni; ++i)
        acc = __dadd_rn(acc, __dmul_rn(sm.W[q * LD + i], sm.W[q * LD + i]));
    const double anorm = sqrt(acc);
    sm.m[0] = 1e-12 * (anorm > 0.0 ? anorm : 1.0);
  }
  __syncwarp(gmask);
  tol = sm.m[0];
  bool deficient = false;
  for (int k = 0; k < nj; ++k)
  {
    const int len = ni - k;
    if (c == k)
    {
      double *x = sm.W + k * LD + k;
      const double sigma = sqrt(dot_serial(x, x, len));
      if (sigma <= tol)
      {
        sm.diag[k] = 0.0;
        sm.tau[k] = 0.0;
        for (int i = 0; i < len; ++i)
          x[i] = 0.0;
      }
      else
      {
        const double alpha = x[0] >= 0.0 ? -sigma : sigma;
        x[0] = __dsub_rn(x[0], alpha);
        const double vtv = dot_serial(x, x, len);
        sm.tau[k] = vtv > 0.0 ? 2.0 / vtv : 0.0;
        sm.diag[k] = alpha;
      }
    }
    __syncwarp(gmask);
    if (sm.diag[k] == 0.0)
      deficient = true;
    if (c > k && c < nj && sm.tau[k] != 0.0)
    {
      const double *v = sm.W + k * LD + k;
      double *y = sm.W + c * LD + k;
      const double s = __dmul_rn(sm.tau[k], dot_serial(v, y, len));
      axpy_serial(len, -s, v, y);
    }
    __syncwarp(gmask);
  }
  if (deficient) // rank < |J|
  {
    if (c == 0)
      report(err, g, MGPU_ERR_NUMERICAL);
    return;
  }
  // ---- Q = H_0 ... H_{nj-1} E, lane c forms column c
  if (c < nj)
  {
    double *q = sm.Q + c * LD;
    for (int i = 0; i < ni; ++i)
      q[i] = 0.0;
    q[c] = 1.0;
    for (int k = c < nj - 1 ? c : nj - 1; k >= 0; --k)
    {
      if (sm.tau[k] == 0.0)
        continue;
      const double *v = sm.W + k * LD + k;
      const int len = ni - k;
      const double s = __dmul_rn(sm.tau[k], dot_serial(v, q + k, len));
      axpy_serial(len, -s, v, q + k);
    }
  }
  __syncwarp(gmask);
  // ---- sign fix (R diagonal nonnegative) and y = Q^T e
  // R(k, q) = W[q][k] for q > k, R(k, k) = diag[k]; row k of R is touched only
  // by column owners q >= k, so every lane flips its own entries.
  if (c < nj)
  {
    for (int k = 0; k <= c; ++k)
    {
      if (sm.diag[k] < 0.0)
      {
        if (k == c)
        {
          for (int i = 0; i < ni; ++i)
            sm.Q[c * LD + i] = __dmul_rn(sm.Q[c * LD + i], -1.0);
        }
        else
          sm.W[c * LD + k] = -sm.W[c * LD + k];
      }
    }
  }
  __syncwarp(gmask);
  if (c < nj)
  {
    const double rkk = sm.diag[c] < 0.0 ? -sm.diag[c] : sm.diag[c];
    sm.tau[c] = rkk; // tau no longer needed: reuse as |R_cc|
    sm.m[c] = dot_serial(sm.Q + c * LD, sm.e, ni); // y_c
  }
  __syncwarp(gmask);
  // ---- back-substitution R m = y (oracle order: acc = y_k; acc -= R_kq m_q, q ascending)
  if (c == 0)
  {
    double mm[G];
    for (int k = nj - 1; k >= 0; --k)
    {
      double acc = sm.m[k];
      for (int q = k + 1; q < nj; ++q)
        acc = __dsub_rn(acc, __dmul_rn(sm.W[q * LD + k], mm[q]));
      mm[k] = acc / sm.tau[k];
    }
    for (int k = 0; k < nj; ++k)
      sm.m[k] = mm[k];
  }
  __syncwarp(gmask);
  if (c < nj)
    out_vals[jb + c] = CS ? __dmul_rn(sm.m[c], sm.dsc[c]) : sm.m[c];
}

// Longest row of a CSR structure (warp max, one atomic per warp).
__global__ void ls_max_row(int64_t nrows, const int64_t *__restrict__ rp, int *out)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int len = i < nrows ? static_cast<int>(rp[i + 1] - rp[i]) : 0;
  for (int off = 16; off > 0; off >>= 1)
    len = max(len, __shfl_xor_sync(0xffffffffu, len, off));
  if ((threadIdx.x & 31) == 0 && len > 0)
    atomicMax(out, len);
}

// ---------------------------------------------------------------- LS columns, one LANE per column
//
// The same column problem as ls_columns, solved start to finish by one thread: 32 columns per
// warp with every lane busy (the group kernel runs the leader-only steps -- union of I, the
// Householder scalars, back-substitution -- on one lane in eight).  Per-lane scratch lives in
// shared memory at an odd stride in 8-byte words, so the 32 lanes' same-offset accesses fall
// in distinct banks.  Q is never stored whole: column c of Q is rebuilt in one NI-vector
// (H_0 .. H_c applied to e_c, the same reflector loop as thin_qr's Q formation), sign-fixed
// and dotted with e, which gives y_c with exactly the operations of the group kernel and the
// oracle (bitwise equal).  That column and e live in registers (loops unrolled to the NJ x NI
// envelope, so every index is a compile-time constant): only W, the reflector scalars and I
// take shared memory, which sets the occupancy.  Envelope: |J| <= NJ, |I| <= NI; a larger column sets `overflow` and
// the host reruns the batch on the group kernels.
template <int NJ, int NI, bool CS = false>
struct LaneLayout
{
  static constexpr int kW = 0;                // W[c * NI + i]: S, then Householder vectors / R
  static constexpr int kDiag = kW + NJ * NI;  // R diagonal (alpha)
  static constexpr int kTau = kDiag + NJ;     // reflector scales, then |R_cc|
  static constexpr int kM = kTau + NJ;        // y, then the solution
  static constexpr int kI = kM + NJ;          // I (int32, NI of them = NI / 2 words)
  static constexpr int kDsc = kI + (NI + 1) / 2; // column scales (CS only)
  static constexpr int kWords0 = kDsc + (CS ? NJ : 0);
  static constexpr int kWords = kWords0 | 1; // odd stride: conflict-free same-offset accesses
};

// The column's least-squares solve once S (= A(I, J), column-major at stride NI in W) and e are
// staged: optional column equilibration, thin_qr, y = Q^T e, back-substitution; m written to out.
// EX: the column fills the envelope exactly (|I| = NI, |J| = NJ -- every interior column of the
// Hermite operators), so every loop has a compile-time trip count and unrolls without per-entry
// guards; otherwise the same operations with run-time bounds.  False: rank deficiency.
template <int NJ, int NI, bool CS, bool EX>
__device__ __forceinline__ bool ls_lane_solve(double *W, double *diag, double *tau, double *mv, double *dsc,
                                              const double (&e)[NI], int ni_rt, int nj_rt, double *out)
{
  const int ni = EX ? NI : ni_rt;
  const int nj = EX ? NJ : nj_rt;
  if (CS) // column equilibration: r_c = 1 / ||S_c|| (in-order dot), S_c *= r_c (oracle.c orc_spai_ls)
  {
    #pragma unroll(EX ? NJ : 1)
    for (int c = 0; c < nj; ++c)
    {
      double *col = W + c * NI;
      const double d = sqrt(dot_serial(col, col, ni));
      if (d == 0.0)
        return false;
      const double r = 1.0 / d;
      dsc[c] = r;
      #pragma unroll(EX ? NI : 1)
      for (int i = 0; i < ni; ++i)
        col[i] = __dmul_rn(col[i], r);
    }
  }
  // ---- thin_qr (dense.cpp:153-246): frob_norm tolerance in column-major order
  double acc = 0.0;
  #pragma unroll(EX ? NJ : 1)
  for (int c = 0; c < nj; ++c)
    #pragma unroll(EX ? NI : 1)
    for (int i = 0; i < ni; ++i)
      acc = __dadd_rn(acc, __dmul_rn(W[c * NI + i], W[c * NI + i]));
  const double anorm = sqrt(acc);
  const double tol = 1e-12 * (anorm > 0.0 ? anorm : 1.0);
  // Householder steps.  The reflector x (column k below the diagonal) is held in registers for
  // the whole trailing update, and the trailing columns are updated two at a time (two
  // independent in-order dot chains, one shared-memory read of x per step): per column the
  // operations and their order are exactly thin_qr's (dense.cpp:168-188).  A flushed column
  // (sigma <= tol) makes the problem rank-deficient, which is an error whatever follows, so the
  // lane stops there.
  #pragma unroll(EX ? NJ : 1)
  for (int k = 0; k < nj; ++k)
  {
    const int len = ni - k;
    double *xs = W + k * NI + k;
    double x[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i)
      x[i] = i < len ? xs[i] : 0.0;
    double acc2 = 0.0;
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (i < len)
        acc2 = __dadd_rn(acc2, __dmul_rn(x[i], x[i]));
    const double sigma = sqrt(acc2);
    if (sigma <= tol)
      return false; // rank < |J|
    const double alpha = x[0] >= 0.0 ? -sigma : sigma;
    x[0] = __dsub_rn(x[0], alpha);
    xs[0] = x[0];
    double vtv = 0.0;
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (i < len)
        vtv = __dadd_rn(vtv, __dmul_rn(x[i], x[i]));
    const double tk = vtv > 0.0 ? 2.0 / vtv : 0.0;
    tau[k] = tk;
    diag[k] = alpha;
    if (tk == 0.0)
      continue;
    int c = k + 1;
    #pragma unroll(EX ? NJ : 1)
    for (; c + 1 < nj; c += 2)
    {
      double *ya = W + c * NI + k, *yb = ya + NI;
      double y0[NI], y1[NI];
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int i = 0; i < NI; ++i)
        if (i < len)
        {
          y0[i] = ya[i];
          y1[i] = yb[i];
          a0 = __dadd_rn(a0, __dmul_rn(x[i], y0[i]));
          a1 = __dadd_rn(a1, __dmul_rn(x[i], y1[i]));
        }
      const double s0 = -__dmul_rn(tk, a0), s1 = -__dmul_rn(tk, a1);
#pragma unroll
      for (int i = 0; i < NI; ++i)
        if (i < len)
        {
          ya[i] = __dadd_rn(y0[i], __dmul_rn(s0, x[i]));
          yb[i] = __dadd_rn(y1[i], __dmul_rn(s1, x[i]));
        }
    }
    if (c < nj)
    {
      double *ya = W + c * NI + k;
      double y0[NI];
      double a0 = 0.0;
#pragma unroll
      for (int i = 0; i < NI; ++i)
        if (i < len)
        {
          y0[i] = ya[i];
          a0 = __dadd_rn(a0, __dmul_rn(x[i], y0[i]));
        }
      const double s0 = -__dmul_rn(tk, a0);
#pragma unroll
      for (int i = 0; i < NI; ++i)
        if (i < len)
          ya[i] = __dadd_rn(y0[i], __dmul_rn(s0, x[i]));
    }
  }
  // ---- y_c = (sign-fixed column c of Q = H_0 ... H_{nj-1} e_c)^T e.  Columns c and c + 1 are
  // formed together in registers: q1 takes reflector c + 1 alone, then both take c .. 0, so each
  // column sees thin_qr's reflector sequence (dense.cpp:200-218) and every reflector is read
  // from shared memory once per pair.
  #pragma unroll(EX ? NJ : 1)
  for (int c = 0; c < nj; c += 2)
  {
    const bool two = c + 1 < nj;
    double q0[NI], q1[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i)
    {
      q0[i] = i == c ? 1.0 : 0.0;
      q1[i] = i == c + 1 ? 1.0 : 0.0;
    }
#pragma unroll
    for (int k = NJ - 1; k >= 0; --k)
    {
      if (k > c + 1 || (k == c + 1 && !two))
        continue;
      const double tk = tau[k];
      if (tk == 0.0)
        continue;
      const double *vs = W + k * NI + k;
      const int len = ni - k;
      double v[NI];
#pragma unroll
      for (int i = 0; i + k < NI; ++i)
        v[i] = i < len ? vs[i] : 0.0;
      if (k == c + 1) // q1 only
      {
        double a1 = 0.0;
#pragma unroll
        for (int i = 0; i + k < NI; ++i)
          if (i < len)
            a1 = __dadd_rn(a1, __dmul_rn(v[i], q1[k + i]));
        const double s1 = -__dmul_rn(tk, a1);
#pragma unroll
        for (int i = 0; i + k < NI; ++i)
          if (i < len)
            q1[k + i] = __dadd_rn(q1[k + i], __dmul_rn(s1, v[i]));
        continue;
      }
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int i = 0; i + k < NI; ++i)
        if (i < len)
        {
          a0 = __dadd_rn(a0, __dmul_rn(v[i], q0[k + i]));
          a1 = __dadd_rn(a1, __dmul_rn(v[i], q1[k + i]));
        }
      const double s0 = -__dmul_rn(tk, a0), s1 = -__dmul_rn(tk, a1);
#pragma unroll
      for (int i = 0; i + k < NI; ++i)
        if (i < len)
        {
          q0[k + i] = __dadd_rn(q0[k + i], __dmul_rn(s0, v[i]));
          if (two)
            q1[k + i] = __dadd_rn(q1[k + i], __dmul_rn(s1, v[i]));
        }
    }
    if (diag[c] < 0.0)
    {
#pragma unroll
      for (int i = 0; i < NI; ++i)
        q0[i] = __dmul_rn(q0[i], -1.0);
    }
    if (two && diag[c + 1] < 0.0)
    {
#pragma unroll
      for (int i = 0; i < NI; ++i)
        q1[i] = __dmul_rn(q1[i], -1.0);
    }
    double y0 = 0.0, y1 = 0.0;
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (i < ni)
      {
        y0 = __dadd_rn(y0, __dmul_rn(q0[i], e[i]));
        y1 = __dadd_rn(y1, __dmul_rn(q1[i], e[i]));
      }
    mv[c] = y0;
    if (two)
      mv[c + 1] = y1;
  }
  // ---- sign fix of R's off-diagonal rows (R(k, c) = W[c][k], c > k), |R_cc|
  #pragma unroll(EX ? NJ : 1)
  for (int c = 0; c < nj; ++c)
  {
    for (int k = 0; k < c; ++k)
      if (diag[k] < 0.0)
        W[c * NI + k] = -W[c * NI + k];
    tau[c] = diag[c] < 0.0 ? -diag[c] : diag[c];
  }
  // ---- back-substitution R m = y (acc = y_k; acc -= R_kq m_q, q ascending)
  #pragma unroll(EX ? NJ : 1)
  for (int k = nj - 1; k >= 0; --k)
  {
    double a = mv[k];
    #pragma unroll(EX ? NJ : 1)
    for (int c = k + 1; c < nj; ++c)
      a = __dsub_rn(a, __dmul_rn(W[c * NI + k], mv[c]));
    mv[k] = a / tau[k];
  }
#pragma unroll(EX ? NJ : 1)
  #pragma unroll(EX ? NJ : 1)
  for (int c = 0; c < nj; ++c)
    out[c] = CS ? __dmul_rn(mv[c], dsc[c]) : mv[c];
  return true;
}

template <int NJ, int NI, bool CS>
__global__ void __launch_bounds__(64) ls_columns_lane(int64_t n, int l, DCsr pat, DCsr At, int64_t at_stride,
                                                       DCsr Kot, int64_t ko_stride, bool update,
                                                       double *__restrict__ out_base, int64_t out_stride,
                                                       unsigned long long *__restrict__ err, int *__restrict__ overflow)
{
  using L = LaneLayout<NJ, NI, CS>;
  extern __shared__ __align__(16) double lane_raw[];
  double *base = lane_raw + static_cast<size_t>(threadIdx.x) * L::kWords;
  double *W = base + L::kW;
  double *diag = base + L::kDiag, *tau = base + L::kTau, *mv = base + L::kM, *dsc = base + L::kDsc;
  int32_t *I = reinterpret_cast<int32_t *>(base + L::kI);
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= static_cast<int64_t>(l) * n)
    return;
  const int p = static_cast<int>(g / n);
  const int64_t j = g - static_cast<int64_t>(p) * n;
  const double *atv = At.v + p * at_stride;
  const double *kov = update ? Kot.v + p * ko_stride : nullptr;
  double *out_vals = out_base + p * out_stride;
  const int64_t jb = pat.rp[j];
  const int nj = static_cast<int>(pat.rp[j + 1] - jb);
  if (nj == 0)
    return;
  if (nj > NJ)
  {
    atomicOr(overflow, 1);
    return;
  }
  // ---- I = sorted union of the rows of A(:, J)
  // Banded operators: the rows of the |J| neighbouring columns fill ONE contiguous range
  // [rmin, rmax] (checked with a bit per row), so I is that range and a row's position is
  // row - rmin -- no insertion, no search.  Same set, same order as the general path below
  // (the index work was ~40% of this kernel's stall samples on the A^2 pattern).
  int ni = 0;
  int32_t rmin = INT_MAX, rmax = -1;
  for (int c = 0; c < nj; ++c)
  {
    const int32_t k = pat.ci[jb + c];
    const int64_t t1 = At.rp[k + 1];
    for (int64_t t = At.rp[k]; t < t1; ++t)
    {
      const int32_t row = At.ci[t];
      rmin = min(rmin, row);
      rmax = max(rmax, row);
    }
  }
  static_assert(NI <= 32, "one bit per row of the range");
  bool contiguous = false;
  if (rmax >= rmin && rmax - rmin < NI)
  {
    const int len = rmax - rmin + 1;
    unsigned mask = 0; // NI <= 32
    for (int c = 0; c < nj; ++c)
    {
      const int32_t k = pat.ci[jb + c];
      const int64_t t1 = At.rp[k + 1];
      for (int64_t t = At.rp[k]; t < t1; ++t)
        mask |= 1u << (At.ci[t] - rmin);
    }
    if (mask == (len == 32 ? 0xffffffffu : (1u << len) - 1u))
    {
      contiguous = true;
      ni = len;
      for (int i = 0; i < len; ++i)
        I[i] = rmin + i;
    }
  }
  if (!contiguous)
  {
    // general: insertion, duplicates skipped
    for (int c = 0; c < nj; ++c)
    {
      const int32_t k = pat.ci[jb + c];
      const int64_t t1 = At.rp[k + 1];
      for (int64_t t = At.rp[k]; t < t1; ++t)
      {
        const int32_t row = At.ci[t];
        int pos = ni;
        while (pos > 0 && I[pos - 1] > row)
          --pos;
        if (pos > 0 && I[pos - 1] == row)
          continue;
        if (ni == NI)
        {
          atomicOr(overflow, 1);
          return;
        }
        for (int u = ni; u > pos; --u)
          I[u] = I[u - 1];
        I[pos] = row;
        ++ni;
      }
    }
  }
  if (ni < nj)
  {
    report(err, g, MGPU_ERR_NUMERICAL);
    return;
  }
  // lower bound of `row` in I
  auto find = [&](int32_t row) {
    if (contiguous)
      return row <= rmin ? 0 : (row - rmin < ni ? static_cast<int>(row - rmin) : ni);
    int lo = 0, hi = ni;
    while (lo < hi)
    {
      const int mid = (lo + hi) >> 1;
      if (I[mid] < row)
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  };
  // ---- S = A(I, J), column-major
  for (int c = 0; c < nj; ++c)
  {
    double *col = W + c * NI;
    for (int i = 0; i < ni; ++i)
      col[i] = 0.0;
    const int32_t k = pat.ci[jb + c];
    const int64_t t1 = At.rp[k + 1];
    for (int64_t t = At.rp[k]; t < t1; ++t)
      col[find(At.ci[t])] = atv[t];
  }
  // ---- e = rhs restricted to I (registers)
  double e[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i)
    e[i] = 0.0;
  if (update)
  {
    for (int64_t t = Kot.rp[j]; t < Kot.rp[j + 1]; ++t)
    {
      const int32_t row = Kot.ci[t];
      const int lo = find(row);
      if (lo < ni && I[lo] == row)
      {
        const double v = kov[t];
#pragma unroll
        for (int i = 0; i < NI; ++i)
          if (i == lo)
            e[i] = v;
      }
    }
  }
  else
  {
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (i < ni && I[i] == j)
        e[i] = 1.0;
  }
  const bool solved = (ni == NI && nj == NJ)
                          ? ls_lane_solve<NJ, NI, CS, true>(W, diag, tau, mv, dsc, e, ni, nj, out_vals + jb)
                          : ls_lane_solve<NJ, NI, CS, false>(W, diag, tau, mv, dsc, e, ni, nj, out_vals + jb);
  if (!solved)
    report(err, g, MGPU_ERR_NUMERICAL);
}

// TPB: threads per block (32 packs the per-lane scratch more tightly for small envelopes)
template <int NJ, int NI, bool CS, int TPB>
void launch_ls_lane_cs(mgpu_ctx *ctx, int64_t n, int l, DCsr pat, DCsr At, int64_t at_stride, DCsr Kot,
                       int64_t ko_stride, bool update, double *out, int64_t out_stride, unsigned long long *err,
                       int *ovf)
{
  constexpr int kThreadsPerBlock = TPB;
  constexpr size_t smem = sizeof(double) * LaneLayout<NJ, NI, CS>::kWords * kThreadsPerBlock;
  static_assert(smem <= 200 * 1024, "LS lane shared memory");
  MG_CUDA(cudaFuncSetAttribute(ls_columns_lane<NJ, NI, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  const int64_t cols = static_cast<int64_t>(l) * n;
  const unsigned grid = static_cast<unsigned>((cols + kThreadsPerBlock - 1) / kThreadsPerBlock);
  ls_columns_lane<NJ, NI, CS><<<grid, kThreadsPerBlock, smem, ctx->stream>>>(n, l, pat, At, at_stride, Kot, ko_stride,
                                                                             update, out, out_stride, err, ovf);
  check_launch(ctx, "ls_columns_lane");
}

template <int NJ, int NI, int TPB = 64>
void launch_ls_lane(mgpu_ctx *ctx, bool cs, int64_t n, int l, DCsr pat, DCsr At, int64_t at_stride, DCsr Kot,
                    int64_t ko_stride, bool update, double *out, int64_t out_stride, unsigned long long *err, int *ovf)
{
  if (cs)
    launch_ls_lane_cs<NJ, NI, true, TPB>(ctx, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, err,
                                         ovf);
  else
    launch_ls_lane_cs<NJ, NI, false, TPB>(ctx, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, err,
                                          ovf);
}

template <int G, int NI, int WARPS, bool CS>
void launch_ls_cs(mgpu_ctx *ctx, int64_t n, int l, DCsr pat, DCsr At, int64_t at_stride, DCsr Kot, int64_t ko_stride,
                  bool update, double *out, int64_t out_stride, unsigned long long *err, int *ovf)
{
  constexpr int per_block = WARPS * (32 / G);
  constexpr size_t smem = sizeof(LsGroupSmem<G, NI>) * per_block;
  static_assert(smem <= 100 * 1024, "LS group shared memory");
  MG_CUDA(cudaFuncSetAttribute(ls_columns<G, NI, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  const int64_t cols = static_cast<int64_t>(l) * n;
  const unsigned grid = static_cast<unsigned>((cols + per_block - 1) / per_block);
  ls_columns<G, NI, CS><<<grid, WARPS * 32, smem, ctx->stream>>>(n, l, pat, At, at_stride, Kot, ko_stride, update,
                                                                 out, out_stride, err, ovf);
  check_launch(ctx, "ls_columns");
}

template <int G, int NI, int WARPS>
void launch_ls(mgpu_ctx *ctx, bool cs, int64_t n, int l, DCsr pat, DCsr At, int64_t at_stride, DCsr Kot,
               int64_t ko_stride, bool update, double *out, int64_t out_stride, unsigned long long *err, int *ovf)
{
  if (cs)
    launch_ls_cs<G, NI, WARPS, true>(ctx, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, err, ovf);
  else
    launch_ls_cs<G, NI, WARPS, false>(ctx, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, err,
                                      ovf);
}

// Runs the LS columns with the smallest lane-group envelope that holds every
// column; throws the lowest failing (point, column) like the reference's
// sequential column loop would.
// abort_dev (optional): a device flag read with the status; nonzero means the batch's shared-
// pattern assumption was wrong, and run_ls returns false without interpreting the results.
bool run_ls(mgpu_ctx *ctx, bool cs, int64_t n, int l, int maxrow, DCsr pat, DCsr At, int64_t at_stride, DCsr Kot,
            int64_t ko_stride, bool update, double *out, int64_t out_stride, const int *extra_dev = nullptr,
            int *extra_host = nullptr, int64_t pat_bw = -1, const int *abort_dev = nullptr,
            const std::function<void()> &after_launch = {})
{
  if (n == 0 || l == 0)
    return true;
  DBuf err(sizeof(unsigned long long), ctx->stream), ovf(sizeof(int), ctx->stream);
  // lane-per-column envelopes first (|J| <= 5 / 6 / 8 pattern entries, |I| <= 13 / 14 / 16 rows),
  // then the lane-group kernels; MGPU_OPT_LS_GROUP skips the lane kernels (diagnostics).  The
  // <5, 13> envelope is taken only when it cannot overflow: a J pattern of bandwidth b gives
  // |I| <= 4 b + 1 (b = 3 on the Hermite beam: 13 rows).
  const bool lanes = ctx->opt[MGPU_OPT_LS_GROUP] == 0;
  // envelopes, tried in order: lane kernels <NJ, NI> (cfg < 0), then lane groups of 8 / 16 / 32
  struct Env
  {
    int nj;
    bool lane;
  };
  // <5, 10> is the exact Hermite A-pattern problem (every interior column: |I| = 10, |J| = 5), which
  // takes ls_lane_solve's fully unrolled path; a column with more rows overflows it and the batch
  // reruns on <5, 13>.  <10, 14> is the exact A^2-pattern problem.
  static constexpr Env kEnv[] = {{5, true}, {5, true}, {6, true}, {8, true}, {10, true}, {10, true}, {8, false},
                                 {16, false}, {32, false}};
  for (int cfg = 0; cfg < 9; ++cfg)
  {
    const int G = kEnv[cfg].nj;
    if (maxrow > G || (kEnv[cfg].lane && !lanes))
      continue;
    if (cfg == 1 && !(pat_bw >= 0 && 4 * pat_bw + 1 <= 13))
      continue;
    MG_CUDA(cudaMemsetAsync(err.ptr, 0xff, sizeof(unsigned long long), ctx->stream));
    MG_CUDA(cudaMemsetAsync(ovf.ptr, 0, sizeof(int), ctx->stream));
    auto *ev = err.as<unsigned long long>();
    switch (cfg)
    {
    case 0:
      launch_ls_lane<5, 10, 32>(ctx, cs, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, ev,
                                ovf.as<int>());
      break;
    case 1:
      launch_ls_lane<5, 13, 32>(ctx, cs, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, ev,
                                ovf.as<int>());
      break;
    case 2:
      launch_ls_lane<6, 14>(ctx, cs, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, ev,
                            ovf.as<int>());
      break;
    case 3:
      launch_ls_lane<8, 16>(ctx, cs, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, ev,
                            ovf.as<int>());
      break;
    case 4: // the A^2 pattern of the Hermite beam: |J| = 10, |I| = 14
      launch_ls_lane<10, 14, 32>(ctx, cs, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, ev,
                                 ovf.as<int>());
      break;
    case 5:
      launch_ls_lane<10, 18, 32>(ctx, cs, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, ev,
                                 ovf.as<int>());
      break;
    case 6:
      launch_ls<8, 16, 4>(ctx, cs, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, ev,
                          ovf.as<int>());
      break;
    case 7:
      launch_ls<16, 32, 2>(ctx, cs, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, ev,
                           ovf.as<int>());
      break;
    default:
      launch_ls<32, 64, 1>(ctx, cs, n, l, pat, At, at_stride, Kot, ko_stride, update, out, out_stride, ev,
                           ovf.as<int>());
    }
    if (after_launch) // caller's dependent work, queued behind the LS kernel before the read-back
      after_launch();
    // one synchronisation returns the error key, the overflow flag and the caller's extra value
    auto *hp = static_cast<unsigned long long *>(pinned_scratch(ctx, 4 * sizeof(unsigned long long)));
    MG_CUDA(cudaMemcpyAsync(hp, err.ptr, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    MG_CUDA(cudaMemcpyAsync(hp + 1, ovf.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (extra_dev)
      MG_CUDA(cudaMemcpyAsync(hp + 2, extra_dev, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (abort_dev)
      MG_CUDA(cudaMemcpyAsync(hp + 3, abort_dev, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    MG_CUDA(cudaStreamSynchronize(ctx->stream));
    const unsigned long long h = hp[0];
    int h_ovf = 0, h_abort = 0;
    std::memcpy(&h_ovf, hp + 1, sizeof(int));
    if (extra_dev)
      std::memcpy(extra_host, hp + 2, sizeof(int));
    if (abort_dev)
      std::memcpy(&h_abort, hp + 3, sizeof(int));
    if (h_abort)
      return false;
    if (h_ovf)
      continue; // a column exceeded this envelope: rerun everything with the next one
    if (h == ULLONG_MAX)
      return true;
    const int64_t g = static_cast<int64_t>(h >> 8);
    const int64_t col = g % n, pt = g / n;
    throw Error(MGPU_ERR_NUMERICAL, "spai_ls: rank-deficient least-squares problem in column " + std::to_string(col),
                col, -1, pt);
  }
  throw Error(MGPU_ERR_UNSUPPORTED,
              "spai_ls: a column exceeds the device envelope (|J| <= 32 pattern entries, |I| <= 64 rows)");
}

struct PatternPtrs
{
  const int64_t *rp[64];
  const int32_t *ci[64];
};

__global__ void pattern_diff(int l, int64_t n, int64_t nnz, PatternPtrs a, const int64_t *rp0, const int32_t *ci0,
                             int *diff)
{
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int p = 0; p < l; ++p)
  {
    if (k <= n && a.rp[p][k] != rp0[k])
      atomicOr(diff, 1);
    if (k < nnz && a.ci[p][k] != ci0[k])
      atomicOr(diff, 1);
  }
}

} // namespace

// True when every matrix in mats (up to 64) has exactly ref's CSR pattern.
bool same_pattern(mgpu_ctx *ctx, int l, const mgpu_csr *const *mats, const mgpu_csr *ref)
{
  if (l > 64)
    return false;
  PatternPtrs pp{};
  for (int p = 0; p < l; ++p)
  {
    if (mats[p]->nrows != ref->nrows || mats[p]->ncols != ref->ncols || mats[p]->nnz != ref->nnz)
      return false;
    pp.rp[p] = mats[p]->row_ptr;
    pp.ci[p] = mats[p]->col_idx;
  }
  DBuf diff(sizeof(int), ctx->stream);
  MG_CUDA(cudaMemsetAsync(diff.ptr, 0, sizeof(int), ctx->stream));
  const int64_t span = std::max<int64_t>(ref->nrows + 1, ref->nnz);
  pattern_diff<<<blocks_for(span), kThreads, 0, ctx->stream>>>(l, ref->nrows, ref->nnz, pp, ref->row_ptr, ref->col_idx,
                                                               diff.as<int>());
  check_launch(ctx, "pattern_diff");
  int h = 0;
  MG_CUDA(cudaMemcpyAsync(&h, diff.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
  return h == 0;
}

// Queues the structure comparison of mats[] against ref, OR-ing a mismatch into *diff_dev; false
// when the host-side sizes already differ (nothing queued: the patterns differ).
bool queue_pattern_diff(mgpu_ctx *ctx, int l, const mgpu_csr *const *mats, const mgpu_csr *ref, int *diff_dev)
{
  if (l > 64)
    return false;
  PatternPtrs pp{};
  for (int p = 0; p < l; ++p)
  {
    if (mats[p]->nrows != ref->nrows || mats[p]->ncols != ref->ncols || mats[p]->nnz != ref->nnz)
      return false;
    pp.rp[p] = mats[p]->row_ptr;
    pp.ci[p] = mats[p]->col_idx;
  }
  const int64_t span = std::max<int64_t>(ref->nrows + 1, ref->nnz);
  pattern_diff<<<blocks_for(span), kThreads, 0, ctx->stream>>>(l, ref->nrows, ref->nnz, pp, ref->row_ptr, ref->col_idx,
                                                               diff_dev);
  check_launch(ctx, "pattern_diff");
  return true;
}

// Symbolic pattern of A*A (values = 1.0 placeholders).
mgpu_csr *pattern_square(mgpu_ctx *ctx, const mgpu_csr *A)
{
  const int64_t n = A->nrows;
  mgpu_csr *S = new mgpu_csr;
  S->ctx = ctx;
  S->nrows = n;
  S->ncols = A->ncols;
  MG_CUDA(mg_malloc(reinterpret_cast<void **>(&S->row_ptr), sizeof(int64_t) * (n + 1), ctx->stream));
  DBuf ovf(sizeof(int), ctx->stream);
  MG_CUDA(cudaMemsetAsync(ovf.ptr, 0, sizeof(int), ctx->stream));
  MG_CUDA(cudaMemsetAsync(S->row_ptr, 0, sizeof(int64_t), ctx->stream));
  if (n > 0)
  {
    square_count<<<blocks_for(n), kThreads, 0, ctx->stream>>>(n, A->view(), S->row_ptr, ovf.as<int>());
    check_launch(ctx, "square_count");
    size_t tmp = 0;
    MG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, S->row_ptr + 1, S->row_ptr + 1, n, ctx->stream));
    DBuf t(tmp, ctx->stream);
    MG_CUDA(cub::DeviceScan::InclusiveSum(t.ptr, tmp, S->row_ptr + 1, S->row_ptr + 1, n, ctx->stream));
    count_launch(ctx);
  }
  int h_ovf = 0;
  int64_t nnz = 0;
  MG_CUDA(cudaMemcpyAsync(&h_ovf, ovf.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA(cudaMemcpyAsync(&nnz, S->row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_ovf)
  {
    mgpu_csr_free(S);
    throw Error(MGPU_ERR_UNSUPPORTED, "spai_ls: A*A pattern row longer than 128 entries");
  }
  S->nnz = nnz;
  MG_CUDA(mg_malloc(reinterpret_cast<void **>(&S->col_idx), sizeof(int32_t) * (nnz > 0 ? nnz : 1), ctx->stream));
  MG_CUDA(mg_malloc(reinterpret_cast<void **>(&S->values), sizeof(double) * (nnz > 0 ? nnz : 1), ctx->stream));
  if (n > 0)
  {
    square_fill<<<blocks_for(n), kThreads, 0, ctx->stream>>>(n, A->view(), S->row_ptr, S->col_idx);
    check_launch(ctx, "square_fill");
  }
  return S;
}

// P (or Q) for one operator.  `pat` may be A itself (pattern 0).
mgpu_csr *spai_ls_one(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *K_old, int pattern)
{
  const bool cs = (pattern & MGPU_LS_COLSCALE) != 0;
  pattern &= ~MGPU_LS_COLSCALE;
  MG_ARG(A->nrows == A->ncols, "spai_ls: operands must be square with equal shape");
  MG_ARG(!K_old || (K_old->nrows == A->nrows && K_old->ncols == A->ncols),
         "spai_ls: operands must be square with equal shape");
  MG_ARG(pattern == MGPU_PATTERN_A || pattern == MGPU_PATTERN_A2, "spai_ls: unknown pattern");
  const int64_t n = A->nrows;
  mgpu_csr *sq = pattern == MGPU_PATTERN_A2 ? pattern_square(ctx, A) : nullptr;
  const mgpu_csr *pat = sq ? sq : A;
  mgpu_csr *At = transpose_csr(ctx, A);
  mgpu_csr *Kot = K_old ? transpose_csr(ctx, K_old) : nullptr;
  // P^T on the J pattern: row j of PT = column j of P
  mgpu_csr *PT = new_csr(ctx, n, n, pat->nnz);
  MG_CUDA(cudaMemcpyAsync(PT->row_ptr, pat->row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, ctx->stream));
  if (pat->nnz > 0)
  {
    MG_CUDA(cudaMemcpyAsync(PT->col_idx, pat->col_idx, sizeof(int32_t) * pat->nnz, cudaMemcpyDeviceToDevice,
                            ctx->stream));
    MG_CUDA(cudaMemsetAsync(PT->values, 0, sizeof(double) * pat->nnz, ctx->stream));
  }
  try
  {
    const int maxrow = static_cast<int>(csr_max_row(ctx, const_cast<mgpu_csr *>(pat)));
    const DCsr kv = Kot ? Kot->view() : DCsr{nullptr, nullptr, nullptr};
    const int64_t bwA = csr_bandwidth(ctx, const_cast<mgpu_csr *>(A));
    run_ls(ctx, cs, n, 1, maxrow, pat->view(), At->view(), 0, kv, 0, Kot != nullptr, PT->values, 0, nullptr, nullptr,
           sq ? 2 * bwA : bwA);
  }
  catch (...)
  {
    mgpu_csr_free(PT);
    mgpu_csr_free(At);
    mgpu_csr_free(Kot);
    mgpu_csr_free(sq);
    throw;
  }
  mgpu_csr *P = transpose_csr(ctx, PT);
  P->may_hold_zeros = true;
  {
    const int64_t ba = csr_bandwidth(ctx, const_cast<mgpu_csr *>(A));
    P->bw = pattern == MGPU_PATTERN_A2 ? 2 * ba : ba; // J pattern bound (A*A at most doubles it)
  }
  mgpu_csr_free(PT);
  mgpu_csr_free(At);
  mgpu_csr_free(Kot);
  mgpu_csr_free(sq);
  return P;
}

// LS-SPAI for l operators that share one CSR pattern (the shifted operators
// of one system do): the pattern work -- J pattern, A^T structure and the
// value permutation, P^T -> P permutation -- is done once, the l * n column
// problems run in ONE launch, and each factor is a gather of its values.
// diff_dev (optional): the speculative shared-pattern flag (queue_pattern_diff); when it turns out
// set, everything is released and an empty vector returned (the caller takes the per-operator path).
std::vector<mgpu_csr *> spai_ls_shared(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, const mgpu_csr *const *K_old,
                                       int pattern, const int *diff_dev = nullptr)
{
  const bool cs = (pattern & MGPU_LS_COLSCALE) != 0;
  pattern &= ~MGPU_LS_COLSCALE;
  const mgpu_csr *A0 = A[0];
  const int64_t n = A0->nrows, nnzA = A0->nnz;
  cudaStream_t s = ctx->stream;
  mgpu_csr *sq = pattern == MGPU_PATTERN_A2 ? pattern_square(ctx, A0) : nullptr;
  const mgpu_csr *pat = sq ? sq : A0;
  const int64_t nnzJ = pat->nnz;
  std::vector<mgpu_csr *> out;
  DBuf perm_t, perm_p;
  mgpu_csr *At0 = nullptr, *PT0 = nullptr, *P0 = nullptr;
  try
  {
    At0 = transpose_perm(ctx, A0, perm_t);
    DBuf at_vals(sizeof(double) * static_cast<size_t>(l) * (nnzA > 0 ? nnzA : 1), s);
    DBuf ko_vals(K_old ? sizeof(double) * static_cast<size_t>(l) * (nnzA > 0 ? nnzA : 1) : 8, s);
    {
      std::vector<const double *> src(static_cast<size_t>(l)), srck(static_cast<size_t>(l));
      std::vector<double *> dst(static_cast<size_t>(l)), dstk(static_cast<size_t>(l));
      for (int p = 0; p < l; ++p)
      {
        src[p] = A[p]->values;
        dst[p] = at_vals.as<double>() + p * nnzA;
        if (K_old)
        {
          srck[p] = K_old[p]->values;
          dstk[p] = ko_vals.as<double>() + p * nnzA;
        }
      }
      gather_batched(ctx, l, nnzA, perm_t.as<int64_t>(), src.data(), dst.data());
      if (K_old)
        gather_batched(ctx, l, nnzA, perm_t.as<int64_t>(), srck.data(), dstk.data());
    }
    DBuf pt_vals(sizeof(double) * static_cast<size_t>(l) * (nnzJ > 0 ? nnzJ : 1), s);
    MG_CUDA(cudaMemsetAsync(pt_vals.ptr, 0, sizeof(double) * static_cast<size_t>(l) * nnzJ, s));
    const int maxrow = static_cast<int>(csr_max_row(ctx, const_cast<mgpu_csr *>(pat)));
    DCsr atv{At0->row_ptr, At0->col_idx, at_vals.as<double>()};
    DCsr kov{At0->row_ptr, At0->col_idx, ko_vals.as<double>()};
    // On A's pattern the factors take At0's structure: its longest row rides along with the
    // LS kernel's status read instead of costing a synchronisation of its own
    DBuf mx(sizeof(int), s);
    int at_maxrow = -1;
    if (!sq && At0->maxrow < 0 && n > 0)
    {
      MG_CUDA(cudaMemsetAsync(mx.ptr, 0, sizeof(int), s));
      ls_max_row<<<blocks_for(n), kThreads, 0, s>>>(n, At0->row_ptr, mx.as<int>());
      check_launch(ctx, "ls_max_row");
    }
    const bool fetch = !sq && At0->maxrow < 0 && n > 0;
    // J pattern bandwidth: A's, doubled for the symbolic A^2
    const int64_t bwA = csr_bandwidth(ctx, const_cast<mgpu_csr *>(A0));
    // P^T (J pattern) -> P: one structure and one permutation for every factor.  On A's
    // pattern P^T has A0's CSR structure, so P has At0's and the values follow perm_t: the
    // factors are made and their value gather queued behind the LS kernel, before its status
    // read-back.  On A^2's the J pattern is transposed once, after the LS solve.
    const int64_t ba = csr_bandwidth(ctx, const_cast<mgpu_csr *>(A0));
    std::vector<const double *> gsrc;
    std::vector<double *> gdst;
    mgpu_ctx *owner_ctx = ctx;
    auto make_factors = [&](mgpu_csr *S, int64_t pmax) {
      // hand S's structure to the factors (shared, freed by the last one)
      int64_t *srp = S->row_ptr;
      int32_t *sci = S->col_idx;
      std::shared_ptr<void> structure(srp, [owner_ctx, sci](void *rp) {
        cudaFreeAsync(rp, owner_ctx->stream);
        cudaFreeAsync(sci, owner_ctx->stream);
      });
      S->row_ptr = nullptr;
      S->col_idx = nullptr;
      // every factor's values in one allocation (slices), released with the last factor
      double *vblock = nullptr;
      MG_CUDA(mg_malloc(reinterpret_cast<void **>(&vblock),
                        sizeof(double) * static_cast<size_t>(l) * (nnzJ > 0 ? nnzJ : 1), s));
      std::shared_ptr<void> values(vblock, [owner_ctx](void *v) { cudaFreeAsync(v, owner_ctx->stream); });
      for (int p = 0; p < l; ++p)
      {
        auto *P = new mgpu_csr;
        P->ctx = ctx;
        P->nrows = n;
        P->ncols = n;
        P->nnz = nnzJ;
        P->row_ptr = srp;
        P->col_idx = sci;
        P->shared_structure = structure;
        out.push_back(P);
        P->values = vblock + static_cast<size_t>(p) * (nnzJ > 0 ? nnzJ : 1);
        P->shared_values = values;
        P->may_hold_zeros = true;
        P->bw = pattern == MGPU_PATTERN_A2 ? 2 * ba : ba;
        P->maxrow = pmax;
        gsrc.push_back(pt_vals.as<double>() + p * nnzJ);
        gdst.push_back(P->values);
      }
    };
    std::function<void()> gather_early;
    if (!sq)
    {
      make_factors(At0, At0->maxrow); // maxrow set below once fetched
      gather_early = [&]() { gather_batched(ctx, l, nnzJ, perm_t.as<int64_t>(), gsrc.data(), gdst.data()); };
    }
    if (!run_ls(ctx, cs, n, l, maxrow, pat->view(), atv, nnzA, kov, nnzA, K_old != nullptr, pt_vals.as<double>(), nnzJ,
                fetch ? mx.as<int>() : nullptr, fetch ? &at_maxrow : nullptr, sq ? 2 * bwA : bwA, diff_dev,
                gather_early))
    {
      for (auto *m : out)
        mgpu_csr_free(m);
      mgpu_csr_free(At0);
      mgpu_csr_free(sq);
      return {};
    }
    if (fetch)
    {
      At0->maxrow = at_maxrow;
      for (auto *P : out)
        P->maxrow = at_maxrow;
    }
    if (sq)
    {
      PT0 = new_csr(ctx, n, n, nnzJ);
      MG_CUDA(cudaMemcpyAsync(PT0->row_ptr, pat->row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
      if (nnzJ > 0)
        MG_CUDA(cudaMemcpyAsync(PT0->col_idx, pat->col_idx, sizeof(int32_t) * nnzJ, cudaMemcpyDeviceToDevice, s));
      P0 = transpose_perm(ctx, PT0, perm_p);
      make_factors(P0, csr_max_row(ctx, P0)); // every factor has P0's stored pattern
      gather_batched(ctx, l, nnzJ, perm_p.as<int64_t>(), gsrc.data(), gdst.data());
    }
    host_mark("spai_ls_shared: factors made");
  }
  catch (...)
  {
    for (auto *m : out)
      mgpu_csr_free(m);
    mgpu_csr_free(P0);
    mgpu_csr_free(PT0);
    mgpu_csr_free(At0);
    mgpu_csr_free(sq);
    throw;
  }
  mgpu_csr_free(P0); // its structure now belongs to the factors
  mgpu_csr_free(PT0);
  mgpu_csr_free(At0);
  mgpu_csr_free(sq);
  host_mark("spai_ls_shared: return");
  return out;
}

} // namespace mgpu

using namespace mgpu;

extern "C" {

int mgpu_spai_ls(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *K_old, int pattern, mgpu_csr **P)
{
  return guard(ctx, [&] {
    MG_ARG(A && P, "spai_ls: null argument");
    *P = spai_ls_one(ctx, A, K_old, pattern);
  });
}

int mgpu_spai_ls_batched(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, const mgpu_csr *const *K_old, int pattern,
                         mgpu_csr **P)
{
  return guard(ctx, [&] {
    MG_ARG(l >= 0 && A && P, "spai_ls: null argument");
    for (int i = 0; i < l; ++i)
      MG_ARG(A[i] && A[i]->nrows == A[i]->ncols && (!K_old || (K_old[i] && K_old[i]->nrows == A[i]->nrows &&
                                                                   K_old[i]->ncols == A[i]->ncols)),
             "spai_ls: operands must be square with equal shape");
    MG_ARG((pattern & ~MGPU_LS_COLSCALE) == MGPU_PATTERN_A || (pattern & ~MGPU_LS_COLSCALE) == MGPU_PATTERN_A2,
           "spai_ls: unknown pattern");
    // shared-pattern path, speculatively: the structure comparison is queued, not awaited; its
    // flag comes back with the LS status, and on a mismatch the batch reruns per operator
    DBuf diff(sizeof(int), ctx->stream);
    MG_CUDA(cudaMemsetAsync(diff.ptr, 0, sizeof(int), ctx->stream));
    if (l >= 2 && queue_pattern_diff(ctx, l, A, A[0], diff.as<int>()) &&
        (!K_old || queue_pattern_diff(ctx, l, K_old, A[0], diff.as<int>())))
    {
      std::vector<mgpu_csr *> made = spai_ls_shared(ctx, l, A, K_old, pattern, diff.as<int>());
      if (!made.empty())
      {
        for (int i = 0; i < l; ++i)
          P[i] = made[i];
        return;
      }
    }
    std::vector<mgpu_csr *> made;
    try
    {
      for (int i = 0; i < l; ++i)
        made.push_back(spai_ls_one(ctx, A[i], K_old ? K_old[i] : nullptr, pattern));
    }
    catch (Error &e)
    {
      for (auto *m : made)
        mgpu_csr_free(m);
      e.point = static_cast<int64_t>(made.size());
      throw;
    }
    for (int i = 0; i < l; ++i)
      P[i] = made[i];
  });
}

} // extern "C"
