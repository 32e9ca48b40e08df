// Streaming CG kernel (cg_stream) for HBM-resident banded systems and its host side
// (stream_solve).  Split from cg.cu; the control flow, reductions and arithmetic are those of
// cg_banded (krylov.cpp:28-174).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "cg_common.cuh"

namespace cgrp = cooperative_groups;

namespace mgpu
{
namespace
{

// =====================================================================
// Streaming kernel for HBM-resident banded systems (cg_stream).
//   * operators in PADDED ROW-MAJOR ELL: values [row][Epad] (Epad even) and
//     the row's int8 column offsets packed in one u64, PADR zero rows at both
//     ends -> every chunk's operator rows are ONE contiguous, 16B-aligned range
//     (no row_ptr, no column index stream: 8 Epad + 8 bytes per row);
//   * vectors interleaved [point][PADR + row][rhs], PADR zero rows per side;
//   * per phase, each CTA walks its rows in chunks of CH = 512 * RPT rows; the
//     inputs of chunk i+1 are fetched with cp.async.bulk (TMA bulk copies,
//     mbarrier transaction counts) into the other half of a double buffer
//     while the CTA computes chunk i from shared memory -> the copy engine
//     keeps HBM busy independent of warp occupancy.
// Control flow, reductions and arithmetic are those of cg_banded.
// =====================================================================
constexpr int kPadR = 64;
constexpr int kEllMax = 64; // widest ELL row the streaming kernel takes (int8 offsets: bandwidth < kPadR)
constexpr int kStreamNB = 4; // bulk-copy ring depth (maximum; StreamParams::nb is the one in use)
constexpr int kTabSlots = 16; // operator-descriptor slots: segments per block
static_assert(kTabSlots >= kMaxSeg, "descriptor table must cover every segment");

__device__ __forceinline__ uint32_t sm_addr(const void *p)
{
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
  asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra WAIT_%=;\n\t}" ::"r"(sm_addr(bar)),
               "r"(parity)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sm_addr(dst)),
               "l"(src), "r"(bytes), "r"(sm_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_addr(bar)) : "memory");
}
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

struct PEll
{
  const double *v;             // logical row 0 (PADR zero rows before / after)
  const unsigned long long *o; // packed int8 offsets, `ow` words per row
  int E;                       // values per row (even, <= 16)
  int ow;                      // offset words per row: ceil(E / 8) (E <= kEllMax)
};

// eq[p] = 1 iff operator p has point 0's CSR structure (then its ELL offsets equal point 0's,
// and the kernel streams point 0's copy for every such point: one DRAM read, L2 hits for the
// rest, since the points advance through the rows together).  eq must be preset to 1.
__global__ void pattern_eq_kernel(int64_t n, int64_t nnz, const int64_t *__restrict__ rp0,
                                  const int32_t *__restrict__ ci0, const int64_t *__restrict__ rp,
                                  const int32_t *__restrict__ ci, int *eq)
{
  bool same = true;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x)
    same = same && rp[i] == rp0[i];
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz; k += gridDim.x * blockDim.x)
    same = same && ci[k] == ci0[k];
  if (!__all_sync(0xffffffffu, same) && (threadIdx.x & 31) == 0)
    *eq = 0;
}

struct StreamParams
{
  int l, m, z, rpt, ch; // ch: rows per chunk (phase A and the check pass)
  int ch_b;             // rows per chunk in phase B (fewer vectors per row: taller chunks fill the same slot)
  int nb;               // ring depth (2..kStreamNB)
  // stage-buffer layout: 0 = row-interleaved [row][c]; > 0 (m == 4) = two planes of double2,
  // (c0, c1) and (c2, c3) per row, plane stride `pst` doubles.  A thread's row loads are then two
  // 16-byte loads from consecutive 16-byte slots across the warp (no bank conflicts; the
  // interleaved 32-byte rows cost two wavefronts per 16-byte load).
  int pst;
  int s0_double; // 1: two stage-0 buffers (chunk parity), no block-wide barrier at the end of a chunk
  int64_t n, ldv; // ldv = (n + 2 PADR) * m rounded up to even: doubles per point block (16-byte aligned)
  int halo[kMaxZ + 1];
  int hmax;
  const PEll *A, *F; // [l], [l * z] newest first
  const int *eqA;     // [l]: operator p shares point 0's structure (use A[0]'s offsets)
  const int *eqF;     // [l * z]: factor (p, f) shares factor (0, f)'s structure
  double rtol;
  int64_t maxit;
  // vectors: logical (point p, row i, col c) at base + p * ldv + (PADR + i) * m + c
  const double *b;
  double *xt, *r, *dbuf0, *dbuf1, *w, *sol;
  double *partial;
  const Seg *seg;
  const int2 *pblk;
  double *X, *REC, *TR;
  int64_t *iters;
  int *conv, *status;
  int64_t *bd_iter;
  double *hist;
  int64_t hist_cap;
  int64_t *loop_iters;
  long long *prof; // optional [16] clock64 totals per phase (block 0, thread 0; MGPU_PROFILE_PHASES)
  // shared-memory carve-up (bytes): two input buffers (phase A layout and
  // phase B layout alias) + stage buffers
  size_t buf_bytes, off_stage0, off_stage0b, off_stage1, off_stage2; // stage 0 is double-buffered (chunk parity)
  size_t a_vr, a_vd, a_vx, a_fv[kMaxZ], a_fo[kMaxZ], a_av, a_ao; // phase A offsets inside a buffer
  size_t b_r, b_w;                                                // phase B offsets inside a buffer
};

// Per-stage entries of StreamParams, copied to shared memory once: indexing the kernel
// parameters with a run-time stage number makes ptxas keep a local-memory copy of the whole
// parameter block (a 700-byte stack frame; configs[3] 1119 -> 1779 us per iteration when it happened).
struct StageTab
{
  int halo[kMaxZ + 1];
  uint32_t a_fv[kMaxZ], a_fo[kMaxZ];
};

__device__ __forceinline__ const double *vrow(const StreamParams &P, const double *base, int p, int64_t i)
{
  return base + static_cast<int64_t>(p) * P.ldv + (kPadR + i) * P.m;
}

// The block's chunks in order: its segments (one point each, masked points skipped), then
// CH-row chunks of the segment.  fn(segment index, point, c0, c1); the producer and the
// consumers walk the same sequence.  Rows are 32-bit (Seg), the loop carries no 64-bit state.
template <int TB, class F>
__device__ __forceinline__ void for_chunks(const BandShared<TB> &sh, int CH, F &&fn)
{
  for (int sg = 0; sg < sh.nseg; ++sg)
  {
    const Seg g = sh.seg[sg];
    if (!sh.pmask[g.p])
      continue;
    for (int c0 = g.rs; c0 < g.re; c0 += CH)
      fn(sg, g.p, c0, min(g.re, c0 + CH));
  }
}

__device__ __forceinline__ int64_t even_up(int64_t x) { return (x + 1) & ~static_cast<int64_t>(1); }

// Producer: issue the bulk copies of one chunk's inputs into buffer `buf`.
// kind 0: phase A step (r, d_old over the halo; x~ on own rows for the deferred
// update), 1: phase A check (x~ and d_old over the halo), 2: phase B (r, w).
template <int TB>
__device__ __forceinline__ void stream_issue(const StreamParams &P, const StageTab &stg, const PEll *tab, unsigned char *buf,
                             uint64_t *bar, int kind, int p, int64_t c0, int64_t c1, const double *dold)
{
  const int m = P.m;
  if (kind == 2)
  {
    const int64_t rows = even_up(c1 - c0);
    const uint32_t vb = static_cast<uint32_t>(rows * m * 8);
    mbar_expect_tx(bar, 2 * vb);
    bulk_g2s(buf + P.b_r, vrow(P, P.r, p, c0), vb, bar);
    bulk_g2s(buf + P.b_w, vrow(P, P.w, p, c0), vb, bar);
    return;
  }
  const int H0 = P.hmax;
  const int64_t vrows = even_up(c1 - c0 + 2 * H0);
  const uint32_t vb = static_cast<uint32_t>(vrows * m * 8);
  const uint32_t xb = static_cast<uint32_t>(even_up(c1 - c0) * m * 8);
  uint32_t total = 2 * vb + (kind == 0 ? xb : 0u);
  for (int st = 0; st < P.z; ++st)
  {
    const int hd = stg.halo[st + 1];
    const PEll F = tab[1 + st];
    const int64_t rows = even_up(c1 - c0 + 2 * hd);
    total += static_cast<uint32_t>(rows * F.E * 8 + rows * F.ow * 8);
  }
  {
    const PEll A = tab[0];
    const int64_t rows = even_up(c1 - c0);
    total += static_cast<uint32_t>(rows * A.E * 8 + rows * A.ow * 8);
  }
  mbar_expect_tx(bar, total);
  bulk_g2s(buf + P.a_vr, vrow(P, kind == 0 ? P.r : P.xt, p, c0 - H0), vb, bar);
  bulk_g2s(buf + P.a_vd, vrow(P, dold, p, c0 - H0), vb, bar); // the check pass reads d_old for the deferred update
  if (kind == 0)
    bulk_g2s(buf + P.a_vx, vrow(P, P.xt, p, c0), xb, bar);
  for (int st = 0; st < P.z; ++st)
  {
    const int hd = stg.halo[st + 1];
    const PEll F = tab[1 + st];
    const int64_t rows = even_up(c1 - c0 + 2 * hd);
    bulk_g2s(buf + stg.a_fv[st], F.v + (c0 - hd) * F.E, static_cast<uint32_t>(rows * F.E * 8), bar);
    bulk_g2s(buf + stg.a_fo[st], F.o + (c0 - hd) * F.ow, static_cast<uint32_t>(rows * F.ow * 8), bar);
  }
  const PEll A = tab[0];
  const int64_t rows = even_up(c1 - c0);
  bulk_g2s(buf + P.a_av, A.v + c0 * A.E, static_cast<uint32_t>(rows * A.E * 8), bar);
  bulk_g2s(buf + P.a_ao, A.o + c0 * A.ow, static_cast<uint32_t>(rows * A.ow * 8), bar);
}

__device__ __forceinline__ int off8s(unsigned long long w, int t)
{
  return static_cast<int>(static_cast<signed char>((w >> (8 * t)) & 0xffull));
}
__device__ __forceinline__ int off16(unsigned long long w0, unsigned long long w1, int t)
{
  return t < 8 ? off8s(w0, t) : off8s(w1, t - 8);
}
// offset t of a row with ow words (the first two held in registers)
__device__ __forceinline__ int off_any(const unsigned long long *offs, unsigned long long w0, unsigned long long w1,
                                       int t)
{
  return t < 16 ? off16(w0, w1, t) : off8s(offs[t >> 3], t & 7);
}

// Column of element e of a row-interleaved block with m columns (MT: compile-time bound, a power of two).
template <int MT>
__device__ __forceinline__ int col_of(int e, int m)
{
  if constexpr (MT == 1)
    return 0;
  else
    return m == MT ? (e & (MT - 1)) : e % m;
}
// acc[c] += v without dynamic register indexing.
template <int MT>
__device__ __forceinline__ void acc_add(double *acc, int c, double v)
{
#pragma unroll
  for (int k = 0; k < MT; ++k)
    if (k == c)
      acc[k] = __dadd_rn(acc[k], v);
}
// m doubles of one row (shared memory); 16-byte vector loads when m == MT >= 2.
template <int MT>
__device__ __forceinline__ void ld_row(const double *x, double (&v)[MT], int m)
{
  if (MT >= 2 && m == MT)
  {
#pragma unroll
    for (int h = 0; h < MT / 2; ++h)
    {
      const double2 t = reinterpret_cast<const double2 *>(x)[h];
      v[2 * h] = t.x;
      v[2 * h + 1] = t.y;
    }
  }
  else
  {
#pragma unroll
    for (int c = 0; c < MT; ++c)
      v[c] = c < m ? x[c] : 0.0;
  }
}
template <int MT>
__device__ __forceinline__ void st_row(double *x, const double (&v)[MT], int m)
{
  if (MT >= 2 && m == MT)
  {
#pragma unroll
    for (int h = 0; h < MT / 2; ++h)
      reinterpret_cast<double2 *>(x)[h] = make_double2(v[2 * h], v[2 * h + 1]);
  }
  else
  {
#pragma unroll
    for (int c = 0; c < MT; ++c)
      if (c < m)
        x[c] = v[c];
  }
}
// Streaming (L2-only) global store of one row.
template <int MT>
__device__ __forceinline__ void stg_row(double *x, const double (&v)[MT], int m)
{
  if (MT >= 2 && m == MT)
  {
#pragma unroll
    for (int h = 0; h < MT / 2; ++h)
      __stcg(reinterpret_cast<double2 *>(x) + h, make_double2(v[2 * h], v[2 * h + 1]));
  }
  else
  {
#pragma unroll
    for (int c = 0; c < MT; ++c)
      if (c < m)
        __stcg(x + c, v[c]);
  }
}
// One padded-ELL row (E even, values 16-byte aligned) times a row-interleaved
// shared-memory block: a2[c] = sum_e val_e * src[(in0 + off_e) * m + c], e ascending.
template <int MT, bool WIDE = false>
__device__ __forceinline__ void ell_row(const double *vals, const unsigned long long *offs, int E, int ow,
                                        const double *src, int in0, int m, double (&a2)[MT])
{
#pragma unroll
  for (int c = 0; c < MT; ++c)
    a2[c] = 0.0;
  const unsigned long long w0 = offs[0];
  const unsigned long long w1 = ow > 1 ? offs[1] : 0ull;
  const double2 *v2 = reinterpret_cast<const double2 *>(vals);
  // wide rows (collapsed update chains): offsets beyond the first two words read per term.  WIDE is
  // a separate instantiation: in the common kernel this path cost the m = 4 instance its registers
  // (123 -> 128 with the parameters in local memory, configs[3] 1119 -> 1779 us per iteration)
  if (WIDE && ow > 2)
  {
    for (int e = 0; e < E; ++e)
    {
      double x[MT];
      ld_row<MT>(src + (in0 + off_any(offs, w0, w1, e)) * m, x, m);
#pragma unroll
      for (int c = 0; c < MT; ++c)
        if (c < m)
          a2[c] = __dadd_rn(a2[c], __dmul_rn(vals[e], x[c]));
    }
    return;
  }
  auto term = [&](double a, int e) {
    double x[MT];
    ld_row<MT>(src + (in0 + off16(w0, w1, e)) * m, x, m);
#pragma unroll
    for (int c = 0; c < MT; ++c)
      if (c < m)
        a2[c] = __dadd_rn(a2[c], __dmul_rn(a, x[c]));
  };
  // single right-hand side: the Hermite operators and their A-pattern LS factors (5 entries)
  // unrolled with constant shifts (configs[2] shape 31.1 -> 27.6 us per iteration; with m = 4
  // the preloaded values cost registers and it measured 2% slower, so MT > 1 keeps the loop)
  if (MT == 1 && E == 5)
  {
    double a5[5];
#pragma unroll
    for (int e = 0; e < 5; ++e)
      a5[e] = vals[e];
#pragma unroll
    for (int e = 0; e < 5; ++e)
      term(a5[e], e);
    return;
  }
  if (E & 1) // odd width (no padding entry): rows are 8-byte aligned only
  {
    for (int e = 0; e < E; ++e)
      term(vals[e], e);
    return;
  }
  for (int h = 0; h < E / 2; ++h)
  {
    const double2 f = v2[h];
    term(f.x, 2 * h);
    term(f.y, 2 * h + 1);
  }
}

// The same row with the width EC and the column count MT known at compile time (m == MT): the
// offsets are byte extracts at constant positions, the loads vectorised, no per-column guards.
// Same terms in the same order as ell_row (bitwise equal).
template <int MT, int EC, bool PL = false>
__device__ __forceinline__ void ell_row_fixed(const double *vals, const unsigned long long *offs, const double *src,
                                              int in0, double (&a2)[MT], int pst = 0)
{
#pragma unroll
  for (int c = 0; c < MT; ++c)
    a2[c] = 0.0;
  const unsigned long long w0 = offs[0];
  const unsigned long long w1 = EC > 8 ? offs[1] : 0ull;
  // even widths: rows are 16-byte aligned, values read as double2 (a quarter warp's 16-byte
  // loads at the 8 EC-byte row stride hit distinct banks; the 8-byte loads conflicted two-way)
  double av[EC];
  if constexpr ((EC & 1) == 0)
  {
#pragma unroll
    for (int h = 0; h < EC / 2; ++h)
    {
      const double2 t = reinterpret_cast<const double2 *>(vals)[h];
      av[2 * h] = t.x;
      av[2 * h + 1] = t.y;
    }
  }
  else
  {
#pragma unroll
    for (int e = 0; e < EC; ++e)
      av[e] = vals[e];
  }
#pragma unroll
  for (int e = 0; e < EC; ++e)
  {
    const double ae = av[e];
    const int off = e < 8 ? off8s(w0, e) : off8s(w1, e - 8);
    double x[MT];
    if constexpr (PL && MT == 4)
    {
      const double2 t0 = reinterpret_cast<const double2 *>(src)[in0 + off];
      const double2 t1 = reinterpret_cast<const double2 *>(src + pst)[in0 + off];
      x[0] = t0.x;
      x[1] = t0.y;
      x[2] = t1.x;
      x[3] = t1.y;
    }
    else if constexpr (MT >= 2)
    {
#pragma unroll
      for (int h = 0; h < MT / 2; ++h)
      {
        const double2 t = reinterpret_cast<const double2 *>(src + (in0 + off) * MT)[h];
        x[2 * h] = t.x;
        x[2 * h + 1] = t.y;
      }
    }
    else
      x[0] = src[in0 + off];
#pragma unroll
    for (int c = 0; c < MT; ++c)
      a2[c] = __dadd_rn(a2[c], __dmul_rn(ae, x[c]));
  }
}

// Planar (m == 4) row of any width: ell_row's terms in ell_row's order.
template <bool WIDE>
__device__ __forceinline__ void ell_row_planar(const double *vals, const unsigned long long *offs, int E, int ow,
                                               const double *src, int in0, int pst, double (&a2)[4])
{
#pragma unroll
  for (int c = 0; c < 4; ++c)
    a2[c] = 0.0;
  const unsigned long long w0 = offs[0];
  const unsigned long long w1 = ow > 1 ? offs[1] : 0ull;
  for (int e = 0; e < E; ++e)
  {
    const int r = in0 + (WIDE ? off_any(offs, w0, w1, e) : off16(w0, w1, e));
    const double a = vals[e];
    const double2 t0 = reinterpret_cast<const double2 *>(src)[r];
    const double2 t1 = reinterpret_cast<const double2 *>(src + pst)[r];
    a2[0] = __dadd_rn(a2[0], __dmul_rn(a, t0.x));
    a2[1] = __dadd_rn(a2[1], __dmul_rn(a, t0.y));
    a2[2] = __dadd_rn(a2[2], __dmul_rn(a, t1.x));
    a2[3] = __dadd_rn(a2[3], __dmul_rn(a, t1.y));
  }
}

// Stage-buffer row access in the P.pst layout.
template <int MT>
__device__ __forceinline__ void ld_stage(const double *buf, int row, double (&v)[MT], int m, int pst)
{
  if constexpr (MT == 4)
  {
    if (pst > 0)
    {
      const double2 t0 = reinterpret_cast<const double2 *>(buf)[row];
      const double2 t1 = reinterpret_cast<const double2 *>(buf + pst)[row];
      v[0] = t0.x;
      v[1] = t0.y;
      v[2] = t1.x;
      v[3] = t1.y;
      return;
    }
  }
  ld_row<MT>(buf + row * m, v, m);
}
template <int MT>
__device__ __forceinline__ void st_stage(double *buf, int row, const double (&v)[MT], int m, int pst)
{
  if constexpr (MT == 4)
  {
    if (pst > 0)
    {
      reinterpret_cast<double2 *>(buf)[row] = make_double2(v[0], v[1]);
      reinterpret_cast<double2 *>(buf + pst)[row] = make_double2(v[2], v[3]);
      return;
    }
  }
  st_row<MT>(buf + row * m, v, m);
}
// Index of element e (= row * m + c) of a stage buffer.
__device__ __forceinline__ int stage_idx(int e, int m, int pst)
{
  if (pst > 0) // m == 4
    return ((e & 2) ? pst : 0) + ((e >> 2) << 1) + (e & 1);
  return e;
}

// ell_row with the common widths (the Hermite operators: 5; their A^2-pattern factors: 10) and
// m == MT dispatched to ell_row_fixed.
// EF: the width this call site expects (the A^2-pattern factors: 10; the Hermite operators: 5),
// unrolled; any other width takes the loop.  One unrolled width per call site keeps the kernel
// inside its 128 registers (two unrolled widths per site pushed the parameters to local memory).
template <int MT, int EF, bool WIDE>
__device__ __forceinline__ void ell_row_any(const double *vals, const unsigned long long *offs, int E, int ow,
                                            const double *src, int in0, int m, double (&a2)[MT], int pst)
{
  if constexpr (MT == 4)
  {
    if (pst > 0)
    {
      if (E == EF)
        ell_row_fixed<4, EF, true>(vals, offs, src, in0, a2, pst);
      else
        ell_row_planar<WIDE>(vals, offs, E, ow, src, in0, pst, a2);
      return;
    }
  }
  ell_row<MT, WIDE>(vals, offs, E, ow, src, in0, m, a2);
}

// Per-phase clock64 totals (MGPU_PROFILE_PHASES); the ON = false instantiation compiles away.
template <bool ON>
struct PhaseClock
{
  bool on;
  long long t, acc[16];
  __device__ void mark(int k)
  {
    if constexpr (ON)
    {
      if (on)
      {
        const long long now = clock64();
        acc[k] += now - t;
        t = now;
      }
    }
  }
};

// Barrier among the TB consumer threads only (the producer warp streams on).
template <int TB>
__device__ __forceinline__ void consumer_sync()
{
  asm volatile("bar.sync 1, %0;" ::"n"(TB) : "memory");
}

// Producer-side state of the bulk-copy ring (lane 0 of the producer warp).
struct RingProducer
{
  uint32_t filled; // bit b: buffer b has been filled at least once
  uint32_t epar;   // bit b: parity of the next empty-barrier phase to wait for
};

// One pass over the block's chunks.  kind: 0 phase A (step), 1 phase A
// (true-residual check), 2 phase B.  Warp-specialised: lane 0 of warp TB/32
// streams chunk inputs into an NB-deep ring of shared buffers (full barrier:
// bulk-copy bytes; empty barrier: consumers done), the TB consumer threads
// compute.  Dot-product partials accumulate per consumer thread over all
// chunks of a point (row order) and are reduced once per point.
//
// Element loops (stage 0, phase B) run on pairs of doubles when m == MT: pair u holds elements
// 2u, 2u + 1 of the row-interleaved block, i.e. columns (2u) % m and (2u + 1) % m (the same
// column twice for m = 1).  2 TB % m == 0 for every MT, so a thread's two columns are fixed
// and their system scalars are read once per chunk.
// (forceinline: as a real call the pass takes the kernel parameters by address, which costs a
// local-memory copy of the parameter block and turns `kind` into run-time branches)
template <int TB, int MT, int NB, class PC, bool WIDE>
__device__ __forceinline__ void stream_pass(const StreamParams &P, BandShared<TB + 32> &sh, const StageTab &stg, const PEll *tab,
                            unsigned char *smem,
                            uint64_t *full, uint64_t *empty, uint32_t &phase_bits, RingProducer &rp, int kind,
                            const double *dold, double *dnew, PC &pc)
{
  const int CH = kind == 2 ? P.ch_b : P.ch;
  const int m = P.m;
  const int nv = kind == 0 ? 2 * m : m;
  __syncthreads();
  if (threadIdx.x >= TB)
  {
    // ---- producer
    if (threadIdx.x == TB)
    {
      fence_async_global(); // generic stores of the previous phase -> async-proxy (bulk copy) reads
      int b = 0;
      for_chunks(sh, CH, [&](int sg, int pp, int c0, int c1) {
        if ((rp.filled >> b) & 1u)
        {
          mbar_wait(&empty[b], (rp.epar >> b) & 1u);
          rp.epar ^= 1u << b;
        }
        rp.filled |= 1u << b;
        stream_issue<TB>(P, stg, tab + sg * (kMaxZ + 1), smem + b * P.buf_bytes, &full[b], kind, pp, c0, c1, dold);
        b = b + 1 == P.nb ? 0 : b + 1;
      });
    }
    __syncthreads();
    return;
  }
  // ---- consumers
  pc.mark(0);
  double acc[2 * MT];
#pragma unroll
  for (int q = 0; q < 2 * MT; ++q)
    acc[q] = 0.0;
  int bi = 0;
  int step = 0;
  int cur_p = -1;
  const bool full_m = m == MT;
  // pairs: this thread's two columns (fixed, see above); scalar fallback (m < MT): TB % m == 0
  // (every m <= 8 but 7) fixes the column of element e = tid + k TB
  const int cA = (2 * static_cast<int>(threadIdx.x)) % m, cB = (2 * static_cast<int>(threadIdx.x) + 1) % m;
  const bool cfix = (TB % m) == 0;
  const int cth = threadIdx.x % m;
  double accA = 0.0, accB = 0.0; // phase B: (r, r) partials of columns cA, cB (pairs) / accA of cth (scalar)
  auto flush = [&](int pnt) {
    if (kind == 2 && (full_m || cfix))
    {
#pragma unroll
      for (int q = 0; q < MT; ++q)
      {
        double v = 0.0;
        if (full_m)
        {
          if (q == cA)
            v = accA;
          if (q == cB)
            v = cB == cA ? __dadd_rn(accA, accB) : accB;
        }
        else if (q == cth)
          v = accA;
        acc[q] = v;
      }
      accA = accB = 0.0;
    }
    double pv[2 * MT];
#pragma unroll
    for (int q = 0; q < 2 * MT; ++q)
      pv[q] = 0.0;
#pragma unroll
    for (int c = 0; c < MT; ++c)
      if (c < m)
      {
        pv[c] = acc[c];
        if (kind == 0)
          pv[m + c] = acc[MT + c];
      }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 2 * MT; ++q)
    {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
        pv[q] = __dadd_rn(pv[q], __shfl_xor_sync(0xffffffffu, pv[q], off));
    }
    if (lane == 0)
    {
#pragma unroll
      for (int q = 0; q < 2 * MT; ++q)
        sh.wsum[warp][q] = pv[q];
    }
    consumer_sync<TB>();
    if (warp == 0)
    {
      for (int q = 0; q < nv; ++q)
      {
        double x = lane < TB / 32 ? sh.wsum[lane][q] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
          x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, off));
        if (lane == 0)
          P.partial[(static_cast<int64_t>(pnt) * 2 * kMaxM + q) * gridDim.x + blockIdx.x] = x;
      }
    }
    consumer_sync<TB>();
#pragma unroll
    for (int q = 0; q < 2 * MT; ++q)
      acc[q] = 0.0;
  };
  for_chunks(sh, CH, [&](int sg, int cp, int cc0, int cc1) {
    pc.mark(1);
    if (cp != cur_p)
    {
      if (cur_p >= 0)
        flush(cur_p);
      cur_p = cp;
    }
    pc.mark(2);
    mbar_wait(&full[bi], (phase_bits >> bi) & 1u);
    phase_bits ^= 1u << bi;
    pc.mark(3);
    unsigned char *buf = smem + bi * P.buf_bytes;
    const int64_t base_i = cc0;
    const int R = cc1 - cc0;
    const int sb = cp * m; // first system of the point
    if (kind == 2)
    {
      // r -= alpha w, partial (r, r).  x~ += alpha d (krylov.cpp:113) is deferred to the next
      // phase A, which streams d anyway.
      const double *rs = reinterpret_cast<const double *>(buf + P.b_r);
      const double *ws = reinterpret_cast<const double *>(buf + P.b_w);
      double *rg = const_cast<double *>(vrow(P, P.r, cp, base_i));
      const int ne = R * m;
      if (full_m)
      {
        const bool runA = sh.state[sb + cA] == kRun, runB = sh.state[sb + cB] == kRun;
        const double alA = sh.alpha[sb + cA], alB = sh.alpha[sb + cB];
        if (runA || runB)
        {
          const int nu = (ne + 1) >> 1;
          for (int u = threadIdx.x; u < nu; u += TB)
          {
            const double2 r2 = reinterpret_cast<const double2 *>(rs)[u];
            const double2 w2 = reinterpret_cast<const double2 *>(ws)[u];
            const double ra = __dadd_rn(r2.x, __dmul_rn(-alA, w2.x));
            const double rb = __dadd_rn(r2.y, __dmul_rn(-alB, w2.y));
            const bool hasB = 2 * u + 1 < ne; // (m = 1, odd row count: the last pair is half empty)
            if (runA && runB && hasB)
              __stcg(reinterpret_cast<double2 *>(rg) + u, make_double2(ra, rb));
            else
            {
              if (runA)
                __stcg(rg + 2 * u, ra);
              if (runB && hasB)
                __stcg(rg + 2 * u + 1, rb);
            }
            if (runA)
              accA = __dadd_rn(accA, __dmul_rn(ra, ra));
            if (runB && hasB)
              accB = __dadd_rn(accB, __dmul_rn(rb, rb));
          }
        }
      }
      else if (cfix)
      {
        if (sh.state[sb + cth] == kRun)
        {
          const double al = sh.alpha[sb + cth];
          for (int e = threadIdx.x; e < ne; e += TB)
          {
            const double rn = __dadd_rn(rs[e], __dmul_rn(-al, ws[e]));
            __stcg(rg + e, rn);
            accA = __dadd_rn(accA, __dmul_rn(rn, rn));
          }
        }
      }
      else
        for (int e = threadIdx.x; e < ne; e += TB)
        {
          const int c = col_of<MT>(e, m);
          if (sh.state[sb + c] != kRun)
            continue;
          const double al = sh.alpha[sb + c];
          const double rn = __dadd_rn(rs[e], __dmul_rn(-al, ws[e]));
          __stcg(rg + e, rn);
          acc_add<MT>(acc, c, __dmul_rn(rn, rn));
        }
    }
    else
    {
      const int H0 = P.hmax;
      const double *vr = reinterpret_cast<const double *>(buf + P.a_vr);
      const double *vd = reinterpret_cast<const double *>(buf + P.a_vd);
      // stage 0 alternates between two buffers: a warp that is done with this chunk starts the next
      // one's stage 0 while slower warps still read this chunk's d_new for their dot products
      double *s0 = reinterpret_cast<double *>(smem + ((step & 1) ? P.off_stage0b : P.off_stage0));
      double *sA = reinterpret_cast<double *>(smem + P.off_stage1);
      double *sB = reinterpret_cast<double *>(smem + P.off_stage2);
      // stage 0: d = fresh ? r : r + beta d_old over the halo-extended chunk; the deferred
      // x~ += alpha_prev d_old on own rows.  Check pass: source x~ + alpha_prev d_old (not
      // written back: neighbours read the same x~ rows as halo during this pass).
      const double *vx = reinterpret_cast<const double *>(buf + P.a_vx);
      const int ne0 = (R + 2 * H0) * m;
      const int lo = H0 * m, hi = (H0 + R) * m; // lo is even (even halos)
      double *dg = kind == 0 ? const_cast<double *>(vrow(P, dnew, cp, base_i - H0)) : nullptr;
      double *xg = kind == 0 ? const_cast<double *>(vrow(P, P.xt, cp, base_i - H0)) : nullptr;
      if (full_m)
      {
        const int sysA = sb + cA, sysB = sb + cB;
        const bool frA = sh.fresh[sysA] != 0, frB = sh.fresh[sysB] != 0;
        const bool pdA = sh.pend[sysA] != 0, pdB = sh.pend[sysB] != 0;
        const bool upA = pdA && sh.state[sysA] == kRun, upB = pdB && sh.state[sysB] == kRun;
        const double beA = sh.beta[sysA], beB = sh.beta[sysB], alA = sh.alpha[sysA], alB = sh.alpha[sysB];
        const int nu = (ne0 + 1) >> 1;
        // pair u -> stage slot: planar (m == 4): plane (u & 1), row u >> 1; else element pair u
        auto st0 = [&](int u, double a, double b) {
          if (MT == 4 && P.pst > 0)
            reinterpret_cast<double2 *>(s0 + ((u & 1) ? P.pst : 0))[u >> 1] = make_double2(a, b);
          else
            reinterpret_cast<double2 *>(s0)[u] = make_double2(a, b);
        };
        if (kind == 1)
          for (int u = threadIdx.x; u < nu; u += TB)
          {
            const double2 r2 = reinterpret_cast<const double2 *>(vr)[u];
            const double2 d2 = reinterpret_cast<const double2 *>(vd)[u];
            st0(u, pdA ? __dadd_rn(r2.x, __dmul_rn(alA, d2.x)) : r2.x, pdB ? __dadd_rn(r2.y, __dmul_rn(alB, d2.y)) : r2.y);
          }
        else
          for (int u = threadIdx.x; u < nu; u += TB)
          {
            const double2 r2 = reinterpret_cast<const double2 *>(vr)[u];
            const double2 d2 = reinterpret_cast<const double2 *>(vd)[u];
            const double va = frA ? r2.x : __dadd_rn(r2.x, __dmul_rn(beA, d2.x));
            const double vb = frB ? r2.y : __dadd_rn(r2.y, __dmul_rn(beB, d2.y));
            const int e = 2 * u;
            const bool ownA = e >= lo && e < hi, ownB = e + 1 >= lo && e + 1 < hi;
            if (ownA && ownB)
            {
              __stcg(reinterpret_cast<double2 *>(dg) + u, make_double2(va, vb));
              if (upA || upB)
              {
                const double2 x2 = reinterpret_cast<const double2 *>(vx)[u - (lo >> 1)];
                const double xa = __dadd_rn(x2.x, __dmul_rn(alA, d2.x)), xb = __dadd_rn(x2.y, __dmul_rn(alB, d2.y));
                if (upA && upB)
                  __stcg(reinterpret_cast<double2 *>(xg) + u, make_double2(xa, xb));
                else if (upA)
                  __stcg(xg + e, xa);
                else
                  __stcg(xg + e + 1, xb);
              }
            }
            else if (ownA) // (m = 1, odd row count: the chunk's last row shares its pair with a halo row)
            {
              __stcg(dg + e, va);
              if (upA)
                __stcg(xg + e, __dadd_rn(vx[e - lo], __dmul_rn(alA, d2.x)));
            }
            else if (ownB)
            {
              __stcg(dg + e + 1, vb);
              if (upB)
                __stcg(xg + e + 1, __dadd_rn(vx[e + 1 - lo], __dmul_rn(alB, d2.y)));
            }
            st0(u, va, vb);
          }
      }
      else if (cfix)
      {
        const int sys = sb + cth;
        const bool fr = sh.fresh[sys] != 0, pd = sh.pend[sys] != 0, run = sh.state[sys] == kRun;
        const double be = sh.beta[sys], al = sh.alpha[sys];
        if (kind == 1)
          for (int e = threadIdx.x; e < ne0; e += TB)
            s0[stage_idx(e, m, P.pst)] = pd ? __dadd_rn(vr[e], __dmul_rn(al, vd[e])) : vr[e];
        else
          for (int e = threadIdx.x; e < ne0; e += TB)
          {
            const double v = fr ? vr[e] : __dadd_rn(vr[e], __dmul_rn(be, vd[e]));
            if (e >= lo && e < hi)
            {
              __stcg(dg + e, v);
              if (pd && run)
                __stcg(xg + e, __dadd_rn(vx[e - lo], __dmul_rn(al, vd[e])));
            }
            s0[stage_idx(e, m, P.pst)] = v;
          }
      }
      else
        for (int e = threadIdx.x; e < ne0; e += TB)
        {
          const int c = col_of<MT>(e, m);
          const int sys = sb + c;
          double v;
          if (kind == 1)
            v = sh.pend[sys] ? __dadd_rn(vr[e], __dmul_rn(sh.alpha[sys], vd[e])) : vr[e];
          else
          {
            v = sh.fresh[sys] ? vr[e] : __dadd_rn(vr[e], __dmul_rn(sh.beta[sys], vd[e]));
            if (e >= lo && e < hi)
            {
              __stcg(dg + e, v);
              if (sh.pend[sys] && sh.state[sys] == kRun)
                __stcg(xg + e, __dadd_rn(vx[e - lo], __dmul_rn(sh.alpha[sys], vd[e])));
            }
          }
          s0[stage_idx(e, m, P.pst)] = v;
        }
      consumer_sync<TB>();
      pc.mark(4);
      const double *src = s0;
      int hs = H0;
      for (int st = 0; st < P.z; ++st)
      {
        const int hd = stg.halo[st + 1];
        const PEll F = tab[sg * (kMaxZ + 1) + 1 + st];
        const double *fv = reinterpret_cast<const double *>(buf + stg.a_fv[st]);
        const unsigned long long *fo = reinterpret_cast<const unsigned long long *>(buf + stg.a_fo[st]);
        double *dst = (st & 1) ? sB : sA;
        const int span = R + 2 * hd;
        for (int q = threadIdx.x; q < span; q += TB)
        {
          double a2[MT];
          ell_row_any<MT, 10, WIDE>(fv + q * F.E, fo + q * F.ow, F.E, F.ow, src, q + hs - hd, m, a2, P.pst);
          st_stage<MT>(dst, q, a2, m, P.pst);
        }
        consumer_sync<TB>();
        src = dst;
        hs = hd;
      }
      pc.mark(5);
      const PEll A = tab[sg * (kMaxZ + 1)];
      const double *av = reinterpret_cast<const double *>(buf + P.a_av);
      const unsigned long long *ao = reinterpret_cast<const unsigned long long *>(buf + P.a_ao);
      double *wg = const_cast<double *>(vrow(P, P.w, cp, base_i));
      for (int lr = threadIdx.x; lr < R; lr += TB)
      {
        double a2[MT];
        ell_row_any<MT, 5, WIDE>(av + lr * A.E, ao + lr * A.ow, A.E, A.ow, src, lr + hs, m, a2, P.pst);
        if (kind == 1)
        {
          const int64_t i = base_i + lr;
#pragma unroll
          for (int c = 0; c < MT; ++c)
          {
            if (c >= m)
              break;
            const double res = __dsub_rn(__ldg(vrow(P, P.b, cp, i) + c), a2[c]);
            __stcg(wg + lr * m + c, res);
            __stcg(const_cast<double *>(vrow(P, P.sol, cp, i)) + c, src[stage_idx((lr + hs) * m + c, m, P.pst)]);
            acc[c] = __dadd_rn(acc[c], __dmul_rn(res, res));
          }
        }
        else
        {
          double dn[MT];
          ld_stage<MT>(s0, H0 + lr, dn, m, P.pst);
          stg_row<MT>(wg + lr * m, a2, m);
          if (full_m)
          {
#pragma unroll
            for (int c = 0; c < MT; ++c)
            {
              acc[c] = __dadd_rn(acc[c], __dmul_rn(dn[c], a2[c]));
              acc[MT + c] = __dadd_rn(acc[MT + c], __dmul_rn(dn[c], dn[c]));
            }
          }
          else
          {
#pragma unroll
            for (int c = 0; c < MT; ++c)
              if (c < m)
              {
                acc[c] = __dadd_rn(acc[c], __dmul_rn(dn[c], a2[c]));
                acc[MT + c] = __dadd_rn(acc[MT + c], __dmul_rn(dn[c], dn[c]));
              }
          }
        }
      }
    }
    pc.mark(kind == 2 ? 7 : 6);
    // this warp is done with buffer bi (the empty barrier counts the consumer warps); no block-wide
    // barrier here: the next chunk's stage 0 writes the other stage-0 buffer, and the chain-stage
    // buffers are next written after that chunk's first barrier, which every warp reaches only
    // after finishing this chunk
    if (P.s0_double || kind == 2)
      __syncwarp();
    else
      consumer_sync<TB>(); // single stage-0 buffer: nobody may start the next chunk's stage 0 yet
    if ((threadIdx.x & 31) == 0)
      mbar_arrive(&empty[bi]);
    pc.mark(8);
    bi = bi + 1 == P.nb ? 0 : bi + 1;
    ++step;
  });
  if (cur_p >= 0)
    flush(cur_p);
  __syncthreads();
  pc.mark(2);
}

template <int TB, int MT, bool PR = false, bool WIDE = false>
__global__ void __launch_bounds__(TB + 32, 1) cg_stream(const __grid_constant__ StreamParams P)
{
  constexpr int TBX = TB + 32; // TB consumer threads + one producer warp
  cgrp::grid_group grid = cgrp::this_grid();
  extern __shared__ __align__(128) unsigned char smem_s[];
  __shared__ BandShared<TBX> sh;
  __shared__ __align__(8) uint64_t bars[2 * kStreamNB]; // full[NB], empty[NB]
  // operator descriptors per segment: A, then stage factors
  __shared__ PEll tab[kTabSlots * (kMaxZ + 1)];
  __shared__ StageTab stg;
  const int m = P.m;
  const int S = P.l * m;
  uint32_t phase_bits = 0;
  RingProducer rp{0u, 0u};
  PhaseClock<PR> pc{PR && P.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0, clock64(), {}};
  if (threadIdx.x == 0)
  {
    int q = 0;
    while (q < kMaxSeg && P.seg[blockIdx.x * kMaxSeg + q].p >= 0)
    {
      sh.seg[q] = P.seg[blockIdx.x * kMaxSeg + q];
      ++q;
    }
    sh.nseg = q;
    for (int g = 0; g < q; ++g)
    {
      const int p = sh.seg[g].p;
      PEll a = P.A[p];
      if (P.eqA[p])
        a.o = P.A[0].o;
      tab[g * (kMaxZ + 1)] = a;
      for (int st = 0; st < P.z; ++st)
      {
        const int f = P.z - 1 - st;
        PEll fe = P.F[p * P.z + f];
        if (P.eqF[p * P.z + f])
          fe.o = P.F[f].o;
        tab[g * (kMaxZ + 1) + 1 + st] = fe;
      }
    }
#pragma unroll
    for (int st = 0; st <= kMaxZ; ++st)
      stg.halo[st] = P.halo[st];
#pragma unroll
    for (int st = 0; st < kMaxZ; ++st)
    {
      stg.a_fv[st] = static_cast<uint32_t>(P.a_fv[st]);
      stg.a_fo[st] = static_cast<uint32_t>(P.a_fo[st]);
    }
    for (int b = 0; b < kStreamNB; ++b)
    {
      mbar_init(&bars[b], 1);                   // full: the producer's arrive.expect_tx
      mbar_init(&bars[kStreamNB + b], TB / 32); // empty: one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int p = threadIdx.x; p < P.l; p += TBX)
    sh.pmask[p] = 1;
  __syncthreads();
  // rows of every masked point this block owns
  auto for_rows = [&](auto &&fn) { for_segments(P, sh, fn); };
  // ---- phase 0: ||b||^2 (one pass, plain loads)
  for_rows([&](int p, int64_t rs, int64_t re) {
    begin_point(sh);
    for (int64_t c0 = rs; c0 < re; c0 += TBX)
    {
      const int64_t i = c0 + threadIdx.x;
      double pk[MT];
#pragma unroll
      for (int c = 0; c < MT; ++c)
      {
        pk[c] = 0.0;
        if (c < m && i < re)
        {
          const double bv = __ldg(vrow(P, P.b, p, i) + c);
          pk[c] = __dmul_rn(bv, bv);
        }
      }
      chunk_sum<TBX, MT>(sh, pk, m);
    }
    end_point(P.partial, sh, p, m);
  });
  grid.sync();
  reduce_blocks<TBX, StreamParams>(P, sh, m);
  for (int s = threadIdx.x; s < S; s += TBX)
  {
    const double bb = sh.tot[s];
    const double bn = sqrt(bb);
    sh.bnorm[s] = bn;
    sh.rho[s] = bb;
    sh.target[s] = P.rtol * bn;
    sh.state[s] = bn == 0.0 ? kZeroRhs : kRun;
    sh.fresh[s] = 1;
    sh.pend[s] = 0;
    sh.beta[s] = 0.0;
    sh.sit[s] = 0;
  }
  __syncthreads();

  auto copy_finish = [&]() {
    for_rows([&](int p, int64_t rs, int64_t re) {
      for (int64_t i = rs + threadIdx.x; i < re; i += TBX)
        for (int c = 0; c < m; ++c)
        {
          const int s = p * m + c;
          const int64_t o = static_cast<int64_t>(s) * P.n + i;
          if (sh.state[s] == kPendingConv || sh.state[s] == kMaxed)
          {
            if (P.X)
              P.X[o] = __ldcg(vrow(P, P.sol, p, i) + c);
            if (P.TR)
              P.TR[o] = __ldcg(vrow(P, P.w, p, i) + c);
          }
          else if (sh.state[s] == kPendingRestart)
            __stcg(const_cast<double *>(vrow(P, P.r, p, i)) + c, __ldcg(vrow(P, P.w, p, i) + c));
        }
    });
    fence_async_global();
  };

  // true-residual check pass over the masked points
  auto check_pass = [&](const double *dcur) {
    stream_pass<TB, MT, kStreamNB, PhaseClock<PR>, WIDE>(P, sh, stg, tab, smem_s, bars, bars + kStreamNB, phase_bits, rp, 1, dcur,
                                                         nullptr, pc);
  };
  // after phase A's reduction: alpha or breakdown for the running systems of masked points
  auto after_a = [&](int64_t itn) {
    for (int s = threadIdx.x; s < S; s += TBX)
    {
      if (!sh.pmask[s / m])
        continue;
      sh.pend[s] = 0; // phase A applied the deferred x~ update
      if (sh.state[s] != kRun)
        continue;
      const int p = s / m, c = s % m;
      const double curv = sh.tot[p * m + c];
      const double dd = sh.tot[S + p * m + c];
      if (!(curv > 1e-30 * dd))
      {
        sh.state[s] = kBreakdown;
        sh.sit[s] = itn;
      }
      else
        sh.alpha[s] = sh.rho[s] / curv;
    }
    __syncthreads();
  };
  // after phase B's reduction: beta, rho for the running systems of masked points (itn: the
  // iteration just completed, 0-based)
  auto after_b = [&](int64_t itn) {
    for (int s = threadIdx.x; s < S; s += TBX)
    {
      if (!sh.pmask[s / m] || sh.state[s] != kRun)
        continue;
      const double rn = sh.tot[s];
      if (P.hist && blockIdx.x == 0 && itn < P.hist_cap)
        P.hist[static_cast<int64_t>(s) * P.hist_cap + itn] = sqrt(rn) / sh.bnorm[s];
      sh.beta[s] = rn / sh.rho[s];
      sh.rho[s] = rn;
      sh.fresh[s] = 0;
      sh.pend[s] = 1; // x~ += alpha d owed to the next phase A / check pass
    }
    __syncthreads();
  };

  int cur = 0;
  int64_t it = 0;
  for (;;)
  {
    if (it >= P.maxit)
      break;
    if (threadIdx.x == 0)
      sh.flag = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < P.l; p += TBX)
    {
      int need = 0;
      for (int c = 0; c < m; ++c)
      {
        const int s = p * m + c;
        need |= sh.state[s] == kRun && sqrt(sh.rho[s]) <= sh.target[s];
      }
      sh.pmask[p] = need;
      if (need)
        atomicOr(&sh.flag, 1);
    }
    __syncthreads();
    if (sh.flag)
    {
      check_pass(cur ? P.dbuf1 : P.dbuf0);
      fence_async_global();
      grid.sync();
      reduce_blocks<TBX, StreamParams>(P, sh, m);
      for (int s = threadIdx.x; s < S; s += TBX)
      {
        if (!(sh.state[s] == kRun && sqrt(sh.rho[s]) <= sh.target[s]))
          continue;
        const double tt = sh.tot[s];
        if (sqrt(tt) <= sh.target[s])
        {
          sh.state[s] = kPendingConv;
          sh.sit[s] = it;
        }
        else
        {
          sh.rho[s] = tt;
          if (sqrt(tt) <= sh.target[s])
          {
            sh.state[s] = kPendingConv;
            sh.sit[s] = it;
          }
          else
          {
            sh.state[s] = kPendingRestart;
            sh.fresh[s] = 1;
          }
        }
      }
      __syncthreads();
      copy_finish();
      grid.sync();
      for (int s = threadIdx.x; s < S; s += TBX)
      {
        if (sh.state[s] == kPendingConv)
          sh.state[s] = kConverged;
        else if (sh.state[s] == kPendingRestart)
          sh.state[s] = kRun;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0)
      sh.flag = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < P.l; p += TBX)
    {
      int live = 0;
      for (int c = 0; c < m; ++c)
        live |= sh.state[p * m + c] == kRun;
      sh.pmask[p] = live;
      if (live)
        atomicOr(&sh.flag, 1);
    }
    __syncthreads();
    if (!sh.flag)
      break;
    double *d_old = cur ? P.dbuf1 : P.dbuf0;
    double *d_new = cur ? P.dbuf0 : P.dbuf1;
    pc.mark(9);
    stream_pass<TB, MT, kStreamNB, PhaseClock<PR>, WIDE>(P, sh, stg, tab, smem_s, bars, bars + kStreamNB, phase_bits, rp, 0, d_old, d_new, pc);
    fence_async_global();
    grid.sync();
    pc.mark(10);
    reduce_blocks<TBX, StreamParams>(P, sh, 2 * m);
    pc.mark(11);
    after_a(it);
    pc.mark(9);
    stream_pass<TB, MT, kStreamNB, PhaseClock<PR>, WIDE>(P, sh, stg, tab, smem_s, bars, bars + kStreamNB, phase_bits, rp, 2, d_old, d_new, pc);
    fence_async_global();
    grid.sync();
    pc.mark(10);
    reduce_blocks<TBX, StreamParams>(P, sh, m);
    pc.mark(11);
    after_b(it);
    ++it;
    cur ^= 1;
  }
  // ---- budget exhausted: final true-residual check
  if (threadIdx.x == 0)
    sh.flag = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < P.l; p += TBX)
  {
    int need = 0;
    for (int c = 0; c < m; ++c)
      need |= sh.state[p * m + c] == kRun;
    sh.pmask[p] = need;
    if (need)
      atomicOr(&sh.flag, 1);
  }
  __syncthreads();
  if (sh.flag)
  {
    check_pass(cur ? P.dbuf1 : P.dbuf0);
    fence_async_global();
    grid.sync();
    reduce_blocks<TBX, StreamParams>(P, sh, m);
    for (int s = threadIdx.x; s < S; s += TBX)
    {
      if (sh.state[s] != kRun)
        continue;
      const double tt = sh.tot[s];
      sh.state[s] = sqrt(tt) <= sh.target[s] ? kPendingConv : kMaxed;
      sh.sit[s] = it;
    }
    __syncthreads();
    copy_finish();
    for (int s = threadIdx.x; s < S; s += TBX)
      if (sh.state[s] == kPendingConv)
        sh.state[s] = kConverged;
    __syncthreads();
  }
  for (int p = threadIdx.x; p < P.l; p += TBX)
    sh.pmask[p] = 1;
  __syncthreads();
  for_rows([&](int p, int64_t rs, int64_t re) {
    for (int64_t i = rs + threadIdx.x; i < re; i += TBX)
      for (int c = 0; c < m; ++c)
      {
        const int s = p * m + c;
        const int64_t o = static_cast<int64_t>(s) * P.n + i;
        if (sh.state[s] == kZeroRhs)
        {
          if (P.X)
            P.X[o] = 0.0;
          if (P.TR)
            P.TR[o] = 0.0;
          if (P.REC)
            P.REC[o] = 0.0;
        }
        else if (sh.state[s] != kBreakdown && P.REC)
          P.REC[o] = __ldcg(vrow(P, P.r, p, i) + c);
      }
  });
  if constexpr (PR)
    if (pc.on)
      for (int k = 0; k < 12; ++k)
        P.prof[k] = pc.acc[k];
  if (blockIdx.x == 0)
  {
    for (int s = threadIdx.x; s < S; s += TBX)
    {
      const int st = sh.state[s];
      P.iters[s] = sh.sit[s];
      P.conv[s] = (st == kConverged || st == kZeroRhs) ? 1 : 0;
      P.status[s] = st == kBreakdown ? MGPU_ERR_BREAKDOWN : MGPU_OK;
      P.bd_iter[s] = st == kBreakdown ? sh.sit[s] : -1;
    }
    if (threadIdx.x == 0)
      *P.loop_iters = it;
  }
}

// CSR -> padded row-major ELL (values [row][E], int8 offsets packed in ow u64 words)
__global__ void csr_to_pell(int64_t n, DCsr M, int E, int ow, double *vals, unsigned long long *offs)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  const int64_t k0 = M.rp[i], k1 = M.rp[i + 1];
  unsigned long long w[kEllMax / 8] = {};
  for (int t = 0; t < E; ++t)
  {
    const bool has = k0 + t < k1;
    vals[i * E + t] = has ? M.v[k0 + t] : 0.0; // padding adds +0 after the row's entries
    if (has)
      w[t >> 3] |=
          static_cast<unsigned long long>(static_cast<unsigned char>(static_cast<signed char>(M.ci[k0 + t] - i)))
          << (8 * (t & 7));
  }
  for (int q = 0; q < ow; ++q)
    offs[i * ow + q] = w[q];
}

__global__ void stream_init(int l, int m, int64_t n, int64_t ldv, const double *__restrict__ B, int64_t ldb,
                            double *b, double *r, double *d, double *xt)
{
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per = n * m;
  if (g >= per * l)
    return;
  const int64_t p = g / per, rem = g - p * per, i = rem / m, c = rem - i * m;
  const double v = B[p * ldb + c * n + i];
  const int64_t o = p * ldv + (kPadR + i) * m + c;
  b[o] = v;
  r[o] = v;
  d[o] = v;
  xt[o] = 0.0;
}

} // namespace

// Host side of cg_stream.  Returns false if the chunk buffers do not fit.
bool stream_solve(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, int z, const mgpu_csr *const *chains, int64_t n,
                  int m, const double *B_dev, int64_t ldb, const int *halo, int hmax, double rtol, int64_t maxit,
                  double *X_dev, double *REC_dev, double *TR_dev, int64_t *d_it, int *d_conv, int *d_st, int64_t *d_bd,
                  double *d_hist, int64_t hist_cap, int64_t *d_loop)
{
  constexpr int TB = 480; // consumer threads; + one producer warp = 512
  cudaStream_t s = ctx->stream;
  // even halos keep every bulk copy 16-byte aligned; rebuilt inside-out so that
  // hal[st] >= hal[st + 1] + bw(factor of stage st) still holds
  std::vector<int> hal(static_cast<size_t>(z + 1));
  hal[z] = (halo[z] + 1) & ~1;
  for (int st = z - 1; st >= 0; --st)
    hal[st] = (hal[st + 1] + (halo[st] - halo[st + 1]) + 1) & ~1;
  const int H0 = hal[0];
  (void)hmax;
  if (H0 >= kPadR || // even_up(c1 - c0 + 2 H0) may reach one row past the kPadR padding when H0 == kPadR
       l > kMaxPoints || static_cast<int64_t>(l) * m > kMaxSys || l > ctx->num_sms * kMaxSeg)
    return false;
  // ---- padded ELL operators
  auto ell_of = [&](const mgpu_csr *M, std::vector<DBuf> &keep) {
    // exact row width (odd widths allowed: a 5-entry row streams 40 bytes, not 48); bulk
    // copies stay 16-byte multiples because chunk row counts are even
    const int E = static_cast<int>(csr_max_row(ctx, const_cast<mgpu_csr *>(M)));
    const int Ee = E < 1 ? 1 : E;
    const int ow = (Ee + 7) / 8;
    const int64_t rows = n + 2 * kPadR;
    keep.emplace_back(sizeof(double) * rows * Ee, s);
    DBuf &v = keep.back();
    keep.emplace_back(sizeof(unsigned long long) * rows * ow, s);
    DBuf &o = keep.back();
    MG_CUDA(cudaMemsetAsync(v.ptr, 0, sizeof(double) * rows * Ee, s));
    MG_CUDA(cudaMemsetAsync(o.ptr, 0, sizeof(unsigned long long) * rows * ow, s));
    double *v0 = v.as<double>() + kPadR * Ee;
    unsigned long long *o0 = o.as<unsigned long long>() + kPadR * ow;
    csr_to_pell<<<blocks_for(n), kThreads, 0, s>>>(n, M->view(), Ee, ow, v0, o0);
    check_launch(ctx, "csr_to_pell");
    return PEll{v0, o0, Ee, ow};
  };
  std::vector<DBuf> keep;
  keep.reserve(static_cast<size_t>(2 * l * (z + 1) + 16));
  for (int p = 0; p < l; ++p)
  {
    // rows of up to kEllMax entries (collapsed update chains widen with every product)
    if (csr_max_row(ctx, const_cast<mgpu_csr *>(A[p])) > kEllMax)
      return false;
    for (int f = 0; f < z; ++f)
      if (csr_max_row(ctx, const_cast<mgpu_csr *>(chains[static_cast<size_t>(p) * z + f])) > kEllMax)
        return false;
  }
  std::vector<PEll> hA(static_cast<size_t>(l)), hF(static_cast<size_t>(l) * (z > 0 ? z : 1));
  int EA = 0;
  std::vector<int> EF(static_cast<size_t>(z > 0 ? z : 1), 0);
  std::vector<int> OWF(static_cast<size_t>(z > 0 ? z : 1), 1); // offset words per row (1: <= 8 entries)
  int OWA = 1;
  for (int p = 0; p < l; ++p)
  {
    hA[p] = ell_of(A[p], keep);
    EA = std::max(EA, hA[p].E);
    for (int f = 0; f < z; ++f)
    {
      hF[static_cast<size_t>(p) * z + f] = ell_of(chains[static_cast<size_t>(p) * z + f], keep);
      const int st = z - 1 - f;
      EF[st] = std::max(EF[st], hF[static_cast<size_t>(p) * z + f].E);
      OWF[st] = std::max(OWF[st], hF[static_cast<size_t>(p) * z + f].ow);
    }
    OWA = std::max(OWA, hA[p].ow);
  }
  // The x~ update is deferred into the next phase A, which streams d_old anyway (one vector pass
  // fewer; configs[3] P = I 1029 -> 1005 us per iteration, configs[4] share 5025 -> 4891,
  // configs[2] shape 36.9 -> 36.1 when it was introduced).
  // ---- shared-memory plan: the largest chunk height whose double buffer fits
  StreamParams P{};
  size_t dyn = 0;
  int64_t CH = 0;
  int optin = 0;
  MG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const size_t stat = sizeof(BandShared<TB + 32>) + sizeof(PEll) * kTabSlots * (kMaxZ + 1) + 128;
  // One plan: fills P's shared-memory layout for (chunk rows, ring depth, stage 0 double-buffered);
  // false when it does not fit.
  auto plan = [&](int64_t ch, int nb, bool dbl) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t o2 = off;
      off += (bytes + 127) & ~static_cast<size_t>(127);
      return o2;
    };
    const int64_t vrows = (ch + 2 * H0 + 1) & ~1ll;
    P.a_vr = take(sizeof(double) * vrows * m);
    P.a_vd = take(sizeof(double) * vrows * m);
    P.a_vx = take(sizeof(double) * ch * m);
    for (int st = 0; st < z; ++st)
    {
      const int64_t rows = (ch + 2 * hal[st + 1] + 1) & ~1ll;
      P.a_fv[st] = take(sizeof(double) * rows * EF[st]);
      P.a_fo[st] = take(sizeof(unsigned long long) * rows * OWF[st]);
    }
    P.a_av = take(sizeof(double) * ch * EA);
    P.a_ao = take(sizeof(unsigned long long) * ch * OWA);
    const size_t a_bytes = off;
    off = 0;
    const size_t b_bytes = sizeof(double) * ch * m * 2;
    P.buf_bytes = (std::max(a_bytes, b_bytes) + 127) & ~static_cast<size_t>(127);
    off = nb * P.buf_bytes;
    // m == 4 with a chain: planar stage buffers, one plane stride (the widest buffer's rows) for all
    const int64_t srows0 = ch + 2 * H0;
    P.pst = (m == 4 && z >= 1) ? static_cast<int>(2 * srows0) : 0; // (P = I measured 842 -> 859 us planar)
    P.off_stage0 = take(sizeof(double) * srows0 * m);
    P.off_stage0b = dbl ? take(sizeof(double) * srows0 * m) : P.off_stage0;
    P.s0_double = dbl ? 1 : 0;
    P.off_stage1 = z >= 1 ? take(sizeof(double) * (P.pst ? srows0 : ch + 2 * hal[1]) * m) : 0; // chain stages
    P.off_stage2 = z >= 2 ? take(sizeof(double) * (P.pst ? srows0 : ch + 2 * hal[2]) * m) : 0;
    if (off + stat > static_cast<size_t>(optin))
      return false;
    dyn = off;
    CH = ch;
    P.nb = nb;
    return true;
  };
  // Chunk height: as tall as shared memory allows (per-chunk barriers and pipeline bookkeeping
  // amortise over its rows), with the double-buffered stage 0 (no block-wide barrier at the end of a
  // chunk) unless that costs more than a tenth of the height.
  //  * m >= 4: 2-deep ring (448 rows 3-deep measured 924 us against 837 2-deep), at most 448 rows,
  //    no multiples of 128 rows (with every block striding through HBM in lock step 512 / 640 rows
  //    measured 872 / 876 us per iteration on configs[3] against 843 / 836 for 576 / 448), in steps
  //    of 16 rows: configs[3] with its factor 1083 us at 320 rows, 1069 at 336, 1060 at 352 (the
  //    tallest with two stage-0 buffers), 1065 at 368 with one.  configs[4] share: 448 rows with one
  //    stage-0 buffer 4841 us, 320 rows with two 5150.
  //  * m < 4 (configs[2] shape): tallest chunk, 3-deep before 2-deep, measured best (26.8 us at
  //    1024 rows, 30.7 at 512 / 3-deep, 39.9 at 256).
  if (ctx->opt[MGPU_OPT_STREAM_CHUNK] > 0) // forced plan (diagnostics)
  {
    const int fd = ctx->opt[MGPU_OPT_STREAM_RING] ? static_cast<int>(ctx->opt[MGPU_OPT_STREAM_RING]) : 2;
    if (!plan(ctx->opt[MGPU_OPT_STREAM_CHUNK], fd, true))
      plan(ctx->opt[MGPU_OPT_STREAM_CHUNK], fd, false);
  }
  if (CH == 0 && m >= 4)
  {
    int64_t ch_single = 0, ch_double = 0;
    for (int64_t ch = 448; ch >= 128 && (ch_single == 0 || ch_double == 0); ch -= 16)
    {
      if (ch % 128 == 0)
        continue;
      if (ch_single == 0 && plan(ch, 2, false))
        ch_single = ch;
      if (ch_double == 0 && plan(ch, 2, true))
        ch_double = ch;
    }
    CH = 0;
    if (ch_double > 0 && 10 * ch_double >= 9 * ch_single)
      plan(ch_double, 2, true);
    else if (ch_single > 0)
      plan(ch_single, 2, false);
  }
  if (CH == 0)
  {
    for (int64_t ch = 1024; ch >= 128 && CH == 0; ch -= 64)
      for (int nb : {3, 2})
      {
        if (m >= 4 && nb == 3)
          continue;
        if (CH == 0 && !plan(ch, nb, true))
          plan(ch, nb, false);
      }
  }
  if (CH == 0)
    return false;
#ifdef MGPU_HOST_TRACE
  {
    char msg[128];
    std::snprintf(msg, sizeof msg, "cg_stream plan: %lld-row chunks, %d-deep ring, %zu B per slot",
                  static_cast<long long>(CH), P.nb, P.buf_bytes);
    host_mark(msg);
  }
#endif
  // ---- vectors (padded) and the per-point block plan
  const int64_t ldv = ((n + 2 * kPadR) * m + 1) & ~1ll; // even: every point block starts 16-byte aligned
  const size_t vb = sizeof(double) * static_cast<size_t>(l) * ldv;
  DBuf b(vb, s), xt(vb, s), r(vb, s), d0(vb, s), d1(vb, s), w(vb, s), sol(vb, s);
  for (DBuf *q : {&b, &xt, &r, &d0, &d1, &w, &sol})
    MG_CUDA(cudaMemsetAsync(q->ptr, 0, vb, s));
  stream_init<<<blocks_for(static_cast<int64_t>(l) * n * m), kThreads, 0, s>>>(
      l, m, n, ldv, B_dev, ldb, b.as<double>(), r.as<double>(), d0.as<double>(), xt.as<double>());
  check_launch(ctx, "stream_init");
  const int G = ctx->num_sms;
  std::vector<Seg> hseg(static_cast<size_t>(G) * kMaxSeg, Seg{-1, 0, 0, 0});
  std::vector<int2> hpb(static_cast<size_t>(l));
  // tile plan: slabs = G / gcd(G, l) (so that slabs * l tiles = tile_seg * G), when a block's
  // tile_seg = l / gcd(G, l) segments fit its table and every slab has rows
  int tile_slabs = 0, tile_seg = 0;
  {
    int a = G, c = l;
    while (c)
    {
      const int t = a % c;
      a = c;
      c = t;
    }
    tile_slabs = G / a;
    tile_seg = l / a;
  }
  // (worth it from about 16 chunks per tile: more segments per block mean more per-point flushes,
  // configs[2] shape measured 26.8 us per iteration contiguous against 29.2 tiled, configs[3] 1106 / 1097)
  const bool tiled = ctx->opt[MGPU_OPT_STREAM_TILES] != 0 && l > 1 && tile_seg <= kMaxSeg &&
                     (ctx->opt[MGPU_OPT_STREAM_TILES] > 1 || n / tile_slabs >= 16 * CH) &&
                     (n + 31) / 32 >= 4 * static_cast<int64_t>(tile_slabs);
  if (tiled)
  {
    // Row-slab x point tiles.  Tile T = (slab T / l, point T % l); block bk takes tiles bk, bk + G,
    // bk + 2 G, ... in that order, so at any time the G blocks work on G consecutive tiles:
    // G / l whole slabs, every point of a slab at the same time.  Whatever the points of a slab
    // share (the ELL offsets; operator values formed from shared M, D, K) is then read from
    // HBM by the first block to get there and from L2 by the others.  (The contiguous plan below
    // puts point p on blocks [p G / l, (p + 1) G / l): with G / l = 9.25 only every fourth
    // point passes the same rows at the same time.)  Every block owns at most one tile of a
    // point (tile_seg * G tiles, G | tile_slabs * l), so one partial-sum slot per (point, block).
    const int64_t groups = (n + 31) / 32;
    for (int bk = 0; bk < G; ++bk)
      for (int t = 0; t < tile_seg; ++t)
      {
        const int64_t T = static_cast<int64_t>(t) * G + bk;
        const int64_t slab = T / l;
        const int p = static_cast<int>(T % l);
        const int64_t g0 = groups * slab / tile_slabs, g1 = groups * (slab + 1) / tile_slabs;
        hseg[static_cast<size_t>(bk) * kMaxSeg + t] =
            Seg{p, static_cast<int>(g0 * 32), static_cast<int>(std::min<int64_t>(n, g1 * 32)), 0};
      }
    // slots of blocks without a tile of the point stay zero (the buffer is cleared below)
    for (int p = 0; p < l; ++p)
      hpb[p] = make_int2(0, G);
  }
  else if (l <= G)
  {
    for (int p = 0; p < l; ++p)
    {
      const int b0 = static_cast<int>(static_cast<int64_t>(p) * G / l);
      const int b1 = static_cast<int>(static_cast<int64_t>(p + 1) * G / l);
      const int64_t groups = (n + 31) / 32;
      // a point spans at most one block per 32-row group: every block in [b0, b0 + nb) owns
      // rows, so every partial-sum slot the reduction reads is written (a block without rows
      // would never flush its slot)
      const int nb = static_cast<int>(std::min<int64_t>(b1 - b0, groups));
      for (int k = 0; k < nb; ++k)
      {
        const int64_t g0 = groups * k / nb, g1 = groups * (k + 1) / nb;
        hseg[static_cast<size_t>(b0 + k) * kMaxSeg] =
            Seg{p, static_cast<int>(g0 * 32), static_cast<int>(std::min<int64_t>(n, g1 * 32)), 0};
      }
      hpb[p] = make_int2(b0, b0 + nb);
    }
  }
  else
  {
    for (int bk = 0; bk < G; ++bk)
    {
      const int p0 = static_cast<int>(static_cast<int64_t>(bk) * l / G);
      const int p1 = static_cast<int>(static_cast<int64_t>(bk + 1) * l / G);
      for (int p = p0; p < p1; ++p)
      {
        hseg[static_cast<size_t>(bk) * kMaxSeg + (p - p0)] = Seg{p, 0, static_cast<int>(n), 0};
        hpb[p] = make_int2(bk, bk + 1);
      }
    }
  }
  DBuf segs(sizeof(Seg) * hseg.size(), s), pblk(sizeof(int2) * hpb.size(), s);
  DBuf dA(sizeof(PEll) * hA.size(), s), dF(sizeof(PEll) * hF.size(), s);
  // structure-equality flags against point 0 (no host round trip: the kernel reads them)
  DBuf eqA(sizeof(int) * static_cast<size_t>(l), s), eqF(sizeof(int) * static_cast<size_t>(l) * (z > 0 ? z : 1), s);
  {
    std::vector<int> ones(static_cast<size_t>(l) * (z > 0 ? z : 1), 1);
    MG_CUDA(cudaMemcpyAsync(eqA.ptr, ones.data(), sizeof(int) * l, cudaMemcpyHostToDevice, s));
    MG_CUDA(cudaMemcpyAsync(eqF.ptr, ones.data(), sizeof(int) * ones.size(), cudaMemcpyHostToDevice, s));
    auto compare = [&](const mgpu_csr *X, const mgpu_csr *X0, int *flag) {
      if (X == X0 || (X->row_ptr == X0->row_ptr && X->col_idx == X0->col_idx))
        return; // stays 1
      if (X->nnz != X0->nnz)
      {
        MG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
        return;
      }
      pattern_eq_kernel<<<std::max(1, std::min(ctx->num_sms * 4, static_cast<int>((n + 255) / 256))), 256, 0, s>>>(
          n, X->nnz, X0->row_ptr, X0->col_idx, X->row_ptr, X->col_idx, flag);
      check_launch(ctx, "pattern_eq_kernel");
    };
    for (int p = 1; p < l; ++p)
    {
      compare(A[p], A[0], eqA.as<int>() + p);
      for (int f = 0; f < z; ++f)
        compare(chains[static_cast<size_t>(p) * z + f], chains[f], eqF.as<int>() + static_cast<size_t>(p) * z + f);
    }
  }
  DBuf partial(sizeof(double) * static_cast<size_t>(l) * 2 * kMaxM * G, s);
  MG_CUDA(cudaMemsetAsync(partial.ptr, 0, partial.bytes, s));
  MG_CUDA(cudaMemcpyAsync(segs.ptr, hseg.data(), sizeof(Seg) * hseg.size(), cudaMemcpyHostToDevice, s));
  MG_CUDA(cudaMemcpyAsync(pblk.ptr, hpb.data(), sizeof(int2) * hpb.size(), cudaMemcpyHostToDevice, s));
  MG_CUDA(cudaMemcpyAsync(dA.ptr, hA.data(), sizeof(PEll) * hA.size(), cudaMemcpyHostToDevice, s));
  MG_CUDA(cudaMemcpyAsync(dF.ptr, hF.data(), sizeof(PEll) * hF.size(), cudaMemcpyHostToDevice, s));
  P.l = l;
  P.m = m;
  P.z = z;
  P.rpt = 1;
  P.ch = static_cast<int>(CH);
  {
    // phase B: r, w -> the tallest chunk (multiple of 64 rows, <= 8192) that fits one slot
    int64_t chb = static_cast<int64_t>(P.buf_bytes / (2 * sizeof(double) * static_cast<size_t>(m))) & ~63ll;
    chb = std::min<int64_t>(std::max<int64_t>(chb, CH), 8192);
    if (ctx->opt[MGPU_OPT_STREAM_SAME_CHB]) // diagnostics: phase B on the phase A chunk height
      chb = CH;
    P.ch_b = static_cast<int>(chb);
    P.b_r = 0;
    P.b_w = static_cast<size_t>(chb) * m * sizeof(double); // multiple of 512 B
  }
  P.n = n;
  P.ldv = ldv;
  for (int q = 0; q <= z; ++q)
    P.halo[q] = hal[q];
  P.hmax = H0;
  P.A = dA.as<PEll>();
  P.F = dF.as<PEll>();
  P.eqA = eqA.as<int>();
  P.eqF = eqF.as<int>();
  P.rtol = rtol;
  P.maxit = maxit;
  P.b = b.as<double>();
  P.xt = xt.as<double>();
  P.r = r.as<double>();
  P.dbuf0 = d0.as<double>();
  P.dbuf1 = d1.as<double>();
  P.w = w.as<double>();
  P.sol = sol.as<double>();
  P.partial = partial.as<double>();
  P.seg = segs.as<Seg>();
  P.pblk = pblk.as<int2>();
  P.X = X_dev;
  P.REC = REC_dev;
  P.TR = TR_dev;
  P.iters = d_it;
  P.conv = d_conv;
  P.status = d_st;
  P.bd_iter = d_bd;
  P.hist = d_hist;
  P.hist_cap = hist_cap;
  P.loop_iters = d_loop;
  P.prof = ctx->prof_dev;
  auto launch = [&](auto kern) {
    MG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
    int per_sm = 0;
    MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TB + 32, dyn));
    if (per_sm < 1)
      return false;
    void *args[] = {&P};
    MG_CUDA(cudaEventRecord(ctx->ev0, s));
    MG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(kern), dim3(static_cast<unsigned>(G)), dim3(TB + 32), args,
                                        dyn, s));
    check_launch(ctx, "cg_stream");
    MG_CUDA(cudaEventRecord(ctx->ev1, s));
    return true;
  };
  bool ok;
  const bool pr = P.prof != nullptr;
  // rows of more than 16 entries (collapsed update chains) take the WIDE instantiation
  bool wide = OWA > 2;
  for (int st = 0; st < z; ++st)
    wide = wide || OWF[st] > 2;
  if (wide)
  {
    if (m == 1)
      ok = launch(cg_stream<TB, 1, false, true>);
    else if (m == 2)
      ok = launch(cg_stream<TB, 2, false, true>);
    else if (m <= 4)
      ok = launch(cg_stream<TB, 4, false, true>);
    else
      ok = launch(cg_stream<TB, 8, false, true>);
  }
  else if (m == 1)
    ok = pr ? launch(cg_stream<TB, 1, true>) : launch(cg_stream<TB, 1>);
  else if (m == 2) // (phase profile instantiated for m = 1 and m <= 4 only)
    ok = launch(cg_stream<TB, 2>);
  else if (m <= 4)
    ok = pr ? launch(cg_stream<TB, 4, true>) : launch(cg_stream<TB, 4>);
  else
    ok = launch(cg_stream<TB, 8>);
  if (ok)
    MG_CUDA(cudaStreamSynchronize(s)); // keep the padded buffers alive until the kernel is done
  return ok;
}

} // namespace mgpu
