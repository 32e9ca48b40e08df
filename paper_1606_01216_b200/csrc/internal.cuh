// Internal declarations shared by the mgpu translation units (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <stdexcept>
#include <memory>
#include <string>
#include <vector>

#include "mgpu.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "mgpu is written for sm_100a (B200) only"
#endif

namespace mgpu
{
// The context's pinned host staging buffer, at least `bytes` long.  Every user copies into it,
// synchronises the stream and unpacks before returning, so one buffer per context suffices.
void *pinned_scratch(mgpu_ctx *ctx, size_t bytes);
// Built with -DMGPU_HOST_TRACE: prints a steady-clock host timestamp and `what` on stderr (diagnostics)
void host_mark(const char *what);

// A C++ exception carrying an mgpu_status; converted at the C boundary.
struct Error : std::runtime_error
{
  int status;
  int64_t index, rhs_column, point;
  Error(int st, const std::string &msg, int64_t idx = -1, int64_t col = -1, int64_t pt = -1)
    : std::runtime_error(msg), status(st), index(idx), rhs_column(col), point(pt)
  {
  }
};

[[noreturn]] inline void cuda_fail(cudaError_t e, const char *what, const char *file, int line)
{
  throw Error(MGPU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" + std::to_string(line) +
                                 ")");
}

#define MG_CUDA(expr)                                                                                                  \
  do                                                                                                                   \
  {                                                                                                                    \
    cudaError_t _e = (expr);                                                                                           \
    if (_e != cudaSuccess)                                                                                             \
      ::mgpu::cuda_fail(_e, #expr, __FILE__, __LINE__);                                                                \
  } while (0)

#define MG_ARG(cond, msg)                                                                                              \
  do                                                                                                                   \
  {                                                                                                                    \
    if (!(cond))                                                                                                       \
      throw ::mgpu::Error(MGPU_ERR_ARG, (msg));                                                                        \
  } while (0)

// Device buffer owned by RAII (cudaMallocAsync on the context stream).
// Every device allocation of the library.  Built with -DMGPU_POISON (diagnostics), fresh memory
// is filled with 0xFF bytes (a NaN pattern) so a read of never-written memory cannot pass silently.
inline constexpr bool mg_poison_enabled()
{
#ifdef MGPU_POISON
  return true;
#else
  return false;
#endif
}
inline cudaError_t mg_malloc(void **p, size_t bytes, cudaStream_t s)
{
  const cudaError_t e = cudaMallocAsync(p, bytes, s);
  if (e == cudaSuccess && bytes > 0 && mg_poison_enabled())
    return cudaMemsetAsync(*p, 0xff, bytes, s);
  return e;
}

struct DBuf
{
  void *ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  DBuf() = default;
  DBuf(size_t n, cudaStream_t s) : bytes(n), stream(s)
  {
    if (n > 0)
      MG_CUDA(mg_malloc(&ptr, n, s));
  }
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : ptr(o.ptr), bytes(o.bytes), stream(o.stream) { o.ptr = nullptr; }
  DBuf &operator=(DBuf &&o) noexcept
  {
    release();
    ptr = o.ptr;
    bytes = o.bytes;
    stream = o.stream;
    o.ptr = nullptr;
    return *this;
  }
  ~DBuf() { release(); }
  void release()
  {
    if (ptr)
      cudaFreeAsync(ptr, stream);
    ptr = nullptr;
  }
  template <class T>
  T *as() const
  {
    return static_cast<T *>(ptr);
  }
};

// Raw device CSR view passed to kernels.
struct DCsr
{
  const int64_t *rp;
  const int32_t *ci;
  const double *v;
};

} // namespace mgpu

struct mgpu_ctx
{
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t launches = 0;
  double last_cg_ms = 0.0;
  int64_t last_cg_iters = 0;
  int last_cg_path = 1; // 0 banded (grid), 1 general, 2 cluster v2 (m = 1), 3 cluster v1
  int cg_path = 0;      // 0 auto, 1 force general, 2 force banded grid kernel, 3 cluster v1 only, 4 stream (no cluster)
  long long *prof_dev = nullptr; // diagnostics: per-phase clock64 totals of the CG kernels (MGPU_OPT_PROFILE_PHASES)
  int64_t opt[MGPU_OPT_COUNT] = {0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0}; // mgpu_ctx_set_option
  void *nccl = nullptr;          // ncclComm_t (mgpu_comm_init), one rank per context
  int nranks = 1, rank = 0;
  cudaEvent_t phase_ev[4] = {nullptr, nullptr, nullptr, nullptr}; // mgpu_shifted_solve phase timing (lazy)
  void *pin = nullptr;           // pinned host staging for small device -> host reads (grown on demand)
  size_t pin_bytes = 0;
  // last error
  int last_status = MGPU_OK;
  int64_t err_index = -1, err_col = -1, err_point = -1;
  std::string err_msg;
};

struct mgpu_csr
{
  mgpu_ctx *ctx = nullptr;
  int64_t nrows = 0, ncols = 0, nnz = 0;
  int64_t *row_ptr = nullptr;
  int32_t *col_idx = nullptr;
  double *values = nullptr;
  bool may_hold_zeros = false; // fixed-pattern factors (LS-SPAI) may store exact zeros
  int64_t bw = -1;              // upper bound of max |i - j| over stored entries (-1: unknown)
  int64_t maxrow = -1;          // longest row (-1: unknown)
  // set when row_ptr / col_idx belong to a structure shared by several matrices (the
  // factors of one batched LS-SPAI build): the last owner frees it (stream-ordered)
  std::shared_ptr<void> shared_structure;
  // set when `values` is a slice of one allocation shared by a batch of factors
  std::shared_ptr<void> shared_values;

  mgpu::DCsr view() const { return {row_ptr, col_idx, values}; }
};

namespace mgpu
{

// Counted launch: every kernel of the library goes through here so the bench
// can report how many of OUR kernels ran (mgpu_launch_count).
inline void count_launch(mgpu_ctx *ctx, int k = 1) { ctx->launches += k; }
inline void check_launch(mgpu_ctx *ctx, const char *name)
{
  count_launch(ctx);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error(MGPU_ERR_CUDA, std::string("launch of ") + name + " failed: " + cudaGetErrorString(e));
}

mgpu_csr *new_csr(mgpu_ctx *ctx, int64_t nrows, int64_t ncols, int64_t nnz);
// Bandwidth bound of A (computed once with a reduction kernel when unknown).
int64_t csr_bandwidth(mgpu_ctx *ctx, mgpu_csr *A);
// Longest row of A (cached).
int64_t csr_max_row(mgpu_ctx *ctx, mgpu_csr *A);
void set_error(mgpu_ctx *ctx, const Error &e);

// FP64 GEMM (dense_gemm.cu): C (M x N) = alpha op(A) B + beta C, column-major, op(A) = A^T when
// transA; tall K split across blocks with an in-order partial sum (deterministic).
void gemm(mgpu_ctx *ctx, bool transA, int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda,
          const double *B, int64_t ldb, double beta, double *C, int64_t ldc);

// Deterministic fixed-shape sum of `count` doubles on the device (two-level,
// grid size independent of the device).  Result written to *out_dev.
void det_sum(mgpu_ctx *ctx, const double *vals, int64_t count, double *out_dev);

// Wrap a C entry point: convert exceptions into a status + ctx error payload.
template <class F>
int guard(mgpu_ctx *ctx, F &&body)
{
  try
  {
    if (ctx) // a context may be driven from any host thread (one per device in the multi-device backend)
      MG_CUDA(cudaSetDevice(ctx->device));
    body();
    if (ctx)
    {
      ctx->last_status = MGPU_OK;
    }
    return MGPU_OK;
  }
  catch (const Error &e)
  {
    if (ctx)
      set_error(ctx, e);
    return e.status;
  }
  catch (const std::bad_alloc &)
  {
    if (ctx)
      set_error(ctx, Error(MGPU_ERR_CUDA, "host allocation failed"));
    return MGPU_ERR_CUDA;
  }
  catch (const std::exception &e)
  {
    if (ctx)
      set_error(ctx, Error(MGPU_ERR_CUDA, e.what()));
    return MGPU_ERR_CUDA;
  }
}

constexpr int kThreads = 256;
inline int blocks_for(int64_t n, int threads = kThreads)
{
  int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 1 ? 1 : (b > (1ll << 30) ? (1ll << 30) : b));
}

} // namespace mgpu
