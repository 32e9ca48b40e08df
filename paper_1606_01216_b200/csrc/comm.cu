// NVLink / NCCL data plane of the shift-sharded path.
//
// The l shifted systems are independent: each rank (one process per GPU) assembles, builds the
// SPAI and solves its own shifts with no communication.  Communication happens only after the
// solves, to turn the shift-sharded solution columns into the row-distributed Arnoldi block and to
// form the reduced matrices (airga.cpp:485-500):
//   columns_to_rows: grouped ncclSend / ncclRecv -- rank s sends to rank d the rows
//                    [ext0_d, ext0_d + next_d) (d's slab plus the operator-bandwidth halo) of each
//                    column s holds; d scatters them into its extended slab at the global column ids;
//   project_reduce:  every rank's slab partials V_slab^T (S V), V_slab^T F, C V_slab
//                    (mgpu_project_reduce_slab, on the device) and ONE ncclAllReduce of them.
// Nothing passes through host memory but the column-id bookkeeping (a few integers per column).
#include <dlfcn.h>
#include <nccl.h> // types only: the library is resolved at run time (see Nccl below)

#include <algorithm>
#include <cstring>
#include <numeric>
#include <type_traits>
#include <vector>

#include "internal.cuh"

namespace mgpu
{
namespace
{

// NCCL is bound on first use, not at load time: libmgpu.so must not pull a libnccl.so.2 into a
// process before PyTorch loads its own (a second NCCL of another version under the same soname
// breaks torch's bindings).  The copy already in the process (RTLD_NOLOAD: torch's, under
// torch.distributed) is preferred; otherwise the system libnccl.so.2.
struct Nccl
{
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const Nccl &nccl()
{
  static const Nccl lib = [] {
    Nccl n;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h)
      return n;
    auto sym = [&](auto &fp, const char *name) { fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name)); };
    sym(n.GetUniqueId, "ncclGetUniqueId");
    sym(n.CommInitRank, "ncclCommInitRank");
    sym(n.CommDestroy, "ncclCommDestroy");
    sym(n.AllReduce, "ncclAllReduce");
    sym(n.AllGather, "ncclAllGather");
    sym(n.Send, "ncclSend");
    sym(n.Recv, "ncclRecv");
    sym(n.GroupStart, "ncclGroupStart");
    sym(n.GroupEnd, "ncclGroupEnd");
    sym(n.GetErrorString, "ncclGetErrorString");
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllReduce && n.AllGather && n.Send && n.Recv &&
           n.GroupStart && n.GroupEnd && n.GetErrorString;
    return n;
  }();
  if (!lib.ok)
    throw Error(MGPU_ERR_NCCL, "NCCL (libnccl.so.2) not available");
  return lib;
}

#define MG_NCCL(fn, ...)                                                                                               \
  do                                                                                                                   \
  {                                                                                                                    \
    const ::mgpu::Nccl &_n = ::mgpu::nccl();                                                                           \
    ncclResult_t _r = _n.fn(__VA_ARGS__);                                                                              \
    if (_r != ncclSuccess)                                                                                             \
      throw ::mgpu::Error(MGPU_ERR_NCCL, std::string("nccl" #fn ": ") + _n.GetErrorString(_r));                       \
  } while (0)

ncclComm_t comm_of(mgpu_ctx *ctx)
{
  MG_ARG(ctx->nccl != nullptr, "comm: no communicator on this context (mgpu_comm_init)");
  return static_cast<ncclComm_t>(ctx->nccl);
}

// Balanced row slab of `rank` and its halo-extended range, clipped to [0, n).
void slab_of(int64_t n, int nranks, int rank, int64_t h, int64_t &r0, int64_t &p, int64_t &e0, int64_t &ne)
{
  r0 = n * rank / nranks;
  const int64_t r1 = n * (rank + 1) / nranks;
  p = r1 - r0;
  e0 = std::max<int64_t>(0, r0 - h);
  ne = std::min<int64_t>(n, r1 + h) - e0;
}

// dst[:, c] (ld_dst) <- src block column j (ld_src = rows) for j < cols, dst column = map[j]
__global__ void scatter_cols(int64_t rows, int64_t cols, const double *__restrict__ src, const int64_t *__restrict__ map,
                             double *__restrict__ dst, int64_t ld_dst)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * cols)
    return;
  const int64_t j = t / rows, i = t - j * rows;
  dst[map[j] * ld_dst + i] = src[t];
}

// CSR rows [r0, r0 + p) of A with global column indices (row_ptr rebased)
__global__ void rebase_rows(int64_t p, const int64_t *__restrict__ rp, int64_t r0, int64_t *__restrict__ out)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i <= p)
    out[i] = rp[r0 + i] - rp[r0];
}

mgpu_csr *row_slab(mgpu_ctx *ctx, const mgpu_csr *A, int64_t r0, int64_t p)
{
  int64_t b[2] = {0, 0};
  MG_CUDA(cudaMemcpyAsync(&b[0], A->row_ptr + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA(cudaMemcpyAsync(&b[1], A->row_ptr + r0 + p, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
  const int64_t nnz = b[1] - b[0];
  mgpu_csr *S = new_csr(ctx, p, A->ncols, nnz);
  rebase_rows<<<blocks_for(p + 1), kThreads, 0, ctx->stream>>>(p, A->row_ptr, r0, S->row_ptr);
  check_launch(ctx, "rebase_rows");
  if (nnz > 0)
  {
    MG_CUDA(cudaMemcpyAsync(S->col_idx, A->col_idx + b[0], sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice,
                            ctx->stream));
    MG_CUDA(cudaMemcpyAsync(S->values, A->values + b[0], sizeof(double) * nnz, cudaMemcpyDeviceToDevice,
                            ctx->stream));
  }
  S->bw = A->bw;
  return S;
}

} // namespace
} // namespace mgpu

using namespace mgpu;

extern "C" {

int mgpu_comm_unique_id(void *id)
{
  if (id == nullptr)
    return MGPU_ERR_ARG;
  try
  {
    ncclUniqueId u;
    if (nccl().GetUniqueId(&u) != ncclSuccess)
      return MGPU_ERR_NCCL;
    std::memcpy(id, &u, sizeof u);
    return MGPU_OK;
  }
  catch (const Error &)
  {
    return MGPU_ERR_NCCL;
  }
}

int mgpu_comm_init(mgpu_ctx *ctx, const void *id, int nranks, int rank)
{
  if (ctx == nullptr)
    return MGPU_ERR_ARG;
  return guard(ctx, [&] {
    MG_ARG(id != nullptr && nranks >= 1 && rank >= 0 && rank < nranks, "comm_init: bad argument");
    MG_ARG(ctx->nccl == nullptr, "comm_init: the context already has a communicator");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclComm_t c = nullptr;
    MG_CUDA(cudaSetDevice(ctx->device));
    MG_NCCL(CommInitRank, &c, nranks, u, rank);
    ctx->nccl = c;
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

int mgpu_comm_destroy(mgpu_ctx *ctx)
{
  if (ctx == nullptr)
    return MGPU_ERR_ARG;
  return guard(ctx, [&] {
    if (ctx->nccl)
    {
      MG_CUDA(cudaStreamSynchronize(ctx->stream));
      MG_NCCL(CommDestroy, static_cast<ncclComm_t>(ctx->nccl));
    }
    ctx->nccl = nullptr;
    ctx->nranks = 1;
    ctx->rank = 0;
  });
}

int mgpu_comm_allreduce_sum(mgpu_ctx *ctx, double *buf, int64_t count)
{
  if (ctx == nullptr)
    return MGPU_ERR_ARG;
  return guard(ctx, [&] {
    MG_ARG(buf != nullptr || count == 0, "comm_allreduce: null buffer");
    if (count > 0)
      MG_NCCL(AllReduce, buf, buf, static_cast<size_t>(count), ncclDouble, ncclSum, comm_of(ctx), ctx->stream);
    MG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mgpu_comm_rows(mgpu_ctx *ctx, int64_t n, int64_t h, int64_t *row0, int64_t *p, int64_t *ext0, int64_t *next)
{
  if (ctx == nullptr || row0 == nullptr || p == nullptr || ext0 == nullptr || next == nullptr || n < 0 || h < 0)
    return MGPU_ERR_ARG;
  slab_of(n, ctx->nranks, ctx->rank, h, *row0, *p, *ext0, *next);
  return MGPU_OK;
}

int mgpu_comm_columns_to_rows(mgpu_ctx *ctx, int64_t n, int64_t h, int64_t c_local, const int64_t *col_ids,
                              const double *X_local, int64_t R, double *Vext)
{
  if (ctx == nullptr)
    return MGPU_ERR_ARG;
  return guard(ctx, [&] {
    MG_ARG(n >= 0 && h >= 0 && c_local >= 0 && R >= 0 && (c_local == 0 || (col_ids && X_local)) && (R == 0 || Vext),
           "comm_columns_to_rows: bad argument");
    ncclComm_t comm = comm_of(ctx);
    const int W = ctx->nranks, me = ctx->rank;
    cudaStream_t s = ctx->stream;
    // every rank's column count and ids (small all-gathers of integers, on the device)
    DBuf cnt_d(sizeof(int64_t) * W, s);
    int64_t mine = c_local;
    MG_CUDA(cudaMemcpyAsync(cnt_d.as<int64_t>() + me, &mine, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    MG_NCCL(AllGather, cnt_d.as<int64_t>() + me, cnt_d.ptr, 1, ncclInt64, comm, s);
    std::vector<int64_t> cnt(static_cast<size_t>(W));
    MG_CUDA(cudaMemcpyAsync(cnt.data(), cnt_d.ptr, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    const int64_t cmax = *std::max_element(cnt.begin(), cnt.end());
    MG_ARG(std::accumulate(cnt.begin(), cnt.end(), int64_t{0}) == R, "comm_columns_to_rows: column counts do not sum to R");
    DBuf ids_d(sizeof(int64_t) * static_cast<size_t>(W) * (cmax > 0 ? cmax : 1), s);
    {
      std::vector<int64_t> pad(static_cast<size_t>(cmax > 0 ? cmax : 1), -1);
      std::copy(col_ids, col_ids + c_local, pad.begin());
      MG_CUDA(cudaMemcpyAsync(ids_d.as<int64_t>() + me * cmax, pad.data(), sizeof(int64_t) * cmax,
                              cudaMemcpyHostToDevice, s));
      if (cmax > 0)
        MG_NCCL(AllGather, ids_d.as<int64_t>() + me * cmax, ids_d.ptr, static_cast<size_t>(cmax), ncclInt64, comm, s);
    }
    int64_t r0, p, e0, ne;
    slab_of(n, W, me, h, r0, p, e0, ne);
    // send buffers: for each destination d, its extended rows of my columns (ne_d x c_local)
    std::vector<int64_t> se0(W), sne(W), soff(W + 1, 0);
    for (int d = 0; d < W; ++d)
    {
      int64_t a, b;
      slab_of(n, W, d, h, a, b, se0[d], sne[d]);
      soff[d + 1] = soff[d] + sne[d] * c_local;
    }
    DBuf sbuf(sizeof(double) * static_cast<size_t>(soff[W] > 0 ? soff[W] : 1), s);
    for (int d = 0; d < W; ++d)
      if (sne[d] > 0 && c_local > 0)
        MG_CUDA(cudaMemcpy2DAsync(sbuf.as<double>() + soff[d], sizeof(double) * sne[d], X_local + se0[d],
                                  sizeof(double) * n, sizeof(double) * sne[d], c_local, cudaMemcpyDeviceToDevice, s));
    // receive buffers: from each source s2, my extended rows of its columns (ne x cnt[s2])
    std::vector<int64_t> roff(W + 1, 0);
    for (int q = 0; q < W; ++q)
      roff[q + 1] = roff[q] + ne * cnt[q];
    DBuf rbuf(sizeof(double) * static_cast<size_t>(roff[W] > 0 ? roff[W] : 1), s);
    MG_NCCL(GroupStart);
    for (int d = 0; d < W; ++d)
      if (sne[d] * c_local > 0)
        MG_NCCL(Send, sbuf.as<double>() + soff[d], static_cast<size_t>(sne[d] * c_local), ncclDouble, d, comm, s);
    for (int q = 0; q < W; ++q)
      if (ne * cnt[q] > 0)
        MG_NCCL(Recv, rbuf.as<double>() + roff[q], static_cast<size_t>(ne * cnt[q]), ncclDouble, q, comm, s);
    MG_NCCL(GroupEnd);
    // scatter every source's block into Vext at its global column ids
    for (int q = 0; q < W; ++q)
      if (ne * cnt[q] > 0)
      {
        scatter_cols<<<blocks_for(ne * cnt[q]), kThreads, 0, s>>>(ne, cnt[q], rbuf.as<double>() + roff[q],
                                                                   ids_d.as<int64_t>() + q * cmax, Vext, ne);
        check_launch(ctx, "scatter_cols");
      }
    MG_CUDA(cudaStreamSynchronize(s));
  });
}

int mgpu_comm_project_reduce(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int64_t h,
                             int64_t r, const double *Vext, int64_t m, const double *F, int64_t q, const double *Cp,
                             const double *Cv, double *Mh, double *Dh, double *Kh, double *Fh, double *Cph,
                             double *Cvh, mgpu_memkind where)
{
  if (ctx == nullptr)
    return MGPU_ERR_ARG;
  mgpu_csr *sl[3] = {nullptr, nullptr, nullptr};
  const int st = guard(ctx, [&] {
    MG_ARG(M && D && K && Vext && Mh && Dh && Kh && r >= 0 && m >= 0 && q >= 0 && h >= 0,
           "comm_project_reduce: null argument");
    MG_ARG(where == MGPU_HOST || where == MGPU_DEVICE, "comm_project_reduce: bad memory kind");
    MG_ARG(m == 0 || (F && Fh), "comm_project_reduce: F / Fh missing");
    MG_ARG(q == 0 || (Cp && Cv && Cph && Cvh), "comm_project_reduce: Cp / Cv missing");
    const int64_t n = M->nrows;
    for (const mgpu_csr *S : {M, D, K})
      MG_ARG(S->nrows == n && S->ncols == n && csr_bandwidth(ctx, const_cast<mgpu_csr *>(S)) <= h,
             "comm_project_reduce: operators must be n x n with bandwidth <= h");
    int64_t r0, p, e0, ne;
    slab_of(n, ctx->nranks, ctx->rank, h, r0, p, e0, ne);
    cudaStream_t s = ctx->stream;
    const mgpu_csr *full[3] = {M, D, K};
    for (int k = 0; k < 3; ++k)
      sl[k] = row_slab(ctx, full[k], r0, p);
    // this slab's partials, packed for one all-reduce: Mh Dh Kh (r x r), Fh (r x m), Cph Cvh (q x r)
    const int64_t tot = 3 * r * r + r * m + 2 * q * r;
    DBuf part(sizeof(double) * static_cast<size_t>(tot > 0 ? tot : 1), s);
    double *P = part.as<double>();
    DBuf Fs(sizeof(double) * static_cast<size_t>(p * m > 0 ? p * m : 1), s);
    if (m > 0 && p > 0) // rows [r0, r0 + p) of the n x m input block (device copy of the slab)
      MG_CUDA(cudaMemcpy2DAsync(Fs.ptr, sizeof(double) * p, F + r0, sizeof(double) * n, sizeof(double) * p, m,
                                where == MGPU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    DBuf Cs(sizeof(double) * static_cast<size_t>(2 * q * p > 0 ? 2 * q * p : 1), s);
    if (q > 0 && p > 0) // columns [r0, r0 + p) of the q x n output maps
    {
      const cudaMemcpyKind kd = where == MGPU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
      MG_CUDA(cudaMemcpyAsync(Cs.ptr, Cp + r0 * q, sizeof(double) * q * p, kd, s));
      MG_CUDA(cudaMemcpyAsync(Cs.as<double>() + q * p, Cv + r0 * q, sizeof(double) * q * p, kd, s));
    }
    const int st2 = mgpu_project_reduce_slab(ctx, sl[0], sl[1], sl[2], r0, e0, ne, r, Vext, m, Fs.as<double>(), q,
                                             Cs.as<double>(), Cs.as<double>() + q * p, P, P + r * r, P + 2 * r * r,
                                             P + 3 * r * r, P + 3 * r * r + r * m, P + 3 * r * r + r * m + q * r,
                                             MGPU_DEVICE);
    if (st2 != MGPU_OK)
      throw Error(st2, ctx->err_msg, ctx->err_index, ctx->err_col, ctx->err_point);
    if (tot > 0)
      MG_NCCL(AllReduce, P, P, static_cast<size_t>(tot), ncclDouble, ncclSum, comm_of(ctx), s);
    double *outs[6] = {Mh, Dh, Kh, Fh, Cph, Cvh};
    const int64_t sizes[6] = {r * r, r * r, r * r, r * m, q * r, q * r};
    int64_t o = 0;
    for (int k = 0; k < 6; ++k)
    {
      if (sizes[k] > 0)
        MG_CUDA(cudaMemcpyAsync(outs[k], P + o, sizeof(double) * sizes[k],
                                where == MGPU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
      o += sizes[k];
    }
    MG_CUDA(cudaStreamSynchronize(s));
  });
  for (auto *x : sl)
    mgpu_csr_free(x);
  return st;
}

int mgpu_csr_bandwidth(mgpu_ctx *ctx, const mgpu_csr *a, int64_t *bw)
{
  if (ctx == nullptr)
    return MGPU_ERR_ARG;
  return guard(ctx, [&] {
    MG_ARG(a && bw, "csr_bandwidth: null argument");
    *bw = csr_bandwidth(ctx, const_cast<mgpu_csr *>(a));
  });
}

} // extern "C"
