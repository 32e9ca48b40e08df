// Binary CSR sidecar.  The reference's interchange is
// Matrix Market text (model_io.cpp:154-351): gigabytes of text and a
// from_triplets sort at n = 1e7.  This is a flat little-endian dump of the
// reference's CSR arrays (sparse.hpp:18-22) that loads straight into device
// memory through the validated upload path:
//
//   bytes 0..7   magic "MGCSR\0\0\1"
//   int64        nrows, ncols, nnz
//   int64[nrows + 1] row_ptr, int32[nnz] col_idx, float64[nnz] values
//
// What is written is the download view (mgpu_csr_download): exact zeros a
// fixed-pattern factor stores are dropped, as the reference stores them.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.cuh"

namespace
{
constexpr char kMagic[8] = {'M', 'G', 'C', 'S', 'R', 0, 0, 1};

struct File
{
  std::FILE *f = nullptr;
  File(const char *path, const char *mode) : f(std::fopen(path, mode)) {}
  ~File()
  {
    if (f)
      std::fclose(f);
  }
};
} // namespace

using namespace mgpu;

extern "C" {

int mgpu_csr_write(mgpu_ctx *ctx, const mgpu_csr *a, const char *path)
{
  return guard(ctx, [&] {
    MG_ARG(a && path, "csr_write: null argument");
    int64_t nr = 0, nc = 0, nnz = 0;
    const int st = mgpu_csr_info(ctx, a, &nr, &nc, &nnz);
    if (st != MGPU_OK)
      throw Error(st, ctx->err_msg);
    std::vector<int64_t> rp(static_cast<size_t>(nr + 1));
    std::vector<int32_t> ci(static_cast<size_t>(nnz > 0 ? nnz : 1));
    std::vector<double> v(static_cast<size_t>(nnz > 0 ? nnz : 1));
    const int st2 = mgpu_csr_download(ctx, a, rp.data(), ci.data(), v.data());
    if (st2 != MGPU_OK)
      throw Error(st2, ctx->err_msg);
    File out(path, "wb");
    if (!out.f)
      throw Error(MGPU_ERR_ARG, std::string("csr_write: cannot open ") + path);
    const int64_t hdr[3] = {nr, nc, nnz};
    bool ok = std::fwrite(kMagic, 1, 8, out.f) == 8 && std::fwrite(hdr, sizeof(int64_t), 3, out.f) == 3 &&
              std::fwrite(rp.data(), sizeof(int64_t), rp.size(), out.f) == rp.size();
    if (nnz > 0)
      ok = ok && std::fwrite(ci.data(), sizeof(int32_t), static_cast<size_t>(nnz), out.f) == static_cast<size_t>(nnz) &&
           std::fwrite(v.data(), sizeof(double), static_cast<size_t>(nnz), out.f) == static_cast<size_t>(nnz);
    if (!ok)
      throw Error(MGPU_ERR_ARG, std::string("csr_write: short write to ") + path);
  });
}

int mgpu_csr_read(mgpu_ctx *ctx, const char *path, mgpu_csr **out)
{
  return guard(ctx, [&] {
    MG_ARG(path && out, "csr_read: null argument");
    File in(path, "rb");
    if (!in.f)
      throw Error(MGPU_ERR_ARG, std::string("csr_read: cannot open ") + path);
    char magic[8];
    int64_t hdr[3];
    if (std::fread(magic, 1, 8, in.f) != 8 || std::memcmp(magic, kMagic, 8) != 0)
      throw Error(MGPU_ERR_ARG, std::string("csr_read: not a binary CSR file: ") + path);
    if (std::fread(hdr, sizeof(int64_t), 3, in.f) != 3 || hdr[0] < 0 || hdr[1] < 0 || hdr[2] < 0)
      throw Error(MGPU_ERR_ARG, std::string("csr_read: bad header in ") + path);
    const int64_t nr = hdr[0], nc = hdr[1], nnz = hdr[2];
    // arrays staged in pinned memory so the upload runs at full PCIe rate
    const size_t bytes = sizeof(int64_t) * (nr + 1) + (sizeof(int32_t) + sizeof(double)) * static_cast<size_t>(nnz);
    void *pinned = nullptr;
    MG_CUDA(cudaMallocHost(&pinned, bytes > 0 ? bytes : 1));
    std::unique_ptr<void, decltype(&cudaFreeHost)> hold(pinned, &cudaFreeHost);
    auto *rp = static_cast<int64_t *>(pinned);
    auto *v = reinterpret_cast<double *>(rp + nr + 1);
    auto *ci = reinterpret_cast<int32_t *>(v + nnz);
    if (std::fread(rp, sizeof(int64_t), static_cast<size_t>(nr + 1), in.f) != static_cast<size_t>(nr + 1) ||
        std::fread(ci, sizeof(int32_t), static_cast<size_t>(nnz), in.f) != static_cast<size_t>(nnz) ||
        std::fread(v, sizeof(double), static_cast<size_t>(nnz), in.f) != static_cast<size_t>(nnz))
      throw Error(MGPU_ERR_ARG, std::string("csr_read: truncated file ") + path);
    const int st = mgpu_csr_upload(ctx, nr, nc, nnz, rp, ci, v, out); // validates the CSR invariants
    if (st != MGPU_OK)
      throw Error(st, ctx->err_msg);
    MG_CUDA(cudaStreamSynchronize(ctx->stream)); // the pinned staging buffer is released below
  });
}

} // extern "C"
