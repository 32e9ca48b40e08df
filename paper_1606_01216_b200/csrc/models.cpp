// Host-side model input for benchmarks and tests (not on the hot path).
//
//   mgpu_model_chain   : the reference's own benchmark family, model_io.cpp:18-87
//   mgpu_model_hermite : BASELINE.json's clamped Euler-Bernoulli cantilever
//                        (SURVEY.md 8(d)), n = 2 * ne after clamping node 0.
//
// Matrices are assembled the way the reference assembles them: triplets ->
// CSR with duplicates summed and exact zeros dropped (sparse.cpp:15-60), and
// D = alpha M + beta K through the union merge of sparse.cpp:167-218.  The
// element coefficient arithmetic is fixed (documented in DESIGN.md) and the
// oracle's generator restates it; tests check both agree bit for bit.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mgpu.h"

namespace
{

struct Trip
{
  int64_t row, col;
  double value;
};

void to_host(int64_t n, const std::vector<int64_t> &rp, const std::vector<int32_t> &ci, const std::vector<double> &v,
             mgpu_host_csr *out)
{
  out->nrows = n;
  out->ncols = n;
  out->nnz = static_cast<int64_t>(v.size());
  out->row_ptr = static_cast<int64_t *>(std::malloc(sizeof(int64_t) * (n + 1)));
  out->col_idx = static_cast<int32_t *>(std::malloc(sizeof(int32_t) * (v.empty() ? 1 : v.size())));
  out->values = static_cast<double *>(std::malloc(sizeof(double) * (v.empty() ? 1 : v.size())));
  std::memcpy(out->row_ptr, rp.data(), sizeof(int64_t) * (n + 1));
  if (!v.empty())
  {
    std::memcpy(out->col_idx, ci.data(), sizeof(int32_t) * v.size());
    std::memcpy(out->values, v.data(), sizeof(double) * v.size());
  }
}

void assemble(int64_t n, std::vector<Trip> t, mgpu_host_csr *out)
{
  std::stable_sort(t.begin(), t.end(), [](const Trip &a, const Trip &b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  std::vector<int64_t> rp(static_cast<size_t>(n + 1), 0);
  std::vector<int32_t> ci;
  std::vector<double> v;
  size_t k = 0;
  for (int64_t i = 0; i < n; ++i)
  {
    while (k < t.size() && t[k].row == i)
    {
      const int64_t col = t[k].col;
      double s = 0.0;
      while (k < t.size() && t[k].row == i && t[k].col == col)
        s += t[k++].value;
      if (s != 0.0)
      {
        ci.push_back(static_cast<int32_t>(col));
        v.push_back(s);
      }
    }
    rp[i + 1] = static_cast<int64_t>(v.size());
  }
  to_host(n, rp, ci, v, out);
}

// a*A + b*B, union pattern, exact zeros dropped.
void add_scaled(const mgpu_host_csr &A, const mgpu_host_csr &B, double a, double b, mgpu_host_csr *out)
{
  const int64_t n = A.nrows;
  std::vector<int64_t> rp(static_cast<size_t>(n + 1), 0);
  std::vector<int32_t> ci;
  std::vector<double> v;
  for (int64_t i = 0; i < n; ++i)
  {
    int64_t ka = A.row_ptr[i], kb = B.row_ptr[i];
    const int64_t ea = A.row_ptr[i + 1], eb = B.row_ptr[i + 1];
    while (ka < ea || kb < eb)
    {
      int32_t col;
      double x;
      if (kb >= eb || (ka < ea && A.col_idx[ka] < B.col_idx[kb]))
      {
        col = A.col_idx[ka];
        x = a * A.values[ka++];
      }
      else if (ka >= ea || B.col_idx[kb] < A.col_idx[ka])
      {
        col = B.col_idx[kb];
        x = b * B.values[kb++];
      }
      else
      {
        col = A.col_idx[ka];
        const double pa = a * A.values[ka++];
        const double pb = b * B.values[kb++];
        x = pa + pb;
      }
      if (x != 0.0)
      {
        ci.push_back(col);
        v.push_back(x);
      }
    }
    rp[i + 1] = static_cast<int64_t>(v.size());
  }
  to_host(n, rp, ci, v, out);
}

} // namespace

extern "C" {

void mgpu_host_free(mgpu_host_csr *a)
{
  if (a == nullptr)
    return;
  std::free(a->row_ptr);
  std::free(a->col_idx);
  std::free(a->values);
  a->row_ptr = nullptr;
  a->col_idx = nullptr;
  a->values = nullptr;
}

int mgpu_model_chain(int64_t n, double alpha, double beta, double stiffness_scale, double mass_scale,
                     int consistent_mass, mgpu_host_csr *M, mgpu_host_csr *D, mgpu_host_csr *K)
{
  if (n < 2 || stiffness_scale <= 0.0 || mass_scale <= 0.0 || !(alpha > 0.0 && alpha < 1.0) ||
      !(beta > 0.0 && beta < 1.0))
    return MGPU_ERR_ARG; // model_io.cpp:20-31
  std::vector<Trip> kt, mt;
  for (int64_t i = 0; i < n; ++i)
  {
    if (i > 0)
      kt.push_back({i, i - 1, -stiffness_scale});
    kt.push_back({i, i, 2.0 * stiffness_scale});
    if (i + 1 < n)
      kt.push_back({i, i + 1, -stiffness_scale});
    if (!consistent_mass)
    {
      mt.push_back({i, i, mass_scale});
      continue;
    }
    if (i > 0)
      mt.push_back({i, i - 1, mass_scale / 6.0});
    mt.push_back({i, i, mass_scale * 2.0 / 3.0});
    if (i + 1 < n)
      mt.push_back({i, i + 1, mass_scale / 6.0});
  }
  assemble(n, std::move(kt), K);
  assemble(n, std::move(mt), M);
  add_scaled(*M, *K, alpha, beta, D);
  return MGPU_OK;
}

int mgpu_model_hermite(int64_t ne, double E, double I, double rho, double area, double L, double alpha, double beta,
                       mgpu_host_csr *M, mgpu_host_csr *D, mgpu_host_csr *K)
{
  if (ne < 1)
    return MGPU_ERR_ARG;
  const int64_t n = 2 * ne;
  const double h = L / static_cast<double>(ne);
  const double kc = (E * I) / (h * h * h);
  const double mc = (rho * area * h) / 420.0;
  const double hh = h * h;
  const double kcoef[4][4] = {{12.0, 6.0 * h, -12.0, 6.0 * h},
                              {6.0 * h, 4.0 * hh, -6.0 * h, 2.0 * hh},
                              {-12.0, -6.0 * h, 12.0, -6.0 * h},
                              {6.0 * h, 2.0 * hh, -6.0 * h, 4.0 * hh}};
  const double mcoef[4][4] = {{156.0, 22.0 * h, 54.0, -13.0 * h},
                              {22.0 * h, 4.0 * hh, 13.0 * h, -3.0 * hh},
                              {54.0, 13.0 * h, 156.0, -22.0 * h},
                              {-13.0 * h, -3.0 * hh, -22.0 * h, 4.0 * hh}};
  std::vector<Trip> kt, mt;
  kt.reserve(static_cast<size_t>(16 * ne));
  mt.reserve(static_cast<size_t>(16 * ne));
  for (int64_t e = 0; e < ne; ++e)
  {
    const int64_t dofs[4] = {2 * e - 2, 2 * e - 1, 2 * e, 2 * e + 1};
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b)
      {
        if (dofs[a] < 0 || dofs[b] < 0)
          continue;
        kt.push_back({dofs[a], dofs[b], kc * kcoef[a][b]});
        mt.push_back({dofs[a], dofs[b], mc * mcoef[a][b]});
      }
  }
  assemble(n, std::move(kt), K);
  assemble(n, std::move(mt), M);
  add_scaled(*M, *K, alpha, beta, D);
  return MGPU_OK;
}

} // extern "C"
