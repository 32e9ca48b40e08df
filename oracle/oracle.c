/* TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.
 * See oracle.h for the pinning story.  Compiled with -ffp-contract=off so every
 * a*b+c is two roundings, like the reference TUs built without -mfma; dot /
 * axpy / gather_dot follow the reference's SCALAR kernel table
 * (kernels_scalar.cpp:13-47: one accumulator, ascending index), which is the
 * canonical oracle variant (MOR_KERNELS=scalar). */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- helpers */

static void set_err(orc_err *err, int64_t index, const char *msg)
{
  if (err)
  {
    err->index = index;
    snprintf(err->msg, sizeof err->msg, "%s", msg);
  }
}

static void clear_err(orc_err *err)
{
  if (err)
  {
    err->index = -1;
    err->msg[0] = '\0';
  }
}

static void csr_alloc(orc_csr *a, int64_t nrows, int64_t ncols, int64_t cap)
{
  a->nrows = nrows;
  a->ncols = ncols;
  a->nnz = 0;
  a->row_ptr = (int64_t *)calloc((size_t)nrows + 1, sizeof(int64_t));
  a->col_idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
  a->values = (double *)malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
}

void orc_csr_free(orc_csr *a)
{
  free(a->row_ptr);
  free(a->col_idx);
  free(a->values);
  a->row_ptr = NULL;
  a->col_idx = NULL;
  a->values = NULL;
}

/* kernels_scalar.cpp:13-21 */
static double dot_s(const double *x, const double *y, int64_t n)
{
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i)
    acc += x[i] * y[i];
  return acc;
}

/* kernels_scalar.cpp:23-29 */
static void axpy_s(int64_t n, double a, const double *x, double *y)
{
  for (int64_t i = 0; i < n; ++i)
    y[i] += a * x[i];
}

/* ---------------------------------------------------------------- CSR core */

typedef struct trip
{
  int64_t row, col;
  double value;
  int64_t seq;
} trip;

static int trip_cmp(const void *pa, const void *pb)
{
  const trip *a = (const trip *)pa, *b = (const trip *)pb;
  if (a->row != b->row)
    return a->row < b->row ? -1 : 1;
  if (a->col != b->col)
    return a->col < b->col ? -1 : 1;
  /* duplicates: the reference's std::sort is unstable; every caller here has
   * at most two duplicates, whose sum is order independent. */
  return a->seq < b->seq ? -1 : (a->seq > b->seq);
}

/* sparse.cpp:15-60: sort, sum duplicates, drop exact zeros. */
int orc_from_triplets(int64_t nrows, int64_t ncols, int64_t count, const int64_t *rows, const int64_t *cols,
                      const double *vals, orc_csr *out, orc_err *err)
{
  clear_err(err);
  if (nrows < 0 || ncols < 0)
  {
    set_err(err, -1, "from_triplets: negative dimension");
    return ORC_ERR_ARG;
  }
  trip *t = (trip *)malloc(sizeof(trip) * (size_t)(count > 0 ? count : 1));
  for (int64_t k = 0; k < count; ++k)
  {
    if (rows[k] < 0 || rows[k] >= nrows || cols[k] < 0 || cols[k] >= ncols)
    {
      free(t);
      set_err(err, -1, "from_triplets: entry index out of range");
      return ORC_ERR_ARG;
    }
    t[k].row = rows[k];
    t[k].col = cols[k];
    t[k].value = vals[k];
    t[k].seq = k;
  }
  qsort(t, (size_t)count, sizeof(trip), trip_cmp);
  csr_alloc(out, nrows, ncols, count);
  int64_t k = 0, nz = 0;
  for (int64_t i = 0; i < nrows; ++i)
  {
    while (k < count && t[k].row == i)
    {
      const int64_t col = t[k].col;
      double v = 0.0;
      while (k < count && t[k].row == i && t[k].col == col)
      {
        v += t[k].value;
        ++k;
      }
      if (v != 0.0)
      {
        out->col_idx[nz] = (int32_t)col;
        out->values[nz] = v;
        ++nz;
      }
    }
    out->row_ptr[i + 1] = nz;
  }
  out->nnz = nz;
  free(t);
  return ORC_OK;
}

/* sparse.cpp:167-218: union merge, a*A + b*B on shared slots, drop exact zeros. */
int orc_sp_add_scaled(const orc_csr *A, const orc_csr *B, double a, double b, orc_csr *out, orc_err *err)
{
  clear_err(err);
  if (A->nrows != B->nrows || A->ncols != B->ncols)
  {
    set_err(err, -1, "sp_add_scaled: shape mismatch");
    return ORC_ERR_ARG;
  }
  csr_alloc(out, A->nrows, A->ncols, A->nnz + B->nnz);
  int64_t nz = 0;
  for (int64_t i = 0; i < A->nrows; ++i)
  {
    int64_t ka = A->row_ptr[i], kb = B->row_ptr[i];
    const int64_t ea = A->row_ptr[i + 1], eb = B->row_ptr[i + 1];
    while (ka < ea || kb < eb)
    {
      int32_t col;
      double v;
      if (kb >= eb || (ka < ea && A->col_idx[ka] < B->col_idx[kb]))
      {
        col = A->col_idx[ka];
        v = a * A->values[ka];
        ++ka;
      }
      else if (ka >= ea || B->col_idx[kb] < A->col_idx[ka])
      {
        col = B->col_idx[kb];
        v = b * B->values[kb];
        ++kb;
      }
      else
      {
        col = A->col_idx[ka];
        v = a * A->values[ka] + b * B->values[kb];
        ++ka;
        ++kb;
      }
      if (v != 0.0)
      {
        out->col_idx[nz] = col;
        out->values[nz] = v;
        ++nz;
      }
    }
    out->row_ptr[i + 1] = nz;
  }
  out->nnz = nz;
  return ORC_OK;
}

/* system.cpp:64-68: (s^2 M + s D) first, then + K. */
int orc_shifted_operator(const orc_csr *M, const orc_csr *D, const orc_csr *K, double s, orc_csr *out, orc_err *err)
{
  orc_csr md;
  int st = orc_sp_add_scaled(M, D, s * s, s, &md, err);
  if (st != ORC_OK)
    return st;
  st = orc_sp_add_scaled(&md, K, 1.0, 1.0, out, err);
  orc_csr_free(&md);
  return st;
}

/* sparse.cpp:220-249: counting transpose, rows visited ascending. */
int orc_transpose(const orc_csr *A, orc_csr *T)
{
  csr_alloc(T, A->ncols, A->nrows, A->nnz);
  T->nnz = A->nnz;
  for (int64_t k = 0; k < A->nnz; ++k)
    T->row_ptr[A->col_idx[k] + 1]++;
  for (int64_t i = 1; i <= A->ncols; ++i)
    T->row_ptr[i] += T->row_ptr[i - 1];
  int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(A->ncols > 0 ? A->ncols : 1));
  memcpy(next, T->row_ptr, sizeof(int64_t) * (size_t)A->ncols);
  for (int64_t i = 0; i < A->nrows; ++i)
    for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k)
    {
      const int64_t slot = next[A->col_idx[k]]++;
      T->col_idx[slot] = (int32_t)i;
      T->values[slot] = A->values[k];
    }
  free(next);
  return ORC_OK;
}

/* sparse.cpp:92-106 */
static double csr_at(const orc_csr *A, int64_t i, int64_t j)
{
  int64_t lo = A->row_ptr[i], hi = A->row_ptr[i + 1];
  while (lo < hi)
  {
    const int64_t mid = lo + (hi - lo) / 2;
    if (A->col_idx[mid] < j)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < A->row_ptr[i + 1] && A->col_idx[lo] == j) ? A->values[lo] : 0.0;
}

/* sparse.cpp:251-260 */
double orc_trace(const orc_csr *A)
{
  double t = 0.0;
  const int64_t n = A->nrows < A->ncols ? A->nrows : A->ncols;
  for (int64_t i = 0; i < n; ++i)
    t += csr_at(A, i, i);
  return t;
}

/* sparse.cpp:262-296: row-major merge over the intersecting pattern. */
double orc_trace_inner(const orc_csr *A, const orc_csr *B)
{
  double acc = 0.0;
  for (int64_t i = 0; i < A->nrows; ++i)
  {
    int64_t ka = A->row_ptr[i], kb = B->row_ptr[i];
    const int64_t ea = A->row_ptr[i + 1], eb = B->row_ptr[i + 1];
    while (ka < ea && kb < eb)
    {
      const int32_t ca = A->col_idx[ka], cb = B->col_idx[kb];
      if (ca < cb)
        ++ka;
      else if (cb < ca)
        ++kb;
      else
      {
        acc += A->values[ka] * B->values[kb];
        ++ka;
        ++kb;
      }
    }
  }
  return acc;
}

/* sparse.cpp:140-158 + kernels_scalar.cpp:39-47 (in-order gather dot per row). */
void orc_spmv(const orc_csr *A, const double *x, double *y)
{
  for (int64_t i = 0; i < A->nrows; ++i)
  {
    double acc = 0.0;
    for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k)
      acc += A->values[k] * x[A->col_idx[k]];
    y[i] = acc;
  }
}

/* ---------------------------------------------------------------- models */

/* model_io.cpp:18-87 */
int orc_chain_generate(int64_t n, double alpha, double beta, double stiffness_scale, double mass_scale,
                       int consistent_mass, orc_csr *M, orc_csr *D, orc_csr *K, orc_err *err)
{
  clear_err(err);
  if (n < 2)
  {
    set_err(err, -1, "beam_generate: n must be at least 2");
    return ORC_ERR_ARG;
  }
  if (stiffness_scale <= 0.0 || mass_scale <= 0.0)
  {
    set_err(err, -1, "beam_generate: scales must be positive");
    return ORC_ERR_ARG;
  }
  if (!(alpha > 0.0 && alpha < 1.0 && beta > 0.0 && beta < 1.0))
  {
    set_err(err, -1, "beam_generate: alpha and beta must lie in (0, 1)");
    return ORC_ERR_ARG;
  }
  const int64_t cap = 3 * n;
  int64_t *r = (int64_t *)malloc(sizeof(int64_t) * cap);
  int64_t *c = (int64_t *)malloc(sizeof(int64_t) * cap);
  double *v = (double *)malloc(sizeof(double) * cap);
  int64_t t = 0;
  for (int64_t i = 0; i < n; ++i)
  {
    if (i > 0)
    {
      r[t] = i; c[t] = i - 1; v[t++] = -stiffness_scale;
    }
    r[t] = i; c[t] = i; v[t++] = 2.0 * stiffness_scale;
    if (i + 1 < n)
    {
      r[t] = i; c[t] = i + 1; v[t++] = -stiffness_scale;
    }
  }
  orc_from_triplets(n, n, t, r, c, v, K, err);
  t = 0;
  for (int64_t i = 0; i < n; ++i)
  {
    if (!consistent_mass)
    {
      r[t] = i; c[t] = i; v[t++] = mass_scale;
      continue;
    }
    if (i > 0)
    {
      r[t] = i; c[t] = i - 1; v[t++] = mass_scale / 6.0;
    }
    r[t] = i; c[t] = i; v[t++] = mass_scale * 2.0 / 3.0;
    if (i + 1 < n)
    {
      r[t] = i; c[t] = i + 1; v[t++] = mass_scale / 6.0;
    }
  }
  orc_from_triplets(n, n, t, r, c, v, M, err);
  free(r);
  free(c);
  free(v);
  return orc_sp_add_scaled(M, K, alpha, beta, D, err);
}

/* Hermite cantilever.  Element coefficient arithmetic is
 * fixed here and restated identically by the product generator
 * (paper_1606_01216_b200/csrc/models.cpp); tests check they agree bitwise. */
int orc_hermite_generate(int64_t ne, double E, double I, double rho, double area, double L, double alpha, double beta,
                         orc_csr *M, orc_csr *D, orc_csr *K, orc_err *err)
{
  clear_err(err);
  if (ne < 1)
  {
    set_err(err, -1, "hermite_generate: need at least one element");
    return ORC_ERR_ARG;
  }
  const int64_t n = 2 * ne;
  const double h = L / (double)ne;
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
  const int64_t cap = 16 * ne;
  int64_t *r = (int64_t *)malloc(sizeof(int64_t) * cap);
  int64_t *c = (int64_t *)malloc(sizeof(int64_t) * cap);
  double *kv = (double *)malloc(sizeof(double) * cap);
  double *mv = (double *)malloc(sizeof(double) * cap);
  int64_t t = 0;
  for (int64_t e = 0; e < ne; ++e)
  {
    const int64_t dofs[4] = {2 * e - 2, 2 * e - 1, 2 * e, 2 * e + 1};
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b)
      {
        if (dofs[a] < 0 || dofs[b] < 0)
          continue;
        r[t] = dofs[a];
        c[t] = dofs[b];
        kv[t] = kc * kcoef[a][b];
        mv[t] = mc * mcoef[a][b];
        ++t;
      }
  }
  orc_from_triplets(n, n, t, r, c, kv, K, err);
  orc_from_triplets(n, n, t, r, c, mv, M, err);
  free(r);
  free(c);
  free(kv);
  free(mv);
  return orc_sp_add_scaled(M, K, alpha, beta, D, err);
}

/* ---------------------------------------------------------------- MR-SPAI */

/* Sparse accumulator (spai.cpp:22-68): dense values, membership, support list.
 * Allocated once per build and cleared in O(support) -- identical values and
 * summation order to the reference's per-column Spa(n). */
typedef struct spa
{
  double *val;
  char *in;
  int64_t *idx;
  int64_t len;
} spa;

static void spa_init(spa *s, int64_t n)
{
  s->val = (double *)calloc((size_t)n, sizeof(double));
  s->in = (char *)calloc((size_t)n, 1);
  s->idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  s->len = 0;
}
static void spa_free(spa *s)
{
  free(s->val);
  free(s->in);
  free(s->idx);
}
static void spa_add(spa *s, int64_t i, double v)
{
  if (!s->in[i])
  {
    s->in[i] = 1;
    s->idx[s->len++] = i;
  }
  s->val[i] += v;
}
static void spa_clear(spa *s)
{
  for (int64_t k = 0; k < s->len; ++k)
  {
    s->val[s->idx[k]] = 0.0;
    s->in[s->idx[k]] = 0;
  }
  s->len = 0;
}
static int cmp_i64(const void *a, const void *b)
{
  const int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return x < y ? -1 : (x > y);
}
static void spa_sort(spa *s) { qsort(s->idx, (size_t)s->len, sizeof(int64_t), cmp_i64); }
/* spai.cpp:53-62 */
static double spa_norm_sq_sorted(spa *s)
{
  spa_sort(s);
  double acc = 0.0;
  for (int64_t k = 0; k < s->len; ++k)
    acc += s->val[s->idx[k]] * s->val[s->idx[k]];
  return acc;
}
/* spai.cpp:70-80 */
static double spa_dot(spa *a, const spa *b)
{
  spa_sort(a);
  double acc = 0.0;
  for (int64_t k = 0; k < a->len; ++k)
    acc += a->val[a->idx[k]] * b->val[a->idx[k]];
  return acc;
}
/* spai.cpp:88-95: out += a * column j of the operand (row j of its transpose). */
static void axpy_col(const orc_csr *T, double a, int64_t j, spa *out)
{
  for (int64_t k = T->row_ptr[j]; k < T->row_ptr[j + 1]; ++k)
    spa_add(out, T->col_idx[k], a * T->values[k]);
}

typedef struct colstore
{
  int64_t *len;
  int64_t **row;
  double **val;
  char *built;
} colstore;

/* spai.cpp:113-209 (build_column) */
static int build_column(int64_t j, double alpha, const orc_csr *Kt, const orc_csr *rhs_t, double tol,
                        int64_t max_col_iters, int mode, colstore *store, spa *p, spa *r, spa *d, spa *w,
                        double *final_res, orc_err *err)
{
  char msg[512];
  spa_clear(p);
  spa_clear(r);
  spa_clear(d);
  spa_clear(w);
  spa_add(p, j, alpha);
  if (rhs_t)
    axpy_col(rhs_t, 1.0, j, r);
  else
    spa_add(r, j, 1.0);
  axpy_col(Kt, -alpha, j, r);

  const double tol_sq = tol * tol;
  double rnorm_sq = spa_norm_sq_sorted(r);
  int64_t iters = 0;
  while (rnorm_sq > tol_sq)
  {
    if (iters >= max_col_iters)
    {
      snprintf(msg, sizeof msg, "spai: column %lld stalled at ||r|| = %f after %lld iterations (tol %f)",
               (long long)j, sqrt(rnorm_sq), (long long)iters, tol);
      set_err(err, j, msg);
      return ORC_ERR_STAGNATION;
    }
    spa_clear(d);
    spa_sort(r);
    for (int64_t k = 0; k < r->len; ++k)
    {
      const int64_t i = r->idx[k];
      const double ri = r->val[i];
      if (ri == 0.0)
        continue;
      if (mode == 0 && store->built[i])
      {
        for (int64_t t = 0; t < store->len[i]; ++t)
          spa_add(d, store->row[i][t], ri * store->val[i][t]);
      }
      else
        spa_add(d, i, alpha * ri);
    }
    spa_clear(w);
    spa_sort(d);
    for (int64_t k = 0; k < d->len; ++k)
    {
      const int64_t i = d->idx[k];
      const double di = d->val[i];
      if (di != 0.0)
        axpy_col(Kt, di, i, w);
    }
    const double ww = spa_dot(w, w);
    const double rw = spa_dot(w, r);
    if (!(ww > 0.0))
    {
      if (!isfinite(ww))
      {
        snprintf(msg, sizeof msg, "spai: non-finite values in column %lld", (long long)j);
        set_err(err, j, msg);
        return ORC_ERR_NUMERICAL;
      }
      snprintf(msg, sizeof msg, "spai: zero curvature in column %lld with ||r|| > tol", (long long)j);
      set_err(err, j, msg);
      return ORC_ERR_STAGNATION;
    }
    const double a = rw / ww;
    if (!isfinite(a))
    {
      snprintf(msg, sizeof msg, "spai: non-finite step in column %lld", (long long)j);
      set_err(err, j, msg);
      return ORC_ERR_NUMERICAL;
    }
    for (int64_t k = 0; k < d->len; ++k)
      spa_add(p, d->idx[k], a * d->val[d->idx[k]]);
    for (int64_t k = 0; k < w->len; ++k)
      spa_add(r, w->idx[k], -a * w->val[w->idx[k]]);
    rnorm_sq = spa_norm_sq_sorted(r);
    ++iters;
  }
  spa_sort(p);
  int64_t cnt = 0;
  for (int64_t k = 0; k < p->len; ++k)
    if (p->val[p->idx[k]] != 0.0)
      ++cnt;
  free(store->row[j]);
  free(store->val[j]);
  store->row[j] = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cnt > 0 ? cnt : 1));
  store->val[j] = (double *)malloc(sizeof(double) * (size_t)(cnt > 0 ? cnt : 1));
  store->len[j] = 0;
  for (int64_t k = 0; k < p->len; ++k)
  {
    const int64_t i = p->idx[k];
    if (p->val[i] != 0.0)
    {
      store->row[j][store->len[j]] = i;
      store->val[j][store->len[j]] = p->val[i];
      store->len[j]++;
    }
  }
  *final_res = sqrt(rnorm_sq);
  return ORC_OK;
}

/* spai.cpp:236-310 (run_build, single-threaded column loop) + assemble (:211-234). */
static int run_build(const orc_csr *K, const orc_csr *rhs_src, double alpha, double tol, int64_t max_col_iters,
                     int mode, orc_csr *out, double *col_residual, orc_err *err)
{
  const int64_t n = K->nrows;
  orc_csr Kt, Rt;
  orc_transpose(K, &Kt);
  if (rhs_src)
    orc_transpose(rhs_src, &Rt);
  colstore store;
  store.len = (int64_t *)calloc((size_t)n, sizeof(int64_t));
  store.row = (int64_t **)calloc((size_t)n, sizeof(int64_t *));
  store.val = (double **)calloc((size_t)n, sizeof(double *));
  store.built = (char *)calloc((size_t)n, 1);
  spa p, r, d, w;
  spa_init(&p, n);
  spa_init(&r, n);
  spa_init(&d, n);
  spa_init(&w, n);
  int st = ORC_OK;
  for (int64_t j = 0; j < n && st == ORC_OK; ++j)
  {
    double res = 0.0;
    st = build_column(j, alpha, &Kt, rhs_src ? &Rt : NULL, tol, max_col_iters, mode, &store, &p, &r, &d, &w, &res,
                      err);
    if (col_residual)
      col_residual[j] = res;
    store.built[j] = 1;
  }
  if (st == ORC_OK)
  {
    int64_t total = 0;
    for (int64_t j = 0; j < n; ++j)
      total += store.len[j];
    int64_t *tr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
    int64_t *tc = (int64_t *)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
    double *tv = (double *)malloc(sizeof(double) * (size_t)(total > 0 ? total : 1));
    int64_t t = 0;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t k = 0; k < store.len[j]; ++k)
      {
        tr[t] = store.row[j][k];
        tc[t] = j;
        tv[t++] = store.val[j][k];
      }
    st = orc_from_triplets(n, n, total, tr, tc, tv, out, err);
    free(tr);
    free(tc);
    free(tv);
  }
  for (int64_t j = 0; j < n; ++j)
  {
    free(store.row[j]);
    free(store.val[j]);
  }
  free(store.len);
  free(store.row);
  free(store.val);
  free(store.built);
  spa_free(&p);
  spa_free(&r);
  spa_free(&d);
  spa_free(&w);
  orc_csr_free(&Kt);
  if (rhs_src)
    orc_csr_free(&Rt);
  return st;
}

/* spai.cpp:314-331 */
int orc_spai_build(const orc_csr *K, double tol, int64_t max_col_iters, int mode, orc_csr *P, double *col_residual,
                   orc_err *err)
{
  clear_err(err);
  if (K->nrows != K->ncols)
  {
    set_err(err, -1, "spai_build: K must be square");
    return ORC_ERR_ARG;
  }
  if (!(tol > 0.0))
  {
    set_err(err, -1, "spai_build: tol must be positive");
    return ORC_ERR_ARG;
  }
  const double denom = orc_trace_inner(K, K);
  if (!(denom > 0.0))
  {
    set_err(err, -1, "spai_build: trace(K K^T) is not positive");
    return ORC_ERR_NUMERICAL;
  }
  const double alpha = orc_trace(K) / denom;
  return run_build(K, NULL, alpha, tol, max_col_iters, mode, P, col_residual, err);
}

/* spai.cpp:333-350 */
int orc_spai_update(const orc_csr *K_old, const orc_csr *K_new, double tol, int64_t max_col_iters, int mode,
                    orc_csr *Q, double *col_residual, orc_err *err)
{
  clear_err(err);
  if (K_old->nrows != K_old->ncols || K_new->nrows != K_new->ncols || K_old->nrows != K_new->nrows)
  {
    set_err(err, -1, "spai_update: operands must be square with equal shape");
    return ORC_ERR_ARG;
  }
  if (!(tol > 0.0))
  {
    set_err(err, -1, "spai_update: tol must be positive");
    return ORC_ERR_ARG;
  }
  const double denom = orc_trace_inner(K_new, K_new);
  if (!(denom > 0.0))
  {
    set_err(err, -1, "spai_update: trace(K_new^T K_new) is not positive");
    return ORC_ERR_NUMERICAL;
  }
  const double alpha = 0.5 * (orc_trace_inner(K_old, K_new) + orc_trace_inner(K_new, K_old)) / denom;
  return run_build(K_new, K_old, alpha, tol, max_col_iters, mode, Q, col_residual, err);
}

/* ---------------------------------------------------------------- thin QR */

/* dense.cpp:153-246 with the scalar kernel table. */
int orc_thin_qr(int64_t m, int64_t n, const double *A, double rank_tol, double *Q, double *R, int64_t *rank)
{
  if (m < n)
    return ORC_ERR_ARG;
  double anorm_sq = 0.0; /* frob_norm(DenseMatrix) = sqrt(dot over all values) */
  anorm_sq = dot_s(A, A, m * n);
  const double anorm = sqrt(anorm_sq);
  const double tol = rank_tol * (anorm > 0.0 ? anorm : 1.0);
  double *W = (double *)malloc(sizeof(double) * (size_t)(m * n > 0 ? m * n : 1));
  memcpy(W, A, sizeof(double) * (size_t)(m * n));
  double *diag = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double *tau = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  for (int64_t k = 0; k < n; ++k)
  {
    double *x = W + k * m + k;
    const int64_t len = m - k;
    const double sigma = sqrt(dot_s(x, x, len));
    if (sigma <= tol)
    {
      diag[k] = 0.0;
      tau[k] = 0.0;
      for (int64_t i = 0; i < len; ++i)
        x[i] = 0.0;
      continue;
    }
    const double alpha = x[0] >= 0.0 ? -sigma : sigma;
    const double v0 = x[0] - alpha;
    x[0] = v0;
    const double vtv = dot_s(x, x, len);
    tau[k] = vtv > 0.0 ? 2.0 / vtv : 0.0;
    diag[k] = alpha;
    for (int64_t j = k + 1; j < n; ++j)
    {
      double *y = W + j * m + k;
      const double s = tau[k] * dot_s(x, y, len);
      axpy_s(len, -s, x, y);
    }
  }
  memset(R, 0, sizeof(double) * (size_t)(n * n));
  for (int64_t k = 0; k < n; ++k)
  {
    for (int64_t i = 0; i < k; ++i)
      R[k * n + i] = W[k * m + i];
    R[k * n + k] = diag[k];
  }
  memset(Q, 0, sizeof(double) * (size_t)(m * n));
  for (int64_t j = 0; j < n; ++j)
  {
    if (diag[j] == 0.0)
      continue;
    double *q = Q + j * m;
    q[j] = 1.0;
    for (int64_t k = (j < n - 1 ? j : n - 1); k >= 0; --k)
    {
      if (tau[k] == 0.0)
        continue;
      const double *v = W + k * m + k;
      const int64_t len = m - k;
      const double s = tau[k] * dot_s(v, q + k, len);
      axpy_s(len, -s, v, q + k);
    }
  }
  int64_t rk = 0;
  for (int64_t k = 0; k < n; ++k)
  {
    if (R[k * n + k] < 0.0)
    {
      for (int64_t j = k; j < n; ++j)
        R[j * n + k] = -R[j * n + k];
      for (int64_t i = 0; i < m; ++i) /* kernels_scalar.cpp:31-37 scal */
        Q[k * m + i] *= -1.0;
    }
    if (R[k * n + k] > 0.0)
      ++rk;
  }
  *rank = rk;
  free(W);
  free(diag);
  free(tau);
  return ORC_OK;
}

/* ---------------------------------------------------------------- LS-SPAI */

int orc_pattern_square(const orc_csr *A, orc_csr *out)
{
  const int64_t n = A->nrows;
  char *mark = (char *)calloc((size_t)A->ncols, 1);
  int64_t *cols = (int64_t *)malloc(sizeof(int64_t) * (size_t)(A->ncols > 0 ? A->ncols : 1));
  int64_t cap = A->nnz * 4 + 16, nz = 0;
  out->nrows = n;
  out->ncols = A->ncols;
  out->row_ptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  out->col_idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
  out->values = (double *)malloc(sizeof(double) * (size_t)cap);
  for (int64_t i = 0; i < n; ++i)
  {
    int64_t c = 0;
    for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k)
    {
      const int64_t t = A->col_idx[k];
      for (int64_t q = A->row_ptr[t]; q < A->row_ptr[t + 1]; ++q)
        if (!mark[A->col_idx[q]])
        {
          mark[A->col_idx[q]] = 1;
          cols[c++] = A->col_idx[q];
        }
    }
    qsort(cols, (size_t)c, sizeof(int64_t), cmp_i64);
    if (nz + c > cap)
    {
      cap = 2 * (nz + c);
      out->col_idx = (int32_t *)realloc(out->col_idx, sizeof(int32_t) * (size_t)cap);
      out->values = (double *)realloc(out->values, sizeof(double) * (size_t)cap);
    }
    for (int64_t q = 0; q < c; ++q)
    {
      out->col_idx[nz] = (int32_t)cols[q];
      out->values[nz++] = 1.0;
      mark[cols[q]] = 0;
    }
    out->row_ptr[i + 1] = nz;
  }
  out->nnz = nz;
  free(mark);
  free(cols);
  return ORC_OK;
}

/* Column-equilibrated variant (pattern | ORC_LS_COLSCALE): before the QR every column c of S
 * is scaled by r_c = 1 / ||S_c|| (in-order dot, sqrt, one division, S_ic * r_c), and the
 * back-substituted solution by r_c again (m_c = u_c * r_c).  In exact arithmetic this is the same least-squares minimiser
 * (S D^-1 (D m) = S m); it removes the spurious global rank flush of thin_qr (sigma <= 1e-12
 * ||S||_F, dense.cpp:162-179), which on the Hermite beam fires once the theta-dof columns
 * (~h^2 smaller than the w-dof ones) drop below 1e-12 of the Frobenius norm (n >= 2e5 on the
 * A^2 pattern, n >= 4e5 on A's).  A zero column (d_c == 0) is rank deficiency.
 *
 * SURVEY.md 8(a') "LS-SPAI oracle definition": J = pattern row j, I = sorted
 * union of the rows of A(:, J), S = A(I, J), (Q, R) = thin_qr(S),
 * y = Q^T e|_I (e = e_j, or K_old(:, j) for the update), R m = y by
 * back-substitution (acc = y_k; acc -= R_kt m_t for t ascending; m_k = acc / R_kk),
 * P(J, j) = m, assembled with from_triplets.  A zero R diagonal raises
 * NumericalError naming the column. */
int orc_spai_ls(const orc_csr *A, const orc_csr *K_old, int pattern, orc_csr *P, orc_err *err)
{
  clear_err(err);
  /* pattern | ORC_LS_COLSCALE: column-equilibrated variant (see the header comment) */
  const int colscale = (pattern & ORC_LS_COLSCALE) != 0;
  pattern &= ~ORC_LS_COLSCALE;
  if (A->nrows != A->ncols || (K_old && (K_old->nrows != A->nrows || K_old->ncols != A->ncols)))
  {
    set_err(err, -1, "spai_ls: operands must be square with equal shape");
    return ORC_ERR_ARG;
  }
  const int64_t n = A->nrows;
  orc_csr pat, At, Kot;
  if (pattern == 1)
    orc_pattern_square(A, &pat);
  else
    pat = *A;
  orc_transpose(A, &At);
  if (K_old)
    orc_transpose(K_old, &Kot);
  int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i)
    pos[i] = -1;
  int64_t *I = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t total = pat.nnz;
  int64_t *tr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
  int64_t *tc = (int64_t *)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
  double *tv = (double *)malloc(sizeof(double) * (size_t)(total > 0 ? total : 1));
  int64_t t = 0;
  int st = ORC_OK;
  for (int64_t j = 0; j < n && st == ORC_OK; ++j)
  {
    const int64_t jb = pat.row_ptr[j], nj = pat.row_ptr[j + 1] - jb;
    if (nj == 0)
      continue;
    int64_t ni = 0;
    for (int64_t c = 0; c < nj; ++c)
    {
      const int64_t k = pat.col_idx[jb + c];
      for (int64_t q = At.row_ptr[k]; q < At.row_ptr[k + 1]; ++q)
        if (pos[At.col_idx[q]] < 0)
        {
          pos[At.col_idx[q]] = 0;
          I[ni++] = At.col_idx[q];
        }
    }
    qsort(I, (size_t)ni, sizeof(int64_t), cmp_i64);
    for (int64_t a = 0; a < ni; ++a)
      pos[I[a]] = a;
    if (ni < nj)
    {
      char msg[256];
      snprintf(msg, sizeof msg, "spai_ls: rank-deficient least-squares problem in column %lld", (long long)j);
      set_err(err, j, msg);
      st = ORC_ERR_NUMERICAL;
    }
    else
    {
      double *S = (double *)calloc((size_t)(ni * nj), sizeof(double));
      double *Qm = (double *)malloc(sizeof(double) * (size_t)(ni * nj));
      double *R = (double *)malloc(sizeof(double) * (size_t)(nj * nj));
      double *e = (double *)calloc((size_t)ni, sizeof(double));
      double *y = (double *)malloc(sizeof(double) * (size_t)nj);
      double *mm = (double *)malloc(sizeof(double) * (size_t)nj);
      double *dsc = (double *)malloc(sizeof(double) * (size_t)nj);
      for (int64_t c = 0; c < nj; ++c)
      {
        const int64_t k = pat.col_idx[jb + c];
        for (int64_t q = At.row_ptr[k]; q < At.row_ptr[k + 1]; ++q)
          S[c * ni + pos[At.col_idx[q]]] = At.values[q];
      }
      if (K_old)
      {
        for (int64_t q = Kot.row_ptr[j]; q < Kot.row_ptr[j + 1]; ++q)
          if (pos[Kot.col_idx[q]] >= 0)
            e[pos[Kot.col_idx[q]]] = Kot.values[q];
      }
      else if (pos[j] >= 0)
        e[pos[j]] = 1.0;
      int64_t rank = 0;
      int zero_col = 0;
      if (colscale)
      {
        /* d_c = sqrt(dot(S_c, S_c)) in index order (kernels_scalar.cpp:13-19), r_c = 1 / d_c,
         * S_c *= r_c */
        for (int64_t c = 0; c < nj; ++c)
        {
          const double d = sqrt(dot_s(S + c * ni, S + c * ni, ni));
          if (d == 0.0)
          {
            zero_col = 1;
            dsc[c] = 0.0;
            continue;
          }
          dsc[c] = 1.0 / d;
          for (int64_t i = 0; i < ni; ++i)
            S[c * ni + i] = S[c * ni + i] * dsc[c];
        }
      }
      if (!zero_col)
        orc_thin_qr(ni, nj, S, 1e-12, Qm, R, &rank);
      if (rank < nj)
      {
        char msg[256];
        snprintf(msg, sizeof msg, "spai_ls: rank-deficient least-squares problem in column %lld", (long long)j);
        set_err(err, j, msg);
        st = ORC_ERR_NUMERICAL;
      }
      else
      {
        for (int64_t c = 0; c < nj; ++c)
          y[c] = dot_s(Qm + c * ni, e, ni);
        for (int64_t k = nj - 1; k >= 0; --k)
        {
          double acc = y[k];
          for (int64_t q = k + 1; q < nj; ++q)
            acc -= R[q * nj + k] * mm[q];
          mm[k] = acc / R[k * nj + k];
        }
        if (colscale)
          for (int64_t c = 0; c < nj; ++c)
            mm[c] = mm[c] * dsc[c];
        for (int64_t c = 0; c < nj; ++c)
        {
          tr[t] = pat.col_idx[jb + c];
          tc[t] = j;
          tv[t++] = mm[c];
        }
      }
      free(S);
      free(Qm);
      free(R);
      free(e);
      free(y);
      free(mm);
      free(dsc);
    }
    for (int64_t a = 0; a < ni; ++a)
      pos[I[a]] = -1;
  }
  if (st == ORC_OK)
    st = orc_from_triplets(n, n, t, tr, tc, tv, P, err);
  free(tr);
  free(tc);
  free(tv);
  free(pos);
  free(I);
  orc_csr_free(&At);
  if (K_old)
    orc_csr_free(&Kot);
  if (pattern == 1)
    orc_csr_free(&pat);
  return st;
}

/* ---------------------------------------------------------------- Krylov */

/* spai.cpp:361-373: oldest factor (last in the newest-first list) applied first. */
void orc_chain_apply(int z, const orc_csr *factors, int64_t n, const double *v, double *out)
{
  double *tmp = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  memcpy(out, v, sizeof(double) * (size_t)n);
  for (int f = z - 1; f >= 0; --f)
  {
    orc_spmv(&factors[f], out, tmp);
    memcpy(out, tmp, sizeof(double) * (size_t)n);
  }
  free(tmp);
}

/* krylov.cpp:28-139: CG on A P (right preconditioning), x~0 = 0, confirm /
 * restart on the true residual, breakdown guard, solution = P x~. */
int orc_pcg_solve(const orc_csr *A, int z, const orc_csr *factors, const double *b, double rtol, int64_t maxit,
                  double *solution, double *residual, double *recurrence, int64_t *iterations, int *converged,
                  double *history, int64_t history_cap, int64_t *history_len, orc_err *err)
{
  clear_err(err);
  const int64_t n = A->nrows;
  for (int f = 0; f < z; ++f)
    if (factors[f].nrows != n)
    {
      set_err(err, -1, "pcg_solve: dimension mismatch");
      return ORC_ERR_ARG;
    }
  if (!(rtol > 0.0))
  {
    set_err(err, -1, "pcg_solve: rtol must be positive");
    return ORC_ERR_ARG;
  }
  *history_len = 0;
  const double bnorm = sqrt(dot_s(b, b, n));
  if (bnorm == 0.0)
  {
    memset(solution, 0, sizeof(double) * (size_t)n);
    memset(residual, 0, sizeof(double) * (size_t)n);
    memset(recurrence, 0, sizeof(double) * (size_t)n);
    *iterations = 0;
    *converged = 1;
    return ORC_OK;
  }
  const double target = rtol * bnorm;
  const size_t bytes = sizeof(double) * (size_t)n;
  double *xt = (double *)calloc((size_t)n, sizeof(double));
  double *r = (double *)malloc(bytes);
  double *d = (double *)malloc(bytes);
  double *t = (double *)malloc(bytes);
  double *w = (double *)malloc(bytes);
  memcpy(r, b, bytes);
  memcpy(d, r, bytes);
  double rho = dot_s(r, r, n);
  int64_t it = 0;
  int done = 0, conv = 0, st = ORC_OK;

  while (it < maxit)
  {
    if (sqrt(rho) <= target)
    {
      orc_chain_apply(z, factors, n, xt, t);
      orc_spmv(A, t, w);
      for (int64_t i = 0; i < n; ++i)
        w[i] = b[i] - w[i];
      const double true_norm = sqrt(dot_s(w, w, n));
      if (true_norm <= target)
      {
        done = 1;
        conv = 1;
        break;
      }
      memcpy(r, w, bytes);
      memcpy(d, r, bytes);
      rho = dot_s(r, r, n);
      if (sqrt(rho) <= target)
      {
        done = 1;
        conv = 1;
        break;
      }
    }
    orc_chain_apply(z, factors, n, d, t);
    orc_spmv(A, t, w);
    const double curvature = dot_s(d, w, n);
    const double dd = dot_s(d, d, n);
    if (!(curvature > 1e-30 * dd))
    {
      char msg[256];
      snprintf(msg, sizeof msg, "pcg_solve: direction curvature breakdown at iteration %lld", (long long)it);
      set_err(err, it, msg);
      st = ORC_ERR_BREAKDOWN;
      break;
    }
    const double alpha = rho / curvature;
    axpy_s(n, alpha, d, xt);
    axpy_s(n, -alpha, w, r);
    ++it;
    const double rho_next = dot_s(r, r, n);
    if (history && *history_len < history_cap)
      history[*history_len] = sqrt(rho_next) / bnorm;
    (*history_len)++;
    const double betak = rho_next / rho;
    rho = rho_next;
    for (int64_t i = 0; i < n; ++i)
      d[i] = r[i] + betak * d[i];
  }
  if (st == ORC_OK)
  {
    /* finish (krylov.cpp:62-73), after the budget-exhausted check (:128-137) when needed */
    orc_chain_apply(z, factors, n, xt, solution);
    orc_spmv(A, solution, w);
    for (int64_t i = 0; i < n; ++i)
      residual[i] = b[i] - w[i];
    if (!done)
    {
      const double true_norm = sqrt(dot_s(residual, residual, n));
      conv = true_norm <= target;
    }
    memcpy(recurrence, r, bytes);
    *iterations = it;
    *converged = conv;
  }
  free(xt);
  free(r);
  free(d);
  free(t);
  free(w);
  return st;
}

/* krylov.cpp:141-174 */
int orc_block_solve(const orc_csr *A, int z, const orc_csr *factors, int64_t m, const double *B, double rtol,
                    int64_t maxit, double *X, double *recurrence, double *true_res, int64_t *iterations,
                    int *all_converged, orc_err *err)
{
  const int64_t n = A->nrows;
  *all_converged = 1;
  for (int64_t j = 0; j < m; ++j)
  {
    int conv = 0;
    int64_t hl = 0;
    const int st = orc_pcg_solve(A, z, factors, B + j * n, rtol, maxit, X + j * n, true_res + j * n,
                                 recurrence + j * n, &iterations[j], &conv, NULL, 0, &hl, err);
    if (st == ORC_ERR_BREAKDOWN)
    {
      char msg[512];
      snprintf(msg, sizeof msg, "block_solve: column %lld: %s", (long long)j, err ? err->msg : "");
      if (err)
        snprintf(err->msg, sizeof err->msg, "%s", msg);
      return st;
    }
    if (st != ORC_OK)
      return st;
    *all_converged = *all_converged && conv;
  }
  return ORC_OK;
}
