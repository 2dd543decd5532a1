/*
 * mstab_oracle.c — TEST INFRASTRUCTURE ONLY (see mstab_oracle.h). Plain-C, real-fp64
 * restatement of the reference Mstab solve path. Each function cites the reference routine it
 * restates; the operation order (accumulations from 0 in index order, products rounded before
 * sums, x * (1/d) where the reference multiplies by an inverse, x / d where it divides) follows
 * the reference so that results agree bit-for-bit with the compiled reference (oracle/_ref).
 * Compiled with -ffp-contract=off (no FMA), like the reference's x86-64 -O3 build.
 */
#include "mstab_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define E_OK 0
#define E_ERROR (-1)
#define E_DIMENSION (-2)
#define E_CONFIG (-3)
#define E_FINGERPRINT (-4)
#define E_STALE (-5)
#define E_SINGULAR (-8)
#define E_RANK (-9)

/* ---- libstdc++ std::mt19937_64 + std::normal_distribution<double> (polar method) ----------- */
typedef struct {
  uint64_t mt[312];
  int idx;
  int saved_available;
  double saved;
} orc_rng;

static void rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->saved_available = 0;
  r->saved = 0.0;
}

static uint64_t rng_next(orc_rng* r) {
  static const uint64_t mag[2] = {0ull, 0xB5026F5AA96619E9ull};
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (r->idx >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag[x & 1ull];
    }
    for (; i < 311; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1ull];
    }
    uint64_t x = (r->mt[311] & UM) | (r->mt[0] & LM);
    r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag[x & 1ull];
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

/* std::generate_canonical<double, 53>(mt19937_64): one draw scaled by 2^64 */
static double rng_canonical(orc_rng* r) {
  double ret = (double)rng_next(r) / 18446744073709551616.0;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret;
}

static double rng_normal(orc_rng* r) {
  double ret;
  if (r->saved_available) {
    r->saved_available = 0;
    ret = r->saved;
  } else {
    double x, y, r2;
    do {
      x = 2.0 * rng_canonical(r) - 1.0;
      y = 2.0 * rng_canonical(r) - 1.0;
      r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = sqrt(-2 * log(r2) / r2);
    r->saved = x * mult;
    r->saved_available = 1;
    ret = y * mult;
  }
  return ret * 1.0 + 0.0;
}

void orc_normal_draws(uint64_t seed, int64_t count, double* out) {
  orc_rng* r = malloc(sizeof(orc_rng));
  rng_seed(r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng_normal(r);
  free(r);
}

/* ---- types.cpp:9-23, dense.cpp:19-48 --------------------------------------------------------- */
static double norm2(const double* v, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += v[i] * v[i];
  return sqrt(acc);
}

static double dot(const double* a, const double* b, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

static void axpy(double alpha, const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}

/* gemv (dense.cpp:19-24): y = 0; y += x_j * A_j in column order */
static void gemv(const double* a, int64_t n, int64_t s, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = 0.0;
  for (int64_t j = 0; j < s; ++j) axpy(x[j], a + j * n, y, n);
}

static int is_zero(const double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (v[i] != 0.0) return 0;
  return 1;
}

static int all_finite(const double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

static double* dalloc(int64_t n) { return calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

static double* dcopy(const double* src, int64_t n) {
  double* d = dalloc(n);
  memcpy(d, src, sizeof(double) * (size_t)n);
  return d;
}

/* ---- csr.cpp:28-43, :103-113 ---------------------------------------------------------------- */
static uint64_t fnv(uint64_t h, const void* p, size_t len) {
  const unsigned char* b = p;
  for (size_t i = 0; i < len; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}

uint64_t orc_fingerprint(const orc_csr* a) {
  uint64_t h = 1469598103934665603ull;
  const uint64_t nnz = (uint64_t)a->row_ptr[a->n];
  const uint64_t dims[3] = {(uint64_t)a->n, (uint64_t)a->n, nnz};
  h = fnv(h, dims, sizeof(dims));
  for (int64_t i = 0; i <= a->n; ++i) {
    uint64_t v = (uint64_t)a->row_ptr[i];
    h = fnv(h, &v, 8);
  }
  for (uint64_t k = 0; k < nnz; ++k) {
    uint64_t v = (uint64_t)a->col_idx[k];
    h = fnv(h, &v, 8);
  }
  for (uint64_t k = 0; k < nnz; ++k) {
    const double z[2] = {a->values[k], 0.0};
    h = fnv(h, z, 16);
  }
  return h;
}

void orc_spmv(const orc_csr* a, const double* x, double* y) {
  for (int64_t i = 0; i < a->n; ++i) {
    double acc = 0.0;
    for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) acc += a->values[k] * x[a->col_idx[k]];
    y[i] = acc;
  }
}

/* ---- kernels.cpp:95-154: LuFactor + solve_small ----------------------------------------------- */
int orc_solve_small(int64_t s, const double* m, const double* rhs, double* x) {
  double* lu = dcopy(m, s * s);
  int64_t* perm = malloc(sizeof(int64_t) * (size_t)s);
#define LU(i, j) lu[(i) + (j) * s]
  double scale = 0.0;
  for (int64_t k = 0; k < s * s; ++k) {
    const double v = fabs(lu[k]);
    scale = (scale < v) ? v : scale;
  }
  for (int64_t i = 0; i < s; ++i) perm[i] = i;
  int singular = 0;
  for (int64_t k = 0; k < s && !singular; ++k) {
    int64_t piv = k;
    double best = fabs(LU(k, k));
    for (int64_t i = k + 1; i < s; ++i) {
      const double mm = fabs(LU(i, k));
      if (mm > best) {
        best = mm;
        piv = i;
      }
    }
    if (best < 1e-14 * scale || scale == 0.0) {
      singular = 1;
      break;
    }
    if (piv != k) {
      int64_t t = perm[k];
      perm[k] = perm[piv];
      perm[piv] = t;
      for (int64_t j = 0; j < s; ++j) {
        double u = LU(k, j);
        LU(k, j) = LU(piv, j);
        LU(piv, j) = u;
      }
    }
    const double inv = 1.0 / LU(k, k);
    for (int64_t i = k + 1; i < s; ++i) {
      const double mm = LU(i, k) * inv;
      LU(i, k) = mm;
      if (mm != 0.0)
        for (int64_t j = k + 1; j < s; ++j) LU(i, j) -= mm * LU(k, j);
    }
  }
  if (!singular) {
    for (int64_t i = 0; i < s; ++i) x[i] = rhs[perm[i]];
    for (int64_t i = 1; i < s; ++i)
      for (int64_t j = 0; j < i; ++j) x[i] -= LU(i, j) * x[j];
    for (int64_t i = s; i-- > 0;) {
      for (int64_t j = i + 1; j < s; ++j) x[i] -= LU(i, j) * x[j];
      x[i] /= LU(i, i);
    }
  }
#undef LU
  free(lu);
  free(perm);
  return singular ? E_SINGULAR : E_OK;
}

/* ---- kernels.cpp:52-93: least_squares_tall (MGS with reiteration) ---------------------------- */
int orc_least_squares(int64_t n, int64_t ell, const double* z, const double* r, double* tau) {
  if (ell < 1 || n < ell) return E_DIMENSION;
  double max_colnorm = 0.0;
  for (int64_t j = 0; j < ell; ++j) {
    const double c = norm2(z + j * n, n);
    max_colnorm = (max_colnorm < c) ? c : max_colnorm;
  }
  double* q = dcopy(z, n * ell);
  double* rr = dalloc(ell * ell);
  double min_diag = INFINITY;
  for (int64_t k = 0; k < ell; ++k) {
    double* qk = q + k * n;
    for (int pass = 0; pass < 2; ++pass)
      for (int64_t i = 0; i < k; ++i) {
        const double c = dot(q + i * n, qk, n);
        axpy(-c, q + i * n, qk, n);
        rr[i + k * ell] += c;
      }
    const double d = norm2(qk, n);
    rr[k + k * ell] = d;
    min_diag = (d < min_diag) ? d : min_diag;
    if (d > 0.0) {
      const double inv = 1.0 / d;
      for (int64_t t = 0; t < n; ++t) qk[t] *= inv;
    }
  }
  int rc = E_OK;
  if (min_diag < 1e-13 * max_colnorm) {
    rc = E_RANK;
  } else {
    for (int64_t j = 0; j < ell; ++j) tau[j] = dot(q + j * n, r, n);
    for (int64_t k = ell; k-- > 0;) {
      for (int64_t j = k + 1; j < ell; ++j) tau[k] -= rr[k + j * ell] * tau[j];
      tau[k] /= rr[k + k * ell];
    }
  }
  free(q);
  free(rr);
  return rc;
}

/* ---- kernels.cpp:21-50 orthonormalize + baselines.cpp:36-47 make_cut_space ------------------- */
static int64_t orthonormalize(const double* v, int64_t n, int64_t cols, double tol, double* out) {
  int64_t rank = 0;
  double* w = dalloc(n);
  double* coeff = dalloc(cols);
  for (int64_t j = 0; j < cols; ++j) {
    const double* vj = v + j * n;
    const double norm0 = norm2(vj, n);
    memcpy(w, vj, sizeof(double) * (size_t)n);
    for (int pass = 0; pass < 2 && rank > 0; ++pass) {
      for (int64_t i = 0; i < rank; ++i) coeff[i] = dot(out + i * n, w, n);
      for (int64_t i = 0; i < rank; ++i) axpy(-coeff[i], out + i * n, w, n);
    }
    const double res = norm2(w, n);
    if (res <= tol * norm0 || norm0 == 0.0) continue;
    const double inv = 1.0 / res;
    for (int64_t t = 0; t < n; ++t) out[rank * n + t] = w[t] * inv;
    ++rank;
  }
  free(w);
  free(coeff);
  return rank;
}

int orc_cut_space(int64_t n, int64_t s, uint64_t seed, double* p) {
  orc_rng* r = malloc(sizeof(orc_rng));
  rng_seed(r, seed);
  double* g = dalloc(n * s);
  int rc = E_ERROR;
  for (int attempt = 0; attempt < 4; ++attempt) {
    for (int64_t k = 0; k < n * s; ++k) g[k] = rng_normal(r);
    if (orthonormalize(g, n, s, 1e-10, p) == s) {
      rc = E_OK;
      break;
    }
  }
  free(g);
  free(r);
  return rc;
}

/* ---- idrstab.cpp:45-87 arnoldi_init ---------------------------------------------------------- */
static int arnoldi(const orc_csr* a, const double* r0, int64_t s, orc_rng* rng, double* u, double* v) {
  const int64_t n = a->n;
  const double r0norm = norm2(r0, n);
  if (r0norm == 0.0) return E_ERROR;
  for (int64_t i = 0; i < n; ++i) u[i] = r0[i] / r0norm;
  double* w = dalloc(n);
  for (int64_t k = 0; k < s; ++k) {
    orc_spmv(a, u + k * n, v + k * n);
    if (k + 1 == s) break;
    memcpy(w, v + k * n, sizeof(double) * (size_t)n);
    const double wnorm0 = norm2(w, n);
    for (int pass = 0; pass < 2; ++pass)
      for (int64_t i = 0; i <= k; ++i) axpy(-dot(u + i * n, w, n), u + i * n, w, n);
    double wnorm = norm2(w, n);
    while (wnorm <= 1e-12 * fmax(wnorm0, 1.0)) {
      for (int64_t i = 0; i < n; ++i) w[i] = rng_normal(rng);
      for (int pass = 0; pass < 2; ++pass)
        for (int64_t i = 0; i <= k; ++i) axpy(-dot(u + i * n, w, n), u + i * n, w, n);
      wnorm = norm2(w, n);
    }
    for (int64_t i = 0; i < n; ++i) u[(k + 1) * n + i] = w[i] / wnorm;
  }
  free(w);
  return E_OK;
}

int orc_arnoldi(const orc_csr* a, const double* r0, int64_t s, uint64_t rng_seed_v, double* u, double* v) {
  orc_rng* r = malloc(sizeof(orc_rng));
  rng_seed(r, rng_seed_v);
  int rc = arnoldi(a, r0, s, r, u, v);
  free(r);
  return rc;
}

/* ---- recycle.cpp:40-83 validate (max deviation + sigma ratio) -------------------------------- */
static void sym_eigenvalues(double* a, int64_t n, double* ev) {
#define A(i, j) a[(i) + (j) * n]
  double off = 0.0, total = 0.0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      const double m = A(i, j) * A(i, j);
      total += m;
      if (i != j) off += m;
    }
  const double stop = 1e-28 * fmax(total, 1e-300);
  for (int sweep = 0; sweep < 60 && off > stop; ++sweep) {
    for (int64_t p = 0; p < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        const double apq = A(p, q), m = fabs(apq);
        if (m == 0.0) continue;
        const double ph = apq / m;
        const double theta = (A(q, q) - A(p, p)) / (2.0 * m);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = t * c;
        for (int64_t k = 0; k < n; ++k) {
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - sn * ph * akq;
          A(k, q) = sn * akp + c * ph * akq;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - sn * ph * aqk;
          A(q, k) = sn * apk + c * ph * aqk;
        }
      }
    off = 0.0;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i)
        if (i != j) off += A(i, j) * A(i, j);
  }
  for (int64_t i = 0; i < n; ++i) ev[i] = A(i, i);
  for (int64_t i = 1; i < n; ++i)
    for (int64_t j = i; j > 0 && ev[j - 1] > ev[j]; --j) {
      const double t = ev[j];
      ev[j] = ev[j - 1];
      ev[j - 1] = t;
    }
#undef A
}

int orc_validate(const orc_csr* a, const orc_recycle* rd, double* max_dev, double* sigma_ratio) {
  if (rd->fingerprint != orc_fingerprint(a)) return E_FINGERPRINT;
  if (rd->n != a->n) return E_DIMENSION;
  if (rd->omega_count != 0 && rd->omega_count != rd->level_j) return E_STALE;
  const int64_t n = rd->n, s = rd->s;
  double dev_num = 0.0, dev_den = 0.0;
  double* au = dalloc(n);
  for (int64_t q = 0; q < s; ++q) {
    orc_spmv(a, rd->u + q * n, au);
    const double* vq = rd->v + q * n;
    for (int64_t i = 0; i < n; ++i) {
      const double d = vq[i] - au[i];
      dev_num += d * d;
    }
    const double nv = norm2(vq, n);
    dev_den += nv * nv;
  }
  free(au);
  const double dev_v = dev_den > 0.0 ? sqrt(dev_num) / sqrt(dev_den) : sqrt(dev_num);
  double dev_p = 0.0;
  for (int64_t j = 0; j < s; ++j)
    for (int64_t i = 0; i < s; ++i) {
      const double g = dot(rd->p + i * n, rd->p + j * n, n);
      const double d = fabs(g - (i == j ? 1.0 : 0.0));
      dev_p = (dev_p < d) ? d : dev_p;
    }
  const double md = (dev_v < dev_p) ? dev_p : dev_v;
  if (max_dev) *max_dev = md;
  if (md > 1e-6) return E_STALE;
  double* vg = dalloc(s * s);
  double* ev = dalloc(s);
  for (int64_t j = 0; j < s; ++j)
    for (int64_t i = 0; i < s; ++i) vg[i + j * s] = dot(rd->v + i * n, rd->v + j * n, n);
  sym_eigenvalues(vg, s, ev);
  const double smin = sqrt(fmax(0.0, ev[0])), smax = sqrt(fmax(0.0, ev[s - 1]));
  if (sigma_ratio) *sigma_ratio = smax > 0.0 ? smin / smax : 0.0;
  free(vg);
  free(ev);
  return E_OK;
}

/* ---- idrstab.cpp:89-191: bicg_projection, level_iteration, poly_combination ---------------- */
typedef struct {
  int64_t n, s, ell;
  double* x0;
  double** r;   /* r^(0..ell) */
  double** v;   /* V^(-1..ell), index level+1, each n x s */
} cycle_state;

/* bicg_projection (idrstab.cpp:89-94): gamma = (P^H B)^-1 P^H t */
static int bicg(const double* p, const double* blk, const double* t, int64_t n, int64_t s, double* gamma) {
  double* m = dalloc(s * s);
  double* rhs = dalloc(s);
  for (int64_t j = 0; j < s; ++j)
    for (int64_t i = 0; i < s; ++i) m[i + j * s] = dot(p + i * n, blk + j * n, n);
  for (int64_t j = 0; j < s; ++j) rhs[j] = dot(p + j * n, t, n);
  int rc = orc_solve_small(s, m, rhs, gamma);
  free(m);
  free(rhs);
  return rc;
}

static int level_iteration(cycle_state* st, const orc_csr* a, const double* p, int64_t k, int64_t* h_mv) {
  const int64_t n = st->n, s = st->s;
  double* gamma = dalloc(s);
  double* corr = dalloc(n);
  int rc = bicg(p, st->v[k + 1], st->r[k], n, s, gamma);
  if (rc) goto done;
  for (int64_t i = 0; i <= k; ++i) {
    gemv(st->v[i + 1], n, s, gamma, corr);
    for (int64_t t = 0; t < n; ++t) st->r[i][t] -= corr[t];
  }
  gemv(st->v[0], n, s, gamma, corr);
  for (int64_t t = 0; t < n; ++t) st->x0[t] += corr[t];
  orc_spmv(a, st->r[k], st->r[k + 1]);
  (*h_mv)++;
  {
    double* rhs = dalloc(s);
    double* msys = dalloc(s * s);
    double* eta = dalloc(s);
    double* newcol = dalloc(n);
    for (int64_t j = 0; j < s; ++j) rhs[j] = dot(p + j * n, st->r[k + 1], n);
    for (int64_t q = 0; q < s && !rc; ++q) {
      for (int64_t c = 0; c < s; ++c) {
        const double* mixed = c < q ? st->v[k + 2] + c * n : st->v[k + 1] + c * n;
        for (int64_t i = 0; i < s; ++i) msys[i + c * s] = dot(p + i * n, mixed, n);
      }
      rc = orc_solve_small(s, msys, rhs, eta);
      if (rc) break;
      for (int64_t i = -1; i <= k; ++i) {
        memcpy(newcol, st->r[i + 1], sizeof(double) * (size_t)n);
        for (int64_t c = 0; c < s; ++c) {
          const double* mixed = c < q ? st->v[i + 2] + c * n : st->v[i + 1] + c * n;
          axpy(-eta[c], mixed, newcol, n);
        }
        memcpy(st->v[i + 1] + q * n, newcol, sizeof(double) * (size_t)n);
      }
      orc_spmv(a, st->v[k + 1] + q * n, st->v[k + 2] + q * n);
      (*h_mv)++;
    }
    free(rhs);
    free(msys);
    free(eta);
    free(newcol);
  }
done:
  free(gamma);
  free(corr);
  return rc;
}

/* poly_combination (idrstab.cpp:154-191); writes x, r, u, v; tau (ell) after the tail guard */
static int poly(const cycle_state* st, double* x, double* r, double* u, double* v, double* tau) {
  const int64_t n = st->n, s = st->s, ell = st->ell;
  double* z = dalloc(n * ell);
  for (int64_t i = 0; i < ell; ++i) memcpy(z + i * n, st->r[i + 1], sizeof(double) * (size_t)n);
  int rc = orc_least_squares(n, ell, z, st->r[0], tau);
  free(z);
  if (rc) return rc;
  double tmax = 0.0;
  for (int64_t i = 0; i < ell; ++i) tmax = (tmax < fabs(tau[i])) ? fabs(tau[i]) : tmax;
  double* tail = &tau[ell - 1];
  if (fabs(*tail) < 1e-12 * tmax || tmax == 0.0) {
    const double target = tmax > 0.0 ? 1e-12 * tmax : 1e-12;
    *tail = fabs(*tail) > 0.0 ? *tail * (target / fabs(*tail)) : target;
  }
  memcpy(r, st->r[0], sizeof(double) * (size_t)n);
  memcpy(x, st->x0, sizeof(double) * (size_t)n);
  for (int64_t i = 1; i <= ell; ++i) {
    axpy(-tau[i - 1], st->r[i], r, n);
    axpy(tau[i - 1], st->r[i - 1], x, n);
  }
  memcpy(u, st->v[0], sizeof(double) * (size_t)(n * s));
  memcpy(v, st->v[1], sizeof(double) * (size_t)(n * s));
  for (int64_t q = 0; q < s; ++q)
    for (int64_t i = 1; i <= ell; ++i) {
      axpy(-tau[i - 1], st->v[i] + q * n, u + q * n, n);
      axpy(-tau[i - 1], st->v[i + 1] + q * n, v + q * n, n);
    }
  return E_OK;
}

/* extract_omegas (idrstab.cpp:28-41) */
static int extract_omegas(const double* tau, int64_t ell, double complex* out, int64_t* cnt) {
  if (ell == 1) {
    out[(*cnt)++] = tau[0];
    return 1;
  }
  if (ell == 2) {
    const double complex t0 = tau[0], t1 = tau[1];
    const double complex disc = csqrt(t0 * t0 + 4.0 * t1);
    out[(*cnt)++] = (t0 + disc) / 2.0;
    out[(*cnt)++] = (t0 - disc) / 2.0;
    return 1;
  }
  return 0;
}

static void make_recycle(orc_recycle* d, int64_t n, int64_t s, const double* p, const double* u,
                         const double* v, const double complex* om, int64_t om_cnt, int64_t level,
                         uint64_t fp) {
  d->n = n;
  d->s = s;
  d->level_j = level;
  d->fingerprint = fp;
  d->p = dcopy(p, n * s);
  d->u = dcopy(u, n * s);
  d->v = dcopy(v, n * s);
  d->omega_count = om_cnt;
  d->omega = dalloc(2 * om_cnt);
  for (int64_t i = 0; i < om_cnt; ++i) {
    d->omega[2 * i] = creal(om[i]);
    d->omega[2 * i + 1] = cimag(om[i]);
  }
}

/* idrstab_solve / mstab_solve (idrstab.cpp:193-307) */
int orc_solve(const orc_csr* a, const double* b, const double* x0, const orc_cfg* cfg,
              const orc_recycle* recycle, int32_t fetch_kind, int64_t fetch_cycle, orc_result* out) {
  memset(out, 0, sizeof(*out));
  if (cfg->s < 1 || cfg->ell < 1 || !(cfg->tol > 0.0) || cfg->max_mv < cfg->s + 1) return E_CONFIG;
  const int64_t n = a->n, s = cfg->s, ell = cfg->ell;
  if (!all_finite(b, n)) return E_ERROR;
  out->bnorm = norm2(b, n);
  double* x = x0 ? dcopy(x0, n) : dalloc(n);
  double* r = dcopy(b, n);
  if (!is_zero(x, n)) {
    if (!all_finite(x, n)) {
      free(x);
      free(r);
      return E_ERROR;
    }
    double* ax = dalloc(n);
    orc_spmv(a, x, ax);
    for (int64_t i = 0; i < n; ++i) r[i] -= ax[i];
    free(ax);
    out->h_mv_aux++;
  }
  const uint64_t fp = orc_fingerprint(a);
  double *p = NULL, *u = NULL, *v = NULL;
  int64_t base_level = 0;
  int64_t om_cap = 2 * (100000 + (recycle ? recycle->omega_count : 0)) + 16;
  double complex* omegas = malloc(sizeof(double complex) * (size_t)om_cap);
  int64_t om_cnt = 0;
  int complete = 1;
  if (recycle) {
    int rc = orc_validate(a, recycle, NULL, NULL);
    if (rc) {
      free(x);
      free(r);
      free(omegas);
      return rc;
    }
    out->h_mv_aux += recycle->s;
    if (recycle->s != s) {
      free(x);
      free(r);
      free(omegas);
      return E_CONFIG;
    }
    p = dcopy(recycle->p, n * s);
    u = dcopy(recycle->u, n * s);
    v = dcopy(recycle->v, n * s);
    base_level = recycle->level_j;
    for (int64_t i = 0; i < recycle->omega_count; ++i)
      omegas[om_cnt++] = recycle->omega[2 * i] + I * recycle->omega[2 * i + 1];
    complete = om_cnt == base_level;
    if (!complete) om_cnt = 0;
  } else {
    p = dalloc(n * s);
    u = dalloc(n * s);
    v = dalloc(n * s);
    if (orc_cut_space(n, s, cfg->seed, p) != E_OK) {
      free(x); free(r); free(omegas); free(p); free(u); free(v);
      return E_ERROR;
    }
    orc_rng* rng = malloc(sizeof(orc_rng));
    rng_seed(rng, cfg->seed ^ 0x9e3779b97f4a7c15ull);
    int rc = arnoldi(a, r, s, rng, u, v);
    free(rng);
    if (rc) {
      free(x); free(r); free(omegas); free(p); free(u); free(v);
      return rc;
    }
    out->h_mv += s;
  }
  double resnorm = norm2(r, n);
  int64_t level = 0;
  int64_t hist_cap = 64;
  out->hist = malloc(sizeof(int64_t) * 3 * (size_t)hist_cap);
  out->hist_resnorm = malloc(sizeof(double) * (size_t)hist_cap);
  int64_t tau_cap = 64;
  out->tau = malloc(sizeof(double) * (size_t)tau_cap);
#define PUSH_HIST(cyc, lvl, rn)                                                     \
  do {                                                                              \
    if (out->hist_len == hist_cap) {                                                \
      hist_cap *= 2;                                                                \
      out->hist = realloc(out->hist, sizeof(int64_t) * 3 * (size_t)hist_cap);       \
      out->hist_resnorm = realloc(out->hist_resnorm, sizeof(double) * (size_t)hist_cap); \
    }                                                                               \
    out->hist[3 * out->hist_len] = (cyc);                                           \
    out->hist[3 * out->hist_len + 1] = out->h_mv + out->h_mv_aux;                   \
    out->hist[3 * out->hist_len + 2] = (lvl);                                       \
    out->hist_resnorm[out->hist_len] = (rn);                                        \
    out->hist_len++;                                                                \
  } while (0)
  PUSH_HIST(0, base_level, resnorm);
  const double threshold = cfg->tol * out->bnorm;
  cycle_state st;
  st.n = n;
  st.s = s;
  st.ell = ell;
  st.x0 = dalloc(n);
  st.r = malloc(sizeof(double*) * (size_t)(ell + 1));
  st.v = malloc(sizeof(double*) * (size_t)(ell + 2));
  for (int64_t i = 0; i <= ell; ++i) st.r[i] = dalloc(n);
  for (int64_t i = 0; i <= ell + 1; ++i) st.v[i] = dalloc(n * s);
  double* tau = dalloc(ell);
  int broke = 0;
  while (resnorm > threshold && out->h_mv < cfg->max_mv) {
    memcpy(st.x0, x, sizeof(double) * (size_t)n);
    memcpy(st.r[0], r, sizeof(double) * (size_t)n);
    memcpy(st.v[0], u, sizeof(double) * (size_t)(n * s));
    memcpy(st.v[1], v, sizeof(double) * (size_t)(n * s));
    int rc = E_OK;
    for (int64_t k = 0; k < ell && !rc; ++k) rc = level_iteration(&st, a, p, k, &out->h_mv);
    if (!rc) {
      double* nx = dalloc(n);
      double* nr = dalloc(n);
      double* nu = dalloc(n * s);
      double* nv = dalloc(n * s);
      rc = poly(&st, nx, nr, nu, nv, tau);
      if (!rc) {
        free(x); free(r); free(u); free(v);
        x = nx; r = nr; u = nu; v = nv;
      } else {
        free(nx); free(nr); free(nu); free(nv);
      }
    }
    if (rc) {
      out->status = 2;
      strcpy(out->reason, rc == E_RANK ? "least_squares_tall: stabilization block lost rank"
                                       : "solve_small: pivot collapse");
      broke = 1;
      break;
    }
    out->cycles++;
    level += ell;
    out->h_rd = level * s + (recycle ? base_level * (s - 1) : 0);
    if (complete) complete = extract_omegas(tau, ell, omegas, &om_cnt);
    if (out->tau_len + ell > tau_cap) {
      tau_cap = 2 * (tau_cap + ell);
      out->tau = realloc(out->tau, sizeof(double) * (size_t)tau_cap);
    }
    for (int64_t i = 0; i < ell; ++i) out->tau[out->tau_len++] = tau[i];
    if (cfg->true_residual) {
      double* ax = dalloc(n);
      orc_spmv(a, x, ax);
      for (int64_t i = 0; i < n; ++i) r[i] = b[i] - ax[i];
      free(ax);
      out->h_mv_aux++;
    }
    resnorm = norm2(r, n);
    PUSH_HIST((int64_t)out->cycles, base_level + level, resnorm);
    if (fetch_kind != 2 && !out->has_fetched) {
      const int hit = (fetch_kind == 0 && out->cycles == fetch_cycle) ||
                      (fetch_kind == 1 && resnorm <= sqrt(cfg->tol) * out->bnorm);
      if (hit) {
        make_recycle(&out->fetched, n, s, p, u, v, omegas, complete ? om_cnt : 0, base_level + level, fp);
        out->has_fetched = 1;
      }
    }
    if (om_cnt + 2 >= om_cap) complete = 0;
  }
#undef PUSH_HIST
  if (!broke) out->status = resnorm <= threshold ? 0 : 1;
  out->final_resnorm = resnorm;
  out->x = x;
  make_recycle(&out->final_data, n, s, p, u, v, omegas, complete ? om_cnt : 0, base_level + level, fp);
  free(r); free(p); free(u); free(v); free(omegas); free(tau);
  free(st.x0);
  for (int64_t i = 0; i <= ell; ++i) free(st.r[i]);
  for (int64_t i = 0; i <= ell + 1; ++i) free(st.v[i]);
  free(st.r);
  free(st.v);
  return E_OK;
}

static void free_recycle(orc_recycle* d) {
  free(d->p);
  free(d->u);
  free(d->v);
  free(d->omega);
  memset(d, 0, sizeof(*d));
}

void orc_result_free(orc_result* r) {
  free(r->x);
  free(r->hist);
  free(r->hist_resnorm);
  free(r->tau);
  free_recycle(&r->final_data);
  if (r->has_fetched) free_recycle(&r->fetched);
  memset(r, 0, sizeof(*r));
}
