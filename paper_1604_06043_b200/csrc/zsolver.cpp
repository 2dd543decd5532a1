// zsolver.cpp — the complex128 solve path: idrstab_solve / mstab_solve, validate,
// make_cut_space and arnoldi_init of the reference (idrstab.cpp:45-307, recycle.cpp:40-83,
// baselines.cpp:36-47, kernels.cpp:20-154) for complex A, b, x0 or recycle data.
//
// Every length-N step runs on the device (kcomplex.cu): the SpMV, the axpy chains of the level
// iteration and the polynomial combination, the P^H products, norms and Gram-Schmidt sweeps. The
// s x s and ell x ell dense steps (LuFactor, the R factor of the least squares, the Hermitian Jacobi
// eigenvalues of validate) run on the host in std::complex<double> between the launches, from the
// reduced values of one small device-to-host copy each. This is the first complex build: one host
// synchronisation per reduction instead of the fused finalisers and cycle graphs of the real path
// (DESIGN.md §3.4 states the cost); the real fp64 path is untouched.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>

#include "solver.h"

#define CUDA_OK(expr)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) throw Error(MSTAB_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace mstab_b200 {

namespace {

using Z = std::complex<double>;
using Clock = std::chrono::steady_clock;
int64_t ns_since(Clock::time_point t0) {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count();
}

struct Breakdown : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Column-major s x s complex matrix on the host.
struct ZMat {
  int n = 0;
  std::vector<Z> a;
  explicit ZMat(int n_ = 0) : n(n_), a((size_t)n_ * n_, Z(0.0)) {}
  Z& operator()(int i, int j) { return a[(size_t)i + (size_t)j * n]; }
  const Z& operator()(int i, int j) const { return a[(size_t)i + (size_t)j * n]; }
};

// solve_small / LuFactor (kernels.cpp:95-154)
std::vector<Z> solve_small(ZMat lu, const std::vector<Z>& rhs) {
  const int n = lu.n;
  std::vector<int> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  double scale = 0.0;
  for (const Z& z : lu.a) scale = std::max(scale, std::abs(z));
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = std::abs(lu(k, k));
    for (int i = k + 1; i < n; ++i) {
      const double m = std::abs(lu(i, k));
      if (m > best) {
        best = m;
        piv = i;
      }
    }
    if (best < 1e-14 * scale || scale == 0.0) throw Breakdown("solve_small: pivot collapse");
    if (piv != k) {
      std::swap(perm[k], perm[piv]);
      for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(piv, j));
    }
    const Z inv = 1.0 / lu(k, k);
    for (int i = k + 1; i < n; ++i) {
      const Z m = lu(i, k) * inv;
      lu(i, k) = m;
      if (m != Z(0.0))
        for (int j = k + 1; j < n; ++j) lu(i, j) -= m * lu(k, j);
    }
  }
  std::vector<Z> x(n);
  for (int i = 0; i < n; ++i) x[i] = rhs[perm[i]];
  for (int i = 1; i < n; ++i)
    for (int j = 0; j < i; ++j) x[i] -= lu(i, j) * x[j];
  for (int i = n; i-- > 0;) {
    for (int j = i + 1; j < n; ++j) x[i] -= lu(i, j) * x[j];
    x[i] /= lu(i, i);
  }
  return x;
}

// hermitian_eigenvalues (kernels.cpp:156-208): cyclic Jacobi with a phase similarity per rotation
std::vector<double> hermitian_eigenvalues(ZMat a) {
  const int n = a.n;
  double off = 0.0, total = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double m = std::norm(a(i, j));
      total += m;
      if (i != j) off += m;
    }
  const double stop = 1e-28 * std::max(total, 1e-300);
  for (int sweep = 0; sweep < 60 && off > stop; ++sweep) {
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const Z apq = a(p, q);
        const double m = std::abs(apq);
        if (m == 0.0) continue;
        const Z phase = apq / m;
        const double theta = (a(q, q).real() - a(p, p).real()) / (2.0 * m);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(1.0 + theta * theta));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = t * c;
        for (int k = 0; k < n; ++k) {
          const Z akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * std::conj(phase) * akq;
          a(k, q) = s * akp + c * std::conj(phase) * akq;
        }
        for (int k = 0; k < n; ++k) {
          const Z apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * phase * aqk;
          a(q, k) = s * apk + c * phase * aqk;
        }
      }
    off = 0.0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        if (i != j) off += std::norm(a(i, j));
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = a(i, i).real();
  std::sort(ev.begin(), ev.end());
  return ev;
}

// extract_omegas (idrstab.cpp:28-41)
bool extract_omegas_z(const std::vector<Z>& tau, std::vector<Z>& out) {
  if (tau.size() == 1) {
    out.push_back(tau[0]);
    return true;
  }
  if (tau.size() == 2) {
    const Z disc = std::sqrt(tau[0] * tau[0] + 4.0 * tau[1]);
    out.push_back((tau[0] + disc) / 2.0);
    out.push_back((tau[0] - disc) / 2.0);
    return true;
  }
  return false;
}

// Device-side toolkit of one context: launches on its stream and reads reduced values back.
struct ZDev {
  Context& ctx;
  int64_t n, ld;
  cudaStream_t st;
  DevPtr red;          // reduction landing area (device)
  DevPtr coef;         // eta / gamma of one level for the deferred rebuild (device)
  double* host = nullptr;  // pinned mirror
  double* host_coef = nullptr;  // pinned staging of coef
  static constexpr int kRed = 2 * kZMaxTerms * kZMaxTerms + 64;
  ZDev(Context& c, int64_t n_) : ctx(c), n(n_), ld(padded_ld(n_)), st(c.stream()) {
    red = ctx.alloc(sizeof(double) * kRed);
    coef = ctx.alloc(sizeof(double) * 2 * (kMaxS * kMaxS + kMaxS));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host), sizeof(double) * kRed));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host_coef), sizeof(double) * 2 * (kMaxS * kMaxS + kMaxS)));
  }
  ~ZDev() {
    if (host) cudaFreeHost(host);
    if (host_coef) cudaFreeHost(host_coef);
  }
  // every launch that read the previous contents is behind a stream synchronisation (the dots of
  // the column loop), so the staging buffer is free to overwrite
  void upload_coef(const std::vector<Z>& c) {
    std::memcpy(host_coef, c.data(), sizeof(Z) * c.size());
    CUDA_OK(cudaMemcpyAsync(coef->ptr, host_coef, sizeof(Z) * c.size(), cudaMemcpyHostToDevice, st));
  }
  DevPtr block(int64_t cols) { return ctx.alloc(sizeof(double) * 2 * (size_t)ld * (size_t)std::max<int64_t>(cols, 1)); }
  double* col(const DevPtr& b, int64_t c) const { return static_cast<double*>(b->ptr) + 2 * ld * c; }
  void check() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(MSTAB_E_CUDA, std::string("launch: ") + cudaGetErrorString(e));
  }
  const double* fetch(int count) {
    CUDA_OK(cudaMemcpyAsync(host, red->ptr, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    return host;
  }
  void copy(double* dst, const double* src, int64_t cols = 1) {
    CUDA_OK(cudaMemcpyAsync(dst, src, sizeof(double) * 2 * (size_t)ld * (size_t)cols, cudaMemcpyDeviceToDevice, st));
  }
  void spmv(const ZOperator& a, const double* x, double* y) {
    launch_zspmv(st, n, a.nnz, static_cast<const int32_t*>(a.rp->ptr), static_cast<const int32_t*>(a.ci->ptr),
                 static_cast<const double*>(a.val->ptr), x, y);
    check();
  }
  // dots of m columns (given by pointer) against y, returned as complex values
  std::vector<Z> dots(const std::vector<const double*>& cols, const double* y) {
    ZTerms t;
    t.m = (int)cols.size();
    for (int c = 0; c < t.m; ++c) t.col[c] = cols[c];
    launch_zdots(st, n, t, y, static_cast<double*>(red->ptr), ctx.reducer());
    check();
    const double* h = fetch(2 * t.m);
    std::vector<Z> out(t.m);
    for (int c = 0; c < t.m; ++c) out[c] = Z(h[2 * c], h[2 * c + 1]);
    return out;
  }
  std::vector<Z> block_dots(const DevPtr& b, int m, const double* y) {
    std::vector<const double*> cols(m);
    for (int c = 0; c < m; ++c) cols[c] = col(b, c);
    return dots(cols, y);
  }
  Z dot(const double* a, const double* y) { return dots({a}, y)[0]; }
  double norm2(const double* x) {
    ZTerms t;
    t.m = 1;
    t.col[0] = x;
    launch_zdots(st, n, t, nullptr, static_cast<double*>(red->ptr), ctx.reducer());
    check();
    return std::sqrt(fetch(2)[0]);
  }
  // y_out = y_in (+ chain | +/- gemv) of coef_c * col_c
  void axpys(int mode, double* y_out, const double* y_in, const std::vector<const double*>& cols,
             const std::vector<Z>& coef) {
    ZTerms t;
    t.m = (int)cols.size();
    for (int c = 0; c < t.m; ++c) {
      t.col[c] = cols[c];
      t.re[c] = coef[c].real();
      t.im[c] = coef[c].imag();
    }
    launch_zaxpys(st, n, mode, y_out, y_in, t);
    check();
  }
  void axpy(Z alpha, const double* x, double* y) { axpys(0, y, y, {x}, {alpha}); }
  void scale(int mode, double* y, const double* x, double a) {
    launch_zscale(st, n, mode, y, x, a);
    check();
  }
  struct Stats {
    double sumsq, nonfinite, nonzero, imag;
  };
  Stats stats(const double* x) {
    launch_zstats(st, n, x, static_cast<double*>(red->ptr), ctx.reducer());
    check();
    const double* h = fetch(4);
    return {h[0], h[1], h[2], h[3]};
  }
};

void upload_z(Context& ctx, double* dst, const double* src, int64_t n, int64_t ld, int64_t cols, int mem) {
  CUDA_OK(cudaMemcpy2DAsync(dst, sizeof(double) * 2 * ld, src, sizeof(double) * 2 * n, sizeof(double) * 2 * n,
                            (size_t)cols, mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            ctx.stream()));
}
void download_z(Context& ctx, double* dst, const double* src, int64_t n, int64_t ld, int64_t cols, int mem) {
  CUDA_OK(cudaMemcpy2DAsync(dst, sizeof(double) * 2 * n, src, sizeof(double) * 2 * ld, sizeof(double) * 2 * n,
                            (size_t)cols, mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                            ctx.stream()));
}

// make_cut_space (baselines.cpp:36-47) with orthonormalize (kernels.cpp:20-50: classical
// Gram-Schmidt applied twice, all coefficients of a pass formed before the updates)
DevPtr make_cut_space_z(ZDev& d, int s, uint64_t seed, bool real) {
  const int64_t n = d.n;
  NormalStream* ns = normal_stream_create(seed);
  struct Guard {
    NormalStream* p;
    ~Guard() { normal_stream_destroy(p); }
  } guard{ns};
  std::vector<double> draws, host((size_t)2 * n * s);
  for (int attempt = 0; attempt < 4; ++attempt) {
    if (real) {
      draws.resize((size_t)n * s);
      normal_stream_fill(ns, draws.data(), (int64_t)draws.size());
      for (size_t i = 0; i < draws.size(); ++i) {
        host[2 * i] = draws[i];
        host[2 * i + 1] = 0.0;
      }
    } else {
      // Complex(normal(rng), normal(rng)) (baselines.cpp:42): g++ evaluates the two arguments right
      // to left, so an entry's FIRST draw is its imaginary part (pinned by tests/test_gpu_complex.py
      // against the reference's P)
      normal_stream_fill(ns, host.data(), (int64_t)host.size());
      for (size_t i = 0; i < host.size(); i += 2) std::swap(host[i], host[i + 1]);
    }
    DevPtr g = d.block(s), q = d.block(s), w = d.block(1);
    upload_z(d.ctx, static_cast<double*>(g->ptr), host.data(), n, d.ld, s, MSTAB_MEM_HOST);
    int rank = 0;
    for (int j = 0; j < s; ++j) {
      const double norm0 = d.norm2(d.col(g, j));
      d.copy(d.col(w, 0), d.col(g, j));
      for (int pass = 0; pass < 2 && rank > 0; ++pass) {
        std::vector<Z> coeff = d.block_dots(q, rank, d.col(w, 0));
        std::vector<const double*> cols(rank);
        for (int i = 0; i < rank; ++i) {
          cols[i] = d.col(q, i);
          coeff[i] = -coeff[i];
        }
        d.axpys(0, d.col(w, 0), d.col(w, 0), cols, coeff);
      }
      const double res = d.norm2(d.col(w, 0));
      if (res <= 1e-10 * norm0 || norm0 == 0.0) continue;
      d.scale(0, d.col(q, rank), d.col(w, 0), 1.0 / res);
      ++rank;
    }
    if (rank == s) return q;
  }
  throw Error(MSTAB_E_ERROR, "make_cut_space: could not draw a full-rank cut-space");
}

// arnoldi_init (idrstab.cpp:45-87)
void arnoldi_init_z(ZDev& d, const ZOperator& a, const double* r0, int s, uint64_t rng_seed, bool real, DevPtr& U,
                    DevPtr& V, int64_t& mv_cost) {
  const int64_t n = d.n;
  const double r0norm = d.norm2(r0);
  if (r0norm == 0.0) throw Error(MSTAB_E_ERROR, "arnoldi_init: zero start vector");
  d.scale(1, d.col(U, 0), r0, r0norm);
  DevPtr w = d.block(1);
  NormalStream* ns = nullptr;
  struct Guard {
    NormalStream*& p;
    ~Guard() {
      if (p) normal_stream_destroy(p);
    }
  } guard{ns};
  auto mgs2 = [&](int k) {
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i <= k; ++i) d.axpy(-d.dot(d.col(U, i), d.col(w, 0)), d.col(U, i), d.col(w, 0));
  };
  for (int k = 0; k < s; ++k) {
    d.spmv(a, d.col(U, k), d.col(V, k));
    mv_cost++;
    if (k + 1 == s) break;
    d.copy(d.col(w, 0), d.col(V, k));
    const double wnorm0 = d.norm2(d.col(w, 0));
    mgs2(k);
    double wnorm = d.norm2(d.col(w, 0));
    while (wnorm <= 1e-12 * std::max(wnorm0, 1.0)) {
      if (!ns) ns = normal_stream_create(rng_seed);
      std::vector<double> host((size_t)2 * n);
      if (real) {
        std::vector<double> draws((size_t)n);
        normal_stream_fill(ns, draws.data(), n);
        for (int64_t i = 0; i < n; ++i) {
          host[2 * i] = draws[i];
          host[2 * i + 1] = 0.0;
        }
      } else {
        normal_stream_fill(ns, host.data(), 2 * n);  // imaginary part drawn first (see make_cut_space_z)
        for (size_t i = 0; i < host.size(); i += 2) std::swap(host[i], host[i + 1]);
      }
      upload_z(d.ctx, d.col(w, 0), host.data(), n, d.ld, 1, MSTAB_MEM_HOST);
      CUDA_OK(cudaStreamSynchronize(d.st));  // host is reused by the next draw
      mgs2(k);
      wnorm = d.norm2(d.col(w, 0));
    }
    d.scale(1, d.col(U, k + 1), d.col(w, 0), wnorm);
  }
}

// least_squares_tall (kernels.cpp:52-93): MGS with reiteration on a copy of Z, tau = R^-1 Q^H r
std::vector<Z> least_squares_z(ZDev& d, const std::vector<const double*>& zcols, const double* r, DevPtr& q) {
  const int ell = (int)zcols.size();
  double max_colnorm = 0.0;
  for (int j = 0; j < ell; ++j) max_colnorm = std::max(max_colnorm, d.norm2(zcols[j]));
  for (int j = 0; j < ell; ++j) d.copy(d.col(q, j), zcols[j]);
  ZMat rr(ell);
  double min_diag = std::numeric_limits<double>::infinity();
  for (int k = 0; k < ell; ++k) {
    double* qk = d.col(q, k);
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < k; ++i) {
        const Z c = d.dot(d.col(q, i), qk);
        d.axpy(-c, d.col(q, i), qk);
        rr(i, k) += c;
      }
    const double dn = d.norm2(qk);
    rr(k, k) = dn;
    min_diag = std::min(min_diag, dn);
    if (dn > 0.0) d.scale(0, qk, qk, 1.0 / dn);
  }
  if (min_diag < 1e-13 * max_colnorm) throw Breakdown("least_squares_tall: stabilization block lost rank");
  std::vector<Z> tau = d.block_dots(q, ell, r);
  for (int k = ell; k-- > 0;) {
    for (int j = k + 1; j < ell; ++j) tau[k] -= rr(k, j) * tau[j];
    tau[k] /= rr(k, k);
  }
  return tau;
}

std::shared_ptr<ZRecycle> fetch_z(ZDev& d, const DevPtr& p, const DevPtr& u, const DevPtr& v, int s,
                                  std::vector<Z> omega, int64_t level_j, uint64_t fp) {
  auto f = std::make_shared<ZRecycle>();
  f->n = d.n;
  f->s = s;
  f->level_j = level_j;
  f->fingerprint = fp;
  f->p = p;  // immutable, shared
  f->u = d.block(s);
  f->v = d.block(s);
  d.copy(static_cast<double*>(f->u->ptr), static_cast<const double*>(u->ptr), s);
  d.copy(static_cast<double*>(f->v->ptr), static_cast<const double*>(v->ptr), s);
  f->omega = std::move(omega);
  return f;
}

}  // namespace

std::shared_ptr<ZOperator> make_operator_z(Context& ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                           const double* values_re_im) {
  // CsrMatrix::validate (csr.cpp:11-24) + square (operator.cpp:21-23)
  if (n < 0 || !row_ptr) throw Error(MSTAB_E_ERROR, "csr: bad dimensions");
  if (row_ptr[0] != 0) throw Error(MSTAB_E_ERROR, "csr: row_ptr[0] != 0");
  for (int64_t i = 0; i < n; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) throw Error(MSTAB_E_ERROR, "csr: row_ptr not monotone");
  const int64_t nnz = row_ptr[n];
  if (nnz >= (int64_t(1) << 31) || n >= (int64_t(1) << 31)) throw Error(MSTAB_E_CONFIG, "b200: nnz and n below 2^31");
  for (int64_t k = 0; k < nnz; ++k)
    if (col_idx[k] < 0 || col_idx[k] >= n) throw Error(MSTAB_E_ERROR, "csr: column index out of range");
  auto op = std::make_shared<ZOperator>();
  op->n = n;
  op->nnz = nnz;
  // CsrMatrix::checksum (csr.cpp:28-43): FNV-1a over dims, row_ptr, col_idx (as u64) and the values
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](const void* p, size_t len) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < len; ++i) {
      h ^= b[i];
      h *= 1099511628211ull;
    }
  };
  const uint64_t dims[3] = {(uint64_t)n, (uint64_t)n, (uint64_t)nnz};
  mix(dims, sizeof(dims));
  for (int64_t i = 0; i <= n; ++i) {
    const uint64_t v = (uint64_t)row_ptr[i];
    mix(&v, 8);
  }
  for (int64_t k = 0; k < nnz; ++k) {
    const uint64_t v = (uint64_t)col_idx[k];
    mix(&v, 8);
  }
  mix(values_re_im, (size_t)nnz * 16);
  op->fingerprint = h;
  op->real = true;
  for (int64_t k = 0; k < nnz; ++k)
    if (values_re_im[2 * k + 1] != 0.0) {
      op->real = false;
      break;
    }
  std::vector<int32_t> rp32((size_t)n + 1), ci32((size_t)nnz);
  for (int64_t i = 0; i <= n; ++i) rp32[(size_t)i] = (int32_t)row_ptr[i];
  for (int64_t k = 0; k < nnz; ++k) ci32[(size_t)k] = (int32_t)col_idx[k];
  op->rp = ctx.alloc(sizeof(int32_t) * ((size_t)n + 1));
  op->ci = ctx.alloc(sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1));
  op->val = ctx.alloc(sizeof(double) * 2 * (size_t)std::max<int64_t>(nnz, 1));
  CUDA_OK(cudaMemcpyAsync(op->rp->ptr, rp32.data(), sizeof(int32_t) * rp32.size(), cudaMemcpyHostToDevice, ctx.stream()));
  if (nnz > 0) {
    CUDA_OK(cudaMemcpyAsync(op->ci->ptr, ci32.data(), sizeof(int32_t) * ci32.size(), cudaMemcpyHostToDevice, ctx.stream()));
    CUDA_OK(cudaMemcpyAsync(op->val->ptr, values_re_im, sizeof(double) * 2 * (size_t)nnz, cudaMemcpyHostToDevice,
                            ctx.stream()));
  }
  ctx.sync();
  return op;
}

void apply_z(Context& ctx, const ZOperator& op, const double* x, double* y, int mem) {
  ZDev d(ctx, op.n);
  DevPtr xv = d.block(1), yv = d.block(1);
  upload_z(ctx, d.col(xv, 0), x, op.n, d.ld, 1, mem);
  d.spmv(op, d.col(xv, 0), d.col(yv, 0));
  download_z(ctx, y, d.col(yv, 0), op.n, d.ld, 1, mem);
  ctx.sync();
}

std::shared_ptr<ZRecycle> make_recycle_z(Context& ctx, int64_t n, int64_t s, const double* p, const double* u,
                                         const double* v, int mem, const double* omega_re_im, int64_t omega_count,
                                         int64_t level_j, uint64_t fingerprint) {
  if (n < 1 || s < 1 || s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: recycle data needs n >= 1, 1 <= s <= 16");
  ZDev d(ctx, n);
  auto r = std::make_shared<ZRecycle>();
  r->n = n;
  r->s = s;
  r->level_j = level_j;
  r->fingerprint = fingerprint;
  r->p = d.block(s);
  r->u = d.block(s);
  r->v = d.block(s);
  upload_z(ctx, static_cast<double*>(r->p->ptr), p, n, d.ld, s, mem);
  upload_z(ctx, static_cast<double*>(r->u->ptr), u, n, d.ld, s, mem);
  upload_z(ctx, static_cast<double*>(r->v->ptr), v, n, d.ld, s, mem);
  for (int64_t i = 0; i < omega_count; ++i) r->omega.emplace_back(omega_re_im[2 * i], omega_re_im[2 * i + 1]);
  ctx.sync();
  return r;
}

void download_recycle_z(Context& ctx, const ZRecycle& rd, double* p, double* u, double* v, double* omega_re_im) {
  const int64_t ld = padded_ld(rd.n);
  if (p) download_z(ctx, p, static_cast<const double*>(rd.p->ptr), rd.n, ld, rd.s, MSTAB_MEM_HOST);
  if (u) download_z(ctx, u, static_cast<const double*>(rd.u->ptr), rd.n, ld, rd.s, MSTAB_MEM_HOST);
  if (v) download_z(ctx, v, static_cast<const double*>(rd.v->ptr), rd.n, ld, rd.s, MSTAB_MEM_HOST);
  if (omega_re_im)
    for (size_t i = 0; i < rd.omega.size(); ++i) {
      omega_re_im[2 * i] = rd.omega[i].real();
      omega_re_im[2 * i + 1] = rd.omega[i].imag();
    }
  ctx.sync();
}

// validate (recycle.cpp:40-83)
mstab_validation_report validate_z(Context& ctx, const ZRecycle& rd, const ZOperator& a) {
  if (rd.fingerprint != a.fingerprint) throw Error(MSTAB_E_FINGERPRINT, "recycle data belongs to a different operator");
  if (rd.n != a.n) throw Error(MSTAB_E_DIMENSION, "recycle data has inconsistent shapes");
  if (!rd.omega.empty() && (int64_t)rd.omega.size() != rd.level_j)
    throw Error(MSTAB_E_STALE, "recycle data: omega history length disagrees with level");
  ZDev d(ctx, rd.n);
  const int s = (int)rd.s;
  DevPtr au = d.block(1);
  double dev_num = 0.0, dev_den = 0.0;
  for (int q = 0; q < s; ++q) {
    d.spmv(a, d.col(rd.u, q), d.col(au, 0));
    launch_zdiff(d.st, d.n, d.col(rd.v, q), d.col(au, 0), static_cast<double*>(d.red->ptr), ctx.reducer());
    d.check();
    const double* h = d.fetch(2);
    dev_num += h[0];
    const double nv = std::sqrt(h[1]);
    dev_den += nv * nv;
  }
  const double dev_v = dev_den > 0.0 ? std::sqrt(dev_num) / std::sqrt(dev_den) : std::sqrt(dev_num);
  double dev_p = 0.0;
  for (int j = 0; j < s; ++j) {
    const std::vector<Z> gj = d.block_dots(rd.p, s, d.col(rd.p, j));  // gram(i, j) = p_i^H p_j
    for (int i = 0; i < s; ++i) dev_p = std::max(dev_p, std::abs(gj[i] - (i == j ? Z(1.0) : Z(0.0))));
  }
  mstab_validation_report rep{};
  rep.max_deviation = std::max(dev_v, dev_p);
  if (rep.max_deviation > 1e-6) throw Error(MSTAB_E_STALE, "recycle data deviates from its invariants");
  ZMat vg(s);
  for (int j = 0; j < s; ++j) {
    const std::vector<Z> gj = d.block_dots(rd.v, s, d.col(rd.v, j));
    for (int i = 0; i < s; ++i) vg(i, j) = gj[i];
  }
  const std::vector<double> ev = hermitian_eigenvalues(vg);
  const double smin = std::sqrt(std::max(0.0, ev.front()));
  const double smax = std::sqrt(std::max(0.0, ev.back()));
  rep.sigma_min_ratio = smax > 0.0 ? smin / smax : 0.0;
  rep.low_rank_warning = rep.sigma_min_ratio < 1e-10 ? 1 : 0;
  return rep;
}

// idrstab_solve / mstab_solve (idrstab.cpp:193-307) on complex data
std::unique_ptr<ZResult> solve_z(Context& ctx, const ZOperator& a, const double* b_in, const double* x0_in, int mem,
                                 const mstab_solver_config& cfg, const ZRecycle* recycle,
                                 const mstab_fetch_policy* fetch) {
  if (cfg.s < 1) throw Error(MSTAB_E_CONFIG, "config: s >= 1 required");
  if (cfg.ell < 1) throw Error(MSTAB_E_CONFIG, "config: ell >= 1 required");
  if (!(cfg.tol > 0.0)) throw Error(MSTAB_E_CONFIG, "config: tol > 0 required");
  if (cfg.max_mv < cfg.s + 1) throw Error(MSTAB_E_CONFIG, "config: max_mv >= s + 1 required");
  if (cfg.s > kMaxS || cfg.ell > kMaxEll) throw Error(MSTAB_E_CONFIG, "b200: s <= 16 and ell <= 8 are supported");
  if (fetch && fetch->kind == MSTAB_FETCH_AT_CYCLE && fetch->cycle < 1)
    throw Error(MSTAB_E_CONFIG, "fetch policy: cycle >= 1 required");
  if (ctx.sharded()) throw Error(MSTAB_E_CONFIG, "b200: the complex path is single-GPU");
  const int s = (int)cfg.s, ell = (int)cfg.ell;
  const int64_t n = a.n;
  ZDev d(ctx, n);
  const auto t0 = Clock::now();
  auto res = std::make_unique<ZResult>();
  res->n = n;
  mstab_report& rep = res->report;
  std::memset(&rep, 0, sizeof(rep));
  rep.ell = ell;

  DevPtr b = d.block(1), x = d.block(1), r = d.block(1), ax = d.block(1);
  upload_z(ctx, d.col(b, 0), b_in, n, d.ld, 1, mem);
  const ZDev::Stats sb = d.stats(d.col(b, 0));
  if (sb.nonfinite > 0.0) throw Error(MSTAB_E_ERROR, "idrstab rhs: non-finite entries");
  rep.bnorm = std::sqrt(sb.sumsq);
  bool x_real = true;
  bool x_zero = true;
  if (x0_in) {
    upload_z(ctx, d.col(x, 0), x0_in, n, d.ld, 1, mem);
    const ZDev::Stats sx = d.stats(d.col(x, 0));
    x_zero = sx.nonzero == 0.0;
    if (!x_zero && sx.nonfinite > 0.0) throw Error(MSTAB_E_ERROR, "idrstab guess: non-finite entries");
    x_real = sx.imag == 0.0;
  } else {
    CUDA_OK(cudaMemsetAsync(x->ptr, 0, x->bytes, d.st));
  }
  if (x_zero) {
    d.copy(d.col(r, 0), d.col(b, 0));
  } else {
    d.spmv(a, d.col(x, 0), d.col(ax, 0));
    launch_zsub(d.st, n, d.col(r, 0), d.col(b, 0), d.col(ax, 0));
    d.check();
    rep.h_mv_aux++;
  }

  DevPtr P, U = d.block(s), V = d.block(s);
  int64_t base_level = 0;
  std::vector<Z> omega_levels;
  bool omegas_complete = true;
  if (recycle) {
    validate_z(ctx, *recycle, a);
    rep.h_mv_aux += recycle->s;
    if (recycle->s != cfg.s) throw Error(MSTAB_E_CONFIG, "idrstab: recycle s != config s");
    P = recycle->p;
    d.copy(static_cast<double*>(U->ptr), static_cast<const double*>(recycle->u->ptr), s);
    d.copy(static_cast<double*>(V->ptr), static_cast<const double*>(recycle->v->ptr), s);
    base_level = recycle->level_j;
    omega_levels = recycle->omega;
    omegas_complete = (int64_t)omega_levels.size() == base_level;
    if (!omegas_complete) omega_levels.clear();
  } else {
    const bool real = a.real && sb.imag == 0.0 && x_real;
    P = make_cut_space_z(d, s, cfg.seed, real);
    // arnoldi_init's own test: real operator and real start vector r (idrstab.cpp:51)
    const bool r_real = d.stats(d.col(r, 0)).imag == 0.0;
    int64_t mv_cost = 0;
    arnoldi_init_z(d, a, d.col(r, 0), s, cfg.seed ^ 0x9e3779b97f4a7c15ull, a.real && r_real, U, V, mv_cost);
    rep.h_mv += mv_cost;
  }

  double resnorm = d.norm2(d.col(r, 0));
  int64_t level = 0;
  res->history.push_back({0, rep.h_mv + rep.h_mv_aux, base_level, resnorm, ns_since(t0)});
  const double threshold = cfg.tol * rep.bnorm;

  // cycle state: r^(0..ell) and V^(-1..ell) (work copies: a mid-cycle breakdown leaves x, r, U, V intact)
  std::vector<DevPtr> R(ell + 1), VL(ell + 2);
  for (auto& v : R) v = d.block(1);
  for (auto& v : VL) v = d.block(s);
  DevPtr xw = d.block(1), lsq = d.block(ell);
  DevPtr xo = d.block(1), ro = d.block(1), Uo = d.block(s), Vo = d.block(s);
  auto vl = [&](int i) -> DevPtr& { return VL[i + 1]; };  // level i in -1..ell
  std::vector<const double*> pcols(s);
  for (int c = 0; c < s; ++c) pcols[c] = d.col(P, c);

  try {
    while (resnorm > threshold && rep.h_mv < cfg.max_mv) {
      d.copy(d.col(xw, 0), d.col(x, 0));
      d.copy(d.col(R[0], 0), d.col(r, 0));
      d.copy(static_cast<double*>(vl(-1)->ptr), static_cast<const double*>(U->ptr), s);
      d.copy(static_cast<double*>(vl(0)->ptr), static_cast<const double*>(V->ptr), s);
      ZMat Ma(s), Mn(s);
      std::vector<Z> g(s);
      for (int k = 0; k < ell; ++k) {
        // (a) BiCG step: gamma = (P^H V^(k))^-1 P^H r^(k) (idrstab.cpp:110-121)
        if (k == 0) {
          for (int c = 0; c < s; ++c) {
            const std::vector<Z> mc = d.dots(pcols, d.col(vl(0), c));
            for (int i = 0; i < s; ++i) Ma(i, c) = mc[i];
          }
          g = d.dots(pcols, d.col(R[0], 0));
        }
        const std::vector<Z> gamma = solve_small(Ma, g);
        // top level now; the levels below (and x) take the same gamma in the deferred pass
        {
          std::vector<const double*> cols(s);
          for (int c = 0; c < s; ++c) cols[c] = d.col(vl(k), c);
          d.axpys(2, d.col(R[k], 0), d.col(R[k], 0), cols, gamma);
        }
        // (b) raise the residual one level
        d.spmv(a, d.col(R[k], 0), d.col(R[k + 1], 0));
        rep.h_mv++;
        // (c) rebuild the columns against the mixed block, raise each one level (idrstab.cpp:127-151).
        // Only the top level's column feeds the next product; levels -1..k-1 are rebuilt after the
        // loop in one pass with the same coefficients (launch_zrebuild_deferred).
        const std::vector<Z> rhs = d.dots(pcols, d.col(R[k + 1], 0));
        std::vector<Z> coef((size_t)s * s + s);
        for (int q = 0; q < s; ++q) {
          ZMat msys(s);
          for (int c = 0; c < s; ++c)
            for (int i = 0; i < s; ++i) msys(i, c) = c < q ? Mn(i, c) : Ma(i, c);
          std::vector<Z> eta = solve_small(msys, rhs);
          for (int c = 0; c < s; ++c) {
            eta[c] = -eta[c];
            coef[(size_t)q * s + c] = eta[c];
          }
          std::vector<const double*> cols(s);
          for (int c = 0; c < s; ++c) cols[c] = c < q ? d.col(vl(k + 1), c) : d.col(vl(k), c);
          // column q of level k is also an input (c == q): each thread reads index t of every
          // input before it writes index t, so the column is rebuilt in place
          d.axpys(0, d.col(vl(k), q), d.col(R[k + 1], 0), cols, eta);
          d.spmv(a, d.col(vl(k), q), d.col(vl(k + 1), q));
          rep.h_mv++;
          const std::vector<Z> mq = d.dots(pcols, d.col(vl(k + 1), q));
          for (int i = 0; i < s; ++i) Mn(i, q) = mq[i];
        }
        {
          for (int c = 0; c < s; ++c) coef[(size_t)s * s + c] = gamma[c];
          d.upload_coef(coef);
          ZDeferredArgs da;
          for (int i = -1; i <= k; ++i) da.lv[i + 1] = d.col(vl(i), 0);
          for (int i = 0; i <= k; ++i) da.r[i] = d.col(R[i], 0);
          da.x = d.col(xw, 0);
          launch_zrebuild_deferred(d.st, n, d.ld, s, k, da, static_cast<const double*>(d.coef->ptr));
          d.check();
        }
        Ma = Mn;   // P^H V^(k+1) for the next level's projection
        g = rhs;   // P^H r^(k+1)
      }
      // poly_combination (idrstab.cpp:154-191)
      std::vector<const double*> zc(ell);
      for (int i = 0; i < ell; ++i) zc[i] = d.col(R[i + 1], 0);
      std::vector<Z> tau = least_squares_z(d, zc, d.col(R[0], 0), lsq);
      double tmax = 0.0;
      for (const Z& t : tau) tmax = std::max(tmax, std::abs(t));
      Z& tail = tau[ell - 1];
      if (std::abs(tail) < 1e-12 * tmax || tmax == 0.0) {
        const double target = tmax > 0.0 ? 1e-12 * tmax : 1e-12;
        tail = std::abs(tail) > 0.0 ? tail * (target / std::abs(tail)) : Z(target);
      }
      {
        std::vector<const double*> rc(ell), xc(ell);
        std::vector<Z> neg(ell);
        for (int i = 1; i <= ell; ++i) {
          rc[i - 1] = d.col(R[i], 0);
          xc[i - 1] = d.col(R[i - 1], 0);
          neg[i - 1] = -tau[i - 1];
        }
        d.axpys(0, d.col(ro, 0), d.col(R[0], 0), rc, neg);
        d.axpys(0, d.col(xo, 0), d.col(xw, 0), xc, tau);
        for (int q = 0; q < s; ++q) {
          std::vector<const double*> uc(ell), vc(ell);
          for (int i = 1; i <= ell; ++i) {
            uc[i - 1] = d.col(vl(i - 1), q);
            vc[i - 1] = d.col(vl(i), q);
          }
          d.axpys(0, d.col(Uo, q), d.col(vl(-1), q), uc, neg);
          d.axpys(0, d.col(Vo, q), d.col(vl(0), q), vc, neg);
        }
      }
      std::swap(x, xo);
      std::swap(r, ro);
      std::swap(U, Uo);
      std::swap(V, Vo);

      rep.cycles++;
      level += ell;
      rep.h_rd = level * s + (recycle ? base_level * (s - 1) : 0);
      if (omegas_complete) omegas_complete = extract_omegas_z(tau, omega_levels);
      res->taus.insert(res->taus.end(), tau.begin(), tau.end());
      if (cfg.true_residual_each_cycle) {
        d.spmv(a, d.col(x, 0), d.col(ax, 0));
        launch_zsub(d.st, n, d.col(r, 0), d.col(b, 0), d.col(ax, 0));
        d.check();
        rep.h_mv_aux++;
      }
      resnorm = d.norm2(d.col(r, 0));
      res->history.push_back({(int64_t)rep.cycles, rep.h_mv + rep.h_mv_aux, base_level + level, resnorm, ns_since(t0)});
      if (fetch && !res->fetched) {
        const bool hit = (fetch->kind == MSTAB_FETCH_AT_CYCLE && rep.cycles == fetch->cycle) ||
                         (fetch->kind == MSTAB_FETCH_AT_HALF_TOLERANCE && resnorm <= std::sqrt(cfg.tol) * rep.bnorm);
        if (hit)
          res->fetched = fetch_z(d, P, U, V, s, omegas_complete ? omega_levels : std::vector<Z>{}, base_level + level,
                                 a.fingerprint);
      }
    }
    rep.status = resnorm <= threshold ? MSTAB_STATUS_CONVERGED : MSTAB_STATUS_MAXMV;
  } catch (const Breakdown& e) {
    rep.status = MSTAB_STATUS_BREAKDOWN;
    std::snprintf(rep.breakdown_reason, sizeof(rep.breakdown_reason), "%s", e.what());
  }
  rep.final_resnorm = resnorm;
  res->x = d.block(1);
  d.copy(d.col(res->x, 0), d.col(x, 0));
  res->final_data = fetch_z(d, P, U, V, s, omegas_complete ? omega_levels : std::vector<Z>{}, base_level + level,
                            a.fingerprint);
  rep.has_fetched = res->fetched ? 1 : 0;
  rep.history_len = (int64_t)res->history.size();
  rep.tau_len = (int64_t)res->taus.size();
  ctx.sync();
  rep.wall_ns_total = ns_since(t0);
  return res;
}

void result_x_z(Context& ctx, const ZResult& res, double* x, int mem) {
  download_z(ctx, x, static_cast<const double*>(res.x->ptr), res.n, padded_ld(res.n), 1, mem);
  ctx.sync();
}

}  // namespace mstab_b200
