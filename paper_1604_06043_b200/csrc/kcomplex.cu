// kcomplex.cu — complex128 device primitives of the complex solve path.
//
// The reference computes everything in std::complex<double> (types.hpp:11-15). For real data the
// imaginary parts stay +0.0 and the fused real kernels of the cycle are exact; complex data (complex
// A, b, x0 or recycle blocks) runs on these kernels instead, orchestrated by zsolver.cpp. Vectors are
// interleaved (re, im) pairs (double2), column stride ld like the real path.
//
// Compiled with --fmad=false: a complex product is (ar*br - ai*bi, ar*bi + ai*br) with every
// product and sum rounded separately, the arithmetic of g++'s complex multiply on finite data
// (x86-64 without FMA contraction), so the element-wise kernels (SpMV, axpy chains, gemv updates)
// are bit-identical to the reference's loops; the length-N reductions are deterministic trees
// (per-CTA partials summed by the last CTA in a fixed order), like the real path.
#include "kcommon.cuh"

namespace mstab_b200 {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// y = A x, one row per thread in CSR order (spmv, csr.cpp:103-113)
__global__ void __launch_bounds__(kBlock) k_zspmv(int64_t n, const int32_t* __restrict__ rp,
                                                  const int32_t* __restrict__ ci, const double2* __restrict__ val,
                                                  const double2* __restrict__ x, double2* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    const int32_t e = rp[i + 1];
    for (int32_t k = rp[i]; k < e; ++k) acc = cadd(acc, cmul(__ldg(val + k), __ldg(x + ci[k])));
    y[i] = acc;
  }
}

// mode 0: y = y_in, then y += coef_c * col_c for c = 0..m-1 (a chain of axpy, types.cpp:21-23)
// mode 1: y = y_in + sum, mode 2: y = y_in - sum, sum = gemv (dense.cpp:19-24: starts at 0, adds
// coef_c * col_c in column order)
__global__ void __launch_bounds__(kBlock) k_zaxpys(int64_t n, int mode, double2* y_out, const double2* y_in,
                                                   ZTerms t) {  // y_out may alias y_in or a column
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 y0 = y_in[i];
    double2 acc = mode == 0 ? y0 : make_double2(0.0, 0.0);
    for (int c = 0; c < t.m; ++c) acc = cadd(acc, cmul(make_double2(t.re[c], t.im[c]), reinterpret_cast<const double2*>(t.col[c])[i]));
    y_out[i] = mode == 0 ? acc : (mode == 1 ? cadd(y0, acc) : csub(y0, acc));
  }
}

// y = x * a (mode 0, complex times the real-valued complex a + 0i: w[i] * inv in orthonormalize) or
// y = x / a (mode 1, complex / double: arnoldi_init's u = w / wnorm)
__global__ void __launch_bounds__(kBlock) k_zscale(int64_t n, int mode, double2* __restrict__ y,
                                                   const double2* __restrict__ x, double a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = x[i];
    // (vr + i vi)(a + i 0) = (vr a - vi 0, vr 0 + vi a): the +-0 terms never change a finite value
    y[i] = mode == 0 ? make_double2(v.x * a - v.y * 0.0, v.x * 0.0 + v.y * a) : make_double2(v.x / a, v.y / a);
  }
}

// r = b - ax (idrstab.cpp:212-215)
__global__ void __launch_bounds__(kBlock) k_zsub(int64_t n, double2* __restrict__ r, const double2* __restrict__ b,
                                                 const double2* __restrict__ ax) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = csub(b[i], ax[i]);
}

template <int NS>
__device__ void commit_to(double (&part)[NS], int nslots, double* out, Reducer red) {
  __shared__ double scratch[NS * 32];
  __shared__ double blk[NS];
  __shared__ double redv[NS];
  block_totals<NS>(part, blk, scratch);
  if (!cta_commit(blk, nslots, red.partials, &red.ds->ticket, redv)) return;
  for (int i = threadIdx.x; i < nslots; i += blockDim.x) out[i] = redv[i];
}

// out[2c], out[2c+1] = sum_i conj(col_c[i]) * y[i] for c < m (dot, types.cpp:15-19); when y is null
// the kernel pairs col_c with itself: out[2c] = sum |col_c|^2 (norm2's sum of std::norm)
constexpr int kZDotCols = 8;
__global__ void __launch_bounds__(kBlock) k_zdots(int64_t n, ZTerms t, const double2* __restrict__ y, double* out,
                                                  Reducer red) {
  double part[2 * kZDotCols];
#pragma unroll
  for (int c = 0; c < 2 * kZDotCols; ++c) part[c] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 yv = make_double2(0.0, 0.0);
    if (y) yv = y[i];
#pragma unroll
    for (int c = 0; c < kZDotCols; ++c) {
      if (c < t.m) {
        const double2 a = reinterpret_cast<const double2*>(t.col[c])[i];
        if (y) {
          const double2 p = cmul(make_double2(a.x, -a.y), yv);
          part[2 * c] += p.x;
          part[2 * c + 1] += p.y;
        } else {
          part[2 * c] += a.x * a.x + a.y * a.y;
        }
      }
    }
  }
  commit_to<2 * kZDotCols>(part, 2 * t.m, out, red);
}

// out[0] = sum |x|^2, out[1] = non-finite entries, out[2] = nonzero entries, out[3] = entries with
// a nonzero imaginary part (ensure_finite, is_zero, is_real: types.cpp:25-40, idrstab.cpp:21-23)
__global__ void __launch_bounds__(kBlock) k_zstats(int64_t n, const double2* __restrict__ x, double* out,
                                                   Reducer red) {
  double part[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = x[i];
    part[0] += v.x * v.x + v.y * v.y;
    if (!isfinite(v.x) || !isfinite(v.y)) part[1] += 1.0;
    if (v.x != 0.0 || v.y != 0.0) part[2] += 1.0;
    if (v.y != 0.0) part[3] += 1.0;
  }
  commit_to<4>(part, 4, out, red);
}

// out[0] = sum |v - au|^2, out[1] = sum |v|^2 (validate, recycle.cpp:53-59)
__global__ void __launch_bounds__(kBlock) k_zdiff(int64_t n, const double2* __restrict__ v,
                                                  const double2* __restrict__ au, double* out, Reducer red) {
  double part[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = v[i];
    const double2 d = csub(a, au[i]);
    part[0] += d.x * d.x + d.y * d.y;
    part[1] += a.x * a.x + a.y * a.y;
  }
  commit_to<2>(part, 2, out, red);
}

// One pass over the rows for ALL lower levels of a level iteration: level k is final; levels
// i = k-1 .. -1 are rebuilt top-down, each needing only level i+1 (final, held in registers from the
// previous step) and level i (updated in q order). Element for element the arithmetic of the
// per-column passes it replaces (axpy chains in column order), so the result is bit-identical.
template <int S>
__global__ void __launch_bounds__(kBlock, S <= 8 ? 2 : 1)
    k_zrebuild_deferred(int64_t n, int64_t ld, int k, ZDeferredArgs a, const double2* __restrict__ coef) {
  __shared__ double2 et[S * S];
  __shared__ double2 gm[S];
  for (int i = threadIdx.x; i < S * S; i += blockDim.x) et[i] = coef[i];
  if (threadIdx.x < S) gm[threadIdx.x] = coef[S * S + threadIdx.x];
  __syncthreads();
  // eta is re-read from shared memory (broadcast) at every use: hoisting its S*S values into
  // registers would spill the level columns
  const volatile double* etv = reinterpret_cast<const volatile double*>(et);
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double2 ln[S], lc[S];
    const double2* top = reinterpret_cast<const double2*>(a.lv[k + 1]);
#pragma unroll
    for (int c = 0; c < S; ++c) ln[c] = top[c * ld + row];
    double2 r_above = reinterpret_cast<const double2*>(a.r[k])[row];
    for (int i = k - 1; i >= -1; --i) {
      double2* cur = reinterpret_cast<double2*>(a.lv[i + 1]);
#pragma unroll
      for (int c = 0; c < S; ++c) lc[c] = cur[c * ld + row];
      // step (a) at this level with its pre-rebuild columns: gemv from zero in column order
      double2 corr = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < S; ++c) corr = cadd(corr, cmul(gm[c], lc[c]));
      double2 ri = make_double2(0.0, 0.0);
      if (i >= 0) {
        double2* rp = reinterpret_cast<double2*>(a.r[i]);
        ri = csub(rp[row], corr);
        rp[row] = ri;
      } else {
        double2* xp = reinterpret_cast<double2*>(a.x);
        xp[row] = cadd(xp[row], corr);
      }
      // step (c) at level i for every column q in order: newcol = r^(i+1) + sum_c (-eta_q[c]) mixed_c
#pragma unroll
      for (int q = 0; q < S; ++q) {
        double2 nc = r_above;
#pragma unroll
        for (int c = 0; c < S; ++c)
          nc = cadd(nc, cmul(make_double2(etv[2 * (q * S + c)], etv[2 * (q * S + c) + 1]), (c < q) ? ln[c] : lc[c]));
        lc[q] = nc;
      }
#pragma unroll
      for (int c = 0; c < S; ++c) {
        cur[c * ld + row] = lc[c];
        ln[c] = lc[c];
      }
      r_above = ri;
    }
  }
}

int zgrid(int64_t n) {
  int64_t want = (n + kBlock - 1) / kBlock;
  const int64_t cap = (int64_t)g_num_sms * 4;
  if (want > cap) want = cap;
  return (int)(want < 1 ? 1 : want);
}

}  // namespace

void launch_zspmv(cudaStream_t st, int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci, const double* val,
                  const double* x, double* y) {
  LaunchScope ls(st, kKSpmv, 20.0 * (double)nnz + 4.0 * (double)(n + 1) + 32.0 * (double)n);
  k_zspmv<<<zgrid(n), kBlock, 0, st>>>(n, rp, ci, reinterpret_cast<const double2*>(val),
                                       reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y));
}

void launch_zaxpys(cudaStream_t st, int64_t n, int mode, double* y_out, const double* y_in, const ZTerms& t) {
  LaunchScope ls(st, kKOther, 16.0 * (double)n * (t.m + 2.0));
  k_zaxpys<<<zgrid(n), kBlock, 0, st>>>(n, mode, reinterpret_cast<double2*>(y_out),
                                        reinterpret_cast<const double2*>(y_in), t);
}

void launch_zscale(cudaStream_t st, int64_t n, int mode, double* y, const double* x, double a) {
  LaunchScope ls(st, kKOther, 32.0 * (double)n);
  k_zscale<<<zgrid(n), kBlock, 0, st>>>(n, mode, reinterpret_cast<double2*>(y), reinterpret_cast<const double2*>(x), a);
}

void launch_zsub(cudaStream_t st, int64_t n, double* r, const double* b, const double* ax) {
  LaunchScope ls(st, kKOther, 48.0 * (double)n);
  k_zsub<<<zgrid(n), kBlock, 0, st>>>(n, reinterpret_cast<double2*>(r), reinterpret_cast<const double2*>(b),
                                      reinterpret_cast<const double2*>(ax));
}

void launch_zdots(cudaStream_t st, int64_t n, const ZTerms& cols, const double* y, double* out, const Reducer& red) {
  // at most kZDotCols columns per launch; the caller's out holds 2 * m doubles
  for (int c0 = 0; c0 < cols.m; c0 += kZDotCols) {
    ZTerms t{};
    t.m = cols.m - c0 < kZDotCols ? cols.m - c0 : kZDotCols;
    for (int c = 0; c < t.m; ++c) t.col[c] = cols.col[c0 + c];
    LaunchScope ls(st, kKOther, 16.0 * (double)n * (t.m + (y ? 1.0 : 0.0)));
    k_zdots<<<zgrid(n), kBlock, 0, st>>>(n, t, reinterpret_cast<const double2*>(y), out + 2 * c0, red);
  }
}

void launch_zrebuild_deferred(cudaStream_t st, int64_t n, int64_t ld, int s, int k, const ZDeferredArgs& a,
                              const double* coef) {
  // reads x, r^(0..k), V^(-1..k); writes x, r^(0..k-1), V^(-1..k-1) (complex: 16 bytes per entry)
  LaunchScope ls(st, kKRebuildDeferred, 2.0 * vbytes(n, (k + 1.0) + 1.0 + (k + 2.0) * s + k + 1.0 + (k + 1.0) * s));
  MSTAB_DISPATCH_S(s, {
    k_zrebuild_deferred<S><<<zgrid(n), kBlock, 0, st>>>(n, ld, k, a, reinterpret_cast<const double2*>(coef));
  });
}

void launch_zstats(cudaStream_t st, int64_t n, const double* x, double* out, const Reducer& red) {
  LaunchScope ls(st, kKOther, 16.0 * (double)n);
  k_zstats<<<zgrid(n), kBlock, 0, st>>>(n, reinterpret_cast<const double2*>(x), out, red);
}

void launch_zdiff(cudaStream_t st, int64_t n, const double* v, const double* au, double* out, const Reducer& red) {
  LaunchScope ls(st, kKOther, 32.0 * (double)n);
  k_zdiff<<<zgrid(n), kBlock, 0, st>>>(n, reinterpret_cast<const double2*>(v), reinterpret_cast<const double2*>(au), out,
                                       red);
}

}  // namespace mstab_b200
