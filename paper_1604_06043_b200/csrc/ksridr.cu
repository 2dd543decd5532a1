// ksridr.cu — the recycled phase of SRIDR (sridr.cpp:57-81): each cycle replays
// one of the donor's relaxations with the auxiliary block fixed, at one matrix-vector product.
//
//   gamma = (P^H V)^-1 P^H r          (LU of the fixed P^H V: finalize_spmv, kFinTrueRes)
//   rt = r - V gamma,  xt = x + U gamma                      k_sridr_corr
//   art = A rt                                                the SpMV kernels
//   r = rt - omega art,  x = xt + omega rt,  P^H r, ||r||^2   k_sridr_update (+ the next gamma)
//
// --fmad=false like every kernel of the cycle: gemv accumulates from 0 in column order
// (dense.cpp:19-24) and every product / sum rounds separately, as the reference's complex
// arithmetic does for real data (omega real: ell = 1 relaxations are real).
#include "kcommon.cuh"

namespace mstab_b200 {

namespace {

template <int S>
__global__ void __launch_bounds__(kBlock) k_sridr_corr(int64_t n, int64_t ld, const double* __restrict__ r,
                                                       const double* __restrict__ x,
                                                       const double* __restrict__ u,
                                                       const double* __restrict__ v, double* __restrict__ rt,
                                                       double* __restrict__ xt, const DevState* ds) {
  pdl_wait();
  double gm[S];
#pragma unroll
  for (int c = 0; c < S; ++c) gm[c] = ds->gamma[c];
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double vc = 0.0, uc = 0.0;
#pragma unroll
    for (int c = 0; c < S; ++c) {
      vc = vc + __ldg(v + c * ld + row) * gm[c];
      uc = uc + __ldg(u + c * ld + row) * gm[c];
    }
    rt[row] = r[row] - vc;
    xt[row] = x[row] + uc;
  }
}

template <int S>
__global__ void __launch_bounds__(kBlock) k_sridr_update(int64_t n, int64_t ld, double omega,
                                                         const double* __restrict__ rt,
                                                         const double* __restrict__ art,
                                                         const double* __restrict__ xt, double* __restrict__ r,
                                                         double* __restrict__ x, const double* __restrict__ p,
                                                         FinParams fin, Reducer red) {
  DevState* ds = red.ds;
  constexpr int NS = S + 1;
  double part[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) part[i] = 0.0;
  pdl_wait();
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    const double t = rt[row];
    const double rn = t - omega * art[row];
    r[row] = rn;
    x[row] = xt[row] + omega * t;
#pragma unroll
    for (int c = 0; c < S; ++c) part[c] = part[c] + __ldg(p + c * ld + row) * rn;
    part[S] = part[S] + rn * rn;
  }
  __shared__ double scratch[NS * 32];
  __shared__ double blk[NS];
  __shared__ double redv[NS];
  __shared__ FinStage fs;
  if (!red.xred) fin_prestage(fin, ds, fs);
  block_totals<NS>(part, blk, scratch);
  if (!cta_commit(blk, NS, red.partials, &ds->ticket, redv, red.xred)) return;
  finalize_spmv<S>(fin, redv, ds, fs);
}

}  // namespace

void launch_sridr_corr(cudaStream_t st, int64_t n, int64_t ld, int s, const double* r, const double* x,
                       const double* u, const double* v, double* rt, double* xt, const DevState* ds) {
  LaunchScope ls(st, kKLevelUpdate, vbytes(n, 2.0 * s + 4.0));
  MSTAB_DISPATCH_S(s, {
    launch_pdl(k_sridr_corr<S>, grid_for(n), kBlock, 0, st, n, ld, r, x, u, v, rt, xt, ds);
  });
}

void launch_sridr_update(cudaStream_t st, int64_t n, int64_t ld, int s, double omega, const double* rt,
                         const double* art, const double* xt, double* r, double* x, const double* p,
                         const FinParams& fin, const Reducer& red) {
  LaunchScope ls(st, kKLevelUpdate, vbytes(n, 5.0 + s));
  MSTAB_DISPATCH_S(s, {
    launch_pdl(k_sridr_update<S>, grid_for(n), kBlock, 0, st, n, ld, omega, rt, art, xt, r, x, p, fin, red);
  });
}

}  // namespace mstab_b200
