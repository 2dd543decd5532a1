// kbase.cu — element-wise updates of the comparison baselines (baselines.cpp:49-262, SURVEY.md
// §8(f3)): BiCGStab and GMRES run their reductions through launch_dots / launch_vec_stats and
// their vector updates here. --fmad=false: each product and sum rounds like the reference's.
#include "kcommon.cuh"

namespace mstab_b200 {

namespace {

// out = x + a * y (axpy(a, y, x) when out == x, types.cpp:21-23; s = r - alpha ap with a = -alpha)
__global__ void k_xpay(int64_t n, const double* x, const double* y, double a, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] + a * y[i];
}

// p = r + beta * (p - omega * ap)   (baselines.cpp:251)
__global__ void k_bicgstab_p(int64_t n, const double* __restrict__ r, const double* __restrict__ ap, double beta,
                             double omega, double* __restrict__ p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = r[i] + beta * (p[i] - omega * ap[i]);
}

}  // namespace

void launch_xpay(cudaStream_t st, int64_t n, const double* x, const double* y, double a, double* out) {
  LaunchScope ls(st, kKOther, vbytes(n, 3.0));
  k_xpay<<<grid_for(n), kBlock, 0, st>>>(n, x, y, a, out);
}

void launch_bicgstab_p(cudaStream_t st, int64_t n, const double* r, const double* ap, double beta, double omega,
                       double* p) {
  LaunchScope ls(st, kKOther, vbytes(n, 4.0));
  k_bicgstab_p<<<grid_for(n), kBlock, 0, st>>>(n, r, ap, beta, omega, p);
}

}  // namespace mstab_b200
