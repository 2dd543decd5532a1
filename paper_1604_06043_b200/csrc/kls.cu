// kls.cu — least squares of the stabilisation step by one-pass Givens TSQR.
//
// Compiled with --fmad=false: every a*b+c below rounds the product and the sum separately,
// exactly like the reference's scalar std::complex<double> loops with zero imaginary parts
// (g++ -O3 without -mfma). Given identical small-solve inputs, the element-wise
// kernels (SpMV, level updates, column rebuilds, poly combination) are therefore bit-identical
// to the reference; only the length-N reductions differ (deterministic trees instead of
// sequential sums), which is why parity is judged teacher-forced (finding 3).
//
// All streaming kernels are HBM-bound; they use persistent grid-stride loops
// sized to the SM count so each CTA leaves exactly one partial per reduced value, and the last
// CTA (ticket counter) reduces the partials in a fixed order and runs the dense step that
// consumes them (s x s LU, Givens-TSQR least squares) without another launch.
#include "kcommon.cuh"

namespace mstab_b200 {

namespace {

// ---------------------------------------------------------------------------------------------
// Least squares by Givens TSQR of [Z | r0] (one HBM pass). R is (L+1)x(L+1) upper triangular,
// packed row-major: row j holds columns j..L at offset j*(L+1) - j*(j-1)/2.
template <int L>
struct Tri {
  static constexpr int D = L + 1;
  static constexpr int NR = D * (D + 1) / 2;
  __host__ __device__ static constexpr int at(int j, int m) { return j * D - j * (j - 1) / 2 + (m - j); }
};

// Absorbs row w (zero before column `start`) into R with Givens rotations.
template <int L>
__device__ __forceinline__ void givens_absorb(double (&R)[Tri<L>::NR], double (&w)[L + 1], int start) {
#pragma unroll
  for (int j = 0; j <= L; ++j) {
    if (j < start) continue;
    const double bj = w[j];
    if (bj == 0.0) continue;
    const double aj = R[Tri<L>::at(j, j)];
    const double h2 = aj * aj + bj * bj;
    const double inv = rsqrt(h2);  // one reciprocal square root instead of sqrt + divide
    const double r = h2 * inv;
    const double c = aj * inv, sn = bj * inv;
    R[Tri<L>::at(j, j)] = r;
#pragma unroll
    for (int m = j + 1; m <= L; ++m) {
      const double t = R[Tri<L>::at(j, m)];
      R[Tri<L>::at(j, m)] = c * t + sn * w[m];
      w[m] = c * w[m] - sn * t;
    }
  }
}

template <int L>
__device__ __forceinline__ void absorb_tri(double (&R)[Tri<L>::NR], const double (&B)[Tri<L>::NR]) {
#pragma unroll
  for (int j = 0; j <= L; ++j) {
    double w[L + 1];
#pragma unroll
    for (int m = 0; m <= L; ++m) w[m] = (m < j) ? 0.0 : B[Tri<L>::at(j, m)];
    givens_absorb<L>(R, w, j);
  }
}

template <int L>
__device__ void ls_finalize(const double* Rf, const double* cn, int s, DevState* ds) {
  // Rf: merged R (packed), cn: column sums of squares of Z (L values)
  double max_colnorm = 0.0;
  for (int j = 0; j < L; ++j) max_colnorm = dmax_ref(max_colnorm, sqrt(cn[j]));
  double min_diag = INFINITY;
  for (int k = 0; k < L; ++k) {
    const double d = fabs(Rf[Tri<L>::at(k, k)]);
    min_diag = (d < min_diag) ? d : min_diag;
  }
  if (min_diag < 1e-13 * max_colnorm) {  // kernels.cpp:83-84
    set_breakdown(ds, kBreakRank, L * (s + 1));
    return;
  }
  double tau[L];
  for (int k = 0; k < L; ++k) tau[k] = Rf[Tri<L>::at(k, L)];
  for (int k = L - 1; k >= 0; --k) {  // kernels.cpp:87-91
    for (int j = k + 1; j < L; ++j) tau[k] = tau[k] - Rf[Tri<L>::at(k, j)] * tau[j];
    tau[k] = tau[k] / Rf[Tri<L>::at(k, k)];
  }
  for (int k = 0; k < L; ++k) ds->scal[32 + k] = tau[k];  // raw least-squares solution
  // tail guard (idrstab.cpp:163-174)
  double tmax = 0.0;
  for (int k = 0; k < L; ++k) tmax = dmax_ref(tmax, fabs(tau[k]));
  int pert = 0;
  double& tail = tau[L - 1];
  if (fabs(tail) < 1e-12 * tmax || tmax == 0.0) {
    const double target = tmax > 0.0 ? 1e-12 * tmax : 1e-12;
    tail = fabs(tail) > 0.0 ? tail * (target / fabs(tail)) : target;
    pert = 1;
  }
  for (int k = 0; k < L; ++k) ds->st.tau[k] = tau[k];
  ds->st.tail_perturbed = pert;
}

struct LsArgs {
  const double* r[kMaxEll + 1];  // r^(0..L)
};

template <int L>
__global__ void __launch_bounds__(kBlock) k_ls_tsqr(int64_t n, int s, LsArgs a, Reducer red) {
  DevState* ds = red.ds;
  pdl_wait();
  constexpr int NR = Tri<L>::NR;
  double R[NR];
  double cn[L];
#pragma unroll
  for (int i = 0; i < NR; ++i) R[i] = 0.0;
#pragma unroll
  for (int j = 0; j < L; ++j) cn[j] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double w[L + 1];
#pragma unroll
    for (int j = 0; j < L; ++j) {
      w[j] = a.r[j + 1][row];
      cn[j] = cn[j] + w[j] * w[j];
    }
    w[L] = a.r[0][row];
    givens_absorb<L>(R, w, 0);
  }
  pdl_trigger();
  // warp tree merge (lane absorbs lane + off)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    double B[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) B[i] = __shfl_down_sync(0xffffffffu, R[i], off);
    if ((lane & (2 * off - 1)) == 0) absorb_tri<L>(R, B);
  }
  __shared__ double wR[32 * NR];
  __shared__ double cns[L * 32];
#pragma unroll
  for (int j = 0; j < L; ++j) {
    const double t = warp_sum(cn[j]);
    if (lane == 0) cns[j * 32 + wid] = t;
  }
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NR; ++i) wR[wid * NR + i] = R[i];
  __syncthreads();
  __shared__ int s_last;
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    double Rc[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) Rc[i] = wR[i];
    for (int w2 = 1; w2 < nw; ++w2) {
      double B[NR];
#pragma unroll
      for (int i = 0; i < NR; ++i) B[i] = wR[w2 * NR + i];
      absorb_tri<L>(Rc, B);
    }
    double* part = red.partials;
#pragma unroll
    for (int i = 0; i < NR; ++i) part[(size_t)i * G + blockIdx.x] = Rc[i];
    for (int j = 0; j < L; ++j) {
      double acc = 0.0;
      for (int k = 0; k < nw; ++k) acc += cns[j * 32 + k];
      part[(size_t)(NR + j) * G + blockIdx.x] = acc;
    }
    __threadfence();
    s_last = (atomicAdd(&ds->ticket, 1u) == (uint32_t)(G - 1));
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last CTA: thread t merges CTAs t, t+blockDim, ... then a fixed tree
  double* part = red.partials;
#pragma unroll
  for (int i = 0; i < NR; ++i) R[i] = 0.0;
  for (int c = threadIdx.x; c < G; c += blockDim.x) {
    double B[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) B[i] = __ldcg(part + (size_t)i * G + c);
    absorb_tri<L>(R, B);
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    double B[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) B[i] = __shfl_down_sync(0xffffffffu, R[i], off);
    if ((lane & (2 * off - 1)) == 0) absorb_tri<L>(R, B);
  }
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NR; ++i) wR[wid * NR + i] = R[i];
  __syncthreads();
  // column sums of squares of Z over all CTAs: warp j reduces column j (fixed lane/tree order)
  __shared__ double cnt[L];
  if (wid < L) {
    const double* p = part + (size_t)(NR + wid) * G;
    double acc = 0.0;
    for (int c = lane; c < G; c += 32) acc += __ldcg(p + c);
    acc = warp_sum(acc);
    if (lane == 0) cnt[wid] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double Rc[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) Rc[i] = wR[i];
    for (int w2 = 1; w2 < nw; ++w2) {
      double B[NR];
#pragma unroll
      for (int i = 0; i < NR; ++i) B[i] = wR[w2 * NR + i];
      absorb_tri<L>(Rc, B);
    }
    ds->ticket = 0u;
    if (red.xred) {  // row-sharded: this rank's R factor and column sums go to the allgather
#pragma unroll
      for (int i = 0; i < NR; ++i) red.xred[i] = Rc[i];
      for (int j = 0; j < L; ++j) red.xred[NR + j] = cnt[j];
      return;
    }
    ls_finalize<L>(Rc, cnt, s, ds);
  }
}

// Row-sharded finaliser: `gath` holds every rank's (R, column sums) back to back, rank-major.
// The factors are merged in rank order by the same Givens absorption as the in-kernel tree and
// the column sums added in rank order, so every rank solves the identical least-squares system.
template <int L>
__global__ void k_fin_ls(int s, int world, const double* __restrict__ gath, DevState* ds) {
  constexpr int NR = Tri<L>::NR;
  if (threadIdx.x != 0) return;
  double Rc[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) Rc[i] = gath[i];
  double cnt[L];
  for (int j = 0; j < L; ++j) cnt[j] = gath[NR + j];
  for (int w = 1; w < world; ++w) {
    const double* g = gath + (size_t)w * (NR + L);
    double B[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) B[i] = g[i];
    absorb_tri<L>(Rc, B);
    for (int j = 0; j < L; ++j) cnt[j] = cnt[j] + g[NR + j];
  }
  ls_finalize<L>(Rc, cnt, s, ds);
}

}  // namespace

void launch_fin_ls(cudaStream_t st, int ell, int s, int world, const double* gath, DevState* ds) {
  static_assert(ls_split_count(8) <= kMaxXred, "LS split payload exceeds xred");
  MSTAB_DISPATCH_L(ell, { k_fin_ls<L><<<1, 32, 0, st>>>(s, world, gath, ds); });
}

void launch_ls(cudaStream_t st, int64_t n, int64_t ld, int ell, int s, const double* const* r,
               const Reducer& red) {
  (void)ld;
  LaunchScope ls(st, kKLs, vbytes(n, ell + 1.0));
  LsArgs a{};
  for (int i = 0; i <= ell; ++i) a.r[i] = r[i];
  MSTAB_DISPATCH_L(ell, {
    auto kfn = k_ls_tsqr<L>;
    const int grid = occupancy_grid(kfn, n, 0);
    launch_pdl(kfn, grid, kBlock, 0, st, n, s, a, red);
  });
}

}  // namespace mstab_b200
