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
#include "kdense.cuh"

namespace mstab_b200 {

namespace {

template <int L>
__global__ void __launch_bounds__(kBlock) k_ls_gram1(int64_t n, LsArgs a, Reducer red) {
  DevState* ds = red.ds;
  pdl_wait();
  constexpr int D = L + 1, NR = Tri<L>::NR;
  double g[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) g[i] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double z[D];
#pragma unroll
    for (int j = 0; j < L; ++j) z[j] = a.r[j + 1][row];
    z[L] = a.r[0][row];
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int m = j; m < D; ++m) g[Tri<L>::at(j, m)] = g[Tri<L>::at(j, m)] + z[j] * z[m];
  }
  pdl_trigger();
  __shared__ double scratch[NR * 32];
  __shared__ double blk[NR];
  __shared__ double redv[NR];
  block_totals<NR>(g, blk, scratch);
  if (!cta_commit(blk, NR, red.partials, &ds->ticket, redv, red.xred)) return;
  if (threadIdx.x == 0) ls_pass1_tail<L>(redv, ds);
}

template <int L>
__global__ void k_fin_ls1(DevState* ds) {
  if (threadIdx.x == 0) ls_pass1_tail<L>(ds->xred, ds);
}

template <int L>
__global__ void __launch_bounds__(kBlock) k_ls_tsqr(int64_t n, int s, int chol, LsArgs a, Reducer red) {
  DevState* ds = red.ds;
  pdl_wait();
  constexpr int NR = Tri<L>::NR;
  if (chol && ds->ls_mode == 1) {  // CholeskyQR2 pass 2: Gram of Q = Z R1^-1, row by row
    constexpr int D = L + 1;
    __shared__ double ri[NR];
    for (int i = threadIdx.x; i < NR; i += blockDim.x) ri[i] = ds->ls_r1inv[i];
    __syncthreads();
    double g[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) g[i] = 0.0;
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
         row += (int64_t)gridDim.x * blockDim.x) {
      double z[D], q[D];
#pragma unroll
      for (int j = 0; j < L; ++j) z[j] = a.r[j + 1][row];
      z[L] = a.r[0][row];
#pragma unroll
      for (int m = 0; m < D; ++m) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j <= m; ++j) t = t + z[j] * ri[Tri<L>::at(j, m)];
        q[m] = t;
      }
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int m = j; m < D; ++m) g[Tri<L>::at(j, m)] = g[Tri<L>::at(j, m)] + q[j] * q[m];
    }
    pdl_trigger();
    __shared__ double scratch2[NR * 32];
    __shared__ double blk2[NR];
    __shared__ double redv2[NR];
    block_totals<NR>(g, blk2, scratch2);
    if (!cta_commit(blk2, NR, red.partials, &ds->ticket, redv2, red.xred)) return;
    if (threadIdx.x == 0) ls_pass2_tail<L>(redv2, s, ds);
    return;
  }
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
__global__ void k_fin_ls(int s, int world, int chol, const double* __restrict__ gath, DevState* ds) {
  constexpr int NR = Tri<L>::NR;
  if (threadIdx.x != 0) return;
  if (chol && ds->ls_mode == 1) {  // CholeskyQR2: the gathered rank-local Grams summed in rank order
    double G2[NR];
    for (int i = 0; i < NR; ++i) G2[i] = gath[i];
    for (int w = 1; w < world; ++w)
      for (int i = 0; i < NR; ++i) G2[i] = G2[i] + gath[(size_t)w * (NR + L) + i];
    ls_pass2_tail<L>(G2, s, ds);
    return;
  }
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

void launch_fin_ls1(cudaStream_t st, int ell, DevState* ds) {
  MSTAB_DISPATCH_L(ell, { k_fin_ls1<L><<<1, 32, 0, st>>>(ds); });
}

void launch_fin_ls(cudaStream_t st, int ell, int s, int world, bool chol, const double* gath, DevState* ds) {
  static_assert(ls_split_count(8) <= kMaxXred, "LS split payload exceeds xred");
  MSTAB_DISPATCH_L(ell, { k_fin_ls<L><<<1, 32, 0, st>>>(s, world, chol ? 1 : 0, gath, ds); });
}

void launch_ls_pass1(cudaStream_t st, int64_t n, int ell, const double* const* r, const Reducer& red) {
  LaunchScope ls(st, kKLs, vbytes(n, ell + 1.0));
  LsArgs a{};
  for (int i = 0; i <= ell; ++i) a.r[i] = r[i];
  MSTAB_DISPATCH_L(ell, {
    auto kfn = k_ls_gram1<L>;
    launch_pdl(kfn, occupancy_grid(kfn, n, 0), kBlock, 0, st, n, a, red);
  });
}

void launch_ls_pass2(cudaStream_t st, int64_t n, int ell, int s, bool chol, const double* const* r,
                     const Reducer& red) {
  LaunchScope ls(st, kKLs, vbytes(n, ell + 1.0));
  LsArgs a{};
  for (int i = 0; i <= ell; ++i) a.r[i] = r[i];
  MSTAB_DISPATCH_L(ell, {
    auto kfn = k_ls_tsqr<L>;
    launch_pdl(kfn, occupancy_grid(kfn, n, 0), kBlock, 0, st, n, s, chol ? 1 : 0, a, red);
  });
}

void launch_ls(cudaStream_t st, int64_t n, int64_t ld, int ell, int s, const double* const* r,
               const Reducer& red) {
  (void)ld;
  const bool chol = ls_use_cholqr(n);
  if (chol) launch_ls_pass1(st, n, ell, r, red);
  launch_ls_pass2(st, n, ell, s, chol, r, red);
}

}  // namespace mstab_b200
