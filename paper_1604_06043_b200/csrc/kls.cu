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

// ---- CholeskyQR2 (two streaming passes, no Q stored) --------------------------------------------
// Pass 1: G1 = Z^T Z of Z = [r^(1..L) | r^(0)] (packed upper, one deterministic reduction), then
// R1 = chol(G1) and R1^-1. Pass 2: G2 = Q^T Q with Q = Z R1^-1 formed row by row, R2 = chol(G2),
// R = R2 R1 (the R factor of Z to working accuracy while cond(Z) <~ 1e8). Used only when every
// Cholesky pivot of G1 keeps more than kCholKeep of its column's squared norm;
// otherwise pass 2 runs the one-pass Givens TSQR instead (same launch, ls_mode = 0), which also
// owns the rank-deficiency regime of the reference's test (kernels.cpp:83-84). Either way the
// least-squares solve, rank test and tail guard are ls_finalize's.
// A Cholesky pivot must keep more than kCholKeep of its column's squared norm (each column adds
// a direction at least 1e-3 of its length away from the previous ones), else the Givens path.
constexpr double kCholKeep = 1e-6;

template <int L>
__device__ bool chol_packed(const double* G, double* R) {
  constexpr int D = L + 1;
  for (int j = 0; j < D; ++j) {
    double d = G[Tri<L>::at(j, j)];
    for (int i = 0; i < j; ++i) d = d - R[Tri<L>::at(i, j)] * R[Tri<L>::at(i, j)];
    if (!(d > kCholKeep * G[Tri<L>::at(j, j)]) || !isfinite(d)) return false;
    const double rjj = sqrt(d);
    R[Tri<L>::at(j, j)] = rjj;
    for (int m = j + 1; m < D; ++m) {
      double t = G[Tri<L>::at(j, m)];
      for (int i = 0; i < j; ++i) t = t - R[Tri<L>::at(i, j)] * R[Tri<L>::at(i, m)];
      R[Tri<L>::at(j, m)] = t / rjj;
    }
  }
  return true;
}

template <int L>
__device__ void tri_inverse(const double* R, double* Ri) {
  constexpr int D = L + 1;
  for (int j = D - 1; j >= 0; --j) {
    Ri[Tri<L>::at(j, j)] = 1.0 / R[Tri<L>::at(j, j)];
    for (int m = j + 1; m < D; ++m) {
      double t = 0.0;
      for (int k = j + 1; k <= m; ++k) t = t + R[Tri<L>::at(j, k)] * Ri[Tri<L>::at(k, m)];
      Ri[Tri<L>::at(j, m)] = -t / R[Tri<L>::at(j, j)];
    }
  }
}

// Dense tail of pass 1 (thread 0): R1, R1^-1, column norms, path choice.
template <int L>
__device__ void ls_pass1_tail(const double* G, DevState* ds) {
  for (int j = 0; j < L; ++j) ds->ls_cn[j] = G[Tri<L>::at(j, j)];
  double R[Tri<L>::NR];
  if (chol_packed<L>(G, R)) {
    for (int i = 0; i < Tri<L>::NR; ++i) ds->ls_r1[i] = R[i];
    tri_inverse<L>(R, ds->ls_r1inv);
    ds->ls_mode = 1;
  } else {
    ds->ls_mode = 0;
  }
}

// Dense tail of the CholeskyQR2 pass 2 (thread 0): R = chol(G2) R1, then the reference's solve.
template <int L>
__device__ void ls_finalize(const double* Rf, const double* cn, int s, DevState* ds);
template <int L>
__device__ void ls_pass2_tail(const double* G2, int s, DevState* ds) {
  constexpr int D = L + 1, NR = Tri<L>::NR;
  double R2[NR], R[NR];
  if (chol_packed<L>(G2, R2)) {
    for (int j = 0; j < D; ++j)
      for (int m = j; m < D; ++m) {
        double t = 0.0;
        for (int k = j; k <= m; ++k) t = t + R2[Tri<L>::at(j, k)] * ds->ls_r1[Tri<L>::at(k, m)];
        R[Tri<L>::at(j, m)] = t;
      }
  } else {  // cannot happen for a well-conditioned Q; keep the first factor
    for (int i = 0; i < NR; ++i) R[i] = ds->ls_r1[i];
  }
  double cn[L];
  for (int j = 0; j < L; ++j) cn[j] = ds->ls_cn[j];
  ls_finalize<L>(R, cn, s, ds);
}

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
