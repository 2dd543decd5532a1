// kernels.cu — sm_100a kernels of the Mstab solve loop (real fp64).
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
#include <cuda_runtime.h>

#include <cmath>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "kernels.h"

namespace mstab_b200 {

namespace {

int g_num_sms = 148;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double dmax_ref(double acc, double v) {
  // std::max(acc, v) == (acc < v) ? v : acc  (NaN keeps acc, like the reference)
  return (acc < v) ? v : acc;
}

// Per-CTA totals of NS per-thread registers into smem `blk` (deterministic tree).
template <int NS>
__device__ void block_totals(const double (&v)[NS], double* blk, double* scratch /*NS*32*/) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    double t = warp_sum(v[i]);
    if (lane == 0) scratch[i * 32 + w] = t;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NS; i += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < nw; ++k) acc += scratch[i * 32 + k];
    blk[i] = acc;
  }
  __syncthreads();
}

// Writes the CTA's `nslots` totals as partials[slot][cta]; the last CTA to arrive reduces every
// slot over all CTAs in a fixed order into `red` (smem) and returns true.
__device__ bool cta_commit(const double* blk, int nslots, double* partials, uint32_t* ticket,
                           double* red) {
  __shared__ int s_last;
  const int G = gridDim.x;
  for (int i = threadIdx.x; i < nslots; i += blockDim.x)
    partials[(size_t)i * G + blockIdx.x] = blk[i];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == (uint32_t)(G - 1));
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = w; i < nslots; i += nw) {
    const double* p = partials + (size_t)i * G;
    double acc = 0.0;
    int c = lane;
    for (; c + 96 < G; c += 128) {
      const double a0 = __ldcg(p + c), a1 = __ldcg(p + c + 32), a2 = __ldcg(p + c + 64),
                   a3 = __ldcg(p + c + 96);
      acc += a0;
      acc += a1;
      acc += a2;
      acc += a3;
    }
    for (; c < G; c += 32) acc += __ldcg(p + c);
    acc = warp_sum(acc);
    if (lane == 0) red[i] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// solve_small / LuFactor (kernels.cpp:95-154): partially pivoted LU with the reference's pivot
// rule (first strictly larger magnitude), singular test |pivot| < 1e-14 * max|M| or max|M| == 0,
// inverse-multiply elimination and in-order substitutions. Single thread; a is s x s col-major
// (destroyed). Returns false on a singular pivot.
__device__ bool dev_lu_solve(int s, double* a, const double* rhs, double* x) {
  int perm[kMaxS];
  double scale = 0.0;
  for (int idx = 0; idx < s * s; ++idx) scale = dmax_ref(scale, fabs(a[idx]));
  for (int i = 0; i < s; ++i) perm[i] = i;
  for (int k = 0; k < s; ++k) {
    int piv = k;
    double best = fabs(a[k + k * s]);
    for (int i = k + 1; i < s; ++i) {
      const double m = fabs(a[i + k * s]);
      if (m > best) {
        best = m;
        piv = i;
      }
    }
    if (best < 1e-14 * scale || scale == 0.0) return false;
    if (piv != k) {
      const int t = perm[k];
      perm[k] = perm[piv];
      perm[piv] = t;
      for (int j = 0; j < s; ++j) {
        const double u = a[k + j * s];
        a[k + j * s] = a[piv + j * s];
        a[piv + j * s] = u;
      }
    }
    const double inv = 1.0 / a[k + k * s];
    for (int i = k + 1; i < s; ++i) {
      const double m = a[i + k * s] * inv;
      a[i + k * s] = m;
      if (m != 0.0)
        for (int j = k + 1; j < s; ++j) a[i + j * s] = a[i + j * s] - m * a[k + j * s];
    }
  }
  for (int i = 0; i < s; ++i) x[i] = rhs[perm[i]];
  for (int i = 1; i < s; ++i)
    for (int j = 0; j < i; ++j) x[i] = x[i] - a[i + j * s] * x[j];
  for (int i = s - 1; i >= 0; --i) {
    for (int j = i + 1; j < s; ++j) x[i] = x[i] - a[i + j * s] * x[j];
    x[i] = x[i] / a[i + i * s];
  }
  return true;
}

__device__ void set_breakdown(DevState* ds, int code, int mv) {
  ds->st.breakdown = code;
  ds->st.mv_at_breakdown = mv;
}

// The dense step after an SpMV reduction (single thread of the last CTA).
__device__ void finalize_spmv(const FinParams& f, const double* red, DevState* ds) {
  __shared__ double lu[kMaxS * kMaxS];
  const int s = f.s;
  switch (f.op) {
    case kFinStore:
      for (int i = 0; i < s; ++i) f.dst[i] = red[i];
      break;
    case kFinRhsEta0: {  // after step (b) of level k: rhs and eta_0 (msys_0 = P^H V^(k))
      for (int i = 0; i < s; ++i) ds->rhs[i] = red[i];
      for (int i = 0; i < s * s; ++i) lu[i] = ds->Ma[i];
      if (!dev_lu_solve(s, lu, ds->rhs, ds->eta)) set_breakdown(ds, kBreakSingular, f.k * (s + 1) + 1);
      break;
    }
    case kFinColEta: {  // after V^(k+1)_q = A v_q^(k)
      const int q = f.q, k = f.k;
      for (int i = 0; i < s; ++i) ds->Mn[i + q * s] = red[i];
      if (q + 1 < s) {
        // msys_{q+1} = [P^H V^(k+1)_{0..q}, P^H V^(k)_{q+1..s-1}]  (idrstab.cpp:133-137)
        for (int c = 0; c < s; ++c)
          for (int i = 0; i < s; ++i) lu[i + c * s] = (c <= q) ? ds->Mn[i + c * s] : ds->Ma[i + c * s];
        if (!dev_lu_solve(s, lu, ds->rhs, ds->eta + (q + 1) * s))
          set_breakdown(ds, kBreakSingular, k * (s + 1) + 1 + (q + 1));
      } else {
        if (k + 1 < f.ell) {  // gamma of level k+1: (P^H V^(k+1)) gamma = P^H r^(k+1)
          for (int i = 0; i < s * s; ++i) lu[i] = ds->Mn[i];
          if (!dev_lu_solve(s, lu, ds->rhs, ds->gamma + (k + 1) * kMaxS))
            set_breakdown(ds, kBreakSingular, (k + 1) * (s + 1));
        }
        for (int i = 0; i < s * s; ++i) ds->Ma[i] = ds->Mn[i];
        for (int i = 0; i < s; ++i) ds->g[i] = ds->rhs[i];
      }
      break;
    }
    case kFinTrueRes: {
      ds->st.resnorm = sqrt(red[s]);
      for (int i = 0; i < s; ++i) ds->g[i] = red[i];
      for (int i = 0; i < s * s; ++i) lu[i] = ds->Ma[i];
      ds->st.pending_singular = dev_lu_solve(s, lu, ds->g, ds->gamma) ? 0 : 1;
      break;
    }
    default:
      break;
  }
}

// ---------------------------------------------------------------------------------------------
// SpMV y = A x (csr.cpp:103-113: sequential accumulation from 0 in CSR order) with fused P^H y.
template <int S, bool TRUE_RES>
__global__ void __launch_bounds__(kBlock) k_spmv_ph(DevCsr a, const double* __restrict__ x,
                                                    double* __restrict__ y,
                                                    const double* __restrict__ p, int64_t ld,
                                                    const double* __restrict__ b, FinParams fin,
                                                    Reducer red) {
  DevState* ds = red.ds;
  if (ds->st.breakdown) return;
  constexpr int NS = S + (TRUE_RES ? 1 : 0);
  double part[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) part[i] = 0.0;
  const int64_t n = a.n;
  const int32_t* __restrict__ rp = a.row_ptr;
  const int32_t* __restrict__ ci = a.col_idx;
  const double* __restrict__ va = a.values;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    const int beg = __ldg(rp + row), end = __ldg(rp + row + 1);
    double acc = 0.0;
    for (int k = beg; k < end; ++k) acc = acc + __ldg(va + k) * __ldg(x + __ldg(ci + k));
    if (TRUE_RES) acc = b[row] - acc;
    y[row] = acc;
#pragma unroll
    for (int c = 0; c < S; ++c) part[c] = part[c] + __ldg(p + c * ld + row) * acc;
    if (TRUE_RES) part[S] = part[S] + acc * acc;
  }
  __shared__ double scratch[NS * 32];
  __shared__ double blk[NS];
  __shared__ double redv[NS];
  block_totals<NS>(part, blk, scratch);
  if (!cta_commit(blk, NS, red.partials, &ds->ticket, redv)) return;
  if (threadIdx.x == 0) finalize_spmv(fin, redv, ds);
}

// step (a), top level: r_out = r_in - (sum_c gamma_c V_c)  (gemv then subtract, idrstab.cpp:113-117)
template <int S>
__global__ void __launch_bounds__(kBlock) k_level_update(int64_t n, int64_t ld, int k,
                                                         const double* __restrict__ r_in,
                                                         double* __restrict__ r_out,
                                                         const double* __restrict__ vk,
                                                         DevState* ds) {
  if (k == 0 && ds->st.pending_singular) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && !ds->st.breakdown) set_breakdown(ds, kBreakSingular, 0);
    return;
  }
  if (ds->st.breakdown) return;
  double gm[S];
#pragma unroll
  for (int c = 0; c < S; ++c) gm[c] = ds->gamma[k * kMaxS + c];
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double corr = 0.0;
#pragma unroll
    for (int c = 0; c < S; ++c) corr = corr + gm[c] * __ldg(vk + c * ld + row);
    r_out[row] = r_in[row] - corr;
  }
}

// step (c), top level, column q (idrstab.cpp:140-148 at i = k)
template <int S>
__global__ void __launch_bounds__(kBlock) k_rebuild_top(int64_t n, int64_t ld, int q,
                                                        const double* __restrict__ rnext,
                                                        const double* __restrict__ vk_in,
                                                        double* __restrict__ vk_out,
                                                        const double* __restrict__ vk1,
                                                        DevState* ds) {
  if (ds->st.breakdown) return;
  double et[S];
#pragma unroll
  for (int c = 0; c < S; ++c) et[c] = ds->eta[q * S + c];
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double nc = rnext[row];
#pragma unroll
    for (int c = 0; c < S; ++c) {
      const double m = (c < q) ? vk1[c * ld + row] : vk_in[c * ld + row];
      nc = nc + (-et[c]) * m;
    }
    vk_out[q * ld + row] = nc;
  }
}

struct DeferredArgs {
  const double* lv_in[kMaxEll + 2];
  double* lv_out[kMaxEll + 2];
  const double* r_in[kMaxEll + 1];
  double* r_out[kMaxEll + 1];
  const double* x_in;
  double* x_out;
};

// Deferred lower levels of level k (see kernels.h). Level k is final; levels i = k-1 .. -1 are
// rebuilt top-down, each needing only level i+1 (final) and level i (being updated in q order).
template <int S>
__global__ void __launch_bounds__(kBlock) k_rebuild_deferred(int64_t n, int64_t ld, int k,
                                                             DeferredArgs a, DevState* ds) {
  if (ds->st.breakdown) return;
  __shared__ double et[S * S];
  __shared__ double gm[S];
  for (int i = threadIdx.x; i < S * S; i += blockDim.x) et[i] = ds->eta[i];
  if (threadIdx.x < S) gm[threadIdx.x] = ds->gamma[k * kMaxS + threadIdx.x];
  __syncthreads();
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double ln[S], lc[S];
    const double* top = a.lv_in[k + 1];
#pragma unroll
    for (int c = 0; c < S; ++c) ln[c] = top[c * ld + row];
    double r_above = a.r_in[k][row];
    for (int i = k - 1; i >= -1; --i) {
      const double* cur = a.lv_in[i + 1];
#pragma unroll
      for (int c = 0; c < S; ++c) lc[c] = cur[c * ld + row];
      // deferred step (a) for this level (idrstab.cpp:113-121), with the level's pre-rebuild V
      double corr = 0.0;
#pragma unroll
      for (int c = 0; c < S; ++c) corr = corr + gm[c] * lc[c];
      double ri = 0.0;
      if (i >= 0) {
        ri = a.r_in[i][row] - corr;
        a.r_out[i][row] = ri;
      } else {
        a.x_out[row] = a.x_in[row] + corr;
      }
      // step (c) at level i for every column q, in q order (idrstab.cpp:140-148)
#pragma unroll
      for (int q = 0; q < S; ++q) {
        double nc = r_above;
#pragma unroll
        for (int c = 0; c < S; ++c) nc = nc + (-et[q * S + c]) * ((c < q) ? ln[c] : lc[c]);
        lc[q] = nc;
      }
      double* out = a.lv_out[i + 1];
#pragma unroll
      for (int c = 0; c < S; ++c) {
        out[c * ld + row] = lc[c];
        ln[c] = lc[c];
      }
      r_above = ri;
    }
  }
}

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
    const double r = sqrt(aj * aj + bj * bj);
    const double inv = 1.0 / r;
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
  if (ds->st.breakdown) return;
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
    double cnt[L];
    for (int j = 0; j < L; ++j) {
      const double* p = part + (size_t)(NR + j) * G;
      double acc = 0.0;
      for (int c = 0; c < G; ++c) acc += __ldcg(p + c);
      cnt[j] = acc;
    }
    ls_finalize<L>(Rc, cnt, s, ds);
    ds->ticket = 0u;
  }
}

// ---------------------------------------------------------------------------------------------
// Tile Gram helper: thread accumulates output o = t % (S*S) over the rows of its part.
template <int S>
struct GramMap {
  static constexpr int O = S * S;
  static constexpr int NP = (kBlock / O) > 0 ? (kBlock / O) : 1;
  static constexpr int LDT = kBlock + 1;  // odd stride: conflict-free column reads
};

template <int S>
__device__ __forceinline__ void gram_tile(const double* A, const double* B, double& acc) {
  using GM = GramMap<S>;
  const int t = threadIdx.x;
  if (t >= GM::O * GM::NP) return;
  const int o = t % GM::O, part = t / GM::O;
  const int i = o % S, j = o / S;
  const double* ai = A + i * GM::LDT;
  const double* bj = B + j * GM::LDT;
  for (int r = part; r < kBlock; r += GM::NP) acc = acc + ai[r] * bj[r];
}

template <int S>
__device__ __forceinline__ void gram_combine(double acc, double* gsc /*kBlock*/, double* out /*O*/) {
  using GM = GramMap<S>;
  gsc[threadIdx.x] = acc;
  __syncthreads();
  for (int o = threadIdx.x; o < GM::O; o += blockDim.x) {
    double v = 0.0;
    for (int part = 0; part < GM::NP; ++part) v += gsc[part * GM::O + o];
    out[o] = v;
  }
  __syncthreads();
}

struct PolyArgs {
  const double* lv[kMaxEll + 2];  // V^(-1..ell)
  const double* r[kMaxEll + 1];   // r^(0..ell)
  double* u_out;
  double* v_out;
  double* r_out;
  const double* x_in;
  double* x_out;
  const double* p;
};

// POLY = true: poly_combination (idrstab.cpp:154-191) + fused reductions.
// POLY = false: prologue (reductions of the given V and r only).
// Slots: [0] ||r||^2, [1..S] P^H r, [1+S ..] P^H V (col-major s x s).
template <int S, bool POLY>
__global__ void __launch_bounds__(kBlock) k_poly(int64_t n, int64_t ld, int ell, PolyArgs a,
                                                 Reducer red) {
  DevState* ds = red.ds;
  if (ds->st.breakdown) return;
  using GM = GramMap<S>;
  extern __shared__ double dsm[];
  double* Vs = dsm;                  // S x LDT
  double* Ps = dsm + S * GM::LDT;    // S x LDT
  __shared__ double taus[kMaxEll];
  if (POLY && threadIdx.x < ell) taus[threadIdx.x] = ds->st.tau[threadIdx.x];
  __syncthreads();
  double pr[S + 1];
#pragma unroll
  for (int c = 0; c <= S; ++c) pr[c] = 0.0;
  double gacc = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * kBlock; base < n; base += (int64_t)gridDim.x * kBlock) {
    const int64_t row = base + threadIdx.x;
    if (row < n) {
      double r = a.r[0][row];
      if (POLY) {
        double x = a.x_in[row];
        for (int i = 1; i <= ell; ++i) {
          const double t = taus[i - 1];
          r = r + (-t) * a.r[i][row];
          x = x + t * a.r[i - 1][row];
        }
        a.r_out[row] = r;
        a.x_out[row] = x;
      }
      pr[S] = pr[S] + r * r;
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const double pq = a.p[q * ld + row];
        double vq;
        if (POLY) {
          double uq = a.lv[0][q * ld + row];
          vq = a.lv[1][q * ld + row];
          for (int i = 1; i <= ell; ++i) {
            const double t = taus[i - 1];
            uq = uq + (-t) * a.lv[i][q * ld + row];
            vq = vq + (-t) * a.lv[i + 1][q * ld + row];
          }
          a.u_out[q * ld + row] = uq;
          a.v_out[q * ld + row] = vq;
        } else {
          vq = a.lv[1][q * ld + row];
        }
        pr[q] = pr[q] + pq * r;
        Vs[q * GM::LDT + threadIdx.x] = vq;
        Ps[q * GM::LDT + threadIdx.x] = pq;
      }
    } else {
#pragma unroll
      for (int q = 0; q < S; ++q) {
        Vs[q * GM::LDT + threadIdx.x] = 0.0;
        Ps[q * GM::LDT + threadIdx.x] = 0.0;
      }
    }
    __syncthreads();
    gram_tile<S>(Ps, Vs, gacc);
    __syncthreads();
  }
  constexpr int NSL = 1 + S + S * S;
  __shared__ double blk[NSL];
  __shared__ double redv[NSL];
  __shared__ double scratch[(S + 1) * 32];
  __shared__ double gsc[kBlock];
  {
    double tot[S + 1];
#pragma unroll
    for (int c = 0; c <= S; ++c) tot[c] = pr[c];
    __shared__ double blk0[S + 1];
    block_totals<S + 1>(tot, blk0, scratch);
    if (threadIdx.x == 0) blk[0] = blk0[S];
    if (threadIdx.x < S) blk[1 + threadIdx.x] = blk0[threadIdx.x];
    gram_combine<S>(gacc, gsc, blk + 1 + S);
  }
  if (!cta_commit(blk, NSL, red.partials, &ds->ticket, redv)) return;
  if (threadIdx.x == 0) {
    __shared__ double lu[kMaxS * kMaxS];
    ds->st.resnorm = sqrt(redv[0]);
    for (int i = 0; i < S; ++i) ds->g[i] = redv[1 + i];
    for (int i = 0; i < S * S; ++i) ds->Ma[i] = redv[1 + S + i];
    for (int i = 0; i < S * S; ++i) lu[i] = ds->Ma[i];
    ds->st.pending_singular = dev_lu_solve(S, lu, ds->g, ds->gamma) ? 0 : 1;
  }
}

// validate(): ||V - A U||^2, sum ||V_q||^2, P^H P, V^H V in one pass.
template <int S>
__global__ void __launch_bounds__(kBlock) k_validate(DevCsr a, const double* __restrict__ p,
                                                     const double* __restrict__ u,
                                                     const double* __restrict__ v, int64_t ld,
                                                     Reducer red) {
  DevState* ds = red.ds;
  using GM = GramMap<S>;
  extern __shared__ double dsm[];
  double* Vs = dsm;
  double* Ps = dsm + S * GM::LDT;
  double dn[2] = {0.0, 0.0};
  double g1 = 0.0, g2 = 0.0;
  const int64_t n = a.n;
  for (int64_t base = (int64_t)blockIdx.x * kBlock; base < n; base += (int64_t)gridDim.x * kBlock) {
    const int64_t row = base + threadIdx.x;
    if (row < n) {
      double acc[S];
#pragma unroll
      for (int q = 0; q < S; ++q) acc[q] = 0.0;
      const int beg = a.row_ptr[row], end = a.row_ptr[row + 1];
      for (int k = beg; k < end; ++k) {
        const double av = a.values[k];
        const int col = a.col_idx[k];
#pragma unroll
        for (int q = 0; q < S; ++q) acc[q] = acc[q] + av * __ldg(u + q * ld + col);
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const double vq = v[q * ld + row];
        const double d = vq - acc[q];
        dn[0] = dn[0] + d * d;
        dn[1] = dn[1] + vq * vq;
        Vs[q * GM::LDT + threadIdx.x] = vq;
        Ps[q * GM::LDT + threadIdx.x] = p[q * ld + row];
      }
    } else {
#pragma unroll
      for (int q = 0; q < S; ++q) {
        Vs[q * GM::LDT + threadIdx.x] = 0.0;
        Ps[q * GM::LDT + threadIdx.x] = 0.0;
      }
    }
    __syncthreads();
    gram_tile<S>(Ps, Ps, g1);
    gram_tile<S>(Vs, Vs, g2);
    __syncthreads();
  }
  constexpr int NSL = 2 + 2 * S * S;
  __shared__ double blk[NSL];
  __shared__ double redv[NSL];
  __shared__ double scratch[2 * 32];
  __shared__ double gsc[kBlock];
  block_totals<2>(dn, blk, scratch);
  gram_combine<S>(g1, gsc, blk + 2);
  gram_combine<S>(g2, gsc, blk + 2 + S * S);
  if (!cta_commit(blk, NSL, red.partials, &ds->ticket, redv)) return;
  if (threadIdx.x == 0) {
    ds->scal[0] = redv[0];
    ds->scal[1] = redv[1];
    for (int i = 0; i < 2 * S * S; ++i) ds->gram[i] = redv[2 + i];
  }
}

// ---------------------------------------------------------------------------------------------
constexpr int kMaxDots = kMaxS + 1;

__global__ void __launch_bounds__(kBlock) k_dots(int64_t n, int64_t ld, const double* __restrict__ a,
                                                 int na, const double* __restrict__ y, int with_norm,
                                                 double* dst, Reducer red) {
  DevState* ds = red.ds;
  double acc[kMaxDots];
#pragma unroll
  for (int j = 0; j < kMaxDots; ++j) acc[j] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    const double yv = y[row];
#pragma unroll
    for (int j = 0; j < kMaxS; ++j)
      if (j < na) acc[j] = acc[j] + a[j * ld + row] * yv;
    if (with_norm) acc[kMaxS] = acc[kMaxS] + yv * yv;
  }
  __shared__ double scratch[kMaxDots * 32];
  __shared__ double blk[kMaxDots];
  __shared__ double redv[kMaxDots];
  block_totals<kMaxDots>(acc, blk, scratch);
  if (!cta_commit(blk, kMaxDots, red.partials, &ds->ticket, redv)) return;
  if (threadIdx.x == 0) {
    for (int j = 0; j < na; ++j) dst[j] = redv[j];
    if (with_norm) dst[na] = redv[kMaxS];
  }
}

__global__ void __launch_bounds__(kBlock) k_axpy_neg(int64_t n, int64_t ld, const double* __restrict__ a,
                                                     int na, const double* __restrict__ coef,
                                                     double* __restrict__ y) {
  double cf[kMaxS];
#pragma unroll
  for (int j = 0; j < kMaxS; ++j) cf[j] = (j < na) ? coef[j] : 0.0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double yv = y[row];
#pragma unroll
    for (int j = 0; j < kMaxS; ++j)
      if (j < na) yv = yv + (-cf[j]) * a[j * ld + row];
    y[row] = yv;
  }
}

__global__ void k_div_by_sqrt(int64_t n, const double* __restrict__ x, const double* d2,
                              double* __restrict__ y) {
  const double d = sqrt(*d2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}

__global__ void k_mul_inv_sqrt(int64_t n, const double* __restrict__ x, const double* d2,
                               double* __restrict__ y) {
  const double inv = 1.0 / sqrt(*d2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * inv;
}

__global__ void k_rsub(int64_t n, const double* __restrict__ b, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = b[i] - y[i];
}

__global__ void __launch_bounds__(kBlock) k_vec_stats(int64_t n, const double* __restrict__ x,
                                                      double* dst, Reducer red) {
  DevState* ds = red.ds;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    acc[0] = acc[0] + v * v;
    if (!isfinite(v)) acc[1] += 1.0;
    if (v != 0.0) acc[2] += 1.0;
  }
  __shared__ double scratch[3 * 32];
  __shared__ double blk[3];
  __shared__ double redv[3];
  block_totals<3>(acc, blk, scratch);
  if (!cta_commit(blk, 3, red.partials, &ds->ticket, redv)) return;
  if (threadIdx.x == 0)
    for (int j = 0; j < 3; ++j) dst[j] = redv[j];
}

__global__ void k_euler_rhs(int64_t n, const double* __restrict__ x, const double* __restrict__ f,
                            double dt, double h2, double* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = h2 * (x[i] / dt + f[i]);
}

__global__ void k_axpby_chain(int64_t n, const double* __restrict__ x, const double* __restrict__ g,
                              double alpha, double* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = x[i] + alpha * g[i];
}

__global__ void k_small_solve(int s, const double* m, const double* rhs, double* x, int32_t* ok) {
  __shared__ double lu[kMaxS * kMaxS];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < s * s; ++i) lu[i] = m[i];
  *ok = dev_lu_solve(s, lu, rhs, x) ? 1 : 0;
}

// Resident CTAs per SM of each kernel, queried once (the occupancy API costs tens of us per
// call, which would starve the GPU between launches).
std::mutex g_occ_mu;
std::unordered_map<const void*, int> g_occ;

template <typename K>
int occupancy_grid(K kernel, int64_t n, size_t dyn_smem) {
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(g_occ_mu);
    auto it = g_occ.find(reinterpret_cast<const void*>(kernel));
    if (it != g_occ.end()) {
      per_sm = it->second;
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, dyn_smem);
      if (per_sm < 1) per_sm = 1;
      g_occ[reinterpret_cast<const void*>(kernel)] = per_sm;
    }
  }
  int64_t want = (n + kBlock - 1) / kBlock;
  int64_t cap = (int64_t)g_num_sms * per_sm;
  if (cap > kMaxGrid) cap = kMaxGrid;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

template <int S>
size_t gram_smem() {
  return sizeof(double) * 2 * S * GramMap<S>::LDT;
}

}  // namespace

// ---- dispatch --------------------------------------------------------------------------------
#define MSTAB_DISPATCH_S(s, ...)                      \
  switch (s) {                                         \
    case 1: { constexpr int S = 1; __VA_ARGS__; } break;      \
    case 2: { constexpr int S = 2; __VA_ARGS__; } break;      \
    case 3: { constexpr int S = 3; __VA_ARGS__; } break;      \
    case 4: { constexpr int S = 4; __VA_ARGS__; } break;      \
    case 5: { constexpr int S = 5; __VA_ARGS__; } break;      \
    case 6: { constexpr int S = 6; __VA_ARGS__; } break;      \
    case 7: { constexpr int S = 7; __VA_ARGS__; } break;      \
    case 8: { constexpr int S = 8; __VA_ARGS__; } break;      \
    case 9: { constexpr int S = 9; __VA_ARGS__; } break;      \
    case 10: { constexpr int S = 10; __VA_ARGS__; } break;    \
    case 11: { constexpr int S = 11; __VA_ARGS__; } break;    \
    case 12: { constexpr int S = 12; __VA_ARGS__; } break;    \
    case 13: { constexpr int S = 13; __VA_ARGS__; } break;    \
    case 14: { constexpr int S = 14; __VA_ARGS__; } break;    \
    case 15: { constexpr int S = 15; __VA_ARGS__; } break;    \
    case 16: { constexpr int S = 16; __VA_ARGS__; } break;    \
    default: break;                                    \
  }

#define MSTAB_DISPATCH_L(l, ...)                      \
  switch (l) {                                         \
    case 1: { constexpr int L = 1; __VA_ARGS__; } break;      \
    case 2: { constexpr int L = 2; __VA_ARGS__; } break;      \
    case 3: { constexpr int L = 3; __VA_ARGS__; } break;      \
    case 4: { constexpr int L = 4; __VA_ARGS__; } break;      \
    case 5: { constexpr int L = 5; __VA_ARGS__; } break;      \
    case 6: { constexpr int L = 6; __VA_ARGS__; } break;      \
    case 7: { constexpr int L = 7; __VA_ARGS__; } break;      \
    case 8: { constexpr int L = 8; __VA_ARGS__; } break;      \
    default: break;                                    \
  }

void kernels_init(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
    g_num_sms = sms;
  // opt in to > 48 KB dynamic shared memory for the Gram tiles (s up to 16)
#define MSTAB_SET_SMEM(S)                                                                      \
  cudaFuncSetAttribute(k_poly<S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem<S>()); \
  cudaFuncSetAttribute(k_poly<S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem<S>()); \
  cudaFuncSetAttribute(k_validate<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem<S>());
  MSTAB_SET_SMEM(1) MSTAB_SET_SMEM(2) MSTAB_SET_SMEM(3) MSTAB_SET_SMEM(4) MSTAB_SET_SMEM(5)
  MSTAB_SET_SMEM(6) MSTAB_SET_SMEM(7) MSTAB_SET_SMEM(8) MSTAB_SET_SMEM(9) MSTAB_SET_SMEM(10)
  MSTAB_SET_SMEM(11) MSTAB_SET_SMEM(12) MSTAB_SET_SMEM(13) MSTAB_SET_SMEM(14) MSTAB_SET_SMEM(15)
  MSTAB_SET_SMEM(16)
#undef MSTAB_SET_SMEM
}

namespace {

// ---- launch accounting -------------------------------------------------------------------------
std::atomic<uint64_t> g_launch_count{0};

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  double bytes;
};

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<ProfRec> pending;
  KernelClassStats stats[kKNumClasses] = {};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
};
Profiler g_prof;
std::mutex g_prof_mu;

// Counts one launch; with profiling on, brackets it with events on its stream.
struct LaunchScope {
  cudaStream_t st;
  int cls;
  double bytes;
  cudaEvent_t a = nullptr;
  LaunchScope(cudaStream_t s, int c, double b) : st(s), cls(c), bytes(b) {
    g_launch_count.fetch_add(1, std::memory_order_relaxed);
    if (g_prof.on) {
      std::lock_guard<std::mutex> lk(g_prof_mu);
      a = g_prof.get();
      cudaEventRecord(a, st);
    }
  }
  ~LaunchScope() {
    if (!a) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t b = g_prof.get();
    cudaEventRecord(b, st);
    g_prof.pending.push_back({cls, a, b, bytes});
  }
};

inline double vbytes(int64_t n, double vectors) { return 8.0 * (double)n * vectors; }
inline double csr_bytes(const DevCsr& a) { return 12.0 * (double)a.nnz + 4.0 * (double)(a.n + 1); }

}  // namespace

uint64_t launch_count() { return g_launch_count.load(); }

void prof_enable(bool on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.on = on;
  // events are created up front and only read back at prof_collect(), so the timed region pays
  // one cudaEventRecord per launch boundary and nothing else
  while (on && g_prof.pool.size() < 65536) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    g_prof.pool.push_back(e);
  }
}

void prof_collect() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (const ProfRec& r : g_prof.pending) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    KernelClassStats& s = g_prof.stats[r.cls];
    s.launches++;
    s.total_ms += ms;
    s.total_bytes += r.bytes;
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.pending.clear();
}

void prof_read(KernelClassStats* out) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int i = 0; i < kKNumClasses; ++i) out[i] = g_prof.stats[i];
}

void prof_reset() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& s : g_prof.stats) s = KernelClassStats{};
}

int grid_for(int64_t n) {
  int64_t want = (n + kBlock - 1) / kBlock;
  int64_t cap = (int64_t)g_num_sms * 4;
  if (want > cap) want = cap;
  return want < 1 ? 1 : (int)want;
}

void launch_spmv_ph(cudaStream_t st, const DevCsr& a, const double* x, double* y, const double* p,
                    int64_t ld, int s, const double* b, const FinParams& fin, const Reducer& red) {
  // CSR + gathered x + y + P^H epilogue (+ b for the true-residual form)
  LaunchScope ls(st, kKSpmv, csr_bytes(a) + vbytes(a.n, 2.0 + s + (b ? 1.0 : 0.0)));
  MSTAB_DISPATCH_S(s, {
    if (b) {
      auto kfn = k_spmv_ph<S, true>;
      const int grid = occupancy_grid(kfn, a.n, 0);
      kfn<<<grid, kBlock, 0, st>>>(a, x, y, p, ld, b, fin, red);
    } else {
      auto kfn = k_spmv_ph<S, false>;
      const int grid = occupancy_grid(kfn, a.n, 0);
      kfn<<<grid, kBlock, 0, st>>>(a, x, y, p, ld, b, fin, red);
    }
  });
}

void launch_level_update(cudaStream_t st, int64_t n, int64_t ld, int s, int k, const double* r_in,
                         double* r_out, const double* vk, DevState* ds) {
  LaunchScope ls(st, kKLevelUpdate, vbytes(n, s + 2.0));
  MSTAB_DISPATCH_S(s, {
    auto kfn = k_level_update<S>;
    const int grid = occupancy_grid(kfn, n, 0);
    kfn<<<grid, kBlock, 0, st>>>(n, ld, k, r_in, r_out, vk, ds);
  });
}

void launch_rebuild_top(cudaStream_t st, int64_t n, int64_t ld, int s, int q, const double* rnext,
                        const double* vk_in, double* vk_out, const double* vk1, DevState* ds) {
  LaunchScope ls(st, kKRebuildTop, vbytes(n, s + 2.0));
  MSTAB_DISPATCH_S(s, {
    auto kfn = k_rebuild_top<S>;
    const int grid = occupancy_grid(kfn, n, 0);
    kfn<<<grid, kBlock, 0, st>>>(n, ld, q, rnext, vk_in, vk_out, vk1, ds);
  });
}

void launch_rebuild_deferred(cudaStream_t st, int64_t n, int64_t ld, int s, int k,
                             const double* const* lv_in, double* const* lv_out,
                             const double* const* r_in, double* const* r_out, const double* x_in,
                             double* x_out, DevState* ds) {
  // reads x, r^(0..k), V^(-1..k); writes x, r^(0..k-1), V^(-1..k-1)
  LaunchScope ls(st, kKRebuildDeferred,
                 vbytes(n, (k + 1.0) + 1.0 + (k + 2.0) * s + k + 1.0 + (k + 1.0) * s));
  DeferredArgs a{};
  for (int i = 0; i <= k + 1; ++i) {
    a.lv_in[i] = lv_in[i];
    a.lv_out[i] = lv_out[i];
  }
  for (int i = 0; i <= k; ++i) {
    a.r_in[i] = r_in[i];
    a.r_out[i] = r_out[i];
  }
  a.x_in = x_in;
  a.x_out = x_out;
  MSTAB_DISPATCH_S(s, {
    auto kfn = k_rebuild_deferred<S>;
    const int grid = occupancy_grid(kfn, n, 0);
    kfn<<<grid, kBlock, 0, st>>>(n, ld, k, a, ds);
  });
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
    kfn<<<grid, kBlock, 0, st>>>(n, s, a, red);
  });
}

void launch_poly(cudaStream_t st, int64_t n, int64_t ld, int s, int ell, const double* const* lv,
                 double* u_out, double* v_out, const double* const* r, double* r_out,
                 const double* x_in, double* x_out, const double* p, const Reducer& red) {
  // reads x, r^(0..ell), V^(-1..ell), P; writes x, r, U, V
  LaunchScope ls(st, kKPoly, vbytes(n, 1.0 + (ell + 1.0) + (ell + 2.0) * s + s + 2.0 + 2.0 * s));
  PolyArgs a{};
  for (int i = 0; i <= ell + 1; ++i) a.lv[i] = lv[i];
  for (int i = 0; i <= ell; ++i) a.r[i] = r[i];
  a.u_out = u_out;
  a.v_out = v_out;
  a.r_out = r_out;
  a.x_in = x_in;
  a.x_out = x_out;
  a.p = p;
  MSTAB_DISPATCH_S(s, {
    auto kfn = k_poly<S, true>;
    const size_t sm = gram_smem<S>();
    const int grid = occupancy_grid(kfn, n, sm);
    kfn<<<grid, kBlock, sm, st>>>(n, ld, ell, a, red);
  });
}

void launch_prologue(cudaStream_t st, int64_t n, int64_t ld, int s, const double* p,
                     const double* v, const double* r, const Reducer& red) {
  LaunchScope ls(st, kKPrologue, vbytes(n, 2.0 * s + 1.0));
  PolyArgs a{};
  a.lv[1] = v;
  a.r[0] = r;
  a.p = p;
  MSTAB_DISPATCH_S(s, {
    auto kfn = k_poly<S, false>;
    const size_t sm = gram_smem<S>();
    const int grid = occupancy_grid(kfn, n, sm);
    kfn<<<grid, kBlock, sm, st>>>(n, ld, 0, a, red);
  });
}

void launch_validate(cudaStream_t st, const DevCsr& a, const double* p, const double* u,
                     const double* v, int64_t ld, int s, const Reducer& red) {
  LaunchScope ls(st, kKValidate, csr_bytes(a) + vbytes(a.n, 3.0 * s));
  MSTAB_DISPATCH_S(s, {
    auto kfn = k_validate<S>;
    const size_t sm = gram_smem<S>();
    const int grid = occupancy_grid(kfn, a.n, sm);
    kfn<<<grid, kBlock, sm, st>>>(a, p, u, v, ld, red);
  });
}

void launch_dots(cudaStream_t st, int64_t n, int64_t ld, const double* a, int na, const double* y,
                 bool with_norm, double* dst, const Reducer& red) {
  LaunchScope ls(st, kKOther, vbytes(n, na + 1.0));
  const int grid = occupancy_grid(k_dots, n, 0);
  k_dots<<<grid, kBlock, 0, st>>>(n, ld, a, na, y, with_norm ? 1 : 0, dst, red);
}

void launch_axpy_neg(cudaStream_t st, int64_t n, int64_t ld, const double* a, int na,
                     const double* coef, double* y) {
  LaunchScope ls(st, kKOther, vbytes(n, na + 2.0));
  const int grid = occupancy_grid(k_axpy_neg, n, 0);
  k_axpy_neg<<<grid, kBlock, 0, st>>>(n, ld, a, na, coef, y);
}

void launch_div_by_sqrt(cudaStream_t st, int64_t n, const double* x, const double* d2, double* y) {
  LaunchScope ls(st, kKOther, vbytes(n, 2.0));
  k_div_by_sqrt<<<grid_for(n), kBlock, 0, st>>>(n, x, d2, y);
}

void launch_mul_inv_sqrt(cudaStream_t st, int64_t n, const double* x, const double* d2, double* y) {
  LaunchScope ls(st, kKOther, vbytes(n, 2.0));
  k_mul_inv_sqrt<<<grid_for(n), kBlock, 0, st>>>(n, x, d2, y);
}

void launch_rsub(cudaStream_t st, int64_t n, const double* b, double* y) {
  LaunchScope ls(st, kKOther, vbytes(n, 3.0));
  k_rsub<<<grid_for(n), kBlock, 0, st>>>(n, b, y);
}

void launch_vec_stats(cudaStream_t st, int64_t n, const double* x, double* dst, const Reducer& red) {
  LaunchScope ls(st, kKOther, vbytes(n, 1.0));
  const int grid = occupancy_grid(k_vec_stats, n, 0);
  k_vec_stats<<<grid, kBlock, 0, st>>>(n, x, dst, red);
}

void launch_euler_rhs(cudaStream_t st, int64_t n, const double* x, const double* f, double dt,
                      double h2, double* b) {
  LaunchScope ls(st, kKOther, vbytes(n, 3.0));
  k_euler_rhs<<<grid_for(n), kBlock, 0, st>>>(n, x, f, dt, h2, b);
}

void launch_axpby_chain(cudaStream_t st, int64_t n, const double* x, const double* g, double alpha,
                        double* b) {
  LaunchScope ls(st, kKOther, vbytes(n, 3.0));
  k_axpby_chain<<<grid_for(n), kBlock, 0, st>>>(n, x, g, alpha, b);
}

void launch_small_solve(cudaStream_t st, int s, const double* m, const double* rhs, double* x,
                        int32_t* ok) {
  LaunchScope ls(st, kKOther, 0.0);
  k_small_solve<<<1, 32, 0, st>>>(s, m, rhs, x, ok);
}

}  // namespace mstab_b200
