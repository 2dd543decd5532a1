// kpoly.cu — poly_combination / prologue (fused Gram reductions) and validate kernels.
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
__global__ void __launch_bounds__(kBlock, S <= 8 ? 3 : 1) k_poly(int64_t n, int64_t ld, int ell, PolyArgs a,
                                                 Reducer red) {
  DevState* ds = red.ds;
  pdl_wait();
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
      // U_q = V^(-1)_q - sum_i tau_i V^(i-1)_q ; V_q = V^(0)_q - sum_i tau_i V^(i)_q, i ascending per
      // column (idrstab.cpp:182-189); the level loop is outermost so each runtime iteration
      // issues S independent loads (level i serves U at i+1 and V at i)
      double uq[S], vq[S], lvl[S];
#pragma unroll
      for (int q = 0; q < S; ++q) {
        uq[q] = POLY ? a.lv[0][q * ld + row] : 0.0;
        vq[q] = a.lv[1][q * ld + row];
      }
      if (POLY) {
#pragma unroll
        for (int q = 0; q < S; ++q) lvl[q] = vq[q];  // V^(0) feeds U's i = 1 term
        for (int i = 1; i <= ell; ++i) {
          const double t = taus[i - 1];
          const double* nxt = a.lv[i + 1];
#pragma unroll
          for (int q = 0; q < S; ++q) {
            const double li1 = nxt[q * ld + row];  // V^(i)
            uq[q] = uq[q] + (-t) * lvl[q];         // - tau_i V^(i-1)
            vq[q] = vq[q] + (-t) * li1;            // - tau_i V^(i)
            lvl[q] = li1;
          }
        }
#pragma unroll
        for (int q = 0; q < S; ++q) {
          a.u_out[q * ld + row] = uq[q];
          a.v_out[q * ld + row] = vq[q];
        }
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const double pq = a.p[q * ld + row];
        pr[q] = pr[q] + pq * r;
        Vs[q * GM::LDT + threadIdx.x] = vq[q];
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
  pdl_trigger();
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
  if (!cta_commit(blk, NSL, red.partials, &ds->ticket, redv, red.xred)) return;
  poly_tail<S>(redv, ds);
}

// Row-sharded finaliser of poly / prologue: the allreduced slots through the same tail.
template <int S>
__global__ void __launch_bounds__(kBlock) k_fin_poly(DevState* ds) {
  constexpr int NSL = 1 + S + S * S;
  __shared__ double redv[NSL];
  pdl_wait();  // ds->xred is written by the collective that precedes this launch
  for (int i = threadIdx.x; i < NSL; i += blockDim.x) redv[i] = ds->xred[i];
  __syncthreads();
  poly_tail<S>(redv, ds);
}

// validate(): ||V - A U||^2, sum ||V_q||^2, P^H P, V^H V in one pass.
template <int S>
__global__ void __launch_bounds__(kBlock) k_validate(DevCsr a, const double* __restrict__ p,
                                                     const double* __restrict__ u,
                                                     const double* __restrict__ v, int64_t ld,
                                                     Reducer red, const double* __restrict__ au) {
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
      if (au) {
#pragma unroll
        for (int q = 0; q < S; ++q) acc[q] = au[q * ld + row];
      } else {
        const int beg = a.row_ptr[row], end = a.row_ptr[row + 1];
        for (int k = beg; k < end; ++k) {
          const double av = a.values[k];
          const int col = a.col_idx[k];
#pragma unroll
          for (int q = 0; q < S; ++q) acc[q] = acc[q] + av * __ldg(u + q * ld + col);
        }
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
  if (!cta_commit(blk, NSL, red.partials, &ds->ticket, redv, red.xred)) return;
  if (threadIdx.x < 2) ds->scal[threadIdx.x] = redv[threadIdx.x];
  for (int i = threadIdx.x; i < 2 * S * S; i += blockDim.x) ds->gram[i] = redv[2 + i];
}

template <int S>
size_t gram_smem() {
  return sizeof(double) * 2 * S * GramMap<S>::LDT;
}

}  // namespace

void launch_fin_poly(cudaStream_t st, int s, DevState* ds) {
  MSTAB_DISPATCH_S(s, { launch_pdl(k_fin_poly<S>, 1, kBlock, 0, st, ds); });
}

void kpoly_init() {
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
    launch_pdl(kfn, grid, kBlock, sm, st, n, ld, ell, a, red);
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
                     const double* v, int64_t ld, int s, const Reducer& red, const double* au) {
  LaunchScope ls(st, kKValidate, (au ? 0.0 : csr_bytes(a)) + vbytes(a.n, 3.0 * s));
  MSTAB_DISPATCH_S(s, {
    auto kfn = k_validate<S>;
    const size_t sm = gram_smem<S>();
    const int grid = occupancy_grid(kfn, a.n, sm);
    kfn<<<grid, kBlock, sm, st>>>(a, p, u, v, ld, red, au);
  });
}

}  // namespace mstab_b200
