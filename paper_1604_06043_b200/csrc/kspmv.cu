// kspmv.cu — SpMV kernels (CSR warp-staged and DIA) with the fused P^H epilogue.
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
  {
  const int32_t* __restrict__ rp = a.row_ptr;
  const int32_t* __restrict__ ci = a.col_idx;
  const double* __restrict__ va = a.values;
  // Each warp owns 32 consecutive rows; their CSR slice is staged through shared memory with
  // fully coalesced loads (the scalar one-thread-per-row walk would issue ~nnz/row strided
  // requests per warp), then every lane accumulates its own row from 0 in CSR order.
  __shared__ double s_val[kBlock / 32][kSpmvStage];
  __shared__ int32_t s_col[kBlock / 32][kSpmvStage];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* sv = s_val[wid];
  int32_t* sc = s_col[wid];
  const int64_t wstride = (int64_t)gridDim.x * (kBlock / 32) * 32;
  for (int64_t base = ((int64_t)blockIdx.x * (kBlock / 32) + wid) * 32; base < n; base += wstride) {
    const int64_t row = base + lane;
    const bool valid = row < n;
    const int64_t last = (base + 32 < n) ? base + 32 : n;
    const int beg = valid ? __ldg(rp + row) : 0;
    const int end = valid ? __ldg(rp + row + 1) : 0;
    const int wbeg = __shfl_sync(0xffffffffu, beg, 0);
    const int wend = __ldg(rp + last);
    double pv[S];
#pragma unroll
    for (int c = 0; c < S; ++c) pv[c] = valid ? __ldg(p + c * ld + row) : 0.0;
    const double bv = (TRUE_RES && valid) ? b[row] : 0.0;
    double acc = 0.0;
    for (int chunk = wbeg; chunk < wend; chunk += kSpmvStage) {
      const int cnt = min(kSpmvStage, wend - chunk);
      for (int i = lane; i < cnt; i += 32) {
        sv[i] = __ldg(va + chunk + i);
        sc[i] = __ldg(ci + chunk + i);
      }
      __syncwarp();
      const int lo = max(beg, chunk) - chunk, hi = min(end, chunk + cnt) - chunk;
      for (int k = lo; k < hi; ++k) acc = acc + sv[k] * __ldg(x + sc[k]);
      __syncwarp();
    }
    if (valid) {
      if (TRUE_RES) acc = bv - acc;
      y[row] = acc;
#pragma unroll
      for (int c = 0; c < S; ++c) part[c] = part[c] + pv[c] * acc;
      if (TRUE_RES) part[S] = part[S] + acc * acc;
    }
  }
  }  // CSR path
  __shared__ double scratch[NS * 32];
  __shared__ double blk[NS];
  __shared__ double redv[NS];
  block_totals<NS>(part, blk, scratch);
  if (!cta_commit(blk, NS, red.partials, &ds->ticket, redv)) return;
  finalize_spmv(fin, redv, ds);
}

// SpMV on the DIA form (kernels.h DevCsr): two rows per thread; every load of the row pair
// (chunks of kDiaChunk value pairs and 2*kDiaChunk x gathers, S P pairs) is independent and
// issued together (guarded unroll), so each warp keeps ~(3*8 + S) requests in flight. Value, P and y
// accesses are 16-byte vectors (ld, dia_ld are multiples of 64); gathers x[row + off] are
// contiguous across the warp. Accumulation d = 0.. is CSR column order (offsets ascending).
constexpr int kDiaChunk = 8;  // diagonals whose loads are issued together

template <int S, bool TRUE_RES>
__global__ void __launch_bounds__(kBlock, 2) k_spmv_dia(DevCsr a, const double* __restrict__ x,
                                                     double* __restrict__ y,
                                                     const double* __restrict__ p, int64_t ld,
                                                     const double* __restrict__ b, FinParams fin,
                                                     Reducer red) {
  DevState* ds = red.ds;
  if (ds->st.breakdown) return;
  constexpr int NS = S + (TRUE_RES ? 1 : 0);
  __shared__ int32_t s_off[kMaxDiag];
  const int nd = a.ndiag;
  for (int d = threadIdx.x; d < kMaxDiag; d += blockDim.x) s_off[d] = d < nd ? a.dia_off[d] : 0;
  __syncthreads();
  double part[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) part[i] = 0.0;
  const int64_t n = a.n;
  const double* __restrict__ dv = a.dia_val;
  const int64_t dld = a.dia_ld;
  const int64_t npair = (n + 1) >> 1;
  for (int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pr < npair;
       pr += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r0 = 2 * pr;
    const bool two = r0 + 1 < n;
    double2 pv[S];
#pragma unroll
    for (int c = 0; c < S; ++c)
      pv[c] = two ? __ldg(reinterpret_cast<const double2*>(p + c * ld + r0))
                  : make_double2(__ldg(p + c * ld + r0), 0.0);
    double acc0 = 0.0, acc1 = 0.0;
    for (int d0 = 0; d0 < nd; d0 += kDiaChunk) {
      double2 vv[kDiaChunk];
      double x0[kDiaChunk], x1[kDiaChunk];
#pragma unroll
      for (int j = 0; j < kDiaChunk; ++j) {
        const int d = d0 + j;
        if (d < nd) {
          vv[j] = __ldg(reinterpret_cast<const double2*>(dv + d * dld + r0));  // dia_ld padding is 0
          int64_t c0 = r0 + s_off[d], c1 = c0 + 1;
          c0 = c0 < 0 ? 0 : (c0 >= n ? n - 1 : c0);  // out-of-range slots hold 0.0
          c1 = c1 < 0 ? 0 : (c1 >= n ? n - 1 : c1);
          x0[j] = __ldg(x + c0);
          x1[j] = __ldg(x + c1);
        }
      }
#pragma unroll
      for (int j = 0; j < kDiaChunk; ++j) {
        if (d0 + j < nd) {
          acc0 = acc0 + vv[j].x * x0[j];
          acc1 = acc1 + vv[j].y * x1[j];
        }
      }
    }
    if (two) {
      if (TRUE_RES) {
        const double2 bv = *reinterpret_cast<const double2*>(b + r0);
        acc0 = bv.x - acc0;
        acc1 = bv.y - acc1;
      }
      *reinterpret_cast<double2*>(y + r0) = make_double2(acc0, acc1);
#pragma unroll
      for (int c = 0; c < S; ++c) part[c] = part[c] + pv[c].x * acc0 + pv[c].y * acc1;
      if (TRUE_RES) part[S] = part[S] + acc0 * acc0 + acc1 * acc1;
    } else {
      if (TRUE_RES) acc0 = b[r0] - acc0;
      y[r0] = acc0;
#pragma unroll
      for (int c = 0; c < S; ++c) part[c] = part[c] + pv[c].x * acc0;
      if (TRUE_RES) part[S] = part[S] + acc0 * acc0;
    }
  }
  __shared__ double scratch[NS * 32];
  __shared__ double blk[NS];
  __shared__ double redv[NS];
  block_totals<NS>(part, blk, scratch);
  if (!cta_commit(blk, NS, red.partials, &ds->ticket, redv)) return;
  finalize_spmv(fin, redv, ds);
}

}  // namespace

void launch_spmv_ph(cudaStream_t st, const DevCsr& a, const double* x, double* y, const double* p,
                    int64_t ld, int s, const double* b, const FinParams& fin, const Reducer& red) {
  // CSR + gathered x + y + P^H epilogue (+ b for the true-residual form)
  LaunchScope ls(st, kKSpmv, csr_bytes(a) + vbytes(a.n, 2.0 + s + (b ? 1.0 : 0.0)));
  if (a.ndiag > 0) {
    MSTAB_DISPATCH_S(s, {
      if (b) {
        auto kfn = k_spmv_dia<S, true>;
        const int grid = occupancy_grid(kfn, (a.n + 1) / 2, 0);
        kfn<<<grid, kBlock, 0, st>>>(a, x, y, p, ld, b, fin, red);
      } else {
        auto kfn = k_spmv_dia<S, false>;
        const int grid = occupancy_grid(kfn, (a.n + 1) / 2, 0);
        kfn<<<grid, kBlock, 0, st>>>(a, x, y, p, ld, b, fin, red);
      }
    });
    return;
  }
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

}  // namespace mstab_b200
