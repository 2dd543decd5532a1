// kcdia.cu — SpMV on the constant-diagonal (stencil) operator form with the fused P^H epilogue.
// Split from kspmv.cu so the 96 instantiations (S x true-residual x mask width) build in parallel.
// Compiled with --fmad=false like every kernel of the cycle (bit-exact element-wise arithmetic).
#include <type_traits>

#include "kcommon.cuh"
#include "ktimeline.cuh"

namespace mstab_b200 {

namespace {

// SpMV on the constant-diagonal form (kernels.h DevCsr::cval / dia_mask): the only matrix
// bytes streamed are the per-row presence masks (mask_bytes per row instead of 8 per diagonal),
// the diagonal values come from the parameter bank. A term is taken only where its presence
// bit is set — exactly the CSR terms in CSR order (offsets ascend) — so the result is
// bit-identical to csr.cpp:103-113: an absent term's gather is predicated off and contributes
// cval * (+0.0) = ±0.0, which leaves the accumulator unchanged (it starts at +0.0 and a
// round-to-nearest sum never produces -0.0 from it; the upload requires finite cval).
//
// ncu on the first versions (c5, s=1): DRAM 24%, issue slots 63% busy, ~250 warp instructions
// per row — instruction-bound, not memory-bound. So the stencil width ND is a template
// parameter: the diagonal loop unrolls completely, each coefficient is a constant-bank operand
// of its DMUL, the presence bits become predicates, and a gather is one 32-bit add, one wide
// address multiply and one predicated load. ND = 0 is the generic (runtime nd) fallback.
template <int ND>
struct MaskOf {
  using T = typename std::conditional<(ND <= 8), uint8_t,
                                      typename std::conditional<(ND <= 16), uint16_t, uint32_t>::type>::type;
};

// 512-thread CTAs, two per SM: the same 32 warps per SM as 4 x 256, but half the per-CTA partials.
// CTA 0 is the finisher (kcommon.cuh, finisher protocol): it streams no rows; CTAs 1..G-1 split the
// rows grid-stride and publish their partial sums through the sentinel slots.
constexpr int kCdiaBlock = 512;

// SEL: the launch covers a row selection (DevCsr::sel_*: the interior or the boundary rows of a row
// slab). A template parameter because the streaming loop is instruction- and register-bound: with
// the selection tested at run time the c2 kernel went from 30.2 to 36.5 us.
template <int S, bool TRUE_RES, int ND, bool SEL>
__global__ void __launch_bounds__(kCdiaBlock, S <= 8 ? 2 : 1)
    k_spmv_cdia(DevCsr a, const double* __restrict__ x, double* __restrict__ y,
                const double* __restrict__ p, int64_t ld, const double* __restrict__ b,
                FinParams fin, Reducer red) {
  DevState* ds = red.ds;
  constexpr int NS = S + (TRUE_RES ? 1 : 0);
  __shared__ double scratch[NS * 32];  // block_totals: up to 32 warps
  __shared__ double blk[NS];
  if (blockIdx.x == 0) {
    // ---- finisher CTA ----
    __shared__ PreLU pl;
    if (threadIdx.x == 0) {
      TL_MIN(0);
      TL_MAX(1);
    }
    pdl_wait();
    pdl_trigger();
    if (!red.xred) finisher_prepare<S>(fin, ds, pl);
    slots_collect(NS, red.slots, blk);
    __syncthreads();
    if (threadIdx.x == 0) {
      TL_SET(7);
      TL_CLK(11);
    }
    if (red.xred) {  // row-sharded: the rank-local totals go to the cross-rank reduction
      if (threadIdx.x < NS)
        red.xred[threadIdx.x] = red.xbase ? red.xbase[threadIdx.x] + blk[threadIdx.x] : blk[threadIdx.x];
      return;
    }
    finisher_finish<S>(fin, blk, ds, pl);
    if (threadIdx.x == 0) {
      TL_SET(9);
      TL_CLK(13);
    }
    return;
  }
  const int64_t n = a.n;
  const int nd = ND > 0 ? ND : a.ndiag;
  const int mb = a.mask_bytes;
  double part[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) part[i] = 0.0;
  // The gathers of a row are predicated on its mask, so the mask is loaded one iteration ahead
  // (the first measured version waited for it: two dependent memory latencies per row).
  // row selection (DevCsr::sel_*): virtual index v -> row
  const int32_t na = SEL ? a.sel_a1 - a.sel_a0 : 0, nb = SEL ? a.sel_b1 - a.sel_b0 : 0;
  const int32_t nv = SEL ? na + nb : (int32_t)n;
  auto row_of = [&](int32_t v) -> int32_t { return !SEL ? v : (v < na ? a.sel_a0 + v : a.sel_b0 + (v - na)); };
  auto load_mask = [&](int32_t v) -> uint32_t {
    if (v >= nv) return 0u;
    const int32_t r = row_of(v);
    if (ND > 0) return (uint32_t)__ldg(static_cast<const typename MaskOf<ND>::T*>(a.dia_mask) + r);
    return mb == 1 ? (uint32_t)__ldg(static_cast<const uint8_t*>(a.dia_mask) + r)
                   : (mb == 2 ? (uint32_t)__ldg(static_cast<const uint16_t*>(a.dia_mask) + r)
                              : __ldg(static_cast<const uint32_t*>(a.dia_mask) + r));
  };
  const int32_t rstride = (gridDim.x - 1) * blockDim.x;
  const int32_t v0 = (blockIdx.x - 1) * blockDim.x + threadIdx.x;
  const int32_t row0 = v0 < nv ? row_of(v0) : (int32_t)n;
  // The masks never change and, inside a cycle, neither do P and b: the first row's mask, P row
  // and b are loaded before waiting on the producer of x (programmatic dependent launch), so that
  // DRAM round trip overlaps the predecessor's tail. A plain product (kFinStore) may pass a
  // producer-written vector as p, so it loads after the wait.
  const bool early = fin.op != kFinStore;
  if (threadIdx.x == 0) {
    TL_MIN(0);
    TL_MAX(1);
  }
  uint32_t mnext = load_mask(v0);
  double pv[S];
  double bv = 0.0;
  if (early && row0 < (int32_t)n) {
#pragma unroll
    for (int c = 0; c < S; ++c) pv[c] = __ldg(p + c * ld + row0);
    if (TRUE_RES) bv = __ldg(b + row0);
  }
  pdl_wait();
  if (threadIdx.x == 0) {
    TL_MIN(2);
    TL_MAX(3);
  }
  bool first = early;
  for (int32_t v = v0; v < nv; v += rstride) {
    const int32_t row = row_of(v);
    const uint32_t m = mnext;
    mnext = load_mask(v + rstride);
    if (!first) {
#pragma unroll
      for (int c = 0; c < S; ++c) pv[c] = __ldg(p + c * ld + row);
      if (TRUE_RES) bv = __ldg(b + row);
    }
    first = false;
    double acc = 0.0;
    if (ND > 0) {
      double xv[ND > 0 ? ND : 1];
#pragma unroll
      for (int d = 0; d < ND; ++d) xv[d] = ((m >> d) & 1u) ? __ldg(x + (row + a.off[d])) : 0.0;
#pragma unroll
      for (int d = 0; d < ND; ++d) acc = acc + a.cval[d] * xv[d];
    } else {
      for (int d0 = 0; d0 < nd; d0 += 8) {
        double xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int d = d0 + j;
          xv[j] = (d < nd && ((m >> d) & 1u)) ? __ldg(x + (row + a.off[d])) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (d0 + j < nd) acc = acc + a.cval[d0 + j] * xv[j];
      }
    }
    if (TRUE_RES) acc = bv - acc;
    y[row] = acc;
#pragma unroll
    for (int c = 0; c < S; ++c) part[c] = part[c] + pv[c] * acc;
    if (TRUE_RES) part[S] = part[S] + acc * acc;
  }
  pdl_trigger();
  block_totals<NS>(part, blk, scratch);
  slots_publish(blk, NS, red.slots);
  if (threadIdx.x == 0) {
    TL_MIN(4);
    TL_MAX(5);
  }
}

}  // namespace
TL_BIND_FN(kcdia_timeline_bind)
namespace {

template <int S, bool TRUE_RES, int ND, bool SEL = false>
void launch_cdia_nd(cudaStream_t st, const DevCsr& a, const double* x, double* y, const double* p,
                    int64_t ld, const double* b, const FinParams& fin, const Reducer& red) {
  auto kfn = k_spmv_cdia<S, TRUE_RES, ND, SEL>;
  // the resident capacity minus the finisher streams; one more CTA (index 0) finishes
  const int64_t rows = (a.sel_a1 | a.sel_b1) ? (int64_t)(a.sel_a1 - a.sel_a0) + (a.sel_b1 - a.sel_b0) : a.n;
  int grid = occupancy_grid(kfn, rows + kCdiaBlock, 0, kCdiaBlock);
  if (grid < 2) grid = 2;
  launch_pdl(kfn, grid, kCdiaBlock, 0, st, a, x, y, p, ld, b, fin, red);
}

// Specialised stencil widths: 5 (2-D 5-point: c1), 7 (3-D 7-point: c2, c5), 27 (27-point: c4).
template <int S, bool TRUE_RES>
void launch_cdia_b(cudaStream_t st, const DevCsr& a, const double* x, double* y, const double* p,
                   int64_t ld, const double* b, const FinParams& fin, const Reducer& red) {
  if (a.sel_a1 | a.sel_b1) {  // split product of a row slab: 3-D stencils specialised, the rest generic
    switch (a.ndiag) {
      case 7: launch_cdia_nd<S, TRUE_RES, 7, true>(st, a, x, y, p, ld, b, fin, red); break;
      case 27: launch_cdia_nd<S, TRUE_RES, 27, true>(st, a, x, y, p, ld, b, fin, red); break;
      default: launch_cdia_nd<S, TRUE_RES, 0, true>(st, a, x, y, p, ld, b, fin, red); break;
    }
    return;
  }
  switch (a.ndiag) {
    case 5: launch_cdia_nd<S, TRUE_RES, 5>(st, a, x, y, p, ld, b, fin, red); break;
    case 7: launch_cdia_nd<S, TRUE_RES, 7>(st, a, x, y, p, ld, b, fin, red); break;
    case 27: launch_cdia_nd<S, TRUE_RES, 27>(st, a, x, y, p, ld, b, fin, red); break;
    default: launch_cdia_nd<S, TRUE_RES, 0>(st, a, x, y, p, ld, b, fin, red); break;
  }
}

template <int S>
void launch_cdia(cudaStream_t st, const DevCsr& a, const double* x, double* y, const double* p,
                 int64_t ld, const double* b, const FinParams& fin, const Reducer& red) {
  if (b)
    launch_cdia_b<S, true>(st, a, x, y, p, ld, b, fin, red);
  else
    launch_cdia_b<S, false>(st, a, x, y, p, ld, b, fin, red);
}

}  // namespace

void launch_spmv_cdia(cudaStream_t st, const DevCsr& a, const double* x, double* y, const double* p,
                      int64_t ld, int s, const double* b, const FinParams& fin, const Reducer& red) {
  MSTAB_DISPATCH_S(s, { launch_cdia<S>(st, a, x, y, p, ld, b, fin, red); });
}

}  // namespace mstab_b200
