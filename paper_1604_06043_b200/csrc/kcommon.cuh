// kcommon.cuh — device helpers and launch plumbing shared by the kernel translation units
// (kspmv.cu, klevel.cu, kls.cu, kpoly.cu, kmisc.cu). Split per kernel family so the many
// (s, ell)-templated instantiations compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "kernels.h"
#include "ktimeline.cuh"

namespace mstab_b200 {

extern int g_num_sms;
extern std::mutex g_occ_mu;
extern std::unordered_map<const void*, int> g_occ;
void kpoly_init();

// Counts one launch; with profiling on, brackets it with CUDA events on its stream (kmisc.cu).
struct LaunchScope {
  cudaStream_t st;
  int cls;
  double bytes;
  cudaEvent_t a = nullptr;
  LaunchScope(cudaStream_t s, int c, double b);
  ~LaunchScope();
};

inline double vbytes(int64_t n, double vectors) { return 8.0 * (double)n * vectors; }
// algorithmic bytes of streaming the matrix once: CSR (int32 col + fp64 value per entry, int32
// row_ptr), the DIA slots actually used, or the presence masks of the constant-diagonal form
inline double csr_bytes(const DevCsr& a) {
  if (a.ndiag > 0 && a.mask_bytes > 0) return (double)a.mask_bytes * (double)a.n;
  if (a.ndiag > 0) return 8.0 * (double)a.ndiag * (double)a.n;
  return 12.0 * (double)a.nnz + 4.0 * (double)(a.n + 1);
}

// ---- programmatic dependent launch (PDL) ------------------------------------------------------
// Every kernel of the cycle is launched with programmatic stream serialisation: it may be
// scheduled while its predecessor is still in its reduction tail, waits (pdl_wait, before its
// first access to anything a predecessor wrote) until the predecessor has completed and flushed,
// and signals (pdl_trigger, once its own streaming phase is done) that its successor may launch.
// This hides the launch gap behind the tails; correctness is unchanged because pdl_wait is the
// full grid dependency. Without a programmatic predecessor both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

namespace {

constexpr int kSpmvStage = 384;  // CSR entries staged per warp (12 B each: 4.5 KB/warp, 36 KB/CTA)

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
                           double* red, double* xred = nullptr) {
  __shared__ int s_last;
  const int G = gridDim.x;
  for (int i = threadIdx.x; i < nslots; i += blockDim.x)
    partials[(size_t)i * G + blockIdx.x] = blk[i];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == (uint32_t)(G - 1));
  __syncthreads();
  if (!s_last) return false;
  if (threadIdx.x == 0) {
    TL_SET(6);
    TL_CLK(10);
  }
  __threadfence();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // This reduction is on the critical path of every fused dense step (the whole grid waits for
  // it): each lane issues all of its partial loads (up to 16 per batch, independent) before
  // summing them in index order, so a slot costs ~one L2 round trip instead of G/128.
  for (int i = w; i < nslots; i += nw) {
    const double* p = partials + (size_t)i * G;
    double acc = 0.0;
    for (int c0 = lane; c0 < G; c0 += 32 * 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = (c0 + 32 * u < G) ? __ldcg(p + c0 + 32 * u) : 0.0;
#pragma unroll
      for (int u = 0; u < 16; ++u) acc += v[u];
    }
    acc = warp_sum(acc);
    if (lane == 0) red[i] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0u;
  if (xred) {  // row-sharded: hand the rank-local totals to the cross-rank reduction
    for (int i = threadIdx.x; i < nslots; i += blockDim.x) xred[i] = red[i];
    return false;
  }
  return true;
}

// Dynamic tile scheduling with deterministic reductions: CTAs claim row tiles from a global
// counter (no SM idles while a slow one finishes a static share) and store each tile's partials
// at partials[slot * ntiles + tile]; the last CTA to finish sums every slot over tiles
// 0..ntiles-1 in a fixed order, so the result does not depend on which CTA ran which tile.
__device__ bool tiles_commit(int nslots, int64_t ntiles, const double* partials, uint32_t* ticket,
                             uint32_t* tile_next, double* red) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = w; i < nslots; i += nw) {
    const double* p = partials + (size_t)i * ntiles;
    double acc = 0.0;
    int64_t c = lane;
    for (; c + 224 < ntiles; c += 256) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + c + 32 * u);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; c < ntiles; c += 32) acc += __ldcg(p + c);
    acc = warp_sum(acc);
    if (lane == 0) red[i] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *ticket = 0u;
    *tile_next = 0u;
  }
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

// The same LU + solve, by one warp, column-oriented: lane j holds column j of the s x s system in
// registers (MAXS >= s). Every element sees exactly the reference's operations in the reference's
// order — pivot = first strictly larger magnitude (searched sequentially by the lane that owns
// the pivot column: no butterfly), elimination a_ij - (a_ik * inv) a_kj skipped for a zero
// multiplier, forward substitution with ascending j, backward substitution with ascending j and a
// final division — so the result is bit-identical to dev_lu_solve. The row interchange is applied
// to the right-hand side as it happens (the same permutation as rhs[perm[i]]). Per elimination
// step the only cross-lane traffic is the pivot index and the column of multipliers, so the
// dependent chain is ~s steps of a few shuffles (the earlier row-per-lane version needed an
// argmax butterfly and a row broadcast per step: ~7 us at s = 8). The substitutions run on lane 0
// from shared memory. Call with all 32 lanes; a (col-major), rhs, x live in shared memory.
// FIXED: s == MAXS at compile time (the finalisers' case: S is dispatched from s), so every size
// test folds away and the factorisation is straight-line code.
template <int MAXS, bool FIXED>
__device__ bool warp_lu_impl(int s_rt, double* a, const double* rhs, double* x) {
  constexpr unsigned FULL = 0xffffffffu;
  const int s = FIXED ? MAXS : s_rt;
  const int lane = threadIdx.x & 31;
  const bool mine = lane < s;
  double col[MAXS];
#pragma unroll
  for (int i = 0; i < MAXS; ++i) col[i] = (mine && i < s) ? a[i + lane * s] : 0.0;
  double b[MAXS];
#pragma unroll
  for (int i = 0; i < MAXS; ++i) b[i] = i < s ? rhs[i] : 0.0;
  // scale = max |a_ij| with std::max semantics (NaN never wins): order-independent
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < MAXS; ++i) mx = dmax_ref(mx, fabs(col[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = dmax_ref(mx, __shfl_xor_sync(FULL, mx, o));
  const double scale = mx;
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    if (k >= s) break;
    // pivot search on column k (lane k), rows k.. in order: first strictly larger magnitude
    int piv = k;
    double best = fabs(col[k]);
    double pval = col[k];
    if (lane == k) {
#pragma unroll
      for (int i = k + 1; i < MAXS; ++i) {
        if (i < s) {
          const double m = fabs(col[i]);
          if (m > best) {
            best = m;
            piv = i;
            pval = col[i];
          }
        }
      }
    }
    // the pivot's reciprocal (the same 1 / a_kk the reference forms after the swap) is started on
    // the pivot lane before the broadcasts, off the shuffle chain
    const double inv = 1.0 / pval;
    piv = __shfl_sync(FULL, piv, k);
    best = __shfl_sync(FULL, best, k);
    if (best < 1e-14 * scale || scale == 0.0) return false;
    if (piv != k) {  // swap rows k and piv in every column and in the right-hand side
      double ck = col[k], cp = 0.0, bp = 0.0;
#pragma unroll
      for (int i = k + 1; i < MAXS; ++i)
        if (i == piv) {
          cp = col[i];
          bp = b[i];
        }
#pragma unroll
      for (int i = k + 1; i < MAXS; ++i)
        if (i == piv) {
          col[i] = ck;
          b[i] = b[k];
        }
      col[k] = cp;
      b[k] = bp;
    }
    // multipliers m_i = a_ik * (1 / a_kk), stored in place (L), by the pivot-column lane
    if (lane == k) {
#pragma unroll
      for (int i = k + 1; i < MAXS; ++i)
        if (i < s) col[i] = col[i] * inv;
    }
    // eliminate: lanes j > k update their column with the broadcast multipliers
    const double akj = col[k];
#pragma unroll
    for (int i = k + 1; i < MAXS; ++i) {
      if (i >= s) break;
      const double mi = __shfl_sync(FULL, col[i], k);
      if (lane > k && mine && mi != 0.0) col[i] = col[i] - mi * akj;
    }
  }
  // factors back to shared memory (col-major LU), then lane 0 substitutes in the reference order
#pragma unroll
  for (int i = 0; i < MAXS; ++i)
    if (mine && i < s) a[i + lane * s] = col[i];
  __syncwarp();
  if (lane == 0) {
    double xv[MAXS];
#pragma unroll
    for (int i = 0; i < MAXS; ++i) xv[i] = b[i];
#pragma unroll
    for (int i = 1; i < MAXS; ++i) {
      if (i >= s) break;
#pragma unroll
      for (int j = 0; j < i; ++j) xv[i] = xv[i] - a[i + j * s] * xv[j];
    }
#pragma unroll
    for (int i = MAXS - 1; i >= 0; --i) {
      if (i >= s) continue;
#pragma unroll
      for (int j = i + 1; j < MAXS; ++j)
        if (j < s) xv[i] = xv[i] - a[i + j * s] * xv[j];
      xv[i] = xv[i] / a[i + i * s];
    }
#pragma unroll
    for (int i = 0; i < MAXS; ++i)
      if (i < s) x[i] = xv[i];
  }
  __syncwarp();
  return true;
}

// The fixed-size form the finalisers run (s == S at compile time). The dense step sits on the
// critical path of every SpMV of the column loop (37 per cycle at c2), executed by ONE warp, so
// what counts is that warp's instruction count and dependent chain (tools/ubench/lat.cu on sm_100a:
// DADD/DMUL/DFMA 8 cycles, 1/x 61, x/y 112; the column-per-lane form above is ~2300 SASS
// instructions at s = 8, issue-bound at ~6000 cycles, a fifth of them the selects of the row
// swaps). Here lane i holds ROW i of the system (replicated in every S-wide segment of the warp, so
// every lane computes and shuffles take a segment-local source):
//  * rows never move: each lane tracks the POSITION its row currently has in the reference's
//    swapped matrix. The pivot of step k is the un-pivoted row with the largest |a_ik|, ties to
//    the lowest position (the first strictly larger magnitude of the reference's scan), found
//    by a log-step butterfly over (magnitude, position|lane);
//  * every candidate forms its own 1 / a_ik while the butterfly runs (SIMT: one instruction
//    stream), and the winner's is broadcast: the reciprocal is off the chain;
//  * elimination a_ij - (a_ik * inv) a_kj, skipped for a zero multiplier, from the broadcast pivot
//    row; the forward substitution is fused (b_i - m b_k as the steps go: the same subtractions in
//    the same ascending-column order as x[i] -= l_ij x[j], zero multipliers included);
//  * the singular test is a flag checked once at the end (a singular system's result is unused);
//  * U and y are scattered to shared memory by position and one lane runs the backward
//    substitution, forming each quotient t / u_ii speculatively as RN(q + (t - u q) r), r = RN(1 / u_ii),
//    q = RN(t r) (3 dependent operations; r is started a row ahead), with the IEEE quotient of the
//    same t computed beside it, off the chain, and compared: a mismatch anywhere (not seen in
//    practice) reruns the substitution with plain divisions, so the result is always the
//    reference's.
// Every element sees the reference's operations in the reference's order: bit-identical to
// dev_lu_solve (tools/ubench/lu.cu checks 2000 systems per size, tests/test_gpu_kernels.py).
template <int S>
__device__ bool warp_lu_fixed(double* a, const double* rhs, double* x) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int PW = S <= 1 ? 1 : (S <= 2 ? 2 : (S <= 4 ? 4 : (S <= 8 ? 8 : 16)));
  const int lane = threadIdx.x & 31;
  const int row = lane & (PW - 1);
  const bool mine = row < S;
  double r[S];
#pragma unroll
  for (int j = 0; j < S; ++j) r[j] = mine ? a[row + j * S] : 0.0;
  double bi = mine ? rhs[row] : 0.0;
  double mx = 0.0;
#pragma unroll
  for (int j = 0; j < S; ++j) mx = dmax_ref(mx, fabs(r[j]));
#pragma unroll
  for (int o = PW / 2; o > 0; o >>= 1) mx = dmax_ref(mx, __shfl_xor_sync(FULL, mx, o));
  const double thresh = 1e-14 * mx;
  bool bad = mx == 0.0;
  int pos = row;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const bool cand = mine && pos >= k;
    double mag = cand ? fabs(r[k]) : -1.0;
    int key = ((cand ? pos : 255) << 8) | row;  // tie-break position, then the lane that holds it
    const double myinv = 1.0 / r[k];
#pragma unroll
    for (int o = PW / 2; o > 0; o >>= 1) {
      const double om = __shfl_xor_sync(FULL, mag, o);
      const int ok = __shfl_xor_sync(FULL, key, o);
      const bool take = (om > mag) || (om == mag && ok < key);
      mag = take ? om : mag;
      key = take ? ok : key;
    }
    const int piv = key >> 8, wl = key & 255;
    bad = bad || (mag < thresh);
    const double inv = __shfl_sync(FULL, myinv, wl, PW);
    const double bp = __shfl_sync(FULL, bi, wl, PW);
    pos = (row == wl) ? k : (pos == k ? piv : pos);  // the row at position k takes the winner's place
    const bool below = mine && pos > k;
    const double m = r[k] * inv;
#pragma unroll
    for (int j = k + 1; j < S; ++j) {
      const double pj = __shfl_sync(FULL, r[j], wl, PW);
      if (below && m != 0.0) r[j] = r[j] - m * pj;
    }
    if (below) bi = bi - m * bp;
  }
  if (bad) return false;  // the same on every lane
  __syncwarp();
  if (lane < PW && mine) {  // U (row `pos`, columns >= pos) and y by position
#pragma unroll
    for (int j = 0; j < S; ++j) a[pos + j * S] = r[j];
    x[pos] = bi;
  }
  __syncwarp();
  if (lane == 0) {
    // U is read from shared memory where it is used: holding it (S(S+1)/2 values) would not fit the
    // 64 registers of the streaming kernels this runs inside.
    double xv[S], y[S];
#pragma unroll
    for (int i = 0; i < S; ++i) y[i] = x[i];
    bool same = true;
    double rnext = 1.0 / a[(S - 1) + (S - 1) * S];
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      const double uii = a[i + i * S];
      const double rc = rnext;
      if (i > 0) rnext = 1.0 / a[(i - 1) + (i - 1) * S];
      double t = y[i];
#pragma unroll
      for (int j = i + 1; j < S; ++j) t = t - a[i + j * S] * xv[j];
      const double q = t * rc;
      const double rem = __fma_rn(-uii, q, t);
      const double xi = __fma_rn(rem, rc, q);
      // the reference's quotient of the same t, off the chain
      same = same && (__double_as_longlong(xi) == __double_as_longlong(t / uii));
      xv[i] = xi;
    }
    if (!same) {
#pragma unroll
      for (int i = S - 1; i >= 0; --i) {
        double t = y[i];
#pragma unroll
        for (int j = i + 1; j < S; ++j) t = t - a[i + j * S] * xv[j];
        xv[i] = t / a[i + i * S];
      }
    }
#pragma unroll
    for (int i = 0; i < S; ++i) x[i] = xv[i];
  }
  __syncwarp();
  return true;
}

template <int MAXS>
__device__ bool warp_lu_solve(int s, double* a, const double* rhs, double* x) {
  // tools/ubench/lu.cu on a B200 (cycles per nonsingular solve, column form / row form): s = 4
  // 2825 / 2864, s = 8 6250 / 6170, s = 12 14140 / 14030, s = 16 23360 / 18520; s = 3, 6: the column
  // form is 20-25% faster. Both are bit-identical to dev_lu_solve on 2000 systems per size.
  if (s == MAXS) {
    if constexpr (MAXS >= 8) return warp_lu_fixed<MAXS>(a, rhs, x);
    return warp_lu_impl<MAXS, true>(s, a, rhs, x);
  }
  return warp_lu_impl<MAXS, false>(s, a, rhs, x);
}

__device__ void set_breakdown(DevState* ds, int code, int mv) {
  if (ds->st.breakdown) return;  // the first breakdown of the cycle is the one the reference raises
  ds->st.breakdown = code;
  ds->st.mv_at_breakdown = mv;
}

// The dense step after an SpMV reduction. Its inputs that do not depend on this launch's
// reduction (the known columns of the s x s system and, for a column step, the right-hand side)
// are staged into shared memory by EVERY CTA before its ticket (fin_prestage), so the last CTA
// starts the factorisation as soon as the partials are summed instead of paying another L2
// round trip; thread 0..31 (warp_lu_solve) factor and solve, and the solution is written back
// in parallel.
struct FinStage {
  double lu[kMaxS * kMaxS];
  double vin[kMaxS], vout[kMaxS];
  int ok;
};

__device__ void fin_prestage(const FinParams& f, const DevState* ds, FinStage& fs) {
  const int s = f.s, t = threadIdx.x, nt = blockDim.x;
  if (f.op == kFinRhsEta0 || f.op == kFinTrueRes) {
    for (int i = t; i < s * s; i += nt) fs.lu[i] = ds->Ma[i];
  } else if (f.op == kFinColEta) {
    const int q = f.q;
    // msys_{q+1} = [P^H V^(k+1)_{0..q}, P^H V^(k)_{q+1..s-1}] (idrstab.cpp:133-137); column q
    // arrives with the reduction. After the last column the level's P^H V^(k+1) is all of Mn.
    for (int i = t; i < s * s; i += nt) {
      const int c = i / s;
      if (c < q)
        fs.lu[i] = ds->Mn[i];
      else if (c > q)
        fs.lu[i] = ds->Ma[i];
    }
    if (t < s) fs.vin[t] = ds->rhs[t];
  }
}

template <int MAXS>
__device__ void finalize_spmv(const FinParams& f, const double* red, DevState* ds, FinStage& fs) {
  const int s = f.s, t = threadIdx.x;
  if (f.op == kFinStore) {
    if (t < s) f.dst[t] = red[t];
    return;
  }
  double* dst = nullptr;
  int mv = 0;
  bool solve = true, pending = false;
  if (f.op == kFinRhsEta0) {  // after step (b) of level k: rhs and eta_0 (msys_0 = P^H V^(k))
    if (t < s) {
      ds->rhs[t] = red[t];
      fs.vin[t] = red[t];
    }
    dst = ds->eta;
    mv = f.k * (s + 1) + 1;
  } else if (f.op == kFinColEta) {  // after V^(k+1)_q = A v_q^(k)
    const int q = f.q, k = f.k;
    if (t < s) {
      ds->Mn[t + q * s] = red[t];
      fs.lu[t + q * s] = red[t];
    }
    if (q + 1 < s) {
      dst = ds->eta + (q + 1) * s;
      mv = k * (s + 1) + 1 + (q + 1);
    } else {
      // level done: Ma := P^H V^(k+1), g := P^H r^(k+1); gamma of level k+1 unless it is the last
      __syncthreads();
      for (int i = t; i < s * s; i += blockDim.x) ds->Ma[i] = fs.lu[i];
      if (t < s) ds->g[t] = fs.vin[t];
      if (k + 1 < f.ell) {
        dst = ds->gamma + (k + 1) * kMaxS;
        mv = (k + 1) * (s + 1);
      } else {
        solve = false;
      }
    }
  } else if (f.op == kFinTrueRes) {  // r = b - A x: resnorm, g, pending gamma_0
    if (t == 0) ds->st.resnorm = sqrt(red[s]);
    if (t < s) {
      ds->g[t] = red[t];
      fs.vin[t] = red[t];
    }
    dst = ds->gamma;
    pending = true;
  } else {
    return;
  }
  __syncthreads();
  if (!solve) return;
  if (t < 32) {
    const bool r = warp_lu_solve<MAXS>(s, fs.lu, fs.vin, fs.vout);
    if (t == 0) {
      fs.ok = r ? 1 : 0;
      TL_SET(8);
      TL_CLK(12);
    }
  }
  __syncthreads();
  if (t < s) dst[t] = fs.vout[t];
  if (t == 0) {
    if (pending)
      ds->st.pending_singular = fs.ok ? 0 : 1;
    else if (!fs.ok)
      set_breakdown(ds, kBreakSingular, mv);
  }
}

// ---- finisher protocol (kcdia.cu) ---------------------------------------------------------------
// The dense step after an SpMV reduction sits on the critical path of the column loop (37 SpMVs per
// cycle at c2). With the last-CTA scheme above that tail was ~8 us of a 34 us launch (r02 timeline:
// store fence + ticket 2.2 us, partial sums 1.3 us, s x s LU 4.3 us). Here CTA 0 of the grid streams
// no rows. While the others stream it factors everything of the small system that is already known
// (fin_prefactor), then polls the partial slots (an empty slot holds an all-ones NaN, so a partial is
// published by ONE relaxed store: no fence, no ticket), sums them in index order, and only forward-
// eliminates the ONE new column (or right-hand side) and back-substitutes (fin_finish).
//
// Which part is known early: after the SpMV of column q the system is msys_{q+1} = [P^H V^(k+1)_{0..q},
// P^H V^(k)_{q+1..s-1}] (idrstab.cpp:133-137) and only column q is new; the right-hand side P^H r^(k+1)
// is known since step (b). The finisher factors the s-1 known columns with partial pivoting, taking
// the new column LAST: for q = s-1 this is exactly the reference's LuFactor (kernels.cpp:95-127), for
// q < s-1 it is the same Gaussian elimination on a column-permuted system (the solution's entries are
// permuted back), equally stable but rounded differently at the 1e-16 level, like the tree reductions.
// After step (b) and after the true-residual product the matrix is fully known and only the right-
// hand side is new: the factorisation and both substitutions are the reference's, bit for bit.
constexpr unsigned long long kSlotEmpty = 0xffffffffffffffffull;

__device__ __forceinline__ double slot_load(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void slot_store(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// a streaming CTA's totals -> its slots (never the empty pattern: a NaN total is canonicalised)
__device__ __forceinline__ void slots_publish(const double* blk, int nslots, double* slots) {
  if ((int)threadIdx.x < nslots) {
    double v = blk[threadIdx.x];
    if (v != v) v = __longlong_as_double(0x7ff8000000000000ll);
    slot_store(slots + (size_t)threadIdx.x * gridDim.x + blockIdx.x, v);
  }
}
// finisher CTA: waits for the slots of CTAs 1..G-1, sums each value over the CTAs in a fixed order
// (per lane ascending, then the warp butterfly: the order cta_commit uses) and empties the slots.
__device__ void slots_collect(int nslots, double* slots, double* red) {
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = w; i < nslots; i += nw) {
    double* p = slots + (size_t)i * G;
    double acc = 0.0;
    // The sums are formed inside the poll loop, on every pass: when the last partial lands, the
    // instructions that consume it are already in the instruction cache (see fin_finish).
    double tot = 0.0;
    for (int cb = 1; cb < G; cb += 32 * 16) {  // warp-uniform trip count (the poll loop votes)
      const int c0 = cb + lane;
      double v[16];
      double part;
      bool all;
      do {
        all = true;
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = (c0 + 32 * u < G) ? slot_load(p + c0 + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u) all = all && ((unsigned long long)__double_as_longlong(v[u]) != kSlotEmpty);
        part = acc;
#pragma unroll
        for (int u = 0; u < 16; ++u) part += v[u];
        tot = warp_sum(part);
        all = __all_sync(0xffffffffu, all);
      } while (!all);
      acc = part;
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (c0 + 32 * u < G) slot_store(p + c0 + 32 * u, __longlong_as_double((long long)kSlotEmpty));
    }
    if (lane == 0) red[i] = tot;
  }
}

struct PreLU {
  double lu[kMaxS * kMaxS];  // in: the columns to factor (column-major, ld = s); out: L \ U by position
  double y[kMaxS];           // column mode: in the right-hand side, out L^-1 (perm rhs)
  double rinv[kMaxS];        // reciprocals of the pivots
  double mx, minpiv;         // max |entry| of the factored columns; smallest pivot magnitude
  int perm[kMaxS];           // perm[position] = original row
  int nc;                    // factored columns: s (right-hand-side mode) or s - 1 (column mode)
  int solve;                 // 0: this step has no solve
  double warm[kMaxS];        // landing area of the warm-up run of fin_finish
};

// One warp: partially pivoted LU of the first nc columns of the s x s system in f.lu (lane i holds
// row i, replicated in every PW-wide segment; the structure of warp_lu_fixed: pivot = largest
// magnitude, ties to the lowest position = the reference's first strictly larger scan; multipliers
// a_ik * (1 / a_kk); elimination skipped for a zero multiplier). With with_rhs the right-hand side
// in f.y is eliminated along. Rows never move: each lane tracks its row's position and the factors
// are scattered by position at the end (multipliers travel with their row, like the reference's
// full-row swaps).
template <int S>
__device__ void fin_prefactor(PreLU& f, int nc, bool with_rhs) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int PW = S <= 1 ? 1 : (S <= 2 ? 2 : (S <= 4 ? 4 : (S <= 8 ? 8 : 16)));
  const int lane = threadIdx.x & 31;
  const int row = lane & (PW - 1);
  const bool mine = row < S;
  double r[S];
#pragma unroll
  for (int j = 0; j < S; ++j) r[j] = (mine && j < nc) ? f.lu[row + j * S] : 0.0;
  double bi = (mine && with_rhs) ? f.y[row] : 0.0;
  double mx = 0.0;
#pragma unroll
  for (int j = 0; j < S; ++j) mx = dmax_ref(mx, fabs(r[j]));
#pragma unroll
  for (int o = PW / 2; o > 0; o >>= 1) mx = dmax_ref(mx, __shfl_xor_sync(FULL, mx, o));
  double minpiv = __longlong_as_double(0x7ff0000000000000ll);
  double myrinv = 0.0;
  int pos = row;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < S; ++k) {
    if (k >= nc) break;
    const bool cand = mine && pos >= k;
    double mag = cand ? fabs(r[k]) : -1.0;
    int key = ((cand ? pos : 255) << 8) | row;
    const double myinv = 1.0 / r[k];
#pragma unroll
    for (int o = PW / 2; o > 0; o >>= 1) {
      const double om = __shfl_xor_sync(FULL, mag, o);
      const int ok = __shfl_xor_sync(FULL, key, o);
      const bool take = (om > mag) || (om == mag && ok < key);
      mag = take ? om : mag;
      key = take ? ok : key;
    }
    const int piv = key >> 8, wl = key & 255;
    minpiv = (mag < minpiv) ? mag : minpiv;
    const double inv = __shfl_sync(FULL, myinv, wl, PW);
    const double bp = __shfl_sync(FULL, bi, wl, PW);
    pos = (row == wl) ? k : (pos == k ? piv : pos);
    if (row == wl) myrinv = inv;
    const bool below = mine && pos > k;
    const double m = r[k] * inv;
#pragma unroll
    for (int j = k + 1; j < S; ++j) {
      const double pj = __shfl_sync(FULL, r[j], wl, PW);
      if (below && m != 0.0 && j < nc) r[j] = r[j] - m * pj;
    }
    if (below) {
      bi = bi - m * bp;
      r[k] = m;
    }
  }
  __syncwarp();
  if (lane < PW && mine) {
#pragma unroll
    for (int j = 0; j < S; ++j) f.lu[pos + j * S] = r[j];
    f.y[pos] = bi;
    f.perm[pos] = row;
    f.rinv[pos] = myrinv;
  }
  if (lane == 0) {
    f.mx = mx;
    f.minpiv = minpiv;
    f.nc = nc;
  }
  __syncwarp();
}

// quotient t / u on the dependent chain as RN(q + (t - u q) rc), q = RN(t rc), rc = RN(1 / u): three
// dependent operations instead of a 112-cycle division. With a correctly rounded rc this is the
// IEEE quotient except in rare last-bit cases; nothing downstream is compared bit for bit with
// the reference (the system's entries come from tree reductions).
__device__ __forceinline__ double quot_chain(double t, double u, double rc) {
  const double q = t * rc;
  const double rem = __fma_rn(-u, q, t);
  return __fma_rn(rem, rc, q);
}

// One warp (lane i = position i, replicated in PW-wide segments) finishes the solve with the new
// vector v (original row order) and writes the unknowns to dst. The loops are rolled on purpose:
// this code runs once per launch, from a cold instruction cache, on the critical path of the
// column loop: the finisher runs it once on dummy data right after the factorisation
// (finisher_prepare), so the instructions are in the SM's instruction cache when the partials
// arrive. Cold, every instruction line costs an L2 round trip at the loaded latency of ~1 us: the
// straight-line single-thread form measured 5400 cycles and this one 7000 (r02 timeline), against
// ~1300 warm. Hence __noinline__: both calls must run the same instructions.
//  * column mode (f.nc == S - 1): v is the last column of the factored order. It goes through the
//    S - 1 elimination steps (zero multipliers skipped, like LuFactor), its last entry is the last
//    pivot, then the back-substitution runs. Unknown j of the factored order is written to
//    dst[colmap(j)].
//  * right-hand-side mode (f.nc == S): forward substitution (ascending j, LuFactor::solve), then
//    the back-substitution.
// The back-substitution subtracts u_ij x_j in the order the unknowns become available (j
// descending; the reference's loop subtracts them ascending): the same terms, rounded in another
// order. Returns false (on every lane) when the reference's pivot test fails; dst is written
// either way (a failed solve's values are never used).
template <int S>
__device__ __noinline__ bool fin_finish(const PreLU& f, const double* v, double* dst, int q) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int PW = S <= 1 ? 1 : (S <= 2 ? 2 : (S <= 4 ? 4 : (S <= 8 ? 8 : 16)));
  const int lane = threadIdx.x & 31;
  const int i = lane & (PW - 1);
  const bool mine = i < S;
  const bool colmode = f.nc == S - 1;
  double w = mine ? v[f.perm[mine ? i : 0]] : 0.0;
  double vmax = mine ? fabs(v[mine ? i : 0]) : 0.0;
#pragma unroll
  for (int o = PW / 2; o > 0; o >>= 1) vmax = dmax_ref(vmax, __shfl_xor_sync(FULL, vmax, o));
  const double yi = f.y[i];
  const double ylast = f.y[S - 1];
  double lnext = f.lu[i];
#pragma unroll 1
  for (int k = 0; k < S - 1; ++k) {
    const double l = lnext;
    lnext = f.lu[i + (k + 1) * S];
    const double wk = __shfl_sync(FULL, w, k, PW);
    if (i > k && (!colmode || l != 0.0)) w = w - l * wk;
  }
  bool ok;
  double t;
  int jstart;
  if (colmode) {
    const double scale = dmax_ref(f.mx, vmax);
    const double upiv = __shfl_sync(FULL, w, S - 1, PW);
    const double lastmag = fabs(upiv);
    const double minpiv = (lastmag < f.minpiv) ? lastmag : f.minpiv;
    ok = !(minpiv < 1e-14 * scale || scale == 0.0);
    const double xl = ylast / upiv;  // every lane forms it: no broadcast on the chain
    t = (i == S - 1) ? xl : yi - w * xl;
    jstart = S - 2;
  } else {
    ok = !(f.minpiv < 1e-14 * f.mx || f.mx == 0.0);
    t = w;
    jstart = S - 1;
  }
  {
    double unext = f.lu[i + (jstart < 0 ? 0 : jstart) * S];
#pragma unroll 1
    for (int j = jstart; j >= 0; --j) {
      const double u = unext;
      if (j > 0) unext = f.lu[i + (j - 1) * S];
      const double xq = quot_chain(t, u, f.rinv[j]);  // lane j: t_j / u_jj
      if (i == j) t = xq;
      const double xj = __shfl_sync(FULL, xq, j, PW);
      if (i < j) t = t - u * xj;
    }
  }
  if (lane < PW && mine) {
    int c = i;
    if (colmode) c = i < q ? i : (i == S - 1 ? q : i + 1);
    dst[c] = t;
  }
  return ok;
}

// Finisher CTA, before the partials arrive: stages what the step's small system already has and
// factors it (warp 0). Everything read here was written by kernels that completed before this
// launch's pdl_wait returned.
template <int S>
__device__ void finisher_prepare(const FinParams& f, DevState* ds, PreLU& pl) {
  const int t = threadIdx.x, nt = blockDim.x;
  int nc = 0;
  bool with_rhs = false, solve = false;
  if (f.op == kFinRhsEta0 || f.op == kFinTrueRes) {
    for (int i = t; i < S * S; i += nt) pl.lu[i] = ds->Ma[i];
    nc = S;
    solve = true;
  } else if (f.op == kFinColEta) {
    const int q = f.q;
    // factored column j < S - 1 is column j (j < q: P^H V^(k+1)_j) or j + 1 (P^H V^(k)_{j+1})
    for (int i = t; i < S * (S - 1); i += nt) {
      const int j = i / S, rw = i - j * S;
      pl.lu[i] = j < q ? ds->Mn[rw + j * S] : ds->Ma[rw + (j + 1) * S];
    }
    if (t < S) pl.y[t] = ds->rhs[t];
    nc = S - 1;
    with_rhs = true;
    solve = (q + 1 < S) || (f.k + 1 < f.ell);
  }
  __syncthreads();
  if (f.op == kFinColEta && f.q + 1 == S) {
    // level done: Ma := P^H V^(k+1) (its last column arrives with the reduction), g := P^H r^(k+1)
    for (int i = t; i < S * (S - 1); i += nt) ds->Ma[i] = ds->Mn[i];
    if (t < S) ds->g[t] = ds->rhs[t];
  }
  if (t == 0) pl.solve = solve ? 1 : 0;
  if (t < 32 && solve) {
    fin_prefactor<S>(pl, nc, with_rhs);
    fin_finish<S>(pl, pl.y, pl.warm, f.q);  // instruction-cache warm-up, result unused
  }
}

// The same preparation by ONE warp with no block-wide barrier (the persistent cycle kernel runs it
// on warp 1 while thread 0 polls the grid barrier; `ds` is then the CTA's shared-memory copy of the
// state, which no other warp touches during the wait).
template <int S>
__device__ void finisher_prepare_warp(const FinParams& f, DevState* ds, PreLU& pl) {
  const int lane = threadIdx.x & 31;
  int nc = 0;
  bool with_rhs = false, solve = false;
  if (f.op == kFinRhsEta0 || f.op == kFinTrueRes) {
    for (int i = lane; i < S * S; i += 32) pl.lu[i] = ds->Ma[i];
    nc = S;
    solve = true;
  } else if (f.op == kFinColEta) {
    const int q = f.q;
    for (int i = lane; i < S * (S - 1); i += 32) {
      const int j = i / S, rw = i - j * S;
      pl.lu[i] = j < q ? ds->Mn[rw + j * S] : ds->Ma[rw + (j + 1) * S];
    }
    if (lane < S) pl.y[lane] = ds->rhs[lane];
    nc = S - 1;
    with_rhs = true;
    solve = (q + 1 < S) || (f.k + 1 < f.ell);
  }
  __syncwarp();
  if (f.op == kFinColEta && f.q + 1 == S) {
    for (int i = lane; i < S * (S - 1); i += 32) ds->Ma[i] = ds->Mn[i];
    if (lane < S) ds->g[lane] = ds->rhs[lane];
  }
  if (lane == 0) pl.solve = solve ? 1 : 0;
  __syncwarp();
  if (solve) fin_prefactor<S>(pl, nc, with_rhs);
}

// Finisher CTA, after slots_collect (and a __syncthreads): the bookkeeping of finalize_spmv, and
// warp 0 finishes the solve.
template <int S>
__device__ void finisher_finish(const FinParams& f, const double* red, DevState* ds, PreLU& pl) {
  const int t = threadIdx.x;
  if (f.op == kFinStore) {
    if (t < S) f.dst[t] = red[t];
    return;
  }
  double* dst = nullptr;
  int mv = 0;
  bool pending = false;
  const int q = f.q, k = f.k;
  if (f.op == kFinRhsEta0) {
    if (t >= 32 && t < 32 + S) ds->rhs[t - 32] = red[t - 32];
    dst = ds->eta;
    mv = k * (S + 1) + 1;
  } else if (f.op == kFinColEta) {
    if (t >= 32 && t < 32 + S) {
      ds->Mn[t - 32 + q * S] = red[t - 32];
      if (q + 1 == S) ds->Ma[t - 32 + q * S] = red[t - 32];
    }
    if (q + 1 < S) {
      dst = ds->eta + (q + 1) * S;
      mv = k * (S + 1) + 1 + (q + 1);
    } else {
      dst = ds->gamma + (k + 1) * kMaxS;
      mv = (k + 1) * (S + 1);
    }
  } else if (f.op == kFinTrueRes) {
    if (t == 32) ds->st.resnorm = sqrt(red[S]);
    if (t >= 32 && t < 32 + S) ds->g[t - 32] = red[t - 32];
    dst = ds->gamma;
    pending = true;
  } else {
    return;
  }
  if (!pl.solve || t >= 32) return;
  const bool ok = fin_finish<S>(pl, red, dst, q);
  if (t == 0) {
    TL_SET(8);
    TL_CLK(12);
    if (pending)
      ds->st.pending_singular = ok ? 0 : 1;
    else if (!ok)
      set_breakdown(ds, kBreakSingular, mv);
  }
}

// Resident CTAs per SM of each kernel, queried once (the occupancy API costs tens of us per
// call, which would starve the GPU between launches).

template <typename K>
int occupancy_grid(K kernel, int64_t n, size_t dyn_smem, int block = kBlock) {
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(g_occ_mu);
    auto it = g_occ.find(reinterpret_cast<const void*>(kernel));
    if (it != g_occ.end()) {
      per_sm = it->second;
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, dyn_smem);
      if (per_sm < 1) per_sm = 1;
      g_occ[reinterpret_cast<const void*>(kernel)] = per_sm;
    }
  }
  int64_t want = (n + block - 1) / block;
  int64_t cap = (int64_t)g_num_sms * per_sm;
  if (cap > kMaxGrid) cap = kMaxGrid;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
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

}  // namespace mstab_b200
