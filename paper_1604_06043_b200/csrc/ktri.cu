// ktri.cu — split preconditioning on the device (precond.cpp:23-219):
// triangular solves with the factors L, R of a SplitPreconditioner and the P^H epilogue that
// follows the preconditioned operator L^-1 A R^-1.
//
// Compiled with --fmad=false like every kernel of the cycle: each row performs exactly the
// reference's operations in the reference's order, so the solves are bit-identical to
// lower_solve / upper_solve (precond.cpp:101-133) for real data:
//   x_i = b_i;  x_i -= f_ik * x_j  for the off-diagonal entries of row i in CSR order;  x_i /= diag
// (complex products and quotients with zero imaginary parts round like the real ones).
#include <cstdlib>
#include <string>

#include "kcommon.cuh"

namespace mstab_b200 {

namespace {

constexpr int kTriRows = 32;  // consecutive rows per work item (one ticket)

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sync-free substitution, one warp per work item of kTriRows consecutive rows taken from a global
// ticket in dependency order (ascending rows for a lower factor, descending for an upper one), so
// every row a warp waits on belongs to an earlier ticket, held by a running warp: no deadlock.
// The lanes stage a row's entries, wait for each off-diagonal dependency's `done` flag
// (acquire), form the products in parallel and lane 0 applies them in CSR order.
// sync[0..n): done flags, sync[n]: ticket; zeroed (memset) before every launch.
__global__ void __launch_bounds__(kBlock) k_tri_solve(int64_t n, const int32_t* __restrict__ rp,
                                                      const int32_t* __restrict__ ci,
                                                      const double* __restrict__ val,
                                                      const double* __restrict__ b, double* x,
                                                      int lower, int* sync) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nitems = (n + kTriRows - 1) / kTriRows;
  int* done = sync;
  int* ticket = sync + n;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= nitems) break;
    const int64_t first = lower ? (int64_t)t * kTriRows : n - 1 - (int64_t)t * kTriRows;
    for (int r = 0; r < kTriRows; ++r) {
      const int64_t i = lower ? first + r : first - r;
      if (i < 0 || i >= n) break;
      const int beg = __ldg(rp + i), end = __ldg(rp + i + 1);
      double xi = __ldg(b + i);
      double diag = 0.0;
      for (int c0 = beg; c0 < end; c0 += 32) {
        const int k = c0 + lane;
        double prod = 0.0, f = 0.0;
        int64_t j = -1;
        bool dep = false;
        if (k < end) {
          j = __ldg(ci + k);
          f = __ldg(val + k);
          dep = lower ? (j < i) : (j > i);
          if (dep) {
            while (ld_acquire(done + j) == 0) {
            }
            prod = f * __ldcg(x + j);
          }
        }
        const unsigned depmask = __ballot_sync(0xffffffffu, dep);
        const unsigned dmask = __ballot_sync(0xffffffffu, k < end && j == i);
        if (dmask) diag = __shfl_sync(0xffffffffu, f, 31 - __clz(dmask));
        const int cnt = min(32, end - c0);
        for (int u = 0; u < cnt; ++u) {
          const double pu = __shfl_sync(0xffffffffu, prod, u);
          if ((depmask >> u) & 1u) xi = xi - pu;
        }
      }
      if (lane == 0) {
        __stcg(x + i, xi / diag);
        __threadfence();
        st_release(done + i, 1);
      }
      __syncwarp();
    }
  }
}

// Level-scheduled sync-free substitution (the default): the host sorts the rows by dependency
// level (solver.cpp level_schedule), so the 32 rows of a work item are mutually independent and
// each lane substitutes its own row, applying the row's products serially in CSR order — exactly
// the reference's operation order. Items are taken from a global ticket in level order, so every
// row a lane waits on belongs to an earlier item, held by a running warp: no deadlock.
// The solution vector is its own done flag: x is filled with kTriPending (an all-ones NaN pattern,
// which no division produces: the GPU's NaN results are the canonical positive quiet NaN) before
// the launch, a row's value is published with one relaxed 64-bit store, and a dependent lane polls
// the value itself — one L2 round trip per level handoff instead of flag + fence + value. The
// entries of a row are loaded and its dependencies polled in batches of 8 independent loads.
// Polling spins without a back-off by default (measured on c2: 1.64 ms per apply against 2.4 ms
// with a 32 ns __nanosleep; MSTAB_TRI_SLEEP_NS sets one) with one 256-thread CTA per SM.
constexpr unsigned long long kTriPending = 0xffffffffffffffffull;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(double* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kBlock) k_tri_levels(int64_t nslots, const int32_t* __restrict__ order,
                                                       const int32_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ b, double* x, int lower,
                                                       int* ticket, int sleep_ns) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nitems = nslots / 32;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= nitems) break;
    const int i = __ldg(order + (int64_t)t * 32 + lane);
    if (i < 0) continue;
    const int beg = __ldg(rp + i), end = __ldg(rp + i + 1);
    double xi = __ldg(b + i);
    double diag = 0.0;
    for (int k0 = beg; k0 < end; k0 += 8) {
      int jj[8];
      double ff[8];
      unsigned long long xb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool in = k0 + u < end;
        jj[u] = in ? __ldg(ci + k0 + u) : i;
        ff[u] = in ? __ldg(val + k0 + u) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool dep = lower ? jj[u] < i : jj[u] > i;
        xb[u] = dep ? ld_relaxed_u64(x + jj[u]) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool dep = lower ? jj[u] < i : jj[u] > i;
        if (dep) {
          while (xb[u] == kTriPending) {
            if (sleep_ns) __nanosleep(sleep_ns);
            xb[u] = ld_relaxed_u64(x + jj[u]);
          }
          xi = xi - ff[u] * __longlong_as_double((long long)xb[u]);
        } else if (k0 + u < end && jj[u] == i) {
          diag = ff[u];
        }
      }
    }
    unsigned long long out = (unsigned long long)__double_as_longlong(xi / diag);
    if (out == kTriPending) out = 0x7fffffffffffffffull;  // never a result; belt and braces
    st_relaxed_u64(x + i, out);
  }
}

// Diagonal factor (split Jacobi: L = R = diag(sqrt(a_ii)), precond.cpp:23-37): x = b ./ d.
__global__ void __launch_bounds__(kBlock) k_diag_solve(int64_t n, const double* __restrict__ d,
                                                       const double* __restrict__ b, double* __restrict__ x) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = b[i] / d[i];
}

// The P^H epilogue of a preconditioned apply: y = w (or the true residual y = b - w), the
// reductions P^H y (+ ||y||^2) and the same finalize_spmv tail as the fused SpMV kernels.
template <int S, bool TRUE_RES>
__global__ void __launch_bounds__(kBlock) k_ph_fin(int64_t n, const double* __restrict__ w,
                                                   double* __restrict__ y, const double* __restrict__ p,
                                                   int64_t ld, const double* __restrict__ b, FinParams fin,
                                                   Reducer red) {
  DevState* ds = red.ds;
  constexpr int NS = S + (TRUE_RES ? 1 : 0);
  double part[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) part[i] = 0.0;
  pdl_wait();
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double v = w[row];
    if (TRUE_RES) v = b[row] - v;
    y[row] = v;
#pragma unroll
    for (int c = 0; c < S; ++c) part[c] = part[c] + __ldg(p + c * ld + row) * v;
    if (TRUE_RES) part[S] = part[S] + v * v;
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

void launch_tri_solve(cudaStream_t st, const DevTri& f, const double* b, double* x, int* sync) {
  LaunchScope ls(st, kKOther, (double)f.nnz * 12.0 + vbytes(f.n, 2.0));
  if (f.diag) {
    launch_pdl(k_diag_solve, grid_for(f.n), kBlock, 0, st, f.n, (const double*)f.diag, b, x);
    return;
  }
  static const bool chain = [] {
    const char* e = std::getenv("MSTAB_TRI_SCHEDULE");
    return e && std::string(e) == "rows";
  }();
  static const int ctas_per_sm = [] {
    const char* e = std::getenv("MSTAB_TRI_CTAS_PER_SM");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  static const int sleep_ns = [] {
    const char* e = std::getenv("MSTAB_TRI_SLEEP_NS");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  if (f.order && !chain) {
    cudaMemsetAsync(x, 0xff, sizeof(double) * (size_t)f.n, st);  // every row kTriPending
    cudaMemsetAsync(sync, 0, sizeof(int), st);                     // ticket
    const int64_t nitems = f.nslots / 32;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)g_num_sms * ctas_per_sm,
                                                                 (nitems + (kBlock / 32) - 1) / (kBlock / 32)));
    launch_pdl(k_tri_levels, grid, kBlock, 0, st, f.nslots, f.order, f.rp, f.ci, f.val, b, x, f.lower ? 1 : 0, sync, sleep_ns);
    return;
  }
  cudaMemsetAsync(sync, 0, sizeof(int) * (size_t)(f.n + 1), st);
  const int grid = std::max(1, std::min(g_num_sms * 4, (int)((f.n + kTriRows * 8 - 1) / (kTriRows * 8))));
  launch_pdl(k_tri_solve, grid, kBlock, 0, st, f.n, f.rp, f.ci, f.val, b, x, f.lower ? 1 : 0, sync);
}

void launch_ph_fin(cudaStream_t st, int64_t n, int64_t ld, int s, const double* w, double* y, const double* p,
                   const double* b, const FinParams& fin, const Reducer& red) {
  LaunchScope ls(st, kKSpmv, vbytes(n, 2.0 + s + (b ? 1.0 : 0.0)));
  MSTAB_DISPATCH_S(s, {
    if (b)
      launch_pdl(k_ph_fin<S, true>, grid_for(n), kBlock, 0, st, n, w, y, p, ld, b, fin, red);
    else
      launch_pdl(k_ph_fin<S, false>, grid_for(n), kBlock, 0, st, n, w, y, p, ld, b, fin, red);
  });
}

}  // namespace mstab_b200
