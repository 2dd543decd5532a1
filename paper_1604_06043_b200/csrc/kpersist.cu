// kpersist.cu — one whole IDR(s)stab(ell) cycle as ONE cooperative kernel, for problems small enough
// that every row's share of the cycle state fits in its thread's registers (BASELINE c1: 256^2).
//
// Why: at N = 65 536 the cycle's working set (~25 vectors of 0.5 MB) is
// L2-resident and the stream-of-kernels cycle is launch-latency-bound: ~26 dependent launches of
// ~5.4 us = 140 us per cycle against a 27 us bandwidth bound. Here each thread owns ONE row of
// x, r^(0..ell), V^(-1..ell), P and b for the whole cycle, so every row-local step of the cycle
// (idrstab.cpp:105-191: BiCG updates, column rebuilds, poly combination) runs out of registers;
// the only traffic is what the algorithm cannot avoid:
//   * an SpMV input is published to a global vector and the neighbours' entries are gathered after
//     a grid barrier (CSR order: constant-diagonal form or plain CSR, bit-identical to csr.cpp:103-113);
//   * every reduction (P^H y, the least-squares Grams, the poly Gram) leaves one partial per CTA;
//     after a grid barrier EVERY CTA sums all partials in the same fixed order and runs the small
//     dense step itself (finalize_spmv / ls tails / poly_tail on a shared-memory copy of DevState),
//     so no CTA waits for another one's solve and no extra barrier broadcasts the result.
// Two grid barriers per operator application, three for the stabilisation step: 25 per cycle at
// (s, ell) = (4, 2). The element-wise arithmetic is the stream-of-kernels path's, expression for
// expression (--fmad=false), so given equal reduced values the two paths agree bit for bit; the
// reductions group rows differently (one partial per 256 rows), which teacher-forced parity covers.
// The least squares is CholeskyQR2 (kdense.cuh); if its first Cholesky factor is refused the
// kernel reports kBreakFallback and the host reruns the cycle on the stream-of-kernels path, whose
// Givens TSQR owns the ill-conditioned regime (the cycle reads set p and writes set 1 - p, so a
// rerun starts from untouched inputs).
#include <cstdio>

#include "kcommon.cuh"
#include "kdense.cuh"

namespace mstab_b200 {

namespace {

constexpr int kPBlock = 512;  // one CTA per SM: half the barrier arrivals and partials of 2 x 256

struct PersistArgs {
  DevCsr a;
  int64_t n, ld;
  const double *x_in, *r_in, *u_in, *v_in;
  double *x_out, *r_out, *u_out, *v_out;
  const double* p;
  const double* b;   // true-residual refresh (nullptr: recurrence residual)
  double* xbuf;      // n doubles: the published SpMV input
  double* partials;  // 2 x kPSlots x gridDim doubles
  DevState* ds;
  unsigned* bar;     // grid barrier counter (zeroed by the host before every launch)
  double stop_below; // residual norm at or below which the cycle ends the solve (DevState::stop)
  HostCycleSlot* hslot;  // mapped host memory: status + sequence number of this launch (or nullptr)
  unsigned long long seq;
  int debug;         // MSTAB_PERSIST_DEBUG: CTA 0 prints phase stamps of the first operator application
};

constexpr int kPSlots = 32;  // widest reduction of an instantiated (s, ell): 1 + s + s^2 = 21 at s = 4

// y_row = sum_k a_row,k x_k accumulated from +0.0 in CSR order
__device__ __forceinline__ double row_product(const DevCsr& a, const double* __restrict__ x, int64_t row) {
  double acc = 0.0;
  if (a.mask_bytes > 0) {
    const uint32_t m = a.mask_bytes == 1 ? (uint32_t) static_cast<const uint8_t*>(a.dia_mask)[row]
                                         : (a.mask_bytes == 2 ? (uint32_t) static_cast<const uint16_t*>(a.dia_mask)[row]
                                                              : static_cast<const uint32_t*>(a.dia_mask)[row]);
    // all gathers of a chunk are issued before the in-order accumulation (one entry at a time the
    // L2 round trips serialise: 0.85 us per product against 0.25 us, r02 phase stamps)
    for (int d0 = 0; d0 < a.ndiag; d0 += 8) {
      double xv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int d = d0 + j;
        xv[j] = (d < a.ndiag && ((m >> d) & 1u)) ? __ldcg(x + (row + a.off[d])) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (d0 + j < a.ndiag && ((m >> (d0 + j)) & 1u)) acc = acc + a.cval[d0 + j] * xv[j];
    }
  } else {
    const int beg = a.row_ptr[row], end = a.row_ptr[row + 1];
    for (int k0 = beg; k0 < end; k0 += 8) {
      double av[8], xv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool in = k0 + j < end;
        av[j] = in ? a.values[k0 + j] : 0.0;
        xv[j] = in ? __ldcg(x + a.col_idx[k0 + j]) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (k0 + j < end) acc = acc + av[j] * xv[j];
    }
  }
  return acc;
}

template <int S, int L, bool TRES>
__global__ void __launch_bounds__(kPBlock, 1) k_cycle(PersistArgs pa) {
  // Grid barrier: one arrival per CTA on a counter the host zeroes before the launch (monotonic
  // targets, so no reset inside the kernel), thread 0 polling with an acquire load. The
  // cooperative launch guarantees that every CTA is resident.
  unsigned bar_target = 0;
  // side(): work for the other warps while thread 0 waits (no block-wide barrier inside)
  auto grid_sync_with = [&](auto&& side) {
    __syncthreads();
    bar_target += gridDim.x;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(pa.bar) : "memory");
      unsigned seen;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(pa.bar) : "memory");
      } while (seen < bar_target);
    } else {
      side();
    }
    __syncthreads();
  };
  auto grid_sync = [&]() {
    __syncthreads();
    bar_target += gridDim.x;
    if (threadIdx.x == 0) {
      // arrival as a fire-and-forget reduction with release semantics (orders the CTA's writes before
      // it, cumulative over the __syncthreads above): unlike atomicAdd the thread does not wait for
      // the old value to come back before it starts polling, one L2 round trip less per barrier
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(pa.bar) : "memory");
      unsigned seen;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(pa.bar) : "memory");
      } while (seen < bar_target);
    }
    __syncthreads();
  };
  __shared__ DevState sds;
  __shared__ PreLU pl;
  __shared__ double scratch[32 * 32];  // block_totals: NS * 32 doubles, NS <= 32 per reduction
  __shared__ double blk[32];
  __shared__ double redv[32];
  const int t = threadIdx.x, G = gridDim.x;
  __shared__ unsigned long long stamps[24];
  int nstamp = 0;
  auto stamp = [&]() {
    if (pa.debug && blockIdx.x == 0 && t == 0 && nstamp < 24) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      stamps[nstamp] = now;
    }
    ++nstamp;
  };
  stamp();  // 0: kernel start
  const int64_t row = (int64_t)blockIdx.x * kPBlock + t;
  const bool valid = row < pa.n;
  const int64_t ld = pa.ld;
  // the device state of the solve, private to the CTA for the cycle
  {
    const double* src = reinterpret_cast<const double*>(pa.ds);
    double* dst = reinterpret_cast<double*>(&sds);
    for (int i = t; i < (int)(sizeof(DevState) / sizeof(double)); i += kPBlock) dst[i] = src[i];
  }
  __syncthreads();
  // CTA 0 hands the cycle's outcome to the host: the status head always; the dense state (P^H V,
  // P^H r, gamma_0 of the next cycle, ...) only when the cycle ran to its end, so that an early exit
  // leaves the inputs of the cycle untouched for the host's rerun.
  auto publish = [&](bool whole) {
    if (blockIdx.x == 0) {
      __syncthreads();
      const double* src = reinterpret_cast<const double*>(&sds);
      double* dst = reinterpret_cast<double*>(pa.ds);
      // the status head, or everything up to (not including) the stop flag and the counters
      const int cnt = whole ? (int)(offsetof(DevState, stop) / sizeof(double)) : (int)(sizeof(CycleStatus) / sizeof(double));
      for (int i = t; i < cnt; i += kPBlock) dst[i] = src[i];
      if (t == 0) {
        // a cycle launched behind this one must not run when this one ended the solve
        const bool stop = sds.st.breakdown != 0 || (whole && sds.st.resnorm <= pa.stop_below);
        pa.ds->stop = stop ? 1 : 0;
        if (pa.hslot) {  // the host polls seq: status first, system-wide fence, then the number
          pa.hslot->st = sds.st;
          __threadfence_system();
          pa.hslot->seq = pa.seq;
        }
      }
    }
  };
  if (sds.stop) return;  // speculative launch behind a cycle that ended the solve (uniform: see DevState::stop)
  if (sds.st.pending_singular) {  // gamma_0 of this cycle came out singular (level_update's check)
    if (t == 0) set_breakdown(&sds, kBreakSingular, 0);
    publish(false);
    return;
  }
  int parity = 0;
  // Sum of NS per-thread values over the whole grid, identical on every CTA, into redv[0..NS).
  auto grid_reduce_with = [&](auto& vals, auto ns_tag, auto&& side) {
    constexpr int NS = decltype(ns_tag)::value;
    static_assert(NS <= 32, "reduction wider than the staging arrays");
    double* part = pa.partials + (size_t)parity * kPSlots * G;
    parity ^= 1;
    block_totals<NS>(vals, blk, scratch);
    for (int i = t; i < NS; i += kPBlock) part[(size_t)i * G + blockIdx.x] = blk[i];
    stamp();  // block totals done
    grid_sync_with(side);
    stamp();  // reduction barrier passed
    const int lane = t & 31, w = t >> 5, nw = kPBlock >> 5;
    for (int i = w; i < NS; i += nw) {
      const double* p = part + (size_t)i * G;
      double acc = 0.0;
      for (int c0 = lane; c0 < G; c0 += 32 * 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = (c0 + 32 * u < G) ? __ldcg(p + c0 + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u) acc += v[u];
      }
      acc = warp_sum(acc);
      if (lane == 0) redv[i] = acc;
    }
    __syncthreads();
    stamp();  // partials summed
  };
  auto grid_reduce = [&](auto& vals, auto ns_tag) { grid_reduce_with(vals, ns_tag, [] {}); };
  // y = A v for this thread's row, v published through xbuf
  auto apply = [&](double v) -> double {
    if (valid) pa.xbuf[row] = v;
    stamp();  // published
    grid_sync();
    stamp();  // publish barrier passed
    const double y = valid ? row_product(pa.a, pa.xbuf, row) : 0.0;
    stamp();  // row product done
    return y;
  };
  // P^H y reduced over the grid, then the dense step `fin` on the CTA's own state
  double pv[S];
#pragma unroll
  for (int c = 0; c < S; ++c) pv[c] = valid ? pa.p[c * ld + row] : 0.0;
  auto ph_step = [&](double y, const FinParams& fin, double extra) {
    double part[S + 1];
#pragma unroll
    for (int c = 0; c < S; ++c) part[c] = pv[c] * y;
    part[S] = extra;
    // The known part of the step's small system is factored by warp 1 WHILE thread 0 waits at the
    // reduction barrier (kcommon.cuh, finisher protocol: the new column is taken last); after the
    // sums only that column's elimination and the substitutions remain (dense step 1.7-2.1 us ->
    // r02 stamps below).
    grid_reduce_with(part, std::integral_constant<int, S + 1>{}, [&] {
      if ((t >> 5) == 1) finisher_prepare_warp<S>(fin, &sds, pl);
    });
    finisher_finish<S>(fin, redv, &sds, pl);
    __syncthreads();
    stamp();  // dense step done
  };

  // ---- the cycle state of this row ------------------------------------------------------------
  double x = valid ? pa.x_in[row] : 0.0;
  double rl[L + 1];
  double vl[L + 2][S];  // vl[i] = V^(i-1)
  rl[0] = valid ? pa.r_in[row] : 0.0;
#pragma unroll
  for (int c = 0; c < S; ++c) {
    vl[0][c] = valid ? pa.u_in[c * ld + row] : 0.0;
    vl[1][c] = valid ? pa.v_in[c * ld + row] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < L; ++k) {
    // (a) BiCG step (idrstab.cpp:110-121): r^(i) -= V^(i) gamma for i <= k, x += V^(-1) gamma
    double gm[S];
#pragma unroll
    for (int c = 0; c < S; ++c) gm[c] = sds.gamma[k * kMaxS + c];
#pragma unroll
    for (int i = 0; i <= k; ++i) {
      double corr = 0.0;
#pragma unroll
      for (int c = 0; c < S; ++c) corr = corr + gm[c] * vl[i + 1][c];
      rl[i] = rl[i] - corr;
    }
    {
      double corr = 0.0;
#pragma unroll
      for (int c = 0; c < S; ++c) corr = corr + gm[c] * vl[0][c];
      x = x + corr;
    }
    // (b) r^(k+1) = A r^(k); rhs = P^H r^(k+1); eta_0
    rl[k + 1] = apply(rl[k]);
    FinParams fb;
    fb.op = kFinRhsEta0;
    fb.s = S;
    fb.k = k;
    fb.ell = L;
    ph_step(rl[k + 1], fb, 0.0);
    // (c) column rebuilds (idrstab.cpp:127-151), every level i = -1..k, then raise the top one
#pragma unroll
    for (int q = 0; q < S; ++q) {
      double et[S];
#pragma unroll
      for (int c = 0; c < S; ++c) et[c] = sds.eta[q * S + c];
#pragma unroll
      for (int i = -1; i <= k; ++i) {
        double nc = rl[i + 1];
#pragma unroll
        for (int c = 0; c < S; ++c) nc = nc + (-et[c]) * ((c < q) ? vl[i + 2][c] : vl[i + 1][c]);
        vl[i + 1][q] = nc;
      }
      vl[k + 2][q] = apply(vl[k + 1][q]);
      FinParams fc;
      fc.op = kFinColEta;
      fc.s = S;
      fc.k = k;
      fc.q = q;
      fc.ell = L;
      ph_step(vl[k + 2][q], fc, 0.0);
    }
  }
  // ---- poly_combination (idrstab.cpp:154-191): CholeskyQR2 least squares (kdense.cuh) ----------
  {
    constexpr int D = L + 1, NR = Tri<L>::NR;
    double z[D];
#pragma unroll
    for (int j = 0; j < L; ++j) z[j] = rl[j + 1];
    z[L] = rl[0];
    double g[NR];
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int m = j; m < D; ++m) g[Tri<L>::at(j, m)] = z[j] * z[m];
    grid_reduce(g, std::integral_constant<int, NR>{});
    if (t == 0) ls_pass1_tail<L>(redv, &sds);
    __syncthreads();
    if (sds.ls_mode != 1) {  // the Givens path owns this regime: ask the host for the other cycle
      if (t == 0 && !sds.st.breakdown) {
        sds.st.breakdown = kBreakFallback;
        sds.st.mv_at_breakdown = 0;
      }
      publish(false);
      return;
    }
    double qv[D];
#pragma unroll
    for (int m = 0; m < D; ++m) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j <= m; ++j) acc = acc + z[j] * sds.ls_r1inv[Tri<L>::at(j, m)];
      qv[m] = acc;
    }
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int m = j; m < D; ++m) g[Tri<L>::at(j, m)] = qv[j] * qv[m];
    grid_reduce(g, std::integral_constant<int, NR>{});
    if (t == 0) ls_pass2_tail<L>(redv, S, &sds);
    __syncthreads();
  }
  double rn = rl[0];
  {
    double tau[L];
#pragma unroll
    for (int i = 0; i < L; ++i) tau[i] = sds.st.tau[i];
#pragma unroll
    for (int i = 1; i <= L; ++i) {
      rn = rn + (-tau[i - 1]) * rl[i];
      x = x + tau[i - 1] * rl[i - 1];
    }
    // U_q = V^(-1)_q - sum_i tau_i V^(i-1)_q, V_q = V^(0)_q - sum_i tau_i V^(i)_q (i ascending)
    double uq[S], vq[S];
#pragma unroll
    for (int q = 0; q < S; ++q) {
      uq[q] = vl[0][q];
      vq[q] = vl[1][q];
#pragma unroll
      for (int i = 1; i <= L; ++i) {
        uq[q] = uq[q] + (-tau[i - 1]) * vl[i][q];
        vq[q] = vq[q] + (-tau[i - 1]) * vl[i + 1][q];
      }
    }
    // ||r||^2, P^H r, P^H V (column-major: entry (i, j) at i + j S) and the next cycle's gamma_0
    constexpr int NSL = 1 + S + S * S;
    double pr[NSL];
    pr[0] = rn * rn;
#pragma unroll
    for (int q = 0; q < S; ++q) pr[1 + q] = pv[q] * rn;
#pragma unroll
    for (int j = 0; j < S; ++j)
#pragma unroll
      for (int i = 0; i < S; ++i) pr[1 + S + i + j * S] = pv[i] * vq[j];
    grid_reduce(pr, std::integral_constant<int, NSL>{});
    poly_tail<S>(redv, &sds);
    __syncthreads();
    if (valid) {
#pragma unroll
      for (int q = 0; q < S; ++q) {
        pa.u_out[q * ld + row] = uq[q];
        pa.v_out[q * ld + row] = vq[q];
      }
    }
  }
  if (TRES) {  // r = b - A x (idrstab.cpp:268-273): resnorm, g, pending gamma_0 from the fixed P^H V
    const double ax = apply(x);
    rn = valid ? pa.b[row] - ax : 0.0;
    FinParams ft;
    ft.op = kFinTrueRes;
    ft.s = S;
    ft.ell = L;
    ph_step(rn, ft, rn * rn);
  }
  if (valid) {
    pa.x_out[row] = x;
    pa.r_out[row] = rn;
  }
  publish(true);
  if (pa.debug && blockIdx.x == 0 && t == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    printf("[persist] ns from start:");
    for (int i = 1; i < 24 && i < nstamp; ++i) printf(" %llu", stamps[i] - stamps[0]);
    printf(" | end %llu (stamps: state loaded+gamma update -> published, barrier, product, totals, barrier, summed, dense; repeated)\n",
           now - stamps[0]);
  }
}

template <typename K>
int coresident_ctas(K kernel) {
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(g_occ_mu);
    auto it = g_occ.find(reinterpret_cast<const void*>(kernel));
    if (it != g_occ.end()) {
      per_sm = it->second;
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kPBlock, 0);
      g_occ[reinterpret_cast<const void*>(kernel)] = per_sm;
    }
  }
  return per_sm * g_num_sms;
}

template <int S, int L>
bool launch_cycle_sl(cudaStream_t st, PersistArgs& pa, bool probe_only) {
  const bool tres = pa.b != nullptr;
  const int grid = (int)((pa.n + kPBlock - 1) / kPBlock);
  void* kfn = tres ? reinterpret_cast<void*>(k_cycle<S, L, true>) : reinterpret_cast<void*>(k_cycle<S, L, false>);
  const int cap = tres ? coresident_ctas(k_cycle<S, L, true>) : coresident_ctas(k_cycle<S, L, false>);
  if (grid > cap) return false;
  if (probe_only) return true;
  void* args[] = {&pa};
  cudaMemsetAsync(pa.bar, 0, sizeof(unsigned), st);
  cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kPBlock), args, 0, st);
  return true;
}

}  // namespace

int64_t persist_partials_doubles(int64_t n) { return 2 * (int64_t)kPSlots * ((n + kPBlock - 1) / kPBlock); }

bool launch_persist_cycle(cudaStream_t st, const DevCsr& a, int64_t n, int64_t ld, int s, int ell,
                          const double* x_in, const double* r_in, const double* u_in, const double* v_in,
                          double* x_out, double* r_out, double* u_out, double* v_out, const double* p,
                          const double* b, double* xbuf, double* partials, DevState* ds, unsigned* bar,
                          bool probe_only, double stop_below, HostCycleSlot* hslot, uint64_t seq) {
  PersistArgs pa;
  pa.stop_below = stop_below;
  pa.hslot = hslot;
  pa.seq = seq;
  pa.a = a;
  pa.n = n;
  pa.ld = ld;
  pa.x_in = x_in;
  pa.r_in = r_in;
  pa.u_in = u_in;
  pa.v_in = v_in;
  pa.x_out = x_out;
  pa.r_out = r_out;
  pa.u_out = u_out;
  pa.v_out = v_out;
  pa.p = p;
  pa.b = b;
  pa.xbuf = xbuf;
  pa.partials = partials;
  pa.ds = ds;
  pa.bar = bar;
  static const bool dbg = std::getenv("MSTAB_PERSIST_DEBUG") != nullptr;
  pa.debug = dbg ? 1 : 0;
  // cycle bytes: every state vector read and written once
  const double vecs = 2.0 * (2.0 + 2.0 * s) + s + (b ? 1.0 : 0.0);
  bool ok = false;
#define MSTAB_PERSIST_CASE(SS, LL)                                   \
  if (s == SS && ell == LL) {                                        \
    if (probe_only) return launch_cycle_sl<SS, LL>(st, pa, true);    \
    LaunchScope ls(st, kKPersistCycle, vbytes(n, vecs));             \
    ok = launch_cycle_sl<SS, LL>(st, pa, false);                     \
    return ok;                                                       \
  }
  MSTAB_PERSIST_CASE(1, 1)
  MSTAB_PERSIST_CASE(2, 1)
  MSTAB_PERSIST_CASE(4, 1)
  MSTAB_PERSIST_CASE(1, 2)
  MSTAB_PERSIST_CASE(2, 2)
  MSTAB_PERSIST_CASE(4, 2)
#undef MSTAB_PERSIST_CASE
  return false;
}

}  // namespace mstab_b200
