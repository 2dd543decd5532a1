// kernels.h — host-callable launchers for the sm_100a kernels in kernels.cu.
//
// Every launcher enqueues on `stream` and never synchronises. Reductions are deterministic:
// per-CTA partials in a fixed order, then the last CTA to finish (ticket counter) reduces all
// partials in a fixed order and runs the small dense step that follows (LU solve, LS solve),
// so no extra kernel and no host round trip sits between a reduction and its consumer.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdlib>

#include "device_state.h"

#include <vector>

typedef struct CUstream_st* cudaStream_t;
typedef struct CUevent_st* cudaEvent_t;

namespace mstab_b200 {

struct DevCsr {
  int64_t n = 0;
  int64_t nnz = 0;
  const int32_t* row_ptr = nullptr;  // n + 1
  const int32_t* col_idx = nullptr;  // nnz (+ padding)
  const double* values = nullptr;    // nnz (+ padding)
  // Optional diagonal (DIA) form chosen at upload when the nonzeros lie on few diagonals
  // (stencils): dia_val[d * dia_ld + row] holds A(row, row + dia_off[d]) (0 where CSR has no
  // entry), offsets ascending, so accumulating d = 0.. is CSR column order.
  int32_t ndiag = 0;
  int64_t dia_ld = 0;
  const double* dia_val = nullptr;
  const int32_t* dia_off = nullptr;
  int32_t off[64] = {};  // the offsets again, by value: kernels read them from the parameter bank
  // Constant-diagonal (stencil) form, chosen at upload when every diagonal holds ONE value
  // (constant-coefficient stencils: c1, c2, c4, c5): cval[d] is that value and dia_mask holds one
  // presence bit per diagonal per row (mask_bytes = 1, 2 or 4 bytes per row, rows padded to
  // dia_ld). A cleared bit means CSR has no entry there (dropped boundary neighbour), so the row
  // accumulates exactly the CSR terms in CSR order. dia_val is unused (nullptr) in this form.
  int32_t mask_bytes = 0;
  const void* dia_mask = nullptr;
  double cval[32] = {};
  // Valid index range [xlo, xhi) of the x vector the SpMV reads: [0, n) on one GPU; in a
  // row-sharded solve the owned rows plus the halo on either side (negative xlo).
  int64_t xlo = 0, xhi = 0;
  // Column band of the stored entries: blo <= col - row <= bhi for every entry (0, 0 when empty).
  // A narrow band lets the CSR SpMV keep a sliding x window in shared memory (kspmv.cu k_spmv_ring).
  int64_t blo = 0, bhi = 0;
  // Largest entry count of any aligned 32-row block (rows 32b .. 32b+31): the TMA-fed banded kernel
  // stages one block's CSR slice at a time (kspmv.cu k_spmv_ring2).
  int32_t blk32_max = 0;
  // Row selection of one launch (constant-diagonal SpMV only): the rows [sel_a0, sel_a1) followed by
  // [sel_b0, sel_b1); all four zero = every row. A row-sharded solve computes the interior rows
  // (no halo column) while the halo exchange is in flight, then the boundary rows (solver.cpp
  // apply_ph_sharded).
  int32_t sel_a0 = 0, sel_a1 = 0, sel_b0 = 0, sel_b1 = 0;
};
constexpr int kMaxDiag = 64;
constexpr int kMaxConstDiag = 32;

// Reduction workspace: `partials` holds at least kMaxGrid * max_slots doubles.
struct Reducer {
  double* partials = nullptr;
  DevState* ds = nullptr;
  // Non-null in row-sharded solves: the last CTA writes its rank-local totals here (ds->xred)
  // and skips the fused dense step (cta_commit), which then runs after the cross-rank reduction.
  double* xred = nullptr;
  // Finisher protocol of the constant-diagonal SpMV (kcdia.cu): (kMaxS + 1) x kMaxGrid partial
  // slots that hold an all-ones NaN pattern while empty. A streaming CTA publishes a partial with
  // one relaxed store; the finisher CTA polls the slots, sums them in index order and re-arms them.
  double* slots = nullptr;
  // Row-sharded, second launch of a split product: totals of the first launch, added (first) to this
  // launch's totals before they go to xred.
  const double* xbase = nullptr;
};

// What the finalising CTA (the last one to finish, or the finisher CTA of kcdia.cu) does with the reduced vector of an SpMV (kcommon.cuh finalize_spmv / finisher_finish).
enum FinOp : int32_t {
  kFinStore = 0,    // copy the reduced values to `dst`
  kFinRhsEta0 = 1,  // level k step (b): rhs := P^H r^(k+1); eta_0 := solve(Ma, rhs)
  kFinColEta = 2,   // level k column q: Mn[:,q] := P^H V^(k+1)_q; eta_{q+1} or gamma_{k+1}
  kFinTrueRes = 3,  // true residual refresh: resnorm, g := P^H r, pending gamma_0
};

struct FinParams {
  int32_t op = kFinStore;
  int32_t s = 0;
  int32_t k = 0;    // level
  int32_t q = 0;    // column
  int32_t ell = 0;
  int32_t _pad = 0;
  double* dst = nullptr;
};

// Occupancy-derived persistent grid size for the streaming kernels (multiple of the SM count).
int grid_for(int64_t n);
void kernels_init(int device);

// ---- launch accounting (bench evidence) ---------------------------------------------------
// Every launcher counts its kernel launches. With profiling on, each launch is also bracketed
// by CUDA events on its stream and tagged with its ALGORITHMIC bytes, so the
// bench can report per-class average duration and achieved GB/s of the timed region.
enum KernelClass : int32_t {
  kKSpmv = 0,
  kKLevelUpdate,
  kKRebuildTop,
  kKRebuildDeferred,
  kKLs,
  kKPoly,
  kKPrologue,
  kKValidate,
  kKOther,
  kKPersistCycle,
  kKNumClasses
};
struct KernelClassStats {
  uint64_t launches;
  double total_ms;
  double total_bytes;
};
uint64_t launch_count();
void count_launches(uint64_t n);  // kernels executed by a CUDA-graph replay
// Graph-captured profiling: while a capture list is set, launchers record their event pair into
// it (event-record graph nodes); after each replay the owner folds the list into the totals.
struct ProfEvent {
  int32_t cls;
  cudaEvent_t a, b;
  double bytes;
};
bool prof_enabled();
void prof_set_capture_list(std::vector<ProfEvent>* list);
void prof_accumulate(const std::vector<ProfEvent>& list);
void prof_release(std::vector<ProfEvent>& list);  // return a destroyed graph's events to the pool
void prof_enable(bool on);
void prof_collect();  // folds completed events into the per-class totals (call after a sync)
void prof_read(KernelClassStats* out);  // kKNumClasses entries
// ktimeline.cuh probes (no-ops unless built with MSTAB_TIMELINE): bind the slot buffer per TU
void kcdia_timeline_bind(unsigned long long* p);
void klevel_timeline_bind(unsigned long long* p);
void prof_reset();

// ---- the Mstab cycle ----------------------------------------------------------------------
// y = A x, fused partial dots P^H y (s of them) and the finaliser `fin`. When `b` != nullptr the
// kernel instead writes y = b - A x and also reduces ||y||^2 (true residual refresh).
void launch_spmv_ph(cudaStream_t st, const DevCsr& a, const double* x, double* y, const double* p,
                    int64_t ld, int s, const double* b, const FinParams& fin, const Reducer& red);

// The same on the constant-diagonal operator form (a.mask_bytes > 0); called by launch_spmv_ph.
void launch_spmv_cdia(cudaStream_t st, const DevCsr& a, const double* x, double* y, const double* p,
                      int64_t ld, int s, const double* b, const FinParams& fin, const Reducer& red);

// ---- row-sharded solves: finalisers run after the cross-rank reduction of ds->xred ---------
// Each replays exactly the dense tail the fused kernel runs in its last CTA (same code), from
// the reduced totals in ds->xred (allreduced) or `gath` (allgathered, rank-major).
void launch_fin_spmv(cudaStream_t st, int s, const FinParams& fin, DevState* ds);
void launch_fin_poly(cudaStream_t st, int s, DevState* ds);
// dots / stats / validate: copy the reduced totals where the fused kernel would have stored them
void launch_fin_copy(cudaStream_t st, const double* src, double* dst, int count);
// LS: merge `world` rank-local R factors (+ column sums of squares) in rank order, then solve.
void launch_fin_ls(cudaStream_t st, int ell, int s, int world, bool chol, const double* gath, DevState* ds);
constexpr int ls_split_count(int ell) { return (ell + 1) * (ell + 2) / 2 + ell; }

// step (a), top level only: r_out = r_in - V^(k) gamma (gemv + subtract, idrstab.cpp:113-117).
// At k == 0 the kernel first raises a pending singular gamma_0 as a breakdown.
void launch_level_update(cudaStream_t st, int64_t n, int64_t ld, int s, int k, const double* r_in,
                         double* r_out, const double* vk, DevState* ds);

// step (c), top level, column q: V^(k)_q = r^(k+1) - sum_c eta_qc * mixed_c (idrstab.cpp:140-148)
void launch_rebuild_top(cudaStream_t st, int64_t n, int64_t ld, int s, int q, const double* rnext,
                        const double* vk_in, double* vk_out, const double* vk1, DevState* ds);

// Deferred lower-level pass of level k: the (a) updates of r^(0..k-1) and x, then the rebuild of
// V^(-1..k-1) for every column, top-down, in one HBM pass. lv_in/lv_out index level+1 (0..k+1).
void launch_rebuild_deferred(cudaStream_t st, int64_t n, int64_t ld, int s, int k,
                             const double* const* lv_in, double* const* lv_out,
                             const double* const* r_in, double* const* r_out, const double* x_in,
                             double* x_out, DevState* ds);

// least_squares_tall(Z=[r^(1)..r^(ell)], r^(0)) by CholeskyQR2 (Givens TSQR fallback) + tail guard.
// The same as two launches (CholeskyQR2 pass 1 / pass 2 with the Givens fallback), for callers
// that reduce across ranks between them.
void launch_ls_pass1(cudaStream_t st, int64_t n, int ell, const double* const* r, const Reducer& red);
void launch_ls_pass2(cudaStream_t st, int64_t n, int ell, int s, bool chol, const double* const* r,
                     const Reducer& red);
// CholeskyQR2 for tall systems (the one-pass Givens TSQR costs a dependent chain of rotations
// per row: 133 us at c2 against 35 us); small systems keep the Givens TSQR, whose rounding the
// reference's own 1e-12 trajectory tests were calibrated against.
constexpr int64_t kCholQrMinRows = 1 << 17;
inline bool ls_use_cholqr(int64_t n_global) {
  static const bool givens_only = std::getenv("MSTAB_LS_GIVENS") != nullptr;  // diagnostics
  return !givens_only && n_global >= kCholQrMinRows;
}
void launch_fin_ls1(cudaStream_t st, int ell, DevState* ds);
void launch_ls(cudaStream_t st, int64_t n, int64_t ld, int ell, int s, const double* const* r,
               const Reducer& red);

// poly_combination + fused ||r||^2, P^H r, P^H V and the pending gamma_0 solve.
void launch_poly(cudaStream_t st, int64_t n, int64_t ld, int s, int ell, const double* const* lv,
                 double* u_out, double* v_out, const double* const* r, double* r_out,
                 const double* x_in, double* x_out, const double* p, const Reducer& red);

// Start of a solve: Ma := P^H V, g := P^H r, pending gamma_0 := solve(Ma, g).
void launch_prologue(cudaStream_t st, int64_t n, int64_t ld, int s, const double* p,
                     const double* v, const double* r, const Reducer& red);

// ---- persistent cycle (kpersist.cu): one cooperative kernel runs a whole cycle out of registers ----
// set p = (x_in, r_in, u_in, v_in) -> set 1-p; b != nullptr adds the true-residual refresh. xbuf: n
// doubles of scratch; partials: persist_partials_doubles(n) doubles; bar: 4 bytes (grid barrier
// counter, zeroed by the launcher). Returns false when (s, ell) is
// not instantiated or the grid cannot be co-resident (probe_only: answer without launching).
int64_t persist_partials_doubles(int64_t n);
bool launch_persist_cycle(cudaStream_t st, const DevCsr& a, int64_t n, int64_t ld, int s, int ell,
                          const double* x_in, const double* r_in, const double* u_in, const double* v_in,
                          double* x_out, double* r_out, double* u_out, double* v_out, const double* p,
                          const double* b, double* xbuf, double* partials, DevState* ds, unsigned* bar,
                          bool probe_only, double stop_below = -1.0, HostCycleSlot* hslot = nullptr,
                          uint64_t seq = 0);
// stop_below: the kernel sets DevState::stop when the cycle breaks down or ends with a residual norm
// <= stop_below (negative: never on convergence); hslot (mapped host memory) receives the status
// and then `seq`.

// ---- validate (recycle.cpp:40-83): ||V - A U||^2, ||V||^2 per column, P^H P, V^H V ----------
// Results land in ds->scal[0..1] (dev_num, dev_den) and ds->gram (P^H P then V^H V).
// ---- split preconditioning (ktri.cu, precond.cpp:23-219) ------------------------------------
// One triangular factor of a SplitPreconditioner on the device: CSR (int32) in ascending column
// order as CsrMatrix::from_triplets leaves it, or, for a diagonal-only factor (split Jacobi),
// just the diagonal (`diag` non-null).
struct DevTri {
  int64_t n = 0, nnz = 0;
  const int32_t* rp = nullptr;
  const int32_t* ci = nullptr;
  const double* val = nullptr;
  const double* diag = nullptr;
  // Level schedule (triangular factors): rows sorted by dependency level, each level padded with
  // -1 to a multiple of 32 slots so a warp's 32 rows are mutually independent.
  const int32_t* order = nullptr;
  int64_t nslots = 0, nlevels = 0;
  bool lower = true;
};
// x = F^-1 b (lower_solve / upper_solve, precond.cpp:101-133), bit-identical; `sync` is n + 1
// ints of scratch (done flags + ticket), zeroed by the launcher.
void launch_tri_solve(cudaStream_t st, const DevTri& f, const double* b, double* x, int* sync);
// y = w (b == nullptr) or y = b - w, with the P^H y (+ ||y||^2) reduction and finalize_spmv(fin).
void launch_ph_fin(cudaStream_t st, int64_t n, int64_t ld, int s, const double* w, double* y, const double* p,
                   const double* b, const FinParams& fin, const Reducer& red);

// ---- comparison baselines (kbase.cu, baselines.cpp:49-262) ------------------------------------
// out = x + a * y (out may alias x)
void launch_xpay(cudaStream_t st, int64_t n, const double* x, const double* y, double a, double* out);
// p = r + beta * (p - omega * ap)
void launch_bicgstab_p(cudaStream_t st, int64_t n, const double* r, const double* ap, double beta, double omega,
                       double* p);

// ---- SRIDR recycled phase (ksridr.cu, sridr.cpp:57-81) ------------------------------------
// rt = r - V gamma, xt = x + U gamma (gamma = ds->gamma[0..s))
void launch_sridr_corr(cudaStream_t st, int64_t n, int64_t ld, int s, const double* r, const double* x,
                       const double* u, const double* v, double* rt, double* xt, const DevState* ds);
// r = rt - omega art, x = xt + omega rt, then P^H r, ||r||^2 and finalize_spmv(fin)
void launch_sridr_update(cudaStream_t st, int64_t n, int64_t ld, int s, double omega, const double* rt,
                         const double* art, const double* xt, double* r, double* x, const double* p,
                         const FinParams& fin, const Reducer& red);

// au: the products A U precomputed by the caller (preconditioned operators), else nullptr and
// the kernel forms them from the CSR.
void launch_validate(cudaStream_t st, const DevCsr& a, const double* p, const double* u,
                     const double* v, int64_t ld, int s, const Reducer& red, const double* au = nullptr);

// ---- generic helpers (initialisation paths; not per-cycle) --------------------------------
// dst[j] = dot(A_j, y) for j < na (A_j = a + j*ld); dst[na] = ||y||^2 when with_norm.
void launch_dots(cudaStream_t st, int64_t n, int64_t ld, const double* a, int na, const double* y,
                 bool with_norm, double* dst, const Reducer& red);
// y += (-coef[j]) * A_j for j = 0..na-1 in order (axpy(-c, a_j, y), types.cpp:21-23)
void launch_axpy_neg(cudaStream_t st, int64_t n, int64_t ld, const double* a, int na,
                     const double* coef, double* y);
// y = x / sqrt(*d2)   (u0 = r0 / ||r0||, idrstab.cpp:57-58 and :83-84)
void launch_div_by_sqrt(cudaStream_t st, int64_t n, const double* x, const double* d2, double* y);
// y = x * (1.0 / sqrt(*d2))   (orthonormalize's q = w * inv, kernels.cpp:43-45)
void launch_mul_inv_sqrt(cudaStream_t st, int64_t n, const double* x, const double* d2, double* y);
// y = b - y (initial residual r = b - A x0)
void launch_rsub(cudaStream_t st, int64_t n, const double* b, double* y);
// out: dst[0] = sum x^2, dst[1] = #non-finite, dst[2] = #non-zero
void launch_vec_stats(cudaStream_t st, int64_t n, const double* x, double* dst, const Reducer& red);
// b_next = h2 * (x / dt + f) (implicit-Euler chain of the BASELINE configs)
void launch_euler_rhs(cudaStream_t st, int64_t n, const double* x, const double* f, double dt,
                      double h2, double* b);
// b_next = x + alpha * g (banded-random chain)
void launch_axpby_chain(cudaStream_t st, int64_t n, const double* x, const double* g, double alpha,
                        double* b);

// ---- standalone kernel helpers (parity tests of the dense steps) --------------------------
// x = solve_small(M, rhs) on the device (single-warp LU, kernels.cpp:95-154); *ok = 1 / 0.
// Fills count doubles with hash-derived values in [-1, 1) (benchmark operands).
void launch_fill_hash(cudaStream_t st, double* p, int64_t count, uint64_t seed);

void launch_small_solve(cudaStream_t st, int s, const double* m, const double* rhs, double* x,
                        int32_t* ok);

// ---- complex128 primitives (kcomplex.cu) ---------------------------------------
// Complex vectors are interleaved (re, im) pairs; every pointer below addresses such pairs.
constexpr int kZMaxTerms = kMaxS + 1;
struct ZTerms {
  int32_t m = 0;
  const double* col[kZMaxTerms] = {};  // m vectors
  double re[kZMaxTerms] = {}, im[kZMaxTerms] = {};  // their complex coefficients (unused by the dots)
};
// y = A x, rows in CSR order (csr.cpp:103-113)
void launch_zspmv(cudaStream_t st, int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci, const double* val,
                  const double* x, double* y);
// mode 0: y_out = y_in then += coef_c col_c in order (axpy chain); mode 1 / 2: y_out = y_in +/- gemv
void launch_zaxpys(cudaStream_t st, int64_t n, int mode, double* y_out, const double* y_in, const ZTerms& t);
// mode 0: y = x * (a + 0i); mode 1: y = x / a
void launch_zscale(cudaStream_t st, int64_t n, int mode, double* y, const double* x, double a);
void launch_zsub(cudaStream_t st, int64_t n, double* r, const double* b, const double* ax);
// out[2c], out[2c+1] = conj(col_c) . y; y == nullptr: out[2c] = sum |col_c|^2
void launch_zdots(cudaStream_t st, int64_t n, const ZTerms& cols, const double* y, double* out, const Reducer& red);
// out: sum |x|^2, #non-finite, #nonzero, #entries with a nonzero imaginary part
void launch_zstats(cudaStream_t st, int64_t n, const double* x, double* out, const Reducer& red);
// Deferred lower levels of level k of the complex level iteration (the complex twin of
// launch_rebuild_deferred): for every row, top-down over the levels i = k-1 .. -1, the BiCG update
// of r^(i) (x for i = -1) with gamma and the column rebuilds of level i for q = 0..s-1 in order
// (idrstab.cpp:113-121,140-148), in place. coef (device, complex pairs): eta as s rows of s
// coefficients ALREADY NEGATED (row q = -eta_q), then gamma (s). lv[i + 1] = V^(i) for i = -1..k,
// r[i] = r^(i) for i = 0..k.
struct ZDeferredArgs {
  double* lv[kMaxEll + 2] = {};
  double* r[kMaxEll + 1] = {};
  double* x = nullptr;
};
void launch_zrebuild_deferred(cudaStream_t st, int64_t n, int64_t ld, int s, int k, const ZDeferredArgs& a,
                              const double* coef);
// out: sum |v - au|^2, sum |v|^2
void launch_zdiff(cudaStream_t st, int64_t n, const double* v, const double* au, double* out, const Reducer& red);

}  // namespace mstab_b200
