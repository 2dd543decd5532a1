// solver.h — C++ objects behind the C-ABI handles of include/mstab_b200.h.
#pragma once
#include <complex>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/mstab_b200.h"
#include "comm.h"
#include "device_state.h"
#include "host_util.h"
#include "kernels.h"

typedef struct CUgraphExec_st* cudaGraphExec_t;

namespace mstab_b200 {

// Device allocation freed stream-ordered on the owning stream (cudaMallocAsync pool).
struct DevMem {
  void* ptr = nullptr;
  size_t bytes = 0;
  int64_t off = 0;  // elements before the owned rows (left halo of a row-sharded vector)
  std::shared_ptr<struct StreamHolder> stream;
  DevMem(std::shared_ptr<StreamHolder> st, size_t b);
  ~DevMem();
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  double* d() const { return static_cast<double*>(ptr) + off; }
};
using DevPtr = std::shared_ptr<DevMem>;

struct StreamHolder {
  int device = 0;
  cudaStream_t stream = nullptr;
  // Size-bucketed cache of released blocks of this stream. A solve hands out fresh, independently
  // owned blocks every time (x, the fetched and final U / V: 550 MB per solve at c2) and the caller
  // drops the previous solve's; routed through cudaFreeAsync / cudaMallocAsync the driver's pool
  // occasionally re-grows mid-solve (r02 step timing: sporadic 5-20 ms cycles at the fetch). A block
  // released here is handed to the next request of the same size on the SAME stream, which is
  // ordered after everything its previous owner enqueued, exactly like a stream-ordered free.
  std::mutex cache_mu;
  std::unordered_map<size_t, std::vector<void*>> cache;
  size_t cached_bytes = 0;
  void* take(size_t bytes);
  bool give(void* p, size_t bytes);
  void drop_cache();  // releases every cached block (stream-ordered)
  ~StreamHolder();
};

int64_t padded_ld(int64_t n);

// One source/destination buffer set of the cycle ping-pong (x, r^(0), U = V^(-1), V = V^(0)).
struct WSet {
  DevPtr x, r, U, V;
};

// An instantiated CUDA graph of one whole cycle (ell level iterations + poly [+ true residual]).
struct CycleGraph {
  cudaGraphExec_t exec = nullptr;
  uint64_t kernels = 0;
  bool profiled = false;
  std::vector<ProfEvent> prof;  // event pairs captured into the graph (profiling mode)
  void reset();
  ~CycleGraph() { reset(); }
};

// Per-context solve workspace, persistent across solves with the same (operator, s, ell,
// true-residual) so the two cycle graphs (A->B, B->A) are captured once and replayed for every
// cycle of every right-hand side of a sequence.
struct Workspace {
  uint64_t op_uid = 0;
  int64_t n = -1;
  int s = 0, ell = 0;
  bool tres = false;
  WSet set[2];
  std::vector<DevPtr> R, VL;  // r^(1..ell), V^(1..ell)
  DevPtr b, P;
  // the buffer P was last copied from, held so its address cannot be recycled by the pool while
  // the copy is trusted (a freed-and-reallocated P at the same address must be copied again)
  DevPtr p_src;
  CycleGraph graph[2];          // graph[p]: set[p] -> set[1-p]
  // persistent cycle kernel (kpersist.cu): chosen once per workspace, dropped for the rest of a
  // solve after a fallback request
  DevPtr xbuf;
  bool persist = false;
};

struct Context {
  std::shared_ptr<StreamHolder> sh;
  int device = 0;
  DevPtr ds_mem;        // DevState
  DevPtr partials;      // reduction partials
  DevPtr slots;         // sentinel-armed partial slots of the finisher protocol (Reducer::slots)
  CycleStatus* host_status = nullptr;  // pinned
  // Pipelined persistent cycles (solver.cpp persist_next): two slots in mapped pinned memory the
  // cycle kernels write their status into, and the launch / consume counters of the current solve.
  HostCycleSlot* hslots = nullptr;
  uint64_t pipe_launched = 0, pipe_consumed = 0;
  double* host_scal = nullptr;         // pinned, 64 doubles
  std::unique_ptr<Workspace> ws;       // cycle buffers + captured cycle graphs
  bool use_graphs = true;
  DevPtr pcache;                       // last make_cut_space result (immutable)
  int64_t pcache_n = -1, pcache_s = -1;
  uint64_t pcache_seed = 0;
  // Row-sharded solves (comm.h): the communicator and the vector layout of the slab operator.
  // Vectors of length lay_n (the slab's rows) get lay_lo halo rows in front of the owned rows
  // and column stride lay_ld; DevMem::d() points at the first owned row.
  std::unique_ptr<Comm> comm;
  DevPtr xgath;  // allgather landing buffer (world * kMaxXred doubles)
  DevPtr val_au;  // validate: the products A U of a large plain operator (n x s scratch)
  int64_t val_au_n = -1;
  int val_au_s = 0;
  int64_t lay_n = -1, lay_lo = 0, lay_ld = 0, lay_row0 = 0, lay_nglobal = 0;
  bool sharded() const { return comm && comm->world() > 1; }
  int64_t ld(int64_t n) const { return n == lay_n ? lay_ld : padded_ld(n); }
  cudaStream_t stream() const { return sh->stream; }
  DevState* ds() const { return static_cast<DevState*>(ds_mem->ptr); }
  Reducer reducer() const { return Reducer{partials->d(), ds(), sharded() ? ds()->xred : nullptr, slots->d()}; }
  DevPtr alloc(size_t bytes) { return std::make_shared<DevMem>(sh, bytes); }
  DevPtr alloc_vecs(int64_t n, int64_t cols);
  void sync();
  void trim();
  explicit Context(int device);
  ~Context();
};

// Split preconditioner L, R of a preconditioned operator L^-1 A R^-1 (precond.hpp:16-24,
// PreconditionedOperator), the factors on the device plus the scratch its applies use.
struct Precond {
  int kind = 0;  // MSTAB_PRECOND_*
  DevPtr l_rp, l_ci, l_val, l_diag, l_ord, r_rp, r_ci, r_val, r_diag, r_ord;
  DevTri L, R;
  DevPtr t1, t2, t3, sync, au;  // chain temporaries, tri-solve flags, A U block of validate
  int au_s = 0;
};

struct Operator {
  uint64_t uid = 0;  // unique per created operator (workspace/graph cache key)
  int64_t n = 0, nnz = 0;
  uint64_t fingerprint = 0;
  DevPtr rp, ci, val;
  // row slab (mstab_operator_create_csr_slab): global size, first row, x index range, halo plan
  int64_t n_global = 0, row0 = 0, xlo = 0, xhi = 0;
  HaloPlan halo;
  // interior rows [int_lo, int_hi) of a row slab: no column outside the owned rows (0, 0: none known)
  int64_t int_lo = 0, int_hi = 0;
  DevCsr csr() const {
    DevCsr c;
    c.n = n;
    c.nnz = nnz;
    c.xlo = xlo;
    c.xhi = xhi;
    c.blo = blo;
    c.bhi = bhi;
    c.blk32_max = blk32_max;
    c.row_ptr = static_cast<const int32_t*>(rp->ptr);
    c.col_idx = static_cast<const int32_t*>(ci->ptr);
    c.values = val->d();
    if (ndiag > 0 && use_dia) {
      c.ndiag = ndiag;
      c.dia_ld = dia_ld;
      c.dia_val = dia_val ? dia_val->d() : nullptr;
      c.dia_off = static_cast<const int32_t*>(dia_off->ptr);
      for (int d = 0; d < ndiag && d < 64; ++d) c.off[d] = offsets[d];
      if (mask_bytes > 0) {
        c.mask_bytes = mask_bytes;
        c.dia_mask = dia_mask->ptr;
        for (int d = 0; d < ndiag && d < kMaxConstDiag; ++d) c.cval[d] = cvals[d];
      }
    }
    return c;
  }
  std::vector<int32_t> offsets;  // DIA offsets (host copy)
  // DIA form of the same matrix (kernels.h DevCsr), built at upload when it pays off
  int64_t blo = 0, bhi = 0;  // column band (kernels.h DevCsr)
  int32_t blk32_max = 0;     // largest aligned 32-row block (kernels.h DevCsr)
  int32_t ndiag = 0;
  int64_t dia_ld = 0;
  DevPtr dia_val, dia_off;
  bool use_dia = true;
  // constant-diagonal form (kernels.h DevCsr::cval / dia_mask); mask_bytes == 0 when not used
  int32_t mask_bytes = 0;
  std::vector<double> cvals;
  DevPtr dia_mask;
  std::shared_ptr<Precond> pc;  // preconditioned operator L^-1 A R^-1 (nullptr: plain CSR)
  // A^H as its own operator (CsrOperator::apply_adjoint), built on first use (adjoint_of)
  mutable std::shared_ptr<Operator> adj;
  mutable std::mutex adj_mu;
};

struct Recycle {
  int64_t n = 0, s = 0, level_j = 0;
  uint64_t fingerprint = 0;
  DevPtr p, u, v;  // n x s blocks with ld = padded_ld(n); immutable
  std::vector<std::complex<double>> omega;
};
using RecyclePtr = std::shared_ptr<const Recycle>;

struct SolveResultImpl {
  DevPtr x;
  int64_t n = 0;
  mstab_report report{};
  std::vector<mstab_history_point> history;
  std::vector<double> taus;  // cycle-major, ell per cycle (real parts; imaginary parts are 0)
  RecyclePtr final_data;
  RecyclePtr fetched;
};

// ---- complex128 path (zsolver.cpp) ---------------------------------------------
// Complex vectors and blocks are interleaved (re, im) pairs with column stride padded_ld(n).
struct ZOperator {
  int64_t n = 0, nnz = 0;
  uint64_t fingerprint = 0;
  bool real = false;  // CsrMatrix::is_real (csr.cpp:26)
  DevPtr rp, ci, val;
};
struct ZRecycle {
  int64_t n = 0, s = 0, level_j = 0;
  uint64_t fingerprint = 0;
  DevPtr p, u, v;
  std::vector<std::complex<double>> omega;
};
struct ZResult {
  DevPtr x;
  int64_t n = 0;
  mstab_report report{};
  std::vector<mstab_history_point> history;
  std::vector<std::complex<double>> taus;
  std::shared_ptr<const ZRecycle> final_data, fetched;
};
std::shared_ptr<ZOperator> make_operator_z(Context& ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                           const double* values_re_im);
void apply_z(Context& ctx, const ZOperator& op, const double* x, double* y, int mem);
std::shared_ptr<ZRecycle> make_recycle_z(Context& ctx, int64_t n, int64_t s, const double* p, const double* u,
                                         const double* v, int mem, const double* omega_re_im, int64_t omega_count,
                                         int64_t level_j, uint64_t fingerprint);
void download_recycle_z(Context& ctx, const ZRecycle& rd, double* p, double* u, double* v, double* omega_re_im);
mstab_validation_report validate_z(Context& ctx, const ZRecycle& rd, const ZOperator& a);
std::unique_ptr<ZResult> solve_z(Context& ctx, const ZOperator& a, const double* b, const double* x0, int mem,
                                 const mstab_solver_config& cfg, const ZRecycle* recycle,
                                 const mstab_fetch_policy* fetch);
void result_x_z(Context& ctx, const ZResult& res, double* x, int mem);

// idrstab_solve / mstab_solve (idrstab.cpp:193-307) on the device.
std::unique_ptr<SolveResultImpl> solve(Context& ctx, const Operator& op, const double* b,
                                       const double* x0, int mem, const mstab_solver_config& cfg,
                                       const Recycle* recycle, const mstab_fetch_policy* fetch);

// sridr_solve (sridr.cpp:23-118) on the device; the result carries x and the report only.
std::unique_ptr<SolveResultImpl> sridr(Context& ctx, const Operator& op, const double* b, const double* x0, int mem,
                                       const mstab_solver_config& cfg, const Recycle& recycle);

// bicgstab_solve / gmres_solve (baselines.cpp:49-262) on the device; x and the report only.
// y = A^H x (CsrOperator::apply_adjoint -> spmv_adjoint, csr.cpp:115-124), bit-identical.
const Operator& adjoint_of(Context& ctx, const Operator& op);
// bicg_solve (baselines.cpp:145-196) on the device; x and the report only.
std::unique_ptr<SolveResultImpl> bicg(Context& ctx, const Operator& op, const double* b, const double* x0, int mem,
                                      double tol, int64_t max_mv, const double* shadow);
std::unique_ptr<SolveResultImpl> bicgstab(Context& ctx, const Operator& op, const double* b, const double* x0, int mem,
                                          double tol, int64_t max_mv, const double* shadow);
std::unique_ptr<SolveResultImpl> gmres(Context& ctx, const Operator& op, const double* b, const double* x0, int mem,
                                       double tol, int64_t max_it);

// validate (recycle.cpp:40-83). Throws Error with the reference's class code.
mstab_validation_report validate(Context& ctx, const Recycle& rd, const Operator& op);

std::shared_ptr<Operator> make_operator(Context& ctx, int64_t n, const int64_t* row_ptr,
                                        const int64_t* col_idx, const double* values);
// Row slab of rank ctx.comm->rank() (slab_starts: world + 1 ascending boundaries).
std::shared_ptr<Operator> make_operator_slab(Context& ctx, int64_t n, const int64_t* row_ptr,
                                             const int64_t* col_idx, const double* values,
                                             const int64_t* slab_starts);

// The same from the rank's own rows only (global column indices), the peers' column spans and the
// global fingerprint supplied by the caller (large systems: no rank holds the global CSR).
std::shared_ptr<Operator> make_operator_slab_local(Context& ctx, int64_t n_global, const int64_t* slab_starts,
                                                   const int64_t* row_ptr, const int64_t* col_idx,
                                                   const double* values, const int64_t* spans,
                                                   uint64_t fingerprint);

void spmv(Context& ctx, const Operator& op, const double* x_dev, double* y_dev);

// build_jacobi / build_ilu0 (precond.cpp:23-99) on the host, real data: the factors in CSR with
// ascending columns (CsrMatrix::from_triplets order). Capacities: nnz(A) + n entries each.
void precond_build(int kind, int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                   int64_t* l_rp, int64_t* l_ci, double* l_val, int64_t* r_rp, int64_t* r_ci, double* r_val);
// PreconditionedOperator(pc, a) (precond.cpp:188-219) with the factors given as CSR.
std::shared_ptr<Operator> make_operator_precond(Context& ctx, int64_t n, const int64_t* row_ptr,
                                                const int64_t* col_idx, const double* values, int kind,
                                                const int64_t* l_rp, const int64_t* l_ci, const double* l_val,
                                                const int64_t* r_rp, const int64_t* r_ci, const double* r_val);
// y = L^-1 x (which = 0, lower_solve) or y = R^-1 x (which = 1, upper_solve) with the operator's factors.
void precond_solve(Context& ctx, const Operator& op, int which, const double* x_dev, double* y_dev);

// make_cut_space (baselines.cpp:36-47): returns the orthonormal n x s block P on the device.
DevPtr make_cut_space(Context& ctx, int64_t n, int s, uint64_t seed);
// arnoldi_init (idrstab.cpp:45-87) with rng seed `rng_seed` for the padding draws.
void arnoldi_init(Context& ctx, const Operator& op, const double* r0, int s, uint64_t rng_seed,
                  double* U, double* V);
// The same with the padding draws supplied by the caller (the reference draws them from the
// caller's std::mt19937_64 through one std::normal_distribution per call, idrstab.cpp:60,77-78).
void arnoldi_init(Context& ctx, const Operator& op, const double* r0, int s,
                  const std::function<void(double*, int64_t)>& draw, double* U, double* V);
// bicg_projection / level_iteration / poly_combination (idrstab.hpp:33-68) on the device, host
// column-major blocks in and out. r_levels holds r^(0..k) on entry and r^(0..k+1) on return
// (capacity n (k+2)); v_levels holds V^(-1..k) on entry and V^(-1..k+1) on return (capacity
// n s (k+3)). Breakdowns throw with the reference's class codes (SINGULAR, RANK).
void bicg_projection_host(Context& ctx, int64_t n, int s, const double* p, const double* block,
                          const double* target, double* gamma);
void projection_gram_host(Context& ctx, int64_t n, int s, const double* p, const double* block,
                          const double* target, double* m, double* g);
void level_iteration_host(Context& ctx, const Operator& op, int s, int k, const double* p, double* x0,
                          double* r_levels, double* v_levels);
void poly_combination_host(Context& ctx, int64_t n, int s, int ell, const double* x0, const double* r_levels,
                           const double* v_levels, double* x, double* r, double* u, double* v, double* tau,
                           int32_t* tail_perturbed);
// Host-visible helpers for the kernel-level C entry points.
const double* read_scal(Context& ctx, int count);
const CycleStatus& read_status(Context& ctx);
void reset_status(Context& ctx);

}  // namespace mstab_b200
