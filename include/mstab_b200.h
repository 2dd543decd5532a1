/*
 * mstab_b200.h — C-ABI drop-in boundary for the M(s,l)stab / IDR(s)stab(l) solve loop.
 *
 * Plain C: opaque handles, plain pointers and sizes, no torch or C++ types.
 * Every entry point below replaces one piece of the reference's proj/core interface;
 * the citation after each declaration names the reference symbol (file:line under
 * /root/reference/proj/core) whose behaviour it keeps.
 *
 * Two libraries export exactly this ABI:
 *   - paper_1604_06043_b200/libmstab_b200.so : the B200 product (sm_100a kernels, device-resident state);
 *   - oracle/_ref/libmstab_ref.so            : the unmodified reference compiled from its own sources
 *                                              (test/bench baseline only, see oracle/Makefile).
 * so a caller (tests, bench.py, a cgo/ctypes binding) can switch implementations by library path.
 *
 * Data model: real fp64 values (the reference stores complex<double>; every real input keeps
 * a zero imaginary part bit-for-bit through the solve), int64 CSR indices at
 * the boundary (the reference uses size_t), column-major N x s blocks (dense.hpp:23-24).
 *
 * Errors: every function returns 0 on success or a negative MSTAB_E_* code that maps 1:1 to the
 * exception class the reference would throw (errors.hpp:9-72). mstab_last_error() returns the
 * message of the last failure on the calling thread. Breakdowns inside a solve are NOT errors:
 * like the reference (idrstab.cpp:290-293) they end the solve with status MSTAB_STATUS_BREAKDOWN.
 *
 * Threading: one in-flight call per context; operators and recycle handles are immutable after
 * creation and may be shared read-only (operator.hpp:12-14, recycle.hpp:14-17).
 */
#ifndef MSTAB_B200_H
#define MSTAB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes (errors.hpp:9-72) ------------------------------------------------------- */
#define MSTAB_OK 0
#define MSTAB_E_ERROR (-1)         /* mstab::Error (non-finite input, zero start vector, csr validate) */
#define MSTAB_E_DIMENSION (-2)     /* mstab::DimensionMismatch */
#define MSTAB_E_CONFIG (-3)        /* mstab::ConfigError */
#define MSTAB_E_FINGERPRINT (-4)   /* mstab::FingerprintMismatch */
#define MSTAB_E_STALE (-5)         /* mstab::StaleData */
#define MSTAB_E_PARSE (-6)         /* mstab::ParseError */
#define MSTAB_E_IO (-7)            /* mstab::IoError */
#define MSTAB_E_SINGULAR (-8)      /* mstab::SingularProjection (only from the kernel helpers) */
#define MSTAB_E_RANK (-9)          /* mstab::RankDeficient (only from the kernel helpers) */
#define MSTAB_E_ZEROPIVOT (-10)    /* mstab::ZeroPivot (build_jacobi / build_ilu0, precond.cpp:33,56-82) */
#define MSTAB_E_MISSING_OMEGAS (-11) /* mstab::MissingOmegas (sridr_solve, sridr.cpp:33-34) */
#define MSTAB_E_CUDA (-20)         /* device/runtime failure (no reference counterpart) */
#define MSTAB_E_NOTREAL (-21)      /* complex data passed to a real fp64 entry point (use the *_z ones) */

/* ---- memory spaces for pointer arguments --------------------------------------------------- */
#define MSTAB_MEM_HOST 0
#define MSTAB_MEM_DEVICE 1

/* ---- status (report.hpp:12) ---------------------------------------------------------------- */
#define MSTAB_STATUS_CONVERGED 0
#define MSTAB_STATUS_MAXMV 1
#define MSTAB_STATUS_BREAKDOWN 2

/* ---- fetch policy kinds (recycle.hpp:31-42) ------------------------------------------------ */
#define MSTAB_FETCH_AT_CYCLE 0
#define MSTAB_FETCH_AT_HALF_TOLERANCE 1
#define MSTAB_FETCH_MANUAL 2

typedef struct mstab_context mstab_context;
typedef struct mstab_operator mstab_operator;
typedef struct mstab_recycle mstab_recycle;
typedef struct mstab_result mstab_result;

/* SolverConfig (report.hpp:24-33; validated as report.cpp:16-22) */
typedef struct mstab_solver_config {
  int64_t s;
  int64_t ell;
  double tol;
  int64_t max_mv;
  int32_t true_residual_each_cycle;
  int32_t _pad;
  uint64_t seed;
} mstab_solver_config;

/* FetchPolicy (recycle.hpp:31-42) */
typedef struct mstab_fetch_policy {
  int32_t kind;
  int32_t _pad;
  int64_t cycle;
} mstab_fetch_policy;

/* HistoryPoint (report.hpp:16-22) */
typedef struct mstab_history_point {
  int64_t cycle;
  int64_t mv;
  int64_t level;
  double resnorm;
  int64_t wall_ns;
} mstab_history_point;

/* SolveReport scalars (report.hpp:35-58); histories come from the accessors below */
typedef struct mstab_report {
  int64_t h_mv;
  int64_t h_mv_aux;
  int64_t h_rd;
  int64_t cycles;
  int32_t status;
  int32_t has_fetched;       /* SolveResult::fetched has a value (idrstab.hpp:76) */
  double bnorm;
  double final_resnorm;
  int64_t wall_ns_total;
  int64_t history_len;       /* residual_history.size() */
  int64_t tau_len;           /* total tau coefficients over all cycles (cycles * ell) */
  int64_t ell;
  char breakdown_reason[128];
} mstab_report;

/* RecycleData header fields (recycle.hpp:18-29) */
typedef struct mstab_recycle_info {
  int64_t n;
  int64_t s;
  int64_t level_j;
  int64_t omega_count;
  uint64_t fingerprint;
} mstab_recycle_info;

/* ValidationReport (recycle.hpp:44-48) */
typedef struct mstab_validation_report {
  double max_deviation;
  double sigma_min_ratio;
  int32_t low_rank_warning;
  int32_t _pad;
} mstab_validation_report;

/* ---- library / context -------------------------------------------------------------------- */
const char* mstab_last_error(void);
/* Row of the last MSTAB_E_ZEROPIVOT on this thread (ZeroPivot::row(), errors.hpp:39-45), -1 when
 * the last error carried no row. */
int64_t mstab_last_error_row(void);
const char* mstab_impl_name(void); /* "b200" or "reference" */
/* Build provenance: "<impl> <git sha>[-dirty] <compiler flags>", fixed at compile time, so every
 * bench line / smoke record names the binary it ran. */
const char* mstab_build_id(void);

/* Binds a device and creates the solver's CUDA stream. device < 0 selects the current device. */
int mstab_context_create(int32_t device, mstab_context** out);
void mstab_context_destroy(mstab_context* ctx);
/* Blocks until all work queued on the context's stream is complete. */
int mstab_context_synchronize(mstab_context* ctx);
/* Releases what the context keeps between solves (cycle workspace and graphs, cached cut-space,
 * recycled result blocks) and returns the memory to the device; the next solve rebuilds them.
 * Handles (operators, recycle data, results) stay valid. */
int mstab_context_trim(mstab_context* ctx);
/* The CUDA stream (cudaStream_t) the context launches on, as an opaque pointer (NULL on host impls). */
void* mstab_context_stream(mstab_context* ctx);

/* ---- operator (operator.hpp:15-50, csr.hpp:17-52) ----------------------------------------- */
/* Builds a CsrOperator from host CSR arrays: validates like CsrMatrix::validate (csr.cpp:11-24),
 * requires a square matrix (operator.cpp:21-23), computes the reference FNV-1a fingerprint
 * once (csr.cpp:28-43 over the size_t/complex<double> byte layout) and uploads the matrix. */
int mstab_operator_create_csr(mstab_context* ctx, int64_t n, const int64_t* row_ptr,
                              const int64_t* col_idx, const double* values, mstab_operator** out);
void mstab_operator_destroy(mstab_operator* op);

/* ---- split preconditioning (precond.hpp, precond.cpp) -----------------------
 * PrecondKind (precond.hpp:12). mstab_precond_build restates build_jacobi / build_ilu0
 * (precond.cpp:23-99) on the host: the factors L (lower, diagonal stored) and R (upper) of A in CSR
 * with ascending columns, like CsrMatrix::from_triplets. Each output array must hold nnz(A) + n
 * entries (row_ptr: n + 1); *l_nnz / *r_nnz receive the counts. Errors: MSTAB_E_ZEROPIVOT
 * (ZeroPivot), MSTAB_E_NOTREAL (Jacobi on a negative diagonal: the reference's square root is
 * imaginary).
 * mstab_operator_create_precond is PreconditionedOperator(pc, a) (precond.hpp:57-74): the operator
 * L^-1 A R^-1 on the device, with the reference's combined fingerprint (precond.cpp:203-210).
 * Every apply runs the upper solve, the SpMV and the lower solve on the device; the triangular
 * solves are bit-identical to upper_solve / lower_solve (precond.cpp:101-133). kind NONE gives
 * the plain CsrOperator (factors ignored). Single-GPU contexts only.
 * mstab_precond_solve: y = L^-1 x (which = 0: lower_solve, preconditioned_rhs) or y = R^-1 x
 * (which = 1: upper_solve, unpreconditioned_solution), mem as in mstab_operator_apply. */
#define MSTAB_PRECOND_NONE 0
#define MSTAB_PRECOND_JACOBI 1
#define MSTAB_PRECOND_ILU0 2
int mstab_precond_build(int32_t kind, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                        const double* values, int64_t* l_row_ptr, int64_t* l_col_idx, double* l_values,
                        int64_t* l_nnz, int64_t* r_row_ptr, int64_t* r_col_idx, double* r_values,
                        int64_t* r_nnz);
int mstab_operator_create_precond(mstab_context* ctx, int64_t n, const int64_t* row_ptr,
                                  const int64_t* col_idx, const double* values, int32_t kind,
                                  const int64_t* l_row_ptr, const int64_t* l_col_idx, const double* l_values,
                                  const int64_t* r_row_ptr, const int64_t* r_col_idx, const double* r_values,
                                  mstab_operator** out);
int32_t mstab_operator_precond_kind(const mstab_operator* op);
int mstab_precond_solve(mstab_context* ctx, const mstab_operator* op, int32_t which, const double* x, double* y,
                        int32_t mem);
int64_t mstab_operator_size(const mstab_operator* op);        /* LinearOperator::size (operator.hpp:21) */
int64_t mstab_operator_nnz(const mstab_operator* op);
uint64_t mstab_operator_fingerprint(const mstab_operator* op); /* operator.cpp:35 */
/* y = A x (CsrOperator::apply, operator.cpp:25-28 -> spmv csr.cpp:103-113). */
int mstab_operator_apply(mstab_context* ctx, const mstab_operator* op, const double* x, double* y,
                         int32_t mem);
/* y = A^H x (CsrOperator::apply_adjoint, operator.cpp:30-33 -> spmv_adjoint csr.cpp:115-124),
 * bit-identical for real data; for a preconditioned operator (L^-1 A R^-1)^H = R^-H A^H L^-H
 * (PreconditionedOperator::apply_adjoint, precond.cpp:190-200), bit-identical to the reference's
 * adjoint solves. Built once per operator on first use. ConfigError for a row slab. */
int mstab_operator_apply_adjoint(mstab_context* ctx, const mstab_operator* op, const double* x, double* y,
                                 int32_t mem);

/* ---- recycle data (recycle.hpp:18-64) ----------------------------------------------------- */
/* fetch(): deep copy of column-major P, U, V (N x s) plus omega history (re,im pairs),
 * level J and the operator fingerprint (recycle.cpp:26-38). */
int mstab_recycle_create(mstab_context* ctx, int64_t n, int64_t s, const double* p, const double* u,
                         const double* v, int32_t mem, const double* omega_re_im,
                         int64_t omega_count, int64_t level_j, uint64_t fingerprint,
                         mstab_recycle** out);
void mstab_recycle_destroy(mstab_recycle* rd);
int mstab_recycle_info_get(const mstab_recycle* rd, mstab_recycle_info* out);
/* Copies P, U, V (each N x s column-major; any may be NULL) and omega (re,im pairs; may be NULL). */
int mstab_recycle_download(mstab_context* ctx, const mstab_recycle* rd, double* p, double* u,
                           double* v, double* omega_re_im);
/* validate() (recycle.cpp:40-83): FingerprintMismatch / DimensionMismatch / StaleData. */
int mstab_recycle_validate(mstab_context* ctx, const mstab_recycle* rd, const mstab_operator* op,
                           mstab_validation_report* out);
/* save()/load() of the bit-exact .mrd file (recycle.cpp:85-192). */
int mstab_recycle_save(mstab_context* ctx, const mstab_recycle* rd, const char* path);
int mstab_recycle_load(mstab_context* ctx, const char* path, mstab_recycle** out);

/* ---- the solve loop (idrstab.hpp:88-96, idrstab.cpp:193-307) ------------------------------ */
/* idrstab_solve / mstab_solve. b and x0 (NULL = empty guess) live in `mem`. recycle == NULL runs
 * the fresh branch (make_cut_space + arnoldi_init); otherwise the recycled branch (validate,
 * then continue in the donor's M-spaces). fetch may be NULL. Returns 0 when the solve ran
 * (status in the report, breakdown included) or a negative error code for the exceptions the
 * reference lets escape (ConfigError, DimensionMismatch, Error, FingerprintMismatch, StaleData). */
int mstab_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                int32_t mem, const mstab_solver_config* cfg, const mstab_recycle* recycle,
                const mstab_fetch_policy* fetch, mstab_result** out);
/* sridr_solve (include/mstab/solvers/sridr.hpp, src/sridr.cpp:23-118): SRIDR with ell = 1 on the
 * recycle data's fixed block for its J recorded relaxations (one product per cycle), then IDR(s)
 * cycles. The result holds x and the report (no final_data / fetched). Errors as sridr_solve:
 * ConfigError (ell != 1, s mismatch), MissingOmegas, and validate's FingerprintMismatch/StaleData. */
int mstab_sridr_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                      int32_t mem, const mstab_solver_config* cfg, const mstab_recycle* recycle,
                      mstab_result** out);
/* The comparison baselines (include/mstab/solvers/baselines.hpp, src/baselines.cpp:49-262) on
 * the device: bicgstab_solve (shadow: N values in `mem`, or NULL for r0) and gmres_solve
 * (full-memory, modified Gram-Schmidt, no restarts). The result holds x and the report. */
int mstab_bicgstab_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                         int32_t mem, double tol, int64_t max_mv, const double* shadow, mstab_result** out);
/* bicg_solve (include/mstab/solvers/baselines.hpp, src/baselines.cpp:145-196): BiCG with the
 * adjoint products on the device (two products per iteration); shadow as in bicgstab_solve. */
int mstab_bicg_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                     int32_t mem, double tol, int64_t max_mv, const double* shadow, mstab_result** out);
int mstab_gmres_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                      int32_t mem, double tol, int64_t max_it, mstab_result** out);
void mstab_result_destroy(mstab_result* res);
int mstab_result_report(const mstab_result* res, mstab_report* out);
/* SolveResult::x, copied into x (N values in `mem`). */
int mstab_result_x(mstab_context* ctx, const mstab_result* res, double* x, int32_t mem);
/* residual_history: copies min(cap, history_len) points; returns the number copied (<0 on error). */
int64_t mstab_result_history(const mstab_result* res, mstab_history_point* out, int64_t cap);
/* omega_history (report.hpp:38-39): tau per cycle, flattened cycle-major, (re,im) pairs.
 * Copies min(cap, tau_len) coefficients; returns the number copied. */
int64_t mstab_result_taus(const mstab_result* res, double* re_im, int64_t cap);
/* New handles on the result's RecycleData: final_data, fetched (MSTAB_E_ERROR if none), and
 * handoff() = fetched if present else final_data (idrstab.hpp:80). Handles share the immutable
 * device buffers with the result; destroy each one independently. */
int mstab_result_final_data(const mstab_result* res, mstab_recycle** out);
int mstab_result_fetched(const mstab_result* res, mstab_recycle** out);
int mstab_result_handoff(const mstab_result* res, mstab_recycle** out);

/* ---- complex128 data (types.hpp:11-15) --------------------------
 * The reference computes in std::complex<double> throughout; the entry points above are its real
 * embedding (imaginary parts +0.0). These take complex arrays as interleaved (re, im) pairs:
 * a complex CsrMatrix (csr.hpp:17-52; fingerprint over the same byte layout, csr.cpp:28-43),
 * idrstab_solve / mstab_solve with complex b, x0 and recycle data (idrstab.cpp:193-307; a real
 * A, b, x0 triple draws the real cut-space, baselines.cpp:36-47), RecycleData with complex P, U,
 * V (recycle.hpp:18-64). The handles are the same types: mstab_recycle_info_get,
 * mstab_recycle_validate, mstab_result_report / _history / _taus / _final_data / _fetched /
 * _handoff and the destroy calls accept both kinds; every other real entry point returns
 * MSTAB_E_NOTREAL for a complex handle. Single-GPU, unpreconditioned operators. */
int mstab_operator_create_csr_z(mstab_context* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                const double* values_re_im, mstab_operator** out);
int32_t mstab_operator_is_complex(const mstab_operator* op);
int32_t mstab_recycle_is_complex(const mstab_recycle* rd);
int32_t mstab_result_is_complex(const mstab_result* res);
/* y = A x (CsrOperator::apply), N complex values each in `mem`. */
int mstab_operator_apply_z(mstab_context* ctx, const mstab_operator* op, const double* x_re_im, double* y_re_im,
                           int32_t mem);
int mstab_recycle_create_z(mstab_context* ctx, int64_t n, int64_t s, const double* p_re_im, const double* u_re_im,
                           const double* v_re_im, int32_t mem, const double* omega_re_im, int64_t omega_count,
                           int64_t level_j, uint64_t fingerprint, mstab_recycle** out);
/* P, U, V as N x s column-major complex blocks on the host (any may be NULL), omega as (re, im) pairs. */
int mstab_recycle_download_z(mstab_context* ctx, const mstab_recycle* rd, double* p_re_im, double* u_re_im,
                             double* v_re_im, double* omega_re_im);
int mstab_solve_z(mstab_context* ctx, const mstab_operator* op, const double* b_re_im, const double* x0_re_im,
                  int32_t mem, const mstab_solver_config* cfg, const mstab_recycle* recycle,
                  const mstab_fetch_policy* fetch, mstab_result** out);
int mstab_result_x_z(mstab_context* ctx, const mstab_result* res, double* x_re_im, int32_t mem);

/* ---- sequence-driver helpers (the caller side of the path: run_sequence's RHS rules) ------- */
/* b = h2 * (x / dt + f) (implicit-Euler chain of the BASELINE conv-diff configs) and
 * b = x + alpha * g (banded-random chain). mem = DEVICE runs on the context stream (synchronised);
 * HOST loops on the host. Both evaluate in exactly this rounding order. */
int mstab_harness_euler_rhs(mstab_context* ctx, int64_t n, const double* x, const double* f,
                            double dt, double h2, double* b, int32_t mem);
int mstab_harness_axpby(mstab_context* ctx, int64_t n, const double* x, const double* g,
                        double alpha, double* b, int32_t mem);

/* ---- row-sharded solves across the GPUs of one node -----------------------
 * One process (one context) per GPU owns a contiguous row slab of A and of every N-vector (x, b,
 * r, P, U, V); the SpMV exchanges halo rows with the neighbouring slabs and every length-N
 * reduction is summed over the ranks (the replicated s x s / least-squares steps then see
 * bit-identical inputs on every rank). The reference is single-process; this is the
 * B200 extension of its solve loop, with the same results up to reduction order.
 *
 * Protocol: rank 0 calls mstab_nccl_unique_id and distributes the 128 bytes; every rank calls
 * mstab_context_set_comm_nccl, then mstab_operator_create_csr_slab with the FULL host CSR and the
 * slab boundaries. From then on every N-length argument of this context (b, x0, x, recycle
 * P/U/V) holds the rank's own rows only, and mstab_solve / validate are collective calls.
 * mstab_context_set_comm_host plugs in a host runtime instead (MPI, gloo...): device buffers are
 * staged through pinned host memory and the callbacks move them (not CUDA-graph capturable). */
typedef struct mstab_host_comm {
  void* user;
  /* in-place sum over the ranks of `count` doubles (host memory); return 0 on success */
  int32_t (*allreduce_sum)(void* user, double* buf, int64_t count);
  /* rank-major concatenation: out[r * count ..] = rank r's in[0 .. count) */
  int32_t (*allgather)(void* user, const double* in, double* out, int64_t count);
  /* send send_bufs[i] (send_counts[i] doubles) to send_peers[i] and receive recv_counts[j]
   * doubles from recv_peers[j] into recv_bufs[j], all concurrently (deadlock-free) */
  int32_t (*halo_exchange)(void* user, int32_t nsend, const int32_t* send_peers,
                           const double* const* send_bufs, const int64_t* send_counts, int32_t nrecv,
                           const int32_t* recv_peers, double* const* recv_bufs,
                           const int64_t* recv_counts);
} mstab_host_comm;

int mstab_nccl_unique_id(uint8_t out[128]);
int mstab_context_set_comm_nccl(mstab_context* ctx, int32_t rank, int32_t world, const uint8_t id[128]);
int mstab_context_set_comm_host(mstab_context* ctx, int32_t rank, int32_t world,
                                const mstab_host_comm* fns);
/* rank / world of the context (0 / 1 without a communicator) */
int mstab_context_comm_info(mstab_context* ctx, int32_t* rank, int32_t* world);
/* Row slab [slab_starts[rank], slab_starts[rank+1]) of the n x n CSR matrix. slab_starts has
 * world + 1 ascending entries (0 .. n). Validation and the FNV fingerprint cover the whole
 * matrix (csr.cpp:11-43), so every rank's operator carries the reference's fingerprint. */
int mstab_operator_create_csr_slab(mstab_context* ctx, int64_t n, const int64_t* row_ptr,
                                   const int64_t* col_idx, const double* values,
                                   const int64_t* slab_starts, mstab_operator** out);
/* The same slab from the rank's OWN rows, for systems no rank can hold whole (c4: 1.5e9 entries):
 * row_ptr (local, from 0, n_local + 1 entries), col_idx (GLOBAL column indices) and values of rows
 * [slab_starts[rank], slab_starts[rank+1]). What the global form derives from the whole matrix is
 * passed in instead:
 *   col_spans    2 x world: [lo_r, hi_r) = the column range rank r's rows reference (each rank
 *                computes its own pair and the caller allgathers them); the halo plans of all ranks
 *                follow from these and match by construction;
 *   fingerprint  the reference checksum of the GLOBAL matrix (csr.cpp:28-43), folded over the ranks
 *                with mstab_fnv_* below (three relays: row_ptr, col_idx, values), or any value
 *                agreed by all ranks when .mrd interchange with the reference is not needed. */
int mstab_operator_create_csr_slab_local(mstab_context* ctx, int64_t n_global, const int64_t* slab_starts,
                                         const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                                         const int64_t* col_spans, uint64_t fingerprint, mstab_operator** out);
/* The reference's CSR checksum as a resumable fold (FNV-1a over dims, every row_ptr entry, every
 * col_idx entry, every value as complex<double>): h = mstab_fnv_begin(n, n, nnz); then in rank
 * order h = mstab_fnv_fold_index(h, row_ptr_local + (rank ? 1 : 0), count, first_entry_of_slab)
 * (local offsets rebased by `add`), again in rank order over col_idx (add = 0), and again over the
 * values. The state is 8 bytes: pass it to the next rank between folds. */
uint64_t mstab_fnv_begin(int64_t n_rows, int64_t n_cols, int64_t nnz);
uint64_t mstab_fnv_fold_index(uint64_t h, const int64_t* v, int64_t count, int64_t add);
uint64_t mstab_fnv_fold_values(uint64_t h, const double* values, int64_t count);
/* First global row of the operator's slab (0 for a whole-matrix operator); size() is the
 * number of local rows. */
int64_t mstab_operator_row_begin(const mstab_operator* op);
int64_t mstab_operator_global_size(const mstab_operator* op);
/* Interior rows [lo, hi) of a row slab (local indices): rows with no column outside the owned rows,
 * computed while the halo exchange of a split product is in flight (0, 0 for a non-slab operator). */
void mstab_operator_interior_rows(const mstab_operator* op, int64_t* lo, int64_t* hi);

/* ---- evidence hooks (no reference counterpart; the reference implementation reports zeros) --- */
/* Number of kernel launches issued by this library since load. */
uint64_t mstab_launch_count(void);
/* Per-launch CUDA-event timing by kernel class, tagged with ALGORITHMIC bytes. */
typedef struct mstab_kernel_class_stats {
  int64_t launches;
  double total_ms;
  double total_bytes;
} mstab_kernel_class_stats;
int mstab_profiling_enable(int32_t on);
int32_t mstab_profiling_read(mstab_kernel_class_stats* out, int32_t cap); /* returns #classes */
void mstab_profiling_reset(void);
const char* mstab_kernel_class_name(int32_t cls);

#ifdef __cplusplus
}
#endif

#endif /* MSTAB_B200_H */
