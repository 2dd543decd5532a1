/*
 * mstab_oracle.h — TEST INFRASTRUCTURE ONLY: plain-C, real-fp64 restatement of the reference's
 * Mstab solve path (proj/core/src/{idrstab,kernels,types,dense,csr,recycle,baselines}.cpp), used
 * by tests/ as a second oracle next to the compiled reference (oracle/_ref). For real inputs the
 * reference's complex<double> arithmetic keeps every imaginary part at +0.0, so this real
 * restatement, evaluated in the same operation order without FMA contraction, reproduces the
 * reference bit-for-bit; tests/test_oracle_pin.py pins that against golden vectors produced by
 * the reference itself (tests/golden/, tests/golden/make_golden.py).
 *
 * Never linked into the product library.
 */
#ifndef MSTAB_ORACLE_H
#define MSTAB_ORACLE_H

#include <stdint.h>

typedef struct {
  int64_t n;
  const int64_t* row_ptr;
  const int64_t* col_idx;
  const double* values;
} orc_csr;

typedef struct {
  int64_t s, ell;
  double tol;
  int64_t max_mv;
  int32_t true_residual;
  int32_t _pad;
  uint64_t seed;
} orc_cfg;

typedef struct {
  int64_t n, s, level_j;
  uint64_t fingerprint;
  double* p;        /* n x s column-major */
  double* u;
  double* v;
  int64_t omega_count;
  double* omega;    /* re, im pairs */
} orc_recycle;

typedef struct {
  int32_t status;   /* 0 converged, 1 maxmv, 2 breakdown */
  int32_t has_fetched;
  int64_t h_mv, h_mv_aux, h_rd, cycles;
  double bnorm, final_resnorm;
  double* x;
  int64_t hist_len;
  int64_t* hist;    /* hist_len x (cycle, mv, level) */
  double* hist_resnorm;
  int64_t tau_len;
  double* tau;      /* real tau per cycle, flattened */
  orc_recycle final_data;
  orc_recycle fetched;
  char reason[128];
} orc_result;

/* Returns 0 or the MSTAB_E_* code of the exception the reference would throw. */
int orc_solve(const orc_csr* a, const double* b, const double* x0, const orc_cfg* cfg,
              const orc_recycle* recycle, int32_t fetch_kind, int64_t fetch_cycle, orc_result* out);
void orc_result_free(orc_result* r);

uint64_t orc_fingerprint(const orc_csr* a);
void orc_spmv(const orc_csr* a, const double* x, double* y);
int orc_solve_small(int64_t s, const double* m, const double* rhs, double* x);
int orc_least_squares(int64_t n, int64_t ell, const double* z, const double* r, double* tau);
int orc_cut_space(int64_t n, int64_t s, uint64_t seed, double* p);
int orc_arnoldi(const orc_csr* a, const double* r0, int64_t s, uint64_t rng_seed, double* u, double* v);
void orc_normal_draws(uint64_t seed, int64_t count, double* out);
int orc_validate(const orc_csr* a, const orc_recycle* rd, double* max_dev, double* sigma_ratio);

#endif
