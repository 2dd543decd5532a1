/*
 * mstab_b200_kernels.h — kernel-level entry points of the drop-in, for parity tests of the dense
 * steps of the solve loop. Both libraries (libmstab_b200.so, oracle/_ref/libmstab_ref.so) export
 * them; the B200 versions run the same device code the solve loop runs.
 * All matrices are column-major real fp64 host arrays.
 */
#ifndef MSTAB_B200_KERNELS_H
#define MSTAB_B200_KERNELS_H

#include "mstab_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* solve_small (kernels.cpp:150-154): x = M^-1 rhs, s x s; MSTAB_E_SINGULAR on pivot collapse. */
int mstab_kernel_solve_small(mstab_context* ctx, int64_t s, const double* m, const double* rhs,
                             double* x);

/* least_squares_tall (kernels.cpp:52-93): tau = argmin ||r - Z tau||, Z n x ell;
 * MSTAB_E_RANK when the block lost rank, MSTAB_E_DIMENSION unless n >= ell >= 1. */
int mstab_kernel_least_squares(mstab_context* ctx, int64_t n, int64_t ell, const double* z,
                               const double* r, double* tau);

/* make_cut_space (baselines.cpp:36-47) for a real problem: P (n x s) orthonormal, seeded. */
int mstab_kernel_cut_space(mstab_context* ctx, int64_t n, int64_t s, uint64_t seed, double* p);

/* arnoldi_init (idrstab.cpp:45-87) with std::mt19937_64 rng(rng_seed) for the padding draws:
 * U (n x s), V = A U, *mv_cost = s. */
int mstab_kernel_arnoldi(mstab_context* ctx, const mstab_operator* op, const double* r0, int64_t s,
                         uint64_t rng_seed, double* u, double* v, int64_t* mv_cost);

/* Micro-benchmark of one kernel class of the cycle on synthetic data shaped like `op` with
 * (s, ell): `iters` back-to-back launches timed with CUDA events; *us = mean microseconds per
 * launch, *bytes = algorithmic bytes per launch. kind: 0 SpMV + P^H + LU finalize, 1 top
 * rebuild, 2 level update, 3 deferred levels (k = ell-1), 4 poly_combination, 5 least squares.
 * (Reference implementation: MSTAB_E_CONFIG.) */
int mstab_kernel_bench(mstab_context* ctx, const mstab_operator* op, int32_t kind, int64_t s,
                       int64_t ell, int32_t iters, double* us, double* bytes);

/* Developer probes: op 0 resets and binds the in-kernel timeline slots, op 1 unbinds and copies
 * the 32 slots to out (globaltimer ns / clock64). Only a timeline build (make timeline) records;
 * the product build leaves out untouched. (Reference implementation: MSTAB_E_CONFIG.) */
int mstab_timeline(mstab_context* ctx, int32_t op, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif
