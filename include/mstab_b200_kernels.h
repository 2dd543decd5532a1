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

/* arnoldi_init with the padding draws supplied by the caller: fill(user, out, count) must write
 * `count` standard normal draws (the reference takes them from the caller's std::mt19937_64
 * through one std::normal_distribution per call, idrstab.cpp:60,77-78; the drop-in shim passes
 * exactly that). Only called on a happy breakdown. */
typedef void (*mstab_normal_fill_fn)(void* user, double* out, int64_t count);
int mstab_kernel_arnoldi_cb(mstab_context* ctx, const mstab_operator* op, const double* r0, int64_t s,
                            mstab_normal_fill_fn fill, void* user, double* u, double* v, int64_t* mv_cost);

/* bicg_projection (idrstab.cpp:89-94): gamma = (P^H block)^-1 P^H target; p and block are n x s.
 * MSTAB_E_SINGULAR when the projection block is singular (solve_small). */
int mstab_kernel_bicg_projection(mstab_context* ctx, int64_t n, int64_t s, const double* p,
                                 const double* block, const double* target, double* gamma);

/* The two reductions of bicg_projection without the solve: m = P^T block (s x s, column-major) and
 * g = P^T target (s). The shim assembles the complex P^H block / P^H target of a complex call from
 * four of these (real and imaginary parts) and solves the s x s system with solve_small. */
int mstab_kernel_projection_gram(mstab_context* ctx, int64_t n, int64_t s, const double* p,
                                 const double* block, const double* target, double* m, double* g);

/* level_iteration (idrstab.cpp:105-152), level k of IterationState (idrstab.hpp:38-46):
 *   x0        n               in/out
 *   r_levels  n x (k + 2)     r^(0..k) on entry, r^(0..k+1) on return
 *   v_levels  n x s x (k + 3) V^(-1..k) on entry (v_levels[i] = level i - 1), V^(-1..k+1) on return
 * Costs s + 1 operator applications. MSTAB_E_SINGULAR on a singular projection block. */
int mstab_kernel_level_iteration(mstab_context* ctx, const mstab_operator* op, int64_t s, int64_t k,
                                 const double* p, double* x0, double* r_levels, double* v_levels);

/* poly_combination (idrstab.cpp:154-191) of a state with levels r^(0..ell), V^(-1..ell):
 * x, r (n), u, v (n x s), tau (ell), *tail_perturbed. MSTAB_E_RANK when the stabilisation block
 * lost rank (least_squares_tall). */
int mstab_kernel_poly_combination(mstab_context* ctx, int64_t n, int64_t s, int64_t ell, const double* x0,
                                  const double* r_levels, const double* v_levels, double* x, double* r,
                                  double* u, double* v, double* tau, int32_t* tail_perturbed);

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
