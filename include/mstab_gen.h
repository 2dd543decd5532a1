/*
 * mstab_gen.h — builder-defined synthetic problem generators for the BASELINE configs
 * (SURVEY.md §8(d) "Common generator conventions"). Host C++ (libmstab_gen.so), used identically
 * by the reference driver (oracle/_ref), the C restatement tests and the B200 bench, so every
 * implementation sees bit-identical matrices and right-hand sides. No external benchmark data.
 *
 * Convection-diffusion: interior unknowns of an n^d grid, lexicographic idx = (k*n + j)*n + i
 * (x fastest), h = 1/(n+1), homogeneous Dirichlet (out-of-domain neighbours dropped), central
 * -Laplacian, first-order upwind beta.grad for beta > 0, implicit Euler multiplied by h^2:
 *   A = h^2 (I/dt + L),   b_{i+1} = h^2 (x_i/dt + f).
 * Stencils: 5-point (d=2), 7-point (d=3), 27-point (d=3: L27 u = (26 u_c - sum_26 u_nb)/(9h^2)
 * plus face upwind convection).
 */
#ifndef MSTAB_GEN_H
#define MSTAB_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Number of nonzeros of the conv-diff matrix (dim 2 with stencil 5, dim 3 with 7 or 27). */
int64_t mstab_gen_convdiff_nnz(int32_t dim, int64_t n, int32_t stencil);
/* Fills row_ptr (N+1), col_idx (nnz), values (nnz); N = n^dim. beta has 3 entries. */
int mstab_gen_convdiff(int32_t dim, int64_t n, int32_t stencil, const double* beta, double dt,
                       int64_t* row_ptr, int64_t* col_idx, double* values);
/* Rows [row0, row1) of the same matrix: row_ptr local (from 0, row1 - row0 + 1 entries), col_idx
 * GLOBAL column indices. Returns the entry count of the range; with row_ptr = col_idx = values =
 * NULL it only counts (a rank of a row-sharded run generates its own slab: no process holds the
 * global matrix). */
int64_t mstab_gen_convdiff_rows(int32_t dim, int64_t n, int32_t stencil, const double* beta, double dt,
                                int64_t row0, int64_t row1, int64_t* row_ptr, int64_t* col_idx,
                                double* values);
/* std::mt19937_64(seed) + std::uniform_real_distribution<double>(0,1): `count` draws. For the
 * conv-diff sequences the first N draws are x0 and the next N are f. */
int mstab_gen_uniform(uint64_t seed, int64_t count, double* out);
/* b = h2 * (x / dt + f)   (the implicit-Euler right-hand side; same rounding order as the GPU). */
void mstab_gen_euler_rhs(int64_t n, const double* x, const double* f, double dt, double h2, double* b);

/* Random banded nonsymmetric matrix (BASELINE config 3): per row the diagonal plus nnz_per_row-1
 * distinct off-diagonal columns drawn uniformly in [max(0,i-hw), min(N-1,i+hw)], sorted; values
 * U[-1,1) in sorted order; diagonal = 1.1 * row abs-sum; std::mt19937_64(seed). */
int mstab_gen_banded(int64_t n, int32_t nnz_per_row, int64_t half_width, uint64_t seed,
                     int64_t* row_ptr, int64_t* col_idx, double* values);
/* make_rhs sinewave (harness.cpp:72-77): v[k-1] = sin(2*pi*k/N), k = 1..N (libm sin). */
void mstab_gen_sinewave(int64_t n, double* out);
/* g ~ N(0,1), N draws from std::mt19937_64(seed) + std::normal_distribution<double>. */
int mstab_gen_normal(uint64_t seed, int64_t count, double* out);

#ifdef __cplusplus
}
#endif

#endif
