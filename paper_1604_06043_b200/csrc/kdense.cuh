// kdense.cuh — the small dense steps shared by the streaming kernels (kls.cu, kpoly.cu) and the
// persistent cycle kernel (kpersist.cu): the least-squares tails (CholeskyQR2 factors, Givens
// absorption, the reference's solve / rank test / tail guard) and the poly / prologue tail.
#pragma once
#include "kcommon.cuh"

namespace mstab_b200 {
namespace {

// ---------------------------------------------------------------------------------------------
// Least squares by Givens TSQR of [Z | r0] (one HBM pass). R is (L+1)x(L+1) upper triangular,
// packed row-major: row j holds columns j..L at offset j*(L+1) - j*(j-1)/2.
template <int L>
struct Tri {
  static constexpr int D = L + 1;
  static constexpr int NR = D * (D + 1) / 2;
  __host__ __device__ static constexpr int at(int j, int m) { return j * D - j * (j - 1) / 2 + (m - j); }
};

// Absorbs row w (zero before column `start`) into R with Givens rotations.
template <int L>
__device__ __forceinline__ void givens_absorb(double (&R)[Tri<L>::NR], double (&w)[L + 1], int start) {
#pragma unroll
  for (int j = 0; j <= L; ++j) {
    if (j < start) continue;
    const double bj = w[j];
    if (bj == 0.0) continue;
    const double aj = R[Tri<L>::at(j, j)];
    const double h2 = aj * aj + bj * bj;
    const double inv = rsqrt(h2);  // one reciprocal square root instead of sqrt + divide
    const double r = h2 * inv;
    const double c = aj * inv, sn = bj * inv;
    R[Tri<L>::at(j, j)] = r;
#pragma unroll
    for (int m = j + 1; m <= L; ++m) {
      const double t = R[Tri<L>::at(j, m)];
      R[Tri<L>::at(j, m)] = c * t + sn * w[m];
      w[m] = c * w[m] - sn * t;
    }
  }
}

template <int L>
__device__ __forceinline__ void absorb_tri(double (&R)[Tri<L>::NR], const double (&B)[Tri<L>::NR]) {
#pragma unroll
  for (int j = 0; j <= L; ++j) {
    double w[L + 1];
#pragma unroll
    for (int m = 0; m <= L; ++m) w[m] = (m < j) ? 0.0 : B[Tri<L>::at(j, m)];
    givens_absorb<L>(R, w, j);
  }
}

template <int L>
__device__ void ls_finalize(const double* Rf, const double* cn, int s, DevState* ds) {
  // Rf: merged R (packed), cn: column sums of squares of Z (L values)
  double max_colnorm = 0.0;
  for (int j = 0; j < L; ++j) max_colnorm = dmax_ref(max_colnorm, sqrt(cn[j]));
  double min_diag = INFINITY;
  for (int k = 0; k < L; ++k) {
    const double d = fabs(Rf[Tri<L>::at(k, k)]);
    min_diag = (d < min_diag) ? d : min_diag;
  }
  if (min_diag < 1e-13 * max_colnorm) {  // kernels.cpp:83-84
    set_breakdown(ds, kBreakRank, L * (s + 1));
    return;
  }
  double tau[L];
  for (int k = 0; k < L; ++k) tau[k] = Rf[Tri<L>::at(k, L)];
  for (int k = L - 1; k >= 0; --k) {  // kernels.cpp:87-91
    for (int j = k + 1; j < L; ++j) tau[k] = tau[k] - Rf[Tri<L>::at(k, j)] * tau[j];
    tau[k] = tau[k] / Rf[Tri<L>::at(k, k)];
  }
  for (int k = 0; k < L; ++k) ds->scal[32 + k] = tau[k];  // raw least-squares solution
  // tail guard (idrstab.cpp:163-174)
  double tmax = 0.0;
  for (int k = 0; k < L; ++k) tmax = dmax_ref(tmax, fabs(tau[k]));
  int pert = 0;
  double& tail = tau[L - 1];
  if (fabs(tail) < 1e-12 * tmax || tmax == 0.0) {
    const double target = tmax > 0.0 ? 1e-12 * tmax : 1e-12;
    tail = fabs(tail) > 0.0 ? tail * (target / fabs(tail)) : target;
    pert = 1;
  }
  for (int k = 0; k < L; ++k) ds->st.tau[k] = tau[k];
  ds->st.tail_perturbed = pert;
}

struct LsArgs {
  const double* r[kMaxEll + 1];  // r^(0..L)
};

// ---- CholeskyQR2 (two streaming passes, no Q stored) --------------------------------------------
// Pass 1: G1 = Z^T Z of Z = [r^(1..L) | r^(0)] (packed upper, one deterministic reduction), then
// R1 = chol(G1) and R1^-1. Pass 2: G2 = Q^T Q with Q = Z R1^-1 formed row by row, R2 = chol(G2),
// R = R2 R1 (the R factor of Z to working accuracy while cond(Z) <~ 1e8). Used only when every
// Cholesky pivot of G1 keeps more than kCholKeep of its column's squared norm;
// otherwise pass 2 runs the one-pass Givens TSQR instead (same launch, ls_mode = 0), which also
// owns the rank-deficiency regime of the reference's test (kernels.cpp:83-84). Either way the
// least-squares solve, rank test and tail guard are ls_finalize's.
// A Cholesky pivot must keep more than kCholKeep of its column's squared norm (each column adds
// a direction at least 1e-3 of its length away from the previous ones), else the Givens path.
constexpr double kCholKeep = 1e-6;

template <int L>
__device__ bool chol_packed(const double* G, double* R) {
  constexpr int D = L + 1;
  for (int j = 0; j < D; ++j) {
    double d = G[Tri<L>::at(j, j)];
    for (int i = 0; i < j; ++i) d = d - R[Tri<L>::at(i, j)] * R[Tri<L>::at(i, j)];
    if (!(d > kCholKeep * G[Tri<L>::at(j, j)]) || !isfinite(d)) return false;
    const double rjj = sqrt(d);
    R[Tri<L>::at(j, j)] = rjj;
    for (int m = j + 1; m < D; ++m) {
      double t = G[Tri<L>::at(j, m)];
      for (int i = 0; i < j; ++i) t = t - R[Tri<L>::at(i, j)] * R[Tri<L>::at(i, m)];
      R[Tri<L>::at(j, m)] = t / rjj;
    }
  }
  return true;
}

template <int L>
__device__ void tri_inverse(const double* R, double* Ri) {
  constexpr int D = L + 1;
  for (int j = D - 1; j >= 0; --j) {
    Ri[Tri<L>::at(j, j)] = 1.0 / R[Tri<L>::at(j, j)];
    for (int m = j + 1; m < D; ++m) {
      double t = 0.0;
      for (int k = j + 1; k <= m; ++k) t = t + R[Tri<L>::at(j, k)] * Ri[Tri<L>::at(k, m)];
      Ri[Tri<L>::at(j, m)] = -t / R[Tri<L>::at(j, j)];
    }
  }
}

// Dense tail of pass 1 (thread 0): R1, R1^-1, column norms, path choice.
template <int L>
__device__ void ls_pass1_tail(const double* G, DevState* ds) {
  for (int j = 0; j < L; ++j) ds->ls_cn[j] = G[Tri<L>::at(j, j)];
  double R[Tri<L>::NR];
  if (chol_packed<L>(G, R)) {
    for (int i = 0; i < Tri<L>::NR; ++i) ds->ls_r1[i] = R[i];
    tri_inverse<L>(R, ds->ls_r1inv);
    ds->ls_mode = 1;
  } else {
    ds->ls_mode = 0;
  }
}

// Dense tail of the CholeskyQR2 pass 2 (thread 0): R = chol(G2) R1, then the reference's solve.
template <int L>
__device__ void ls_finalize(const double* Rf, const double* cn, int s, DevState* ds);
template <int L>
__device__ void ls_pass2_tail(const double* G2, int s, DevState* ds) {
  constexpr int D = L + 1, NR = Tri<L>::NR;
  double R2[NR], R[NR];
  if (chol_packed<L>(G2, R2)) {
    for (int j = 0; j < D; ++j)
      for (int m = j; m < D; ++m) {
        double t = 0.0;
        for (int k = j; k <= m; ++k) t = t + R2[Tri<L>::at(j, k)] * ds->ls_r1[Tri<L>::at(k, m)];
        R[Tri<L>::at(j, m)] = t;
      }
  } else {  // cannot happen for a well-conditioned Q; keep the first factor
    for (int i = 0; i < NR; ++i) R[i] = ds->ls_r1[i];
  }
  double cn[L];
  for (int j = 0; j < L; ++j) cn[j] = ds->ls_cn[j];
  ls_finalize<L>(R, cn, s, ds);
}


// The dense tail of poly / prologue (run by every thread of one CTA): ||r||, g = P^H r,
// Ma = P^H V and the next cycle's gamma_0 = (P^H V)^-1 P^H r, staged in parallel and solved by
// one warp in shared memory.
template <int S>
__device__ void poly_tail(const double* redv, DevState* ds) {
  __shared__ double lu[kMaxS * kMaxS];
  __shared__ double vin[kMaxS], vout[kMaxS];
  __shared__ int ok;
  const int t = threadIdx.x;
  if (t == 0) ds->st.resnorm = sqrt(redv[0]);
  if (t < S) {
    ds->g[t] = redv[1 + t];
    vin[t] = redv[1 + t];
  }
  for (int i = t; i < S * S; i += blockDim.x) {
    ds->Ma[i] = redv[1 + S + i];
    lu[i] = redv[1 + S + i];
  }
  __syncthreads();
  if (t < 32) {
    const bool r2 = warp_lu_solve<S>(S, lu, vin, vout);
    if (t == 0) ok = r2 ? 1 : 0;
  }
  __syncthreads();
  if (t < S) ds->gamma[t] = vout[t];
  if (t == 0) ds->st.pending_singular = ok ? 0 : 1;
}


}  // namespace
}  // namespace mstab_b200
