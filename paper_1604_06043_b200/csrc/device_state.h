// device_state.h — POD structures shared by the sm_100a kernels (kernels.cu) and the host
// orchestration (solver.cpp). No CUDA headers here so g++ can include it.
//
// Layout conventions:
//   * every N-vector / block column is fp64 with column stride `ld` (N rounded up to 64);
//   * an N x s block is s consecutive columns (column-major, like DenseMatrix, dense.hpp:23-24);
//   * CSR is int32 row_ptr / col_idx + fp64 values (all BASELINE configs have nnz < 2^31).
#pragma once
#include <cstdint>

namespace mstab_b200 {

constexpr int kMaxS = 16;    // s in {1..16} (BASELINE c5 sweep tops at 16)
constexpr int kMaxEll = 8;   // ell in {1..8}
constexpr int kBlock = 256;  // threads per CTA for every streaming kernel
constexpr int kMaxGrid = 148 * 8;
constexpr int kMaxXred = 2 + 2 * kMaxS * kMaxS + 6;  // largest split payload (validate)

// Breakdown codes written by the device finalizers (idrstab.cpp:290-293 reasons).
// kBreakFallback is not a breakdown of the method: the persistent cycle kernel (kpersist.cu) asks
// the host to rerun the cycle on the stream-of-kernels path (its least squares left the
// CholeskyQR2 regime); the host never reports it.
enum : int32_t { kBreakNone = 0, kBreakSingular = 1, kBreakRank = 2, kBreakFallback = 3 };

// Small, per-solve scalar state living in device memory. The "status" head is copied back to
// the host once per cycle (one small D2H); the rest stays on the device.
struct CycleStatus {
  double resnorm;          // ||r|| after the cycle (norm2, types.cpp:9-13)
  double tau[kMaxEll];     // stabilisation coefficients of the cycle (after the tail guard)
  int32_t breakdown;       // kBreak*
  int32_t mv_at_breakdown; // operator applications done in the cycle before the failing solve
  int32_t tail_perturbed;  // PolyOut::tail_perturbed (idrstab.cpp:165-174)
  int32_t pending_singular;// gamma_0 for the NEXT cycle came out singular (raised when it starts)
};

// What a persistent cycle writes straight into mapped host memory (one slot per in-flight cycle):
// the cycle's status and, last, the launch's sequence number the host polls for.
struct HostCycleSlot {
  CycleStatus st;
  volatile uint64_t seq;
};

struct DevState {
  CycleStatus st;
  double Ma[kMaxS * kMaxS];    // P^H V^(k), column-major s x s (ld = s)
  double Mn[kMaxS * kMaxS];    // P^H V^(k+1), filled column by column during step (c)
  double g[kMaxS];             // P^H r^(k)
  double rhs[kMaxS];           // P^H r^(k+1)
  double gamma[kMaxEll * kMaxS];  // BiCG coefficients per level k (bicg_projection), row k
  double eta[kMaxS * kMaxS];   // eta_q of the current level, row q = eta for column q
  double scal[64];             // misc reduced scalars (norms, dots for init/validate)
  double gram[2 * kMaxS * kMaxS];  // validate: P^H P then V^H V
  // Row-sharded solves (comm world > 1): the last CTA of a reduction kernel leaves its rank-local
  // totals here instead of running the dense step; the host allreduces (or allgathers) them over
  // the ranks and launches the matching finaliser kernel (kernels.h launch_fin_*).
  double xred[kMaxXred];
  double xred2[kMaxS + 1];  // totals of the interior launch of a split SpMV (Reducer::xbase)
  // least squares (kls.cu): CholeskyQR2 state between its two passes
  int32_t ls_mode;                      // 1: CholeskyQR2 path, 0: Givens TSQR fallback
  int32_t _pad_ls;
  double ls_r1[(kMaxEll + 1) * (kMaxEll + 2) / 2];     // first Cholesky factor (packed upper)
  double ls_r1inv[(kMaxEll + 1) * (kMaxEll + 2) / 2];  // its inverse
  double ls_cn[kMaxEll];                // column sums of squares of Z
  // Set by the persistent cycle kernel when its cycle ended the solve (converged below the
  // threshold it was given, or broke down): a cycle launched speculatively behind it returns at once
  // without touching anything (solver.cpp, pipelined persistent cycles). Cleared by reset_status.
  int32_t stop;
  uint32_t ticket;             // last-CTA-done counter (reset by the finaliser)
  uint32_t tile_next;          // dynamic tile scheduler counter (reset by the finaliser)
};

}  // namespace mstab_b200
