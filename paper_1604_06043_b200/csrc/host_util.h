// host_util.h — host-side pieces of the drop-in that are not per-cycle device work:
// error classes mirroring errors.hpp, the reference's FNV-1a operator fingerprint, the .mrd
// byte format, the small Jacobi eigensolver used by validate(), and omega extraction.
#pragma once
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mstab_b200 {

// Error carrying the C-ABI code of the reference exception class it stands for (errors.hpp).
struct Error : std::runtime_error {
  int code;
  int64_t row = -1;  // ZeroPivot::row() (errors.hpp:39-45) for MSTAB_E_ZEROPIVOT
  Error(int c, const std::string& msg, int64_t r = -1) : std::runtime_error(msg), code(c), row(r) {}
};

// FNV-1a over the reference CsrMatrix byte layout (csr.cpp:28-43): dims {n_rows, n_cols, nnz}
// as 3 x u64, row_ptr and col_idx widened to u64 (size_t), values as complex<double> with a
// +0.0 imaginary part. Zero bytes are folded in as multiplications by powers of the prime.
uint64_t fnv_csr_fingerprint(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                             const double* values, int64_t nnz);
// Resumable form of the same fold (a row-distributed matrix is hashed in three relays): the
// dims, then row_ptr entries (each + add: a slab's local offsets rebased to global), col_idx, values.
uint64_t fnv_begin(int64_t n_rows, int64_t n_cols, int64_t nnz);
uint64_t fnv_fold_u64(uint64_t h, const int64_t* v, int64_t count, int64_t add);
uint64_t fnv_fold_values(uint64_t h, const double* values, int64_t count);

// Cyclic Jacobi eigenvalues (ascending) of a real symmetric s x s matrix (column-major);
// the real specialisation of hermitian_eigenvalues (kernels.cpp:156-208).
std::vector<double> symmetric_eigenvalues(const double* h, int s);

// extract_omegas (idrstab.cpp:28-41): ell = 1 -> tau_1; ell = 2 -> roots of w^2 - tau1 w - tau2.
bool extract_omegas(const std::vector<double>& tau, std::vector<std::complex<double>>& out);

// .mrd file (recycle.cpp:85-192): 56-byte header, P, U, V column-major (fp64 when the real flag
// is set, re/im pairs otherwise), then omega as re/im pairs.
struct MrdData {
  int64_t n = 0, s = 0, level_j = 0;
  uint64_t fingerprint = 0;
  std::vector<double> p, u, v;                 // real parts, n*s each
  std::vector<std::complex<double>> omega;
};
void mrd_write(const std::string& path, const MrdData& d);
MrdData mrd_read(const std::string& path);  // throws ParseError / IoError / NotReal

// mt19937_64 + std::normal_distribution<double>(0,1) draws in the reference's order.
struct NormalStream;
NormalStream* normal_stream_create(uint64_t seed);
void normal_stream_fill(NormalStream* st, double* out, int64_t count);
void normal_stream_destroy(NormalStream* st);

}  // namespace mstab_b200
