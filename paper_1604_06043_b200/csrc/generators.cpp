// generators.cpp — see include/mstab_gen.h. Host-only; builder-defined stand-ins for the
// BASELINE configs (no external data set is involved).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "../../include/mstab_gen.h"

namespace {

struct Nb {
  int dx, dy, dz;
};

// Neighbour offsets of each stencil in increasing column order (z slowest).
std::vector<Nb> stencil_offsets(int dim, int stencil) {
  std::vector<Nb> out;
  if (dim == 2 && stencil == 5) {
    out = {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}};
  } else if (dim == 3 && stencil == 7) {
    out = {{0, 0, -1}, {0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  } else if (dim == 3 && stencil == 27) {
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) out.push_back({dx, dy, dz});
  }
  return out;
}

}  // namespace

extern "C" {

int64_t mstab_gen_convdiff_nnz(int32_t dim, int64_t n, int32_t stencil) {
  if (dim == 2 && stencil == 5) return 5 * n * n - 4 * n;
  if (dim == 3 && stencil == 7) return 7 * n * n * n - 6 * n * n;
  if (dim == 3 && stencil == 27) return (3 * n - 2) * (3 * n - 2) * (3 * n - 2);
  return -1;
}

int mstab_gen_convdiff(int32_t dim, int64_t n, int32_t stencil, const double* beta, double dt,
                       int64_t* row_ptr, int64_t* col_idx, double* values) {
  const int64_t N = dim == 3 ? n * n * n : n * n;
  return mstab_gen_convdiff_rows(dim, n, stencil, beta, dt, 0, N, row_ptr, col_idx, values) < 0 ? -3 : 0;
}

int64_t mstab_gen_convdiff_rows(int32_t dim, int64_t n, int32_t stencil, const double* beta, double dt,
                                int64_t row0, int64_t row1, int64_t* row_ptr, int64_t* col_idx,
                                double* values) {
  const std::vector<Nb> offs = stencil_offsets(dim, stencil);
  if (offs.empty() || n < 1) return -3;
  const double h = 1.0 / (double)(n + 1);
  const double h2 = h * h;
  const int64_t nz = dim == 3 ? n : 1;
  // coefficients (already multiplied by h^2)
  double diag = h2 / dt;
  double off_plain, off_upwind[3];
  if (stencil == 27) {
    diag += 26.0 / 9.0;
    off_plain = -1.0 / 9.0;
  } else {
    diag += 2.0 * dim;
    off_plain = -1.0;
  }
  for (int d = 0; d < dim; ++d) {
    diag += h * beta[d];
    off_upwind[d] = off_plain - h * beta[d];
  }
  int64_t k_nz = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (int64_t row = row0; row < row1; ++row) {
      const int64_t x = row % n, y = (row / n) % n, z = row / (n * n);
      {
        for (const Nb& o : offs) {
          const int64_t xx = x + o.dx, yy = y + o.dy, zz = z + o.dz;
          if (xx < 0 || xx >= n || yy < 0 || yy >= n || zz < 0 || zz >= nz) continue;
          double v;
          const int nonzero_axes = (o.dx != 0) + (o.dy != 0) + (o.dz != 0);
          if (nonzero_axes == 0) {
            v = diag;
          } else if (nonzero_axes == 1 && (o.dx == -1 || o.dy == -1 || o.dz == -1)) {
            const int axis = o.dx ? 0 : (o.dy ? 1 : 2);
            v = off_upwind[axis];  // upstream face neighbour: diffusion + upwind convection
          } else {
            v = off_plain;
          }
          if (col_idx) {
            col_idx[k_nz] = (zz * n + yy) * n + xx;
            values[k_nz] = v;
          }
          ++k_nz;
        }
        if (row_ptr) row_ptr[row - row0 + 1] = k_nz;
      }
  }
  return k_nz;
}

int mstab_gen_uniform(uint64_t seed, int64_t count, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  for (int64_t i = 0; i < count; ++i) out[i] = uni(rng);
  return 0;
}

void mstab_gen_euler_rhs(int64_t n, const double* x, const double* f, double dt, double h2, double* b) {
  for (int64_t i = 0; i < n; ++i) {
    const volatile double q = x[i] / dt;  // keep the GPU's rounding order: h2 * ((x/dt) + f)
    const volatile double t = q + f[i];
    b[i] = h2 * t;
  }
}

int mstab_gen_banded(int64_t n, int32_t nnz_per_row, int64_t half_width, uint64_t seed,
                     int64_t* row_ptr, int64_t* col_idx, double* values) {
  if (nnz_per_row < 1 || n < 1) return -3;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  std::vector<int64_t> cols;
  row_ptr[0] = 0;
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = std::max<int64_t>(0, i - half_width);
    const int64_t hi = std::min<int64_t>(n - 1, i + half_width);
    const int64_t want = std::min<int64_t>(nnz_per_row - 1, hi - lo);  // excluding the diagonal
    std::uniform_int_distribution<int64_t> pick(lo, hi);
    cols.clear();
    while ((int64_t)cols.size() < want) {
      const int64_t c = pick(rng);
      if (c == i || std::find(cols.begin(), cols.end(), c) != cols.end()) continue;
      cols.push_back(c);
    }
    cols.push_back(i);
    std::sort(cols.begin(), cols.end());
    double abs_sum = 0.0;
    int64_t diag_pos = -1;
    for (int64_t c : cols) {
      col_idx[k] = c;
      if (c == i) {
        diag_pos = k;
        values[k] = 0.0;
      } else {
        values[k] = uni(rng);
        abs_sum += std::abs(values[k]);
      }
      ++k;
    }
    values[diag_pos] = 1.1 * abs_sum;
    row_ptr[i + 1] = k;
  }
  return 0;
}

void mstab_gen_sinewave(int64_t n, double* out) {
  const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
  for (int64_t k = 1; k <= n; ++k) out[k - 1] = std::sin(two_pi * static_cast<double>(k) / static_cast<double>(n));
}

int mstab_gen_normal(uint64_t seed, int64_t count, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> normal(0.0, 1.0);
  for (int64_t i = 0; i < count; ++i) out[i] = normal(rng);
  return 0;
}

}  // extern "C"
