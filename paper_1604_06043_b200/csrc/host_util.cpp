// host_util.cpp — see host_util.h.
#include "host_util.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <random>

#include "../../include/mstab_b200.h"

namespace mstab_b200 {

namespace {

constexpr uint64_t kFnvOffset = 1469598103934665603ull;
constexpr uint64_t kFnvPrime = 1099511628211ull;

inline uint64_t fnv_bytes(uint64_t h, const unsigned char* b, size_t len) {
  for (size_t i = 0; i < len; ++i) {
    h ^= b[i];
    h *= kFnvPrime;
  }
  return h;
}

// h after mixing a little-endian u64 value: low bytes explicitly, zero high bytes as prime powers.
struct U64Mixer {
  uint64_t pow[9];
  U64Mixer() {
    pow[0] = 1;
    for (int i = 1; i <= 8; ++i) pow[i] = pow[i - 1] * kFnvPrime;
  }
  inline uint64_t mix(uint64_t h, uint64_t v) const {
    int nb = 0;
    while (nb < 8 && (v >> (8 * nb)) != 0) ++nb;
    for (int i = 0; i < nb; ++i) {
      h ^= (v >> (8 * i)) & 0xffu;
      h *= kFnvPrime;
    }
    return h * pow[8 - nb];  // (h ^ 0) * prime == h * prime
  }
};

}  // namespace

uint64_t fnv_csr_fingerprint(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                             const double* values, int64_t nnz) {
  static const U64Mixer mx;
  uint64_t h = kFnvOffset;
  h = mx.mix(h, (uint64_t)n);
  h = mx.mix(h, (uint64_t)n);
  h = mx.mix(h, (uint64_t)nnz);
  for (int64_t i = 0; i <= n; ++i) h = mx.mix(h, (uint64_t)row_ptr[i]);
  for (int64_t k = 0; k < nnz; ++k) h = mx.mix(h, (uint64_t)col_idx[k]);
  for (int64_t k = 0; k < nnz; ++k) {
    h = fnv_bytes(h, reinterpret_cast<const unsigned char*>(values + k), sizeof(double));
    h *= mx.pow[8];  // imaginary part +0.0: eight zero bytes
  }
  return h;
}

std::vector<double> symmetric_eigenvalues(const double* h, int n) {
  std::vector<double> a(h, h + (size_t)n * n);
  auto A = [&](int i, int j) -> double& { return a[(size_t)j * n + i]; };
  double off = 0.0, total = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double m = A(i, j) * A(i, j);
      total += m;
      if (i != j) off += m;
    }
  const double stop = 1e-28 * std::max(total, 1e-300);
  for (int sweep = 0; sweep < 60 && off > stop; ++sweep) {
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        const double m = std::abs(apq);
        if (m == 0.0) continue;
        const double phase = apq / m;  // +-1 for real symmetric input
        const double theta = (A(q, q) - A(p, p)) / (2.0 * m);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(1.0 + theta * theta));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * phase * akq;
          A(k, q) = s * akp + c * phase * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * phase * aqk;
          A(q, k) = s * apk + c * phase * aqk;
        }
      }
    off = 0.0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        if (i != j) off += A(i, j) * A(i, j);
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = A(i, i);
  std::sort(ev.begin(), ev.end());
  return ev;
}

bool extract_omegas(const std::vector<double>& tau, std::vector<std::complex<double>>& out) {
  using C = std::complex<double>;
  if (tau.size() == 1) {
    out.push_back(C(tau[0]));
    return true;
  }
  if (tau.size() == 2) {
    const C t0(tau[0]), t1(tau[1]);
    const C disc = std::sqrt(t0 * t0 + 4.0 * t1);
    out.push_back((t0 + disc) / 2.0);
    out.push_back((t0 - disc) / 2.0);
    return true;
  }
  return false;
}

namespace {

constexpr char kMagic[8] = {'M', 'S', 'T', 'A', 'B', 'M', 'R', 'D'};
struct Header {
  char magic[8];
  uint32_t version;
  uint32_t flags;
  uint64_t n;
  uint64_t s;
  uint64_t level_j;
  uint64_t omega_count;
  uint64_t fingerprint;
};
static_assert(sizeof(Header) == 56, "mrd header");

}  // namespace

void mrd_write(const std::string& path, const MrdData& d) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw Error(MSTAB_E_IO, "cannot open " + path + " for writing");
  Header h{};
  std::memcpy(h.magic, kMagic, 8);
  h.version = 1;
  h.flags = 1u;  // real blocks: every imaginary part is +0.0 on this path
  h.n = (uint64_t)d.n;
  h.s = (uint64_t)d.s;
  h.level_j = (uint64_t)d.level_j;
  h.omega_count = d.omega.size();
  h.fingerprint = d.fingerprint;
  f.write(reinterpret_cast<const char*>(&h), sizeof(h));
  const size_t cnt = (size_t)d.n * (size_t)d.s;
  f.write(reinterpret_cast<const char*>(d.p.data()), (std::streamsize)(cnt * sizeof(double)));
  f.write(reinterpret_cast<const char*>(d.u.data()), (std::streamsize)(cnt * sizeof(double)));
  f.write(reinterpret_cast<const char*>(d.v.data()), (std::streamsize)(cnt * sizeof(double)));
  for (const auto& w : d.omega) {
    const double re = w.real(), im = w.imag();
    f.write(reinterpret_cast<const char*>(&re), sizeof(double));
    f.write(reinterpret_cast<const char*>(&im), sizeof(double));
  }
  if (!f) throw Error(MSTAB_E_IO, "write failed: " + path);
}

MrdData mrd_read(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error(MSTAB_E_IO, "cannot open " + path);
  Header h{};
  f.read(reinterpret_cast<char*>(&h), sizeof(h));
  if (!f || std::memcmp(h.magic, kMagic, 8) != 0) throw Error(MSTAB_E_PARSE, path + ": not a .mrd file");
  if (h.version != 1) throw Error(MSTAB_E_PARSE, path + ": unsupported version " + std::to_string(h.version));
  const bool real = (h.flags & 1u) != 0;
  const uint64_t scalar = real ? sizeof(double) : 2 * sizeof(double);
  const uint64_t expect = sizeof(Header) + 3 * h.n * h.s * scalar + h.omega_count * 2 * sizeof(double);
  std::error_code ec;
  const auto actual = std::filesystem::file_size(path, ec);
  if (ec || actual != expect) throw Error(MSTAB_E_PARSE, path + ": truncated or padded file");
  MrdData d;
  d.n = (int64_t)h.n;
  d.s = (int64_t)h.s;
  d.level_j = (int64_t)h.level_j;
  d.fingerprint = h.fingerprint;
  const size_t cnt = (size_t)h.n * (size_t)h.s;
  auto read_block = [&](std::vector<double>& out) {
    out.resize(cnt);
    if (real) {
      f.read(reinterpret_cast<char*>(out.data()), (std::streamsize)(cnt * sizeof(double)));
    } else {
      for (size_t i = 0; i < cnt; ++i) {
        double re = 0.0, im = 0.0;
        f.read(reinterpret_cast<char*>(&re), sizeof(double));
        f.read(reinterpret_cast<char*>(&im), sizeof(double));
        if (im != 0.0) throw Error(MSTAB_E_NOTREAL, path + ": complex recycle blocks are not supported");
        out[i] = re;
      }
    }
  };
  read_block(d.p);
  read_block(d.u);
  read_block(d.v);
  d.omega.resize(h.omega_count);
  for (auto& w : d.omega) {
    double re = 0.0, im = 0.0;
    f.read(reinterpret_cast<char*>(&re), sizeof(double));
    f.read(reinterpret_cast<char*>(&im), sizeof(double));
    w = std::complex<double>(re, im);
  }
  if (!f) throw Error(MSTAB_E_PARSE, path + ": unexpected end of file");
  return d;
}

struct NormalStream {
  std::mt19937_64 rng;
  std::normal_distribution<double> normal{0.0, 1.0};
  explicit NormalStream(uint64_t seed) : rng(seed) {}
};

NormalStream* normal_stream_create(uint64_t seed) { return new NormalStream(seed); }
void normal_stream_fill(NormalStream* st, double* out, int64_t count) {
  for (int64_t i = 0; i < count; ++i) out[i] = st->normal(st->rng);
}
void normal_stream_destroy(NormalStream* st) { delete st; }

}  // namespace mstab_b200
