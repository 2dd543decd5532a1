// host_util.cpp — see host_util.h.
#include "host_util.h"

#include <algorithm>
#include <limits>
#include <cstdlib>
#include <vector>
#include <thread>
#include <mutex>
#include <atomic>
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

// The same fold, resumable: a rank that holds only a slice of the matrix continues the hash a
// peer started (csr.cpp:28-43 folds dims, then every row_ptr entry, then every col_idx entry, then
// every value, so a distributed matrix is hashed in three relays over the ranks).
uint64_t fnv_begin(int64_t n_rows, int64_t n_cols, int64_t nnz) {
  static const U64Mixer mx;
  uint64_t h = kFnvOffset;
  h = mx.mix(h, (uint64_t)n_rows);
  h = mx.mix(h, (uint64_t)n_cols);
  return mx.mix(h, (uint64_t)nnz);
}
uint64_t fnv_fold_u64(uint64_t h, const int64_t* v, int64_t count, int64_t add) {
  static const U64Mixer mx;
  for (int64_t i = 0; i < count; ++i) h = mx.mix(h, (uint64_t)(v[i] + add));
  return h;
}
uint64_t fnv_fold_values(uint64_t h, const double* values, int64_t count) {
  static const U64Mixer mx;
  for (int64_t k = 0; k < count; ++k) {
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

// The draws of std::normal_distribution<double>(0, 1) over std::mt19937_64(seed), value for
// value (libstdc++'s Marsaglia polar method, bits/random.tcc: attempts (u1, u2) from
// generate_canonical, x = 2 u1 - 1, y = 2 u2 - 1, accepted when 0 < x^2 + y^2 <= 1, then
// mult = sqrt(-2 log(r2) / r2) and the pair is returned as y mult, x mult), but produced in bulk:
// the engine itself is sequential and cheap (~2 ns per 64-bit output); everything after it is a
// pure function of the attempt's two raw outputs, so attempts are evaluated by a few threads in
// blocks — acceptance and the two factors first, positions by a running count, then log / sqrt /
// divide (~15 ns per pair on one core: what made make_cut_space cost 0.3 s at c2 and 4.6 s at
// c5 s = 16). Raw outputs drawn but not consumed by a fill stay buffered for the next one, and an
// odd count leaves the pair's second value saved, exactly like the distribution's state.
struct NormalStream {
  std::mt19937_64 rng;
  std::vector<uint64_t> ahead;  // raw engine outputs drawn but not yet consumed (attempt-aligned)
  size_t ahead_pos = 0;
  bool saved_available = false;
  double saved = 0.0;
  explicit NormalStream(uint64_t seed) : rng(seed) {}
};

namespace {

// generate_canonical<double, 53> over a pre-drawn engine output: the library's own code run on a
// one-shot generator with mt19937_64's range, so the value is the distribution adaptor's
// (bits/random.h _Adaptor::operator()) by construction.
struct RawOnce {
  using result_type = uint64_t;
  uint64_t v;
  static constexpr result_type min() { return std::mt19937_64::min(); }
  static constexpr result_type max() { return std::mt19937_64::max(); }
  result_type operator()() { return v; }
};
inline double canonical_from_raw(uint64_t raw) {
  RawOnce g{raw};
  return std::generate_canonical<double, std::numeric_limits<double>::digits>(g);
}

int normal_threads() {
  static const int n = [] {
    if (const char* e = std::getenv("MSTAB_HOST_THREADS")) return std::max(1, std::atoi(e));
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::min<unsigned>(16u, std::max<unsigned>(1u, hc));
  }();
  return n;
}

template <typename F>
void parallel_blocks(int64_t count, int64_t grain, F&& fn) {
  const int64_t nblocks = (count + grain - 1) / grain;
  const int nt = (int)std::min<int64_t>(normal_threads(), nblocks);
  if (nt <= 1) {
    for (int64_t b = 0; b < nblocks; ++b) fn(b * grain, std::min(count, (b + 1) * grain));
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> th;
  auto work = [&] {
    for (int64_t b = next.fetch_add(1); b < nblocks; b = next.fetch_add(1))
      fn(b * grain, std::min(count, (b + 1) * grain));
  };
  for (int t = 1; t < nt; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
}

}  // namespace

NormalStream* normal_stream_create(uint64_t seed) { return new NormalStream(seed); }

void normal_stream_fill(NormalStream* st, double* out, int64_t count) {
  int64_t done = 0;
  if (count > 0 && st->saved_available) {
    st->saved_available = false;
    out[done++] = st->saved * 1.0 + 0.0;
  }
  std::vector<double> xs, ys, r2;
  std::vector<int64_t> slot;
  while (done < count) {
    const int64_t pairs_needed = (count - done + 1) / 2;
    // attempts to evaluate this round: the expected number (acceptance pi / 4) plus slack; a
    // round that accepts more than needed leaves its surplus raw outputs buffered
    // (rounds are capped so the attempt arrays stay cache-sized instead of paging in hundreds of MB)
    const int64_t attempts =
        std::min<int64_t>(int64_t(1) << 19, std::max<int64_t>(64, (int64_t)((double)pairs_needed * 1.30) + 64));
    // compact the look-ahead buffer and top it up to 2 * attempts raw outputs (sequential)
    if (st->ahead_pos > 0) {
      st->ahead.erase(st->ahead.begin(), st->ahead.begin() + (std::ptrdiff_t)st->ahead_pos);
      st->ahead_pos = 0;
    }
    const size_t have = st->ahead.size();
    if (have < (size_t)(2 * attempts)) {
      st->ahead.resize((size_t)(2 * attempts));
      for (size_t i = have; i < st->ahead.size(); ++i) st->ahead[i] = st->rng();
    }
    const int64_t navail = (int64_t)(st->ahead.size() / 2);
    xs.resize(navail);
    ys.resize(navail);
    r2.resize(navail);
    const uint64_t* raw = st->ahead.data();
    parallel_blocks(navail, 1 << 15, [&](int64_t lo, int64_t hi) {
      for (int64_t t = lo; t < hi; ++t) {
        const double x = 2.0 * canonical_from_raw(raw[2 * t]) - 1.0;
        const double y = 2.0 * canonical_from_raw(raw[2 * t + 1]) - 1.0;
        xs[t] = x;
        ys[t] = y;
        r2[t] = x * x + y * y;
      }
    });
    // accepted attempts in order, up to the number of pairs still needed
    slot.clear();
    int64_t used_attempts = navail;
    for (int64_t t = 0; t < navail; ++t) {
      if (!(r2[t] > 1.0 || r2[t] == 0.0)) {
        slot.push_back(t);
        if ((int64_t)slot.size() == pairs_needed) {
          used_attempts = t + 1;
          break;
        }
      }
    }
    const int64_t npairs = (int64_t)slot.size();
    double* dst = out + done;
    const int64_t room = count - done;
    double last_saved = 0.0;
    bool has_saved = false;
    std::mutex mu;
    parallel_blocks(npairs, 1 << 14, [&](int64_t lo, int64_t hi) {
      for (int64_t k = lo; k < hi; ++k) {
        const int64_t t = slot[(size_t)k];
        const double mult = std::sqrt(-2 * std::log(r2[t]) / r2[t]);
        const double first = ys[t] * mult, second = xs[t] * mult;
        dst[2 * k] = first * 1.0 + 0.0;
        if (2 * k + 1 < room) {
          dst[2 * k + 1] = second * 1.0 + 0.0;
        } else {  // odd count: the pair's second value stays saved (un-scaled, as _M_saved)
          std::lock_guard<std::mutex> lk(mu);
          last_saved = second;
          has_saved = true;
        }
      }
    });
    done += std::min<int64_t>(room, 2 * npairs);
    if (has_saved) {
      st->saved = last_saved;
      st->saved_available = true;
    }
    st->ahead_pos = (size_t)(2 * used_attempts);
  }
}

void normal_stream_destroy(NormalStream* st) { delete st; }

}  // namespace mstab_b200
