// kmisc.cu — init, launch accounting/profiling, and the small helper kernels.
//
// Compiled with --fmad=false: every a*b+c below rounds the product and the sum separately,
// exactly like the reference's scalar std::complex<double> loops with zero imaginary parts
// (g++ -O3 without -mfma). Given identical small-solve inputs, the element-wise
// kernels (SpMV, level updates, column rebuilds, poly combination) are therefore bit-identical
// to the reference; only the length-N reductions differ (deterministic trees instead of
// sequential sums), which is why parity is judged teacher-forced (finding 3).
//
// All streaming kernels are HBM-bound; they use persistent grid-stride loops
// sized to the SM count so each CTA leaves exactly one partial per reduced value, and the last
// CTA (ticket counter) reduces the partials in a fixed order and runs the dense step that
// consumes them (s x s LU, Givens-TSQR least squares) without another launch.
#include "kcommon.cuh"

namespace mstab_b200 {

int g_num_sms = 148;
std::mutex g_occ_mu;
std::unordered_map<const void*, int> g_occ;

namespace {

// ---------------------------------------------------------------------------------------------
constexpr int kMaxDots = kMaxS + 1;

__global__ void __launch_bounds__(kBlock) k_dots(int64_t n, int64_t ld, const double* __restrict__ a,
                                                 int na, const double* __restrict__ y, int with_norm,
                                                 double* dst, Reducer red) {
  DevState* ds = red.ds;
  double acc[kMaxDots];
#pragma unroll
  for (int j = 0; j < kMaxDots; ++j) acc[j] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    const double yv = y[row];
#pragma unroll
    for (int j = 0; j < kMaxS; ++j)
      if (j < na) acc[j] = acc[j] + a[j * ld + row] * yv;
    if (with_norm) acc[kMaxS] = acc[kMaxS] + yv * yv;
  }
  __shared__ double scratch[kMaxDots * 32];
  __shared__ double blk[kMaxDots];
  __shared__ double redv[kMaxDots];
  block_totals<kMaxDots>(acc, blk, scratch);
  if (!cta_commit(blk, kMaxDots, red.partials, &ds->ticket, redv, red.xred)) return;
  if (threadIdx.x == 0) {
    for (int j = 0; j < na; ++j) dst[j] = redv[j];
    if (with_norm) dst[na] = redv[kMaxS];
  }
}

__global__ void __launch_bounds__(kBlock) k_axpy_neg(int64_t n, int64_t ld, const double* __restrict__ a,
                                                     int na, const double* __restrict__ coef,
                                                     double* __restrict__ y) {
  double cf[kMaxS];
#pragma unroll
  for (int j = 0; j < kMaxS; ++j) cf[j] = (j < na) ? coef[j] : 0.0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double yv = y[row];
#pragma unroll
    for (int j = 0; j < kMaxS; ++j)
      if (j < na) yv = yv + (-cf[j]) * a[j * ld + row];
    y[row] = yv;
  }
}

__global__ void k_div_by_sqrt(int64_t n, const double* __restrict__ x, const double* d2,
                              double* __restrict__ y) {
  const double d = sqrt(*d2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}

__global__ void k_mul_inv_sqrt(int64_t n, const double* __restrict__ x, const double* d2,
                               double* __restrict__ y) {
  const double inv = 1.0 / sqrt(*d2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * inv;
}

__global__ void k_rsub(int64_t n, const double* __restrict__ b, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = b[i] - y[i];
}

__global__ void __launch_bounds__(kBlock) k_vec_stats(int64_t n, const double* __restrict__ x,
                                                      double* dst, Reducer red) {
  DevState* ds = red.ds;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    acc[0] = acc[0] + v * v;
    if (!isfinite(v)) acc[1] += 1.0;
    if (v != 0.0) acc[2] += 1.0;
  }
  __shared__ double scratch[3 * 32];
  __shared__ double blk[3];
  __shared__ double redv[3];
  block_totals<3>(acc, blk, scratch);
  if (!cta_commit(blk, 3, red.partials, &ds->ticket, redv, red.xred)) return;
  if (threadIdx.x == 0)
    for (int j = 0; j < 3; ++j) dst[j] = redv[j];
}

__global__ void k_euler_rhs(int64_t n, const double* __restrict__ x, const double* __restrict__ f,
                            double dt, double h2, double* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = h2 * (x[i] / dt + f[i]);
}

__global__ void k_axpby_chain(int64_t n, const double* __restrict__ x, const double* __restrict__ g,
                              double alpha, double* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = x[i] + alpha * g[i];
}

template <int S>
__global__ void k_small_solve(int s, const double* m, const double* rhs, double* x, int32_t* ok) {
  // the warp LU the finalizers run (bit-identical to the scalar dev_lu_solve), at the same
  // compile-time size bound the finalizers use (MAXS = S)
  __shared__ double lu[kMaxS * kMaxS], vin[kMaxS], vout[kMaxS];
  for (int i = threadIdx.x; i < s * s; i += blockDim.x) lu[i] = m[i];
  if ((int)threadIdx.x < s) vin[threadIdx.x] = rhs[threadIdx.x];
  __syncwarp();
  const bool r = warp_lu_solve<S>(s, lu, vin, vout);
  __syncwarp();
  if ((int)threadIdx.x < s) x[threadIdx.x] = vout[threadIdx.x];
  if (threadIdx.x == 0) *ok = r ? 1 : 0;
}

// ---- launch accounting -------------------------------------------------------------------------
std::atomic<uint64_t> g_launch_count{0};

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  double bytes;
};

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<ProfRec> pending;
  KernelClassStats stats[kKNumClasses] = {};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
};
Profiler g_prof;
std::mutex g_prof_mu;
thread_local std::vector<ProfEvent>* t_capture_list = nullptr;
thread_local cudaStream_t t_capture_stream = nullptr;  // stream of the capture list's last event

// Counts one launch; with profiling on, brackets it with events on its stream.
}  // namespace

void kernels_init(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
    g_num_sms = sms;
  kpoly_init();
}

LaunchScope::LaunchScope(cudaStream_t s, int c, double b) : st(s), cls(c), bytes(b) {
  g_launch_count.fetch_add(1, std::memory_order_relaxed);
  if (g_prof.on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    // Inside a captured cycle consecutive launches share ONE boundary event (the previous launch's
    // end is this launch's start: nothing else is enqueued between the kernels of a cycle), which
    // halves the event-record nodes the profiling pass puts between kernels. (Row-sharded captures
    // have the cross-rank collective between two kernels: it is charged to the kernel after it.)
    if (t_capture_list && !t_capture_list->empty() && t_capture_stream == st) {
      a = t_capture_list->back().b;
      return;
    }
    a = g_prof.get();
    // inside a stream capture an event-record NODE needs the External flag (a plain record only
    // adds a dependency edge)
    cudaEventRecordWithFlags(a, st, t_capture_list ? cudaEventRecordExternal : cudaEventRecordDefault);
    t_capture_stream = st;
  }
}

LaunchScope::~LaunchScope() {
  if (!a) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t b = g_prof.get();
  cudaEventRecordWithFlags(b, st, t_capture_list ? cudaEventRecordExternal : cudaEventRecordDefault);
  if (t_capture_list)
    t_capture_list->push_back({cls, a, b, bytes});
  else
    g_prof.pending.push_back({cls, a, b, bytes});
}

uint64_t launch_count() { return g_launch_count.load(); }
void count_launches(uint64_t n) { g_launch_count.fetch_add(n, std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool on = std::getenv("MSTAB_NO_PDL") == nullptr;
  return on;
}

bool prof_enabled() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  return g_prof.on;
}

void prof_set_capture_list(std::vector<ProfEvent>* list) {
  t_capture_list = list;
  t_capture_stream = nullptr;
}

void prof_accumulate(const std::vector<ProfEvent>& list) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (const ProfEvent& r : list) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) continue;
    KernelClassStats& s = g_prof.stats[r.cls];
    s.launches++;
    s.total_ms += ms;
    s.total_bytes += r.bytes;
  }
}

void prof_release(std::vector<ProfEvent>& list) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t prev_b = nullptr;
  for (const ProfEvent& r : list) {
    if (r.a != prev_b) g_prof.pool.push_back(r.a);  // a shared boundary event is returned once
    g_prof.pool.push_back(r.b);
    prev_b = r.b;
  }
  list.clear();
}

void prof_enable(bool on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.on = on;
  // events are created up front and only read back at prof_collect(), so the timed region pays
  // one cudaEventRecord per launch boundary and nothing else
  while (on && g_prof.pool.size() < 65536) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    g_prof.pool.push_back(e);
  }
}

void prof_collect() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (const ProfRec& r : g_prof.pending) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    KernelClassStats& s = g_prof.stats[r.cls];
    s.launches++;
    s.total_ms += ms;
    s.total_bytes += r.bytes;
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.pending.clear();
}

void prof_read(KernelClassStats* out) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int i = 0; i < kKNumClasses; ++i) out[i] = g_prof.stats[i];
}

void prof_reset() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& s : g_prof.stats) s = KernelClassStats{};
}

int grid_for(int64_t n) {
  int64_t want = (n + kBlock - 1) / kBlock;
  int64_t cap = (int64_t)g_num_sms * 4;
  if (want > cap) want = cap;
  return want < 1 ? 1 : (int)want;
}

void launch_dots(cudaStream_t st, int64_t n, int64_t ld, const double* a, int na, const double* y,
                 bool with_norm, double* dst, const Reducer& red) {
  LaunchScope ls(st, kKOther, vbytes(n, na + 1.0));
  const int grid = occupancy_grid(k_dots, n, 0);
  k_dots<<<grid, kBlock, 0, st>>>(n, ld, a, na, y, with_norm ? 1 : 0, dst, red);
}

void launch_axpy_neg(cudaStream_t st, int64_t n, int64_t ld, const double* a, int na,
                     const double* coef, double* y) {
  LaunchScope ls(st, kKOther, vbytes(n, na + 2.0));
  const int grid = occupancy_grid(k_axpy_neg, n, 0);
  k_axpy_neg<<<grid, kBlock, 0, st>>>(n, ld, a, na, coef, y);
}

void launch_div_by_sqrt(cudaStream_t st, int64_t n, const double* x, const double* d2, double* y) {
  LaunchScope ls(st, kKOther, vbytes(n, 2.0));
  k_div_by_sqrt<<<grid_for(n), kBlock, 0, st>>>(n, x, d2, y);
}

void launch_mul_inv_sqrt(cudaStream_t st, int64_t n, const double* x, const double* d2, double* y) {
  LaunchScope ls(st, kKOther, vbytes(n, 2.0));
  k_mul_inv_sqrt<<<grid_for(n), kBlock, 0, st>>>(n, x, d2, y);
}

void launch_rsub(cudaStream_t st, int64_t n, const double* b, double* y) {
  LaunchScope ls(st, kKOther, vbytes(n, 3.0));
  k_rsub<<<grid_for(n), kBlock, 0, st>>>(n, b, y);
}

void launch_vec_stats(cudaStream_t st, int64_t n, const double* x, double* dst, const Reducer& red) {
  LaunchScope ls(st, kKOther, vbytes(n, 1.0));
  const int grid = occupancy_grid(k_vec_stats, n, 0);
  k_vec_stats<<<grid, kBlock, 0, st>>>(n, x, dst, red);
}

void launch_euler_rhs(cudaStream_t st, int64_t n, const double* x, const double* f, double dt,
                      double h2, double* b) {
  LaunchScope ls(st, kKOther, vbytes(n, 3.0));
  k_euler_rhs<<<grid_for(n), kBlock, 0, st>>>(n, x, f, dt, h2, b);
}

void launch_axpby_chain(cudaStream_t st, int64_t n, const double* x, const double* g, double alpha,
                        double* b) {
  LaunchScope ls(st, kKOther, vbytes(n, 3.0));
  k_axpby_chain<<<grid_for(n), kBlock, 0, st>>>(n, x, g, alpha, b);
}

namespace {
__global__ void k_fin_copy(const double* __restrict__ src, double* __restrict__ dst, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
}
}  // namespace

void launch_fin_copy(cudaStream_t st, const double* src, double* dst, int count) {
  k_fin_copy<<<1, kBlock, 0, st>>>(src, dst, count);
}

void launch_small_solve(cudaStream_t st, int s, const double* m, const double* rhs, double* x,
                        int32_t* ok) {
  LaunchScope ls(st, kKOther, 0.0);
  MSTAB_DISPATCH_S(s, { k_small_solve<S><<<1, 32, 0, st>>>(s, m, rhs, x, ok); });
}

namespace {
__global__ void k_fill_hash(double* p, int64_t count, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ull * (uint64_t)(i + 1);  // splitmix64
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    p[i] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}
}  // namespace

void launch_fill_hash(cudaStream_t st, double* p, int64_t count, uint64_t seed) {
  k_fill_hash<<<grid_for(count), kBlock, 0, st>>>(p, count, seed);
}

}  // namespace mstab_b200
