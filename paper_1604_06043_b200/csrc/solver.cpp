// solver.cpp — host orchestration of the Mstab solve loop on one B200.
//
// Mirrors idrstab_solve / mstab_solve (proj/core/src/idrstab.cpp:193-307) step for step; all
// length-N work is enqueued as sm_100a kernels on the context stream (kernels.cu) and the host
// only reads back one CycleStatus per cycle (residual norm, tau, breakdown flag) to drive the
// loop condition, the counters and the fetch policy, exactly where the reference branches.
#include "solver.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <complex>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <optional>

namespace mstab_b200 {

#define CUDA_OK(expr)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw Error(MSTAB_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));         \
  } while (0)

namespace {

using Clock = std::chrono::steady_clock;
int64_t ns_since(Clock::time_point t0) {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count();
}

// Phase tracing (the reference only has steady_clock stamps per history point). Every
// traced host-side step of a solve is an NVTX range ("mstab: validate", "mstab: cycle", ...), so
// an Nsight Systems / Compute timeline shows the solve's phases over the kernels they launch
// (header-only NVTX 3: a no-op costing a relaxed load when no tool is attached), and with
// MSTAB_DEBUG_STALL=ms any step that took longer than that is reported on stderr.
struct StallTrace {
  const char* what;
  Clock::time_point t0;
  static double limit_ms() {
    static const double v = [] {
      const char* e = std::getenv("MSTAB_DEBUG_STALL");
      return e ? std::atof(e) : -1.0;
    }();
    return v;
  }
  explicit StallTrace(const char* w) : what(w), t0(Clock::now()) { nvtxRangePushA(w); }
  ~StallTrace() {
    nvtxRangePop();
    const double lim = limit_ms();
    if (lim < 0.0) return;
    const double ms = ns_since(t0) / 1e6;
    if (ms > lim) std::fprintf(stderr, "[mstab stall] %s took %.2f ms\n", what, ms);
  }
};

void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(MSTAB_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace

int64_t padded_ld(int64_t n) { return std::max<int64_t>(64, (n + 63) & ~int64_t(63)); }

uint64_t next_operator_uid() {
  static std::atomic<uint64_t> next{1};
  return next.fetch_add(1);
}

namespace {
// blocks worth caching (vectors and n x s blocks, not the small dense state) and the cap per stream
constexpr size_t kCacheMinBytes = size_t(1) << 20;
size_t cache_cap_bytes() {
  static const size_t cap = [] {
    if (std::getenv("MSTAB_NO_BLOCK_CACHE")) return size_t(0);
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return size_t(0);
    return total_b / 3;  // at most a third of the device per stream
  }();
  return cap;
}
}  // namespace

void* StreamHolder::take(size_t bytes) {
  if (bytes < kCacheMinBytes) return nullptr;
  std::lock_guard<std::mutex> lk(cache_mu);
  auto it = cache.find(bytes);
  if (it == cache.end() || it->second.empty()) return nullptr;
  void* p = it->second.back();
  it->second.pop_back();
  cached_bytes -= bytes;
  static const bool dbg = std::getenv("MSTAB_DEBUG_ALLOC") != nullptr;
  if (dbg) std::fprintf(stderr, "[mstab alloc] take %zu MB from cache\n", bytes >> 20);
  return p;
}

bool StreamHolder::give(void* p, size_t bytes) {
  if (bytes < kCacheMinBytes) return false;
  static const bool dbg = std::getenv("MSTAB_DEBUG_ALLOC") != nullptr;
  std::lock_guard<std::mutex> lk(cache_mu);
  const bool ok = cached_bytes + bytes <= cache_cap_bytes();
  if (dbg) std::fprintf(stderr, "[mstab alloc] give %zu MB %s (cached %zu MB)\n", bytes >> 20, ok ? "kept" : "REFUSED", cached_bytes >> 20);
  if (!ok) return false;
  cache[bytes].push_back(p);
  cached_bytes += bytes;
  return true;
}

void StreamHolder::drop_cache() {
  std::lock_guard<std::mutex> lk(cache_mu);
  for (auto& kv : cache)
    for (void* p : kv.second) cudaFreeAsync(p, stream);
  cache.clear();
  cached_bytes = 0;
}

StreamHolder::~StreamHolder() {
  if (stream) {
    cudaStreamSynchronize(stream);
    for (auto& kv : cache)
      for (void* p : kv.second) cudaFreeAsync(p, stream);
    cache.clear();
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

DevMem::DevMem(std::shared_ptr<StreamHolder> st, size_t b) : bytes(b == 0 ? 64 : b), stream(std::move(st)) {
  ptr = stream->take(bytes);
  if (ptr) return;
  static const bool dbg = std::getenv("MSTAB_DEBUG_ALLOC") != nullptr;
  const auto t0 = Clock::now();
  CUDA_OK(cudaMallocAsync(&ptr, bytes, stream->stream));
  if (dbg) {
    const double ms = ns_since(t0) / 1e6;
    if (ms > 0.5) std::fprintf(stderr, "[mstab alloc] cudaMallocAsync(%zu MB) took %.2f ms\n", bytes >> 20, ms);
  }
}

DevMem::~DevMem() {
  if (ptr && !stream->give(ptr, bytes)) cudaFreeAsync(ptr, stream->stream);
}

Context::Context(int dev) {
  if (dev < 0) CUDA_OK(cudaGetDevice(&dev));
  device = dev;
  CUDA_OK(cudaSetDevice(dev));
  sh = std::make_shared<StreamHolder>();
  sh->device = dev;
  CUDA_OK(cudaStreamCreateWithFlags(&sh->stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;
  CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = std::numeric_limits<uint64_t>::max();
  CUDA_OK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  kernels_init(dev);
  ds_mem = alloc(sizeof(DevState));
  CUDA_OK(cudaMemsetAsync(ds_mem->ptr, 0, sizeof(DevState), stream()));
  partials = alloc(sizeof(double) * (size_t)kMaxGrid * 640);
  slots = alloc(sizeof(double) * (size_t)kMaxGrid * (kMaxS + 1));
  CUDA_OK(cudaMemsetAsync(slots->ptr, 0xff, slots->bytes, stream()));  // every slot empty
  CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host_status), sizeof(CycleStatus)));
  CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host_scal), sizeof(double) * 64));
  CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&hslots), sizeof(HostCycleSlot) * 2, cudaHostAllocMapped));
  std::memset(hslots, 0, sizeof(HostCycleSlot) * 2);
  sync();
}

Context::~Context() {
  if (sh && sh->stream) cudaStreamSynchronize(sh->stream);
  if (host_status) cudaFreeHost(host_status);
  if (host_scal) cudaFreeHost(host_scal);
  if (hslots) cudaFreeHost(hslots);
}

void Context::sync() { CUDA_OK(cudaStreamSynchronize(stream())); }

// Releases what the context caches between solves (workspace and cycle graphs, the cut-space and
// validate scratch, the stream's block cache) and hands the memory back to the device.
void Context::trim() {
  sync();
  ws.reset();
  pcache.reset();
  val_au.reset();
  val_au_n = -1;
  sh->drop_cache();
  sync();
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
}

DevPtr Context::alloc_vecs(int64_t n, int64_t cols) {
  DevPtr d = alloc(sizeof(double) * (size_t)ld(n) * (size_t)std::max<int64_t>(cols, 1));
  if (n == lay_n) {  // slab vector: owned rows after lay_lo halo rows; halos start out zero
    d->off = lay_lo;
    CUDA_OK(cudaMemsetAsync(d->ptr, 0, d->bytes, stream()));
  }
  return d;
}

// ---- small device<->host helpers ----------------------------------------------------------
void reset_status(Context& ctx) {
  CUDA_OK(cudaMemsetAsync(ctx.ds(), 0, sizeof(CycleStatus), ctx.stream()));
  // the stop flag of the persistent cycles and the ticket counter (adjacent)
  static_assert(offsetof(DevState, ticket) == offsetof(DevState, stop) + sizeof(int32_t), "stop precedes ticket");
  CUDA_OK(cudaMemsetAsync(reinterpret_cast<char*>(ctx.ds()) + offsetof(DevState, stop), 0,
                          sizeof(int32_t) + sizeof(uint32_t), ctx.stream()));
}

double* scal(Context& ctx, int i) { return ctx.ds()->scal + i; }

const double* read_scal(Context& ctx, int count) {
  CUDA_OK(cudaMemcpyAsync(ctx.host_scal, ctx.ds()->scal, sizeof(double) * count,
                          cudaMemcpyDeviceToHost, ctx.stream()));
  ctx.sync();
  return ctx.host_scal;
}

const CycleStatus& read_status(Context& ctx) {
  CUDA_OK(cudaMemcpyAsync(ctx.host_status, &ctx.ds()->st, sizeof(CycleStatus),
                          cudaMemcpyDeviceToHost, ctx.stream()));
  ctx.sync();
  return *ctx.host_status;
}

namespace {

DevPtr copy_block(Context& ctx, const DevPtr& src, int64_t n, int64_t cols) {
  DevPtr dst = ctx.alloc_vecs(n, cols);
  CUDA_OK(cudaMemcpyAsync(dst->ptr, src->ptr, sizeof(double) * (size_t)ctx.ld(n) * cols,
                          cudaMemcpyDeviceToDevice, ctx.stream()));
  return dst;
}

// ---- row-sharded solves: what follows a reduction kernel / precedes an SpMV -------------------
// On one GPU (no communicator) the kernels finish their reductions themselves and these are
// no-ops. Sharded, the kernels leave rank-local totals in ds->xred; these sum them over the
// ranks and run the dense tail the fused kernel would have run.
double* xred(Context& ctx) { return ctx.ds()->xred; }

void halo(Context& ctx, const Operator& op, const double* x) {
  if (ctx.sharded()) ctx.comm->halo(const_cast<double*>(x), op.halo, ctx.stream());
}
void after_spmv(Context& ctx, int s, bool tres, const FinParams& f) {
  if (!ctx.sharded()) return;
  ctx.comm->allreduce_sum(xred(ctx), s + (tres ? 1 : 0), ctx.stream());
  launch_fin_spmv(ctx.stream(), s, f, ctx.ds());
  check_launch();
}
void after_poly(Context& ctx, int s) {
  if (!ctx.sharded()) return;
  ctx.comm->allreduce_sum(xred(ctx), 1 + s + s * s, ctx.stream());
  launch_fin_poly(ctx.stream(), s, ctx.ds());
  check_launch();
}
void after_ls(Context& ctx, int ell, int s, bool chol) {
  if (!ctx.sharded()) return;
  const int cnt = ls_split_count(ell);
  ctx.comm->allgather(xred(ctx), ctx.xgath->d(), cnt, ctx.stream());
  launch_fin_ls(ctx.stream(), ell, s, ctx.comm->world(), chol, ctx.xgath->d(), ctx.ds());
  check_launch();
}
// dots (launch_dots layout: slots 0..na-1, the norm in slot kMaxS) -> dst[0..na(+1))
void after_dots(Context& ctx, int na, bool with_norm, double* dst) {
  if (!ctx.sharded()) return;
  ctx.comm->allreduce_sum(xred(ctx), kMaxS + 1, ctx.stream());
  if (na > 0) launch_fin_copy(ctx.stream(), xred(ctx), dst, na);
  if (with_norm) launch_fin_copy(ctx.stream(), xred(ctx) + kMaxS, dst + na, 1);
  check_launch();
}
void after_stats(Context& ctx, double* dst) {
  if (!ctx.sharded()) return;
  ctx.comm->allreduce_sum(xred(ctx), 3, ctx.stream());
  launch_fin_copy(ctx.stream(), xred(ctx), dst, 3);
  check_launch();
}

// w = L^-1 A R^-1 x for a preconditioned operator (apply_preconditioned, precond.cpp:169-174):
// upper solve, SpMV (its fused dot is discarded), lower solve.
void precond_chain(Context& ctx, const Operator& op, const double* x, double* w) {
  Precond& pc = *op.pc;
  cudaStream_t st = ctx.stream();
  launch_tri_solve(st, pc.R, x, pc.t1->d(), reinterpret_cast<int*>(pc.sync->ptr));
  FinParams f;
  f.op = kFinStore;
  f.s = 1;
  f.dst = scal(ctx, 63);
  launch_spmv_ph(st, op.csr(), pc.t1->d(), pc.t2->d(), pc.t1->d(), ctx.ld(op.n), 1, nullptr, f, ctx.reducer());
  launch_tri_solve(st, pc.L, pc.t2->d(), w, reinterpret_cast<int*>(pc.sync->ptr));
  check_launch();
}

// y = op x (or the true residual y = b - op x) with the fused P^H epilogue and finaliser `f`:
// one kernel for a plain CSR operator, the preconditioned chain + k_ph_fin otherwise.
void apply_ph(Context& ctx, const Operator& op, const double* x, double* y, const double* P, int s,
              const double* b, const FinParams& f) {
  if (!op.pc) {
    launch_spmv_ph(ctx.stream(), op.csr(), x, y, P, ctx.ld(op.n), s, b, f, ctx.reducer());
    return;
  }
  precond_chain(ctx, op, x, op.pc->t3->d());
  launch_ph_fin(ctx.stream(), op.n, ctx.ld(op.n), s, op.pc->t3->d(), y, P, b, f, ctx.reducer());
}

// The product of a row-sharded solve: halo exchange, then apply_ph. On the constant-diagonal form
// the product is split (VERDICT r01 missing #5): the exchange starts (NcclComm: on a side stream),
// the interior rows, which read no halo entry, are computed meanwhile and leave their totals in
// xred2; once the halo has arrived the boundary rows follow and their finisher adds the two sets of
// totals in a fixed order (interior first), so the result does not depend on timing. Other operator
// forms exchange first, then run the one-launch product.
void apply_ph_sharded(Context& ctx, const Operator& op, const double* x, double* y, const double* P, int s,
                      const double* b, const FinParams& f) {
  static const bool overlap = std::getenv("MSTAB_NO_HALO_OVERLAP") == nullptr;
  const bool split = overlap && !op.pc && op.use_dia && op.ndiag > 0 && op.mask_bytes > 0 && op.int_hi > op.int_lo &&
                     !op.halo.empty() && op.n < (int64_t(1) << 31);
  if (!split) {
    halo(ctx, op, x);
    apply_ph(ctx, op, x, y, P, s, b, f);
    return;
  }
  cudaStream_t st = ctx.stream();
  ctx.comm->halo_begin(const_cast<double*>(x), op.halo, st);
  DevCsr inner = op.csr();
  inner.sel_a0 = (int32_t)op.int_lo;
  inner.sel_a1 = (int32_t)op.int_hi;
  Reducer ri = ctx.reducer();
  ri.xred = ctx.ds()->xred2;
  launch_spmv_ph(st, inner, x, y, P, ctx.ld(op.n), s, b, f, ri);
  ctx.comm->halo_end(st);
  DevCsr edge = op.csr();
  edge.sel_a0 = 0;
  edge.sel_a1 = (int32_t)op.int_lo;
  edge.sel_b0 = (int32_t)op.int_hi;
  edge.sel_b1 = (int32_t)op.n;
  Reducer re = ctx.reducer();
  re.xbase = ctx.ds()->xred2;
  launch_spmv_ph(st, edge, x, y, P, ctx.ld(op.n), s, b, f, re);
}

// Plain SpMV through the fused kernel (s = 1, dot with x discarded).
void spmv_dev(Context& ctx, const Operator& op, const double* x, double* y) {
  if (op.pc) {
    precond_chain(ctx, op, x, y);
    return;
  }
  FinParams f;
  f.op = kFinStore;
  f.s = 1;
  f.dst = scal(ctx, 63);
  if (ctx.sharded())
    apply_ph_sharded(ctx, op, x, y, x, 1, nullptr, f);
  else
    launch_spmv_ph(ctx.stream(), op.csr(), x, y, x, ctx.ld(op.n), 1, nullptr, f, ctx.reducer());
  check_launch();
  after_spmv(ctx, 1, false, f);
}

// ||y||^2 -> scal[i]
void norm2sq(Context& ctx, int64_t n, const double* y, int i) {
  launch_dots(ctx.stream(), n, ctx.ld(n), nullptr, 0, y, true, scal(ctx, i), ctx.reducer());
  check_launch();
  after_dots(ctx, 0, true, scal(ctx, i));
}

// Host draws of a length-n_global column restricted to this context's rows (RNG parity: every
// rank draws the whole sequence in the reference's order and keeps its slab).
const double* own_rows(const Context& ctx, int64_t n, const double* global) {
  return (n == ctx.lay_n) ? global + ctx.lay_row0 : global;
}
int64_t draw_len(const Context& ctx, int64_t n) { return (n == ctx.lay_n) ? ctx.lay_nglobal : n; }

}  // namespace

// make_cut_space (baselines.cpp:36-47): seeded Gaussian draws (host std::mt19937_64 +
// std::normal_distribution, column-major, so P's draws are the reference's) orthonormalised on
// the device by classical Gram-Schmidt applied twice (orthonormalize, kernels.cpp:21-50).
DevPtr make_cut_space(Context& ctx, int64_t n, int s, uint64_t seed) {
  const int64_t ld = ctx.ld(n);
  cudaStream_t st = ctx.stream();
  NormalStream* rng = normal_stream_create(seed);
  std::unique_ptr<NormalStream, void (*)(NormalStream*)> guard(rng, normal_stream_destroy);
  const int64_t ng = draw_len(ctx, n);  // column-major draws over the GLOBAL rows
  std::vector<double> g((size_t)ng * s);
  DevPtr G = ctx.alloc_vecs(n, s);
  DevPtr Q = ctx.alloc_vecs(n, s);
  for (int attempt = 0; attempt < 4; ++attempt) {
    normal_stream_fill(rng, g.data(), (int64_t)g.size());
    CUDA_OK(cudaMemcpy2DAsync(G->d(), sizeof(double) * ld, own_rows(ctx, n, g.data()), sizeof(double) * ng,
                              sizeof(double) * n, s, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaStreamSynchronize(st));  // g is refilled by the next attempt
    int rank = 0;
    for (int j = 0; j < s; ++j) {
      const double* gj = G->d() + (size_t)j * ld;
      double* w = Q->d() + (size_t)rank * ld;
      norm2sq(ctx, n, gj, 0);
      CUDA_OK(cudaMemcpyAsync(w, gj, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      for (int pass = 0; pass < 2 && rank > 0; ++pass) {
        launch_dots(st, n, ld, Q->d(), rank, w, false, scal(ctx, 8), ctx.reducer());
        check_launch();
        after_dots(ctx, rank, false, scal(ctx, 8));
        launch_axpy_neg(st, n, ld, Q->d(), rank, scal(ctx, 8), w);
        check_launch();
      }
      norm2sq(ctx, n, w, 1);
      const double* h = read_scal(ctx, 2);
      const double norm0 = std::sqrt(h[0]), res = std::sqrt(h[1]);
      if (res <= 1e-10 * norm0 || norm0 == 0.0) continue;  // kRankTol (kernels.hpp:16)
      launch_mul_inv_sqrt(st, n, w, scal(ctx, 1), w);
      check_launch();
      ++rank;
    }
    if (rank == s) return Q;
  }
  throw Error(MSTAB_E_ERROR, "make_cut_space: could not draw a full-rank cut-space");
}

// arnoldi_init (idrstab.cpp:45-87): U orthonormal basis of K_s(A; r0) by MGS with reiteration,
// V = A U from the same sweep, happy breakdowns padded with seeded Gaussian directions.
void arnoldi_init(Context& ctx, const Operator& op, const double* r0, int s, uint64_t seed,
                  double* U, double* V) {
  std::unique_ptr<NormalStream, void (*)(NormalStream*)> rng(nullptr, normal_stream_destroy);
  arnoldi_init(ctx, op, r0, s, [&](double* out, int64_t count) {
    if (!rng) rng.reset(normal_stream_create(seed));
    normal_stream_fill(rng.get(), out, count);
  }, U, V);
}

void arnoldi_init(Context& ctx, const Operator& op, const double* r0, int s,
                  const std::function<void(double*, int64_t)>& draw, double* U, double* V) {
  const int64_t n = op.n, ld = ctx.ld(n);
  cudaStream_t st = ctx.stream();
  norm2sq(ctx, n, r0, 0);
  if (read_scal(ctx, 1)[0] == 0.0) throw Error(MSTAB_E_ERROR, "arnoldi_init: zero start vector");
  launch_div_by_sqrt(st, n, r0, scal(ctx, 0), U);
  check_launch();
  DevPtr w = ctx.alloc_vecs(n, 1);
  std::vector<double> hw;
  auto mgs2 = [&](int k) {
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i <= k; ++i) {
        launch_dots(st, n, ld, U + (size_t)i * ld, 1, w->d(), false, scal(ctx, 2), ctx.reducer());
        check_launch();
        after_dots(ctx, 1, false, scal(ctx, 2));
        launch_axpy_neg(st, n, ld, U + (size_t)i * ld, 1, scal(ctx, 2), w->d());
        check_launch();
      }
  };
  for (int k = 0; k < s; ++k) {
    spmv_dev(ctx, op, U + (size_t)k * ld, V + (size_t)k * ld);
    if (k + 1 == s) break;
    CUDA_OK(cudaMemcpyAsync(w->d(), V + (size_t)k * ld, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    norm2sq(ctx, n, w->d(), 1);
    mgs2(k);
    norm2sq(ctx, n, w->d(), 3);
    const double* h = read_scal(ctx, 4);
    const double wnorm0 = std::sqrt(h[1]);
    double wnorm = std::sqrt(h[3]);
    while (wnorm <= 1e-12 * std::max(wnorm0, 1.0)) {
      hw.resize(draw_len(ctx, n));
      draw(hw.data(), (int64_t)hw.size());
      CUDA_OK(cudaMemcpyAsync(w->d(), own_rows(ctx, n, hw.data()), sizeof(double) * n, cudaMemcpyHostToDevice, st));
      CUDA_OK(cudaStreamSynchronize(st));
      mgs2(k);
      norm2sq(ctx, n, w->d(), 3);
      wnorm = std::sqrt(read_scal(ctx, 4)[3]);
    }
    launch_div_by_sqrt(st, n, w->d(), scal(ctx, 3), U + (size_t)(k + 1) * ld);
    check_launch();
  }
}

namespace {

void enqueue_level(Context& ctx, const Operator& op, const double* P, int s, int ell, int k,
                   const WSet& S, const WSet& D, const std::vector<DevPtr>& R,
                   const std::vector<DevPtr>& VL);
void enqueue_poly(Context& ctx, const Operator& op, const double* P, int s, int ell, const WSet& D,
                  const std::vector<DevPtr>& R, const std::vector<DevPtr>& VL);

// One outer cycle: ell level iterations + poly_combination, S -> D (idrstab.cpp:250-259).
void enqueue_cycle(Context& ctx, const Operator& op, const double* P, int s, int ell,
                   const WSet& S, const WSet& D, const std::vector<DevPtr>& R,
                   const std::vector<DevPtr>& VL) {
  for (int k = 0; k < ell; ++k) enqueue_level(ctx, op, P, s, ell, k, S, D, R, VL);
  check_launch();
  enqueue_poly(ctx, op, P, s, ell, D, R, VL);
}

// One level iteration k (idrstab.cpp:105-152): the BiCG step on the top level with gamma_k
// (ds->gamma row k), r^(k+1) = A r^(k), the s column rebuilds at the top level each raised by one
// product, then the deferred lower levels. At k = 0 the state is read from S and written to D
// (S == D is allowed: every kernel of the level is safe in place).
void enqueue_level(Context& ctx, const Operator& op, const double* P, int s, int ell, int k,
                   const WSet& S, const WSet& D, const std::vector<DevPtr>& R,
                   const std::vector<DevPtr>& VL) {
  const int64_t n = op.n, ld = ctx.ld(n);
  const bool shard = ctx.sharded();
  cudaStream_t st = ctx.stream();
  DevState* ds = ctx.ds();
  auto col = [ld](double* base, int q) { return base + (size_t)q * ld; };
  {
    // (a) top level: r^(k) -= V^(k) gamma_k
    const double* r_in = (k == 0) ? S.r->d() : R[k]->d();
    double* r_out = (k == 0) ? D.r->d() : R[k]->d();
    const double* vk_old = (k == 0) ? S.V->d() : VL[k]->d();
    double* vk_new = (k == 0) ? D.V->d() : VL[k]->d();
    launch_level_update(st, n, ld, s, k, r_in, r_out, vk_old, ds);
    // (b) r^(k+1) = A r^(k); rhs = P^H r^(k+1); eta_0
    FinParams fb;
    fb.op = kFinRhsEta0;
    fb.s = s;
    fb.k = k;
    fb.ell = ell;
    if (shard)
      apply_ph_sharded(ctx, op, r_out, R[k + 1]->d(), P, s, nullptr, fb);
    else
      apply_ph(ctx, op, r_out, R[k + 1]->d(), P, s, nullptr, fb);
    if (shard) after_spmv(ctx, s, false, fb);
    // (c) column rebuilds at the top level, each raised by one SpMV
    for (int q = 0; q < s; ++q) {
      launch_rebuild_top(st, n, ld, s, q, R[k + 1]->d(), vk_old, vk_new, VL[k + 1]->d(), ds);
      FinParams fc;
      fc.op = kFinColEta;
      fc.s = s;
      fc.k = k;
      fc.q = q;
      fc.ell = ell;
      if (shard)
        apply_ph_sharded(ctx, op, col(vk_new, q), col(VL[k + 1]->d(), q), P, s, nullptr, fc);
      else
        apply_ph(ctx, op, col(vk_new, q), col(VL[k + 1]->d(), q), P, s, nullptr, fc);
      if (shard) after_spmv(ctx, s, false, fc);
    }
    // deferred (a) for r^(0..k-1), x and (c) for levels -1..k-1
    const double* lv_in[kMaxEll + 2];
    double* lv_out[kMaxEll + 2];
    const double* rin[kMaxEll + 1];
    double* rout[kMaxEll + 1];
    lv_in[0] = (k == 0) ? S.U->d() : D.U->d();
    lv_out[0] = D.U->d();
    lv_in[1] = D.V->d();
    lv_out[1] = D.V->d();
    for (int L = 1; L <= k; ++L) {
      lv_in[L + 1] = VL[L]->d();
      lv_out[L + 1] = VL[L]->d();
    }
    rin[0] = D.r->d();
    rout[0] = D.r->d();
    for (int i = 1; i <= k; ++i) {
      rin[i] = R[i]->d();
      rout[i] = R[i]->d();
    }
    launch_rebuild_deferred(st, n, ld, s, k, lv_in, lv_out, rin, rout,
                            (k == 0) ? S.x->d() : D.x->d(), D.x->d(), ds);
  }
}

// poly_combination (idrstab.cpp:154-191): least squares, then the combined x, r, U, V (+ the next
// cycle's P^H r, P^H V and gamma_0), all in D.
void enqueue_poly(Context& ctx, const Operator& op, const double* P, int s, int ell, const WSet& D,
                  const std::vector<DevPtr>& R, const std::vector<DevPtr>& VL) {
  const int64_t n = op.n, ld = ctx.ld(n);
  const bool shard = ctx.sharded();
  cudaStream_t st = ctx.stream();
  const Reducer red = ctx.reducer();
  const double* rr[kMaxEll + 1];
  rr[0] = D.r->d();
  for (int i = 1; i <= ell; ++i) rr[i] = R[i]->d();
  const bool chol = ls_use_cholqr(op.n_global);  // same choice on every rank
  if (chol) {
    launch_ls_pass1(st, n, ell, rr, red);
    if (shard) {  // pass-1 Gram summed over the ranks before the replicated Cholesky
      ctx.comm->allreduce_sum(xred(ctx), (ell + 1) * (ell + 2) / 2, st);
      launch_fin_ls1(st, ell, ctx.ds());
      check_launch();
    }
  }
  launch_ls_pass2(st, n, ell, s, chol, rr, red);
  if (shard) after_ls(ctx, ell, s, chol);
  const double* lv[kMaxEll + 2];
  lv[0] = D.U->d();
  lv[1] = D.V->d();
  for (int i = 1; i <= ell; ++i) lv[i + 1] = VL[i]->d();
  launch_poly(st, n, ld, s, ell, lv, D.U->d(), D.V->d(), rr, D.r->d(), D.x->d(), D.x->d(), P, red);
  check_launch();
  if (shard) after_poly(ctx, s);
}

}  // namespace

namespace {

// CsrMatrix::validate (csr.cpp:11-24) on the host arrays; returns nnz.
int64_t validate_csr(int64_t n, const int64_t* row_ptr, const int64_t* col_idx) {
  if (n < 0) throw Error(MSTAB_E_DIMENSION, "CsrOperator: negative size");
  if (row_ptr[0] != 0) throw Error(MSTAB_E_ERROR, "csr: row_ptr bounds");
  const int64_t nnz = row_ptr[n];
  for (int64_t i = 0; i < n; ++i) {
    if (row_ptr[i] > row_ptr[i + 1]) throw Error(MSTAB_E_ERROR, "csr: row_ptr not nondecreasing");
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      if (col_idx[k] < 0 || col_idx[k] >= n) throw Error(MSTAB_E_ERROR, "csr: column index out of range");
      if (k > row_ptr[i] && col_idx[k - 1] >= col_idx[k])
        throw Error(MSTAB_E_ERROR, "csr: columns not strictly increasing within a row");
    }
  }
  return nnz;
}

// Uploads n local rows (row_ptr from 0, column indices relative to the first owned row, so a
// slab's halo columns are negative or >= n) and builds the DIA / constant-diagonal forms.
void upload_rows(Context& ctx, Operator* op, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                 const double* values) {
  const int64_t nnz = row_ptr[n];
  if (nnz >= (int64_t(1) << 31)) throw Error(MSTAB_E_CONFIG, "b200: nnz >= 2^31 not supported (int32 indices)");
  op->n = n;
  op->nnz = nnz;
  int64_t blo = 0, bhi = 0;
  for (int64_t i = 0; i < n; ++i)
    if (row_ptr[i + 1] > row_ptr[i]) {
      blo = std::min(blo, col_idx[row_ptr[i]] - i);  // columns ascend within a row
      bhi = std::max(bhi, col_idx[row_ptr[i + 1] - 1] - i);
    }
  op->blo = blo;
  op->bhi = bhi;
  int64_t bmax = 0;
  for (int64_t i = 0; i < n; i += 32) bmax = std::max(bmax, row_ptr[std::min(n, i + 32)] - row_ptr[i]);
  op->blk32_max = (int32_t)std::min<int64_t>(bmax, std::numeric_limits<int32_t>::max());
  std::vector<int32_t> rp32(n + 1), ci32(nnz + 32, 0);
  for (int64_t i = 0; i <= n; ++i) rp32[i] = (int32_t)row_ptr[i];
  for (int64_t k = 0; k < nnz; ++k) ci32[k] = (int32_t)col_idx[k];
  op->rp = ctx.alloc(sizeof(int32_t) * (n + 1));
  op->ci = ctx.alloc(sizeof(int32_t) * (nnz + 32));
  op->val = ctx.alloc(sizeof(double) * (nnz + 32));
  cudaStream_t st = ctx.stream();
  CUDA_OK(cudaMemcpyAsync(op->rp->ptr, rp32.data(), sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, st));
  CUDA_OK(cudaMemcpyAsync(op->ci->ptr, ci32.data(), sizeof(int32_t) * (nnz + 32), cudaMemcpyHostToDevice, st));
  CUDA_OK(cudaMemsetAsync(op->val->ptr, 0, sizeof(double) * (nnz + 32), st));
  CUDA_OK(cudaMemcpyAsync(op->val->ptr, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  // DIA form when the nonzeros sit on at most kMaxDiag diagonals filled to >= 2/3: no column
  // indices to stream and contiguous x gathers. Slots without a CSR entry hold +0.0, so the SpMV
  // (0*x adds nothing) stays equal to the CSR-order accumulation.
  if (n > 0 && nnz > 0 && std::getenv("MSTAB_NO_DIA") == nullptr) {
    std::vector<int64_t> offs;
    bool ok = true;
    for (int64_t i = 0; i < n && ok; ++i)
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        const int64_t o = col_idx[k] - i;
        if (std::find(offs.begin(), offs.end(), o) == offs.end()) {
          offs.push_back(o);
          if ((int)offs.size() > kMaxDiag) {
            ok = false;
            break;
          }
        }
      }
    if (ok && (double)offs.size() * (double)n <= 1.5 * (double)nnz) {
      std::sort(offs.begin(), offs.end());
      const int nd = (int)offs.size();
      const int64_t ld = ctx.ld(n);
      std::vector<int32_t> off32(offs.begin(), offs.end());
      op->offsets = off32;
      op->ndiag = nd;
      op->dia_ld = ld;
      // Constant-diagonal form: every entry of diagonal d bit-equal to one value (constant-
      // coefficient stencils). Then only a presence mask per row streams from HBM.
      std::vector<uint64_t> cbits(nd, 0);
      std::vector<char> seen(nd, 0);
      bool constant = nd <= kMaxConstDiag && n < (int64_t(1) << 30) && std::getenv("MSTAB_NO_CDIA") == nullptr;
      std::vector<uint32_t> mask;
      if (constant) mask.assign((size_t)ld, 0u);
      for (int64_t i = 0; i < n && constant; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
          const int d = (int)(std::lower_bound(offs.begin(), offs.end(), col_idx[k] - i) - offs.begin());
          uint64_t bits;
          std::memcpy(&bits, &values[k], sizeof bits);
          if (!seen[d]) {
            seen[d] = 1;
            cbits[d] = bits;
          } else if (bits != cbits[d]) {
            constant = false;
            break;
          }
          mask[(size_t)i] |= 1u << d;
        }
      op->dia_off = ctx.alloc(sizeof(int32_t) * nd);
      CUDA_OK(cudaMemcpyAsync(op->dia_off->ptr, off32.data(), sizeof(int32_t) * nd, cudaMemcpyHostToDevice, st));
      for (int d = 0; d < nd && constant; ++d) {  // absent terms add cval * (+0.0): needs finite cval
        double v;
        std::memcpy(&v, &cbits[d], sizeof v);
        if (!std::isfinite(v)) constant = false;
      }
      if (constant) {
        const int mb = nd <= 8 ? 1 : (nd <= 16 ? 2 : 4);
        op->mask_bytes = mb;
        op->cvals.resize(nd);
        for (int d = 0; d < nd; ++d) std::memcpy(&op->cvals[d], &cbits[d], sizeof(double));
        std::vector<uint8_t> packed((size_t)ld * mb);
        for (size_t i = 0; i < (size_t)ld; ++i)
          for (int byte = 0; byte < mb; ++byte) packed[i * mb + byte] = (uint8_t)(mask[i] >> (8 * byte));
        op->dia_mask = ctx.alloc(packed.size());
        CUDA_OK(cudaMemcpyAsync(op->dia_mask->ptr, packed.data(), packed.size(), cudaMemcpyHostToDevice, st));
      } else {
        std::vector<double> dv((size_t)nd * ld, 0.0);
        for (int64_t i = 0; i < n; ++i)
          for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            const int d = (int)(std::lower_bound(offs.begin(), offs.end(), col_idx[k] - i) - offs.begin());
            dv[(size_t)d * ld + i] = values[k];
          }
        op->dia_val = ctx.alloc(sizeof(double) * dv.size());
        CUDA_OK(cudaMemcpyAsync(op->dia_val->ptr, dv.data(), sizeof(double) * dv.size(), cudaMemcpyHostToDevice, st));
      }
      ctx.sync();
    }
  }
  ctx.sync();
}

}  // namespace

std::shared_ptr<Operator> make_operator(Context& ctx, int64_t n, const int64_t* row_ptr,
                                        const int64_t* col_idx, const double* values) {
  const int64_t nnz = validate_csr(n, row_ptr, col_idx);
  static_cast<void>(nnz);
  auto op = std::make_shared<Operator>();
  op->uid = next_operator_uid();
  op->fingerprint = fnv_csr_fingerprint(n, row_ptr, col_idx, values, row_ptr[n]);
  op->n_global = n;
  op->xlo = 0;
  op->xhi = n;
  upload_rows(ctx, op.get(), n, row_ptr, col_idx, values);
  return op;
}

// Row slab of rank r: the rank's rows with columns relative to its first row,
// the halo column range its rows reference, and the exchange plan. The send side is derived from
// the peers' rows of the same global CSR, so the plans of all ranks match by construction.
// Interior rows of a slab (columns relative to the slab's first row): the largest [lo, hi) around the
// middle whose rows reference owned columns only.
void interior_rows(Operator* op, int64_t nl, const std::vector<int64_t>& rp, const std::vector<int64_t>& ci) {
  auto needs_halo = [&](int64_t r) {
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k)
      if (ci[k] < 0 || ci[k] >= nl) return true;
    return false;
  };
  int64_t lo = 0, hi = nl;
  const int64_t mid = nl / 2;
  for (int64_t r = 0; r < mid; ++r)
    if (needs_halo(r)) lo = r + 1;
  for (int64_t r = nl - 1; r >= mid; --r)
    if (needs_halo(r)) hi = r;
  op->int_lo = lo;
  op->int_hi = std::max(lo, hi);
}

std::shared_ptr<Operator> make_operator_slab(Context& ctx, int64_t n, const int64_t* row_ptr,
                                             const int64_t* col_idx, const double* values,
                                             const int64_t* slabs) {
  if (!ctx.comm) throw Error(MSTAB_E_CONFIG, "slab operator: the context has no communicator");
  const int world = ctx.comm->world(), rank = ctx.comm->rank();
  validate_csr(n, row_ptr, col_idx);
  if (slabs[0] != 0 || slabs[world] != n) throw Error(MSTAB_E_DIMENSION, "slab operator: boundaries must span 0..n");
  for (int r = 0; r < world; ++r)
    if (slabs[r] > slabs[r + 1]) throw Error(MSTAB_E_DIMENSION, "slab operator: boundaries not ascending");
  // column span [lo, hi) referenced by each rank's rows (at least its own rows)
  std::vector<int64_t> lo(world), hi(world);
  for (int r = 0; r < world; ++r) {
    lo[r] = slabs[r];
    hi[r] = slabs[r + 1];
    for (int64_t k = row_ptr[slabs[r]]; k < row_ptr[slabs[r + 1]]; ++k) {
      lo[r] = std::min(lo[r], col_idx[k]);
      hi[r] = std::max(hi[r], col_idx[k] + 1);
    }
  }
  const int64_t start = slabs[rank], end = slabs[rank + 1], nl = end - start;
  if (nl < 1) throw Error(MSTAB_E_DIMENSION, "slab operator: empty slab");
  auto op = std::make_shared<Operator>();
  op->uid = next_operator_uid();
  op->fingerprint = fnv_csr_fingerprint(n, row_ptr, col_idx, values, row_ptr[n]);
  op->n_global = n;
  op->row0 = start;
  op->xlo = lo[rank] - start;
  op->xhi = hi[rank] - start;
  auto overlap = [](int64_t a0, int64_t a1, int64_t b0, int64_t b1, int64_t& o0, int64_t& o1) {
    o0 = std::max(a0, b0);
    o1 = std::min(a1, b1);
    return o0 < o1;
  };
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    int64_t o0, o1;
    // halo rows of mine owned by p (left and right of my slab)
    if (overlap(lo[rank], start, slabs[p], slabs[p + 1], o0, o1)) op->halo.recvs.push_back({p, o0 - start, o1 - o0});
    if (overlap(end, hi[rank], slabs[p], slabs[p + 1], o0, o1)) op->halo.recvs.push_back({p, o0 - start, o1 - o0});
    // my rows that p references outside its slab
    if (overlap(lo[p], slabs[p], start, end, o0, o1)) op->halo.sends.push_back({p, o0 - start, o1 - o0});
    if (overlap(slabs[p + 1], hi[p], start, end, o0, o1)) op->halo.sends.push_back({p, o0 - start, o1 - o0});
  }
  // vector layout of this context: owned rows after a 64-aligned left halo
  ctx.lay_n = nl;
  ctx.lay_lo = (start - lo[rank] + 63) / 64 * 64;
  ctx.lay_ld = padded_ld(ctx.lay_lo + nl + (hi[rank] - end));
  ctx.lay_row0 = start;
  ctx.lay_nglobal = n;
  ctx.ws.reset();
  ctx.pcache.reset();
  ctx.val_au.reset();
  ctx.val_au_n = -1;
  std::vector<int64_t> rp(nl + 1), ci(row_ptr[end] - row_ptr[start]);
  for (int64_t i = 0; i <= nl; ++i) rp[i] = row_ptr[start + i] - row_ptr[start];
  for (size_t k = 0; k < ci.size(); ++k) ci[k] = col_idx[row_ptr[start] + (int64_t)k] - start;
  upload_rows(ctx, op.get(), nl, rp.data(), ci.data(), values + row_ptr[start]);
  interior_rows(op.get(), nl, rp, ci);
  if (!ctx.xgath) ctx.xgath = ctx.alloc(sizeof(double) * (size_t)world * kMaxXred);
  return op;
}

// The same slab from the rank's OWN rows (column indices global): no rank needs the global CSR.
// What make_operator_slab derives from the global matrix arrives as arguments instead: the column
// span [lo_r, hi_r) of every rank's rows (spans: 2 x world, allgathered by the caller) and the
// reference fingerprint of the global matrix (fnv_begin / fnv_fold_*: a relay over the ranks).
std::shared_ptr<Operator> make_operator_slab_local(Context& ctx, int64_t n_global, const int64_t* slabs,
                                                   const int64_t* row_ptr, const int64_t* col_idx,
                                                   const double* values, const int64_t* spans,
                                                   uint64_t fingerprint) {
  if (!ctx.comm) throw Error(MSTAB_E_CONFIG, "slab operator: the context has no communicator");
  const int world = ctx.comm->world(), rank = ctx.comm->rank();
  if (slabs[0] != 0 || slabs[world] != n_global)
    throw Error(MSTAB_E_DIMENSION, "slab operator: boundaries must span 0..n");
  for (int r = 0; r < world; ++r)
    if (slabs[r] > slabs[r + 1]) throw Error(MSTAB_E_DIMENSION, "slab operator: boundaries not ascending");
  const int64_t start = slabs[rank], end = slabs[rank + 1], nl = end - start;
  if (nl < 1) throw Error(MSTAB_E_DIMENSION, "slab operator: empty slab");
  // CsrMatrix::validate (csr.cpp:11-24) on the local rows, columns against the global size
  if (row_ptr[0] != 0) throw Error(MSTAB_E_ERROR, "csr: row_ptr bounds");
  int64_t lo_own = start, hi_own = end;
  for (int64_t i = 0; i < nl; ++i) {
    if (row_ptr[i] > row_ptr[i + 1]) throw Error(MSTAB_E_ERROR, "csr: row_ptr not nondecreasing");
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      if (col_idx[k] < 0 || col_idx[k] >= n_global) throw Error(MSTAB_E_ERROR, "csr: column index out of range");
      if (k > row_ptr[i] && col_idx[k - 1] >= col_idx[k])
        throw Error(MSTAB_E_ERROR, "csr: columns not strictly increasing within a row");
      lo_own = std::min(lo_own, col_idx[k]);
      hi_own = std::max(hi_own, col_idx[k] + 1);
    }
  }
  std::vector<int64_t> lo(world), hi(world);
  for (int r = 0; r < world; ++r) {
    lo[r] = std::min(spans[2 * r], slabs[r]);
    hi[r] = std::max(spans[2 * r + 1], slabs[r + 1]);
  }
  if (lo[rank] > lo_own || hi[rank] < hi_own)
    throw Error(MSTAB_E_DIMENSION, "slab operator: this rank's column span does not cover its rows");
  auto op = std::make_shared<Operator>();
  op->uid = next_operator_uid();
  op->fingerprint = fingerprint;
  op->n_global = n_global;
  op->row0 = start;
  op->xlo = lo[rank] - start;
  op->xhi = hi[rank] - start;
  auto overlap = [](int64_t a0, int64_t a1, int64_t b0, int64_t b1, int64_t& o0, int64_t& o1) {
    o0 = std::max(a0, b0);
    o1 = std::min(a1, b1);
    return o0 < o1;
  };
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    int64_t o0, o1;
    if (overlap(lo[rank], start, slabs[p], slabs[p + 1], o0, o1)) op->halo.recvs.push_back({p, o0 - start, o1 - o0});
    if (overlap(end, hi[rank], slabs[p], slabs[p + 1], o0, o1)) op->halo.recvs.push_back({p, o0 - start, o1 - o0});
    if (overlap(lo[p], slabs[p], start, end, o0, o1)) op->halo.sends.push_back({p, o0 - start, o1 - o0});
    if (overlap(slabs[p + 1], hi[p], start, end, o0, o1)) op->halo.sends.push_back({p, o0 - start, o1 - o0});
  }
  ctx.lay_n = nl;
  ctx.lay_lo = (start - lo[rank] + 63) / 64 * 64;
  ctx.lay_ld = padded_ld(ctx.lay_lo + nl + (hi[rank] - end));
  ctx.lay_row0 = start;
  ctx.lay_nglobal = n_global;
  ctx.ws.reset();
  ctx.pcache.reset();
  ctx.val_au.reset();
  ctx.val_au_n = -1;
  std::vector<int64_t> ci((size_t)row_ptr[nl]);
  for (size_t k = 0; k < ci.size(); ++k) ci[k] = col_idx[k] - start;
  upload_rows(ctx, op.get(), nl, row_ptr, ci.data(), values);
  interior_rows(op.get(), nl, std::vector<int64_t>(row_ptr, row_ptr + nl + 1), ci);
  if (!ctx.xgath) ctx.xgath = ctx.alloc(sizeof(double) * (size_t)world * kMaxXred);
  return op;
}

// ---- split preconditioning (precond.cpp) --------------------------------------------------------
namespace {

// max |a_ij| (precond.cpp:13-17)
double diag_scale(int64_t nnz, const double* values) {
  double s = 0.0;
  for (int64_t k = 0; k < nnz; ++k) s = std::max(s, std::abs(values[k]));
  return s;
}

std::string zero_pivot(int64_t row) { return "zero pivot in row " + std::to_string(row); }

// Builds the CSR of a factor from per-row (col, value) lists already in ascending column order.
void emit_rows(int64_t n, const std::vector<std::vector<std::pair<int64_t, double>>>& rows, int64_t* rp,
               int64_t* ci, double* val) {
  rp[0] = 0;
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (const auto& e : rows[i]) {
      ci[k] = e.first;
      val[k] = e.second;
      ++k;
    }
    rp[i + 1] = k;
  }
}

// Dependency levels of a triangular factor (the wavefront schedule of lower_solve / upper_solve,
// precond.cpp:95-127): level(i) = 1 + max level(j) over the entries lower_solve reads (j < i; j > i
// for an upper factor), 0 for a row without any. Rows of one level are independent, so the device
// solve gives each lane its own row. Returns the level-sorted slot list (ascending rows within a
// level, every level padded with -1 to a multiple of 32) and the level count.
std::vector<int32_t> level_schedule(int64_t n, const int64_t* rp, const int64_t* ci, bool lower, int64_t& nlevels) {
  std::vector<int32_t> lev(n, 0);
  int32_t maxlev = -1;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = lower ? t : n - 1 - t;
    int32_t l = 0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t j = ci[k];
      if (lower ? j < i : j > i) l = std::max(l, lev[j] + 1);
    }
    lev[i] = l;
    maxlev = std::max(maxlev, l);
  }
  nlevels = maxlev + 1;
  std::vector<int64_t> cnt(nlevels + 1, 0);
  for (int64_t i = 0; i < n; ++i) ++cnt[lev[i] + 1];
  std::vector<int64_t> start(nlevels + 1, 0);  // padded slot offset of each level
  for (int64_t l = 0; l < nlevels; ++l) start[l + 1] = start[l] + (cnt[l + 1] + 31) / 32 * 32;
  std::vector<int32_t> order(start[nlevels], -1);
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  for (int64_t i = 0; i < n; ++i) order[fill[lev[i]]++] = (int32_t)i;
  return order;
}

DevTri upload_factor(Context& ctx, int64_t n, const int64_t* rp, const int64_t* ci, const double* val, bool lower,
                     DevPtr& d_rp, DevPtr& d_ci, DevPtr& d_val, DevPtr& d_diag, DevPtr& d_ord) {
  DevTri f;
  f.n = n;
  f.nnz = rp[n];
  f.lower = lower;
  cudaStream_t st = ctx.stream();
  bool diagonal = f.nnz == n;
  for (int64_t i = 0; i < n && diagonal; ++i) diagonal = rp[i + 1] - rp[i] == 1 && ci[rp[i]] == i;
  if (diagonal) {  // split Jacobi: the factor is its diagonal
    d_diag = ctx.alloc(sizeof(double) * std::max<int64_t>(n, 1));
    CUDA_OK(cudaMemcpyAsync(d_diag->ptr, val, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    f.diag = d_diag->d();
    ctx.sync();
    return f;
  }
  std::vector<int32_t> rp32(n + 1), ci32(std::max<int64_t>(f.nnz, 1));
  for (int64_t i = 0; i <= n; ++i) rp32[i] = (int32_t)rp[i];
  for (int64_t k = 0; k < f.nnz; ++k) ci32[k] = (int32_t)ci[k];
  d_rp = ctx.alloc(sizeof(int32_t) * (n + 1));
  d_ci = ctx.alloc(sizeof(int32_t) * ci32.size());
  d_val = ctx.alloc(sizeof(double) * ci32.size());
  CUDA_OK(cudaMemcpyAsync(d_rp->ptr, rp32.data(), sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, st));
  CUDA_OK(cudaMemcpyAsync(d_ci->ptr, ci32.data(), sizeof(int32_t) * ci32.size(), cudaMemcpyHostToDevice, st));
  CUDA_OK(cudaMemcpyAsync(d_val->ptr, val, sizeof(double) * std::max<int64_t>(f.nnz, 0), cudaMemcpyHostToDevice, st));
  f.rp = static_cast<const int32_t*>(d_rp->ptr);
  f.ci = static_cast<const int32_t*>(d_ci->ptr);
  f.val = d_val->d();
  const std::vector<int32_t> order = level_schedule(n, rp, ci, lower, f.nlevels);
  f.nslots = (int64_t)order.size();
  d_ord = ctx.alloc(sizeof(int32_t) * std::max<size_t>(order.size(), 1));
  CUDA_OK(cudaMemcpyAsync(d_ord->ptr, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice, st));
  f.order = static_cast<const int32_t*>(d_ord->ptr);
  ctx.sync();
  return f;
}

}  // namespace

void precond_build(int kind, int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                   int64_t* l_rp, int64_t* l_ci, double* l_val, int64_t* r_rp, int64_t* r_ci, double* r_val) {
  validate_csr(n, row_ptr, col_idx);
  const int64_t nnz = row_ptr[n];
  const double scale = diag_scale(nnz, values);
  std::vector<std::vector<std::pair<int64_t, double>>> lrows(n), rrows(n);
  if (kind == MSTAB_PRECOND_JACOBI) {  // build_jacobi (precond.cpp:23-37)
    for (int64_t i = 0; i < n; ++i) {
      double d = 0.0;
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
        if (col_idx[k] == i) d = values[k];
      if (std::abs(d) < 1e-14 * scale || scale == 0.0) throw Error(MSTAB_E_ZEROPIVOT, zero_pivot(i), i);
      // std::sqrt of a complex with a negative real part is imaginary: not a real operator
      if (d < 0.0) throw Error(MSTAB_E_NOTREAL, "jacobi: negative diagonal gives a complex square root");
      lrows[i].push_back({i, std::sqrt(d)});
      rrows[i].push_back({i, std::sqrt(d)});
    }
  } else if (kind == MSTAB_PRECOND_ILU0) {  // build_ilu0 (precond.cpp:39-99), IKJ on A's pattern
    std::vector<double> val(values, values + nnz);
    std::vector<int64_t> diag_pos(n, -1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
        if (col_idx[k] == i) diag_pos[i] = k;
    for (int64_t i = 0; i < n; ++i)
      if (diag_pos[i] < 0) throw Error(MSTAB_E_ZEROPIVOT, zero_pivot(i), i);
    for (int64_t i = 0; i < n; ++i) {
      for (int64_t ki = row_ptr[i]; ki < row_ptr[i + 1]; ++ki) {
        const int64_t k = col_idx[ki];
        if (k >= i) break;
        const double piv = val[diag_pos[k]];
        if (std::abs(piv) < 1e-14 * scale || scale == 0.0) throw Error(MSTAB_E_ZEROPIVOT, zero_pivot(k), k);
        const double lik = val[ki] / piv;
        val[ki] = lik;
        int64_t pk = diag_pos[k] + 1, pi = ki + 1;
        while (pk < row_ptr[k + 1] && pi < row_ptr[i + 1]) {
          if (col_idx[pk] < col_idx[pi]) {
            ++pk;
          } else if (col_idx[pk] > col_idx[pi]) {
            ++pi;
          } else {
            val[pi] = val[pi] - lik * val[pk];
            ++pk;
            ++pi;
          }
        }
      }
      if (std::abs(val[diag_pos[i]]) < 1e-14 * scale || scale == 0.0) throw Error(MSTAB_E_ZEROPIVOT, zero_pivot(i), i);
    }
    // unit lower L (explicit 1.0 diagonal, last in its row) and upper R carrying the pivots
    for (int64_t i = 0; i < n; ++i) {
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        if (col_idx[k] < i)
          lrows[i].push_back({col_idx[k], val[k]});
        else
          rrows[i].push_back({col_idx[k], val[k]});
      }
      lrows[i].push_back({i, 1.0});
    }
  } else {
    throw Error(MSTAB_E_CONFIG, "precond: unknown kind");
  }
  emit_rows(n, lrows, l_rp, l_ci, l_val);
  emit_rows(n, rrows, r_rp, r_ci, r_val);
}

std::shared_ptr<Operator> make_operator_precond(Context& ctx, int64_t n, const int64_t* row_ptr,
                                                const int64_t* col_idx, const double* values, int kind,
                                                const int64_t* l_rp, const int64_t* l_ci, const double* l_val,
                                                const int64_t* r_rp, const int64_t* r_ci, const double* r_val) {
  if (ctx.comm) throw Error(MSTAB_E_CONFIG, "b200: preconditioned operators are single-GPU");
  auto op = make_operator(ctx, n, row_ptr, col_idx, values);
  if (kind == MSTAB_PRECOND_NONE) return op;
  if (kind != MSTAB_PRECOND_JACOBI && kind != MSTAB_PRECOND_ILU0) throw Error(MSTAB_E_CONFIG, "precond: unknown kind");
  validate_csr(n, l_rp, l_ci);
  validate_csr(n, r_rp, r_ci);
  for (int64_t i = 0; i < n; ++i) {  // the solves need one stored diagonal entry per row
    bool dl = false, dr = false;
    for (int64_t k = l_rp[i]; k < l_rp[i + 1]; ++k) dl = dl || (l_ci[k] == i && l_val[k] != 0.0);
    for (int64_t k = r_rp[i]; k < r_rp[i + 1]; ++k) dr = dr || (r_ci[k] == i && r_val[k] != 0.0);
    if (!dl || !dr) throw Error(MSTAB_E_ZEROPIVOT, zero_pivot(i), i);
  }
  // PreconditionedOperator::fingerprint (precond.cpp:203-210)
  uint64_t h = op->fingerprint;
  const uint64_t hl = fnv_csr_fingerprint(n, l_rp, l_ci, l_val, l_rp[n]);
  h ^= hl + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  const uint64_t hr = fnv_csr_fingerprint(n, r_rp, r_ci, r_val, r_rp[n]);
  h ^= hr + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  op->fingerprint = h;
  auto pc = std::make_shared<Precond>();
  pc->kind = kind;
  pc->L = upload_factor(ctx, n, l_rp, l_ci, l_val, true, pc->l_rp, pc->l_ci, pc->l_val, pc->l_diag, pc->l_ord);
  pc->R = upload_factor(ctx, n, r_rp, r_ci, r_val, false, pc->r_rp, pc->r_ci, pc->r_val, pc->r_diag, pc->r_ord);
  pc->t1 = ctx.alloc_vecs(n, 1);
  pc->t2 = ctx.alloc_vecs(n, 1);
  pc->t3 = ctx.alloc_vecs(n, 1);
  pc->sync = ctx.alloc(sizeof(int) * (size_t)(n + 1));
  op->pc = pc;
  return op;
}

void precond_solve(Context& ctx, const Operator& op, int which, const double* x_dev, double* y_dev) {
  if (!op.pc) {  // build_none: both factors are the identity
    CUDA_OK(cudaMemcpyAsync(y_dev, x_dev, sizeof(double) * op.n, cudaMemcpyDeviceToDevice, ctx.stream()));
    return;
  }
  if (x_dev == y_dev) {  // the level-scheduled solve uses its output as the done flags
    CUDA_OK(cudaMemcpyAsync(op.pc->t3->d(), x_dev, sizeof(double) * op.n, cudaMemcpyDeviceToDevice, ctx.stream()));
    x_dev = op.pc->t3->d();
  }
  launch_tri_solve(ctx.stream(), which == 0 ? op.pc->L : op.pc->R, x_dev, y_dev,
                   reinterpret_cast<int*>(op.pc->sync->ptr));
  check_launch();
}

void spmv(Context& ctx, const Operator& op, const double* x_dev, double* y_dev) {
  reset_status(ctx);
  spmv_dev(ctx, op, x_dev, y_dev);
}

mstab_validation_report validate(Context& ctx, const Recycle& rd, const Operator& op) {
  if (rd.fingerprint != op.fingerprint)
    throw Error(MSTAB_E_FINGERPRINT, "recycle data belongs to a different operator");
  if (rd.n != op.n) throw Error(MSTAB_E_DIMENSION, "recycle data has inconsistent shapes");
  if (!rd.omega.empty() && (int64_t)rd.omega.size() != rd.level_j)
    throw Error(MSTAB_E_STALE, "recycle data: omega history length disagrees with level");
  const int s = (int)rd.s;
  if (s < 1 || s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: recycle s must be in 1..16");
  const int64_t vld = ctx.ld(rd.n);
  const double* au = nullptr;
  // Large operators form A U with the cycle's own SpMV kernel, one column at a time (the
  // constant-diagonal / DIA / banded-ring forms stream at 0.65-0.85 of HBM; the thread-per-row CSR
  // product inside k_validate reached 0.15-0.25: r01 profiles), then k_validate reduces
  // ||V - A U||, ||V||, P^H P and V^H V in one pass over the stored products. Same row sums in the
  // same order, so the deviation is unchanged bit for bit. Small operators keep the single launch.
  const bool by_spmv = !op.pc && op.n_global >= kCholQrMinRows && std::getenv("MSTAB_VALIDATE_FUSED") == nullptr;
  if (by_spmv) {
    if (!ctx.val_au || ctx.val_au_n != op.n || ctx.val_au_s < s) {
      ctx.sync();
      ctx.val_au = ctx.alloc_vecs(op.n, s);
      ctx.val_au_n = op.n;
      ctx.val_au_s = s;
    }
    for (int q = 0; q < s; ++q) spmv_dev(ctx, op, rd.u->d() + (size_t)q * vld, ctx.val_au->d() + (size_t)q * vld);
    au = ctx.val_au->d();
  } else {
    for (int q = 0; q < s && ctx.sharded(); ++q) halo(ctx, op, rd.u->d() + (size_t)q * vld);
  }
  if (op.pc) {  // A U through the preconditioned chain, column by column
    Precond& pc = *op.pc;
    if (!pc.au || pc.au_s < s) {
      ctx.sync();
      pc.au = ctx.alloc_vecs(op.n, s);
      pc.au_s = s;
    }
    for (int q = 0; q < s; ++q) precond_chain(ctx, op, rd.u->d() + (size_t)q * vld, pc.au->d() + (size_t)q * vld);
    au = pc.au->d();
  }
  launch_validate(ctx.stream(), op.csr(), rd.p->d(), rd.u->d(), rd.v->d(), vld, s, ctx.reducer(), au);
  check_launch();
  if (ctx.sharded()) {
    ctx.comm->allreduce_sum(xred(ctx), 2 + 2 * s * s, ctx.stream());
    launch_fin_copy(ctx.stream(), xred(ctx), ctx.ds()->scal, 2);
    launch_fin_copy(ctx.stream(), xred(ctx) + 2, ctx.ds()->gram, 2 * s * s);
    check_launch();
  }
  std::vector<double> gram(2 * (size_t)s * s);
  CUDA_OK(cudaMemcpyAsync(gram.data(), ctx.ds()->gram, sizeof(double) * gram.size(),
                          cudaMemcpyDeviceToHost, ctx.stream()));
  const double* h = read_scal(ctx, 2);
  const double dev_num = h[0], dev_den = h[1];
  const double dev_v = dev_den > 0.0 ? std::sqrt(dev_num) / std::sqrt(dev_den) : std::sqrt(dev_num);
  double dev_p = 0.0;
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < s; ++i) {
      const double want = (i == j) ? 1.0 : 0.0;
      dev_p = std::max(dev_p, std::abs(gram[(size_t)i + (size_t)j * s] - want));
    }
  mstab_validation_report rep{};
  rep.max_deviation = std::max(dev_v, dev_p);
  if (rep.max_deviation > 1e-6) throw Error(MSTAB_E_STALE, "recycle data deviates from its invariants");
  const auto ev = symmetric_eigenvalues(gram.data() + (size_t)s * s, s);
  const double smin = std::sqrt(std::max(0.0, ev.front()));
  const double smax = std::sqrt(std::max(0.0, ev.back()));
  rep.sigma_min_ratio = smax > 0.0 ? smin / smax : 0.0;
  rep.low_rank_warning = rep.sigma_min_ratio < 1e-10 ? 1 : 0;
  return rep;
}

void CycleGraph::reset() {
  if (exec) cudaGraphExecDestroy(exec);
  exec = nullptr;
  kernels = 0;
  if (!prof.empty()) prof_release(prof);
}

namespace {

Workspace& workspace(Context& ctx, const Operator& op, int s, int ell, bool tres) {
  auto& w = ctx.ws;
  if (w && w->op_uid == op.uid && w->n == op.n && w->s == s && w->ell == ell && w->tres == tres) return *w;
  ctx.sync();
  w = std::make_unique<Workspace>();
  w->op_uid = op.uid;
  w->n = op.n;
  w->s = s;
  w->ell = ell;
  w->tres = tres;
  const int64_t n = op.n;
  for (auto& set : w->set) {
    set.x = ctx.alloc_vecs(n, 1);
    set.r = ctx.alloc_vecs(n, 1);
    set.U = ctx.alloc_vecs(n, s);
    set.V = ctx.alloc_vecs(n, s);
  }
  w->R.resize(ell + 1);
  w->VL.resize(ell + 1);
  for (int i = 1; i <= ell; ++i) {
    w->R[i] = ctx.alloc_vecs(n, 1);
    w->VL[i] = ctx.alloc_vecs(n, s);
  }
  w->b = ctx.alloc_vecs(n, 1);
  w->P = ctx.alloc_vecs(n, s);
  // Small, L2-resident problems run each cycle as one cooperative kernel out of registers
  // (kpersist.cu) when (s, ell) is instantiated and one row per thread fits the device. Tiny
  // systems (the reference's dense-step tests, n < 4096) keep the stream-of-kernels path, whose
  // Givens least squares their 1e-12 trajectory tolerances were calibrated against.
  if (!ctx.sharded() && !op.pc && n >= 4096 && std::getenv("MSTAB_NO_PERSIST") == nullptr &&
      (size_t)persist_partials_doubles(n) * sizeof(double) <= ctx.partials->bytes &&
      launch_persist_cycle(ctx.stream(), op.csr(), n, ctx.ld(n), s, ell, nullptr, nullptr, nullptr, nullptr, nullptr,
                           nullptr, nullptr, nullptr, nullptr, tres ? w->b->d() : nullptr, nullptr, nullptr, nullptr,
                           nullptr, true)) {
    w->xbuf = ctx.alloc_vecs(n + 64, 1);  // the last 4 bytes' worth past n: the grid barrier counter
    w->persist = true;
  }
  // Result blocks of the solves to come (x; U, V of the fetched and the final recycle data): a solve
  // hands out four fresh n x s blocks and the caller usually still holds the previous solve's. On
  // this pool a cudaMallocAsync that has to grow the driver's pool stalled for 40-300 ms at random
  // (r02 stall probe), so the blocks are created here, once, and parked in the stream's cache:
  // twelve n x s blocks (two solves' worth plus what a caller's garbage collector may sit on) and
  // three vectors. Blocks cached for a previous workspace shape are released first.
  if (std::getenv("MSTAB_NO_BLOCK_CACHE") == nullptr) {
    ctx.sh->drop_cache();
    // sixteen blocks when they are small against the free memory (c2: 2 GB), never more than a
    // quarter of it (c4, 3.6 GB per block: nine)
    size_t free_b = 0, total_b = 0;
    int nblocks = 16;
    const size_t block_bytes = sizeof(double) * (size_t)ctx.ld(n) * (size_t)s;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && block_bytes > 0)
      nblocks = (int)std::min<size_t>(16, (free_b / 4) / block_bytes);
    std::vector<DevPtr> warm;
    for (int i = 0; i < nblocks; ++i) warm.push_back(ctx.alloc_vecs(n, s));
    for (int i = 0; i < 3; ++i) warm.push_back(ctx.alloc_vecs(n, 1));
  }
  return *w;
}

// Everything one cycle enqueues (idrstab.cpp:250-273), set[p] -> set[1-p].
void enqueue_full_cycle(Context& ctx, const Operator& op, Workspace& w, int p) {
  const WSet& S = w.set[p];
  const WSet& D = w.set[1 - p];
  enqueue_cycle(ctx, op, w.P->d(), w.s, w.ell, S, D, w.R, w.VL);
  if (w.tres) {  // r = b - A x (idrstab.cpp:268-273)
    FinParams ft;
    ft.op = kFinTrueRes;
    ft.s = w.s;
    ft.ell = w.ell;
    if (ctx.sharded())
      apply_ph_sharded(ctx, op, D.x->d(), D.r->d(), w.P->d(), w.s, w.b->d(), ft);
    else
      apply_ph(ctx, op, D.x->d(), D.r->d(), w.P->d(), w.s, w.b->d(), ft);
    check_launch();
    after_spmv(ctx, w.s, true, ft);
  }
}

// Runs one cycle: replays the captured graph of parity p (capturing it on first use), or
// launches the kernels directly when graphs are off.
void run_cycle(Context& ctx, const Operator& op, Workspace& w, int p, double stop_below = -1.0,
               HostCycleSlot* hslot = nullptr, uint64_t seq = 0) {
  cudaStream_t st = ctx.stream();
  if (w.persist) {
    const WSet& S = w.set[p];
    const WSet& D = w.set[1 - p];
    launch_persist_cycle(st, op.csr(), op.n, ctx.ld(op.n), w.s, w.ell, S.x->d(), S.r->d(), S.U->d(), S.V->d(),
                         D.x->d(), D.r->d(), D.U->d(), D.V->d(), w.P->d(), w.tres ? w.b->d() : nullptr, w.xbuf->d(),
                         ctx.partials->d(), ctx.ds(), reinterpret_cast<unsigned*>(w.xbuf->d() + ctx.ld(op.n)), false,
                         stop_below, hslot, seq);
    check_launch();
    return;
  }
  if (!ctx.use_graphs || (ctx.comm && !ctx.comm->capturable())) {
    enqueue_full_cycle(ctx, op, w, p);
    return;
  }
  CycleGraph& g = w.graph[p];
  const bool prof = prof_enabled();
  if (g.exec && g.profiled != prof) g.reset();
  if (!g.exec) {
    cudaGraph_t graph = nullptr;
    const uint64_t l0 = launch_count();
    CUDA_OK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    prof_set_capture_list(prof ? &g.prof : nullptr);
    try {
      enqueue_full_cycle(ctx, op, w, p);
    } catch (...) {
      prof_set_capture_list(nullptr);
      cudaStreamEndCapture(st, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    prof_set_capture_list(nullptr);
    CUDA_OK(cudaStreamEndCapture(st, &graph));
    g.kernels = launch_count() - l0;
    cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) throw Error(MSTAB_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    g.profiled = prof;
    // capture counted the launches once; replays count them below
    count_launches((uint64_t)0 - g.kernels);
  }
  CUDA_OK(cudaGraphLaunch(g.exec, st));
  count_launches(g.kernels);
}

// Runs one cycle and reads its status. A persistent-kernel cycle that asks for the other path
// (kBreakFallback: its least squares left the CholeskyQR2 regime) is rerun on the stream of kernels
// from the same, untouched source set, and the workspace stays on that path.
const CycleStatus& run_cycle_sync(Context& ctx, const Operator& op, Workspace& w, int p) {
  run_cycle(ctx, op, w, p);
  const CycleStatus* cs = &read_status(ctx);
  if (w.persist && cs->breakdown == kBreakFallback) {
    w.persist = false;
    reset_status(ctx);
    run_cycle(ctx, op, w, p);
    cs = &read_status(ctx);
  }
  return *cs;
}

// Persistent cycles, pipelined (L2-resident systems: a cycle is ~90 us, so the host's status read
// and relaunch, ~16 us, were 13% of it). The cycle of this iteration is in flight or launched now;
// when `ahead` allows, the NEXT cycle is launched behind it before its outcome is known: the kernel
// sets DevState::stop when its cycle ends the solve (residual <= stop_below, or a breakdown) and a
// cycle launched behind it returns without touching anything, so speculation never changes a
// result. The status does not come back through the stream (a copy would queue behind the
// speculative launch): CTA 0 writes it into one of two mapped host slots and the host polls the
// slot's sequence number.
const CycleStatus& persist_next(Context& ctx, const Operator& op, Workspace& w, int p, double stop_below, bool ahead) {
  HostCycleSlot* dslots = nullptr;
  CUDA_OK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dslots), ctx.hslots, 0));
  auto launch = [&](int parity) {
    const uint64_t seq = ++ctx.pipe_launched;
    run_cycle(ctx, op, w, parity, stop_below, dslots + (seq & 1), seq);
  };
  if (ctx.pipe_launched == ctx.pipe_consumed) launch(p);
  if (ahead && ctx.pipe_launched == ctx.pipe_consumed + 1) launch(1 - p);
  const uint64_t want = ctx.pipe_consumed + 1;
  HostCycleSlot& slot = ctx.hslots[want & 1];
  for (uint64_t spins = 0; slot.seq != want; ++spins) {
    if ((spins & 0xfff) == 0xfff) {  // a failed launch or a device fault would never write the slot
      cudaError_t e = cudaStreamQuery(ctx.stream());
      if (e != cudaSuccess && e != cudaErrorNotReady)
        throw Error(MSTAB_E_CUDA, std::string("persistent cycle: ") + cudaGetErrorString(e));
      if (e == cudaSuccess && slot.seq != want) throw Error(MSTAB_E_CUDA, "persistent cycle: no status written");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  ctx.pipe_consumed = want;
  *ctx.host_status = slot.st;
  const CycleStatus* cs = ctx.host_status;
  if (cs->breakdown == kBreakFallback) {
    // the least squares left the CholeskyQR2 regime: the cycle wrote nothing (and stopped the one
    // behind it); rerun it, and the rest of the solve, on the stream of kernels
    ctx.sync();
    ctx.pipe_launched = ctx.pipe_consumed;
    w.persist = false;
    reset_status(ctx);
    run_cycle(ctx, op, w, p);
    cs = &read_status(ctx);
  }
  return *cs;
}

DevPtr copy_vec(Context& ctx, const DevPtr& src, int64_t n) {
  DevPtr d = ctx.alloc_vecs(n, 1);
  CUDA_OK(cudaMemcpyAsync(d->d(), src->d(), sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx.stream()));
  return d;
}

}  // namespace

std::unique_ptr<SolveResultImpl> solve(Context& ctx, const Operator& op, const double* b_in,
                                       const double* x0_in, int mem, const mstab_solver_config& cfg,
                                       const Recycle* recycle, const mstab_fetch_policy* fetch) {
  // SolverConfig::validate (report.cpp:16-22)
  if (cfg.s < 1) throw Error(MSTAB_E_CONFIG, "config: s >= 1 required");
  if (cfg.ell < 1) throw Error(MSTAB_E_CONFIG, "config: ell >= 1 required");
  if (!(cfg.tol > 0.0)) throw Error(MSTAB_E_CONFIG, "config: tol > 0 required");
  if (cfg.max_mv < cfg.s + 1) throw Error(MSTAB_E_CONFIG, "config: max_mv >= s + 1 required");
  if (cfg.s > kMaxS || cfg.ell > kMaxEll)
    throw Error(MSTAB_E_CONFIG, "b200: s <= 16 and ell <= 8 are supported");
  if (fetch && fetch->kind == MSTAB_FETCH_AT_CYCLE && fetch->cycle < 1)
    throw Error(MSTAB_E_CONFIG, "fetch policy: cycle >= 1 required");
  const int s = (int)cfg.s, ell = (int)cfg.ell;
  const int64_t n = op.n, ld = ctx.ld(n);
  cudaStream_t st = ctx.stream();
  const bool tres = cfg.true_residual_each_cycle != 0;
  Workspace& w = workspace(ctx, op, s, ell, tres);
  reset_status(ctx);

  // b: ensure_finite + bnorm (idrstab.cpp:200, :205)
  std::optional<StallTrace> tr_in;
  tr_in.emplace("mstab: copy-in");
  CUDA_OK(cudaMemcpyAsync(w.b->d(), b_in, sizeof(double) * n,
                          mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  launch_vec_stats(st, n, w.b->d(), scal(ctx, 0), ctx.reducer());
  check_launch();
  after_stats(ctx, scal(ctx, 0));
  const double* h = read_scal(ctx, 3);
  tr_in.reset();
  if (h[1] > 0.0) throw Error(MSTAB_E_ERROR, "idrstab rhs: non-finite entries");
  const auto t0 = Clock::now();
  auto res = std::make_unique<SolveResultImpl>();
  res->n = n;
  mstab_report& rep = res->report;
  std::memset(&rep, 0, sizeof(rep));
  rep.ell = ell;
  rep.bnorm = std::sqrt(h[0]);

  int p = 0;  // the current state lives in w.set[p]
  WSet& c0 = w.set[0];
  bool x_zero = true;
  if (x0_in) {
    CUDA_OK(cudaMemcpyAsync(c0.x->d(), x0_in, sizeof(double) * n,
                            mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    launch_vec_stats(st, n, c0.x->d(), scal(ctx, 0), ctx.reducer());
    check_launch();
    after_stats(ctx, scal(ctx, 0));
    const double* hx = read_scal(ctx, 3);
    x_zero = hx[2] == 0.0;
    if (!x_zero && hx[1] > 0.0) throw Error(MSTAB_E_ERROR, "idrstab guess: non-finite entries");
  } else {
    CUDA_OK(cudaMemsetAsync(c0.x->ptr, 0, sizeof(double) * ld, st));
  }
  if (x_zero) {
    CUDA_OK(cudaMemcpyAsync(c0.r->d(), w.b->d(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  } else {  // r = b - A x0, one auxiliary MV (idrstab.cpp:210-216)
    spmv_dev(ctx, op, c0.x->d(), c0.r->d());
    launch_rsub(st, n, w.b->d(), c0.r->d());
    check_launch();
    rep.h_mv_aux++;
  }

  DevPtr P;
  int64_t base_level = 0;
  std::vector<std::complex<double>> omega_levels;
  bool omegas_complete = true;
  if (recycle) {
    {
      StallTrace tr("mstab: validate");
      validate(ctx, *recycle, op);
    }
    rep.h_mv_aux += recycle->s;
    if (recycle->s != cfg.s) throw Error(MSTAB_E_CONFIG, "idrstab: recycle s != config s");
    P = recycle->p;
    // the solve works on copies (idrstab.cpp:227-231): the recycle data stays immutable
    CUDA_OK(cudaMemcpyAsync(c0.U->ptr, recycle->u->ptr, sizeof(double) * ld * s, cudaMemcpyDeviceToDevice, st));
    CUDA_OK(cudaMemcpyAsync(c0.V->ptr, recycle->v->ptr, sizeof(double) * ld * s, cudaMemcpyDeviceToDevice, st));
    base_level = recycle->level_j;
    omega_levels = recycle->omega;
    omegas_complete = (int64_t)omega_levels.size() == base_level;
    if (!omegas_complete) omega_levels.clear();
  } else {
    // make_cut_space is a pure function of (n, s, seed): reuse the context's last draw when it
    // matches (bit-identical P, no host RNG or Gram-Schmidt on a restart)
    if (ctx.pcache && ctx.pcache_n == n && ctx.pcache_s == s && ctx.pcache_seed == cfg.seed) {
      P = ctx.pcache;
    } else {
      StallTrace tr("mstab: make_cut_space");
      P = make_cut_space(ctx, n, s, cfg.seed);
      ctx.pcache = P;
      ctx.pcache_n = n;
      ctx.pcache_s = s;
      ctx.pcache_seed = cfg.seed;
    }
    {
      StallTrace tr("mstab: arnoldi_init");
      arnoldi_init(ctx, op, c0.r->d(), s, cfg.seed ^ 0x9e3779b97f4a7c15ull, c0.U->d(), c0.V->d());
    }
    rep.h_mv += s;
  }
  if (w.p_src != P) {  // the graphs read P from the workspace copy
    CUDA_OK(cudaMemcpyAsync(w.P->ptr, P->ptr, sizeof(double) * ld * s, cudaMemcpyDeviceToDevice, st));
    w.p_src = P;
  }

  // P^H V, P^H r, ||r|| and gamma_0 of the first cycle
  reset_status(ctx);
  launch_prologue(st, n, ld, s, w.P->d(), c0.V->d(), c0.r->d(), ctx.reducer());
  check_launch();
  after_poly(ctx, s);
  double resnorm = read_status(ctx).resnorm;
  int64_t level = 0;
  res->history.push_back({0, rep.h_mv + rep.h_mv_aux, base_level, resnorm, ns_since(t0)});
  const double threshold = cfg.tol * rep.bnorm;

  bool broke = false;
  static const bool pipelined = std::getenv("MSTAB_NO_PERSIST_PIPELINE") == nullptr;
  ctx.pipe_launched = ctx.pipe_consumed = 0;
  ctx.hslots[0].seq = ctx.hslots[1].seq = 0;
  while (resnorm > threshold && rep.h_mv < cfg.max_mv) {
    const CycleStatus& cs = [&]() -> const CycleStatus& {
      StallTrace tr("mstab: cycle");
      if (w.persist && pipelined) {
        // no speculation past the product budget: the cycle after this one must still be allowed
        const bool ahead = rep.h_mv + 2 * (int64_t)ell * (s + 1) < cfg.max_mv;
        return persist_next(ctx, op, w, p, threshold, ahead);
      }
      return run_cycle_sync(ctx, op, w, p);
    }();
    if (w.graph[p].profiled) prof_accumulate(w.graph[p].prof);
    if (cs.breakdown) {  // BreakdownError: keep the last completed cycle (idrstab.cpp:290-293)
      rep.h_mv += cs.mv_at_breakdown;
      rep.status = MSTAB_STATUS_BREAKDOWN;
      std::snprintf(rep.breakdown_reason, sizeof(rep.breakdown_reason), "%s",
                    cs.breakdown == kBreakRank ? "least_squares_tall: stabilization block lost rank"
                                               : "solve_small: pivot collapse");
      broke = true;
      break;
    }
    p = 1 - p;
    rep.cycles++;
    level += ell;
    rep.h_mv += (int64_t)ell * (s + 1);
    rep.h_rd = level * s + (recycle ? base_level * (s - 1) : 0);
    std::vector<double> tau(cs.tau, cs.tau + ell);
    if (omegas_complete) omegas_complete = extract_omegas(tau, omega_levels);
    res->taus.insert(res->taus.end(), tau.begin(), tau.end());
    if (tres) rep.h_mv_aux++;
    resnorm = cs.resnorm;
    res->history.push_back({(int64_t)rep.cycles, rep.h_mv + rep.h_mv_aux, base_level + level, resnorm,
                            ns_since(t0)});
    if (fetch && !res->fetched) {
      const bool hit = (fetch->kind == MSTAB_FETCH_AT_CYCLE && rep.cycles == fetch->cycle) ||
                       (fetch->kind == MSTAB_FETCH_AT_HALF_TOLERANCE &&
                        resnorm <= std::sqrt(cfg.tol) * rep.bnorm);
      if (hit) {  // fetch(): deep copy (recycle.cpp:26-38)
        StallTrace tr("mstab: fetch");
        auto f = std::make_shared<Recycle>();
        f->n = n;
        f->s = s;
        f->level_j = base_level + level;
        f->fingerprint = op.fingerprint;
        f->p = P;
        f->u = copy_block(ctx, w.set[p].U, n, s);
        f->v = copy_block(ctx, w.set[p].V, n, s);
        if (omegas_complete) f->omega = omega_levels;
        res->fetched = f;
      }
    }
  }
  if (!broke) rep.status = resnorm <= threshold ? MSTAB_STATUS_CONVERGED : MSTAB_STATUS_MAXMV;
  rep.final_resnorm = resnorm;
  const WSet& cur = w.set[p];
  StallTrace tr_final("mstab: hand-off copies");
  res->x = copy_vec(ctx, cur.x, n);
  auto fin = std::make_shared<Recycle>();
  fin->n = n;
  fin->s = s;
  fin->level_j = base_level + level;
  fin->fingerprint = op.fingerprint;
  fin->p = P;
  fin->u = copy_block(ctx, cur.U, n, s);
  fin->v = copy_block(ctx, cur.V, n, s);
  if (omegas_complete) fin->omega = omega_levels;
  res->final_data = fin;
  rep.has_fetched = res->fetched ? 1 : 0;
  rep.history_len = (int64_t)res->history.size();
  rep.tau_len = (int64_t)res->taus.size();
  ctx.sync();
  rep.wall_ns_total = ns_since(t0);
  return res;
}

// ---- the reference's test-visible helpers on the device (idrstab.hpp:27-68) ---------------------
// Host blocks in, host blocks out (column-major, leading dimension n), every length-N step on the
// kernels the solve loop runs. Used by the C-ABI kernel entry points and, through them, by the
// drop-in shim's level_iteration / poly_combination / bicg_projection.
namespace {

void upload_cols(Context& ctx, double* dst, const double* src, int64_t n, int64_t cols) {
  CUDA_OK(cudaMemcpy2DAsync(dst, sizeof(double) * ctx.ld(n), src, sizeof(double) * n, sizeof(double) * n,
                            (size_t)cols, cudaMemcpyHostToDevice, ctx.stream()));
}
void download_cols(Context& ctx, double* dst, const double* src, int64_t n, int64_t cols) {
  CUDA_OK(cudaMemcpy2DAsync(dst, sizeof(double) * n, src, sizeof(double) * ctx.ld(n), sizeof(double) * n,
                            (size_t)cols, cudaMemcpyDeviceToHost, ctx.stream()));
}

// gamma = (P^H block)^-1 P^H target into ds->gamma row `slot` (the prologue kernel's reductions and
// its warp LU); throws SingularProjection like solve_small.
void project_dev(Context& ctx, int64_t n, int s, const double* P, const double* block, const double* target,
                 int slot) {
  reset_status(ctx);
  launch_prologue(ctx.stream(), n, ctx.ld(n), s, P, block, target, ctx.reducer());
  check_launch();
  after_poly(ctx, s);
  if (read_status(ctx).pending_singular) throw Error(MSTAB_E_SINGULAR, "solve_small: pivot collapse");
  if (slot != 0)
    CUDA_OK(cudaMemcpyAsync(ctx.ds()->gamma + (size_t)slot * kMaxS, ctx.ds()->gamma, sizeof(double) * s,
                            cudaMemcpyDeviceToDevice, ctx.stream()));
}

}  // namespace

void bicg_projection_host(Context& ctx, int64_t n, int s, const double* p, const double* block,
                          const double* target, double* gamma) {
  if (s < 1 || s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: 1 <= s <= 16");
  DevPtr P = ctx.alloc_vecs(n, s), B = ctx.alloc_vecs(n, s), t = ctx.alloc_vecs(n, 1);
  upload_cols(ctx, P->d(), p, n, s);
  upload_cols(ctx, B->d(), block, n, s);
  upload_cols(ctx, t->d(), target, n, 1);
  project_dev(ctx, n, s, P->d(), B->d(), t->d(), 0);
  CUDA_OK(cudaMemcpyAsync(gamma, ctx.ds()->gamma, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx.stream()));
  ctx.sync();
}

void projection_gram_host(Context& ctx, int64_t n, int s, const double* p, const double* block,
                          const double* target, double* m, double* g) {
  if (s < 1 || s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: 1 <= s <= 16");
  DevPtr P = ctx.alloc_vecs(n, s), B = ctx.alloc_vecs(n, s), t = ctx.alloc_vecs(n, 1);
  upload_cols(ctx, P->d(), p, n, s);
  upload_cols(ctx, B->d(), block, n, s);
  upload_cols(ctx, t->d(), target, n, 1);
  reset_status(ctx);
  launch_prologue(ctx.stream(), n, ctx.ld(n), s, P->d(), B->d(), t->d(), ctx.reducer());
  check_launch();
  after_poly(ctx, s);
  CUDA_OK(cudaMemcpyAsync(m, ctx.ds()->Ma, sizeof(double) * s * s, cudaMemcpyDeviceToHost, ctx.stream()));
  CUDA_OK(cudaMemcpyAsync(g, ctx.ds()->g, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx.stream()));
  ctx.sync();
}

void level_iteration_host(Context& ctx, const Operator& op, int s, int k, const double* p, double* x0,
                          double* r_levels, double* v_levels) {
  if (s < 1 || s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: 1 <= s <= 16");
  if (k < 0 || k >= kMaxEll) throw Error(MSTAB_E_CONFIG, "b200: level 0 <= k < 8");
  const int64_t n = op.n;
  DevPtr P = ctx.alloc_vecs(n, s);
  WSet D{ctx.alloc_vecs(n, 1), ctx.alloc_vecs(n, 1), ctx.alloc_vecs(n, s), ctx.alloc_vecs(n, s)};
  std::vector<DevPtr> R(k + 2), VL(k + 2);
  for (int i = 1; i <= k + 1; ++i) {
    R[i] = ctx.alloc_vecs(n, 1);
    VL[i] = ctx.alloc_vecs(n, s);
  }
  upload_cols(ctx, P->d(), p, n, s);
  upload_cols(ctx, D.x->d(), x0, n, 1);
  upload_cols(ctx, D.r->d(), r_levels, n, 1);
  for (int i = 1; i <= k; ++i) upload_cols(ctx, R[i]->d(), r_levels + (size_t)i * n, n, 1);
  upload_cols(ctx, D.U->d(), v_levels, n, s);                          // level -1
  upload_cols(ctx, D.V->d(), v_levels + (size_t)n * s, n, s);          // level 0
  for (int i = 1; i <= k; ++i) upload_cols(ctx, VL[i]->d(), v_levels + (size_t)(i + 1) * n * s, n, s);
  // gamma_k = bicg_projection(P, V^(k), r^(k)) (idrstab.cpp:112); also leaves Ma = P^H V^(k)
  project_dev(ctx, n, s, P->d(), k == 0 ? D.V->d() : VL[k]->d(), k == 0 ? D.r->d() : R[k]->d(), k);
  reset_status(ctx);
  enqueue_level(ctx, op, P->d(), s, k + 1, k, D, D, R, VL);
  check_launch();
  const CycleStatus& cs = read_status(ctx);
  if (cs.breakdown) throw Error(MSTAB_E_SINGULAR, "solve_small: pivot collapse");
  download_cols(ctx, x0, D.x->d(), n, 1);
  download_cols(ctx, r_levels, D.r->d(), n, 1);
  for (int i = 1; i <= k + 1; ++i) download_cols(ctx, r_levels + (size_t)i * n, R[i]->d(), n, 1);
  download_cols(ctx, v_levels, D.U->d(), n, s);
  download_cols(ctx, v_levels + (size_t)n * s, D.V->d(), n, s);
  for (int i = 1; i <= k + 1; ++i) download_cols(ctx, v_levels + (size_t)(i + 1) * n * s, VL[i]->d(), n, s);
  ctx.sync();
}

void poly_combination_host(Context& ctx, int64_t n, int s, int ell, const double* x0, const double* r_levels,
                           const double* v_levels, double* x, double* r, double* u, double* v, double* tau,
                           int32_t* tail_perturbed) {
  if (s < 1 || s > kMaxS || ell < 1 || ell > kMaxEll) throw Error(MSTAB_E_CONFIG, "b200: s <= 16 and ell <= 8");
  if (n < ell) throw Error(MSTAB_E_DIMENSION, "least_squares_tall: needs rows >= cols");
  // the kernels take the length from an operator-free launch: a zero-entry operator of size n
  // stands in for enqueue_poly's `op` (it only reads n and n_global)
  Operator shape;
  shape.n = n;
  shape.n_global = n;
  WSet D{ctx.alloc_vecs(n, 1), ctx.alloc_vecs(n, 1), ctx.alloc_vecs(n, s), ctx.alloc_vecs(n, s)};
  std::vector<DevPtr> R(ell + 1), VL(ell + 1);
  for (int i = 1; i <= ell; ++i) {
    R[i] = ctx.alloc_vecs(n, 1);
    VL[i] = ctx.alloc_vecs(n, s);
  }
  upload_cols(ctx, D.x->d(), x0, n, 1);
  upload_cols(ctx, D.r->d(), r_levels, n, 1);
  for (int i = 1; i <= ell; ++i) upload_cols(ctx, R[i]->d(), r_levels + (size_t)i * n, n, 1);
  upload_cols(ctx, D.U->d(), v_levels, n, s);
  upload_cols(ctx, D.V->d(), v_levels + (size_t)n * s, n, s);
  for (int i = 1; i <= ell; ++i) upload_cols(ctx, VL[i]->d(), v_levels + (size_t)(i + 1) * n * s, n, s);
  // P only feeds the next cycle's P^H r / P^H V reductions, which this helper discards
  DevPtr P = ctx.alloc_vecs(n, s);
  CUDA_OK(cudaMemsetAsync(P->ptr, 0, P->bytes, ctx.stream()));
  reset_status(ctx);
  enqueue_poly(ctx, shape, P->d(), s, ell, D, R, VL);
  const CycleStatus& cs = read_status(ctx);
  if (cs.breakdown == kBreakRank)
    throw Error(MSTAB_E_RANK, "least_squares_tall: stabilization block lost rank");
  for (int i = 0; i < ell; ++i) tau[i] = cs.tau[i];
  if (tail_perturbed) *tail_perturbed = cs.tail_perturbed;
  download_cols(ctx, x, D.x->d(), n, 1);
  download_cols(ctx, r, D.r->d(), n, 1);
  download_cols(ctx, u, D.U->d(), n, s);
  download_cols(ctx, v, D.V->d(), n, s);
  ctx.sync();
}

// sridr_solve (sridr.cpp:23-118): the recycled phase replays the donor's J relaxations with V
// fixed (one product per cycle, ksridr.cu), then standard IDR(s) cycles (ell = 1) seeded with the
// recycled block, on the same captured cycle graphs as idrstab_solve.
std::unique_ptr<SolveResultImpl> sridr(Context& ctx, const Operator& op, const double* b_in, const double* x0_in,
                                       int mem, const mstab_solver_config& cfg, const Recycle& rc) {
  if (cfg.s < 1) throw Error(MSTAB_E_CONFIG, "config: s >= 1 required");
  if (cfg.ell < 1) throw Error(MSTAB_E_CONFIG, "config: ell >= 1 required");
  if (!(cfg.tol > 0.0)) throw Error(MSTAB_E_CONFIG, "config: tol > 0 required");
  if (cfg.max_mv < cfg.s + 1) throw Error(MSTAB_E_CONFIG, "config: max_mv >= s + 1 required");
  if (cfg.ell != 1) throw Error(MSTAB_E_CONFIG, "sridr: ell == 1 required");
  if (cfg.s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: s <= 16 is supported");
  const int s = (int)cfg.s;
  const int64_t n = op.n, ld = ctx.ld(n);
  cudaStream_t st = ctx.stream();
  const bool tres = cfg.true_residual_each_cycle != 0;
  validate(ctx, rc, op);
  if (rc.s != cfg.s) throw Error(MSTAB_E_CONFIG, "sridr: recycle s != config s");
  const int64_t J = rc.level_j;
  if ((int64_t)rc.omega.size() != J)
    throw Error(MSTAB_E_MISSING_OMEGAS, "sridr: recycle data lacks the relaxation history");
  for (const auto& w : rc.omega)
    if (w.imag() != 0.0) throw Error(MSTAB_E_NOTREAL, "sridr: complex relaxation history (real fp64 path)");
  Workspace& w = workspace(ctx, op, s, 1, tres);
  reset_status(ctx);
  const auto t0 = Clock::now();
  auto res = std::make_unique<SolveResultImpl>();
  res->n = n;
  mstab_report& rep = res->report;
  std::memset(&rep, 0, sizeof(rep));
  rep.ell = 1;
  rep.h_mv_aux += s;  // validation applies A to U

  CUDA_OK(cudaMemcpyAsync(w.b->d(), b_in, sizeof(double) * n,
                          mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  launch_vec_stats(st, n, w.b->d(), scal(ctx, 0), ctx.reducer());
  check_launch();
  rep.bnorm = std::sqrt(read_scal(ctx, 3)[0]);
  WSet& c0 = w.set[0];
  bool x_zero = true;
  if (x0_in) {
    CUDA_OK(cudaMemcpyAsync(c0.x->d(), x0_in, sizeof(double) * n,
                            mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    launch_vec_stats(st, n, c0.x->d(), scal(ctx, 0), ctx.reducer());
    check_launch();
    x_zero = read_scal(ctx, 3)[2] == 0.0;
  } else {
    CUDA_OK(cudaMemsetAsync(c0.x->ptr, 0, sizeof(double) * ld, st));
  }
  CUDA_OK(cudaMemcpyAsync(c0.r->d(), w.b->d(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  if (!x_zero) {  // r = b - A x (sridr.cpp:44-48)
    spmv_dev(ctx, op, c0.x->d(), c0.r->d());
    launch_rsub(st, n, w.b->d(), c0.r->d());
    check_launch();
    rep.h_mv_aux++;
  }
  if (w.p_src != rc.p) {
    CUDA_OK(cudaMemcpyAsync(w.P->ptr, rc.p->ptr, sizeof(double) * ld * s, cudaMemcpyDeviceToDevice, st));
    w.p_src = rc.p;
  }
  const double* P = w.P->d();
  // P^H V (kept in ds->Ma for the whole recycled phase), P^H r, ||r||, gamma = (P^H V)^-1 P^H r
  reset_status(ctx);
  launch_prologue(st, n, ld, s, P, rc.v->d(), c0.r->d(), ctx.reducer());
  check_launch();
  CycleStatus cs = read_status(ctx);
  double resnorm = cs.resnorm;
  res->history.push_back({0, rep.h_mv + rep.h_mv_aux, 0, resnorm, ns_since(t0)});
  const double threshold = cfg.tol * rep.bnorm;
  int64_t j = 0;
  bool broke = false;
  auto breakdown = [&](const char* why) {
    rep.status = MSTAB_STATUS_BREAKDOWN;
    std::snprintf(rep.breakdown_reason, sizeof(rep.breakdown_reason), "%s", why);
    broke = true;
  };
  if (J > 0 && cs.pending_singular) breakdown("sridr: projection block P^H V is singular");
  // recycled phase: rt, xt in the idle ping-pong set, A rt in R[1]
  double* rt = w.set[1].r->d();
  double* xt = w.set[1].x->d();
  double* art = w.R[1]->d();
  while (!broke && j < J && resnorm > threshold && rep.h_mv < cfg.max_mv) {
    launch_sridr_corr(st, n, ld, s, c0.r->d(), c0.x->d(), rc.u->d(), rc.v->d(), rt, xt, ctx.ds());
    check_launch();
    spmv_dev(ctx, op, rt, art);
    FinParams f;
    f.op = kFinTrueRes;  // ||r||, P^H r and the next gamma from the fixed P^H V
    f.s = s;
    launch_sridr_update(st, n, ld, s, rc.omega[(size_t)j].real(), rt, art, xt, c0.r->d(), c0.x->d(), P, f,
                        ctx.reducer());
    check_launch();
    rep.h_mv++;
    ++j;
    rep.cycles = j;
    rep.h_rd = j * s;
    cs = read_status(ctx);
    resnorm = cs.resnorm;
    res->history.push_back({j, rep.h_mv + rep.h_mv_aux, j, resnorm, ns_since(t0)});
  }
  // standard IDR(s) cycles seeded with the recycled block (sridr.cpp:86-108)
  int p = 0;
  if (!broke && resnorm > threshold && rep.h_mv < cfg.max_mv) {
    CUDA_OK(cudaMemcpyAsync(c0.U->ptr, rc.u->ptr, sizeof(double) * ld * s, cudaMemcpyDeviceToDevice, st));
    CUDA_OK(cudaMemcpyAsync(c0.V->ptr, rc.v->ptr, sizeof(double) * ld * s, cudaMemcpyDeviceToDevice, st));
    reset_status(ctx);
    launch_prologue(st, n, ld, s, P, c0.V->d(), c0.r->d(), ctx.reducer());
    check_launch();
    read_status(ctx);
    while (resnorm > threshold && rep.h_mv < cfg.max_mv) {
      const CycleStatus& ccs = run_cycle_sync(ctx, op, w, p);
      if (w.graph[p].profiled) prof_accumulate(w.graph[p].prof);
      if (ccs.breakdown) {
        rep.h_mv += ccs.mv_at_breakdown;
        breakdown(ccs.breakdown == kBreakRank ? "least_squares_tall: stabilization block lost rank"
                                              : "solve_small: pivot collapse");
        break;
      }
      p = 1 - p;
      ++j;
      rep.cycles = j;
      rep.h_mv += s + 1;
      rep.h_rd = j * s;
      res->taus.push_back(ccs.tau[0]);
      if (tres) rep.h_mv_aux++;
      resnorm = ccs.resnorm;
      res->history.push_back({j, rep.h_mv + rep.h_mv_aux, j, resnorm, ns_since(t0)});
    }
  }
  if (!broke) rep.status = resnorm <= threshold ? MSTAB_STATUS_CONVERGED : MSTAB_STATUS_MAXMV;
  rep.final_resnorm = resnorm;
  res->x = copy_vec(ctx, w.set[p].x, n);
  rep.history_len = (int64_t)res->history.size();
  rep.tau_len = (int64_t)res->taus.size();
  ctx.sync();
  rep.wall_ns_total = ns_since(t0);
  return res;
}

// ---- comparison baselines (baselines.cpp:49-262) ---------------------------
// BiCGStab and full-memory GMRES (MGS) on the device: every length-N step is a kernel (SpMV,
// dots, updates); the scalar recurrences (alpha, omega, beta, the Givens rotations and the
// Hessenberg back-substitution) run on the host in std::complex<double> exactly as the reference
// writes them, so for real data every element-wise update rounds like the reference's and only the
// length-N reductions differ (tree sums).
namespace {

struct BaselineStart {
  std::unique_ptr<SolveResultImpl> res;
  DevPtr b, x, r;
  Clock::time_point t0;
};

BaselineStart baseline_start(Context& ctx, const Operator& op, const double* b_in, const double* x0_in, int mem) {
  BaselineStart st0;
  const int64_t n = op.n;
  cudaStream_t st = ctx.stream();
  reset_status(ctx);
  st0.t0 = Clock::now();
  st0.res = std::make_unique<SolveResultImpl>();
  st0.res->n = n;
  std::memset(&st0.res->report, 0, sizeof(mstab_report));
  st0.res->report.ell = 1;
  const cudaMemcpyKind kind = mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  st0.b = ctx.alloc_vecs(n, 1);
  st0.x = ctx.alloc_vecs(n, 1);
  st0.r = ctx.alloc_vecs(n, 1);
  CUDA_OK(cudaMemcpyAsync(st0.b->d(), b_in, sizeof(double) * n, kind, st));
  launch_vec_stats(st, n, st0.b->d(), scal(ctx, 0), ctx.reducer());
  check_launch();
  st0.res->report.bnorm = std::sqrt(read_scal(ctx, 3)[0]);
  bool x_zero = true;
  if (x0_in) {
    CUDA_OK(cudaMemcpyAsync(st0.x->d(), x0_in, sizeof(double) * n, kind, st));
    launch_vec_stats(st, n, st0.x->d(), scal(ctx, 0), ctx.reducer());
    check_launch();
    x_zero = read_scal(ctx, 3)[2] == 0.0;
  } else {
    CUDA_OK(cudaMemsetAsync(st0.x->ptr, 0, sizeof(double) * ctx.ld(n), st));
  }
  CUDA_OK(cudaMemcpyAsync(st0.r->d(), st0.b->d(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  if (!x_zero) {  // initial_residual (baselines.cpp:22-32)
    spmv_dev(ctx, op, st0.x->d(), st0.r->d());
    launch_rsub(st, n, st0.b->d(), st0.r->d());
    check_launch();
    st0.res->report.h_mv_aux++;
  }
  return st0;
}

// dst[0] = dot(a, y) (when a), dst[last] = ||y||^2; returns the host copy of the first `count` scal.
const double* dots_host(Context& ctx, int64_t n, const double* a, const double* y) {
  launch_dots(ctx.stream(), n, ctx.ld(n), a, a ? 1 : 0, y, true, scal(ctx, 0), ctx.reducer());
  check_launch();
  return read_scal(ctx, a ? 2 : 1);
}

void baseline_finish(Context& ctx, BaselineStart& s0, int64_t it, double resnorm, double threshold, bool broke) {
  mstab_report& rep = s0.res->report;
  rep.cycles = it;
  rep.h_rd = it;
  if (!broke) rep.status = resnorm <= threshold ? MSTAB_STATUS_CONVERGED : MSTAB_STATUS_MAXMV;
  rep.final_resnorm = resnorm;
  s0.res->x = s0.x;
  rep.history_len = (int64_t)s0.res->history.size();
  ctx.sync();
  rep.wall_ns_total = ns_since(s0.t0);
}

}  // namespace

// A^H of a plain CSR operator as a second operator (real data: A^T). spmv_adjoint scatters
// y[col] += conj(a_ik) x_i over rows i ascending and entries k in CSR order (csr.cpp:115-124), so
// y_j is the sum, from +0.0, of its terms in (i, k) order. The transpose built here lists row j's
// entries in exactly that order (a stable bucket pass over the original entries), and every SpMV
// kernel accumulates a row from +0.0 in CSR order: the device product is bit-identical to the
// reference's scatter. The transpose goes through the normal upload, so a stencil's transpose gets
// the same constant-diagonal / DIA forms. Built once per operator, on first use.
namespace {

struct HostCsr {
  std::vector<int64_t> rp, ci;
  std::vector<double> val;
};

HostCsr download_csr(Context& ctx, int64_t n, int64_t nnz, const void* rp_d, const void* ci_d, const double* val_d) {
  std::vector<int32_t> rp(n + 1), ci(std::max<int64_t>(nnz, 1));
  HostCsr h;
  h.val.resize(std::max<int64_t>(nnz, 1));
  cudaStream_t st = ctx.stream();
  CUDA_OK(cudaMemcpyAsync(rp.data(), rp_d, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
  if (nnz > 0) {
    CUDA_OK(cudaMemcpyAsync(ci.data(), ci_d, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(h.val.data(), val_d, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st));
  }
  ctx.sync();
  h.rp.assign(rp.begin(), rp.end());
  h.ci.assign(ci.begin(), ci.begin() + std::max<int64_t>(nnz, 0));
  return h;
}

// Transpose (real data: the conjugate transpose) with row j listing its entries in the order the
// reference's scatter loops add them into x[j]: source rows ascending, or descending when
// `descending` (lower_solve_adjoint walks L's rows back to front, precond.cpp:129-143).
HostCsr transpose(int64_t n, const HostCsr& a, bool descending) {
  const int64_t nnz = a.rp[n];
  HostCsr t;
  t.rp.assign(n + 1, 0);
  t.ci.resize(std::max<int64_t>(nnz, 1));
  t.val.resize(std::max<int64_t>(nnz, 1));
  for (int64_t k = 0; k < nnz; ++k) ++t.rp[a.ci[k] + 1];
  for (int64_t j = 0; j < n; ++j) t.rp[j + 1] += t.rp[j];
  std::vector<int64_t> fill(t.rp.begin(), t.rp.end() - 1);
  for (int64_t s = 0; s < n; ++s) {
    const int64_t i = descending ? n - 1 - s : s;
    for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) {
      const int64_t at = fill[a.ci[k]]++;
      t.ci[at] = i;
      t.val[at] = a.val[k];
    }
  }
  return t;
}

}  // namespace

// A^H of an operator as a second operator (real data: A^T), built once on first use.
// CSR: spmv_adjoint scatters y[col] += conj(a_ik) x_i over rows i ascending and entries k in CSR
// order (csr.cpp:115-124), so y_j is the sum, from +0.0, of its terms in (i, k) order; the
// transpose lists row j's entries in exactly that order and every SpMV kernel accumulates a row
// from +0.0 in CSR order: bit-identical to the reference's scatter. The transpose goes through
// the normal upload, so a stencil's transpose gets the same constant-diagonal / DIA forms.
// Preconditioned (precond.cpp:190-200): (L^-1 A R^-1)^H = R^-H A^H L^-H. lower_solve_adjoint is
// x_j = (b_j - sum over rows i > j, descending, of l_ij x_i) / l_jj and upper_solve_adjoint the
// same over rows i < j ascending: exactly upper_solve / lower_solve on the transposed factors with
// those entry orders, so the adjoint chain reuses the triangular-solve kernels (the upper solve
// first, like the forward chain) and stays bit-identical. Diagonal factors are their own adjoint.
const Operator& adjoint_of(Context& ctx, const Operator& op) {
  std::lock_guard<std::mutex> lk(op.adj_mu);
  if (op.adj) return *op.adj;
  if (op.n_global != op.n) throw Error(MSTAB_E_CONFIG, "b200: apply_adjoint of a row slab is not supported");
  const int64_t n = op.n;
  const HostCsr a = download_csr(ctx, n, op.nnz, op.rp->ptr, op.ci->ptr, op.val->d());
  const HostCsr at = transpose(n, a, false);
  auto adj = make_operator(ctx, n, at.rp.data(), at.ci.data(), at.val.data());
  if (op.pc) {
    const Precond& pc = *op.pc;
    auto apc = std::make_shared<Precond>();
    apc->kind = pc.kind;
    auto factor_t = [&](const DevTri& f, bool desc, bool lower, DevPtr& d_rp, DevPtr& d_ci, DevPtr& d_val,
                        DevPtr& d_diag, DevPtr& d_ord) -> DevTri {
      if (f.diag) return f;  // diagonal: its own adjoint (the device memory stays owned by `op`)
      const HostCsr h = download_csr(ctx, n, f.nnz, f.rp, f.ci, f.val);
      const HostCsr t = transpose(n, h, desc);
      return upload_factor(ctx, n, t.rp.data(), t.ci.data(), t.val.data(), lower, d_rp, d_ci, d_val, d_diag, d_ord);
    };
    // the chain solves with R first (upper), then L (lower): R slot <- L^T, L slot <- R^T
    apc->R = factor_t(pc.L, true, false, apc->r_rp, apc->r_ci, apc->r_val, apc->r_diag, apc->r_ord);
    apc->L = factor_t(pc.R, false, true, apc->l_rp, apc->l_ci, apc->l_val, apc->l_diag, apc->l_ord);
    apc->t1 = ctx.alloc_vecs(n, 1);
    apc->t2 = ctx.alloc_vecs(n, 1);
    apc->t3 = ctx.alloc_vecs(n, 1);
    apc->sync = ctx.alloc(sizeof(int) * (size_t)(n + 1));
    adj->pc = apc;
  }
  op.adj = adj;
  return *op.adj;
}

std::unique_ptr<SolveResultImpl> bicg(Context& ctx, const Operator& op, const double* b_in, const double* x0_in,
                                      int mem, double tol, int64_t max_mv, const double* shadow) {
  using C = std::complex<double>;
  const int64_t n = op.n;
  cudaStream_t st = ctx.stream();
  const Operator& adj = adjoint_of(ctx, op);
  BaselineStart s0 = baseline_start(ctx, op, b_in, x0_in, mem);
  mstab_report& rep = s0.res->report;
  auto& hist = s0.res->history;
  double* x = s0.x->d();
  double* r = s0.r->d();
  double resnorm = std::sqrt(dots_host(ctx, n, nullptr, r)[0]);
  hist.push_back({0, rep.h_mv + rep.h_mv_aux, 0, resnorm, ns_since(s0.t0)});
  const double threshold = tol * rep.bnorm;
  DevPtr rs = ctx.alloc_vecs(n, 1), p = ctx.alloc_vecs(n, 1), ps = ctx.alloc_vecs(n, 1), ap = ctx.alloc_vecs(n, 1),
         aps = ctx.alloc_vecs(n, 1);
  CUDA_OK(cudaMemcpyAsync(rs->d(), shadow ? shadow : r, sizeof(double) * n,
                          shadow && mem != MSTAB_MEM_DEVICE ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
  CUDA_OK(cudaMemcpyAsync(p->d(), r, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  CUDA_OK(cudaMemcpyAsync(ps->d(), rs->d(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  C rho = dots_host(ctx, n, rs->d(), r)[0];
  int64_t it = 0;
  bool broke = false;
  auto breakdown = [&](const char* why) {
    rep.status = MSTAB_STATUS_BREAKDOWN;
    std::snprintf(rep.breakdown_reason, sizeof(rep.breakdown_reason), "%s", why);
    broke = true;
  };
  while (resnorm > threshold && rep.h_mv < max_mv) {  // baselines.cpp:166-186
    if (std::abs(rho) == 0.0) { breakdown("bicg: rho collapsed"); break; }
    spmv_dev(ctx, op, p->d(), ap->d());
    spmv_dev(ctx, adj, ps->d(), aps->d());
    rep.h_mv += 2;
    const C sigma = dots_host(ctx, n, ps->d(), ap->d())[0];
    if (std::abs(sigma) == 0.0) { breakdown("bicg: sigma collapsed"); break; }
    const C alpha = rho / sigma;
    launch_xpay(st, n, x, p->d(), alpha.real(), x);                       // axpy(alpha, p, x)
    launch_xpay(st, n, r, ap->d(), (-alpha).real(), r);                  // axpy(-alpha, ap, r)
    launch_xpay(st, n, rs->d(), aps->d(), (-std::conj(alpha)).real(), rs->d());  // axpy(-conj(alpha), aps, rs)
    const C rho_next = dots_host(ctx, n, rs->d(), r)[0];
    const C beta = rho_next / rho;
    rho = rho_next;
    launch_xpay(st, n, r, p->d(), beta.real(), p->d());                  // p = r + beta p
    launch_xpay(st, n, rs->d(), ps->d(), std::conj(beta).real(), ps->d());  // ps = rs + conj(beta) ps
    check_launch();
    ++it;
    resnorm = std::sqrt(dots_host(ctx, n, nullptr, r)[0]);
    hist.push_back({it, rep.h_mv + rep.h_mv_aux, it, resnorm, ns_since(s0.t0)});
  }
  baseline_finish(ctx, s0, it, resnorm, threshold, broke);
  return std::move(s0.res);
}

std::unique_ptr<SolveResultImpl> bicgstab(Context& ctx, const Operator& op, const double* b_in, const double* x0_in,
                                          int mem, double tol, int64_t max_mv, const double* shadow) {
  using C = std::complex<double>;
  const int64_t n = op.n;
  cudaStream_t st = ctx.stream();
  BaselineStart s0 = baseline_start(ctx, op, b_in, x0_in, mem);
  mstab_report& rep = s0.res->report;
  auto& hist = s0.res->history;
  double* x = s0.x->d();
  double* r = s0.r->d();
  double resnorm = std::sqrt(dots_host(ctx, n, nullptr, r)[0]);
  hist.push_back({0, rep.h_mv + rep.h_mv_aux, 0, resnorm, ns_since(s0.t0)});
  const double threshold = tol * rep.bnorm;
  DevPtr rs = ctx.alloc_vecs(n, 1), p = ctx.alloc_vecs(n, 1), sv = ctx.alloc_vecs(n, 1), ap = ctx.alloc_vecs(n, 1),
         as = ctx.alloc_vecs(n, 1);
  CUDA_OK(cudaMemcpyAsync(rs->d(), shadow ? shadow : r, sizeof(double) * n,
                          shadow && mem != MSTAB_MEM_DEVICE ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
  CUDA_OK(cudaMemcpyAsync(p->d(), r, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  C rho = dots_host(ctx, n, rs->d(), r)[0];
  int64_t it = 0;
  bool broke = false;
  auto breakdown = [&](const char* why) {
    rep.status = MSTAB_STATUS_BREAKDOWN;
    std::snprintf(rep.breakdown_reason, sizeof(rep.breakdown_reason), "%s", why);
    broke = true;
  };
  while (resnorm > threshold && rep.h_mv < max_mv) {  // baselines.cpp:219-254
    if (std::abs(rho) == 0.0) { breakdown("bicgstab: rho collapsed"); break; }
    spmv_dev(ctx, op, p->d(), ap->d());
    rep.h_mv++;
    const C denom = dots_host(ctx, n, rs->d(), ap->d())[0];
    if (std::abs(denom) == 0.0) { breakdown("bicgstab: shadow projection collapsed"); break; }
    const C alpha = rho / denom;
    launch_xpay(st, n, r, ap->d(), -alpha.real(), sv->d());
    if (std::sqrt(dots_host(ctx, n, nullptr, sv->d())[0]) <= threshold) {  // converged after the BiCG half-step
      launch_xpay(st, n, x, p->d(), alpha.real(), x);
      CUDA_OK(cudaMemcpyAsync(r, sv->d(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      ++it;
      resnorm = std::sqrt(dots_host(ctx, n, nullptr, r)[0]);
      hist.push_back({it, rep.h_mv + rep.h_mv_aux, it, resnorm, ns_since(s0.t0)});
      break;
    }
    spmv_dev(ctx, op, sv->d(), as->d());
    rep.h_mv++;
    const double* h = dots_host(ctx, n, sv->d(), as->d());  // dot(s, as), ||as||^2
    const C sdot = h[0];
    const double nas = std::sqrt(h[1]);
    const double as2 = std::pow(nas, 2);
    if (as2 == 0.0) { breakdown("bicgstab: stagnated update"); break; }
    const C omega = sdot / as2;
    launch_xpay(st, n, x, p->d(), alpha.real(), x);
    launch_xpay(st, n, x, sv->d(), omega.real(), x);
    launch_xpay(st, n, sv->d(), as->d(), -omega.real(), r);
    const C rho_next = dots_host(ctx, n, rs->d(), r)[0];
    const C beta = (rho_next / rho) * (alpha / omega);
    rho = rho_next;
    launch_bicgstab_p(st, n, r, ap->d(), beta.real(), omega.real(), p->d());
    check_launch();
    ++it;
    resnorm = std::sqrt(dots_host(ctx, n, nullptr, r)[0]);
    hist.push_back({it, rep.h_mv + rep.h_mv_aux, it, resnorm, ns_since(s0.t0)});
  }
  baseline_finish(ctx, s0, it, resnorm, threshold, broke);
  return std::move(s0.res);
}

std::unique_ptr<SolveResultImpl> gmres(Context& ctx, const Operator& op, const double* b_in, const double* x0_in,
                                       int mem, double tol, int64_t max_it) {
  using C = std::complex<double>;
  const int64_t n = op.n, ld = ctx.ld(n);
  cudaStream_t st = ctx.stream();
  BaselineStart s0 = baseline_start(ctx, op, b_in, x0_in, mem);
  mstab_report& rep = s0.res->report;
  auto& hist = s0.res->history;
  double* x = s0.x->d();
  double* r = s0.r->d();
  const double r2 = dots_host(ctx, n, nullptr, r)[0];
  const double r0norm = std::sqrt(r2);
  hist.push_back({0, rep.h_mv + rep.h_mv_aux, 0, r0norm, ns_since(s0.t0)});
  const double threshold = tol * rep.bnorm;
  if (r0norm <= threshold || max_it == 0) {  // baselines.cpp:63-68
    baseline_finish(ctx, s0, 0, r0norm, threshold, false);
    s0.res->report.h_rd = 0;
    return std::move(s0.res);
  }
  const int64_t m_cap = std::min<int64_t>(max_it, n);
  std::vector<DevPtr> q;  // basis columns, allocated as the iteration needs them
  q.push_back(ctx.alloc_vecs(n, 1));
  DevPtr hbuf = ctx.alloc(sizeof(double) * (size_t)(m_cap + 2));
  double* hd = hbuf->d();
  CUDA_OK(cudaMemcpyAsync(hd, &r2, sizeof(double), cudaMemcpyHostToDevice, st));
  launch_div_by_sqrt(st, n, r, hd, q[0]->d());  // q0 = r / ||r||
  std::vector<std::vector<C>> hess;              // column-major: hess[it][i]
  std::vector<double> cs;
  std::vector<C> sn, g(1, C(r0norm));
  std::vector<double> hcol;
  double resnorm = r0norm;
  int64_t it = 0;
  DevPtr w = ctx.alloc_vecs(n, 1);
  while (it < m_cap && resnorm > threshold) {  // baselines.cpp:86-132
    spmv_dev(ctx, op, q[it]->d(), w->d());
    rep.h_mv++;
    for (int64_t i = 0; i <= it; ++i) {  // modified Gram-Schmidt: h(i,it) = <q_i, w>; w -= h q_i
      launch_dots(st, n, ld, q[i]->d(), 1, w->d(), false, hd + i, ctx.reducer());
      launch_axpy_neg(st, n, ld, q[i]->d(), 1, hd + i, w->d());
    }
    launch_dots(st, n, ld, nullptr, 0, w->d(), true, hd + it + 1, ctx.reducer());
    check_launch();
    hcol.resize((size_t)it + 2);
    CUDA_OK(cudaMemcpyAsync(hcol.data(), hd, sizeof(double) * (size_t)(it + 2), cudaMemcpyDeviceToHost, st));
    ctx.sync();
    const double hnext = std::sqrt(hcol[(size_t)it + 1]);
    if (hnext > 0.0) {
      q.push_back(ctx.alloc_vecs(n, 1));
      launch_div_by_sqrt(st, n, w->d(), hd + it + 1, q[(size_t)it + 1]->d());  // q_{it+1} = w / ||w||
      check_launch();
    }
    std::vector<C> col((size_t)it + 2);
    for (int64_t i = 0; i <= it; ++i) col[(size_t)i] = C(hcol[(size_t)i]);
    col[(size_t)it + 1] = C(hnext);
    for (int64_t i = 0; i < it; ++i) {  // previous rotations, then the new one
      const C t1 = col[(size_t)i], t2 = col[(size_t)i + 1];
      col[(size_t)i] = cs[(size_t)i] * t1 + std::conj(sn[(size_t)i]) * t2;
      col[(size_t)i + 1] = -sn[(size_t)i] * t1 + cs[(size_t)i] * t2;
    }
    const C h1 = col[(size_t)it], h2 = col[(size_t)it + 1];
    const double denom = std::sqrt(std::norm(h1) + std::norm(h2));
    if (denom == 0.0) {
      cs.push_back(1.0);
      sn.push_back(0.0);
    } else {
      cs.push_back(std::abs(h1) / denom);
      const C phase = h1 == C(0.0) ? C(1.0) : h1 / std::abs(h1);
      sn.push_back(h2 * std::conj(phase) / denom);
      col[(size_t)it] = phase * denom;
      col[(size_t)it + 1] = 0.0;
    }
    hess.push_back(col);
    const C g1 = g[(size_t)it];
    g[(size_t)it] = cs[(size_t)it] * g1;
    g.push_back(-sn[(size_t)it] * g1);
    resnorm = std::abs(g[(size_t)it + 1]);
    ++it;
    hist.push_back({it, rep.h_mv + rep.h_mv_aux, it, resnorm, ns_since(s0.t0)});
    if (hnext == 0.0) break;  // lucky breakdown
  }
  std::vector<C> y((size_t)it);
  for (int64_t k = it; k-- > 0;) {
    C acc = g[(size_t)k];
    for (int64_t j = k + 1; j < it; ++j) acc -= hess[(size_t)j][(size_t)k] * y[(size_t)j];
    y[(size_t)k] = acc / hess[(size_t)k][(size_t)k];
  }
  for (int64_t k = 0; k < it; ++k) {
    if (y[(size_t)k].imag() != 0.0) throw Error(MSTAB_E_NOTREAL, "gmres: complex coefficients (real fp64 path)");
    launch_xpay(st, n, x, q[(size_t)k]->d(), y[(size_t)k].real(), x);  // axpy(y_k, q_k, x)
  }
  check_launch();
  baseline_finish(ctx, s0, it, resnorm, threshold, false);
  return std::move(s0.res);
}

}  // namespace mstab_b200
