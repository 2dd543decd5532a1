// capi.cpp — extern "C" entry points of include/mstab_b200.h over solver.cpp.
// Exceptions never cross the boundary: each call returns the MSTAB_E_* code of the reference
// exception class (errors.hpp) and leaves the message in mstab_last_error().
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "solver.h"

#include <cstdio>
#include <cstdlib>

using namespace mstab_b200;

struct mstab_context {
  std::unique_ptr<Context> impl;
};
// A handle holds either the real object (impl) or, for complex128 data, the
// complex one (z); the *_z entry points create and consume the latter.
struct mstab_operator {
  std::shared_ptr<Operator> impl;
  std::shared_ptr<ZOperator> z;
};
struct mstab_recycle {
  RecyclePtr impl;
  std::shared_ptr<const ZRecycle> z;
};
struct mstab_result {
  std::unique_ptr<SolveResultImpl> impl;
  std::unique_ptr<ZResult> z;
};

namespace {

thread_local std::string g_last_error;
thread_local int64_t g_last_row = -1;

#ifndef MSTAB_GIT_SHA
#define MSTAB_GIT_SHA "unknown"
#endif
#ifndef MSTAB_BUILD_FLAGS
#define MSTAB_BUILD_FLAGS ""
#endif

template <typename F>
int guarded(F&& f) {
  g_last_row = -1;
  try {
    f();
    return MSTAB_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    g_last_row = e.row;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    g_last_row = -1;
    return MSTAB_E_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    g_last_row = -1;
    return MSTAB_E_ERROR;
  }
}

void bind(mstab_context* ctx) {
  if (!ctx || !ctx->impl) throw Error(MSTAB_E_CONFIG, "null context");
  cudaSetDevice(ctx->impl->device);
}

// the real fp64 entry points reject complex handles (use the *_z entry points)
const Operator& real_of(const mstab_operator* op) {
  if (!op || !op->impl) throw Error(MSTAB_E_NOTREAL, "complex operator: use the *_z entry points");
  return *op->impl;
}
const Recycle* real_of(const mstab_recycle* rd) {
  if (!rd) return nullptr;
  if (!rd->impl) throw Error(MSTAB_E_NOTREAL, "complex recycle data: use the *_z entry points");
  return rd->impl.get();
}
const ZOperator& complex_of(const mstab_operator* op) {
  if (!op || !op->z) throw Error(MSTAB_E_CONFIG, "real operator: create it with mstab_operator_create_csr_z");
  return *op->z;
}

}  // namespace

extern "C" {

const char* mstab_last_error(void) { return g_last_error.c_str(); }
int64_t mstab_last_error_row(void) { return g_last_row; }
const char* mstab_impl_name(void) { return "b200"; }
const char* mstab_build_id(void) { return "b200 " MSTAB_GIT_SHA " " MSTAB_BUILD_FLAGS; }

int mstab_context_create(int32_t device, mstab_context** out) {
  return guarded([&] {
    auto c = std::make_unique<mstab_context>();
    c->impl = std::make_unique<Context>(device);
    *out = c.release();
  });
}

void mstab_context_destroy(mstab_context* ctx) { delete ctx; }

int mstab_context_synchronize(mstab_context* ctx) {
  return guarded([&] {
    bind(ctx);
    ctx->impl->sync();
  });
}

int mstab_context_trim(mstab_context* ctx) {
  return guarded([&] {
    bind(ctx);
    ctx->impl->trim();
  });
}

void* mstab_context_stream(mstab_context* ctx) {
  return ctx && ctx->impl ? static_cast<void*>(ctx->impl->stream()) : nullptr;
}

int mstab_operator_create_csr(mstab_context* ctx, int64_t n, const int64_t* row_ptr,
                              const int64_t* col_idx, const double* values, mstab_operator** out) {
  return guarded([&] {
    bind(ctx);
    auto o = std::make_unique<mstab_operator>();
    o->impl = make_operator(*ctx->impl, n, row_ptr, col_idx, values);
    *out = o.release();
  });
}

int mstab_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] { nccl_unique_id(out); });
}

int mstab_context_set_comm_nccl(mstab_context* ctx, int32_t rank, int32_t world, const uint8_t id[128]) {
  return guarded([&] {
    bind(ctx);
    if (world < 1 || rank < 0 || rank >= world) throw Error(MSTAB_E_CONFIG, "comm: bad rank/world");
    ctx->impl->sync();
    ctx->impl->comm = make_nccl_comm(rank, world, id, ctx->impl->device);
  });
}

int mstab_context_set_comm_host(mstab_context* ctx, int32_t rank, int32_t world, const mstab_host_comm* fns) {
  return guarded([&] {
    bind(ctx);
    if (world < 1 || rank < 0 || rank >= world || !fns) throw Error(MSTAB_E_CONFIG, "comm: bad rank/world");
    ctx->impl->sync();
    ctx->impl->comm = make_host_comm(rank, world, *fns);
  });
}

int mstab_context_comm_info(mstab_context* ctx, int32_t* rank, int32_t* world) {
  return guarded([&] {
    const Context& c = *ctx->impl;
    if (rank) *rank = c.comm ? c.comm->rank() : 0;
    if (world) *world = c.comm ? c.comm->world() : 1;
  });
}

int mstab_operator_create_csr_slab(mstab_context* ctx, int64_t n, const int64_t* row_ptr,
                                   const int64_t* col_idx, const double* values,
                                   const int64_t* slab_starts, mstab_operator** out) {
  return guarded([&] {
    bind(ctx);
    auto o = std::make_unique<mstab_operator>();
    o->impl = make_operator_slab(*ctx->impl, n, row_ptr, col_idx, values, slab_starts);
    *out = o.release();
  });
}

int mstab_operator_create_csr_slab_local(mstab_context* ctx, int64_t n_global, const int64_t* slab_starts,
                                         const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                                         const int64_t* col_spans, uint64_t fingerprint, mstab_operator** out) {
  return guarded([&] {
    bind(ctx);
    auto o = std::make_unique<mstab_operator>();
    o->impl = make_operator_slab_local(*ctx->impl, n_global, slab_starts, row_ptr, col_idx, values, col_spans,
                                       fingerprint);
    *out = o.release();
  });
}

uint64_t mstab_fnv_begin(int64_t n_rows, int64_t n_cols, int64_t nnz) { return fnv_begin(n_rows, n_cols, nnz); }
uint64_t mstab_fnv_fold_index(uint64_t h, const int64_t* v, int64_t count, int64_t add) {
  return fnv_fold_u64(h, v, count, add);
}
uint64_t mstab_fnv_fold_values(uint64_t h, const double* values, int64_t count) {
  return fnv_fold_values(h, values, count);
}

int64_t mstab_operator_row_begin(const mstab_operator* op) { return op->impl->row0; }
int64_t mstab_operator_global_size(const mstab_operator* op) { return op->impl->n_global; }
void mstab_operator_interior_rows(const mstab_operator* op, int64_t* lo, int64_t* hi) {
  if (lo) *lo = op && op->impl ? op->impl->int_lo : 0;
  if (hi) *hi = op && op->impl ? op->impl->int_hi : 0;
}

void mstab_operator_destroy(mstab_operator* op) { delete op; }
int64_t mstab_operator_size(const mstab_operator* op) { return op->z ? op->z->n : op->impl->n; }
int64_t mstab_operator_nnz(const mstab_operator* op) { return op->z ? op->z->nnz : op->impl->nnz; }
uint64_t mstab_operator_fingerprint(const mstab_operator* op) {
  return op->z ? op->z->fingerprint : op->impl->fingerprint;
}

namespace {

// y = A x (adjoint: A^H x) with caller buffers in `mem`.
void apply_mem(mstab_context* ctx, const mstab_operator* op, const double* x, double* y, int32_t mem, bool adjoint) {
    bind(ctx);
    Context& c = *ctx->impl;
    const Operator& a = adjoint ? adjoint_of(c, real_of(op)) : real_of(op);
    const int64_t n = a.n;
    // The SpMV kernels move row pairs with 16-byte accesses: caller buffers are used in place
    // only when 16-byte aligned and of even length, otherwise staged through padded buffers.
    const bool direct = !c.sharded() && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15u) == 0 &&
                        (n % 2) == 0;
    if (mem == MSTAB_MEM_DEVICE && direct) {
      spmv(c, a, x, y);
      c.sync();
      return;
    }
    const cudaMemcpyKind in = mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const cudaMemcpyKind out = mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    DevPtr dx = c.alloc_vecs(n, 1), dy = c.alloc_vecs(n, 1);
    if (cudaMemcpyAsync(dx->d(), x, sizeof(double) * n, in, c.stream()) != cudaSuccess)
      throw Error(MSTAB_E_CUDA, "upload x");
    spmv(c, a, dx->d(), dy->d());
    if (cudaMemcpyAsync(y, dy->d(), sizeof(double) * n, out, c.stream()) != cudaSuccess)
      throw Error(MSTAB_E_CUDA, "download y");
    c.sync();
}

}  // namespace

int mstab_operator_apply(mstab_context* ctx, const mstab_operator* op, const double* x, double* y,
                         int32_t mem) {
  return guarded([&] { apply_mem(ctx, op, x, y, mem, false); });
}

int mstab_operator_apply_adjoint(mstab_context* ctx, const mstab_operator* op, const double* x, double* y,
                                 int32_t mem) {
  return guarded([&] { apply_mem(ctx, op, x, y, mem, true); });
}

int mstab_precond_build(int32_t kind, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                        const double* values, int64_t* l_row_ptr, int64_t* l_col_idx, double* l_values,
                        int64_t* l_nnz, int64_t* r_row_ptr, int64_t* r_col_idx, double* r_values,
                        int64_t* r_nnz) {
  return guarded([&] {
    precond_build(kind, n, row_ptr, col_idx, values, l_row_ptr, l_col_idx, l_values, r_row_ptr, r_col_idx,
                  r_values);
    *l_nnz = l_row_ptr[n];
    *r_nnz = r_row_ptr[n];
  });
}

int mstab_operator_create_precond(mstab_context* ctx, int64_t n, const int64_t* row_ptr,
                                  const int64_t* col_idx, const double* values, int32_t kind,
                                  const int64_t* l_row_ptr, const int64_t* l_col_idx, const double* l_values,
                                  const int64_t* r_row_ptr, const int64_t* r_col_idx, const double* r_values,
                                  mstab_operator** out) {
  return guarded([&] {
    bind(ctx);
    auto o = std::make_unique<mstab_operator>();
    o->impl = make_operator_precond(*ctx->impl, n, row_ptr, col_idx, values, kind, l_row_ptr, l_col_idx, l_values,
                                    r_row_ptr, r_col_idx, r_values);
    *out = o.release();
  });
}

int32_t mstab_operator_precond_kind(const mstab_operator* op) {
  return op && op->impl && op->impl->pc ? op->impl->pc->kind : MSTAB_PRECOND_NONE;
}

int mstab_precond_solve(mstab_context* ctx, const mstab_operator* op, int32_t which, const double* x, double* y,
                        int32_t mem) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    const int64_t n = real_of(op).n;
    if (which != 0 && which != 1) throw Error(MSTAB_E_CONFIG, "precond_solve: which must be 0 (L) or 1 (R)");
    const cudaMemcpyKind in = mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const cudaMemcpyKind out = mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    DevPtr dx = c.alloc_vecs(n, 1), dy = c.alloc_vecs(n, 1);
    if (cudaMemcpyAsync(dx->d(), x, sizeof(double) * n, in, c.stream()) != cudaSuccess)
      throw Error(MSTAB_E_CUDA, "upload x");
    precond_solve(c, *op->impl, which, dx->d(), dy->d());
    if (cudaMemcpyAsync(y, dy->d(), sizeof(double) * n, out, c.stream()) != cudaSuccess)
      throw Error(MSTAB_E_CUDA, "download y");
    c.sync();
  });
}

int mstab_recycle_create(mstab_context* ctx, int64_t n, int64_t s, const double* p, const double* u,
                         const double* v, int32_t mem, const double* omega_re_im,
                         int64_t omega_count, int64_t level_j, uint64_t fingerprint,
                         mstab_recycle** out) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    if (n < 1 || s < 1) throw Error(MSTAB_E_DIMENSION, "recycle data has inconsistent shapes");
    auto r = std::make_shared<Recycle>();
    r->n = n;
    r->s = s;
    r->level_j = level_j;
    r->fingerprint = fingerprint;
    const int64_t ld = c.ld(n);
    const auto kind = mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    auto up = [&](const double* src) {
      DevPtr d = c.alloc_vecs(n, s);
      if (cudaMemcpy2DAsync(d->d(), sizeof(double) * ld, src, sizeof(double) * n, sizeof(double) * n, s,
                            kind, c.stream()) != cudaSuccess)
        throw Error(MSTAB_E_CUDA, "recycle upload");
      return d;
    };
    r->p = up(p);
    r->u = up(u);
    r->v = up(v);
    for (int64_t i = 0; i < omega_count; ++i)
      r->omega.emplace_back(omega_re_im[2 * i], omega_re_im[2 * i + 1]);
    c.sync();
    auto h = std::make_unique<mstab_recycle>();
    h->impl = r;
    *out = h.release();
  });
}

void mstab_recycle_destroy(mstab_recycle* rd) { delete rd; }

int mstab_recycle_info_get(const mstab_recycle* rd, mstab_recycle_info* out) {
  return guarded([&] {
    if (rd->z) {
      out->n = rd->z->n;
      out->s = rd->z->s;
      out->level_j = rd->z->level_j;
      out->omega_count = (int64_t)rd->z->omega.size();
      out->fingerprint = rd->z->fingerprint;
      return;
    }
    out->n = rd->impl->n;
    out->s = rd->impl->s;
    out->level_j = rd->impl->level_j;
    out->omega_count = (int64_t)rd->impl->omega.size();
    out->fingerprint = rd->impl->fingerprint;
  });
}

int mstab_recycle_download(mstab_context* ctx, const mstab_recycle* rd, double* p, double* u,
                           double* v, double* omega_re_im) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    const Recycle& r = *real_of(rd);
    const int64_t ld = c.ld(r.n);
    auto down = [&](const DevPtr& src, double* dst) {
      if (!dst) return;
      if (cudaMemcpy2DAsync(dst, sizeof(double) * r.n, src->d(), sizeof(double) * ld, sizeof(double) * r.n,
                            r.s, cudaMemcpyDeviceToHost, c.stream()) != cudaSuccess)
        throw Error(MSTAB_E_CUDA, "recycle download");
    };
    down(r.p, p);
    down(r.u, u);
    down(r.v, v);
    if (omega_re_im)
      for (size_t i = 0; i < r.omega.size(); ++i) {
        omega_re_im[2 * i] = r.omega[i].real();
        omega_re_im[2 * i + 1] = r.omega[i].imag();
      }
    c.sync();
  });
}

int mstab_recycle_validate(mstab_context* ctx, const mstab_recycle* rd, const mstab_operator* op,
                           mstab_validation_report* out) {
  return guarded([&] {
    bind(ctx);
    if (rd->z || op->z) {  // complex data: both sides must be complex (a real side has another fingerprint space)
      if (!rd->z || !op->z) throw Error(MSTAB_E_FINGERPRINT, "recycle data belongs to a different operator");
      mstab_validation_report rz = validate_z(*ctx->impl, *rd->z, *op->z);
      if (out) *out = rz;
      return;
    }
    mstab_validation_report r = validate(*ctx->impl, *rd->impl, *op->impl);
    if (out) *out = r;
  });
}

int mstab_recycle_save(mstab_context* ctx, const mstab_recycle* rd, const char* path) {
  return guarded([&] {
    bind(ctx);
    if (ctx->impl->sharded())
      throw Error(MSTAB_E_CONFIG, "recycle save: a row-sharded context holds a slab; gather P/U/V on the host");
    const Recycle& r = *real_of(rd);
    MrdData d;
    d.n = r.n;
    d.s = r.s;
    d.level_j = r.level_j;
    d.fingerprint = r.fingerprint;
    d.p.resize((size_t)r.n * r.s);
    d.u.resize(d.p.size());
    d.v.resize(d.p.size());
    d.omega = r.omega;
    int rc = mstab_recycle_download(ctx, rd, d.p.data(), d.u.data(), d.v.data(), nullptr);
    if (rc != MSTAB_OK) throw Error(rc, g_last_error);
    mrd_write(path, d);
  });
}

int mstab_recycle_load(mstab_context* ctx, const char* path, mstab_recycle** out) {
  return guarded([&] {
    bind(ctx);
    if (ctx->impl->sharded())
      throw Error(MSTAB_E_CONFIG, "recycle load: a row-sharded context holds a slab; scatter P/U/V on the host");
    MrdData d = mrd_read(path);
    std::vector<double> om(2 * d.omega.size());
    for (size_t i = 0; i < d.omega.size(); ++i) {
      om[2 * i] = d.omega[i].real();
      om[2 * i + 1] = d.omega[i].imag();
    }
    int rc = mstab_recycle_create(ctx, d.n, d.s, d.p.data(), d.u.data(), d.v.data(), MSTAB_MEM_HOST,
                                  om.data(), (int64_t)d.omega.size(), d.level_j, d.fingerprint, out);
    if (rc != MSTAB_OK) throw Error(rc, g_last_error);
  });
}

int mstab_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                int32_t mem, const mstab_solver_config* cfg, const mstab_recycle* recycle,
                const mstab_fetch_policy* fetch, mstab_result** out) {
  return guarded([&] {
    bind(ctx);
    auto r = std::make_unique<mstab_result>();
    r->impl = solve(*ctx->impl, real_of(op), b, x0, mem, *cfg, real_of(recycle), fetch);
    *out = r.release();
  });
}

int mstab_sridr_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                      int32_t mem, const mstab_solver_config* cfg, const mstab_recycle* recycle,
                      mstab_result** out) {
  return guarded([&] {
    bind(ctx);
    if (!recycle) throw Error(MSTAB_E_CONFIG, "sridr: recycle data required");
    auto r = std::make_unique<mstab_result>();
    r->impl = sridr(*ctx->impl, real_of(op), b, x0, mem, *cfg, *real_of(recycle));
    *out = r.release();
  });
}

int mstab_bicgstab_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                         int32_t mem, double tol, int64_t max_mv, const double* shadow, mstab_result** out) {
  return guarded([&] {
    bind(ctx);
    auto r = std::make_unique<mstab_result>();
    r->impl = bicgstab(*ctx->impl, real_of(op), b, x0, mem, tol, max_mv, shadow);
    *out = r.release();
  });
}

int mstab_bicg_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                     int32_t mem, double tol, int64_t max_mv, const double* shadow, mstab_result** out) {
  return guarded([&] {
    bind(ctx);
    auto r = std::make_unique<mstab_result>();
    r->impl = bicg(*ctx->impl, real_of(op), b, x0, mem, tol, max_mv, shadow);
    *out = r.release();
  });
}

int mstab_gmres_solve(mstab_context* ctx, const mstab_operator* op, const double* b, const double* x0,
                      int32_t mem, double tol, int64_t max_it, mstab_result** out) {
  return guarded([&] {
    bind(ctx);
    auto r = std::make_unique<mstab_result>();
    r->impl = gmres(*ctx->impl, real_of(op), b, x0, mem, tol, max_it);
    *out = r.release();
  });
}

void mstab_result_destroy(mstab_result* res) { delete res; }

int mstab_result_report(const mstab_result* res, mstab_report* out) {
  return guarded([&] { *out = res->z ? res->z->report : res->impl->report; });
}

int mstab_result_x(mstab_context* ctx, const mstab_result* res, double* x, int32_t mem) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    if (!res->impl) throw Error(MSTAB_E_NOTREAL, "complex result: use mstab_result_x_z");
    if (cudaMemcpyAsync(x, res->impl->x->d(), sizeof(double) * res->impl->n,
                        mem == MSTAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                        c.stream()) != cudaSuccess)
      throw Error(MSTAB_E_CUDA, "download x");
    c.sync();
  });
}

int64_t mstab_result_history(const mstab_result* res, mstab_history_point* out, int64_t cap) {
  const auto& h = res->z ? res->z->history : res->impl->history;
  const int64_t cnt = std::min<int64_t>(cap, (int64_t)h.size());
  if (cnt > 0) std::memcpy(out, h.data(), sizeof(mstab_history_point) * cnt);
  return cnt;
}

int64_t mstab_result_taus(const mstab_result* res, double* re_im, int64_t cap) {
  if (res->z) {
    const auto& tz = res->z->taus;
    const int64_t cz = std::min<int64_t>(cap, (int64_t)tz.size());
    for (int64_t i = 0; i < cz; ++i) {
      re_im[2 * i] = tz[i].real();
      re_im[2 * i + 1] = tz[i].imag();
    }
    return cz;
  }
  const auto& t = res->impl->taus;
  const int64_t cnt = std::min<int64_t>(cap, (int64_t)t.size());
  for (int64_t i = 0; i < cnt; ++i) {
    re_im[2 * i] = t[i];
    re_im[2 * i + 1] = 0.0;
  }
  return cnt;
}

int mstab_result_final_data(const mstab_result* res, mstab_recycle** out) {
  return guarded([&] {
    auto h = std::make_unique<mstab_recycle>();
    if (res->z) {
      h->z = res->z->final_data;
      *out = h.release();
      return;
    }
    if (!res->impl->final_data) throw Error(MSTAB_E_ERROR, "no final recycle data (sridr result)");
    h->impl = res->impl->final_data;
    *out = h.release();
  });
}

int mstab_result_fetched(const mstab_result* res, mstab_recycle** out) {
  return guarded([&] {
    auto h = std::make_unique<mstab_recycle>();
    if (res->z) {
      if (!res->z->fetched) throw Error(MSTAB_E_ERROR, "no fetched recycle data");
      h->z = res->z->fetched;
      *out = h.release();
      return;
    }
    if (!res->impl->fetched) throw Error(MSTAB_E_ERROR, "no fetched recycle data");
    h->impl = res->impl->fetched;
    *out = h.release();
  });
}

int mstab_result_handoff(const mstab_result* res, mstab_recycle** out) {
  return guarded([&] {
    auto h = std::make_unique<mstab_recycle>();
    if (res->z) {
      h->z = res->z->fetched ? res->z->fetched : res->z->final_data;
      *out = h.release();
      return;
    }
    if (!res->impl->fetched && !res->impl->final_data) throw Error(MSTAB_E_ERROR, "no recycle data (sridr result)");
    h->impl = res->impl->fetched ? res->impl->fetched : res->impl->final_data;
    *out = h.release();
  });
}

// ---- complex128 data -------------------------------------------------------
int mstab_operator_create_csr_z(mstab_context* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                const double* values_re_im, mstab_operator** out) {
  return guarded([&] {
    bind(ctx);
    auto o = std::make_unique<mstab_operator>();
    o->z = make_operator_z(*ctx->impl, n, row_ptr, col_idx, values_re_im);
    *out = o.release();
  });
}
int32_t mstab_operator_is_complex(const mstab_operator* op) { return op && op->z ? 1 : 0; }
int32_t mstab_recycle_is_complex(const mstab_recycle* rd) { return rd && rd->z ? 1 : 0; }
int32_t mstab_result_is_complex(const mstab_result* res) { return res && res->z ? 1 : 0; }

int mstab_operator_apply_z(mstab_context* ctx, const mstab_operator* op, const double* x_re_im, double* y_re_im,
                           int32_t mem) {
  return guarded([&] {
    bind(ctx);
    apply_z(*ctx->impl, complex_of(op), x_re_im, y_re_im, mem);
  });
}

int mstab_recycle_create_z(mstab_context* ctx, int64_t n, int64_t s, const double* p, const double* u, const double* v,
                           int32_t mem, const double* omega_re_im, int64_t omega_count, int64_t level_j,
                           uint64_t fingerprint, mstab_recycle** out) {
  return guarded([&] {
    bind(ctx);
    auto h = std::make_unique<mstab_recycle>();
    h->z = make_recycle_z(*ctx->impl, n, s, p, u, v, mem, omega_re_im, omega_count, level_j, fingerprint);
    *out = h.release();
  });
}

int mstab_recycle_download_z(mstab_context* ctx, const mstab_recycle* rd, double* p, double* u, double* v,
                             double* omega_re_im) {
  return guarded([&] {
    bind(ctx);
    if (!rd || !rd->z) throw Error(MSTAB_E_CONFIG, "real recycle data: use mstab_recycle_download");
    download_recycle_z(*ctx->impl, *rd->z, p, u, v, omega_re_im);
  });
}

int mstab_solve_z(mstab_context* ctx, const mstab_operator* op, const double* b_re_im, const double* x0_re_im,
                  int32_t mem, const mstab_solver_config* cfg, const mstab_recycle* recycle,
                  const mstab_fetch_policy* fetch, mstab_result** out) {
  return guarded([&] {
    bind(ctx);
    if (recycle && !recycle->z) throw Error(MSTAB_E_CONFIG, "real recycle data in a complex solve");
    auto r = std::make_unique<mstab_result>();
    r->z = solve_z(*ctx->impl, complex_of(op), b_re_im, x0_re_im, mem, *cfg, recycle ? recycle->z.get() : nullptr, fetch);
    *out = r.release();
  });
}

int mstab_result_x_z(mstab_context* ctx, const mstab_result* res, double* x_re_im, int32_t mem) {
  return guarded([&] {
    bind(ctx);
    if (!res || !res->z) throw Error(MSTAB_E_CONFIG, "real result: use mstab_result_x");
    result_x_z(*ctx->impl, *res->z, x_re_im, mem);
  });
}

}  // extern "C"

// ---- kernel-level entry points (include/mstab_b200_kernels.h) -------------------------------
#include "../../include/mstab_b200_kernels.h"

extern "C" {

int mstab_kernel_solve_small(mstab_context* ctx, int64_t s, const double* m, const double* rhs,
                             double* x) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    if (s < 1 || s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: solve_small supports 1 <= s <= 16");
    DevPtr buf = c.alloc(sizeof(double) * (size_t)(s * s + 2 * s + 1));
    double* dm = buf->d();
    double* drhs = dm + s * s;
    double* dx = drhs + s;
    int32_t* dok = reinterpret_cast<int32_t*>(dx + s);
    cudaMemcpyAsync(dm, m, sizeof(double) * s * s, cudaMemcpyHostToDevice, c.stream());
    cudaMemcpyAsync(drhs, rhs, sizeof(double) * s, cudaMemcpyHostToDevice, c.stream());
    launch_small_solve(c.stream(), (int)s, dm, drhs, dx, dok);
    int32_t ok = 0;
    cudaMemcpyAsync(x, dx, sizeof(double) * s, cudaMemcpyDeviceToHost, c.stream());
    cudaMemcpyAsync(&ok, dok, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream());
    c.sync();
    if (!ok) throw Error(MSTAB_E_SINGULAR, "solve_small: pivot collapse");
  });
}

int mstab_kernel_least_squares(mstab_context* ctx, int64_t n, int64_t ell, const double* z,
                               const double* r, double* tau) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    if (ell < 1 || n < ell) throw Error(MSTAB_E_DIMENSION, "least_squares_tall: need N >= ell >= 1");
    if (ell > kMaxEll) throw Error(MSTAB_E_CONFIG, "b200: least squares supports ell <= 8");
    const int64_t ld = c.ld(n);
    DevPtr zr = c.alloc_vecs(n, ell + 1);
    cudaMemcpyAsync(zr->d(), r, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream());
    cudaMemcpy2DAsync(zr->d() + ld, sizeof(double) * ld, z, sizeof(double) * n, sizeof(double) * n, ell,
                      cudaMemcpyHostToDevice, c.stream());
    const double* cols[kMaxEll + 1];
    for (int64_t i = 0; i <= ell; ++i) cols[i] = zr->d() + i * ld;
    reset_status(c);
    launch_ls(c.stream(), n, ld, (int)ell, 1, cols, c.reducer());
    const CycleStatus& st = read_status(c);
    if (st.breakdown == kBreakRank) throw Error(MSTAB_E_RANK, "least_squares_tall: stabilization block lost rank");
    const double* h = read_scal(c, 32 + (int)ell);
    for (int64_t i = 0; i < ell; ++i) tau[i] = h[32 + i];
  });
}

int mstab_kernel_cut_space(mstab_context* ctx, int64_t n, int64_t s, uint64_t seed, double* p) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    if (s < 1 || s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: 1 <= s <= 16");
    DevPtr P = make_cut_space(c, n, (int)s, seed);
    cudaMemcpy2DAsync(p, sizeof(double) * n, P->d(), sizeof(double) * c.ld(n), sizeof(double) * n, s,
                      cudaMemcpyDeviceToHost, c.stream());
    c.sync();
  });
}

int mstab_kernel_arnoldi(mstab_context* ctx, const mstab_operator* op, const double* r0, int64_t s,
                         uint64_t rng_seed, double* u, double* v, int64_t* mv_cost) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    if (s < 1 || s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: 1 <= s <= 16");
    const int64_t n = real_of(op).n, ld = c.ld(n);
    DevPtr r = c.alloc_vecs(n, 1), U = c.alloc_vecs(n, s), V = c.alloc_vecs(n, s);
    cudaMemcpyAsync(r->d(), r0, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream());
    reset_status(c);
    arnoldi_init(c, *op->impl, r->d(), (int)s, rng_seed, U->d(), V->d());
    cudaMemcpy2DAsync(u, sizeof(double) * n, U->d(), sizeof(double) * ld, sizeof(double) * n, s,
                      cudaMemcpyDeviceToHost, c.stream());
    cudaMemcpy2DAsync(v, sizeof(double) * n, V->d(), sizeof(double) * ld, sizeof(double) * n, s,
                      cudaMemcpyDeviceToHost, c.stream());
    c.sync();
    if (mv_cost) *mv_cost = s;
  });
}

int mstab_kernel_arnoldi_cb(mstab_context* ctx, const mstab_operator* op, const double* r0, int64_t s,
                            mstab_normal_fill_fn fill, void* user, double* u, double* v, int64_t* mv_cost) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    if (s < 1 || s > kMaxS) throw Error(MSTAB_E_CONFIG, "b200: 1 <= s <= 16");
    if (!fill) throw Error(MSTAB_E_CONFIG, "arnoldi: no draw callback");
    const int64_t n = real_of(op).n, ld = c.ld(n);
    DevPtr r = c.alloc_vecs(n, 1), U = c.alloc_vecs(n, s), V = c.alloc_vecs(n, s);
    cudaMemcpyAsync(r->d(), r0, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream());
    reset_status(c);
    arnoldi_init(c, *op->impl, r->d(), (int)s, [&](double* out, int64_t count) { fill(user, out, count); },
                 U->d(), V->d());
    cudaMemcpy2DAsync(u, sizeof(double) * n, U->d(), sizeof(double) * ld, sizeof(double) * n, s,
                      cudaMemcpyDeviceToHost, c.stream());
    cudaMemcpy2DAsync(v, sizeof(double) * n, V->d(), sizeof(double) * ld, sizeof(double) * n, s,
                      cudaMemcpyDeviceToHost, c.stream());
    c.sync();
    if (mv_cost) *mv_cost = s;
  });
}

int mstab_kernel_bicg_projection(mstab_context* ctx, int64_t n, int64_t s, const double* p,
                                 const double* block, const double* target, double* gamma) {
  return guarded([&] {
    bind(ctx);
    if (n < 1) throw Error(MSTAB_E_DIMENSION, "bicg_projection: empty vectors");
    bicg_projection_host(*ctx->impl, n, (int)s, p, block, target, gamma);
  });
}

int mstab_kernel_projection_gram(mstab_context* ctx, int64_t n, int64_t s, const double* p,
                                 const double* block, const double* target, double* m, double* g) {
  return guarded([&] {
    bind(ctx);
    if (n < 1) throw Error(MSTAB_E_DIMENSION, "projection_gram: empty vectors");
    projection_gram_host(*ctx->impl, n, (int)s, p, block, target, m, g);
  });
}

int mstab_kernel_level_iteration(mstab_context* ctx, const mstab_operator* op, int64_t s, int64_t k,
                                 const double* p, double* x0, double* r_levels, double* v_levels) {
  return guarded([&] {
    bind(ctx);
    level_iteration_host(*ctx->impl, real_of(op), (int)s, (int)k, p, x0, r_levels, v_levels);
  });
}

int mstab_kernel_poly_combination(mstab_context* ctx, int64_t n, int64_t s, int64_t ell, const double* x0,
                                  const double* r_levels, const double* v_levels, double* x, double* r,
                                  double* u, double* v, double* tau, int32_t* tail_perturbed) {
  return guarded([&] {
    bind(ctx);
    poly_combination_host(*ctx->impl, n, (int)s, (int)ell, x0, r_levels, v_levels, x, r, u, v, tau,
                          tail_perturbed);
  });
}

}  // extern "C"

// ---- sequence-driver helpers ------------------------------------------------------------------
extern "C" {

}  // extern "C"

namespace {
// Element-wise host loops of the sequence driver, split over host threads (each element is
// computed by exactly one thread with the same operations, so the result does not depend on the
// split). The .cpp is compiled with -ffp-contract=off: x/dt, +f, *h2 round separately.
template <typename F>
void host_parallel(int64_t n, F&& body) {
  const int64_t grain = 1 << 16;
  unsigned hw = std::thread::hardware_concurrency();
  int nt = (int)std::min<int64_t>(hw ? hw : 1, std::max<int64_t>(1, n / grain));
  nt = std::min(nt, 16);
  if (nt <= 1) {
    body(0, n);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(nt - 1);
  const int64_t chunk = (n + nt - 1) / nt;
  for (int t = 1; t < nt; ++t) {
    const int64_t a = std::min<int64_t>(n, t * chunk), b = std::min<int64_t>(n, a + chunk);
    pool.emplace_back([&body, a, b] { body(a, b); });
  }
  body(0, std::min<int64_t>(n, chunk));
  for (auto& th : pool) th.join();
}
}  // namespace

extern "C" {

int mstab_harness_euler_rhs(mstab_context* ctx, int64_t n, const double* x, const double* f,
                            double dt, double h2, double* b, int32_t mem) {
  return guarded([&] {
    if (mem == MSTAB_MEM_DEVICE) {
      bind(ctx);
      launch_euler_rhs(ctx->impl->stream(), n, x, f, dt, h2, b);
      ctx->impl->sync();
    } else {
      host_parallel(n, [=](int64_t a, int64_t e) {
        for (int64_t i = a; i < e; ++i) b[i] = h2 * (x[i] / dt + f[i]);
      });
    }
  });
}

int mstab_harness_axpby(mstab_context* ctx, int64_t n, const double* x, const double* g,
                        double alpha, double* b, int32_t mem) {
  return guarded([&] {
    if (mem == MSTAB_MEM_DEVICE) {
      bind(ctx);
      launch_axpby_chain(ctx->impl->stream(), n, x, g, alpha, b);
      ctx->impl->sync();
    } else {
      host_parallel(n, [=](int64_t a, int64_t e) {
        for (int64_t i = a; i < e; ++i) b[i] = x[i] + alpha * g[i];
      });
    }
  });
}

}  // extern "C"

// ---- evidence hooks -------------------------------------------------------------------------
extern "C" {

uint64_t mstab_launch_count(void) { return launch_count(); }

namespace {
// MSTAB_REPORT_LAUNCHES=1: the kernel launch total on stderr at process exit (evidence that a
// host program linked against the drop-in ran its work on the device, tests/test_refsuite.py).
struct LaunchReport {
  ~LaunchReport() {
    if (std::getenv("MSTAB_REPORT_LAUNCHES"))
      std::fprintf(stderr, "[mstab] kernel launches: %llu\n", (unsigned long long)launch_count());
  }
} g_launch_report;
}  // namespace

int mstab_profiling_enable(int32_t on) {
  return guarded([&] {
    prof_collect();
    prof_enable(on != 0);
  });
}

int32_t mstab_profiling_read(mstab_kernel_class_stats* out, int32_t cap) {
  prof_collect();
  KernelClassStats st[kKNumClasses];
  prof_read(st);
  const int32_t cnt = std::min<int32_t>(cap, kKNumClasses);
  for (int32_t i = 0; i < cnt; ++i) out[i] = {(int64_t)st[i].launches, st[i].total_ms, st[i].total_bytes};
  return kKNumClasses;
}

void mstab_profiling_reset(void) {
  prof_collect();
  prof_reset();
}

const char* mstab_kernel_class_name(int32_t cls) {
  static const char* names[kKNumClasses] = {"spmv_ph", "level_update", "rebuild_top", "rebuild_deferred",
                                            "ls_tsqr", "poly", "prologue", "validate", "other", "persist_cycle"};
  return (cls >= 0 && cls < kKNumClasses) ? names[cls] : "?";
}

int mstab_kernel_bench(mstab_context* ctx, const mstab_operator* op, int32_t kind, int64_t s64,
                       int64_t ell64, int32_t iters, double* us, double* bytes) {
  return guarded([&] {
    bind(ctx);
    Context& c = *ctx->impl;
    const Operator& o = real_of(op);
    const int s = (int)s64, ell = (int)ell64;
    if (s < 1 || s > kMaxS || ell < 1 || ell > kMaxEll) throw Error(MSTAB_E_CONFIG, "bench: bad s/ell");
    const int64_t n = o.n, ld = c.ld(n);
    cudaStream_t st = c.stream();
    uint64_t seed = 1;
    auto vec = [&](int64_t cols) {
      DevPtr d = c.alloc_vecs(n, cols);
      launch_fill_hash(st, d->d(), ld * cols, seed++);
      return d;
    };
    DevPtr P = vec(s), b = vec(1);
    WSet A{vec(1), vec(1), vec(s), vec(s)}, B{vec(1), vec(1), vec(s), vec(s)};
    std::vector<DevPtr> R(ell + 1), VL(ell + 1);
    for (int i = 1; i <= ell; ++i) {
      R[i] = vec(1);
      VL[i] = vec(s);
    }
    // benign small-system state: identity projections, small coefficients, no breakdown
    DevState hs{};
    for (int i = 0; i < s; ++i) {
      hs.Ma[i + i * s] = 1.0;
      hs.Mn[i + i * s] = 1.0;
      hs.rhs[i] = hs.g[i] = 1.0;
      for (int k = 0; k < kMaxEll; ++k) hs.gamma[k * kMaxS + i] = 0.1;
      for (int q = 0; q < s; ++q) hs.eta[q * s + i] = 0.01;
    }
    for (int i = 0; i < kMaxEll; ++i) hs.st.tau[i] = 0.1;
    cudaMemcpyAsync(c.ds(), &hs, sizeof(DevState), cudaMemcpyHostToDevice, st);
    const Reducer red = c.reducer();
    DevState* ds = c.ds();
    const DevCsr csr = o.csr();
    const double* lv_in[kMaxEll + 2];
    double* lv_out[kMaxEll + 2];
    const double* rin[kMaxEll + 1];
    double* rout[kMaxEll + 1];
    const double* rr[kMaxEll + 1];
    const double* lv[kMaxEll + 2];
    const int k = ell - 1;
    lv_in[0] = lv_out[0] = A.U->d();
    lv_in[1] = lv_out[1] = A.V->d();
    lv[0] = A.U->d();
    lv[1] = A.V->d();
    for (int i = 1; i <= ell; ++i) {
      lv_in[i + 1] = lv_out[i + 1] = VL[i]->d();
      lv[i + 1] = VL[i]->d();
    }
    rin[0] = rout[0] = A.r->d();
    rr[0] = A.r->d();
    for (int i = 1; i <= ell; ++i) {
      rout[i] = R[i]->d();
      rin[i] = rr[i] = R[i]->d();
    }
    auto launch = [&]() {
      switch (kind) {
        case 0: {
          FinParams f;
          f.op = kFinRhsEta0;
          f.s = s;
          f.ell = ell;
          launch_spmv_ph(st, csr, A.r->d(), R[1]->d(), P->d(), ld, s, nullptr, f, red);
          break;
        }
        case 1:
          launch_rebuild_top(st, n, ld, s, s / 2, R[1]->d(), A.V->d(), B.V->d(), VL[1]->d(), ds);
          break;
        case 2:
          launch_level_update(st, n, ld, s, 1, A.r->d(), B.r->d(), A.V->d(), ds);
          break;
        case 3:
          launch_rebuild_deferred(st, n, ld, s, k, lv_in, lv_out, rin, rout, A.x->d(), B.x->d(), ds);
          break;
        case 4:
          launch_poly(st, n, ld, s, ell, lv, B.U->d(), B.V->d(), rr, B.r->d(), A.x->d(), B.x->d(), P->d(), red);
          break;
        case 5:
          launch_ls(st, n, ld, ell, s, rr, red);
          break;
        case 6: {  // the SpMV alone: reduced P^H y stored, no dense step in the tail
          FinParams f;
          f.op = kFinStore;
          f.s = s;
          f.dst = ds->scal;
          launch_spmv_ph(st, csr, A.r->d(), R[1]->d(), P->d(), ld, s, nullptr, f, red);
          break;
        }
        case 7:  // the s x s LU solve alone (one warp): latency of the finalizers' dense step
          launch_small_solve(st, s, ds->Ma, ds->rhs, ds->scal, reinterpret_cast<int32_t*>(ds->scal + 32));
          break;
        case 8: {  // the column-loop pair: SpMV of column q (P^H + LU for eta_{q+1}), then rebuild q+1
          const int q = s / 2 - 1 < 0 ? 0 : s / 2 - 1;
          FinParams f;
          f.op = kFinColEta;
          f.s = s;
          f.ell = ell;
          f.k = 0;
          f.q = q;
          launch_spmv_ph(st, csr, B.V->d() + q * ld, VL[1]->d() + q * ld, P->d(), ld, s, nullptr, f, red);
          launch_rebuild_top(st, n, ld, s, q + 1, R[1]->d(), A.V->d(), B.V->d(), VL[1]->d(), ds);
          break;
        }
        default:
          throw Error(MSTAB_E_CONFIG, "bench: unknown kind");
      }
    };
    launch();
    launch();
    c.sync();
    prof_collect();
    KernelClassStats before[kKNumClasses], after[kKNumClasses];
    prof_read(before);
    const bool was_on = prof_enabled();
    prof_enable(true);  // bytes per launch come from the launchers' accounting
    launch();
    c.sync();
    prof_collect();
    prof_read(after);
    prof_enable(was_on);
    double b1 = 0.0;
    for (int i = 0; i < kKNumClasses; ++i) b1 += after[i].total_bytes - before[i].total_bytes;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    for (int i = 0; i < iters; ++i) launch();
    cudaEventRecord(e1, st);
    c.sync();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaGetLastError() != cudaSuccess) throw Error(MSTAB_E_CUDA, "bench launch failed");
    *us = 1e3 * ms / iters;
    *bytes = b1;
  });
}

// Developer probes (ktimeline.cuh): with a timeline build, bind a 32-slot device buffer, run one
// kernel_bench kind, then read the slots (globaltimer ns / clock64). Product build: no-op + 0.
int mstab_timeline(mstab_context* ctx, int32_t op, uint64_t* out) {
  return guarded([&] {
    bind(ctx);
    static unsigned long long* buf = nullptr;
    if (!buf) cudaMalloc(&buf, 32 * sizeof(unsigned long long));
    if (op == 0) {  // reset + bind
      std::vector<unsigned long long> init(32, 0ull);
      for (int i = 0; i < 32; i += 2) init[i] = ~0ull;  // even slots are minima
      cudaMemcpy(buf, init.data(), 32 * sizeof(unsigned long long), cudaMemcpyHostToDevice);
      kcdia_timeline_bind(buf);
      klevel_timeline_bind(buf);
    } else if (op == 1) {  // unbind + read
      kcdia_timeline_bind(nullptr);
      klevel_timeline_bind(nullptr);
      cudaMemcpy(out, buf, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    }
  });
}

}  // extern "C"
