// ref_capi.cpp — TEST INFRASTRUCTURE ONLY. The C-ABI of include/mstab_b200.h implemented over
// the unmodified reference library (mstab:: from /root/reference/proj/core), so tests and the
// bench's reference arm drive the reference through exactly the boundary the B200 library
// exports. Host memory only (MSTAB_MEM_DEVICE -> MSTAB_E_CONFIG). Built by oracle/Makefile.
#include <complex>
#include <cstring>
#include <memory>
#include <optional>
#include <random>
#include <string>

#include "mstab/csr.hpp"
#include "mstab/errors.hpp"
#include "mstab/kernels.hpp"
#include "mstab/operator.hpp"
#include "mstab/precond.hpp"
#include "mstab/recycle.hpp"
#include "mstab/solvers/baselines.hpp"
#include "mstab/solvers/idrstab.hpp"
#include "mstab/solvers/sridr.hpp"
#include "mstab_b200.h"
#include "mstab_b200_kernels.h"

using mstab::Complex;

struct mstab_context {
  int device = -1;
};
struct mstab_operator {
  mstab::CsrMatrix m;
  mstab::SplitPreconditioner pc;  // build_none() unless created by mstab_operator_create_precond
  std::unique_ptr<mstab::LinearOperator> op;  // CsrOperator or PreconditionedOperator(pc, m)
  uint64_t fp = 0;
};
struct mstab_recycle {
  std::shared_ptr<const mstab::RecycleData> d;
};
struct mstab_result {
  mstab::SolveResult r;
  bool sridr = false;  // sridr_solve and the baselines return x and the report only
};

namespace {

thread_local std::string g_err;
thread_local int64_t g_row = -1;

struct ConfigErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NotRealErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename F>
int guarded(F&& f) {
  g_row = -1;
  try {
    f();
    return MSTAB_OK;
  } catch (const mstab::FingerprintMismatch& e) {
    g_err = e.what();
    return MSTAB_E_FINGERPRINT;
  } catch (const mstab::StaleData& e) {
    g_err = e.what();
    return MSTAB_E_STALE;
  } catch (const mstab::DimensionMismatch& e) {
    g_err = e.what();
    return MSTAB_E_DIMENSION;
  } catch (const mstab::ConfigError& e) {
    g_err = e.what();
    return MSTAB_E_CONFIG;
  } catch (const mstab::ParseError& e) {
    g_err = e.what();
    return MSTAB_E_PARSE;
  } catch (const mstab::IoError& e) {
    g_err = e.what();
    return MSTAB_E_IO;
  } catch (const mstab::SingularProjection& e) {
    g_err = e.what();
    return MSTAB_E_SINGULAR;
  } catch (const mstab::RankDeficient& e) {
    g_err = e.what();
    return MSTAB_E_RANK;
  } catch (const mstab::MissingOmegas& e) {
    g_err = e.what();
    return MSTAB_E_MISSING_OMEGAS;
  } catch (const mstab::ZeroPivot& e) {
    g_err = e.what();
    g_row = (int64_t)e.row();
    return MSTAB_E_ZEROPIVOT;
  } catch (const mstab::Error& e) {
    g_err = e.what();
    return MSTAB_E_ERROR;
  } catch (const ConfigErr& e) {
    g_err = e.what();
    return MSTAB_E_CONFIG;
  } catch (const NotRealErr& e) {
    g_err = e.what();
    return MSTAB_E_NOTREAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MSTAB_E_ERROR;
  }
}

void host_only(int32_t mem) {
  if (mem != MSTAB_MEM_HOST) throw ConfigErr("reference implementation: host memory only");
}

mstab::CsrMatrix to_csr(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* values) {
  mstab::CsrMatrix m;
  m.n_rows = m.n_cols = (size_t)n;
  const int64_t nnz = row_ptr[n];
  m.row_ptr.assign(row_ptr, row_ptr + n + 1);
  m.col_idx.assign(col_idx, col_idx + nnz);
  m.values.resize((size_t)nnz);
  for (int64_t k = 0; k < nnz; ++k) m.values[(size_t)k] = Complex(values[k], 0.0);
  m.validate();
  return m;
}

void from_csr(const mstab::CsrMatrix& m, int64_t* rp, int64_t* ci, double* val, int64_t* nnz) {
  for (size_t i = 0; i <= m.n_rows; ++i) rp[i] = (int64_t)m.row_ptr[i];
  for (size_t k = 0; k < m.col_idx.size(); ++k) {
    if (m.values[k].imag() != 0.0) throw NotRealErr("precond: complex factor");
    ci[k] = (int64_t)m.col_idx[k];
    val[k] = m.values[k].real();
  }
  *nnz = (int64_t)m.col_idx.size();
}

mstab::Vector to_vec(const double* x, int64_t n) {
  mstab::Vector v((size_t)n);
  for (int64_t i = 0; i < n; ++i) v[(size_t)i] = Complex(x[i], 0.0);
  return v;
}

mstab::DenseMatrix to_dense(const double* a, int64_t n, int64_t s) {
  mstab::DenseMatrix m((size_t)n, (size_t)s);
  for (int64_t j = 0; j < s; ++j)
    for (int64_t i = 0; i < n; ++i) m((size_t)i, (size_t)j) = Complex(a[i + j * n], 0.0);
  return m;
}

void from_dense(const mstab::DenseMatrix& m, double* out) {
  if (!out) return;
  for (size_t j = 0; j < m.cols(); ++j)
    for (size_t i = 0; i < m.rows(); ++i) out[i + j * m.rows()] = m(i, j).real();
}

}  // namespace

extern "C" {

const char* mstab_last_error(void) { return g_err.c_str(); }
int64_t mstab_last_error_row(void) { return g_row; }
const char* mstab_impl_name(void) { return "reference"; }
const char* mstab_build_id(void) { return "reference (unmodified /root/reference sources, oracle/Makefile)"; }

int mstab_context_create(int32_t device, mstab_context** out) {
  return guarded([&] {
    *out = new mstab_context();
    (*out)->device = device;
  });
}
void mstab_context_destroy(mstab_context* ctx) { delete ctx; }
int mstab_context_synchronize(mstab_context*) { return MSTAB_OK; }
int mstab_context_trim(mstab_context*) { return MSTAB_OK; }
void mstab_operator_interior_rows(const mstab_operator*, int64_t* lo, int64_t* hi) {
  if (lo) *lo = 0;
  if (hi) *hi = 0;
}
void* mstab_context_stream(mstab_context*) { return nullptr; }

int mstab_operator_create_csr(mstab_context*, int64_t n, const int64_t* row_ptr,
                              const int64_t* col_idx, const double* values, mstab_operator** out) {
  return guarded([&] {
    auto o = std::make_unique<mstab_operator>();
    o->m.n_rows = o->m.n_cols = (size_t)n;
    const int64_t nnz = row_ptr[n];
    o->m.row_ptr.assign(row_ptr, row_ptr + n + 1);
    o->m.col_idx.assign(col_idx, col_idx + nnz);
    o->m.values.resize((size_t)nnz);
    for (int64_t k = 0; k < nnz; ++k) o->m.values[(size_t)k] = Complex(values[k], 0.0);
    o->m.validate();
    o->op = std::make_unique<mstab::CsrOperator>(o->m);
    o->fp = o->op->fingerprint();
    *out = o.release();
  });
}

int mstab_precond_build(int32_t kind, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                        const double* values, int64_t* l_row_ptr, int64_t* l_col_idx, double* l_values,
                        int64_t* l_nnz, int64_t* r_row_ptr, int64_t* r_col_idx, double* r_values,
                        int64_t* r_nnz) {
  return guarded([&] {
    const mstab::CsrMatrix a = to_csr(n, row_ptr, col_idx, values);
    mstab::SplitPreconditioner pc;
    if (kind == MSTAB_PRECOND_JACOBI)
      pc = mstab::build_jacobi(a);
    else if (kind == MSTAB_PRECOND_ILU0)
      pc = mstab::build_ilu0(a);
    else
      throw ConfigErr("precond: unknown kind");
    from_csr(pc.l_factor, l_row_ptr, l_col_idx, l_values, l_nnz);
    from_csr(pc.r_factor, r_row_ptr, r_col_idx, r_values, r_nnz);
  });
}

int mstab_operator_create_precond(mstab_context*, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                  const double* values, int32_t kind, const int64_t* l_row_ptr,
                                  const int64_t* l_col_idx, const double* l_values, const int64_t* r_row_ptr,
                                  const int64_t* r_col_idx, const double* r_values, mstab_operator** out) {
  return guarded([&] {
    auto o = std::make_unique<mstab_operator>();
    o->m = to_csr(n, row_ptr, col_idx, values);
    if (kind == MSTAB_PRECOND_NONE) {
      o->op = std::make_unique<mstab::CsrOperator>(o->m);
    } else {
      if (kind != MSTAB_PRECOND_JACOBI && kind != MSTAB_PRECOND_ILU0) throw ConfigErr("precond: unknown kind");
      o->pc.kind = kind == MSTAB_PRECOND_JACOBI ? mstab::PrecondKind::Jacobi : mstab::PrecondKind::Ilu0;
      o->pc.l_factor = to_csr(n, l_row_ptr, l_col_idx, l_values);
      o->pc.r_factor = to_csr(n, r_row_ptr, r_col_idx, r_values);
      o->op = std::make_unique<mstab::PreconditionedOperator>(o->pc, o->m);
    }
    o->fp = o->op->fingerprint();
    *out = o.release();
  });
}

int32_t mstab_operator_precond_kind(const mstab_operator* op) {
  if (!op) return MSTAB_PRECOND_NONE;
  return op->pc.kind == mstab::PrecondKind::Jacobi ? MSTAB_PRECOND_JACOBI
         : op->pc.kind == mstab::PrecondKind::Ilu0 ? MSTAB_PRECOND_ILU0
                                                    : MSTAB_PRECOND_NONE;
}

int mstab_precond_solve(mstab_context*, const mstab_operator* op, int32_t which, const double* x, double* y,
                        int32_t mem) {
  return guarded([&] {
    host_only(mem);
    const int64_t n = (int64_t)op->m.n_rows;
    if (which != 0 && which != 1) throw ConfigErr("precond_solve: which must be 0 (L) or 1 (R)");
    const mstab::Vector xv = to_vec(x, n);
    const mstab::Vector out = which == 0 ? mstab::preconditioned_rhs(op->pc, xv)
                                         : mstab::unpreconditioned_solution(op->pc, xv);
    for (int64_t i = 0; i < n; ++i) y[i] = out[(size_t)i].real();
  });
}
// Row-sharded solves are a B200 extension (the reference is single-process): the
// reference implementation of the ABI reports one rank and rejects communicators and slabs.
int mstab_nccl_unique_id(uint8_t*) {
  g_err = "reference: row-sharded solves are not part of the reference";
  return MSTAB_E_CONFIG;
}
int mstab_context_set_comm_nccl(mstab_context*, int32_t, int32_t, const uint8_t*) { return mstab_nccl_unique_id(nullptr); }
int mstab_context_set_comm_host(mstab_context*, int32_t, int32_t, const mstab_host_comm*) {
  return mstab_nccl_unique_id(nullptr);
}
int mstab_context_comm_info(mstab_context*, int32_t* rank, int32_t* world) {
  if (rank) *rank = 0;
  if (world) *world = 1;
  return MSTAB_OK;
}
int mstab_operator_create_csr_slab(mstab_context*, int64_t, const int64_t*, const int64_t*, const double*,
                                   const int64_t*, mstab_operator**) {
  return mstab_nccl_unique_id(nullptr);
}
int mstab_operator_create_csr_slab_local(mstab_context*, int64_t, const int64_t*, const int64_t*, const int64_t*,
                                         const double*, const int64_t*, uint64_t, mstab_operator**) {
  return mstab_nccl_unique_id(nullptr);
}
// The resumable checksum fold: the reference's own mixing (csr.cpp:28-43), byte for byte.
namespace {
uint64_t fnv_mix(uint64_t h, const void* p, size_t len) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < len; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}
}  // namespace
uint64_t mstab_fnv_begin(int64_t n_rows, int64_t n_cols, int64_t nnz) {
  const uint64_t dims[3] = {(uint64_t)n_rows, (uint64_t)n_cols, (uint64_t)nnz};
  return fnv_mix(1469598103934665603ull, dims, sizeof(dims));
}
uint64_t mstab_fnv_fold_index(uint64_t h, const int64_t* v, int64_t count, int64_t add) {
  for (int64_t i = 0; i < count; ++i) {
    const uint64_t w = (uint64_t)(v[i] + add);
    h = fnv_mix(h, &w, sizeof(w));
  }
  return h;
}
uint64_t mstab_fnv_fold_values(uint64_t h, const double* values, int64_t count) {
  for (int64_t k = 0; k < count; ++k) {
    const Complex z(values[k], 0.0);
    h = fnv_mix(h, &z, sizeof(z));
  }
  return h;
}
int64_t mstab_operator_row_begin(const mstab_operator*) { return 0; }
int64_t mstab_operator_global_size(const mstab_operator* op) { return (int64_t)op->m.n_rows; }

void mstab_operator_destroy(mstab_operator* op) { delete op; }
int64_t mstab_operator_size(const mstab_operator* op) { return (int64_t)op->m.n_rows; }
int64_t mstab_operator_nnz(const mstab_operator* op) { return (int64_t)op->m.nnz(); }
uint64_t mstab_operator_fingerprint(const mstab_operator* op) { return op->fp; }

int mstab_operator_apply(mstab_context*, const mstab_operator* op, const double* x, double* y,
                         int32_t mem) {
  return guarded([&] {
    host_only(mem);
    const int64_t n = (int64_t)op->m.n_rows;
    mstab::Vector out = op->op->apply(to_vec(x, n));
    for (int64_t i = 0; i < n; ++i) y[i] = out[(size_t)i].real();
  });
}

int mstab_operator_apply_adjoint(mstab_context*, const mstab_operator* op, const double* x, double* y,
                                 int32_t mem) {
  return guarded([&] {
    host_only(mem);
    const int64_t n = (int64_t)op->m.n_rows;
    mstab::Vector out = op->op->apply_adjoint(to_vec(x, n));
    for (int64_t i = 0; i < n; ++i) y[i] = out[(size_t)i].real();
  });
}

int mstab_recycle_create(mstab_context*, int64_t n, int64_t s, const double* p, const double* u,
                         const double* v, int32_t mem, const double* omega_re_im,
                         int64_t omega_count, int64_t level_j, uint64_t fingerprint,
                         mstab_recycle** out) {
  return guarded([&] {
    host_only(mem);
    std::vector<Complex> om;
    for (int64_t i = 0; i < omega_count; ++i) om.emplace_back(omega_re_im[2 * i], omega_re_im[2 * i + 1]);
    auto d = std::make_shared<mstab::RecycleData>(mstab::fetch(to_dense(p, n, s), to_dense(u, n, s),
                                                               to_dense(v, n, s), om, (size_t)level_j,
                                                               fingerprint));
    *out = new mstab_recycle{d};
  });
}
void mstab_recycle_destroy(mstab_recycle* rd) { delete rd; }

int mstab_recycle_info_get(const mstab_recycle* rd, mstab_recycle_info* out) {
  return guarded([&] {
    out->n = (int64_t)rd->d->p.rows();
    out->s = (int64_t)rd->d->s;
    out->level_j = (int64_t)rd->d->level_J;
    out->omega_count = (int64_t)rd->d->omega_history.size();
    out->fingerprint = rd->d->matrix_fingerprint;
  });
}

int mstab_recycle_download(mstab_context*, const mstab_recycle* rd, double* p, double* u,
                           double* v, double* omega_re_im) {
  return guarded([&] {
    from_dense(rd->d->p, p);
    from_dense(rd->d->u, u);
    from_dense(rd->d->v, v);
    if (omega_re_im)
      for (size_t i = 0; i < rd->d->omega_history.size(); ++i) {
        omega_re_im[2 * i] = rd->d->omega_history[i].real();
        omega_re_im[2 * i + 1] = rd->d->omega_history[i].imag();
      }
  });
}

int mstab_recycle_validate(mstab_context*, const mstab_recycle* rd, const mstab_operator* op,
                           mstab_validation_report* out) {
  return guarded([&] {
    mstab::ValidationReport r = mstab::validate(*rd->d, *op->op);
    if (out) {
      out->max_deviation = r.max_deviation;
      out->sigma_min_ratio = r.sigma_min_ratio;
      out->low_rank_warning = r.low_rank_warning ? 1 : 0;
    }
  });
}

int mstab_recycle_save(mstab_context*, const mstab_recycle* rd, const char* path) {
  return guarded([&] { mstab::save(*rd->d, path); });
}

int mstab_recycle_load(mstab_context*, const char* path, mstab_recycle** out) {
  return guarded([&] {
    auto d = std::make_shared<mstab::RecycleData>(mstab::load(path));
    *out = new mstab_recycle{d};
  });
}

int mstab_solve(mstab_context*, const mstab_operator* op, const double* b, const double* x0,
                int32_t mem, const mstab_solver_config* cfg, const mstab_recycle* recycle,
                const mstab_fetch_policy* fetch, mstab_result** out) {
  return guarded([&] {
    host_only(mem);
    const int64_t n = (int64_t)op->m.n_rows;
    mstab::SolverConfig sc{(size_t)cfg->s, (size_t)cfg->ell, cfg->tol, cfg->max_mv,
                           cfg->true_residual_each_cycle != 0, cfg->seed};
    std::optional<mstab::FetchPolicy> fp;
    if (fetch) {
      if (fetch->kind == MSTAB_FETCH_AT_CYCLE) fp = mstab::FetchPolicy::at_cycle((size_t)fetch->cycle);
      else if (fetch->kind == MSTAB_FETCH_AT_HALF_TOLERANCE) fp = mstab::FetchPolicy::at_half_tolerance();
      else fp = mstab::FetchPolicy::manual();
    }
    mstab::Vector bv = to_vec(b, n);
    mstab::Vector xv = x0 ? to_vec(x0, n) : mstab::Vector{};
    auto r = std::make_unique<mstab_result>();
    r->r = mstab::idrstab_solve(*op->op, bv, xv, sc, recycle ? recycle->d.get() : nullptr,
                                fp ? &*fp : nullptr);
    *out = r.release();
  });
}

int mstab_sridr_solve(mstab_context*, const mstab_operator* op, const double* b, const double* x0, int32_t mem,
                      const mstab_solver_config* cfg, const mstab_recycle* recycle, mstab_result** out) {
  return guarded([&] {
    host_only(mem);
    if (!recycle) throw ConfigErr("sridr: recycle data required");
    const int64_t n = (int64_t)op->m.n_rows;
    mstab::SolverConfig sc{(size_t)cfg->s, (size_t)cfg->ell, cfg->tol, cfg->max_mv,
                           cfg->true_residual_each_cycle != 0, cfg->seed};
    mstab::Vector bv = to_vec(b, n);
    mstab::Vector xv = x0 ? to_vec(x0, n) : mstab::Vector{};
    auto [x, rep] = mstab::sridr_solve(*op->op, bv, xv, sc, *recycle->d);
    auto r = std::make_unique<mstab_result>();
    r->r.x = std::move(x);
    r->r.report = std::move(rep);
    r->sridr = true;
    *out = r.release();
  });
}

int mstab_bicgstab_solve(mstab_context*, const mstab_operator* op, const double* b, const double* x0, int32_t mem,
                         double tol, int64_t max_mv, const double* shadow, mstab_result** out) {
  return guarded([&] {
    host_only(mem);
    const int64_t n = (int64_t)op->m.n_rows;
    const mstab::Vector bv = to_vec(b, n);
    const mstab::Vector xv = x0 ? to_vec(x0, n) : mstab::Vector{};
    const mstab::Vector sv = shadow ? to_vec(shadow, n) : mstab::Vector{};
    auto [x, rep] = mstab::bicgstab_solve(*op->op, bv, xv, tol, max_mv, shadow ? &sv : nullptr);
    auto r = std::make_unique<mstab_result>();
    r->r.x = std::move(x);
    r->r.report = std::move(rep);
    r->sridr = true;
    *out = r.release();
  });
}

int mstab_bicg_solve(mstab_context*, const mstab_operator* op, const double* b, const double* x0, int32_t mem,
                     double tol, int64_t max_mv, const double* shadow, mstab_result** out) {
  return guarded([&] {
    host_only(mem);
    const int64_t n = (int64_t)op->m.n_rows;
    const mstab::Vector bv = to_vec(b, n);
    const mstab::Vector xv = x0 ? to_vec(x0, n) : mstab::Vector{};
    const mstab::Vector sv = shadow ? to_vec(shadow, n) : mstab::Vector{};
    auto [x, rep] = mstab::bicg_solve(*op->op, bv, xv, tol, max_mv, shadow ? &sv : nullptr);
    auto r = std::make_unique<mstab_result>();
    r->r.x = std::move(x);
    r->r.report = std::move(rep);
    r->sridr = true;
    *out = r.release();
  });
}

int mstab_gmres_solve(mstab_context*, const mstab_operator* op, const double* b, const double* x0, int32_t mem,
                      double tol, int64_t max_it, mstab_result** out) {
  return guarded([&] {
    host_only(mem);
    const int64_t n = (int64_t)op->m.n_rows;
    const mstab::Vector bv = to_vec(b, n);
    const mstab::Vector xv = x0 ? to_vec(x0, n) : mstab::Vector{};
    auto [x, rep] = mstab::gmres_solve(*op->op, bv, xv, tol, max_it);
    auto r = std::make_unique<mstab_result>();
    r->r.x = std::move(x);
    r->r.report = std::move(rep);
    r->sridr = true;
    *out = r.release();
  });
}

void mstab_result_destroy(mstab_result* res) { delete res; }

int mstab_result_report(const mstab_result* res, mstab_report* out) {
  return guarded([&] {
    const mstab::SolveReport& rep = res->r.report;
    std::memset(out, 0, sizeof(*out));
    out->h_mv = rep.h_mv;
    out->h_mv_aux = rep.h_mv_aux;
    out->h_rd = rep.h_rd;
    out->cycles = (int64_t)rep.cycles;
    out->status = rep.status == mstab::SolveStatus::Converged ? MSTAB_STATUS_CONVERGED
                  : rep.status == mstab::SolveStatus::MaxMV   ? MSTAB_STATUS_MAXMV
                                                              : MSTAB_STATUS_BREAKDOWN;
    out->has_fetched = res->r.fetched ? 1 : 0;
    out->bnorm = rep.bnorm;
    out->final_resnorm = rep.final_resnorm;
    out->wall_ns_total = rep.wall_ns_total;
    out->history_len = (int64_t)rep.residual_history.size();
    int64_t taus = 0;
    for (const auto& t : rep.omega_history) taus += (int64_t)t.size();
    out->tau_len = taus;
    out->ell = rep.omega_history.empty() ? 0 : (int64_t)rep.omega_history.front().size();
    std::snprintf(out->breakdown_reason, sizeof(out->breakdown_reason), "%s", rep.breakdown_reason.c_str());
  });
}

int mstab_result_x(mstab_context*, const mstab_result* res, double* x, int32_t mem) {
  return guarded([&] {
    host_only(mem);
    for (size_t i = 0; i < res->r.x.size(); ++i) x[i] = res->r.x[i].real();
  });
}

int64_t mstab_result_history(const mstab_result* res, mstab_history_point* out, int64_t cap) {
  const auto& h = res->r.report.residual_history;
  int64_t cnt = std::min<int64_t>(cap, (int64_t)h.size());
  for (int64_t i = 0; i < cnt; ++i)
    out[i] = {(int64_t)h[i].cycle, h[i].mv, (int64_t)h[i].level, h[i].resnorm, h[i].wall_ns};
  return cnt;
}

int64_t mstab_result_taus(const mstab_result* res, double* re_im, int64_t cap) {
  int64_t k = 0;
  for (const auto& t : res->r.report.omega_history)
    for (const Complex& z : t) {
      if (k >= cap) return k;
      re_im[2 * k] = z.real();
      re_im[2 * k + 1] = z.imag();
      ++k;
    }
  return k;
}

int mstab_result_final_data(const mstab_result* res, mstab_recycle** out) {
  return guarded([&] {
    if (res->sridr) throw mstab::Error("no final recycle data (sridr result)");
    *out = new mstab_recycle{std::make_shared<mstab::RecycleData>(res->r.final_data)};
  });
}

int mstab_result_fetched(const mstab_result* res, mstab_recycle** out) {
  return guarded([&] {
    if (!res->r.fetched) throw mstab::Error("no fetched recycle data");
    *out = new mstab_recycle{std::make_shared<mstab::RecycleData>(*res->r.fetched)};
  });
}

int mstab_result_handoff(const mstab_result* res, mstab_recycle** out) {
  return guarded([&] {
    if (res->sridr) throw mstab::Error("no recycle data (sridr result)");
    *out = new mstab_recycle{std::make_shared<mstab::RecycleData>(res->r.handoff())};
  });
}

// ---- kernel-level helpers -----------------------------------------------------------------
int mstab_kernel_solve_small(mstab_context*, int64_t s, const double* m, const double* rhs, double* x) {
  return guarded([&] {
    mstab::Vector out = mstab::solve_small(to_dense(m, s, s), to_vec(rhs, s));
    for (int64_t i = 0; i < s; ++i) x[i] = out[(size_t)i].real();
  });
}

int mstab_kernel_least_squares(mstab_context*, int64_t n, int64_t ell, const double* z,
                               const double* r, double* tau) {
  return guarded([&] {
    mstab::Vector t = mstab::least_squares_tall(to_dense(z, n, ell), to_vec(r, n));
    for (int64_t i = 0; i < ell; ++i) tau[i] = t[(size_t)i].real();
  });
}

int mstab_kernel_cut_space(mstab_context*, int64_t n, int64_t s, uint64_t seed, double* p) {
  return guarded([&] { from_dense(mstab::make_cut_space((size_t)n, (size_t)s, seed, true), p); });
}

int mstab_kernel_arnoldi(mstab_context*, const mstab_operator* op, const double* r0, int64_t s,
                         uint64_t rng_seed, double* u, double* v, int64_t* mv_cost) {
  return guarded([&] {
    std::mt19937_64 rng(rng_seed);
    mstab::Vector r = to_vec(r0, (int64_t)op->m.n_rows);
    mstab::ArnoldiResult ar = mstab::arnoldi_init(*op->op, r, (size_t)s, rng);
    from_dense(ar.u, u);
    from_dense(ar.v, v);
    if (mv_cost) *mv_cost = ar.mv_cost;
  });
}

// The reference's arnoldi_init draws its padding from a std::mt19937_64 it is handed, so a draw
// callback cannot be injected: the callback form exists on the B200 library only (the shim passes
// the caller's engine through it); this library answers the seed form, mstab_kernel_arnoldi.
int mstab_kernel_arnoldi_cb(mstab_context*, const mstab_operator*, const double*, int64_t,
                            mstab_normal_fill_fn, void*, double*, double*, int64_t*) {
  return guarded([&] { throw ConfigErr("reference build: use mstab_kernel_arnoldi (seed form)"); });
}

int mstab_kernel_bicg_projection(mstab_context*, int64_t n, int64_t s, const double* p, const double* block,
                                 const double* target, double* gamma) {
  return guarded([&] {
    mstab::Vector g = mstab::bicg_projection(to_dense(p, n, s), to_dense(block, n, s), to_vec(target, n));
    for (int64_t i = 0; i < s; ++i) gamma[i] = g[(size_t)i].real();
  });
}

int mstab_kernel_projection_gram(mstab_context*, int64_t n, int64_t s, const double* p, const double* block,
                                 const double* target, double* m, double* g) {
  return guarded([&] {
    const mstab::DenseMatrix pm = to_dense(p, n, s);
    from_dense(mstab::gemm(mstab::adjoint(pm), to_dense(block, n, s)), m);
    const mstab::Vector gv = mstab::gemv_adjoint(pm, to_vec(target, n));
    for (int64_t i = 0; i < s; ++i) g[i] = gv[(size_t)i].real();
  });
}

int mstab_kernel_level_iteration(mstab_context*, const mstab_operator* op, int64_t s, int64_t k, const double* p,
                                 double* x0, double* r_levels, double* v_levels) {
  return guarded([&] {
    const int64_t n = (int64_t)op->m.n_rows;
    mstab::IterationState st;
    st.x0 = to_vec(x0, n);
    for (int64_t i = 0; i <= k; ++i) st.r_levels.push_back(to_vec(r_levels + i * n, n));
    for (int64_t i = 0; i <= k + 1; ++i) st.v_levels.push_back(to_dense(v_levels + i * n * s, n, s));
    mstab::SolveReport rep;
    mstab::level_iteration(st, *op->op, to_dense(p, n, s), (size_t)k, rep);
    for (int64_t t = 0; t < n; ++t) x0[t] = st.x0[(size_t)t].real();
    for (int64_t i = 0; i <= k + 1; ++i)
      for (int64_t t = 0; t < n; ++t) r_levels[i * n + t] = st.r_levels[(size_t)i][(size_t)t].real();
    for (int64_t i = 0; i <= k + 2; ++i) from_dense(st.v_levels[(size_t)i], v_levels + i * n * s);
  });
}

int mstab_kernel_poly_combination(mstab_context*, int64_t n, int64_t s, int64_t ell, const double* x0,
                                  const double* r_levels, const double* v_levels, double* x, double* r,
                                  double* u, double* v, double* tau, int32_t* tail_perturbed) {
  return guarded([&] {
    mstab::IterationState st;
    st.x0 = to_vec(x0, n);
    for (int64_t i = 0; i <= ell; ++i) st.r_levels.push_back(to_vec(r_levels + i * n, n));
    for (int64_t i = 0; i <= ell + 1; ++i) st.v_levels.push_back(to_dense(v_levels + i * n * s, n, s));
    mstab::PolyOut po = mstab::poly_combination(st, (size_t)ell);
    for (int64_t t = 0; t < n; ++t) {
      x[t] = po.x[(size_t)t].real();
      r[t] = po.r[(size_t)t].real();
    }
    from_dense(po.u, u);
    from_dense(po.v, v);
    for (int64_t i = 0; i < ell; ++i) tau[i] = po.tau[(size_t)i].real();
    if (tail_perturbed) *tail_perturbed = po.tail_perturbed ? 1 : 0;
  });
}

}  // extern "C"

// ---- bench reference arm: the reference solve loop advanced one level iteration at a time ------
// (idrstab.cpp:250-259 split into steps: start + level_iteration(0), level_iteration(1), ...,
// level_iteration(ell-1) + poly_combination), so a bounded number of steps times the reference's
// own cycle cost on the workload's real system. Initialised like a fresh solve (make_cut_space +
// arnoldi_init), outside the timed steps.
namespace {
struct RefSample {
  const mstab_operator* op = nullptr;
  mstab::DenseMatrix p, u, v;
  mstab::Vector x, r;
  mstab::IterationState st;
  mstab::SolveReport rep;
  size_t k = 0, ell = 1;
};
}  // namespace

extern "C" {
void* mstab_ref_sample_create(const mstab_operator* op, const double* b, int64_t s, int64_t ell,
                              uint64_t seed) {
  try {
    auto* h = new RefSample();
    const size_t n = op->m.n_rows;
    h->op = op;
    h->ell = (size_t)ell;
    h->r = to_vec(b, (int64_t)n);
    h->x = mstab::Vector(n, Complex(0.0));
    h->p = mstab::make_cut_space(n, (size_t)s, seed, true);
    std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ull);
    mstab::ArnoldiResult ai = mstab::arnoldi_init(*op->op, h->r, (size_t)s, rng);
    h->u = std::move(ai.u);
    h->v = std::move(ai.v);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// One step; returns 0, or MSTAB_E_* on a breakdown (the sample is then restarted from its x, r).
int mstab_ref_sample_step(void* handle) {
  auto* h = static_cast<RefSample*>(handle);
  return guarded([&] {
    if (h->k == 0) h->st = mstab::IterationState::start(h->x, h->r, h->u, h->v);
    try {
      mstab::level_iteration(h->st, *h->op->op, h->p, h->k, h->rep);
      if (h->k + 1 == h->ell) {
        mstab::PolyOut po = mstab::poly_combination(h->st, h->ell);
        h->x = std::move(po.x);
        h->r = std::move(po.r);
        h->u = std::move(po.u);
        h->v = std::move(po.v);
        h->k = 0;
      } else {
        h->k++;
      }
    } catch (...) {
      h->k = 0;
      throw;
    }
  });
}

void mstab_ref_sample_destroy(void* handle) { delete static_cast<RefSample*>(handle); }
}

// ---- sequence-driver helpers (host only) ---------------------------------------------------------
extern "C" {
int mstab_harness_euler_rhs(mstab_context*, int64_t n, const double* x, const double* f, double dt,
                            double h2, double* b, int32_t mem) {
  return guarded([&] {
    host_only(mem);
    for (int64_t i = 0; i < n; ++i) {
      const volatile double q = x[i] / dt;
      const volatile double t = q + f[i];
      b[i] = h2 * t;
    }
  });
}

int mstab_harness_axpby(mstab_context*, int64_t n, const double* x, const double* g, double alpha,
                        double* b, int32_t mem) {
  return guarded([&] {
    host_only(mem);
    for (int64_t i = 0; i < n; ++i) {
      const volatile double t = alpha * g[i];
      b[i] = x[i] + t;
    }
  });
}
}

// ---- evidence hooks: the reference launches no kernels -------------------------------------
extern "C" {
uint64_t mstab_launch_count(void) { return 0; }
int mstab_profiling_enable(int32_t) { return MSTAB_OK; }
int32_t mstab_profiling_read(mstab_kernel_class_stats*, int32_t) { return 0; }
void mstab_profiling_reset(void) {}
const char* mstab_kernel_class_name(int32_t) { return "?"; }
}

extern "C" int mstab_kernel_bench(mstab_context*, const mstab_operator*, int32_t, int64_t, int64_t, int32_t,
                                  double*, double*) {
  g_err = "reference implementation: no kernels to benchmark";
  return MSTAB_E_CONFIG;
}

extern "C" int mstab_timeline(mstab_context*, int32_t, uint64_t*) {
  g_err = "reference implementation: no kernel timeline";
  return MSTAB_E_CONFIG;
}

// ---- complex128 data (include/mstab_b200.h, *_z entry points): the reference's native types ----
extern "C" {
int mstab_operator_create_csr_z(mstab_context*, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                const double* values_re_im, mstab_operator** out) {
  return guarded([&] {
    auto o = std::make_unique<mstab_operator>();
    o->m.n_rows = o->m.n_cols = (size_t)n;
    const int64_t nnz = row_ptr[n];
    o->m.row_ptr.assign(row_ptr, row_ptr + n + 1);
    o->m.col_idx.assign(col_idx, col_idx + nnz);
    o->m.values.resize((size_t)nnz);
    for (int64_t k = 0; k < nnz; ++k) o->m.values[(size_t)k] = Complex(values_re_im[2 * k], values_re_im[2 * k + 1]);
    o->m.validate();
    o->op = std::make_unique<mstab::CsrOperator>(o->m);
    o->fp = o->op->fingerprint();
    *out = o.release();
  });
}
// the reference has one (complex) type: every handle can serve both kinds of entry points; "complex"
// means some imaginary part is nonzero (is_real, types.cpp:25-29)
int32_t mstab_operator_is_complex(const mstab_operator* op) { return op && !op->m.is_real() ? 1 : 0; }
int32_t mstab_recycle_is_complex(const mstab_recycle* rd) {
  if (!rd || !rd->d) return 0;
  auto cplx = [](const mstab::DenseMatrix& m) { return !mstab::is_real(std::span<const Complex>(m.data())); };
  return cplx(rd->d->p) || cplx(rd->d->u) || cplx(rd->d->v) ? 1 : 0;
}
int32_t mstab_result_is_complex(const mstab_result* res) {
  return res && !mstab::is_real(std::span<const Complex>(res->r.x)) ? 1 : 0;
}

static mstab::Vector to_vec_z(const double* x, int64_t n) {
  mstab::Vector v((size_t)n);
  for (int64_t i = 0; i < n; ++i) v[(size_t)i] = Complex(x[2 * i], x[2 * i + 1]);
  return v;
}
static mstab::DenseMatrix to_dense_z(const double* a, int64_t n, int64_t s) {
  mstab::DenseMatrix m((size_t)n, (size_t)s);
  for (int64_t j = 0; j < s; ++j)
    for (int64_t i = 0; i < n; ++i) m((size_t)i, (size_t)j) = Complex(a[2 * (i + j * n)], a[2 * (i + j * n) + 1]);
  return m;
}
static void from_dense_z(const mstab::DenseMatrix& m, double* out) {
  if (!out) return;
  for (size_t j = 0; j < m.cols(); ++j)
    for (size_t i = 0; i < m.rows(); ++i) {
      out[2 * (i + j * m.rows())] = m(i, j).real();
      out[2 * (i + j * m.rows()) + 1] = m(i, j).imag();
    }
}

int mstab_operator_apply_z(mstab_context*, const mstab_operator* op, const double* x, double* y, int32_t mem) {
  return guarded([&] {
    host_only(mem);
    const int64_t n = (int64_t)op->m.n_rows;
    mstab::Vector r = op->op->apply(to_vec_z(x, n));
    for (int64_t i = 0; i < n; ++i) {
      y[2 * i] = r[(size_t)i].real();
      y[2 * i + 1] = r[(size_t)i].imag();
    }
  });
}

int mstab_recycle_create_z(mstab_context*, int64_t n, int64_t s, const double* p, const double* u, const double* v,
                           int32_t mem, const double* omega_re_im, int64_t omega_count, int64_t level_j,
                           uint64_t fingerprint, mstab_recycle** out) {
  return guarded([&] {
    host_only(mem);
    std::vector<Complex> om;
    for (int64_t i = 0; i < omega_count; ++i) om.emplace_back(omega_re_im[2 * i], omega_re_im[2 * i + 1]);
    auto d = std::make_shared<mstab::RecycleData>(mstab::fetch(to_dense_z(p, n, s), to_dense_z(u, n, s),
                                                               to_dense_z(v, n, s), std::move(om), (size_t)level_j,
                                                               fingerprint));
    *out = new mstab_recycle{d};
  });
}

int mstab_recycle_download_z(mstab_context*, const mstab_recycle* rd, double* p, double* u, double* v,
                             double* omega_re_im) {
  return guarded([&] {
    from_dense_z(rd->d->p, p);
    from_dense_z(rd->d->u, u);
    from_dense_z(rd->d->v, v);
    if (omega_re_im)
      for (size_t i = 0; i < rd->d->omega_history.size(); ++i) {
        omega_re_im[2 * i] = rd->d->omega_history[i].real();
        omega_re_im[2 * i + 1] = rd->d->omega_history[i].imag();
      }
  });
}

int mstab_solve_z(mstab_context*, const mstab_operator* op, const double* b, const double* x0, int32_t mem,
                  const mstab_solver_config* cfg, const mstab_recycle* recycle, const mstab_fetch_policy* fetch,
                  mstab_result** out) {
  return guarded([&] {
    host_only(mem);
    const int64_t n = (int64_t)op->m.n_rows;
    mstab::SolverConfig sc{(size_t)cfg->s, (size_t)cfg->ell, cfg->tol, cfg->max_mv,
                           cfg->true_residual_each_cycle != 0, cfg->seed};
    std::optional<mstab::FetchPolicy> fp;
    if (fetch) {
      if (fetch->kind == MSTAB_FETCH_AT_CYCLE) fp = mstab::FetchPolicy::at_cycle((size_t)fetch->cycle);
      else if (fetch->kind == MSTAB_FETCH_AT_HALF_TOLERANCE) fp = mstab::FetchPolicy::at_half_tolerance();
      else fp = mstab::FetchPolicy::manual();
    }
    mstab::Vector bv = to_vec_z(b, n);
    mstab::Vector xv = x0 ? to_vec_z(x0, n) : mstab::Vector{};
    auto r = std::make_unique<mstab_result>();
    r->r = mstab::idrstab_solve(*op->op, bv, xv, sc, recycle ? recycle->d.get() : nullptr, fp ? &*fp : nullptr);
    *out = r.release();
  });
}

int mstab_result_x_z(mstab_context*, const mstab_result* res, double* x, int32_t mem) {
  return guarded([&] {
    host_only(mem);
    for (size_t i = 0; i < res->r.x.size(); ++i) {
      x[2 * i] = res->r.x[i].real();
      x[2 * i + 1] = res->r.x[i].imag();
    }
  });
}
}  // extern "C"
