// idrstab_b200.cpp — C++ drop-in shim: the reference's solve entry points
//
//   mstab::idrstab_solve(const LinearOperator&, const Vector& b, const Vector& x0,
//                        const SolverConfig&, const RecycleData*, const FetchPolicy*)
//   mstab::mstab_solve  (..., const RecycleData&, const FetchPolicy*)
//
// (proj/core/include/mstab/solvers/idrstab.hpp:88-96) defined on top of the B200 C-ABI
// (include/mstab_b200.h), so a reference build that compiles this file instead of the two entry
// points of src/idrstab.cpp runs every solve on the GPU. The test-visible
// helpers of the same header (idrstab.hpp:27-68: arnoldi_init, bicg_projection,
// IterationState::start, level_iteration, poly_combination) are defined here too, device-backed
// through the kernel-level C-ABI (include/mstab_b200_kernels.h: host blocks copied in, the solve
// loop's own kernels, results copied out), so this file replaces src/idrstab.cpp as a whole.
// Everything else of the reference library (CsrMatrix, CsrOperator, RecycleData,
// fetch/validate/save/load, the harness) stays the reference's own.
//
// Behaviour kept from idrstab.cpp:193-307:
//   * check order: SolverConfig::validate (report.cpp:16-22) -> DimensionMismatch for b / x0
//     (:198-199) -> ensure_finite(b) (:200) -> (recycle) validate / s mismatch;
//   * exceptions escaping to the caller are the reference's classes (errors.hpp:9-72), mapped 1:1
//     from the C-ABI codes; breakdowns are a status with the reason string (:290-293);
//   * SolveResult owns deep copies of x, the report (histories, per-cycle tau), final_data and
//     the fetched snapshot (recycle.cpp:26-38).
// B200 restrictions (no CPU fallback): the operator must be a CsrOperator or a
// PreconditionedOperator over one (split Jacobi / ILU(0), precond.hpp) and all data real
// (imaginary parts exactly 0); anything else is rejected with ConfigError.
#include <complex>
#include <cstdint>
#include <list>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "mstab/csr.hpp"
#include "mstab/errors.hpp"
#include "mstab/kernels.hpp"
#include "mstab/operator.hpp"
#include "mstab/precond.hpp"
#include "mstab/recycle.hpp"
#include "mstab/solvers/idrstab.hpp"
#include "mstab/solvers/baselines.hpp"
#include "mstab/solvers/report.hpp"
#include "mstab/solvers/sridr.hpp"
#include "mstab/types.hpp"
#include "mstab_b200.h"
#include "mstab_b200_kernels.h"

namespace mstab {

namespace {

[[noreturn]] void rethrow(int code) {
  const std::string msg = std::string("b200: ") + mstab_last_error();
  switch (code) {
    case MSTAB_E_DIMENSION: throw DimensionMismatch(msg);
    case MSTAB_E_CONFIG: throw ConfigError(msg);
    case MSTAB_E_FINGERPRINT: throw FingerprintMismatch(msg);
    case MSTAB_E_STALE: throw StaleData(msg);
    case MSTAB_E_PARSE: throw ParseError(msg);
    case MSTAB_E_IO: throw IoError(msg);
    case MSTAB_E_SINGULAR: throw SingularProjection(msg);
    case MSTAB_E_RANK: throw RankDeficient(msg);
    case MSTAB_E_NOTREAL: throw ConfigError(msg);
    case MSTAB_E_ZEROPIVOT: {  // ZeroPivot(row) builds its own message, like precond.cpp
      const int64_t row = mstab_last_error_row();
      if (row >= 0) throw ZeroPivot(static_cast<std::size_t>(row));
      throw Error(msg);
    }
    case MSTAB_E_MISSING_OMEGAS: throw MissingOmegas(msg);
    default: throw Error(msg);
  }
}

void check(int code) {
  if (code != MSTAB_OK) rethrow(code);
}

// One B200 context per host thread (a solve is single-threaded and owns its state, like the
// reference's; operators are shared read-only).
struct Session {
  mstab_context* ctx = nullptr;
  struct CachedOp {
    const CsrMatrix* m = nullptr;
    uint64_t fp = 0;
    size_t nnz = 0;
    mstab_operator* op = nullptr;
    bool complex = false;  // uploaded through mstab_operator_create_csr_z
  };
  std::list<CachedOp> ops;  // most recent first
  Session() { check(mstab_context_create(-1, &ctx)); }
  ~Session() {
    for (auto& c : ops) mstab_operator_destroy(c.op);
    if (ctx) mstab_context_destroy(ctx);
  }
};

Session& session() {
  thread_local Session s;
  return s;
}

std::vector<double> real_parts(std::span<const Complex> v, const char* what) {
  std::vector<double> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    if (v[i].imag() != 0.0)
      throw ConfigError(std::string("b200: complex ") + what + " not supported (real fp64 path)");
    out[i] = v[i].real();
  }
  return out;
}

// PreconditionedOperator keeps its preconditioner and matrix private (precond.hpp:71-72) and has
// no accessors. The shim reads them without touching the reference: an explicit instantiation
// may name a private member ([temp.spec.general]/6), and the friend defined inside it hands the
// member pointer out.
template <typename Tag, typename Tag::type M>
struct MemberOf {
  friend typename Tag::type member(Tag) { return M; }
};
struct PcOf {
  using type = const SplitPreconditioner* PreconditionedOperator::*;
  friend type member(PcOf);
};
struct MatOf {
  using type = const CsrMatrix* PreconditionedOperator::*;
  friend type member(MatOf);
};
template struct MemberOf<PcOf, &PreconditionedOperator::pc_>;
template struct MemberOf<MatOf, &PreconditionedOperator::a_>;

struct Csr64 {
  std::vector<int64_t> rp, ci;
  std::vector<double> va;
  Csr64(const CsrMatrix& m, const char* what)
      : rp(m.row_ptr.begin(), m.row_ptr.end()), ci(m.col_idx.begin(), m.col_idx.end()), va(real_parts(m.values, what)) {}
};

// Uploads the operator once per content (keyed by address, re-checked by the reference's own
// fingerprint, csr.cpp:28-43 / precond.cpp:203-210, which the reference recomputes on every
// solve anyway). A PreconditionedOperator goes up with its factors: L^-1 A R^-1 on the device.
mstab_operator* device_operator(Session& ss, const LinearOperator& a) {
  const CsrMatrix* mp = nullptr;
  const SplitPreconditioner* pc = nullptr;
  if (const auto* csr = dynamic_cast<const CsrOperator*>(&a)) {
    mp = &csr->matrix();
  } else if (const auto* pre = dynamic_cast<const PreconditionedOperator*>(&a)) {
    mp = pre->*member(MatOf{});
    pc = pre->*member(PcOf{});
    if (pc->kind == PrecondKind::None) pc = nullptr;
  } else {
    throw ConfigError("b200: only CsrOperator and PreconditionedOperator are supported on the device path");
  }
  const CsrMatrix& m = *mp;
  const uint64_t fp = a.fingerprint();
  for (auto it = ss.ops.begin(); it != ss.ops.end(); ++it)
    if (!it->complex && it->m == &m && it->fp == fp && it->nnz == m.nnz()) {
      ss.ops.splice(ss.ops.begin(), ss.ops, it);
      return it->op;
    }
  if (!m.is_real()) throw ConfigError("b200: complex operator on a real fp64 entry point (only idrstab_solve / mstab_solve take complex data)");
  const int64_t n = (int64_t)m.n_rows;
  const Csr64 am(m, "operator");
  mstab_operator* op = nullptr;
  if (pc) {
    const Csr64 l(pc->l_factor, "preconditioner"), r(pc->r_factor, "preconditioner");
    const int32_t kind = pc->kind == PrecondKind::Jacobi ? MSTAB_PRECOND_JACOBI : MSTAB_PRECOND_ILU0;
    check(mstab_operator_create_precond(ss.ctx, n, am.rp.data(), am.ci.data(), am.va.data(), kind, l.rp.data(),
                                        l.ci.data(), l.va.data(), r.rp.data(), r.ci.data(), r.va.data(), &op));
  } else {
    check(mstab_operator_create_csr(ss.ctx, n, am.rp.data(), am.ci.data(), am.va.data(), &op));
  }
  ss.ops.push_front({&m, fp, m.nnz(), op, false});
  while (ss.ops.size() > 8) {
    mstab_operator_destroy(ss.ops.back().op);
    ss.ops.pop_back();
  }
  return op;
}

// ---- complex128 data: std::complex<double> arrays are the interleaved (re, im)
// layout of the *_z entry points ----
bool has_imag(std::span<const Complex> v) {
  for (const Complex& z : v)
    if (z.imag() != 0.0) return true;
  return false;
}
const double* as_re_im(const Complex* p) { return reinterpret_cast<const double*>(p); }

// The operator with complex values (a real matrix goes up with +0.0 imaginary parts when the
// vectors are complex: the reference has a single complex type). Plain CsrOperator only.
mstab_operator* device_operator_z(Session& ss, const LinearOperator& a) {
  const auto* csr = dynamic_cast<const CsrOperator*>(&a);
  if (!csr) throw ConfigError("b200: complex data needs a plain CsrOperator (no preconditioner) on the device path");
  const CsrMatrix& m = csr->matrix();
  const uint64_t fp = a.fingerprint();
  for (auto it = ss.ops.begin(); it != ss.ops.end(); ++it)
    if (it->complex && it->m == &m && it->fp == fp && it->nnz == m.nnz()) {
      ss.ops.splice(ss.ops.begin(), ss.ops, it);
      return it->op;
    }
  const std::vector<int64_t> rp(m.row_ptr.begin(), m.row_ptr.end()), ci(m.col_idx.begin(), m.col_idx.end());
  mstab_operator* op = nullptr;
  check(mstab_operator_create_csr_z(ss.ctx, (int64_t)m.n_rows, rp.data(), ci.data(), as_re_im(m.values.data()), &op));
  ss.ops.push_front({&m, fp, m.nnz(), op, true});
  while (ss.ops.size() > 8) {
    mstab_operator_destroy(ss.ops.back().op);
    ss.ops.pop_back();
  }
  return op;
}

struct RecycleHandle {
  mstab_recycle* h = nullptr;
  ~RecycleHandle() {
    if (h) mstab_recycle_destroy(h);
  }
};

void upload_recycle(Session& ss, const RecycleData& rd, RecycleHandle& out) {
  const int64_t n = (int64_t)rd.p.rows(), s = (int64_t)rd.s;
  if ((int64_t)rd.p.cols() != s || (int64_t)rd.u.rows() != n || (int64_t)rd.u.cols() != s ||
      (int64_t)rd.v.rows() != n || (int64_t)rd.v.cols() != s)
    throw DimensionMismatch("recycle data has inconsistent shapes");
  const auto p = real_parts(rd.p.data(), "recycle P");
  const auto u = real_parts(rd.u.data(), "recycle U");
  const auto v = real_parts(rd.v.data(), "recycle V");
  std::vector<double> om(2 * rd.omega_history.size());
  for (size_t i = 0; i < rd.omega_history.size(); ++i) {
    om[2 * i] = rd.omega_history[i].real();
    om[2 * i + 1] = rd.omega_history[i].imag();
  }
  check(mstab_recycle_create(ss.ctx, n, s, p.data(), u.data(), v.data(), MSTAB_MEM_HOST,
                             om.empty() ? nullptr : om.data(), (int64_t)rd.omega_history.size(),
                             (int64_t)rd.level_J, rd.matrix_fingerprint, &out.h));
}

void upload_recycle_z(Session& ss, const RecycleData& rd, RecycleHandle& out) {
  const int64_t n = (int64_t)rd.p.rows(), s = (int64_t)rd.s;
  if ((int64_t)rd.p.cols() != s || (int64_t)rd.u.rows() != n || (int64_t)rd.u.cols() != s ||
      (int64_t)rd.v.rows() != n || (int64_t)rd.v.cols() != s)
    throw DimensionMismatch("recycle data has inconsistent shapes");
  check(mstab_recycle_create_z(ss.ctx, n, s, as_re_im(rd.p.data().data()), as_re_im(rd.u.data().data()),
                               as_re_im(rd.v.data().data()), MSTAB_MEM_HOST,
                               rd.omega_history.empty() ? nullptr : as_re_im(rd.omega_history.data()),
                               (int64_t)rd.omega_history.size(), (int64_t)rd.level_J, rd.matrix_fingerprint, &out.h));
}

RecycleData download_recycle(Session& ss, mstab_recycle* h) {
  mstab_recycle_info info{};
  check(mstab_recycle_info_get(h, &info));
  const size_t n = (size_t)info.n, s = (size_t)info.s;
  if (mstab_recycle_is_complex(h)) {
    RecycleData rz;
    rz.p = DenseMatrix(n, s);
    rz.u = DenseMatrix(n, s);
    rz.v = DenseMatrix(n, s);
    rz.omega_history.resize((size_t)info.omega_count);
    check(mstab_recycle_download_z(ss.ctx, h, reinterpret_cast<double*>(rz.p.data().data()),
                                   reinterpret_cast<double*>(rz.u.data().data()),
                                   reinterpret_cast<double*>(rz.v.data().data()),
                                   rz.omega_history.empty() ? nullptr
                                                            : reinterpret_cast<double*>(rz.omega_history.data())));
    rz.level_J = (size_t)info.level_j;
    rz.s = s;
    rz.matrix_fingerprint = info.fingerprint;
    return rz;
  }
  std::vector<double> p(n * s), u(n * s), v(n * s), om(2 * (size_t)info.omega_count);
  check(mstab_recycle_download(ss.ctx, h, p.data(), u.data(), v.data(), om.empty() ? nullptr : om.data()));
  RecycleData rd;
  rd.p = DenseMatrix(n, s);
  rd.u = DenseMatrix(n, s);
  rd.v = DenseMatrix(n, s);
  for (size_t i = 0; i < n * s; ++i) {
    rd.p.data()[i] = Complex(p[i]);
    rd.u.data()[i] = Complex(u[i]);
    rd.v.data()[i] = Complex(v[i]);
  }
  for (int64_t i = 0; i < info.omega_count; ++i) rd.omega_history.emplace_back(om[2 * i], om[2 * i + 1]);
  rd.level_J = (size_t)info.level_j;
  rd.s = s;
  rd.matrix_fingerprint = info.fingerprint;
  return rd;
}

// SolveResult::x and SolveReport (histories, per-cycle tau) from a C-ABI result.
void read_result(Session& ss, mstab_result* res, size_t n, size_t cfg_ell, Vector& x_out, SolveReport& rep) {
  mstab_report r{};
  check(mstab_result_report(res, &r));
  x_out.resize(n);
  if (mstab_result_is_complex(res)) {
    check(mstab_result_x_z(ss.ctx, res, reinterpret_cast<double*>(x_out.data()), MSTAB_MEM_HOST));
  } else {
    std::vector<double> x(n);
    check(mstab_result_x(ss.ctx, res, x.data(), MSTAB_MEM_HOST));
    for (size_t i = 0; i < n; ++i) x_out[i] = Complex(x[i]);
  }
  rep.h_mv = r.h_mv;
  rep.h_mv_aux = r.h_mv_aux;
  rep.h_rd = r.h_rd;
  rep.cycles = (size_t)r.cycles;
  rep.status = r.status == MSTAB_STATUS_CONVERGED ? SolveStatus::Converged
               : r.status == MSTAB_STATUS_MAXMV   ? SolveStatus::MaxMV
                                                  : SolveStatus::Breakdown;
  rep.breakdown_reason = r.breakdown_reason;
  rep.bnorm = r.bnorm;
  rep.final_resnorm = r.final_resnorm;
  rep.wall_ns_total = r.wall_ns_total;
  std::vector<mstab_history_point> hist((size_t)r.history_len);
  if (r.history_len > 0 && mstab_result_history(res, hist.data(), r.history_len) != r.history_len)
    throw Error("b200: history read failed");
  for (const auto& h : hist)
    rep.residual_history.push_back({(size_t)h.cycle, h.mv, (size_t)h.level, h.resnorm, h.wall_ns});
  std::vector<double> taus(2 * (size_t)r.tau_len);
  if (r.tau_len > 0 && mstab_result_taus(res, taus.data(), r.tau_len) != r.tau_len)
    throw Error("b200: tau read failed");
  const int64_t ell = r.ell > 0 ? r.ell : (int64_t)cfg_ell;
  for (int64_t c0 = 0; c0 + ell <= r.tau_len; c0 += ell) {
    std::vector<Complex> t;
    for (int64_t j = 0; j < ell; ++j) t.emplace_back(taus[2 * (c0 + j)], taus[2 * (c0 + j) + 1]);
    rep.omega_history.push_back(std::move(t));
  }
}

mstab_solver_config to_c(const SolverConfig& cfg) {
  mstab_solver_config c{};
  c.s = (int64_t)cfg.s;
  c.ell = (int64_t)cfg.ell;
  c.tol = cfg.tol;
  c.max_mv = cfg.max_mv;
  c.true_residual_each_cycle = cfg.true_residual_each_cycle ? 1 : 0;
  c.seed = cfg.seed;
  return c;
}

}  // namespace

SolveResult idrstab_solve(const LinearOperator& a, const Vector& b, const Vector& x0,
                          const SolverConfig& cfg, const RecycleData* recycle,
                          const FetchPolicy* fetch_policy) {
  cfg.validate();
  const std::size_t n = a.size();
  if (b.size() != n) throw DimensionMismatch("idrstab: rhs size");
  if (!x0.empty() && x0.size() != n) throw DimensionMismatch("idrstab: guess size");
  ensure_finite(b, "idrstab rhs");
  if (!x0.empty()) ensure_finite(x0, "idrstab guess");

  Session& ss = session();
  // complex data anywhere (operator, b, x0, recycle blocks) takes the complex128 entry points
  const bool cplx = !a.is_real() || has_imag(b) || has_imag(x0) ||
                    (recycle && (has_imag(recycle->p.data()) || has_imag(recycle->u.data()) ||
                                 has_imag(recycle->v.data())));
  mstab_operator* op = cplx ? device_operator_z(ss, a) : device_operator(ss, a);
  std::vector<double> bh, xh;
  if (!cplx) {
    bh = real_parts(b, "rhs");
    xh = real_parts(x0, "guess");
  }
  RecycleHandle rh;
  if (recycle) {
    if (cplx)
      upload_recycle_z(ss, *recycle, rh);
    else
      upload_recycle(ss, *recycle, rh);
  }

  mstab_solver_config c = to_c(cfg);
  mstab_fetch_policy fp{};
  if (fetch_policy) {
    fp.kind = fetch_policy->kind == FetchPolicy::Kind::AtCycle          ? MSTAB_FETCH_AT_CYCLE
              : fetch_policy->kind == FetchPolicy::Kind::AtHalfTolerance ? MSTAB_FETCH_AT_HALF_TOLERANCE
                                                                         : MSTAB_FETCH_MANUAL;
    fp.cycle = (int64_t)fetch_policy->cycle;
  }
  mstab_result* res = nullptr;
  if (cplx)
    check(::mstab_solve_z(ss.ctx, op, as_re_im(b.data()), x0.empty() ? nullptr : as_re_im(x0.data()), MSTAB_MEM_HOST,
                          &c, rh.h, fetch_policy ? &fp : nullptr, &res));
  else
    check(::mstab_solve(ss.ctx, op, bh.data(), x0.empty() ? nullptr : xh.data(), MSTAB_MEM_HOST, &c, rh.h,
                        fetch_policy ? &fp : nullptr, &res));
  std::unique_ptr<mstab_result, void (*)(mstab_result*)> guard(res, mstab_result_destroy);

  SolveResult out;
  read_result(ss, res, n, cfg.ell, out.x, out.report);
  mstab_report r{};
  check(mstab_result_report(res, &r));

  RecycleHandle fin;
  check(mstab_result_final_data(res, &fin.h));
  out.final_data = download_recycle(ss, fin.h);
  if (r.has_fetched) {
    RecycleHandle fh;
    check(mstab_result_fetched(res, &fh.h));
    out.fetched = download_recycle(ss, fh.h);
  }
  return out;
}

SolveResult mstab_solve(const LinearOperator& a, const Vector& b, const Vector& x0,
                        const SolverConfig& cfg, const RecycleData& recycle,
                        const FetchPolicy* fetch_policy) {
  return idrstab_solve(a, b, x0, cfg, &recycle, fetch_policy);
}

// sridr_solve (sridr.hpp, sridr.cpp:23-118) on the device: the recycled phase and the IDR(s)
// cycles both run on the B200 (ksridr.cu + the cycle graphs).
std::pair<Vector, SolveReport> sridr_solve(const LinearOperator& a, const Vector& b, const Vector& x0,
                                           const SolverConfig& cfg, const RecycleData& recycle) {
  cfg.validate();
  if (cfg.ell != 1) throw ConfigError("sridr: ell == 1 required");
  const std::size_t n = a.size();
  if (b.size() != n) throw DimensionMismatch("sridr: rhs size");
  Session& ss = session();
  mstab_operator* op = device_operator(ss, a);
  const std::vector<double> bh = real_parts(b, "rhs");
  const std::vector<double> xh = real_parts(x0, "guess");
  RecycleHandle rh;
  upload_recycle(ss, recycle, rh);
  const mstab_solver_config c = to_c(cfg);
  mstab_result* res = nullptr;
  check(::mstab_sridr_solve(ss.ctx, op, bh.data(), x0.empty() ? nullptr : xh.data(), MSTAB_MEM_HOST, &c, rh.h,
                            &res));
  std::unique_ptr<mstab_result, void (*)(mstab_result*)> guard(res, mstab_result_destroy);
  std::pair<Vector, SolveReport> out;
  read_result(ss, res, n, 1, out.first, out.second);
  return out;
}

// The comparison baselines (baselines.hpp, baselines.cpp:49-262) on the device.
std::pair<Vector, SolveReport> gmres_solve(const LinearOperator& a, const Vector& b, const Vector& x0, double tol,
                                           std::int64_t max_it) {
  const std::size_t n = a.size();
  if (b.size() != n) throw DimensionMismatch("gmres: rhs size");
  Session& ss = session();
  mstab_operator* op = device_operator(ss, a);
  const std::vector<double> bh = real_parts(b, "rhs");
  const std::vector<double> xh = real_parts(x0, "guess");
  mstab_result* res = nullptr;
  check(::mstab_gmres_solve(ss.ctx, op, bh.data(), x0.empty() ? nullptr : xh.data(), MSTAB_MEM_HOST, tol, max_it,
                            &res));
  std::unique_ptr<mstab_result, void (*)(mstab_result*)> guard(res, mstab_result_destroy);
  std::pair<Vector, SolveReport> out;
  read_result(ss, res, n, 1, out.first, out.second);
  out.second.omega_history.clear();
  return out;
}

std::pair<Vector, SolveReport> bicg_solve(const LinearOperator& a, const Vector& b, const Vector& x0, double tol,
                                          std::int64_t max_mv, const Vector* shadow) {
  const std::size_t n = a.size();
  if (b.size() != n) throw DimensionMismatch("bicg: rhs size");
  Session& ss = session();
  mstab_operator* op = device_operator(ss, a);
  const std::vector<double> bh = real_parts(b, "rhs");
  const std::vector<double> xh = real_parts(x0, "guess");
  std::vector<double> sh;
  if (shadow) sh = real_parts(*shadow, "shadow");
  mstab_result* res = nullptr;
  check(::mstab_bicg_solve(ss.ctx, op, bh.data(), x0.empty() ? nullptr : xh.data(), MSTAB_MEM_HOST, tol, max_mv,
                           shadow ? sh.data() : nullptr, &res));
  std::unique_ptr<mstab_result, void (*)(mstab_result*)> guard(res, mstab_result_destroy);
  std::pair<Vector, SolveReport> out;
  read_result(ss, res, n, 1, out.first, out.second);
  out.second.omega_history.clear();
  return out;
}

std::pair<Vector, SolveReport> bicgstab_solve(const LinearOperator& a, const Vector& b, const Vector& x0, double tol,
                                              std::int64_t max_mv, const Vector* shadow) {
  const std::size_t n = a.size();
  if (b.size() != n) throw DimensionMismatch("bicgstab: rhs size");
  Session& ss = session();
  mstab_operator* op = device_operator(ss, a);
  const std::vector<double> bh = real_parts(b, "rhs");
  const std::vector<double> xh = real_parts(x0, "guess");
  std::vector<double> sh;
  if (shadow) sh = real_parts(*shadow, "shadow");
  mstab_result* res = nullptr;
  check(::mstab_bicgstab_solve(ss.ctx, op, bh.data(), x0.empty() ? nullptr : xh.data(), MSTAB_MEM_HOST, tol, max_mv,
                               shadow ? sh.data() : nullptr, &res));
  std::unique_ptr<mstab_result, void (*)(mstab_result*)> guard(res, mstab_result_destroy);
  std::pair<Vector, SolveReport> out;
  read_result(ss, res, n, 1, out.first, out.second);
  out.second.omega_history.clear();
  return out;
}

// ---- the test-visible helpers (idrstab.hpp:27-68), device-backed --------------------------------
namespace {

std::vector<double> dense_real(const DenseMatrix& m, const char* what) { return real_parts(m.data(), what); }

DenseMatrix dense_from(const double* a, size_t n, size_t s) {
  DenseMatrix m(n, s);
  for (size_t i = 0; i < n * s; ++i) m.data()[i] = Complex(a[i]);
  return m;
}

struct DrawCtx {
  std::mt19937_64* rng;
  std::normal_distribution<double> normal{0.0, 1.0};  // one per arnoldi_init call (idrstab.cpp:60)
};
void draw_normals(void* user, double* out, int64_t count) {
  auto* d = static_cast<DrawCtx*>(user);
  for (int64_t i = 0; i < count; ++i) out[i] = d->normal(*d->rng);  // real problems: one draw per entry (:77-78)
}

}  // namespace

ArnoldiResult arnoldi_init(const LinearOperator& a, std::span<const Complex> r0, std::size_t s,
                           std::mt19937_64& rng) {
  const std::size_t n = a.size();
  if (s < 1) throw ConfigError("arnoldi_init: s >= 1 required");
  if (r0.size() != n) throw DimensionMismatch("arnoldi_init: start vector length");
  Session& ss = session();
  mstab_operator* op = device_operator(ss, a);
  const auto r = real_parts(r0, "start vector");
  std::vector<double> u(n * s), v(n * s);
  DrawCtx dc{&rng};
  int64_t mv = 0;
  check(mstab_kernel_arnoldi_cb(ss.ctx, op, r.data(), (int64_t)s, draw_normals, &dc, u.data(), v.data(), &mv));
  ArnoldiResult res;
  res.u = dense_from(u.data(), n, s);
  res.v = dense_from(v.data(), n, s);
  res.mv_cost = mv;
  return res;
}

namespace {
bool all_real(std::span<const Complex> v) {
  for (const Complex& z : v)
    if (z.imag() != 0.0) return false;
  return true;
}
void split(std::span<const Complex> v, std::vector<double>& re, std::vector<double>& im) {
  re.resize(v.size());
  im.resize(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    re[i] = v[i].real();
    im[i] = v[i].imag();
  }
}
}  // namespace

Vector bicg_projection(const DenseMatrix& p, const DenseMatrix& block, std::span<const Complex> target) {
  const std::size_t n = p.rows(), s = p.cols();
  if (block.rows() != n || block.cols() != s || target.size() != n)
    throw DimensionMismatch("bicg_projection: shapes");
  Session& ss = session();
  if (!all_real(p.data()) || !all_real(block.data()) || !all_real(target)) {
    // Complex data (the reference's BicgProjection tests): the length-n reductions still run on
    // the device, on real and imaginary parts,
    //   P^H B = (Pr^T Br + Pi^T Bi) + i (Pr^T Bi - Pi^T Br),  P^H t likewise,
    // and the s x s complex system goes to the reference's own solve_small (kernels.cpp:150-154).
    std::vector<double> pr, pi, br, bi, tr, ti;
    split(p.data(), pr, pi);
    split(block.data(), br, bi);
    split(target, tr, ti);
    std::vector<double> m[4], g[4];
    const double* lhs[4] = {pr.data(), pi.data(), pr.data(), pi.data()};
    const double* rb[4] = {br.data(), bi.data(), bi.data(), br.data()};
    const double* rt[4] = {tr.data(), ti.data(), ti.data(), tr.data()};
    for (int k = 0; k < 4; ++k) {
      m[k].resize(s * s);
      g[k].resize(s);
      check(mstab_kernel_projection_gram(ss.ctx, (int64_t)n, (int64_t)s, lhs[k], rb[k], rt[k], m[k].data(),
                                         g[k].data()));
    }
    DenseMatrix msys(s, s);
    Vector rhs(s);
    for (std::size_t i = 0; i < s * s; ++i) msys.data()[i] = Complex(m[0][i] + m[1][i], m[2][i] - m[3][i]);
    for (std::size_t i = 0; i < s; ++i) rhs[i] = Complex(g[0][i] + g[1][i], g[2][i] - g[3][i]);
    return solve_small(msys, rhs);
  }
  const auto pp = dense_real(p, "P"), bb = dense_real(block, "block"), tt = real_parts(target, "target");
  std::vector<double> g(s);
  check(mstab_kernel_bicg_projection(ss.ctx, (int64_t)n, (int64_t)s, pp.data(), bb.data(), tt.data(), g.data()));
  Vector out(s);
  for (std::size_t i = 0; i < s; ++i) out[i] = Complex(g[i]);
  return out;
}

IterationState IterationState::start(Vector x, Vector r, DenseMatrix u, DenseMatrix v) {
  IterationState st;
  st.x0 = std::move(x);
  st.r_levels.push_back(std::move(r));
  st.v_levels.push_back(std::move(u));  // level -1
  st.v_levels.push_back(std::move(v));  // level 0
  return st;
}

void level_iteration(IterationState& st, const LinearOperator& a, const DenseMatrix& p, std::size_t k,
                     SolveReport& rep) {
  const std::size_t n = a.size(), s = p.cols();
  if (st.r_levels.size() < k + 1 || st.v_levels.size() < k + 2) throw Error("level_iteration: missing levels");
  Session& ss = session();
  mstab_operator* op = device_operator(ss, a);
  const auto pp = dense_real(p, "P");
  auto x0 = real_parts(st.x0, "x0");
  std::vector<double> r((k + 2) * n), v((k + 3) * n * s);
  for (std::size_t i = 0; i <= k; ++i) {
    const auto ri = real_parts(st.r_levels[i], "residual level");
    std::copy(ri.begin(), ri.end(), r.begin() + (std::ptrdiff_t)(i * n));
  }
  for (std::size_t i = 0; i <= k + 1; ++i) {
    const auto vi = dense_real(st.v_levels[i], "auxiliary level");
    std::copy(vi.begin(), vi.end(), v.begin() + (std::ptrdiff_t)(i * n * s));
  }
  check(mstab_kernel_level_iteration(ss.ctx, op, (int64_t)s, (int64_t)k, pp.data(), x0.data(), r.data(), v.data()));
  for (std::size_t t = 0; t < n; ++t) st.x0[t] = Complex(x0[t]);
  st.r_levels.resize(k + 1);
  st.v_levels.resize(k + 2);
  for (std::size_t i = 0; i <= k; ++i)
    for (std::size_t t = 0; t < n; ++t) st.r_levels[i][t] = Complex(r[i * n + t]);
  Vector rnew(n);
  for (std::size_t t = 0; t < n; ++t) rnew[t] = Complex(r[(k + 1) * n + t]);
  st.r_levels.push_back(std::move(rnew));
  for (std::size_t i = 0; i <= k + 1; ++i) st.v_levels[i] = dense_from(v.data() + i * n * s, n, s);
  st.v_levels.push_back(dense_from(v.data() + (k + 2) * n * s, n, s));
  rep.h_mv += (std::int64_t)(s + 1);
}

PolyOut poly_combination(const IterationState& st, std::size_t ell) {
  const std::size_t n = st.x0.size();
  const std::size_t s = st.v_levels[0].cols();
  if (st.r_levels.size() < ell + 1 || st.v_levels.size() < ell + 2) throw Error("poly_combination: missing levels");
  Session& ss = session();
  const auto x0 = real_parts(st.x0, "x0");
  std::vector<double> r((ell + 1) * n), v((ell + 2) * n * s);
  for (std::size_t i = 0; i <= ell; ++i) {
    const auto ri = real_parts(st.r_levels[i], "residual level");
    std::copy(ri.begin(), ri.end(), r.begin() + (std::ptrdiff_t)(i * n));
  }
  for (std::size_t i = 0; i <= ell + 1; ++i) {
    const auto vi = dense_real(st.v_levels[i], "auxiliary level");
    std::copy(vi.begin(), vi.end(), v.begin() + (std::ptrdiff_t)(i * n * s));
  }
  std::vector<double> x(n), rr(n), u(n * s), vv(n * s), tau(ell);
  int32_t pert = 0;
  check(mstab_kernel_poly_combination(ss.ctx, (int64_t)n, (int64_t)s, (int64_t)ell, x0.data(), r.data(), v.data(),
                                      x.data(), rr.data(), u.data(), vv.data(), tau.data(), &pert));
  PolyOut out;
  out.x.resize(n);
  out.r.resize(n);
  for (std::size_t t = 0; t < n; ++t) {
    out.x[t] = Complex(x[t]);
    out.r[t] = Complex(rr[t]);
  }
  out.u = dense_from(u.data(), n, s);
  out.v = dense_from(vv.data(), n, s);
  for (std::size_t i = 0; i < ell; ++i) out.tau.emplace_back(tau[i]);
  out.tail_perturbed = pert != 0;
  return out;
}

}  // namespace mstab
