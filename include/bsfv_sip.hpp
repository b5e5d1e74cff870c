// bsfv_sip.hpp -- header-only C++ shim that gives the reference's sip module
// interface on top of the B200 C-ABI (sip_c.h).
//
// Drop-in use from the reference code base (proj/):
//
//   #include "bsfv/error.hpp"      // optional: throw the reference's own classes
//   #include "bsfv/field.hpp"
//   #define BSFV_SIP_USE_REFERENCE_ERRORS 1
//   #include "bsfv_sip.hpp"
//
//   bsfv::b200::StencilSystemT<bsfv::FieldD> A{...};  // Field3<double> members
//   ... fill A.ap, A.aw, ..., A.q ...
//   bsfv::b200::SipConfig cfg;                     // alpha 0.92, max_iters, target
//   auto F = bsfv::b200::sip_factor(A, cfg);       // SingularFactorError names the cell
//   auto [fi, report] = bsfv::b200::solve(A, fi0, cfg, &F);
//
// The field type is a template parameter: anything with nx()/ny()/nz() and
// data() over (nx+2)(ny+2)(nz+2) doubles in Field3 order
// (proj/include/bsfv/field.hpp:21-44) works, including bsfv::FieldD itself.
//
// Error mapping (proj/include/bsfv/error.hpp:34-50):
//   SIP_ERR_SINGULAR -> SingularFactorError, SIP_ERR_STALE -> StaleFactorsError,
//   SIP_ERR_MISUSE -> MisuseError, SIP_ERR_CONFIG -> ConfigError,
//   SIP_ERR_NOCONV -> NonConvergenceError (PressureSolver), else Error.
//
// The caller of the SIP: PressureSolver assembles
// the pressure-correction Laplacian on a block lattice, factors it once and
// runs pressure_correct steps on a device-resident flow state.
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sip_c.h"

namespace bsfv {
namespace b200 {

#if defined(BSFV_SIP_USE_REFERENCE_ERRORS) && BSFV_SIP_USE_REFERENCE_ERRORS
using Error = ::bsfv::Error;
using ConfigError = ::bsfv::ConfigError;
using SingularFactorError = ::bsfv::SingularFactorError;
using StaleFactorsError = ::bsfv::StaleFactorsError;
using MisuseError = ::bsfv::MisuseError;
using FormatError = ::bsfv::FormatError;
using ProtocolError = ::bsfv::ProtocolError;
using NonConvergenceError = ::bsfv::NonConvergenceError;
#else
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
class ConfigError : public Error {
 public:
  explicit ConfigError(const std::string& w) : Error(w) {}
};
class SingularFactorError : public Error {
 public:
  explicit SingularFactorError(const std::string& w) : Error(w) {}
};
class StaleFactorsError : public Error {
 public:
  explicit StaleFactorsError(const std::string& w) : Error(w) {}
};
class MisuseError : public Error {
 public:
  explicit MisuseError(const std::string& w) : Error(w) {}
};
class FormatError : public Error {  // error.hpp:22-31: the message carries the offset
 public:
  FormatError(const std::string& w, std::size_t offset)
      : Error(w + " (at byte offset " + std::to_string(offset) + ")"), offset_(offset) {}
  std::size_t offset() const { return offset_; }

 private:
  std::size_t offset_;
};
class ProtocolError : public Error {
 public:
  explicit ProtocolError(const std::string& w) : Error(w) {}
};
class NonConvergenceError : public Error {  // error.hpp:72-80: carries the defect
 public:
  NonConvergenceError(const std::string& w, double defect) : Error(w), defect_(defect) {}
  double defect() const { return defect_; }

 private:
  double defect_;
};
#endif

inline void check(int status, const sip_ctx* ctx, const char* what) {
  if (status == SIP_OK) return;
  const std::string msg = std::string(what) + ": " + ::sip_status_string(status) + ": " +
                          ::sip_last_error(ctx);
  switch (status) {
    case SIP_ERR_SINGULAR: throw SingularFactorError(msg);
    case SIP_ERR_STALE: throw StaleFactorsError(msg);
    case SIP_ERR_MISUSE: throw MisuseError(msg);
    case SIP_ERR_CONFIG: throw ConfigError(msg);
    case SIP_ERR_PROTOCOL: throw ProtocolError(::sip_last_error(ctx));
    default: throw Error(msg);
  }
}

/// SPEC.md:124-127
struct SipConfig {
  double alpha = 0.92;
  int max_iters = 50;
  double target = 0.0;  // <= 0: fixed iteration count
  bool single_precision = false;
  int check_every = 8;  // target mode: norm-evaluation interval (sip_solve_ex)
};

/// iterations used, initial / final norms, per-iteration
/// history, wall time in factorisation vs relaxation (host clock around the
/// library calls; both calls synchronise before returning).
struct SolveReport {
  int iterations = 0;
  std::vector<double> norms;
  double factor_seconds = 0.0;  // 0 on the reuse path (no factorisation)
  double relax_seconds = 0.0;   // su / fi0 upload, sweeps, fi and norms download
  double initial() const { return norms.empty() ? 0.0 : norms.front(); }
  double final_norm() const { return norms.empty() ? 0.0 : norms.back(); }
};

/// StencilSystem over any Field3-compatible type; matrix
/// entries (A_nb = -a_nb).
template <class Field>
struct StencilSystemT {
  Field ap, aw, ae, as, an, ab, at, q;
  long long revision = 0;  // bump after editing the coefficients
  bool symmetric = false;  // ae(i) = aw(i+1), an(j) = as(j+1), at(k) = ab(k+1)
};

/// SipFactors: a device context holding the factors,
/// stamped with the revision they were computed from.
class SipFactors {
 public:
  SipFactors() = default;
  SipFactors(sip_ctx* ctx, long long stamp, bool single) : ctx_(ctx), stamp_(stamp), single_(single) {}
  SipFactors(const SipFactors&) = delete;
  SipFactors& operator=(const SipFactors&) = delete;
  SipFactors(SipFactors&& o) noexcept { *this = std::move(o); }
  SipFactors& operator=(SipFactors&& o) noexcept {
    std::swap(ctx_, o.ctx_);
    stamp_ = o.stamp_;
    single_ = o.single_;
    return *this;
  }
  ~SipFactors() {
    if (ctx_) ::sip_destroy(ctx_);
  }
  sip_ctx* ctx() const { return ctx_; }
  long long stamp() const { return stamp_; }
  /// Library-side factorisation counter of the context.
  long long factorizations() const { return ctx_ ? ::sip_factor_count(ctx_) : 0; }
  bool single_precision() const { return single_; }

 private:
  sip_ctx* ctx_ = nullptr;
  long long stamp_ = -1;
  bool single_ = false;
};

/// sip_factor
template <class Field>
SipFactors sip_factor(const StencilSystemT<Field>& A, const SipConfig& cfg, int device = 0) {
  sip_ctx* ctx = nullptr;
  check(::sip_create(device, A.ap.nx(), A.ap.ny(), A.ap.nz(),
                     cfg.single_precision ? SIP_PREC_SINGLE : SIP_PREC_DOUBLE, &ctx),
        nullptr, "sip_create");
  SipFactors F(ctx, A.revision, cfg.single_precision);  // owns ctx from here on
  check(::sip_set_system(ctx, 0, A.ap.data(), A.aw.data(), A.ae.data(), A.as.data(), A.an.data(),
                         A.ab.data(), A.at.data(), A.q.data()),
        ctx, "sip_set_system");
  long long bb = -1, bc = -1;
  check(::sip_factor(ctx, cfg.alpha, &bb, &bc), ctx, "sip_factor");
  return F;
}

/// solve on the reuse path (factors given) or with one
/// factorisation at entry.  Returns (fi, report).
template <class Field>
std::pair<Field, SolveReport> solve(const StencilSystemT<Field>& A, const Field& fi0,
                                    const SipConfig& cfg, SipFactors* F = nullptr,
                                    int device = 0) {
  using clock = std::chrono::steady_clock;
  SipFactors own;
  double t_factor = 0.0;
  if (!F) {
    const auto t0 = clock::now();
    own = sip_factor(A, cfg, device);
    t_factor = std::chrono::duration<double>(clock::now() - t0).count();
    F = &own;
  } else if (F->stamp() != A.revision) {
    throw StaleFactorsError("solve: factors stamped with revision " + std::to_string(F->stamp()) +
                            " used against system revision " + std::to_string(A.revision));
  } else if (F->single_precision() != cfg.single_precision) {
    throw MisuseError("solve: factors were computed for another precision");
  }
  Field fi = fi0;
  SolveReport rep;
  rep.factor_seconds = t_factor;
  if (cfg.target >= 1.0) return {fi, rep};
  const auto t0 = clock::now();
  check(::sip_set_source(F->ctx(), 0, A.q.data()), F->ctx(), "sip_set_source");
  rep.norms.assign(static_cast<size_t>(cfg.max_iters), 0.0);
  double* phis[1] = {fi.data()};
  int used = 0;
  check(::sip_solve_ex(F->ctx(), phis, cfg.max_iters, cfg.target, cfg.check_every, rep.norms.data(),
                       &used),
        F->ctx(), "sip_solve");
  rep.relax_seconds = std::chrono::duration<double>(clock::now() - t0).count();
  rep.norms.resize(static_cast<size_t>(used));
  rep.iterations = used;
  return {fi, rep};
}

/// residual_general / residual_symmetric
/// of fi on the device; returns a Field of the same shape (interior written).
/// residual_symmetric throws MisuseError unless A.symmetric, ConfigError if
/// the coefficients contradict the flag.
template <class Field>
Field residual(const StencilSystemT<Field>& A, const Field& fi, bool symmetric, int device = 0) {
  if (symmetric && !A.symmetric)
    throw MisuseError("residual_symmetric: system not flagged symmetric");
  sip_ctx* ctx = nullptr;
  check(::sip_create(device, A.ap.nx(), A.ap.ny(), A.ap.nz(), SIP_PREC_DOUBLE, &ctx), nullptr,
        "sip_create");
  SipFactors holder(ctx, A.revision, false);  // owns ctx
  check(::sip_set_system(ctx, 0, A.ap.data(), A.aw.data(), A.ae.data(), A.as.data(), A.an.data(),
                         A.ab.data(), A.at.data(), A.q.data()),
        ctx, "sip_set_system");
  if (symmetric) check(::sip_set_symmetric(ctx, 0, 1), ctx, "sip_set_symmetric");
  const double* in[1] = {fi.data()};
  check(::sip_load_phi(ctx, const_cast<double* const*>(in)), ctx, "sip_load_phi");
  Field res = fi;
  double* out[1] = {res.data()};
  check(::sip_residual(ctx, symmetric ? 1 : 0, out), ctx, "sip_residual");
  return res;
}
template <class Field>
Field residual_general(const StencilSystemT<Field>& A, const Field& fi, int device = 0) {
  return residual(A, fi, false, device);
}
template <class Field>
Field residual_symmetric(const StencilSystemT<Field>& A, const Field& fi, int device = 0) {
  return residual(A, fi, true, device);
}

/// FTT1 transfer tables (tables.hpp:57-71): one vector of int[12] rows per rank
/// (dir, kind, face, peer, owner, neighbor, ilo, ihi, jlo, jhi, klo, khi).
using TableRows = std::vector<std::vector<std::array<int, 12>>>;

inline TableRows read_tables(const std::vector<unsigned char>& image) {
  int nranks = 0;
  long long total = 0, off = -1;
  auto fail = [&](int st) {
    if (st == SIP_ERR_FORMAT) {
      // sip_last_error carries " (at byte offset N)"; rebuild the typed error
      std::string m = ::sip_last_error(nullptr);
      const auto cut = m.rfind(" (at byte offset ");
      throw FormatError(cut == std::string::npos ? m : m.substr(0, cut), (std::size_t)off);
    }
    check(st, nullptr, "sip_ftt1_read");
  };
  int st = ::sip_ftt1_read(image.data(), image.size(), &nranks, nullptr, nullptr, 0, &total, &off);
  if (st != SIP_OK) fail(st);
  std::vector<int> counts((std::size_t)std::max(1, nranks)), rows((std::size_t)std::max(1LL, total) * 12);
  st = ::sip_ftt1_read(image.data(), image.size(), &nranks, counts.data(), rows.data(), total, &total,
                       &off);
  if (st != SIP_OK) fail(st);
  TableRows t((std::size_t)nranks);
  std::size_t at = 0;
  for (int r = 0; r < nranks; ++r)
    for (int k = 0; k < counts[r]; ++k, ++at) {
      std::array<int, 12> row;
      for (int f = 0; f < 12; ++f) row[f] = rows[at * 12 + f];
      t[r].push_back(row);
    }
  return t;
}

inline void flatten_tables(const TableRows& t, std::vector<int>& counts, std::vector<int>& rows) {
  counts.clear();
  rows.clear();
  for (const auto& r : t) {
    counts.push_back((int)r.size());
    for (const auto& e : r) rows.insert(rows.end(), e.begin(), e.end());
  }
}

inline std::vector<unsigned char> write_tables(const TableRows& t) {
  std::vector<int> counts, rows;
  flatten_tables(t, counts, rows);
  std::size_t len = 0;
  check(::sip_ftt1_write((int)t.size(), counts.data(), rows.data(), nullptr, 0, &len), nullptr,
        "sip_ftt1_write");
  std::vector<unsigned char> out(len);
  check(::sip_ftt1_write((int)t.size(), counts.data(), rows.data(), out.data(), len, &len), nullptr,
        "sip_ftt1_write");
  return out;
}

/// tables.cpp:185-235: throws ProtocolError on an unmatched / orphan entry.
inline void validate_matching(const TableRows& t) {
  std::vector<int> counts, rows;
  flatten_tables(t, counts, rows);
  check(::sip_ftt1_validate((int)t.size(), counts.data(), rows.data()), nullptr, "sip_ftt1_validate");
}

/// sip_sweep: one inner iteration in place, returns the L1 norm.
template <class Field>
double sip_sweep(const StencilSystemT<Field>& A, SipFactors& F, Field& fi) {
  if (F.stamp() != A.revision) throw StaleFactorsError("sip_sweep: stale factors");
  check(::sip_set_source(F.ctx(), 0, A.q.data()), F.ctx(), "sip_set_source");
  double norm = 0.0;
  int used = 0;
  double* phis[1] = {fi.data()};
  check(::sip_solve(F.ctx(), phis, 1, 0.0, &norm, &used), F.ctx(), "sip_solve");
  return norm;
}

/// Boundary kind per domain face (GridSpec bc), order W,E,S,N,B,T.
enum class Bc { Wall = SIP_BC_WALL, Periodic = SIP_BC_PERIODIC, Symmetry = SIP_BC_SYMMETRY };

/// Result of one pressure_correct call: outer iterations run and the
/// divergence L1 before each mass check.
struct CorrectionReport {
  int outer = 0;
  std::vector<double> divergence;
};

/// assemble_poisson + sip_factor + pressure_correct with factor reuse
/// (SPEC.md:134-142, 341-349): one device context over a block lattice of one
/// rank, the pressure system assembled and factored once at construction,
/// FlowState (u, v, w, p) resident on the device.  factorizations() is the
/// work-avoidance counter: it stays 1 for the object's life.
class PressureSolver {
 public:
  PressureSolver(std::array<int, 3> cells, std::array<int, 3> blocks, std::array<double, 3> lengths,
                 std::array<Bc, 6> bc, const SipConfig& cfg = SipConfig(), int device = 0) {
    check(::sip_create_lattice(device, cells[0], cells[1], cells[2], blocks[0], blocks[1], blocks[2],
                               nullptr, 0, 1, nullptr,
                               cfg.single_precision ? SIP_PREC_SINGLE : SIP_PREC_DOUBLE, &ctx_),
          nullptr, "sip_create_lattice");
    try {
      int b[6];
      for (int f = 0; f < 6; ++f) b[f] = static_cast<int>(bc[f]);
      check(::sip_assemble_poisson(ctx_, lengths.data(), b), ctx_, "assemble_poisson");
      long long bb = -1, bcell = -1;
      check(::sip_factor(ctx_, cfg.alpha, &bb, &bcell), ctx_, "sip_factor");
      ++factorizations_;
      check(::sip_flow_create(ctx_, &flow_), ctx_, "sip_flow_create");
      int n = 0;
      ::sip_num_local_blocks(ctx_, &n);
      for (int lb = 0; lb < n; ++lb) {
        std::array<int, 3> d{}, o{};
        int id = 0;
        ::sip_local_block(ctx_, lb, &id, d.data(), o.data());
        dims_.push_back(d);
      }
    } catch (...) {
      release();
      throw;
    }
  }
  PressureSolver(const PressureSolver&) = delete;
  PressureSolver& operator=(const PressureSolver&) = delete;
  ~PressureSolver() { release(); }

  int num_blocks() const { return static_cast<int>(dims_.size()); }
  std::array<int, 3> block_dims(int b) const { return dims_.at(static_cast<std::size_t>(b)); }
  long long factorizations() const { return factorizations_; }

  /// field: SIP_FLOW_U .. SIP_FLOW_P; one Field3 array per local block.
  void set(int field, const std::vector<const double*>& per_block) {
    std::vector<double*> p(per_block.size());
    for (std::size_t b = 0; b < p.size(); ++b) p[b] = const_cast<double*>(per_block[b]);
    check(::sip_flow_set(flow_, field, p.data()), ctx_, "sip_flow_set");
  }
  void get(int field, const std::vector<double*>& per_block) {
    check(::sip_flow_get(flow_, field, per_block.data()), ctx_, "sip_flow_get");
  }
  double divergence() {
    double d = 0.0;
    check(::sip_flow_divergence(flow_, &d), ctx_, "sip_flow_divergence");
    return d;
  }
  /// pressure_correct; NonConvergenceError carries the defect.
  CorrectionReport pressure_correct(double dt, double threshold, int max_outer, int sweeps = 5) {
    CorrectionReport r;
    r.divergence.assign(static_cast<std::size_t>(max_outer) + 1, 0.0);
    const int st = ::sip_pressure_correct(flow_, dt, threshold, max_outer, sweeps, &r.outer,
                                          r.divergence.data());
    r.divergence.resize(static_cast<std::size_t>(r.outer) + 1);
    if (st == SIP_ERR_NOCONV) throw NonConvergenceError(::sip_last_error(ctx_), r.divergence.back());
    check(st, ctx_, "pressure_correct");
    return r;
  }

 private:
  void release() {
    if (flow_) ::sip_flow_destroy(flow_);
    if (ctx_) ::sip_destroy(ctx_);
    flow_ = nullptr;
    ctx_ = nullptr;
  }
  sip_ctx* ctx_ = nullptr;
  sip_flow* flow_ = nullptr;
  long long factorizations_ = 0;
  std::vector<std::array<int, 3>> dims_;
};

}  // namespace b200
}  // namespace bsfv
