// bsfv_perf.hpp -- header-only profiling and parallel-efficiency reporting
// with the reference's perf module interface (SPEC.md:384-450,
// proj/include/bsfv/perf.hpp), fed by the B200 library's CUDA-event timings.
//
//   TimerSet / profile_report / profile_csv / profile_table   Tables 1-3 format
//   efficiency (Eq. 1)  eps(N) = T_s / (N * T_p(N))
//   efficiency_based (Eq. 2)  eps(N) = T_p(M) / ((N/M) * T_p(N))
//   threshold_point / iso_efficiency_compare   acceptable-efficiency limit (sec. 5)
//   scaling_csv / format_double   CSV outputs (label,N,Tp,inv_Tp,eps), shortest
//                                 round-trip decimals: same records -> same bytes
//   add_gpu_profile   device time of the SIP routines of a sip_ctx (K2 forward
//                     incl. its edge-record build, K3 backward, K4 halo)
//
// Errors follow the reference: MisuseError for invalid records / baselines.
#pragma once

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "bsfv_sip.hpp"

namespace bsfv {
namespace b200 {

/// Accumulating wall-clock region timers of one rank; "self" excludes
/// enclosed child regions (perf.hpp:11-50).
class TimerSet {
 public:
  struct Rec {
    double self_s = 0.0;
    std::uint64_t calls = 0;
  };
  void enter(const std::string& name) { stack_.push_back(Frame{name, now_s(), 0.0}); }
  void exit() {
    if (stack_.empty()) throw MisuseError("TimerSet::exit without enter");
    const Frame f = stack_.back();
    stack_.pop_back();
    const double elapsed = now_s() - f.start;
    Rec& r = recs_[f.name];
    r.self_s += elapsed - f.child;
    r.calls += 1;
    if (!stack_.empty()) stack_.back().child += elapsed;
  }
  /// Adds an externally timed region (e.g. CUDA-event device time).
  void add(const std::string& name, double self_s, std::uint64_t calls) {
    Rec& r = recs_[name];
    r.self_s += self_s;
    r.calls += calls;
  }
  const std::map<std::string, Rec>& records() const { return recs_; }
  void clear() { recs_.clear(); }

  class Scope {
   public:
    Scope(TimerSet* ts, const std::string& name) : ts_(ts) {
      if (ts_) ts_->enter(name);
    }
    ~Scope() {
      if (ts_) ts_->exit();
    }
    Scope(const Scope&) = delete;
    Scope& operator=(const Scope&) = delete;

   private:
    TimerSet* ts_;
  };

 private:
  static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  struct Frame {
    std::string name;
    double start = 0.0;
    double child = 0.0;
  };
  std::map<std::string, Rec> recs_;
  std::vector<Frame> stack_;
};

struct ProfileEntry {
  std::string name;
  double self_s = 0.0;
  std::uint64_t calls = 0;
  double pct = 0.0;
};

/// Shortest round-trip decimal (std::to_chars), stable across runs.
inline std::string format_double(double v) {
  char buf[32];
  const auto res = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, res.ptr);
}

/// Per-rank timers -> profile: max self time over ranks, summed calls,
/// share of the total, sorted by self time (ties by name); optional top-N.
inline std::vector<ProfileEntry> profile_report(const std::vector<const TimerSet*>& per_rank,
                                                std::optional<std::size_t> top = std::nullopt) {
  // region name -> (max self seconds over ranks, summed calls); map order =
  // name order, which breaks self-time ties below
  std::map<std::string, std::pair<double, std::uint64_t>> merged;
  for (std::size_t r = 0; r < per_rank.size(); ++r) {
    if (per_rank[r] == nullptr) continue;
    for (const auto& rec : per_rank[r]->records()) {
      auto& slot = merged[rec.first];
      if (rec.second.self_s > slot.first) slot.first = rec.second.self_s;
      slot.second += rec.second.calls;
    }
  }
  double sum = 0.0;
  for (const auto& m : merged) sum += m.second.first;
  std::vector<ProfileEntry> rows;
  rows.reserve(merged.size());
  for (const auto& m : merged)
    rows.push_back({m.first, m.second.first, m.second.second,
                    sum > 0.0 ? 100.0 * m.second.first / sum : 0.0});
  std::stable_sort(rows.begin(), rows.end(), [](const ProfileEntry& x, const ProfileEntry& y) {
    return x.self_s > y.self_s;  // stable: equal times keep name order
  });
  if (top.has_value() && rows.size() > top.value()) rows.erase(rows.begin() + top.value(), rows.end());
  return rows;
}

inline std::string profile_csv(const std::vector<ProfileEntry>& entries) {
  std::string s = "name,self_s,calls,pct\n";
  for (const auto& e : entries)
    s += e.name + "," + format_double(e.self_s) + "," + std::to_string(e.calls) + "," +
         format_double(e.pct) + "\n";
  return s;
}

inline std::string profile_table(const std::vector<ProfileEntry>& entries) {
  std::string s = "time %   self [s]     calls  name\n";
  char buf[160];
  for (const auto& e : entries) {
    std::snprintf(buf, sizeof(buf), "%6.2f  %9.4f  %8llu  %s\n", e.pct, e.self_s,
                  static_cast<unsigned long long>(e.calls), e.name.c_str());
    s += buf;
  }
  return s;
}

struct ScalingRecord {
  std::string label;
  int n = 1;
  double tp = 0.0;  // seconds per step
};

struct EfficiencyEntry {
  std::string label;
  int n = 1;
  double tp = 0.0;
  double eps = 0.0;
};

struct EfficiencyReport {
  std::string baseline;
  double threshold = 0.5;
  std::vector<EfficiencyEntry> entries;
  /// Largest sampled N of `label` with eps >= threshold.
  std::optional<int> max_n_meeting(const std::string& label) const {
    std::optional<int> best;
    for (const auto& e : entries)
      if (e.label == label && e.eps >= threshold) best = best ? std::max(*best, e.n) : e.n;
    return best;
  }
};

/// Eq. (1).
inline EfficiencyReport efficiency(const std::vector<ScalingRecord>& records, double t_s,
                                   double threshold = 0.5) {
  if (records.empty()) throw MisuseError("efficiency: no records");
  if (!(t_s > 0.0)) throw MisuseError("efficiency: nonpositive baseline time");
  EfficiencyReport rep;
  rep.baseline = "single-rank T_s";
  rep.threshold = threshold;
  for (const auto& r : records) {
    if (!(r.tp > 0.0) || r.n < 1)
      throw MisuseError("efficiency: record " + r.label + " has invalid N=" + std::to_string(r.n) +
                        " or T_p");
    rep.entries.push_back({r.label, r.n, r.tp, t_s / (r.n * r.tp)});
  }
  return rep;
}

/// Eq. (2): M-rank baseline; every record's N must be divisible by M.
inline EfficiencyReport efficiency_based(const std::vector<ScalingRecord>& records, int m,
                                         double t_pm, double threshold = 0.5) {
  if (records.empty()) throw MisuseError("efficiency_based: no records");
  if (m < 1 || !(t_pm > 0.0)) throw MisuseError("efficiency_based: invalid baseline");
  EfficiencyReport rep;
  rep.baseline = "baseline of M=" + std::to_string(m) + " ranks";
  rep.threshold = threshold;
  for (const auto& r : records) {
    if (!(r.tp > 0.0)) throw MisuseError("efficiency_based: nonpositive T_p");
    if (r.n % m != 0)
      throw MisuseError("efficiency_based: record N=" + std::to_string(r.n) +
                        " not divisible by M=" + std::to_string(m));
    const double units = static_cast<double>(r.n) / m;
    rep.entries.push_back({r.label, r.n, r.tp, t_pm / (units * r.tp)});
  }
  return rep;
}

struct OperatingPoint {
  bool reached = false;
  double n = 0.0;
  double rate = 0.0;  // 1 / T_p
};

/// Largest N of one curve still meeting the threshold, linearly interpolated
/// toward the first sample below it, and the rate 1/T_p there.
inline OperatingPoint threshold_point(const std::vector<EfficiencyEntry>& curve, double threshold) {
  std::vector<EfficiencyEntry> byn(curve);
  std::stable_sort(byn.begin(), byn.end(),
                   [](const EfficiencyEntry& x, const EfficiencyEntry& y) { return x.n < y.n; });
  // the last sample (in N order) that still meets the threshold
  std::size_t hit = byn.size();
  for (std::size_t i = byn.size(); i-- > 0;)
    if (byn[i].eps >= threshold) {
      hit = i;
      break;
    }
  OperatingPoint op;
  if (hit == byn.size()) return op;  // never meets it
  op.reached = true;
  const EfficiencyEntry& lo = byn[hit];
  if (hit + 1 == byn.size()) {  // still meeting it at the largest sampled N
    op.n = lo.n;
    op.rate = 1.0 / lo.tp;
    return op;
  }
  const EfficiencyEntry& hi = byn[hit + 1];  // first sample below the threshold
  const double frac = (hi.eps == lo.eps) ? 0.0 : (threshold - lo.eps) / (hi.eps - lo.eps);
  const double rate_lo = 1.0 / lo.tp, rate_hi = 1.0 / hi.tp;
  op.n = lo.n + frac * (hi.n - lo.n);
  op.rate = rate_lo + frac * (rate_hi - rate_lo);
  return op;
}

struct IsoEfficiencyResult {
  bool comparable = false;
  OperatingPoint a, b;
  double speedup_b_over_a = 0.0;
  std::string note;
};

inline IsoEfficiencyResult iso_efficiency_compare(const std::vector<EfficiencyEntry>& curve_a,
                                                  const std::vector<EfficiencyEntry>& curve_b,
                                                  double threshold = 0.5) {
  IsoEfficiencyResult res;
  res.a = threshold_point(curve_a, threshold);
  res.b = threshold_point(curve_b, threshold);
  res.comparable = res.a.reached && res.b.reached;
  if (res.comparable) {
    res.speedup_b_over_a = res.b.rate / res.a.rate;
  } else {
    std::vector<std::string> missing;
    if (!res.a.reached) missing.push_back("first curve");
    if (!res.b.reached) missing.push_back("second curve");
    res.note = "below threshold at all N: " + missing[0];
    if (missing.size() == 2) res.note += " and " + missing[1];
  }
  return res;
}

inline std::string scaling_csv(const EfficiencyReport& report) {
  std::string s = "label,N,Tp,inv_Tp,eps\n";
  for (const auto& e : report.entries)
    s += e.label + "," + std::to_string(e.n) + "," + format_double(e.tp) + "," +
         format_double(1.0 / e.tp) + "," + format_double(e.eps) + "\n";
  return s;
}

/// Device time of the SIP routines of one context since sip_set_profiling(1)
/// (CUDA events on the launch stream) added to `ts` under the paper's routine
/// names; `iterations` = inner iterations run meanwhile (the call count).
inline void add_gpu_profile(TimerSet& ts, sip_ctx* ctx, std::uint64_t iterations) {
  double f = 0, b = 0, h = 0;
  long long launches = 0;
  check(::sip_get_profile(ctx, &f, &b, &h, &launches), ctx, "sip_get_profile");
  ts.add("resforward3d (K2)", f * 1e-3, iterations);
  ts.add("backward3d (K3)", b * 1e-3, iterations);
  if (h > 0.0) ts.add("halo exchange (K4)", h * 1e-3, iterations);
}

}  // namespace b200
}  // namespace bsfv
