// coinfer/offline_solvers.hpp — drop-in for the reference's offline solvers
// (/root/reference/proj/include/coinfer/offline_solvers.hpp) on the B200
// engine.
//
// Same namespace, types and signatures as the reference; every solver below
// runs in the engine's sm_100a kernels through the C ABI
// (include/coinfer_b200.h), which also builds and normalises the returned
// Schedule on the device.  The host side only validates shapes, packs the
// inputs, and maps status codes back onto the reference's exceptions and
// messages.  Results are bit-identical to the reference's (tests/).
//
//   batch_start_times, sum_latency        :18-47   (profile arithmetic, host)
//   detail::local_only_choice             :62-75   -> coinfer_best_partition(s = NULL)
//   best_partition                        :83-117  -> coinfer_best_partition
//   detail::try_fixed_batch               :137-188 -> coinfer_fixed_batch + coinfer_ipssa_schedule
//   detail::try_ip_ssa, ip_ssa            :192-224 -> coinfer_ipssa_batch + coinfer_ipssa_schedule
//   fixed_batch_schedule                  :208-214
//   groups_fit                            :229-232 (profile arithmetic, host)
//   GroupingPlan, og                      :234-388 -> coinfer_og_batch + coinfer_og_schedule
//   detail::subscenario, detail::lc_solve :245-276
//   BaselineMode, baseline                :390-612 -> coinfer_baseline_batch
//   ScheduleMetrics, schedule_metrics     :621-657 (evaluation of a given schedule, host)
//
// Batched entry points for many scenarios per launch live in
// coinfer::b200 (end of this file).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <limits>
#include <optional>
#include <stdexcept>
#include <utility>
#include <vector>

#include "b200.hpp"
#include "core_model.hpp"
#include "schedule.hpp"

namespace coinfer {

constexpr double kInf = std::numeric_limits<double>::infinity();

// s*_n: latest batch starts that run the pipeline back to back at batch
// size b and end at the deadline; infeasible if s*_1 < 0.
struct BatchStartTimes {
  std::vector<double> s;
  bool feasible = false;
};

inline BatchStartTimes batch_start_times(const DnnProfile& p, double deadline, std::size_t b) {
  if (b == 0) throw std::invalid_argument("batch_start_times: b must be >= 1");
  BatchStartTimes r;
  r.s.assign(p.subtasks(), 0.0);
  double t = deadline;
  for (std::size_t n = p.subtasks(); n >= 1; --n) {
    t -= edge_batch_latency(p, n, b);
    r.s[n - 1] = t;
  }
  r.feasible = r.s[0] >= 0.0;
  return r;
}

inline double sum_latency(const DnnProfile& p, std::size_t b) {
  double sum = 0.0;
  for (std::size_t n = 1; n <= p.subtasks(); ++n) sum += edge_batch_latency(p, n, b);
  return sum;
}

// split = number of leading sub-tasks run on the device; freq is NaN when
// none is.
struct PartitionChoice {
  std::size_t split = 0;
  double freq = std::numeric_limits<double>::quiet_NaN();
  double energy = kInf;
  bool feasible = false;
};

namespace detail {

inline PartitionChoice partition_query(const UserSpec& u, const DnnProfile& p, const double* s,
                                       double deadline) {
  b200::FlatProfile fp(p);
  coinfer_users q{};
  q.n_inst = 1;
  q.M = 1;
  q.mem = COINFER_MEM_HOST;
  q.f_min = &u.f_min;
  q.f_max = &u.f_max;
  q.kappa = &u.kappa;
  q.rate_up = &u.rate_up;
  q.power_up = &u.power_up;
  q.arrival = &u.arrival;
  q.deadline = &deadline;
  int32_t split = 0;
  double freq = 0.0, energy = 0.0;
  uint8_t feas = 0;
  b200::check_call(coinfer_best_partition(b200::context().get(), &fp.view, &q, s, &split, &freq,
                                          &energy, &feas));
  PartitionChoice c;
  c.split = (std::size_t)split;
  c.freq = freq;
  c.energy = energy;
  c.feasible = feas != 0;
  return c;
}

// All-local candidate against the user's own deadline (GPU).
inline PartitionChoice local_only_choice(const UserSpec& u, const DnnProfile& p, double deadline) {
  return partition_query(u, p, nullptr, deadline);
}

}  // namespace detail

// Minimum-energy split against fixed batch starts s (GPU).
inline PartitionChoice best_partition(const UserSpec& u, const DnnProfile& p,
                                      const std::vector<double>& s, double deadline) {
  if (s.size() != p.subtasks())
    throw std::invalid_argument("best_partition: need one start time per sub-task");
  return detail::partition_query(u, p, s.data(), deadline);
}

struct SolveResult {
  Schedule schedule;
  double energy = 0.0;
  std::vector<std::size_t> split;
  std::vector<std::size_t> batch_size;  // realized size per sub-task, index n-1
  bool pipeline_feasible = true;
  std::size_t batch_bound = 0;
};

inline bool groups_fit(double earlier_deadline, double later_deadline, const DnnProfile& p,
                       std::size_t later_size) {
  return earlier_deadline + sum_latency(p, later_size) <= later_deadline;
}

struct GroupingPlan {
  std::vector<std::vector<std::size_t>> groups;  // original ids, by rising deadline
  std::vector<double> group_deadline;
  std::vector<double> group_energy;
  double energy = 0.0;
  Schedule schedule;
  bool fallback = false;
};

enum class BaselineMode { LC, PS, FIFO, IPSSA_NP };

struct ScheduleMetrics {
  double total_energy = 0.0;
  std::vector<double> per_user_energy;
  std::vector<double> mean_batch_size;  // per sub-task; 0 when never offloaded
};

namespace b200 {

// Shape checks the flat ABI cannot express, in Scenario::check's order: the
// profile, then one deadline per user.  The per-user contract (and the
// table length) is checked by the kernels, in the same order.
inline void check_shapes(const Scenario& sc) {
  sc.profile.check();
  if (sc.deadline.size() != sc.users.size())
    throw std::invalid_argument("scenario: one deadline per user required");
}

// All scenarios of a batch share one profile and one user count.
inline void check_batch(const std::vector<Scenario>& scs) {
  for (const Scenario& s : scs) check_shapes(s);
  for (const Scenario& s : scs) {
    const DnnProfile& p = s.profile;
    const DnnProfile& q = scs[0].profile;
    if (s.n_users() != scs[0].n_users() || p.work != q.work || p.data_bits != q.data_bits ||
        p.latency != q.latency)
      throw std::invalid_argument("coinfer::b200: a batch needs one profile and one user count");
  }
}

inline std::vector<const Scenario*> ptrs(const std::vector<Scenario>& scs) {
  std::vector<const Scenario*> v;
  for (const Scenario& s : scs) v.push_back(&s);
  return v;
}

inline SolveResult take_result(const SolveBuffers& b, const ScheduleBuffers& sb, std::size_t k,
                               std::size_t M, std::size_t N) {
  SolveResult r;
  r.energy = b.energy[k];
  r.pipeline_feasible = b.pipe[k] != 0;
  r.batch_bound = (std::size_t)b.batch_bound[k];
  r.split.assign(M, 0);
  for (std::size_t m = 0; m < M; ++m) r.split[m] = b.split[k * M + m];
  r.batch_size.assign(N, 0);
  for (std::size_t n = 0; n < N; ++n) r.batch_size[n] = (std::size_t)b.batch_size[k * N + n];
  r.schedule = sb.take(k);
  return r;
}

// IP-SSA (bounds == nullptr) or Alg. 1 at bound bounds[k] for every
// scenario, statuses left to the caller.
inline std::vector<int32_t> solve_raw(const std::vector<const Scenario*>& scs,
                                      const std::vector<double>& deadline,
                                      const std::vector<int32_t>* bounds,
                                      std::vector<SolveResult>& out) {
  const std::size_t K = scs.size();
  out.clear();
  if (K == 0) return {};
  const std::size_t M = scs[0]->n_users(), N = scs[0]->profile.subtasks();
  FlatProfile fp(scs[0]->profile);
  UserBatch ub(scs.data(), K, M);
  SolveBuffers sb(K, M, N);
  ScheduleBuffers sch(K, M, N);
  coinfer_ctx* ctx = context().get();
  if (bounds)
    check_call(coinfer_fixed_batch(ctx, &fp.view, &ub.view, deadline.data(), bounds->data(), &sb.out));
  else
    check_call(coinfer_ipssa_batch(ctx, &fp.view, &ub.view, deadline.data(), &sb.out));
  check_call(coinfer_ipssa_schedule(ctx, &fp.view, &ub.view, deadline.data(), &sb.out, &sch.out));
  for (std::size_t k = 0; k < K; ++k)
    out.push_back(sb.status[k] == COINFER_ST_OK ? take_result(sb, sch, k, M, N) : SolveResult{});
  return sb.status;
}

inline std::vector<int32_t> og_raw(const std::vector<const Scenario*>& scs,
                                   std::vector<GroupingPlan>& out) {
  const std::size_t K = scs.size();
  out.clear();
  if (K == 0) return {};
  const std::size_t M = scs[0]->n_users(), N = scs[0]->profile.subtasks();
  FlatProfile fp(scs[0]->profile);
  UserBatch ub(scs.data(), K, M);
  OgBuffers ob(K, M, N);
  ScheduleBuffers sch(K, M, N);
  coinfer_ctx* ctx = context().get();
  check_call(coinfer_og_batch(ctx, &fp.view, &ub.view, &ob.out));
  check_call(coinfer_og_schedule(ctx, &fp.view, &ub.view, &ob.out, &sch.out));
  for (std::size_t k = 0; k < K; ++k) {
    GroupingPlan plan;
    if (ob.status[k] == COINFER_ST_OK) {
      const std::size_t G = (std::size_t)ob.n_groups[k];
      for (std::size_t g = 0; g < G; ++g) {
        const std::size_t gi = k * M + g;
        std::vector<std::size_t> ids;
        for (int32_t q = ob.group_lo[gi]; q < ob.group_lo[gi] + ob.group_size[gi]; ++q)
          ids.push_back((std::size_t)ob.order[k * M + q]);
        plan.groups.push_back(std::move(ids));
        plan.group_deadline.push_back(ob.group_deadline[gi]);
        plan.group_energy.push_back(ob.group_energy[gi]);
      }
      plan.energy = ob.energy[k];
      plan.fallback = ob.fallback[k] != 0;
      plan.schedule = sch.take(k);
    }
    out.push_back(std::move(plan));
  }
  return ob.status;
}

inline std::vector<int32_t> baseline_raw(const std::vector<const Scenario*>& scs, BaselineMode mode,
                                         std::vector<SolveResult>& out) {
  const std::size_t K = scs.size();
  out.clear();
  if (K == 0) return {};
  const std::size_t M = scs[0]->n_users(), N = scs[0]->profile.subtasks();
  FlatProfile fp(scs[0]->profile);
  UserBatch ub(scs.data(), K, M);
  SolveBuffers sb(K, M, N);
  ScheduleBuffers sch(K, M, N);
  check_call(coinfer_baseline_batch(context().get(), &fp.view, &ub.view, (int32_t)mode, &sb.out,
                                    &sch.out));
  for (std::size_t k = 0; k < K; ++k)
    out.push_back(sb.status[k] == COINFER_ST_OK ? take_result(sb, sch, k, M, N) : SolveResult{});
  return sb.status;
}

inline const char* baseline_solver_name(BaselineMode mode) {
  switch (mode) {
    case BaselineMode::LC: return "lc";
    case BaselineMode::PS: return "ps";
    case BaselineMode::FIFO: return "fifo";
    case BaselineMode::IPSSA_NP: return "np";
  }
  return "np";
}

// An empty scenario: nothing to launch (the reference returns the same
// default-constructed results structurally).
inline SolveResult empty_baseline(const Scenario& sc) {
  SolveResult r;
  r.batch_size.assign(sc.profile.subtasks(), 0);
  return r;
}

}  // namespace b200

namespace detail {

inline std::optional<SolveResult> try_fixed_batch(const Scenario& sc, double deadline,
                                                  std::size_t b) {
  b200::check_shapes(sc);
  if (b == 0) throw std::invalid_argument("batch_start_times: b must be >= 1");
  if (b > sc.profile.max_batch())
    throw std::out_of_range("edge_batch_latency: batch size beyond table");
  if (sc.n_users() == 0) {  // nothing to place: the pipeline alone decides
    SolveResult r;
    r.batch_bound = b;
    r.pipeline_feasible = batch_start_times(sc.profile, deadline, b).feasible;
    r.batch_size.assign(sc.profile.subtasks(), 0);
    return r;
  }
  std::vector<SolveResult> out;
  const std::vector<int32_t> bv(1, (int32_t)b);
  const std::vector<int32_t> st = b200::solve_raw({&sc}, {deadline}, &bv, out);
  if (st[0] == COINFER_ST_INFEASIBLE) return std::nullopt;
  b200::check_status(st[0], "fixed");
  return std::move(out[0]);
}

inline std::optional<SolveResult> try_ip_ssa(const Scenario& sc, double deadline) {
  b200::check_shapes(sc);
  if (sc.n_users() == 0) return SolveResult{};
  std::vector<SolveResult> out;
  const std::vector<int32_t> st = b200::solve_raw({&sc}, {deadline}, nullptr, out);
  if (st[0] == COINFER_ST_INFEASIBLE) return std::nullopt;
  b200::check_status(st[0], "ipssa");
  return std::move(out[0]);
}

inline Scenario subscenario(const Scenario& sc, const std::vector<std::size_t>& ids) {
  Scenario sub;
  sub.profile = sc.profile;
  sub.users.reserve(ids.size());
  sub.deadline.reserve(ids.size());
  for (std::size_t id : ids) {
    sub.users.push_back(sc.users[id]);
    sub.deadline.push_back(sc.deadline[id]);
  }
  return sub;
}

inline SolveResult lc_solve(const Scenario& sc) {
  b200::check_shapes(sc);
  if (sc.n_users() == 0) return b200::empty_baseline(sc);
  std::vector<SolveResult> out;
  const std::vector<int32_t> st = b200::baseline_raw({&sc}, BaselineMode::LC, out);
  b200::check_status(st[0], "lc");
  return std::move(out[0]);
}

}  // namespace detail

inline SolveResult fixed_batch_schedule(const Scenario& sc, double deadline, std::size_t b) {
  sc.check();
  std::optional<SolveResult> r = detail::try_fixed_batch(sc, deadline, b);
  if (!r) throw std::domain_error("fixed_batch_schedule: user cannot meet the deadline");
  return std::move(*r);
}

inline SolveResult ip_ssa(const Scenario& sc, double deadline) {
  b200::check_shapes(sc);
  if (sc.n_users() == 0) return SolveResult{};
  std::vector<SolveResult> out;
  const std::vector<int32_t> st = b200::solve_raw({&sc}, {deadline}, nullptr, out);
  b200::check_status(st[0], "ipssa");
  return std::move(out[0]);
}

inline GroupingPlan og(const Scenario& sc) {
  b200::check_shapes(sc);
  if (sc.n_users() == 0) return GroupingPlan{};
  std::vector<GroupingPlan> out;
  const std::vector<int32_t> st = b200::og_raw({&sc}, out);
  b200::check_status(st[0], "og");
  return std::move(out[0]);
}

inline SolveResult baseline(const Scenario& sc, BaselineMode mode) {
  b200::check_shapes(sc);
  if (sc.n_users() == 0) return b200::empty_baseline(sc);
  std::vector<SolveResult> out;
  const std::vector<int32_t> st = b200::baseline_raw({&sc}, mode, out);
  b200::check_status(st[0], b200::baseline_solver_name(mode));
  return std::move(out[0]);
}

// Per-user energies in total_energy's term order, plus the mean size of the
// batches of every sub-task (an evaluation of a given schedule).
inline ScheduleMetrics schedule_metrics(const Schedule& s, const Scenario& sc) {
  check_shapes(s, sc);
  const DnnProfile& p = sc.profile;
  const std::size_t N = p.subtasks();
  ScheduleMetrics out;
  out.per_user_energy.assign(sc.n_users(), 0.0);
  for (std::size_t m = 0; m < sc.n_users(); ++m) {
    const UserSpec& u = sc.users[m];
    double e = 0.0;
    for (std::size_t n = 1; n <= N; ++n)
      if (s.x[m][n - 1] == kLocal) e += local_energy(u.kappa, p.work[n - 1], s.freq[m]);
    for (std::size_t n = 0; n < N; ++n) {
      if (upload_needed(s, m, n)) e += link_cost(p.data_bits[n], u.rate_up, u.power_up).energy;
      if (download_needed(s, m, n)) e += link_cost(p.data_bits[n], u.rate_down, u.power_down).energy;
    }
    out.per_user_energy[m] = e;
    out.total_energy += e;
  }
  std::vector<std::size_t> copies(N, 0), count(N, 0);
  for (const BatchView& v : batch_views(s)) {
    if (v.members.empty()) continue;
    copies[v.subtask - 1] += v.size();
    count[v.subtask - 1] += 1;
  }
  for (std::size_t n = 0; n < N; ++n)
    out.mean_batch_size.push_back(count[n] == 0 ? 0.0 : double(copies[n]) / double(count[n]));
  return out;
}

// ----------------------------------------------------------------------
// Batched API: one launch for many scenarios with one profile and one user
// count (the offline Monte Carlo sweep).  Each entry is what the
// single-scenario call returns; an instance that would throw is reported by
// its status (COINFER_ST_*, message via coinfer_status_message) and a
// default-constructed result, so one bad draw does not abort the batch.
namespace b200 {

template <class R>
struct Batch {
  std::vector<R> results;
  std::vector<int32_t> status;
};

inline Batch<SolveResult> ip_ssa(const std::vector<Scenario>& scs,
                                 const std::vector<double>& deadline) {
  check_batch(scs);
  if (deadline.size() != scs.size())
    throw std::invalid_argument("coinfer::b200::ip_ssa: one deadline per scenario");
  Batch<SolveResult> b;
  if (!scs.empty() && scs[0].n_users() == 0) {
    b.results.assign(scs.size(), SolveResult{});
    b.status.assign(scs.size(), COINFER_ST_OK);
    return b;
  }
  b.status = solve_raw(ptrs(scs), deadline, nullptr, b.results);
  return b;
}

inline Batch<GroupingPlan> og(const std::vector<Scenario>& scs) {
  check_batch(scs);
  Batch<GroupingPlan> b;
  if (!scs.empty() && scs[0].n_users() == 0) {
    b.results.assign(scs.size(), GroupingPlan{});
    b.status.assign(scs.size(), COINFER_ST_OK);
    return b;
  }
  b.status = og_raw(ptrs(scs), b.results);
  return b;
}

inline Batch<SolveResult> baseline(const std::vector<Scenario>& scs, BaselineMode mode) {
  check_batch(scs);
  Batch<SolveResult> b;
  if (!scs.empty() && scs[0].n_users() == 0) {
    b.results.assign(scs.size(), empty_baseline(scs[0]));
    b.status.assign(scs.size(), COINFER_ST_OK);
    return b;
  }
  b.status = baseline_raw(ptrs(scs), mode, b.results);
  return b;
}

}  // namespace b200

}  // namespace coinfer
