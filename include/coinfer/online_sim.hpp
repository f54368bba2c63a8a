// coinfer/online_sim.hpp — drop-in for the reference's online slot simulator
// (/root/reference/proj/include/coinfer/online_sim.hpp), on the B200 engine.
//
//   ArrivalModel (+check)                 online_sim.hpp:26-41
//   MdpState, ActionVec, OnlineSolver     :43-53
//   StepInfo                              :55-65
//   OnlineEnv (ctor checks, reset,        :69-261
//     load_state, step, invoke_solver,
//     process_all_local, sample_arrivals)
//   TraceRow, EpisodeMetrics              :263-296
//   PolicyFn, local_policy                :298-307
//   TimeWindowPolicy                      :309-336
//   run_episode (both overloads)          :338-371
//   write_trace_csv, write_episode_summary :373-400
//
// Two execution paths, identical results:
//   * run_episode(env, policy, horizon) with the fixed policies
//     (TimeWindowPolicy, local_policy) runs the WHOLE episode on the GPU in
//     one coinfer_online_run call (one warp; the per-slot OG / IP-SSA solves
//     happen on the device) and then leaves `env` in exactly the state the
//     reference's slot loop would: pending deadlines, expiries, edge_busy,
//     time, and the mt19937_64 stream position (seed + discard(draws)).
//   * OnlineEnv::step (and run_episode with any other policy) advances one
//     slot on the host; the solver call of a slot is coinfer::og /
//     coinfer::ip_ssa, i.e. the GPU engine through the C ABI.
// Arrivals use std::mt19937_64 + std::uniform_real_distribution from the
// host's libstdc++, the same generator the reference draws from (the device
// kernels reproduce that stream bit for bit; tests/golden/online*.json pins
// it to the reference).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <json.hpp>

#include "b200.hpp"
#include "core_model.hpp"
#include "offline_solvers.hpp"
#include "schedule.hpp"

namespace coinfer {

// Task process: a user whose previous constraint window has lapsed draws a
// new task each slot with probability p_arrive (Bernoulli) or at once
// (Immediate); deadlines ~ U[l_low, l_high].
struct ArrivalModel {
  enum class Kind { Bernoulli, Immediate };
  Kind kind = Kind::Bernoulli;
  double p_arrive = 0.25;
  double l_low = 0.25;
  double l_high = 1.0;

  void check() const {
    // comparisons as the reference writes them (NaN passes the same way)
    if (l_low <= 0.0 || l_high < l_low) throw std::invalid_argument("arrivals: bad deadline range");
    if (kind == Kind::Bernoulli && (p_arrive < 0.0 || p_arrive > 1.0))
      throw std::invalid_argument("arrivals: p_arrive must lie in [0, 1]");
  }
};

struct MdpState {
  std::vector<double> deadline;  // remaining time per user; 0 = no task
  double edge_busy = 0.0;        // time until the planned batches are done
};

struct ActionVec {
  int mode = 0;            // 0 wait, 1 all pending tasks local now, 2 call the solver
  double threshold = 0.0;  // deadline clip for mode 2
};

enum class OnlineSolver { IPSSA, OG };

struct StepInfo {
  double energy = 0.0;
  double forced_cost = 0.0;
  std::size_t forced_count = 0;
  std::size_t pending_before = 0;
  double busy_before = 0.0;
  bool solver_invoked = false;
  std::size_t solver_tasks = 0;
  std::size_t solver_groups = 0;
  std::vector<std::size_t> batch_sizes;
};

namespace detail {
#ifndef COINFER_DETAIL_FMT_G17
#define COINFER_DETAIL_FMT_G17
inline std::string fmt_g17(double v) {
  char text[40];
  std::snprintf(text, sizeof text, "%.17g", v);
  return std::string(text);
}
#endif
}  // namespace detail

class OnlineEnv {
 public:
  OnlineEnv(Scenario base, ArrivalModel arrivals, OnlineSolver solver = OnlineSolver::OG,
            double slot = 0.025, std::uint64_t seed = 1)
      : sc_(std::move(base)), arr_(arrivals), solver_(solver), slot_(slot), seed_(seed) {
    sc_.check();
    arr_.check();
    if (slot_ <= 0.0) throw std::invalid_argument("online: slot must be positive");
    const double W = sc_.profile.total_work();
    floor_.reserve(sc_.n_users());
    for (const UserSpec& u : sc_.users) {
      if (u.arrival != 0.0)
        throw std::invalid_argument("online: users must be released at time zero");
      floor_.push_back(W / u.f_max);  // all-local run at full speed
      if (floor_.back() > arr_.l_low)
        throw std::invalid_argument("online: l_low below a user's all-local processing floor");
    }
    reset();
  }

  const MdpState& state() const { return st_; }
  const Scenario& scenario() const { return sc_; }
  const ArrivalModel& arrivals() const { return arr_; }
  OnlineSolver solver() const { return solver_; }
  double slot() const { return slot_; }
  std::uint64_t seed() const { return seed_; }
  double now() const { return double(tick_) * slot_; }
  double local_floor(std::size_t m) const { return floor_[m]; }

  MdpState reset() {
    rng_.seed(seed_);
    tick_ = 0;
    const std::size_t M = sc_.n_users();
    st_.deadline.assign(M, 0.0);
    st_.edge_busy = 0.0;
    expiry_.assign(M, -1.0);
    draw_tasks();
    return st_;
  }
  MdpState reset(std::uint64_t seed) {
    seed_ = seed;
    return reset();
  }

  void load_state(const MdpState& s) {
    const std::size_t M = sc_.n_users();
    if (s.deadline.size() != M)
      throw std::invalid_argument("load_state: one deadline per user required");
    if (std::any_of(s.deadline.begin(), s.deadline.end(), [](double l) { return l < 0.0; }))
      throw std::invalid_argument("load_state: negative deadline");
    if (s.edge_busy < 0.0) throw std::invalid_argument("load_state: negative busy time");
    st_ = s;
    const double t = now();
    for (std::size_t m = 0; m < M; ++m) expiry_[m] = st_.deadline[m] > 0.0 ? t + st_.deadline[m] : t - 1.0;
  }

  // One slot: apply the (clamped) action, rescue tasks that could no longer
  // finish locally by the next decision, advance time, draw arrivals.
  double step(const ActionVec& act, StepInfo* info_out = nullptr) {
    StepInfo info;
    info.pending_before = pending();
    info.busy_before = st_.edge_busy;
    const int mode = act.mode < 0 ? 0 : (act.mode > 2 ? 2 : act.mode);
    const double l_th = std::min(std::max(act.threshold, 0.0), arr_.l_high);
    if (mode == 1) {
      run_local(info);
    } else if (mode == 2 && !(st_.edge_busy > 0.0)) {
      call_solver(l_th, info);
    }
    rescue(info);
    advance();
    const double reward = -(info.energy + info.forced_cost);
    if (info_out) *info_out = std::move(info);
    return reward;
  }

  // Replaces the state with the one the device episode ended in (run_episode's
  // GPU path): deadlines, expiries, edge_busy, the slot count, and the
  // generator advanced by the draws the episode consumed.
  void adopt_episode_end(std::size_t slots, const double* fin, std::uint64_t draws) {
    const std::size_t M = sc_.n_users();
    st_.deadline.assign(fin, fin + M);
    expiry_.assign(fin + M, fin + 2 * M);
    st_.edge_busy = fin[2 * M];
    tick_ = slots;
    rng_.seed(seed_);
    rng_.discard(draws);
  }

 private:
  std::size_t pending() const {
    return (std::size_t)std::count_if(st_.deadline.begin(), st_.deadline.end(),
                                      [](double l) { return l > 0.0; });
  }

  // mode 1: every pending task runs locally at the slowest frequency that
  // meets its remaining time (clamped to [f_min, f_max]).
  void run_local(StepInfo& info) {
    const double W = sc_.profile.total_work();
    for (std::size_t m = 0; m < sc_.n_users(); ++m) {
      double& l = st_.deadline[m];
      if (l <= 0.0) continue;
      const UserSpec& u = sc_.users[m];
      const double f = std::min(std::max(W / l, u.f_min), u.f_max);
      info.energy += local_energy(u.kappa, W, f);
      l = 0.0;
    }
  }

  // mode 2 on an idle edge: the pending users (ascending id) form a
  // sub-scenario whose deadlines at or above the threshold are pulled down to
  // it (never below the user's local floor); OG plans it, or IP-SSA at the
  // tightest deadline.  Both solves run on the GPU engine.
  void call_solver(double l_th, StepInfo& info) {
    Scenario sub;
    sub.profile = sc_.profile;
    std::vector<std::size_t> ids;
    for (std::size_t m = 0; m < sc_.n_users(); ++m) {
      const double l = st_.deadline[m];
      if (!(l > 0.0)) continue;
      ids.push_back(m);
      sub.users.push_back(sc_.users[m]);
      sub.deadline.push_back(l >= l_th ? std::max(l_th, floor_[m]) : l);
    }
    if (ids.empty()) return;
    info.solver_invoked = true;
    info.solver_tasks = ids.size();
    auto record = [&](const Schedule& s) {
      for (const BatchView& b : batch_views(s)) info.batch_sizes.push_back(b.size());
    };
    if (solver_ == OnlineSolver::OG) {
      const GroupingPlan plan = og(sub);
      info.energy += plan.energy;
      info.solver_groups = plan.groups.size();
      st_.edge_busy = plan.schedule.batch_start.empty() ? 0.0 : plan.group_deadline.back();
      record(plan.schedule);
    } else {
      double lc = sub.deadline.front();
      for (double l : sub.deadline) lc = std::min(lc, l);
      const SolveResult r = ip_ssa(sub, lc);
      info.energy += r.energy;
      info.solver_groups = 1;
      st_.edge_busy = r.schedule.batch_start.empty() ? 0.0 : lc;
      record(r.schedule);
    }
    for (std::size_t m : ids) st_.deadline[m] = 0.0;
  }

  // A task whose remaining time after this slot would drop below its
  // all-local floor runs now at f_max.
  void rescue(StepInfo& info) {
    const double W = sc_.profile.total_work();
    for (std::size_t m = 0; m < sc_.n_users(); ++m) {
      double& l = st_.deadline[m];
      if (l <= 0.0 || !(l - slot_ < floor_[m])) continue;
      const UserSpec& u = sc_.users[m];
      info.forced_cost += local_energy(u.kappa, W, u.f_max);
      info.forced_count += 1;
      l = 0.0;
    }
  }

  void advance() {
    ++tick_;
    for (double& l : st_.deadline)
      if (l > 0.0) l -= slot_;
    st_.edge_busy = std::max(0.0, st_.edge_busy - slot_);
    draw_tasks();
    for (std::size_t m = 0; m < sc_.n_users(); ++m) {
      const double l = st_.deadline[m];
      if (l > 0.0 && l < floor_[m] - 1e-12)
        throw std::logic_error("online: task slipped below its local floor");
    }
  }

  // Arrivals for the slot starting now: users without a task whose last
  // window has passed draw a coin (Bernoulli, 0 < p < 1), then a deadline.
  void draw_tasks() {
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    std::uniform_real_distribution<double> span(arr_.l_low, arr_.l_high);
    const bool bern = arr_.kind == ArrivalModel::Kind::Bernoulli;
    const double t = now();
    for (std::size_t m = 0; m < sc_.n_users(); ++m) {
      if (st_.deadline[m] > 0.0 || !(t > expiry_[m])) continue;
      if (bern && arr_.p_arrive <= 0.0) continue;
      if (bern && arr_.p_arrive < 1.0 && unit(rng_) >= arr_.p_arrive) continue;
      const double l = arr_.l_low < arr_.l_high ? span(rng_) : arr_.l_low;
      st_.deadline[m] = l;
      expiry_[m] = t + l;
    }
  }

  Scenario sc_;
  ArrivalModel arr_;
  OnlineSolver solver_;
  double slot_;
  std::uint64_t seed_;
  std::mt19937_64 rng_;
  std::size_t tick_ = 0;
  MdpState st_;
  std::vector<double> floor_;
  std::vector<double> expiry_;
};

struct TraceRow {
  std::size_t slot = 0;
  int action_c = 0;
  double action_lth = 0.0;
  double reward = 0.0;
  double energy = 0.0;
  std::size_t forced_count = 0;
  std::size_t pending_count = 0;
  double edge_busy = 0.0;
};

struct EpisodeMetrics {
  std::size_t slots = 0;
  double total_energy = 0.0;
  double total_forced_cost = 0.0;
  double total_reward = 0.0;
  std::size_t forced_count = 0;
  std::size_t solver_calls = 0;
  std::size_t solver_tasks = 0;
  std::size_t solver_groups = 0;
  std::size_t batches = 0;
  std::size_t batched_tasks = 0;
  std::vector<TraceRow> trace;

  double mean_tasks_per_call() const { return ratio(solver_tasks, solver_calls); }
  double mean_tasks_per_group() const { return ratio(solver_tasks, solver_groups); }
  double mean_batch_size() const { return ratio(batched_tasks, batches); }

 private:
  static double ratio(std::size_t a, std::size_t b) { return b ? double(a) / double(b) : 0.0; }
};

using PolicyFn = std::function<ActionVec(const MdpState&)>;

namespace detail {
// local_policy's callable, a named type so run_episode can recognise it.
struct LocalPolicy {
  ActionVec operator()(const MdpState& s) const {
    const bool any = std::any_of(s.deadline.begin(), s.deadline.end(), [](double l) { return l > 0.0; });
    return any ? ActionVec{1, 0.0} : ActionVec{0, 0.0};
  }
};
}  // namespace detail

inline PolicyFn local_policy() { return detail::LocalPolicy{}; }

// Fires the solver `window` slots after the edge goes idle with work
// pending (0: at once); the threshold is l_high, so nothing is clipped.
class TimeWindowPolicy {
 public:
  TimeWindowPolicy(std::size_t window, double l_high) : window_(window), l_th_(l_high) {}

  ActionVec operator()(const MdpState& s) {
    const bool any = std::any_of(s.deadline.begin(), s.deadline.end(), [](double l) { return l > 0.0; });
    if (!any || s.edge_busy > 0.0) {
      waited_ = 0;
      return {0, 0.0};
    }
    if (waited_ < window_) {
      ++waited_;
      return {0, 0.0};
    }
    waited_ = 0;
    return {2, l_th_};
  }

  std::size_t window() const { return window_; }
  double threshold() const { return l_th_; }
  std::size_t waited() const { return waited_; }

 private:
  std::size_t window_;
  double l_th_;
  std::size_t waited_ = 0;
};

namespace detail {

// The whole episode on the GPU (coinfer_online_run, one episode, full trace);
// false when the policy is not one of the fixed policies the device driver
// implements, or the instance is outside its limits.
inline bool run_episode_device(OnlineEnv& env, const PolicyFn& policy, std::size_t horizon,
                               EpisodeMetrics& m) {
  coinfer_online_cfg cfg{};
  if (const TimeWindowPolicy* tw = policy.target<TimeWindowPolicy>()) {
    if (tw->waited() != 0 || tw->window() > (std::size_t)INT32_MAX) return false;
    cfg.policy = COINFER_POLICY_TW;
    cfg.window = (int32_t)tw->window();
    cfg.threshold = tw->threshold();
  } else if (policy.target<LocalPolicy>()) {
    cfg.policy = COINFER_POLICY_LOCAL;
  } else {
    return false;
  }
  const Scenario& sc = env.scenario();
  const std::size_t M = sc.n_users();
  const ArrivalModel& am = env.arrivals();
  cfg.arrival = am.kind == ArrivalModel::Kind::Bernoulli ? COINFER_ARRIVAL_BERNOULLI : COINFER_ARRIVAL_IMMEDIATE;
  cfg.solver = env.solver() == OnlineSolver::OG ? COINFER_SOLVER_OG : COINFER_SOLVER_IPSSA;
  cfg.p_arrive = am.p_arrive;
  cfg.l_low = am.l_low;
  cfg.l_high = am.l_high;
  cfg.slot = env.slot();
  cfg.horizon = (int64_t)horizon;

  b200::FlatProfile prof(sc.profile);
  const Scenario* one[1] = {&sc};
  b200::UserBatch users(one, 1, M);
  const std::uint64_t seed = env.seed();
  int32_t status = 0;
  double totals[3];
  int64_t counts[6];
  int64_t draws = 0;
  std::vector<double> tr_reward(horizon), tr_energy(horizon), tr_busy(horizon), fin(2 * M + 1);
  std::vector<int32_t> tr_pending(horizon), tr_action(horizon), tr_forced(horizon);
  coinfer_online_out out{};
  out.status = &status;
  out.totals = totals;
  out.counts = counts;
  out.n_trace = 1;
  out.trace_reward = tr_reward.data();
  out.trace_energy = tr_energy.data();
  out.trace_pending = tr_pending.data();
  out.trace_edge_busy = tr_busy.data();
  out.trace_action = tr_action.data();
  out.trace_forced = tr_forced.data();
  out.final_state = fin.data();
  out.draws = &draws;
  const int rc = coinfer_online_run(b200::context().get(), &prof.view, &users.view, &cfg, &seed, 1, &out);
  if (rc == COINFER_E_UNSUPPORTED) return false;  // e.g. more users than the device driver holds
  b200::check_call(rc);
  b200::check_status(status, env.solver() == OnlineSolver::OG ? "og" : "ip_ssa");

  m.total_energy = totals[0];
  m.total_forced_cost = totals[1];
  m.total_reward = totals[2];
  m.forced_count = (std::size_t)counts[0];
  m.solver_calls = (std::size_t)counts[1];
  m.solver_tasks = (std::size_t)counts[2];
  m.solver_groups = (std::size_t)counts[3];
  m.batches = (std::size_t)counts[4];
  m.batched_tasks = (std::size_t)counts[5];
  m.trace.resize(horizon);
  for (std::size_t t = 0; t < horizon; ++t) {
    TraceRow& r = m.trace[t];
    r.slot = t;
    r.action_c = tr_action[t];
    r.action_lth = tr_action[t] == 2 ? cfg.threshold : 0.0;
    r.reward = tr_reward[t];
    r.energy = tr_energy[t];
    r.forced_count = (std::size_t)tr_forced[t];
    r.pending_count = (std::size_t)tr_pending[t];
    r.edge_busy = tr_busy[t];
  }
  env.adopt_episode_end(horizon, fin.data(), (std::uint64_t)draws);
  return true;
}

}  // namespace detail

inline EpisodeMetrics run_episode(OnlineEnv& env, PolicyFn policy, std::size_t horizon) {
  if (horizon == 0) throw std::invalid_argument("run_episode: empty horizon");
  EpisodeMetrics m;
  m.slots = horizon;
  env.reset();
  if (detail::run_episode_device(env, policy, horizon, m)) return m;
  // any other policy: the host slot loop, solver calls on the GPU
  m.trace.reserve(horizon);
  for (std::size_t t = 0; t < horizon; ++t) {
    const ActionVec a = policy(env.state());
    StepInfo info;
    const double r = env.step(a, &info);
    m.total_energy += info.energy;
    m.total_forced_cost += info.forced_cost;
    m.forced_count += info.forced_count;
    m.solver_calls += info.solver_invoked ? 1 : 0;
    m.solver_tasks += info.solver_tasks;
    m.solver_groups += info.solver_groups;
    m.batches += info.batch_sizes.size();
    for (std::size_t b : info.batch_sizes) m.batched_tasks += b;
    m.trace.push_back({t, a.mode, a.threshold, r, info.energy, info.forced_count, info.pending_before,
                       info.busy_before});
  }
  m.total_reward = -(m.total_energy + m.total_forced_cost);  // the totals' identity, exactly
  return m;
}

inline EpisodeMetrics run_episode(OnlineEnv& env, PolicyFn policy, std::size_t horizon,
                                  std::uint64_t seed) {
  env.reset(seed);
  return run_episode(env, std::move(policy), horizon);
}

inline void write_trace_csv(const std::vector<TraceRow>& trace, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw std::runtime_error("write_trace_csv: cannot open " + path);
  f << "slot,action_c,action_lth,reward,energy,forced_count,pending_count,edge_busy\n";
  for (const TraceRow& r : trace) {
    f << r.slot << ',' << r.action_c << ',' << detail::fmt_g17(r.action_lth) << ','
      << detail::fmt_g17(r.reward) << ',' << detail::fmt_g17(r.energy) << ',' << r.forced_count << ','
      << r.pending_count << ',' << detail::fmt_g17(r.edge_busy) << '\n';
  }
}

inline void write_episode_summary(const EpisodeMetrics& m, const std::string& path) {
  nlohmann::json j = {{"slots", m.slots},
                      {"total_energy", m.total_energy},
                      {"total_forced_cost", m.total_forced_cost},
                      {"total_reward", m.total_reward},
                      {"forced_count", m.forced_count},
                      {"solver_calls", m.solver_calls},
                      {"mean_tasks_per_call", m.mean_tasks_per_call()},
                      {"mean_tasks_per_group", m.mean_tasks_per_group()},
                      {"mean_batch_size", m.mean_batch_size()}};
  std::ofstream f(path);
  if (!f) throw std::runtime_error("write_episode_summary: cannot open " + path);
  f << j.dump(2) << '\n';
}

}  // namespace coinfer
