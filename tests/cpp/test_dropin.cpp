// Drop-in C++ API (include/coinfer/) on the B200 engine vs the reference's
// golden vectors (tests/golden/*.json, made from the reference by
// tests/golden/make_golden.py): every solve through the reference's own
// signatures (ip_ssa, fixed_batch_schedule, og), decisions and energies bit
// for bit, the device-built schedule checked by validate() and total_energy,
// errors mapped to the reference's exception types.  Plus the batched API
// and the baselines' invariants.  Needs a GPU.
#include <gtest/gtest.h>
#include <unistd.h>

#include <cstring>
#include <fstream>
#include <json.hpp>
#include <random>
#include <string>

#include "coinfer/offline_solvers.hpp"
#include "coinfer/online_sim.hpp"
#include <memory>

using namespace coinfer;
using json = nlohmann::json;

namespace {

std::string golden_dir() {
  if (const char* g = std::getenv("COINFER_GOLDEN")) return g;
  char buf[4096];
  const ssize_t n = readlink("/proc/self/exe", buf, sizeof buf - 1);
  std::string exe(buf, n > 0 ? (size_t)n : 0);
  return exe.substr(0, exe.rfind('/')) + "/../../golden";  // tests/cpp/_bin -> tests/golden
}

std::vector<json> load(const std::string& name) {
  std::ifstream f(golden_dir() + "/" + name + ".json");
  if (!f) throw std::runtime_error("golden file missing: " + name);
  json j;
  f >> j;
  return j.get<std::vector<json>>();
}

std::vector<json> all_cases() {
  std::vector<json> v;
  for (const char* n : {"kat", "random", "cli"}) {
    auto c = load(n);
    v.insert(v.end(), c.begin(), c.end());
  }
  return v;
}

Scenario scenario(const json& c, size_t k) {
  Scenario sc;
  sc.profile.work = c["profile"]["work"].get<std::vector<double>>();
  sc.profile.data_bits = c["profile"]["data_bits"].get<std::vector<double>>();
  sc.profile.latency = c["profile"]["latency"].get<std::vector<std::vector<double>>>();
  const json& u = c["users"];
  const size_t M = u["deadline"][k].size();
  for (size_t m = 0; m < M; ++m) {
    UserSpec s;
    s.f_min = u["f_min"][k][m];
    s.f_max = u["f_max"][k][m];
    s.kappa = u["kappa"][k][m];
    s.rate_up = u["rate_up"][k][m];
    s.rate_down = u["rate_down"][k][m];
    s.power_up = u["power_up"][k][m];
    s.power_down = u["power_down"][k][m];
    s.arrival = u["arrival"][k][m];
    sc.users.push_back(s);
    sc.deadline.push_back(u["deadline"][k][m]);
  }
  return sc;
}

size_t n_inst(const json& c) { return c["users"]["deadline"].size(); }

double ip_deadline(const json& c, const Scenario& sc, size_t k) {
  if (!c["deadline"].is_null()) return c["deadline"][k];
  double l = kInf;
  for (double d : sc.deadline) l = std::min(l, d);
  return l;
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

// The exception family of a per-instance status, as the reference throws it.
template <class F>
void expect_throws_for_status(int st, F&& f, const std::string& where) {
  if (st == COINFER_ST_INFEASIBLE) {
    EXPECT_THROW(f(), std::domain_error) << where;
  } else if (st == COINFER_ST_BOUND_PAST_TABLE) {
    EXPECT_THROW(f(), std::out_of_range) << where;
  } else {
    EXPECT_THROW(f(), std::invalid_argument) << where;
  }
}

void check_solve(const SolveResult& r, const json& e, size_t k, const Scenario& sc, const std::string& where) {
  const size_t M = sc.n_users(), N = sc.profile.subtasks();
  EXPECT_EQ(r.batch_bound, e["batch_bound"][k].get<size_t>()) << where;
  EXPECT_EQ(r.pipeline_feasible, e["pipeline_feasible"][k].get<int>() != 0) << where;
  EXPECT_TRUE(same_bits(r.energy, e["energy"][k].get<double>())) << where;
  for (size_t m = 0; m < M; ++m) {
    EXPECT_EQ(r.split[m], e["split"][k][m].get<size_t>()) << where << " user " << m;
    EXPECT_TRUE(same_bits(r.schedule.freq[m], e["freq"][k][m].get<double>())) << where << " user " << m;
  }
  for (size_t n = 0; n < N; ++n) EXPECT_EQ(r.batch_size[n], e["batch_size"][k][n].get<size_t>()) << where;
  const ScheduleMetrics mt = schedule_metrics(r.schedule, sc);
  for (size_t m = 0; m < M; ++m)
    EXPECT_TRUE(same_bits(mt.per_user_energy[m], e["user_energy"][k][m].get<double>())) << where;
  EXPECT_TRUE(same_bits(total_energy(r.schedule, sc), r.energy)) << where;
  EXPECT_TRUE(validate(r.schedule, sc).empty()) << where;
}

}  // namespace

TEST(Golden, IpSsaAndFixedBatchThroughTheDropIn) {
  int n = 0;
  for (const json& c : all_cases()) {
    const std::string kind = c["kind"];
    if (kind == "og") continue;
    const json& e = c["expect"];
    for (size_t k = 0; k < n_inst(c); ++k) {
      const Scenario sc = scenario(c, k);
      const double l = ip_deadline(c, sc, k);
      const std::string where = c["name"].get<std::string>() + "[" + std::to_string(k) + "]";
      const int st = e["status"][k];
      auto run = [&]() {
        return kind == "ipssa" ? ip_ssa(sc, l) : fixed_batch_schedule(sc, l, c["b"][k].get<size_t>());
      };
      if (st != COINFER_ST_OK) {
        expect_throws_for_status(st, run, where);
        continue;
      }
      check_solve(run(), e, k, sc, where);
      ++n;
    }
  }
  EXPECT_GT(n, 100);
}

TEST(Golden, OgThroughTheDropIn) {
  int n = 0;
  for (const json& c : all_cases()) {
    if (c["kind"] != "og") continue;
    const json& e = c["expect"];
    for (size_t k = 0; k < n_inst(c); ++k) {
      const Scenario sc = scenario(c, k);
      const std::string where = c["name"].get<std::string>() + "[" + std::to_string(k) + "]";
      const int st = e["status"][k];
      if (st != COINFER_ST_OK) {
        expect_throws_for_status(st, [&]() { return og(sc); }, where);
        continue;
      }
      const GroupingPlan p = og(sc);
      const size_t M = sc.n_users();
      EXPECT_EQ(p.fallback, e["fallback"][k].get<int>() != 0) << where;
      EXPECT_TRUE(same_bits(p.energy, e["energy"][k].get<double>())) << where;
      const size_t G = e["n_groups"][k];
      ASSERT_EQ(p.groups.size(), G) << where;
      for (size_t g = 0; g < G; ++g) {
        const int lo = e["group_lo"][k][g], sz = e["group_size"][k][g];
        std::vector<size_t> ids;
        for (int q = lo; q < lo + sz; ++q) ids.push_back(e["order"][k][q].get<size_t>());
        EXPECT_EQ(p.groups[g], ids) << where << " group " << g;
        EXPECT_TRUE(same_bits(p.group_deadline[g], e["group_deadline"][k][g].get<double>())) << where;
        EXPECT_TRUE(same_bits(p.group_energy[g], e["group_energy"][k][g].get<double>())) << where;
      }
      for (size_t m = 0; m < M; ++m) {
        size_t split = 0;
        while (split < sc.profile.subtasks() && p.schedule.x[m][split] == kLocal) ++split;
        EXPECT_EQ(split, e["split"][k][m].get<size_t>()) << where << " user " << m;
        EXPECT_TRUE(same_bits(p.schedule.freq[m], e["freq"][k][m].get<double>())) << where;
      }
      const ScheduleMetrics mt = schedule_metrics(p.schedule, sc);
      for (size_t m = 0; m < M; ++m)
        EXPECT_TRUE(same_bits(mt.per_user_energy[m], e["user_energy"][k][m].get<double>())) << where;
      EXPECT_TRUE(validate(p.schedule, sc).empty()) << where;
      // the plan's energy is the left fold of the group energies (og:385-386;
      // a fallback plan carries lc_solve's user-order fold instead)
      double fold = 0.0;
      for (double x : p.group_energy) fold += x;
      if (!p.fallback) {
        EXPECT_TRUE(same_bits(fold, p.energy)) << where;
      }
      Schedule norm = p.schedule;
      normalize(norm);
      EXPECT_EQ(norm.x, p.schedule.x) << where << " (device schedule is normalised)";
      ++n;
    }
  }
  EXPECT_GT(n, 50);
}

TEST(Batched, MatchesSingleCallsBitForBit) {
  // the CLI-style C3 instances (one profile, one user count) in one launch
  for (const json& c : load("cli")) {
    if (n_inst(c) < 2) continue;
    std::vector<Scenario> scs;
    std::vector<double> l;
    for (size_t k = 0; k < n_inst(c); ++k) {
      scs.push_back(scenario(c, k));
      l.push_back(ip_deadline(c, scs.back(), k));
    }
    if (c["kind"] == "og") {
      const auto b = b200::og(scs);
      for (size_t k = 0; k < scs.size(); ++k) {
        const GroupingPlan one = og(scs[k]);
        EXPECT_EQ(b.status[k], COINFER_ST_OK);
        EXPECT_TRUE(same_bits(b.results[k].energy, one.energy));
        EXPECT_EQ(b.results[k].groups, one.groups);
        EXPECT_EQ(b.results[k].schedule.x, one.schedule.x);
        EXPECT_EQ(b.results[k].schedule.batch_start, one.schedule.batch_start);
      }
    } else if (c["kind"] == "ipssa") {
      const auto b = b200::ip_ssa(scs, l);
      for (size_t k = 0; k < scs.size(); ++k) {
        const SolveResult one = ip_ssa(scs[k], l[k]);
        EXPECT_TRUE(same_bits(b.results[k].energy, one.energy));
        EXPECT_EQ(b.results[k].split, one.split);
        EXPECT_EQ(b.results[k].schedule.completion, one.schedule.completion);
      }
    }
  }
}

TEST(Batched, BadDrawReportedByStatus) {
  const json c = load("kat")[0];
  std::vector<Scenario> scs{scenario(c, 0), scenario(c, 0)};
  scs[1].users[0].kappa = -1.0;
  const auto b = b200::ip_ssa(scs, {0.1, 0.1});
  EXPECT_EQ(b.status[0], COINFER_ST_OK);
  EXPECT_EQ(b.status[1], COINFER_ST_NEG_KAPPA);
  EXPECT_THROW(ip_ssa(scs[1], 0.1), std::invalid_argument);
}

TEST(Baselines, SchedulesValidateAndFoldTheirEnergy) {
  int n = 0;
  for (const json& c : all_cases()) {
    if (c["kind"] != "og" || c["expect"]["status"][0] != 0) continue;
    const Scenario sc = scenario(c, 0);
    for (BaselineMode mode : {BaselineMode::LC, BaselineMode::PS, BaselineMode::FIFO, BaselineMode::IPSSA_NP}) {
      SolveResult r;
      try {
        r = baseline(sc, mode);
      } catch (const std::domain_error&) {
        continue;  // a baseline may find no feasible plan where OG does
      }
      const std::string where = c["name"].get<std::string>() + " mode " + std::to_string((int)mode);
      EXPECT_TRUE(validate(r.schedule, sc).empty()) << where;
      EXPECT_TRUE(same_bits(total_energy(r.schedule, sc), r.energy)) << where;
      Schedule norm = r.schedule;
      normalize(norm);
      EXPECT_EQ(norm.x, r.schedule.x) << where;
      EXPECT_EQ(norm.batch_start, r.schedule.batch_start) << where;
      ++n;
    }
  }
  EXPECT_GT(n, 100);
}

template <class F>
std::string invalid_argument_message(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument& e) {
    return e.what();
  }
  return "<no invalid_argument>";
}

TEST(Errors, ShapeAndContractMessages) {
  const Scenario sc = scenario(load("kat")[0], 0);
  Scenario bad = sc;
  bad.deadline.push_back(1.0);
  EXPECT_EQ(invalid_argument_message([&] { og(bad); }), "scenario: one deadline per user required");
  bad = sc;
  bad.profile.latency[1].pop_back();
  EXPECT_EQ(invalid_argument_message([&] { ip_ssa(bad, 0.1); }), "profile: ragged latency table");
  bad = sc;
  bad.users[0].rate_up = 0.0;
  EXPECT_EQ(invalid_argument_message([&] { ip_ssa(bad, 0.1); }), "scenario: rates must be positive");
  bad = sc;
  bad.profile.work[0] = 0.0;
  EXPECT_EQ(invalid_argument_message([&] { baseline(bad, BaselineMode::PS); }),
            "profile: work must be positive");
  EXPECT_THROW(fixed_batch_schedule(sc, 0.1, 0), std::invalid_argument);
  EXPECT_THROW(fixed_batch_schedule(sc, 0.1, 1000), std::out_of_range);
  Scenario empty = sc;
  empty.users.clear();
  empty.deadline.clear();
  EXPECT_EQ(ip_ssa(empty, 0.1).split.size(), 0u);
  EXPECT_EQ(og(empty).groups.size(), 0u);
  EXPECT_EQ(baseline(empty, BaselineMode::FIFO).batch_size.size(), sc.profile.subtasks());
}

// ---------------------------------------------------------------- online_sim

namespace {

struct OnlineCase {
  Scenario sc;
  ArrivalModel am;
  OnlineSolver solver;
  double slot;
  bool local;
  std::size_t window;
  double threshold;
  std::size_t horizon;
  std::uint64_t seed;
};

OnlineCase online_case(const json& c) {
  OnlineCase o;
  o.sc = scenario(c, 0);
  const json& g = c["cfg"];
  o.am.kind = g["arrival"] == "immediate" ? ArrivalModel::Kind::Immediate : ArrivalModel::Kind::Bernoulli;
  o.am.p_arrive = g["p_arrive"];
  o.am.l_low = g["l_low"];
  o.am.l_high = g["l_high"];
  o.solver = g["solver"] == "og" ? OnlineSolver::OG : OnlineSolver::IPSSA;
  o.slot = g["slot"];
  o.local = g["policy"] == "local";
  o.window = g["window"].get<std::size_t>();
  o.threshold = g["threshold"].is_null() ? o.am.l_high : g["threshold"].get<double>();
  o.horizon = g["horizon"].get<std::size_t>();
  o.seed = c["seed"].get<std::uint64_t>();
  return o;
}

void expect_episode(const EpisodeMetrics& m, const json& e, const std::string& where) {
  EXPECT_TRUE(same_bits(m.total_energy, e["totals"][0].get<double>())) << where;
  EXPECT_TRUE(same_bits(m.total_forced_cost, e["totals"][1].get<double>())) << where;
  EXPECT_TRUE(same_bits(m.total_reward, e["totals"][2].get<double>())) << where;
  const std::size_t got[6] = {m.forced_count, m.solver_calls, m.solver_tasks,
                              m.solver_groups, m.batches,     m.batched_tasks};
  for (int i = 0; i < 6; ++i) EXPECT_EQ(got[i], e["counts"][i].get<std::size_t>()) << where << " count " << i;
  ASSERT_EQ(m.trace.size(), e["trace_reward"].size()) << where;
  std::size_t bad = 0;
  for (std::size_t t = 0; t < m.trace.size(); ++t) {
    const TraceRow& r = m.trace[t];
    bad += r.slot != t || !same_bits(r.reward, e["trace_reward"][t].get<double>()) ||
           !same_bits(r.energy, e["trace_energy"][t].get<double>()) ||
           r.pending_count != e["trace_pending"][t].get<std::size_t>() ||
           !same_bits(r.edge_busy, e["trace_edge_busy"][t].get<double>());
  }
  EXPECT_EQ(bad, 0u) << where << ": slots differing from the reference trace";
}

}  // namespace

// run_episode with the fixed policies is ONE device episode; the same episode
// stepped on the host (a policy the device driver does not know, so
// OnlineEnv::step runs each slot and calls the GPU og / ip_ssa) must give the
// same reference trace, the same trace actions, and leave the env in the same
// state (deadlines, edge_busy, time, random stream position).
TEST(Online, RunEpisodeDeviceAndHostStepMatchTheReference) {
  for (const json& c : load("online")) {
    const OnlineCase o = online_case(c);
    const std::string where = c["name"];
    OnlineEnv dev(o.sc, o.am, o.solver, o.slot, 1);
    OnlineEnv host(o.sc, o.am, o.solver, o.slot, 1);
    const PolicyFn fixed = o.local ? local_policy() : PolicyFn(TimeWindowPolicy(o.window, o.threshold));
    const EpisodeMetrics md = run_episode(dev, fixed, o.horizon, o.seed);
    auto inner = std::make_shared<PolicyFn>(fixed);  // opaque wrapper: forces the host slot loop
    const EpisodeMetrics mh = run_episode(host, [inner](const MdpState& s) { return (*inner)(s); }, o.horizon, o.seed);
    expect_episode(md, c["expect"], where + " (device episode)");
    expect_episode(mh, c["expect"], where + " (host steps)");
    for (std::size_t t = 0; t < md.trace.size(); ++t) {
      ASSERT_EQ(md.trace[t].action_c, mh.trace[t].action_c) << where << " slot " << t;
      ASSERT_TRUE(same_bits(md.trace[t].action_lth, mh.trace[t].action_lth)) << where << " slot " << t;
      ASSERT_EQ(md.trace[t].forced_count, mh.trace[t].forced_count) << where << " slot " << t;
    }
    EXPECT_EQ(md.mean_batch_size(), mh.mean_batch_size()) << where;
    // state after the episode, and after more host slots from it
    for (int extra = 0; extra < 60; ++extra) {
      ASSERT_TRUE(same_bits(dev.now(), host.now())) << where;
      ASSERT_TRUE(same_bits(dev.state().edge_busy, host.state().edge_busy)) << where << " +" << extra;
      for (std::size_t m = 0; m < o.sc.n_users(); ++m)
        ASSERT_TRUE(same_bits(dev.state().deadline[m], host.state().deadline[m])) << where << " user " << m << " +" << extra;
      const ActionVec a{extra % 3 == 2 ? 1 : 0, 0.0};
      ASSERT_TRUE(same_bits(dev.step(a), host.step(a))) << where << " +" << extra;
    }
  }
}

TEST(Online, StepSolverCallEqualsOgOnTheClippedScenario) {
  const json c = load("online")[0];
  OnlineCase o = online_case(c);
  o.am.p_arrive = 0.0;  // no arrivals: only the loaded state
  OnlineEnv env(o.sc, o.am, OnlineSolver::OG, o.slot, 3);
  const std::size_t M = o.sc.n_users();
  MdpState s;
  s.deadline.assign(M, 0.0);
  for (std::size_t m = 0; m < M; m += 2) s.deadline[m] = 0.15 + 0.05 * double(m % 5);
  env.load_state(s);
  StepInfo info;
  const double r = env.step({2, 0.25}, &info);
  Scenario sub;
  sub.profile = o.sc.profile;
  for (std::size_t m = 0; m < M; ++m)
    if (s.deadline[m] > 0.0) {
      sub.users.push_back(o.sc.users[m]);
      sub.deadline.push_back(s.deadline[m] >= 0.25 ? std::max(0.25, env.local_floor(m)) : s.deadline[m]);
    }
  const GroupingPlan plan = og(sub);
  EXPECT_TRUE(same_bits(info.energy, plan.energy));
  EXPECT_TRUE(same_bits(-r, plan.energy + info.forced_cost));
  EXPECT_EQ(info.solver_groups, plan.groups.size());
  EXPECT_EQ(info.solver_tasks, sub.users.size());
}
