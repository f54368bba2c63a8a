// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference headers (/root/reference/proj/include,
// included in place, never copied) behind the same SoA C ABI as the product
// library, so tests and bench.py can drive the reference solvers on exactly
// the bytes the CUDA engine sees.  Built by oracle/Makefile into
// oracle/_ref/libcoinfer_ref.so (git-ignored; travels to the GPU box with the
// snapshot).  Nothing in the product path links it.
//
// Entry points:
//   ref_ipssa_batch / ref_fixed_batch / ref_og_batch   coinfer::ip_ssa,
//       fixed_batch_schedule, og + schedule_metrics (offline_solvers.hpp)
//   ref_sweep_threads       the CLI's IPSSA+OG pair per instance
//       (coinfer_main.cpp:237-245), on n threads, wall-clock timed
//   ref_random_scenario     testutil::random_scenario (tests/helpers.hpp:42-101)
//   ref_sample_scenario     coinfer::sample_scenario + profile_heavy/light
//       (scenario_gen.hpp:113-216), seeded like the CLI (coinfer_main.cpp:47-50)
//   ref_online_episode      run_episode(OnlineEnv, TimeWindowPolicy) (online_sim.hpp)
//   ref_schedule_batch      the Schedule ip_ssa / og return, in the product's
//       SoA schedule layout (coinfer_schedule_out)
//   ref_baseline_batch      baseline(sc, BaselineMode) + its Schedule
//   ref_validate_batch      validate(Schedule, Scenario, tol) as counts per constraint id

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <thread>
#include <vector>

#include "coinfer/ddpg.hpp"
#include "coinfer/offline_solvers.hpp"
#include "coinfer/online_sim.hpp"
#include "coinfer/oracles.hpp"
#include "coinfer/scenario_gen.hpp"
#include "helpers.hpp"

#include "../include/coinfer_b200.h"

using namespace coinfer;

namespace {

DnnProfile make_profile(const coinfer_profile* p) {
  DnnProfile d;
  d.work.assign(p->work, p->work + p->N);
  d.data_bits.assign(p->data_bits, p->data_bits + p->N + 1);
  for (int n = 0; n < p->N; ++n)
    d.latency.emplace_back(p->latency + (size_t)n * p->b_max, p->latency + (size_t)(n + 1) * p->b_max);
  return d;
}

Scenario make_scenario(const DnnProfile& prof, const coinfer_users* u, int64_t k) {
  Scenario sc;
  sc.profile = prof;
  const size_t o = (size_t)k * u->M;
  for (int m = 0; m < u->M; ++m) {
    UserSpec s;
    s.f_min = u->f_min[o + m];
    s.f_max = u->f_max[o + m];
    s.kappa = u->kappa[o + m];
    s.rate_up = u->rate_up[o + m];
    s.rate_down = u->rate_down ? u->rate_down[o + m] : s.rate_up;
    s.power_up = u->power_up[o + m];
    s.power_down = u->power_down ? u->power_down[o + m] : s.power_up;
    s.arrival = u->arrival[o + m];
    sc.users.push_back(s);
    sc.deadline.push_back(u->deadline[o + m]);
  }
  return sc;
}

int status_of_invalid(const std::string& what) {
  if (what == "scenario: bad frequency range") return COINFER_ST_BAD_FREQ;
  if (what == "scenario: negative kappa") return COINFER_ST_NEG_KAPPA;
  if (what == "scenario: rates must be positive") return COINFER_ST_BAD_RATE;
  if (what == "scenario: negative link power") return COINFER_ST_NEG_POWER;
  if (what == "scenario: negative arrival") return COINFER_ST_NEG_ARRIVAL;
  if (what == "scenario: deadline before arrival") return COINFER_ST_EARLY_DEADLINE;
  if (what == "scenario: latency table shorter than user count") return COINFER_ST_SHORT_TABLE;
  if (what == "batch_start_times: b must be >= 1") return COINFER_ST_ZERO_BOUND;
  return -1;
}

void write_solve(const SolveResult& r, const Scenario& sc, int64_t k, int M, int N,
                 coinfer_ipssa_out* out) {
  if (out->batch_bound) out->batch_bound[k] = (int32_t)r.batch_bound;
  if (out->pipeline_feasible) out->pipeline_feasible[k] = r.pipeline_feasible;
  if (out->energy) out->energy[k] = r.energy;
  const ScheduleMetrics met = M ? schedule_metrics(r.schedule, sc) : ScheduleMetrics{};
  for (int m = 0; m < M; ++m) {
    const size_t x = (size_t)k * M + m;
    if (out->split) out->split[x] = (uint8_t)r.split[m];
    if (out->freq) out->freq[x] = r.schedule.freq[m];
    if (out->user_energy) out->user_energy[x] = met.per_user_energy[m];
  }
  if (out->batch_size)
    for (int n = 0; n < N; ++n)
      out->batch_size[(size_t)k * N + n] = r.batch_size.empty() ? 0 : (int32_t)r.batch_size[n];
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const std::domain_error&) {
    return COINFER_ST_INFEASIBLE;
  } catch (const std::out_of_range&) {
    return COINFER_ST_BOUND_PAST_TABLE;
  } catch (const std::invalid_argument& e) {
    return status_of_invalid(e.what());
  }
}

int og_into(const Scenario& sc, int64_t k, int M, int N, coinfer_og_out* out) {
  const GroupingPlan plan = og(sc);
  if (out->fallback) out->fallback[k] = plan.fallback;
  if (out->energy) out->energy[k] = plan.energy;
  if (out->n_groups) out->n_groups[k] = (int32_t)plan.groups.size();
  std::vector<size_t> order(M);
  for (int m = 0; m < M; ++m) order[m] = m;
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return std::tie(sc.deadline[a], a) < std::tie(sc.deadline[b], b);
  });
  std::vector<int> pos(M);
  for (int i = 0; i < M; ++i) pos[order[i]] = i;
  if (out->order)
    for (int i = 0; i < M; ++i) out->order[(size_t)k * M + i] = (int32_t)order[i];
  const ScheduleMetrics met = M ? schedule_metrics(plan.schedule, sc) : ScheduleMetrics{};
  for (size_t g = 0; g < plan.groups.size(); ++g) {
    const auto& ids = plan.groups[g];
    const size_t gi = (size_t)k * M + g;
    if (out->group_lo) out->group_lo[gi] = pos[ids[0]];
    if (out->group_size) out->group_size[gi] = (int32_t)ids.size();
    if (out->group_deadline) out->group_deadline[gi] = plan.group_deadline[g];
    if (out->group_energy) out->group_energy[gi] = plan.group_energy[g];
    // batch bound and sizes of the group's own solve (the reference keeps
    // them only transiently; recompute the identical call og makes)
    int32_t bb = 0;
    std::vector<size_t> bs(N, 0);
    if (!plan.fallback) {
      const Scenario sub = detail::subscenario(sc, ids);
      const SolveResult r = *detail::try_ip_ssa(sub, plan.group_deadline[g]);
      bb = (int32_t)r.batch_bound;
      for (int n = 0; n < N; ++n) bs[n] = r.batch_size[n];
    }
    if (out->group_b) out->group_b[gi] = bb;
    if (out->group_batch_size)
      for (int n = 0; n < N; ++n) out->group_batch_size[gi * N + n] = (int32_t)bs[n];
    for (size_t id : ids)
      if (out->group_of_user) out->group_of_user[(size_t)k * M + id] = (int32_t)g;
  }
  for (int m = 0; m < M; ++m) {
    const size_t x = (size_t)k * M + m;
    size_t split = N;
    for (int n = 0; n < N; ++n)
      if (plan.schedule.x[m][n] != kLocal) {
        split = n;
        break;
      }
    if (out->split) out->split[x] = (uint8_t)split;
    if (out->freq) out->freq[x] = plan.schedule.freq[m];
    if (out->user_energy) out->user_energy[x] = met.per_user_energy[m];
  }
  return COINFER_ST_OK;
}

void write_schedule(const Schedule& s, int64_t k, int M, int N, coinfer_schedule_out* o) {
  o->n_batches[k] = (int32_t)s.batch_start.size();
  for (size_t i = 0; i < s.batch_start.size(); ++i) o->batch_start[(size_t)k * M * N + i] = s.batch_start[i];
  for (int m = 0; m < M; ++m) {
    o->freq[(size_t)k * M + m] = s.freq[m];
    for (int n = 0; n < N; ++n) o->x[((size_t)k * M + m) * N + n] = (int32_t)s.x[m][n];
    for (int n = 0; n <= N; ++n) o->completion[((size_t)k * M + m) * (N + 1) + n] = s.completion[m][n];
  }
}

}  // namespace

extern "C" {

// kind 0: ip_ssa(sc, deadline[k] or the smallest deadline); kind 1: og(sc).
// Returns per-instance statuses in status[k].
int ref_schedule_batch(const coinfer_profile* p, const coinfer_users* u, const double* deadline,
                       int kind, int32_t* status, coinfer_schedule_out* out) {
  const DnnProfile prof = make_profile(p);
  for (int64_t k = 0; k < u->n_inst; ++k) {
    const Scenario sc = make_scenario(prof, u, k);
    status[k] = guarded([&] {
      if (kind == 0) {
        double l = kInf;
        for (double d : sc.deadline) l = std::min(l, d);
        write_schedule(ip_ssa(sc, deadline ? deadline[k] : l).schedule, k, u->M, p->N, out);
      } else {
        write_schedule(og(sc).schedule, k, u->M, p->N, out);
      }
      return 0;
    });
  }
  return COINFER_OK;
}

int ref_validate_batch(const coinfer_profile* p, const coinfer_users* u,
                       const coinfer_schedule_out* sc_in, double tol, int32_t* status,
                       int32_t* counts, double* min_slack) {
  static const char* ids[COINFER_N_CONSTRAINTS] = {"C7-batchsize", "C8-samesubtask", "C9-batchready",
                                                   "C11-occupancy", "C12-precedence", "C15-deadline",
                                                   "C17-initial"};
  const DnnProfile prof = make_profile(p);
  const int M = u->M, N = p->N;
  for (int64_t k = 0; k < u->n_inst; ++k) {
    const Scenario sc = make_scenario(prof, u, k);
    Schedule s;
    s.x.assign(M, std::vector<std::size_t>(N));
    s.completion.assign(M, std::vector<double>(N + 1));
    for (int m = 0; m < M; ++m) {
      for (int n = 0; n < N; ++n) s.x[m][n] = (std::size_t)sc_in->x[((size_t)k * M + m) * N + n];
      for (int n = 0; n <= N; ++n) s.completion[m][n] = sc_in->completion[((size_t)k * M + m) * (N + 1) + n];
      s.freq.push_back(sc_in->freq[(size_t)k * M + m]);
    }
    for (int i = 0; i < sc_in->n_batches[k]; ++i) s.batch_start.push_back(sc_in->batch_start[(size_t)k * M * N + i]);
    for (int c = 0; c < COINFER_N_CONSTRAINTS; ++c) counts[(size_t)k * COINFER_N_CONSTRAINTS + c] = 0;
    double worst = 0.0;
    try {
      for (const Violation& v : validate(s, sc, tol)) {
        for (int c = 0; c < COINFER_N_CONSTRAINTS; ++c)
          if (v.constraint_id == ids[c]) ++counts[(size_t)k * COINFER_N_CONSTRAINTS + c];
        worst = v.slack < worst ? v.slack : worst;
      }
      status[k] = COINFER_ST_OK;
    } catch (const std::invalid_argument&) {
      status[k] = COINFER_ST_BAD_BATCH_ID;
    } catch (const std::out_of_range&) {
      status[k] = COINFER_ST_BOUND_PAST_TABLE;
    } catch (const std::domain_error&) {
      status[k] = COINFER_ST_NONPOS_FREQ;
    }
    if (min_slack) min_slack[k] = status[k] == COINFER_ST_OK ? worst : 0.0;
  }
  return COINFER_OK;
}

int ref_baseline_batch(const coinfer_profile* p, const coinfer_users* u, int mode,
                       coinfer_ipssa_out* out, coinfer_schedule_out* sched) {
  const DnnProfile prof = make_profile(p);
  try {
    prof.check();
  } catch (const std::invalid_argument&) {
    return COINFER_E_PROFILE;
  }
  for (int64_t k = 0; k < u->n_inst; ++k) {
    const Scenario sc = make_scenario(prof, u, k);
    const int st = guarded([&] {
      const SolveResult r = baseline(sc, (BaselineMode)mode);
      write_solve(r, sc, k, u->M, p->N, out);
      if (sched) write_schedule(r.schedule, k, u->M, p->N, sched);
      return 0;
    });
    if (out->status) out->status[k] = st;
  }
  return COINFER_OK;
}


int ref_ipssa_batch(const coinfer_profile* p, const coinfer_users* u, const double* deadline,
                    coinfer_ipssa_out* out) {
  const DnnProfile prof = make_profile(p);
  try {
    prof.check();
  } catch (const std::invalid_argument&) {
    return COINFER_E_PROFILE;
  }
  for (int64_t k = 0; k < u->n_inst; ++k) {
    const Scenario sc = make_scenario(prof, u, k);
    const int st = guarded([&] {
      double l = deadline ? deadline[k] : (u->M ? sc.deadline[0] : 0.0);
      if (!deadline)
        for (double d : sc.deadline) l = std::min(l, d);
      const SolveResult r = ip_ssa(sc, l);
      write_solve(r, sc, k, u->M, p->N, out);
      return COINFER_ST_OK;
    });
    if (out->status) out->status[k] = st;
  }
  return COINFER_OK;
}

int ref_fixed_batch(const coinfer_profile* p, const coinfer_users* u, const double* deadline,
                    const int32_t* b, coinfer_ipssa_out* out) {
  const DnnProfile prof = make_profile(p);
  try {
    prof.check();
  } catch (const std::invalid_argument&) {
    return COINFER_E_PROFILE;
  }
  for (int64_t k = 0; k < u->n_inst; ++k) {
    const Scenario sc = make_scenario(prof, u, k);
    const int st = guarded([&] {
      double l = deadline ? deadline[k] : (u->M ? sc.deadline[0] : 0.0);
      if (!deadline)
        for (double d : sc.deadline) l = std::min(l, d);
      const SolveResult r = fixed_batch_schedule(sc, l, (size_t)b[k]);
      write_solve(r, sc, k, u->M, p->N, out);
      return COINFER_ST_OK;
    });
    if (out->status) out->status[k] = st;
  }
  return COINFER_OK;
}

int ref_og_batch(const coinfer_profile* p, const coinfer_users* u, coinfer_og_out* out) {
  const DnnProfile prof = make_profile(p);
  try {
    prof.check();
  } catch (const std::invalid_argument&) {
    return COINFER_E_PROFILE;
  }
  for (int64_t k = 0; k < u->n_inst; ++k) {
    const Scenario sc = make_scenario(prof, u, k);
    const int st = guarded([&] { return og_into(sc, k, u->M, p->N, out); });
    if (out->status) out->status[k] = st;
  }
  return COINFER_OK;
}

// Brute-force oracles (oracles.hpp), for the Theorem 1/2 parity tests.
double ref_oracle_grouping_contiguous(const coinfer_profile* p, const coinfer_users* u, int64_t k,
                                      int32_t* n_groups) {
  const Scenario sc = make_scenario(make_profile(p), u, k);
  const GroupingOracle o = oracle_grouping_contiguous(sc);
  *n_groups = o.feasible ? (int32_t)o.groups.size() : -1;
  return o.energy;
}

// oracle_structured with outputs; the group ids of the grouping oracles
// (index of the user's group in the oracle's rising-deadline order).
double ref_oracle_structured(const coinfer_profile* p, const coinfer_users* u, int64_t k,
                             double deadline, int32_t b, uint8_t* split, uint8_t* fallback,
                             uint8_t* feasible) {
  const Scenario sc = make_scenario(make_profile(p), u, k);
  const StructuredOracle o = oracle_structured(sc, deadline, (std::size_t)b);
  *fallback = o.fallback;
  *feasible = o.feasible;
  for (int m = 0; m < u->M; ++m) split[m] = o.feasible ? (uint8_t)o.split[m] : 0;
  return o.energy;
}

double ref_oracle_groups(const coinfer_profile* p, const coinfer_users* u, int64_t k, int contiguous,
                         int32_t* n_groups, int32_t* group_of_user) {
  const Scenario sc = make_scenario(make_profile(p), u, k);
  const GroupingOracle o = contiguous ? oracle_grouping_contiguous(sc) : oracle_grouping(sc);
  *n_groups = o.feasible ? (int32_t)o.groups.size() : 0;
  if (o.feasible)
    for (std::size_t g = 0; g < o.groups.size(); ++g)
      for (std::size_t m : o.groups[g]) group_of_user[m] = (int32_t)g;
  return o.energy;
}

double ref_oracle_grouping(const coinfer_profile* p, const coinfer_users* u, int64_t k,
                           int32_t* n_groups) {
  const Scenario sc = make_scenario(make_profile(p), u, k);
  const GroupingOracle o = oracle_grouping(sc);
  *n_groups = o.feasible ? (int32_t)o.groups.size() : -1;
  return o.energy;
}

// The CLI's IPSSA + OG pair on every listed instance, spread over n_threads
// workers (the solvers are pure and reentrant).  Returns wall
// seconds of the solve loop; energies written for cross-checking.
double ref_sweep_threads(const coinfer_profile* p, const coinfer_users* u, const int64_t* idx,
                         int64_t count, int n_threads, int do_ipssa, int do_og,
                         double* ipssa_energy, double* og_energy) {
  const DnnProfile prof = make_profile(p);
  std::vector<Scenario> scs;
  scs.reserve(count);
  for (int64_t c = 0; c < count; ++c) scs.push_back(make_scenario(prof, u, idx[c]));
  std::atomic<int64_t> next{0};
  auto worker = [&] {
    for (int64_t c; (c = next.fetch_add(1)) < count;) {
      const Scenario& sc = scs[c];
      if (do_ipssa) {
        double l = sc.deadline[0];
        for (double d : sc.deadline) l = std::min(l, d);
        try {
          ipssa_energy[c] = ip_ssa(sc, l).energy;
        } catch (const std::exception&) {
          ipssa_energy[c] = -1.0;
        }
      }
      if (do_og) {
        try {
          og_energy[c] = og(sc).energy;
        } catch (const std::exception&) {
          og_energy[c] = -1.0;
        }
      }
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < n_threads; ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  const std::chrono::duration<double> dt = std::chrono::steady_clock::now() - t0;
  return dt.count();
}

// ---------------------------------------------------------------- inputs --

uint64_t ref_mix_seed(uint64_t root, uint64_t salt) { return testutil::mix_seed(root, salt); }

uint64_t ref_sub_seed(uint64_t root, uint64_t component, uint64_t index) {
  // coinfer_main.cpp:47-50
  return detail::mix64(detail::mix64(root ^ (component * 0x9e3779b97f4a7c15ull)) + index);
}

void* ref_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
uint64_t ref_rng_next(void* r) { return (*static_cast<std::mt19937_64*>(r))(); }
uint64_t ref_uniform_int(void* r, uint64_t lo, uint64_t hi) {
  std::uniform_int_distribution<std::size_t> d(lo, hi);
  return d(*static_cast<std::mt19937_64*>(r));
}
double ref_uniform_real(void* r, double lo, double hi) {
  std::uniform_real_distribution<double> d(lo, hi);
  return d(*static_cast<std::mt19937_64*>(r));
}

// testutil::random_scenario; profile arrays sized N, N+1, N*(users+2).
void ref_random_scenario(void* r, int users, int subtasks, double growth_max, int equal_deadlines,
                         double margin_max, double* work, double* bits, double* lat, double* fmin,
                         double* fmax, double* kappa, double* ru, double* pu, double* arr,
                         double* dl) {
  const Scenario sc = testutil::random_scenario(*static_cast<std::mt19937_64*>(r), users, subtasks,
                                                growth_max, equal_deadlines != 0, margin_max);
  const size_t bmax = sc.profile.max_batch();
  for (int n = 0; n < subtasks; ++n) {
    work[n] = sc.profile.work[n];
    for (size_t b = 0; b < bmax; ++b) lat[n * bmax + b] = sc.profile.latency[n][b];
  }
  for (int n = 0; n <= subtasks; ++n) bits[n] = sc.profile.data_bits[n];
  for (int m = 0; m < users; ++m) {
    fmin[m] = sc.users[m].f_min;
    fmax[m] = sc.users[m].f_max;
    kappa[m] = sc.users[m].kappa;
    ru[m] = sc.users[m].rate_up;
    pu[m] = sc.users[m].power_up;
    arr[m] = sc.users[m].arrival;
    dl[m] = sc.deadline[m];
  }
}

// profile_heavy / profile_light at b_max (scenario_gen.hpp:208-216).
void ref_profile(int heavy, int b_max, double* work, double* bits, double* lat) {
  const DnnProfile p = heavy ? profile_heavy(b_max) : profile_light(b_max);
  for (int n = 0; n < 4; ++n) {
    work[n] = p.work[n];
    for (int b = 0; b < b_max; ++b) lat[n * b_max + b] = p.latency[n][b];
  }
  for (int n = 0; n <= 4; ++n) bits[n] = p.data_bits[n];
}

// sample_scenario with ScenarioConfig defaults, users=M, deadlines fixed
// (lo == hi) or uniform [lo, hi], rng = mt19937_64(seed).  Writes one
// instance of the SoA arrays (plus rate_down/power_down).
int ref_sample_scenario(int heavy, int M, double lo, double hi, double bandwidth, uint64_t seed,
                        double* fmin, double* fmax, double* kappa, double* ru, double* pu,
                        double* arr, double* dl, double* rd, double* pd) {
  ScenarioConfig cfg;
  cfg.users = M;
  cfg.bandwidth = bandwidth;
  cfg.deadline = lo == hi ? DeadlineSpec::fixed(lo) : DeadlineSpec::uniform(lo, hi);
  std::mt19937_64 rng(seed);
  try {
    const GeneratedScenario g =
        sample_scenario(cfg, heavy ? profile_heavy(M) : profile_light(M), rng);
    for (int m = 0; m < M; ++m) {
      const UserSpec& u = g.scenario.users[m];
      fmin[m] = u.f_min;
      fmax[m] = u.f_max;
      kappa[m] = u.kappa;
      ru[m] = u.rate_up;
      pu[m] = u.power_up;
      arr[m] = u.arrival;
      dl[m] = g.scenario.deadline[m];
      if (rd) rd[m] = u.rate_down;
      if (pd) pd[m] = u.power_down;
    }
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

// One episode of run_episode(OnlineEnv(sample_scenario(users=M, fixed(l_high)),
// ArrivalModel{Bernoulli, p, [l_low, l_high]}, solver, slot, seed),
// TimeWindowPolicy(window, threshold) or local_policy (window < 0), horizon) — the CLI's online path
// (coinfer_main.cpp:482-573).  Scenario given as SoA (one instance).
// trace arrays (may be NULL) get per-slot reward, energy, pending, busy.
int ref_online_episode(const coinfer_profile* p, const coinfer_users* u, int solver_og,
                       double p_arrive, int immediate, double l_low, double l_high, double slot,
                       uint64_t seed, int window, double threshold, int64_t horizon,
                       double* totals /*[4]*/,
                       int64_t* counts /*[6]*/, double* tr_reward, double* tr_energy,
                       int32_t* tr_pending, double* tr_busy) {
  try {
    const Scenario sc = make_scenario(make_profile(p), u, 0);
    ArrivalModel a;
    a.kind = immediate ? ArrivalModel::Kind::Immediate : ArrivalModel::Kind::Bernoulli;
    a.p_arrive = p_arrive;
    a.l_low = l_low;
    a.l_high = l_high;
    OnlineEnv env(sc, a, solver_og ? OnlineSolver::OG : OnlineSolver::IPSSA, slot, seed);
    // window < 0 selects local_policy (online_sim.hpp:301-307)
    const PolicyFn pol = window < 0 ? local_policy() : PolicyFn(TimeWindowPolicy(window, threshold));
    const EpisodeMetrics m = run_episode(env, pol, horizon, seed);
    totals[0] = m.total_energy;
    totals[1] = m.total_forced_cost;
    totals[2] = m.total_reward;
    totals[3] = m.mean_batch_size();
    counts[0] = m.forced_count;
    counts[1] = m.solver_calls;
    counts[2] = m.solver_tasks;
    counts[3] = m.solver_groups;
    counts[4] = m.batches;
    counts[5] = m.batched_tasks;
    for (size_t t = 0; t < m.trace.size(); ++t) {
      if (tr_reward) tr_reward[t] = m.trace[t].reward;
      if (tr_energy) tr_energy[t] = m.trace[t].energy;
      if (tr_pending) tr_pending[t] = (int32_t)m.trace[t].pending_count;
      if (tr_busy) tr_busy[t] = m.trace[t].edge_busy;
    }
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

}  // extern "C"
