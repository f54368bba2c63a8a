// coinfer/b200.hpp — glue between the drop-in C++ API (value types,
// exceptions) and the engine's C ABI (include/coinfer_b200.h: SoA arrays,
// status codes).  Link with -lcoinfer_b200 (paper_2206_06304_b200/).
//
// One engine context per host thread (the ABI's contract), created lazily
// on CUDA device $COINFER_DEVICE (default 0).  There is no CPU solver: if no
// GPU is present, the first solve throws std::runtime_error.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../coinfer_b200.h"
#include "core_model.hpp"
#include "schedule.hpp"

namespace coinfer {
namespace b200 {

class Context {
 public:
  explicit Context(int device) : ctx_(coinfer_ctx_create(device)) {
    if (!ctx_)
      throw std::runtime_error("coinfer: cannot create a B200 engine context on CUDA device " +
                               std::to_string(device) + " (the engine has no CPU path)");
  }
  ~Context() { coinfer_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  coinfer_ctx* get() const { return ctx_; }

 private:
  coinfer_ctx* ctx_;
};

inline Context& context() {
  static thread_local Context ctx([] {
    const char* d = std::getenv("COINFER_DEVICE");
    return d ? std::atoi(d) : 0;
  }());
  return ctx;
}

// Call-level return code -> the reference's exception family.
inline void check_call(int rc) {
  if (rc == COINFER_OK) return;
  const std::string msg = coinfer_last_error(context().get());
  if (rc == COINFER_E_ARG || rc == COINFER_E_PROFILE) throw std::invalid_argument(msg);
  throw std::runtime_error("coinfer engine: " + msg);
}

// Per-instance status -> the exception the reference solver would throw.
inline void check_status(int32_t st, const char* solver) {
  if (st == COINFER_ST_OK) return;
  const std::string msg = coinfer_status_message(st, solver);
  if (st == COINFER_ST_INFEASIBLE) throw std::domain_error(msg);
  if (st == COINFER_ST_BOUND_PAST_TABLE) throw std::out_of_range(msg);
  if (st == COINFER_ST_SLIPPED) throw std::logic_error(msg);
  throw std::invalid_argument(msg);
}

// A profile flattened for the ABI (latency row-major [n][b-1]).
struct FlatProfile {
  std::vector<double> latency;
  coinfer_profile view;
  explicit FlatProfile(const DnnProfile& p) {
    const std::size_t N = p.subtasks(), B = p.max_batch();
    latency.reserve(N * B);
    for (std::size_t n = 0; n < N; ++n) {
      if (p.latency[n].size() != B) throw std::invalid_argument("profile: ragged latency table");
      latency.insert(latency.end(), p.latency[n].begin(), p.latency[n].end());
    }
    view.N = (int32_t)N;
    view.b_max = (int32_t)B;
    view.work = p.work.data();
    view.data_bits = p.data_bits.data();
    view.latency = latency.data();
  }
};

// A batch of scenarios with one profile and one user count, as SoA host
// arrays (field[k*M + m]).
struct UserBatch {
  std::vector<double> f_min, f_max, kappa, rate_up, power_up, arrival, deadline, rate_down,
      power_down;
  coinfer_users view;
  UserBatch(const Scenario* const* sc, std::size_t K, std::size_t M) {
    for (auto* v : {&f_min, &f_max, &kappa, &rate_up, &power_up, &arrival, &deadline, &rate_down,
                    &power_down})
      v->resize(K * M);
    for (std::size_t k = 0; k < K; ++k) {
      const Scenario& s = *sc[k];
      for (std::size_t m = 0; m < M; ++m) {
        const UserSpec& u = s.users[m];
        const std::size_t i = k * M + m;
        f_min[i] = u.f_min;
        f_max[i] = u.f_max;
        kappa[i] = u.kappa;
        rate_up[i] = u.rate_up;
        power_up[i] = u.power_up;
        arrival[i] = u.arrival;
        deadline[i] = s.deadline[m];
        rate_down[i] = u.rate_down;
        power_down[i] = u.power_down;
      }
    }
    view.n_inst = (int64_t)K;
    view.M = (int32_t)M;
    view.mem = COINFER_MEM_HOST;
    view.f_min = f_min.data();
    view.f_max = f_max.data();
    view.kappa = kappa.data();
    view.rate_up = rate_up.data();
    view.power_up = power_up.data();
    view.arrival = arrival.data();
    view.deadline = deadline.data();
    view.rate_down = rate_down.data();
    view.power_down = power_down.data();
  }
};

// Output storage of a SolveResult batch (coinfer_ipssa_out + schedule).
struct SolveBuffers {
  std::vector<int32_t> status, batch_bound, batch_size;
  std::vector<uint8_t> pipe, split;
  std::vector<double> energy, freq, user_energy;
  coinfer_ipssa_out out;
  SolveBuffers(std::size_t K, std::size_t M, std::size_t N)
      : status(K), batch_bound(K), batch_size(K * N), pipe(K), split(K * M), energy(K),
        freq(K * M), user_energy(K * M) {
    out.status = status.data();
    out.batch_bound = batch_bound.data();
    out.pipeline_feasible = pipe.data();
    out.energy = energy.data();
    out.split = split.data();
    out.freq = freq.data();
    out.user_energy = user_energy.data();
    out.batch_size = batch_size.data();
  }
};

struct OgBuffers {
  std::vector<int32_t> status, n_groups, order, group_of_user, group_lo, group_size, group_b,
      group_batch_size;
  std::vector<uint8_t> fallback, split;
  std::vector<double> energy, freq, user_energy, group_deadline, group_energy;
  coinfer_og_out out;
  OgBuffers(std::size_t K, std::size_t M, std::size_t N)
      : status(K), n_groups(K), order(K * M), group_of_user(K * M), group_lo(K * M),
        group_size(K * M), group_b(K * M), group_batch_size(K * M * N), fallback(K), split(K * M),
        energy(K), freq(K * M), user_energy(K * M), group_deadline(K * M), group_energy(K * M) {
    out.status = status.data();
    out.fallback = fallback.data();
    out.energy = energy.data();
    out.n_groups = n_groups.data();
    out.order = order.data();
    out.group_of_user = group_of_user.data();
    out.split = split.data();
    out.freq = freq.data();
    out.user_energy = user_energy.data();
    out.group_lo = group_lo.data();
    out.group_size = group_size.data();
    out.group_b = group_b.data();
    out.group_deadline = group_deadline.data();
    out.group_energy = group_energy.data();
    out.group_batch_size = group_batch_size.data();
  }
};

struct ScheduleBuffers {
  std::size_t M, N;
  std::vector<int32_t> x, n_batches;
  std::vector<double> batch_start, completion, freq;
  coinfer_schedule_out out;
  ScheduleBuffers(std::size_t K, std::size_t M_, std::size_t N_)
      : M(M_), N(N_), x(K * M_ * N_), n_batches(K), batch_start(K * M_ * N_),
        completion(K * M_ * (N_ + 1)), freq(K * M_) {
    out.x = x.data();
    out.n_batches = n_batches.data();
    out.batch_start = batch_start.data();
    out.completion = completion.data();
    out.freq = freq.data();
  }
  // The device-built Schedule of instance k as the reference's value type.
  Schedule take(std::size_t k) const {
    Schedule s;
    s.x.assign(M, std::vector<std::size_t>(N));
    s.completion.assign(M, std::vector<double>(N + 1));
    s.freq.assign(freq.begin() + k * M, freq.begin() + (k + 1) * M);
    for (std::size_t m = 0; m < M; ++m) {
      for (std::size_t n = 0; n < N; ++n) s.x[m][n] = (std::size_t)x[(k * M + m) * N + n];
      for (std::size_t n = 0; n <= N; ++n) s.completion[m][n] = completion[(k * M + m) * (N + 1) + n];
    }
    const std::size_t nb = (std::size_t)n_batches[k];
    s.batch_start.assign(batch_start.begin() + k * M * N, batch_start.begin() + k * M * N + nb);
    return s;
  }
};

}  // namespace b200
}  // namespace coinfer
