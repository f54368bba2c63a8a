/*
 * coinfer_b200.h — C ABI of the B200 solver engine for the offloading and
 * scheduling hot path of arXiv 2206.06304 (IP-SSA, same-sub-task
 * aggregation, OG optimal grouping, online slot driver).
 *
 * The reference is a header-only C++ library (namespace `coinfer`, value
 * semantics, exceptions).  This ABI is what a foreign caller binds instead:
 * plain pointers and sizes, structure-of-arrays fp64 inputs, integer status
 * codes, no exceptions and no C++ or torch types.  The C++ drop-in layer in
 * include/coinfer/ rebuilds the reference's value types on top of it and
 * rethrows the reference's exceptions.
 *
 * Reference interfaces replaced (all under /root/reference/proj/include/coinfer):
 *   coinfer_ipssa_batch   <- ip_ssa(const Scenario&, double)           offline_solvers.hpp:219-224
 *                            detail::try_ip_ssa                          offline_solvers.hpp:192-204
 *   coinfer_fixed_batch   <- fixed_batch_schedule(const Scenario&, double, size_t)
 *                                                                       offline_solvers.hpp:208-214
 *                            detail::try_fixed_batch (+ aggregation)     offline_solvers.hpp:137-188
 *   coinfer_og_batch      <- og(const Scenario&)                         offline_solvers.hpp:286-388
 *                            detail::lc_solve (OG fallback)              offline_solvers.hpp:255-276
 *   coinfer_sweep_batch   <- the CLI's per-instance pair of solves
 *                            run_offline_solver("IPSSA"/"OG")           tools/coinfer_main.cpp:237-245
 *   (per-user energies)   <- schedule_metrics(...).per_user_energy      offline_solvers.hpp:627-646
 *   (contract checks)     <- Scenario::check / DnnProfile::check        core_model.hpp:31-52,80-101
 *   coinfer_ipssa_schedule / coinfer_og_schedule
 *                         <- the Schedule built by try_fixed_batch / og + normalize
 *                                                                       offline_solvers.hpp:155-185,357-386
 *                                                                       schedule.hpp:93-113
 *   coinfer_baseline_batch <- baseline(const Scenario&, BaselineMode)   offline_solvers.hpp:390-612
 *   coinfer_validate_batch <- validate(const Schedule&, const Scenario&, double) schedule.hpp:139-209
 *   coinfer_sample_batch  <- sample_scenario(cfg, profile, rng)        scenario_gen.hpp:113-173
 *   coinfer_oracle_*_batch <- oracle_structured / oracle_grouping(_contiguous) oracles.hpp:28-225
 *   coinfer_best_partition <- best_partition / detail::local_only_choice offline_solvers.hpp:62-117
 *   coinfer_online_run    <- run_episode(OnlineEnv&, TimeWindowPolicy, horizon, seed)
 *                                                                       online_sim.hpp:131-249,312-371
 *
 * Threading: a context owns one CUDA stream and its workspace; calls on one
 * context must be serialised by the caller (the reference solvers are pure
 * and reentrant; use one context per host thread).
 *
 * Memory: every array in coinfer_users and the output structs is either all
 * host memory or all device memory of the context's GPU, selected by
 * coinfer_users.mem.  Host inputs are copied in and outputs copied back
 * inside the call (synchronously); device arrays are used in place and the
 * call only enqueues work on the context stream (call coinfer_ctx_synchronize
 * before reading results).  Profile arrays are always host memory.
 * Any output pointer may be NULL: that output is then not produced.
 */
#ifndef COINFER_B200_H
#define COINFER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COINFER_ABI_VERSION 3

/* Call-level return codes. */
#define COINFER_OK 0
#define COINFER_E_ARG 1         /* null/ill-shaped argument (std::invalid_argument) */
#define COINFER_E_PROFILE 2     /* DnnProfile::check failed; message in coinfer_last_error */
#define COINFER_E_CUDA 3        /* CUDA runtime error; message in coinfer_last_error */
#define COINFER_E_UNSUPPORTED 4 /* shape outside what the kernels were built for */

/* Per-instance status codes (out->status[k]). */
#define COINFER_ST_OK 0
#define COINFER_ST_INFEASIBLE 1 /* std::domain_error (see coinfer_status_message) */
/* std::invalid_argument from Scenario::check, first failing user, first failing test
   (core_model.hpp:90-99, in that order) */
#define COINFER_ST_BAD_FREQ 10      /* "scenario: bad frequency range" */
#define COINFER_ST_NEG_KAPPA 11     /* "scenario: negative kappa" */
#define COINFER_ST_BAD_RATE 12      /* "scenario: rates must be positive" */
#define COINFER_ST_NEG_POWER 13     /* "scenario: negative link power" */
#define COINFER_ST_NEG_ARRIVAL 14   /* "scenario: negative arrival" */
#define COINFER_ST_EARLY_DEADLINE 15 /* "scenario: deadline before arrival" */
#define COINFER_ST_SHORT_TABLE 16   /* "scenario: latency table shorter than user count" */
#define COINFER_ST_ZERO_BOUND 17    /* b == 0: "batch_start_times: b must be >= 1" (invalid_argument) */
#define COINFER_ST_BOUND_PAST_TABLE 18 /* b > b_max: std::out_of_range "edge_batch_latency: batch size beyond table" */

/* online driver (OnlineEnv, online_sim.hpp) */
#define COINFER_ST_NOT_RELEASED 20     /* "online: users must be released at time zero" */
#define COINFER_ST_FLOOR_ABOVE_LLOW 21 /* "online: l_low below a user's all-local floor" */
#define COINFER_ST_SLIPPED 22          /* std::logic_error "online: task slipped below its local floor" */

#define COINFER_MEM_HOST 0
#define COINFER_MEM_DEVICE 1

/* Largest sub-task count N the kernels are instantiated for. */
#define COINFER_MAX_SUBTASKS 16

typedef struct coinfer_ctx coinfer_ctx;

/* DnnProfile (core_model.hpp:17-53).  latency is row-major [n][b-1]:
   latency[(n-1)*b_max + (b-1)] = F_n(b).  Host memory. */
typedef struct coinfer_profile {
  int32_t N;
  int32_t b_max;
  const double* work;      /* [N]        A_n                 */
  const double* data_bits; /* [N+1]      B_0..B_N            */
  const double* latency;   /* [N*b_max]  F_n(b)              */
} coinfer_profile;

/* A batch of n_inst independent scenarios, each with M users, stored as
   structure of arrays: field[k*M + m] is user m of instance k (UserSpec,
   core_model.hpp:56-66, plus Scenario::deadline).  rate_down/power_down are
   read only by the contract check and may be NULL (treated as valid). */
typedef struct coinfer_users {
  int64_t n_inst;
  int32_t M;
  int32_t mem; /* COINFER_MEM_HOST or COINFER_MEM_DEVICE, for inputs and outputs */
  const double* f_min;
  const double* f_max;
  const double* kappa;
  const double* rate_up;
  const double* power_up;
  const double* arrival;
  const double* deadline;
  const double* rate_down;  /* optional */
  const double* power_down; /* optional */
} coinfer_users;

/* SolveResult (offline_solvers.hpp:119-126) in SoA form, plus the per-user
   energies of schedule_metrics (offline_solvers.hpp:627-646). */
typedef struct coinfer_ipssa_out {
  int32_t* status;           /* [n_inst] COINFER_ST_*                                  */
  int32_t* batch_bound;      /* [n_inst] SolveResult::batch_bound                      */
  uint8_t* pipeline_feasible;/* [n_inst] SolveResult::pipeline_feasible                */
  double* energy;            /* [n_inst] SolveResult::energy (total_energy fold)       */
  uint8_t* split;            /* [n_inst*M] SolveResult::split                          */
  double* freq;              /* [n_inst*M] Schedule::freq (f_max placeholder, split 0) */
  double* user_energy;       /* [n_inst*M] ScheduleMetrics::per_user_energy            */
  int32_t* batch_size;       /* [n_inst*N] SolveResult::batch_size                     */
} coinfer_ipssa_out;

/* GroupingPlan (offline_solvers.hpp:234-241) in SoA form.  Groups are listed
   in rising-deadline order g = 0..n_groups-1; group g holds the sorted users
   order[group_lo[g] .. group_lo[g]+group_size[g]-1].  Per-group arrays have
   capacity M per instance. */
typedef struct coinfer_og_out {
  int32_t* status;          /* [n_inst]                                               */
  uint8_t* fallback;        /* [n_inst] GroupingPlan::fallback                        */
  double* energy;           /* [n_inst] GroupingPlan::energy                          */
  int32_t* n_groups;        /* [n_inst] groups.size()                                 */
  int32_t* order;           /* [n_inst*M] users sorted by (deadline, id)              */
  int32_t* group_of_user;   /* [n_inst*M] group index of original user m              */
  uint8_t* split;           /* [n_inst*M] split of original user m in the plan        */
  double* freq;             /* [n_inst*M] Schedule::freq of user m                    */
  double* user_energy;      /* [n_inst*M] per_user_energy of user m                   */
  int32_t* group_lo;        /* [n_inst*M] first sorted index of group g               */
  int32_t* group_size;      /* [n_inst*M] member count of group g                     */
  int32_t* group_b;         /* [n_inst*M] batch bound the group was solved with (0 in fallback) */
  double* group_deadline;   /* [n_inst*M] GroupingPlan::group_deadline                */
  double* group_energy;     /* [n_inst*M] GroupingPlan::group_energy                  */
  int32_t* group_batch_size;/* [n_inst*M*N] realized batch size per sub-task per group */
} coinfer_og_out;

/* Schedule (schedule.hpp:26-36) in SoA form, normalised like
   coinfer::normalize (schedule.hpp:93-113): batch ids 1..n_batches ordered by
   (start time, sub-task).  x[(k*M + m)*N + n-1] is the placement of sub-task
   n of user m (0 = local, COINFER kLocal); batch_start has capacity M*N per
   instance; completion[(k*M + m)*(N+1) + n] = t_{m,n}. */
typedef struct coinfer_schedule_out {
  int32_t* x;           /* [n_inst*M*N]      */
  int32_t* n_batches;   /* [n_inst]          */
  double* batch_start;  /* [n_inst*M*N]      */
  double* completion;   /* [n_inst*M*(N+1)]  */
  double* freq;         /* [n_inst*M]        */
} coinfer_schedule_out;

/* Offline comparison baselines (BaselineMode, offline_solvers.hpp:390-612). */
#define COINFER_BASELINE_LC 0       /* detail::lc_solve        :255-276 */
#define COINFER_BASELINE_PS 1       /* detail::ps_solve        :404-487 */
#define COINFER_BASELINE_FIFO 2     /* detail::fifo_solve      :489-555 */
#define COINFER_BASELINE_IPSSA_NP 3 /* detail::ipssa_np_solve  :560-600 */

/* Online slot driver: run_episode(OnlineEnv(scenario, ArrivalModel, solver,
   slot, seed), policy, horizon, seed) (online_sim.hpp:69-371), one episode
   per seed.  Policies: the fixed TimeWindowPolicy(window, l_high) and
   local_policy (DDPG is out of scope). */
#define COINFER_ARRIVAL_BERNOULLI 0
#define COINFER_ARRIVAL_IMMEDIATE 1
#define COINFER_SOLVER_IPSSA 0
#define COINFER_SOLVER_OG 1
#define COINFER_POLICY_TW 0
#define COINFER_POLICY_LOCAL 1

typedef struct coinfer_online_cfg {
  int32_t arrival;  /* COINFER_ARRIVAL_*  (ArrivalModel::kind)   */
  int32_t solver;   /* COINFER_SOLVER_*   (OnlineSolver)         */
  int32_t policy;   /* COINFER_POLICY_*                          */
  int32_t window;   /* TimeWindowPolicy window, in slots          */
  double p_arrive;  /* ArrivalModel::p_arrive                     */
  double l_low;     /* ArrivalModel::l_low                        */
  double l_high;    /* ArrivalModel::l_high (also the TW threshold) */
  double slot;      /* slot length, seconds                       */
  double threshold; /* TimeWindowPolicy threshold (the CLI uses l_high) */
  int64_t horizon;  /* slots per episode                          */
} coinfer_online_cfg;

/* EpisodeMetrics (online_sim.hpp:274-296) per episode, plus an optional
   per-slot trace (TraceRow reward / energy / pending_count / edge_busy) for
   the first n_trace episodes. */
typedef struct coinfer_online_out {
  int32_t* status;  /* [n_ep] COINFER_ST_*                                   */
  double* totals;   /* [n_ep*3] total_energy, total_forced_cost, total_reward */
  int64_t* counts;  /* [n_ep*6] forced_count, solver_calls, solver_tasks,
                       solver_groups, batches, batched_tasks                 */
  int64_t n_trace;
  double* trace_reward;      /* [n_trace*horizon] */
  double* trace_energy;      /* [n_trace*horizon] */
  int32_t* trace_pending;    /* [n_trace*horizon] */
  double* trace_edge_busy;   /* [n_trace*horizon] */
  /* optional (NULL: not written) */
  int32_t* trace_action;     /* [n_trace*horizon] TraceRow::action_c, the policy's mode */
  int32_t* trace_forced;     /* [n_trace*horizon] TraceRow::forced_count */
  double* final_state;       /* [n_ep*(2*M+1)] OnlineEnv state after the last slot:
                                MdpState::deadline[M], expiry_[M], MdpState::edge_busy */
  int64_t* draws;            /* [n_ep] mt19937_64 outputs consumed (rng_ = seed, discard(draws)) */
} coinfer_online_out;

int coinfer_abi_version(void);

/* Context: one CUDA device, one stream, a workspace.  NULL on failure. */
coinfer_ctx* coinfer_ctx_create(int device);
void coinfer_ctx_destroy(coinfer_ctx* ctx);
/* Enqueue on an existing cudaStream_t (passed as void*; NULL is the legacy
   default stream, as in CUDA) instead of the context's private stream. */
int coinfer_ctx_set_stream(coinfer_ctx* ctx, void* stream);
/* Go back to the context's private stream. */
int coinfer_ctx_reset_stream(coinfer_ctx* ctx);
int coinfer_ctx_synchronize(coinfer_ctx* ctx);
/* Message of the last call-level error on this context ("" if none). */
const char* coinfer_last_error(const coinfer_ctx* ctx);
/* The reference's exception message for a per-instance status code and solver
   ("ipssa", "fixed", "og"). */
const char* coinfer_status_message(int32_t status, const char* solver);
/* Number of kernels this context launched so far (for launch accounting). */
int64_t coinfer_ctx_launch_count(const coinfer_ctx* ctx);
/* Diagnostic: measured fp64-pipe throughput of the context's GPU in lane
   operations per second (independent DADD/DMUL/DFMA streams on every SM);
   the denominator of the engine's roofline (MEASURED_PEAKS.json has none). */
int coinfer_probe_fp64(coinfer_ctx* ctx, double* lane_ops_per_s);

/* IP-SSA (Alg. 2) for every instance.  deadline[k] is the common batch
   deadline l of instance k (same memory kind as the users); NULL means the
   smallest user deadline of the instance, as the CLI does
   (coinfer_main.cpp:240-243). */
int coinfer_ipssa_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                        const coinfer_users* users, const double* deadline,
                        coinfer_ipssa_out* out);

/* Alg. 1 at one assumed batch bound b[k] (fixed_batch_schedule).  deadline
   may be NULL as above.  status COINFER_ST_INFEASIBLE when some user cannot
   meet the deadline. */
int coinfer_fixed_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                        const coinfer_users* users, const double* deadline,
                        const int32_t* b, coinfer_ipssa_out* out);

/* OG optimal grouping (Alg. 3) for every instance. */
int coinfer_og_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                     const coinfer_users* users, coinfer_og_out* out);

/* IP-SSA at the smallest deadline AND OG for every instance in one fused
   pass (the offline Monte Carlo sweep).  Either output may be NULL. */
int coinfer_sweep_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                        const coinfer_users* users, coinfer_ipssa_out* ipssa,
                        coinfer_og_out* og);

/* Measurement aid (bench.py's roofline): the same fused IP-SSA + OG solve
   with work counters -- counters[0] OG chain steps ((user, chain)
   evaluations), [1] IP-SSA chain steps, [2] all-local user steps, [3] b*
   re-derivation steps, [4] chain starts (start-time recursions), [5] DP
   cells, [6] instances, [7] the b* steps of instances
   whose groups do not all take their largest admissible bound (the
   pipelined kernel's speculative b* re-runs only those).  Decisions are the solver's; M <= 255
   (the shared-memory path). */
int coinfer_count_work(coinfer_ctx* ctx, const coinfer_profile* profile, const coinfer_users* users,
                       coinfer_ipssa_out* ipssa, coinfer_og_out* og, uint64_t* counters);

/* Schedule materialisation on the device (try_fixed_batch:155-185, the
   og stitch :357-386 and normalize).  `solved` holds the decisions of an
   earlier coinfer_ipssa_batch / coinfer_fixed_batch (status, batch_bound,
   pipeline_feasible, split, freq, batch_size required) or coinfer_og_batch
   call (status, fallback, n_groups, order, group_lo, group_size, group_b,
   group_deadline, group_batch_size, split, freq required) on the same
   inputs, in the same memory kind; deadline as in coinfer_ipssa_batch.
   Instances whose status is not COINFER_ST_OK get n_batches 0 and untouched
   rows.  Every member of `out` is required. */
int coinfer_ipssa_schedule(coinfer_ctx* ctx, const coinfer_profile* profile,
                           const coinfer_users* users, const double* deadline,
                           const coinfer_ipssa_out* solved, coinfer_schedule_out* out);
int coinfer_og_schedule(coinfer_ctx* ctx, const coinfer_profile* profile,
                        const coinfer_users* users, const coinfer_og_out* solved,
                        coinfer_schedule_out* out);

/* baseline(sc, mode) (offline_solvers.hpp:602-612) for every instance:
   SolveResult fields in `out` (batch_bound / pipeline_feasible are those of
   the collapsed IP-SSA for IPSSA_NP, 0 / 1 otherwise), the schedule in
   `sched` (optional; all members required when given).  Infeasible
   instances get COINFER_ST_INFEASIBLE; the message per mode is
   coinfer_status_message(status, "lc" | "ps" | "fifo" | "np"). */
int coinfer_baseline_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                           const coinfer_users* users, int32_t mode, coinfer_ipssa_out* out,
                           coinfer_schedule_out* sched);

/* best_partition (offline_solvers.hpp:83-117) for n independent (user,
   start-time vector, deadline) queries, or detail::local_only_choice
   (:62-75) when s is NULL.  Users are the n rows of `users` (n_inst = n,
   M = 1); s is [n*N].  Outputs: PartitionChoice split / freq (NaN when
   nothing runs locally) / energy (+inf when infeasible) / feasible.
   Host memory only. */
int coinfer_best_partition(coinfer_ctx* ctx, const coinfer_profile* profile,
                           const coinfer_users* users, const double* s, int32_t* split,
                           double* freq, double* energy, uint8_t* feasible);

/* validate(schedule, scenario, tol) (schedule.hpp:139-209) for every
   instance, as violation counts per constraint id (the reference returns
   the list; here one row of counts per instance, in this order):
     C7-batchsize, C8-samesubtask, C9-batchready, C11-occupancy,
     C12-precedence, C15-deadline, C17-initial.
   `sched` is a coinfer_schedule_out as produced by the solvers (x,
   n_batches, batch_start, completion, freq; same memory kind as the users;
   rate_down / power_down used when given, else rate_up / power_up).
   status[k]: COINFER_ST_OK, COINFER_ST_BAD_BATCH_ID ("schedule: batch id
   beyond start-time table", invalid_argument), COINFER_ST_BOUND_PAST_TABLE
   (a batch larger than the table, out_of_range) or COINFER_ST_NONPOS_FREQ
   (local_latency with f <= 0, domain_error).  min_slack[k] (optional) is
   the most negative slack found (0 if none). */
#define COINFER_N_CONSTRAINTS 7
#define COINFER_ST_BAD_BATCH_ID 19
#define COINFER_ST_NONPOS_FREQ 23
int coinfer_validate_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                           const coinfer_users* users, const coinfer_schedule_out* sched,
                           double tol, int32_t* status, int32_t* counts, double* min_slack);

/* Scenario generation on the device: sample_scenario(cfg, profile,
   std::mt19937_64(seeds[k])) (scenario_gen.hpp:113-173) for every k.  The
   RNG stream, positions, deadlines, f_max and kappa are the reference
   generator's bit for bit; rates go through CUDA's log10/pow/log2 (within
   1-2 ulp of glibc's).  The CLI seeds instance k of its sweep with
   coinfer_sub_seed(root, 1, k) (coinfer_main.cpp:47-50,346-350). */
typedef struct coinfer_sample_cfg {  /* ScenarioConfig (scenario_gen.hpp:49-84) */
  double cell_radius, bandwidth, noise_dbm_hz, tx_power, uplink_power, downlink_power;
  double edge_power, edge_efficiency, device_efficiency, alpha, shadow_sigma_db;
  int32_t deadline_uniform; /* 0: DeadlineSpec::fixed(deadline_low); 1: uniform(low, high) */
  int32_t reserved;
  double deadline_low, deadline_high;
} coinfer_sample_cfg;

/* The same layout as coinfer_users, with writable arrays (an output). */
typedef struct coinfer_users_mut {
  int64_t n_inst;
  int32_t M;
  int32_t mem;
  double *f_min, *f_max, *kappa, *rate_up, *power_up, *arrival, *deadline, *rate_down, *power_down;
} coinfer_users_mut;

#define COINFER_ST_NO_DEADLINE 24 /* runtime_error "sample_scenario: cannot draw a feasible deadline" */
#define COINFER_ST_TOO_LARGE 25   /* invalid_argument "...: instance too large to enumerate" (oracles) */

void coinfer_sample_cfg_defaults(coinfer_sample_cfg* cfg); /* ScenarioConfig{} with fixed(0.5) */
uint64_t coinfer_sub_seed(uint64_t root, uint64_t component, uint64_t index);
/* out->n_inst instances of out->M users; seeds[n_inst] in out->mem memory,
   status[n_inst] (optional, same memory).  Config / profile errors return
   COINFER_E_ARG with the reference's message (ScenarioConfig::check,
   DnnProfile::check, sample_scenario's own tests). */
int coinfer_sample_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                         const coinfer_sample_cfg* cfg, const uint64_t* seeds,
                         coinfer_users_mut* out, int32_t* status);

/* The reference's brute-force oracles (oracles.hpp), one CTA per instance:
     oracle_structured(sc, deadline[k], b[k])      :28-93  ((N+1)^M <= 2e6)
     oracle_grouping_contiguous(sc) / oracle_grouping(sc)   :131-225
                                                   (M <= 16 / M <= 9)
   Outputs mirror StructuredOracle / GroupingOracle: energy (+inf when
   infeasible), split or group_of_user (index of the user's group in rising
   deadline order), fallback, n_groups, feasible; status COINFER_ST_TOO_LARGE
   when the reference would refuse to enumerate.  No contract checks (the
   oracles do none).  Every output array is required. */
int coinfer_oracle_structured_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                                    const coinfer_users* users, const double* deadline,
                                    const int32_t* b, int32_t* status, double* energy,
                                    uint8_t* split, uint8_t* fallback, uint8_t* feasible);
int coinfer_oracle_grouping_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                                  const coinfer_users* users, int32_t contiguous, int32_t* status,
                                  double* energy, int32_t* n_groups, int32_t* group_of_user,
                                  uint8_t* feasible);

/* Run n_ep episodes; episode e simulates scenario e % users->n_inst (each a
   Scenario of users->M users; deadlines are only contract-checked) with
   std::mt19937_64 seeded by seeds[e].  seeds and all outputs live in the
   same memory kind as the users.  Config errors (ArrivalModel::check, slot,
   horizon) return COINFER_E_ARG with the reference's message. */
int coinfer_online_run(coinfer_ctx* ctx, const coinfer_profile* profile,
                       const coinfer_users* scenarios, const coinfer_online_cfg* cfg,
                       const uint64_t* seeds, int64_t n_ep, coinfer_online_out* out);

#ifdef __cplusplus
}
#endif

#endif /* COINFER_B200_H */
