// kernels.h — host-visible launch interface of the solver kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/coinfer_b200.h"
#include "device_common.cuh"

namespace cfb {

// Byte offsets of the fused kernel's shared-memory regions; computed on the
// host once per launch so the kernel reads them from the constant bank.
struct SmemLayout {
  int rec, tri, dls, sumlat, ipe, fsc;
  int rowoff, b0, order, rank, gid, glo, ghi, gitem, gbest, misc;
  int pfit, argpm, parent, spsc, ipb, lat;
  int total;
};

// Arguments of the per-instance kernels; all pointers are device memory.
struct SmallArgs {
  SmemLayout L;
  ProfileConst P;
  const double* lat;  // [N*bmax] F_n(b)
  int64_t n_inst;
  int M;
  const double *fmin, *fmax, *kappa, *ru, *pu, *arr, *dl, *rd, *pd;
  const double* l_ip;  // IP-SSA / fixed deadline per instance, NULL = min deadline
  int do_ip, do_og;
  coinfer_ipssa_out ip;
  coinfer_og_out og;
  // work counters of the counting kernel (solve_count_kernel), else unused:
  // [0] OG chain steps, [1] IP-SSA chain steps, [2] all-local user steps,
  // [3] b* re-derivation steps, [4] chain starts, [5] DP cells, [6] instances
  unsigned long long* ctr;
  // instance claim counter of the pipelined kernel (zeroed before each launch)
  unsigned long long* claim;
  // pipelined kernel: G tables in global memory, 2 per CTA (pipe_gg_doubles), or NULL
  double* gg;
};
enum { CTR_OG = 0, CTR_IP, CTR_LOCAL, CTR_BSTAR, CTR_STARTS, CTR_DP, CTR_INST, CTR_BSTAR_MISS, CTR_N = 8 };

// One instance's users (global or shared memory), already offset.
struct InstIn {
  const double *fmin, *fmax, *kappa, *ru, *pu, *arr, *dl, *rd, *pd;
  double l_ip;    // IP-SSA common deadline when has_l_ip
  bool has_l_ip;  // else the smallest user deadline
};

// Arguments of the online driver (one warp per episode).
struct OnlineArgs {
  SmallArgs solve;  // profile, latency table, solver choice, per-episode scratch outputs
  SmemLayout L;     // solver workspace for M users, one warp
  int M;
  int64_t n_scen;   // episode e runs scenario e % n_scen
  const double *fmin, *fmax, *kappa, *ru, *pu, *arr, *dl, *rd, *pd;
  int immediate;
  double p_arrive, l_low, l_high, slot, threshold;
  int policy, window;
  int64_t horizon, n_ep;
  const unsigned long long* seeds;
  int32_t* status;
  double* totals;
  long long* counts;
  int64_t n_trace;
  double *tr_reward, *tr_energy, *tr_busy;
  int32_t* tr_pending;
  int32_t *tr_action, *tr_forced;  // optional
  double* fin_state;               // optional: [n_ep][2M+1] deadline, expiry, edge_busy
  long long* draws;                // optional: [n_ep] rng outputs consumed
};

// Arguments of the large-instance path (solve_large.cu); one instance per
// launch sequence, all pointers device memory.
struct LargeArgs {
  ProfileConst P;
  const double* lat;
  int M;
  const double *fmin, *fmax, *kappa, *ru, *pu, *arr, *dl, *rd, *pd;  // this instance
  double l_ip;
  int has_l_ip, do_ip, do_og;
  const double* l_ip_dev;  // else: this instance's IP-SSA deadline in device memory (read on the device)
  int64_t k;    // output instance index
  size_t base;  // output row (k * M)
  // workspace
  int* status;  // INT_MAX, or the first failing user * 32 + code
  int* simple;  // all arrivals and f_min zero
  double *rec, *dls, *sumlat, *G, *St, *ipres, *fpos, *genergy, *slast;
  int *order, *rank, *b0, *spos, *gid, *rlen;
  uint16_t *bstar, *par, *ipb, *pfit, *argpm;
  coinfer_ipssa_out ip;
  coinfer_og_out og;
};

// Arguments of the schedule-materialisation and baseline kernels
// (baselines.cu): one thread per instance, all pointers device memory.
struct AuxArgs {
  ProfileConst P;
  const double* lat;  // the caller's profile table [N*bmax]
  int64_t n_inst;
  int M;
  const double *fmin, *fmax, *kappa, *ru, *pu, *arr, *dl, *rd, *pd;
  const double* l_ip;       // IP-SSA / fixed deadline per instance, NULL = smallest user deadline
  coinfer_ipssa_out ip;     // baseline results, or the IP-SSA decisions to materialise
  coinfer_og_out og;        // the OG decisions to materialise
  coinfer_ipssa_out flat;   // IPSSA_NP: the collapsed-profile IP-SSA decisions
  coinfer_schedule_out sch; // Schedule (x, batch_start, completion, freq)
  int mode;                 // COINFER_BASELINE_*
  unsigned char* scratch;   // per-thread scratch, scratch_per_thread bytes each
  size_t scratch_per_thread;
  // validate: tolerance and outputs
  double tol;
  int32_t* vstatus;         // [n_inst]
  int32_t* vcounts;         // [n_inst * COINFER_N_CONSTRAINTS]
  double* vslack;           // [n_inst] (optional)
};

// Arguments of the brute-force oracle kernels (oracles.cu), device memory.
struct OracleArgs {
  ProfileConst P;
  const double* lat;
  int64_t n_inst;
  int M;
  const double *fmin, *fmax, *kappa, *ru, *pu, *arr, *dl;
  const double* deadline;  // structured: common deadline per instance
  const int32_t* b;        // structured: bound per instance
  int contiguous;          // grouping: 1 = cut patterns only
  int32_t* status;
  double* energy;
  uint8_t* split;          // structured [K*M]
  uint8_t* fallback;       // structured [K]
  uint8_t* feasible;       // [K]
  int32_t* n_groups;       // grouping [K]
  int32_t* group_of_user;  // grouping [K*M]
};

cudaError_t launch_oracle_structured(const OracleArgs& a, cudaStream_t st);
cudaError_t launch_oracle_grouping(const OracleArgs& a, cudaStream_t st);

size_t aux_scratch_bytes(int M, int N);
int aux_grid(int64_t n_inst);
cudaError_t launch_materialize_ip(const AuxArgs& a, cudaStream_t st);
cudaError_t launch_materialize_og(const AuxArgs& a, cudaStream_t st);
cudaError_t launch_baseline(const AuxArgs& a, cudaStream_t st);
cudaError_t launch_validate(const AuxArgs& a, cudaStream_t st);
cudaError_t launch_sample(const coinfer_sample_cfg& cfg, double total_work, int M, int64_t n_inst,
                          const unsigned long long* seeds, const coinfer_users_mut& out, int32_t* status,
                          cudaStream_t st);
cudaError_t launch_partition(const AuxArgs& a, const double* s, int32_t* split, double* freq,
                             double* energy, uint8_t* feasible, cudaStream_t st);

int small_smem_bytes(int M, int N, int W);
int online_smem_bytes(int M, int N);
size_t large_ws_bytes(int M, int N);
cudaError_t launch_large(const LargeArgs& a, cudaStream_t st);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize [, carveout 100%]) for
// kernel f on the current device, only when the request grows (a cached
// per-(kernel, device) high-water mark: single-instance calls pay no
// attribute round trips).
cudaError_t ensure_smem(const void* f, int smem, bool carveout = false);
cudaError_t launch_online(const OnlineArgs& a, int grid, cudaStream_t st);
int fixed_smem_bytes(int M, int N);
cudaError_t launch_small(const SmallArgs& a, int threads, int grid, cudaStream_t st);
// The pipelined persistent kernel (solve_small.cu: solve_pipe_kernel); a.claim
// must be set.  Returns cudaErrorInvalidValue when two instance buffers of
// this size do not fit (the caller then uses launch_small).
cudaError_t launch_pipe(const SmallArgs& a, cudaStream_t st);
bool pipe_fits(int M, int N);
// Whether the pipelined kernel beats the one-CTA kernel at this size (by
// the instances each keeps in flight per SM; measured crossovers, see there)
bool pipe_preferred(int M, int N);
size_t pipe_gg_doubles(int M, int N);  // the global G-table workspace the pipelined kernel wants
// per team shape (solve_pipe{0,1,2}.cu): resident CTAs, launch
int pipe_max_grid_s0(int M, int N);
int pipe_max_grid_s1(int M, int N);
int pipe_max_grid_s2(int M, int N);
cudaError_t launch_pipe_s0(const SmallArgs& a, cudaStream_t st);
cudaError_t launch_pipe_s1(const SmallArgs& a, cudaStream_t st);
cudaError_t launch_pipe_s2(const SmallArgs& a, cudaStream_t st);
cudaError_t launch_fixed(const SmallArgs& a, const int32_t* b, int grid, cudaStream_t st);

#ifdef CFB_ONLY_N  // development builds: one sub-task count only (fast compiles)
#define CFB_DISPATCH_N(NVAL, CALL)                   \
  switch (NVAL) {                                    \
    case CFB_ONLY_N: CALL(CFB_ONLY_N); break;        \
    default: return cudaErrorInvalidValue;           \
  }
#else
#define CFB_DISPATCH_N(NVAL, CALL) \
  switch (NVAL) {                  \
    case 1: CALL(1); break;        \
    case 2: CALL(2); break;        \
    case 3: CALL(3); break;        \
    case 4: CALL(4); break;        \
    case 5: CALL(5); break;        \
    case 6: CALL(6); break;        \
    case 7: CALL(7); break;        \
    case 8: CALL(8); break;        \
    case 9: CALL(9); break;        \
    case 10: CALL(10); break;      \
    case 11: CALL(11); break;      \
    case 12: CALL(12); break;      \
    case 13: CALL(13); break;      \
    case 14: CALL(14); break;      \
    case 15: CALL(15); break;      \
    case 16: CALL(16); break;      \
    default: return cudaErrorInvalidValue; \
  }
#endif

}  // namespace cfb
