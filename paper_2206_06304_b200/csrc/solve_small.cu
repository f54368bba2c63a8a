// solve_small.cu — fused IP-SSA + OG solver, one CTA per problem instance,
// everything resident in shared memory (M up to ~180 users).
//
// Reference (all under /root/reference/proj/include/coinfer):
//   ip_ssa / detail::try_ip_ssa            offline_solvers.hpp:192-224
//   detail::try_fixed_batch + aggregation  offline_solvers.hpp:137-188
//   og (sort, G table, DP, backtrack, stitch, lc fallback)
//                                          offline_solvers.hpp:255-388
//   total_energy fold                      schedule.hpp:214-231
//   schedule_metrics per-user energy       offline_solvers.hpp:627-646
//
// Algorithm (bit-identical restatement):
//  * Users are deadline-sorted once; every per-user quantity the reference
//    recomputes in its inner loops is hoisted into a shared-memory record.
//  * A "chain" is one (group start i, assumed batch bound b) pair.  For a
//    fixed chain the per-user split choices do not depend on the group end j
//    and total_energy is a left fold, so one pass over j = i..M-1 yields the
//    energies of all groups i..j at that b (the reference re-solves every
//    (i, j) cell from scratch: O(M^4 N) -> O(M^3 N)).  Bounds b whose
//    pipeline does not fit dl[i] all give the same all-local plan, so they
//    collapse into one "all-local" chain keyed with the largest admissible b.
//    The IP-SSA solve is one more chain set over the users in original order.
//  * A chain dies once its offloader count exceeds b (it never decreases),
//    and OG rows stop at their last cell the DP can read (a cell no group
//    fits before has S = +inf whatever G holds).
//  * Chains are dealt to 4-lane slots in chunks of one row; a slot steps
//    its row's users together (one broadcast record read) and merges its
//    candidates into the G cell with an order-free 64-bit min.  The bound
//    attaining each chosen cell (the reference's descending-b scan with
//    strict '<') is re-derived only for the groups the DP picks.
//  * The grouping DP runs in place over the G triangle: per cell, the
//    feasible prevs are a prefix (binary search before the G phase) and the
//    minimum over them is a column prefix minimum kept in the triangle,
//    one barrier per stage.  Backtrack, b*, then every chosen group is
//    re-derived to produce the per-user outputs.
//  See solve_core.cuh for the details and DESIGN.md §2 for the proofs.

#include "solve_core.cuh"

namespace cfb {


int small_smem_bytes(int M, int N, int W) { return small_smem_bytes_impl(M, N, W); }

// The batch kernel: up to 256 threads and several CTAs per SM (throughput),
// or -- for a handful of instances, where SMs would idle -- one CTA of up to
// 1024 threads per instance, so each instance's chains spread over more
// lanes (latency).  Same body, same 64-register budget.
template <int N, bool COUNT = false>
__device__ __forceinline__ void solve_batch(const SmallArgs& a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int M = a.M;
  for (int64_t k = blockIdx.x; k < a.n_inst; k += gridDim.x) {
    const size_t base = (size_t)k * M;
    InstIn in;
    in.fmin = a.fmin + base;
    in.fmax = a.fmax + base;
    in.kappa = a.kappa + base;
    in.ru = a.ru + base;
    in.pu = a.pu + base;
    in.arr = a.arr + base;
    in.dl = a.dl + base;
    in.rd = a.rd ? a.rd + base : nullptr;
    in.pd = a.pd ? a.pd + base : nullptr;
    in.has_l_ip = a.l_ip != nullptr;
    in.l_ip = a.l_ip ? a.l_ip[k] : 0.0;
    solve_one<N, false, COUNT>(a, k, base, M, in, sm, a.L);
  }
}

template <int N>
__global__ void __launch_bounds__(256, CFB_SMALL_MINB) solve_small_kernel(SmallArgs a) {
  solve_batch<N>(a);
}

template <int N>
__global__ void __launch_bounds__(1024, 1) solve_wide_kernel(SmallArgs a) {
  solve_batch<N>(a);
}

// The same solve counting the work units it executes (SmallArgs::ctr).
template <int N>
__global__ void __launch_bounds__(256, CFB_SMALL_MINB) solve_count_kernel(SmallArgs a) {
  solve_batch<N, true>(a);
}

// fixed_batch_schedule (offline_solvers.hpp:208-214): one CTA per instance.
template <int N>
__global__ void __launch_bounds__(128) fixed_batch_kernel(SmallArgs a, const int32_t* bvec) {
  using R = Rec<N>;
  constexpr int REC = R::SIZE;
  extern __shared__ __align__(16) unsigned char sm[];
  const int M = a.M;
  const int tid = threadIdx.x, NT = blockDim.x;
  double* rec = reinterpret_cast<double*>(sm);
  double* fsc = rec + (size_t)M * REC;
  int* spsc = reinterpret_cast<int*>(fsc + M);
  __shared__ int st;
  __shared__ double lmin;
  const ProfileConst& P = a.P;
  for (int64_t k = blockIdx.x; k < a.n_inst; k += gridDim.x) {
    const size_t base = (size_t)k * M;
    if (tid == 0) st = INT_MAX;
    __syncthreads();
    for (int m = tid; m < M; m += NT) {
      const size_t x = base + m;
      const double rd = a.rd ? a.rd[x] : 1.0, pd = a.pd ? a.pd[x] : 0.0;
      const int code = check_user(a.fmin[x], a.fmax[x], a.kappa[x], a.ru[x], rd, a.pu[x], pd,
                                  a.arr[x], a.dl[x]);
      if (code != COINFER_ST_OK) atomicMin(&st, m * 32 + code);
      build_rec<N>(rec + m * REC, P, a.fmin[x], a.fmax[x], a.kappa[x], a.ru[x], a.pu[x], a.arr[x],
                   a.dl[x]);
    }
    if (tid == 0) {
      double l = M ? a.dl[base] : 0.0;
      for (int m = 0; m < M; ++m) l = smin(l, a.dl[base + m]);
      lmin = l;
    }
    __syncthreads();
    int status = st;
    if (P.bmax < M) status = COINFER_ST_SHORT_TABLE;
    else if (status != INT_MAX) status &= 31;
    else status = COINFER_ST_OK;
    const int b = bvec[k];
    if (status == COINFER_ST_OK && b < 1) status = COINFER_ST_ZERO_BOUND;
    if (status == COINFER_ST_OK && b > P.bmax) status = COINFER_ST_BOUND_PAST_TABLE;
    if (status != COINFER_ST_OK) {
      if (tid == 0 && a.ip.status) a.ip.status[k] = status;
      __syncthreads();
      continue;
    }
    const double l = a.l_ip ? a.l_ip[k] : lmin;
    double s[N];
    const bool pipe = start_times<N>(a.lat, P.bmax, l, b, s);
    for (int m = tid; m < M; m += NT) {
      int sp;
      double f;
      choose<N>(rec + m * REC, P, s, pipe, sp, f);
      spsc[m] = sp;
      fsc[m] = f;
    }
    __syncthreads();
    if (tid == 0) {
      bool ok = true;
      for (int m = 0; m < M; ++m) ok = ok && spsc[m] >= 0;
      st = ok ? COINFER_ST_OK : COINFER_ST_INFEASIBLE;
    }
    __syncthreads();
    if (st != COINFER_ST_OK) {
      if (tid == 0 && a.ip.status) a.ip.status[k] = st;
      __syncthreads();
      continue;
    }
    for (int m = tid; m < M; m += NT) {
      const size_t x = base + m;
      if (a.ip.split) a.ip.split[x] = (uint8_t)spsc[m];
      if (a.ip.freq) a.ip.freq[x] = fsc[m];
      if (a.ip.user_energy) a.ip.user_energy[x] = fold<N>(rec + m * REC, spsc[m], fsc[m], 0.0);
    }
    if (a.ip.batch_size)
      for (int n = 1 + tid; n <= N; n += NT) {
        int c = 0;
        for (int m = 0; m < M; ++m) c += spsc[m] < n;
        a.ip.batch_size[(size_t)k * N + n - 1] = c;
      }
    if (tid == 0) {
      double total = 0.0;
      for (int m = 0; m < M; ++m) total = fold<N>(rec + m * REC, spsc[m], fsc[m], total);
      if (a.ip.status) a.ip.status[k] = COINFER_ST_OK;
      if (a.ip.batch_bound) a.ip.batch_bound[k] = b;
      if (a.ip.pipeline_feasible) a.ip.pipeline_feasible[k] = pipe;
      if (a.ip.energy) a.ip.energy[k] = total;
    }
    __syncthreads();
  }
}


// Pipelined persistent kernel.  Per instance the fused solve is a latency-
// bound front (check, sort, hoist, row layout, DP feasibility), the
// issue-bound G table, and a latency-bound tail (IP-SSA output, DP,
// backtrack, b*, stitch) with a barrier per DP stage; in the one-CTA-per-
// instance kernel every warp of the CTA sits through the front and tail.
// Here a CTA holds two instance buffers and splits its warps: CFB_PIPE_GW
// warps run only G phases, alternating buffers, while CFB_PIPE_LW warps run
// the tail of one instance and then the front of the next into the same
// buffer.  Named barriers 1 (G team) and 2 (front/tail team) are the teams'
// own; the hand-offs are mbarriers: F[b] "front done in buffer b" (every
// front/tail thread arrives, G warps wait on its phase) and D[b] "G done in
// buffer b" (every G thread arrives, the front/tail team waits).  G warps
// are not synchronised with each other: one that runs out of chains starts
// the next instance as soon as its front is done.  Instances are claimed
// from a global counter, so CTAs stay busy to the end.
#ifndef CFB_PIPE_GW
#define CFB_PIPE_GW 6
#endif
#ifndef CFB_PIPE_LW
#define CFB_PIPE_LW 2
#endif
#ifndef CFB_PIPE_SUSPEND_NS
#define CFB_PIPE_SUSPEND_NS 1000000  // mbarrier wait suspend-time hint
#endif
#ifndef CFB_PIPE_GW1
#define CFB_PIPE_GW1 16  // when one CTA of two buffers fits an SM: 24 warps (M=100 target,
#endif                   // 100k instances: 20+4 / 18+6 / 16+8 / 14+10 -> 45.1 / 43.3 / 42.6 / 42.3 ms)
#ifndef CFB_PIPE_LW1
#define CFB_PIPE_LW1 8
#endif
#ifndef CFB_PIPE_GW2
#define CFB_PIPE_GW2 10  // ... when two fit: 16 warps (M=64: 12+4 / 11+5 / 10+6 -> 17.3 / 17.1 / 16.9 ms)
#endif
#ifndef CFB_PIPE_LW2
#define CFB_PIPE_LW2 6
#endif
// Team shapes by how many CTAs (two instance buffers each) fit an SM's
// shared memory: 0 = four (8 warps each), 2 = two (16), 1 = one (24);
// 64 registers per thread in every case.
template <int S>
struct PipeShape {
  static constexpr int GW = S == 0 ? CFB_PIPE_GW : S == 1 ? CFB_PIPE_GW1 : CFB_PIPE_GW2;
  static constexpr int LW = S == 0 ? CFB_PIPE_LW : S == 1 ? CFB_PIPE_LW1 : CFB_PIPE_LW2;
  static constexpr int GT = 32 * GW, LT = 32 * LW, T = GT + LT;
  static constexpr int MINB = S == 0 ? 4 : S == 2 ? 2 : 1;
};

__device__ __forceinline__ void mb_init(uint32_t addr, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" : : "r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint32_t addr) {  // release
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" : : "r"(addr) : "memory");
}
// acquire; the thread is suspended in the hardware until the phase completes
// (or the time hint runs out), instead of spinning on issue slots the
// other warps need
__device__ __forceinline__ void mb_wait(uint32_t addr, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}"
      : : "r"(addr), "r"(parity), "r"(CFB_PIPE_SUSPEND_NS) : "memory");
}

__host__ __device__ inline int pipe_buf_bytes(int M, int N) { return (make_layout(M, N, CFB_SLOT_PIPE).total + 127) & ~127; }

#ifdef CFB_PIPE_PROF  // development: cycles each team spends waiting on the other
static __device__ unsigned long long g_pipe_cyc[4];  // G wait, G busy, L wait, L busy (per warp-0 lane 0 of each team)
extern "C" int coinfer_debug_pipe_cycles(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_pipe_cyc, sizeof(unsigned long long) * 4);
  if (reset) {
    unsigned long long z[4] = {0};
    cudaMemcpyToSymbol(g_pipe_cyc, z, sizeof z);
  }
  return 0;
}
#define PIPE_T0 const long long _t0 = clock64();
#define PIPE_ACC(i) if (T.t == 0) atomicAdd(&g_pipe_cyc[i], (unsigned long long)(clock64() - _t0));
#else
#define PIPE_T0
#define PIPE_ACC(i)
#endif

template <int N, int S>
__global__ void __launch_bounds__(PipeShape<S>::T, PipeShape<S>::MINB) solve_pipe_kernel(SmallArgs a) {
  using PS = PipeShape<S>;
  constexpr int kPipeGT = PS::GT, kPipeLT = PS::LT, CFB_PIPE_GW_ = PS::GW;
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ long long kb[2];  // instance in buffer b, -1: none (stop)
  __shared__ __align__(8) unsigned long long mbar[4];  // F[0], F[1], D[0], D[1]
  const int M = a.M;
  const int bufb = pipe_buf_bytes(M, N);
  const int w = threadIdx.x >> 5;
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(mbar);
  auto F = [&](int b) { return mb0 + 8u * (uint32_t)b; };
  auto D = [&](int b) { return mb0 + 16u + 8u * (uint32_t)b; };
  // this CTA's two G tables in global memory (L2-resident)
  const size_t gstride = ((size_t)M * (M + 1) / 2 + 31) & ~(size_t)31;
  auto gbuf = [&](int b) { return a.gg + (2 * (size_t)blockIdx.x + b) * gstride; };
  if (threadIdx.x == 0) {
    mb_init(F(0), kPipeLT);
    mb_init(F(1), kPipeLT);
    mb_init(D(0), kPipeGT);
    mb_init(D(1), kPipeGT);
  }
  __syncthreads();
  auto input = [&](long long k) {
    const size_t base = (size_t)k * M;
    InstIn in;
    in.fmin = a.fmin + base;
    in.fmax = a.fmax + base;
    in.kappa = a.kappa + base;
    in.ru = a.ru + base;
    in.pu = a.pu + base;
    in.arr = a.arr + base;
    in.dl = a.dl + base;
    in.rd = a.rd ? a.rd + base : nullptr;
    in.pd = a.pd ? a.pd + base : nullptr;
    in.has_l_ip = a.l_ip != nullptr;
    in.l_ip = a.l_ip ? a.l_ip[k] : 0.0;
    return in;
  };
  // Team roles by warp: the last warps run the front/tail.  (The SM places
  // warp w of its c-th resident CTA on sub-partition (w + c) % 4, measured
  // with %warpid, so each sub-partition hosts two front/tail warps and six
  // G warps.  Putting all front/tail warps on one sub-partition cut their
  // tail from ~80k to ~57k cycles but left the G warps three sub-partitions:
  // G ~105k, 93.6 vs 90.5 ms per 1M C3 instances.)
  const bool lteam = w >= CFB_PIPE_GW_;
  const int lw = w - CFB_PIPE_GW_;  // rank among the front/tail warps
  const int gw = w;                 // rank among the G warps
  if (!lteam) {  // G team
    const Team T{gw * 32 + (int)(threadIdx.x & 31), kPipeGT, gw, 1};
    for (int i = 0;; ++i) {
      const int b = i & 1;
      {
        PIPE_T0
        mb_wait(F(b), (unsigned)(i >> 1) & 1u);
        PIPE_ACC(0)
      }
      const long long k = kb[b];
      if (k < 0) break;
      {
        PIPE_T0
        solve_one<N, false, false, PH_G>(a, k, (size_t)k * M, M, input(k), sm + b * bufb, a.L, T, gbuf(b));
        PIPE_ACC(1)
      }
      mb_arrive(D(b));
    }
  } else {  // front/tail team
    const Team T{lw * 32 + (int)(threadIdx.x & 31), kPipeLT, lw, 2};
    int nprod = 0, stop = INT_MAX;
    auto produce = [&]() {
      const int j = nprod++, b = j & 1;
      if (T.t == 0) {
        const unsigned long long c = atomicAdd(a.claim, 1ull);
        kb[b] = c < (unsigned long long)a.n_inst ? (long long)c : -1;
      }
      T.sync();
      const long long k = kb[b];
      if (k >= 0)
        solve_one<N, false, false, PH_FRONT>(a, k, (size_t)k * M, M, input(k), sm + b * bufb, a.L, T, gbuf(b));
      else stop = j;
      mb_arrive(F(b));
    };
    // fills j = 0, 1, 2, ... go to buffer j & 1; the tail of fill i runs
    // before fill i + 2 (one call site each: the phases are large)
    for (int step = 0;; ++step) {
      if (step >= 2) {
        const int i = step - 2, b = i & 1;
        if (i >= stop) break;
        {
          PIPE_T0
          mb_wait(D(b), (unsigned)(i >> 1) & 1u);
          PIPE_ACC(2)
        }
        PIPE_T0
        const long long k = kb[b];
        solve_one<N, false, false, PH_TAIL, PS::LW>(a, k, (size_t)k * M, M, input(k), sm + b * bufb, a.L, T,
                                                    gbuf(b));
        PIPE_ACC(3)
      }
      if (stop == INT_MAX) produce();
    }
  }
}

int fixed_smem_bytes(int M, int N) { return 8 * M * rec_size(N) + 8 * M + 4 * M + 16; }

// ------------------------------------------------------------ host launch
template <int N>
static cudaError_t launch_small_n(const SmallArgs& a_in, int threads, int grid, cudaStream_t st) {
  if (a_in.ctr && threads > 256) threads = 256;  // the counting kernel is built for <= 256
  SmallArgs a = a_in;
  a.L = make_layout(a.M, N);
  const int smem = a.L.total;
  auto kern = a.ctr ? solve_count_kernel<N> : threads > 256 ? solve_wide_kernel<N> : solve_small_kernel<N>;
  cudaError_t e = ensure_smem((const void*)kern, smem, true);
  if (e != cudaSuccess) return e;
  kern<<<grid, threads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_fixed_n(const SmallArgs& a, const int32_t* b, int grid, cudaStream_t st) {
  const int smem = fixed_smem_bytes(a.M, N);
  cudaError_t e = ensure_smem((const void*)fixed_batch_kernel<N>, smem);
  if (e != cudaSuccess) return e;
  fixed_batch_kernel<N><<<grid, 128, smem, st>>>(a, b);
  return cudaGetLastError();
}


#ifdef CFB_PHASE_TIMING
extern "C" int coinfer_debug_phase_cycles(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 8);
  cudaMemcpyFromSymbol(out + 8, g_ip_steps, sizeof(unsigned long long) * 2);
  cudaMemcpyFromSymbol(out + 10, g_tail_cycles, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
    cudaMemcpyToSymbol(g_ip_steps, z, sizeof(unsigned long long) * 2);
    cudaMemcpyToSymbol(g_tail_cycles, z, sizeof(unsigned long long) * 8);
  }
  return 0;
}
#endif

cudaError_t launch_small(const SmallArgs& a, int threads, int grid, cudaStream_t st) {
#define CFB_CALL(n) return launch_small_n<n>(a, threads, grid, st)
  CFB_DISPATCH_N(a.P.N, CFB_CALL)
#undef CFB_CALL
}


bool pipe_fits(int M, int N) { return M >= 1 && 2 * pipe_buf_bytes(M, N) + 64 <= 227 * 1024; }
static int pipe_shape(int M, int N) {
  const int cta = 2 * pipe_buf_bytes(M, N) + 64 + 1024;  // + the per-CTA reservation
  return 4 * cta <= 228 * 1024 ? 0 : 2 * cta <= 228 * 1024 ? 2 : 1;
}
// Measured at N = 4, 100k instances (pipelined vs one-CTA, ms): M = 40
// 7.6 / 8.3, 50 90.6 / 111.6 (1M), 56 14.8 / 14.5, 64 16.9 / 19.0, 72
// 19.7 / 25.6, 80 33.2 / 29.8, 84 35.1 / 40.1, 88 36.9 / 42.1, 90 37.7 /
// 42.6, 100 42.6 / 49.4.
bool pipe_preferred(int M, int N) {
  if (!pipe_fits(M, N)) return false;
  const int sh = pipe_shape(M, N);
  if (sh == 0) return true;
  if (sh == 1) return M >= 82;  // one CTA per SM: only past the measured crossover (80 -> 84)
  const int one = make_layout(M, N).total + 1024;  // one-CTA kernel: instances per SM by shared memory
  const int small_inst = (228 * 1024) / one;
  return 4 >= small_inst - 1;
}

// CTAs of the pipelined kernel resident at once (its persistent grid)
template <int N, int S>
static int pipe_max_grid(int M) {
  const int smem = 2 * pipe_buf_bytes(M, N);
  static thread_local int last_smem = -1, per_sm = 1, sms = 148;
  if (smem != last_smem) {  // occupancy of this buffer size
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    ensure_smem((const void*)solve_pipe_kernel<N, S>, smem, true);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_pipe_kernel<N, S>, PipeShape<S>::T, smem);
    if (per_sm < 1) per_sm = 1;
    last_smem = smem;
  }
  return per_sm * sms;
}

template <int N>
static int pipe_max_grid_m(int M) {
  const int sh = pipe_shape(M, N);
  return sh == 0 ? pipe_max_grid<N, 0>(M) : sh == 2 ? pipe_max_grid<N, 2>(M) : pipe_max_grid<N, 1>(M);
}

static cudaError_t pipe_grid_of(int M, int N, int* g) {
#define CFB_CALL(n) *g = pipe_max_grid_m<n>(M); return cudaSuccess
  CFB_DISPATCH_N(N, CFB_CALL)
#undef CFB_CALL
}

size_t pipe_gg_doubles(int M, int N) {
  int g = 0;
  if (pipe_grid_of(M, N, &g) != cudaSuccess) return 0;
  return (size_t)g * 2 * (((size_t)M * (M + 1) / 2 + 31) & ~(size_t)31);
}

template <int N, int S>
static cudaError_t launch_pipe_ns(const SmallArgs& a_in, cudaStream_t st) {
  SmallArgs a = a_in;
  a.L = make_layout(a.M, N, CFB_SLOT_PIPE);
  const int smem = 2 * pipe_buf_bytes(a.M, N);
  if (!pipe_fits(a.M, N) || !a.claim || !a.gg) return cudaErrorInvalidValue;
  cudaError_t e = ensure_smem((const void*)solve_pipe_kernel<N, S>, smem, true);
  if (e != cudaSuccess) return e;
  const long long maxg = pipe_max_grid<N, S>(a.M);
  const long long want = (a.n_inst + 1) / 2;  // two instances in flight per CTA
  const int grid = (int)(want < maxg ? want : maxg);
  e = cudaMemsetAsync(a.claim, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  solve_pipe_kernel<N, S><<<grid, PipeShape<S>::T, smem, st>>>(a);
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_pipe_n(const SmallArgs& a, cudaStream_t st) {
  const int sh = pipe_shape(a.M, N);
  return sh == 0 ? launch_pipe_ns<N, 0>(a, st) : sh == 2 ? launch_pipe_ns<N, 2>(a, st) : launch_pipe_ns<N, 1>(a, st);
}

cudaError_t launch_pipe(const SmallArgs& a, cudaStream_t st) {
#define CFB_CALL(n) return launch_pipe_n<n>(a, st)
  CFB_DISPATCH_N(a.P.N, CFB_CALL)
#undef CFB_CALL
}

cudaError_t launch_fixed(const SmallArgs& a, const int32_t* b, int grid, cudaStream_t st) {
#define CFB_CALL(n) return launch_fixed_n<n>(a, b, grid, st)
  CFB_DISPATCH_N(a.P.N, CFB_CALL)
#undef CFB_CALL
}

}  // namespace cfb
