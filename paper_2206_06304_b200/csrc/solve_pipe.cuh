// solve_pipe.cuh -- the pipelined persistent kernel (solve_pipe_kernel) and
// its launch, instantiated per team shape by solve_pipe{0,1,2}.cu so the
// shapes compile side by side.  See solve_small.cu for the one-CTA kernel.
#pragma once

#include <climits>

#include "solve_core.cuh"

namespace cfb {

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
#endif                   // 100k instances: 20+4 / 18+6 / 16+8 / 14+10 -> 45.1 / 43.3 / 42.6 / 42.3 ms;
                         // 28 warps 18+10: 42.0 vs 42.0, 32 warps 20+12: 43.3)
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
// G wait, G busy, L wait, L busy (per translation unit: solve_pipe0.cu's, shape 0, is exported)
static __device__ unsigned long long g_pipe_cyc[4];
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

template <int N, int S>
static cudaError_t launch_pipe_ns(const SmallArgs& a_in, cudaStream_t st) {
  SmallArgs a = a_in;
  a.L = make_layout(a.M, N, CFB_SLOT_PIPE);
  const int smem = 2 * pipe_buf_bytes(a.M, N);
  if (2 * pipe_buf_bytes(a.M, N) + 64 > 227 * 1024 || !a.claim || !a.gg) return cudaErrorInvalidValue;
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

// the pipelined kernel runs N <= CFB_PIPE_MAXN sub-tasks (others: one-CTA kernel)
#ifndef CFB_PIPE_MAXN
#define CFB_PIPE_MAXN 8
#endif
#ifdef CFB_ONLY_N
#define CFB_PIPE_DISPATCH(NVAL, CALL)          \
  switch (NVAL) {                              \
    case CFB_ONLY_N: CALL(CFB_ONLY_N); break;  \
    default: return cudaErrorInvalidValue;     \
  }
#else
#define CFB_PIPE_DISPATCH(NVAL, CALL) \
  switch (NVAL) {                     \
    case 1: CALL(1); break;           \
    case 2: CALL(2); break;           \
    case 3: CALL(3); break;           \
    case 4: CALL(4); break;           \
    case 5: CALL(5); break;           \
    case 6: CALL(6); break;           \
    case 7: CALL(7); break;           \
    case 8: CALL(8); break;           \
    default: return cudaErrorInvalidValue; \
  }
#endif

}  // namespace cfb
