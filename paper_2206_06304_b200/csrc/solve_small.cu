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
#include "solve_pipe.cuh"

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


bool pipe_fits(int M, int N) {
  return M >= 1 && N <= CFB_PIPE_MAXN && 2 * pipe_buf_bytes(M, N) + 64 <= 227 * 1024;
}
static int pipe_shape(int M, int N) {
  const int cta = 2 * pipe_buf_bytes(M, N) + 64 + 1024;  // + the per-CTA reservation
  return 4 * cta <= 228 * 1024 ? 0 : 2 * cta <= 228 * 1024 ? 2 : 1;
}
// Measured at N = 4, 100k instances (pipelined vs one-CTA, ms): M = 40
// 7.6 / 8.3, 50 90.6 / 111.6 (1M), 56 14.8 / 14.5, 64 16.0 / 19.0, 72
// 18.9 / 25.6, 80 33.2 / 29.8, 84 35.1 / 40.1, 88 36.9 / 42.1, 90 37.7 /
// 42.6, 100 42.0 / 49.4.
bool pipe_preferred(int M, int N) {
  if (!pipe_fits(M, N)) return false;
  const int sh = pipe_shape(M, N);
  if (sh == 0) return true;
  if (sh == 1) return M >= 82;  // one CTA per SM: only past the measured crossover (80 -> 84)
  const int one = make_layout(M, N).total + 1024;  // one-CTA kernel: instances per SM by shared memory
  const int small_inst = (228 * 1024) / one;
  return 4 >= small_inst - 1;
}

size_t pipe_gg_doubles(int M, int N) {
  const int sh = pipe_shape(M, N);
  const int g = sh == 0 ? pipe_max_grid_s0(M, N) : sh == 2 ? pipe_max_grid_s2(M, N) : pipe_max_grid_s1(M, N);
  return (size_t)g * 2 * (((size_t)M * (M + 1) / 2 + 31) & ~(size_t)31);
}

cudaError_t launch_pipe(const SmallArgs& a, cudaStream_t st) {
  if (!pipe_fits(a.M, a.P.N)) return cudaErrorInvalidValue;
  const int sh = pipe_shape(a.M, a.P.N);
  return sh == 0 ? launch_pipe_s0(a, st) : sh == 2 ? launch_pipe_s2(a, st) : launch_pipe_s1(a, st);
}

cudaError_t launch_fixed(const SmallArgs& a, const int32_t* b, int grid, cudaStream_t st) {
#define CFB_CALL(n) return launch_fixed_n<n>(a, b, grid, st)
  CFB_DISPATCH_N(a.P.N, CFB_CALL)
#undef CFB_CALL
}

}  // namespace cfb
