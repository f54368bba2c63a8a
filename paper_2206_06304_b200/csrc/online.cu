// online.cu — the online slot driver on the GPU: run_episode(OnlineEnv,
// policy, horizon, seed) for many independent episodes, one warp each.
//
// Reference (under /root/reference/proj/include/coinfer/online_sim.hpp):
//   OnlineEnv ctor checks        :71-91     reset / sample_arrivals  :100-108, 235-249
//   step (modes, clip, rescue)   :131-173   process_all_local        :182-191
//   invoke_solver (OG / IP-SSA)  :193-233   TimeWindowPolicy         :312-336
//   local_policy                 :301-307   run_episode + metrics    :338-371
//
// An episode is strictly sequential: lane 0 walks the slots
// (policy, rescue, time, arrivals — M users each), and the whole warp joins
// for every solver call, which runs the same per-instance solver as the
// batch kernel (solve_one) on the pending users held in shared memory.
// Random numbers are std::mt19937_64 + libstdc++ 13 uniform_real_distribution
// reproduced exactly (generate_canonical<double,53> with one 64-bit draw:
// double(x) / 2^64, clamped below 1; then u*(b-a)+a without contraction), so a
// device episode replays the reference episode slot for slot.

#include "solve_core.cuh"

namespace cfb {

namespace {

// std::mt19937_64 (the standard's parameters), state in shared memory.
struct Mt64 {
  static constexpr int n = 312, m = 156;
  unsigned long long* x;
  int* idx;

  __device__ void seed(unsigned long long v) {
    x[0] = v;
    for (int i = 1; i < n; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + (unsigned long long)i;
    *idx = n;
  }
  __device__ void twist() {
    constexpr unsigned long long up = 0xffffffff80000000ULL, lo = 0x7fffffffULL, a = 0xb5026f5aa96619e9ULL;
    for (int i = 0; i < n - m; ++i) {
      const unsigned long long y = (x[i] & up) | (x[i + 1] & lo);
      x[i] = x[i + m] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    for (int i = n - m; i < n - 1; ++i) {
      const unsigned long long y = (x[i] & up) | (x[i + 1] & lo);
      x[i] = x[i + m - n] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    const unsigned long long y = (x[n - 1] & up) | (x[0] & lo);
    x[n - 1] = x[m - 1] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    *idx = 0;
  }
  __device__ unsigned long long next() {
    if (*idx >= n) twist();
    unsigned long long z = x[(*idx)++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71d67fffeda60000ULL;
    z ^= (z << 37) & 0xfff7eee000000000ULL;
    z ^= z >> 43;
    return z;
  }
  // uniform_real_distribution<double>(a, b)(*this), libstdc++ 13
  __device__ double uniform(double a, double b) {
    double u = __dmul_rn(__ull2double_rn(next()), 0x1p-64);  // exact: power-of-two scaling
    if (u >= 1.0) u = 0x1.fffffffffffffp-1;                   // nextafter(1, 0)
    return __dadd_rn(__dmul_rn(u, __dsub_rn(b, a)), a);
  }
};

}  // namespace

template <int N>
__global__ void __launch_bounds__(32) online_kernel(OnlineArgs o) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int M = o.M;
  const int tid = threadIdx.x;
  // shared memory: solver workspace | episode state
  unsigned char* st = sm + o.L.total;
  double* lrem = reinterpret_cast<double*>(st);           // remaining deadline per user
  double* expiry = lrem + M;
  double* floor_ = expiry + M;
  double* sub = floor_ + M;                                // 7 SoA arrays of the sub-scenario
  double* sfmin = sub, *sfmax = sub + M, *skap = sub + 2 * M, *sru = sub + 3 * M, *spu = sub + 4 * M,
         *sarr = sub + 5 * M, *sdl = sub + 6 * M;
  unsigned long long* mtx = reinterpret_cast<unsigned long long*>(sub + 7 * M);
  int* ivars = reinterpret_cast<int*>(mtx + Mt64::n);      // [0] mt idx, [1] call, [2] status, [3] n_sub
  int* ids = ivars + 8;

  const double W = o.solve.P.prefix[N];  // total_work()
  for (int64_t e = blockIdx.x; e < o.n_ep; e += gridDim.x) {
    const size_t sbase = (size_t)(e % o.n_scen) * M;
    const size_t obase = (size_t)e * M;  // solver scratch rows of this episode
    Mt64 rng{mtx, ivars};
    // ---------------------------------------------------------------- reset
    if (tid == 0) {
      int status = COINFER_ST_OK;
      for (int m = 0; m < M; ++m) {
        const size_t x = sbase + m;
        const double rd = o.rd ? o.rd[x] : 1.0, pd = o.pd ? o.pd[x] : 0.0;
        const int c = check_user(o.fmin[x], o.fmax[x], o.kappa[x], o.ru[x], rd, o.pu[x], pd, o.arr[x], o.dl[x]);
        if (c != COINFER_ST_OK && status == COINFER_ST_OK) status = c;
      }
      if (status == COINFER_ST_OK && o.solve.P.bmax < M) status = COINFER_ST_SHORT_TABLE;
      for (int m = 0; m < M && status == COINFER_ST_OK; ++m) {
        if (o.arr[sbase + m] != 0.0) status = COINFER_ST_NOT_RELEASED;
        floor_[m] = __ddiv_rn(W, o.fmax[sbase + m]);
        if (status == COINFER_ST_OK && floor_[m] > o.l_low) status = COINFER_ST_FLOOR_ABOVE_LLOW;
      }
      ivars[2] = status;
      rng.seed(o.seeds[e]);
      for (int m = 0; m < M; ++m) {
        lrem[m] = 0.0;
        expiry[m] = -1.0;
      }
    }
    __syncthreads();
    if (ivars[2] != COINFER_ST_OK) {
      if (tid == 0 && o.status) o.status[e] = ivars[2];
      __syncthreads();
      continue;
    }
    long long tick = 0;
    int wait = 0;        // TimeWindowPolicy state
    double ebusy = 0.0;  // MdpState::edge_busy
    double tot_energy = 0.0, tot_forced = 0.0;
    long long n_forced = 0, n_calls = 0, n_tasks = 0, n_groups = 0, n_batches = 0, n_batched = 0;
    const bool trace = e < o.n_trace;
    const size_t tbase = (size_t)e * (size_t)o.horizon;

    // sample_arrivals (online_sim.hpp:235-249), lane 0
    auto sample_arrivals = [&]() {
      const double now = __dmul_rn((double)tick, o.slot);
      for (int m = 0; m < M; ++m) {
        if (lrem[m] > 0.0) continue;
        if (!(now > expiry[m])) continue;
        if (!o.immediate) {
          if (o.p_arrive <= 0.0) continue;
          if (o.p_arrive < 1.0 && rng.uniform(0.0, 1.0) >= o.p_arrive) continue;
        }
        const double l = o.l_low < o.l_high ? rng.uniform(o.l_low, o.l_high) : o.l_low;
        lrem[m] = l;
        expiry[m] = __dadd_rn(now, l);
      }
    };
    if (tid == 0) sample_arrivals();
    __syncthreads();

    for (long long t = 0; t < o.horizon; ++t) {
      double energy = 0.0, forced = 0.0, busy_before = 0.0;
      int pending_before = 0;
      long long f_count = 0;
      // ------------------------------------------- policy + step (lane 0)
      if (tid == 0) {
        bool pending = false;
        for (int m = 0; m < M; ++m) {
          pending = pending || lrem[m] > 0.0;
          pending_before += lrem[m] > 0.0;
        }
        busy_before = ebusy;
        int mode = 0;
        double th = 0.0;
        if (o.policy == COINFER_POLICY_LOCAL) {
          mode = pending ? 1 : 0;
        } else if (ebusy > 0.0 || !pending) {  // TimeWindowPolicy (online_sim.hpp:317-330)
          wait = 0;
        } else if (wait >= o.window) {
          wait = 0;
          mode = 2;
          th = o.threshold;
        } else {
          ++wait;
        }
        const double l_th = smin(smax(th, 0.0), o.l_high);
        if (mode == 2 && ebusy > 0.0) mode = 0;
        ivars[1] = 0;
        if (mode == 1) {  // process_all_local (online_sim.hpp:182-191)
          for (int m = 0; m < M; ++m) {
            if (lrem[m] <= 0.0) continue;
            const size_t x = sbase + m;
            const double f = smin(smax(__ddiv_rn(W, lrem[m]), o.fmin[x]), o.fmax[x]);
            energy = __dadd_rn(energy, __dmul_rn(__dmul_rn(__dmul_rn(o.kappa[x], W), f), f));
            lrem[m] = 0.0;
          }
        } else if (mode == 2) {  // invoke_solver: pending users, ascending id, clipped deadlines
          int ns = 0;
          for (int m = 0; m < M; ++m) {
            if (!(lrem[m] > 0.0)) continue;
            const size_t x = sbase + m;
            const double l = lrem[m];
            ids[ns] = m;
            sfmin[ns] = o.fmin[x];
            sfmax[ns] = o.fmax[x];
            skap[ns] = o.kappa[x];
            sru[ns] = o.ru[x];
            spu[ns] = o.pu[x];
            sarr[ns] = 0.0;
            sdl[ns] = l >= l_th ? smax(l_th, floor_[m]) : l;
            ++ns;
          }
          ivars[3] = ns;
          ivars[1] = ns > 0;
        }
      }
      __syncthreads();
      if (ivars[1]) {  // the whole warp runs the solver on the pending users
        const int ns = ivars[3];
        InstIn in;
        in.fmin = sfmin;
        in.fmax = sfmax;
        in.kappa = skap;
        in.ru = sru;
        in.pu = spu;
        in.arr = sarr;
        in.dl = sdl;
        in.rd = nullptr;
        in.pd = nullptr;
        in.has_l_ip = false;  // IP-SSA at min deadline, as invoke_solver does
        in.l_ip = 0.0;
        const Layout L = make_layout(ns, N, 1);
        solve_one<N>(o.solve, e, obase, ns, in, sm, L);
        __syncthreads();
        if (tid == 0) {
          const int ns2 = ivars[3];
          const bool og = o.solve.do_og;
          const int stt = og ? o.solve.og.status[e] : o.solve.ip.status[e];
          if (stt != COINFER_ST_OK) {
            ivars[2] = stt;  // og/ip_ssa would throw out of step()
          } else {
            long long nb = 0, nbt = 0;
            double busy = 0.0;
            if (og) {
              energy = __dadd_rn(energy, o.solve.og.energy[e]);
              const int ng = o.solve.og.n_groups[e];
              n_groups += ng;
              for (int g = 0; g < ng; ++g)
                for (int n = 0; n < N; ++n) {
                  const int c = o.solve.og.group_batch_size[(obase + g) * N + n];
                  nb += c > 0;
                  nbt += c;
                }
              if (nb > 0) busy = o.solve.og.group_deadline[obase + ng - 1];
            } else {
              energy = __dadd_rn(energy, o.solve.ip.energy[e]);
              n_groups += 1;
              double lc = sdl[0];
              for (int x = 0; x < ns2; ++x) lc = smin(lc, sdl[x]);
              for (int n = 0; n < N; ++n) {
                const int c = o.solve.ip.batch_size[(size_t)e * N + n];
                nb += c > 0;
                nbt += c;
              }
              if (nb > 0) busy = lc;
            }
            ebusy = busy;
            n_batches += nb;
            n_batched += nbt;
            n_calls += 1;
            n_tasks += ns2;
            for (int x = 0; x < ns2; ++x) lrem[ids[x]] = 0.0;
          }
        }
        __syncthreads();
        if (ivars[2] != COINFER_ST_OK) break;
      }
      if (tid == 0) {
        // forced rescue at f_max (online_sim.hpp:149-158)
        for (int m = 0; m < M; ++m) {
          if (lrem[m] <= 0.0) continue;
          if (__dsub_rn(lrem[m], o.slot) < floor_[m]) {
            const size_t x = sbase + m;
            forced = __dadd_rn(forced, __dmul_rn(__dmul_rn(__dmul_rn(o.kappa[x], W), o.fmax[x]), o.fmax[x]));
            ++f_count;
            lrem[m] = 0.0;
          }
        }
        ++tick;
        for (int m = 0; m < M; ++m)
          if (lrem[m] > 0.0) lrem[m] = __dsub_rn(lrem[m], o.slot);
        ebusy = smax(0.0, __dsub_rn(ebusy, o.slot));
        sample_arrivals();
        for (int m = 0; m < M; ++m)
          if (lrem[m] > 0.0 && lrem[m] < __dsub_rn(floor_[m], 1e-12)) ivars[2] = COINFER_ST_SLIPPED;
        const double reward = -__dadd_rn(energy, forced);
        tot_energy = __dadd_rn(tot_energy, energy);
        tot_forced = __dadd_rn(tot_forced, forced);
        n_forced += f_count;
        if (trace) {
          if (o.tr_reward) o.tr_reward[tbase + t] = reward;
          if (o.tr_energy) o.tr_energy[tbase + t] = energy;
          if (o.tr_pending) o.tr_pending[tbase + t] = pending_before;
          if (o.tr_busy) o.tr_busy[tbase + t] = busy_before;
        }
      }
      __syncthreads();
      if (ivars[2] != COINFER_ST_OK) break;
    }
    if (tid == 0) {
      if (o.status) o.status[e] = ivars[2];
      if (o.totals) {
        o.totals[(size_t)e * 3 + 0] = tot_energy;
        o.totals[(size_t)e * 3 + 1] = tot_forced;
        o.totals[(size_t)e * 3 + 2] = -__dadd_rn(tot_energy, tot_forced);  // run_episode:362
      }
      if (o.counts) {
        long long* c = o.counts + (size_t)e * 6;
        c[0] = n_forced;
        c[1] = n_calls;
        c[2] = n_tasks;
        c[3] = n_groups;
        c[4] = n_batches;
        c[5] = n_batched;
      }
    }
    __syncthreads();
  }
}

int online_smem_bytes(int M, int N) {
  const int solver = make_layout(M, N, 1).total;
  return solver + 8 * (3 * M + 7 * M) + 8 * Mt64::n + 4 * (8 + M) + 16;
}

template <int N>
static cudaError_t launch_online_n(const OnlineArgs& a_in, int grid, cudaStream_t st) {
  OnlineArgs a = a_in;
  a.L = make_layout(a.M, N, 1);
  const int smem = online_smem_bytes(a.M, N);
  cudaError_t e = cudaFuncSetAttribute(online_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  online_kernel<N><<<grid, 32, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_online(const OnlineArgs& a, int grid, cudaStream_t st) {
#define CFB_CALL(n) return launch_online_n<n>(a, grid, st)
  CFB_DISPATCH_N(a.solve.P.N, CFB_CALL)
#undef CFB_CALL
}

}  // namespace cfb
