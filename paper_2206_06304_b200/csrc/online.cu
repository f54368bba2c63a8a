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

#include <cstdlib>

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
    long long ndraw = 0;  // mt19937_64 outputs consumed

    // sample_arrivals (online_sim.hpp:235-249), lane 0
    auto sample_arrivals = [&]() {
      const double now = __dmul_rn((double)tick, o.slot);
      for (int m = 0; m < M; ++m) {
        if (lrem[m] > 0.0) continue;
        if (!(now > expiry[m])) continue;
        if (!o.immediate) {
          if (o.p_arrive <= 0.0) continue;
          if (o.p_arrive < 1.0) {
            ++ndraw;
            if (rng.uniform(0.0, 1.0) >= o.p_arrive) continue;
          }
        }
        ndraw += o.l_low < o.l_high;
        const double l = o.l_low < o.l_high ? rng.uniform(o.l_low, o.l_high) : o.l_low;
        lrem[m] = l;
        expiry[m] = __dadd_rn(now, l);
      }
    };
    if (tid == 0) sample_arrivals();
    __syncthreads();

    for (long long t = 0; t < o.horizon; ++t) {
      double energy = 0.0, forced = 0.0, busy_before = 0.0;
      int pending_before = 0, pmode = 0;
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
        pmode = mode;  // TraceRow::action_c: the policy's action, before step() clamps it
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
        const Layout L = make_layout(ns, N);
        solve_one<N, true>(o.solve, e, obase, ns, in, sm, L);
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
          if (o.tr_action) o.tr_action[tbase + t] = pmode;
          if (o.tr_forced) o.tr_forced[tbase + t] = (int32_t)f_count;
        }
      }
      __syncthreads();
      if (ivars[2] != COINFER_ST_OK) break;
    }
    if (tid == 0) {
      if (o.status) o.status[e] = ivars[2];
      if (o.draws) o.draws[e] = ndraw;
      if (o.fin_state) {
        double* fs = o.fin_state + (size_t)e * (2 * M + 1);
        for (int m = 0; m < M; ++m) {
          fs[m] = lrem[m];
          fs[M + m] = expiry[m];
        }
        fs[2 * M] = ebusy;
      }
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

// ---------------------------------------------------------------------------
// The same episode with the per-user work spread over the warp (M <= 32):
// lane m holds user m's remaining deadline, expiry and contract values in
// registers, so policy, rescue, time and arrivals are ballots, scans and
// ordered shuffle folds instead of lane 0 walking M users.  Sums keep the
// reference's user order (an ordered fold over lanes); the random stream
// stays the reference's one sequence: each slot's draws are assigned to
// users by a prefix sum over how many each consumes (a Bernoulli coin, then
// a deadline if it arrives), resolved by iterating the coins to a fixed
// point, and read from a window of tempered outputs refilled in order (the
// mt19937_64 twist runs warp-wide).
namespace {

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71d67fffeda60000ULL;
  z ^= (z << 37) & 0xfff7eee000000000ULL;
  z ^= z >> 43;
  return z;
}

// std::mt19937_64 twist, warp-wide: each 32-element chunk reads the old
// values it needs before any lane writes (the sequential update reads
// x[i+1] before it changes and x[i+m] / x[i+m-n] as the loop leaves them).
__device__ void mt_twist_warp(unsigned long long* x, int lane) {
  constexpr int n = 312, m = 156;
  constexpr unsigned long long up = 0xffffffff80000000ULL, lo = 0x7fffffffULL, a = 0xb5026f5aa96619e9ULL;
  for (int c = 0; c < n - m; c += 32) {  // i < n-m: x[i+m] old
    const int i = c + lane;
    unsigned long long v = 0;
    if (i < n - m) {
      const unsigned long long y = (x[i] & up) | (x[i + 1] & lo);
      v = x[i + m] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    __syncwarp();
    if (i < n - m) x[i] = v;
    __syncwarp();
  }
  for (int c = n - m; c < n - 1; c += 32) {  // x[i+m-n] already updated
    const int i = c + lane;
    unsigned long long v = 0;
    if (i < n - 1) {
      const unsigned long long y = (x[i] & up) | (x[i + 1] & lo);
      v = x[i + m - n] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    __syncwarp();
    if (i < n - 1) x[i] = v;
    __syncwarp();
  }
  if (lane == 0) {
    const unsigned long long y = (x[n - 1] & up) | (x[0] & lo);
    x[n - 1] = x[m - 1] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
  }
  __syncwarp();
}

// generate_canonical<double, 53> from one output, libstdc++ 13
__device__ __forceinline__ double mt_canonical(unsigned long long z) {
  double u = __dmul_rn(__ull2double_rn(z), 0x1p-64);
  return u >= 1.0 ? 0x1.fffffffffffffp-1 : u;
}

// ordered left fold over lanes: acc + v[0] + v[1] + ... (lanes with take set)
__device__ __forceinline__ double lane_fold(double acc, double v, unsigned take, int M) {
  for (int m = 0; m < M; ++m) {
    const double t = __shfl_sync(kFull, v, m);
    if ((take >> m) & 1u) acc = __dadd_rn(acc, t);
  }
  return acc;
}

}  // namespace

template <int N>
#ifndef CFB_ONLINE_WARP_MINB
#define CFB_ONLINE_WARP_MINB 16  // 128 registers: 16 episodes per SM (measured best of 1/16/21/32)
#endif
__global__ void __launch_bounds__(32, CFB_ONLINE_WARP_MINB) online_warp_kernel(OnlineArgs o) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int M = o.M;  // <= 32
  const int lane = threadIdx.x;
  unsigned char* st = sm + o.L.total;
  double* sub = reinterpret_cast<double*>(st);  // 7 SoA arrays of the sub-scenario
  double *sfmin = sub, *sfmax = sub + M, *skap = sub + 2 * M, *sru = sub + 3 * M, *spu = sub + 4 * M,
         *sarr = sub + 5 * M, *sdl = sub + 6 * M;
  unsigned long long* mtx = reinterpret_cast<unsigned long long*>(sub + 7 * M);  // [312]
  unsigned long long* win = mtx + 312;                                           // [128] tempered outputs
  int* ids = reinterpret_cast<int*>(win + 128);                                  // [32]
  constexpr int WIN = 128;

  const double W = o.solve.P.prefix[N];  // total_work()
  const bool own = lane < M;
  const unsigned users = M >= 32 ? 0xffffffffu : ((1u << M) - 1u);
  for (int64_t e = blockIdx.x; e < o.n_ep; e += gridDim.x) {
    const size_t sbase = (size_t)(e % o.n_scen) * M;
    const size_t obase = (size_t)e * M;
    // ---------------------------------------------------------------- reset
    double ufmin = 0.0, ufmax = 1.0, ukap = 0.0, uru = 1.0, upu = 0.0, floor_ = 0.0;
    int code = COINFER_ST_OK, code2 = COINFER_ST_OK;
    if (own) {
      const size_t x = sbase + lane;
      const double rd = o.rd ? o.rd[x] : 1.0, pd = o.pd ? o.pd[x] : 0.0;
      ufmin = o.fmin[x];
      ufmax = o.fmax[x];
      ukap = o.kappa[x];
      uru = o.ru[x];
      upu = o.pu[x];
      code = check_user(ufmin, ufmax, ukap, uru, rd, upu, pd, o.arr[x], o.dl[x]);
      floor_ = __ddiv_rn(W, ufmax);
      code2 = o.arr[x] != 0.0 ? COINFER_ST_NOT_RELEASED
                              : (floor_ > o.l_low ? COINFER_ST_FLOOR_ABOVE_LLOW : COINFER_ST_OK);
    }
    int status = COINFER_ST_OK;
    {  // first failing user, checks in the reference's order
      const unsigned b1 = __ballot_sync(kFull, code != COINFER_ST_OK);
      if (b1) status = __shfl_sync(kFull, code, __ffs(b1) - 1);
      if (status == COINFER_ST_OK && o.solve.P.bmax < M) status = COINFER_ST_SHORT_TABLE;
      const unsigned b2 = __ballot_sync(kFull, code2 != COINFER_ST_OK);
      if (status == COINFER_ST_OK && b2) status = __shfl_sync(kFull, code2, __ffs(b2) - 1);
    }
    if (status != COINFER_ST_OK) {
      if (lane == 0 && o.status) o.status[e] = status;
      continue;
    }
    if (lane == 0) {  // mt19937_64 seeding is a sequential recurrence
      mtx[0] = o.seeds[e];
      for (int i = 1; i < 312; ++i)
        mtx[i] = 6364136223846793005ULL * (mtx[i - 1] ^ (mtx[i - 1] >> 62)) + (unsigned long long)i;
    }
    __syncwarp();
    int mtpos = 312;   // next state element to temper (312: twist first)
    int wbeg = 0, wcnt = 0;
    // make >= need tempered outputs available in win[wbeg .. wbeg+wcnt)
    auto ensure = [&](int need) {
      if (wcnt >= need) return;
      // compact, then append outputs in stream order up to a full window
      unsigned long long keep = lane < wcnt ? win[wbeg + lane] : 0ULL;
      unsigned long long keep2 = lane + 32 < wcnt ? win[wbeg + lane + 32] : 0ULL;
      __syncwarp();
      if (lane < wcnt) win[lane] = keep;
      if (lane + 32 < wcnt) win[lane + 32] = keep2;
      wbeg = 0;
      while (wcnt < WIN) {
        if (mtpos >= 312) {
          mt_twist_warp(mtx, lane);
          mtpos = 0;
        }
        const int take = min(WIN - wcnt, 312 - mtpos);
        for (int k = lane; k < take; k += 32) win[wcnt + k] = mt_temper(mtx[mtpos + k]);
        wcnt += take;
        mtpos += take;
      }
      __syncwarp();
    };
    double lrem = 0.0, expiry = -1.0;
    long long tick = 0, ndraw = 0;  // ndraw: mt19937_64 outputs consumed
    const bool imm = o.immediate != 0;
    const bool coin = !imm && o.p_arrive > 0.0 && o.p_arrive < 1.0;  // a Bernoulli draw per eligible user
    const bool never = !imm && !(o.p_arrive > 0.0);
    const bool ranged = o.l_low < o.l_high;
    // sample_arrivals (online_sim.hpp:235-249) for every user at once
    auto sample_arrivals = [&]() {
      const double now = __dmul_rn((double)tick, o.slot);
      const bool elig = own && !never && !(lrem > 0.0) && now > expiry;
      const unsigned em = __ballot_sync(kFull, elig);
      if (!em) return;
      ensure(2 * M);
      const int c1 = (elig && coin) ? 1 : 0;
      bool arrived = elig && !coin;  // coins decide the rest
      int off = 0;
      for (;;) {
        const int cons = elig ? c1 + ((arrived && ranged) ? 1 : 0) : 0;
        int incl = cons;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int t = __shfl_up_sync(kFull, incl, d);
          if (lane >= d) incl += t;
        }
        off = incl - cons;
        bool na = arrived;
        if (elig && coin) na = !(mt_canonical(win[wbeg + off]) >= o.p_arrive);
        const unsigned changed = __ballot_sync(kFull, na != arrived);
        arrived = na;
        if (!changed) {
          const int total = __shfl_sync(kFull, incl, 31);
          if (arrived) {
            double l = o.l_low;
            if (ranged) {
              const double u = mt_canonical(win[wbeg + off + c1]);
              l = __dadd_rn(__dmul_rn(u, __dsub_rn(o.l_high, o.l_low)), o.l_low);
            }
            lrem = l;
            expiry = __dadd_rn(now, l);
          }
          wbeg += total;
          wcnt -= total;
          ndraw += total;
          return;
        }
      }
    };
    sample_arrivals();

    int wait = 0;        // TimeWindowPolicy state
    double ebusy = 0.0;  // MdpState::edge_busy
    double tot_energy = 0.0, tot_forced = 0.0;
    long long n_forced = 0, n_calls = 0, n_tasks = 0, n_groups = 0, n_batches = 0, n_batched = 0;
    const bool trace = e < o.n_trace;
    const size_t tbase = (size_t)e * (size_t)o.horizon;
    for (long long t = 0; t < o.horizon; ++t) {
      double energy = 0.0, forced = 0.0;
      const double busy_before = ebusy;
      const unsigned pend = __ballot_sync(kFull, own && lrem > 0.0);
      const int pending_before = __popc(pend);
      // ------------------------------------------------------------ policy
      int mode = 0;
      double th = 0.0;
      if (o.policy == COINFER_POLICY_LOCAL) {
        mode = pend ? 1 : 0;
      } else if (ebusy > 0.0 || !pend) {  // TimeWindowPolicy (online_sim.hpp:317-330)
        wait = 0;
      } else if (wait >= o.window) {
        wait = 0;
        mode = 2;
        th = o.threshold;
      } else {
        ++wait;
      }
      const int pmode = mode;  // TraceRow::action_c: the policy's action, before step() clamps it
      const double l_th = smin(smax(th, 0.0), o.l_high);
      if (mode == 2 && ebusy > 0.0) mode = 0;
      int n_resc = 0;
      if (mode == 1) {  // process_all_local (online_sim.hpp:182-191), user order
        double term = 0.0;
        if ((pend >> lane) & 1u) {
          const double f = smin(smax(__ddiv_rn(W, lrem), ufmin), ufmax);
          term = __dmul_rn(__dmul_rn(__dmul_rn(ukap, W), f), f);
          lrem = 0.0;
        }
        energy = lane_fold(energy, term, pend, M);
      } else if (mode == 2 && pend) {  // invoke_solver: pending users, ascending id, clipped deadlines
        const int ns = __popc(pend);
        if ((pend >> lane) & 1u) {
          const int q = __popc(pend & ((1u << lane) - 1u));
          ids[q] = lane;
          sfmin[q] = ufmin;
          sfmax[q] = ufmax;
          skap[q] = ukap;
          sru[q] = uru;
          spu[q] = upu;
          sarr[q] = 0.0;
          sdl[q] = lrem >= l_th ? smax(l_th, floor_) : lrem;
        }
        __syncwarp();
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
        const Layout L = make_layout(ns, N);
        solve_one<N, true>(o.solve, e, obase, ns, in, sm, L);
        __syncthreads();
        const bool og = o.solve.do_og;
        const int stt = og ? o.solve.og.status[e] : o.solve.ip.status[e];
        if (stt != COINFER_ST_OK) {  // og/ip_ssa would throw out of step()
          status = stt;
          break;
        }
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
          for (int x = 0; x < ns; ++x) lc = smin(lc, sdl[x]);
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
        n_tasks += ns;
        if ((pend >> lane) & 1u) lrem = 0.0;
        __syncwarp();
      }
      // forced rescue at f_max (online_sim.hpp:149-158), user order
      {
        const bool resc = own && lrem > 0.0 && __dsub_rn(lrem, o.slot) < floor_;
        const unsigned rm = __ballot_sync(kFull, resc);
        if (rm) {
          const double term = resc ? __dmul_rn(__dmul_rn(__dmul_rn(ukap, W), ufmax), ufmax) : 0.0;
          forced = lane_fold(forced, term, rm, M);
          n_resc = __popc(rm);
          n_forced += n_resc;
          if (resc) lrem = 0.0;
        }
      }
      ++tick;
      if (lrem > 0.0) lrem = __dsub_rn(lrem, o.slot);
      ebusy = smax(0.0, __dsub_rn(ebusy, o.slot));
      sample_arrivals();
      if (__ballot_sync(kFull, own && lrem > 0.0 && lrem < __dsub_rn(floor_, 1e-12)) != 0u)
        status = COINFER_ST_SLIPPED;
      tot_energy = __dadd_rn(tot_energy, energy);
      tot_forced = __dadd_rn(tot_forced, forced);
      if (trace && lane == 0) {
        const double reward = -__dadd_rn(energy, forced);
        if (o.tr_reward) o.tr_reward[tbase + t] = reward;
        if (o.tr_energy) o.tr_energy[tbase + t] = energy;
        if (o.tr_pending) o.tr_pending[tbase + t] = pending_before;
        if (o.tr_busy) o.tr_busy[tbase + t] = busy_before;
        if (o.tr_action) o.tr_action[tbase + t] = pmode;
        if (o.tr_forced) o.tr_forced[tbase + t] = n_resc;
      }
      if (status != COINFER_ST_OK) break;
    }
    (void)users;
    if (o.fin_state && own) {
      double* fs = o.fin_state + (size_t)e * (2 * M + 1);
      fs[lane] = lrem;
      fs[M + lane] = expiry;
      if (lane == 0) fs[2 * M] = ebusy;
    }
    if (lane == 0) {
      if (o.status) o.status[e] = status;
      if (o.draws) o.draws[e] = ndraw;
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
    __syncwarp();
  }
}

#ifdef CFB_PHASE_TIMING
extern "C" int coinfer_debug_online_phase_cycles(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
  }
  return 0;
}
#endif

int online_warp_smem_bytes(int M, int N) {
  const int solver = make_layout(M, N).total;
  return solver + 8 * 7 * M + 8 * 312 + 8 * 128 + 4 * 32 + 16;
}

int online_smem_bytes(int M, int N) {
  const int solver = make_layout(M, N).total;
  return solver + 8 * (3 * M + 7 * M) + 8 * Mt64::n + 4 * (8 + M) + 16;
}

template <int N>
static cudaError_t launch_online_n(const OnlineArgs& a_in, int grid, cudaStream_t st) {
  OnlineArgs a = a_in;
  a.L = make_layout(a.M, N);
  static const bool serial = std::getenv("COINFER_ONLINE_SERIAL") != nullptr;  // testing aid
  if (a.M <= 32 && !serial) {
    const int smem = online_warp_smem_bytes(a.M, N);
    cudaError_t e = ensure_smem((const void*)online_warp_kernel<N>, smem);
    if (e != cudaSuccess) return e;
    online_warp_kernel<N><<<grid, 32, smem, st>>>(a);
    return cudaGetLastError();
  }
  const int smem = online_smem_bytes(a.M, N);
  cudaError_t e = ensure_smem((const void*)online_kernel<N>, smem);
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
