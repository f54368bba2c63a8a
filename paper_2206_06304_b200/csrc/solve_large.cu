// solve_large.cu — IP-SSA / OG for instances too large for shared memory
// (BASELINE config 4: M = 4096 users in one instance).
//
// Same algorithm and bit-exact semantics as solve_core.cuh (see the comments
// there and in solve_small.cu); only the data placement and the work split
// differ:
//   large_prep    one warp per user: contract check, stable deadline rank,
//                 hoisted records (global, sorted order), sum_latency table
//   large_rows    one thread per row: first infeasible bound b0 (row 0 is the
//                 IP-SSA row when requested)
//   large_grow    one warp per G row (group start i): chains b = 1..cnt in
//                 passes of 32 lanes, each pass one left fold over j; the
//                 warp-wide lexicographic argmin (energy asc, b desc) per cell
//                 merges into the row with `<=` (later passes carry larger b)
//   large_pfit    one warp per row, a lane per useful DP cell: the
//                 feasible-prev prefix length (groups_fit is monotone in prev)
//   large_dp      one warp: the grouping DP over M sequential stages when
//                 every row has <= 96 useful cells (dense prefix-minimum ring)
//   large_finish  one CTA: otherwise the grouping DP over M sequential stages
//                 (offline_solvers.hpp:313-330), the same O(1)-per-cell scheme
//                 as solve_core.cuh: the triangle holds column prefix minima
//                 and their first positions (running values of each column in
//                 shared memory), so a cell is one gather plus a rare binary
//                 search; best_i, backtrack, stitch, lc fallback, IP-SSA outputs.
// G, the prefix minima (St) and the u16 triangles are upper triangles in
// global memory, row-major.

#include <type_traits>

#include "solve_core.cuh"

namespace cfb {

namespace {

__device__ __forceinline__ long long tri_u(long long i, long long j, long long M) {
  return i * M - ((i * (i - 1)) >> 1) + (j - i);  // upper triangle, row-major
}
[[maybe_unused]] __device__ __forceinline__ long long tri_l(long long j, long long p) {
  return ((j * (j + 1)) >> 1) + p;  // lower triangle: row j holds p = 0..j
}

// fast DP (large_dp): rows of <= kFastDW useful cells, live columns in a
// shared-memory ring of kFastDR slots
constexpr int kFastDW = 96, kFastDR = 128;

}  // namespace

// The IP-SSA deadline: the caller's (host value or device pointer), else `dflt`.
__device__ __forceinline__ double ip_deadline(const LargeArgs& a, double dflt) {
  return a.l_ip_dev ? *a.l_ip_dev : (a.has_l_ip ? a.l_ip : dflt);
}

template <int N>
__global__ void large_prep(LargeArgs a) {  // one warp per user m (and per sumlat entry m)
  using R = Rec<N>;
  const int M = a.M;
  const int m = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (m < M) {
    const double d = a.dl[m];
    int r = 0;
    for (int o = lane; o < M; o += 32) {  // stable rank by (deadline, id), offline_solvers.hpp:292-296
      const double e = __ldg(a.dl + o);
      r += (e < d) || (e == d && o < m);
    }
    r = __reduce_add_sync(kFull, r);
    if (lane == 0) {
      const double rd = a.rd ? a.rd[m] : 1.0, pd = a.pd ? a.pd[m] : 0.0;
      const int code = check_user(a.fmin[m], a.fmax[m], a.kappa[m], a.ru[m], rd, a.pu[m], pd,
                                  a.arr[m], a.dl[m]);
      if (code != COINFER_ST_OK && *a.status != COINFER_ST_SHORT_TABLE) atomicMin(a.status, m * 32 + code);
      // SIMPLE path conditions (solve_core.cuh, device_common.cuh: fast_div_*)
      if (!(a.arr[m] == 0.0 && a.fmin[m] == 0.0 && fast_div_deadline(a.dl[m]))) atomicAnd(a.simple, 0);
      a.rank[m] = r;
      a.order[r] = m;
      a.dls[r] = d;
      build_rec<N>(a.rec + (size_t)r * R::SIZE, a.P, a.fmin[m], a.fmax[m], a.kappa[m], a.ru[m], a.pu[m],
                   a.arr[m], d);
    }
  }
  if (lane == 0 && m >= 1 && m <= M) {  // sum_latency(size = m), offline_solvers.hpp:42-47
    double t = 0.0;
    for (int n = 1; n <= N; ++n) t = __dadd_rn(t, __ldg(a.lat + (size_t)(n - 1) * a.P.bmax + m - 1));
    a.sumlat[m] = t;
  }
}

template <int N>
__global__ void large_rows(LargeArgs a) {
  if (*a.status != INT_MAX) return;
  const int M = a.M, nip = a.do_ip ? 1 : 0, Q = nip + (a.do_og ? M : 0);
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  const bool isip = q < nip;
  const int len = isip ? M : M - (q - nip);
  const double d = isip ? ip_deadline(a, a.dls[0]) : a.dls[q - nip];
  a.b0[q] = first_infeasible<N>(a.lat, a.P.bmax, d, len);
  if (!isip) {
    // useful length (solve_core.cuh, "Useful cells"): cells (row, j) with
    // dl[0] + sumlat(j-row+1) > dl[row] have no fitting prev, so the DP
    // never reads their G; the row's chains stop before them and bounds
    // b > rlen do not run
    const int row = q - nip;
    int lo = 0, hi = len;
    if (row > 0)
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__dadd_rn(a.dls[0], a.sumlat[mid]) <= d) lo = mid; else hi = mid - 1;
      }
    else
      lo = len;
    a.rlen[row] = lo;
  }
}

template <int N, bool SIMPLE>
__device__ __forceinline__ void grow_row(const LargeArgs& a, int q, int lane) {
  using R = Rec<N>;
  const int M = a.M, nip = a.do_ip ? 1 : 0;
  const bool isip = q < nip;
  const int row = q - nip;
  const int len = isip ? M : M - row;
  const int b0q = a.b0[q];
  const double dlq = isip ? ip_deadline(a, a.dls[0]) : a.dls[row];
  const double INF = dinf();
  double* gE = isip ? a.ipres : a.G + tri_u(row, row, M);
  uint16_t* gB = isip ? a.ipb : a.bstar + tri_u(row, row, M);
  if (!isip)
    for (int kk = lane; kk < len; kk += 32) gE[kk] = INF;
  else if (lane == 0)
    gE[0] = INF;
  __syncwarp();
  bool num_ok = true;
#pragma unroll
  for (int n = 1; n < N; ++n) num_ok = num_ok && numerator_fast_ok(a.P.prefix[n]);
  const int rl = isip ? M : a.rlen[row];  // useful length (large_rows)
  // regular chains b < b0, 32 per pass, in b order; a chain is dropped once
  // a user is infeasible or its offloader count exceeds b (it never
  // decreases), and a pass ends when all its chains are dropped
  const int creg = b0q - 1 < rl ? b0q - 1 : rl;
  for (int base = 0; base < creg; base += 32) {
    const int b = base + lane + 1;
    bool alive[1] = {b <= creg};
    const bool al[1] = {false};
    const int kmin = isip ? M - 1 : b - 1;
    double s[1][N], tot[1] = {0.0};
    if (alive[0]) {
      start_times<N>(a.lat, a.P.bmax, dlq, b, s[0]);
    } else {
#pragma unroll
      for (int n = 0; n < N; ++n) s[0][n] = -1.0;
    }
    int off = 0;
    // the pass's winner for cell kk (the min energy, largest b on ties) is
    // parked in lane kk % 32 and merged into the row 32 cells at a time
    // (coalesced, off the per-step critical path)
    double pv = INF;
    int pb = 0;
    auto flush = [&](int w0) {
      const int cellk = w0 + lane;
      if (pv != INF && cellk < rl && pv <= gE[cellk]) {  // later passes carry larger b: they win ties
        gE[cellk] = pv;
        gB[cellk] = (uint16_t)pb;
      }
      pv = INF;
    };
    int kk = 0;
    for (; kk < rl && __any_sync(kFull, alive[0]); ++kk) {
      if (alive[0]) {
        const int ri = isip ? a.rank[kk] : row + kk;
        int sp[1] = {0};
        const bool live[1] = {true};
        eval_multi<N, 1, SIMPLE>(a.rec + (size_t)ri * R::SIZE, a.P, s, al, num_ok, live, tot, sp);
        off += (sp[0] >= 0 && sp[0] < N);
        alive[0] = sp[0] >= 0 && off <= b;
      }
      const bool cand = alive[0] && kk >= kmin;
      const unsigned long long key = (unsigned long long)__double_as_longlong(tot[0]);
      const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
      const unsigned mh = __reduce_min_sync(kFull, cand ? khi : 0xffffffffu);
      const bool hit = cand && khi == mh;
      unsigned wm = __ballot_sync(kFull, hit);
      if (__popc(wm) > 1) {
        const unsigned ml = __reduce_min_sync(kFull, hit ? klo : 0xffffffffu);
        wm = __ballot_sync(kFull, hit && klo == ml);
      }
      if (isip) {
        if (wm != 0u && lane == 31 - __clz(wm) && tot[0] <= gE[0]) {
          gE[0] = tot[0];
          gB[0] = (uint16_t)b;
        }
        continue;
      }
      const int win = 31 - __clz(wm);  // -1: no candidate
      const double wv = __shfl_sync(kFull, tot[0], win & 31);
      if (lane == (kk & 31) && wm != 0u) {
        pv = wv;
        pb = base + win + 1;
      }
      if ((kk & 31) == 31) flush(kk - 31);
    }
    if (!isip && (kk & 31) != 0) flush(kk & ~31);
    __syncwarp();
  }
  // the all-local chain (every bound >= b0): each user runs local_only_choice
  // at f_L, so a step is that user's N local fold terms; its key is the
  // largest admissible bound (j-i+1, IP: M), larger than every regular b.
  // The fold stays one sequential sum; the warp computes 32 users' terms at
  // a time, every lane runs the (identical) sum over them through shuffles
  // and keeps the partial sum after its own user, then the 32 cells merge
  // at once.
  if (b0q <= rl) {
    const int kmin = isip ? M - 1 : b0q - 1;
    double t = 0.0;
    for (int c0 = 0; c0 < rl; c0 += 32) {
      const int kk = c0 + lane;
      double x[N];
      bool feas = false;
      if (kk < rl) {
        const double* r = a.rec + (size_t)(isip ? a.rank[kk] : row + kk) * R::SIZE;
        feas = r[R::FEAS] != 0.0;
        const double fL = r[R::FL];
#pragma unroll
        for (int n = 1; n <= N; ++n) x[n - 1] = __dmul_rn(__dmul_rn(r[R::KA(n)], fL), fL);
      } else {
#pragma unroll
        for (int n = 0; n < N; ++n) x[n] = 0.0;
      }
      // users up to the first one that cannot meet its deadline locally
      const unsigned bad = __ballot_sync(kFull, kk < rl && !feas);
      const int stop = bad ? __ffs(bad) - 1 : (rl - c0 < 32 ? rl - c0 : 32);
      double mine = INF;
      for (int u = 0; u < stop; ++u) {
#pragma unroll
        for (int n = 0; n < N; ++n) t = __dadd_rn(t, __shfl_sync(kFull, x[n], u));
        if (lane == u) mine = t;
      }
      if (lane < stop && kk >= kmin) {
        const int slot = isip ? 0 : kk;
        if (mine <= gE[slot]) {
          gE[slot] = mine;
          gB[slot] = (uint16_t)(isip ? M : kk + 1);
        }
      }
      if (bad) break;
    }
  }
  __syncwarp();
}

template <int N>
__global__ void __launch_bounds__(128) large_grow(LargeArgs a) {
  if (*a.status != INT_MAX) return;
  const int nip = a.do_ip ? 1 : 0, Q = nip + (a.do_og ? a.M : 0);
  const int q = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (q >= Q) return;
  if (*a.simple)
    grow_row<N, true>(a, q, threadIdx.x & 31);
  else
    grow_row<N, false>(a, q, threadIdx.x & 31);
}

// One CTA: DP, backtrack, stitch, outputs (and the IP-SSA outputs).
#ifndef CFB_LARGE_SHORT
#define CFB_LARGE_SHORT 3  // DP rows of <= 32*this useful cells run on one warp
#endif
#ifdef CFB_LARGE_TIMING
__device__ unsigned long long g_large_t[8];
extern "C" int coinfer_debug_large_times(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_large_t, sizeof(unsigned long long) * 8);
  return 0;
}
#endif
// The grouping DP when every row i >= 1 has <= kFastDW useful cells (C4:
// ~35, peaks in the 70s), one row per stage (offline_solvers.hpp:313-330).  Column c's useful rows are row 0 and a suffix [q1(c), c], so
// its prefix minima live dense over that suffix: S0[c] (row 0) below
// q1(c), then one entry per row; only columns i-1 .. i+DW are live at
// stage i, so they sit in a ring of DR column slots.
//   Stage i needs column i-1 complete and nothing else new: its critical
// path is one shared load of column i-1 and of each cell's running
// minimum, an add, a compare and the stores.  Two warps run it (32 and 64
// cells of the row), so every dependency is exposed: the stage is
// straight-line code over only the
// row's live 32-cell chunks (stores of lanes past the row go to a dummy
// slot instead of branching), the parent's tie check (rounding that merges
// an earlier, larger S into the same sum) reads column i-1 beside the
// critical chain, and the rows' G / pfit are staged by cp.async in a
// producer warp (dp_producer), which hands each stage a record (G, pfit
// masked to the useful cells, the column's q1) two stages ahead.
namespace {
constexpr int kPD = 4;  // rows of G / pfit in flight (power of 2)
constexpr int kQ = 4;   // stage records in the ring the producer warp fills (power of 2)
constexpr int kDpSmemMax = 227 * 1024;  // large_dp runs when its shared memory fits (M <= ~8,000)
template <int NW>
struct DpIn {  // one stage's inputs, per lane: cells i + 32(C0 + k) + lane of this warp's chunks
  double g[NW], s0j[NW];
  int p[NW], qj[NW];
  int rl, q1c;
  double s0c;
};
struct DpPtrs {  // large_dp's shared-memory arrays
  double *S0, *ringV, *runV, *stG, *recG, *recS0c;
  uint16_t *ringA, *runA, *q1, *rlS;
  uint32_t *stP, *recPQ;
  int* recRl;  // [kQ] row length, [kQ] q1(i-1)
};
__device__ __forceinline__ void dp_bar() { asm volatile("bar.sync 1, 96;" : : : "memory"); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" : : "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" : : "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" : : : "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" : : "n"(K) : "memory"); }
// large_dp's shared memory: S0 | ring values (+1 dummy) | running values
// (+1 dummy) | ring positions | running positions | q1 | rlen | staged G |
// staged pfit words
struct DpSmem {
  int oRingV, oRunV, oRingA, oRunA, oQ1, oRl, oStG, oStP, oRecG, oRecPQ, oRecS0c, oRecRl, bytes;
  __host__ __device__ explicit DpSmem(int M) {
    auto al = [](int x) { return (x + 15) & ~15; };
    oRingV = al(8 * M);
    oRunV = al(oRingV + 8 * (kFastDR * kFastDW + 1));
    oRingA = al(oRunV + 8 * (kFastDR + 1));
    oRunA = al(oRingA + 2 * (kFastDR * kFastDW + 1));
    oQ1 = al(oRunA + 2 * (kFastDR + 1));
    oRl = al(oQ1 + 2 * M);
    oStG = al(oRl + 2 * M);
    oStP = al(oStG + 8 * kPD * kFastDW);
    oRecG = al(oStP + 4 * kPD * kFastDW);
    oRecPQ = al(oRecG + 8 * kQ * kFastDW);
    oRecS0c = al(oRecPQ + 4 * kQ * kFastDW);
    oRecRl = al(oRecS0c + 8 * kQ);
    bytes = al(oRecRl + 8 * kQ);
  }
};
}  // namespace

// large_dp's producer warp: G and pfit rows staged by cp.async kPD rows
// ahead (kPD), and per row the stage record the DP warps read -- each cell's G
// and (pfit masked to the row's useful cells | q1 of its column), the row
// length, q1(i-1), S0[i-1] -- into a ring of kQ records, two rows ahead of
// the stage that reads them (one named barrier per stage orders both).
__device__ __forceinline__ void dp_producer(const LargeArgs& a, const DpPtrs& sp, int lane) {
  constexpr int DW = kFastDW;
  const int M = a.M;
  const double* __restrict__ G = a.G;
  const uint16_t* __restrict__ PF = a.pfit;
  auto xrow = [&](int i) {
    const uint32_t ui = (uint32_t)i;
    return ui * (uint32_t)M - ui * (ui - 1u) / 2u - ui;
  };
  auto issue = [&](int r) {
    if (r < M) {
      const int s = (r & (kPD - 1)) * DW;
      const uint32_t xr = xrow(r);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const uint32_t x = xr + (uint32_t)min(r + 32 * c + lane, M - 1);
        cp_async8(sp.stG + s + 32 * c + lane, G + x);
        cp_async4(sp.stP + s + 32 * c + lane,
                  reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(PF + x) & ~(uintptr_t)3));
      }
    }
    cp_async_commit();
  };
  auto produce = [&](int r) {  // record of row r (1 <= r < M)
    issue(r + kPD - 1);
    cp_async_wait<kPD - 1>();  // row r has landed
    const int s = (r & (kPD - 1)) * DW, q = (r & (kQ - 1)) * DW;
    const uint32_t xr = xrow(r);
    const int rl = sp.rlS[r];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int jt = r + 32 * c + lane, j = min(jt, M - 1);
      const uint32_t pw = jt < r + rl  // past the row's useful cells pfit is not computed
                              ? (sp.stP[s + 32 * c + lane] >> (((xr + (uint32_t)j) & 1u) * 16u)) & 0xffffu : 0u;
      sp.recG[q + 32 * c + lane] = sp.stG[s + 32 * c + lane];
      sp.recPQ[q + 32 * c + lane] = pw | ((uint32_t)sp.q1[j] << 16);
    }
    if (lane == 0) {
      sp.recRl[r & (kQ - 1)] = rl;
      sp.recRl[kQ + (r & (kQ - 1))] = sp.q1[r - 1];
      sp.recS0c[r & (kQ - 1)] = sp.S0[r - 1];
    }
  };
  for (int r = 1; r < kPD; ++r) issue(r);
  produce(1);
  if (2 < M) produce(2);
  dp_bar();  // records 1 and 2
  for (int i = 1; i < M; ++i) {
    if (i + 2 < M) produce(i + 2);
    dp_bar();  // end of stage i
  }
  cp_async_wait<0>();
}

// One of large_dp's two DP warps: chunks C0 .. C0+NCW-1 (32 cells each) of
// every row; the warps meet at a named barrier after each stage (a stage
// reads ring entries the other warp wrote in the stages before).
template <int C0, int NCW>
__device__ __forceinline__ void dp_warp(const LargeArgs& a, const DpPtrs& sp, int lane) {
  constexpr int DW = kFastDW, DR = kFastDR;
  const int M = a.M;
  const double INF = dinf();
  double* __restrict__ ringV = sp.ringV;
  double* __restrict__ runV = sp.runV;
  uint16_t* __restrict__ ringA = sp.ringA;
  uint16_t* __restrict__ runA = sp.runA;
  uint16_t* __restrict__ PAR = a.par;
  // 32-bit triangle offsets (M <= 8192: < 2^26 cells): x(i, j) = xr(i) + j
  auto xrow = [&](int i) {
    const uint32_t ui = (uint32_t)i;
    return ui * (uint32_t)M - ui * (ui - 1u) / 2u - ui;
  };
  auto fetch = [&](DpIn<NCW>& R, int i) {  // row i's stage record into registers
    if (i >= M) return;
    const int q = (i & (kQ - 1)) * DW;
    R.rl = sp.recRl[i & (kQ - 1)];
    R.q1c = sp.recRl[kQ + (i & (kQ - 1))];
    R.s0c = sp.recS0c[i & (kQ - 1)];
#pragma unroll
    for (int k = 0; k < NCW; ++k) {
      const int c = C0 + k;
      const uint32_t pq = sp.recPQ[q + 32 * c + lane];
      R.g[k] = sp.recG[q + 32 * c + lane];
      R.p[k] = (int)(pq & 0xffffu);
      R.qj[k] = (int)(pq >> 16);
      R.s0j[k] = sp.S0[min(i + 32 * c + lane, M - 1)];
    }
  };
  auto stage = [&](const DpIn<NCW>& R, int i, auto nc_tag) {
    constexpr int NC = decltype(nc_tag)::value;  // live chunks of this warp
    const int jend = i + R.rl, q1c = R.q1c;
    const double s0c = R.s0c;
    const int cs = ((i - 1) & (DR - 1)) * DW - q1c;  // column i-1: entry of row r at cs + r, r >= q1c
    double best[NC], cand[NC], vC[NC], vR[NC], npm[NC], vT[NC];
    int bp[NC], aC[NC], aR[NC], na[NC], ws[NC], wr[NC];
    bool tie[NC];
    // all loads of the stage first (the compiler cannot move a load of one
    // chunk above a store of another), then the selects, then the stores
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int slot = min(i + 32 * (C0 + k) + lane, M - 1) & (DR - 1), rc = max(R.p[k] - 1, q1c);
      vC[k] = ringV[cs + rc];
      aC[k] = ringA[cs + rc];
      vR[k] = runV[slot];
      aR[k] = runA[slot];
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int pma = R.p[k] - 1 < q1c ? 0 : aC[k];
      vT[k] = ringV[cs + max(pma - 1, q1c)];  // the row before the minimum's first position
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int jt = i + 32 * (C0 + k) + lane, slot = min(jt, M - 1) & (DR - 1);
      const bool in = jt < jend;
      const int p = R.p[k], r = p - 1;
      const double rv = r < q1c ? s0c : vC[k];
      const int pma = r < q1c ? 0 : aC[k];
      const bool first = i == R.qj[k];
      const double pmj = first ? R.s0j[k] : vR[k];
      const int paj = first ? 0 : aR[k];
      const double g = R.g[k];
      const bool valid = in && g != INF && p > 0;
      cand[k] = __dadd_rn(rv, g);
      best[k] = valid ? cand[k] : INF;   // (rv = INF gives cand = INF)
      const bool lower = best[k] < pmj;  // strict: the first position is kept
      npm[k] = lower ? best[k] : pmj;
      na[k] = lower ? i : paj;
      ws[k] = in ? slot : DR;  // lanes past the row store to the dummy slot
      wr[k] = in ? slot * DW + (i - R.qj[k]) : DR * DW;
      const bool fin = valid && cand[k] != INF;
      bp[k] = fin ? pma : 0xffff;
      tie[k] = fin && pma > 0 && __dadd_rn(pma - 1 < q1c ? s0c : vT[k], g) == cand[k];
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      runV[ws[k]] = npm[k];
      runA[ws[k]] = (uint16_t)na[k];
      ringV[wr[k]] = npm[k];
      ringA[wr[k]] = (uint16_t)na[k];
    }
    bool anytie = false;
#pragma unroll
    for (int k = 0; k < NC; ++k) anytie = anytie || tie[k];
    if (__any_sync(kFull, anytie)) {
#pragma unroll
      for (int k = 0; k < NC; ++k)
        if (tie[k]) {  // the first row whose S sums to the same value
          const double g = R.g[k];
          int qa = 0, qb = bp[k] - 1;
          while (qa < qb) {
            const int mid = (qa + qb) >> 1;
            if (__dadd_rn(mid < q1c ? s0c : ringV[cs + mid], g) == cand[k]) qb = mid; else qa = mid + 1;
          }
          bp[k] = qb;
        }
    }
    const uint32_t xr = xrow(i);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int jt = i + 32 * (C0 + k) + lane;
      if (jt < jend) {
        PAR[xr + (uint32_t)jt] = (uint16_t)bp[k];
        if (jt == M - 1) a.slast[i] = best[k];
      }
    }
  };
  auto step = [&](const DpIn<NCW>& cur, DpIn<NCW>& nxt, int i) {
    // the next stage's record first (the producer wrote it before the last
    // barrier): its loads then run beside this stage's chain
    fetch(nxt, i + 1);
    const int live = ((cur.rl + 31) >> 5) - C0;  // this warp's chunks holding useful cells
    if (C0 == 0 && lane == 0 && i + cur.rl < M) a.slast[i] = INF;
    if (live >= NCW) stage(cur, i, std::integral_constant<int, NCW>{});
    else if (NCW > 1 && live == 1) stage(cur, i, std::integral_constant<int, 1>{});
    dp_bar();                      // both warps' stores of stage i before stage i + 1's loads
  };
  dp_bar();  // records 1 and 2
  DpIn<NCW> A, B;
  fetch(A, 1);
  for (int i = 1; i < M; i += 2) {
    step(A, B, i);
    if (i + 1 >= M) break;
    step(B, A, i + 1);
  }
}

__global__ void __launch_bounds__(256) large_dp(LargeArgs a) {
  if (*a.status != INT_MAX) return;
  extern __shared__ __align__(16) unsigned char smb[];
  constexpr int DW = kFastDW;
  const int M = a.M, tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  __shared__ int ired[8];
  int rlmax = 0;
  for (int j = 1 + tid; j < M; j += NT) rlmax = max(rlmax, a.rlen[j]);
  rlmax = __reduce_max_sync(kFull, rlmax);
  if (lane == 0) ired[warp] = rlmax;
  __syncthreads();
  rlmax = 0;
  for (int w = 0; w < NW; ++w) rlmax = max(rlmax, ired[w]);
  if (rlmax > DW || DpSmem(M).bytes > kDpSmemMax) return;  // large_finish runs the change-point DP
  const double INF = dinf();
  const DpSmem L(M);
  double* S0 = reinterpret_cast<double*>(smb);                   // [M] row 0: S = G = PM
  double* ringV = reinterpret_cast<double*>(smb + L.oRingV);      // [DR*DW] PM_c over rows q1(c).. | dummy
  double* runV = reinterpret_cast<double*>(smb + L.oRunV);        // [DR] running PM of live columns | dummy
  uint16_t* ringA = reinterpret_cast<uint16_t*>(smb + L.oRingA);  // first positions of the PMs
  uint16_t* runA = reinterpret_cast<uint16_t*>(smb + L.oRunA);
  uint16_t* q1 = reinterpret_cast<uint16_t*>(smb + L.oQ1);        // [M] first useful row >= 1 per column (M: none)
  uint16_t* rlS = reinterpret_cast<uint16_t*>(smb + L.oRl);       // [M] useful row lengths
  double* stG = reinterpret_cast<double*>(smb + L.oStG);          // [kPD*DW] staged G rows
  uint32_t* stP = reinterpret_cast<uint32_t*>(smb + L.oStP);      // [kPD*DW] staged pfit words
  for (int j = tid; j < M; j += NT) {
    S0[j] = a.G[tri_u(0, j, M)];
    a.par[tri_u(0, j, M)] = 0xffff;
    q1[j] = (uint16_t)M;
    rlS[j] = (uint16_t)a.rlen[j];
  }
  if (tid == 0) a.slast[0] = a.G[tri_u(0, M - 1, M)];
  __syncthreads();
  for (int q = 1 + tid; q < M; q += NT) {  // columns whose first useful row >= 1 is q
    const int e0 = q == 1 ? 1 : (q - 1) + a.rlen[q - 1], e1 = q + a.rlen[q];
    for (int c = max(e0, 1); c < e1 && c < M; ++c) q1[c] = (uint16_t)q;
  }
  __syncthreads();
  const DpPtrs sp{S0, ringV, runV, stG,
                  reinterpret_cast<double*>(smb + L.oRecG), reinterpret_cast<double*>(smb + L.oRecS0c),
                  ringA, runA, q1, rlS, stP, reinterpret_cast<uint32_t*>(smb + L.oRecPQ),
                  reinterpret_cast<int*>(smb + L.oRecRl)};
  if (warp == 0) dp_warp<0, 1>(a, sp, lane);       // cells i .. i+31 of each row
  else if (warp == 1) dp_warp<1, 2>(a, sp, lane);  // cells i+32 .. i+95
  else if (warp == 2) dp_producer(a, sp, lane);    // G / pfit staging and the stage records
}

template <int N>
__global__ void __launch_bounds__(1024) large_finish(LargeArgs a) {
  using R = Rec<N>;
  extern __shared__ __align__(16) unsigned char smb[];
  const int M = a.M, nip = a.do_ip ? 1 : 0;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  // shared memory: DP running column minima + the cached column i-1;
  // after the DP the group bounds reuse the column cache
  constexpr int RING = 128, CAP = 16;  // shared-memory mirror of recent columns (DP)
  double* runPM = reinterpret_cast<double*>(smb);        // [M] running column minima
  double* colV = runPM + M;                               // [M] a column staged from global
  double* ringV = colV + M;                               // [RING*CAP]
  int* ringOwn = reinterpret_cast<int*>(ringV + RING * CAP);  // [RING]
  uint16_t* ringR = reinterpret_cast<uint16_t*>(ringOwn + RING);  // [RING*CAP]
  uint16_t* ccount = ringR + RING * CAP;                  // [M] change points per column
  uint16_t* colR = ccount + M;                            // [M]
  uint16_t* rlenS = colR + M;                             // [M] useful row lengths
  uint16_t* runRow = rlenS + M;                           // [M] row of the last change point
  int* gl = reinterpret_cast<int*>(colV);  // after the DP
  int* gh = gl + M;
  const double* dls = a.dls;
  __shared__ double wred[32];
  __shared__ int ired[32];
  __shared__ int s_best, s_ng, s_st;
  const double INF = dinf();
  const ProfileConst& P = a.P;
  const size_t base = a.base;
  if (*a.status != INT_MAX) {  // Scenario::check failed: first failing user, first test
    if (tid == 0) {
      if (a.do_ip && a.ip.status) a.ip.status[a.k] = *a.status & 31;
      if (a.do_og && a.og.status) a.og.status[a.k] = *a.status & 31;
    }
    return;
  }
  // ------------------------------------------------------------- IP-SSA out
  if (a.do_ip) {
    const double ipE = a.ipres[0];
    const int ipbv = a.ipb[0];
    if (ipE == INF) {
      if (tid == 0 && a.ip.status) a.ip.status[a.k] = COINFER_ST_INFEASIBLE;
    } else {
      const double l_ip = ip_deadline(a, dls[0]);
      const bool pipe = ipbv < a.b0[0];
      double s[N];
      if (pipe) start_times<N>(a.lat, P.bmax, l_ip, ipbv, s);
      else
#pragma unroll
        for (int n = 0; n < N; ++n) s[n] = 0.0;
      for (int m = tid; m < M; m += NT) {
        const double* r = a.rec + (size_t)a.rank[m] * R::SIZE;
        int sp;
        double f;
        choose<N>(r, P, s, pipe, sp, f);
        if (a.ip.split) a.ip.split[base + m] = (uint8_t)sp;
        if (a.ip.freq) a.ip.freq[base + m] = f;
        if (a.ip.user_energy) a.ip.user_energy[base + m] = fold<N>(r, sp, f, 0.0);
        a.spos[a.rank[m]] = sp;
      }
      __syncthreads();
      if (a.ip.batch_size)
        for (int n = 1 + tid; n <= N; n += NT) {
          int c = 0;
          for (int x = 0; x < M; ++x) c += a.spos[x] < n;
          a.ip.batch_size[(size_t)a.k * N + n - 1] = c;
        }
      if (tid == 0) {
        if (a.ip.status) a.ip.status[a.k] = COINFER_ST_OK;
        if (a.ip.batch_bound) a.ip.batch_bound[a.k] = ipbv;
        if (a.ip.pipeline_feasible) a.ip.pipeline_feasible[a.k] = pipe;
        if (a.ip.energy) a.ip.energy[a.k] = ipE;
      }
    }
    __syncthreads();
  }
  if (!a.do_og) return;

  // ------------------------------------------------------------------ DP
  // S[i][j] = min over feasible prev of fl(S[prev][i-1] + G[i][j]), smallest
  // prev on ties: feasible prevs are the prefix [0, pfit) and the minimum
  // is fl(PM + g) with PM the column prefix minimum; the parent is the first
  // position of that minimum unless rounding merges an earlier, larger S
  // into the same sum (then the earliest such position).  A column's prefix
  // minimum is a step function of the row that drops only where S sets a
  // new strict minimum, so each column keeps just its change points (row,
  // value) -- about ln(M) of them -- appended in global memory (column c
  // at c(c+1)/2, the worst case fits).  Stage i loads the finished column
  // i-1's change points into shared memory; PM(p-1) is the last change
  // point at a row <= p-1, its row is the first position of the minimum,
  // and earlier rows with the same sum are earlier change points (binary
  // searches over a handful of entries).  Cells past a row's useful length
  // have no fitting prev (pfit 0).
  //   Change points always go to global memory (chgV/chgR, complete); a
  // column whose first change after row 0 comes in a short-row stage also
  // gets a slot in a shared-memory ring (column c in slot c % 128, up to 16
  // points, claimed only once the slot's previous column has been read), so
  // stage i usually finds column i-1 in shared memory: in the ring, or --
  // when it has a single change point -- in runPM/runRow.  Only a column
  // that overflowed or missed the ring is staged from global memory.
  // Fast DP when every row i >= 1 has <= DW useful cells (C4: ~35, peaks in
  // the 70s).  Column c's useful rows are row 0 and a suffix [q1(c), c]
  // (c - q < rlen(q) is monotone in q >= 1), so the column prefix minima
  // live DENSE over that suffix: S0[c] (row 0) below q1(c), then one entry
  // per row -- the small path's in-place scheme (solve_core.cuh) with O(1)
  // lookups instead of change-point searches.  Only columns i-1 .. i+DW are
  // live at stage i, so they sit in a shared-memory ring of DR columns.
  // That DP is its own kernel, large_dp (below), launched just before this
  // one; it and this kernel take the same decision from the row lengths.
  int rlmax = 0;
  for (int j = 1 + tid; j < M; j += NT) rlmax = max(rlmax, a.rlen[j]);
  rlmax = __reduce_max_sync(kFull, rlmax);
  if (lane == 0) ired[warp] = rlmax;
  __syncthreads();
  rlmax = 0;
  for (int w = 0; w < NW; ++w) rlmax = max(rlmax, ired[w]);
  __syncthreads();
  const bool fastdp = rlmax <= kFastDW && DpSmem(M).bytes <= kDpSmemMax;  // (the test large_dp made)
  if (fastdp) {
    // the whole DP ran in large_dp (same rlmax test): S row M-1 in slast, parents in par
  } else {
    double* chgV = a.St;
    uint16_t* chgR = a.argpm;
    auto coff = [](int c) { return (long long)c * (c + 1) / 2; };
    for (int r = tid; r < RING; r += NT) ringOwn[r] = -1;
    for (int j = tid; j < M; j += NT) rlenS[j] = (uint16_t)a.rlen[j];
    for (int j = tid; j < M; j += NT) {  // row 0: S[0][j] = G[0][j]
      const double g = a.G[tri_u(0, j, M)];
      runPM[j] = g;
      runRow[j] = 0;
      ccount[j] = g < INF ? 1 : 0;
      if (g < INF) {
        chgV[coff(j)] = g;
        chgR[coff(j)] = 0;
      }
      a.par[tri_u(0, j, M)] = 0xffff;
    }
    if (tid == 0) a.slast[0] = a.G[tri_u(0, M - 1, M)];
    __syncthreads();
    // S[i][j] for cell (i, j) given G, pfit and column i-1's change points
    // (V, Rr, nc); appends (i, S) to column j when it is a new strict minimum
    // (`claim`: short-row stages, whose <= 96 columns are distinct mod RING)
    auto cell = [&](int i, int j, long long x, double g, int p, const double* V, const uint16_t* Rr, int nc,
                    bool claim) {
      double best = INF;
      int bp = 0xffff;
      if (g != INF && p > 0) {
        int lo = 0, hi = nc;  // change points at rows <= p-1
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (Rr[mid] <= p - 1) lo = mid + 1; else hi = mid;
        }
        if (lo > 0) {
          int k = lo - 1;
          const double cand = __dadd_rn(V[k], g);
          if (cand != INF) {
            best = cand;
            if (k > 0 && __dadd_rn(V[k - 1], g) == best) {  // rounding merged earlier minima
              int ka = 0;
              --k;
              while (ka < k) {
                const int mid = (ka + k) >> 1;
                if (__dadd_rn(V[mid], g) == best) k = mid; else ka = mid + 1;
              }
            }
            bp = Rr[k];
          }
        }
      }
      if (j == M - 1) a.slast[i] = best;
      a.par[x] = (uint16_t)bp;
      if (best < runPM[j]) {  // strict: the first position is kept
        const int n = ccount[j];
        chgV[coff(j) + n] = best;
        chgR[coff(j) + n] = (uint16_t)i;
        const int slot = j & (RING - 1), own = ringOwn[slot];
        double* rv = ringV + slot * CAP;
        uint16_t* rr = ringR + slot * CAP;
        if (own == j) {
          if (n < CAP) {
            rv[n] = best;
            rr[n] = (uint16_t)i;
          } else {
            ringOwn[slot] = -1;  // overflow: the column is read from global memory
          }
        } else if (claim && n <= 1 && own < i - 1) {  // free, or its column already read
          if (n == 1) {
            rv[0] = runPM[j];
            rr[0] = runRow[j];
          }
          rv[n] = best;
          rr[n] = (uint16_t)i;
          ringOwn[slot] = j;
        }
        ccount[j] = (uint16_t)(n + 1);
        runPM[j] = best;
        runRow[j] = (uint16_t)i;
      }
    };
    // column c's change points in shared memory, or nullptr (stage them from global)
    auto column = [&](int c, int nc, const double*& V, const uint16_t*& Rr) {
      if (nc <= 1) {
        V = runPM + c;
        Rr = runRow + c;
        return true;
      }
      if (ringOwn[c & (RING - 1)] == c) {
        V = ringV + (c & (RING - 1)) * CAP;
        Rr = ringR + (c & (RING - 1)) * CAP;
        return true;
      }
      V = colV;
      Rr = colR;
      return false;
    };
    // Only a row's useful cells j < i + rlen[i] are computed: past them no
    // prev fits, S = +inf changes no running minimum and no parent is ever
    // followed.  Rows of <= 96 useful cells (all of them on C4, where rlen
    // averages ~35 and peaks in the 70s) run on warp 0 alone, synchronised by __syncwarp, with
    // the next row's G and pfit loads in flight; the other warps skip ahead to
    // the next long row, which runs on the whole CTA between barriers (<= 8
    // cells per thread since M <= 8*NT).
    constexpr int SHORT = CFB_LARGE_SHORT;  // short rows: <= 32*SHORT useful cells
    int pref = -1;  // warp 0: the row whose first 32*SHORT cells gq/pq hold
    double gq[SHORT];
    int pq[SHORT];
    auto prefetch = [&](int r) {
      const int je = r + rlenS[r];
      const long long xr = tri_u(r, r, M) - r;
  #pragma unroll
      for (int c = 0; c < SHORT; ++c) {
        const int j = r + 32 * c + lane;
        gq[c] = j < je ? a.G[xr + j] : INF;
        pq[c] = j < je ? a.pfit[xr + j] : 0;
      }
      pref = r;
    };
    for (int i = 1; i < M; ++i) {
      const int rl = rlenS[i];
      if (rl <= 32 * SHORT && warp != 0) continue;  // short row: warp 0's
      const int jend = i + rl;
      const long long xr = tri_u(i, i, M) - i;  // x(i, j) = xr + j
      const long long c0 = coff(i - 1);
      if (rl <= 32 * SHORT) {
  #ifdef CFB_LARGE_TIMING
        long long t0 = clock64();
  #endif
        if (pref != i) prefetch(i);
        double gc[SHORT];
        int pc[SHORT];
  #pragma unroll
        for (int c = 0; c < SHORT; ++c) {
          gc[c] = gq[c];
          pc[c] = pq[c];
        }
        if (i + 1 < M) prefetch(i + 1);  // in flight during this stage
        if (lane == 0 && jend < M) a.slast[i] = INF;
        const int nc = ccount[i - 1];
        const double* V;
        const uint16_t* Rr;
        const bool insm = column(i - 1, nc, V, Rr);
        if (!insm) {
          for (int q = lane; q < nc; q += 32) {
            colV[q] = chgV[c0 + q];
            colR[q] = chgR[c0 + q];
          }
          __syncwarp();
        }
  #ifdef CFB_LARGE_TIMING
        long long t1 = clock64();
        const double gsink = gc[0] + (double)pc[0];
        long long t2 = clock64();
  #endif
  #pragma unroll
        for (int c = 0; c < SHORT; ++c) {
          const int j = i + 32 * c + lane;
          if (j < jend) cell(i, j, xr + j, gc[c], pc[c], V, Rr, nc, true);
        }
        __syncwarp();
  #ifdef CFB_LARGE_TIMING
        long long t3 = clock64();
        if (lane == 0) {
          g_large_t[0] += t1 - t0;
          g_large_t[1] += t2 - t1 + (gsink == 12345.0);
          g_large_t[2] += t3 - t2;
          g_large_t[3] += 1;
          g_large_t[4] += insm ? 0 : 1;
        }
  #endif
        continue;
      }
      __syncthreads();  // warp 0's short rows are done
      const int nc = ccount[i - 1];
      if (tid == 0 && jend < M) a.slast[i] = INF;
      double gv[8];
      int pv[8];
  #pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int j = i + tid + c * NT;
        gv[c] = j < jend ? a.G[xr + j] : INF;
        pv[c] = j < jend ? a.pfit[xr + j] : 0;
      }
      const double* V;
      const uint16_t* Rr;
      if (!column(i - 1, nc, V, Rr))
        for (int q = tid; q < nc; q += NT) {
          colV[q] = chgV[c0 + q];
          colR[q] = chgR[c0 + q];
        }
      __syncthreads();
  #pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int j = i + tid + c * NT;
        if (j >= jend) break;
        cell(i, j, xr + j, gv[c], pv[c], V, Rr, nc, false);
      }
      __syncthreads();
    }
  }
  __syncthreads();

  // best_i: strict '<', smallest i (offline_solvers.hpp:332-334); S[i][M-1] = St row M-1
  {
    double bv = INF;
    int bi = M;
    for (int i = tid; i < M; i += NT) {
      const double v = a.slast[i];
      if (v < bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
      }
    }
    for (int off = 16; off; off >>= 1) {
      const double ov = __shfl_xor_sync(kFull, bv, off);
      const int oi = __shfl_xor_sync(kFull, bi, off);
      if (ov < bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      wred[warp] = bv;
      ired[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double v = INF;
      int b = M;
      for (int w = 0; w < NW; ++w)
        if (wred[w] < v || (wred[w] == v && ired[w] < b)) {
          v = wred[w];
          b = ired[w];
        }
      s_best = v == INF ? -1 : b;
      s_st = COINFER_ST_OK;
    }
    __syncthreads();
  }
  const int best_i = s_best;
  if (a.og.order)
    for (int i = tid; i < M; i += NT) a.og.order[base + i] = a.order[i];

  if (best_i < 0) {  // lc_solve fallback (offline_solvers.hpp:336-348)
    for (int i = tid; i < M; i += NT)
      if (a.rec[(size_t)i * R::SIZE + R::FEAS] == 0.0) s_st = COINFER_ST_INFEASIBLE;
    __syncthreads();
    if (s_st != COINFER_ST_OK) {
      if (tid == 0 && a.og.status) a.og.status[a.k] = COINFER_ST_INFEASIBLE;
      return;
    }
    for (int i = tid; i < M; i += NT) {
      const double* r = a.rec + (size_t)i * R::SIZE;
      const double fL = r[R::FL];
      const double e = fold<N>(r, N, fL, 0.0);
      const int m = a.order[i];
      const size_t g = base + i;
      if (a.og.group_lo) a.og.group_lo[g] = i;
      if (a.og.group_size) a.og.group_size[g] = 1;
      if (a.og.group_b) a.og.group_b[g] = 0;
      if (a.og.group_deadline) a.og.group_deadline[g] = dls[i];
      if (a.og.group_energy) a.og.group_energy[g] = e;
      if (a.og.group_batch_size)
        for (int n = 0; n < N; ++n) a.og.group_batch_size[g * N + n] = 0;
      if (a.og.group_of_user) a.og.group_of_user[base + m] = i;
      if (a.og.split) a.og.split[base + m] = (uint8_t)N;
      if (a.og.freq) a.og.freq[base + m] = fL;
      if (a.og.user_energy) a.og.user_energy[base + m] = e;
    }
    if (tid == 0) {
      double total = 0.0;  // lc_solve folds users in original order
      for (int m = 0; m < M; ++m) {
        const double* r = a.rec + (size_t)a.rank[m] * R::SIZE;
        total = fold<N>(r, N, r[R::FL], total);
      }
      if (a.og.status) a.og.status[a.k] = COINFER_ST_OK;
      if (a.og.fallback) a.og.fallback[a.k] = 1;
      if (a.og.energy) a.og.energy[a.k] = total;
      if (a.og.n_groups) a.og.n_groups[a.k] = M;
    }
    return;
  }

  // backtrack (offline_solvers.hpp:350-360)
  if (tid == 0) {
    int ng = 0, i = best_i, j = M - 1;
    while (true) {
      gl[ng] = i;
      gh[ng] = j;
      ++ng;
      if (i == 0) break;
      const int prev = a.par[tri_u(i, j, M)];
      j = i - 1;
      i = prev;
    }
    for (int x = 0, y = ng - 1; x < y; ++x, --y) {
      int t = gl[x];
      gl[x] = gl[y];
      gl[y] = t;
      t = gh[x];
      gh[x] = gh[y];
      gh[y] = t;
    }
    s_ng = ng;
  }
  __syncthreads();
  const int ng = s_ng;
  for (int x = tid; x < M; x += NT) {  // the group holding sorted user x: the last lo <= x
    int g0 = 0, g1 = ng - 1;
    while (g0 < g1) {
      const int mid = (g0 + g1 + 1) >> 1;
      if (gl[mid] <= x) g0 = mid; else g1 = mid - 1;
    }
    a.gid[x] = g0;
  }
  __syncthreads();
  // stitch: re-derive each chosen group's plan from its stored bound
  for (int x = tid; x < M; x += NT) {
    const int g = a.gid[x];
    const int lo = gl[g], hi = gh[g];
    const int bb = a.bstar[tri_u(lo, hi, M)];
    const bool pipe = bb < a.b0[nip + lo];
    double s[N];
    if (pipe) start_times<N>(a.lat, P.bmax, dls[lo], bb, s);
    else
#pragma unroll
      for (int n = 0; n < N; ++n) s[n] = 0.0;
    const double* r = a.rec + (size_t)x * R::SIZE;
    int sp;
    double f;
    choose<N>(r, P, s, pipe, sp, f);
    a.spos[x] = sp;
    a.fpos[x] = f;
    const int m = a.order[x];
    if (a.og.group_of_user) a.og.group_of_user[base + m] = g;
    if (a.og.split) a.og.split[base + m] = (uint8_t)sp;
    if (a.og.freq) a.og.freq[base + m] = f;
    if (a.og.user_energy) a.og.user_energy[base + m] = fold<N>(r, sp, f, 0.0);
  }
  __syncthreads();
  // group energies and batch sizes: one warp per group, 32 members at a
  // time; each lane computes its member's terms (fold<N>'s products), and
  // every lane runs the group's left fold over them in member order through
  // shuffles (the adds are the only serial part)
  for (int g = warp; g < ng; g += NW) {
    const int lo = gl[g], hi = gh[g];
    double total = 0.0;
    int cnt[N];
#pragma unroll
    for (int n = 0; n < N; ++n) cnt[n] = 0;
    for (int x0 = lo; x0 <= hi; x0 += 32) {
      const int x = x0 + lane;
      const bool live = x <= hi;
      double t[N + 1];
      int sp = N;
      if (live) {
        const double* r = a.rec + (size_t)x * R::SIZE;
        sp = a.spos[x];
        const double f = a.fpos[x];
#pragma unroll
        for (int n = 1; n <= N; ++n) t[n - 1] = __dmul_rn(__dmul_rn(r[R::KA(n)], f), f);
        t[N] = sp < N ? (sp == 0 ? r[R::E0] : r[R::U(sp)]) : 0.0;
      } else {
#pragma unroll
        for (int n = 0; n <= N; ++n) t[n] = 0.0;
      }
      const int nu = min(32, hi - x0 + 1);
      auto member = [&](int u) {  // member x0 + u's terms onto the running total
        const int su = __shfl_sync(kFull, sp, u);
#pragma unroll
        for (int n = 1; n <= N; ++n) {
          const double tv = __shfl_sync(kFull, t[n - 1], u);
          if (n <= su) total = __dadd_rn(total, tv);
        }
        const double up = __shfl_sync(kFull, t[N], u);
        if (su < N) total = __dadd_rn(total, up);
      };
      if (nu == 32) {  // unrolled: the shuffles run ahead of the serial adds
#pragma unroll
        for (int u = 0; u < 32; ++u) member(u);
      } else {
        for (int u = 0; u < nu; ++u) member(u);
      }
#pragma unroll
      for (int n = 1; n <= N; ++n) cnt[n - 1] += __popc(__ballot_sync(kFull, live && sp < n));
    }
    if (lane == 0) {
      a.genergy[g] = total;
      const size_t gi = base + g;
      if (a.og.group_lo) a.og.group_lo[gi] = lo;
      if (a.og.group_size) a.og.group_size[gi] = hi - lo + 1;
      if (a.og.group_b) a.og.group_b[gi] = a.bstar[tri_u(lo, hi, M)];
      if (a.og.group_deadline) a.og.group_deadline[gi] = dls[lo];
      if (a.og.group_energy) a.og.group_energy[gi] = total;
      if (a.og.group_batch_size)
#pragma unroll
        for (int n = 1; n <= N; ++n) a.og.group_batch_size[gi * N + n - 1] = cnt[n - 1];
    }
  }
  __syncthreads();
  if (tid == 0) {
    double e = 0.0;  // plan.energy: left fold of group energies (:385-386)
    for (int g = 0; g < ng; ++g) e = __dadd_rn(e, a.genergy[g]);
    if (a.og.status) a.og.status[a.k] = COINFER_ST_OK;
    if (a.og.fallback) a.og.fallback[a.k] = 0;
    if (a.og.energy) a.og.energy[a.k] = e;
    if (a.og.n_groups) a.og.n_groups[a.k] = ng;
  }
}

size_t large_ws_bytes(int M, int N) {
  const size_t T = (size_t)M * (M + 1) / 2;
  const size_t rec = (size_t)M * rec_size(N) * 8;
  // G, St (fp64) + bstar, par, pfit, argpm (u16) + records + dls/sumlat/fpos/genergy/slast + 6 int arrays
  // (every take() rounds up to 256 bytes: 32 * 256 covers all of them)
  return 16 * T + 8 * T + rec + 8 * ((size_t)M + 2) * 5 + 4 * ((size_t)M + 2) * 6 + 32 * 256;
}

// Feasible-prev prefix length of every DP cell (i >= 1): the number of prevs
// in [0, i) with groups_fit(dl[prev], dl[i], j-i+1) (offline_solvers.hpp:229-232).
__global__ void large_pfit(LargeArgs a) {  // one warp per row i >= 1, its useful cells only
  const int M = a.M, lane = threadIdx.x & 31;
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  for (int i = 1 + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < M; i += nw) {
    const int jend = i + a.rlen[i];  // past it no prev fits (pfit 0); no DP reads those cells
    const double di = a.dls[i];
    const long long xr = tri_u(i, i, M) - i;
    for (int j = i + lane; j < jend; j += 32) {
      const double thr = a.sumlat[j - i + 1];
      int l2 = 0, h2 = i;  // useful: dls[0] + thr <= di, so prev 0 fits
      while (l2 < h2) {
        const int mid = (l2 + h2) >> 1;
        if (__dadd_rn(a.dls[mid], thr) <= di) l2 = mid + 1; else h2 = mid;
      }
      a.pfit[xr + j] = (uint16_t)l2;
    }
  }
}

__global__ void large_init(LargeArgs a) {
  // Scenario::check tests the table length before any user (core_model.hpp:86-87)
  *a.status = a.P.bmax < a.M ? COINFER_ST_SHORT_TABLE : INT_MAX;
  const bool given = a.has_l_ip || a.l_ip_dev;
  *a.simple = fast_div_profile(a.P) && (!a.do_ip || !given || fast_div_deadline(ip_deadline(a, 0.0))) ? 1 : 0;
}

template <int N>
static cudaError_t launch_large_n(LargeArgs a, cudaStream_t st) {
  const int M = a.M, Q = (a.do_ip ? 1 : 0) + (a.do_og ? M : 0);
  large_init<<<1, 1, 0, st>>>(a);
  large_prep<N><<<(M + 8) / 8, 256, 0, st>>>(a);  // warps for m = 0..M
  large_rows<N><<<(Q + 255) / 256, 256, 0, st>>>(a);
  large_grow<N><<<(Q + 3) / 4, 128, 0, st>>>(a);
  if (a.do_og) large_pfit<<<(M + 7) / 8 < 148 * 8 ? (M + 7) / 8 : 148 * 8, 256, 0, st>>>(a);
  const int smem_fast = DpSmem(M).bytes;  // large_dp
  // large_finish: running PM, staged column | ring (128 x 16 points + owners) | counts, staged rows, rlen, last rows
  const int smem = 8 * 2 * M + 128 * 16 * 10 + 128 * 4 + 2 * 4 * M;
  if (M > 8 * 1024 || smem > 227 * 1024) return cudaErrorInvalidValue;  // <= 8 DP cells per thread
  cudaError_t e;
  if (a.do_og && smem_fast <= kDpSmemMax) {
    e = ensure_smem((const void*)large_dp, smem_fast);
    if (e != cudaSuccess) return e;
    large_dp<<<1, 256, smem_fast, st>>>(a);
  }
  e = ensure_smem((const void*)large_finish<N>, smem);
  if (e != cudaSuccess) return e;
  large_finish<N><<<1, 1024, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_large(const LargeArgs& a, cudaStream_t st) {
#define CFB_CALL(n) return launch_large_n<n>(a, st)
  CFB_DISPATCH_N(a.P.N, CFB_CALL)
#undef CFB_CALL
}

}  // namespace cfb
