// oracles.cu — the reference's brute-force oracles on the device (SURVEY.md
// §8f row 4), so the Theorem 1/2 checks (tests/test_oracles.cpp) run on far
// more instances than a CPU can enumerate.
//
// Reference (all under /root/reference/proj/include/coinfer/oracles.hpp):
//   oracle_structured           :28-93    every split vector in {0..N}^M
//                                          against the start times for bound b
//   oracle_grouping_contiguous  :165-225  every cut pattern of the sorted order
//   oracle_grouping             :131-163  every set partition (restricted
//                                          growth strings), groups served at
//                                          their earliest member deadline
//   detail::grouping_cost       :106-127
//
// One CTA per instance.  Enumerations are split across the threads by index;
// each thread keeps a lexicographic (energy, index) minimum, so the CTA
// reduction returns the reference's choice (strict '<' in enumeration order
// = the smallest index among the minima).  Grouping costs are re-derived
// with the plain per-group batch-bound search (choose() + fold(), the
// O(M^4 N) direct form), not the engine's chain sweeps.

#include <climits>

#include "kernels.h"

namespace cfb {
namespace {

constexpr int kOT = 256;  // threads per instance


__device__ __forceinline__ bool lex_less(double e, long long i, double be, long long bi) {
  return e < be || (e == be && i < bi);
}

// Block-wide lexicographic (energy, index) minimum.
__device__ void block_lexmin(double& e, long long& i) {
  __shared__ double se[kOT / 32];
  __shared__ long long si[kOT / 32];
  for (int o = 16; o; o >>= 1) {
    const double oe = __shfl_xor_sync(kFull, e, o);
    const long long oi = __shfl_xor_sync(kFull, i, o);
    if (lex_less(oe, oi, e, i)) {
      e = oe;
      i = oi;
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    se[w] = e;
    si[w] = i;
  }
  __syncthreads();
  e = se[0];
  i = si[0];
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
    if (lex_less(se[k], si[k], e, i)) {
      e = se[k];
      i = si[k];
    }
}

// ---------------------------------------------------------- structured
template <int N>
__global__ void __launch_bounds__(kOT) structured_kernel(OracleArgs a) {
  __shared__ double cost[16][COINFER_MAX_SUBTASKS + 1];
  __shared__ unsigned char ok[16][COINFER_MAX_SUBTASKS + 1];
  const ProfileConst& P = a.P;
  const int M = a.M, tid = threadIdx.x;
  for (int64_t k = blockIdx.x; k < a.n_inst; k += gridDim.x) {
    const size_t base = (size_t)k * M;
    const double l = a.deadline[k];
    const int b = a.b[k];
    // start times first (edge_batch_latency: b past the table throws,
    // b == 0 is F = 0), then the enumeration guard (oracles.hpp:34-40,82-84)
    if (b > P.bmax || b < 0) {
      if (tid == 0) a.status[k] = COINFER_ST_BOUND_PAST_TABLE;
      continue;
    }
    double combos = 1.0;
    for (int m = 0; m < M; ++m) combos *= double(N + 1);
    if (combos > 2e6 || M > 16) {
      if (tid == 0) a.status[k] = COINFER_ST_TOO_LARGE;
      continue;
    }
    double s[N];
    if (b >= 1) {
      start_times<N>(a.lat, P.bmax, l, b, s);
    } else {
#pragma unroll
      for (int n = 0; n < N; ++n) s[n] = l;
    }
    const bool fb = s[0] < 0.0;
    // split_cost (oracles.hpp:44-69), straight from the model
    for (int x = tid; x < M * (N + 1); x += blockDim.x) {
      const int m = x / (N + 1), n = x % (N + 1);
      const size_t i = base + m;
      const double arr = a.arr[i], fmx = a.fmax[i], fmn = a.fmin[i], kap = a.kappa[i];
      double c = 0.0;
      bool good = false;
      if (n == N) {
        const double window = __dsub_rn(a.dl[i], arr);
        if (window > 0.0) {
          double f = __ddiv_rn(P.prefix[N], window);
          if (!(f > __dmul_rn(fmx, 1.0 + 1e-12))) {
            f = smin(smax(f, fmn), fmx);
            c = __dmul_rn(__dmul_rn(__dmul_rn(kap, P.prefix[N]), f), f);
            good = true;
          }
        }
      } else if (!fb) {
        if (n == 0) {
          const double lat0 = __ddiv_rn(P.bits[0], a.ru[i]);
          if (!(__dadd_rn(arr, lat0) > s[0])) {
            c = __dmul_rn(lat0, a.pu[i]);
            good = true;
          }
        } else {
          double prefix = 0.0;
          for (int q = 0; q < n; ++q) prefix = __dadd_rn(prefix, P.work[q]);
          const double up = __ddiv_rn(P.bits[n], a.ru[i]);
          const double window = __dsub_rn(__dsub_rn(s[n], up), arr);
          if (window > 0.0) {
            double f = __ddiv_rn(prefix, window);
            if (!(f > fmx)) {
              f = smin(smax(f, fmn), fmx);
              c = __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(kap, prefix), f), f), __dmul_rn(up, a.pu[i]));
              good = true;
            }
          }
        }
      }
      cost[m][n] = c;
      ok[m][n] = good;
    }
    __syncthreads();
    const long long total = (long long)combos;
    double be = dinf();
    long long bi = LLONG_MAX;
    for (long long c = tid; c < total; c += blockDim.x) {
      long long r = c;
      double e = 0.0;
      bool good = true;
      for (int m = 0; m < M; ++m) {  // pick[0] varies fastest (oracles.hpp:87-90)
        const int n = (int)(r % (N + 1));
        r /= (N + 1);
        good = good && ok[m][n];
        e = __dadd_rn(e, cost[m][n]);
      }
      if (good && lex_less(e, c, be, bi)) {
        be = e;
        bi = c;
      }
    }
    block_lexmin(be, bi);
    if (tid == 0) {
      a.status[k] = COINFER_ST_OK;
      a.fallback[k] = fb;
      a.feasible[k] = bi != LLONG_MAX;
      a.energy[k] = bi != LLONG_MAX ? be : dinf();
      long long r = bi != LLONG_MAX ? bi : 0;
      for (int m = 0; m < M; ++m) {
        a.split[base + m] = bi != LLONG_MAX ? (uint8_t)(r % (N + 1)) : 0;
        r /= (N + 1);
      }
    }
    __syncthreads();
  }
}

// The batch-bound search on one group of users (try_ip_ssa of the
// subscenario, offline_solvers.hpp:192-204 with :137-188), members in the
// given order, common deadline l.  +inf when no bound admits everyone.
template <int N>
__device__ double group_ipssa(const double* rec, const int* mem, int size, const ProfileConst& P,
                              const double* lat, double l) {
  using R = Rec<N>;
  double best = dinf();
  for (int b = size; b >= 1; --b) {
    double s[N];
    const bool pipe = start_times<N>(lat, P.bmax, l, b, s);
    double e = 0.0;
    int off = 0;
    bool good = true;
    for (int q = 0; q < size && good; ++q) {
      const double* r = rec + mem[q] * R::SIZE;
      int sp;
      double f;
      choose<N>(r, P, s, pipe, sp, f);
      if (sp < 0) {
        good = false;
        break;
      }
      e = fold<N>(r, sp, f, e);
      off += sp < N;
    }
    // realised max batch = offloaders (suffix splits), must stay <= b
    if (good && off <= b && e < best) best = e;
  }
  return best;
}

// ------------------------------------------------------------ grouping
// Restricted growth strings of length M (oracles.hpp:146-160), ranked in
// the recursion's order: cnt[m][u] = completions of positions m..M-1 when
// u labels are in use.
template <int N>
__global__ void __launch_bounds__(kOT) grouping_kernel(OracleArgs a) {
  using R = Rec<N>;
  __shared__ double rec[16 * R::SIZE];
  __shared__ double dls[16];
  __shared__ int order[16], rank_[16];
  __shared__ double G[16][16];
  __shared__ double sumlat[17];
  __shared__ long long tab[17][17];
  const ProfileConst& P = a.P;
  const int M = a.M, tid = threadIdx.x;
  for (int64_t k = blockIdx.x; k < a.n_inst; k += gridDim.x) {
    const size_t base = (size_t)k * M;
    if ((a.contiguous && M > 16) || (!a.contiguous && M > 9)) {
      if (tid == 0) a.status[k] = COINFER_ST_TOO_LARGE;
      continue;
    }
    if (M == 0) {
      if (tid == 0) {
        a.status[k] = COINFER_ST_OK;
        a.energy[k] = 0.0;
        a.feasible[k] = 1;
        a.n_groups[k] = 0;
      }
      continue;
    }
    // sort by (deadline, id), records in sorted order
    for (int m = tid; m < M; m += blockDim.x) {
      const double d = a.dl[base + m];
      int r = 0;
      for (int o = 0; o < M; ++o) {
        const double e = a.dl[base + o];
        r += (e < d) || (e == d && o < m);
      }
      rank_[m] = r;
      order[r] = m;
      dls[r] = d;
      const size_t i = base + m;
      build_rec<N>(rec + r * R::SIZE, P, a.fmin[i], a.fmax[i], a.kappa[i], a.ru[i], a.pu[i], a.arr[i], d);
    }
    for (int sz = tid + 1; sz <= M; sz += blockDim.x) {  // sum_latency
      double t = 0.0;
      for (int n = 1; n <= N; ++n) t = __dadd_rn(t, __ldg(a.lat + (size_t)(n - 1) * P.bmax + sz - 1));
      sumlat[sz] = t;
    }
    if (tid == 0) {  // RGS completion counts
      for (int u = 0; u <= M; ++u) tab[0][u] = 1;
      for (int rem = 1; rem <= M; ++rem)
        for (int u = 0; u <= M; ++u) tab[rem][u] = (long long)u * tab[rem - 1][u] + (u < M ? tab[rem - 1][u + 1] : 0);
    }
    __syncthreads();
    double be = dinf();
    long long bi = LLONG_MAX;
    if (a.contiguous) {
      // G[i][j]: the batch-bound search on sorted users i..j at dl[i]
      for (int x = tid; x < M * M; x += blockDim.x) {
        const int i = x / M, j = x % M;
        if (j < i) continue;
        int mem[16];
        for (int q = i; q <= j; ++q) mem[q - i] = q;
        G[i][j] = group_ipssa<N>(rec, mem, j - i + 1, P, a.lat, dls[i]);
      }
      __syncthreads();
      const long long total = 1LL << (M - 1);
      for (long long mask = tid; mask < total; mask += blockDim.x) {
        double e = 0.0;
        bool good = true;
        int lo = 0, plo = -1;
        for (int i = 0; i < M && good; ++i) {
          if (i + 1 == M || ((mask >> i) & 1)) {  // group lo..i
            if (plo >= 0) good = __dadd_rn(dls[plo], sumlat[i - lo + 1]) <= dls[lo];  // groups_fit
            const double g = G[lo][i];
            if (g == dinf()) good = false;
            e = __dadd_rn(e, g);
            plo = lo;
            lo = i + 1;
          }
        }
        if (good && lex_less(e, mask, be, bi)) {
          be = e;
          bi = mask;
        }
      }
    } else {
      const long long total = tab[M][0];
      for (long long rk = tid; rk < total; rk += blockDim.x) {
        int label[9];
        long long r = rk;
        int used = 0;
        for (int m = 0; m < M; ++m) {  // unrank: label of original user m
          int v = 0;
          for (; v <= used; ++v) {
            const long long c = tab[M - m - 1][used > v ? used : v + 1];
            if (r < c) break;
            r -= c;
          }
          label[m] = v;
          if (v == used) ++used;
        }
        // groups: members sorted by (deadline, id); groups ordered by their
        // first member (detail::grouping_cost, oracles.hpp:106-121)
        int first[9], size[9];
        for (int g = 0; g < used; ++g) {
          first[g] = 16;
          size[g] = 0;
        }
        for (int m = 0; m < M; ++m) {
          const int g = label[m], p = rank_[m];
          if (p < first[g]) first[g] = p;
          ++size[g];
        }
        int gord[9];  // groups by first sorted position
        for (int g = 0; g < used; ++g) gord[g] = g;
        for (int x = 1; x < used; ++x)
          for (int y = x; y > 0 && first[gord[y]] < first[gord[y - 1]]; --y) {
            const int t = gord[y];
            gord[y] = gord[y - 1];
            gord[y - 1] = t;
          }
        bool good = true;
        for (int x = 1; x < used && good; ++x)
          good = __dadd_rn(dls[first[gord[x - 1]]], sumlat[size[gord[x]]]) <= dls[first[gord[x]]];
        double e = 0.0;
        for (int x = 0; x < used && good; ++x) {
          const int g = gord[x];
          int mem[9], c = 0;
          for (int p = 0; p < M; ++p)
            if (label[order[p]] == g) mem[c++] = p;  // sorted positions = (deadline, id) order
          const double ge = group_ipssa<N>(rec, mem, c, P, a.lat, dls[first[g]]);
          if (ge == dinf()) good = false;
          e = __dadd_rn(e, ge);
        }
        if (good && lex_less(e, rk, be, bi)) {
          be = e;
          bi = rk;
        }
      }
    }
    block_lexmin(be, bi);
    if (tid == 0) {
      a.status[k] = COINFER_ST_OK;
      const bool feas = bi != LLONG_MAX;
      a.feasible[k] = feas;
      a.energy[k] = feas ? be : dinf();
      int ng = 0;
      if (feas && a.contiguous) {
        int g = 0;
        for (int i = 0; i < M; ++i) {
          a.group_of_user[base + order[i]] = g;
          if (i + 1 == M || ((bi >> i) & 1)) ++g;
        }
        ng = g;
      } else if (feas) {
        int label[9], used = 0;
        long long r = bi;
        for (int m = 0; m < M; ++m) {
          int v = 0;
          for (; v <= used; ++v) {
            const long long c = tab[M - m - 1][used > v ? used : v + 1];
            if (r < c) break;
            r -= c;
          }
          label[m] = v;
          if (v == used) ++used;
        }
        int first[9];
        for (int g = 0; g < used; ++g) first[g] = 16;
        for (int m = 0; m < M; ++m)
          if (rank_[m] < first[label[m]]) first[label[m]] = rank_[m];
        for (int m = 0; m < M; ++m) {  // group index in rising-deadline order
          int pos = 0;
          for (int g = 0; g < used; ++g) pos += first[g] < first[label[m]];
          a.group_of_user[base + m] = pos;
        }
        ng = used;
      }
      a.n_groups[k] = ng;
    }
    __syncthreads();
  }
}

}  // namespace

template <int N>
static cudaError_t launch_structured_n(const OracleArgs& a, int grid, cudaStream_t st) {
  structured_kernel<N><<<grid, kOT, 0, st>>>(a);
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_grouping_n(const OracleArgs& a, int grid, cudaStream_t st) {
  grouping_kernel<N><<<grid, kOT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_oracle_structured(const OracleArgs& a, cudaStream_t st) {
  const int grid = (int)(a.n_inst < 148 * 8 ? (a.n_inst > 0 ? a.n_inst : 1) : 148 * 8);
#define CFB_CALL(n) return launch_structured_n<n>(a, grid, st)
  CFB_DISPATCH_N(a.P.N, CFB_CALL)
#undef CFB_CALL
}

cudaError_t launch_oracle_grouping(const OracleArgs& a, cudaStream_t st) {
  const int grid = (int)(a.n_inst < 148 * 8 ? (a.n_inst > 0 ? a.n_inst : 1) : 148 * 8);
#define CFB_CALL(n) return launch_grouping_n<n>(a, grid, st)
  CFB_DISPATCH_N(a.P.N, CFB_CALL)
#undef CFB_CALL
}

}  // namespace cfb
