// baselines.cu — the step right after the solve:
// Schedule materialisation on the device, and the offline comparison
// baselines LC / PS / FIFO / IPSSA_NP.
//
// Reference (all under /root/reference/proj/include/coinfer):
//   try_fixed_batch schedule build        offline_solvers.hpp:155-185
//   og stitch + batch-id offset           offline_solvers.hpp:357-386
//   normalize                             schedule.hpp:93-113
//   detail::lc_solve                      offline_solvers.hpp:255-276
//   detail::ps_solve                      offline_solvers.hpp:404-487
//   detail::fifo_solve                    offline_solvers.hpp:489-555
//   detail::ipssa_np_solve (expansion)    offline_solvers.hpp:560-600
//   best_partition / local_only_choice    offline_solvers.hpp:62-117
//   total_energy / schedule_metrics fold  schedule.hpp:214-231, offline_solvers.hpp:627-646
//
// These are sequential per instance in the reference (serialised edge
// reservations, a demotion fixpoint), so the mapping is one thread per
// instance, grid-stride over the batch, per-thread scratch in global memory.
// They are not the throughput path (the fused IP-SSA/OG kernel is); the bar
// here is bit-exact agreement with the reference, so every operation keeps
// the reference's order with explicit round-to-nearest intrinsics.

#include <cmath>

#include "kernels.h"

namespace cfb {
namespace {

__device__ __forceinline__ double dnan() { return __longlong_as_double(0x7ff8000000000000LL); }

// edge_batch_latency (core_model.hpp:128-136): F_n(0) = 0.
__device__ __forceinline__ double F(const AuxArgs& a, int n, int b) {
  return b == 0 ? 0.0 : a.lat[(size_t)(n - 1) * a.P.bmax + (b - 1)];
}

// PartitionChoice (offline_solvers.hpp:51-56)
struct PC {
  int split;
  double freq, energy;
  bool feasible;
};

struct User {
  double fmin, fmax, kappa, ru, pu, arr, dl;
};

__device__ __forceinline__ User load_user(const AuxArgs& a, size_t i) {
  return {a.fmin[i], a.fmax[i], a.kappa[i], a.ru[i], a.pu[i], a.arr[i], a.dl[i]};
}

// detail::local_only_choice (offline_solvers.hpp:62-75)
__device__ PC local_choice(const ProfileConst& P, const User& u, double deadline) {
  PC c{P.N, dnan(), dinf(), false};
  double f, E;
  if (local_only(deadline, u.arr, u.fmin, u.fmax, u.kappa, P.prefix[P.N], f, E)) {
    c.freq = f;
    c.energy = E;
    c.feasible = true;
  }
  return c;
}

// best_partition (offline_solvers.hpp:83-117), runtime N.
__device__ PC best_partition(const ProfileConst& P, const User& u, const double* s, double deadline) {
  const int N = P.N;
  PC best{0, dnan(), dinf(), false};
  const double lat0 = __ddiv_rn(P.bits[0], u.ru);
  if (__dadd_rn(u.arr, lat0) <= s[0]) {
    best.split = 0;
    best.energy = __dmul_rn(lat0, u.pu);
    best.feasible = true;
  }
  for (int n = 1; n <= N; ++n) {
    PC c{0, dnan(), dinf(), false};
    if (n == N) {
      c = local_choice(P, u, deadline);
    } else {
      const double upload = __ddiv_rn(P.bits[n], u.ru);
      const double budget = __dsub_rn(__dsub_rn(s[n], upload), u.arr);
      if (budget <= 0.0) continue;
      const double f_req = __ddiv_rn(P.prefix[n], budget);
      if (f_req > u.fmax) continue;
      c.split = n;
      c.freq = smin(smax(f_req, u.fmin), u.fmax);
      c.energy = __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(u.kappa, P.prefix[n]), c.freq), c.freq),
                           __dmul_rn(upload, u.pu));
      c.feasible = true;
    }
    if (c.feasible && c.energy <= best.energy) best = c;
  }
  return best;
}

// One user's total_energy terms (schedule.hpp:214-231) for a suffix
// schedule: local sub-tasks 1..split at f, then the single upload of
// B_split (downloads never fire when the edge part is a suffix).
__device__ __forceinline__ double user_terms(const ProfileConst& P, const User& u, int split, double f,
                                             double acc) {
  for (int n = 1; n <= split; ++n)
    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(u.kappa, P.work[n - 1]), f), f));
  if (split < P.N) acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn(P.bits[split], u.ru), u.pu));
  return acc;
}

// Scenario::check (core_model.hpp:80-101) for instance k: the table length
// first, then users in order, first failing test.
__device__ int check_instance(const AuxArgs& a, size_t base) {
  if (a.P.bmax < a.M) return COINFER_ST_SHORT_TABLE;
  for (int m = 0; m < a.M; ++m) {
    const size_t i = base + m;
    const int c = check_user(a.fmin[i], a.fmax[i], a.kappa[i], a.ru[i], a.rd ? a.rd[i] : 1.0, a.pu[i],
                             a.pd ? a.pd[i] : 0.0, a.arr[i], a.dl[i]);
    if (c != COINFER_ST_OK) return c;
  }
  return COINFER_ST_OK;
}

// In-place heap sort of idx[0..n) under a strict weak order.
template <class Less>
__device__ void heap_sort(int* idx, int n, Less less) {
  auto sift = [&](int root, int end) {
    while (2 * root + 1 < end) {
      int child = 2 * root + 1;
      if (child + 1 < end && less(idx[child], idx[child + 1])) ++child;
      if (!less(idx[root], idx[child])) return;
      const int t = idx[root];
      idx[root] = idx[child];
      idx[child] = t;
      root = child;
    }
  };
  for (int s = n / 2 - 1; s >= 0; --s) sift(s, n);
  for (int end = n - 1; end > 0; --end) {
    const int t = idx[0];
    idx[0] = idx[end];
    idx[end] = t;
    sift(0, end);
  }
}

// Per-instance views of the schedule output.
struct Sched {
  int* x;
  double* bstart;
  double* comp;
  double* freq;
  int* nb;
};

__device__ __forceinline__ Sched sched_of(const AuxArgs& a, int64_t k) {
  const int M = a.M, N = a.P.N;
  return {a.sch.x + (size_t)k * M * N, a.sch.batch_start + (size_t)k * M * N,
          a.sch.completion + (size_t)k * M * (N + 1), a.sch.freq + (size_t)k * M, a.sch.n_batches + k};
}

// normalize (schedule.hpp:93-113): batches renumbered by (start, sub-task).
// Every path here creates batches with strictly increasing start times
// (serialised reservations, back-to-back pipelines, groups_fit spacing), so
// the order is almost always already normal and the sort is one pass.
// bsub[i]: sub-task of batch i+1.  perm/tmp: scratch of nb entries.
__device__ void normalize(const Sched& S, int M, int N, int nb, int* bsub, int* perm, double* tmp) {
  for (int i = 0; i < nb; ++i) perm[i] = i;
  bool moved = false;
  for (int i = 1; i < nb; ++i) {  // insertion sort of batch indices
    const int v = perm[i];
    int j = i;
    while (j > 0) {
      const int u = perm[j - 1];
      const bool gt = S.bstart[u] != S.bstart[v] ? S.bstart[v] < S.bstart[u] : bsub[v] < bsub[u];
      if (!gt) break;
      perm[j] = u;
      --j;
      moved = true;
    }
    perm[j] = v;
  }
  if (!moved) return;
  for (int i = 0; i < nb; ++i) tmp[i] = S.bstart[perm[i]];
  int* newid = bsub;  // reuse: bsub no longer needed
  for (int i = 0; i < nb; ++i) newid[perm[i]] = i + 1;
  for (int i = 0; i < nb; ++i) S.bstart[i] = tmp[i];
  for (int q = 0; q < M * N; ++q)
    if (S.x[q] != 0) S.x[q] = newid[S.x[q] - 1];
}

// Completion times of user m's local prefix: t_0 = arrival,
// t_n = t_{n-1} + A_n / f (try_fixed_batch:173-175).
__device__ __forceinline__ void local_chain(const ProfileConst& P, double* t, double arr, int split,
                                            double f) {
  t[0] = arr;
  for (int n = 1; n <= split; ++n) t[n] = __dadd_rn(t[n - 1], __ddiv_rn(P.work[n - 1], f));
}

struct Scratch {
  unsigned char* p;
  __device__ explicit Scratch(const AuxArgs& a)
      : p(a.scratch + (size_t)(blockIdx.x * blockDim.x + threadIdx.x) * a.scratch_per_thread) {}
  template <class T>
  __device__ T* take(size_t n) {
    T* r = reinterpret_cast<T*>(p);
    p += (n * sizeof(T) + 15) & ~size_t(15);
    return r;
  }
};

__device__ void zero_result(const AuxArgs& a, int64_t k, int status) {
  const int M = a.M, N = a.P.N;
  if (a.ip.status) a.ip.status[k] = status;
  if (a.ip.batch_bound) a.ip.batch_bound[k] = 0;
  if (a.ip.pipeline_feasible) a.ip.pipeline_feasible[k] = 1;
  if (a.ip.energy) a.ip.energy[k] = 0.0;
  for (int n = 0; n < N; ++n)
    if (a.ip.batch_size) a.ip.batch_size[(size_t)k * N + n] = 0;
  for (int m = 0; m < M; ++m) {
    if (a.ip.split) a.ip.split[(size_t)k * M + m] = 0;
    if (a.ip.freq) a.ip.freq[(size_t)k * M + m] = 0.0;
    if (a.ip.user_energy) a.ip.user_energy[(size_t)k * M + m] = 0.0;
  }
  if (a.sch.n_batches) a.sch.n_batches[k] = 0;
}

// ------------------------------------------------------------------ kernels

// Schedule of an IP-SSA / fixed-bound solve (try_fixed_batch:155-185):
// batches at s*_n for every sub-task with a nonzero realised size, in n
// order (already normal: s*_n is strictly increasing).
__global__ void materialize_ip_kernel(AuxArgs a) {
  const ProfileConst& P = a.P;
  const int M = a.M, N = P.N;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.n_inst;
       k += (int64_t)gridDim.x * blockDim.x) {
    const Sched S = sched_of(a, k);
    const size_t base = (size_t)k * M;
    if (a.ip.status[k] != COINFER_ST_OK) {
      *S.nb = 0;
      continue;
    }
    double l;
    if (a.l_ip) {
      l = a.l_ip[k];
    } else {
      l = dinf();
      for (int m = 0; m < M; ++m) l = smin(l, a.dl[base + m]);
    }
    const int b = a.ip.batch_bound[k];
    const int* bs = a.ip.batch_size + (size_t)k * N;
    double s[COINFER_MAX_SUBTASKS];
    if (a.ip.pipeline_feasible[k] && b >= 1) {
      double t = l;
      for (int n = N; n >= 1; --n) {
        t = __dsub_rn(t, F(a, n, b));
        s[n - 1] = t;
      }
    }
    int id[COINFER_MAX_SUBTASKS];
    int nb = 0;
    for (int n = 1; n <= N; ++n) {
      id[n - 1] = 0;
      if (bs[n - 1] > 0) {
        S.bstart[nb] = s[n - 1];
        id[n - 1] = ++nb;
      }
    }
    *S.nb = nb;
    for (int m = 0; m < M; ++m) {
      const int sp = a.ip.split[base + m];
      const double f = a.ip.freq[base + m];
      double* t = S.comp + (size_t)m * (N + 1);
      int* x = S.x + (size_t)m * N;
      local_chain(P, t, a.arr[base + m], sp, f);
      for (int n = 1; n <= N; ++n) {
        if (n <= sp) {
          x[n - 1] = 0;
        } else {
          x[n - 1] = id[n - 1];
          t[n] = __dadd_rn(s[n - 1], F(a, n, bs[n - 1]));
        }
      }
      S.freq[m] = f;
    }
  }
}

// Schedule of an OG plan (og:357-386): each group's batches at its own s*_n
// (deadline dl[lo], bound b), ids offset by the batches before it, then
// normalize.  Fallback plans are the all-local lc_solve schedule.
__global__ void materialize_og_kernel(AuxArgs a) {
  const ProfileConst& P = a.P;
  const int M = a.M, N = P.N;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.n_inst;
       k += (int64_t)gridDim.x * blockDim.x) {
    const Sched S = sched_of(a, k);
    const size_t base = (size_t)k * M;
    if (a.og.status[k] != COINFER_ST_OK) {
      *S.nb = 0;
      continue;
    }
    Scratch sc(a);
    int* bsub = sc.take<int>((size_t)M * N);
    int* perm = sc.take<int>((size_t)M * N);
    double* tmp = sc.take<double>((size_t)M * N);
    int nb = 0;
    const bool fb = a.og.fallback[k] != 0;
    const int G = fb ? 0 : a.og.n_groups[k];
    for (int g = 0; g < G; ++g) {
      const size_t gi = base + g;
      const int lo = a.og.group_lo[gi], sz = a.og.group_size[gi], b = a.og.group_b[gi];
      const int* bs = a.og.group_batch_size + gi * N;
      double s[COINFER_MAX_SUBTASKS];
      bool any = false;
      for (int n = 0; n < N; ++n) any = any || bs[n] > 0;
      if (any) {
        double t = a.og.group_deadline[gi];
        for (int n = N; n >= 1; --n) {
          t = __dsub_rn(t, F(a, n, b));
          s[n - 1] = t;
        }
      }
      int id[COINFER_MAX_SUBTASKS];
      for (int n = 1; n <= N; ++n) {
        id[n - 1] = 0;
        if (bs[n - 1] > 0) {
          S.bstart[nb] = s[n - 1];
          bsub[nb] = n;
          id[n - 1] = ++nb;
        }
      }
      for (int q = lo; q < lo + sz; ++q) {
        const int m = a.og.order[base + q];
        const int sp = a.og.split[base + m];
        const double f = a.og.freq[base + m];
        double* t = S.comp + (size_t)m * (N + 1);
        int* x = S.x + (size_t)m * N;
        local_chain(P, t, a.arr[base + m], sp, f);
        for (int n = 1; n <= N; ++n) {
          if (n <= sp) {
            x[n - 1] = 0;
          } else {
            x[n - 1] = id[n - 1];
            t[n] = __dadd_rn(s[n - 1], F(a, n, bs[n - 1]));
          }
        }
        S.freq[m] = f;
      }
    }
    if (fb) {
      for (int m = 0; m < M; ++m) {
        const double f = a.og.freq[base + m];
        local_chain(P, S.comp + (size_t)m * (N + 1), a.arr[base + m], N, f);
        for (int n = 0; n < N; ++n) S.x[(size_t)m * N + n] = 0;
        S.freq[m] = f;
      }
    }
    normalize(S, M, N, nb, bsub, perm, tmp);
    *S.nb = nb;
  }
}

// Writes the per-user outputs (split, freq, per-user energy) and the
// total_energy fold in user order for a suffix schedule.
__device__ void finish_result(const AuxArgs& a, int64_t k, const int* split, const double* freq) {
  const ProfileConst& P = a.P;
  const int M = a.M;
  const size_t base = (size_t)k * M;
  double total = 0.0;
  for (int m = 0; m < M; ++m) {
    const User u = load_user(a, base + m);
    total = user_terms(P, u, split[m], freq[m], total);
    if (a.ip.user_energy) a.ip.user_energy[base + m] = user_terms(P, u, split[m], freq[m], 0.0);
    if (a.ip.split) a.ip.split[base + m] = (uint8_t)split[m];
    if (a.ip.freq) a.ip.freq[base + m] = freq[m];
  }
  if (a.ip.energy) a.ip.energy[k] = total;
  if (a.ip.status) a.ip.status[k] = COINFER_ST_OK;
}

__device__ void baseline_lc(const AuxArgs& a, int64_t k, Scratch& sc) {
  const ProfileConst& P = a.P;
  const int M = a.M, N = P.N;
  const size_t base = (size_t)k * M;
  int* split = sc.take<int>(M);
  double* freq = sc.take<double>(M);
  for (int m = 0; m < M; ++m) {
    const User u = load_user(a, base + m);
    const PC c = local_choice(P, u, u.dl);
    if (!c.feasible) return zero_result(a, k, COINFER_ST_INFEASIBLE);
    split[m] = N;
    freq[m] = c.freq;
  }
  if (a.sch.x) {
    const Sched S = sched_of(a, k);
    for (int m = 0; m < M; ++m) {
      local_chain(P, S.comp + (size_t)m * (N + 1), a.arr[base + m], N, freq[m]);
      for (int n = 0; n < N; ++n) S.x[(size_t)m * N + n] = 0;
      S.freq[m] = freq[m];
    }
    *S.nb = 0;
  }
  for (int n = 0; n < N; ++n)
    if (a.ip.batch_size) a.ip.batch_size[(size_t)k * N + n] = 0;
  if (a.ip.batch_bound) a.ip.batch_bound[k] = 0;
  if (a.ip.pipeline_feasible) a.ip.pipeline_feasible[k] = 1;
  finish_result(a, k, split, freq);
}

// detail::ps_solve: private timelines at M x the unit latency, then the
// edge serialises the reserved unit batches by (nominal start, sub-task,
// user); users pushed past their deadline are demoted to local and the
// placement reruns until nobody moves.
__device__ void baseline_ps(const AuxArgs& a, int64_t k, Scratch& sc) {
  const ProfileConst& P = a.P;
  const int M = a.M, N = P.N;
  const size_t base = (size_t)k * M;
  double* nominal = sc.take<double>((size_t)M * N);
  int* jobs = sc.take<int>((size_t)M * N);
  double* jstart = sc.take<double>((size_t)M * N);
  double* job_end = sc.take<double>(M);
  int* split = sc.take<int>(M);
  double* cfreq = sc.take<double>(M);
  int* bsub = sc.take<int>((size_t)M * N);
  int* perm = sc.take<int>((size_t)M * N);
  double* tmp = sc.take<double>((size_t)M * N);
  for (int m = 0; m < M; ++m) {
    const User u = load_user(a, base + m);
    double* s = nominal + (size_t)m * N;
    double t = u.dl;
    for (int n = N; n >= 1; --n) {
      t = __dsub_rn(t, __dmul_rn((double)M, F(a, n, 1)));
      s[n - 1] = t;
    }
    const PC c = s[0] < 0.0 ? local_choice(P, u, u.dl) : best_partition(P, u, s, u.dl);
    if (!c.feasible) return zero_result(a, k, COINFER_ST_INFEASIBLE);
    split[m] = c.split;
    cfreq[m] = c.freq;
    job_end[m] = 0.0;
  }
  int nj;
  while (true) {
    nj = 0;
    for (int m = 0; m < M; ++m)
      for (int n = split[m] + 1; n <= N; ++n) jobs[nj++] = m * N + (n - 1);
    // std::tie(nominal, subtask, user) <
    heap_sort(jobs, nj, [&](int p, int q) {
      if (nominal[p] != nominal[q]) return nominal[p] < nominal[q];
      const int np = p % N, nq = q % N;
      if (np != nq) return np < nq;
      return p / N < q / N;
    });
    double cursor = 0.0;
    for (int i = 0; i < nj; ++i) {
      const int j = jobs[i], m = j / N, n = j % N + 1;
      const double st = smax(nominal[j], cursor);
      jstart[i] = st;
      cursor = __dadd_rn(st, F(a, n, 1));
      job_end[m] = cursor;
    }
    bool demoted = false;
    for (int m = 0; m < M; ++m) {
      if (split[m] < N && job_end[m] > __dadd_rn(a.dl[base + m], 1e-12)) {
        const User u = load_user(a, base + m);
        const PC c = local_choice(P, u, u.dl);
        if (!c.feasible) return zero_result(a, k, COINFER_ST_INFEASIBLE);
        split[m] = c.split;
        cfreq[m] = c.freq;
        demoted = true;
      }
    }
    if (!demoted) break;
  }
  if (a.ip.batch_size)
    for (int n = 0; n < N; ++n) a.ip.batch_size[(size_t)k * N + n] = 0;
  double* freq = cfreq;
  for (int m = 0; m < M; ++m)
    if (split[m] == 0) freq[m] = a.fmax[base + m];
  if (a.sch.x) {
    const Sched S = sched_of(a, k);
    for (int m = 0; m < M; ++m) {
      local_chain(P, S.comp + (size_t)m * (N + 1), a.arr[base + m], split[m], freq[m]);
      for (int n = 1; n <= split[m]; ++n) S.x[(size_t)m * N + n - 1] = 0;
      S.freq[m] = freq[m];
    }
    for (int i = 0; i < nj; ++i) {
      const int j = jobs[i], m = j / N, n = j % N + 1;
      S.bstart[i] = jstart[i];
      bsub[i] = n;
      S.x[(size_t)m * N + n - 1] = i + 1;
      S.comp[(size_t)m * (N + 1) + n] = __dadd_rn(jstart[i], F(a, n, 1));
    }
    normalize(S, M, N, nj, bsub, perm, tmp);
    *S.nb = nj;
  }
  for (int i = 0; i < nj; ++i)
    if (a.ip.batch_size) a.ip.batch_size[(size_t)k * N + jobs[i] % N] += 1;
  if (a.ip.batch_bound) a.ip.batch_bound[k] = 0;
  if (a.ip.pipeline_feasible) a.ip.pipeline_feasible[k] = 1;
  finish_result(a, k, split, freq);
}

// detail::fifo_solve: users by (rate_up desc, id); each takes its cheapest
// split that fits behind the edge cursor with everything local at f_max,
// and reserves unit batches back to back.
__device__ void baseline_fifo(const AuxArgs& a, int64_t k, Scratch& sc) {
  const ProfileConst& P = a.P;
  const int M = a.M, N = P.N;
  const size_t base = (size_t)k * M;
  int* order = sc.take<int>(M);
  int* split = sc.take<int>(M);
  double* freq = sc.take<double>(M);
  double* ready_t = sc.take<double>(M);  // best_start per user
  int* bsub = sc.take<int>((size_t)M * N);
  int* perm = sc.take<int>((size_t)M * N);
  double* tmp = sc.take<double>((size_t)M * N);
  const double* ru = a.ru + base;
  for (int m = 0; m < M; ++m) order[m] = m;
  heap_sort(order, M, [&](int p, int q) {
    if (ru[p] != ru[q]) return ru[p] > ru[q];
    return p < q;
  });
  const double tw = P.prefix[N];  // DnnProfile::total_work, a left fold
  const bool want = a.sch.x != nullptr;
  Sched S{};
  if (want) S = sched_of(a, k);
  double cursor = 0.0;
  int nb = 0;
  if (a.ip.batch_size)
    for (int n = 0; n < N; ++n) a.ip.batch_size[(size_t)k * N + n] = 0;
  for (int oi = 0; oi < M; ++oi) {
    const int m = order[oi];
    const User u = load_user(a, base + m);
    int best_n = N;
    double best_e = __dmul_rn(__dmul_rn(__dmul_rn(u.kappa, tw), u.fmax), u.fmax);
    double best_start = 0.0;
    if (__ddiv_rn(tw, u.fmax) > __dadd_rn(__dsub_rn(u.dl, u.arr), 1e-12))
      return zero_result(a, k, COINFER_ST_INFEASIBLE);
    double prefix = 0.0;
    for (int n = 0; n < N; ++n) {
      if (n > 0) prefix = __dadd_rn(prefix, P.work[n - 1]);
      const double ready =
          __dadd_rn(__dadd_rn(u.arr, __ddiv_rn(prefix, u.fmax)), __ddiv_rn(P.bits[n], u.ru));
      const double start = smax(ready, cursor);
      double done = start;
      for (int i = n + 1; i <= N; ++i) done = __dadd_rn(done, F(a, i, 1));
      if (done > u.dl) continue;
      const double e = __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(u.kappa, prefix), u.fmax), u.fmax),
                                 __dmul_rn(__ddiv_rn(P.bits[n], u.ru), u.pu));
      if (e <= best_e) {
        best_e = e;
        best_n = n;
        best_start = start;
      }
    }
    split[m] = best_n;
    freq[m] = u.fmax;
    ready_t[m] = best_start;
    double t = best_start;
    if (want) local_chain(P, S.comp + (size_t)m * (N + 1), u.arr, best_n, u.fmax);
    if (best_n < N) {
      for (int n = best_n + 1; n <= N; ++n) {
        if (want) {
          S.bstart[nb] = t;
          bsub[nb] = n;
          S.x[(size_t)m * N + n - 1] = nb + 1;
        }
        ++nb;
        t = __dadd_rn(t, F(a, n, 1));
        if (want) S.comp[(size_t)m * (N + 1) + n] = t;
        if (a.ip.batch_size) a.ip.batch_size[(size_t)k * N + n - 1] += 1;
      }
      cursor = t;
    }
    if (want)
      for (int n = 1; n <= best_n; ++n) S.x[(size_t)m * N + n - 1] = 0;
  }
  if (want) {
    for (int m = 0; m < M; ++m) S.freq[m] = freq[m];
    normalize(S, M, N, nb, bsub, perm, tmp);
    *S.nb = nb;
  }
  if (a.ip.batch_bound) a.ip.batch_bound[k] = 0;
  if (a.ip.pipeline_feasible) a.ip.pipeline_feasible[k] = 1;
  finish_result(a, k, split, freq);
}

// detail::ipssa_np_solve after the collapsed IP-SSA (run by the caller on
// the one-sub-task profile whose table is sum_latency): offloaders send B_0
// and run every sub-task in shared batches of `offloaders` copies back to
// back from the collapsed batch start; everyone else stays local.
__device__ void baseline_np(const AuxArgs& a, int64_t k, Scratch& sc) {
  const ProfileConst& P = a.P;
  const int M = a.M, N = P.N;
  const size_t base = (size_t)k * M;
  const int st = a.flat.status[k];
  if (st != COINFER_ST_OK) return zero_result(a, k, st);
  int* split = sc.take<int>(M);
  double* freq = sc.take<double>(M);
  const int b = a.flat.batch_bound[k];
  const int off = M > 0 ? a.flat.batch_size[k] : 0;  // collapsed batch_size[0]
  for (int m = 0; m < M; ++m) {
    split[m] = a.flat.split[base + m] == 0 ? 0 : N;
    freq[m] = a.flat.freq[base + m];
  }
  if (a.ip.batch_size)
    for (int n = 0; n < N; ++n) a.ip.batch_size[(size_t)k * N + n] = off;
  if (a.sch.x) {
    const Sched S = sched_of(a, k);
    double t = 0.0;
    if (off > 0) {
      // the collapsed schedule's batch_start[0]: l - sum_latency(b), with l
      // the smallest deadline (std::min fold from +inf) and sum_latency the
      // left fold of F_n(b)
      double l = dinf();
      for (int m = 0; m < M; ++m) l = smin(l, a.dl[base + m]);
      double sum = 0.0;
      for (int n = 1; n <= N; ++n) sum = __dadd_rn(sum, F(a, n, b));
      t = __dsub_rn(l, sum);
      for (int n = 1; n <= N; ++n) {
        S.bstart[n - 1] = t;
        t = __dadd_rn(t, F(a, n, off));
      }
    }
    for (int m = 0; m < M; ++m) {
      double* tc = S.comp + (size_t)m * (N + 1);
      int* x = S.x + (size_t)m * N;
      if (split[m] == 0) {
        tc[0] = a.arr[base + m];
        for (int n = 1; n <= N; ++n) {
          x[n - 1] = n;
          tc[n] = __dadd_rn(S.bstart[n - 1], F(a, n, off));
        }
      } else {
        local_chain(P, tc, a.arr[base + m], N, freq[m]);
        for (int n = 0; n < N; ++n) x[n] = 0;
      }
      S.freq[m] = freq[m];
    }
    *S.nb = off > 0 ? N : 0;
  }
  if (a.ip.batch_bound) a.ip.batch_bound[k] = b;
  if (a.ip.pipeline_feasible) a.ip.pipeline_feasible[k] = a.flat.pipeline_feasible[k];
  finish_result(a, k, split, freq);
}

__global__ void baseline_kernel(AuxArgs a) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.n_inst;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (a.mode != COINFER_BASELINE_IPSSA_NP) {  // NP: checked by the collapsed IP-SSA
      const int st = check_instance(a, (size_t)k * a.M);
      if (st != COINFER_ST_OK) {
        zero_result(a, k, st);
        continue;
      }
    }
    Scratch sc(a);
    switch (a.mode) {
      case COINFER_BASELINE_LC: baseline_lc(a, k, sc); break;
      case COINFER_BASELINE_PS: baseline_ps(a, k, sc); break;
      case COINFER_BASELINE_FIFO: baseline_fifo(a, k, sc); break;
      default: baseline_np(a, k, sc); break;
    }
  }
}

// best_partition / local_only_choice queries, one thread each.
__global__ void partition_kernel(AuxArgs a, const double* s, int32_t* split, double* freq, double* energy,
                                 uint8_t* feasible) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.n_inst;
       k += (int64_t)gridDim.x * blockDim.x) {
    const User u = load_user(a, k);
    const PC c = s ? best_partition(a.P, u, s + (size_t)k * a.P.N, u.dl) : local_choice(a.P, u, u.dl);
    split[k] = c.split;
    freq[k] = c.freq;
    energy[k] = c.energy;
    feasible[k] = c.feasible ? 1 : 0;
  }
}

// validate (schedule.hpp:139-209) as counts per constraint id, one thread
// per instance; the same checks, in the same order (so the same first
// exception), with the reference's arithmetic.
__global__ void validate_kernel(AuxArgs a) {
  const ProfileConst& P = a.P;
  const int M = a.M, N = P.N;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.n_inst;
       k += (int64_t)gridDim.x * blockDim.x) {
    const Sched S = sched_of(a, k);
    const size_t base = (size_t)k * M;
    const int nb = *S.nb;
    Scratch sc(a);
    int* bsize = sc.take<int>((size_t)M * N);
    int* bsub = sc.take<int>((size_t)M * N);
    int* bmix = sc.take<int>((size_t)M * N);
    int cnt[COINFER_N_CONSTRAINTS] = {0, 0, 0, 0, 0, 0, 0};
    double worst = 0.0;
    int st = COINFER_ST_OK;
    auto hit = [&](int c, double slack) {
      ++cnt[c];
      worst = slack < worst ? slack : worst;
    };
    for (int q = 0; q < nb; ++q) bsize[q] = bsub[q] = bmix[q] = 0;
    // batch_views (schedule.hpp:78-91): members in (m, n) order
    for (int m = 0; m < M && st == COINFER_ST_OK; ++m)
      for (int i = 0; i < N; ++i) {
        const int id = S.x[(size_t)m * N + i];
        if (id == 0) continue;
        if (id > nb || id < 0) {
          st = COINFER_ST_BAD_BATCH_ID;
          break;
        }
        if (bsize[id - 1] == 0) bsub[id - 1] = i + 1;
        else if (bsub[id - 1] != i + 1) bmix[id - 1] = 1;
        ++bsize[id - 1];
      }
    const double tol = a.tol, ntol = -a.tol;
    auto local_at = [&](int m, int n) { return n == 0 || S.x[(size_t)m * N + n - 1] == 0; };
    auto comp = [&](int m, int n) { return S.comp[(size_t)m * (N + 1) + n]; };
    if (st == COINFER_ST_OK) {
      // C7 / C8
      for (int q = 0; q < nb; ++q) {
        if (bsize[q] == 0) hit(0, -1.0);
        else if (bmix[q]) hit(1, -1.0);
      }
      // C17
      for (int m = 0; m < M; ++m) {
        const double d = __dsub_rn(comp(m, 0), a.arr[base + m]);
        if (d < ntol || d > tol) hit(6, -(d < 0 ? -d : d));
      }
      // C9: every member's input at the edge by s_k
      for (int m = 0; m < M; ++m)
        for (int n = 1; n <= N; ++n) {
          const int id = S.x[(size_t)m * N + n - 1];
          if (id == 0) continue;
          double ready = comp(m, n - 1);
          if (local_at(m, n - 1)) ready = __dadd_rn(ready, __ddiv_rn(P.bits[n - 1], a.ru[base + m]));
          const double slack = __dsub_rn(S.bstart[id - 1], ready);
          if (slack < ntol) hit(2, slack);
        }
      // C11: consecutive batch ids
      for (int q = 0; q + 1 < nb && st == COINFER_ST_OK; ++q) {
        double busy = 0.0;
        if (bsize[q] != 0) {
          if (bsize[q] > P.bmax) {
            st = COINFER_ST_BOUND_PAST_TABLE;
            break;
          }
          busy = F(a, bsub[q], bsize[q]);
        }
        const double slack = __dsub_rn(__dsub_rn(S.bstart[q + 1], S.bstart[q]), busy);
        if (slack < ntol) hit(3, slack);
      }
      // C12 / C15
      for (int m = 0; m < M && st == COINFER_ST_OK; ++m) {
        const double rd = a.rd ? a.rd[base + m] : a.ru[base + m];
        for (int n = 1; n <= N; ++n) {
          const int id = S.x[(size_t)m * N + n - 1];
          double need;
          if (id == 0) {
            need = comp(m, n - 1);
            if (n - 1 >= 1 && !local_at(m, n - 1)) need = __dadd_rn(need, __ddiv_rn(P.bits[n - 1], rd));
            const double f = S.freq[m];
            if (f <= 0.0) {  // local_latency throws (core_model.hpp:104-105)
              st = COINFER_ST_NONPOS_FREQ;
              break;
            }
            need = __dadd_rn(need, __ddiv_rn(P.work[n - 1], f));
          } else {
            if (bsize[id - 1] > P.bmax) {
              st = COINFER_ST_BOUND_PAST_TABLE;
              break;
            }
            need = __dadd_rn(S.bstart[id - 1], F(a, n, bsize[id - 1]));
          }
          const double slack = __dsub_rn(comp(m, n), need);
          if (slack < ntol) hit(4, slack);
        }
        if (st != COINFER_ST_OK) break;
        const double slack = __dsub_rn(a.dl[base + m], comp(m, N));
        if (slack < ntol) hit(5, slack);
      }
    }
    a.vstatus[k] = st;
    for (int c = 0; c < COINFER_N_CONSTRAINTS; ++c)
      a.vcounts[(size_t)k * COINFER_N_CONSTRAINTS + c] = st == COINFER_ST_OK ? cnt[c] : 0;
    if (a.vslack) a.vslack[k] = st == COINFER_ST_OK ? worst : 0.0;
  }
}

constexpr int kThreads = 128;

}  // namespace

size_t aux_scratch_bytes(int M, int N) {
  const size_t MN = (size_t)M * N;
  return MN * (8 + 4 + 8 + 4 + 4 + 8) + (size_t)M * (8 + 4 + 8 + 8 + 4) + 16 * 16;
}

int aux_grid(int64_t n_inst) {
  const int64_t cap = 148 * 8;  // one resident wave of 128-thread CTAs bounds the scratch
  const int64_t want = (n_inst + kThreads - 1) / kThreads;
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

cudaError_t launch_materialize_ip(const AuxArgs& a, cudaStream_t st) {
  materialize_ip_kernel<<<aux_grid(a.n_inst), kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_materialize_og(const AuxArgs& a, cudaStream_t st) {
  materialize_og_kernel<<<aux_grid(a.n_inst), kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_baseline(const AuxArgs& a, cudaStream_t st) {
  baseline_kernel<<<aux_grid(a.n_inst), kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_validate(const AuxArgs& a, cudaStream_t st) {
  validate_kernel<<<aux_grid(a.n_inst), kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_partition(const AuxArgs& a, const double* s, int32_t* split, double* freq,
                             double* energy, uint8_t* feasible, cudaStream_t st) {
  partition_kernel<<<aux_grid(a.n_inst), kThreads, 0, st>>>(a, s, split, freq, energy, feasible);
  return cudaGetLastError();
}

}  // namespace cfb
