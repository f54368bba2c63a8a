/*
 * coinfer_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference's offloading and
 * scheduling hot path (arXiv 2206.06304 C++ reference,
 * /root/reference/proj/include/coinfer).  It exists to CHECK the CUDA
 * engine: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.  The product library never links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks this restatement against
 * the reference's own known-answer tests (test_offline_solvers.cpp,
 * test_schedule.cpp, test_oracles.cpp) and against fixtures produced by the
 * unmodified reference headers (tests/golden/, made by
 * tests/golden/make_golden.py through oracle/_ref).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off: the reference is built
 * for baseline x86-64 without FMA contraction, so every a*b+c below rounds
 * twice, exactly like the reference).
 *
 * Semantics followed, function by function:
 *   F()                   edge_batch_latency       core_model.hpp:129-136
 *   total_work()          DnnProfile::total_work   core_model.hpp:25-29
 *   check_instance()      Scenario::check          core_model.hpp:80-101
 *   check_profile()       DnnProfile::check        core_model.hpp:31-52
 *   batch_start_times()   batch_start_times        offline_solvers.hpp:28-40
 *   sum_latency()         sum_latency              offline_solvers.hpp:42-47
 *   local_only_choice()   detail::local_only_choice offline_solvers.hpp:62-75
 *   best_partition()      best_partition           offline_solvers.hpp:83-117
 *   try_fixed_batch()     detail::try_fixed_batch  offline_solvers.hpp:137-188
 *                         + total_energy           schedule.hpp:214-231
 *   try_ip_ssa()          detail::try_ip_ssa       offline_solvers.hpp:192-204
 *   og_one()              og                       offline_solvers.hpp:286-388
 *                         detail::lc_solve         offline_solvers.hpp:255-276
 *   user_energy()         schedule_metrics         offline_solvers.hpp:627-646
 */
#include "coinfer_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int N, bmax, M;
  const double *work, *bits, *lat;
  double total_work;
  const double *fmin, *fmax, *kappa, *ru, *pu, *arr, *dl, *rd, *pd;
} inst_t;

typedef struct {
  int split;
  double freq;
  double energy;
  int feasible;
} choice_t;

/* libstdc++ std::max / std::min (select form, not fmax/fmin). */
static double smax(double a, double b) { return (a < b) ? b : a; }
static double smin(double a, double b) { return (b < a) ? b : a; }

static double F(const inst_t* s, int n, int b) {
  if (b == 0) return 0.0;
  return s->lat[(size_t)(n - 1) * s->bmax + (b - 1)];
}

static double total_work(const coinfer_profile* p) {
  double a = 0.0;
  for (int n = 0; n < p->N; ++n) a += p->work[n];
  return a;
}

int oracle_check_profile(const coinfer_profile* p) {
  if (p->N <= 0) return 1;
  if (p->b_max <= 0) return 1;
  for (int i = 0; i < p->N; ++i) {
    if (p->work[i] <= 0.0) return 1;
    if (p->latency[(size_t)i * p->b_max] <= 0.0) return 1;
    for (int b = 1; b < p->b_max; ++b)
      if (p->latency[(size_t)i * p->b_max + b] < p->latency[(size_t)i * p->b_max + b - 1]) return 1;
  }
  for (int n = 0; n <= p->N; ++n)
    if (p->data_bits[n] < 0.0) return 1;
  return 0;
}

/* Scenario::check per-user part, first failing user, first failing test. */
static int check_instance(const inst_t* s) {
  if (s->bmax < s->M) return COINFER_ST_SHORT_TABLE;
  for (int m = 0; m < s->M; ++m) {
    if (s->fmax[m] <= 0.0 || s->fmin[m] < 0.0 || s->fmin[m] > s->fmax[m]) return COINFER_ST_BAD_FREQ;
    if (s->kappa[m] < 0.0) return COINFER_ST_NEG_KAPPA;
    if (s->ru[m] <= 0.0 || (s->rd && s->rd[m] <= 0.0)) return COINFER_ST_BAD_RATE;
    if (s->pu[m] < 0.0 || (s->pd && s->pd[m] < 0.0)) return COINFER_ST_NEG_POWER;
    if (s->arr[m] < 0.0) return COINFER_ST_NEG_ARRIVAL;
    if (s->dl[m] <= s->arr[m]) return COINFER_ST_EARLY_DEADLINE;
  }
  return COINFER_ST_OK;
}

static int batch_start_times(const inst_t* s, double deadline, int b, double* st) {
  double t = deadline;
  for (int n = s->N; n >= 1; --n) {
    t -= F(s, n, b);
    st[n - 1] = t;
  }
  return st[0] >= 0.0;
}

static double sum_latency(const inst_t* s, int b) {
  double total = 0.0;
  for (int n = 1; n <= s->N; ++n) total += F(s, n, b);
  return total;
}

static choice_t local_only_choice(const inst_t* s, int m, double deadline) {
  choice_t c = {s->N, NAN, INFINITY, 0};
  const double budget = deadline - s->arr[m];
  if (budget <= 0.0) return c;
  const double work = s->total_work;
  const double f_req = work / budget;
  if (f_req > s->fmax[m] * (1.0 + 1e-12)) return c;
  c.freq = smin(smax(f_req, s->fmin[m]), s->fmax[m]);
  c.energy = s->kappa[m] * work * c.freq * c.freq;
  c.feasible = 1;
  return c;
}

static choice_t best_partition(const inst_t* s, int m, const double* st, double deadline) {
  choice_t best = {0, NAN, INFINITY, 0};
  if (s->arr[m] + s->bits[0] / s->ru[m] <= st[0]) {
    best.split = 0;
    best.energy = (s->bits[0] / s->ru[m]) * s->pu[m];
    best.feasible = 1;
  }
  double prefix = 0.0;
  for (int n = 1; n <= s->N; ++n) {
    prefix += s->work[n - 1];
    choice_t c = {0, NAN, INFINITY, 0};
    if (n == s->N) {
      c = local_only_choice(s, m, deadline);
    } else {
      const double upload = s->bits[n] / s->ru[m];
      const double budget = st[n] - upload - s->arr[m];
      if (budget <= 0.0) continue;
      const double f_req = prefix / budget;
      if (f_req > s->fmax[m]) continue;
      c.split = n;
      c.freq = smin(smax(f_req, s->fmin[m]), s->fmax[m]);
      c.energy = s->kappa[m] * prefix * c.freq * c.freq + (s->bits[n] / s->ru[m]) * s->pu[m];
      c.feasible = 1;
    }
    if (c.feasible && c.energy <= best.energy) best = c;
  }
  return best;
}

/* Schedule frequency of a choice (try_fixed_batch:170). */
static double sched_freq(const inst_t* s, int m, const choice_t* c) {
  return c->split == 0 ? s->fmax[m] : c->freq;
}

/* One user's contribution, in total_energy's term order, added onto acc. */
static double fold_user(const inst_t* s, int m, int split, double f, double acc) {
  for (int n = 1; n <= split; ++n) acc += s->kappa[m] * s->work[n - 1] * f * f;
  if (split < s->N) acc += (s->bits[split] / s->ru[m]) * s->pu[m];
  return acc;
}

typedef struct {
  int ok;
  int b;
  int pipe;
  double energy;
  int* split; /* [cnt] */
  double* freq;
} fixed_t;

/* try_fixed_batch over the sub-scenario ids[0..cnt-1]. */
static int try_fixed_batch(const inst_t* s, const int* ids, int cnt, double deadline, int b,
                           int* split, double* freq, double* energy, int* pipe) {
  double st[COINFER_MAX_SUBTASKS];
  const int feas = batch_start_times(s, deadline, b, st);
  *pipe = feas;
  for (int k = 0; k < cnt; ++k) {
    const int m = ids[k];
    const choice_t c = feas ? best_partition(s, m, st, s->dl[m]) : local_only_choice(s, m, s->dl[m]);
    if (!c.feasible) return 0;
    split[k] = c.split;
    freq[k] = sched_freq(s, m, &c);
  }
  double total = 0.0;
  for (int k = 0; k < cnt; ++k) total = fold_user(s, ids[k], split[k], freq[k], total);
  *energy = total;
  return 1;
}

/* try_ip_ssa over ids; returns 1 and fills best_* when some b admits all. */
static int try_ip_ssa(const inst_t* s, const int* ids, int cnt, double deadline, int* best_b,
                      int* best_pipe, double* best_e, int* best_split, double* best_freq,
                      int* scratch_split, double* scratch_freq) {
  if (cnt == 0) {
    *best_b = 0;
    *best_pipe = 1;
    *best_e = 0.0;
    return 1;
  }
  int have = 0;
  for (int b = cnt; b >= 1; --b) {
    double e;
    int pipe;
    if (!try_fixed_batch(s, ids, cnt, deadline, b, scratch_split, scratch_freq, &e, &pipe)) continue;
    int realized = 0;
    for (int k = 0; k < cnt; ++k) realized += scratch_split[k] < s->N;
    if (realized <= b && (!have || e < *best_e)) {
      have = 1;
      *best_b = b;
      *best_pipe = pipe;
      *best_e = e;
      if (best_split) memcpy(best_split, scratch_split, sizeof(int) * cnt);
      if (best_freq) memcpy(best_freq, scratch_freq, sizeof(double) * cnt);
    }
  }
  return have;
}

static void make_inst(inst_t* s, const coinfer_profile* p, const coinfer_users* u, int64_t k) {
  s->N = p->N;
  s->bmax = p->b_max;
  s->M = u->M;
  s->work = p->work;
  s->bits = p->data_bits;
  s->lat = p->latency;
  s->total_work = total_work(p);
  const size_t o = (size_t)k * u->M;
  s->fmin = u->f_min + o;
  s->fmax = u->f_max + o;
  s->kappa = u->kappa + o;
  s->ru = u->rate_up + o;
  s->pu = u->power_up + o;
  s->arr = u->arrival + o;
  s->dl = u->deadline + o;
  s->rd = u->rate_down ? u->rate_down + o : NULL;
  s->pd = u->power_down ? u->power_down + o : NULL;
}

/* schedule_metrics per-user energy for a suffix schedule. */
static double user_energy(const inst_t* s, int m, int split, double f) {
  return fold_user(s, m, split, f, 0.0);
}

static void write_solve(const inst_t* s, const coinfer_users* u, int64_t k, const int* split,
                        const double* freq, int b, int pipe, double e, coinfer_ipssa_out* out) {
  const int M = s->M, N = s->N;
  if (out->batch_bound) out->batch_bound[k] = b;
  if (out->pipeline_feasible) out->pipeline_feasible[k] = (uint8_t)pipe;
  if (out->energy) out->energy[k] = e;
  for (int m = 0; m < M; ++m) {
    if (out->split) out->split[(size_t)k * M + m] = (uint8_t)split[m];
    if (out->freq) out->freq[(size_t)k * M + m] = freq[m];
    if (out->user_energy) out->user_energy[(size_t)k * M + m] = user_energy(s, m, split[m], freq[m]);
  }
  if (out->batch_size)
    for (int n = 1; n <= N; ++n) {
      int c = 0;
      for (int m = 0; m < M; ++m) c += split[m] < n;
      out->batch_size[(size_t)k * N + n - 1] = c;
    }
  (void)u;
}

static double min_deadline(const inst_t* s) {
  double l = s->dl[0];
  for (int m = 0; m < s->M; ++m) l = smin(l, s->dl[m]);
  return l;
}

int oracle_ipssa_batch(const coinfer_profile* p, const coinfer_users* u, const double* deadline,
                       coinfer_ipssa_out* out) {
  if (oracle_check_profile(p)) return COINFER_E_PROFILE;
  if (p->N > COINFER_MAX_SUBTASKS) return COINFER_E_UNSUPPORTED;
  const int M = u->M;
  int* ids = malloc(sizeof(int) * (M + 1));
  int* split = malloc(sizeof(int) * (M + 1));
  int* ssplit = malloc(sizeof(int) * (M + 1));
  double* freq = malloc(sizeof(double) * (M + 1));
  double* sfreq = malloc(sizeof(double) * (M + 1));
  for (int m = 0; m < M; ++m) ids[m] = m;
  for (int64_t k = 0; k < u->n_inst; ++k) {
    inst_t s;
    make_inst(&s, p, u, k);
    int st = check_instance(&s);
    if (st == COINFER_ST_OK) {
      if (M == 0) {
        write_solve(&s, u, k, split, freq, 0, 1, 0.0, out);
      } else {
        const double l = deadline ? deadline[k] : min_deadline(&s);
        int b, pipe;
        double e;
        if (try_ip_ssa(&s, ids, M, l, &b, &pipe, &e, split, freq, ssplit, sfreq))
          write_solve(&s, u, k, split, freq, b, pipe, e, out);
        else
          st = COINFER_ST_INFEASIBLE;
      }
    }
    if (out->status) out->status[k] = st;
  }
  free(ids);
  free(split);
  free(ssplit);
  free(freq);
  free(sfreq);
  return COINFER_OK;
}

int oracle_fixed_batch(const coinfer_profile* p, const coinfer_users* u, const double* deadline,
                       const int32_t* b, coinfer_ipssa_out* out) {
  if (oracle_check_profile(p)) return COINFER_E_PROFILE;
  if (p->N > COINFER_MAX_SUBTASKS) return COINFER_E_UNSUPPORTED;
  const int M = u->M;
  int* ids = malloc(sizeof(int) * (M + 1));
  int* split = malloc(sizeof(int) * (M + 1));
  double* freq = malloc(sizeof(double) * (M + 1));
  for (int m = 0; m < M; ++m) ids[m] = m;
  for (int64_t k = 0; k < u->n_inst; ++k) {
    inst_t s;
    make_inst(&s, p, u, k);
    int st = check_instance(&s);
    if (st == COINFER_ST_OK) {
      if (b[k] < 1) {
        st = COINFER_ST_ZERO_BOUND;
      } else if (b[k] > s.bmax) {
        st = COINFER_ST_BOUND_PAST_TABLE;
      } else {
        const double l = deadline ? deadline[k] : min_deadline(&s);
        double e;
        int pipe;
        if (try_fixed_batch(&s, ids, M, l, b[k], split, freq, &e, &pipe))
          write_solve(&s, u, k, split, freq, b[k], pipe, e, out);
        else
          st = COINFER_ST_INFEASIBLE;
      }
    }
    if (out->status) out->status[k] = st;
  }
  free(ids);
  free(split);
  free(freq);
  return COINFER_OK;
}

/* ---------------------------------------------------------------- OG ---- */

/* G row i by the shared left fold: for a fixed group
   start i and assumed bound b, the per-user choices do not depend on the
   group end j, and total_energy is a prefix-consistent left fold, so the
   energies of all groups i..j come out of one pass over j.  Two exact cuts
   (SURVEY §7 "b-pruning"):
     * every bound b >= b0 (the first whose pipeline does not fit dl[i];
       feasibility is monotone in b) sends every user local-only
       (try_fixed_batch:148-150) with the same energies, so those bounds
       collapse into one pass keyed with the largest admissible bound,
       b = j-i+1 (the reference's descending-b scan with strict '<' keeps
       the largest b among equal energies);
     * a chain whose offloader count exceeds b is never admissible again
       (the count never decreases along j), so it stops there.
   Bit-identical to calling try_ip_ssa(subscenario(i..j), dl[i]) per cell
   (tests compare the two forms cell by cell and against the reference). */
static void g_row_fast(const inst_t* s, const int* order, int i, double* G, int* B) {
  const int M = s->M, N = s->N;
  const double dli = s->dl[order[i]];
  for (int j = i; j < M; ++j) {
    G[j] = INFINITY;
    B[j] = 0;
  }
  int b0 = 1;  /* first bound whose pipeline does not fit dl[i] (or M-i+1) */
  {
    int lo = 1, hi = M - i + 1;
    while (lo < hi) {
      const int mid = (lo + hi) / 2;
      double st[COINFER_MAX_SUBTASKS];
      if (batch_start_times(s, dli, mid, st)) lo = mid + 1; else hi = mid;
    }
    b0 = lo;
  }
  for (int b = 1; b < b0; ++b) {
    double st[COINFER_MAX_SUBTASKS];
    batch_start_times(s, dli, b, st);
    double total = 0.0;
    int offl = 0;
    for (int j = i; j < M; ++j) {
      const int m = order[j];
      const choice_t c = best_partition(s, m, st, s->dl[m]);
      if (!c.feasible) break;
      const double f = sched_freq(s, m, &c);
      total = fold_user(s, m, c.split, f, total);
      offl += c.split < N;
      if (offl > b) break;
      if (b <= j - i + 1 && (total < G[j] || (total == G[j] && b > B[j]))) {
        G[j] = total;
        B[j] = b;
      }
    }
  }
  if (b0 <= M - i) { /* the all-local pass: bounds b0..j-i+1 */
    double total = 0.0;
    for (int j = i; j < M; ++j) {
      const int m = order[j];
      const choice_t c = local_only_choice(s, m, s->dl[m]);
      if (!c.feasible) break;
      total = fold_user(s, m, N, c.freq, total);
      const int b = j - i + 1;
      if (b >= b0 && (total < G[j] || (total == G[j] && b > B[j]))) {
        G[j] = total;
        B[j] = b;
      }
    }
  }
}

static int cmp_deadline_ctx_dl_sort(const double* dl, int a, int b) {
  if (dl[a] < dl[b]) return -1;
  if (dl[b] < dl[a]) return 1;
  return (a > b) - (a < b);
}

/* Stable sort of user ids by (deadline, id): insertion sort keeps the code
   obviously equal to std::sort with std::tie (a strict total order). */
static void sort_by_deadline(const double* dl, int* order, int M) {
  for (int m = 0; m < M; ++m) order[m] = m;
  for (int a = 1; a < M; ++a) {
    const int v = order[a];
    int k = a - 1;
    while (k >= 0 && cmp_deadline_ctx_dl_sort(dl, order[k], v) > 0) {
      order[k + 1] = order[k];
      --k;
    }
    order[k + 1] = v;
  }
}

static int og_one(const inst_t* s, int fast, int64_t k, coinfer_og_out* out) {
  const int M = s->M, N = s->N;
  if (out->energy) out->energy[k] = 0.0;
  if (out->fallback) out->fallback[k] = 0;
  if (out->n_groups) out->n_groups[k] = 0;
  if (M == 0) return COINFER_ST_OK;
  const size_t MM = (size_t)M * M;
  int* order = malloc(sizeof(int) * M);
  double* dl = malloc(sizeof(double) * M);
  double* G = malloc(sizeof(double) * MM);
  int* GB = malloc(sizeof(int) * MM);
  double* S = malloc(sizeof(double) * MM);
  int* parent = malloc(sizeof(int) * MM);
  int* sp = malloc(sizeof(int) * M);
  int* sp2 = malloc(sizeof(int) * M);
  double* fq = malloc(sizeof(double) * M);
  double* fq2 = malloc(sizeof(double) * M);
  int st = COINFER_ST_OK;

  sort_by_deadline(s->dl, order, M);
  for (int i = 0; i < M; ++i) dl[i] = s->dl[order[i]];

  /* G[i][j] (offline_solvers.hpp:304-311) */
  for (int i = 0; i < M; ++i) {
    if (fast) {
      g_row_fast(s, order, i, G + (size_t)i * M, GB + (size_t)i * M);
      continue;
    }
    for (int j = 0; j < M; ++j) {
      G[(size_t)i * M + j] = INFINITY;
      GB[(size_t)i * M + j] = 0;
    }
    for (int j = i; j < M; ++j) {
      int b, pipe;
      double e;
      if (try_ip_ssa(s, order + i, j - i + 1, dl[i], &b, &pipe, &e, NULL, NULL, sp, fq)) {
        G[(size_t)i * M + j] = e;
        GB[(size_t)i * M + j] = b;
      }
    }
  }

  /* DP (offline_solvers.hpp:313-330).  S is stored transposed (column i-1
     is contiguous: the prev loop reads it in order) and sum_latency(size)
     is tabulated once; the comparisons and their order are the reference's. */
  double* sl = malloc(sizeof(double) * (M + 1));
  for (int z = 1; z <= M; ++z) sl[z] = sum_latency(s, z);
  for (size_t x = 0; x < MM; ++x) {
    S[x] = INFINITY;
    parent[x] = -1;
  }
#define ST(row, col) S[(size_t)(col) * M + (row)]
  for (int j = 0; j < M; ++j) ST(0, j) = G[j];
  for (int i = 1; i < M; ++i) {
    const double* col = &ST(0, i - 1);
    for (int j = i; j < M; ++j) {
      const double g = G[(size_t)i * M + j];
      if (g == INFINITY) continue;
      const double thr = sl[j - i + 1];
      double best = INFINITY;
      int bp = -1;
      for (int prev = 0; prev < i; ++prev) {
        const double sp_ = col[prev];
        if (sp_ == INFINITY) continue;
        if (!(dl[prev] + thr <= dl[i])) continue;  /* groups_fit */
        const double cand = sp_ + g;
        if (cand < best) {
          best = cand;
          bp = prev;
        }
      }
      ST(i, j) = best;
      parent[(size_t)i * M + j] = bp;
    }
  }
  int best_i = 0;
  for (int i = 1; i < M; ++i)
    if (ST(i, M - 1) < ST(best_i, M - 1)) best_i = i;
  const double s_best = ST(best_i, M - 1);
#undef ST
  free(sl);

  if (out->order)
    for (int i = 0; i < M; ++i) out->order[(size_t)k * M + i] = order[i];

  if (s_best == INFINITY) {
    /* lc_solve fallback (offline_solvers.hpp:336-348, 255-276) */
    double total = 0.0;
    for (int m = 0; m < M; ++m) {
      const choice_t c = local_only_choice(s, m, s->dl[m]);
      if (!c.feasible) {
        st = COINFER_ST_INFEASIBLE;
        goto done;
      }
      sp[m] = N;
      fq[m] = c.freq;
      total = fold_user(s, m, N, c.freq, total);
    }
    if (out->fallback) out->fallback[k] = 1;
    if (out->energy) out->energy[k] = total;
    if (out->n_groups) out->n_groups[k] = M;
    for (int i = 0; i < M; ++i) {
      const int m = order[i];
      const size_t g = (size_t)k * M + i;
      if (out->group_lo) out->group_lo[g] = i;
      if (out->group_size) out->group_size[g] = 1;
      if (out->group_b) out->group_b[g] = 0;
      if (out->group_deadline) out->group_deadline[g] = dl[i];
      if (out->group_energy) out->group_energy[g] = fold_user(s, m, N, fq[m], 0.0);
      if (out->group_batch_size)
        for (int n = 0; n < N; ++n) out->group_batch_size[g * N + n] = 0;
      if (out->group_of_user) out->group_of_user[(size_t)k * M + m] = i;
    }
    for (int m = 0; m < M; ++m) {
      if (out->split) out->split[(size_t)k * M + m] = (uint8_t)N;
      if (out->freq) out->freq[(size_t)k * M + m] = fq[m];
      if (out->user_energy) out->user_energy[(size_t)k * M + m] = fold_user(s, m, N, fq[m], 0.0);
    }
    goto done;
  }

  {
    /* backtrack (offline_solvers.hpp:350-360) */
    int lo_list[4096], hi_list[4096];
    int* los = M <= 4096 ? lo_list : malloc(sizeof(int) * M);
    int* his = M <= 4096 ? hi_list : malloc(sizeof(int) * M);
    int ng = 0;
    int i = best_i, j = M - 1;
    while (1) {
      los[ng] = i;
      his[ng] = j;
      ++ng;
      if (i == 0) break;
      const int prev = parent[(size_t)i * M + j];
      j = i - 1;
      i = prev;
    }
    /* reverse */
    for (int a = 0, b = ng - 1; a < b; ++a, --b) {
      int t = los[a];
      los[a] = los[b];
      los[b] = t;
      t = his[a];
      his[a] = his[b];
      his[b] = t;
    }
    double energy = 0.0;
    for (int g = 0; g < ng; ++g) {
      const int lo = los[g], hi = his[g], cnt = hi - lo + 1;
      int b, pipe;
      double e;
      try_ip_ssa(s, order + lo, cnt, dl[lo], &b, &pipe, &e, sp, fq, sp2, fq2);
      energy += e;
      const size_t gi = (size_t)k * M + g;
      if (out->group_lo) out->group_lo[gi] = lo;
      if (out->group_size) out->group_size[gi] = cnt;
      if (out->group_b) out->group_b[gi] = b;
      if (out->group_deadline) out->group_deadline[gi] = dl[lo];
      if (out->group_energy) out->group_energy[gi] = e;
      if (out->group_batch_size)
        for (int n = 1; n <= N; ++n) {
          int c = 0;
          for (int x = 0; x < cnt; ++x) c += sp[x] < n;
          out->group_batch_size[gi * N + n - 1] = c;
        }
      for (int x = 0; x < cnt; ++x) {
        const int m = order[lo + x];
        const size_t um = (size_t)k * M + m;
        if (out->group_of_user) out->group_of_user[um] = g;
        if (out->split) out->split[um] = (uint8_t)sp[x];
        if (out->freq) out->freq[um] = fq[x];
        if (out->user_energy) out->user_energy[um] = fold_user(s, m, sp[x], fq[x], 0.0);
      }
    }
    if (out->energy) out->energy[k] = energy;
    if (out->n_groups) out->n_groups[k] = ng;
    if (los != lo_list) free(los);
    if (his != hi_list) free(his);
  }
done:
  free(order);
  free(dl);
  free(G);
  free(GB);
  free(S);
  free(parent);
  free(sp);
  free(sp2);
  free(fq);
  free(fq2);
  return st;
}

int oracle_og_batch(const coinfer_profile* p, const coinfer_users* u, coinfer_og_out* out, int fast) {
  if (oracle_check_profile(p)) return COINFER_E_PROFILE;
  if (p->N > COINFER_MAX_SUBTASKS) return COINFER_E_UNSUPPORTED;
  for (int64_t k = 0; k < u->n_inst; ++k) {
    inst_t s;
    make_inst(&s, p, u, k);
    int st = check_instance(&s);
    if (st == COINFER_ST_OK) st = og_one(&s, fast, k, out);
    if (out->status) out->status[k] = st;
  }
  return COINFER_OK;
}

/* G table only (fast or direct), row-major [i][j] over the sorted order;
   used by tests to compare the two forms cell by cell. */
int oracle_og_gtable(const coinfer_profile* p, const coinfer_users* u, int64_t k, int fast,
                     double* G, int32_t* B) {
  inst_t s;
  make_inst(&s, p, u, k);
  const int M = s.M;
  int* order = malloc(sizeof(int) * (M + 1));
  int* sp = malloc(sizeof(int) * (M + 1));
  double* fq = malloc(sizeof(double) * (M + 1));
  int* row = malloc(sizeof(int) * (M + 1));
  sort_by_deadline(s.dl, order, M);
  for (int i = 0; i < M; ++i) {
    if (fast) {
      g_row_fast(&s, order, i, G + (size_t)i * M, row);
      for (int j = 0; j < M; ++j) B[(size_t)i * M + j] = j >= i ? row[j] : 0;
      for (int j = 0; j < i; ++j) G[(size_t)i * M + j] = INFINITY;
      continue;
    }
    for (int j = 0; j < M; ++j) {
      G[(size_t)i * M + j] = INFINITY;
      B[(size_t)i * M + j] = 0;
    }
    for (int j = i; j < M; ++j) {
      int b, pipe;
      double e;
      if (try_ip_ssa(&s, order + i, j - i + 1, s.dl[order[i]], &b, &pipe, &e, NULL, NULL, sp, fq)) {
        G[(size_t)i * M + j] = e;
        B[(size_t)i * M + j] = b;
      }
    }
  }
  free(order);
  free(sp);
  free(fq);
  free(row);
  return 0;
}
