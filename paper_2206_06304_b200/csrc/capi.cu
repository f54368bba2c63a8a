// capi.cu — the extern "C" boundary (include/coinfer_b200.h).
//
// No exceptions cross this boundary; errors are return codes plus a
// per-context message.  There is no CPU solver behind it: every solve runs
// in the sm_100a kernels, host memory is only staged through.

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/coinfer_b200.h"
#include "kernels.h"

namespace cfb {
cudaError_t probe_fp64(cudaStream_t st, double* ops_per_s);
}

struct coinfer_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  // latency table on the device, re-uploaded only when it changes
  double* d_lat = nullptr;
  size_t lat_cap = 0;
  std::vector<double> lat_host;
  // host-memory calls: chunks alternate over two streams / two workspaces so
  // the copies of one chunk overlap the solve of the other
  cudaStream_t pipe[2] = {nullptr, nullptr};
  unsigned char* ws2[2] = {nullptr, nullptr};
  size_t ws2_cap[2] = {0, 0};
  // large-instance path: instances of a batch run round-robin on up to
  // kLargeStreams streams, each with its own workspace (G/S triangles etc.)
  static constexpr int kLargeStreams = 16;
  cudaStream_t lst[kLargeStreams] = {};
  cudaEvent_t lev[kLargeStreams] = {};
  unsigned char* big[kLargeStreams] = {};
  size_t big_cap[kLargeStreams] = {};
  cudaEvent_t lstart = nullptr;
  // schedule / baseline / partition calls: staging + scratch (baselines.cu)
  unsigned char* aux = nullptr;
  size_t aux_cap = 0;
  // coinfer_count_work: device work counters while a counting solve runs
  unsigned long long* ctr = nullptr;
  // pipelined kernel: instance claim counters, one per launch in rotation
  // (each launch zeroes its own on its stream first)
  static constexpr int kClaims = 64;
  unsigned long long* claim = nullptr;
  int claim_next = 0;
  // pipelined kernel: global G tables, one workspace per stream it runs on
  // (ctx->stream, pipe[0], pipe[1]: launches on different streams may overlap)
  double* gg[3] = {nullptr, nullptr, nullptr};
  size_t gg_cap[3] = {0, 0, 0};
};

namespace cfb {
cudaError_t ensure_smem(const void* f, int smem, bool carveout) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> smem set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({f, dev});
  if (it != done.end() && it->second >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (carveout) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
  }
  done[{f, dev}] = smem;
  return cudaSuccess;
}
}  // namespace cfb

namespace {

int fail(coinfer_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_fail(coinfer_ctx* ctx, cudaError_t e, const char* what) {
  return fail(ctx, COINFER_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// DnnProfile::check (core_model.hpp:31-52), same messages.
int check_profile(coinfer_ctx* ctx, const coinfer_profile* p) {
  if (!p || !p->work || !p->data_bits || !p->latency)
    return fail(ctx, COINFER_E_ARG, "profile: null array");
  if (p->N <= 0) return fail(ctx, COINFER_E_PROFILE, "profile: no sub-tasks");
  if (p->b_max <= 0) return fail(ctx, COINFER_E_PROFILE, "profile: empty latency row");
  for (int i = 0; i < p->N; ++i) {
    if (p->work[i] <= 0.0) return fail(ctx, COINFER_E_PROFILE, "profile: work must be positive");
    const double* row = p->latency + (size_t)i * p->b_max;
    if (row[0] <= 0.0) return fail(ctx, COINFER_E_PROFILE, "profile: F_n(1) must be positive");
    for (int b = 1; b < p->b_max; ++b)
      if (row[b] < row[b - 1])
        return fail(ctx, COINFER_E_PROFILE, "profile: F_n(b) must be nondecreasing in b");
  }
  for (int n = 0; n <= p->N; ++n)
    if (p->data_bits[n] < 0.0) return fail(ctx, COINFER_E_PROFILE, "profile: negative data size");
  if (p->N > COINFER_MAX_SUBTASKS)
    return fail(ctx, COINFER_E_UNSUPPORTED, "profile: more sub-tasks than COINFER_MAX_SUBTASKS");
  return COINFER_OK;
}

cfb::ProfileConst make_const(const coinfer_profile* p) {
  cfb::ProfileConst P;
  std::memset(&P, 0, sizeof P);
  P.N = p->N;
  P.bmax = p->b_max;
  double acc = 0.0;
  P.prefix[0] = 0.0;
  for (int n = 0; n < p->N; ++n) {
    P.work[n] = p->work[n];
    acc += p->work[n];  // left fold, as DnnProfile::total_work / best_partition
    P.prefix[n + 1] = acc;
  }
  for (int n = 0; n <= p->N; ++n) P.bits[n] = p->data_bits[n];
  return P;
}

int upload_latency(coinfer_ctx* ctx, const coinfer_profile* p) {
  const size_t n = (size_t)p->N * p->b_max;
  if (ctx->lat_host.size() == n && std::memcmp(ctx->lat_host.data(), p->latency, n * 8) == 0)
    return COINFER_OK;
  if (ctx->d_lat) {
    // a different table: kernels still in flight on any stream may read the
    // old one, so drain the device before overwriting it (profiles change rarely)
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "synchronize before latency upload");
  }
  if (n > ctx->lat_cap) {
    if (ctx->d_lat) cudaFree(ctx->d_lat);
    ctx->d_lat = nullptr;
    cudaError_t e = cudaMalloc(&ctx->d_lat, n * 8);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(latency)");
    ctx->lat_cap = n;
  }
  ctx->lat_host.assign(p->latency, p->latency + n);
  cudaError_t e =
      cudaMemcpyAsync(ctx->d_lat, ctx->lat_host.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "upload latency");
  e = cudaStreamSynchronize(ctx->stream);  // lat_host may change on the next call
  if (e != cudaSuccess) return cuda_fail(ctx, e, "upload latency");
  return COINFER_OK;
}

// Host-memory calls: inputs are copied into one device workspace, outputs
// are produced there and copied back.
struct Stager {
  coinfer_ctx* ctx;
  size_t used = 0;
  struct Back {
    void* host;
    size_t off;
    size_t bytes;
  };
  std::vector<Back> back;
  struct In {
    const void* host;
    size_t off;
    size_t bytes;
  };
  std::vector<In> in;
  size_t reserve(size_t bytes) {
    const size_t off = used;
    used += (bytes + 255) & ~size_t(255);
    return off;
  }
};

template <class T>
void plan_in(Stager& s, const T*& p, size_t count) {
  if (!p) return;
  const size_t off = s.reserve(count * sizeof(T));
  s.in.push_back({p, off, count * sizeof(T)});
  p = reinterpret_cast<const T*>(off + 1);  // placeholder, patched after allocation
}

template <class T>
void plan_out(Stager& s, T*& p, size_t count) {
  if (!p) return;
  const size_t off = s.reserve(count * sizeof(T));
  s.back.push_back({p, off, count * sizeof(T)});
  p = reinterpret_cast<T*>(off + 1);
}

template <class T>
void patch(unsigned char* base, T*& p) {
  if (p) p = reinterpret_cast<T*>(base + (reinterpret_cast<uintptr_t>(p) - 1));
}

int ensure_ws(coinfer_ctx* ctx, int slot, size_t bytes) {
  if (!ctx->pipe[slot]) {
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->pipe[slot], cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamCreate");
  }
  if (bytes <= ctx->ws2_cap[slot]) return COINFER_OK;
  if (ctx->ws2[slot]) {
    cudaStreamSynchronize(ctx->pipe[slot]);
    cudaFree(ctx->ws2[slot]);
  }
  ctx->ws2[slot] = nullptr;
  ctx->ws2_cap[slot] = 0;
  cudaError_t e = cudaMalloc(&ctx->ws2[slot], bytes);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(workspace)");
  ctx->ws2_cap[slot] = bytes;
  return COINFER_OK;
}

void plan_ip_out(Stager& s, coinfer_ipssa_out& o, size_t K, size_t M, size_t N) {
  plan_out(s, o.status, K);
  plan_out(s, o.batch_bound, K);
  plan_out(s, o.pipeline_feasible, K);
  plan_out(s, o.energy, K);
  plan_out(s, o.split, K * M);
  plan_out(s, o.freq, K * M);
  plan_out(s, o.user_energy, K * M);
  plan_out(s, o.batch_size, K * N);
}

void patch_ip_out(unsigned char* b, coinfer_ipssa_out& o) {
  patch(b, o.status);
  patch(b, o.batch_bound);
  patch(b, o.pipeline_feasible);
  patch(b, o.energy);
  patch(b, o.split);
  patch(b, o.freq);
  patch(b, o.user_energy);
  patch(b, o.batch_size);
}

void plan_og_out(Stager& s, coinfer_og_out& o, size_t K, size_t M, size_t N) {
  plan_out(s, o.status, K);
  plan_out(s, o.fallback, K);
  plan_out(s, o.energy, K);
  plan_out(s, o.n_groups, K);
  plan_out(s, o.order, K * M);
  plan_out(s, o.group_of_user, K * M);
  plan_out(s, o.split, K * M);
  plan_out(s, o.freq, K * M);
  plan_out(s, o.user_energy, K * M);
  plan_out(s, o.group_lo, K * M);
  plan_out(s, o.group_size, K * M);
  plan_out(s, o.group_b, K * M);
  plan_out(s, o.group_deadline, K * M);
  plan_out(s, o.group_energy, K * M);
  plan_out(s, o.group_batch_size, K * M * N);
}

void patch_og_out(unsigned char* b, coinfer_og_out& o) {
  patch(b, o.status);
  patch(b, o.fallback);
  patch(b, o.energy);
  patch(b, o.n_groups);
  patch(b, o.order);
  patch(b, o.group_of_user);
  patch(b, o.split);
  patch(b, o.freq);
  patch(b, o.user_energy);
  patch(b, o.group_lo);
  patch(b, o.group_size);
  patch(b, o.group_b);
  patch(b, o.group_deadline);
  patch(b, o.group_energy);
  patch(b, o.group_batch_size);
}

#ifndef CFB_E2E_CHUNKS
#define CFB_E2E_CHUNKS 64  // host-memory batches: up to this many chunks pipelined over two streams
#endif
#ifndef CFB_E2E_MINCHUNK
// instances per chunk, at least (measured, 1M C3 instances: 8 / 16 / 32 chunks 8.17 / 8.40 / 8.53M/s e2e
// in round 1; 32 / 64 / 128 chunks 11.25 / 11.31 / 11.21M/s e2e on the round-2 kernel)
#define CFB_E2E_MINCHUNK 16384
#endif
constexpr int kSmallMaxM = 255;
#ifndef CFB_PIPE_MAXM
#define CFB_PIPE_MAXM 64  // largest M run by the pipelined kernel (measured: see DESIGN.md §4)
#endif  // u8 group/bound indices in shared memory

// Instances too large for one CTA's shared memory: the multi-kernel path of
// solve_large.cu, one instance at a time.  `a` carries device pointers.
int run_large_device(coinfer_ctx* ctx, const cfb::SmallArgs& a, cudaStream_t st) {
  // One instance = 6 dependent launches (solve_large.cu).  A batch runs its
  // instances round-robin on up to kLargeStreams streams, each with its own
  // workspace (bounded to ~4 GB in total), ordered after everything already
  // queued on `st`; `st` then waits for all of them.
  const int M = a.M, N = a.P.N;
  const size_t need = cfb::large_ws_bytes(M, N);
  int S = (int)std::min<int64_t>(coinfer_ctx::kLargeStreams, std::max<int64_t>(1, a.n_inst));
  S = (int)std::max<size_t>(1, std::min<size_t>((size_t)S, ((size_t)4 << 30) / std::max<size_t>(need, 1)));
  cudaError_t e;
  if (!ctx->lstart) {
    e = cudaEventCreateWithFlags(&ctx->lstart, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaEventCreate");
  }
  e = cudaEventRecord(ctx->lstart, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaEventRecord");
  for (int w = 0; w < S; ++w) {
    if (!ctx->lst[w]) {
      e = cudaStreamCreateWithFlags(&ctx->lst[w], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->lev[w], cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "large-path stream");
    }
    if (need > ctx->big_cap[w]) {
      cudaStreamSynchronize(ctx->lst[w]);
      if (ctx->big[w]) cudaFree(ctx->big[w]);
      ctx->big[w] = nullptr;
      ctx->big_cap[w] = 0;
      e = cudaMalloc(&ctx->big[w], need);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(large workspace)");
      ctx->big_cap[w] = need;
    }
    e = cudaStreamWaitEvent(ctx->lst[w], ctx->lstart, 0);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamWaitEvent");
  }
  const size_t T = (size_t)M * (M + 1) / 2;
  auto workspace = [&](int w) {
    unsigned char* p = ctx->big[w];
    auto take = [&](size_t bytes) {
      unsigned char* q = p;
      p += (bytes + 255) & ~size_t(255);
      return q;
    };
    cfb::LargeArgs L;
    std::memset(&L, 0, sizeof L);
    L.P = a.P;
    L.lat = a.lat;
    L.M = M;
    L.do_ip = a.do_ip;
    L.do_og = a.do_og;
    L.G = reinterpret_cast<double*>(take(8 * T));
    L.St = reinterpret_cast<double*>(take(8 * T));
    L.bstar = reinterpret_cast<uint16_t*>(take(2 * T));
    L.par = reinterpret_cast<uint16_t*>(take(2 * T));
    L.pfit = reinterpret_cast<uint16_t*>(take(2 * T));
    L.argpm = reinterpret_cast<uint16_t*>(take(2 * T));
    L.slast = reinterpret_cast<double*>(take(8 * (size_t)M));
    L.rec = reinterpret_cast<double*>(take((size_t)M * cfb::rec_size(N) * 8));
    L.dls = reinterpret_cast<double*>(take(8 * (size_t)M));
    L.sumlat = reinterpret_cast<double*>(take(8 * ((size_t)M + 2)));
    L.fpos = reinterpret_cast<double*>(take(8 * (size_t)M));
    L.genergy = reinterpret_cast<double*>(take(8 * (size_t)M));
    L.ipres = reinterpret_cast<double*>(take(8));
    L.order = reinterpret_cast<int*>(take(4 * (size_t)M));
    L.rank = reinterpret_cast<int*>(take(4 * (size_t)M));
    L.b0 = reinterpret_cast<int*>(take(4 * ((size_t)M + 2)));
    L.spos = reinterpret_cast<int*>(take(4 * (size_t)M));
    L.gid = reinterpret_cast<int*>(take(4 * (size_t)M));
    L.rlen = reinterpret_cast<int*>(take(4 * (size_t)M));
    L.status = reinterpret_cast<int*>(take(4));
    L.simple = reinterpret_cast<int*>(take(4));
    L.ipb = reinterpret_cast<uint16_t*>(take(4));
    L.ip = a.ip;
    L.og = a.og;
    return L;
  };
  for (int64_t k = 0; k < a.n_inst; ++k) {
    const int w = (int)(k % S);
    cfb::LargeArgs L = workspace(w);
    const size_t base = (size_t)k * M;
    L.k = k;
    L.base = base;
    L.fmin = a.fmin + base;
    L.fmax = a.fmax + base;
    L.kappa = a.kappa + base;
    L.ru = a.ru + base;
    L.pu = a.pu + base;
    L.arr = a.arr + base;
    L.dl = a.dl + base;
    L.rd = a.rd ? a.rd + base : nullptr;
    L.pd = a.pd ? a.pd + base : nullptr;
    L.l_ip_dev = a.l_ip ? a.l_ip + k : nullptr;  // read on the device
    e = cfb::launch_large(L, ctx->lst[w]);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "large-instance launch");
    ctx->launches += 6;
  }
  for (int w = 0; w < S; ++w) {
    e = cudaEventRecord(ctx->lev[w], ctx->lst[w]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ctx->lev[w], 0);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "large-path join");
  }
  return COINFER_OK;
}

enum class Mode { Solve, Fixed };

int run(coinfer_ctx* ctx, const coinfer_profile* prof, const coinfer_users* users,
        const double* deadline, const int32_t* bvec, const coinfer_ipssa_out* ip_in,
        const coinfer_og_out* og_in, Mode mode) {
  if (!ctx) return COINFER_E_ARG;
  ctx->err.clear();
  if (!users) return fail(ctx, COINFER_E_ARG, "users: null");
  int rc = check_profile(ctx, prof);
  if (rc != COINFER_OK) return rc;
  if (users->n_inst < 0 || users->M < 0) return fail(ctx, COINFER_E_ARG, "users: negative size");
  if (users->mem != COINFER_MEM_HOST && users->mem != COINFER_MEM_DEVICE)
    return fail(ctx, COINFER_E_ARG, "users: bad mem kind");
  if (users->M > 0 && users->n_inst > 0 &&
      (!users->f_min || !users->f_max || !users->kappa || !users->rate_up || !users->power_up ||
       !users->arrival || !users->deadline))
    return fail(ctx, COINFER_E_ARG, "users: null input array");
  if (mode == Mode::Fixed && users->n_inst > 0 && !bvec)
    return fail(ctx, COINFER_E_ARG, "fixed: null batch-bound array");
  if (users->n_inst == 0) return COINFER_OK;

  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  rc = upload_latency(ctx, prof);
  if (rc != COINFER_OK) return rc;

  const size_t K = (size_t)users->n_inst, M = (size_t)users->M, N = (size_t)prof->N;
  cfb::SmallArgs a;
  std::memset(&a, 0, sizeof a);
  a.P = make_const(prof);
  a.lat = ctx->d_lat;
  a.n_inst = users->n_inst;
  a.M = users->M;
  a.fmin = users->f_min;
  a.fmax = users->f_max;
  a.kappa = users->kappa;
  a.ru = users->rate_up;
  a.pu = users->power_up;
  a.arr = users->arrival;
  a.dl = users->deadline;
  a.rd = users->rate_down;
  a.pd = users->power_down;
  a.l_ip = deadline;
  a.ctr = ctx->ctr;
  a.do_ip = ip_in != nullptr;
  a.do_og = og_in != nullptr;
  if (ip_in) a.ip = *ip_in;
  if (og_in) a.og = *og_in;
  const int32_t* bdev = bvec;

  auto launch = [&](const cfb::SmallArgs& args, const int32_t* bd, size_t Kc, cudaStream_t st) {
    const int grid = (int)(Kc < (size_t)(1u << 30) ? Kc : (size_t)(1u << 30));
    if (mode == Mode::Fixed) return cfb::launch_fixed(args, bd, grid, st);
    // Many instances: 4 warps per CTA and several CTAs per SM.  Fewer: 8
    // warps per CTA to spread each instance's chains wider; a handful (SMs
    // would idle anyway): 16 warps per instance (measured best of 8/16/32 at
    // M = 50..176; COINFER_WIDE overrides, for experiments).
    // Many instances: large instances (fewer CTAs fit the shared memory)
    // get more warps per CTA, about 36 / (CTAs per SM), 4..16 -- measured
    // best at M = 50 (8 CTAs: 4 warps), 75 (5: 7), 100 (3: 12), 150 (1: 16).
    // Many small instances: the pipelined kernel (two instances per CTA,
    // G-phase warps apart from front/tail warps) when two buffers fit.
    static const char* pipe_env = std::getenv("COINFER_PIPE");
    const bool pipe_force = pipe_env && pipe_env[0] == '1';  // testing aid: whenever it fits
    if (!args.ctr && Kc >= 2048 &&
        (pipe_force ? cfb::pipe_fits((int)M, (int)N) : cfb::pipe_preferred((int)M, (int)N)) &&
        !(pipe_env && pipe_env[0] == '0')) {
      if (!ctx->claim) {
        cudaError_t e = cudaMalloc(&ctx->claim, sizeof(unsigned long long) * coinfer_ctx::kClaims);
        if (e != cudaSuccess) return e;
      }
      cfb::SmallArgs ap = args;
      ap.claim = ctx->claim + (ctx->claim_next++ % coinfer_ctx::kClaims);
      {  // its G tables live in global memory (L2)
        const int gs = st == ctx->pipe[1] ? 2 : st == ctx->pipe[0] ? 1 : 0;
        const size_t need = cfb::pipe_gg_doubles((int)M, (int)N);
        if (need > ctx->gg_cap[gs]) {
          cudaStreamSynchronize(st);
          if (ctx->gg[gs]) cudaFree(ctx->gg[gs]);
          ctx->gg[gs] = nullptr;
          ctx->gg_cap[gs] = 0;
          cudaError_t e = cudaMalloc(&ctx->gg[gs], need * sizeof(double));
          if (e != cudaSuccess) return e;
          ctx->gg_cap[gs] = need;
        }
        ap.gg = ctx->gg[gs];
      }
      return cfb::launch_pipe(ap, st);
    }
    static const int wide = std::getenv("COINFER_WIDE") ? std::atoi(std::getenv("COINFER_WIDE")) : 512;
    static const int many = std::getenv("COINFER_THREADS") ? std::atoi(std::getenv("COINFER_THREADS")) : 0;
    int threads = Kc >= 148 ? 256 : wide;
    if (Kc >= 1024) {
      const int smem = cfb::small_smem_bytes((int)M, (int)N, 4);
      const int ctas = std::max(1, std::min(8, (227 * 1024) / std::max(smem, 1)));
      threads = many > 0 ? many : 32 * std::max(4, std::min(16, 36 / ctas));
    }
    return cfb::launch_small(args, threads, grid, st);
  };
  static const bool force_large = std::getenv("COINFER_FORCE_LARGE") != nullptr;  // testing aid
  const bool large = M > (size_t)kSmallMaxM || cfb::small_smem_bytes((int)M, (int)N, 8) > 227 * 1024 ||
                     (force_large && mode != Mode::Fixed && M > 0);
  if (large && mode == Mode::Fixed &&
      (size_t)cfb::fixed_smem_bytes((int)M, (int)N) > 227 * 1024)
    return fail(ctx, COINFER_E_UNSUPPORTED, "fixed_batch: instance does not fit in shared memory");
  if (large && mode != Mode::Fixed) {
    // solve_large.cu, instances spread over the large-path streams; host
    // batches are staged whole (the workspaces are per worker stream, so
    // successive calls order themselves on those streams)
    if (users->mem == COINFER_MEM_DEVICE) return run_large_device(ctx, a, ctx->stream);
    Stager st{ctx};
    plan_in(st, a.fmin, K * M);
    plan_in(st, a.fmax, K * M);
    plan_in(st, a.kappa, K * M);
    plan_in(st, a.ru, K * M);
    plan_in(st, a.pu, K * M);
    plan_in(st, a.arr, K * M);
    plan_in(st, a.dl, K * M);
    plan_in(st, a.rd, K * M);
    plan_in(st, a.pd, K * M);
    plan_in(st, a.l_ip, K);
    if (ip_in) plan_ip_out(st, a.ip, K, M, N);
    if (og_in) plan_og_out(st, a.og, K, M, N);
    rc = ensure_ws(ctx, 0, st.used);
    if (rc != COINFER_OK) return rc;
    unsigned char* b = ctx->ws2[0];
    cudaStream_t sp = ctx->pipe[0];
    patch(b, a.fmin);
    patch(b, a.fmax);
    patch(b, a.kappa);
    patch(b, a.ru);
    patch(b, a.pu);
    patch(b, a.arr);
    patch(b, a.dl);
    patch(b, a.rd);
    patch(b, a.pd);
    patch(b, a.l_ip);
    if (ip_in) patch_ip_out(b, a.ip);
    if (og_in) patch_og_out(b, a.og);
    for (const auto& x : st.in) {
      e = cudaMemcpyAsync(b + x.off, x.host, x.bytes, cudaMemcpyHostToDevice, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D inputs");
    }
    rc = run_large_device(ctx, a, sp);
    if (rc != COINFER_OK) return rc;
    for (const auto& x : st.back) {
      e = cudaMemcpyAsync(x.host, b + x.off, x.bytes, cudaMemcpyDeviceToHost, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H outputs");
    }
    e = cudaStreamSynchronize(sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "solve");
    return COINFER_OK;
  }

  if (users->mem == COINFER_MEM_DEVICE) {
    e = launch(a, bdev, K, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
    ctx->launches += 1;
    return COINFER_OK;
  }

  // Host memory: chunk the batch and alternate two streams, so the H2D copy
  // of chunk c+1 and the D2H copy of chunk c-1 overlap the solve of chunk c.
  size_t nch = K / CFB_E2E_MINCHUNK < CFB_E2E_CHUNKS ? K / CFB_E2E_MINCHUNK : CFB_E2E_CHUNKS;
  if (K < 4 * (size_t)CFB_E2E_MINCHUNK || nch < 1) nch = 1;  // small batches: one chunk
  for (size_t c = 0; c < nch; ++c) {
    const size_t k0 = K * c / nch, k1 = K * (c + 1) / nch, Kc = k1 - k0;
    const int slot = (int)(c & 1);
    cfb::SmallArgs ac = a;
    ac.n_inst = (int64_t)Kc;
    auto off = [&](auto*& p, size_t per) {
      if (p) p += k0 * per;
    };
    off(ac.fmin, M);
    off(ac.fmax, M);
    off(ac.kappa, M);
    off(ac.ru, M);
    off(ac.pu, M);
    off(ac.arr, M);
    off(ac.dl, M);
    off(ac.rd, M);
    off(ac.pd, M);
    off(ac.l_ip, 1);
    const int32_t* bc = bdev;
    off(bc, 1);
    if (ip_in) {
      off(ac.ip.status, 1);
      off(ac.ip.batch_bound, 1);
      off(ac.ip.pipeline_feasible, 1);
      off(ac.ip.energy, 1);
      off(ac.ip.split, M);
      off(ac.ip.freq, M);
      off(ac.ip.user_energy, M);
      off(ac.ip.batch_size, N);
    }
    if (og_in) {
      off(ac.og.status, 1);
      off(ac.og.fallback, 1);
      off(ac.og.energy, 1);
      off(ac.og.n_groups, 1);
      off(ac.og.order, M);
      off(ac.og.group_of_user, M);
      off(ac.og.split, M);
      off(ac.og.freq, M);
      off(ac.og.user_energy, M);
      off(ac.og.group_lo, M);
      off(ac.og.group_size, M);
      off(ac.og.group_b, M);
      off(ac.og.group_deadline, M);
      off(ac.og.group_energy, M);
      off(ac.og.group_batch_size, M * N);
    }
    Stager st{ctx};
    plan_in(st, ac.fmin, Kc * M);
    plan_in(st, ac.fmax, Kc * M);
    plan_in(st, ac.kappa, Kc * M);
    plan_in(st, ac.ru, Kc * M);
    plan_in(st, ac.pu, Kc * M);
    plan_in(st, ac.arr, Kc * M);
    plan_in(st, ac.dl, Kc * M);
    plan_in(st, ac.rd, Kc * M);
    plan_in(st, ac.pd, Kc * M);
    plan_in(st, ac.l_ip, Kc);
    plan_in(st, bc, Kc);
    if (ip_in) plan_ip_out(st, ac.ip, Kc, M, N);
    if (og_in) plan_og_out(st, ac.og, Kc, M, N);
    rc = ensure_ws(ctx, slot, st.used);
    if (rc != COINFER_OK) return rc;
    unsigned char* b = ctx->ws2[slot];
    cudaStream_t sp = ctx->pipe[slot];
    patch(b, ac.fmin);
    patch(b, ac.fmax);
    patch(b, ac.kappa);
    patch(b, ac.ru);
    patch(b, ac.pu);
    patch(b, ac.arr);
    patch(b, ac.dl);
    patch(b, ac.rd);
    patch(b, ac.pd);
    patch(b, ac.l_ip);
    patch(b, bc);
    if (ip_in) patch_ip_out(b, ac.ip);
    if (og_in) patch_og_out(b, ac.og);
    for (const auto& x : st.in) {
      e = cudaMemcpyAsync(b + x.off, x.host, x.bytes, cudaMemcpyHostToDevice, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D inputs");
    }
    e = launch(ac, bc, Kc, sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
    ctx->launches += 1;
    for (const auto& x : st.back) {
      e = cudaMemcpyAsync(x.host, b + x.off, x.bytes, cudaMemcpyDeviceToHost, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H outputs");
    }
  }
  for (int slot = 0; slot < 2; ++slot)
    if (ctx->pipe[slot]) {
      e = cudaStreamSynchronize(ctx->pipe[slot]);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "solve");
    }
  return COINFER_OK;
}

// ------------------------------------------------ schedule / baseline calls

int ensure_aux(coinfer_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->aux_cap) return COINFER_OK;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->aux) cudaFree(ctx->aux);
  ctx->aux = nullptr;
  ctx->aux_cap = 0;
  cudaError_t e = cudaMalloc(&ctx->aux, bytes);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(aux workspace)");
  ctx->aux_cap = bytes;
  return COINFER_OK;
}

template <class T>
void plan_in_mut(Stager& s, T*& p, size_t count) {
  const T* q = p;
  plan_in(s, q, count);
  p = const_cast<T*>(q);
}

enum class Aux { MatIp, MatOg, Baseline };

int check_users(coinfer_ctx* ctx, const coinfer_users* users) {
  if (!users) return fail(ctx, COINFER_E_ARG, "users: null");
  if (users->n_inst < 0 || users->M < 0) return fail(ctx, COINFER_E_ARG, "users: negative size");
  if (users->mem != COINFER_MEM_HOST && users->mem != COINFER_MEM_DEVICE)
    return fail(ctx, COINFER_E_ARG, "users: bad mem kind");
  if (users->M > 0 && users->n_inst > 0 &&
      (!users->f_min || !users->f_max || !users->kappa || !users->rate_up || !users->power_up ||
       !users->arrival || !users->deadline))
    return fail(ctx, COINFER_E_ARG, "users: null input array");
  return COINFER_OK;
}

bool sched_complete(const coinfer_schedule_out* o) {
  return o && o->x && o->n_batches && o->batch_start && o->completion && o->freq;
}

// Shared driver of coinfer_{ipssa,og}_schedule and coinfer_baseline_batch:
// host batches are staged whole through ctx->aux; device batches run in place.
int run_aux(coinfer_ctx* ctx, const coinfer_profile* prof, const coinfer_users* users,
            const double* deadline, Aux kind, int mode, coinfer_ipssa_out* ip,
            const coinfer_og_out* og, coinfer_schedule_out* sch) {
  if (!ctx) return COINFER_E_ARG;
  ctx->err.clear();
  int rc = check_users(ctx, users);
  if (rc != COINFER_OK) return rc;
  rc = check_profile(ctx, prof);
  if (rc != COINFER_OK) return rc;
  if (users->n_inst == 0) return COINFER_OK;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");

  const size_t K = (size_t)users->n_inst, M = (size_t)users->M, N = (size_t)prof->N;
  const bool host = users->mem == COINFER_MEM_HOST;
  cfb::AuxArgs a;
  std::memset(&a, 0, sizeof a);
  a.P = make_const(prof);
  a.n_inst = users->n_inst;
  a.M = users->M;
  a.mode = mode;
  a.fmin = users->f_min;
  a.fmax = users->f_max;
  a.kappa = users->kappa;
  a.ru = users->rate_up;
  a.pu = users->power_up;
  a.arr = users->arrival;
  a.dl = users->deadline;
  a.rd = users->rate_down;
  a.pd = users->power_down;
  a.l_ip = deadline;
  if (kind == Aux::MatIp) {  // only the decision arrays the materialiser reads
    a.ip.status = ip->status;
    a.ip.batch_bound = ip->batch_bound;
    a.ip.pipeline_feasible = ip->pipeline_feasible;
    a.ip.split = ip->split;
    a.ip.freq = ip->freq;
    a.ip.batch_size = ip->batch_size;
  } else if (kind == Aux::MatOg) {
    a.og.status = og->status;
    a.og.fallback = og->fallback;
    a.og.n_groups = og->n_groups;
    a.og.order = og->order;
    a.og.split = og->split;
    a.og.freq = og->freq;
    a.og.group_lo = og->group_lo;
    a.og.group_size = og->group_size;
    a.og.group_b = og->group_b;
    a.og.group_deadline = og->group_deadline;
    a.og.group_batch_size = og->group_batch_size;
  } else {
    a.ip = *ip;
  }
  if (sch) a.sch = *sch;

  Stager st{ctx};
  if (host) {
    plan_in(st, a.fmin, K * M);
    plan_in(st, a.fmax, K * M);
    plan_in(st, a.kappa, K * M);
    plan_in(st, a.ru, K * M);
    plan_in(st, a.pu, K * M);
    plan_in(st, a.arr, K * M);
    plan_in(st, a.dl, K * M);
    plan_in(st, a.rd, K * M);
    plan_in(st, a.pd, K * M);
    plan_in(st, a.l_ip, K);
    if (kind == Aux::MatIp) {
      plan_in_mut(st, a.ip.status, K);
      plan_in_mut(st, a.ip.batch_bound, K);
      plan_in_mut(st, a.ip.pipeline_feasible, K);
      plan_in_mut(st, a.ip.split, K * M);
      plan_in_mut(st, a.ip.freq, K * M);
      plan_in_mut(st, a.ip.batch_size, K * N);
    } else if (kind == Aux::MatOg) {
      plan_in_mut(st, a.og.status, K);
      plan_in_mut(st, a.og.fallback, K);
      plan_in_mut(st, a.og.n_groups, K);
      plan_in_mut(st, a.og.order, K * M);
      plan_in_mut(st, a.og.split, K * M);
      plan_in_mut(st, a.og.freq, K * M);
      plan_in_mut(st, a.og.group_lo, K * M);
      plan_in_mut(st, a.og.group_size, K * M);
      plan_in_mut(st, a.og.group_b, K * M);
      plan_in_mut(st, a.og.group_deadline, K * M);
      plan_in_mut(st, a.og.group_batch_size, K * M * N);
    } else {
      plan_ip_out(st, a.ip, K, M, N);
    }
    if (sch) {
      plan_out(st, a.sch.x, K * M * N);
      plan_out(st, a.sch.n_batches, K);
      plan_out(st, a.sch.batch_start, K * M * N);
      plan_out(st, a.sch.completion, K * M * (N + 1));
      plan_out(st, a.sch.freq, K * M);
    }
  }
  const size_t nlat = N * (size_t)prof->b_max;
  const size_t lat_off = st.reserve(nlat * 8);
  const int grid = cfb::aux_grid(users->n_inst);
  a.scratch_per_thread = (cfb::aux_scratch_bytes((int)M, (int)N) + 255) & ~size_t(255);
  const size_t scr_off = st.reserve((size_t)grid * 128 * a.scratch_per_thread);
  const bool np = kind == Aux::Baseline && mode == COINFER_BASELINE_IPSSA_NP;
  size_t f_st = 0, f_bb = 0, f_pf = 0, f_sp = 0, f_fr = 0, f_bs = 0;
  if (np) {
    f_st = st.reserve(4 * K);
    f_bb = st.reserve(4 * K);
    f_pf = st.reserve(K);
    f_sp = st.reserve(K * M);
    f_fr = st.reserve(8 * K * M);
    f_bs = st.reserve(4 * K);
  }
  rc = ensure_aux(ctx, st.used);
  if (rc != COINFER_OK) return rc;
  unsigned char* b = ctx->aux;
  cudaStream_t sp = ctx->stream;
  if (host) {
    patch(b, a.fmin);
    patch(b, a.fmax);
    patch(b, a.kappa);
    patch(b, a.ru);
    patch(b, a.pu);
    patch(b, a.arr);
    patch(b, a.dl);
    patch(b, a.rd);
    patch(b, a.pd);
    patch(b, a.l_ip);
    patch_ip_out(b, a.ip);
    patch_og_out(b, a.og);
    if (sch) {
      patch(b, a.sch.x);
      patch(b, a.sch.n_batches);
      patch(b, a.sch.batch_start);
      patch(b, a.sch.completion);
      patch(b, a.sch.freq);
    }
    for (const auto& x : st.in) {
      e = cudaMemcpyAsync(b + x.off, x.host, x.bytes, cudaMemcpyHostToDevice, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D inputs");
    }
  }
  a.lat = reinterpret_cast<const double*>(b + lat_off);
  e = cudaMemcpyAsync(b + lat_off, prof->latency, nlat * 8, cudaMemcpyHostToDevice, sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D latency");
  a.scratch = b + scr_off;

  if (np) {
    // the collapsed one-sub-task profile (ipssa_np_solve:563-569): work =
    // total_work, bits = {B_0, B_N}, F(b) = sum_latency(b) (a left fold)
    std::vector<double> fw(1, a.P.prefix[N]), fb{prof->data_bits[0], prof->data_bits[N]};
    std::vector<double> fl((size_t)prof->b_max);
    for (int bb = 0; bb < prof->b_max; ++bb) {
      double t = 0.0;
      for (size_t n = 0; n < N; ++n) t += prof->latency[n * prof->b_max + bb];
      fl[bb] = t;
    }
    coinfer_profile flat{1, prof->b_max, fw.data(), fb.data(), fl.data()};
    coinfer_users du = *users;
    du.mem = COINFER_MEM_DEVICE;
    du.f_min = a.fmin;
    du.f_max = a.fmax;
    du.kappa = a.kappa;
    du.rate_up = a.ru;
    du.power_up = a.pu;
    du.arrival = a.arr;
    du.deadline = a.dl;
    du.rate_down = a.rd;
    du.power_down = a.pd;
    std::memset(&a.flat, 0, sizeof a.flat);
    a.flat.status = reinterpret_cast<int32_t*>(b + f_st);
    a.flat.batch_bound = reinterpret_cast<int32_t*>(b + f_bb);
    a.flat.pipeline_feasible = b + f_pf;
    a.flat.split = b + f_sp;
    a.flat.freq = reinterpret_cast<double*>(b + f_fr);
    a.flat.batch_size = reinterpret_cast<int32_t*>(b + f_bs);
    rc = run(ctx, &flat, &du, nullptr, nullptr, &a.flat, nullptr, Mode::Solve);
    if (rc != COINFER_OK) return rc;
  }
  if (kind == Aux::MatIp)
    e = cfb::launch_materialize_ip(a, sp);
  else if (kind == Aux::MatOg)
    e = cfb::launch_materialize_og(a, sp);
  else
    e = cfb::launch_baseline(a, sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
  ctx->launches += 1;
  if (host) {
    for (const auto& x : st.back) {
      e = cudaMemcpyAsync(x.host, b + x.off, x.bytes, cudaMemcpyDeviceToHost, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H outputs");
    }
  }
  // the latency table was copied from pageable host memory the caller owns;
  // host calls are synchronous anyway
  e = cudaStreamSynchronize(sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "aux kernel");
  return COINFER_OK;
}

}  // namespace

extern "C" {

int coinfer_abi_version(void) { return COINFER_ABI_VERSION; }

coinfer_ctx* coinfer_ctx_create(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  coinfer_ctx* ctx = new coinfer_ctx;
  ctx->device = device;
  if (cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return nullptr;
  }
  ctx->stream = ctx->own;
  return ctx;
}

void coinfer_ctx_destroy(coinfer_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->d_lat) cudaFree(ctx->d_lat);
  for (int w = 0; w < coinfer_ctx::kLargeStreams; ++w) {
    if (ctx->lst[w]) cudaStreamSynchronize(ctx->lst[w]);
    if (ctx->big[w]) cudaFree(ctx->big[w]);
    if (ctx->lev[w]) cudaEventDestroy(ctx->lev[w]);
    if (ctx->lst[w]) cudaStreamDestroy(ctx->lst[w]);
  }
  if (ctx->lstart) cudaEventDestroy(ctx->lstart);
  if (ctx->aux) cudaFree(ctx->aux);
  if (ctx->claim) cudaFree(ctx->claim);
  for (int i = 0; i < 3; ++i)
    if (ctx->gg[i]) cudaFree(ctx->gg[i]);
  for (int i = 0; i < 2; ++i) {
    if (ctx->pipe[i]) cudaStreamSynchronize(ctx->pipe[i]);
    if (ctx->ws2[i]) cudaFree(ctx->ws2[i]);
    if (ctx->pipe[i]) cudaStreamDestroy(ctx->pipe[i]);
  }
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
}

int coinfer_ctx_set_stream(coinfer_ctx* ctx, void* stream) {
  if (!ctx) return COINFER_E_ARG;
  ctx->stream = static_cast<cudaStream_t>(stream);
  return COINFER_OK;
}

int coinfer_ctx_reset_stream(coinfer_ctx* ctx) {
  if (!ctx) return COINFER_E_ARG;
  ctx->stream = ctx->own;
  return COINFER_OK;
}

int coinfer_ctx_synchronize(coinfer_ctx* ctx) {
  if (!ctx) return COINFER_E_ARG;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "synchronize");
  return COINFER_OK;
}

const char* coinfer_last_error(const coinfer_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t coinfer_ctx_launch_count(const coinfer_ctx* ctx) { return ctx ? ctx->launches : 0; }

int coinfer_probe_fp64(coinfer_ctx* ctx, double* lane_ops_per_s) {
  if (!ctx || !lane_ops_per_s) return COINFER_E_ARG;
  cudaSetDevice(ctx->device);
  cudaError_t e = cfb::probe_fp64(ctx->stream, lane_ops_per_s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "probe_fp64");
  return COINFER_OK;
}

const char* coinfer_status_message(int32_t status, const char* solver) {
  const std::string s = solver ? solver : "";
  switch (status) {
    case COINFER_ST_OK: return "";
    case COINFER_ST_INFEASIBLE:
      if (s == "og") return "baseline: user cannot meet the deadline locally";
      if (s == "fixed") return "fixed_batch_schedule: user cannot meet the deadline";
      if (s == "lc") return "baseline: user cannot meet the deadline locally";
      if (s == "ps" || s == "fifo") return "baseline: user cannot meet the deadline";
      return "ip_ssa: no batch bound admits every user";
    case COINFER_ST_BAD_FREQ: return "scenario: bad frequency range";
    case COINFER_ST_NEG_KAPPA: return "scenario: negative kappa";
    case COINFER_ST_BAD_RATE: return "scenario: rates must be positive";
    case COINFER_ST_NEG_POWER: return "scenario: negative link power";
    case COINFER_ST_NEG_ARRIVAL: return "scenario: negative arrival";
    case COINFER_ST_EARLY_DEADLINE: return "scenario: deadline before arrival";
    case COINFER_ST_SHORT_TABLE: return "scenario: latency table shorter than user count";
    case COINFER_ST_ZERO_BOUND: return "batch_start_times: b must be >= 1";
    case COINFER_ST_BOUND_PAST_TABLE: return "edge_batch_latency: batch size beyond table";
    case COINFER_ST_NOT_RELEASED: return "online: users must be released at time zero";
    case COINFER_ST_FLOOR_ABOVE_LLOW: return "online: l_low below a user's all-local floor";
    case COINFER_ST_SLIPPED: return "online: task slipped below its local floor";
    case COINFER_ST_BAD_BATCH_ID: return "schedule: batch id beyond start-time table";
    case COINFER_ST_NONPOS_FREQ: return "local_latency: f must be positive";
    case COINFER_ST_NO_DEADLINE: return "sample_scenario: cannot draw a feasible deadline";
    case COINFER_ST_TOO_LARGE:
      if (s == "structured") return "oracle_structured: instance too large to enumerate";
      if (s == "contiguous") return "oracle_grouping_contiguous: instance too large to enumerate";
      return "oracle_grouping: instance too large to enumerate";
  }
  return "unknown status";
}

int coinfer_ipssa_batch(coinfer_ctx* ctx, const coinfer_profile* profile, const coinfer_users* users,
                        const double* deadline, coinfer_ipssa_out* out) {
  if (!out) return fail(ctx, COINFER_E_ARG, "ipssa: null output");
  return run(ctx, profile, users, deadline, nullptr, out, nullptr, Mode::Solve);
}

int coinfer_fixed_batch(coinfer_ctx* ctx, const coinfer_profile* profile, const coinfer_users* users,
                        const double* deadline, const int32_t* b, coinfer_ipssa_out* out) {
  if (!out) return fail(ctx, COINFER_E_ARG, "fixed: null output");
  return run(ctx, profile, users, deadline, b, out, nullptr, Mode::Fixed);
}

int coinfer_og_batch(coinfer_ctx* ctx, const coinfer_profile* profile, const coinfer_users* users,
                     coinfer_og_out* out) {
  if (!out) return fail(ctx, COINFER_E_ARG, "og: null output");
  return run(ctx, profile, users, nullptr, nullptr, nullptr, out, Mode::Solve);
}

int coinfer_online_run(coinfer_ctx* ctx, const coinfer_profile* profile,
                       const coinfer_users* sc, const coinfer_online_cfg* cfg,
                       const uint64_t* seeds, int64_t n_ep, coinfer_online_out* out) {
  if (!ctx) return COINFER_E_ARG;
  ctx->err.clear();
  if (!sc || !cfg || !out) return fail(ctx, COINFER_E_ARG, "online: null argument");
  int rc = check_profile(ctx, profile);
  if (rc != COINFER_OK) return rc;
  // ArrivalModel::check, OnlineEnv ctor, run_episode (online_sim.hpp:33-38,81,340)
  if (cfg->l_low <= 0.0 || cfg->l_high < cfg->l_low)
    return fail(ctx, COINFER_E_ARG, "arrivals: bad deadline range");
  if (cfg->arrival == COINFER_ARRIVAL_BERNOULLI && (cfg->p_arrive < 0.0 || cfg->p_arrive > 1.0))
    return fail(ctx, COINFER_E_ARG, "arrivals: p_arrive must lie in [0, 1]");
  if (cfg->arrival != COINFER_ARRIVAL_BERNOULLI && cfg->arrival != COINFER_ARRIVAL_IMMEDIATE)
    return fail(ctx, COINFER_E_ARG, "arrivals: unknown kind");
  if (!(cfg->slot > 0.0)) return fail(ctx, COINFER_E_ARG, "online: slot must be positive");
  if (cfg->horizon <= 0) return fail(ctx, COINFER_E_ARG, "run_episode: empty horizon");
  if (cfg->solver != COINFER_SOLVER_OG && cfg->solver != COINFER_SOLVER_IPSSA)
    return fail(ctx, COINFER_E_ARG, "online: unknown solver");
  if (cfg->policy != COINFER_POLICY_TW && cfg->policy != COINFER_POLICY_LOCAL)
    return fail(ctx, COINFER_E_ARG, "online: unknown policy");
  if (sc->n_inst <= 0 || sc->M <= 0) return fail(ctx, COINFER_E_ARG, "online: need a scenario with users");
  if (sc->M > kSmallMaxM) return fail(ctx, COINFER_E_UNSUPPORTED, "online: M above the solver limit");
  if (n_ep <= 0) return COINFER_OK;
  if (!seeds) return fail(ctx, COINFER_E_ARG, "online: null seeds");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  rc = upload_latency(ctx, profile);
  if (rc != COINFER_OK) return rc;

  const size_t S = (size_t)sc->n_inst, M = (size_t)sc->M, N = (size_t)profile->N, E = (size_t)n_ep;
  const size_t T = out->n_trace > 0 ? (size_t)out->n_trace * (size_t)cfg->horizon : 0;
  cfb::OnlineArgs a;
  std::memset(&a, 0, sizeof a);
  a.solve.P = make_const(profile);
  a.solve.lat = ctx->d_lat;
  a.solve.n_inst = 1;
  a.solve.do_og = cfg->solver == COINFER_SOLVER_OG;
  a.solve.do_ip = !a.solve.do_og;
  a.M = sc->M;
  a.n_scen = sc->n_inst;
  a.fmin = sc->f_min;
  a.fmax = sc->f_max;
  a.kappa = sc->kappa;
  a.ru = sc->rate_up;
  a.pu = sc->power_up;
  a.arr = sc->arrival;
  a.dl = sc->deadline;
  a.rd = sc->rate_down;
  a.pd = sc->power_down;
  a.immediate = cfg->arrival == COINFER_ARRIVAL_IMMEDIATE;
  a.p_arrive = cfg->p_arrive;
  a.l_low = cfg->l_low;
  a.l_high = cfg->l_high;
  a.slot = cfg->slot;
  a.threshold = cfg->threshold;
  a.policy = cfg->policy;
  a.window = cfg->window;
  a.horizon = cfg->horizon;
  a.n_ep = n_ep;
  a.seeds = reinterpret_cast<const unsigned long long*>(seeds);
  a.status = out->status;
  a.totals = out->totals;
  a.counts = reinterpret_cast<long long*>(out->counts);
  a.n_trace = out->n_trace;
  a.tr_reward = out->trace_reward;
  a.tr_energy = out->trace_energy;
  a.tr_pending = out->trace_pending;
  a.tr_busy = out->trace_edge_busy;
  a.tr_action = out->trace_action;
  a.tr_forced = out->trace_forced;
  a.fin_state = out->final_state;
  a.draws = reinterpret_cast<long long*>(out->draws);

  const bool host = sc->mem == COINFER_MEM_HOST;
  Stager st{ctx};
  if (host) {
    plan_in(st, a.fmin, S * M);
    plan_in(st, a.fmax, S * M);
    plan_in(st, a.kappa, S * M);
    plan_in(st, a.ru, S * M);
    plan_in(st, a.pu, S * M);
    plan_in(st, a.arr, S * M);
    plan_in(st, a.dl, S * M);
    plan_in(st, a.rd, S * M);
    plan_in(st, a.pd, S * M);
    plan_in(st, a.seeds, E);
    plan_out(st, a.status, E);
    plan_out(st, a.totals, 3 * E);
    plan_out(st, a.counts, 6 * E);
    plan_out(st, a.tr_reward, T);
    plan_out(st, a.tr_energy, T);
    plan_out(st, a.tr_pending, T);
    plan_out(st, a.tr_busy, T);
    plan_out(st, a.tr_action, T);
    plan_out(st, a.tr_forced, T);
    plan_out(st, a.fin_state, E * (2 * M + 1));
    plan_out(st, a.draws, E);
  }
  // per-episode solver scratch, device only
  int32_t* s_status = reinterpret_cast<int32_t*>(st.reserve(4 * E) + 1);
  double* s_energy = reinterpret_cast<double*>(st.reserve(8 * E) + 1);
  int32_t* s_ng = reinterpret_cast<int32_t*>(st.reserve(4 * E) + 1);
  double* s_gdl = reinterpret_cast<double*>(st.reserve(8 * E * M) + 1);
  int32_t* s_gbs = reinterpret_cast<int32_t*>(st.reserve(4 * E * M * N) + 1);
  int32_t* s_ibs = reinterpret_cast<int32_t*>(st.reserve(4 * E * N) + 1);
  rc = ensure_ws(ctx, 0, st.used);
  if (rc != COINFER_OK) return rc;
  unsigned char* b = ctx->ws2[0];
  cudaStream_t sp = host ? ctx->pipe[0] : ctx->stream;
  if (host) {
    patch(b, a.fmin);
    patch(b, a.fmax);
    patch(b, a.kappa);
    patch(b, a.ru);
    patch(b, a.pu);
    patch(b, a.arr);
    patch(b, a.dl);
    patch(b, a.rd);
    patch(b, a.pd);
    patch(b, a.seeds);
    patch(b, a.status);
    patch(b, a.totals);
    patch(b, a.counts);
    patch(b, a.tr_reward);
    patch(b, a.tr_energy);
    patch(b, a.tr_pending);
    patch(b, a.tr_busy);
    patch(b, a.tr_action);
    patch(b, a.tr_forced);
    patch(b, a.fin_state);
    patch(b, a.draws);
    for (const auto& x : st.in) {
      e = cudaMemcpyAsync(b + x.off, x.host, x.bytes, cudaMemcpyHostToDevice, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D online inputs");
    }
  }
  patch(b, s_status);
  patch(b, s_energy);
  patch(b, s_ng);
  patch(b, s_gdl);
  patch(b, s_gbs);
  patch(b, s_ibs);
  a.solve.og.status = s_status;
  a.solve.og.energy = s_energy;
  a.solve.og.n_groups = s_ng;
  a.solve.og.group_deadline = s_gdl;
  a.solve.og.group_batch_size = s_gbs;
  a.solve.ip.status = s_status;
  a.solve.ip.energy = s_energy;
  a.solve.ip.batch_size = s_ibs;
  const int grid = (int)(E < (size_t)(1u << 30) ? E : (size_t)(1u << 30));
  e = cfb::launch_online(a, grid, sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "online kernel launch");
  ctx->launches += 1;
  if (host) {
    for (const auto& x : st.back) {
      e = cudaMemcpyAsync(x.host, b + x.off, x.bytes, cudaMemcpyDeviceToHost, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H online outputs");
    }
    e = cudaStreamSynchronize(sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "online run");
  }
  return COINFER_OK;
}

int coinfer_sweep_batch(coinfer_ctx* ctx, const coinfer_profile* profile, const coinfer_users* users,
                        coinfer_ipssa_out* ipssa, coinfer_og_out* og) {
  if (!ipssa && !og) return fail(ctx, COINFER_E_ARG, "sweep: no output requested");
  return run(ctx, profile, users, nullptr, nullptr, ipssa, og, Mode::Solve);
}

int coinfer_count_work(coinfer_ctx* ctx, const coinfer_profile* profile, const coinfer_users* users,
                       coinfer_ipssa_out* ipssa, coinfer_og_out* og, uint64_t* counters) {
  if (!ctx) return COINFER_E_ARG;
  if (!counters) return fail(ctx, COINFER_E_ARG, "count_work: null counters");
  if (!ipssa && !og) return fail(ctx, COINFER_E_ARG, "count_work: no output requested");
  if (users && users->M > kSmallMaxM)
    return fail(ctx, COINFER_E_UNSUPPORTED, "count_work: the counting solve covers M <= 255");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  unsigned long long* d = nullptr;
  e = cudaMalloc(&d, sizeof(unsigned long long) * cfb::CTR_N);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc counters");
  e = cudaMemsetAsync(d, 0, sizeof(unsigned long long) * cfb::CTR_N, ctx->stream);
  int rc = e == cudaSuccess ? COINFER_OK : cuda_fail(ctx, e, "memset counters");
  if (rc == COINFER_OK) {
    ctx->ctr = d;
    rc = run(ctx, profile, users, nullptr, nullptr, ipssa, og, Mode::Solve);
    ctx->ctr = nullptr;
  }
  if (rc == COINFER_OK) {
    e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(counters, d, sizeof(unsigned long long) * cfb::CTR_N, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(ctx, e, "count_work");
  }
  cudaFree(d);
  return rc;
}

int coinfer_ipssa_schedule(coinfer_ctx* ctx, const coinfer_profile* profile,
                           const coinfer_users* users, const double* deadline,
                           const coinfer_ipssa_out* solved, coinfer_schedule_out* out) {
  if (!solved || !solved->status || !solved->batch_bound || !solved->pipeline_feasible ||
      !solved->split || !solved->freq || !solved->batch_size)
    return fail(ctx, COINFER_E_ARG, "ipssa_schedule: decision arrays missing");
  if (!sched_complete(out)) return fail(ctx, COINFER_E_ARG, "ipssa_schedule: schedule arrays missing");
  coinfer_ipssa_out in = *solved;
  return run_aux(ctx, profile, users, deadline, Aux::MatIp, 0, &in, nullptr, out);
}

int coinfer_og_schedule(coinfer_ctx* ctx, const coinfer_profile* profile, const coinfer_users* users,
                        const coinfer_og_out* solved, coinfer_schedule_out* out) {
  if (!solved || !solved->status || !solved->fallback || !solved->n_groups || !solved->order ||
      !solved->split || !solved->freq || !solved->group_lo || !solved->group_size ||
      !solved->group_b || !solved->group_deadline || !solved->group_batch_size)
    return fail(ctx, COINFER_E_ARG, "og_schedule: decision arrays missing");
  if (!sched_complete(out)) return fail(ctx, COINFER_E_ARG, "og_schedule: schedule arrays missing");
  return run_aux(ctx, profile, users, nullptr, Aux::MatOg, 0, nullptr, solved, out);
}

int coinfer_baseline_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                           const coinfer_users* users, int32_t mode, coinfer_ipssa_out* out,
                           coinfer_schedule_out* sched) {
  if (!out) return fail(ctx, COINFER_E_ARG, "baseline: null output");
  if (mode < COINFER_BASELINE_LC || mode > COINFER_BASELINE_IPSSA_NP)
    return fail(ctx, COINFER_E_ARG, "baseline: unknown mode");
  if (sched && !sched_complete(sched))
    return fail(ctx, COINFER_E_ARG, "baseline: schedule arrays missing");
  return run_aux(ctx, profile, users, nullptr, Aux::Baseline, mode, out, nullptr, sched);
}

int coinfer_validate_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                           const coinfer_users* users, const coinfer_schedule_out* sched,
                           double tol, int32_t* status, int32_t* counts, double* min_slack) {
  if (!ctx) return COINFER_E_ARG;
  ctx->err.clear();
  int rc = check_users(ctx, users);
  if (rc != COINFER_OK) return rc;
  if (!sched_complete(sched)) return fail(ctx, COINFER_E_ARG, "validate: schedule arrays missing");
  if (!status || !counts) return fail(ctx, COINFER_E_ARG, "validate: null output");
  rc = check_profile(ctx, profile);
  if (rc != COINFER_OK) return rc;
  if (users->n_inst == 0) return COINFER_OK;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  const size_t K = (size_t)users->n_inst, M = (size_t)users->M, N = (size_t)profile->N;
  const bool host = users->mem == COINFER_MEM_HOST;
  cfb::AuxArgs a;
  std::memset(&a, 0, sizeof a);
  a.P = make_const(profile);
  a.n_inst = users->n_inst;
  a.M = users->M;
  a.arr = users->arrival;
  a.dl = users->deadline;
  a.ru = users->rate_up;
  a.rd = users->rate_down;
  a.sch = *sched;
  a.tol = tol;
  a.vstatus = status;
  a.vcounts = counts;
  a.vslack = min_slack;
  Stager st{ctx};
  if (host) {
    plan_in(st, a.arr, K * M);
    plan_in(st, a.dl, K * M);
    plan_in(st, a.ru, K * M);
    plan_in(st, a.rd, K * M);
    plan_in_mut(st, a.sch.x, K * M * N);
    plan_in_mut(st, a.sch.n_batches, K);
    plan_in_mut(st, a.sch.batch_start, K * M * N);
    plan_in_mut(st, a.sch.completion, K * M * (N + 1));
    plan_in_mut(st, a.sch.freq, K * M);
    plan_out(st, a.vstatus, K);
    plan_out(st, a.vcounts, K * COINFER_N_CONSTRAINTS);
    plan_out(st, a.vslack, K);
  }
  const size_t nlat = N * (size_t)profile->b_max;
  const size_t lat_off = st.reserve(nlat * 8);
  const int grid = cfb::aux_grid(users->n_inst);
  a.scratch_per_thread = (cfb::aux_scratch_bytes((int)M, (int)N) + 255) & ~size_t(255);
  const size_t scr_off = st.reserve((size_t)grid * 128 * a.scratch_per_thread);
  rc = ensure_aux(ctx, st.used);
  if (rc != COINFER_OK) return rc;
  unsigned char* b = ctx->aux;
  cudaStream_t sp = ctx->stream;
  if (host) {
    patch(b, a.arr);
    patch(b, a.dl);
    patch(b, a.ru);
    patch(b, a.rd);
    patch(b, a.sch.x);
    patch(b, a.sch.n_batches);
    patch(b, a.sch.batch_start);
    patch(b, a.sch.completion);
    patch(b, a.sch.freq);
    patch(b, a.vstatus);
    patch(b, a.vcounts);
    patch(b, a.vslack);
    for (const auto& x : st.in) {
      e = cudaMemcpyAsync(b + x.off, x.host, x.bytes, cudaMemcpyHostToDevice, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D inputs");
    }
  }
  a.lat = reinterpret_cast<const double*>(b + lat_off);
  e = cudaMemcpyAsync(b + lat_off, profile->latency, nlat * 8, cudaMemcpyHostToDevice, sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D latency");
  a.scratch = b + scr_off;
  e = cfb::launch_validate(a, sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
  ctx->launches += 1;
  if (host) {
    for (const auto& x : st.back) {
      e = cudaMemcpyAsync(x.host, b + x.off, x.bytes, cudaMemcpyDeviceToHost, sp);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H outputs");
    }
  }
  e = cudaStreamSynchronize(sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "validate");
  return COINFER_OK;
}

void coinfer_sample_cfg_defaults(coinfer_sample_cfg* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->cell_radius = 100.0;
  c->bandwidth = 1e6;
  c->noise_dbm_hz = -174.0;
  c->tx_power = 0.05;
  c->uplink_power = 1.0;
  c->downlink_power = 1.0;
  c->edge_power = 300.0;
  c->edge_efficiency = 48.75;
  c->device_efficiency = 48.75;
  c->alpha = 1.0;
  c->shadow_sigma_db = 8.0;
  c->deadline_uniform = 0;
  c->deadline_low = 0.5;
  c->deadline_high = 0.5;
}

uint64_t coinfer_sub_seed(uint64_t root, uint64_t component, uint64_t index) {
  auto mix64 = [](uint64_t x) {  // splitmix64 finalizer (ddpg.hpp:272-277)
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d4a9749d57afbbull;
    return x ^ (x >> 31);
  };
  return mix64(mix64(root ^ (component * 0x9e3779b97f4a7c15ull)) + index);
}

int coinfer_sample_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                         const coinfer_sample_cfg* cfg, const uint64_t* seeds,
                         coinfer_users_mut* out, int32_t* status) {
  if (!ctx) return COINFER_E_ARG;
  ctx->err.clear();
  if (!cfg || !out) return fail(ctx, COINFER_E_ARG, "sample: null argument");
  const coinfer_sample_cfg& c = *cfg;
  // ScenarioConfig::check (scenario_gen.hpp:68-82)
  if (out->M <= 0) return fail(ctx, COINFER_E_ARG, "config: users must be positive");
  if (c.cell_radius <= 0.0 || c.bandwidth <= 0.0 || c.tx_power <= 0.0 || c.uplink_power < 0.0 ||
      c.downlink_power < 0.0 || c.edge_power <= 0.0 || c.edge_efficiency <= 0.0 ||
      c.device_efficiency <= 0.0 || c.alpha <= 0.0 || c.shadow_sigma_db < 0.0)
    return fail(ctx, COINFER_E_ARG, "config: physical quantities must be positive");
  if (!c.deadline_uniform) {
    if (c.deadline_low <= 0.0) return fail(ctx, COINFER_E_ARG, "config: deadline must be positive");
  } else if (c.deadline_low <= 0.0 || c.deadline_high < c.deadline_low) {
    return fail(ctx, COINFER_E_ARG, "config: bad deadline range");
  }
  int rc = check_profile(ctx, profile);
  if (rc != COINFER_OK) return fail(ctx, COINFER_E_ARG, ctx->err);
  if (profile->b_max < out->M)
    return fail(ctx, COINFER_E_ARG, "sample_scenario: latency table shorter than user count");
  const cfb::ProfileConst P = make_const(profile);
  const double total_work = P.prefix[P.N];
  const double fmax = 1.0 / c.alpha, floor_ = total_work / fmax;
  if (!c.deadline_uniform && c.deadline_low < floor_)
    return fail(ctx, COINFER_E_ARG, "sample_scenario: deadline below the all-local floor");
  if (c.deadline_uniform && c.deadline_high < floor_)
    return fail(ctx, COINFER_E_ARG, "sample_scenario: deadline range below the all-local floor");
  if (out->n_inst < 0) return fail(ctx, COINFER_E_ARG, "sample: negative size");
  if (out->n_inst == 0) return COINFER_OK;
  if (!seeds || !out->f_min || !out->f_max || !out->kappa || !out->rate_up || !out->power_up ||
      !out->arrival || !out->deadline)
    return fail(ctx, COINFER_E_ARG, "sample: null array");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  const size_t K = (size_t)out->n_inst, M = (size_t)out->M;
  cudaStream_t sp = ctx->stream;
  if (out->mem == COINFER_MEM_DEVICE) {
    e = cfb::launch_sample(c, total_work, out->M, out->n_inst,
                           reinterpret_cast<const unsigned long long*>(seeds), *out, status, sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
    ctx->launches += 1;
    return COINFER_OK;
  }
  Stager st{ctx};
  coinfer_users_mut d = *out;
  const uint64_t* sd = seeds;
  plan_in(st, sd, K);
  plan_out(st, d.f_min, K * M);
  plan_out(st, d.f_max, K * M);
  plan_out(st, d.kappa, K * M);
  plan_out(st, d.rate_up, K * M);
  plan_out(st, d.power_up, K * M);
  plan_out(st, d.arrival, K * M);
  plan_out(st, d.deadline, K * M);
  plan_out(st, d.rate_down, K * M);
  plan_out(st, d.power_down, K * M);
  plan_out(st, status, K);
  rc = ensure_aux(ctx, st.used);
  if (rc != COINFER_OK) return rc;
  unsigned char* b = ctx->aux;
  patch(b, sd);
  patch(b, d.f_min);
  patch(b, d.f_max);
  patch(b, d.kappa);
  patch(b, d.rate_up);
  patch(b, d.power_up);
  patch(b, d.arrival);
  patch(b, d.deadline);
  patch(b, d.rate_down);
  patch(b, d.power_down);
  patch(b, status);
  for (const auto& x : st.in) {
    e = cudaMemcpyAsync(b + x.off, x.host, x.bytes, cudaMemcpyHostToDevice, sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D seeds");
  }
  e = cfb::launch_sample(c, total_work, out->M, out->n_inst, reinterpret_cast<const unsigned long long*>(sd),
                         d, status, sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
  ctx->launches += 1;
  for (const auto& x : st.back) {
    e = cudaMemcpyAsync(x.host, b + x.off, x.bytes, cudaMemcpyDeviceToHost, sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H users");
  }
  e = cudaStreamSynchronize(sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "sample");
  return COINFER_OK;
}

namespace {
// Shared driver of the two oracle entry points (host batches staged whole).
int run_oracle(coinfer_ctx* ctx, const coinfer_profile* profile, const coinfer_users* users,
               cfb::OracleArgs a, bool structured) {
  if (!ctx) return COINFER_E_ARG;
  ctx->err.clear();
  int rc = check_users(ctx, users);
  if (rc != COINFER_OK) return rc;
  rc = check_profile(ctx, profile);
  if (rc != COINFER_OK) return rc;
  if (users->n_inst == 0) return COINFER_OK;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  rc = upload_latency(ctx, profile);
  if (rc != COINFER_OK) return rc;
  const size_t K = (size_t)users->n_inst, M = (size_t)users->M;
  a.P = make_const(profile);
  a.lat = ctx->d_lat;
  a.n_inst = users->n_inst;
  a.M = users->M;
  a.fmin = users->f_min;
  a.fmax = users->f_max;
  a.kappa = users->kappa;
  a.ru = users->rate_up;
  a.pu = users->power_up;
  a.arr = users->arrival;
  a.dl = users->deadline;
  cudaStream_t sp = ctx->stream;
  if (users->mem == COINFER_MEM_DEVICE) {
    e = structured ? cfb::launch_oracle_structured(a, sp) : cfb::launch_oracle_grouping(a, sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
    ctx->launches += 1;
    return COINFER_OK;
  }
  Stager st{ctx};
  plan_in(st, a.fmin, K * M);
  plan_in(st, a.fmax, K * M);
  plan_in(st, a.kappa, K * M);
  plan_in(st, a.ru, K * M);
  plan_in(st, a.pu, K * M);
  plan_in(st, a.arr, K * M);
  plan_in(st, a.dl, K * M);
  plan_in(st, a.deadline, K);
  plan_in(st, a.b, K);
  plan_out(st, a.status, K);
  plan_out(st, a.energy, K);
  plan_out(st, a.split, K * M);
  plan_out(st, a.fallback, K);
  plan_out(st, a.feasible, K);
  plan_out(st, a.n_groups, K);
  plan_out(st, a.group_of_user, K * M);
  rc = ensure_aux(ctx, st.used);
  if (rc != COINFER_OK) return rc;
  unsigned char* b = ctx->aux;
  patch(b, a.fmin);
  patch(b, a.fmax);
  patch(b, a.kappa);
  patch(b, a.ru);
  patch(b, a.pu);
  patch(b, a.arr);
  patch(b, a.dl);
  patch(b, a.deadline);
  patch(b, a.b);
  patch(b, a.status);
  patch(b, a.energy);
  patch(b, a.split);
  patch(b, a.fallback);
  patch(b, a.feasible);
  patch(b, a.n_groups);
  patch(b, a.group_of_user);
  for (const auto& x : st.in) {
    e = cudaMemcpyAsync(b + x.off, x.host, x.bytes, cudaMemcpyHostToDevice, sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D inputs");
  }
  e = structured ? cfb::launch_oracle_structured(a, sp) : cfb::launch_oracle_grouping(a, sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
  ctx->launches += 1;
  for (const auto& x : st.back) {
    e = cudaMemcpyAsync(x.host, b + x.off, x.bytes, cudaMemcpyDeviceToHost, sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H outputs");
  }
  e = cudaStreamSynchronize(sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "oracle");
  return COINFER_OK;
}
}  // namespace

int coinfer_oracle_structured_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                                    const coinfer_users* users, const double* deadline,
                                    const int32_t* b, int32_t* status, double* energy,
                                    uint8_t* split, uint8_t* fallback, uint8_t* feasible) {
  if (!deadline || !b || !status || !energy || !split || !fallback || !feasible)
    return fail(ctx, COINFER_E_ARG, "oracle_structured: null argument");
  cfb::OracleArgs a;
  std::memset(&a, 0, sizeof a);
  a.deadline = deadline;
  a.b = b;
  a.status = status;
  a.energy = energy;
  a.split = split;
  a.fallback = fallback;
  a.feasible = feasible;
  return run_oracle(ctx, profile, users, a, true);
}

int coinfer_oracle_grouping_batch(coinfer_ctx* ctx, const coinfer_profile* profile,
                                  const coinfer_users* users, int32_t contiguous, int32_t* status,
                                  double* energy, int32_t* n_groups, int32_t* group_of_user,
                                  uint8_t* feasible) {
  if (!status || !energy || !n_groups || !group_of_user || !feasible)
    return fail(ctx, COINFER_E_ARG, "oracle_grouping: null argument");
  cfb::OracleArgs a;
  std::memset(&a, 0, sizeof a);
  a.contiguous = contiguous ? 1 : 0;
  a.status = status;
  a.energy = energy;
  a.n_groups = n_groups;
  a.group_of_user = group_of_user;
  a.feasible = feasible;
  return run_oracle(ctx, profile, users, a, false);
}

int coinfer_best_partition(coinfer_ctx* ctx, const coinfer_profile* profile,
                           const coinfer_users* users, const double* s, int32_t* split,
                           double* freq, double* energy, uint8_t* feasible) {
  if (!ctx) return COINFER_E_ARG;
  ctx->err.clear();
  int rc = check_users(ctx, users);
  if (rc != COINFER_OK) return rc;
  if (users->mem != COINFER_MEM_HOST || users->M != 1)
    return fail(ctx, COINFER_E_ARG, "best_partition: host memory, one user per query");
  if (!split || !freq || !energy || !feasible) return fail(ctx, COINFER_E_ARG, "best_partition: null output");
  rc = check_profile(ctx, profile);
  if (rc != COINFER_OK) return rc;
  if (users->n_inst == 0) return COINFER_OK;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  const size_t K = (size_t)users->n_inst, N = (size_t)profile->N;
  cfb::AuxArgs a;
  std::memset(&a, 0, sizeof a);
  a.P = make_const(profile);
  a.n_inst = users->n_inst;
  a.M = 1;
  a.fmin = users->f_min;
  a.fmax = users->f_max;
  a.kappa = users->kappa;
  a.ru = users->rate_up;
  a.pu = users->power_up;
  a.arr = users->arrival;
  a.dl = users->deadline;
  Stager st{ctx};
  plan_in(st, a.fmin, K);
  plan_in(st, a.fmax, K);
  plan_in(st, a.kappa, K);
  plan_in(st, a.ru, K);
  plan_in(st, a.pu, K);
  plan_in(st, a.arr, K);
  plan_in(st, a.dl, K);
  const double* sd = s;
  plan_in(st, sd, K * N);
  plan_out(st, split, K);
  plan_out(st, freq, K);
  plan_out(st, energy, K);
  plan_out(st, feasible, K);
  rc = ensure_aux(ctx, st.used);
  if (rc != COINFER_OK) return rc;
  unsigned char* b = ctx->aux;
  cudaStream_t sp = ctx->stream;
  patch(b, a.fmin);
  patch(b, a.fmax);
  patch(b, a.kappa);
  patch(b, a.ru);
  patch(b, a.pu);
  patch(b, a.arr);
  patch(b, a.dl);
  patch(b, sd);
  patch(b, split);
  patch(b, freq);
  patch(b, energy);
  patch(b, feasible);
  for (const auto& x : st.in) {
    e = cudaMemcpyAsync(b + x.off, x.host, x.bytes, cudaMemcpyHostToDevice, sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D inputs");
  }
  e = cfb::launch_partition(a, sd, split, freq, energy, feasible, sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
  ctx->launches += 1;
  for (const auto& x : st.back) {
    e = cudaMemcpyAsync(x.host, b + x.off, x.bytes, cudaMemcpyDeviceToHost, sp);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H outputs");
  }
  e = cudaStreamSynchronize(sp);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "best_partition");
  return COINFER_OK;
}

}  // extern "C"
