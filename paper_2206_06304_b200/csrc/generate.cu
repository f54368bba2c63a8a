// generate.cu — scenario generation on the device:
// sample_scenario (scenario_gen.hpp:113-173) for a batch of seeds, one
// thread per instance, the input side of the offline sweep.
//
// The random stream is the reference's bit for bit: std::mt19937_64 seeded
// per instance (the CLI seeds sub_seed(root, 1, k), coinfer_main.cpp:47-50,
// 346-350), libstdc++ 13 generate_canonical<double, 53> (one 64-bit draw,
// scaled by 2^-64, clamped below 1), uniform_real_distribution `(b-a)*u + a`,
// and normal_distribution's Marsaglia polar method with its cached second
// variate (random.tcc:1811-1844), in the same draw order (radius, angle,
// retry while r < 1 m, shadowing, deadline redraws below the all-local
// floor).  So positions, deadlines, f_max and kappa are bit-identical to the
// reference generator.  The libm calls (log for the polar method, log10 /
// pow / log2 in uplink_rate, scenario_gen.hpp:86-93) use CUDA's
// implementations, within 1-2 ulp of glibc's, so shadowing and rates agree to
// ~1e-15 relative rather than bit for bit — generator bits are not pinned
// across platforms anyway; parity tests feed the same input
// bytes to the engine and the checkers.

#include <cmath>

#include "kernels.h"

namespace cfb {
namespace {

// std::mt19937_64 with its state in (per-thread) local memory.
struct Mt64L {
  static constexpr int n = 312, m = 156;
  unsigned long long x[n];
  int idx;
  __device__ void seed(unsigned long long v) {
    x[0] = v;
    for (int i = 1; i < n; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + (unsigned long long)i;
    idx = n;
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
    idx = 0;
  }
  __device__ unsigned long long next() {
    if (idx >= n) twist();
    unsigned long long z = x[idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71d67fffeda60000ULL;
    z ^= (z << 37) & 0xfff7eee000000000ULL;
    z ^= z >> 43;
    return z;
  }
  // generate_canonical<double, 53>: one draw, exact power-of-two scaling
  __device__ double canonical() {
    double u = __dmul_rn(__ull2double_rn(next()), 0x1p-64);
    return u >= 1.0 ? 0x1.fffffffffffffp-1 : u;
  }
  __device__ double uniform(double a, double b) { return __dadd_rn(__dmul_rn(canonical(), __dsub_rn(b, a)), a); }
};

// normal_distribution<double>(mean, stddev), libstdc++ 13 (Marsaglia polar)
struct Normal {
  double saved = 0.0;
  bool have = false;
  __device__ double operator()(Mt64L& g, double mean, double stddev) {
    double ret;
    if (have) {
      have = false;
      ret = saved;
    } else {
      double x, y, r2;
      do {
        x = __dsub_rn(__dmul_rn(2.0, g.canonical()), 1.0);
        y = __dsub_rn(__dmul_rn(2.0, g.canonical()), 1.0);
        r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
      } while (r2 > 1.0 || r2 == 0.0);
      const double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
      saved = __dmul_rn(x, mult);
      have = true;
      ret = __dmul_rn(y, mult);
    }
    return __dadd_rn(__dmul_rn(ret, stddev), mean);
  }
};

struct GenArgs {
  coinfer_sample_cfg cfg;
  double total_work;
  int M;
  int64_t n_inst;
  const unsigned long long* seeds;
  double *fmin, *fmax, *kappa, *ru, *pu, *arr, *dl, *rd, *pd;
  int32_t* status;
};

__global__ void __launch_bounds__(128) sample_kernel(GenArgs g) {
  const coinfer_sample_cfg& c = g.cfg;
  // calibrate_device (core_model.hpp:147-151) with rho = edge / device efficiency
  const double rho = __ddiv_rn(c.edge_efficiency, c.device_efficiency);
  const double fmax = __ddiv_rn(1.0, c.alpha);
  const double kappa = __dmul_rn(__dmul_rn(__dmul_rn(rho, c.edge_power), c.alpha), c.alpha);
  const double floor_ = __ddiv_rn(g.total_work, fmax);
  const double noise = pow(10.0, __ddiv_rn(__dsub_rn(c.noise_dbm_hz, 30.0), 10.0));
  const double two_pi = __dmul_rn(2.0, acos(-1.0));
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < g.n_inst;
       k += (int64_t)gridDim.x * blockDim.x) {
    Mt64L rng;
    rng.seed(g.seeds[k]);
    Normal shadow;
    int st = COINFER_ST_OK;
    for (int m = 0; m < g.M && st == COINFER_ST_OK; ++m) {
      double r, theta;
      do {
        r = __dmul_rn(c.cell_radius, __dsqrt_rn(rng.uniform(0.0, 1.0)));
        theta = __dmul_rn(two_pi, rng.uniform(0.0, 1.0));
      } while (r < 1.0);
      (void)theta;  // positions are not part of the solver input
      const double sh = c.shadow_sigma_db > 0.0 ? shadow(rng, 0.0, c.shadow_sigma_db) : 0.0;
      // uplink_rate (scenario_gen.hpp:86-93)
      const double d_km = __ddiv_rn(r, 1000.0);
      const double pl = __dadd_rn(__dadd_rn(128.1, __dmul_rn(37.6, log10(d_km))), sh);
      const double gain = pow(10.0, __ddiv_rn(-pl, 10.0));
      const double snr = __ddiv_rn(__dmul_rn(c.tx_power, gain), __dmul_rn(c.bandwidth, noise));
      const double rate = __dmul_rn(c.bandwidth, log2(__dadd_rn(1.0, snr)));
      double l;
      if (!c.deadline_uniform) {
        l = c.deadline_low;
      } else {
        int guard = 0;
        do {
          l = rng.uniform(c.deadline_low, c.deadline_high);
          if (++guard > 100000) {
            st = COINFER_ST_NO_DEADLINE;
            break;
          }
        } while (l < floor_);
      }
      const size_t i = (size_t)k * g.M + m;
      g.fmin[i] = 0.0;
      g.fmax[i] = fmax;
      g.kappa[i] = kappa;
      g.ru[i] = rate;
      g.pu[i] = c.uplink_power;
      g.arr[i] = 0.0;
      g.dl[i] = l;
      if (g.rd) g.rd[i] = rate;
      if (g.pd) g.pd[i] = c.downlink_power;
    }
    if (g.status) g.status[k] = st;
  }
}

}  // namespace

cudaError_t launch_sample(const coinfer_sample_cfg& cfg, double total_work, int M, int64_t n_inst,
                          const unsigned long long* seeds, const coinfer_users_mut& out, int32_t* status,
                          cudaStream_t st) {
  GenArgs g;
  g.cfg = cfg;
  g.total_work = total_work;
  g.M = M;
  g.n_inst = n_inst;
  g.seeds = seeds;
  g.fmin = out.f_min;
  g.fmax = out.f_max;
  g.kappa = out.kappa;
  g.ru = out.rate_up;
  g.pu = out.power_up;
  g.arr = out.arrival;
  g.dl = out.deadline;
  g.rd = out.rate_down;
  g.pd = out.power_down;
  g.status = status;
  const int64_t want = (n_inst + 127) / 128;
  const int grid = (int)(want < 148 * 16 ? (want > 0 ? want : 1) : 148 * 16);
  sample_kernel<<<grid, 128, 0, st>>>(g);
  return cudaGetLastError();
}

}  // namespace cfb
