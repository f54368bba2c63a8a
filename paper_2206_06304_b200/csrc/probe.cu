// probe.cu — fp64-pipe throughput microbenchmark (roofline denominator).
// Each thread runs 8 independent DFMA chains (no FMA contraction concerns:
// this is a throughput probe, not a solver path), full occupancy, loop
// unrolled so loop overhead stays far below the fp64 pipe's issue share.
// ops = threads * iters * 8; best of 5 launches of ~10 ms.
#include <cuda_runtime.h>

#include "../../include/coinfer_b200.h"

namespace cfb {

__global__ void __launch_bounds__(256) dfma_probe(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
  double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
#pragma unroll 8
  for (int i = 0; i < iters; ++i) {
    x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
    x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 1234.5) out[0] = s;  // keep the chains live
}

cudaError_t probe_fp64(cudaStream_t st, double* ops_per_s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  cudaError_t e = cudaMalloc(&out, 8);
  if (e != cudaSuccess) return e;
  // ~10 ms per launch at full occupancy, so ramp-up and tail are < 1%
  const int blocks = sms * 8, threads = 256, iters = 65536;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  dfma_probe<<<blocks, threads, 0, st>>>(out, iters, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(t0, st);
    dfma_probe<<<blocks, threads, 0, st>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(t1, st);
    cudaEventSynchronize(t1);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    if (ms < best) best = ms;
  }
  e = cudaGetLastError();
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(out);
  *ops_per_s = (double)blocks * threads * iters * 8 / (best * 1e-3);
  return e;
}

}  // namespace cfb
