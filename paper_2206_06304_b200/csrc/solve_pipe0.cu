// solve_pipe0.cu -- the pipelined kernel's team shape 0 (solve_pipe.cuh),
// for N <= CFB_PIPE_MAXN sub-tasks; a translation unit of its own so the
// shapes compile in parallel.
#include "solve_pipe.cuh"

namespace cfb {

int pipe_max_grid_s0(int M, int N) {
  int g = 0;
  auto get = [&]() -> cudaError_t {
#define CFB_CALL(n) g = pipe_max_grid<n, 0>(M); return cudaSuccess
    CFB_PIPE_DISPATCH(N, CFB_CALL)
#undef CFB_CALL
  };
  return get() == cudaSuccess ? g : 0;
}

cudaError_t launch_pipe_s0(const SmallArgs& a, cudaStream_t st) {
#define CFB_CALL(n) return launch_pipe_ns<n, 0>(a, st)
  CFB_PIPE_DISPATCH(a.P.N, CFB_CALL)
#undef CFB_CALL
}

#ifdef CFB_PIPE_PROF
extern "C" int coinfer_debug_pipe_cycles(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_pipe_cyc, sizeof(unsigned long long) * 4);
  if (reset) {
    unsigned long long z[4] = {0};
    cudaMemcpyToSymbol(g_pipe_cyc, z, sizeof z);
  }
  return 0;
}
#endif

}  // namespace cfb
