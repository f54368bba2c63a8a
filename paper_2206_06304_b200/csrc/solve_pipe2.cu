// solve_pipe2.cu -- the pipelined kernel's team shape 2 (solve_pipe.cuh),
// for N <= CFB_PIPE_MAXN sub-tasks; a translation unit of its own so the
// shapes compile in parallel.
#include "solve_pipe.cuh"

namespace cfb {

int pipe_max_grid_s2(int M, int N) {
  int g = 0;
  auto get = [&]() -> cudaError_t {
#define CFB_CALL(n) g = pipe_max_grid<n, 2>(M); return cudaSuccess
    CFB_PIPE_DISPATCH(N, CFB_CALL)
#undef CFB_CALL
  };
  return get() == cudaSuccess ? g : 0;
}

cudaError_t launch_pipe_s2(const SmallArgs& a, cudaStream_t st) {
#define CFB_CALL(n) return launch_pipe_ns<n, 2>(a, st)
  CFB_PIPE_DISPATCH(a.P.N, CFB_CALL)
#undef CFB_CALL
}

}  // namespace cfb
