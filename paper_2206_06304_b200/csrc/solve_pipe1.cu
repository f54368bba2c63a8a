// solve_pipe1.cu -- the pipelined kernel's team shape 1 (solve_pipe.cuh),
// for N <= CFB_PIPE_MAXN sub-tasks; a translation unit of its own so the
// shapes compile in parallel.
#include "solve_pipe.cuh"

namespace cfb {

int pipe_max_grid_s1(int M, int N) {
  int g = 0;
  auto get = [&]() -> cudaError_t {
#define CFB_CALL(n) g = pipe_max_grid<n, 1>(M); return cudaSuccess
    CFB_PIPE_DISPATCH(N, CFB_CALL)
#undef CFB_CALL
  };
  return get() == cudaSuccess ? g : 0;
}

cudaError_t launch_pipe_s1(const SmallArgs& a, cudaStream_t st) {
#define CFB_CALL(n) return launch_pipe_ns<n, 1>(a, st)
  CFB_PIPE_DISPATCH(a.P.N, CFB_CALL)
#undef CFB_CALL
}

}  // namespace cfb
