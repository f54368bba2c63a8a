// kernels.h — host-visible launch interface of the solver kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/coinfer_b200.h"
#include "device_common.cuh"

namespace cfb {

// Byte offsets of the fused kernel's shared-memory regions; computed on the
// host once per launch so the kernel reads them from the constant bank.
struct SmemLayout {
  int rec, tri, dls, sumlat, headE, fsc;
  int rowoff, b0, order, rank, gid, glo, ghi, headq, headlen, tpre, misc;
  int headb, bstar, parent, spsc, ipb;
  int total;
};

// Arguments of the per-instance kernels; all pointers are device memory.
struct SmallArgs {
  SmemLayout L;
  ProfileConst P;
  const double* lat;  // [N*bmax] F_n(b)
  int64_t n_inst;
  int M;
  const double *fmin, *fmax, *kappa, *ru, *pu, *arr, *dl, *rd, *pd;
  const double* l_ip;  // IP-SSA / fixed deadline per instance, NULL = min deadline
  int do_ip, do_og;
  coinfer_ipssa_out ip;
  coinfer_og_out og;
};

int small_smem_bytes(int M, int N, int W);
int fixed_smem_bytes(int M, int N);
cudaError_t launch_small(const SmallArgs& a, int threads, int grid, cudaStream_t st);
cudaError_t launch_fixed(const SmallArgs& a, const int32_t* b, int grid, cudaStream_t st);

}  // namespace cfb
