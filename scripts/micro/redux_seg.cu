// Checks that redux.sync / ballot with per-lane segment membermasks (disjoint
// groups inside one warp, executed convergently) reduce within each segment.
#include <cstdio>
#include <cstdlib>
__global__ void k(const unsigned* v, const unsigned* seg_end, unsigned* out, unsigned* bal) {
  const int gi = blockIdx.x * blockDim.x + threadIdx.x; const int lane = gi & 31, w = gi >> 5;
  const unsigned* se = seg_end + w * 32;
  // segment of this lane: [start, end)
  int start = 0;
  for (int l = 0; l < lane; ++l) if (se[l] != se[lane]) start = l + 1;
  const int end = se[lane];
  const unsigned mask = (end >= 32 ? 0xffffffffu : ((1u << end) - 1u)) & ~((1u << start) - 1u);
  out[gi] = __reduce_min_sync(mask, v[gi]);
  bal[gi] = __ballot_sync(mask, v[gi] & 1) & mask;
}
int main() {
  const int W = 64, T = W * 32;
  unsigned *v, *se, *o, *b;
  cudaMallocManaged(&v, T * 4); cudaMallocManaged(&se, T * 4); cudaMallocManaged(&o, T * 4); cudaMallocManaged(&b, T * 4);
  srand(1);
  for (int w = 0; w < W; ++w) {
    int l = 0;
    while (l < 32) { int len = 1 + rand() % 12; int e = l + len > 32 ? 32 : l + len; for (int x = l; x < e; ++x) se[w * 32 + x] = e; l = e; }
    for (int x = 0; x < 32; ++x) v[w * 32 + x] = rand();
  }

  cudaDeviceSynchronize();
  k<<<W / 32, 1024>>>(v, se, o, b);
  cudaDeviceSynchronize();
  int bad = 0;
  for (int w = 0; w < W; ++w) for (int x = 0; x < 32; ++x) {
    int i = w * 32 + x; int end = se[i]; int start = 0;
    for (int l = 0; l < x; ++l) if (se[w*32+l] != se[i]) start = l + 1;
    unsigned m = 0xffffffffu, bb = 0;
    for (int l = start; l < end; ++l) { if (v[w*32+l] < m) m = v[w*32+l]; if (v[w*32+l] & 1) bb |= 1u << l; }
    if (o[i] != m || b[i] != bb) ++bad;
  }
  printf("segmented redux/ballot mismatches: %d of %d\n", bad, T);
  return bad != 0;
}
