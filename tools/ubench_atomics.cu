// FP64 global reduction throughput (red.global.add.f64) for the symmetric interaction kernel's
// column-sum flush (tools, not product).  Pattern: runs of 14 consecutive doubles (one cell's pivots)
// at scattered bases inside a 16 MB array, like u_in of a level.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void red_runs(double* a, int64_t nslots, int runs_per_warp, int run) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  unsigned h = (unsigned)warp * 2654435761u;
  for (int r = 0; r < runs_per_warp; r++) {
    h = h * 1664525u + 1013904223u;
    const int64_t base = (int64_t)(h % (unsigned)(nslots - 64));
    // each lane owns a few slots of a 32 x 3 register tile: 3 runs of `run` per lane-group
    if (lane < run) atomicAdd(a + base + lane, 1.0);
  }
}
__global__ void red_dense(double* a, int64_t n, int iters) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; it++) atomicAdd(a + (i + it * 7919) % n, 1.0);
}
template <class F> float timeit(F f) { cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n = 2 << 20;  // 16 MB
  double* a; cudaMalloc(&a, n * 8); cudaMemset(a, 0, n * 8);
  for (int run : {14, 32}) {
    const int blocks = nsm * 8, threads = 256, rpw = 200;
    float ms = timeit([&] { red_runs<<<blocks, threads>>>(a, n, rpw, run); });
    double ops = (double)blocks * threads / 32 * rpw * run;
    printf("runs of %d: %.3f ms, %.3g atomics/s\n", run, ms, ops / ms * 1e3);
  }
  {
    const int blocks = nsm * 16, threads = 256, it = 64;
    float ms = timeit([&] { red_dense<<<blocks, threads>>>(a, n, it); });
    double ops = (double)blocks * threads * it;
    printf("coalesced warps: %.3f ms, %.3g atomics/s\n", ms, ops / ms * 1e3);
  }
  return 0;
}
