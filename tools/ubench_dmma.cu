// DMMA (mma.sync m8n8k4 f64) throughput alone and mixed with DFMA (tools, not product).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int MM, int FF>
__global__ void mix(double* out, int n) {
  double c[MM > 0 ? MM : 1][2];
  for (int i = 0; i < (MM > 0 ? MM : 1); i++) { c[i][0] = threadIdx.x; c[i][1] = i; }
  double f[FF > 0 ? FF : 1];
  for (int i = 0; i < (FF > 0 ? FF : 1); i++) f[i] = threadIdx.x + i;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  for (int it = 0; it < n; it++) {
#pragma unroll
    for (int i = 0; i < MM; i++) dmma(c[i][0], c[i][1], a, b);
#pragma unroll
    for (int i = 0; i < FF; i++) f[i] = fma(f[i], 0.999999, 1e-7);
  }
  double s = 0;
  for (int i = 0; i < MM; i++) s += c[i][0] + c[i][1];
  for (int i = 0; i < FF; i++) s += f[i];
  if (s == 1.2345) out[0] = s;
}
template <class F> float timeit(F f) { cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
int main() {
  double* d; cudaMalloc(&d, 8); int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int blocks = nsm * 8, threads = 256, n = 4000;
  float ms = timeit([&] { mix<8, 0><<<blocks, threads>>>(d, n); });
  double mmas = 8.0 * n * blocks * threads / 32; printf("DMMA only: %.1f TFLOP/s (512 flop per m8n8k4)\n", mmas * 512 / ms / 1e9);
  ms = timeit([&] { mix<0, 8><<<blocks, threads>>>(d, n); });
  printf("DFMA only: %.1f TFLOP/s\n", 8.0 * n * blocks * threads * 2 / ms / 1e9);
  ms = timeit([&] { mix<4, 8><<<blocks, threads>>>(d, n); });
  printf("mixed 4 DMMA + 8 DFMA per iter: %.3f ms (DMMA %.1f TF + DFMA %.1f TF)\n", ms, 4.0 * n * blocks * threads / 32 * 512 / ms / 1e9, 8.0 * n * blocks * threads * 2 / ms / 1e9);
  ms = timeit([&] { mix<4, 0><<<blocks, threads>>>(d, n); });
  printf("4 DMMA only: %.3f ms\n", ms);
  ms = timeit([&] { mix<0, 8><<<blocks, threads>>>(d, n); });
  printf("8 DFMA only: %.3f ms\n", ms);
  return 0;
}
