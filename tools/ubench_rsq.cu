// Accuracy of the MUFU.RSQ64H seed (rsqrt.approx.ftz.f64) and of the one-step
// Newton forms used by the interaction kernel, over inputs spanning 1e-12..1e12.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ double rsq_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__global__ void k(int n, unsigned long long seed, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long s = seed + 0x9E3779B97F4A7C15ull * (i + 1);
  s ^= s >> 33; s *= 0xff51afd7ed558ccdull; s ^= s >> 33; s *= 0xc4ceb9fe1a85ec53ull; s ^= s >> 33;
  double u = (double)(s >> 11) * (1.0 / 9007199254740992.0);
  double x = pow(10.0, -12.0 + 24.0 * u);
  double ex = 1.0 / sqrt(x);
  double y = rsq_approx(x);
  double q = 0.5 * y * fma(-x, y * y, 3.0);
  double e = fma(-x, y * y, 1.0);
  double c = fma(y * e, fma(0.375, e, 0.5), y);
  out[3 * i] = fabs(y - ex) / ex;
  out[3 * i + 1] = fabs(q - ex) / ex;
  out[3 * i + 2] = fabs(c - ex) / ex;
}

int main() {
  const int n = 1 << 22;
  double* d;
  cudaMalloc(&d, 3 * sizeof(double) * n);
  k<<<n / 256, 256>>>(n, 12345, d);
  double* h = new double[3 * n];
  cudaMemcpy(h, d, 3 * sizeof(double) * n, cudaMemcpyDeviceToHost);
  double mx[3] = {0, 0, 0}, mean[3] = {0, 0, 0};
  for (int i = 0; i < n; i++)
    for (int j = 0; j < 3; j++) {
      mx[j] = fmax(mx[j], h[3 * i + j]);
      mean[j] += h[3 * i + j] / n;
    }
  printf("rsqrt.approx.f64 seed: max rel err %.3e (2^%.1f), mean %.3e\n", mx[0], log2(mx[0]), mean[0]);
  printf("seed + quadratic Newton: max rel err %.3e, mean %.3e\n", mx[1], mean[1]);
  printf("seed + cubic correction: max rel err %.3e, mean %.3e\n", mx[2], mean[2]);
  return 0;
}
