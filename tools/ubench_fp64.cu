// FP64 / MUFU.RSQ64H latency and throughput probes on the B200 (tools, not product).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsq(double x){double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;":"=d"(y):"d"(x)); return y;}
__global__ void lat_dfma(double* out, long long* cyc, int n){ double x=threadIdx.x+1.0; long long t0=clock64(); for(int i=0;i<n;i++) x=fma(x,0.999999,1e-7); long long t1=clock64(); out[0]=x; cyc[0]=t1-t0;}
__global__ void lat_rsq(double* out, long long* cyc, int n){ double x=threadIdx.x+2.0; long long t0=clock64(); for(int i=0;i<n;i++) x=rsq(x)+1.0; long long t1=clock64(); out[0]=x; cyc[0]=t1-t0;}
template<int C> __global__ void thr_dfma(double* out, int n){ double x[C]; for(int c=0;c<C;c++) x[c]=threadIdx.x+c; for(int i=0;i<n;i++){
#pragma unroll
 for(int c=0;c<C;c++) x[c]=fma(x[c],0.999999,1e-7);} double s=0; for(int c=0;c<C;c++) s+=x[c]; if(s==1.5) out[0]=s;}
template<int C> __global__ void thr_rsq(double* out, int n){ double x[C]; for(int c=0;c<C;c++) x[c]=threadIdx.x+c+1.0; for(int i=0;i<n;i++){
#pragma unroll
 for(int c=0;c<C;c++) x[c]=rsq(x[c]+2.0);} double s=0; for(int c=0;c<C;c++) s+=x[c]; if(s==1.5) out[0]=s;}
template<class F> float timeit(F f){ cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); f(); cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); return ms;}
int main(){ double* d; long long* c; cudaMalloc(&d,8); cudaMalloc(&c,8); long long h;
 int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
 lat_dfma<<<1,1>>>(d,c,4096); lat_dfma<<<1,1>>>(d,c,4096); cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost); printf("DFMA dependent latency: %.2f cycles\n", h/4096.0);
 lat_rsq<<<1,1>>>(d,c,4096); lat_rsq<<<1,1>>>(d,c,4096); cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost); printf("RSQ64H+DADD dependent latency: %.2f cycles\n", h/4096.0);
 int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
 for (int wps : {4, 8, 16, 32}) { // warps per SM
   int threads = 128, blocks = nsm * wps / 4; int n = 2000;
   float ms = timeit([&]{ thr_dfma<4><<<blocks,threads>>>(d,n); });
   double flops = 2.0*4*n*(double)threads*blocks; printf("DFMA 4 chains, %2d warps/SM: %.1f TFLOP/s\n", wps, flops/ms/1e9);
   ms = timeit([&]{ thr_dfma<8><<<blocks,threads>>>(d,n); });
   flops = 2.0*8*n*(double)threads*blocks; printf("DFMA 8 chains, %2d warps/SM: %.1f TFLOP/s\n", wps, flops/ms/1e9);
   ms = timeit([&]{ thr_rsq<8><<<blocks,threads>>>(d,n); });
   double ops = 8.0*n*(double)threads*blocks; printf("RSQ64H(+DADD) 8 chains, %2d warps/SM: %.1f Gop/s = %.2f per SM per clk\n", wps, ops/ms/1e6, ops/ms/1e6*1e9/(nsm*clk*1e3)/1e9*1e9/1e9);
 }
 return 0; }
