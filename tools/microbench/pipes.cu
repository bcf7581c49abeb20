// Pipe-throughput microbenchmark for the B200 design decisions (fp64 DFMA
// rate, f32<->f64 conversion rate, copy bandwidth).  Not product code.
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
__global__ void dfma_k(double* out, int iters, double a, double b) {
  double v[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) v[c] = fma(v[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += v[c];
  if (s == 12345.678) out[0] = s;
}
__global__ void ffma_k(float* out, int iters, float a, float b) {
  float v[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) v[c] = fmaf(v[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += v[c];
  if (s == 12345.678f) out[0] = s;
}
// dependent-chain latency of DFMA (1 chain per thread, 1 warp per SM)
__global__ void dfma_lat_k(double* out, int iters, double a, double b, long long* cyc) {
  double v = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = fma(v, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (v == 12345.678) out[0] = v;
}
__global__ void cvt_k(float* out, int iters) {
  float f[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) f[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      double d;
      asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f[c]));
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[c]) : "d"(d));
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += f[c];
  if (s == 12345.678f) out[0] = s;
}
__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("name=%s sms=%d l2=%d MB smem/blk optin=%zu regs/sm=%d clock_khz=%d memclk_khz=%d busw=%d\n",
         p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin,
         p.regsPerMultiprocessor, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  int sms = p.multiProcessorCount;
  double* dout; float* fout; long long* cyc;
  cudaMalloc(&dout, 8); cudaMalloc(&fout, 8); cudaMalloc(&cyc, 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int iters = 4096;
  for (int bps = 4; bps <= 8; bps *= 2) {
    dim3 g(sms * bps), b(256);
    dfma_k<<<g, b>>>(dout, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_k<<<g, b>>>(dout, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)g.x * b.x * iters * CHAINS;
    printf("DFMA  blocks/sm=%d: %.3f ms  %.2f TFMA/s  (%.1f fp64 TFLOP/s)\n", bps, ms, ops / ms / 1e9, 2 * ops / ms / 1e9);
    ffma_k<<<g, b>>>(fout, 16, 1.0000001f, 1e-9f);
    cudaEventRecord(e0); ffma_k<<<g, b>>>(fout, iters, 1.0000001f, 1e-9f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA  blocks/sm=%d: %.3f ms  %.2f TFMA/s\n", bps, ms, ops / ms / 1e9);
    cvt_k<<<g, b>>>(fout, 16);
    cudaEventRecord(e0); cvt_k<<<g, b>>>(fout, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("CVT pair f32->f64->f32 blocks/sm=%d: %.3f ms  %.2f Tpairs/s\n", bps, ms, ops / ms / 1e9);
  }
  dfma_lat_k<<<sms, 32>>>(dout, 16, 1.0000001, 1e-9, cyc);
  dfma_lat_k<<<sms, 32>>>(dout, 100000, 1.0000001, 1e-9, cyc);
  long long c0; cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", c0 / 100000.0);
  size_t n = (size_t)1 << 28;  // 1 GiB per buffer
  float4 *a, *bb; cudaMalloc(&a, n * 4); cudaMalloc(&bb, n * 4);
  cudaMemset(a, 0, n * 4);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); copy_k<<<sms * 8, 512>>>(a, bb, n / 4); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 1GiB: %.3f ms  %.1f GB/s\n", ms, 2.0 * n * 4 / ms / 1e6);
  }
  // 64 MiB copy (fits L2): L2-resident repeated
  size_t n2 = (size_t)1 << 24;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); copy_k<<<sms * 8, 512>>>(a, bb, n2 / 4); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 64MiB (warm): %.3f ms  %.1f GB/s\n", ms, 2.0 * n2 * 4 / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
