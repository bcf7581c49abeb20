// Which pipe do 64-bit warp shuffles use, and do they contend with F2F
// (f32<->f64) conversions?  Times N iterations of: (a) 8 independent
// shfl.up/down pairs of doubles, (b) 8 independent f32->f64->f32 pairs,
// (c) both interleaved.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(256) mix(float *out, int iters) {
  double d[8];
  float f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    d[i] = threadIdx.x * 1.0001 + i;
    f[i] = threadIdx.x * 0.5f + i;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE & 1) {
        double u = __shfl_up_sync(0xffffffffu, d[i], 1);
        double w = __shfl_down_sync(0xffffffffu, d[i], 1);
        d[i] = u + w;  // one DADD per pair keeps the values live
      }
      if (MODE & 2) {
        double x = (double)f[i];
        f[i] = (float)(x * 1.0000001);
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += (float)d[i] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  float *out;
  const int blocks = 148 * 8, threads = 256, iters = 2000;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char *names[4] = {"", "shfl64 pair + dadd", "f2f pair + dmul", "both"};
  for (int mode = 1; mode <= 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 1) mix<1><<<blocks, threads>>>(out, iters);
      if (mode == 2) mix<2><<<blocks, threads>>>(out, iters);
      if (mode == 3) mix<3><<<blocks, threads>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double items = (double)blocks * threads * iters * 8;  // per-thread pairs
      double per_sm_clk = items / (ms * 1e-3) / 148 / 1.965e9;
      if (rep) printf("%-20s %.3f ms  %.2f pairs/clk/SM\n", names[mode], ms, per_sm_clk);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
