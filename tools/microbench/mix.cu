// Does F2F (f32<->f64) issue concurrently with DFMA on sm_100a?  And what does
// an integer-pipe f32->f64 conversion cost next to DFMA?  Not product code.
#include <cstdio>
#include <cuda_runtime.h>
#define CH 8
__device__ __forceinline__ double i2d(float f) {  // exact for normal floats
  unsigned b = __float_as_uint(f);
  unsigned hi = (b & 0x80000000u) | (((b & 0x7fffffffu) >> 3) + (896u << 20));
  unsigned lo = b << 29;
  hi = (b & 0x7fffffffu) ? hi : (b & 0x80000000u);
  return __hiloint2double(hi, lo);
}
template <int MODE>
__global__ void k(float* out, int iters, double a, double b) {
  double v[CH]; float f[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { v[c] = threadIdx.x * 1e-3 + c; f[c] = threadIdx.x * 1e-3f + c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MODE == 0 || MODE == 2 || MODE == 3) {  // 4 DFMA per chain
        v[c] = fma(v[c], a, b); v[c] = fma(v[c], a, b); v[c] = fma(v[c], a, b); v[c] = fma(v[c], a, b);
      }
      if (MODE == 1 || MODE == 2) {  // 1 cvt pair per chain (2 F2F)
        double d; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f[c]));
        asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[c]) : "d"(d));
      }
      if (MODE == 3) {  // int-trick up-conversion, consumed
        double d = i2d(f[c]);
        v[c] += d * 1e-30;
        f[c] = __uint_as_float(__float_as_uint(f[c]) ^ 1u);
      }
      if (MODE == 4) {  // int-trick alone
        double d = i2d(f[c]);
        asm volatile("" :: "d"(d));
        f[c] = __uint_as_float(__float_as_uint(f[c]) + 3u);
      }
    }
  }
  double s = 0; float t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) { s += v[c]; t += f[c]; }
  if (s == 1.2345 || t == 1.2345f) out[0] = (float)s + t;
}
int main() {
  float* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dim3 g(148 * 8), bl(256); int it = 2048; float ms;
  const char* names[] = {"4 DFMA", "1 cvt pair (2 F2F)", "4 DFMA + 2 F2F", "4 DFMA + int cvt + DADD/DFMA", "int cvt alone"};
  for (int m = 0; m < 5; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k<0><<<g, bl>>>(o, it, 1.0000001, 1e-9);
      if (m == 1) k<1><<<g, bl>>>(o, it, 1.0000001, 1e-9);
      if (m == 2) k<2><<<g, bl>>>(o, it, 1.0000001, 1e-9);
      if (m == 3) k<3><<<g, bl>>>(o, it, 1.0000001, 1e-9);
      if (m == 4) k<4><<<g, bl>>>(o, it, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double units = (double)g.x * bl.x * it * CH;
    printf("%-32s %.3f ms  (%.2f G chain-iters/s)\n", names[m], ms, units / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
