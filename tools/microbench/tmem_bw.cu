// TMEM load / store throughput: every warp issues 4 independent
// tcgen05.{st,ld}.32x32b.x16 (64 columns) per round and waits once.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdint>
#include <cstdio>

#define ST16(ta, r)                                                                               \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, "  \
               "%9, %10, %11, %12, %13, %14, %15, %16};\n" ::"r"(ta),                             \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),      \
               "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),  \
               "r"(r[14]), "r"(r[15]))
#define LD16(ta, r)                                                                               \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, " \
               "%10, %11, %12, %13, %14, %15}, [%16];\n"                                         \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),         \
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),       \
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                              \
               : "r"(ta))

template <int MODE>  // 1 = store only, 2 = load only, 3 = store + load
__global__ void __launch_bounds__(128, 8) bw(int rounds, unsigned *out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(
        (unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t ta = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t a[16], b[16], c[16], d[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = b[i] = c[i] = d[i] = threadIdx.x + i;
  unsigned acc = 0;
  for (int it = 0; it < rounds; ++it) {
    if (MODE & 1) {
      ST16(ta, a);
      ST16(ta + 16, b);
      ST16(ta + 32, c);
      ST16(ta + 48, d);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    if (MODE & 2) {
      LD16(ta, a);
      LD16(ta + 16, b);
      LD16(ta + 32, c);
      LD16(ta + 48, d);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      acc += a[it & 15] + b[3] + c[7] + d[11];
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tbase));
}

int main() {
  unsigned *out;
  const int grid = 148 * 8, rounds = 4000;
  cudaMalloc(&out, grid * 128 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 1; mode <= 3; ++mode)
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 1) bw<1><<<grid, 128>>>(rounds, out);
      if (mode == 2) bw<2><<<grid, 128>>>(rounds, out);
      if (mode == 3) bw<3><<<grid, 128>>>(rounds, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)grid * 128 * 64 * 4 * rounds * (mode == 3 ? 2 : 1);
      if (rep)
        printf("mode %d (%s): %.3f ms  %.0f B/clk/SM\n", mode,
               mode == 1 ? "st" : (mode == 2 ? "ld" : "st+ld"), ms,
               bytes / (ms * 1e-3) / 148 / 1.965e9);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
