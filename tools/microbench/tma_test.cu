// Standalone check of the TMA helpers in vmf_tma.cuh (not product code).
#include <cstdio>
#include <vector>
#include "../../paper_1912_07133_b200/csrc/vmf_tma.cuh"
using namespace vmf;

__device__ void body(const CUtensorMap *tm, float *out, int c, int r) {
  extern __shared__ __align__(128) unsigned char sm[];
  float *tile = reinterpret_cast<float *>(((uintptr_t)sm + 127) & ~(uintptr_t)127);
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(1));
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
    mbar_expect_tx(&bar, 70 * 128 * 4);
    tma_load_2d(tile, tm, &bar, c, r);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 70 * 128; i += blockDim.x) out[i] = tile[i];
}
__global__ void kparam(const __grid_constant__ CUtensorMap tmap, float *out, int c, int r) {
  body(&tmap, out, c, r);
}
__global__ void kglobal(const CUtensorMap *tmap, float *out, int c, int r) { body(tmap, out, c, r); }
template <int BOXC, int BOXR, int FORM>
__global__ void ksmall(const __grid_constant__ CUtensorMap tmap, float *out, int c, int r) {
  extern __shared__ __align__(128) unsigned char sm[];
  float *tile = reinterpret_cast<float *>(((uintptr_t)sm + 127) & ~(uintptr_t)127);
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(1));
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
    mbar_expect_tx(&bar, BOXC * BOXR * 4);
    unsigned d = (unsigned)__cvta_generic_to_shared(tile);
    if (FORM == 0)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(d), "l"((uint64_t)&tmap), "r"(c), "r"(r), "r"(a) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(d), "l"((uint64_t)&tmap), "r"(c), "r"(r), "r"(a) : "memory");
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < BOXC * BOXR; i += blockDim.x) out[i] = tile[i];
}
__global__ void kbulk(const float *src, float *out) {  // 1-D bulk copy
  __shared__ __align__(128) float tile[1024];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(1));
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
    mbar_expect_tx(&bar, 4096);
    unsigned d = (unsigned)__cvta_generic_to_shared(tile);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];\n"
                 ::"r"(d), "l"(src), "r"(a) : "memory");
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = tile[i];
}
__global__ void kbar(float *out) {  // mbarrier only, plain arrive
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a));
  }
  mbar_wait(&bar, 0);
  out[threadIdx.x] = 1.0f;
}

int check(const char *name, cudaError_t e, float *o, const std::vector<float> &h, int W) {
  printf("%s: %s\n", name, cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> ho(70 * 128);
  cudaMemcpy(ho.data(), o, 70 * 128 * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int rr = 0; rr < 70; ++rr)
    for (int cc = 0; cc < 128; ++cc)
      if (ho[rr * 128 + cc] != h[(61 + rr) * W + 122 + cc]) ++bad;
  printf("%s mismatches %d\n", name, bad);
  return 0;
}

int main(int argc, char **argv) {
  int which = argc > 1 ? atoi(argv[1]) : 0;
  int H = 512, W = 512;
  std::vector<float> h(H * W);
  for (int i = 0; i < H * W; ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, H * W * 4);
  cudaMalloc(&o, 70 * 128 * 4);
  cudaMemcpy(d, h.data(), H * W * 4, cudaMemcpyHostToDevice);
  CUtensorMap map;
  bool ok = make_tmap_2d_f32(&map, d, H, W, W, 128, 70);
  if (which == 6 || which == 7) {  // link-time libcuda encode
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
    cuuint64_t strides[1] = {(cuuint64_t)(W * 4)};
    cuuint32_t box[2] = {32, 8};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("libcuda encode rc=%d\n", (int)r);
    const unsigned char *b = (const unsigned char *)&map;
    for (int i = 0; i < 128; ++i) printf("%02x%s", b[i], (i % 32 == 31) ? "\n" : "");
    if (which == 6) ksmall<32, 8, 0><<<1, 128, 2048>>>(map, o, 122, 61);
    else ksmall<32, 8, 0><<<1, 128, 2048>>>(map, o, 0, 0);
    cudaError_t e = cudaDeviceSynchronize(); printf("libcuda small: %s\n", cudaGetErrorString(e));
    return 0;
  }
  printf("encode ok=%d sizeof=%zu\n", ok, sizeof(map));
  int smem = 70 * 128 * 4 + 256;
  if (which >= 3) {
    cudaError_t e;
    if (which == 3) { kbulk<<<1, 128>>>(d, o); e = cudaDeviceSynchronize(); printf("bulk1d: %s\n", cudaGetErrorString(e)); return 0; }
    CUtensorMap m2;
    bool ok2 = make_tmap_2d_f32(&m2, d, H, W, W, 32, 8);
    printf("encode small ok=%d\n", ok2);
    if (which == 4) ksmall<32, 8, 0><<<1, 128, 2048>>>(m2, o, 122, 61);
    if (which == 5) ksmall<32, 8, 1><<<1, 128, 2048>>>(m2, o, 122, 61);
    e = cudaDeviceSynchronize(); printf("small form %d: %s\n", which - 4, cudaGetErrorString(e));
    return 0;
  }
  if (which == 0) {
    kbar<<<1, 32>>>(o);
    printf("kbar: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  } else if (which == 1) {
    CUtensorMap *dm;
    cudaMalloc(&dm, sizeof(map));
    cudaMemcpy(dm, &map, sizeof(map), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(kglobal, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kglobal<<<1, 128, smem>>>(dm, o, 122, 61);
    return check("global desc", cudaDeviceSynchronize(), o, h, W);
  } else {
    cudaFuncSetAttribute(kparam, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kparam<<<1, 128, smem>>>(map, o, 122, 61);
    return check("param desc", cudaDeviceSynchronize(), o, h, W);
  }
  return 0;
}
