// vmf_tma.cuh -- TMA (cp.async.bulk.tensor) helpers: host-side tensor-map
// encoding through the driver entry point (no libcuda link), device-side
// mbarrier + 2-D tile load.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

namespace vmf {

// 2-D fp32 tensor map over a row-major [rows][cols] image with pitch ld
// (elements); box = box_cols x box_rows.  Returns false if TMA is unavailable.
bool make_tmap_2d_f32(CUtensorMap *map, const float *base, int64_t rows, int64_t cols,
                      int64_t ld, int box_cols, int box_rows);

// Rows of a row-major fp32 image as 3-D boxes [chunks][32] with 128-byte
// swizzle: dims {32, w / 32, rows}; box = nrows whole rows.  w % 32 == 0.
bool make_tmap_rows_swz_f32(CUtensorMap *map, const float *base, int64_t rows, int64_t w,
                            int64_t ld, int nrows);

// 2-D fp32 [rows][cols] map with 128-byte swizzle and box {32 cols, box_rows}:
// the K-major SWIZZLE_128B operand layout of tcgen05.mma (8-row x 128-byte
// atoms, 1024 bytes apart).  OOB elements read as zero.
bool make_tmap_2d_f32_sw128(CUtensorMap *map, const float *base, int64_t rows, int64_t cols,
                            int64_t ld, int box_rows);

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  asm volatile("fence.proxy.async.shared::cta;\n" ::);
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes));
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c, int r) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(r), "r"(b)
      : "memory");
}

// Same load with an L2 eviction-priority policy (see l2_policy_* in
// vmf_common.cuh).
__device__ __forceinline__ void tma_load_2d_hint(void *dst, const CUtensorMap *map, uint64_t *bar,
                                                 int c, int r, uint64_t policy) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(r), "r"(b), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d_hint(void *dst, const CUtensorMap *map, uint64_t *bar,
                                                 int c0, int c1, int c2, uint64_t policy) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(b), "l"(policy)
      : "memory");
}

// shared -> global tile store (bulk-group completion; the caller commits and
// waits with cp.async.bulk.commit_group / wait_group).
__device__ __forceinline__ void tma_store_3d_hint(const CUtensorMap *map, const void *src, int c0,
                                                  int c1, int c2, uint64_t policy) {
  unsigned s = (unsigned)__cvta_generic_to_shared(src);
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint"
      " [%0, {%1, %2, %3}], [%4], %5;\n" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(s), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}

}  // namespace vmf
