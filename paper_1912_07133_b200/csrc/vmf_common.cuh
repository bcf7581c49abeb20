// vmf_common.cuh -- shared device helpers and host-side error plumbing for the
// B200-native vmfilt hot path.  See include/vmfilt_b200.h for the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <utility>

#include "../../include/vmfilt_b200.h"

namespace vmf {

enum Orient { ROWS = 0, COLS = 1 };

// ---------------------------------------------------------------------------
// host: thread-local last error + status helpers
// ---------------------------------------------------------------------------
void set_error(const char *fmt, ...);
int fail(int code, const char *fmt, ...);
int cuda_status(const char *what);  // VMF_OK or VMF_ECUDA after a launch

// Per-device one-time host setup.  Kernel attributes (the dynamic shared
// memory opt-in) and occupancy-derived sizes belong to a device, so a
// process driving several GPUs must set them once per device, not once.
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
struct PerDevice {
  uint64_t done = 0;  // bit d: device d set up
  bool first() {
    const int d = current_device();
    if (d < 0 || d >= 64) return true;  // (not cached)
    const uint64_t b = 1ull << d;
    if (done & b) return false;
    done |= b;
    return true;
  }
};

// ---------------------------------------------------------------------------
// device: element loads (fp32 / u16 -> fp64) through the read-only path
// ---------------------------------------------------------------------------
// Input sample types of the first pass: fp32, u16 (native order), u8 and
// big-endian u16 (PGM P5 with maxval > 255, read straight from the file
// bytes; the byte swap is one PRMT in the load).
struct u16be {
  uint16_t raw;
};
__device__ __forceinline__ float ldf32(const float *p) { return __ldg(p); }
__device__ __forceinline__ float ldf32(const uint16_t *p) { return (float)__ldg(p); }
__device__ __forceinline__ float ldf32(const uint8_t *p) { return (float)__ldg(p); }
__device__ __forceinline__ float ldf32(const u16be *p) {
  const unsigned r = __ldg(&p->raw);
  return (float)__byte_perm(r, 0u, 0x3201u);  // bytes 1,0 -> 0,1 (upper half zero)
}
// Eight consecutive samples from a 16-byte (u16) / 8-byte (u8) aligned
// address with one vector load, widened to fp32 (exact).
__device__ __forceinline__ void ld8f(const uint16_t *p, float *o) {
  const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
  const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[2 * i] = (float)(w[i] & 0xffffu);
    o[2 * i + 1] = (float)(w[i] >> 16);
  }
}
__device__ __forceinline__ void ld8f(const u16be *p, float *o) {
  const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
  const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[2 * i] = (float)__byte_perm(w[i], 0u, 0x4401u);      // bytes 1,0 of the first sample
    o[2 * i + 1] = (float)__byte_perm(w[i], 0u, 0x4423u);  // bytes 3,2 of the second
  }
}
__device__ __forceinline__ void ld8f(const uint8_t *p, float *o) {
  const uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[i] = (float)((v.x >> (8 * i)) & 0xffu);
    o[4 + i] = (float)((v.y >> (8 * i)) & 0xffu);
  }
}
__device__ __forceinline__ void ld8f(const float *p, float *o) {
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = __ldg(p + i);
}

template <typename T>
__device__ __forceinline__ double ld64(const T *p) {
  return (double)ldf32(p);  // exact for every input type
}

// Host: call f((const T *)x) with T the sample type of dtype code `code`
// (VMF_F32 / VMF_U16 / VMF_U8 / VMF_U16BE); VMF_EVALUE for anything else.
template <class F>
int with_sample_type(int code, const void *x, F &&f) {
  switch (code) {
    case VMF_F32: return f((const float *)x);
    case VMF_U16: return f((const uint16_t *)x);
    case VMF_U8: return f((const uint8_t *)x);
    case VMF_U16BE: return f((const u16be *)x);
  }
  return fail(VMF_EVALUE, "unsupported dtype code %d", code);
}

// ---------------------------------------------------------------------------
// device: L2 residency hints.  The intermediate T (row-pass output) is read
// twice by the column pass, so it is written and first read with
// evict_last; the frame X and the final L stream through with evict_first.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_v4_hint(float *addr, float4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(policy)
               : "memory");
}
// 256-bit store (sm_100: STG.256, one full 32-byte sector per lane)
// Packed fp32 FMA (sm_100 FFMA2: two lanes' worth of FMAs per issue slot):
// (a.x b.x + c.x, a.y b.y + c.y).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

__device__ __forceinline__ void st_v8_hint(float *addr, const float *v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;\n" ::"l"(addr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]),
               "f"(v[7]), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void *smem_dst, const void *src, uint64_t policy) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa),
               "l"(src), "l"(policy));
}

// ---------------------------------------------------------------------------
// programmatic dependent launch: the fused path's kernels are launched with
// the PDL attribute, so each may be scheduled while its predecessor drains.
// pdl_wait() blocks until the predecessor grid has completed and its memory
// is visible (a no-op without the attribute); pdl_trigger() lets the next
// grid launch once every CTA of this grid has issued it or exited.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

template <typename... Exp, typename... Act>
inline cudaError_t launch_pdl(void (*kern)(Exp...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Act &&...args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}

// Element n of line `line` for a pass along rows (line = row) or columns
// (line = column).
template <int O, typename T>
__device__ __forceinline__ const T *line_ptr(const T *base, int64_t ld, int64_t line,
                                             int64_t n) {
  return O == ROWS ? base + line * ld + n : base + n * ld + line;
}
template <int O>
__device__ __forceinline__ float *line_ptr_out(float *base, int64_t ld, int64_t line,
                                               int64_t n) {
  return O == ROWS ? base + line * ld + n : base + n * ld + line;
}

// Non-negative float max via integer atomics (bit patterns of non-negative
// IEEE floats order like unsigned integers).
__device__ __forceinline__ void atomic_max_nonneg(float *addr, float v) {
  atomicMax(reinterpret_cast<unsigned int *>(addr), __float_as_uint(v));
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace vmf
