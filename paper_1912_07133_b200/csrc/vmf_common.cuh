// vmf_common.cuh -- shared device helpers and host-side error plumbing for the
// B200-native vmfilt hot path.  See include/vmfilt_b200.h for the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/vmfilt_b200.h"

namespace vmf {

enum Orient { ROWS = 0, COLS = 1 };

// ---------------------------------------------------------------------------
// host: thread-local last error + status helpers
// ---------------------------------------------------------------------------
void set_error(const char *fmt, ...);
int fail(int code, const char *fmt, ...);
int cuda_status(const char *what);  // VMF_OK or VMF_ECUDA after a launch

// ---------------------------------------------------------------------------
// device: element loads (fp32 / u16 -> fp64) through the read-only path
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ld64(const float *p) { return (double)__ldg(p); }
__device__ __forceinline__ double ld64(const uint16_t *p) { return (double)__ldg(p); }

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
