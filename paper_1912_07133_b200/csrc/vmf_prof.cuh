// vmf_prof.cuh -- launch accounting for the C ABI: every kernel launch is
// counted (vmf_launch_count) and, while profiling is on, bracketed with CUDA
// events on its own stream so bench.py can time individual kernels inside
// the timed region (vmf_profile_begin / vmf_profile_end).
#pragma once
#include <cuda_runtime.h>

namespace vmf {

enum KernelId {
  K_IIR_CARRY = 0,
  K_IIR_SCAN,
  K_IIR_APPLY,
  K_IIR_SCALE,
  K_FIR_ROWS,
  K_FIR_COLS,
  K_LAPLACIAN,
  K_ABSMAX,
  K_NMS_COUNT,
  K_NMS_SCAN,
  K_NMS_WRITE,
  K_IIR_ROWS_FUSED,
  K_IIR_COLS_FUSED,
  K_FINALIZE,
  K_COL_CARRY,
  K_COL_SCAN,
  K_ROW_BORDER,
  K_SWEEP_ROWS,
  K_COL_APPLY,
  K_FIRTC_PREP,
  K_FIRTC_ROWS,
  K_FIRTC_COLS,
  K_NUM_IDS
};

extern const char *const kKernelNames[K_NUM_IDS];

// RAII bracket around exactly one kernel launch.
class Launch {
 public:
  Launch(KernelId id, cudaStream_t st);
  ~Launch();

 private:
  int slot_;
  cudaStream_t st_;
};

}  // namespace vmf
