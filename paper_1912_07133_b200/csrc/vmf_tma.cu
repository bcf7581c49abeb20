// vmf_tma.cu -- see vmf_tma.cuh.
#include <mutex>

#include "vmf_tma.cuh"

namespace vmf {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    // request the CUDA 12.0 ABI of the symbol explicitly (the installed
    // driver may be newer than this runtime)
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

bool make_tmap_2d_f32(CUtensorMap *map, const float *base, int64_t rows, int64_t cols,
                      int64_t ld, int box_cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  if (((uintptr_t)base & 15) || ((ld * 4) & 15) || box_cols > 256 || box_rows > 256) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_rows_swz_f32(CUtensorMap *map, const float *base, int64_t rows, int64_t w,
                            int64_t ld, int nrows) {
  auto fn = encode_fn();
  if (!fn) return false;
  if (((uintptr_t)base & 15) || ((ld * 4) & 15) || (w % 32) || w / 32 > 256) return false;
  cuuint64_t dims[3] = {32, (cuuint64_t)(w / 32), (cuuint64_t)rows};
  cuuint64_t strides[2] = {128, (cuuint64_t)(ld * 4)};
  cuuint32_t box[3] = {32, (cuuint32_t)(w / 32), (cuuint32_t)nrows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_2d_f32_sw128(CUtensorMap *map, const float *base, int64_t rows, int64_t cols,
                            int64_t ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  if (((uintptr_t)base & 15) || ((ld * 4) & 15) || box_rows > 256) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace vmf
