// Library-level entry points: ABI version, last-error string, device check,
// and the TMA tensor-map encoder (driver entry point fetched through the
// runtime so the library does not link libcuda directly).
#include <string.h>

#include <mutex>
#include <map>
#include <utility>

#include "common.cuh"

static thread_local char g_last_error[512] = "";

void omni_set_last_error(const char* msg) {
  strncpy(g_last_error, msg ? msg : "", sizeof(g_last_error) - 1);
  g_last_error[sizeof(g_last_error) - 1] = '\0';
}

void omni_set_cuda_error(const char* what, cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, cudaGetErrorString(e));
}

cudaError_t omni_smem_attr_raw(const void* fn, int bytes) {
  // the attribute only ever grows per (kernel, device): a later, smaller
  // request must not lower the limit a concurrent or later launch relies on
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cur;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_pair(fn, dev);
  std::lock_guard<std::mutex> lock(mu);
  const auto it = cur.find(key);
  if (it != cur.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur[key] = bytes;
  return e;
}

extern "C" int omni_abi_version(void) { return OMNI_ABI_VERSION; }

extern "C" const char* omni_last_error(void) { return g_last_error; }

extern "C" int omni_device_check(void) {
  omni_begin();
  int dev = 0;
  OMNI_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  OMNI_CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10 || prop.minor != 0) {
    omni_set_last_error("libomnisparse is built for sm_100a (B200) only");
    return OMNI_E_CUDA;
  }
  return OMNI_OK;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D row-major tensor map [rows, cols] with a (box_rows x box_cols) box and
// 128-byte swizzle (box_cols * elem_bytes must be 128). Out-of-range rows read
// as zero.
int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    omni_set_last_error("cuTensorMapEncodeTiled unavailable");
    return OMNI_E_CUDA;
  }
  cuuint64_t dims[2] = {cols_elems, rows};
  cuuint64_t strides[1] = {cols_elems * (cuuint64_t)elem_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapDataType dt = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    omni_set_last_error("cuTensorMapEncodeTiled failed");
    return OMNI_E_CUDA;
  }
  return OMNI_OK;
}
