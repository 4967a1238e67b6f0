// C-ABI plumbing shared by every entry point: thread-local error messages,
// launch checking, device properties and driver entry-point lookup.
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace mosaic {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error.assign(buf);
}

int fail(int status, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error.assign(buf);
  return status;
}

int check_launch(const char* what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(MOSAIC_E_CUDA, "%s launch: %s", what, cudaGetErrorString(err));
  return MOSAIC_OK;
}

int num_sms() {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  cache[dev] = n;
  return n;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

void* driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return fn;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int encode_tma_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld, int box_rows,
                    int box_cols) {
  static EncodeTiledFn fn = reinterpret_cast<EncodeTiledFn>(driver_fn("cuTensorMapEncodeTiled"));
  if (!fn) return fail(MOSAIC_E_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t elem_strides[2] = {1, 1};
  // L2 promotion of TMA reads (experiment knob MOSAIC_TMA_L2_PROMOTION: 0 none, 1 64B, 2 128B, 3 256B)
  static const int promo = [] {
    const char* e = getenv("MOSAIC_TMA_L2_PROMOTION");
    return e ? atoi(e) : 3;
  }();
  const CUtensorMapL2promotion pr = promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                    : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                 : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                  elem_strides, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MOSAIC_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return MOSAIC_OK;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MOSAIC_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace mosaic

extern "C" int mosaic_abi_version(void) { return 100; }

extern "C" const char* mosaic_last_error(void) { return mosaic::g_last_error.c_str(); }

// L2 set-aside for persisting accesses (the evict_last class of createpolicy /
// access-policy windows). K3 marks its A operand (the gathered masked rows,
// re-read once per vocab tile) evict_last; without a set-aside the hint has no
// reserved capacity to protect those lines from the streamed LM-head weights.
extern "C" int mosaic_l2_persisting_limit(int64_t bytes, int64_t* applied_out) {
  int dev = 0;
  MOSAIC_CUDA(cudaGetDevice(&dev));
  int max_bytes = 0;
  MOSAIC_CUDA(cudaDeviceGetAttribute(&max_bytes, cudaDevAttrMaxPersistingL2CacheSize, dev));
  size_t want = bytes < 0 ? 0 : static_cast<size_t>(bytes);
  if (want > static_cast<size_t>(max_bytes)) want = static_cast<size_t>(max_bytes);
  MOSAIC_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
  size_t got = 0;
  MOSAIC_CUDA(cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize));
  if (applied_out) *applied_out = static_cast<int64_t>(got);
  return MOSAIC_OK;
}
