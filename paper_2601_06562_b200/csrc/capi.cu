// C-ABI plumbing shared by every entry point: thread-local error messages,
// launch checking, device properties and driver entry-point lookup.
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
