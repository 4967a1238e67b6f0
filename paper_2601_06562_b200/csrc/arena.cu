// K7: contiguous device workspace with lazy physical commitment over the CUDA
// virtual-memory API (cuMemAddressReserve / cuMemCreate / cuMemMap /
// cuMemSetAccess / cuMemUnmap / cuMemRelease).
//
// Mirrors the reference Workspace (mosaic/vmm.py:48-139): one virtual range is
// reserved up front (vmm.py:68-76 does mmap PROT_NONE) and a prefix
// [0, round_up(target, granularity)) is backed by physical memory
// (vmm.py:78-100 does mprotect/madvise). Physical memory is created one
// allocation granule (2 MiB on B200) per handle, so the prefix can grow or
// shrink at granule resolution without moving or losing the bytes below the
// new target. The invariant committed - target < granularity is the device
// analogue of the reference's "within one page of the planned peak".
#include <vector>

#include "common.cuh"

struct mosaic_arena {
  int device = 0;
  CUdeviceptr base = 0;
  uint64_t reserved = 0;
  uint64_t committed = 0;
  uint64_t granularity = 0;
  std::vector<CUmemGenericAllocationHandle> handles;  // one per mapped granule, in order
};

namespace mosaic {
namespace {

struct Driver {
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  bool ok = false;
};

const Driver& drv() {
  static Driver d = [] {
    Driver x;
    x.granularity = reinterpret_cast<decltype(x.granularity)>(driver_fn("cuMemGetAllocationGranularity"));
    x.reserve = reinterpret_cast<decltype(x.reserve)>(driver_fn("cuMemAddressReserve"));
    x.addr_free = reinterpret_cast<decltype(x.addr_free)>(driver_fn("cuMemAddressFree"));
    x.create = reinterpret_cast<decltype(x.create)>(driver_fn("cuMemCreate"));
    x.release = reinterpret_cast<decltype(x.release)>(driver_fn("cuMemRelease"));
    x.map = reinterpret_cast<decltype(x.map)>(driver_fn("cuMemMap"));
    x.unmap = reinterpret_cast<decltype(x.unmap)>(driver_fn("cuMemUnmap"));
    x.set_access = reinterpret_cast<decltype(x.set_access)>(driver_fn("cuMemSetAccess"));
    x.ok = x.granularity && x.reserve && x.addr_free && x.create && x.release && x.map && x.unmap &&
           x.set_access;
    return x;
  }();
  return d;
}

CUmemAllocationProp device_prop(int device) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  return prop;
}

int shrink_to(mosaic_arena* a, uint64_t new_bytes) {
  const Driver& d = drv();
  while (a->committed > new_bytes) {
    const uint64_t off = a->committed - a->granularity;
    CUresult r = d.unmap(a->base + off, a->granularity);
    if (r != CUDA_SUCCESS) return fail(MOSAIC_E_RESOURCE, "cuMemUnmap failed (%d)", int(r));
    d.release(a->handles.back());
    a->handles.pop_back();
    a->committed = off;
  }
  return MOSAIC_OK;
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

extern "C" int mosaic_arena_reserve(int32_t device, uint64_t reserve_bytes, mosaic_arena** out) {
  MOSAIC_REQUIRE(out != nullptr, "null output handle");
  MOSAIC_REQUIRE(reserve_bytes > 0, "reserve size must be positive");
  const Driver& d = drv();
  if (!d.ok) return fail(MOSAIC_E_RESOURCE, "CUDA VMM driver entry points unavailable");
  MOSAIC_CUDA(cudaSetDevice(device));
  MOSAIC_CUDA(cudaFree(nullptr));  // make sure the primary context exists
  CUmemAllocationProp prop = device_prop(device);
  size_t gran = 0;
  CUresult r = d.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  if (r != CUDA_SUCCESS || gran == 0)
    return fail(MOSAIC_E_RESOURCE, "cuMemGetAllocationGranularity failed (%d)", int(r));
  auto* a = new mosaic_arena();
  a->device = device;
  a->granularity = gran;
  a->reserved = ceil_div(static_cast<int64_t>(reserve_bytes), static_cast<int64_t>(gran)) * gran;
  r = d.reserve(&a->base, a->reserved, gran, 0, 0);
  if (r != CUDA_SUCCESS) {
    delete a;
    return fail(MOSAIC_E_RESOURCE, "cuMemAddressReserve of %llu bytes failed (%d)",
                (unsigned long long)reserve_bytes, int(r));
  }
  *out = a;
  return MOSAIC_OK;
}

extern "C" int mosaic_arena_commit(mosaic_arena* a, uint64_t target_bytes) {
  MOSAIC_REQUIRE(a != nullptr, "null arena");
  if (target_bytes > a->reserved)
    return fail(MOSAIC_E_CAPACITY, "commit target %llu exceeds reservation %llu",
                (unsigned long long)target_bytes, (unsigned long long)a->reserved);
  const Driver& d = drv();
  const uint64_t want = ceil_div(static_cast<int64_t>(target_bytes), a->granularity) * a->granularity;
  if (want < a->committed) return shrink_to(a, want);
  if (want == a->committed) return MOSAIC_OK;
  const uint64_t start = a->committed;
  CUmemAllocationProp prop = device_prop(a->device);
  while (a->committed < want) {
    CUmemGenericAllocationHandle h;
    CUresult r = d.create(&h, a->granularity, &prop, 0);
    if (r != CUDA_SUCCESS) {
      shrink_to(a, start);
      return fail(MOSAIC_E_RESOURCE, "cuMemCreate failed at %llu bytes (%d)",
                  (unsigned long long)a->committed, int(r));
    }
    r = d.map(a->base + a->committed, a->granularity, 0, h, 0);
    if (r != CUDA_SUCCESS) {
      d.release(h);
      shrink_to(a, start);
      return fail(MOSAIC_E_RESOURCE, "cuMemMap failed (%d)", int(r));
    }
    a->handles.push_back(h);
    a->committed += a->granularity;
  }
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = a->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUresult r = d.set_access(a->base + start, want - start, &acc, 1);
  if (r != CUDA_SUCCESS) {
    shrink_to(a, start);
    return fail(MOSAIC_E_RESOURCE, "cuMemSetAccess failed (%d)", int(r));
  }
  return MOSAIC_OK;
}

extern "C" int mosaic_arena_info(const mosaic_arena* a, uint64_t* base, uint64_t* reserved,
                                 uint64_t* committed, uint64_t* granularity) {
  MOSAIC_REQUIRE(a != nullptr, "null arena");
  if (base) *base = a->base;
  if (reserved) *reserved = a->reserved;
  if (committed) *committed = a->committed;
  if (granularity) *granularity = a->granularity;
  return MOSAIC_OK;
}

extern "C" int mosaic_arena_release(mosaic_arena* a) {
  if (a == nullptr) return MOSAIC_OK;
  cudaDeviceSynchronize();  // no kernel may still touch the range
  int st = shrink_to(a, 0);
  drv().addr_free(a->base, a->reserved);
  delete a;
  return st;
}

// ---------------------------------------------------------------- canaries
// Plan-executor canaries on the device (mosaic/vmm.py:188-291 `execute_plan`):
// a defined group's range is filled with its 8-byte tag repeated from the
// range start; a read verifies the whole range still carries it, so any
// overlap between simultaneously live groups shows up even away from the
// range start.
namespace mosaic {
namespace {

__device__ __forceinline__ uint8_t tag_byte(uint64_t tag, int64_t i) {
  return static_cast<uint8_t>(tag >> (8 * (i & 7)));
}

__global__ void k7_tag_fill(uint8_t* p, int64_t n, uint64_t tag) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n8 = n / 8;
  uint64_t* p8 = reinterpret_cast<uint64_t*>(p);  // range starts are plan-aligned (>= 8 B)
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8; i += stride) p8[i] = tag;
  for (int64_t i = n8 * 8 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    p[i] = tag_byte(tag, i);
}

__global__ void k7_tag_check(const uint8_t* p, int64_t n, uint64_t tag, unsigned int* bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n8 = n / 8;
  const uint64_t* p8 = reinterpret_cast<const uint64_t*>(p);
  bool ok = true;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8; i += stride) ok &= p8[i] == tag;
  for (int64_t i = n8 * 8 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    ok &= p[i] == tag_byte(tag, i);
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicAdd(bad, 1u);
}

int tag_grid(int64_t n) {
  const int64_t want = ceil_div(n / 8 > 0 ? n / 8 : 1, 256);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 4;
  return static_cast<int>(want < cap ? want : cap);
}

}  // namespace
}  // namespace mosaic

extern "C" int mosaic_tag_fill(void* ptr, int64_t nbytes, uint64_t tag, void* stream) {
  MOSAIC_REQUIRE(nbytes >= 0, "negative size");
  if (nbytes == 0) return MOSAIC_OK;
  MOSAIC_REQUIRE(ptr && (reinterpret_cast<uintptr_t>(ptr) & 7) == 0, "range must be 8-byte aligned");
  k7_tag_fill<<<tag_grid(nbytes), 256, 0, as_stream(stream)>>>(static_cast<uint8_t*>(ptr), nbytes, tag);
  return check_launch("mosaic_tag_fill");
}

extern "C" int mosaic_tag_check(const void* ptr, int64_t nbytes, uint64_t tag, uint32_t* mismatch_count,
                                void* stream) {
  MOSAIC_REQUIRE(nbytes >= 0 && mismatch_count, "bad arguments");
  if (nbytes == 0) return MOSAIC_OK;
  MOSAIC_REQUIRE(ptr && (reinterpret_cast<uintptr_t>(ptr) & 7) == 0, "range must be 8-byte aligned");
  k7_tag_check<<<tag_grid(nbytes), 256, 0, as_stream(stream)>>>(static_cast<const uint8_t*>(ptr), nbytes, tag,
                                                                 mismatch_count);
  return check_launch("mosaic_tag_check");
}
