// K7b: the arena's torch-scratch region as a PyTorch pluggable allocator.
//
// The reference's contract is one workspace per step, reserved once and
// committed up to the plan's size (mosaic/vmm.py:48-147), with the budget
// covering everything the step holds (mosaic/workload.py:362-369). The step
// executor plans every activation at a first-fit offset of the cuMem arena;
// what it cannot plan are the temporaries library calls make through torch's
// allocator (the attention output of scaled_dot_product_attention). Those are
// routed into a region at the start of the same arena: each executor binds its
// arena's [base, base + size), selects it before a step, and runs the step's
// ops under a torch.cuda.MemPool whose allocator is mosaic_pool_alloc /
// mosaic_pool_free. torch's caching allocator asks for a few segments on the
// first step and recycles them afterwards, so steady-state steps make no
// allocator calls at all, and nothing the step touches lies outside the
// arena. Host-only code: per region, first-fit over an offset-ordered free
// map with coalescing frees; no device calls (the region is committed cuMem).
#include <cstdint>
#include <iterator>
#include <map>
#include <mutex>

#include "common.cuh"

namespace mosaic {
namespace {

constexpr int kMaxDevices = 64;
constexpr uint64_t kAlign = 512;

struct Region {
  uint64_t size = 0;
  std::map<uint64_t, uint64_t> free_;  // offset -> length
  std::map<uint64_t, uint64_t> used;   // offset -> length
  uint64_t in_use = 0, high = 0, n_alloc = 0, n_fail = 0;
};

struct DevicePools {
  std::map<uintptr_t, Region> regions;  // by base address (one per executor arena)
  uintptr_t current = 0;                // region new allocations come from
};

std::mutex& mu() {
  static std::mutex m;
  return m;
}

DevicePools& pools(int device) {
  static DevicePools p[kMaxDevices];
  return p[device];
}

void add_free(Region& r, uint64_t start, uint64_t len) {
  auto next = r.free_.lower_bound(start);
  if (next != r.free_.end() && start + len == next->first) {  // coalesce with the following hole
    len += next->second;
    next = r.free_.erase(next);
  }
  if (next != r.free_.begin()) {  // and with the preceding one
    auto prev = std::prev(next);
    if (prev->first + prev->second == start) {
      start = prev->first;
      len += prev->second;
      r.free_.erase(prev);
    }
  }
  r.free_[start] = len;
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

extern "C" int mosaic_pool_bind(int32_t device, void* base, uint64_t size) {
  MOSAIC_REQUIRE(device >= 0 && device < kMaxDevices, "device %d out of range", device);
  MOSAIC_REQUIRE(base != nullptr && size > 0, "empty region");
  MOSAIC_REQUIRE((reinterpret_cast<uintptr_t>(base) & (kAlign - 1)) == 0, "region must be %llu-byte aligned",
                 (unsigned long long)kAlign);
  std::lock_guard<std::mutex> lock(mu());
  Region& r = pools(device).regions[reinterpret_cast<uintptr_t>(base)];
  if (size < r.size) {  // shrink: only the untouched tail may go
    for (const auto& u : r.used)
      if (u.first + u.second > size)
        return fail(MOSAIC_E_INPUT, "cannot shrink the scratch region below a live block");
    auto last = r.free_.empty() ? r.free_.end() : std::prev(r.free_.end());
    if (last == r.free_.end() || last->first + last->second != r.size || last->first > size)
      return fail(MOSAIC_E_INPUT, "cannot shrink the scratch region below a live block");
    const uint64_t start = last->first;
    r.free_.erase(last);
    if (start < size) r.free_[start] = size - start;
  } else if (size > r.size) {  // create or grow in place: live blocks stay valid
    add_free(r, r.size, size - r.size);
  }
  r.size = size;
  return MOSAIC_OK;
}

extern "C" int mosaic_pool_select(int32_t device, void* base) {
  MOSAIC_REQUIRE(device >= 0 && device < kMaxDevices, "device %d out of range", device);
  std::lock_guard<std::mutex> lock(mu());
  DevicePools& p = pools(device);
  const uintptr_t b = reinterpret_cast<uintptr_t>(base);
  MOSAIC_REQUIRE(b == 0 || p.regions.count(b), "no scratch region bound at %p", base);
  p.current = b;
  return MOSAIC_OK;
}

extern "C" int mosaic_pool_unbind(int32_t device, void* base) {
  MOSAIC_REQUIRE(device >= 0 && device < kMaxDevices, "device %d out of range", device);
  std::lock_guard<std::mutex> lock(mu());
  DevicePools& p = pools(device);
  const uintptr_t b = reinterpret_cast<uintptr_t>(base);
  p.regions.erase(b);  // the arena is going away: its blocks with it
  if (p.current == b) p.current = 0;
  return MOSAIC_OK;
}

extern "C" void* mosaic_pool_alloc(ssize_t size, int device, void* /*stream*/) {
  if (device < 0 || device >= kMaxDevices || size < 0) return nullptr;
  std::lock_guard<std::mutex> lock(mu());
  DevicePools& p = pools(device);
  auto reg = p.regions.find(p.current);
  if (reg == p.regions.end()) return nullptr;
  Region& r = reg->second;
  const uint64_t want = (static_cast<uint64_t>(size) + kAlign - 1) & ~(kAlign - 1);
  for (auto it = r.free_.begin(); it != r.free_.end(); ++it) {
    if (it->second < want) continue;
    const uint64_t off = it->first, len = it->second;
    r.free_.erase(it);
    if (len > want) r.free_[off + want] = len - want;
    r.used[off] = want;
    r.in_use += want;
    r.high = r.in_use > r.high ? r.in_use : r.high;
    ++r.n_alloc;
    return reinterpret_cast<void*>(reg->first + off);
  }
  ++r.n_fail;  // torch raises its out-of-memory error: the region was sized too small, loudly
  return nullptr;
}

extern "C" void mosaic_pool_free(void* ptr, ssize_t /*size*/, int device, void* /*stream*/) {
  if (ptr == nullptr || device < 0 || device >= kMaxDevices) return;
  std::lock_guard<std::mutex> lock(mu());
  DevicePools& p = pools(device);
  const uintptr_t a = reinterpret_cast<uintptr_t>(ptr);
  auto reg = p.regions.upper_bound(a);  // the region with the largest base <= a
  if (reg == p.regions.begin()) return;
  --reg;
  Region& r = reg->second;
  const uint64_t off = a - reg->first;
  auto u = r.used.find(off);
  if (u == r.used.end()) return;  // not a block of a live region: ignore
  const uint64_t len = u->second;
  r.in_use -= len;
  r.used.erase(u);
  add_free(r, off, len);
}

extern "C" int mosaic_pool_stats(int32_t device, void* base, uint64_t* in_use, uint64_t* high_water,
                                 uint64_t* n_alloc, uint64_t* n_fail) {
  MOSAIC_REQUIRE(device >= 0 && device < kMaxDevices, "device %d out of range", device);
  MOSAIC_REQUIRE(in_use && high_water && n_alloc && n_fail, "null outputs");
  std::lock_guard<std::mutex> lock(mu());
  DevicePools& p = pools(device);
  auto reg = p.regions.find(reinterpret_cast<uintptr_t>(base));
  MOSAIC_REQUIRE(reg != p.regions.end(), "no scratch region bound at %p", base);
  *in_use = reg->second.in_use;
  *high_water = reg->second.high;
  *n_alloc = reg->second.n_alloc;
  *n_fail = reg->second.n_fail;
  return MOSAIC_OK;
}
