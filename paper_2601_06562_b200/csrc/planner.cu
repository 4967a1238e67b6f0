// Native first-fit workspace planner (host code): the production placement of
// mosaic/planner.py:107-142 (`_first_fit_offsets` / `plan_first_fit`), whose
// offsets become arena offsets on the device. The Python control plane sorts
// the storage groups into placement order (def asc, size desc, id asc) and
// hands the sizes and live intervals here; each group goes to the lowest
// aligned offset that collides with no already-placed, lifetime-overlapping
// group. Called once per denoising step, so it must cost well under a
// millisecond at thousands of groups: when the defs arrive non-decreasing (the
// default order) groups whose interval ended before the current def are
// retired from the active set, so each placement only scans live neighbours.
#include <algorithm>
#include <utility>
#include <vector>

#include "common.cuh"

extern "C" int mosaic_first_fit(int64_t n, const int64_t* sizes, const int64_t* def_idx,
                                const int64_t* last_idx, int64_t alignment, int64_t* offsets_out,
                                int64_t* workspace_out) {
  MOSAIC_REQUIRE(n >= 0, "negative group count");
  MOSAIC_REQUIRE(alignment >= 1 && (alignment & (alignment - 1)) == 0,
                 "alignment must be a power of two >= 1, got %lld", (long long)alignment);
  MOSAIC_REQUIRE(n == 0 || (sizes && def_idx && last_idx && offsets_out), "null arrays");
  auto up = [alignment](int64_t x) { return (x + alignment - 1) & ~(alignment - 1); };
  std::vector<int64_t> active;  // placed groups that may still overlap later ones
  active.reserve(static_cast<size_t>(n < 4096 ? n : 4096));
  std::vector<std::pair<int64_t, int64_t>> busy;
  bool sorted_defs = true;  // retiring is only sound when later defs never go back in time
  for (int64_t i = 0; i < n; ++i) {
    MOSAIC_REQUIRE(sizes[i] >= 0 && def_idx[i] <= last_idx[i], "group %lld: bad size/interval", (long long)i);
    if (i > 0 && def_idx[i] < def_idx[i - 1]) sorted_defs = false;
  }
  int64_t workspace = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (sizes[i] == 0) {
      offsets_out[i] = 0;
      continue;
    }
    busy.clear();
    size_t keep = 0;
    for (size_t a = 0; a < active.size(); ++a) {
      const int64_t j = active[a];
      if (sorted_defs && last_idx[j] < def_idx[i]) continue;  // retired: ends before every later def
      active[keep++] = j;
      if (def_idx[j] <= last_idx[i] && def_idx[i] <= last_idx[j])
        busy.emplace_back(offsets_out[j], offsets_out[j] + sizes[j]);
    }
    active.resize(keep);
    std::sort(busy.begin(), busy.end());
    int64_t at = 0;
    for (const auto& r : busy) {
      if (at + sizes[i] <= r.first) break;  // the gap below this range holds the group
      at = std::max(at, up(r.second));
    }
    offsets_out[i] = at;
    workspace = std::max(workspace, at + sizes[i]);
    active.push_back(i);
  }
  if (workspace_out) *workspace_out = workspace;
  return MOSAIC_OK;
}
