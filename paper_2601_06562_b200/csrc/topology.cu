// SM -> L2-die map of this GPU, measured (the split is per physical part on
// B200: two dies, each L2 caching for its own SMs). The optional die split of
// K3's dynamic unit schedule uses it (die-0 pairs claim units from the front
// of the order, die-1 pairs from the back), so each die's m-groups stay in its
// own L2; off by default -- the undivided dynamic schedule measured better
// (DESIGN.md §4).
//
// Method (validated on B200, profiles/r01_die_probe.txt): one CTA reads a
// pool of lines (bringing each into its own die's L2 and into the line's home
// L2); then every SM times one cold read per line of a private 64 KB slice of
// the pool. Lines are homed on a die per 2 KB chunk; an SM on the reader's die
// finds every line near (~330 cycles), an SM on the other die finds the lines
// homed on the reader's die only across the die fabric (~690 cycles) -- about
// half of its slice. SMs with <10% slow reads share the reader's die.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace mosaic {
namespace {

constexpr int kLinesPerSm = 512;  // 64 KB = 32 two-KB homing chunks per SM
constexpr int kLineWords = 32;    // 128-byte lines

__global__ void topo_touch(const uint32_t* buf, int64_t n_lines, uint32_t* sink) {
  uint32_t acc = 0;
  for (int64_t i = threadIdx.x; i < n_lines; i += blockDim.x) acc += __ldcg(buf + i * kLineWords);
  if (acc == 0xFFFFFFFFu) sink[0] = acc;
  if (threadIdx.x == 0) {
    uint32_t s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    sink[1] = s;
  }
}

__global__ void topo_probe(const uint32_t* buf, uint32_t* lat, uint32_t* claimed, uint32_t* sink, int n_sm) {
  if (threadIdx.x != 0) return;
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (smid >= static_cast<uint32_t>(n_sm) || atomicCAS(claimed + smid, 0u, 1u) != 0u) return;
  for (int i = 0; i < kLinesPerSm; ++i) {
    const uint32_t* p = buf + (static_cast<int64_t>(smid) * kLinesPerSm + i) * kLineWords;
    const long long t0 = clock64();
    const uint32_t v = __ldcg(p);
    if (v == 0xFFFFFFFFu) sink[0] = v;  // keeps the load ahead of the second clock read
    const long long t1 = clock64();
    lat[smid * kLinesPerSm + i] = static_cast<uint32_t>(t1 - t0);
  }
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

// Eviction region: written in full before every round so the pool's lines are
// out of both dies' L2 (2x the L2 size). A discard.global.L2 of the pool
// instead left ~30 SMs with intermediate slow fractions; the full write gives
// a clean 0% / 50% split (profiles/r01_die_probe.txt).
static size_t flush_bytes() {
  int dev = 0, l2 = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  return 2 * static_cast<size_t>(l2 > 0 ? l2 : (128 << 20));
}

extern "C" size_t mosaic_die_map_scratch_bytes(int32_t n_sm) {
  return static_cast<size_t>(n_sm) * kLinesPerSm * (kLineWords * 4 + 4) + static_cast<size_t>(n_sm + 2) * 4 + 256 +
         flush_bytes();
}

extern "C" int mosaic_die_map(uint8_t* die_of_sm_host, int32_t n_sm, void* scratch, int32_t* n_die0_out,
                              int32_t* ambiguous_out, void* stream) {
  MOSAIC_REQUIRE(die_of_sm_host && scratch && n_sm >= 2 && n_sm <= 1024, "bad arguments");
  cudaStream_t s = as_stream(stream);
  const int64_t n_lines = static_cast<int64_t>(n_sm) * kLinesPerSm;
  uint32_t* buf = static_cast<uint32_t*>(scratch);
  uint32_t* lat = buf + n_lines * kLineWords;
  uint32_t* claimed = lat + n_lines;
  uint32_t* sink = claimed + n_sm;  // 2 words
  uint8_t* flush = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(sink + 2) + 255) & ~static_cast<uintptr_t>(255));
  // Three probe rounds (each: evict, touch from one CTA, time cold reads), the
  // slow-read counts summed per SM before classifying.
  constexpr int kRounds = 3;
  std::vector<int> slow(static_cast<size_t>(n_sm), 0), seen(static_cast<size_t>(n_sm), 0);
  std::vector<uint32_t> L(static_cast<size_t>(n_lines)), cl(static_cast<size_t>(n_sm));
  MOSAIC_CUDA(cudaMemsetAsync(buf, 1, static_cast<size_t>(n_lines) * kLineWords * 4, s));
  for (int round = 0; round < kRounds; ++round) {
    MOSAIC_CUDA(cudaMemsetAsync(claimed, 0, static_cast<size_t>(n_sm + 2) * 4, s));
    MOSAIC_CUDA(cudaMemsetAsync(flush, round + 2, flush_bytes(), s));  // pool out of every L2
    topo_touch<<<1, 256, 0, s>>>(buf, n_lines, sink);
    topo_probe<<<n_sm * 8, 32, 0, s>>>(buf, lat, claimed, sink, n_sm);
    MOSAIC_CUDA(cudaGetLastError());
    MOSAIC_CUDA(cudaMemcpyAsync(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost, s));
    MOSAIC_CUDA(cudaMemcpyAsync(cl.data(), claimed, cl.size() * 4, cudaMemcpyDeviceToHost, s));
    MOSAIC_CUDA(cudaStreamSynchronize(s));
    // the touching CTA's die is the reference: keep rounds consistent by
    // recording its SM and flipping a round whose toucher sits on the other die
    std::vector<uint32_t> all(L);
    std::nth_element(all.begin(), all.begin() + all.size() / 2, all.end());
    const uint32_t med = all[all.size() / 2];
    std::vector<int> round_slow(static_cast<size_t>(n_sm), -1);
    for (int sm = 0; sm < n_sm; ++sm) {
      if (!cl[sm]) continue;
      int c = 0;
      for (int i = 0; i < kLinesPerSm; ++i) c += L[static_cast<size_t>(sm) * kLinesPerSm + i] > med + 60;
      round_slow[sm] = c;
    }
    uint32_t toucher = 0;
    MOSAIC_CUDA(cudaMemcpy(&toucher, sink + 1, 4, cudaMemcpyDeviceToHost));
    // orientation: die 0 = round 0's toucher die. If this round's toucher reads
    // as slow in the accumulated map, its labels are inverted.
    bool flip = false;
    if (round > 0 && toucher < static_cast<uint32_t>(n_sm) && seen[toucher] > 0)
      flip = 100 * slow[toucher] / (seen[toucher] * kLinesPerSm) >= 25;
    for (int sm = 0; sm < n_sm; ++sm) {
      if (round_slow[sm] < 0) continue;
      slow[sm] += flip ? kLinesPerSm - round_slow[sm] : round_slow[sm];
      ++seen[sm];
    }
  }
  int n0 = 0, amb = 0;
  for (int sm = 0; sm < n_sm; ++sm) {
    if (!seen[sm]) {  // no probe CTA landed on this SM in any round: unknown
      die_of_sm_host[sm] = 255;
      ++amb;
      continue;
    }
    const int pct = 100 * slow[sm] / (seen[sm] * kLinesPerSm);
    if (pct >= 10 && pct < 25) ++amb;
    die_of_sm_host[sm] = pct < 10 ? 0 : 1;  // 0 = the first reading CTA's die
    n0 += pct < 10;
  }
  if (n_die0_out) *n_die0_out = n0;
  if (ambiguous_out) *ambiguous_out = amb;
  return MOSAIC_OK;
}
