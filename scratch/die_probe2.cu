// Probe v2: which L2 die serves each SM? SM0 (the first CTA's SM) first touches
// a pool of lines; then every SM times ONE cold load per line of its own
// private subset of that pool. A line homed on SM0's die and read from the
// other die misses the near L2 and crosses the die fabric; lines homed on the
// other die are replicated near SM0 and... (see notes in the printout). The
// per-SM fraction of slow lines should split the SMs into two groups.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

constexpr int LINES_PER_SM = 512;

__global__ void touch(const uint32_t* buf, int n_lines, uint32_t* sink, uint32_t* smid_out) {
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < n_lines; i += blockDim.x) acc += __ldcg(buf + i * 32);
  if (acc == 0xFFFFFFFF) sink[0] = acc;
  if (threadIdx.x == 0) {
    uint32_t s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    *smid_out = s;
  }
}

__global__ void probe(const uint32_t* buf, uint32_t* lat /*[n_sm][LINES_PER_SM]*/, uint32_t* sink) {
  if (threadIdx.x != 0) return;
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  // only the first CTA that lands on an SM measures (others exit)
  if (atomicCAS(sink + 1 + smid, 0u, 1u) != 0u) return;
  for (int i = 0; i < LINES_PER_SM; ++i) {
    const uint32_t* p = buf + (static_cast<int64_t>(smid) * LINES_PER_SM + i) * 32;
    long long t0 = clock64();
    uint32_t v = __ldcg(p);
    if (v == 0xFFFFFFFF) sink[0] = v;  // dependence: clock after the load returns
    long long t1 = clock64();
    lat[smid * LINES_PER_SM + i] = static_cast<uint32_t>(t1 - t0);
  }
}

int main() {
  int n_sm = 0;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  const int n_lines = n_sm * LINES_PER_SM;
  uint32_t *buf, *lat, *sink, *sm0;
  cudaMalloc(&buf, (size_t)n_lines * 128 * 4);
  cudaMemset(buf, 1, (size_t)n_lines * 128 * 4);
  cudaMalloc(&lat, n_sm * LINES_PER_SM * 4);
  cudaMalloc(&sink, (1 + 1024) * 4);
  cudaMalloc(&sm0, 4);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(sink, 0, (1 + 1024) * 4);
    // flush L2 by streaming a large buffer
    void* big;
    cudaMalloc(&big, 512ull << 20);
    cudaMemset(big, rep, 512ull << 20);
    cudaFree(big);
    touch<<<1, 256>>>(buf, n_lines, sink, sm0);
    probe<<<n_sm * 8, 32>>>(buf, lat, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<uint32_t> L(n_sm * LINES_PER_SM);
    uint32_t s0;
    cudaMemcpy(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&s0, sm0, 4, cudaMemcpyDeviceToHost);
    // per SM: median and fraction of "slow" loads (above global median + 60 cycles)
    std::vector<uint32_t> all(L);
    std::nth_element(all.begin(), all.begin() + all.size() / 2, all.end());
    const uint32_t med = all[all.size() / 2];
    printf("rep %d: toucher SM %u, global median %u cycles\n", rep, s0, med);
    int groupA = 0;
    std::vector<int> frac(n_sm);
    for (int s = 0; s < n_sm; ++s) {
      int slow = 0;
      for (int i = 0; i < LINES_PER_SM; ++i) slow += L[s * LINES_PER_SM + i] > med + 60;
      frac[s] = 100 * slow / LINES_PER_SM;
      groupA += frac[s] >= 25;
    }
    printf("  SMs with >=25%% slow lines: %d of %d\n  slow%%:", groupA, n_sm);
    for (int s = 0; s < n_sm; ++s) printf(" %d", frac[s]);
    printf("\n  die map (1 = toucher's die):\n  ");
    for (int s = 0; s < n_sm; ++s) printf("%d", frac[s] < 10 ? 1 : 0);
    printf("\n  ambiguous (10..25%%): ");
    for (int s = 0; s < n_sm; ++s) if (frac[s] >= 10 && frac[s] < 25) printf("%d ", s);
    printf("\n");
  }
  return 0;
}
