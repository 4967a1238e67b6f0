// Microbenchmark: L2 -> shared memory feed rate per SM with cp.async (16-byte
// per lane, software-pipelined with commit/wait groups) versus a register-staged
// copy (ld.global.v4 -> st.shared.v4), from an L2-resident buffer, no MMA.
// Question: is K3 gather mode's A feed (~22 B/clk/SM) the ceiling of the
// per-lane copy paths, or an interaction with the tensor core's smem reads?
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

constexpr int kStageBytes = 16384;

template <int WARPS, int DEPTH>
__global__ void __launch_bounds__(WARPS * 32, 1) cpasync_feed(const uint4* src, int64_t n_vec, int iters,
                                                               unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  constexpr int kVecPerStage = kStageBytes / 16;
  constexpr int kPerThread = kVecPerStage / (WARPS * 32);
  const long long t0 = clock64();
  int64_t base = (static_cast<int64_t>(blockIdx.x) * 7919) % (n_vec - kVecPerStage);
  for (int it = 0; it < iters; ++it) {
    const int stage = it % DEPTH;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem + stage * kStageBytes));
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const int v = j * WARPS * 32 + tid;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + v * 16), "l"(src + base + v) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1) : "memory");
    base += kVecPerStage * 3;
    if (base + kVecPerStage >= n_vec) base -= n_vec - kVecPerStage - 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (tid == 0) atomicAdd(cycles, static_cast<unsigned long long>(clock64() - t0));
}

template <int WARPS, int DEPTH>
__global__ void __launch_bounds__(WARPS * 32, 1) reg_feed(const uint4* src, int64_t n_vec, int iters,
                                                           unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  constexpr int kVecPerStage = kStageBytes / 16;
  constexpr int kPerThread = kVecPerStage / (WARPS * 32);
  uint4 buf[DEPTH][kPerThread];
  const long long t0 = clock64();
  int64_t base = (static_cast<int64_t>(blockIdx.x) * 7919) % (n_vec - kVecPerStage);
  for (int it = 0; it < iters + DEPTH; ++it) {
    const int slot = it % DEPTH;
    if (it >= DEPTH) {  // store the stage loaded DEPTH iterations ago
      uint4* d = reinterpret_cast<uint4*>(smem + ((it - DEPTH) % 4) * kStageBytes);
#pragma unroll
      for (int j = 0; j < kPerThread; ++j) d[j * WARPS * 32 + tid] = buf[slot][j];
    }
    if (it < iters) {
#pragma unroll
      for (int j = 0; j < kPerThread; ++j) buf[slot][j] = __ldcg(src + base + j * WARPS * 32 + tid);
      base += kVecPerStage * 3;
      if (base + kVecPerStage >= n_vec) base -= n_vec - kVecPerStage - 1;
    }
  }
  __syncthreads();
  if (tid == 0) atomicAdd(cycles, static_cast<unsigned long long>(clock64() - t0) + (smem[5] == 255 ? 1 : 0));
}

template <typename K>
void run(const char* name, K kern, int threads, int smem_bytes, const uint4* src, int64_t n_vec, int n_sm) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  const int iters = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<n_sm, threads, smem_bytes>>>(src, n_vec, iters, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double bytes = double(n_sm) * iters * kStageBytes;
    const double avg_cyc = double(c) / n_sm;
    if (rep == 1)
      printf("%-28s %8.3f ms  %7.1f GB/s total  %6.1f B/clk/SM\n", name, ms, bytes / ms / 1e6,
             kStageBytes * double(iters) / avg_cyc);
  }
  cudaFree(cyc);
}

int main() {
  int n_sm = 0;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 48ll << 20;  // L2-resident source
  uint4* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  const int64_t n_vec = bytes / 16;
  run("cp.async 4 warps depth 2", cpasync_feed<4, 2>, 128, 2 * kStageBytes, src, n_vec, n_sm);
  run("cp.async 4 warps depth 4", cpasync_feed<4, 4>, 128, 4 * kStageBytes, src, n_vec, n_sm);
  run("cp.async 4 warps depth 8", cpasync_feed<4, 8>, 128, 8 * kStageBytes, src, n_vec, n_sm);
  run("cp.async 8 warps depth 4", cpasync_feed<8, 4>, 256, 4 * kStageBytes, src, n_vec, n_sm);
  run("cp.async 8 warps depth 8", cpasync_feed<8, 8>, 256, 8 * kStageBytes, src, n_vec, n_sm);
  run("cp.async 16 warps depth 8", cpasync_feed<16, 8>, 512, 8 * kStageBytes, src, n_vec, n_sm);
  run("regs 4 warps depth 2", reg_feed<4, 2>, 128, 4 * kStageBytes, src, n_vec, n_sm);
  run("regs 8 warps depth 2", reg_feed<8, 2>, 256, 4 * kStageBytes, src, n_vec, n_sm);
  run("regs 16 warps depth 2", reg_feed<16, 2>, 512, 4 * kStageBytes, src, n_vec, n_sm);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
