// Probe: TMA tile::gather4 semantics on sm_100a. Loads a 128-row x 64-col bf16
// A tile (128B swizzle) two ways -- (1) 32 gather4 ops from H by row index,
// (2) one plain 2D TMA box from the pre-gathered dense Hc -- and compares the
// shared-memory bytes. Tries tensor-map box heights 1 and 4.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstring>

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tg, const __grid_constant__ CUtensorMap td,
                      const int* idx, int col0, uint8_t* out_g, uint8_t* out_d) {
  extern __shared__ uint8_t raw[];
  uint8_t* s = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sg = s;            // 16 KB
  uint8_t* sd = s + 16384;    // 16 KB
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[0])), "r"(16384) : "memory");
    for (int i = 0; i < 32; ++i) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(sg + i * 512)),
          "l"((uint64_t)&tg), "r"(smem_u32(&bar[0])), "r"(col0), "r"(idx[4 * i]), "r"(idx[4 * i + 1]),
          "r"(idx[4 * i + 2]), "r"(idx[4 * i + 3])
          : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[1])), "r"(16384) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(sd)), "l"((uint64_t)&td), "r"(smem_u32(&bar[1])), "r"(col0), "r"(0)
        : "memory");
  }
  for (int b = 0; b < 2; ++b) {
    uint32_t ok = 0;
    long spins = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar[b])) : "memory");
      if (++spins > (1l << 26)) { if (threadIdx.x == 0) printf("timeout bar %d\n", b); return; }
    }
  }
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) {
    out_g[i] = sg[i];
    out_d[i] = sd[i];
  }
}

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  const int L = 1000, d = 256, M = 128;
  std::vector<uint16_t> H(L * d);
  for (int i = 0; i < L * d; ++i) H[i] = (uint16_t)(i * 2654435761u >> 16);
  std::vector<int> idx(M);
  for (int i = 0; i < M; ++i) idx[i] = (i * 7 + 3) % L;
  std::vector<uint16_t> Hc(M * d);
  for (int i = 0; i < M; ++i) memcpy(&Hc[i * d], &H[idx[i] * d], d * 2);
  uint16_t *dH, *dHc;
  int* didx;
  uint8_t *og, *od;
  cudaMalloc(&dH, L * d * 2); cudaMalloc(&dHc, M * d * 2); cudaMalloc(&didx, M * 4);
  cudaMalloc(&og, 16384); cudaMalloc(&od, 16384);
  cudaMemcpy(dH, H.data(), L * d * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dHc, Hc.data(), M * d * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(didx, idx.data(), M * 4, cudaMemcpyHostToDevice);
  int* hidx_dev_unused = nullptr; (void)hidx_dev_unused;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int boxh : {1, 4}) {
    CUtensorMap tg, td;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)L}, strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxh}, es[2] = {1, 1};
    CUresult r1 = enc(&tg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dH, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t dims2[2] = {(cuuint64_t)d, (cuuint64_t)M};
    cuuint32_t box2[2] = {64, 128};
    CUresult r2 = enc(&td, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dHc, dims2, strides, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("boxh=%d encode gather=%d dense=%d\n", boxh, (int)r1, (int)r2);
    if (r1 || r2) continue;
    // row indices passed as kernel args through a host copy: kernel reads idx from device memory
    for (int col0 : {0, 64, 192}) {
      cudaMemset(og, 0xAB, 16384); cudaMemset(od, 0xCD, 16384);
      probe<<<1, 128, 40000>>>(tg, td, didx, col0, og, od);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("  col0=%d launch error %s\n", col0, cudaGetErrorString(e)); return 1; }
      std::vector<uint8_t> a(16384), b(16384);
      cudaMemcpy(a.data(), og, 16384, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), od, 16384, cudaMemcpyDeviceToHost);
      int diff = 0, first = -1;
      for (int i = 0; i < 16384; ++i) if (a[i] != b[i]) { if (first < 0) first = i; ++diff; }
      printf("  col0=%d differing bytes=%d first=%d\n", col0, diff, first);
    }
  }
  return 0;
}
