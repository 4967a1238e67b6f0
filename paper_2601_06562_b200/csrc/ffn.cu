// K6: fused SwiGLU of one FFN chunk, in place over the `up` rows:
// up[i] = silu(gate[i]) * up[i] (bf16 storage, fp32 math).
//
// Realises the `glu` op of the chunked FFN loop (mosaic/workload.py:249-259,
// in_place act <- up) whose rows are ceil(L / K_FFN) (x top_k for MoE). Pure
// streaming: 6 bytes of HBM traffic per element (read gate + up, write act),
// 16-byte vectors, grid sized to a whole number of waves over the SMs.
#include <cuda_bf16.h>

#include "common.cuh"

namespace mosaic {
namespace {

__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.f + __expf(-g)); }

__device__ __forceinline__ uint4 swiglu8(uint4 g, uint4 u) {
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
  __nv_bfloat162* u2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 gf = __bfloat1622float2(g2[j]);
    const float2 uf = __bfloat1622float2(u2[j]);
    u2[j] = __floats2bfloat162_rn(silu(gf.x) * uf.x, silu(gf.y) * uf.y);
  }
  return u;
}

// Each block streams contiguous 1024-vector (16 KB per operand) tiles: all of
// a thread's 4 (gate, up) vector pairs are loaded before any math, so 8
// independent 16-byte loads per thread are in flight; evict-first loads and
// streaming stores keep the chunk from displacing the GEMM operands in L2.
constexpr int kVecPerThread = 4;
constexpr int kK6Threads = 256;

__global__ void __launch_bounds__(kK6Threads) k6_swiglu(const uint4* __restrict__ gate, uint4* __restrict__ up,
                                                        int64_t n_vec) {
  constexpr int64_t kTile = static_cast<int64_t>(kK6Threads) * kVecPerThread;
  const int64_t n_full = n_vec / kTile;
  for (int64_t t = blockIdx.x; t < n_full; t += gridDim.x) {
    const int64_t base = t * kTile + threadIdx.x;
    uint4 g[kVecPerThread], u[kVecPerThread];
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      g[j] = __ldcs(gate + base + j * kK6Threads);
      u[j] = __ldcs(up + base + j * kK6Threads);
    }
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) __stcs(up + base + j * kK6Threads, swiglu8(g[j], u[j]));
  }
  // ragged vector tail (< one tile): plain grid-stride
  for (int64_t i = n_full * kTile + blockIdx.x * static_cast<int64_t>(kK6Threads) + threadIdx.x; i < n_vec;
       i += static_cast<int64_t>(gridDim.x) * kK6Threads)
    up[i] = swiglu8(__ldg(gate + i), up[i]);
}

__global__ void k6_swiglu_tail(const __nv_bfloat16* __restrict__ gate, __nv_bfloat16* __restrict__ up,
                               int64_t begin, int64_t n) {
  const int64_t i = begin + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) up[i] = __float2bfloat16(silu(__bfloat162float(gate[i])) * __bfloat162float(up[i]));
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

extern "C" int mosaic_swiglu(const uint16_t* gate, uint16_t* up, int64_t n, void* stream) {
  MOSAIC_REQUIRE(n >= 0, "negative element count");
  if (n == 0) return MOSAIC_OK;
  MOSAIC_REQUIRE(gate && up, "null operands");
  MOSAIC_REQUIRE((reinterpret_cast<uintptr_t>(gate) & 15) == 0 && (reinterpret_cast<uintptr_t>(up) & 15) == 0,
                 "gate/up must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  const int64_t n_vec = n / 8;
  if (n_vec > 0) {
    const int64_t want = ceil_div(n_vec, kK6Threads * kVecPerThread);
    const int64_t cap = static_cast<int64_t>(num_sms()) * 8;  // 8 resident 256-thread blocks per SM
    k6_swiglu<<<static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap), kK6Threads, 0, s>>>(
        reinterpret_cast<const uint4*>(gate), reinterpret_cast<uint4*>(up), n_vec);
  }
  const int64_t rest = n - n_vec * 8;
  if (rest > 0)
    k6_swiglu_tail<<<1, 32, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(gate),
                                   reinterpret_cast<__nv_bfloat16*>(up), n_vec * 8, n);
  return check_launch("mosaic_swiglu");
}
