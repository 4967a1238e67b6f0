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

__device__ __forceinline__ float silu(float g) { return g / (1.f + __expf(-g)); }

__global__ void __launch_bounds__(256) k6_swiglu(const uint4* __restrict__ gate, uint4* __restrict__ up,
                                                 int64_t n_vec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_vec; i += stride) {
    const uint4 g = __ldg(gate + i);
    uint4 u = up[i];
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
    __nv_bfloat162* u2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 gf = __bfloat1622float2(g2[j]);
      const float2 uf = __bfloat1622float2(u2[j]);
      u2[j] = __floats2bfloat162_rn(silu(gf.x) * uf.x, silu(gf.y) * uf.y);
    }
    up[i] = u;
  }
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
    const int64_t want = ceil_div(n_vec, 256);
    const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
    k6_swiglu<<<static_cast<int>(want < cap ? want : cap), 256, 0, s>>>(
        reinterpret_cast<const uint4*>(gate), reinterpret_cast<uint4*>(up), n_vec);
  }
  const int64_t rest = n - n_vec * 8;
  if (rest > 0)
    k6_swiglu_tail<<<1, 32, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(gate),
                                   reinterpret_cast<__nv_bfloat16*>(up), n_vec * 8, n);
  return check_launch("mosaic_swiglu");
}
