// K11: rotary position embedding of the attention queries and keys, in place
// (bf16 storage, fp32 math), applied by the step executor's `fused_attention`
// op before the attention itself.
//
// The reference's layer template (mosaic/workload.py:207-229) is memory-only:
// q/k/v projections feed `fused_attention` and positions never appear. A
// numeric step needs them -- without positions every masked row of a
// random-init model sees the same MASK embedding and the same bidirectional
// context, so all masked rows end with identical hidden states and the remask
// has nothing to rank ("configs[0] selection check proves
// nothing"). This is the rotate-half RoPE of LLaDA / LLaMA: for head h and
// pair i < dh/2 at position p,
//   (x_i, x_{i+dh/2}) <- (x_i c - x_{i+dh/2} s, x_{i+dh/2} c + x_i s),
//   c, s = cos, sin(p * theta^(-2i/dh)),
// the angle formed in fp32 exactly as the torch reference
// (tests/torch_reference.py) forms it. Streaming: 8 B of HBM traffic per pair
// (read + write two bf16), one 16-byte vector of each half per thread.
#include <cuda_bf16.h>

#include "common.cuh"

namespace mosaic {
namespace {

constexpr int kRopeThreads = 256;

__global__ void __launch_bounds__(kRopeThreads)
    k11_rope(uint16_t* __restrict__ q, uint16_t* __restrict__ k, int64_t L, int32_t n_heads, int32_t head_dim,
             int64_t ld, const float* __restrict__ inv_freq, int64_t pos0) {
  const int half = head_dim / 2;
  const int vec_per_head = half / 8;
  const int64_t per_row = static_cast<int64_t>(n_heads) * vec_per_head;
  const int64_t total = 2 * L * per_row;  // q then k
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRopeThreads) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * kRopeThreads) {
    const int64_t which = i / (L * per_row);
    const int64_t rem = i - which * L * per_row;
    const int64_t row = rem / per_row;
    const int64_t hv = rem - row * per_row;
    const int h = static_cast<int>(hv / vec_per_head);
    const int j0 = static_cast<int>(hv - static_cast<int64_t>(h) * vec_per_head) * 8;  // first pair of the vector
    uint16_t* base = (which == 0 ? q : k) + row * ld + static_cast<int64_t>(h) * head_dim;
    uint4* lo_p = reinterpret_cast<uint4*>(base + j0);
    uint4* hi_p = reinterpret_cast<uint4*>(base + half + j0);
    uint4 lo = *lo_p, hi = *hi_p;
    __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&lo);
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&hi);
    const float p = static_cast<float>(row + pos0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 a = __bfloat1622float2(l2[j]);
      const float2 b = __bfloat1622float2(h2[j]);
      float s0, c0, s1, c1;
      sincosf(p * __ldg(inv_freq + j0 + 2 * j), &s0, &c0);
      sincosf(p * __ldg(inv_freq + j0 + 2 * j + 1), &s1, &c1);
      l2[j] = __floats2bfloat162_rn(a.x * c0 - b.x * s0, a.y * c1 - b.y * s1);
      h2[j] = __floats2bfloat162_rn(b.x * c0 + a.x * s0, b.y * c1 + a.y * s1);
    }
    *lo_p = lo;
    *hi_p = hi;
  }
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

extern "C" int mosaic_rope_qk(uint16_t* q, uint16_t* k, int64_t L, int32_t n_heads, int32_t head_dim, int64_t ld,
                              const float* inv_freq, int64_t pos0, void* stream) {
  MOSAIC_REQUIRE(L >= 0 && n_heads >= 1 && head_dim >= 16 && head_dim % 16 == 0,
                 "rope needs head_dim a multiple of 16 (got %d)", head_dim);
  MOSAIC_REQUIRE(ld >= static_cast<int64_t>(n_heads) * head_dim && ld % 8 == 0, "row stride %lld", (long long)ld);
  if (L == 0) return MOSAIC_OK;
  MOSAIC_REQUIRE(q && k && inv_freq, "null operands");
  MOSAIC_REQUIRE((reinterpret_cast<uintptr_t>(q) & 15) == 0 && (reinterpret_cast<uintptr_t>(k) & 15) == 0,
                 "q/k must be 16-byte aligned");
  const int64_t total = 2 * L * n_heads * (head_dim / 16);
  const int64_t want = ceil_div(total, kRopeThreads);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  k11_rope<<<static_cast<int>(want < cap ? want : cap), kRopeThreads, 0, as_stream(stream)>>>(
      q, k, L, n_heads, head_dim, ld, inv_freq, pos0);
  return check_launch("mosaic_rope_qk");
}
