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
// (read + write two bf16), 16-byte vectors of each half.
#include <cuda_bf16.h>

#include "common.cuh"

namespace mosaic {
namespace {

constexpr int kRopeThreads = 256;
constexpr int kHeadsPerThread = 8;  // heads sharing one thread's angles

// One thread: row `row`, pair vector jv (8 consecutive pairs of every head),
// a chunk of kHeadsPerThread heads, q and k. The 8 angles depend on (row, jv)
// only, so they are formed once and applied to 2 x kHeadsPerThread vector
// pairs (round 1 formed them per head and per tensor: 64x the sincosf work,
// which made the pass compute-bound at 0.58 of HBM). Consecutive threads take
// consecutive jv, then head chunks, so each head-iteration of a warp touches
// whole 128-byte runs of the lo and hi halves.
__global__ void __launch_bounds__(kRopeThreads)
    k11_rope(uint16_t* __restrict__ q, uint16_t* __restrict__ k, int64_t L, int32_t n_heads, int32_t head_dim,
             int64_t ld, const float* __restrict__ inv_freq, int64_t pos0) {
  const int half = head_dim / 2;
  const int vec_per_half = half / 8;
  const int chunks = (n_heads + kHeadsPerThread - 1) / kHeadsPerThread;
  const int per_row = vec_per_half * chunks;
  const int64_t total = L * per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRopeThreads) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * kRopeThreads) {
    const int64_t row = i / per_row;
    const int r = static_cast<int>(i - row * per_row);
    const int chunk = r / vec_per_half;
    const int j0 = (r - chunk * vec_per_half) * 8;  // first pair of the vector
    const float p = static_cast<float>(row + pos0);
    float c[8], sn[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) sincosf(p * __ldg(inv_freq + j0 + j), &sn[j], &c[j]);
    const int h_end = min(n_heads, (chunk + 1) * kHeadsPerThread);
    for (int h = chunk * kHeadsPerThread; h < h_end; ++h) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        uint16_t* base = (t == 0 ? q : k) + row * ld + static_cast<int64_t>(h) * head_dim;
        uint4* lo_p = reinterpret_cast<uint4*>(base + j0);
        uint4* hi_p = reinterpret_cast<uint4*>(base + half + j0);
        uint4 lo = *lo_p, hi = *hi_p;
        __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&lo);
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&hi);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 a = __bfloat1622float2(l2[j]);
          const float2 b = __bfloat1622float2(h2[j]);
          l2[j] = __floats2bfloat162_rn(a.x * c[2 * j] - b.x * sn[2 * j], a.y * c[2 * j + 1] - b.y * sn[2 * j + 1]);
          h2[j] = __floats2bfloat162_rn(b.x * c[2 * j] + a.x * sn[2 * j], b.y * c[2 * j + 1] + a.y * sn[2 * j + 1]);
        }
        *lo_p = lo;
        *hi_p = hi;
      }
    }
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
  const int64_t total = L * ((n_heads + kHeadsPerThread - 1) / kHeadsPerThread) * (head_dim / 16);
  const int64_t want = ceil_div(total, kRopeThreads);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
  k11_rope<<<static_cast<int>(want < cap ? want : cap), kRopeThreads, 0, as_stream(stream)>>>(
      q, k, L, n_heads, head_dim, ld, inv_freq, pos0);
  return check_launch("mosaic_rope_qk");
}
