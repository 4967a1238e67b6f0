// K8 expert routing + dispatch order and K9 weighted combine for the lazily
// chunked MoE FFN (BASELINE configs[3], "LLaDA-MoE shape at seq 64k").
//
// The reference models MoE only as a footprint multiplier: the FFN chunk's
// up/gate/act tensors have ceil(L/K_FFN) * top_k rows (mosaic/workload.py:195,
// 238-253). Executing it needs the routing those rows stand for:
//
//   K8a  per token row: top-k experts of the router logits (logit desc, expert
//        id asc on ties), weights = softmax over the k selected logits, and a
//        per-CTA expert histogram;
//   K8b  one exclusive scan over the (expert, CTA) histogram in expert-major
//        order -> expert segment offsets and every CTA's base per expert;
//   K8c  stable scatter: assignment (row, j) gets position base[e][cta] + its
//        rank among the CTA's earlier assignments to e (warp match_any), so
//        the dispatch order is (expert, row, j) ascending -- deterministic,
//        no atomics on global memory.
//
// The dispatch rows then go through K2 (gather), the per-expert GEMMs, K6
// (SwiGLU), and K9 folds the k expert outputs of every token back into its
// row: out[r] = sum_j w[r, j] * down_e[pos[r, j]] in fp32, fixed j order.
#include <cuda_bf16.h>

#include "common.cuh"

namespace mosaic {
namespace {

constexpr int kRouteThreads = 256;                 // 8 warps
constexpr int kRowsPerWarp = 8;
constexpr int kRowsPerCta = (kRouteThreads / 32) * kRowsPerWarp;  // 64 token rows per CTA
constexpr int kMaxExperts = 256;
constexpr int kMaxTopK = 16;
constexpr int kScanThreads = 1024;

// K8a: top-k + softmax weights per row, expert histogram per CTA.
__global__ void __launch_bounds__(kRouteThreads)
    k8_topk(const float* __restrict__ logits, int64_t ld, int64_t rows, int32_t E, int32_t k,
            int32_t* __restrict__ sel_e, float* __restrict__ sel_w, int32_t* __restrict__ hist) {
  __shared__ int32_t cnt[kMaxExperts];
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per_lane = (E + 31) / 32;  // <= 8
  for (int rr = 0; rr < kRowsPerWarp; ++rr) {
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + warp * kRowsPerWarp + rr;
    if (row >= rows) break;  // warp-uniform
    float v[kMaxExperts / 32];
#pragma unroll
    for (int i = 0; i < kMaxExperts / 32; ++i) {
      const int e = i * 32 + lane;
      v[i] = (i < per_lane && e < E) ? logits[row * ld + e] : -INFINITY;
    }
    float top_logit[kMaxTopK];
    int top_e[kMaxTopK];
    for (int j = 0; j < k; ++j) {
      // lane-local best (lowest expert id on ties: i ascending, strict >)
      float bv = -INFINITY;
      int be = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < kMaxExperts / 32; ++i) {
        const int e = i * 32 + lane;
        if (i < per_lane && e < E && (v[i] > bv || (v[i] == bv && e < be))) {
          bv = v[i];
          be = e;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oe = __shfl_xor_sync(0xffffffffu, be, o);
        if (ov > bv || (ov == bv && oe < be)) {
          bv = ov;
          be = oe;
        }
      }
      top_logit[j] = bv;
      top_e[j] = be;
#pragma unroll
      for (int i = 0; i < kMaxExperts / 32; ++i)
        if (i * 32 + lane == be) v[i] = -INFINITY;  // the owning lane drops it
    }
    // softmax over the selected logits (top_logit[0] is the max)
    float z = 0.f;
    for (int j = 0; j < k; ++j) z += __expf(top_logit[j] - top_logit[0]);
    if (lane < k) {
      float lj = top_logit[0];
      int ej = top_e[0];
      for (int j = 1; j < k; ++j)
        if (j == lane) {
          lj = top_logit[j];
          ej = top_e[j];
        }
      sel_e[row * k + lane] = ej;
      sel_w[row * k + lane] = __expf(lj - top_logit[0]) / z;
      atomicAdd(&cnt[ej], 1);  // shared memory; only the per-CTA total matters
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[static_cast<int64_t>(e) * gridDim.x + blockIdx.x] = cnt[e];
}

// K8b: exclusive scan over hist[E][n_cta] (expert-major) in one CTA; writes the
// scanned bases back in place and expert_off[0..E].
__global__ void __launch_bounds__(kScanThreads)
    k8_scan(int32_t* __restrict__ hist, int64_t n, int32_t E, int32_t n_cta, int32_t* __restrict__ expert_off) {
  __shared__ int32_t warp_tot[kScanThreads / 32];
  __shared__ int32_t carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    const int32_t x = i < n ? hist[i] : 0;
    int32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int32_t t = warp_tot[lane];
      int32_t ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += y;
      }
      warp_tot[lane] = ti - t;  // exclusive warp prefix
    }
    __syncthreads();
    const int32_t excl = carry + warp_tot[warp] + incl - x;
    if (i < n) {
      hist[i] = excl;
      if (i % n_cta == 0) expert_off[i / n_cta] = excl;  // first CTA of expert e
    }
    __syncthreads();
    if (threadIdx.x == kScanThreads - 1) carry = excl + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) expert_off[E] = carry;
}

// K8c: stable scatter of every assignment to its dispatch position.
__global__ void __launch_bounds__(kRouteThreads)
    k8_scatter(const int32_t* __restrict__ base, int64_t rows, int32_t E, int32_t k, int32_t row_base,
               int32_t* __restrict__ sel_e_pos, float* __restrict__ sel_w, int32_t* __restrict__ disp_row,
               float* __restrict__ disp_w) {
  __shared__ int32_t cnt[kMaxExperts];
  __shared__ int32_t ids[kRowsPerCta * kMaxTopK];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRowsPerCta;
  const int64_t n_rows = min(static_cast<int64_t>(kRowsPerCta), rows - r0);
  const int n = static_cast<int>(n_rows) * k;
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    cnt[e] = base[static_cast<int64_t>(e) * gridDim.x + blockIdx.x];
  for (int i = threadIdx.x; i < n; i += blockDim.x) ids[i] = sel_e_pos[r0 * k + i];
  __syncthreads();
  if (threadIdx.x < 32) {  // one warp walks the CTA's assignments in order
    const int lane = threadIdx.x;
    for (int c = 0; c < n; c += 32) {
      const int i = c + lane;
      const bool valid = i < n;
      const int e = valid ? ids[i] : -1 - lane;  // invalid lanes never match a real expert
      const unsigned peers = __match_any_sync(0xffffffffu, e);
      if (valid) {
        const int rank = __popc(peers & ((1u << lane) - 1u));
        const int pos = cnt[e] + rank;
        const int64_t g = r0 * k + i;
        const int64_t row = r0 + i / k;
        disp_row[pos] = row_base + static_cast<int32_t>(row);
        if (disp_w) disp_w[pos] = sel_w[g];
        sel_e_pos[g] = pos;  // becomes the combine position
        const int leader = 31 - __clz(peers);
        __syncwarp(peers);
        if (lane == leader) cnt[e] += __popc(peers);
      }
      __syncwarp();
    }
  }
}

// K9: out[r, :] = sum_j w[r, j] * src[pos[r, j], :], one warp per row, 16-byte vectors.
__global__ void __launch_bounds__(256)
    k9_combine(const uint4* __restrict__ src, int64_t ld_src_vec, const int32_t* __restrict__ pos,
               const float* __restrict__ w, int64_t rows, int32_t k, int64_t d_vec, uint4* __restrict__ out,
               int64_t ld_out_vec) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    for (int64_t c = lane; c < d_vec; c += 32) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < k; ++j) {
        const int32_t p = __ldg(pos + r * k + j);
        const float wj = __ldg(w + r * k + j);
        const uint4 v = __ldg(src + p * ld_src_vec + c);
        const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(v2[q]);
          acc[2 * q] = fmaf(wj, f.x, acc[2 * q]);
          acc[2 * q + 1] = fmaf(wj, f.y, acc[2 * q + 1]);
        }
      }
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int q = 0; q < 4; ++q) o2[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
      out[r * ld_out_vec + c] = o;
    }
  }
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

extern "C" size_t mosaic_moe_route_scratch_bytes(int64_t rows, int32_t n_experts) {
  if (rows <= 0 || n_experts <= 0) return 256;
  const int64_t n_cta = ceil_div(rows, kRowsPerCta);
  return static_cast<size_t>(n_cta * n_experts * 4 + 256);
}

extern "C" int mosaic_moe_route(const float* logits, int64_t ld, int64_t rows, int32_t n_experts,
                                int32_t top_k, int32_t row_base, int32_t* disp_row, float* disp_w,
                                int32_t* comb_pos, float* comb_w, int32_t* expert_off, void* scratch,
                                void* stream) {
  MOSAIC_REQUIRE(n_experts >= 1 && n_experts <= kMaxExperts, "n_experts=%d not in [1, %d]", n_experts,
                 kMaxExperts);
  MOSAIC_REQUIRE(top_k >= 1 && top_k <= kMaxTopK && top_k <= n_experts, "top_k=%d not in [1, min(%d, E)]",
                 top_k, kMaxTopK);
  MOSAIC_REQUIRE(rows >= 0 && rows * top_k < (int64_t(1) << 31), "rows out of range");
  MOSAIC_REQUIRE(ld >= n_experts, "router logits row stride %lld < E", (long long)ld);
  MOSAIC_REQUIRE(expert_off && scratch, "null outputs");
  cudaStream_t s = as_stream(stream);
  if (rows == 0) {
    MOSAIC_CUDA(cudaMemsetAsync(expert_off, 0, sizeof(int32_t) * (n_experts + 1), s));
    return MOSAIC_OK;
  }
  MOSAIC_REQUIRE(logits && disp_row && comb_pos && comb_w, "null operands");
  const int n_cta = static_cast<int>(ceil_div(rows, kRowsPerCta));
  int32_t* hist = static_cast<int32_t*>(scratch);
  k8_topk<<<n_cta, kRouteThreads, 0, s>>>(logits, ld, rows, n_experts, top_k, comb_pos, comb_w, hist);
  k8_scan<<<1, kScanThreads, 0, s>>>(hist, static_cast<int64_t>(n_cta) * n_experts, n_experts, n_cta,
                                      expert_off);
  k8_scatter<<<n_cta, kRouteThreads, 0, s>>>(hist, rows, n_experts, top_k, row_base, comb_pos, comb_w,
                                             disp_row, disp_w);
  return check_launch("mosaic_moe_route");
}

extern "C" int mosaic_moe_combine(const uint16_t* src, int64_t ld_src, const int32_t* pos, const float* w,
                                  int64_t rows, int32_t top_k, int64_t d, uint16_t* out, int64_t ld_out,
                                  void* stream) {
  MOSAIC_REQUIRE(rows >= 0 && top_k >= 1 && d >= 0, "bad sizes");
  if (rows == 0 || d == 0) return MOSAIC_OK;
  MOSAIC_REQUIRE(src && pos && w && out, "null operands");
  MOSAIC_REQUIRE(d % 8 == 0 && ld_src % 8 == 0 && ld_out % 8 == 0, "d and row strides must be multiples of 8");
  MOSAIC_REQUIRE((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0,
                 "src/out must be 16-byte aligned");
  const int64_t want = ceil_div(rows, 8);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  k9_combine<<<static_cast<int>(want < cap ? want : cap), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(src), ld_src / 8, pos, w, rows, top_k, d / 8,
      reinterpret_cast<uint4*>(out), ld_out / 8);
  return check_launch("mosaic_moe_combine");
}
