// K4 split/rank merge of the softmax-statistics triples, and K5 the
// low-confidence remasking commit.
//
// Both realise ops that are memory-only in the reference template: `sample`
// writes token_out/confidence [rows] (mosaic/workload.py:281-285,306-308) and
// `commit` consumes them (mosaic/workload.py:315), with the per-step unmask
// count coming from ScenarioConfig.masked_at (mosaic/workload.py:140-146).
//
// Merge rule (associative, applied in fixed ascending order so every rank and
// every run produces the same bits):
//   (m1,S1,a1) + (m2,S2,a2) = (max, S1 e^(m1-max) + S2 e^(m2-max),
//                              a of the larger m, lower index on equal m).
// Remask rule: keep the k masked rows with the highest confidence, ties broken
// towards the lower sequence position. Implemented as an exact radix select on
// the 64-bit key (conf bits << 32 | ~pos), unique per row, 8 passes of 8 bits.
#include <cfloat>
#include <cstdlib>

#include "common.cuh"

namespace mosaic {
namespace {

__global__ void k4_merge(const float* __restrict__ in_max, const float* __restrict__ in_sum,
                         const int32_t* __restrict__ in_arg, int32_t S, int64_t stride,
                         const int32_t* __restrict__ m_dev, int64_t m_host, int64_t m_cap,
                         float* __restrict__ out_max, float* __restrict__ out_sum,
                         int32_t* __restrict__ out_arg, int32_t* __restrict__ token,
                         float* __restrict__ lse, float* __restrict__ conf) {
  pdl_wait();
  pdl_trigger();
  const int64_t M = min(static_cast<int64_t>(load_count(m_dev, m_host)), m_cap);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < M;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float m, sum;
    int32_t arg;
    merge_triples_row(in_max, in_sum, in_arg, S, stride, r, m, sum, arg);
    if (out_max) out_max[r] = m;
    if (out_sum) out_sum[r] = sum;
    if (out_arg) out_arg[r] = arg;
    if (token) token[r] = arg;
    if (lse) lse[r] = m + logf(sum);
    if (conf) conf[r] = 1.f / sum;
  }
}

// K4 for few rows and many splits (a decoding block against one split per SM):
// one warp per row, the lanes load 32 splits' triples at once (one L2 round
// trip instead of 32), and every lane replays the same ascending-order merge
// from warp shuffles -- bit-identical to merge_triples_row.
__global__ void __launch_bounds__(256) k4_merge_warp(const float* __restrict__ in_max, const float* __restrict__ in_sum,
                                                     const int32_t* __restrict__ in_arg, int32_t S, int64_t stride,
                                                     const int32_t* __restrict__ m_dev, int64_t m_host, int64_t m_cap,
                                                     float* __restrict__ out_max, float* __restrict__ out_sum,
                                                     int32_t* __restrict__ out_arg, int32_t* __restrict__ token,
                                                     float* __restrict__ lse, float* __restrict__ conf) {
  pdl_wait();
  pdl_trigger();
  const int64_t M = min(static_cast<int64_t>(load_count(m_dev, m_host)), m_cap);
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); r < M; r += warps) {
    float m = -INFINITY, sum = 0.f;
    int32_t arg = INT32_MAX;
    for (int s0 = 0; s0 < S; s0 += 32) {
      const int s = s0 + lane;
      float mi_l = -INFINITY, si_l = 0.f;
      int32_t ai_l = INT32_MAX;
      if (s < S) {
        const int64_t o = static_cast<int64_t>(s) * stride + r;
        mi_l = in_max[o];
        si_l = in_sum[o];
        ai_l = in_arg[o];
      }
      const int n = min(32, S - s0);
      for (int j = 0; j < n; ++j) {
        const float mi = __shfl_sync(0xffffffffu, mi_l, j);
        const float si = __shfl_sync(0xffffffffu, si_l, j);
        const int32_t ai = __shfl_sync(0xffffffffu, ai_l, j);
        if (mi > m) {
          sum = sum * expf(m - mi) + si;
          m = mi;
          arg = ai;
        } else if (mi == m) {
          sum += si;
          arg = min(arg, ai);
        } else {
          sum += si * expf(mi - m);
        }
      }
    }
    if (lane == 0) {
      if (out_max) out_max[r] = m;
      if (out_sum) out_sum[r] = sum;
      if (out_arg) out_arg[r] = arg;
      if (token) token[r] = arg;
      if (lse) lse[r] = m + logf(sum);
      if (conf) conf[r] = 1.f / sum;
    }
  }
}

// K4 for the sampling variant: (max, sum) merge as merge_triples_row; the
// token is the noisy argmax (larger noisy score wins, lower vocab id on ties)
// and conf = p(token) under the untempered logits = exp(x_token - lse), as
// LLaDA's generate scores a sampled token.
__global__ void __launch_bounds__(256) k4_sample_merge(const float* __restrict__ in_max, const float* __restrict__ in_sum,
                                                       const int32_t* __restrict__ in_arg,
                                                       const float* __restrict__ in_y, const float* __restrict__ in_x,
                                                       int32_t S, int64_t stride, const int32_t* __restrict__ m_dev,
                                                       int64_t m_host, int64_t m_cap, int32_t* __restrict__ token,
                                                       float* __restrict__ lse, float* __restrict__ conf) {
  pdl_wait();
  pdl_trigger();
  const int64_t M = min(static_cast<int64_t>(load_count(m_dev, m_host)), m_cap);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < M;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float m, sum;
    int32_t unused;
    merge_triples_row(in_max, in_sum, in_arg, S, stride, r, m, sum, unused);
    float ybest = -INFINITY, xbest = -INFINITY;
    int32_t abest = INT32_MAX;
    constexpr int kChunk = 8;  // loads issued ahead of the compare chain (few rows, many splits)
    for (int s0 = 0; s0 < S; s0 += kChunk) {
      float y[kChunk], xv[kChunk];
      int32_t a[kChunk];
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        if (s0 + j < S) {
          const int64_t o = static_cast<int64_t>(s0 + j) * stride + r;
          y[j] = in_y[o];
          a[j] = in_arg[o];
          xv[j] = in_x[o];
        }
      }
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        if (s0 + j < S && (y[j] > ybest || (y[j] == ybest && a[j] < abest))) {
          ybest = y[j];
          abest = a[j];
          xbest = xv[j];
        }
      }
    }
    const float l = m + logf(sum);
    token[r] = abest;
    if (lse) lse[r] = l;
    conf[r] = expf(xbest - l);
  }
}

struct SelectState {
  unsigned long long prefix;
  uint32_t k_rem;
  uint32_t active;
  uint32_t hist[256];
};

__device__ __forceinline__ unsigned long long remask_key(float c, int32_t pos) {
  return (static_cast<unsigned long long>(__float_as_uint(c)) << 32) |
         static_cast<unsigned long long>(~static_cast<uint32_t>(pos));
}

__global__ void k5_init(SelectState* st, const int32_t* __restrict__ m_dev, int64_t m_host,
                        int64_t m_cap, int64_t k) {
  const int64_t M = min(static_cast<int64_t>(load_count(m_dev, m_host)), m_cap);
  const int64_t kk = k < M ? k : M;
  if (threadIdx.x == 0) {
    st->prefix = 0ull;
    st->k_rem = static_cast<uint32_t>(kk > 0 ? kk : 0);
    st->active = kk > 0 ? 1u : 0u;
  }
  st->hist[threadIdx.x] = 0u;
}

__global__ void __launch_bounds__(256) k5_hist(const float* __restrict__ conf,
                                               const int32_t* __restrict__ pos,
                                               const int32_t* __restrict__ m_dev, int64_t m_host,
                                               int64_t m_cap, int pass, SelectState* st) {
  __shared__ uint32_t h[256];
  if (st->k_rem == 0) return;  // uniform across the grid
  h[threadIdx.x] = 0u;
  __syncthreads();
  const int64_t M = min(static_cast<int64_t>(load_count(m_dev, m_host)), m_cap);
  const unsigned long long prefix = st->prefix;
  const int hi_shift = 64 - 8 * pass;  // bits already fixed: [hi_shift, 64)
  const int lo_shift = 56 - 8 * pass;
  for (int64_t r = blockIdx.x * 256ll + threadIdx.x; r < M; r += gridDim.x * 256ll) {
    const unsigned long long key = remask_key(conf[r], pos[r]);
    if (pass == 0 || (key >> hi_shift) == (prefix >> hi_shift))
      atomicAdd(&h[(key >> lo_shift) & 255u], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k5_pick(SelectState* st, int pass) {
  __shared__ uint32_t cum[256];
  const int t = threadIdx.x;
  const uint32_t k_rem = st->k_rem;
  const uint32_t cnt = st->hist[255 - t];  // descending digit order
  cum[t] = cnt;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const uint32_t add = t >= o ? cum[t - o] : 0u;
    __syncthreads();
    cum[t] += add;
    __syncthreads();
  }
  if (k_rem > 0) {
    const uint32_t incl = cum[t], above = incl - cnt;
    if (above < k_rem && incl >= k_rem) {
      st->prefix |= static_cast<unsigned long long>(255 - t) << (56 - 8 * pass);
      st->k_rem = k_rem - above;
    }
  }
  st->hist[255 - t] = 0u;
}

__global__ void __launch_bounds__(256) k5_commit(const float* __restrict__ conf,
                                                 const int32_t* __restrict__ pos,
                                                 const int32_t* __restrict__ token,
                                                 const int32_t* __restrict__ m_dev, int64_t m_host,
                                                 int64_t m_cap, const SelectState* st,
                                                 int32_t* __restrict__ x,
                                                 int32_t* __restrict__ selected) {
  const int64_t M = min(static_cast<int64_t>(load_count(m_dev, m_host)), m_cap);
  const bool active = st->active != 0u;
  const unsigned long long thr = st->prefix;
  for (int64_t r = blockIdx.x * 256ll + threadIdx.x; r < M; r += gridDim.x * 256ll) {
    const int32_t p = pos[r];
    const bool sel = active && remask_key(conf[r], p) >= thr;
    if (sel) x[p] = token[r];
    if (selected) selected[r] = sel ? 1 : 0;
  }
}

// Single-CTA K5 for capacities up to kFusedRemaskCap rows: the same 8-pass
// radix select (one 8-bit digit of the 64-bit key per pass, histogram in
// shared memory) and the commit, in one launch instead of 18 -- at LLaDA 32k
// (M = 16384) the 18 dependent launches cost more than the work.
constexpr int64_t kFusedRemaskCap = 40960;  // measured crossover (profiles/r01i_k5_crossover.txt)
constexpr int kFusedThreads = 1024;
constexpr int kRankCountRows = 256;  // rank-by-counting K5 up to this many rows per segment

// One CTA selects and commits among rows [r0, r1): the k most confident
// (ties -> lower position), exactly, by an 8-pass radix select of the 64-bit
// key with the histogram in shared memory.
__device__ __forceinline__ void select_commit_cta(const float* __restrict__ conf, const int32_t* __restrict__ pos,
                                                  const int32_t* __restrict__ token, int64_t r0, int64_t r1,
                                                  int64_t k, int32_t* __restrict__ x,
                                                  int32_t* __restrict__ selected) {
  __shared__ uint32_t h[256];
  __shared__ uint32_t cum[256];
  __shared__ unsigned long long s_prefix;
  __shared__ uint32_t s_krem;
  __shared__ unsigned long long s_keys[kRankCountRows];
  const int t = threadIdx.x;
  const int64_t M = r1 - r0;
  const int64_t kk = k < M ? k : M;
  if (M <= kRankCountRows) {
    // short segments (decoding blocks): rank every key by counting the larger
    // ones -- keys are unique (position tie-break), so exactly kk ranks fall
    // below kk; one barrier instead of 8 radix passes. O(M^2) compares, so
    // only up to kRankCountRows (at 1024 rows it cost ~60 us more than radix)
    if (t < M) s_keys[t] = remask_key(conf[r0 + t], pos[r0 + t]);
    __syncthreads();
    if (t < M) {
      const unsigned long long mine = s_keys[t];
      int64_t rank = 0;
      for (int64_t j = 0; j < M; ++j) rank += s_keys[j] > mine;
      const bool sel = rank < kk;
      const int32_t p = pos[r0 + t];
      if (sel) x[p] = token[r0 + t];
      if (selected) selected[r0 + t] = sel ? 1 : 0;
    }
    return;
  }
  if (t == 0) {
    s_prefix = 0ull;
    s_krem = static_cast<uint32_t>(kk > 0 ? kk : 0);
  }
  for (int pass = 0; pass < 8; ++pass) {
    if (t < 256) h[t] = 0u;
    __syncthreads();
    // every thread snapshots the pass state here; the single qualifying thread
    // below is the only writer, and nobody re-reads s_krem / s_prefix before
    // the closing barrier (racecheck/synccheck clean)
    const uint32_t k_rem = s_krem;
    if (k_rem == 0u) break;  // only when k == 0 (uniform)
    const unsigned long long prefix = s_prefix;
    const int hi_shift = 64 - 8 * pass;
    const int lo_shift = 56 - 8 * pass;
    for (int64_t r = r0 + t; r < r1; r += kFusedThreads) {
      const unsigned long long key = remask_key(conf[r], pos[r]);
      if (pass == 0 || (key >> hi_shift) == (prefix >> hi_shift)) atomicAdd(&h[(key >> lo_shift) & 255u], 1u);
    }
    __syncthreads();
    uint32_t cnt = 0u;
    if (t < 256) {
      cnt = h[255 - t];  // descending digit order
      cum[t] = cnt;
    }
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
      const uint32_t add = (t < 256 && t >= o) ? cum[t - o] : 0u;
      __syncthreads();
      if (t < 256) cum[t] += add;
      __syncthreads();
    }
    if (t < 256) {
      const uint32_t incl = cum[t], above = incl - cnt;
      if (above < k_rem && incl >= k_rem) {  // exactly one digit qualifies
        s_prefix = prefix | (static_cast<unsigned long long>(255 - t) << lo_shift);
        s_krem = k_rem - above;
      }
    }
    __syncthreads();
  }
  const bool active = kk > 0;
  const unsigned long long thr = s_prefix;
  for (int64_t r = r0 + t; r < r1; r += kFusedThreads) {
    const int32_t p = pos[r];
    const bool sel = active && remask_key(conf[r], p) >= thr;
    if (sel) x[p] = token[r];
    if (selected) selected[r] = sel ? 1 : 0;
  }
}

__global__ void __launch_bounds__(kFusedThreads) k5_fused(const float* __restrict__ conf,
                                                          const int32_t* __restrict__ pos,
                                                          const int32_t* __restrict__ token,
                                                          const int32_t* __restrict__ m_dev, int64_t m_host,
                                                          int64_t m_cap, int64_t k, int32_t* __restrict__ x,
                                                          int32_t* __restrict__ selected) {
  pdl_wait();
  pdl_trigger();
  const int64_t M = min(static_cast<int64_t>(load_count(m_dev, m_host)), m_cap);
  select_commit_cta(conf, pos, token, 0, M, k, x, selected);
}

// Segmented K5 (batched sequences / blocks): CTA b owns the rows whose
// position lies in [b * seg_len, (b + 1) * seg_len) -- a contiguous run of the
// ascending compacted list, found by binary search -- and commits its own k_b.
__device__ __forceinline__ int64_t lower_bound_pos(const int32_t* __restrict__ pos, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (pos[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kFusedThreads) k5_segmented(const float* __restrict__ conf,
                                                              const int32_t* __restrict__ pos,
                                                              const int32_t* __restrict__ token,
                                                              const int32_t* __restrict__ m_dev, int64_t m_host,
                                                              int64_t m_cap, int64_t seg_len,
                                                              const int32_t* __restrict__ k_per_seg, int64_t k,
                                                              int32_t* __restrict__ x,
                                                              int32_t* __restrict__ selected) {
  __shared__ int64_t s_bounds[2];
  pdl_wait();
  pdl_trigger();
  const int64_t M = min(static_cast<int64_t>(load_count(m_dev, m_host)), m_cap);
  const int64_t b = blockIdx.x;
  if (threadIdx.x < 2) s_bounds[threadIdx.x] = lower_bound_pos(pos, M, (b + threadIdx.x) * seg_len);
  __syncthreads();
  const int64_t kb = k_per_seg ? static_cast<int64_t>(k_per_seg[b]) : k;
  select_commit_cta(conf, pos, token, s_bounds[0], s_bounds[1], kb < 0 ? 0 : kb, x, selected);
}

int grid_for(int64_t n, int per_block) {
  const int64_t want = ceil_div(n > 0 ? n : 1, per_block);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  return static_cast<int>(want < cap ? want : cap);
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

extern "C" int mosaic_stats_merge(const float* in_max, const float* in_sum, const int32_t* in_arg,
                                  int32_t S, int64_t stride, const int32_t* m_dev, int64_t m_host,
                                  int64_t m_cap, float* out_max, float* out_sum, int32_t* out_arg,
                                  int32_t* token, float* lse, float* conf, void* stream) {
  MOSAIC_REQUIRE(S >= 1, "need at least one partial, got S=%d", S);
  MOSAIC_REQUIRE(stride >= m_cap, "partial stride %lld < m_cap %lld", (long long)stride,
                 (long long)m_cap);
  MOSAIC_REQUIRE(in_max && in_sum && in_arg, "null partial inputs");
  MOSAIC_REQUIRE(m_dev != nullptr || (m_host >= 0 && m_host <= m_cap), "m_host > m_cap");
  if (m_cap == 0) return MOSAIC_OK;
  if (m_cap <= 8192 && S >= 8) {  // few rows, many splits: warp per row (r01i_k5_crossover.txt has the K4 note)
    MOSAIC_CUDA(launch_pdl(k4_merge_warp, dim3(grid_for(m_cap * 32, 256)), dim3(256), 0, as_stream(stream), in_max,
                           in_sum, in_arg, S, stride, m_dev, m_host, m_cap, out_max, out_sum, out_arg, token, lse,
                           conf));
  } else {
    MOSAIC_CUDA(launch_pdl(k4_merge, dim3(grid_for(m_cap, 256)), dim3(256), 0, as_stream(stream), in_max, in_sum,
                           in_arg, S, stride, m_dev, m_host, m_cap, out_max, out_sum, out_arg, token, lse, conf));
  }
  return check_launch("mosaic_stats_merge");
}

extern "C" size_t mosaic_remask_scratch_bytes(void) { return sizeof(SelectState); }

extern "C" int mosaic_remask_commit(const float* conf, const int32_t* pos, const int32_t* token,
                                    const int32_t* m_dev, int64_t m_host, int64_t m_cap, int64_t k,
                                    int32_t* x, int32_t* selected, void* scratch, void* stream) {
  MOSAIC_REQUIRE(k >= 0, "negative unmask count %lld", (long long)k);
  MOSAIC_REQUIRE(scratch != nullptr, "scratch required");
  MOSAIC_REQUIRE(m_dev != nullptr || (m_host >= 0 && m_host <= m_cap), "m_host > m_cap");
  if (m_cap == 0) return MOSAIC_OK;
  MOSAIC_REQUIRE(conf && pos && token && x, "null inputs");
  cudaStream_t s = as_stream(stream);
  static const int64_t fused_cap = [] {  // experiment knob; default measured (profiles/r01i_k5_crossover.txt)
    const char* e = getenv("MOSAIC_K5_FUSED_CAP");
    return e ? static_cast<int64_t>(atoll(e)) : kFusedRemaskCap;
  }();
  if (m_cap <= fused_cap) {
    MOSAIC_CUDA(launch_pdl(k5_fused, dim3(1), dim3(kFusedThreads), 0, s, conf, pos, token, m_dev, m_host, m_cap, k,
                           x, selected));
    return check_launch("mosaic_remask_commit");
  }
  SelectState* st = static_cast<SelectState*>(scratch);
  const int grid = grid_for(m_cap, 256);
  k5_init<<<1, 256, 0, s>>>(st, m_dev, m_host, m_cap, k);
  for (int pass = 0; pass < 8; ++pass) {
    k5_hist<<<grid, 256, 0, s>>>(conf, pos, m_dev, m_host, m_cap, pass, st);
    k5_pick<<<1, 256, 0, s>>>(st, pass);
  }
  k5_commit<<<grid, 256, 0, s>>>(conf, pos, token, m_dev, m_host, m_cap, st, x, selected);
  return check_launch("mosaic_remask_commit");
}

extern "C" int mosaic_remask_commit_segmented(const float* conf, const int32_t* pos, const int32_t* token,
                                              const int32_t* m_dev, int64_t m_host, int64_t m_cap, int64_t seg_len,
                                              int32_t n_seg, const int32_t* k_per_seg, int64_t k, int32_t* x,
                                              int32_t* selected, void* stream) {
  MOSAIC_REQUIRE(k >= 0, "negative unmask count %lld", (long long)k);
  MOSAIC_REQUIRE(seg_len >= 1 && n_seg >= 1 && n_seg <= (1 << 20), "bad segments (%lld x %d)", (long long)seg_len,
                 n_seg);
  MOSAIC_REQUIRE(m_dev != nullptr || (m_host >= 0 && m_host <= m_cap), "m_host > m_cap");
  if (m_cap == 0) return MOSAIC_OK;
  MOSAIC_REQUIRE(conf && pos && token && x, "null inputs");
  MOSAIC_CUDA(launch_pdl(k5_segmented, dim3(n_seg), dim3(kFusedThreads), 0, as_stream(stream), conf, pos, token,
                         m_dev, m_host, m_cap, seg_len, k_per_seg, k, x, selected));
  return check_launch("mosaic_remask_commit_segmented");
}

extern "C" int mosaic_sample_merge(const float* in_max, const float* in_sum, const int32_t* in_arg, const float* in_y,
                                   const float* in_x, int32_t S, int64_t stride, const int32_t* m_dev, int64_t m_host,
                                   int64_t m_cap, int32_t* token, float* lse, float* conf, void* stream) {
  MOSAIC_REQUIRE(S >= 1 && stride >= m_cap, "bad split layout");
  MOSAIC_REQUIRE(in_max && in_sum && in_arg && in_y && in_x && token && conf, "null operands");
  MOSAIC_REQUIRE(m_dev != nullptr || (m_host >= 0 && m_host <= m_cap), "m_host > m_cap");
  if (m_cap == 0) return MOSAIC_OK;
  MOSAIC_CUDA(launch_pdl(k4_sample_merge, dim3(grid_for(m_cap, 256)), dim3(256), 0, as_stream(stream), in_max, in_sum,
                         in_arg, in_y, in_x, S, stride, m_dev, m_host, m_cap, token, lse, conf));
  return check_launch("mosaic_sample_merge");
}
