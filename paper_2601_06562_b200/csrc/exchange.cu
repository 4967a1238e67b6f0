// K4x: the vocab-shard exchange fused into the split merge, over NVLink peer
// memory (north_star item 4). Replaces "K4 local merge -> NCCL all-gather of
// the per-row triples -> K4 rank merge" by
//
//   push:  each row's S split triples are merged (the K4 rule) and the merged
//          (max, sum, argmax) is stored straight into slot [epoch & 1][rank] of
//          EVERY rank's gathered buffer [2][P][3][m_cap] through its peer pointer
//          (st.global over NVLink); the last CTA to finish publishes `epoch`
//          into every rank's signal pad slot [rank] (release, system scope);
//   wait:  one CTA spins until all P slots of the local signal pad have
//          reached `epoch` (acquire, system scope; wraparound-safe "not
//          behind" test, since a peer may already have published epoch + 1
//          -- it needs only this rank's push of `epoch`, not this wait),
//          bounded so a missing peer traps instead of hanging;
//
// after which the ordinary K4 (mosaic_stats_merge) merges the P triples in
// rank order on the local buffer, exactly as after the all-gather. Buffers and
// signal pads are symmetric allocations (torch symmetric memory) whose peer
// pointers the host passes in as device arrays. Every rank runs the same
// deterministic K5 afterwards, so no broadcast is needed.
//
// Reference: rows are independent (mosaic/kernel.py:70-84) and the merge is
// associative; the reference itself has no distribution.
#include "common.cuh"

namespace mosaic {
namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(256)
    k4x_push(const float* __restrict__ in_max, const float* __restrict__ in_sum, const int32_t* __restrict__ in_arg,
             int32_t S, int64_t stride, const int32_t* __restrict__ m_dev, int64_t m_host, int64_t m_cap,
             float* const* __restrict__ peer_gathered, uint32_t* const* __restrict__ peer_signal, int32_t rank,
             int32_t world, uint32_t epoch, uint32_t* __restrict__ done) {
  const int64_t M = min(static_cast<int64_t>(load_count(m_dev, m_host)), m_cap);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < M;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float m, sum;
    int32_t arg;
    merge_triples_row(in_max, in_sum, in_arg, S, stride, r, m, sum, arg);  // the K4 rule, ascending splits
    // half (epoch & 1) of the double-buffered [2][P][3][m_cap] gathered block:
    // a rank can be at most one step ahead of a peer's merge (its next push
    // needs every rank's signal of this step, which each rank gives only after
    // merging the previous one), so alternating halves rules out overwriting
    // triples a slower peer has not merged yet
    const int64_t slot = (static_cast<int64_t>(epoch & 1u) * world + rank) * 3 * m_cap + r;
    for (int p = 0; p < world; ++p) {  // peer stores over NVLink (p == rank: local)
      float* g = peer_gathered[p];
      g[slot] = m;
      g[slot + m_cap] = sum;
      reinterpret_cast<int32_t*>(g)[slot + 2 * m_cap] = arg;
    }
  }
  // publish once every CTA's stores are visible system-wide
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t prev = atomicAdd(done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      *done = 0u;  // ready for the next step
      for (int p = 0; p < world; ++p) st_release_sys(peer_signal[p] + rank, epoch);
    }
  }
}

__global__ void k4x_wait(const uint32_t* __restrict__ local_signal, int32_t world, uint32_t epoch) {
  const int p = threadIdx.x;
  if (p < world) {
    uint32_t spins = 0;
    // a peer is at most one epoch ahead (its next push needs this rank's push
    // of the next epoch, which follows this wait), so "slot - epoch >= 0" in
    // wraparound arithmetic is exactly "the peer's push of `epoch` landed"
    while (static_cast<int32_t>(ld_acquire_sys(local_signal + p) - epoch) < 0) {
      if (++spins == (1u << 27)) __trap();  // a peer never arrived (~tens of s): fail the launch, do not hang
    }
  }
  __syncthreads();
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

extern "C" int mosaic_stats_exchange_push(const float* in_max, const float* in_sum, const int32_t* in_arg, int32_t S,
                                          int64_t stride, const int32_t* m_dev, int64_t m_host, int64_t m_cap,
                                          float* const* peer_gathered, uint32_t* const* peer_signal, int32_t rank,
                                          int32_t world, uint32_t epoch, uint32_t* done_counter, void* stream) {
  MOSAIC_REQUIRE(S >= 1 && stride >= m_cap, "bad split layout");
  MOSAIC_REQUIRE(world >= 1 && world <= 64 && rank >= 0 && rank < world, "rank %d / world %d", rank, world);
  MOSAIC_REQUIRE(in_max && in_sum && in_arg && peer_gathered && peer_signal && done_counter, "null operands");
  MOSAIC_REQUIRE(m_dev != nullptr || (m_host >= 0 && m_host <= m_cap), "m_host > m_cap");
  const int64_t want = ceil_div(m_cap > 0 ? m_cap : 1, 256);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 4;
  k4x_push<<<static_cast<int>(want < cap ? want : cap), 256, 0, as_stream(stream)>>>(
      in_max, in_sum, in_arg, S, stride, m_dev, m_host, m_cap, peer_gathered, peer_signal, rank, world, epoch,
      done_counter);
  return check_launch("mosaic_stats_exchange_push");
}

extern "C" int mosaic_stats_exchange_wait(const uint32_t* local_signal, int32_t world, uint32_t epoch, void* stream) {
  MOSAIC_REQUIRE(local_signal && world >= 1 && world <= 64, "bad arguments");
  k4x_wait<<<1, 64, 0, as_stream(stream)>>>(local_signal, world, epoch);
  return check_launch("mosaic_stats_exchange_wait");
}
