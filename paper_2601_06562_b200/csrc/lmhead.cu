// K3: mask-only LM head as a persistent, warp-specialised tcgen05 GEMM whose
// epilogue folds every FP32 accumulator tile into per-row online softmax
// statistics (max, sum-exp, argmax) and never writes the logits.
//
// Reference counterpart: gather_gemm (mosaic/kernel.py:62-86) computes
// logits[i, :] = H[mask_idx[i], :] @ W and materialises [m, V] (:68); the
// `sample` op that consumes them is memory-only (mosaic/workload.py:306-308).
// Here the gathered rows Hc (K2) and the vocab shard W [V, d] (K-major) stream
// through TMA into a shared-memory ring (in gather mode the A rows come from H
// itself through cp.async loader warps); one elected thread issues tcgen05.mma (BF16 -> FP32 in TMEM) and four
// epilogue warps drain a double-buffered TMEM accumulator with tcgen05.ld while
// the next tile's MMAs run. Default cta_group::2: a CTA pair computes 256 x 256
// tiles (UMMA M=256, N=256, K=16) out of a 6-stage ring; cta_group::1 (128 x 256,
// 4 stages) serves M <= 128.
//
// Work decomposition: the vocab tiles (256 columns) are cut into n_splits
// contiguous splits; a work unit is (row block, split). Each pair takes the
// units the dynamic schedule hands it (claimed from a global counter by the
// pair leader and published to both CTAs through a shared-memory ring; the
// static order u = cluster, cluster + n_clusters, ... without a scratch) and
// keeps the per-row statistics of the current unit in registers across the
// split's tiles, so the only global output is one (max, sum, arg) triple per
// row and split. Units are numbered m-fastest inside groups of `group_m` row
// blocks, so the ~74 units in flight share a handful of W tiles and row blocks
// through L2.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace mosaic {
namespace {

constexpr int BM = 128;          // accumulator rows per CTA (TMEM lanes)
constexpr int BN = 256;          // vocab columns per tile (UMMA N)
constexpr int BK = 64;           // K per stage: one 128-byte swizzle atom of bf16
constexpr int UK = 16;           // K per tcgen05.mma (kind::f16)
constexpr int NUM_ACC = 2;       // TMEM accumulator double buffer
constexpr int TMEM_COLS = 512;   // 2 x 256 fp32 columns
constexpr int kThreads = 192;    // warp0 TMEM alloc + TMA, warp1 MMA, warps 2..5 epilogue
#ifndef MOSAIC_K3_AWARPS
#define MOSAIC_K3_AWARPS 4  // measured: 4 >= 8 once the per-stage sync is CTA-scope
#endif
constexpr int kAWarps = MOSAIC_K3_AWARPS;  // cp.async gather path: A loader warps (warp 0 + warps 6..)
// (A hybrid that fetched part of each block by TMA gather4 was measured slower
// for every split, profiles/r01_k3_gather_modes.txt, and is gone.)
constexpr int kRowsPerAWarp = BM / kAWarps;  // 32
static_assert(kRowsPerAWarp * kAWarps == BM, "gather rows must tile the block");
static_assert(kRowsPerAWarp % 4 == 0 && kRowsPerAWarp <= 32, "loader warp covers 4-row groups");
constexpr int kThreadsCpAsync = kThreads + (kAWarps - 1) * 32;
constexpr int kEpiWarps = 4;
// The sampling variant's epilogue (hash + two logs per logit) runs 8 epilogue
// warps: warps 2-5 take the first 128 columns of each tile, warps 6-9 the last
// 128 (each warp still owns one TMEM lane quarter), and each half writes its
// own partial, so the split count doubles for K4.
constexpr int kSampleHalves = 2;
#ifndef MOSAIC_K3_EPI_HALVES
#define MOSAIC_K3_EPI_HALVES 1  // experiment: 2 = eight epilogue warps on the argmax path too (partials x2)
#endif
constexpr int threads_for(int gather, bool sample) {
  return gather == 2 ? kThreadsCpAsync
                     : ((sample || MOSAIC_K3_EPI_HALVES == 2) ? kThreads + kEpiWarps * 32 : kThreads);
}
constexpr int kMaxSplits = 64;
// Dynamic unit schedule: the pair leader's producer thread claims units from
// global counters and publishes each id into this ring in both CTAs; every
// other role of the pair reads it. No free-slot barrier: the producer runs at
// most STAGES k-blocks (so <= STAGES units) ahead of the MMA issuer, which runs
// at most NUM_ACC tiles ahead of the slowest epilogue, so the reader furthest
// behind lags the publisher by < STAGES + NUM_ACC + 2 < kURing units.
constexpr int kURing = 16;
#ifndef MOSAIC_K3_EPI_SLEEP_NS
#define MOSAIC_K3_EPI_SLEEP_NS 0   // epilogue poll backoff while the next accumulator fills
#endif
#ifndef MOSAIC_K3_PROD_SLEEP_NS
#define MOSAIC_K3_PROD_SLEEP_NS 0  // producer poll backoff while the ring is full
#endif
constexpr float kLog2e = 1.4426950408889634f;

// Per cta_group configuration. CG = 2 pairs two SMs on one 256 x 256 tile
// (tcgen05.mma.cta_group::2): each CTA stages half of the rows (A) and half of
// the vocab columns (B) of every K step, so shared-memory and L2 traffic per
// FLOP drop by a third against CG = 1 and the ring can be 6 stages deep.
template <int CG>
struct Cfg {
  static constexpr int ROWS = BM * CG;             // tile rows (UMMA M)
  static constexpr int B_ROWS = BN / CG;           // vocab rows staged per CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
#ifndef MOSAIC_K3_STAGES2
#define MOSAIC_K3_STAGES2 6
#endif
  static constexpr int STAGES = CG == 1 ? 4 : MOSAIC_K3_STAGES2;
  static constexpr int OFF_BAR = STAGES * STAGE_BYTES;  // mbarriers + TMEM slot (256 B)
  static constexpr int OFF_SIDX = OFF_BAR + 256;          // gather4 rows (BM int32)
  static constexpr int OFF_RING = OFF_SIDX + BM * 4;      // unit ring: kURing mbarriers + kURing ids
  static constexpr int SMEM = OFF_RING + kURing * 12 + 1024;  // + 1 KB alignment slack
  static constexpr uint32_t IDESC = umma_idesc_bf16(ROWS, BN);
};

struct Params {
  const int32_t* m_dev;
  int64_t m_host;
  int64_t m_cap;
  int64_t V;
  int32_t K;
  int32_t n_tiles;
  int32_t tiles_per_split;
  int32_t n_splits;
  int32_t group_m;
  int32_t seg_splits;  // vocab segments of this many splits, processed segment-major (0 = one segment)
  const uint8_t* die_of_sm;  // die-aware dynamic schedule: SM -> L2 die (null = every pair claims from the front)
  int32_t n_sm;              // entries of die_of_sm (%smid need not be below it: treated as die 0)
  uint32_t* sched;           // dynamic schedule: [claimed (die split only), front, back, unused] counters,
                             // zeroed per launch;
                             // null = static schedule (pair c takes units c, c + pairs, ...)
  int32_t policy;   // L2 policy of (A, B) loads: 0 = (normal, normal), 1 = (evict_last, normal), 2 = (normal, evict_first), 3 = (evict_last, evict_first)
  int64_t v_offset;
  float* part_max;
  float* part_sum;
  int32_t* part_arg;
  float* out;   // logits (debug path)
  int64_t ldo;
  const int32_t* idx;  // gather mode: masked positions, A rows are H[src(idx[r])]
  const uint16_t* h;   // gather mode: H base (cp.async path)
  int64_t ld_h;        // gather mode: H row stride (elements)
  int32_t shift;       // gather/runs modes: bit 0 src(p) = max(p - 1, 0) (Dream token shift); bit 1 idx may
                       // repeat rows (not strictly ascending): no tile is treated as a contiguous run
  int32_t w_blocked;   // W pre-tiled as [n_tiles][K/64][256][64] (each TMA box contiguous)
  // sampling variant (temperature > 0): token = argmax_v (x_v + T * g(pos, v)),
  // g Gumbel noise from a counter-based hash of (seed, position, vocab id)
  const int32_t* spos;  // masked positions (K1 output), the noise's row key
  float temperature;
  uint32_t seed;
  float* part_y;        // max noisy score per split
  float* part_x;        // raw logit at that argmax
};

// Unit order: vocab segments of `seg_splits` consecutive splits, outermost;
// inside a segment, groups of `group_m` m-blocks, then the segment's splits,
// then m-blocks fastest. With segments sized so one segment's LM-head rows fit
// in L2 (like a 1/8 vocab shard), every m-group re-reads them from L2 instead
// of DRAM, while each group's gathered rows stay resident across the
// segment's splits.
__device__ __forceinline__ void unit_coords(const Params& p, int m_blocks, int64_t u, int& mb,
                                            int& s) {
  const int64_t seg_splits = p.seg_splits > 0 ? p.seg_splits : p.n_splits;
  const int64_t per_seg = static_cast<int64_t>(m_blocks) * seg_splits;
  const int64_t seg = u / per_seg;
  const int64_t su = u - seg * per_seg;
  const int64_t s_in = min(seg_splits, static_cast<int64_t>(p.n_splits) - seg * seg_splits);
  const int64_t per_group = static_cast<int64_t>(p.group_m) * s_in;
  const int64_t g = su / per_group;
  const int64_t rem = su - g * per_group;
  const int64_t gm = min(static_cast<int64_t>(p.group_m), m_blocks - g * p.group_m);
  s = static_cast<int>(seg * seg_splits + rem / gm);
  mb = static_cast<int>(g * p.group_m + rem % gm);
}

// TMA coordinates (col, row) of this CTA's W box for vocab tile t, k-block kb.
__device__ __forceinline__ void w_box(const Params& p, int t, int kb, int k_blocks, int b_rows_off, int& col,
                                      int& row) {
  if (p.w_blocked) {
    col = 0;
    row = (t * k_blocks + kb) * BN + b_rows_off;
  } else {
    col = kb * BK;
    row = t * BN + b_rows_off;
  }
}

// Counter-based noise for the sampling variant (murmur3 finaliser); restated
// bit for bit in oracle/mosaic_oracle.py (gumbel_u24).
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}


// 2-D TMA gather of four K-major rows (64 bf16 columns each) by row index,
// 128-byte swizzled like a plain box load; with CG == 2 the transaction bytes
// complete on the pair leader's mbarrier.
template <int CG>
__device__ __forceinline__ void tma_gather4(void* smem_dst, const void* tmap, uint64_t* bar, int32_t col,
                                            int4 rows, uint64_t policy) {
  if constexpr (CG == 1)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(col), "r"(rows.x), "r"(rows.y), "r"(rows.z),
        "r"(rows.w), "l"(policy)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(col), "r"(rows.x),
        "r"(rows.y), "r"(rows.z), "r"(rows.w), "l"(policy)
        : "memory");
}

// kGather: the A operand is not a compacted [m, d] buffer but the hidden
// states H themselves, fetched row by row with TMA gather4 at the masked
// positions idx[] -- the gather-GEMM of the paper with no intermediate
// buffer (K2 is skipped entirely).
// kGather selects the A path: 0 = dense TMA box of Hc, 1 = TMA gather4 from
// H, 2 = cp.async 16-byte row segments from H issued by the whole producer
// warp (swizzled in software to the 128-byte TMA layout).
// 3 = runs: a pair tile whose source rows are one contiguous run of H loads A
// as a TMA box of H (no copy); any other tile loads its box from Hc, where K2
// (mosaic_gather_rows_scattered) compacted only the rows of such tiles.
constexpr int kGatherNone = 0, kGatherTma4 = 1, kGatherCpAsync = 2, kGatherRuns = 3;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// cp.async A path: a gathered slot is released LAG stages after it is issued,
// so up to LAG + 1 stages of each loader thread's copies stay in flight. LAG <
// STAGES leaves the producer a free slot to issue into (no deadlock): 4 of 6
// stages on pairs, 2 of 4 on single CTAs. Slots of contiguous-run tiles (TMA
// A) carry no copies and are released as soon as they are issued, after the
// pending gathered ones (each barrier sees its arrivals in stage order).
template <int STAGES>
constexpr int a_lag() { return STAGES - 2 < 4 ? STAGES - 2 : 4; }

// Release the oldest of `pend` pending slots (the one issued pend - 1 stages
// before `stage`): wait until at most LAG of this thread's copy groups are in
// flight -- that slot's group has landed --, fence its generic-proxy writes to
// the async proxy (the writer-side fence of the PTX memory model), arrive
// (release); the MMA issuer acquires the barrier before tcgen05.mma reads.
// (One arrival per thread: electing one lane per warp after a __syncwarp was
// measured slower, 17 vs 14 ms at LLaDA 32k scattered.)
template <int STAGES>
__device__ __forceinline__ void a_release_oldest(uint64_t* afull, uint32_t stage, int pend) {
  constexpr int LAG = a_lag<STAGES>();
  static_assert(LAG >= 1 && LAG < STAGES, "bad lag");
  asm volatile("cp.async.wait_group %0;" ::"n"(LAG) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_arrive(&afull[(stage + STAGES - (pend - 1)) % STAGES]);
}

// Release every pending slot (oldest first); `next` is the next stage to issue.
template <int STAGES>
__device__ __forceinline__ void a_release_all(uint64_t* afull, uint32_t next, int& pend) {
  if (pend == 0) return;
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  for (int i = pend; i >= 1; --i) mbar_arrive(&afull[(next + STAGES - i) % STAGES]);
  pend = 0;
}

// Gather mode: the pair tile of row block `mb` (ROWS rows) reads one
// contiguous run of H -- its source rows are consecutive (idx ascends
// strictly, so first and last ROWS - 1 apart means consecutive; with the
// shift, src = p - 1 stays consecutive unless the run starts at position 0) --
// so its A operand is a plain TMA box. Evaluated identically by the producer,
// the MMA issuer and the peer relay: every role agrees which slots carry
// gathered rows (and so take part in the afull protocol).
template <int ROWS>
__device__ __forceinline__ bool contiguous_tile(const int32_t* idx, int shift, int64_t M, int mb, int* p0_out) {
  const int64_t r0 = static_cast<int64_t>(mb) * ROWS;
  if (r0 + ROWS > M) return false;
  if (shift & 2) return false;  // caller's idx may repeat rows (batched windows with the shift)
  const int p0 = __ldg(idx + r0), p1 = __ldg(idx + r0 + ROWS - 1);
  *p0_out = p0;
  return p1 - p0 == ROWS - 1 && !((shift & 1) && p0 == 0);
}

template <int CG, bool kStoreLogits, int kGather = kGatherNone, bool kSample = false>
__global__ void __launch_bounds__(threads_for(kGather, kSample), 1)
    k3_lmhead(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
              const __grid_constant__ CUtensorMap tmap_h, const Params p) {
  using C = Cfg<CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + NUM_ACC;
  // cp.async A path: the producer lanes' copies of a slot landed (32 async
  // arrivals per CTA; the pair leader's barrier also takes one relayed
  // arrival from the peer CTA)
  uint64_t* afull = tempty + NUM_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(afull + C::STAGES);
  int32_t* sidx = reinterpret_cast<int32_t*>(smem + C::OFF_SIDX);  // gather rows
  uint64_t* ufull = reinterpret_cast<uint64_t*>(smem + C::OFF_RING);  // unit ring: id published
  int32_t* uring = reinterpret_cast<int32_t*>(ufull + kURing);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;  // position in the SM pair
  const int64_t cluster = blockIdx.x / CG;
  const int64_t n_clusters = gridDim.x / CG;
  const int k_blocks = p.K / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    if constexpr (kGather == kGatherRuns) tma_prefetch_desc(&tmap_h);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&afull[i], kAWarps * 32 + (CG == 2 && rank == 0 ? 1 : 0));  // one arrival per loader thread
    }
    for (int i = 0; i < NUM_ACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps * ((kSample || (kGather != 2 && MOSAIC_K3_EPI_HALVES == 2)) ? 2 : 1) * CG);
    }
    for (int i = 0; i < kURing; ++i) mbar_init(&ufull[i], 1);
    fence_mbar_init();
  }
  // TMEM is allocated (and freed) by warp 0, the warp that also runs the block's
  // prologue: allocating from warp 1 showed up in compute-sanitizer racecheck as a
  // RAW hazard on the allocator's reserved shared word (1025 reports per launch,
  // 0 with warp 0; profiles/r02w_racecheck_tmem_alloc.txt)
  if (warp == 0) {
    __syncwarp();  // lane 0 initialised the barriers above; tcgen05.alloc is .sync.aligned
    tmem_alloc<CG>(tmem_slot, TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: everything above (barriers, TMEM, descriptor prefetch) overlapped the
  // predecessor's tail; from here on K2's rows and K1's count are read
  pdl_wait();
  pdl_trigger();
  const int64_t M = min(static_cast<int64_t>(load_count(p.m_dev, p.m_host)), p.m_cap);
  const int m_blocks = static_cast<int>((M + C::ROWS - 1) / C::ROWS);

  // Unit schedule. Units (m-block, split) are numbered m-fastest inside groups
  // of group_m m-blocks (unit_coords), so a contiguous range of unit ids shares
  // the group's row blocks and each split's W tiles through L2.
  //  * static (p.sched == null): pair c runs units c, c + pairs, ... -- the
  //    pairs drift apart over many units (equal work, unequal speed), and the
  //    units of one split stop sharing W fetches (Dream 128k: 77 GB of DRAM per
  //    launch against ~25 GB in lockstep, profiles/r02h_k3_shapes.json);
  //  * dynamic: the pair leader's producer claims the next unit from global
  //    counters when it starts one, so the units in flight are always one
  //    contiguous window of ids; with a die map, pairs on die 0 claim from the
  //    front of the range and pairs on die 1 from the back, so each die walks its
  //    own m-groups (its L2 holds them) and the two meet wherever their speeds
  //    put them -- no registration, no per-die pair counts, no idle tail.
  //    Claimed ids reach the pair's other roles through the unit ring.
  const int64_t units = static_cast<int64_t>(m_blocks) * p.n_splits;
  const bool dyn = p.sched != nullptr;
  int die = 0;
  if (dyn && p.die_of_sm != nullptr) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    die = (static_cast<int32_t>(smid) < p.n_sm && p.die_of_sm[smid] == 1) ? 1 : 0;
  }
  // the n-th unit of this pair (-1: no more); `publisher`: the pair leader's
  // producer thread, which claims it and publishes it to both CTAs' rings
  // claim: without a die map one atomic on the front counter; with it, a claim
  // on the shared total first, then the front or back counter of this die
  auto claim = [&]() -> int32_t {
    if (p.die_of_sm == nullptr) {
      const uint32_t c = atomicAdd(p.sched + 1, 1u);
      return c < static_cast<uint32_t>(units) ? static_cast<int32_t>(c) : -1;
    }
    if (atomicAdd(p.sched + 0, 1u) >= static_cast<uint32_t>(units)) return -1;
    return die == 0 ? static_cast<int32_t>(atomicAdd(p.sched + 1, 1u))
                    : static_cast<int32_t>(units - 1 - static_cast<int64_t>(atomicAdd(p.sched + 2, 1u)));
  };
  // the publisher claims one unit ahead: the atomic for unit n + 1 is issued
  // when unit n is published and its result is first used a whole unit later,
  // so its latency never stalls the TMA stream (units of 2 tiles at 1/8 vocab
  // shards last ~50 us)
  int32_t claimed_next = (dyn && rank == 0 && warp == 0 && lane == 0) ? claim() : -1;
  auto unit_at = [&](int n, bool publisher) -> int64_t {
    if (!dyn) {
      const int64_t u = cluster + static_cast<int64_t>(n) * n_clusters;
      return u < units ? u : -1;
    }
    const int slot = n & (kURing - 1);
    if (publisher) {
      const int32_t u = claimed_next;
      claimed_next = u >= 0 ? claim() : -1;
      uring[slot] = u;
      if constexpr (CG == 2) {
        asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(mapa_shared(smem_u32(uring + slot), 1)), "r"(u)
                     : "memory");
        mbar_arrive_cluster(mapa_shared(smem_u32(&ufull[slot]), 1));  // release.cluster: orders the store
      }
      mbar_arrive(&ufull[slot]);
      return u;
    }
    if (CG == 2 && rank == 1) mbar_wait_cluster(&ufull[slot], (n / kURing) & 1);
    else mbar_wait(&ufull[slot], (n / kURing) & 1);
    return *reinterpret_cast<volatile int32_t*>(uring + slot);
  };
  const bool is_publisher = dyn && rank == 0 && warp == 0 && lane == 0;

  if (warp == 0 || (kGather == kGatherCpAsync && warp >= 6)) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    // A is re-read for every tile of a unit and by the units of its m-group;
    // a W tile is shared by the m-blocks in flight at the same moment.
    const uint64_t pol_a = (p.policy == 1 || p.policy == 3) ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_b = (p.policy == 2 || p.policy == 3) ? policy_evict_first() : policy_evict_normal();
    uint32_t stage = 0, phase = 0;
    int a_pend = 0;  // cp.async A path: slots issued by this thread and not yet released
    for (int n = 0;; ++n) {
      // lane 0 of each producer warp learns the unit (the leader's warp 0 lane 0 claims it)
      int64_t u = 0;
      if (lane == 0) u = unit_at(n, is_publisher);
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u < 0) break;
      int mb, s;
      unit_coords(p, m_blocks, u, mb, s);
      const int t0 = s * p.tiles_per_split;
      const int t1 = min(t0 + p.tiles_per_split, p.n_tiles);
      const int a_row = mb * C::ROWS + rank * BM;
      if constexpr (kGather == kGatherTma4) {
        // this CTA's 128 source rows, once per unit (rows past M read row 0;
        // their statistics are never stored)
#pragma unroll
        for (int j = 0; j < BM / 32; ++j) {
          const int r = a_row + j * 32 + lane;
          int v = r < M ? __ldg(p.idx + r) : 0;
          if (p.shift & 1) v = max(v - 1, 0);
          sidx[j * 32 + lane] = v;
        }
        __syncwarp();
      }
      if constexpr (kGather == kGatherCpAsync) {
        // A rows of a pair tile whose 256 source rows are consecutive rows of H
        // (a contiguous masked run: the reference schedule's step-0 suffix,
        // semi-autoregressive blocks) come in one TMA box per CTA-stage, exactly
        // the dense path's load; any other tile is gathered by the kAWarps
        // loader warps with 16-byte cp.async (kRowsPerAWarp rows each, lane
        // copies chunk (lane & 7) of rows (lane >> 3) + 4 i, swizzled in software
        // to the 128-byte TMA layout). The choice is per unit and the same in
        // both CTAs of the pair (it depends on the pair tile's rows only); idx
        // ascends strictly, so first/last 255 apart means consecutive.
        int p0 = 0;
        const bool contig = contiguous_tile<C::ROWS>(p.idx, p.shift, M, mb, &p0);
        const int a_src = p0 + static_cast<int>(rank) * BM - (p.shift & 1);  // this CTA's first source row
        if (contig) {
          // the unit runs exactly like the dense path: warp 0 lane 0 issues A and
          // B boxes, no afull traffic; the other loader warps skip its slots
          // (the MMA issuer and the peer relay skip them in the afull protocol)
          a_release_all<C::STAGES>(afull, stage, a_pend);  // gathered slots of earlier units first
          const int n_st = (t1 - t0) * k_blocks;
          if (warp == 0 && lane == 0) {
            for (int t = t0; t < t1; ++t)
              for (int kb = 0; kb < k_blocks; ++kb) {
                mbar_wait(&empty[(stage + (t - t0) * k_blocks + kb) % C::STAGES],
                          (phase ^ (((stage + (t - t0) * k_blocks + kb) / C::STAGES) & 1)) ^ 1);
                const uint32_t st = (stage + (t - t0) * k_blocks + kb) % C::STAGES;
                int bc, br;
                w_box(p, t, kb, k_blocks, rank * C::B_ROWS, bc, br);
                if (rank == 0) mbar_arrive_expect_tx(&full[st], C::STAGE_BYTES * CG);
                if constexpr (CG == 1) {
                  tma_load_2d(sB + st * C::B_BYTES, &tmap_b, &full[st], bc, br, pol_b);
                  tma_load_2d(sA + st * C::A_BYTES, &tmap_a, &full[st], kb * BK, a_src, pol_a);
                } else {
                  tma_load_2d_cg2(sB + st * C::B_BYTES, &tmap_b, &full[st], bc, br, pol_b);
                  tma_load_2d_cg2(sA + st * C::A_BYTES, &tmap_a, &full[st], kb * BK, a_src, pol_a);
                }
              }
          }
          // the other loader warps wait here (a hardware barrier, no polling) until
          // warp 0 has issued the whole unit, i.e. waited on every slot's
          // free-barrier in ring order: skipping ahead without it would let them
          // poll a slot's barrier several phases early, where its 1-bit parity
          // aliases. bar.sync is the .aligned form: warp 0 reconverges first (its
          // lane 0 issued the boxes), or the barrier sees a divergent warp
          __syncwarp();
          asm volatile("bar.sync 1, %0;" ::"n"(kAWarps * 32) : "memory");
          phase ^= ((stage + n_st) / C::STAGES) & 1;
          stage = (stage + n_st) % C::STAGES;
          continue;
        }
        const int slot = warp == 0 ? 0 : warp - 5;
        const int chunk = lane & 7;
        const int row0 = slot * kRowsPerAWarp;  // this warp's first row in the CTA's block
        const int my_row = a_row + row0 + (lane % kRowsPerAWarp);
        int src = my_row < M ? __ldg(p.idx + my_row) : 0;  // rows past M read row 0, never stored
        if (p.shift & 1) src = max(src - 1, 0);
        int64_t off[kRowsPerAWarp / 4];
#pragma unroll
        for (int i = 0; i < kRowsPerAWarp / 4; ++i)
          off[i] = static_cast<int64_t>(__shfl_sync(0xffffffffu, src, 4 * i + (lane >> 3))) * p.ld_h + chunk * 8;
        for (int t = t0; t < t1; ++t) {
          const int b_row_off = rank * C::B_ROWS;
          for (int kb = 0; kb < k_blocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            int bc, br;
            w_box(p, t, kb, k_blocks, b_row_off, bc, br);
            if (warp == 0 && lane == 0) {
              if (rank == 0) mbar_arrive_expect_tx(&full[stage], C::B_BYTES * CG);
              if constexpr (CG == 1)
                tma_load_2d(sB + stage * C::B_BYTES, &tmap_b, &full[stage], bc, br, pol_b);
              else
                tma_load_2d_cg2(sB + stage * C::B_BYTES, &tmap_b, &full[stage], bc, br, pol_b);
            }
            const uint32_t dst0 = smem_u32(sA + stage * C::A_BYTES);
            const uint16_t* hk = p.h + static_cast<int64_t>(kb) * BK;
#pragma unroll
            for (int i = 0; i < kRowsPerAWarp / 4; ++i) {
              const int r = row0 + 4 * i + (lane >> 3);  // row within the CTA's 128-row block
              cp_async16(dst0 + r * (BK * 2) + ((chunk ^ (r & 7)) << 4), hk + off[i], pol_a);
            }
            // writer-side release of the slot issued LAG stages ago (a_release_oldest)
            cp_async_commit();
            if (++a_pend > a_lag<C::STAGES>()) a_release_oldest<C::STAGES>(afull, stage, a_pend--);
            if (++stage == C::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      } else if (lane == 0) {
        // runs mode: this unit's A box comes from H (contiguous run) or from Hc
        const CUtensorMap* amap = &tmap_a;
        int a_box_row = a_row;
        if constexpr (kGather == kGatherRuns) {
          int p0 = 0;
          if (contiguous_tile<C::ROWS>(p.idx, p.shift, M, mb, &p0)) {
            amap = &tmap_h;
            a_box_row = p0 + static_cast<int>(rank) * BM - (p.shift & 1);
          }
        }
        for (int t = t0; t < t1; ++t) {
          const int b_row_off = rank * C::B_ROWS;
          for (int kb = 0; kb < k_blocks; ++kb) {
            mbar_wait_sleep(&empty[stage], phase ^ 1, MOSAIC_K3_PROD_SLEEP_NS);
            int bc, br;
            w_box(p, t, kb, k_blocks, b_row_off, bc, br);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES * CG);
            if constexpr (CG == 1)
              tma_load_2d(sB + stage * C::B_BYTES, &tmap_b, &full[stage], bc, br, pol_b);
            else
              tma_load_2d_cg2(sB + stage * C::B_BYTES, &tmap_b, &full[stage], bc, br, pol_b);
            if constexpr (kGather == kGatherTma4) {
              const uint32_t rows_addr = smem_u32(sidx);
#pragma unroll 4
              for (int i = 0; i < BM / 4; ++i) {
                int4 r4;
                asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(r4.x), "=r"(r4.y), "=r"(r4.z), "=r"(r4.w)
                             : "r"(rows_addr + i * 16));
                tma_gather4<CG>(sA + stage * C::A_BYTES + i * 4 * (BK * 2), &tmap_a, &full[stage], kb * BK,
                                r4, pol_a);
              }
            } else if constexpr (CG == 1) {
              tma_load_2d(sA + stage * C::A_BYTES, amap, &full[stage], kb * BK, a_box_row, pol_a);
            } else {
              tma_load_2d_cg2(sA + stage * C::A_BYTES, amap, &full[stage], kb * BK, a_box_row, pol_a);
            }
            if (++stage == C::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      __syncwarp();
    }
    if constexpr (kGather == kGatherCpAsync) {
      a_release_all<C::STAGES>(afull, stage, a_pend);  // drain: the last pending slots, oldest first
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    if (lane == 0 && rank == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      uint32_t abits = 0;  // gather mode: expected afull parity per slot (only gathered uses flip it)
      for (int n = 0;; ++n) {
        const int64_t u = unit_at(n, false);
        if (u < 0) break;
        int mb, s;
        unit_coords(p, m_blocks, u, mb, s);
        const int t0 = s * p.tiles_per_split;
        const int t1 = min(t0 + p.tiles_per_split, p.n_tiles);
        int p0_unused;
        const bool gathered = kGather == kGatherCpAsync && !contiguous_tile<C::ROWS>(p.idx, p.shift, M, mb, &p0_unused);
        for (int t = t0; t < t1; ++t) {
          if constexpr (CG == 2) mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
          else mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < k_blocks; ++kb) {
            mbar_wait(&full[stage], phase);
            if (gathered) {
              // the gathered rows of this slot landed and were fenced to the
              // async proxy by their writers (and, on a pair, the peer's rows:
              // relayed below). Only CTA-scope operations on the per-stage path:
              // cluster-scope fences and release.cluster arrives compile to
              // MEMBAR.ALL.GPU, which serialised the pair ring at ~0.9 us per
              // stage (profiles/r01_k3_gather_modes.txt).
              mbar_wait(&afull[stage], (abits >> stage) & 1u);
              abits ^= 1u << stage;
            }
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
            const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / UK; ++kk)
              umma_bf16<CG>(d_tmem, umma_desc_sw128(a0 + kk * UK * 2),
                            umma_desc_sw128(b0 + kk * UK * 2), C::IDESC, (kb | kk) != 0);
            umma_commit<CG>(&empty[stage]);  // frees the smem slot(s) when these MMAs retire
            if (++stage == C::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit<CG>(&tfull[acc]);  // accumulator ready for the epilogue(s)
          if (++acc == NUM_ACC) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
    if constexpr (kGather == kGatherCpAsync && CG == 2) {
      // peer CTA of the pair: relay "A slot landed" to the leader's barrier
      if (lane == 0 && rank == 1) {
        uint32_t stage = 0, phase = 0, abits = 0;
        for (int n = 0;; ++n) {
          const int64_t u = unit_at(n, false);
          if (u < 0) break;
          int mb, s;
          unit_coords(p, m_blocks, u, mb, s);
          const int t0 = s * p.tiles_per_split;
          const int t1 = min(t0 + p.tiles_per_split, p.n_tiles);
          int p0_unused;
          if (contiguous_tile<C::ROWS>(p.idx, p.shift, M, mb, &p0_unused)) {  // no gathered slots to relay
            const int n_st = (t1 - t0) * k_blocks;
            phase ^= ((stage + n_st) / C::STAGES) & 1;
            stage = (stage + n_st) % C::STAGES;
            continue;
          }
          for (int t = t0; t < t1; ++t)
            for (int kb = 0; kb < k_blocks; ++kb) {
              mbar_wait(&afull[stage], (abits >> stage) & 1u);
              abits ^= 1u << stage;
              // the peer's writers fenced their rows to the async proxy before
              // arriving; forward with a default-semantics remote arrive on the
              // leader's barrier: the form CUTLASS's cluster pipelines use for
              // remote arrives (cutlass/arch/barrier.h ClusterBarrier::arrive)
              asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(
                               mapa_shared(smem_u32(&afull[stage]), 0))
                           : "memory");
              if (++stage == C::STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;  // TMEM lane quarter accessible to this warp
    const int row_local = q * 32 + lane;
    constexpr int kHalves = (kSample || (kGather != 2 && MOSAIC_K3_EPI_HALVES == 2)) ? kSampleHalves : 1;
    const int half = (kHalves == 2 && warp >= 2 + kEpiWarps) ? 1 : 0;  // which 128 columns of each tile
    constexpr int kChunksPerHalf = BN / 32 / kHalves;
    // tempty lives in the pair leader: arrive locally or through the cluster window
    const uint32_t tempty_addr0 = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]);
    uint32_t acc = 0, acc_phase = 0;
    for (int n = 0;; ++n) {
      int64_t u = 0;
      if (lane == 0) u = unit_at(n, false);
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u < 0) break;
      int mb, s;
      unit_coords(p, m_blocks, u, mb, s);
      const int t0 = s * p.tiles_per_split;
      const int t1 = min(t0 + p.tiles_per_split, p.n_tiles);
      const int64_t row = static_cast<int64_t>(mb) * C::ROWS + rank * BM + row_local;
      float run_max = -INFINITY, run_sum = 0.f;
      int64_t run_arg = 0;
      float s_ymax = -INFINITY, s_xarg = 0.f;  // sampling variant: noisy max and its raw logit
      uint32_t row_key = 0;
      if constexpr (kSample) {
        if (row < M) row_key = fmix32(static_cast<uint32_t>(__ldg(p.spos + row)) ^ p.seed);
      }
      for (int t = t0; t < t1; ++t) {
        mbar_wait_sleep(&tfull[acc], acc_phase, MOSAIC_K3_EPI_SLEEP_NS);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
        const int64_t col_base = static_cast<int64_t>(t) * BN;
#pragma unroll 1
        for (int c = half * kChunksPerHalf; c < (half + 1) * kChunksPerHalf; ++c) {
          const int64_t col0 = col_base + c * 32;
          if (col0 >= p.V) break;  // warp-uniform: vocab tail
          float v[32];
          tmem_ld32(taddr + c * 32, v);
          if constexpr (kStoreLogits) {
            if (row < M) {
              float* dst = p.out + row * p.ldo + col0;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j < p.V) dst[j] = v[j];
            }
          } else {
            if (col0 + 32 > p.V) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j >= p.V) v[j] = -INFINITY;
            }
            float cmax = v[0];
#pragma unroll
            for (int j = 1; j < 32; ++j) cmax = fmaxf(cmax, v[j]);
            if (cmax > run_max) {  // strict: earlier columns win ties
              if constexpr (!kSample) {  // (the sampling variant's token is the noisy argmax below)
                int jf = 31;
#pragma unroll
                for (int j = 31; j >= 0; --j)
                  if (v[j] == cmax) jf = j;
                run_arg = col0 + jf;
              }
              run_sum *= fast_exp2((run_max - cmax) * kLog2e);
              run_max = cmax;
            }
            const float mb2 = run_max * kLog2e;
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              s0 += fast_exp2(fmaf(v[j + 0], kLog2e, -mb2));
              s1 += fast_exp2(fmaf(v[j + 1], kLog2e, -mb2));
              s2 += fast_exp2(fmaf(v[j + 2], kLog2e, -mb2));
              s3 += fast_exp2(fmaf(v[j + 3], kLog2e, -mb2));
            }
            run_sum += (s0 + s1) + (s2 + s3);
            if constexpr (kSample) {
              // y = x + T * g, g = -ln(-ln u), u from (seed, position, global vocab id);
              // strict > in ascending columns: the lowest id wins ties. g <= 16.64 for every
              // u the hash can produce, so a chunk with cmax + T * 16.7 < s_ymax cannot win
              // and its noise is skipped when that holds for all 32 rows of the warp (exact)
              const bool cannot_win = cmax + p.temperature * 16.7f < s_ymax;
              const uint32_t cg0 = static_cast<uint32_t>(p.v_offset + col0);
              if (!__all_sync(0xffffffffu, cannot_win))
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const uint32_t h = fmix32(row_key ^ (cg0 + j) * 0x9E3779B1u);
                // u = (h23 + 0.5) / 2^23 is exact in fp32 and strictly inside (0, 1); the inner log
                // is the accurate logf (u can sit within 2^-24 of 1), the outer one the fast MUFU form
                const float u = (static_cast<float>(h >> 9) + 0.5f) * 1.1920928955078125e-7f;
                const float g = -__logf(-logf(u));
                const float y = fmaf(p.temperature, g, v[j]);
                if (y > s_ymax) {  // v[j] = -inf past the vocab tail: never chosen
                  s_ymax = y;
                  s_xarg = v[j];
                  run_arg = col0 + j;
                }
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(tempty_addr0 + acc * 8);
          else mbar_arrive(&tempty[acc]);
        }
        if (++acc == NUM_ACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if constexpr (!kStoreLogits) {
        if (row < M) {
          const int64_t o = (static_cast<int64_t>(s) * kHalves + half) * p.m_cap + row;
          p.part_max[o] = run_max;
          p.part_sum[o] = run_sum;
          p.part_arg[o] = static_cast<int32_t>(p.v_offset + run_arg);  // sampling: the noisy argmax
          if constexpr (kSample) {
            p.part_y[o] = s_ymax;
            p.part_x[o] = s_xarg;
          }
        }
      }
    }
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {  // the allocating warp frees
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, TMEM_COLS);
  }
}

int cta_group_for(int64_t m_cap) {
  static int forced = [] {
    const char* e = getenv("MOSAIC_CTA_GROUP");
    return e ? atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2) return forced;
  return m_cap > BM ? 2 : 1;  // a lone 128-row block would leave half a pair idle
}

int env_int(const char* name, int fallback) {
  const char* e = getenv(name);
  return e ? atoi(e) : fallback;
}

int group_m_default() {
  static int g = [] {
    const char* e = getenv("MOSAIC_GROUP_M");
    return e ? atoi(e) : 0;
  }();
  return g;
}

void plan_splits(int64_t m_cap, int64_t V, int32_t* n_splits, int32_t* tps) {
  const int cg = cta_group_for(m_cap);
  const int64_t n_tiles = ceil_div(V, BN);
  const int64_t m_blocks = ceil_div(m_cap > 0 ? m_cap : 1, BM * cg);
  const int64_t workers = num_sms() / cg;
  int64_t best_cost = INT64_MAX, best_tps = n_tiles;
  // Split cap: kMaxSplits bounds the [S][m_cap] partials for large M; with a
  // single row block (M <= 256, e.g. semi-autoregressive block decoding) the
  // splits are the only parallelism and the launch streams the whole W shard,
  // so the cap rises to one split per worker (profiles/r01h_k3_small_m.txt).
  const int64_t max_splits = std::max<int64_t>(kMaxSplits, ceil_div(workers, m_blocks));
  static const int forced_tps = env_int("MOSAIC_K3_TPS", 0);  // schedule experiments only
  if (forced_tps > 0 && ceil_div(n_tiles, std::min<int64_t>(forced_tps, n_tiles)) <= max_splits) {
    *tps = static_cast<int32_t>(std::min<int64_t>(forced_tps, n_tiles));
    *n_splits = static_cast<int32_t>(ceil_div(n_tiles, *tps));
    return;
  }
  // Pass 1: the least busiest-pair load (tiles). Pass 2: among loads within
  // 0.5% of it, the unit length closest to kPreferTps tiles -- measured on B200
  // (profiles/r01b_k3_schedule_sweep.txt): ~13-tile units keep the m-group's
  // rows and the shared LM-head tiles L2-resident best, which lowers DRAM
  // traffic and with it the power-capped clock penalty.
  constexpr int64_t kPreferTps = 13;
  auto cost_of = [&](int64_t t) { return ceil_div(m_blocks * ceil_div(n_tiles, t), workers) * t; };
  for (int64_t t = n_tiles; t >= 1; --t) {
    const int64_t S = ceil_div(n_tiles, t);
    if (S > max_splits) break;
    if (ceil_div(n_tiles, S) != t) continue;  // same split count as a larger t
    best_cost = std::min(best_cost, cost_of(t));
  }
  int64_t best_dist = INT64_MAX;
  for (int64_t t = n_tiles; t >= 1; --t) {
    const int64_t S = ceil_div(n_tiles, t);
    if (S > max_splits) break;
    if (ceil_div(n_tiles, S) != t) continue;
    if (cost_of(t) * 1000 > best_cost * 1005) continue;
    const int64_t dist = t > kPreferTps ? t - kPreferTps : kPreferTps - t;
    if (dist < best_dist) {
      best_dist = dist;
      best_tps = t;
    }
  }
  *tps = static_cast<int32_t>(best_tps);
  *n_splits = static_cast<int32_t>(ceil_div(n_tiles, best_tps));
}

template <int CG, bool kStore, int kGather, bool kSample = false>
int launch_cg(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& th, const Params& p,
              int64_t m_cap, cudaStream_t stream) {
  using C = Cfg<CG>;
  auto kern = k3_lmhead<CG, kStore, kGather, kSample>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    MOSAIC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  const int64_t units_cap = ceil_div(m_cap, C::ROWS) * p.n_splits;
  static const int max_clusters = env_int("MOSAIC_K3_MAX_CLUSTERS", 0);  // experiment: fewer SMs
  const int64_t workers = max_clusters > 0 ? std::min<int64_t>(max_clusters, num_sms() / CG) : num_sms() / CG;
  const int64_t clusters = units_cap < workers ? units_cap : workers;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * CG));
  cfg.blockDim = dim3(threads_for(kGather, kSample));
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (common.cuh)
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  MOSAIC_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, th, p));
  return MOSAIC_OK;
}

// A operand source: a dense [m_cap, d] buffer (Hc, K2's output) or, in gather
// mode, the hidden states H [n_rows, d] (row stride ld_h) read at idx[].
struct ASource {
  const uint16_t* base;
  int64_t rows;
  int64_t ld;
  const int32_t* idx;  // non-null = gather mode
  int32_t shift;
  const uint16_t* hc = nullptr;  // runs mode: the [m_cap, d] buffer of the scattered tiles' rows (base = H)
};

template <bool kStore>
int launch(const ASource& a, int64_t m_cap, const int32_t* m_dev, int64_t m_host, const uint16_t* W, int64_t V,
           int64_t d, Params p, void* stream) {
  MOSAIC_REQUIRE(d > 0 && d % BK == 0, "d=%lld must be a positive multiple of %d", (long long)d, BK);
  MOSAIC_REQUIRE(V >= 1 && V < (int64_t(1) << 31), "vocab shard %lld out of range", (long long)V);
  MOSAIC_REQUIRE(m_cap >= 0 && m_cap < (int64_t(1) << 31), "m_cap out of range");
  MOSAIC_REQUIRE(m_dev != nullptr || (m_host >= 0 && m_host <= m_cap), "m_host=%lld > m_cap=%lld",
                 (long long)m_host, (long long)m_cap);
  MOSAIC_REQUIRE((reinterpret_cast<uintptr_t>(a.base) & 15) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0,
                 "A rows and W must be 16-byte aligned");
  MOSAIC_REQUIRE(a.ld >= d && a.ld % 8 == 0, "row stride %lld must be >= d and a multiple of 8", (long long)a.ld);
  if (m_cap == 0) return MOSAIC_OK;
  const bool runs = a.hc != nullptr;
  const bool gather = a.idx != nullptr && !runs;
  MOSAIC_REQUIRE(!runs || (a.idx != nullptr && !kStore && p.part_y == nullptr), "runs mode: stats path only");
  MOSAIC_REQUIRE(!runs || (reinterpret_cast<uintptr_t>(a.hc) & 15) == 0, "Hc must be 16-byte aligned");
  const int cg = cta_group_for(m_cap);  // gather mode included: pairs measured faster since the
                                        // per-stage sync is CTA-scope only (r01_k3_gather_modes.txt)
  CUtensorMap ta, tb, th;
  static const int gmode = env_int("MOSAIC_K3_GATHER", kGatherCpAsync);  // 1 = TMA gather4 (measured slower)
  // gather4 reads single rows of H; the cp.async path's contiguous-run tiles read 128-row boxes of H
  int st = gather ? encode_tma_bf16(&ta, a.base, a.rows, d, a.ld, (gmode == kGatherTma4 && !kStore) ? 1 : BM, BK)
           : runs ? encode_tma_bf16(&ta, a.hc, m_cap, d, d, BM, BK)
                  : encode_tma_bf16(&ta, a.base, m_cap, d, a.ld, BM, BK);
  if (st) return st;
  if (runs) {
    st = encode_tma_bf16(&th, a.base, a.rows, d, a.ld, BM, BK);  // H: contiguous-run tiles' boxes
    if (st) return st;
  } else {
    th = ta;  // unused
  }
  // experiment: W handed over pre-tiled as [n_tiles][d/64][256][64] (each TMA box one contiguous 32 KB block)
  static const int w_blocked = env_int("MOSAIC_K3_WBLOCKED", 0);
  p.w_blocked = w_blocked;
  st = w_blocked ? encode_tma_bf16(&tb, W, ceil_div(V, BN) * (d / BK) * BN, BK, BK, BN / cg, BK)
                 : encode_tma_bf16(&tb, W, V, d, d, BN / cg, BK);
  if (st) return st;
  p.m_dev = m_dev;
  p.m_host = m_host;
  p.m_cap = m_cap;
  p.V = V;
  p.K = static_cast<int32_t>(d);
  p.n_tiles = static_cast<int32_t>(ceil_div(V, BN));
  p.idx = a.idx;
  p.shift = a.shift;
  if (p.group_m <= 0) p.group_m = group_m_default() > 0 ? group_m_default() : 16;
  static const int seg_splits = env_int("MOSAIC_K3_SEG_SPLITS", 0);
  p.seg_splits = seg_splits;
  // L2 policy of the (A, B) loads: A (the m-group's rows, re-read for every vocab tile) evict_last, B
  // (an LM-head tile, consumed by the group's units within one wave and dead after) evict_first --
  // measured best under the dynamic schedule (+2.2% steady over evict_last A alone,
  // profiles/r02r_k3_l2_policy_dynamic.txt)
  static const int policy = env_int("MOSAIC_L2_POLICY", 3);
  p.policy = policy;
  cudaStream_t s = as_stream(stream);
  MOSAIC_REQUIRE(p.die_of_sm == nullptr || p.sched != nullptr, "the die map needs the dynamic schedule's scratch");
  MOSAIC_REQUIRE(p.sched == nullptr || !kStore, "materialised logits use the static schedule");
  static const int force_static = env_int("MOSAIC_K3_STATIC", 0);  // experiment: the static schedule
  // a launch of at most two units per pair gains nothing from claiming (and
  // the counters' memset would cost a launch): small heads keep the static order
  const int64_t pairs = num_sms() / cg;
  const bool few_units = ceil_div(m_cap, static_cast<int64_t>(BM) * cg) * p.n_splits <= 2 * pairs;
  if (force_static || few_units) {
    p.sched = nullptr;
    p.die_of_sm = nullptr;
  }
  if (p.sched != nullptr) {  // dynamic schedule: counters start at zero every launch
    p.n_sm = num_sms();      // the die table holds one entry per SM (hotpath.die_map)
    MOSAIC_CUDA(cudaMemsetAsync(p.sched, 0, 16, s));
  }
  if (runs) {
    st = cg == 2 ? launch_cg<2, false, kGatherRuns>(ta, tb, th, p, m_cap, s)
                 : launch_cg<1, false, kGatherRuns>(ta, tb, th, p, m_cap, s);
  } else if (gather) {
    p.h = a.base;
    p.ld_h = a.ld;
    if constexpr (kStore) {  // materialised logits straight from H at idx (the drop-in gather_gemm)
      st = cg == 2 ? launch_cg<2, true, kGatherCpAsync>(ta, tb, th, p, m_cap, s)
                   : launch_cg<1, true, kGatherCpAsync>(ta, tb, th, p, m_cap, s);
    } else if (gmode == kGatherTma4) {
      st = cg == 2 ? launch_cg<2, false, kGatherTma4>(ta, tb, th, p, m_cap, s)
                   : launch_cg<1, false, kGatherTma4>(ta, tb, th, p, m_cap, s);
    } else {
      st = cg == 2 ? launch_cg<2, false, kGatherCpAsync>(ta, tb, th, p, m_cap, s)
                   : launch_cg<1, false, kGatherCpAsync>(ta, tb, th, p, m_cap, s);
    }
  } else {
    if (p.part_y != nullptr) {  // sampling variant (buffered A only)
      st = cg == 2 ? launch_cg<2, false, kGatherNone, true>(ta, tb, th, p, m_cap, s)
                   : launch_cg<1, false, kGatherNone, true>(ta, tb, th, p, m_cap, s);
    } else {
      st = cg == 2 ? launch_cg<2, kStore, kGatherNone>(ta, tb, th, p, m_cap, s)
                   : launch_cg<1, kStore, kGatherNone>(ta, tb, th, p, m_cap, s);
    }
  }
  if (st) return st;
  return check_launch(kStore ? "mosaic_lmhead_logits" : "mosaic_lmhead_stats");
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

extern "C" int mosaic_lmhead_plan(int64_t m_cap, int64_t V_shard, int64_t d, int32_t* n_splits_out,
                                  int32_t* tiles_per_split_out) {
  MOSAIC_REQUIRE(V_shard >= 1 && d >= 1, "empty shard");
  MOSAIC_REQUIRE(n_splits_out && tiles_per_split_out, "null outputs");
  plan_splits(m_cap, V_shard, n_splits_out, tiles_per_split_out);
  return MOSAIC_OK;
}

extern "C" int mosaic_lmhead_stats(const uint16_t* Hc, int64_t m_cap, const int32_t* m_dev,
                                   int64_t m_host, const uint16_t* W, int64_t V_shard, int64_t d,
                                   int64_t v_offset, int32_t n_splits, float* part_max,
                                   float* part_sum, int32_t* part_arg, void* stream) {
  MOSAIC_REQUIRE(part_max && part_sum && part_arg, "null partial buffers");
  const int64_t n_tiles = ceil_div(V_shard, BN);
  MOSAIC_REQUIRE(n_splits >= 1 && n_splits <= n_tiles, "n_splits=%d not in [1, %lld]", n_splits,
                 (long long)n_tiles);
  Params p{};
  p.tiles_per_split = static_cast<int32_t>(ceil_div(n_tiles, n_splits));
  p.n_splits = static_cast<int32_t>(ceil_div(n_tiles, p.tiles_per_split));
  MOSAIC_REQUIRE(p.n_splits == n_splits, "n_splits=%d does not tile %lld vocab tiles evenly; use mosaic_lmhead_plan",
                 n_splits, (long long)n_tiles);
  p.v_offset = v_offset;
  p.part_max = part_max;
  p.part_sum = part_sum;
  p.part_arg = part_arg;
  return launch<false>(ASource{Hc, m_cap, d, nullptr, 0}, m_cap, m_dev, m_host, W, V_shard, d, p, stream);
}

extern "C" int mosaic_lmhead_stats_die(const uint16_t* Hc, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                                       const uint16_t* W, int64_t V_shard, int64_t d, int64_t v_offset,
                                       int32_t n_splits, float* part_max, float* part_sum, int32_t* part_arg,
                                       const uint8_t* die_of_sm, uint32_t* sched_scratch, void* stream) {
  MOSAIC_REQUIRE(part_max && part_sum && part_arg, "null partial buffers");
  const int64_t n_tiles = ceil_div(V_shard, BN);
  MOSAIC_REQUIRE(n_splits >= 1 && n_splits <= n_tiles, "n_splits=%d not in [1, %lld]", n_splits,
                 (long long)n_tiles);
  Params p{};
  p.tiles_per_split = static_cast<int32_t>(ceil_div(n_tiles, n_splits));
  p.n_splits = static_cast<int32_t>(ceil_div(n_tiles, p.tiles_per_split));
  MOSAIC_REQUIRE(p.n_splits == n_splits, "n_splits=%d does not tile %lld vocab tiles evenly; use mosaic_lmhead_plan",
                 n_splits, (long long)n_tiles);
  p.v_offset = v_offset;
  p.part_max = part_max;
  p.part_sum = part_sum;
  p.part_arg = part_arg;
  p.die_of_sm = die_of_sm;
  p.sched = sched_scratch;
  return launch<false>(ASource{Hc, m_cap, d, nullptr, 0}, m_cap, m_dev, m_host, W, V_shard, d, p, stream);
}

extern "C" int mosaic_lmhead_sample(const uint16_t* Hc, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                                    const uint16_t* W, int64_t V_shard, int64_t d, int64_t v_offset,
                                    int32_t n_splits, const int32_t* pos, float temperature, uint32_t seed,
                                    float* part_max, float* part_sum, int32_t* part_arg, float* part_y,
                                    float* part_x, const uint8_t* die_of_sm, uint32_t* sched_scratch,
                                    void* stream) {
  MOSAIC_REQUIRE(part_max && part_sum && part_arg && part_y && part_x && pos, "null operands");
  MOSAIC_REQUIRE(temperature > 0.f && temperature < 1e30f, "temperature must be positive (0 = argmax: use "
                 "mosaic_lmhead_stats)");
  MOSAIC_REQUIRE(die_of_sm == nullptr || sched_scratch != nullptr, "the die map needs the dynamic schedule's scratch");
  const int64_t n_tiles = ceil_div(V_shard, BN);
  MOSAIC_REQUIRE(n_splits >= 1 && n_splits <= n_tiles, "n_splits=%d not in [1, %lld]", n_splits,
                 (long long)n_tiles);
  Params p{};
  p.tiles_per_split = static_cast<int32_t>(ceil_div(n_tiles, n_splits));
  p.n_splits = static_cast<int32_t>(ceil_div(n_tiles, p.tiles_per_split));
  MOSAIC_REQUIRE(p.n_splits == n_splits, "n_splits=%d does not tile %lld vocab tiles evenly; use mosaic_lmhead_plan",
                 n_splits, (long long)n_tiles);
  p.v_offset = v_offset;
  p.part_max = part_max;
  p.part_sum = part_sum;
  p.part_arg = part_arg;
  p.part_y = part_y;
  p.part_x = part_x;
  p.spos = pos;
  p.temperature = temperature;
  p.seed = seed;
  p.die_of_sm = die_of_sm;
  p.sched = sched_scratch;
  return launch<false>(ASource{Hc, m_cap, d, nullptr, 0}, m_cap, m_dev, m_host, W, V_shard, d, p, stream);
}

namespace {
int lmhead_stats_gather_impl(const uint16_t* H, int64_t n_rows, int64_t ld_h, const int32_t* idx, int32_t shift,
                             int64_t m_cap, const int32_t* m_dev, int64_t m_host, const uint16_t* W,
                             int64_t V_shard, int64_t d, int64_t v_offset, int32_t n_splits, float* part_max,
                             float* part_sum, int32_t* part_arg, const uint8_t* die_of_sm, uint32_t* sched,
                             void* stream) {
  MOSAIC_REQUIRE(H && idx && part_max && part_sum && part_arg, "null operands");
  MOSAIC_REQUIRE(n_rows >= 1 && n_rows < (int64_t(1) << 31), "n_rows out of range");
  const int64_t n_tiles = ceil_div(V_shard, BN);
  MOSAIC_REQUIRE(n_splits >= 1 && n_splits <= n_tiles, "n_splits=%d not in [1, %lld]", n_splits,
                 (long long)n_tiles);
  Params p{};
  p.tiles_per_split = static_cast<int32_t>(ceil_div(n_tiles, n_splits));
  p.n_splits = static_cast<int32_t>(ceil_div(n_tiles, p.tiles_per_split));
  MOSAIC_REQUIRE(p.n_splits == n_splits, "n_splits=%d does not tile %lld vocab tiles evenly; use mosaic_lmhead_plan",
                 n_splits, (long long)n_tiles);
  p.v_offset = v_offset;
  p.part_max = part_max;
  p.part_sum = part_sum;
  p.part_arg = part_arg;
  p.die_of_sm = die_of_sm;
  p.sched = sched;
  return launch<false>(ASource{H, n_rows, ld_h, idx, shift & 3}, m_cap, m_dev, m_host, W, V_shard, d, p,
                       stream);
}
}  // namespace

extern "C" int mosaic_lmhead_stats_gather(const uint16_t* H, int64_t n_rows, int64_t ld_h, const int32_t* idx,
                                          int32_t shift, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                                          const uint16_t* W, int64_t V_shard, int64_t d, int64_t v_offset,
                                          int32_t n_splits, float* part_max, float* part_sum, int32_t* part_arg,
                                          void* stream) {
  return lmhead_stats_gather_impl(H, n_rows, ld_h, idx, shift, m_cap, m_dev, m_host, W, V_shard, d, v_offset,
                                  n_splits, part_max, part_sum, part_arg, nullptr, nullptr, stream);
}

extern "C" int mosaic_lmhead_stats_gather_die(const uint16_t* H, int64_t n_rows, int64_t ld_h, const int32_t* idx,
                                              int32_t shift, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                                              const uint16_t* W, int64_t V_shard, int64_t d, int64_t v_offset,
                                              int32_t n_splits, float* part_max, float* part_sum,
                                              int32_t* part_arg, const uint8_t* die_of_sm, uint32_t* sched_scratch,
                                              void* stream) {
  MOSAIC_REQUIRE(sched_scratch, "the dynamic schedule needs its 16-byte scratch (die_of_sm optional)");
  return lmhead_stats_gather_impl(H, n_rows, ld_h, idx, shift, m_cap, m_dev, m_host, W, V_shard, d, v_offset,
                                  n_splits, part_max, part_sum, part_arg, die_of_sm, sched_scratch, stream);
}

extern "C" int mosaic_lmhead_stats_runs(const uint16_t* H, int64_t n_rows, int64_t ld_h, const int32_t* idx,
                                        int32_t shift, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                                        const uint16_t* Hc, const uint16_t* W, int64_t V_shard, int64_t d,
                                        int64_t v_offset, int32_t n_splits, float* part_max, float* part_sum,
                                        int32_t* part_arg, const uint8_t* die_of_sm, uint32_t* sched_scratch,
                                        void* stream) {
  MOSAIC_REQUIRE(H && idx && Hc && part_max && part_sum && part_arg, "null operands");
  MOSAIC_REQUIRE(n_rows >= 1 && n_rows < (int64_t(1) << 31), "n_rows out of range");
  MOSAIC_REQUIRE(die_of_sm == nullptr || sched_scratch != nullptr, "the die map needs the dynamic schedule's 16-byte scratch");
  const int64_t n_tiles = ceil_div(V_shard, BN);
  MOSAIC_REQUIRE(n_splits >= 1 && n_splits <= n_tiles, "n_splits=%d not in [1, %lld]", n_splits,
                 (long long)n_tiles);
  Params p{};
  p.tiles_per_split = static_cast<int32_t>(ceil_div(n_tiles, n_splits));
  p.n_splits = static_cast<int32_t>(ceil_div(n_tiles, p.tiles_per_split));
  MOSAIC_REQUIRE(p.n_splits == n_splits, "n_splits=%d does not tile %lld vocab tiles evenly; use mosaic_lmhead_plan",
                 n_splits, (long long)n_tiles);
  p.v_offset = v_offset;
  p.part_max = part_max;
  p.part_sum = part_sum;
  p.part_arg = part_arg;
  p.die_of_sm = die_of_sm;
  p.sched = sched_scratch;
  ASource a{H, n_rows, ld_h, idx, shift & 3};
  a.hc = Hc;
  return launch<false>(a, m_cap, m_dev, m_host, W, V_shard, d, p, stream);
}

extern "C" int mosaic_lmhead_logits_gather(const uint16_t* H, int64_t n_rows, int64_t ld_h, const int32_t* idx,
                                           int32_t shift, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                                           const uint16_t* W, int64_t V_shard, int64_t d, float* out, int64_t ldo,
                                           void* stream) {
  MOSAIC_REQUIRE(H && idx, "null operands");
  MOSAIC_REQUIRE(n_rows >= 1 && n_rows < (int64_t(1) << 31), "n_rows out of range");
  MOSAIC_REQUIRE(out != nullptr && ldo >= V_shard, "bad logits output");
  Params p{};
  p.tiles_per_split = static_cast<int32_t>(ceil_div(V_shard, BN));
  p.n_splits = 1;
  p.out = out;
  p.ldo = ldo;
  return launch<true>(ASource{H, n_rows, ld_h, idx, shift & 3}, m_cap, m_dev, m_host, W, V_shard, d, p, stream);
}

extern "C" int mosaic_lmhead_config(int64_t m_cap, int32_t gather, int64_t* out) {
  MOSAIC_REQUIRE(out != nullptr, "null output");
  const int cg = cta_group_for(m_cap);
  const bool cp = gather != 0;
  out[0] = cg;                                                   // SMs per tile (cta_group)
  out[1] = cg == 2 ? Cfg<2>::STAGES : Cfg<1>::STAGES;            // shared-memory ring stages
  out[2] = BM;                                                   // A rows staged per CTA
  out[3] = BK;                                                   // K per stage
  out[4] = BN / cg;                                              // W rows staged per CTA
  out[5] = TMEM_COLS;                                            // TMEM columns (fp32 x 128 lanes)
  out[6] = cg == 2 ? Cfg<2>::SMEM : Cfg<1>::SMEM;                // dynamic shared memory per CTA (bytes)
  out[7] = threads_for(cp ? kGatherCpAsync : kGatherNone, false);
  return MOSAIC_OK;
}

extern "C" int mosaic_lmhead_logits(const uint16_t* Hc, int64_t m_cap, const int32_t* m_dev,
                                    int64_t m_host, const uint16_t* W, int64_t V_shard, int64_t d,
                                    float* out, int64_t ldo, void* stream) {
  MOSAIC_REQUIRE(out != nullptr && ldo >= V_shard, "bad logits output");
  Params p{};
  const int64_t n_tiles = ceil_div(V_shard, BN);
  p.tiles_per_split = static_cast<int32_t>(n_tiles);
  p.n_splits = 1;
  p.out = out;
  p.ldo = ldo;
  return launch<true>(ASource{Hc, m_cap, d, nullptr, 0}, m_cap, m_dev, m_host, W, V_shard, d, p, stream);
}
