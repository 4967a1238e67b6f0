// K10: grouped tcgen05 GEMM for the lazily chunked FFN, with an optional
// SwiGLU epilogue -- the FFN chunk's up/gate projections and activation in one
// kernel (act = silu(x Wg) * (x Wu) straight from the TMEM accumulators, so
// neither `gate` nor `up` is ever written), and the down projection.
//
// Reference counterpart: the FFN chunk loop of the step template
// (mosaic/workload.py:231-273: ffn_up / ffn_gate / glu / ffn_down per chunk of
// ceil(L/K_FFN) rows, x top_k rows for MoE, :195,238-253). The MoE routing
// (K8) orders the chunk's dispatch rows by expert, so the experts' GEMMs are
// one grouped GEMM over contiguous row segments whose bounds stay on the
// device (no host round trip): group g multiplies rows
// [group_off[g], group_off[g+1]) of A by its own weight block W[g].
//
// Layout: A [rows, K] bf16 (row stride lda), W [G * N, K] bf16 K-major (the
// transpose of torch's [K, N] weight), C [rows, N or N/2] bf16 (row stride
// ldc). SwiGLU mode expects W rows interleaved in 128-row blocks (gate block
// j, then up block j) so one 256-column tile holds matching gate and up
// columns; it writes 128 act columns per tile. Residual mode (the dense FFN's
// down projection) accumulates in place, C = C + A W^T, rounding the fp32 sum
// once to bf16: the chunk's `ffn_down` -> `chunk_write` -> `ffn_res` add
// (mosaic/workload.py:261-272) in one epilogue, so neither the chunk's `down`
// rows nor the [L, d] `ffn_acc` accumulator is ever written.
//
// Structure as K3 (csrc/lmhead.cu): warp 0 TMEM allocator + TMA producer, warp 1
// single-thread tcgen05.mma issuer (cta_group::2 256x256 tiles over
// an SM pair by default, cta_group::1 128x256 for tiny row counts; BF16 ->
// FP32), warps 2-5 epilogue draining a double-buffered TMEM accumulator;
// persistent CTAs walk (m-block, n-tile) units rasterised in groups of
// `group_m` m-blocks so the weight tiles in flight are shared through L2.
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"

namespace mosaic {
namespace {

constexpr int BM = 128;   // rows per CTA (TMEM lanes)
constexpr int BN = 256;   // output (or gate|up) columns per tile
constexpr int BK = 64;
constexpr int UK = 16;
constexpr int NUM_ACC = 2;
constexpr int TMEM_COLS = 512;
constexpr int kThreads = 192;
constexpr int kEpiWarps = 4;
constexpr int kMaxGroups = 256;
constexpr int kGroupM = 16;
constexpr int kURing = 16;  // dynamic schedule's unit ring (as K3, csrc/lmhead.cu)

// CG = 2: a CTA pair computes a 256 x 256 tile (tcgen05.mma.cta_group::2),
// each CTA staging half of the rows and half of the weight columns, as K3.
template <int CG>
struct GCfg {
  static constexpr int ROWS = BM * CG;   // rows per unit (UMMA M)
  static constexpr int B_ROWS = BN / CG;  // weight rows staged per CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = CG == 1 ? 4 : 6;
  static constexpr int OFF_RING = STAGES * STAGE_BYTES + 256 + 2 * (kMaxGroups + 1) * 4;  // 8-byte aligned
  static constexpr int SMEM = OFF_RING + kURing * 12 + 1024;
  static constexpr uint32_t IDESC = umma_idesc_bf16(ROWS, BN);
};

struct GParams {
  const int32_t* group_off;  // [G + 1] device row offsets, or null: one group of m_host rows
  int32_t G;
  int64_t m_host;
  int64_t N;        // weight rows per group (output columns; 2 x act columns with SwiGLU)
  int32_t K;
  int32_t n_tiles;  // ceil(N / BN)
  int32_t swiglu;
  int32_t residual;  // C += A W^T (read-modify-write of each output vector)
  uint16_t* C;
  int64_t ldc;
  uint32_t* sched;  // dynamic schedule: [unused, next unit, ...], zeroed per launch; null = static schedule
  int32_t group_m;  // m-blocks per raster group (units m-fastest inside a group)
  int32_t b_evict_first;  // L2 policy of the weight tiles: evict_first (default) or evict_normal
};

__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.f + __expf(-g)); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// unit -> (group, first row, end row of the group, n-tile)
struct Unit {
  int g;
  int64_t row0;
  int64_t row_end;
  int nt;
};

template <int ROWS>
__device__ __forceinline__ Unit unit_of(int64_t u, int n_tiles, int total_mb, const int32_t* s_off,
                                        const int32_t* s_mbp, int G, int group_m) {
  const int64_t per_group = static_cast<int64_t>(group_m) * n_tiles;
  const int64_t gi = u / per_group;
  const int64_t rem = u - gi * per_group;
  const int64_t gm = min(static_cast<int64_t>(group_m), total_mb - gi * group_m);
  const int nt = static_cast<int>(rem / gm);
  const int gmb = static_cast<int>(gi * group_m + rem % gm);
  int lo = 0, hi = G - 1;  // largest g with s_mbp[g] <= gmb
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_mbp[mid] <= gmb) lo = mid;
    else hi = mid - 1;
  }
  Unit r;
  r.g = lo;
  r.row0 = s_off[lo] + static_cast<int64_t>(gmb - s_mbp[lo]) * ROWS;
  r.row_end = s_off[lo + 1];
  r.nt = nt;
  return r;
}

template <int CG>
__global__ void __launch_bounds__(kThreads, 1)
    k10_ffn_gemm(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                 const GParams p) {
  using C = GCfg<CG>;
  constexpr int STAGES = C::STAGES, A_BYTES = C::A_BYTES, B_BYTES = C::B_BYTES, STAGE_BYTES = C::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + NUM_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NUM_ACC);
  int32_t* s_off = reinterpret_cast<int32_t*>(smem + STAGES * STAGE_BYTES + 256);
  int32_t* s_mbp = s_off + kMaxGroups + 1;
  uint64_t* ufull = reinterpret_cast<uint64_t*>(smem + C::OFF_RING);  // unit ring: id published
  int32_t* uring = reinterpret_cast<int32_t*>(ufull + kURing);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = p.G;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const int64_t cluster = blockIdx.x / CG;
  const int64_t n_clusters = gridDim.x / CG;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < NUM_ACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps * CG);
    }
    for (int i = 0; i < kURing; ++i) mbar_init(&ufull[i], 1);
    fence_mbar_init();
    // group row offsets and the exclusive prefix of their m-block counts
    int32_t mb = 0;
    for (int g = 0; g <= G; ++g) {
      const int32_t o = p.group_off ? __ldg(p.group_off + g) : (g == 0 ? 0 : static_cast<int32_t>(p.m_host));
      s_off[g] = o;
      s_mbp[g] = mb;
      if (g < G) {
        const int32_t cnt = (p.group_off ? __ldg(p.group_off + g + 1) : static_cast<int32_t>(p.m_host)) - o;
        mb += (cnt + C::ROWS - 1) / C::ROWS;
      }
    }
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
  const int total_mb = s_mbp[G];
  const int64_t units = static_cast<int64_t>(total_mb) * p.n_tiles;
  const int k_blocks = p.K / BK;

  // Unit schedule as K3's (csrc/lmhead.cu): static striding, or -- with a
  // sched scratch -- units claimed from a global counter by the pair leader's
  // producer (one claim ahead) and published to both CTAs through the ring, so
  // the tiles in flight stay one contiguous window of the m-grouped order
  // instead of drifting apart.
  const bool dyn = p.sched != nullptr;
  auto claim = [&]() -> int32_t {
    const uint32_t c = atomicAdd(p.sched + 1, 1u);
    return c < static_cast<uint32_t>(units) ? static_cast<int32_t>(c) : -1;
  };
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
        mbar_arrive_cluster(mapa_shared(smem_u32(&ufull[slot]), 1));
      }
      mbar_arrive(&ufull[slot]);
      return u;
    }
    if (CG == 2 && rank == 1) mbar_wait_cluster(&ufull[slot], (n / kURing) & 1);
    else mbar_wait(&ufull[slot], (n / kURing) & 1);
    return *reinterpret_cast<volatile int32_t*>(uring + slot);
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_last();
      const uint64_t pol_b = p.b_evict_first ? policy_evict_first() : policy_evict_normal();
      uint32_t stage = 0, phase = 0;
      for (int n = 0;; ++n) {
        const int64_t u = unit_at(n, dyn && rank == 0);
        if (u < 0) break;
        const Unit w = unit_of<C::ROWS>(u, p.n_tiles, total_mb, s_off, s_mbp, G, p.group_m);
        const int32_t a_row = static_cast<int32_t>(w.row0 + rank * BM);
        const int32_t b_row = static_cast<int32_t>(w.g * p.N + static_cast<int64_t>(w.nt) * BN + rank * C::B_ROWS);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], STAGE_BYTES * CG);
          if constexpr (CG == 1) {
            tma_load_2d(sA + stage * A_BYTES, &tmap_a, &full[stage], kb * BK, a_row, pol_a);
            tma_load_2d(sB + stage * B_BYTES, &tmap_b, &full[stage], kb * BK, b_row, pol_b);
          } else {
            tma_load_2d_cg2(sA + stage * A_BYTES, &tmap_a, &full[stage], kb * BK, a_row, pol_a);
            tma_load_2d_cg2(sB + stage * B_BYTES, &tmap_b, &full[stage], kb * BK, b_row, pol_b);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (int n = 0;; ++n) {
        if (unit_at(n, false) < 0) break;
        if constexpr (CG == 2) mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
        else mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk)
            umma_bf16<CG>(d_tmem, umma_desc_sw128(a0 + kk * UK * 2), umma_desc_sw128(b0 + kk * UK * 2), C::IDESC,
                          (kb | kk) != 0);
          umma_commit<CG>(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit<CG>(&tfull[acc]);
        if (++acc == NUM_ACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int row_local = q * 32 + lane;
    const uint32_t tempty_addr0 = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]);
    uint32_t acc = 0, acc_phase = 0;
    for (int n = 0;; ++n) {
      int64_t u = 0;
      if (lane == 0) u = unit_at(n, false);
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u < 0) break;
      const Unit w = unit_of<C::ROWS>(u, p.n_tiles, total_mb, s_off, s_mbp, G, p.group_m);
      const int64_t row = w.row0 + rank * BM + row_local;
      const bool live = row < w.row_end;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      if (p.swiglu) {
        const int64_t n_out = p.N >> 1;
#pragma unroll 1
        for (int c = 0; c < BN / 64; ++c) {
          const int64_t col0 = static_cast<int64_t>(w.nt) * (BN / 2) + c * 32;
          float gv[32], uv[32];
          tmem_ld32(taddr + c * 32, gv);             // gate block columns
          tmem_ld32(taddr + BN / 2 + c * 32, uv);    // matching up block columns
          if (live && col0 < n_out) {
            uint4* dst = reinterpret_cast<uint4*>(p.C + row * p.ldc + col0);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 o;
              o.x = pack_bf16x2(silu(gv[8 * v + 0]) * uv[8 * v + 0], silu(gv[8 * v + 1]) * uv[8 * v + 1]);
              o.y = pack_bf16x2(silu(gv[8 * v + 2]) * uv[8 * v + 2], silu(gv[8 * v + 3]) * uv[8 * v + 3]);
              o.z = pack_bf16x2(silu(gv[8 * v + 4]) * uv[8 * v + 4], silu(gv[8 * v + 5]) * uv[8 * v + 5]);
              o.w = pack_bf16x2(silu(gv[8 * v + 6]) * uv[8 * v + 6], silu(gv[8 * v + 7]) * uv[8 * v + 7]);
              dst[v] = o;
            }
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          const int64_t col0 = static_cast<int64_t>(w.nt) * BN + c * 32;
          if (col0 >= p.N) break;  // warp-uniform (N % 32 == 0)
          float v32[32];
          tmem_ld32(taddr + c * 32, v32);
          if (live) {
            uint4* dst = reinterpret_cast<uint4*>(p.C + row * p.ldc + col0);
            if (p.residual) {
              uint4 r[4];
#pragma unroll
              for (int v = 0; v < 4; ++v) r[v] = dst[v];  // all four loads in flight before the adds
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&r[v]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float2 rf = __bfloat1622float2(r2[j]);
                  v32[8 * v + 2 * j] += rf.x;
                  v32[8 * v + 2 * j + 1] += rf.y;
                }
              }
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 o;
              o.x = pack_bf16x2(v32[8 * v + 0], v32[8 * v + 1]);
              o.y = pack_bf16x2(v32[8 * v + 2], v32[8 * v + 3]);
              o.z = pack_bf16x2(v32[8 * v + 4], v32[8 * v + 5]);
              o.w = pack_bf16x2(v32[8 * v + 6], v32[8 * v + 7]);
              dst[v] = o;
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
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {  // the allocating warp frees
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, TMEM_COLS);
  }
}

template <int CG>
int launch_k10(const CUtensorMap& ta, const CUtensorMap& tb, const GParams& p, int64_t rows_cap,
               cudaStream_t stream) {
  using C = GCfg<CG>;
  static bool attr_set = false;
  if (!attr_set) {
    MOSAIC_CUDA(cudaFuncSetAttribute(k10_ffn_gemm<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  const int64_t units_cap = (ceil_div(rows_cap, C::ROWS) + p.G) * p.n_tiles;
  const int64_t workers = num_sms() / CG;
  const int64_t clusters = units_cap < workers ? units_cap : workers;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * CG));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (p.sched != nullptr) MOSAIC_CUDA(cudaMemsetAsync(p.sched, 0, 16, stream));  // counters start at zero
  MOSAIC_CUDA(cudaLaunchKernelEx(&cfg, k10_ffn_gemm<CG>, ta, tb, p));
  return MOSAIC_OK;
}

}  // namespace
}  // namespace mosaic

using namespace mosaic;

extern "C" int mosaic_ffn_gemm(const uint16_t* A, int64_t rows_cap, int64_t lda, const int32_t* group_off, int32_t G,
                               int64_t m_host, const uint16_t* W, int64_t N, int64_t K, int32_t swiglu, uint16_t* C,
                               int64_t ldc, void* stream) {
  return mosaic_ffn_gemm_ex(A, rows_cap, lda, group_off, G, m_host, W, N, K, swiglu ? 1 : 0, C, ldc, stream);
}

extern "C" int mosaic_ffn_gemm_ex(const uint16_t* A, int64_t rows_cap, int64_t lda, const int32_t* group_off,
                                  int32_t G, int64_t m_host, const uint16_t* W, int64_t N, int64_t K, int32_t epilogue,
                                  uint16_t* C, int64_t ldc, void* stream) {
  return mosaic_ffn_gemm_sched(A, rows_cap, lda, group_off, G, m_host, W, N, K, epilogue, C, ldc, nullptr, stream);
}

extern "C" int mosaic_ffn_gemm_sched(const uint16_t* A, int64_t rows_cap, int64_t lda, const int32_t* group_off,
                                     int32_t G, int64_t m_host, const uint16_t* W, int64_t N, int64_t K,
                                     int32_t epilogue, uint16_t* C, int64_t ldc, uint32_t* sched_scratch,
                                     void* stream) {
  MOSAIC_REQUIRE(epilogue >= 0 && epilogue <= 2, "epilogue %d not in {0 store, 1 SwiGLU, 2 residual}", epilogue);
  const int32_t swiglu = epilogue == 1;
  MOSAIC_REQUIRE(A && W && C, "null operands");
  MOSAIC_REQUIRE(G >= 1 && G <= kMaxGroups, "G=%d not in [1, %d]", G, kMaxGroups);
  MOSAIC_REQUIRE(group_off != nullptr || G == 1, "several groups need device offsets");
  MOSAIC_REQUIRE(K >= BK && K % BK == 0, "K=%lld must be a positive multiple of %d", (long long)K, BK);
  MOSAIC_REQUIRE(N >= 32 && N % 32 == 0, "N=%lld must be a positive multiple of 32", (long long)N);
  MOSAIC_REQUIRE(!swiglu || N % BN == 0, "SwiGLU mode needs N (2 x d_ff) to be a multiple of %d", BN);
  MOSAIC_REQUIRE(lda >= K && lda % 8 == 0 && ldc % 8 == 0, "row strides must be multiples of 8 elements");
  MOSAIC_REQUIRE(ldc >= (swiglu ? N / 2 : N), "ldc too small");
  MOSAIC_REQUIRE(rows_cap >= 0 && rows_cap < (int64_t(1) << 31) && G * N < (int64_t(1) << 31), "sizes out of range");
  MOSAIC_REQUIRE(group_off != nullptr || (m_host >= 0 && m_host <= rows_cap), "m_host out of range");
  MOSAIC_REQUIRE((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(C) & 15) == 0,
                 "A, W, C must be 16-byte aligned");
  if (rows_cap == 0) return MOSAIC_OK;
  static const int forced = [] {
    const char* e = getenv("MOSAIC_K10_CTA_GROUP");
    return e ? atoi(e) : 0;
  }();
  const int cg = forced == 1 || forced == 2 ? forced : (rows_cap > BM ? 2 : 1);
  CUtensorMap ta, tb;
  int st = encode_tma_bf16(&ta, A, rows_cap, K, lda, BM, BK);
  if (st) return st;
  st = encode_tma_bf16(&tb, W, G * N, K, K, BN / cg, BK);
  if (st) return st;
  GParams p{};
  p.group_off = group_off;
  p.G = G;
  p.m_host = m_host;
  p.N = N;
  p.K = static_cast<int32_t>(K);
  p.n_tiles = static_cast<int32_t>(ceil_div(N, BN));
  p.swiglu = swiglu ? 1 : 0;
  p.residual = epilogue == 2 ? 1 : 0;
  p.C = C;
  p.ldc = ldc;
  static const int force_static = [] {
    const char* e = getenv("MOSAIC_K10_STATIC");
    return e ? atoi(e) : 0;
  }();
  // at most two tiles per pair: nothing to balance, keep the static order (and skip the counter memset)
  const int64_t tiles_cap = (ceil_div(rows_cap, static_cast<int64_t>(BM) * cg) + G) * p.n_tiles;
  p.sched = (force_static || tiles_cap <= 2 * (num_sms() / cg)) ? nullptr : sched_scratch;
  // raster group: the ~74 tiles in flight span g m-blocks x 74/g weight tiles, (g + 74/g) x 512 x K bytes
  // of L2. At K = 4096 the default 16 fits (41 MB); at the down projection's K = d_ff = 12288 it is 129 MB
  // and g = 8 (the minimum of g + 74/g) measured best: DRAM 6.0 -> 4.0 GB, 2.31 -> 2.20 ms per LLaDA
  // chunk (profiles/r02p_k10_group_m.txt; MOSAIC_K10_GROUP_M overrides)
  static const int forced_gm = [] {
    const char* e = getenv("MOSAIC_K10_GROUP_M");
    return e ? atoi(e) : 0;
  }();
  p.group_m = forced_gm > 0 ? forced_gm : (K > 8192 ? 8 : kGroupM);
  // weight tiles evict_first (as K3's LM-head tiles): gate/up 4.29 -> 4.24 ms, down 2.31 -> 2.25 ms per
  // LLaDA chunk under ncu (profiles/r02s_k10_l2_policy.txt); MOSAIC_K10_B_EVICT_FIRST=0 restores evict_normal
  static const int b_first = [] {
    const char* e = getenv("MOSAIC_K10_B_EVICT_FIRST");
    return e ? atoi(e) : 1;
  }();
  p.b_evict_first = b_first;
  st = cg == 2 ? launch_k10<2>(ta, tb, p, rows_cap, as_stream(stream))
               : launch_k10<1>(ta, tb, p, rows_cap, as_stream(stream));
  if (st) return st;
  return check_launch("mosaic_ffn_gemm");
}
