/*
 * mosaic_b200.h — C ABI of the B200-native mask-only logits + remask hot path.
 *
 * This is the drop-in boundary for the reference's hot-path operator
 * (`gather_gemm`, /root/reference/pkg/src/mosaic/kernel.py:62-86) and for the
 * memory-only graph ops that surround it in the step template
 * (`gather_logits` / `sample` / `commit`, mosaic/workload.py:287-315), plus the
 * workspace reservation/commit it runs out of (mosaic/vmm.py:48-147).
 *
 * Conventions (every entry point):
 *   - returns an int status: MOSAIC_OK (0) or one of the error codes below; the
 *     Python host maps them onto the reference exception hierarchy
 *     (mosaic/errors.py: InputError / CapacityError / ResourceError);
 *     mosaic_last_error() returns a thread-local message for the last failure;
 *   - all device buffers are caller-owned (arena views); nothing allocates
 *     device memory except the arena functions;
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *     all kernels are enqueued asynchronously on it, no host synchronisation;
 *   - element types: hidden states / LM-head weights are bf16 (uint16 bits),
 *     indices int32, statistics fp32;
 *   - a masked-row count may be given on the device (`m_dev`, int32, e.g. the
 *     output of mosaic_mask_compact) so that a whole step can be enqueued or
 *     graph-captured without a device->host round trip; when m_dev is NULL the
 *     host value m_host is used. Buffers are sized for the capacity m_cap.
 */
#ifndef MOSAIC_B200_H_
#define MOSAIC_B200_H_

#include <stddef.h>
#include <stdint.h>
#include <sys/types.h> /* ssize_t (the pluggable-allocator signature) */

#if defined(__GNUC__)
#define MOSAIC_API __attribute__((visibility("default")))
#else
#define MOSAIC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum mosaic_status {
  MOSAIC_OK = 0,
  MOSAIC_E_INPUT = 1,       /* malformed arguments  -> InputError     (errors.py:41-42) */
  MOSAIC_E_CAPACITY = 2,    /* commit > reservation -> CapacityError  (errors.py:33-34) */
  MOSAIC_E_RESOURCE = 3,    /* VA/physical alloc    -> ResourceError  (errors.py:29-30) */
  MOSAIC_E_CUDA = 4,        /* CUDA runtime/driver failure                              */
  MOSAIC_E_UNSUPPORTED = 5  /* shape the kernels do not support (e.g. d % 64 != 0)      */
};

/* ABI version (major*100 + minor) and the last error message of this thread. */
MOSAIC_API int mosaic_abi_version(void);
MOSAIC_API const char* mosaic_last_error(void);

/* L2 set-aside for persisting (evict_last) lines on the current device:
 * min(bytes, device maximum); *applied_out receives the limit now in force.
 * K3 keeps its A operand evict_last, so the set-aside decides whether the
 * gathered rows survive the LM-head weight stream in L2. Device-global.     */
MOSAIC_API int mosaic_l2_persisting_limit(int64_t bytes, int64_t* applied_out);

/* Native first-fit planner (host): groups given in placement order (the
 * reference's def asc, size desc, id asc; mosaic/planner.py:107-142) with
 * byte sizes and inclusive live intervals [def_idx, last_idx]; offsets_out[i]
 * = lowest multiple of `alignment` that collides with no earlier-placed,
 * lifetime-overlapping group; *workspace_out = max(offset + size).          */
MOSAIC_API int mosaic_first_fit(int64_t n, const int64_t* sizes, const int64_t* def_idx,
                     const int64_t* last_idx, int64_t alignment, int64_t* offsets_out,
                     int64_t* workspace_out);

/* ---------------------------------------------------------------- K1 ------
 * Mask compaction: idx_out[0..M) = ascending positions p with x[p] == mask_id,
 * *m_out = M (device int32). Restates np.flatnonzero(x == MASK_ID); the
 * reference takes mask_idx as a ready graph input (workload.py:199-200) and
 * only validates it (kernel.py:42-49).
 * `scratch` must hold mosaic_mask_compact_scratch_bytes(L) bytes.            */
MOSAIC_API size_t mosaic_mask_compact_scratch_bytes(int64_t L);
MOSAIC_API int mosaic_mask_compact(const int32_t* x, int64_t L, int32_t mask_id,
                        int32_t* idx_out, int32_t* m_out,
                        void* scratch, void* stream);

/* Batched windows (MaskOnlyHead.step_batch): rows[r] = b * ls + src(lo + j)
 * for the compacted window coordinate q[r] = b * wn + j, r < M; src(p) =
 * max(p - 1, 0) with shift = 1. One launch instead of host-side index math. */
MOSAIC_API int mosaic_window_rows(const int32_t* q, const int32_t* m_dev, int64_t m_host, int64_t m_cap,
                       int64_t wn, int64_t ls, int64_t lo, int32_t shift, int32_t* rows, void* stream);

/* ---------------------------------------------------------------- K2 ------
 * Row gather: Hc[i, :] = H[src(idx[i]), :] for i < M, src(p) = p (shift=0) or
 * max(p-1, 0) (shift=1, Dream's token-level shift, workload.py:295-303).
 * Replaces the indirect panel fetch `H[rows, k0:k1]` of kernel.py:77.
 * H: [n_rows, d] with row stride ld_h (elements); Hc: [m_cap, d] dense.
 * d must be a multiple of 8 and ld_h too (16-byte rows).                    */
MOSAIC_API int mosaic_gather_rows(const uint16_t* H, int64_t n_rows, int64_t ld_h, int64_t d,
                       const int32_t* idx, const int32_t* m_dev, int64_t m_host,
                       int64_t m_cap, int32_t shift, uint16_t* Hc, void* stream);

/* Runs mode of K2: as mosaic_gather_rows, but the rows of every full K3 tile
 * (tile_rows consecutive compacted rows: 256 with cta_group::2, 128 with
 * cta_group::1 -- mosaic_lmhead_config out[0] * out[2]) whose source rows are
 * one contiguous run of H are skipped: mosaic_lmhead_stats_runs reads those
 * tiles straight from H. Same indirect fetch it replaces (kernel.py:77).     */
MOSAIC_API int mosaic_gather_rows_scattered(const uint16_t* H, int64_t n_rows, int64_t ld_h, int64_t d,
                                 const int32_t* idx, const int32_t* m_dev, int64_t m_host,
                                 int64_t m_cap, int32_t shift, int32_t tile_rows, uint16_t* Hc,
                                 void* stream);

/* ---------------------------------------------------------------- K3 ------
 * Mask-only LM head with the fused softmax-statistics epilogue.
 * For every row r < M of Hc [m_cap, d] and every vocab split s of the shard
 * W [V_shard, d] (row-major, K-major for TMA/UMMA; the reference stores the
 * transpose [d, V], kernel.py:26):
 *   part_max[s*m_cap + r] = max_{v in split s} logit(r, v)
 *   part_sum[s*m_cap + r] = sum_{v in split s} exp(logit(r, v) - part_max)
 *   part_arg[s*m_cap + r] = v_offset + argmax (lowest index on ties)
 * with logit(r, v) = <Hc[r, :], W[v, :]> in fp32 (tcgen05, bf16 operands).
 * The [M, V] logits are never written. n_splits is chosen by
 * mosaic_lmhead_plan() and the partial buffers hold n_splits*m_cap entries.
 * d must be a multiple of 64, V_shard >= 1.                                  */
MOSAIC_API int mosaic_lmhead_plan(int64_t m_cap, int64_t V_shard, int64_t d, int32_t* n_splits_out,
                       int32_t* tiles_per_split_out);
MOSAIC_API int mosaic_lmhead_stats(const uint16_t* Hc, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                        const uint16_t* W, int64_t V_shard, int64_t d, int64_t v_offset,
                        int32_t n_splits, float* part_max, float* part_sum, int32_t* part_arg,
                        void* stream);

/* K3 with the dynamic unit schedule (MaskOnlyHead's default): the pairs claim
 * work units (row block x vocab split, numbered m-fastest inside groups of 16
 * row blocks) from counters in sched_scratch (16 caller-owned device bytes,
 * zeroed by the call; one launch at a time per scratch), so the units in flight
 * stay one contiguous window of the order and each split's LM-head tiles are
 * shared through L2 (DRAM per LLaDA 32k launch 5.8 GB vs 12.1 GB for the
 * static order the plain entry point keeps). die_of_sm (optional, device
 * uint8 [num SMs] from mosaic_die_map, 0/1): pairs on die 1 claim from the back
 * of the order instead of the front. Same outputs bit for bit as
 * mosaic_lmhead_stats for any schedule and any map.                          */
MOSAIC_API int mosaic_lmhead_stats_die(const uint16_t* Hc, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                            const uint16_t* W, int64_t V_shard, int64_t d, int64_t v_offset,
                            int32_t n_splits, float* part_max, float* part_sum, int32_t* part_arg,
                            const uint8_t* die_of_sm, uint32_t* sched_scratch, void* stream);

/* SM -> L2-die map, measured (two cold-read latency classes; see
 * csrc/topology.cu), for the optional die split of the dynamic schedule.
 * die_of_sm_host receives 0/1 per SM (255 = unknown); scratch holds
 * mosaic_die_map_scratch_bytes(n_sm) device bytes. Synchronises `stream`.
 * *ambiguous_out counts SMs without a clear class.                          */
MOSAIC_API size_t mosaic_die_map_scratch_bytes(int32_t n_sm);
MOSAIC_API int mosaic_die_map(uint8_t* die_of_sm_host, int32_t n_sm, void* scratch, int32_t* n_die0_out,
                   int32_t* ambiguous_out, void* stream);

/* Gather mode of K3 -- the paper's gather-GEMM with no intermediate buffer:
 * the A rows are read straight from the hidden states H [n_rows, d] (row
 * stride ld_h elements) at the masked positions idx[0..M) (src(p) = p, or
 * max(p-1, 0) with shift = 1) by cp.async loader warps (16-byte segments,
 * swizzled in software to the UMMA layout), so K2 and the [m_cap, d]
 * compacted buffer disappear. Outputs as mosaic_lmhead_stats. The _die form
 * takes the dynamic schedule (arguments as mosaic_lmhead_stats_die).         */
MOSAIC_API int mosaic_lmhead_stats_gather(const uint16_t* H, int64_t n_rows, int64_t ld_h, const int32_t* idx,
                               int32_t shift, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                               const uint16_t* W, int64_t V_shard, int64_t d, int64_t v_offset,
                               int32_t n_splits, float* part_max, float* part_sum, int32_t* part_arg,
                               void* stream);
MOSAIC_API int mosaic_lmhead_stats_gather_die(const uint16_t* H, int64_t n_rows, int64_t ld_h, const int32_t* idx,
                                   int32_t shift, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                                   const uint16_t* W, int64_t V_shard, int64_t d, int64_t v_offset,
                                   int32_t n_splits, float* part_max, float* part_sum, int32_t* part_arg,
                                   const uint8_t* die_of_sm, uint32_t* sched_scratch, void* stream);

/* Runs mode of K3 (the product default): per 256-row pair tile (128 with
 * cta_group::1) the A operand is one TMA box of H itself when the tile's
 * source rows src(idx[r]) are consecutive -- the reference schedule's step-0
 * suffix, semi-autoregressive blocks -- and otherwise one TMA box of Hc, where
 * mosaic_gather_rows_scattered compacted that tile's rows. Both A sources
 * feed the dense TMA pipeline, so every tile runs at the dense rate and the
 * gathered copy shrinks to the scattered tiles. Replaces gather_gemm
 * (kernel.py:62-86) like mosaic_lmhead_stats, with identical outputs;
 * sched_scratch (16 B) selects the dynamic schedule, die_of_sm its optional
 * die split (both null = static schedule).                                  */
MOSAIC_API int mosaic_lmhead_stats_runs(const uint16_t* H, int64_t n_rows, int64_t ld_h, const int32_t* idx,
                             int32_t shift, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                             const uint16_t* Hc, const uint16_t* W, int64_t V_shard, int64_t d,
                             int64_t v_offset, int32_t n_splits, float* part_max, float* part_sum,
                             int32_t* part_arg, const uint8_t* die_of_sm, uint32_t* sched_scratch,
                             void* stream);

/* Sampling variant of K3 (temperature > 0; the reference's `sample` op is
 * memory-only, this follows LLaDA's generate): per masked row r the token is
 * argmax_v (x_v + temperature * g), g = -ln(-ln u), u = ((h >> 9) + 0.5) / 2^23,
 * h = fmix32(fmix32(pos[r] ^ seed) ^ (v * 0x9E3779B1)) with v the global vocab
 * id (murmur3 finaliser; so samples do not depend on the split, the vocab
 * shard or the chunking) -- lowest id on ties. Partials per split: the usual
 * (max, sum-exp) of the untempered logits, part_arg = the noisy argmax,
 * part_y = its noisy score, part_x = its raw logit; every partial buffer holds
 * 2 * n_splits * m_cap entries (each split's two 128-column halves are written
 * separately: merge with S = 2 * n_splits). mosaic_sample_merge gives token,
 * lse and conf = exp(x_token - lse) (the untempered p(token)).                */
MOSAIC_API int mosaic_lmhead_sample(const uint16_t* Hc, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                         const uint16_t* W, int64_t V_shard, int64_t d, int64_t v_offset,
                         int32_t n_splits, const int32_t* pos, float temperature, uint32_t seed,
                         float* part_max, float* part_sum, int32_t* part_arg, float* part_y,
                         float* part_x, const uint8_t* die_of_sm, uint32_t* sched_scratch, void* stream);
MOSAIC_API int mosaic_sample_merge(const float* in_max, const float* in_sum, const int32_t* in_arg,
                        const float* in_y, const float* in_x, int32_t S, int64_t stride,
                        const int32_t* m_dev, int64_t m_host, int64_t m_cap, int32_t* token,
                        float* lse, float* conf, void* stream);

/* Debug / parity path for the reference operator itself: out[r, v] =
 * <Hc[r, :], W[v, :]> in fp32, row stride ldo. Materialises the logits like
 * gather_gemm (kernel.py:68); the product path never calls it.               */
/* Materialised logits with the A rows read from H at idx (gather mode: no
 * [m, d] gathered copy), the parity form of gather_gemm (kernel.py:62-86)
 * under the ScratchAccount contract ("no [m x d] gathered copy is
 * ever materialized"). out [m_cap, ldo] fp32; shift = Dream src(p)=max(p-1,0). */
MOSAIC_API int mosaic_lmhead_logits_gather(const uint16_t* H, int64_t n_rows, int64_t ld_h, const int32_t* idx,
                                           int32_t shift, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                                           const uint16_t* W, int64_t V_shard, int64_t d, float* out, int64_t ldo,
                                           void* stream);
/* The launched K3 configuration for a problem of m_cap rows, the device
 * counterpart of ScratchAccount (kernel.py:52-59): out[8] = {cta_group,
 * smem stages, A rows per CTA, K per stage, W rows per CTA, TMEM columns,
 * dynamic shared memory bytes per CTA, threads per CTA}; gather != 0 selects
 * the gather-mode (cp.async A) kernel.                                        */
MOSAIC_API int mosaic_lmhead_config(int64_t m_cap, int32_t gather, int64_t* out);
MOSAIC_API int mosaic_lmhead_logits(const uint16_t* Hc, int64_t m_cap, const int32_t* m_dev, int64_t m_host,
                         const uint16_t* W, int64_t V_shard, int64_t d,
                         float* out, int64_t ldo, void* stream);

/* ---------------------------------------------------------------- K4 ------
 * Merge S partial triples per row (fixed ascending-s order; larger max wins,
 * lower index on equal max), in layout [S][stride]. Any of the outputs may be
 * NULL: (out_max, out_sum, out_arg) receive the merged triple (used before the
 * cross-rank exchange); (token, lse, conf) the finalised sample:
 * token = argmax, lse = max + ln(sum), conf = p(token) = 1/sum.
 * Realises the memory-only `sample` op (workload.py:306-308).                */
MOSAIC_API int mosaic_stats_merge(const float* in_max, const float* in_sum, const int32_t* in_arg,
                       int32_t S, int64_t stride, const int32_t* m_dev, int64_t m_host,
                       int64_t m_cap, float* out_max, float* out_sum, int32_t* out_arg,
                       int32_t* token, float* lse, float* conf, void* stream);

/* ---------------------------------------------------------------- K4x -----
 * Vocab-shard exchange fused into the split merge, over NVLink peer memory:
 * push merges the S split triples of every row r < M (K4 rule) and stores the
 * merged (max, sum, arg-bits) into slot [epoch & 1][rank] of every rank's
 * double-buffered gathered block [2][world][3][m_cap] fp32 (peer_gathered:
 * device array of `world` pointers to those blocks), then publishes `epoch`
 * into every rank's signal pad slot [rank] (peer_signal: device array of
 * `world` uint32 pointers; release.sys); wait blocks the stream until the
 * local pad's `world` slots equal `epoch` (acquire.sys, bounded: traps if a
 * peer never arrives). Then mosaic_stats_merge over half (epoch & 1) of the
 * local block (S=world, stride=3*m_cap) finalises. Alternating halves keep a
 * rank that is one step ahead from overwriting triples a peer has not merged.
 * Replaces K4 + all-gather + K4 of the NCCL path. done_counter: one local
 * uint32, 0. epoch: 1, 2, 3, ... (never 0, the pads' initial value).      */
MOSAIC_API int mosaic_stats_exchange_push(const float* in_max, const float* in_sum, const int32_t* in_arg,
                               int32_t S, int64_t stride, const int32_t* m_dev, int64_t m_host,
                               int64_t m_cap, float* const* peer_gathered, uint32_t* const* peer_signal,
                               int32_t rank, int32_t world, uint32_t epoch, uint32_t* done_counter,
                               void* stream);
MOSAIC_API int mosaic_stats_exchange_wait(const uint32_t* local_signal, int32_t world, uint32_t epoch,
                               void* stream);

/* ---------------------------------------------------------------- K5 ------
 * Low-confidence remasking commit (memory-only `commit` op, workload.py:315):
 * among the M masked rows keep the k with the highest confidence (ties ->
 * lower position pos[r]) and write x[pos[r]] = token[r] for them; the others
 * stay masked. selected (optional, int32 [m_cap]) receives 1/0 per row.
 * `scratch` must hold mosaic_remask_scratch_bytes() bytes. k is clamped to M. */
MOSAIC_API size_t mosaic_remask_scratch_bytes(void);
MOSAIC_API int mosaic_remask_commit(const float* conf, const int32_t* pos, const int32_t* token,
                         const int32_t* m_dev, int64_t m_host, int64_t m_cap, int64_t k,
                         int32_t* x, int32_t* selected, void* scratch, void* stream);

/* K5 per segment (batched sequences / semi-autoregressive blocks): the rows
 * whose position pos[r] lies in [b * seg_len, (b + 1) * seg_len) form segment
 * b (a contiguous run of the ascending compacted list; one CTA each), which
 * keeps its own k_b most confident rows (ties -> lower position) and commits
 * x[pos[r]] = token[r] for them. k_b = k_per_seg[b] (device int32 [n_seg]) or
 * `k` when k_per_seg is null; k_b is clamped to the segment's row count.
 * Extends the reference's single-sequence `commit` (workload.py:315) to a
 * batch; no scratch needed.                                                  */
MOSAIC_API int mosaic_remask_commit_segmented(const float* conf, const int32_t* pos, const int32_t* token,
                                   const int32_t* m_dev, int64_t m_host, int64_t m_cap, int64_t seg_len,
                                   int32_t n_seg, const int32_t* k_per_seg, int64_t k, int32_t* x,
                                   int32_t* selected, void* stream);

/* ---------------------------------------------------------------- K6 ------
 * Fused SwiGLU of one FFN chunk, in place: up[i] = silu(gate[i]) * up[i],
 * bf16, n elements (the in-place `glu` op of the chunked FFN loop,
 * workload.py:249-259). gate/up 16-byte aligned.                              */
MOSAIC_API int mosaic_swiglu(const uint16_t* gate, uint16_t* up, int64_t n, void* stream);

/* ---------------------------------------------------------------- K11 -----
 * Rotary position embedding (rotate-half, LLaDA/LLaMA form) of the attention
 * queries and keys, in place: q, k [L, ld] bf16 rows of n_heads x head_dim;
 * inv_freq [head_dim / 2] fp32 (theta^(-2i/head_dim)); row r has position
 * pos0 + r. The reference's `fused_attention` op (workload.py:207-229) is
 * memory-only; the executor applies this before the attention so masked rows
 * carry their positions. head_dim a multiple of 16, q/k 16-byte aligned.     */
MOSAIC_API int mosaic_rope_qk(uint16_t* q, uint16_t* k, int64_t L, int32_t n_heads, int32_t head_dim, int64_t ld,
                              const float* inv_freq, int64_t pos0, void* stream);

/* ---------------------------------------------------------------- K8/K9 ---
 * MoE expert routing and combine for the chunked expert FFN (BASELINE
 * configs[3]). The reference models MoE only as a top_k multiplier on the FFN
 * chunk rows (mosaic/workload.py:195,238-253); these realise the routing those
 * rows stand for.
 * mosaic_moe_route: for each of `rows` router-logit rows (fp32, stride ld):
 *   top_k experts by (logit desc, expert asc), weights = softmax over the
 *   selected logits; assignments are ordered (expert, row, j) ascending:
 *   disp_row[p] = row_base + row of dispatch slot p (and disp_w[p], optional),
 *   comb_pos[row*top_k + j] = p, comb_w[row*top_k + j] = weight,
 *   expert_off[0..E] = segment offsets (device int32, E+1 entries).
 * `scratch` holds mosaic_moe_route_scratch_bytes(rows, E) bytes. E <= 256,
 * top_k <= 16.
 * mosaic_moe_combine: out[r, :] = sum_j comb_w[r*k+j] * src[comb_pos[r*k+j], :]
 *   (bf16 in/out, fp32 accumulation in ascending j), d % 8 == 0.             */
MOSAIC_API size_t mosaic_moe_route_scratch_bytes(int64_t rows, int32_t n_experts);
MOSAIC_API int mosaic_moe_route(const float* logits, int64_t ld, int64_t rows, int32_t n_experts,
                     int32_t top_k, int32_t row_base, int32_t* disp_row, float* disp_w,
                     int32_t* comb_pos, float* comb_w, int32_t* expert_off, void* scratch,
                     void* stream);
MOSAIC_API int mosaic_moe_combine(const uint16_t* src, int64_t ld_src, const int32_t* comb_pos,
                       const float* comb_w, int64_t rows, int32_t top_k, int64_t d,
                       uint16_t* out, int64_t ld_out, void* stream);

/* ---------------------------------------------------------------- K10 -----
 * Grouped tcgen05 GEMM of the FFN chunk (workload.py:231-273, MoE rows
 * :238-253): for each group g < G, rows [off[g], off[g+1]) of A [rows_cap, K]
 * (row stride lda) times W[g] = W rows [g*N, (g+1)*N) (K-major, i.e. torch's
 * [K, N] weight transposed) into C (row stride ldc), bf16 in/out, fp32
 * accumulation. group_off is a device int32 array of G+1 offsets (the K8
 * expert_off output), or NULL for one group of m_host rows. swiglu = 1: W
 * rows alternate 128-row gate / up blocks and C receives silu(gate) * up,
 * N/2 columns -- the ffn_up + ffn_gate + glu ops of a chunk in one kernel.
 * K % 64 == 0, N % 32 == 0 (N % 256 == 0 with swiglu), G <= 256.            */
MOSAIC_API int mosaic_ffn_gemm(const uint16_t* A, int64_t rows_cap, int64_t lda, const int32_t* group_off,
                    int32_t G, int64_t m_host, const uint16_t* W, int64_t N, int64_t K, int32_t swiglu,
                    uint16_t* C, int64_t ldc, void* stream);
/* The same GEMM with an epilogue selector: 0 store C = A W^T, 1 SwiGLU (as
 * swiglu = 1 above), 2 residual C += A W^T in place (fp32 sum rounded once):
 * the dense chunk's ffn_down + chunk_write + ffn_res add (workload.py:261-272)
 * in one launch, written straight into the chunk's rows of the hidden state.  */
MOSAIC_API int mosaic_ffn_gemm_ex(const uint16_t* A, int64_t rows_cap, int64_t lda, const int32_t* group_off,
                                  int32_t G, int64_t m_host, const uint16_t* W, int64_t N, int64_t K,
                                  int32_t epilogue, uint16_t* C, int64_t ldc, void* stream);
/* mosaic_ffn_gemm_ex with K3's dynamic unit schedule: sched_scratch (16
 * caller-owned device bytes, zeroed by the call; one launch at a time per
 * scratch) holds the counter the SM pairs claim output tiles from, so the
 * tiles in flight stay one contiguous window of the m-grouped order (null =
 * the static order of mosaic_ffn_gemm_ex). Identical outputs.               */
MOSAIC_API int mosaic_ffn_gemm_sched(const uint16_t* A, int64_t rows_cap, int64_t lda, const int32_t* group_off,
                                     int32_t G, int64_t m_host, const uint16_t* W, int64_t N, int64_t K,
                                     int32_t epilogue, uint16_t* C, int64_t ldc, uint32_t* sched_scratch,
                                     void* stream);

/* ---------------------------------------------------------------- K7 ------
 * Contiguous device workspace with lazy physical commitment (cuMem VMM):
 * reserve a VA range once, map physical granules for the prefix
 * [0, round_up(target, granularity)). Mirrors Workspace/reserve/commit_to of
 * mosaic/vmm.py:48-147 with a `cuda` backend.                                */
typedef struct mosaic_arena mosaic_arena;
MOSAIC_API int mosaic_arena_reserve(int32_t device, uint64_t reserve_bytes, mosaic_arena** out);
MOSAIC_API int mosaic_arena_commit(mosaic_arena* arena, uint64_t target_bytes);
MOSAIC_API int mosaic_arena_info(const mosaic_arena* arena, uint64_t* base, uint64_t* reserved,
                      uint64_t* committed, uint64_t* granularity);
MOSAIC_API int mosaic_arena_release(mosaic_arena* arena);

/* The arena's torch-scratch region as a PyTorch pluggable allocator
 * (torch.cuda.memory.CUDAPluggableAllocator(lib, "mosaic_pool_alloc",
 * "mosaic_pool_free") inside a torch.cuda.MemPool): library temporaries of the
 * step (attention outputs) are carved from a committed region at the start of
 * the executor's own arena instead of fresh cudaMallocs -- the reference's
 * single-workspace contract (vmm.py:48-147, budget workload.py:362-369).
 * Regions are keyed by base address (one per arena): bind creates or resizes
 * one in place (live blocks stay valid; a shrink below one fails), select
 * picks the region new allocations come from, unbind forgets one whose arena
 * is released. alloc returns NULL when the selected region is exhausted (torch
 * then raises out-of-memory); stats reports bytes in use, the high-water
 * mark, allocations served and refused.                                      */
MOSAIC_API int mosaic_pool_bind(int32_t device, void* base, uint64_t size);
MOSAIC_API int mosaic_pool_select(int32_t device, void* base);
MOSAIC_API int mosaic_pool_unbind(int32_t device, void* base);
MOSAIC_API void* mosaic_pool_alloc(ssize_t size, int device, void* stream);
MOSAIC_API void mosaic_pool_free(void* ptr, ssize_t size, int device, void* stream);
MOSAIC_API int mosaic_pool_stats(int32_t device, void* base, uint64_t* in_use, uint64_t* high_water,
                                 uint64_t* n_alloc, uint64_t* n_fail);

/* Plan-executor canaries (execute_plan, mosaic/vmm.py:188-291) on device
 * memory: fill [ptr, ptr+nbytes) with the 8-byte tag repeated from ptr; check
 * adds to *mismatch_count (device uint32) when any byte differs. ptr 8-byte
 * aligned (plan offsets are).                                                 */
MOSAIC_API int mosaic_tag_fill(void* ptr, int64_t nbytes, uint64_t tag, void* stream);
MOSAIC_API int mosaic_tag_check(const void* ptr, int64_t nbytes, uint64_t tag, uint32_t* mismatch_count,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOSAIC_B200_H_ */
