/* One fused mask-only logits + remask step through the C ABI alone -- what a
 * non-Python host (the reference's FFI) links against: plain
 * C, the CUDA runtime for device buffers, include/mosaic_b200.h, and
 * libmosaic_b200.so. K1 compact -> K2 gather -> K3 statistics GEMM (dynamic
 * unit schedule) -> K4 merge -> K5 remask commit, then a host check: argmax of
 * fp64 dot products of the same bf16 operands on the rows whose top-1 margin
 * exceeds 1e-3, and exactly k commits.
 *
 *   gcc -O2 -std=c11 examples/capi_step.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2601_06562_b200 -lmosaic_b200 -L/usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,paper_2601_06562_b200 -o build/capi_step && build/capi_step
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mosaic_b200.h"

#define CK(call)                                                                       \
  do {                                                                                 \
    int st_ = (call);                                                                  \
    if (st_) {                                                                         \
      fprintf(stderr, "%s failed (%d): %s\n", #call, st_, mosaic_last_error());        \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)
#define CUDA(call)                                                                     \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));                      \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

static uint64_t rng = 0x9E3779B97F4A7C15ull;
static double uniform(void) { /* xorshift64*, (0, 1) */
  rng ^= rng >> 12; rng ^= rng << 25; rng ^= rng >> 27;
  return ((rng * 0x2545F4914F6CDD1Dull) >> 11) * (1.0 / 9007199254740992.0) + 1e-17;
}
static double normal(void) { return sqrt(-2.0 * log(uniform())) * cos(6.283185307179586 * uniform()); }
static uint16_t to_bf16(float f) { /* round to nearest even */
  uint32_t u; memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static double from_bf16(uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; }

int main(void) {
  const int64_t L = 4096, d = 256, V = 8192;
  const int32_t mask_id = (int32_t)V - 1;
  const int64_t k = 64;
  printf("mosaic ABI %d\n", mosaic_abi_version());
  int32_t* x = (int32_t*)malloc(L * 4);
  uint16_t* H = (uint16_t*)malloc(L * d * 2);
  uint16_t* W = (uint16_t*)malloc(V * d * 2);
  for (int64_t i = 0; i < L; ++i) x[i] = uniform() < 0.5 ? mask_id : (int32_t)(uniform() * (V - 1));
  for (int64_t i = 0; i < L * d; ++i) H[i] = to_bf16((float)normal());
  for (int64_t i = 0; i < V * d; ++i) W[i] = to_bf16((float)(0.05 * normal()));

  int32_t S = 0, tps = 0;
  CK(mosaic_lmhead_plan(L, V, d, &S, &tps));
  int32_t *dx, *didx, *dm, *dtok, *dsel, *darg;
  uint16_t *dH, *dW, *dHc;
  float *dmax, *dsum, *dlse, *dconf;
  void *csc, *rsc;
  uint32_t* dsched;
  const size_t csb = mosaic_mask_compact_scratch_bytes(L), rsb = mosaic_remask_scratch_bytes();
  CUDA(cudaMalloc((void**)&dx, L * 4)); CUDA(cudaMalloc((void**)&didx, L * 4)); CUDA(cudaMalloc((void**)&dm, 4));
  CUDA(cudaMalloc((void**)&dH, L * d * 2)); CUDA(cudaMalloc((void**)&dW, V * d * 2));
  CUDA(cudaMalloc((void**)&dHc, L * d * 2));
  CUDA(cudaMalloc((void**)&dmax, (size_t)S * L * 4)); CUDA(cudaMalloc((void**)&dsum, (size_t)S * L * 4));
  CUDA(cudaMalloc((void**)&darg, (size_t)S * L * 4));
  CUDA(cudaMalloc((void**)&dtok, L * 4)); CUDA(cudaMalloc((void**)&dlse, L * 4)); CUDA(cudaMalloc((void**)&dconf, L * 4));
  CUDA(cudaMalloc((void**)&dsel, L * 4)); CUDA(cudaMalloc(&csc, csb)); CUDA(cudaMalloc(&rsc, rsb));
  CUDA(cudaMalloc((void**)&dsched, 16));
  CUDA(cudaMemcpy(dx, x, L * 4, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dH, H, L * d * 2, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dW, W, V * d * 2, cudaMemcpyHostToDevice));
  cudaStream_t s;
  CUDA(cudaStreamCreate(&s));

  /* the step: every launch reads the masked count from the device (dm) */
  CK(mosaic_mask_compact(dx, L, mask_id, didx, dm, csc, s));
  CK(mosaic_gather_rows(dH, L, d, d, didx, dm, 0, L, 0, dHc, s));
  CK(mosaic_lmhead_stats_die(dHc, L, dm, 0, dW, V, d, 0, S, dmax, dsum, darg, NULL, dsched, s));
  CK(mosaic_stats_merge(dmax, dsum, darg, S, L, dm, 0, L, NULL, NULL, NULL, dtok, dlse, dconf, s));
  CK(mosaic_remask_commit(dconf, didx, dtok, dm, 0, L, k, dx, dsel, rsc, s));
  CUDA(cudaStreamSynchronize(s));

  int32_t M = 0;
  CUDA(cudaMemcpy(&M, dm, 4, cudaMemcpyDeviceToHost));
  int32_t* idx = (int32_t*)malloc(L * 4); int32_t* tok = (int32_t*)malloc(L * 4);
  int32_t* sel = (int32_t*)malloc(L * 4); int32_t* xo = (int32_t*)malloc(L * 4);
  CUDA(cudaMemcpy(idx, didx, M * 4, cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(tok, dtok, M * 4, cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(sel, dsel, M * 4, cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(xo, dx, L * 4, cudaMemcpyDeviceToHost));

  int64_t expect_m = 0, n_sel = 0, checked = 0, bad = 0;
  for (int64_t i = 0; i < L; ++i) expect_m += x[i] == mask_id;
  if (M != expect_m) { fprintf(stderr, "masked count %d != %lld\n", M, (long long)expect_m); return 1; }
  for (int32_t r = 0; r < M; ++r) {
    n_sel += sel[r];
    if (r % 16) continue; /* argmax of fp64 logits on every 16th row */
    double best = -1e300, second = -1e300; int32_t arg = 0;
    for (int64_t v = 0; v < V; ++v) {
      double z = 0;
      for (int64_t j = 0; j < d; ++j) z += from_bf16(H[idx[r] * d + j]) * from_bf16(W[v * d + j]);
      if (z > best) { second = best; best = z; arg = (int32_t)v; } else if (z > second) second = z;
    }
    if (best - second > 1e-3) { ++checked; bad += tok[r] != arg; }
    if (sel[r] && xo[idx[r]] != tok[r]) { fprintf(stderr, "row %d committed wrong token\n", r); return 1; }
  }
  if (n_sel != (k < M ? k : M) || bad) {
    fprintf(stderr, "commits %lld (want %lld), argmax mismatches %lld of %lld\n", (long long)n_sel,
            (long long)(k < M ? k : M), (long long)bad, (long long)checked);
    return 1;
  }
  printf("capi ok: L=%lld M=%d splits=%d, %lld rows' argmax vs fp64, %lld committed\n", (long long)L, M, S,
         (long long)checked, (long long)n_sel);
  return 0;
}
