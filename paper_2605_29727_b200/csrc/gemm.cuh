// Stream-K schedule helpers shared by the GEMM and its consumer kernels.
#pragma once
#include <cuda.h>
#include "../../include/bastion.h"

namespace bst {

// CTA c owns units [floor(c*U/G), floor((c+1)*U/G)); unit = tile*n_kb + k_block.
__host__ __device__ __forceinline__ int sched_first_cta(const bst_gemm_sched_t& s, int tile) {
  int64_t a = ((int64_t)tile * s.n_kb + 1) * s.grid;
  int64_t c = (a + s.units - 1) / s.units - 1;
  return (int)(c < 0 ? 0 : (c >= s.grid ? s.grid - 1 : c));
}
__host__ __device__ __forceinline__ int sched_last_cta(const bst_gemm_sched_t& s, int tile) {
  int64_t a = ((int64_t)(tile + 1) * s.n_kb) * s.grid;
  int64_t c = (a + s.units - 1) / s.units - 1;
  return (int)(c < 0 ? 0 : (c >= s.grid ? s.grid - 1 : c));
}

// Y[t, n] = sum of the tile's partial slots, lowest k range first (deterministic).
__device__ __forceinline__ float gemm_load(const float* __restrict__ partial, const bst_gemm_sched_t& s, int t,
                                           int n) {
  const int tile = n >> 7, r = n & 127;
  const int nslot = sched_last_cta(s, tile) - sched_first_cta(s, tile) + 1;
  const float* p = partial + ((int64_t)tile * s.s_max * s.bn + t) * 128 + r;
  float acc = 0.f;
  for (int k = 0; k < nslot; ++k) acc += p[(int64_t)k * s.bn * 128];
  return acc;
}

int make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t row_stride,
                   uint32_t box_rows, uint32_t box_cols);
int cached_tmap(CUtensorMap* out, const void* ptr, uint64_t rows, uint64_t cols, uint64_t stride, uint32_t br,
                uint32_t bc);

}  // namespace bst
