// Stream-K schedule helpers shared by the GEMM and its consumer kernels.
#pragma once
#include <cuda.h>
#include "../../include/bastion.h"

namespace bst {

// Stream-K over units = (super-tile, k_block); a super-tile is s.pair (1 or 2)
// consecutive 128-row weight tiles that share each X k-block.  CTA c owns units
// [floor(c*U/G), floor((c+1)*U/G)); unit = st*n_kb + k_block.
__host__ __device__ __forceinline__ int tile_st(const bst_gemm_sched_t& s, int tile) { return tile >> (s.pair >> 1); }
__host__ __device__ __forceinline__ int sched_first_st(const bst_gemm_sched_t& s, int st) {
  int64_t a = ((int64_t)st * s.n_kb + 1) * s.grid;
  int64_t c = (a + s.units - 1) / s.units - 1;
  return (int)(c < 0 ? 0 : (c >= s.grid ? s.grid - 1 : c));
}
__host__ __device__ __forceinline__ int sched_last_st(const bst_gemm_sched_t& s, int st) {
  int64_t a = ((int64_t)(st + 1) * s.n_kb) * s.grid;
  int64_t c = (a + s.units - 1) / s.units - 1;
  return (int)(c < 0 ? 0 : (c >= s.grid ? s.grid - 1 : c));
}
__host__ __device__ __forceinline__ int sched_first_cta(const bst_gemm_sched_t& s, int tile) {
  return sched_first_st(s, tile_st(s, tile));
}
__host__ __device__ __forceinline__ int sched_last_cta(const bst_gemm_sched_t& s, int tile) {
  return sched_last_st(s, tile_st(s, tile));
}

// 32-bit fast path of the slot lookup (units * grid < 2^32 for every verify shape).
__device__ __forceinline__ int tile_nslot(const bst_gemm_sched_t& s, int tile) {
  const uint32_t U = (uint32_t)s.units, G = (uint32_t)s.grid, kb = (uint32_t)s.n_kb;
  const uint32_t st = (uint32_t)tile_st(s, tile);
  const uint32_t first = (st * kb + 1) * G;
  const uint32_t last = ((st + 1) * kb) * G;
  int f = (int)((first + U - 1) / U) - 1, l = (int)((last + U - 1) / U) - 1;
  f = f < 0 ? 0 : (f >= (int)G ? (int)G - 1 : f);
  l = l < 0 ? 0 : (l >= (int)G ? (int)G - 1 : l);
  return l - f + 1;
}

// Four consecutive outputs Y[t, n0..n0+3] (n0 % 4 == 0, same 128-wide tile): one
// slot lookup, float4 loads, slots summed lowest k range first.  B > 1 issues that many
// slot loads before their adds (same sums); the default GEMM_LOAD_BATCH keeps the register
// count of the epilogues that share SMs with the next GEMM's early CTAs.
#ifndef GEMM_LOAD_BATCH
#define GEMM_LOAD_BATCH 1
#endif
template <int B = GEMM_LOAD_BATCH>
__device__ __forceinline__ float4 gemm_load4(const float* __restrict__ partial, const bst_gemm_sched_t& s, int t,
                                             int n0) {
  const int tile = n0 >> 7;
  const int nslot = tile_nslot(s, tile);
  const float4* p = reinterpret_cast<const float4*>(partial + ((int64_t)tile * s.s_max * s.bn + t) * 128 + (n0 & 127));
  const int64_t stride = (int64_t)s.bn * 32;  // in float4
  float4 acc = __ldg(p);
  for (int k0 = 1; k0 < nslot; k0 += B) {
    float4 v[B];
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (k0 + u < nslot) v[u] = __ldg(p + (k0 + u) * stride);
#pragma unroll
    for (int u = 0; u < B; ++u) {
      if (k0 + u < nslot) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
  }
  return acc;
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
