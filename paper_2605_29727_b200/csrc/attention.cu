// K3 — tree-masked verification attention over the paged KV cache.
//
// Replaces the reference's simulated mask (linearize, verify_sim.py:336-355):
// query row i may see every cached prefix slot (< c) and, inside the tree
// block, only its ancestor-or-self slots (bit j of ancestor-bitmask row i).
// The same kernel serves chunked prefill (CAUSAL: slot <= c + i) and the
// drafter's non-causal block attention (FULL).
//
// Layout: KV cache [layer][page][K|V][n_kv][64 slots][128] bf16, so one
// 64-slot page of one head is a contiguous 16 KiB tile.  A CTA owns one KV
// head and a contiguous run of pages (flash-decoding split); all GQA query
// rows of that head (group x tokens) are processed against each tile, so
// every K/V byte is read from HBM once.  Tiles arrive by TMA (two 64-column
// boxes with 128-byte swizzle) into a 3-stage mbarrier ring; QK^T and PV run
// on mma.sync bf16 (the bytes/flop ratio at s <= 64 is HBM bound); softmax is
// the online exp2 form in fp32.  Splits are merged by attn_combine_kernel.
#include <cuda_bf16.h>

#include "common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"

namespace bst {

constexpr int A_D = 128;
constexpr int A_PAGE = 64;
constexpr int A_WARPS = 8;
constexpr int A_THREADS = A_WARPS * 32;
constexpr int A_STAGES = 3;
constexpr int A_TILE_BYTES = A_PAGE * A_D * 2;      // 16 KiB per K or V tile
constexpr int A_STAGE_BYTES = 2 * A_TILE_BYTES;      // K + V
constexpr int A_ROWS_PER_CTA = A_WARPS * 16;

struct AttnArgs {
  const __nv_bfloat16* q;  // [s][n_q][128]
  int64_t q_tok_stride;
  __nv_bfloat16* out;      // [s][n_q][128]
  int64_t o_tok_stride;
  const int32_t* page_table;
  const uint32_t* anc;     // TREE: [s][mask_words]
  int mask_words;
  int n_q, n_kv, group;
  int s;                   // query tokens
  int c;                   // prefix slots visible to every row (host value)
  int keys_after_c;        // keys considered: slots [0, c + keys_after_c)
  const int32_t* state;    // optional device scalar array; c = state[c_idx]
  int c_idx;
  int n_keys;              // derived in-kernel
  int mode;                // 0 tree, 1 causal, 2 full
  int layer, n_pages_total;
  int pages_per_split, n_splits;
  int row_blocks;          // CTAs along the query-row dimension (blockIdx.z)
  float scale_log2;        // softmax scale * log2(e)
  float* ws_o;             // [split][s*n_q][128] unnormalised partial O
  float* ws_ml;            // [split][s*n_q][2] (running max (log2 domain), sum)
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// Byte address of (row, 16B-chunk q in 0..15) inside a K/V tile written by TMA as
// two [64 rows][128 B] boxes with the 128B swizzle (chunk ^= row % 8).
__device__ __forceinline__ uint32_t tile_addr(uint32_t tile, int row, int q) {
  const int half = q >> 3, cq = q & 7;
  return tile + half * (A_PAGE * 128) + row * 128 + ((cq ^ (row & 7)) << 4);
}

__device__ __forceinline__ bool visible(const AttnArgs& a, int tok, int slot, const uint32_t* mrow) {
  if (slot >= a.n_keys) return false;
  if (a.mode == 2) return true;
  if (slot < a.c) return true;
  if (a.mode == 1) return slot <= a.c + tok;
  const int j = slot - a.c;
  return (mrow[j >> 5] >> (j & 31)) & 1u;
}

__global__ void __launch_bounds__(A_THREADS, 1)
    attn_tree_kernel(const __grid_constant__ CUtensorMap tmKV, AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[A_STAGES], empty[A_STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = (sm100::smem_u32(smem_raw) + 1023) & ~1023u;
  uint8_t* smem = smem_raw + (base - sm100::smem_u32(smem_raw));

  sm100::grid_dep_launch();
  const int head = blockIdx.x;  // kv head
  const int split = blockIdx.y;
  if (a.state) a.c = a.state[a.c_idx];
  a.n_keys = a.c + a.keys_after_c;
  const int R = a.group * a.s;  // query rows of this kv head: r = t * group + g
  const int page0 = split * a.pages_per_split;
  const int n_pages_keys = (a.n_keys + A_PAGE - 1) / A_PAGE;
  const int page1 = min(page0 + a.pages_per_split, n_pages_keys);
  const int n_tiles = max(page1 - page0, 0);

  if (threadIdx.x == 0) {
    sm100::prefetch_tmap(&tmKV);
    for (int i = 0; i < A_STAGES; ++i) { sm100::mbar_init(&full[i], 1); sm100::mbar_init(&empty[i], A_WARPS); }
    sm100::fence_mbar_init();
  }
  __syncthreads();

  // producer: thread 0 issues TMA for tile i into stage i % A_STAGES
  auto issue = [&](int i) {
    const int st = i % A_STAGES;
    const int phys = a.page_table[page0 + i];
    const int64_t rowK = ((((int64_t)a.layer * a.n_pages_total + phys) * 2 + 0) * a.n_kv + head) * A_PAGE;
    const int64_t rowV = rowK + (int64_t)a.n_kv * A_PAGE;
    uint8_t* dst = smem + st * A_STAGE_BYTES;
    sm100::mbar_expect_tx(&full[st], A_STAGE_BYTES);
    sm100::tma_load_2d(dst, &tmKV, &full[st], 0, (int)rowK);
    sm100::tma_load_2d(dst + A_PAGE * 128, &tmKV, &full[st], 64, (int)rowK);
    sm100::tma_load_2d(dst + A_TILE_BYTES, &tmKV, &full[st], 0, (int)rowV);
    sm100::tma_load_2d(dst + A_TILE_BYTES + A_PAGE * 128, &tmKV, &full[st], 64, (int)rowV);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < min(n_tiles, A_STAGES); ++i) issue(i);

  // this warp's 16 query rows
  const int row0 = (blockIdx.z * A_WARPS + warp) * 16;
  const bool active = row0 < R;
  const int g = lane >> 2, cq = lane & 3;
  int tok[2], qh[2];
  bool rv[2];
  const uint32_t* mrow[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = row0 + g + 8 * h;
    rv[h] = r < R;
    const int rr = rv[h] ? r : 0;
    tok[h] = rr / a.group;
    qh[h] = head * a.group + rr % a.group;
    mrow[h] = a.mode == 0 ? a.anc + (int64_t)tok[h] * a.mask_words : nullptr;
  }
  // Q fragments: 8 k-steps of 16 dims
  uint32_t qf[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const __nv_bfloat16* qp = a.q + (int64_t)tok[h] * a.q_tok_stride + (int64_t)qh[h] * A_D + ks * 16 + 2 * cq;
      qf[ks][h] = rv[h] ? *reinterpret_cast<const uint32_t*>(qp) : 0u;
      qf[ks][h + 2] = rv[h] ? *reinterpret_cast<const uint32_t*>(qp + 8) : 0u;
    }
  }
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};

  for (int i = 0; i < n_tiles; ++i) {
    const int st = i % A_STAGES;
    sm100::mbar_wait(&full[st], (i / A_STAGES) & 1);
    const uint32_t kt = base + st * A_STAGE_BYTES;
    const uint32_t vt = kt + A_TILE_BYTES;
    const int slot0 = (page0 + i) * A_PAGE;
    if (active) {
      // S = Q K^T : 16 rows x 64 keys (8 n-tiles of 8 keys)
      float sacc[8][4];
#pragma unroll
      for (int n = 0; n < 8; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) {  // two n-tiles per ldmatrix.x4
          // matrices: (keys n2*16+0..7, chunk 2ks), (same keys, chunk 2ks+1), (keys +8.., 2ks), (+8.., 2ks+1)
          const int mi = lane >> 3, rr = lane & 7;
          const int key = n2 * 16 + (mi >> 1) * 8 + rr;
          const int q = 2 * ks + (mi & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(tile_addr(kt, key, q), b0, b1, b2, b3);
          mma_bf16(sacc[2 * n2], qf[ks], b0, b1);
          mma_bf16(sacc[2 * n2 + 1], qf[ks], b2, b3);
        }
      }
      // mask + online softmax (rows g and g+8 of this warp's block)
      float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int n = 0; n < 8; ++n) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int h = e >> 1;
          const int slot = slot0 + n * 8 + 2 * cq + (e & 1);
          float v = sacc[n][e] * a.scale_log2;
          if (!rv[h] || !visible(a, tok[h], slot, mrow[h])) v = -INFINITY;
          sacc[n][e] = v;
          mx[h] = fmaxf(mx[h], v);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
        mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
      }
      float alpha[2], mnew[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mnew[h] = fmaxf(m_run[h], mx[h]);
        alpha[h] = (mnew[h] == -INFINITY) ? 1.f : exp2f(m_run[h] - mnew[h]);
        m_run[h] = mnew[h];
      }
      float rs[2] = {0.f, 0.f};
      uint32_t pf[4][4];  // P as A fragments: 4 k-steps of 16 keys
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        float p[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int h = e >> 1;
          p[e] = (mnew[h] == -INFINITY) ? 0.f : exp2f(sacc[n][e] - mnew[h]);
          rs[h] += p[e];
        }
        const int ks = n >> 1, hi = n & 1;
        pf[ks][hi * 2 + 0] = pack_bf16(p[0], p[1]);
        pf[ks][hi * 2 + 1] = pack_bf16(p[2], p[3]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) l_run[h] = l_run[h] * alpha[h] + rs[h];
#pragma unroll
      for (int n = 0; n < 16; ++n) {
        o[n][0] *= alpha[0];
        o[n][1] *= alpha[0];
        o[n][2] *= alpha[1];
        o[n][3] *= alpha[1];
      }
      // O += P V : V tile [64 keys][128 d], B fragments via ldmatrix.trans
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        // A regs order expected: a0=(g, k 0-7), a1=(g+8, k 0-7), a2=(g, k 8-15), a3=(g+8, k 8-15)
        uint32_t af[4] = {pf[ks][0], pf[ks][1], pf[ks][2], pf[ks][3]};
#pragma unroll
        for (int dn = 0; dn < 8; ++dn) {  // 16 d-columns per ldmatrix.x4.trans -> two n-tiles
          const int mi = lane >> 3, rr = lane & 7;
          const int key = ks * 16 + (mi & 1) * 8 + rr;
          const int q = dn * 2 + (mi >> 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(tile_addr(vt, key, q), b0, b1, b2, b3);
          mma_bf16(o[2 * dn], af, b0, b1);
          mma_bf16(o[2 * dn + 1], af, b2, b3);
        }
      }
    }
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(&empty[st]);
    if (threadIdx.x == 0 && i + A_STAGES < n_tiles) {
      sm100::mbar_wait(&empty[st], (i / A_STAGES) & 1);
      issue(i + A_STAGES);
    }
    __syncwarp();
  }
  if (!active) return;
  // row sums across the 4 lanes of a row
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l_run[h] += __shfl_xor_sync(0xffffffffu, l_run[h], 1);
    l_run[h] += __shfl_xor_sync(0xffffffffu, l_run[h], 2);
  }
  if (a.n_splits == 1) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!rv[h]) continue;
      const float inv = l_run[h] > 0.f ? 1.f / l_run[h] : 0.f;
      __nv_bfloat16* op = a.out + (int64_t)tok[h] * a.o_tok_stride + (int64_t)qh[h] * A_D;
#pragma unroll
      for (int n = 0; n < 16; ++n)
        *reinterpret_cast<uint32_t*>(op + n * 8 + 2 * cq) = pack_bf16(o[n][2 * h] * inv, o[n][2 * h + 1] * inv);
    }
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!rv[h]) continue;
      const int64_t row = (int64_t)split * a.s * a.n_q + (int64_t)tok[h] * a.n_q + qh[h];
      float* op = a.ws_o + row * A_D;
#pragma unroll
      for (int n = 0; n < 16; ++n)
        *reinterpret_cast<float2*>(op + n * 8 + 2 * cq) = make_float2(o[n][2 * h], o[n][2 * h + 1]);
      if (cq == 0) {
        a.ws_ml[row * 2 + 0] = m_run[h];
        a.ws_ml[row * 2 + 1] = l_run[h];
      }
    }
  }
}

// merge flash-decoding splits: one warp per (token, q-head) row, single pass
// with online rescaling, 4 splits in flight per iteration
__global__ void attn_combine_kernel(AttnArgs a) {
  sm100::grid_dep_launch();
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int rows = a.s * a.n_q;
  if (row >= rows) return;
  float M = -INFINITY, L = 0.f;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int sp0 = 0; sp0 < a.n_splits; sp0 += 4) {
    float m[4], l[4];
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int sp = sp0 + j;
      if (sp < a.n_splits) {
        const int64_t r = (int64_t)sp * rows + row;
        m[j] = a.ws_ml[r * 2];
        l[j] = a.ws_ml[r * 2 + 1];
        v[j] = *reinterpret_cast<const float4*>(a.ws_o + r * A_D + lane * 4);
      } else {
        m[j] = -INFINITY;
        l[j] = 0.f;
        v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    float Mn = M;
#pragma unroll
    for (int j = 0; j < 4; ++j) Mn = fmaxf(Mn, m[j]);
    if (Mn == -INFINITY) continue;
    const float sc = (M == -INFINITY) ? 0.f : exp2f(M - Mn);
    L *= sc;
    acc[0] *= sc; acc[1] *= sc; acc[2] *= sc; acc[3] *= sc;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float w = (m[j] == -INFINITY) ? 0.f : exp2f(m[j] - Mn);
      L += w * l[j];
      acc[0] += w * v[j].x; acc[1] += w * v[j].y; acc[2] += w * v[j].z; acc[3] += w * v[j].w;
    }
    M = Mn;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  const int tok = row / a.n_q, qh = row % a.n_q;
  __nv_bfloat16* op = a.out + (int64_t)tok * a.o_tok_stride + (int64_t)qh * A_D + lane * 4;
  *reinterpret_cast<uint2*>(op) = make_uint2(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv));
}

}  // namespace bst

extern "C" int bst_attention(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride, const void* kv_cache,
                             int n_layers, int n_pages_total, int layer, const int32_t* page_table, int n_q, int n_kv,
                             int s, int c, int keys_after_c, int max_keys, const int32_t* state, int c_idx, int mode,
                             const uint32_t* anc, int mask_words, int n_splits, float* ws, size_t ws_bytes,
                             bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(q && out && kv_cache && page_table, "null pointer argument");
  BST_REQUIRE(n_kv >= 1 && n_q % n_kv == 0, "n_q must be a multiple of n_kv");
  BST_REQUIRE(s >= 1 && c >= 0 && keys_after_c >= 0, "bad sizes");
  BST_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0 (tree), 1 (causal) or 2 (full)");
  BST_REQUIRE(mode != 0 || (anc && mask_words * 32 >= keys_after_c), "tree mode needs the ancestor mask");
  if (max_keys < c + keys_after_c) max_keys = c + keys_after_c;
  const int group = n_q / n_kv;
  const int R = group * s;
  const int row_blocks = (R + A_ROWS_PER_CTA - 1) / A_ROWS_PER_CTA;
  const int pages = (max_keys + A_PAGE - 1) / A_PAGE;
  BST_REQUIRE(pages <= n_pages_total, "context exceeds the page table");
  if (n_splits <= 0) {
    // one wave of CTAs: per-tile work (GQA group x tokens rows against 64 keys)
    // dominates a CTA's fixed cost, so spread the pages over every SM
    int want = 148 / (n_kv * row_blocks);
    n_splits = want < 1 ? 1 : want;
  }
  if (n_splits > pages) n_splits = pages;
  const int pps = (pages + n_splits - 1) / n_splits;
  n_splits = (pages + pps - 1) / pps;
  if (n_splits > 1) {
    const size_t need = (size_t)n_splits * s * n_q * (A_D + 2) * sizeof(float);
    BST_REQUIRE(ws && ws_bytes >= need, "attention workspace too small: %zu < %zu", ws_bytes, need);
  }
  CUtensorMap tm;
  const uint64_t rows = (uint64_t)n_layers * n_pages_total * 2 * n_kv * A_PAGE;
  int rc = cached_tmap(&tm, kv_cache, rows, A_D, A_D, A_PAGE, 64);
  if (rc) return rc;
  AttnArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.q_tok_stride = q_tok_stride;
  a.out = static_cast<__nv_bfloat16*>(out);
  a.o_tok_stride = o_tok_stride;
  a.page_table = page_table;
  a.anc = anc;
  a.mask_words = mask_words;
  a.n_q = n_q;
  a.n_kv = n_kv;
  a.group = group;
  a.s = s;
  a.c = c;
  a.keys_after_c = keys_after_c;
  a.state = state;
  a.c_idx = c_idx;
  a.n_keys = c + keys_after_c;
  a.mode = mode;
  a.layer = layer;
  a.n_pages_total = n_pages_total;
  a.pages_per_split = pps;
  a.n_splits = n_splits;
  a.row_blocks = row_blocks;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)A_D);
  a.ws_o = ws;
  a.ws_ml = ws ? ws + (size_t)n_splits * s * n_q * A_D : nullptr;
  const int smem = A_STAGES * A_STAGE_BYTES + 1024;
  static bool attr = false;
  if (!attr) {
    BST_CUDA(cudaFuncSetAttribute(attn_tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  cudaStream_t st = as_stream(stream);
  attn_tree_kernel<<<dim3(n_kv, n_splits, row_blocks), A_THREADS, smem, st>>>(tm, a);
  if (n_splits > 1) {
    const int rows_total = s * n_q;
    attn_combine_kernel<<<(rows_total + 7) / 8, 256, 0, st>>>(a);
  }
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" size_t bst_attention_workspace(int n_q, int s, int n_splits) {
  return (size_t)(n_splits < 1 ? 1 : n_splits) * s * n_q * (128 + 2) * sizeof(float);
}
