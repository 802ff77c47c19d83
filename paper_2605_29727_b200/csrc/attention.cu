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
// boxes with 128-byte swizzle) into an mbarrier ring; S = QK^T and O += PV run on
// tcgen05 with TMEM accumulators; softmax is the online exp2 form in fp32.
// Splits merge in-kernel (last-arriving CTA) or in attn_combine_kernel.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdlib.h>

#include "common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"

namespace bst {

BST_BND_TRACE_DEF

constexpr int A_D = 128;
constexpr int A_PAGE = 64;
constexpr int A_WARPS = 8;
constexpr int A_THREADS = A_WARPS * 32;
constexpr int A_STAGES = 3;
constexpr int A_TILE_BYTES = A_PAGE * A_D * 2;      // 16 KiB per K or V tile
constexpr int A_STAGE_BYTES = 2 * A_TILE_BYTES;      // K + V
constexpr int A_ROWS_PER_CTA = A_WARPS * 16;
constexpr size_t A_WS_CNT_BYTES = 4096;  // workspace head: split-arrival counters (zero-initialised once)

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
  unsigned long long* cnt; // [row_blocks][n_kv] split barrier words (generation | arrivals)
  int merge;               // 1: splits merged in-kernel (one-wave grid), 0: attn_combine_kernel
  // batched requests (blockIdx.z = req * row_blocks + rb): request req owns query rows
  // [req * s, req * s + s), page-table entries [req * req_pages, ...), state words
  // [req * req_state, ...) and ws partials [req][split][s * n_q]
  int n_req, req_pages, req_state;
  // ragged batch (nullable): request req's query rows are q/out rows [row_off[req],
  // row_off[req] + row_cnt[req]) of a packed layout; masks and partials keep the
  // uniform [req][s] stride (s = the per-request row capacity)
  const int32_t* row_off;
  const int32_t* row_cnt;
  int rows_per_block;      // key-major kernel: query rows per CTA (row blocks balanced over R)
  bst_prefetch_t pf;       // next-GEMM weights to pull into L2 while we run
  int seq;                 // boundary-trace launch number (BST_TRACE builds)
};

// First packed q/out row of request req, and its query-row count (ragged batches).
__device__ __forceinline__ int64_t req_row0(const AttnArgs& a, int req) {
  return a.row_off ? (int64_t)a.row_off[req] : (int64_t)req * a.s;
}
__device__ __forceinline__ int req_rows(const AttnArgs& a, int req) { return a.row_cnt ? a.row_cnt[req] : a.s; }


__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t pack_f16(float a, float b) {
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float2 unpack_f16(uint32_t u) {
  return __half22float2(*reinterpret_cast<__half2*>(&u));
}


// 64-bit visibility of keys slot0..slot0+63 for query row `tok`:
// prefix (< c) always, tree/causal part per mode, nothing at or beyond n_keys.
__device__ __forceinline__ uint64_t bits_from(int lo, int hi) {  // bits [lo, hi] (clamped to 0..63)
  lo = lo < 0 ? 0 : lo;
  hi = hi > 63 ? 63 : hi;
  if (hi < lo) return 0ull;
  const uint64_t upto = hi == 63 ? ~0ull : ((1ull << (hi + 1)) - 1);
  return upto & ~((1ull << lo) - 1);
}
__device__ __forceinline__ uint64_t mask_get64(const uint32_t* m, int words, int start) {
  const int w = start >> 5, sh = start & 31;
  const uint64_t w0 = w < words ? m[w] : 0u, w1 = w + 1 < words ? m[w + 1] : 0u, w2 = w + 2 < words ? m[w + 2] : 0u;
  const uint64_t lo = w0 | (w1 << 32);
  return sh ? (lo >> sh) | (w2 << (64 - sh)) : lo;
}
__device__ __forceinline__ uint64_t row_vis64(int mode, int c, int n_keys, int tok, int slot0, const uint32_t* mrow,
                                              int words) {
  const uint64_t lim = bits_from(0, n_keys - slot0 - 1);
  if (mode == 2) return lim;
  const int np = c - slot0;  // prefix keys in this tile
  const uint64_t pre = bits_from(0, np - 1);
  if (np >= 64) return pre & lim;
  const int j0 = slot0 - c;  // tree index of key 0 (< 0: the tile starts in the prefix)
  uint64_t tail;
  if (mode == 1) {
    tail = bits_from(-j0, tok - j0);
  } else if (j0 >= 0) {
    tail = mask_get64(mrow, words, j0);
  } else {
    tail = mask_get64(mrow, words, 0) << (-j0);
  }
  return (pre | tail) & lim;
}

__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2, ex2(-inf) = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (x <= 0; -inf -> 0): round-to-nearest split by the 1.5 * 2^23
// trick, degree-3 fit of 2^f on [-1/2, 1/2] (max rel. error 7.6e-5, far below the bf16
// rounding P goes through), exponent added as integer bits.  Takes part of the
// softmax's exponentials off the MUFU pipe.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.05517030f, 0.24260803f);
  p = fmaf(f, p, 0.69326091f);
  p = fmaf(f, p, 0.99992830f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

__device__ long long* g_attn_trace = nullptr;  // debug: [32 tiles][8] globaltimer stamps of CTA (0,0,0)
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ int g_attn_trace_y = 0;               // debug: which split's CTA (0, y, 0) is traced
__device__ int g_kt_ablate = 0;                  // debug (profiling only): skip key-major softmax phases
#ifdef BST_TRACE  // phase tracing (scripts/attn_trace.py); compiled out by default
#define TRACE(i, k)                                                                                   \
  do {                                                                                                \
    if (g_attn_trace && blockIdx.x == 0 && blockIdx.y == g_attn_trace_y && blockIdx.z == 0 && (i) < 32) \
      g_attn_trace[(i) * 8 + (k)] = gtimer();                                                         \
  } while (0)
#define TRACE_MAX(k)                                                                                  \
  do {                                                                                                \
    if (g_attn_trace) atomicMax(reinterpret_cast<unsigned long long*>(g_attn_trace) + 29 * 8 + (k),   \
                                (unsigned long long)gtimer());                                        \
  } while (0)
#define TRACE_MIN(k)                                                                                  \
  do {                                                                                                \
    if (g_attn_trace) atomicMin(reinterpret_cast<unsigned long long*>(g_attn_trace) + 28 * 8 + (k),   \
                                (unsigned long long)gtimer());                                        \
  } while (0)
#else
#define TRACE_MIN(k) \
  do {               \
  } while (0)
#define TRACE(i, k) \
  do {              \
  } while (0)
#define TRACE_MAX(k) \
  do {               \
  } while (0)
#endif

__device__ __forceinline__ unsigned long long ld_acquire_gpu64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long atom_add_acq_rel_gpu(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ long long gtimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// In-kernel flash-decoding merge (a.merge == 1).  The NT epilogue threads of a CTA
// have staged its unnormalised partial O in shared memory, `stg` = [128 rows][128]
// fp32 with 16-byte chunks swizzled by row % 8, and written (m, l) to ws_ml.
// 1. warp-per-row coalesced copy of the partial rows to ws_o (L2-resident);
// 2. arrive on the (head, row-block) counter and wait until every split has arrived:
//    the grid is one wave (host checks grid <= #SMs at one CTA per SM) and every CTA
//    has started before a dependent kernel can launch (griddepcontrol at entry), so
//    all splits are co-resident;
// 3. merge rows [split * per, split * per + per) of the row block across splits
//    (fixed split order: deterministic) and store bf16;
// 4. second arrival; the last one resets the counter to zero for the next launch.
// STAGED = false: the caller has already written its partial rows to ws_o / ws_ml.
template <int NT, bool STAGED = true>
__device__ void split_merge(const AttnArgs& a, const float* stg, int head, int split, int req, int rb, int row0, int Rb,
                            int t) {
  constexpr int NW = NT / 32;
  const int warp = t >> 5, lane = t & 31;
  const int64_t rows_all = (int64_t)a.s * a.n_q;
  for (int r = warp; STAGED && r < Rb; r += NW) {
    const int rg = row0 + r, tok = rg / a.group, qh = head * a.group + rg % a.group;
    const int64_t gr = ((int64_t)req * a.n_splits + split) * rows_all + (int64_t)tok * a.n_q + qh;
    const float4 v = *reinterpret_cast<const float4*>(stg + r * A_D + ((lane ^ (r & 7)) << 2));
    __stcg(reinterpret_cast<float4*>(a.ws_o + gr * A_D) + lane, v);
  }
  // generation barrier over the splits of this (head, row block): the counter word is
  // (generation << 32 | arrivals); the last arrival clears the arrivals and bumps the
  // generation in one release RMW, the others spin (acquire) until the generation moves.
  named_bar_sync(1, NT);
  if (t == 0) TRACE(30, 2);
  unsigned long long* cnt = a.cnt + ((int64_t)req * a.row_blocks + rb) * a.n_kv + head;
  if (t == 0) {
    const unsigned long long old = atom_add_acq_rel_gpu(cnt, 1ull);
    TRACE_MAX(3);
    if ((unsigned)(old & 0xffffffffu) == (unsigned)a.n_splits - 1u) {
      red_add_release_gpu(cnt, (1ull << 32) - (unsigned long long)a.n_splits);
    } else {
      const unsigned gen = (unsigned)(old >> 32);
      const long long t0 = gtimer_ns();
      for (uint32_t it = 1; (unsigned)(ld_acquire_gpu64(cnt) >> 32) == gen; ++it) {
        if ((it & 1023u) == 0 && gtimer_ns() - t0 > 2000000000ll) __trap();  // a split never arrived: fail, do not hang
      }
    }
  }
  if (t == 0) TRACE_MAX(4);
  if (t == 0) TRACE(30, 3);
  named_bar_sync(1, NT);
  // thread item = (row, DI-dim slice); the loads of up to 20 splits are issued at once
  // (DI = 8 for the 192-thread kernel, 4 for the 384-thread one: register budget)
  constexpr int MS = 20, DI = NT == 128 ? 8 : 4, IPR = A_D / DI;
  const int per = (Rb + a.n_splits - 1) / a.n_splits;
  const int r0 = split * per, r1 = min(r0 + per, Rb);
  for (int it = t; it < (r1 - r0) * IPR; it += NT) {
    const int r = r0 + it / IPR, d0 = (it % IPR) * DI;
    const int rg = row0 + r, tok = rg / a.group, qh = head * a.group + rg % a.group;
    const int64_t base = (int64_t)req * a.n_splits * rows_all + (int64_t)tok * a.n_q + qh;
    float M = -INFINITY, L = 0.f, acc[DI];
#pragma unroll
    for (int e = 0; e < DI; ++e) acc[e] = 0.f;
    for (int j0 = 0; j0 < a.n_splits; j0 += MS) {
      float2 ml[MS];
      float4 va[MS][DI / 4];
#pragma unroll
      for (int u = 0; u < MS; ++u) {
        if (j0 + u < a.n_splits) {
          const int64_t gr = (j0 + u) * rows_all + base;
          ml[u] = __ldcg(reinterpret_cast<const float2*>(a.ws_ml + gr * 2));
#pragma unroll
          for (int h = 0; h < DI / 4; ++h) va[u][h] = __ldcg(reinterpret_cast<const float4*>(a.ws_o + gr * A_D + d0) + h);
        } else {
          ml[u] = make_float2(-INFINITY, 0.f);
#pragma unroll
          for (int h = 0; h < DI / 4; ++h) va[u][h] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      float Mn = M;
#pragma unroll
      for (int u = 0; u < MS; ++u) Mn = fmaxf(Mn, ml[u].x);
      if (Mn == -INFINITY) continue;
      const float sc = M == -INFINITY ? 0.f : ex2(M - Mn);
      L *= sc;
#pragma unroll
      for (int e = 0; e < DI; ++e) acc[e] *= sc;
#pragma unroll
      for (int u = 0; u < MS; ++u) {
        const float w = ml[u].x == -INFINITY ? 0.f : ex2(ml[u].x - Mn);
        L += w * ml[u].y;
#pragma unroll
        for (int h = 0; h < DI / 4; ++h) {
          acc[4 * h + 0] += w * va[u][h].x;
          acc[4 * h + 1] += w * va[u][h].y;
          acc[4 * h + 2] += w * va[u][h].z;
          acc[4 * h + 3] += w * va[u][h].w;
        }
      }
      M = Mn;
    }
    if (t == 0) TRACE(30, 4);
    const float inv = L > 0.f ? 1.f / L : 0.f;
    __nv_bfloat16* op = a.out + (req_row0(a, req) + tok) * a.o_tok_stride + (int64_t)qh * A_D + d0;
    if constexpr (DI == 8) {
      *reinterpret_cast<uint4*>(op) = make_uint4(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv),
                                                 pack_bf16(acc[4] * inv, acc[5] * inv), pack_bf16(acc[6] * inv, acc[7] * inv));
    } else {
      *reinterpret_cast<uint2*>(op) = make_uint2(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv));
    }
  }
}

// Global split merge of the key-major kernel.  Partials live in a head-major, dim-chunk
// major layout so both the writers (one query row per thread) and the readers are
// coalesced: ws_o float4 index ((req, split, head) * 32 + d4) * R + row, ws_ml float2
// index (req, split, head) * R + row (row = the GQA row index inside the head).  The
// arrival protocol is split_merge's generation counter.
__device__ __forceinline__ int64_t kt_ws_base(const AttnArgs& a, int req, int split, int head) {
  return ((int64_t)req * a.n_splits + split) * a.n_kv + head;
}
__device__ void kt_global_merge(const AttnArgs& a, int head, int split, int req, int rb, int row0, int Rb, int t) {
  const int R = a.group * a.s;
  named_bar_sync(1, 256);
  unsigned long long* cnt = a.cnt + ((int64_t)req * a.row_blocks + rb) * a.n_kv + head;
  if (t == 0) {
    const unsigned long long old = atom_add_acq_rel_gpu(cnt, 1ull);
    TRACE_MAX(3);
    if ((unsigned)(old & 0xffffffffu) == (unsigned)a.n_splits - 1u) {
      red_add_release_gpu(cnt, (1ull << 32) - (unsigned long long)a.n_splits);
    } else {
      const unsigned gen = (unsigned)(old >> 32);
      const long long t0 = gtimer_ns();
      for (uint32_t it = 1; (unsigned)(ld_acquire_gpu64(cnt) >> 32) == gen; ++it) {
        if ((it & 1023u) == 0 && gtimer_ns() - t0 > 2000000000ll) __trap();  // a split never arrived
      }
    }
  }
  if (t == 0) TRACE_MAX(4);
  named_bar_sync(1, 256);
  const int ns = a.n_splits;
  const int per = (Rb + ns - 1) / ns, r0 = split * per, nr = min(r0 + per, Rb) - r0;
  const float2* ml_all = reinterpret_cast<const float2*>(a.ws_ml);
  const float4* o_all = reinterpret_cast<const float4*>(a.ws_o);
  // two lanes per (row, 16-byte chunk) item: lane h merges the splits h, h + 2, ... (one
  // batch of loads for up to 20 splits), then the pair combines over a shuffle; fixed
  // assignment and combine order: deterministic
  constexpr int MH = 10;
  for (int it2 = t; it2 < nr * 64; it2 += 256) {
    const unsigned am = __activemask();  // pairs (2i, 2i+1) are always active together
    const int it = it2 >> 1, h = it2 & 1;
    const int rr = row0 + r0 + it % nr, d4 = it / nr;  // lanes walk rows: coalesced
    float M = -INFINITY, L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j0 = h; j0 < ns; j0 += 2 * MH) {
      float2 ml[MH];
      float4 v[MH];
#pragma unroll
      for (int u = 0; u < MH; ++u) {
        const int q = j0 + 2 * u;
        if (q < ns) {
          const int64_t b = kt_ws_base(a, req, q, head);
          ml[u] = __ldcg(ml_all + b * R + rr);
          v[u] = __ldcg(o_all + (b * 32 + d4) * R + rr);
        } else {
          ml[u] = make_float2(-INFINITY, 0.f);
          v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      float Mn = M;
#pragma unroll
      for (int u = 0; u < MH; ++u) Mn = fmaxf(Mn, ml[u].x);
      if (Mn == -INFINITY) continue;
      const float sc = M == -INFINITY ? 0.f : ex2(M - Mn);
      L *= sc;
      acc.x *= sc; acc.y *= sc; acc.z *= sc; acc.w *= sc;
#pragma unroll
      for (int u = 0; u < MH; ++u) {
        const float w = ml[u].x == -INFINITY ? 0.f : ex2(ml[u].x - Mn);
        L += w * ml[u].y;
        acc.x += w * v[u].x; acc.y += w * v[u].y; acc.z += w * v[u].z; acc.w += w * v[u].w;
      }
      M = Mn;
    }
    // combine the pair: half 0's terms first, then half 1's
    const float Mo = __shfl_xor_sync(am, M, 1), Lo = __shfl_xor_sync(am, L, 1);
    const float4 ao = make_float4(__shfl_xor_sync(am, acc.x, 1), __shfl_xor_sync(am, acc.y, 1),
                                  __shfl_xor_sync(am, acc.z, 1), __shfl_xor_sync(am, acc.w, 1));
    if (h == 0) {
      const float Mt = fmaxf(M, Mo);
      const float w0 = M == -INFINITY ? 0.f : ex2(M - Mt), w1 = Mo == -INFINITY ? 0.f : ex2(Mo - Mt);
      const float Lt = w0 * L + w1 * Lo;
      const float4 at = make_float4(w0 * acc.x + w1 * ao.x, w0 * acc.y + w1 * ao.y, w0 * acc.z + w1 * ao.z,
                                    w0 * acc.w + w1 * ao.w);
      const float inv = Lt > 0.f ? 1.f / Lt : 0.f;
      const int tok = rr / a.group, qh = head * a.group + rr % a.group;
      __nv_bfloat16* op = a.out + (req_row0(a, req) + tok) * a.o_tok_stride + (int64_t)qh * A_D + 4 * d4;
      *reinterpret_cast<uint2*>(op) = make_uint2(pack_bf16(at.x * inv, at.y * inv), pack_bf16(at.z * inv, at.w * inv));
    }
  }
}

// Slots the previous kernel cannot be writing, so their pages may be loaded before
// griddepcontrol.wait: the committed prefix below c, except that in FULL mode (the
// drafter block) the keys_after_c context slots just below c are written by the
// preceding qkv_rope as well (newly committed tokens' context K/V).
__device__ __forceinline__ int pdl_safe_slots(const AttnArgs& a, int c_ctx) {
  return max(c_ctx - (a.mode == 2 ? a.keys_after_c : 0), 0);
}

// Pages [page0, page0 + n_tiles) of this split: the live pages (those holding keys
// < n_keys, read from device state at run time) are balanced over the splits, so a
// graph captured for the capacity still gives every split the same share.
__device__ __forceinline__ void split_pages(const AttnArgs& a, int n_keys, int split, int& page0, int& n_tiles) {
  const int live = (n_keys + A_PAGE - 1) / A_PAGE;
  page0 = split * live / a.n_splits;
  n_tiles = (split + 1) * live / a.n_splits - page0;
}

// ---- distributed shared memory (thread-block clusters)
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float ld_dsmem_f1(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 ld_dsmem_u4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 ld_dsmem_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Cluster split merge (a.merge == 2): the n_splits (<= 16) CTAs of one (head, row block)
// form a thread-block cluster (rank = split).  Each has staged its partial rows
// normalised by its own row sum l, as fp16 [128][128] (16-byte chunks swizzled by
// row % 8; half the DSMEM requests of fp32 partials — the merge is bound by DSMEM
// requests), at shared address `stg`, and (m, l) per row in `ml`.  A normalised row is a
// convex combination of V rows, so fp16 holds it whenever |V| < 65504 (bf16 LLM value
// activations are orders of magnitude below; bf16 staging measured the same speed but
// its 8-bit mantissa flips a near-tie argmax of the tiny test model, and a per-half
// scale cost 0.6 us per launch).  After a cluster
// barrier CTA `split` merges rows [split * per, split * per + per) from every rank over
// DSMEM in rank order, weighting rank q by 2^(m_q - M) l_q (deterministic), and stores
// bf16; a second barrier
// keeps the staging alive until every remote read is done.  This replaces the L2 merge's
// partial stores, arrival atomic, poll and partial loads (three dependent gpu-scope round
// trips, ~3 us per launch at c = 2K) by two cluster barriers and DSMEM loads.
constexpr int T2_CLUSTER_MAX = 16;
template <int NT>
__device__ void cluster_split_merge(const AttnArgs& a, const float2* ml, uint32_t stg, int head,
                                    int split, int req, int rb, int R) {
  cluster_sync_all();
  if (threadIdx.x == 64) TRACE(30, 5);
  if (threadIdx.x == 64) TRACE_MAX(3);
  if (threadIdx.x >= 64 && threadIdx.x < 64 + NT) {
    const int t = threadIdx.x - 64, ns = a.n_splits;
    const int Rb = min(128, R - rb * 128);
    const int per = (Rb + ns - 1) / ns, r0 = split * per, r1 = min(r0 + per, Rb);
    const uint32_t ml_u = sm100::smem_u32(ml);
    for (int it = t; it < (r1 - r0) * 16; it += NT) {
      const int r = r0 + (it >> 4), cq = it & 15;  // dims [8 cq, 8 cq + 8) of row r
      const uint32_t off = (uint32_t)(r * 256 + ((cq ^ (r & 7)) << 4));
      float m[T2_CLUSTER_MAX], l[T2_CLUSTER_MAX];
      uint4 v[T2_CLUSTER_MAX];
#pragma unroll
      for (int q = 0; q < T2_CLUSTER_MAX; ++q) {
        if (q < ns) {
          const float2 v2 = ld_dsmem_f2(mapa_shared(ml_u + r * 8, q));  // (m, l) in one request
          m[q] = v2.x;
          l[q] = v2.y;
          v[q] = ld_dsmem_u4(mapa_shared(stg + off, q));
        }
      }
      float M = -INFINITY;
#pragma unroll
      for (int q = 0; q < T2_CLUSTER_MAX; ++q)
        if (q < ns) M = fmaxf(M, m[q]);
      float Lsum = 0.f;
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
      for (int q = 0; q < T2_CLUSTER_MAX; ++q) {
        if (q < ns && m[q] != -INFINITY) {
          const float w = ex2(m[q] - M) * l[q];  // the rank's softmax mass (its rows were staged normalised)
          const float2 p0 = unpack_f16(v[q].x), p1 = unpack_f16(v[q].y), p2 = unpack_f16(v[q].z), p3 = unpack_f16(v[q].w);
          Lsum += w;
          acc[0] += w * p0.x; acc[1] += w * p0.y; acc[2] += w * p1.x; acc[3] += w * p1.y;
          acc[4] += w * p2.x; acc[5] += w * p2.y; acc[6] += w * p3.x; acc[7] += w * p3.y;
        }
      }
      const float inv = Lsum > 0.f ? 1.f / Lsum : 0.f;
      const int rg = rb * 128 + r, tok = rg / a.group, qh = head * a.group + rg % a.group;
      __nv_bfloat16* op = a.out + (req_row0(a, req) + tok) * a.o_tok_stride + (int64_t)qh * A_D + 8 * cq;
      *reinterpret_cast<uint4*>(op) = make_uint4(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv),
                                                 pack_bf16(acc[4] * inv, acc[5] * inv), pack_bf16(acc[6] * inv, acc[7] * inv));
    }
  }
  if (threadIdx.x == 64) TRACE(30, 6);
  cluster_sync_all();
}

// ===========================================================================
// tcgen05 variant (default): S = Q K^T and O += P V on the 5th-gen tensor cores.
// One CTA = one KV head x one KV split x up to 128 query rows (UMMA M = 128).
// warp 0: TMA producer (K/V pages, 4-stage ring); warp 1: TMEM owner + single
// issuing thread; warps 2-5: one thread per query row — Q staging, tcgen05.ld of
// S, mask + online softmax (lazy O rescale when the row max grows by > 2^8),
// bf16 P -> tensor memory (tcgen05.st), epilogue.  TMEM: S double buffer (2 x 64
// columns), O (128 columns), P double buffer (2 x 32 columns, 2 bf16 per column).
// O += P V reads P from TMEM as the A operand (TS-mode tcgen05.mma: no shared-memory
// P, no async-proxy fence per tile) and V from shared memory as an MN-major operand.
// ===========================================================================
constexpr int T_THREADS = 192;
constexpr int T_STAGES = 4;
constexpr int T_Q_BYTES = 128 * A_D * 2;   // 32 KiB: two [128 rows][64] SW128 halves
constexpr int T_PCOL = 256;  // TMEM: S 0-127 (double buffer), O 128-255, bf16 P 256-319 (double buffer, 32 each)
constexpr float T_RESCALE = 8.f;            // log2 units

__global__ void __launch_bounds__(T_THREADS, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap tmKV, AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[T_STAGES], empty[T_STAGES], s_full[2], s_free[2], p_full, o_done[2], q_ready;
  __shared__ uint32_t tmem_sh;
  __shared__ float2 cml[128];  // cluster merge: (m, l) per row
  sm100::grid_dep_launch();
  if (threadIdx.x == 0) TRACE(31, 0);
  if (threadIdx.x == 0) BND(a.seq, 0);
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) BND_KIND(a.seq, 5);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = (sm100::smem_u32(smem_raw) + 1023) & ~1023u;
  uint8_t* smem = smem_raw + (base - sm100::smem_u32(smem_raw));
  const uint32_t sQ = base, sKV = base + T_Q_BYTES;
  uint8_t* gQ = smem;
  uint8_t* gKV = smem + T_Q_BYTES;

  const int head = blockIdx.x, split = blockIdx.y, req = blockIdx.z / a.row_blocks, rb = blockIdx.z % a.row_blocks;
  const int c_ctx = a.state ? a.state[req * a.req_state + a.c_idx] : a.c;
  const int n_keys = c_ctx + a.keys_after_c;
  int R = a.group * a.s;
  if (a.row_cnt) {  // ragged batch: the row counts come from an earlier kernel of the graph
    sm100::grid_dep_wait();
    R = a.group * req_rows(a, req);
    if (rb * 128 >= R) return;  // every split of this (head, row block) exits: no barrier waits on it
  }
  int page0, n_tiles;
  split_pages(a, n_keys, split, page0, n_tiles);

  if (threadIdx.x == 0) {
    sm100::prefetch_tmap(&tmKV);
    for (int i = 0; i < T_STAGES; ++i) { sm100::mbar_init(&full[i], 1); sm100::mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { sm100::mbar_init(&s_full[i], 1); sm100::mbar_init(&s_free[i], 4); }
    sm100::mbar_init(&p_full, 4);
    sm100::mbar_init(&o_done[0], 1);
    sm100::mbar_init(&o_done[1], 1);
    sm100::mbar_init(&q_ready, 4);
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc(&tmem_sh, 512);  // S, O and P: 320 columns
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  if (threadIdx.x == 0) TRACE(31, 1);

  if (warp == 0) {
    if (lane == 0) {
      issue_prefetch(a.pf, (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x,
                     gridDim.x * gridDim.y * gridDim.z);
      // PDL: pages entirely below c hold committed K/V the previous kernel does not
      // touch; the page holding slot c onwards is written by qkv_rope right before us.
      const int safe_tiles = max(min(pdl_safe_slots(a, c_ctx) / A_PAGE - page0, n_tiles), 0);
      bool waited = false;
      for (int i = 0; i < n_tiles; ++i) {
        const int st = i % T_STAGES;
        if (i >= T_STAGES) sm100::mbar_wait(&empty[st], ((i / T_STAGES) & 1) ^ 1);
        if (!waited && (i >= safe_tiles || i >= T_STAGES)) {
          sm100::grid_dep_wait();
          waited = true;
        }
        const int phys = a.page_table[(int64_t)req * a.req_pages + page0 + i];
        const int64_t rowK = ((((int64_t)a.layer * a.n_pages_total + phys) * 2 + 0) * a.n_kv + head) * A_PAGE;
        const int64_t rowV = rowK + (int64_t)a.n_kv * A_PAGE;
        uint8_t* dst = gKV + st * A_STAGE_BYTES;
        sm100::mbar_expect_tx(&full[st], A_STAGE_BYTES);
        sm100::tma_load_2d(dst, &tmKV, &full[st], 0, (int)rowK);
        sm100::tma_load_2d(dst + A_PAGE * 128, &tmKV, &full[st], 64, (int)rowK);
        sm100::tma_load_2d(dst + A_TILE_BYTES, &tmKV, &full[st], 0, (int)rowV);
        sm100::tma_load_2d(dst + A_TILE_BYTES + A_PAGE * 128, &tmKV, &full[st], 64, (int)rowV);
        TRACE(i, 0);
      }
    }
  } else if (warp == 1) {
    const uint32_t idS = sm100::idesc_bf16(128, A_PAGE);
    const uint32_t idO = sm100::idesc_bf16_bmn(128, A_D);
    sm100::mbar_wait(&q_ready, 0);
    for (int i = 0; i <= n_tiles; ++i) {
      if (i < n_tiles) {
        const int st = i % T_STAGES, b = i & 1;
        sm100::mbar_wait(&full[st], (i / T_STAGES) & 1);
        if (lane == 0) TRACE(i, 1);
        if (i >= 2) sm100::mbar_wait(&s_free[b], ((i - 2) >> 1) & 1);
        sm100::tc_fence_after();
        if (sm100::elect_one()) {
          const uint32_t kb = sKV + st * A_STAGE_BYTES;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint64_t ad = sm100::desc_k_sw128(sQ + (j >> 2) * (128 * 128) + (j & 3) * 32);
            const uint64_t bd = sm100::desc_k_sw128(kb + (j >> 2) * (A_PAGE * 128) + (j & 3) * 32);
            sm100::umma_f16(tmem + b * A_PAGE, ad, bd, idS, j > 0 ? 1u : 0u);
          }
          sm100::umma_commit(&s_full[b]);
        }
        __syncwarp();
      }
      if (i >= 1) {
        const int j = i - 1, stj = j % T_STAGES;
        sm100::mbar_wait(&p_full, j & 1);
        if (lane == 0) TRACE(j, 2);
        sm100::tc_fence_after();
        if (sm100::elect_one()) {
          const uint32_t vb = sKV + stj * A_STAGE_BYTES + A_TILE_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t bd = sm100::desc_mn_sw128(vb + kk * 2048, A_PAGE * 128);
            sm100::umma_f16_ts(tmem + 128, tmem + T_PCOL + 32 * (j & 1) + 8 * kk, bd, idO, (j > 0 || kk > 0) ? 1u : 0u);
          }
          sm100::umma_commit(&o_done[j & 1]);
          sm100::umma_commit(&empty[stj]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- one thread per query row
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const int rg = rb * 128 + row;
    const bool valid = rg < R;
    const int rr = valid ? rg : 0;
    const int tok = rr / a.group;
    const int qh = head * a.group + rr % a.group;
    const uint32_t* mrow = a.mode == 0 ? a.anc + ((int64_t)req * a.s + tok) * a.mask_words : nullptr;
    const int mode = a.mode, mwords = a.mask_words;
    const float scale = a.scale_log2;
    sm100::grid_dep_wait();  // q is produced by the previous kernel (PDL)
    if (threadIdx.x == 64) TRACE(31, 2);
    if (threadIdx.x == 64) BND(a.seq, 2);
    if (threadIdx.x == 64) BND(a.seq, 3);
    if (threadIdx.x == 64) TRACE_MAX(0);
    {  // stage Q row (256 B) into the swizzled K-major tile
      const int4* src = reinterpret_cast<const int4*>(a.q + (req_row0(a, req) + tok) * a.q_tok_stride + (int64_t)qh * A_D);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int4 v = valid ? src[q] : make_int4(0, 0, 0, 0);
        *reinterpret_cast<int4*>(gQ + (q >> 3) * (128 * 128) + row * 128 + (((q & 7) ^ (row & 7)) << 4)) = v;
      }
    }
    sm100::fence_async_shared();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(&q_ready);
    if (threadIdx.x == 64) TRACE(31, 3);
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    float m_run = -INFINITY, l_run = 0.f;
    for (int i = 0; i < n_tiles; ++i) {
      const int b = i & 1;
      sm100::mbar_wait(&s_full[b], (i >> 1) & 1);
      if (threadIdx.x == 64) TRACE(i, 3);
      sm100::tc_fence_after();
      float sv[64];
      {  // the tile's 64 score columns: four loads in flight, one wait
        uint32_t r[4][16];
#pragma unroll
        for (int k = 0; k < 4; ++k) sm100::tmem_ld16_nw(lane_base + b * A_PAGE + 16 * k, r[k]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int e = 0; e < 16; ++e) sv[16 * k + e] = __uint_as_float(r[k][e]);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&s_free[b]);
      if (threadIdx.x == 64) TRACE(i, 7);
      const int slot0 = (page0 + i) * A_PAGE;
      const uint64_t vis = valid ? row_vis64(mode, c_ctx, n_keys, tok, slot0, mrow, mwords) : 0ull;
      float mx8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
      // max over the raw scores (scale > 0 commutes with max); the scale is folded into
      // the exponent's FMA below (as in tc2)
      if (__all_sync(0xffffffffu, vis == ~0ull)) {  // prefix tile: no masking
#pragma unroll
        for (int k = 0; k < 64; ++k) mx8[k & 7] = fmaxf(mx8[k & 7], sv[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 64; ++k) {
          const float v = ((vis >> k) & 1ull) ? sv[k] : -INFINITY;
          sv[k] = v;
          mx8[k & 7] = fmaxf(mx8[k & 7], v);
        }
      }
      const float mt = scale * fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                     fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float m_new = fmaxf(m_run, mt);
      const bool rescale = (m_run == -INFINITY) ? (m_new != -INFINITY) : (m_new > m_run + T_RESCALE);
      const float m_ref = rescale ? m_new : m_run;
      const float alpha = (rescale && m_run != -INFINITY) ? ex2(m_run - m_ref) : (rescale ? 0.f : 1.f);
      const float nsub = m_ref == -INFINITY ? 0.f : -m_ref;  // all-masked row: ex2(-inf) = 0
      float rs8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) rs8[k] = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int k = 0; k < 64; k += 2) {
        const float p0 = ex2(fmaf(sv[k], scale, nsub));
        const float p1 = ex2(fmaf(sv[k + 1], scale, nsub));
        rs8[(k >> 1) & 7] += p0 + p1;
        pk[k >> 1] = pack_bf16(p0, p1);
      }
      const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
      if (threadIdx.x == 64) TRACE(i, 4);
      // P buffer i&1 was last read by PV(i-2); O only needs PV(i-1) when it is rescaled
      const bool need_o = __any_sync(0xffffffffu, rescale && i >= 1);
      if (need_o) sm100::mbar_wait(&o_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
      else if (i >= 2) sm100::mbar_wait(&o_done[i & 1], ((i - 2) >> 1) & 1);
      if (threadIdx.x == 64) TRACE(i, 5);
      sm100::tc_fence_after();
      // tcgen05.ld/st are warp-collective: rescale if any row of the warp needs it
      if (need_o) {
        const float f = (rescale && i >= 1) ? alpha : 1.f;
#pragma unroll 1
        for (int cc = 0; cc < 8; ++cc) {
          float ov[16];
          sm100::tmem_ld16(lane_base + 128 + 16 * cc, ov);
#pragma unroll
          for (int e = 0; e < 16; ++e) ov[e] *= f;
          sm100::tmem_st16(lane_base + 128 + 16 * cc, ov);
        }
        sm100::tmem_st_wait();
      }
      l_run = rescale ? l_run * alpha + rs : l_run + rs;
      m_run = m_ref;
      // bf16 P into tensor memory (A operand of the PV MMA), buffer i & 1
      sm100::tmem_st32u(lane_base + T_PCOL + 32 * (i & 1), pk);
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&p_full);
      if (threadIdx.x == 64) TRACE(i, 6);
    }
    // ---------------- epilogue
    float o[128];
    if (n_tiles > 0) {
      sm100::mbar_wait(&o_done[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1);
      if (threadIdx.x == 64) TRACE(31, 4);
      sm100::tc_fence_after();
      {
        uint32_t r[8][16];
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) sm100::tmem_ld16_nw(lane_base + 128 + 16 * cc, r[cc]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
#pragma unroll
          for (int e = 0; e < 16; ++e) o[16 * cc + e] = __uint_as_float(r[cc][e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 128; ++e) o[e] = 0.f;
    }
    if (a.n_splits > 1 && a.merge == 2) {
      // normalised rows as fp16 (the merge re-weights them by each rank's mass m, l): half
      // the DSMEM bytes of fp32 partials; the K/V ring is idle once the last PV is done
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        *reinterpret_cast<uint4*>(gKV + row * 256 + ((q ^ (row & 7)) << 4)) =
            make_uint4(pack_f16(o[8 * q] * inv, o[8 * q + 1] * inv), pack_f16(o[8 * q + 2] * inv, o[8 * q + 3] * inv),
                       pack_f16(o[8 * q + 4] * inv, o[8 * q + 5] * inv), pack_f16(o[8 * q + 6] * inv, o[8 * q + 7] * inv));
      cml[row] = make_float2(m_run, l_run);
    } else if (a.n_splits > 1 && a.merge) {
      float* stg = reinterpret_cast<float*>(gKV);  // the K/V ring is idle once the last PV is done
#pragma unroll
      for (int q = 0; q < 32; ++q)
        *reinterpret_cast<float4*>(stg + row * A_D + ((q ^ (row & 7)) << 2)) =
            make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
      if (valid) {
        const int64_t r = (((int64_t)req * a.n_splits + split) * a.s + tok) * a.n_q + qh;
        *reinterpret_cast<float2*>(a.ws_ml + r * 2) = make_float2(m_run, l_run);
      }
      named_bar_sync(1, 128);
      if (threadIdx.x == 64) TRACE(31, 5);
      if (threadIdx.x == 64) TRACE_MAX(1);
      split_merge<128>(a, stg, head, split, req, rb, rb * 128, min(128, R - rb * 128), threadIdx.x - 64);
    } else if (valid) {
      if (a.n_splits == 1) {
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        uint4* op = reinterpret_cast<uint4*>(a.out + (req_row0(a, req) + tok) * a.o_tok_stride + (int64_t)qh * A_D);
#pragma unroll
        for (int q = 0; q < 16; ++q)
          op[q] = make_uint4(pack_bf16(o[8 * q] * inv, o[8 * q + 1] * inv), pack_bf16(o[8 * q + 2] * inv, o[8 * q + 3] * inv),
                             pack_bf16(o[8 * q + 4] * inv, o[8 * q + 5] * inv), pack_bf16(o[8 * q + 6] * inv, o[8 * q + 7] * inv));
      } else {
        const int64_t r = (((int64_t)req * a.n_splits + split) * a.s + tok) * a.n_q + qh;
        float4* op = reinterpret_cast<float4*>(a.ws_o + r * A_D);
#pragma unroll
        for (int q = 0; q < 32; ++q) op[q] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        a.ws_ml[r * 2 + 0] = m_run;
        a.ws_ml[r * 2 + 1] = l_run;
      }
    }
    if (threadIdx.x == 64) TRACE(31, 6);
    if (threadIdx.x == 64) TRACE_MAX(2);
  }
  if (a.n_splits > 1 && a.merge == 2) cluster_split_merge<128>(a, cml, sm100::smem_u32(gKV), head, split, req, rb, R);
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 512);
  }
  if (threadIdx.x == 0) BND(a.seq, 1);
}


// K and V pages stream through separate rings: a K stage is released when its S
// MMA completes, a V stage when its PV MMA completes, so K runs further ahead of
// the softmax than a joint K+V ring of the same size allows.
#ifndef BST_T2_KS  // ring depths (measurement builds may override: BST_NVCC_EXTRA=-DBST_T2_KS=..)
#define BST_T2_KS 5
#endif
#ifndef BST_T2_VS
#define BST_T2_VS 4
#endif
constexpr int T2_KS = BST_T2_KS, T2_VS = BST_T2_VS;
#ifndef BST_T2_MIN_PAGES  // measurement builds may override
#define BST_T2_MIN_PAGES 4
#endif
constexpr int T2_MIN_PAGES = BST_T2_MIN_PAGES;  // per-CTA page run from which the two-group kernel is used
constexpr int T2_LCOL = 384;  // TMEM: S 0-127, O 128-383, row sums 384-415 (16 columns per group)
constexpr int T2_PCOL = 416;  // bf16 P of group g in columns 416 + 32 g .. + 32 (A operand of PV / row sums)
constexpr int T2_THREADS = 384;  // warps 0-1 K TMA / S issuer, 2-9 softmax groups, 10 V TMA, 11 PV issuer

__global__ void __launch_bounds__(T2_THREADS, 1) attn_tc2_kernel(const __grid_constant__ CUtensorMap tmKV, AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t fullK[T2_KS], emptyK[T2_KS], fullV[T2_VS], emptyV[T2_VS], s_full[2], s_free[2],
      p_full[2], o_done[2], q_ready;
  __shared__ uint32_t tmem_sh;
  __shared__ float xm[2][128], xl[2][128];
  __shared__ float2 cml[128];
  sm100::grid_dep_launch();
  if (threadIdx.x == 0) TRACE(31, 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = (sm100::smem_u32(smem_raw) + 1023) & ~1023u;
  uint8_t* smem = smem_raw + (base - sm100::smem_u32(smem_raw));
  const uint32_t sQ = base, sK = base + T_Q_BYTES, sV = sK + T2_KS * A_TILE_BYTES;
  const uint32_t sOnes = sV + T2_VS * A_TILE_BYTES;  // [16][64] bf16 ones: B operand of the row-sum MMA
  uint8_t* gQ = smem;
  uint8_t* gKV = smem + T_Q_BYTES;  // K ring, then V ring; reused as the merge staging buffer

  const int head = blockIdx.x, split = blockIdx.y, req = blockIdx.z / a.row_blocks, rb = blockIdx.z % a.row_blocks;
  const int c_ctx = a.state ? a.state[req * a.req_state + a.c_idx] : a.c;
  const int n_keys = c_ctx + a.keys_after_c;
  int R = a.group * a.s;
  if (a.row_cnt) {  // ragged batch: the row counts come from an earlier kernel of the graph
    sm100::grid_dep_wait();
    R = a.group * req_rows(a, req);
    if (rb * 128 >= R) return;  // every split of this (head, row block) exits: no barrier waits on it
  }
  int page0, n_tiles;
  split_pages(a, n_keys, split, page0, n_tiles);

  if (threadIdx.x == 0) {
    sm100::prefetch_tmap(&tmKV);
    for (int i = 0; i < T2_KS; ++i) { sm100::mbar_init(&fullK[i], 1); sm100::mbar_init(&emptyK[i], 1); }
    for (int i = 0; i < T2_VS; ++i) { sm100::mbar_init(&fullV[i], 1); sm100::mbar_init(&emptyV[i], 1); }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&s_free[i], 4);
      sm100::mbar_init(&p_full[i], 4);
      sm100::mbar_init(&o_done[i], 1);
    }
    sm100::mbar_init(&q_ready, 8);
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc(&tmem_sh, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_sh;

  if (warp == 0 || warp == 10) {
    if (lane == 0) {
      const bool isK = warp == 0;
      if (isK)
        issue_prefetch(a.pf, (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x,
                       gridDim.x * gridDim.y * gridDim.z);
      const int ns = isK ? T2_KS : T2_VS;
      uint64_t* fb = isK ? fullK : fullV;
      uint64_t* eb = isK ? emptyK : emptyV;
      uint8_t* ring = isK ? gKV : gKV + T2_KS * A_TILE_BYTES;
      // PDL: pages entirely below c hold committed K/V the previous kernel does not
      // touch; the page holding slot c onwards is written by qkv_rope right before us.
      const int safe_tiles = max(min(pdl_safe_slots(a, c_ctx) / A_PAGE - page0, n_tiles), 0);
      bool waited = false;
      for (int i = 0; i < n_tiles; ++i) {
        const int st = i % ns;
        if (i >= ns) sm100::mbar_wait(&eb[st], ((i / ns) & 1) ^ 1);
        if (!waited && (i >= safe_tiles || i >= ns)) {
          sm100::grid_dep_wait();
          waited = true;
        }
        const int phys = a.page_table[(int64_t)req * a.req_pages + page0 + i];
        const int64_t row = ((((int64_t)a.layer * a.n_pages_total + phys) * 2 + (isK ? 0 : 1)) * a.n_kv + head) * A_PAGE;
        uint8_t* dst = ring + st * A_TILE_BYTES;
        sm100::mbar_expect_tx(&fb[st], A_TILE_BYTES);
        sm100::tma_load_2d(dst, &tmKV, &fb[st], 0, (int)row);
        sm100::tma_load_2d(dst + A_PAGE * 128, &tmKV, &fb[st], 64, (int)row);
        if (isK) TRACE(i, 0);
      }
    }
  } else if (warp == 1) {
    const uint32_t idS = sm100::idesc_bf16(128, A_PAGE);
    sm100::mbar_wait(&q_ready, 0);
    // S issuer: S(i) (group i & 1) as soon as K(i) has landed and the group has read
    // S(i - 2) out of TMEM.  PV runs on its own issuing warp (warp 11), so neither kind
    // of MMA waits behind the other and the two softmax groups stay decoupled.
    for (int i = 0; i < n_tiles; ++i) {
      const int st = i % T2_KS, b = i & 1;
      sm100::mbar_wait(&fullK[st], (i / T2_KS) & 1);
      if (i >= 2) sm100::mbar_wait(&s_free[b], ((i - 2) >> 1) & 1);
      if (lane == 0) TRACE(i, 1);
      sm100::tc_fence_after();
      if (sm100::elect_one()) {
        const uint32_t kb = sK + st * A_TILE_BYTES;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint64_t ad = sm100::desc_k_sw128(sQ + (j >> 2) * (128 * 128) + (j & 3) * 32);
          const uint64_t bd = sm100::desc_k_sw128(kb + (j >> 2) * (A_PAGE * 128) + (j & 3) * 32);
          sm100::umma_f16(tmem + b * A_PAGE, ad, bd, idS, j > 0 ? 1u : 0u);
        }
        sm100::umma_commit(&s_full[b]);
        sm100::umma_commit(&emptyK[st]);
      }
      __syncwarp();
    }
  } else if (warp == 11) {
    const uint32_t idO = sm100::idesc_bf16_bmn(128, A_D);
    const uint32_t idL = sm100::idesc_bf16(128, 16);
    for (int j = 0; j < n_tiles; ++j) {
      const int stj = j % T2_VS;
      sm100::mbar_wait(&p_full[j & 1], (j >> 1) & 1);
      sm100::mbar_wait(&fullV[stj], (j / T2_VS) & 1);
      if (lane == 0) TRACE(j, 2);
      sm100::tc_fence_after();
      if (sm100::elect_one()) {
        const uint32_t vb = sV + stj * A_TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = sm100::desc_mn_sw128(vb + kk * 2048, A_PAGE * 128);
          sm100::umma_f16_ts(tmem + 128 + (j & 1) * A_D, tmem + T2_PCOL + 32 * (j & 1) + 8 * kk, bd, idO,
                             (j > 1 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // row sums of P: l += P x ones (the same bf16 P as the numerator)
          const uint64_t bd = sm100::desc_k_sw128(sOnes + kk * 32);
          sm100::umma_f16_ts(tmem + T2_LCOL + (j & 1) * 16, tmem + T2_PCOL + 32 * (j & 1) + 8 * kk, bd, idL,
                             (j > 1 || kk > 0) ? 1u : 0u);
        }
        sm100::umma_commit(&o_done[j & 1]);
        sm100::umma_commit(&emptyV[stj]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- two groups x one thread per query row; group g takes tiles g, g+2, ...
    const int g = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const int rg = rb * 128 + row;
    const bool valid = rg < R;
    const int rr = valid ? rg : 0;
    const int tok = rr / a.group;
    const int qh = head * a.group + rr % a.group;
    const uint32_t* mrow = a.mode == 0 ? a.anc + ((int64_t)req * a.s + tok) * a.mask_words : nullptr;
    const int mode = a.mode, mwords = a.mask_words;
    const float scale = a.scale_log2;
    sm100::grid_dep_wait();  // q is produced by the previous kernel (PDL)
    if (threadIdx.x == 64) TRACE(31, 2);
    if (threadIdx.x == 64) TRACE_MAX(0);
    {  // each group stages one 64-dim half of the row
      const int4* src = reinterpret_cast<const int4*>(a.q + (req_row0(a, req) + tok) * a.q_tok_stride + (int64_t)qh * A_D) + 8 * g;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int4 v = valid ? src[q] : make_int4(0, 0, 0, 0);
        *reinterpret_cast<int4*>(gQ + g * (128 * 128) + row * 128 + ((q ^ (row & 7)) << 4)) = v;
      }
    }
    *reinterpret_cast<uint2*>(gKV + (T2_KS + T2_VS) * A_TILE_BYTES + (threadIdx.x - 64) * 8) =
        make_uint2(0x3F803F80u, 0x3F803F80u);  // bf16 1.0 x 4
    sm100::fence_async_shared();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(&q_ready);
    if (threadIdx.x == 64) TRACE(31, 3);
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    const uint32_t o_col = 128 + g * A_D;
    float m_run = -INFINITY;
    int u = 0;
    for (int i = g; i < n_tiles; i += 2, ++u) {
      sm100::mbar_wait(&s_full[g], u & 1);
      if (threadIdx.x == 64 || threadIdx.x == 192) TRACE(i, 3);
      sm100::tc_fence_after();
      float sv[64];
      {  // the tile's 64 score columns: four loads in flight, one wait
        uint32_t r[4][16];
#pragma unroll
        for (int k = 0; k < 4; ++k) sm100::tmem_ld16_nw(lane_base + g * A_PAGE + 16 * k, r[k]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int e = 0; e < 16; ++e) sv[16 * k + e] = __uint_as_float(r[k][e]);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&s_free[g]);
      if (threadIdx.x == 64 || threadIdx.x == 192) TRACE(i, 7);
      const int slot0 = (page0 + i) * A_PAGE;
      const uint64_t vis = valid ? row_vis64(mode, c_ctx, n_keys, tok, slot0, mrow, mwords) : 0ull;
      // max over the raw scores (scale > 0 commutes with max); masked keys -> -inf
      if (!__all_sync(0xffffffffu, vis == ~0ull)) {
#pragma unroll
        for (int k = 0; k < 64; ++k) sv[k] = ((vis >> k) & 1ull) ? sv[k] : -INFINITY;
      }
      float mx8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mx8[k] = fmaxf(fmaxf(sv[k], sv[k + 8]), fmaxf(sv[k + 16], sv[k + 24]));
#pragma unroll
      for (int k = 0; k < 8; ++k) mx8[k] = fmaxf(mx8[k], fmaxf(fmaxf(sv[k + 32], sv[k + 40]), fmaxf(sv[k + 48], sv[k + 56])));
      const float mt = scale * fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                     fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float m_new = fmaxf(m_run, mt);
      const bool rescale = (m_run == -INFINITY) ? (m_new != -INFINITY) : (m_new > m_run + T_RESCALE);
      const float m_ref = rescale ? m_new : m_run;
      const float alpha = (rescale && m_run != -INFINITY) ? ex2(m_run - m_ref) : (rescale ? 0.f : 1.f);
      const float nsub = m_ref == -INFINITY ? 0.f : -m_ref;
      uint32_t pk[32];
#pragma unroll
      for (int k = 0; k < 64; k += 2) {
        const float x0 = fmaf(sv[k], scale, nsub), x1 = fmaf(sv[k + 1], scale, nsub);
        // every fourth exponential on the FMA pipe, the rest on MUFU
        const float p0 = ex2(x0);
        const float p1 = (k & 2) ? ex2_poly(x1) : ex2(x1);
        pk[k >> 1] = pack_bf16(p0, p1);
      }
      if (threadIdx.x == 64 || threadIdx.x == 192) TRACE(i, 4);
      // this group's previous PV (tile i-2) must be done before P/O are touched
      if (u >= 1) sm100::mbar_wait(&o_done[g], (u - 1) & 1);
      if (threadIdx.x == 64 || threadIdx.x == 192) TRACE(i, 5);
      sm100::tc_fence_after();
      if (__any_sync(0xffffffffu, rescale && u >= 1)) {
        const float f = (rescale && u >= 1) ? alpha : 1.f;
#pragma unroll 1
        for (int cc = 0; cc < 8; ++cc) {
          float ov[16];
          sm100::tmem_ld16(lane_base + o_col + 16 * cc, ov);
#pragma unroll
          for (int e = 0; e < 16; ++e) ov[e] *= f;
          sm100::tmem_st16(lane_base + o_col + 16 * cc, ov);
        }
        float lv[16];
        sm100::tmem_ld16(lane_base + T2_LCOL + 16 * g, lv);
#pragma unroll
        for (int e = 0; e < 16; ++e) lv[e] *= f;
        sm100::tmem_st16(lane_base + T2_LCOL + 16 * g, lv);
        sm100::tmem_st_wait();
      }
      m_run = m_ref;
      // bf16 P straight into tensor memory: the PV / row-sum MMAs read it as their A
      // operand (no shared-memory round trip, no proxy fence)
      sm100::tmem_st32u(lane_base + T2_PCOL + 32 * g, pk);
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&p_full[g]);
      if (threadIdx.x == 64 || threadIdx.x == 192) TRACE(i, 6);
    }
    // ---------------- merge the two groups; thread (g, row) writes dims [64 g, 64 g + 64)
    if (u >= 1) sm100::mbar_wait(&o_done[g], (u - 1) & 1);
    if (threadIdx.x == 64) TRACE(31, 4);
    xm[g][row] = m_run;
    sm100::tc_fence_before();
    named_bar_sync(1, 256);
    sm100::tc_fence_after();
    const float mA = xm[0][row], mB = xm[1][row];
    const float M = fmaxf(mA, mB);
    const float wA = (mA == -INFINITY) ? 0.f : ex2(mA - M), wB = (mB == -INFINITY) ? 0.f : ex2(mB - M);
    const bool hasA = n_tiles >= 1, hasB = n_tiles >= 2;
    float L = 0.f;
    {
      float la[16], lb[16];
      if (hasA) sm100::tmem_ld16(lane_base + T2_LCOL, la);
      if (hasB) sm100::tmem_ld16(lane_base + T2_LCOL + 16, lb);
      L = (hasA ? wA * la[0] : 0.f) + (hasB ? wB * lb[0] : 0.f);
    }
    float o[64];
    {  // group A's 64 columns in flight together (one wait), then group B's (register budget)
      uint32_t r[4][16];
#pragma unroll
      for (int e = 0; e < 64; ++e) o[e] = 0.f;
      if (hasA) {
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) sm100::tmem_ld16_nw(lane_base + 128 + 64 * g + 16 * cc, r[cc]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
#pragma unroll
          for (int e = 0; e < 16; ++e) o[16 * cc + e] = wA * __uint_as_float(r[cc][e]);
      }
      if (hasB) {
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) sm100::tmem_ld16_nw(lane_base + 128 + A_D + 64 * g + 16 * cc, r[cc]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
#pragma unroll
          for (int e = 0; e < 16; ++e) o[16 * cc + e] = (hasA ? o[16 * cc + e] : 0.f) + wB * __uint_as_float(r[cc][e]);
      }
    }
    if (a.n_splits > 1 && a.merge == 2) {  // normalised fp16 rows (see attn_tc_kernel)
      const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint4*>(gKV + row * 256 + (((8 * g + q) ^ (row & 7)) << 4)) =
            make_uint4(pack_f16(o[8 * q] * inv, o[8 * q + 1] * inv), pack_f16(o[8 * q + 2] * inv, o[8 * q + 3] * inv),
                       pack_f16(o[8 * q + 4] * inv, o[8 * q + 5] * inv), pack_f16(o[8 * q + 6] * inv, o[8 * q + 7] * inv));
      if (g == 0) cml[row] = make_float2(M, L);
    } else if (a.n_splits > 1 && a.merge) {
      const int Rws = a.group * a.s;  // the workspace keeps the uniform per-request row stride
      if (valid) {  // unnormalised partial straight to the L2 workspace, coalesced over rows
        const int64_t bse = kt_ws_base(a, req, split, head);
        float4* op = reinterpret_cast<float4*>(a.ws_o) + (bse * 32 + 16 * g) * Rws + rg;
#pragma unroll
        for (int q = 0; q < 16; ++q) __stcg(op + (int64_t)q * Rws, make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]));
        if (g == 0) __stcg(reinterpret_cast<float2*>(a.ws_ml) + bse * Rws + rg, make_float2(M, L));
      }
      if (threadIdx.x == 64) TRACE(31, 5);
      if (threadIdx.x == 64) TRACE_MAX(1);
      kt_global_merge(a, head, split, req, rb, rb * 128, min(128, R - rb * 128), threadIdx.x - 64);
    } else if (valid) {
      if (a.n_splits == 1) {
        const float inv = L > 0.f ? 1.f / L : 0.f;
        uint4* op = reinterpret_cast<uint4*>(a.out + (req_row0(a, req) + tok) * a.o_tok_stride + (int64_t)qh * A_D + 64 * g);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          op[q] = make_uint4(pack_bf16(o[8 * q] * inv, o[8 * q + 1] * inv), pack_bf16(o[8 * q + 2] * inv, o[8 * q + 3] * inv),
                             pack_bf16(o[8 * q + 4] * inv, o[8 * q + 5] * inv), pack_bf16(o[8 * q + 6] * inv, o[8 * q + 7] * inv));
      } else {
        const int64_t r = (((int64_t)req * a.n_splits + split) * a.s + tok) * a.n_q + qh;
        float4* op = reinterpret_cast<float4*>(a.ws_o + r * A_D + 64 * g);
#pragma unroll
        for (int q = 0; q < 16; ++q) op[q] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        if (g == 0) {
          a.ws_ml[r * 2 + 0] = M;
          a.ws_ml[r * 2 + 1] = L;
        }
      }
    }
  }
  if (threadIdx.x == 64) TRACE(31, 6);
  if (a.n_splits > 1 && a.merge == 2) cluster_split_merge<256>(a, cml, sm100::smem_u32(gKV), head, split, req, rb, R);
  if (threadIdx.x == 64) TRACE_MAX(2);
  if (threadIdx.x == 0) TRACE(31, 0);
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 512);
  }
}

// ===========================================================================
// Key-major tcgen05 variant (default): S^T = K Q^T, so a TMEM lane holds one KEY and
// its columns hold every query row of the CTA.  Decode-time trees have few rows
// (GQA group x tree tokens, e.g. 4 x 17 = 68), which in the row-major kernels above
// leave most TMEM lanes / softmax threads idle and serialise 64 exponentials per
// thread per tile; here all 128 lanes (4 warps, one per SM sub-partition) are busy
// for any row count and each thread does one exponential per row.
//   * 128-key tiles (two 64-slot pages), K and V in separate 2-stage TMA rings.
//   * S^T: M = 128 keys, N = NP (rows rounded up to 16), K = 128 dims; double buffer.
//   * softmax against a per-row REFERENCE maximum (smem), not a per-tile max: the
//     fast path is p = 2^(s*scale - ref) with no cross-lane reduction; one barrier
//     with an OR reduction per tile detects any row whose score exceeds its reference
//     by > 2^KT_OVF, and only then (always on a row's first visible tile) the slow path
//     reduces per-row tile maxima (redux.sync.max.f32 + 4-warp smem), raises the
//     references, rescales those rows of O/l in TMEM and recomputes P.  Any reference
//     within the headroom gives the same softmax (the factor cancels in O / l).
//   * P^T is written key-major (MN-major A operand): [row half][128 keys][128 B].
//   * O += P V (A and B MN-major) and l += P 1 (a second MMA against a ones matrix),
//     so the row sums use the same bf16 P as the numerator and need no shuffles.
// warp 0: K TMA, warp 1: TMEM owner + S issuer, warps 2-9: softmax (warp w owns TMEM
// lanes 32 (w % 4) ..; two warps per SM sub-partition split the rows), warp 10: V TMA,
// warp 11: PV issuer.
// ===========================================================================
constexpr int KT_SM_WARPS = 8;                     // softmax warps 2 .. 9
constexpr int KT_VTMA_WARP = 10, KT_PV_WARP = 11;
constexpr int KT_THREADS = 384;
constexpr int KT_KEYS = 128;
constexpr int KT_TILE_BYTES = KT_KEYS * A_D * 2;  // 32 KiB: K or V of one tile
constexpr int KT_KS = 2, KT_VS = 2;
constexpr int KT_P_BYTES = 128 * KT_KEYS * 2;     // one P^T buffer: [2 row halves][128 keys][128 B]
constexpr int KT_ONES_BYTES = 16 * 128;           // [16][64 keys] bf16 ones (every K step reads the same block)
// per row count: Q [2 dim halves][NP rows][128 B]; P^T double-buffered while it fits
__host__ __device__ constexpr int kt_pbufs(int nch) { return nch <= 6 ? 2 : 1; }
__host__ __device__ constexpr int kt_smem(int nch) {
  return nch * 16 * 256 + kt_pbufs(nch) * KT_P_BYTES + KT_ONES_BYTES + 4 * KT_TILE_BYTES + 1024;
}
constexpr int KT_O_COL = 256, KT_L_COL = 384;     // TMEM: S 0-255 (two buffers), O, l
constexpr float KT_OVF = 48.f;                     // log2 headroom above the reference

__device__ __forceinline__ float redux_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
// named barrier over `n` threads returning whether any thread's predicate was true
__device__ __forceinline__ bool bar_or(int id, int n, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred q, o;\n\t"
      "setp.ne.u32 q, %1, 0;\n\t"
      "barrier.red.or.pred o, %2, %3, q;\n\t"
      "selp.u32 %0, 1, 0, o;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}


// p = 2^(s * scale - ref) for the NP rows of this thread's key (all chunks loaded from
// TMEM with one wait); masked entries -> 0.  Returns the largest exponent (overflow
// check).  Unmasked tiles run every fourth exponential on the FMA pipe (ex2_poly).
template <int NCH, bool MASKED, int NA>
__device__ __forceinline__ float kt_tile(uint32_t taddr, const float* nmref, float scale, const uint32_t (&vis)[NA],
                                         uint32_t (&pk)[NA][8]) {
  static_assert(NCH <= NA, "chunk count exceeds the register arrays");
  uint32_t r[NCH > 0 ? NCH : 1][16];
#pragma unroll
  for (int c = 0; c < NCH; ++c) sm100::tmem_ld16_nw(taddr + 16 * c, r[c]);
  sm100::tmem_ld_wait();
  float em = -INFINITY;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const float4* nm4 = reinterpret_cast<const float4*>(nmref + 16 * c);
    float d[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 v = nm4[q];
      d[4 * q + 0] = fmaf(__uint_as_float(r[c][4 * q + 0]), scale, v.x);
      d[4 * q + 1] = fmaf(__uint_as_float(r[c][4 * q + 1]), scale, v.y);
      d[4 * q + 2] = fmaf(__uint_as_float(r[c][4 * q + 2]), scale, v.z);
      d[4 * q + 3] = fmaf(__uint_as_float(r[c][4 * q + 3]), scale, v.w);
    }
    if (MASKED) {
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (!((vis[c] >> e) & 1u)) d[e] = -INFINITY;
    }
    float m = fmax3(d[0], d[1], d[2]);
#pragma unroll
    for (int e = 3; e < 15; e += 2) m = fmax3(m, d[e], d[e + 1]);
    em = fmax3(em, m, d[15]);
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
      const float p0 = ex2(d[e]);
      const float p1 = (!MASKED && (e & 2)) ? ex2_poly(d[e + 1]) : ex2(d[e + 1]);
      pk[c][e >> 1] = pack_bf16(p0, p1);
    }
  }
  return em;
}

template <int NCH>
__global__ void __launch_bounds__(KT_THREADS, 1) attn_kt_kernel(const __grid_constant__ CUtensorMap tmKV, AttnArgs a) {
  constexpr int NP = NCH * 16;
  constexpr int C0 = (NCH + 1) / 2, C1 = NCH / 2;  // row chunks of softmax half 0 / half 1
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t fullK[KT_KS], emptyK[KT_KS], fullV[KT_VS], emptyV[KT_VS], s_full[2], s_free[2],
      p_full[2], o_done[2], q_ready;
  __shared__ uint32_t tmem_sh;
  __shared__ __align__(16) float nmref[NP];  // -(reference max), log2 domain; +inf: row has seen no key yet
  __shared__ float alpha_sh[128];
  __shared__ float wmax[4][NP];
  __shared__ uint32_t colm[KT_KEYS][4];  // tree tile: bit r of colm[k][r / 32] = row r sees key k
  __shared__ float2 ml_sh[128];          // cluster merge: (reference max, row sum) of this CTA's rows
  sm100::grid_dep_launch();
  if (threadIdx.x == 0) TRACE(31, 1);
  if (threadIdx.x == 0) TRACE_MIN(0);
  if (threadIdx.x == 0) TRACE_MAX(5);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = (sm100::smem_u32(smem_raw) + 1023) & ~1023u;
  uint8_t* smem = smem_raw + (base - sm100::smem_u32(smem_raw));
  constexpr int PB = kt_pbufs(NCH);  // P^T buffers: tile i uses buffer i % PB, barriers p_full / o_done[i % PB]
  const uint32_t sQ = base, sP = sQ + NP * 256, sOnes = sP + PB * KT_P_BYTES, sK = sOnes + KT_ONES_BYTES;
  const uint32_t sV = sK + KT_KS * KT_TILE_BYTES;
  uint8_t* gQ = smem;
  uint8_t* gP = smem + NP * 256;
  uint8_t* gOnes = gP + PB * KT_P_BYTES;
  uint8_t* gK = gOnes + KT_ONES_BYTES;  // K ring, then V ring; reused as the merge staging buffer
  uint8_t* gV = gK + KT_KS * KT_TILE_BYTES;

  const int head = blockIdx.x, split = blockIdx.y, req = blockIdx.z / a.row_blocks, rb = blockIdx.z % a.row_blocks;
  const int c_ctx = a.state ? a.state[req * a.req_state + a.c_idx] : a.c;
  const int n_keys = c_ctx + a.keys_after_c;
  int R = a.group * a.s;
  if (a.row_cnt) {  // ragged batch: the row counts come from an earlier kernel of the graph
    sm100::grid_dep_wait();
    R = a.group * req_rows(a, req);
    if (rb * 128 >= R) return;  // every split of this (head, row block) exits: no barrier waits on it
  }
  const int row0 = rb * a.rows_per_block;
  const int Rb = min(a.rows_per_block, R - row0);
  int page0, n_pages;
  split_pages(a, n_keys, split, page0, n_pages);
  const int n_tiles = (n_pages + 1) >> 1;

  if (threadIdx.x == 0) {
    sm100::prefetch_tmap(&tmKV);
    for (int i = 0; i < KT_KS; ++i) { sm100::mbar_init(&fullK[i], 1); sm100::mbar_init(&emptyK[i], 1); }
    for (int i = 0; i < KT_VS; ++i) { sm100::mbar_init(&fullV[i], 1); sm100::mbar_init(&emptyV[i], 1); }
    for (int i = 0; i < 2; ++i) { sm100::mbar_init(&s_full[i], 1); sm100::mbar_init(&s_free[i], KT_SM_WARPS); }
    for (int i = 0; i < 2; ++i) { sm100::mbar_init(&p_full[i], KT_SM_WARPS); sm100::mbar_init(&o_done[i], 1); }
    sm100::mbar_init(&q_ready, KT_SM_WARPS);
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc(&tmem_sh, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_sh;

  if (warp == 0 || warp == KT_VTMA_WARP) {
    if (lane == 0) {
      const bool isK = warp == 0;
      if (isK)
        issue_prefetch(a.pf, (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x,
                       gridDim.x * gridDim.y * gridDim.z);
      uint64_t* fb = isK ? fullK : fullV;
      uint64_t* eb = isK ? emptyK : emptyV;
      uint8_t* ring = isK ? gK : gV;
      // PDL: pages entirely below c hold committed K/V the previous kernel does not touch
      const int safe_pages = max(min(pdl_safe_slots(a, c_ctx) / A_PAGE - page0, n_pages), 0);
      const int64_t pt = (int64_t)req * a.req_pages + page0;
      bool waited = false;
      for (int i = 0; i < n_tiles; ++i) {
        const int st = i & 1;
        if (i >= 2) sm100::mbar_wait(&eb[st], ((i >> 1) & 1) ^ 1);
        // the second page of an odd split's last tile re-loads the first (finite data; its keys are masked)
        const int pA = 2 * i, pB = min(2 * i + 1, n_pages - 1);
        if (!waited && (pB >= safe_pages || i >= 2)) {
          sm100::grid_dep_wait();
          waited = true;
        }
        const int kv = isK ? 0 : 1;
        const int64_t rowA = ((((int64_t)a.layer * a.n_pages_total + a.page_table[pt + pA]) * 2 + kv) * a.n_kv + head) * A_PAGE;
        const int64_t rowB = ((((int64_t)a.layer * a.n_pages_total + a.page_table[pt + pB]) * 2 + kv) * a.n_kv + head) * A_PAGE;
        uint8_t* dst = ring + st * KT_TILE_BYTES;
        sm100::mbar_expect_tx(&fb[st], KT_TILE_BYTES);
        sm100::tma_load_2d(dst, &tmKV, &fb[st], 0, (int)rowA);
        sm100::tma_load_2d(dst + 8192, &tmKV, &fb[st], 0, (int)rowB);
        sm100::tma_load_2d(dst + 16384, &tmKV, &fb[st], 64, (int)rowA);
        sm100::tma_load_2d(dst + 24576, &tmKV, &fb[st], 64, (int)rowB);
        if (isK) TRACE(i, 0);
      }
    }
  } else if (warp == 1) {
    const uint32_t idS = sm100::idesc_bf16(128, NP);
    sm100::mbar_wait(&q_ready, 0);
    for (int i = 0; i < n_tiles; ++i) {
      const int st = i & 1, b = i & 1;
      sm100::mbar_wait(&fullK[st], (i >> 1) & 1);
      if (i >= 2) sm100::mbar_wait(&s_free[b], ((i - 2) >> 1) & 1);
      if (lane == 0) TRACE(i, 1);
      sm100::tc_fence_after();
      if (sm100::elect_one()) {
        const uint32_t kb = sK + st * KT_TILE_BYTES;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint64_t ad = sm100::desc_k_sw128(kb + (j >> 2) * 16384 + (j & 3) * 32);
          const uint64_t bd = sm100::desc_k_sw128(sQ + (j >> 2) * (NP * 128) + (j & 3) * 32);
          sm100::umma_f16(tmem + b * 128, ad, bd, idS, j > 0 ? 1u : 0u);
        }
        sm100::umma_commit(&s_full[b]);
        sm100::umma_commit(&emptyK[st]);
      }
      __syncwarp();
    }
  } else if (warp == KT_PV_WARP) {
    const uint32_t idO = sm100::idesc_bf16_abmn(128, A_D);
    const uint32_t idL = sm100::idesc_bf16_amn(128, 16);
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j & 1;
      sm100::mbar_wait(&p_full[j % PB], (j / PB) & 1);
      sm100::mbar_wait(&fullV[st], (j >> 1) & 1);
      if (lane == 0) TRACE(j, 2);
      sm100::tc_fence_after();
      if (sm100::elect_one()) {
        const uint32_t vb = sV + st * KT_TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = sm100::desc_mn_sw128(sP + (j % PB) * KT_P_BYTES + kk * 2048, 16384);
          const uint64_t bd = sm100::desc_mn_sw128(vb + kk * 2048, 16384);
          sm100::umma_f16(tmem + KT_O_COL, ad, bd, idO, (j > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = sm100::desc_mn_sw128(sP + (j % PB) * KT_P_BYTES + kk * 2048, 16384);
          const uint64_t bd = sm100::desc_k_sw128(sOnes + (kk & 3) * 32);
          sm100::umma_f16(tmem + KT_L_COL, ad, bd, idL, (j > 0 || kk > 0) ? 1u : 0u);
        }
        sm100::umma_commit(&o_done[j % PB]);
        sm100::umma_commit(&emptyV[st]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- softmax: warps 2 .. 9.  Warp w owns TMEM lanes 32 (w % 4) .. (key kk of
    // each S^T tile, query row kk of O); half h = (w - 2) / 4 takes row chunks
    // [h C0, h C0 + (h ? C1 : C0)) of the tile and O columns / dims [64 h, 64 h + 64).
    const int t = threadIdx.x - 64;  // 0 .. 255
    const int quad = warp & 3, h = (warp - 2) >> 2;
    const int kk = quad * 32 + lane;
    const int c0 = h ? C0 : 0;
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    const float scale = a.scale_log2;
    if (t < NP) nmref[t] = t < Rb ? INFINITY : 0.f;  // padding rows (zero Q): p = 1, never overflow
    sm100::grid_dep_wait();  // q is produced by the previous kernel (PDL)
    if (t == 0) TRACE(31, 2);
    {  // stage query rows (K-major, 128B swizzle): thread t stages dim half t / 128 of row t % 128
      const int row = t & 127, hq = t >> 7;
      if (row < NP) {
        const bool valid = row < Rb;
        const int rg = row0 + (valid ? row : 0);
        const int tok = rg / a.group, qh = head * a.group + rg % a.group;
        const int4* src =
            reinterpret_cast<const int4*>(a.q + (req_row0(a, req) + tok) * a.q_tok_stride + (int64_t)qh * A_D) + 8 * hq;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int4 v = valid ? src[q] : make_int4(0, 0, 0, 0);
          *reinterpret_cast<int4*>(gQ + hq * (NP * 128) + row * 128 + ((q ^ (row & 7)) << 4)) = v;
        }
      }
    }
    if (t < KT_ONES_BYTES / 16)
      *reinterpret_cast<uint4*>(gOnes + t * 16) = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    sm100::fence_async_shared();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(&q_ready);
    named_bar_sync(2, 256);  // nmref initialised
    if (t == 0) TRACE(31, 3);

    const uint32_t* anc = a.mode == 0 ? a.anc + (int64_t)req * a.s * a.mask_words : nullptr;
    const int my_tok = (row0 + min(t & 127, Rb - 1)) / a.group;
    const int abl = g_kt_ablate;
    for (int i = 0; i < n_tiles; ++i) {
      const int b = i & 1;
      const int tslot0 = (page0 + 2 * i) * A_PAGE;
      const int slot = tslot0 + kk;
      // key class: 0 visible to no row, 1 to every row, 2 per row (tree / causal part)
      int cls;
      if (2 * i + (kk >> 6) >= n_pages || slot >= n_keys) cls = 0;
      else if (a.mode == 2 || slot < c_ctx) cls = 1;
      else cls = 2;
      if (a.mode == 0 && tslot0 + KT_KEYS > c_ctx && tslot0 < n_keys) {
        // tree keys in this tile: column masks by ballots; thread t evaluates row t % 128
        // for the keys of parity t / 128
        const int k_lo = max(c_ctx - tslot0, 0), k_hi = min(n_keys - tslot0, KT_KEYS);
        const int rr = t & 127;
        int wi = -1;
        uint32_t wv = 0;
        for (int k2 = k_lo + h; k2 < k_hi; k2 += 2) {
          const int j = tslot0 + k2 - c_ctx;
          bool bit = false;
          if (rr < Rb) {
            if ((j >> 5) != wi) {
              wi = j >> 5;
              wv = anc[(int64_t)my_tok * a.mask_words + wi];
            }
            bit = (wv >> (j & 31)) & 1u;
          }
          const uint32_t bal = __ballot_sync(0xffffffffu, bit);
          if (lane == 0) colm[k2][rr >> 5] = bal;
        }
        named_bar_sync(2, 256);
      }
      uint32_t vis[C0];
#pragma unroll
      for (int u = 0; u < C0; ++u) {
        const int c = c0 + u;
        uint32_t v;
        if (cls == 2) {
          if (a.mode == 1) {  // causal: rows whose token is >= the key's tree index
            const int rmin = max((slot - c_ctx) * a.group - row0, 0), lo = 16 * c;
            v = rmin <= lo ? 0xFFFFu : (rmin >= lo + 16 ? 0u : ((0xFFFFu << (rmin - lo)) & 0xFFFFu));
          } else {
            v = (colm[kk][c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
          }
        } else {
          v = cls == 1 ? 0xFFFFu : 0u;
        }
        vis[u] = v;
      }
      const bool masked = !__all_sync(0xffffffffu, cls == 1);
      sm100::mbar_wait(&s_full[b], (i >> 1) & 1);
      if (t == 0) TRACE(i, 3);
      sm100::tc_fence_after();
      const uint32_t sb = lane_base + b * 128 + 16 * c0;
      const float* nmr = nmref + 16 * c0;
      uint32_t pk[C0][8];
      float emax = -INFINITY;
      bool need;
      if (i == 0) {
        // first tile: references = the scores of key 0 when every row sees it (any visible
        // score is <= the row max, so only the overflow side needs checking)
        const bool cheap = n_pages > 0 && (a.mode == 2 ? tslot0 < n_keys : tslot0 < c_ctx);
        if (cheap) {
          if (quad == 0) {
            uint32_t r0[C0][16];
            if (h == 0) {
#pragma unroll
              for (int u = 0; u < C0; ++u) sm100::tmem_ld16_nw(sb + 16 * u, r0[u]);
            } else {
#pragma unroll
              for (int u = 0; u < C1; ++u) sm100::tmem_ld16_nw(sb + 16 * u, r0[u]);
            }
            sm100::tmem_ld_wait();
            if (lane == 0) {
              const int nu = h ? C1 : C0;
#pragma unroll
              for (int u = 0; u < C0; ++u)
#pragma unroll
                for (int e = 0; e < 16; ++e)
                  if (u < nu && 16 * (c0 + u) + e < Rb) nmref[16 * (c0 + u) + e] = -(__uint_as_float(r0[u][e]) * scale);
            }
          }
          named_bar_sync(2, 256);
        }
        if (cheap) {
          if (h == 0) emax = masked ? kt_tile<C0, true>(sb, nmr, scale, vis, pk) : kt_tile<C0, false>(sb, nmr, scale, vis, pk);
          else if (C1 > 0) emax = masked ? kt_tile<C1, true>(sb, nmr, scale, vis, pk) : kt_tile<C1, false>(sb, nmr, scale, vis, pk);
        }
        need = !cheap || emax > KT_OVF;
      } else if (abl & 1) {
#pragma unroll
        for (int u = 0; u < C0; ++u)
#pragma unroll
          for (int e = 0; e < 8; ++e) pk[u][e] = 0u;
        need = false;
      } else {
        if (h == 0) emax = masked ? kt_tile<C0, true>(sb, nmr, scale, vis, pk) : kt_tile<C0, false>(sb, nmr, scale, vis, pk);
        else if (C1 > 0) emax = masked ? kt_tile<C1, true>(sb, nmr, scale, vis, pk) : kt_tile<C1, false>(sb, nmr, scale, vis, pk);
        need = emax > KT_OVF;
      }
      if (t == 0) TRACE(i, 4);
      if ((abl & 4) ? need : bar_or(3, 256, need)) {
        // slow path: per-row maxima of this tile -> raise the references -> rescale O, l
        const int nu = h ? C1 : C0;
#pragma unroll
        for (int u = 0; u < C0; ++u) {
          if (u < nu) {
            uint32_t r[16];
            sm100::tmem_ld16_nw(sb + 16 * u, r);
            sm100::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float x = ((vis[u] >> e) & 1u) ? __uint_as_float(r[e]) * scale : -INFINITY;
              const float wm = redux_max(x);
              if (lane == e + (u & 1) * 16) wmax[quad][16 * (c0 + u) + e] = wm;
            }
          }
        }
        named_bar_sync(2, 256);
        if (t < 128) {
          if (t < Rb) {
            const float tm = fmaxf(fmaxf(wmax[0][t], wmax[1][t]), fmaxf(wmax[2][t], wmax[3][t]));
            const float old = -nmref[t];
            float al = 1.f;
            if (tm > old) {
              al = old == -INFINITY ? 0.f : ex2(old - tm);
              nmref[t] = -tm;
            }
            alpha_sh[t] = al;
          } else {
            alpha_sh[t] = 1.f;
          }
        }
        named_bar_sync(2, 256);
        if (i >= 1) {
          sm100::mbar_wait(&o_done[(i - 1) % PB], ((i - 1) / PB) & 1);  // O, l hold PV(0 .. i-1)
          sm100::tc_fence_after();
          const float f = alpha_sh[kk];
          if (__any_sync(0xffffffffu, f != 1.f)) {  // O columns 0-79 (half 0), 80-143 (half 1, incl. l)
#pragma unroll 1
            for (int cc = 5 * h; cc < (h ? 9 : 5); ++cc) {
              float ov[16];
              sm100::tmem_ld16(lane_base + KT_O_COL + 16 * cc, ov);
#pragma unroll
              for (int e = 0; e < 16; ++e) ov[e] *= f;
              sm100::tmem_st16(lane_base + KT_O_COL + 16 * cc, ov);
            }
            sm100::tmem_st_wait();
          }
        }
        if (h == 0) kt_tile<C0, true>(sb, nmr, scale, vis, pk);
        else if (C1 > 0) kt_tile<C1, true>(sb, nmr, scale, vis, pk);
        if (t == 0) TRACE(i, 7);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&s_free[b]);
      if (i >= PB) sm100::mbar_wait(&o_done[i % PB], ((i - PB) / PB) & 1);  // PV(i-PB) has read this P buffer
      if (t == 0) TRACE(i, 5);
      // my key's column of P^T: rows 16c .. 16c+15 are 16-byte chunks 2c, 2c+1
      if (!(abl & 2)) {
        const int nu = h ? C1 : C0;
#pragma unroll
        for (int u = 0; u < C0; ++u) {
          if (u < nu) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int q = 2 * (c0 + u) + hh;
              *reinterpret_cast<uint4*>(gP + (i % PB) * KT_P_BYTES + (q >> 3) * 16384 + kk * 128 + (((q & 7) ^ (kk & 7)) << 4)) =
                  make_uint4(pk[u][4 * hh], pk[u][4 * hh + 1], pk[u][4 * hh + 2], pk[u][4 * hh + 3]);
            }
          }
        }
      }
      sm100::fence_async_shared();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&p_full[i % PB]);
      if (t == 0) TRACE(i, 6);
    }
    // ---------------- epilogue: thread (h, kk) owns dims [64 h, 64 h + 64) of query row kk
    float o[64];
    float L = 0.f;
    if (n_tiles > 0) {
      sm100::mbar_wait(&o_done[(n_tiles - 1) % PB], ((n_tiles - 1) / PB) & 1);
      if (t == 0) TRACE(31, 4);
      sm100::tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        float t16[16];
        sm100::tmem_ld16(lane_base + KT_O_COL + 64 * h + 16 * cc, t16);
#pragma unroll
        for (int e = 0; e < 16; ++e) o[16 * cc + e] = t16[e];
      }
      float lv[16];
      sm100::tmem_ld16(lane_base + KT_L_COL, lv);
      L = lv[0];
    } else {
#pragma unroll
      for (int e = 0; e < 64; ++e) o[e] = 0.f;
    }
    const bool valid = kk < Rb;
    const float m = valid ? -nmref[kk] : -INFINITY;
    const int rg = row0 + (valid ? kk : 0);
    const int tok = rg / a.group, qh = head * a.group + rg % a.group;
    if (a.n_splits > 1 && a.merge == 2) {
      // cluster merge: stage the partial rows in this CTA's shared memory (the idle K ring)
      float* stg = reinterpret_cast<float*>(gK);
#pragma unroll
      for (int q = 0; q < 16; ++q)
        *reinterpret_cast<float4*>(stg + kk * A_D + (((16 * h + q) ^ (kk & 7)) << 2)) =
            make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
      if (h == 0) ml_sh[kk] = make_float2(m, L);
    } else if (a.n_splits > 1 && a.merge) {
      if (valid) {  // unnormalised partial straight to the (L2-resident) workspace, coalesced over rows
        const int Rt = a.group * a.s, rr = row0 + kk;
        const int64_t bse = kt_ws_base(a, req, split, head);
        float4* op = reinterpret_cast<float4*>(a.ws_o) + (bse * 32 + 16 * h) * Rt + rr;
#pragma unroll
        for (int q = 0; q < 16; ++q) __stcg(op + (int64_t)q * Rt, make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]));
        if (h == 0) __stcg(reinterpret_cast<float2*>(a.ws_ml) + bse * Rt + rr, make_float2(m, L));
      }
      if (t == 0) TRACE(31, 5);
      if (t == 0) TRACE_MAX(1);
      kt_global_merge(a, head, split, req, rb, row0, Rb, t);
    } else if (valid) {
      if (a.n_splits == 1) {
        const float inv = L > 0.f ? 1.f / L : 0.f;
        uint4* op = reinterpret_cast<uint4*>(a.out + (req_row0(a, req) + tok) * a.o_tok_stride + (int64_t)qh * A_D + 64 * h);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          op[q] = make_uint4(pack_bf16(o[8 * q] * inv, o[8 * q + 1] * inv), pack_bf16(o[8 * q + 2] * inv, o[8 * q + 3] * inv),
                             pack_bf16(o[8 * q + 4] * inv, o[8 * q + 5] * inv), pack_bf16(o[8 * q + 6] * inv, o[8 * q + 7] * inv));
      } else {
        const int64_t r = (((int64_t)req * a.n_splits + split) * a.s + tok) * a.n_q + qh;
        float4* op = reinterpret_cast<float4*>(a.ws_o + r * A_D + 64 * h);
#pragma unroll
        for (int q = 0; q < 16; ++q) op[q] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        if (h == 0) {
          a.ws_ml[r * 2 + 0] = m;
          a.ws_ml[r * 2 + 1] = L;
        }
      }
    }
  }
  if (a.n_splits > 1 && a.merge == 2) {
    // the splits of this (head, row block) form one cluster (rank = split): every CTA
    // merges rows [rank * per, rank * per + per) from all ranks' staged partials over
    // DSMEM, in rank order (deterministic); a second cluster barrier keeps the staging
    // alive until every remote read is done
    if (threadIdx.x == 64) TRACE_MAX(1);
    cluster_sync_all();
    if (threadIdx.x == 64) TRACE_MAX(3);
    if (warp >= 2 && warp < 2 + KT_SM_WARPS) {
      const int t = threadIdx.x - 64, ns = a.n_splits;
      const int per = (Rb + ns - 1) / ns, r0 = split * per, r1 = min(r0 + per, Rb);
      const uint32_t stg_u = sK, ml_u = sm100::smem_u32(ml_sh);
      for (int it = t; it < (r1 - r0) * 32; it += 256) {
        const int r = r0 + (it >> 5), cq = it & 31;
        const uint32_t off = (uint32_t)(r * A_D + ((cq ^ (r & 7)) << 2)) * 4u;
        float2 ml[8];
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // every rank's loads in flight at once
          if (q < ns) {
            ml[q] = ld_dsmem_f2(mapa_shared(ml_u + r * 8, q));
            v[q] = ld_dsmem_f4(mapa_shared(stg_u + off, q));
          }
        }
        float M = -INFINITY;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < ns) M = fmaxf(M, ml[q].x);
        float Lsum = 0.f;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < ns && ml[q].x != -INFINITY) {
            const float w = ex2(ml[q].x - M);
            Lsum += w * ml[q].y;
            acc.x += w * v[q].x; acc.y += w * v[q].y; acc.z += w * v[q].z; acc.w += w * v[q].w;
          }
        }
        const float inv = Lsum > 0.f ? 1.f / Lsum : 0.f;
        const int rg = row0 + r, tok = rg / a.group, qh = head * a.group + rg % a.group;
        __nv_bfloat16* op = a.out + (req_row0(a, req) + tok) * a.o_tok_stride + (int64_t)qh * A_D + 4 * cq;
        *reinterpret_cast<uint2*>(op) = make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
      }
    }
    if (threadIdx.x == 64) TRACE_MAX(4);
    cluster_sync_all();
  }
  if (threadIdx.x == 64) TRACE_MAX(2);
  if (threadIdx.x == 64) TRACE(31, 6);
  sm100::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TRACE(31, 0);
  if (threadIdx.x == 0) TRACE_MAX(6);
  if (threadIdx.x == 0) TRACE_MIN(1);
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 512);
  }
}

// merge flash-decoding splits: one warp per (token, q-head) row, single pass
// with online rescaling, 4 splits in flight per iteration
__global__ void attn_combine_kernel(AttnArgs a) {
  pdl_enter();
  if (blockIdx.x == 0 && threadIdx.x == 0) TRACE(30, 0);
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), req = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int rows = a.s * a.n_q;
  if (row >= rows) return;
  if (a.row_cnt && row / a.n_q >= req_rows(a, req)) return;  // ragged: past this request's rows
  float M = -INFINITY, L = 0.f;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int sp0 = 0; sp0 < a.n_splits; sp0 += 4) {
    float m[4], l[4];
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int sp = sp0 + j;
      if (sp < a.n_splits) {
        const int64_t r = ((int64_t)req * a.n_splits + sp) * rows + row;
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
  __nv_bfloat16* op = a.out + (req_row0(a, req) + tok) * a.o_tok_stride + (int64_t)qh * A_D + lane * 4;
  *reinterpret_cast<uint2*>(op) = make_uint2(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv));
  if (blockIdx.x == 0 && threadIdx.x == 0) TRACE(30, 1);
}

}  // namespace bst

namespace bst {
// resident clusters of `cs` key-major CTAs (cudaOccupancyMaxActiveClusters)
static int kt_cluster_occupancy(int nch, int cs) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(8, cs, 1);
  cfg.blockDim = dim3(KT_THREADS);
  cfg.dynamicSmemBytes = kt_smem(nch);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = cs;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  cudaError_t e = cudaSuccess;
  switch (nch) {
    case 1: cudaFuncSetAttribute(attn_kt_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kt_smem(1)); e = cudaOccupancyMaxActiveClusters(&n, attn_kt_kernel<1>, &cfg); break;
    case 2: cudaFuncSetAttribute(attn_kt_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kt_smem(2)); e = cudaOccupancyMaxActiveClusters(&n, attn_kt_kernel<2>, &cfg); break;
    case 3: cudaFuncSetAttribute(attn_kt_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kt_smem(3)); e = cudaOccupancyMaxActiveClusters(&n, attn_kt_kernel<3>, &cfg); break;
    case 4: cudaFuncSetAttribute(attn_kt_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kt_smem(4)); e = cudaOccupancyMaxActiveClusters(&n, attn_kt_kernel<4>, &cfg); break;
    case 5: cudaFuncSetAttribute(attn_kt_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, kt_smem(5)); e = cudaOccupancyMaxActiveClusters(&n, attn_kt_kernel<5>, &cfg); break;
    case 6: cudaFuncSetAttribute(attn_kt_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, kt_smem(6)); e = cudaOccupancyMaxActiveClusters(&n, attn_kt_kernel<6>, &cfg); break;
    case 7: cudaFuncSetAttribute(attn_kt_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, kt_smem(7)); e = cudaOccupancyMaxActiveClusters(&n, attn_kt_kernel<7>, &cfg); break;
    default: cudaFuncSetAttribute(attn_kt_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kt_smem(8)); e = cudaOccupancyMaxActiveClusters(&n, attn_kt_kernel<8>, &cfg); break;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}


// resident clusters of `cs` row-major attention CTAs (cudaOccupancyMaxActiveClusters), per kernel
static int rm_cluster_fits(bool two_groups, int cs, int smem) {
  static int occ[2][T2_CLUSTER_MAX + 1];
  static bool init = false;
  if (!init) {
    for (int k = 0; k < 2; ++k)
      for (int i = 0; i <= T2_CLUSTER_MAX; ++i) occ[k][i] = -1;
    init = true;
  }
  if (cs < 2 || cs > T2_CLUSTER_MAX) return 0;
  int& o = occ[two_groups ? 1 : 0][cs];
  if (o >= 0) return o;
  auto kern = two_groups ? attn_tc2_kernel : attn_tc_kernel;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1, cs, 1);
  cfg.blockDim = dim3(two_groups ? T2_THREADS : T_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = cs;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  o = n;
  return n;
}

static int attention_impl(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride, const void* kv_cache,
                          int n_layers, int n_pages_total, int layer, const int32_t* page_table, int n_q, int n_kv, int s,
                          int c, int keys_after_c, int max_keys, const int32_t* state, int c_idx, int mode,
                          const uint32_t* anc, int mask_words, int n_splits, float* ws, size_t ws_bytes, int n_req,
                          int req_pages, int req_state, bool keymajor, const int32_t* row_off,
                          const int32_t* row_cnt, bst_stream_t stream) {
  BST_REQUIRE(q && out && kv_cache && page_table, "null pointer argument");
  BST_REQUIRE(n_req >= 1 && (n_req == 1 || (req_pages >= 1 && (state == nullptr || req_state >= 1))),
              "batched attention needs per-request page and state strides");
  BST_REQUIRE(n_kv >= 1 && n_q % n_kv == 0, "n_q must be a multiple of n_kv");
  BST_REQUIRE(s >= 1 && c >= 0 && keys_after_c >= 0, "bad sizes");
  BST_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0 (tree), 1 (causal) or 2 (full)");
  BST_REQUIRE(mode != 0 || (anc && mask_words * 32 >= keys_after_c), "tree mode needs the ancestor mask");
  BST_REQUIRE(!row_off == !row_cnt, "ragged batches need both row offsets and row counts");
  BST_REQUIRE(!row_off || (!keymajor && state), "ragged batches run on the row-major kernels with device contexts");
  if (max_keys < c + keys_after_c) max_keys = c + keys_after_c;
  const int group = n_q / n_kv;
  const int R = group * s;
  const int row_blocks = (R + A_ROWS_PER_CTA - 1) / A_ROWS_PER_CTA;
  const int pages = (max_keys + A_PAGE - 1) / A_PAGE;
  BST_REQUIRE(pages <= n_pages_total, "context exceeds the page table");
  if (n_req > 1) BST_REQUIRE(req_pages >= pages, "request page slice (%d) smaller than the context (%d pages)", req_pages, pages);
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    BST_CUDA(cudaGetDevice(&dev));
    BST_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  }
  const int n_splits_arg = n_splits;
  if (n_splits <= 0) {
    // one wave of CTAs: per-tile work (GQA group x tokens rows against 64 keys)
    // dominates a CTA's fixed cost, so spread the pages over every SM
    int want = n_sm / (n_kv * row_blocks * n_req);
    static int split_cap = -1;  // measurement knob: leave SMs free for the next GEMM's early CTAs
    if (split_cap < 0) split_cap = getenv("BST_ATTN_SPLIT_CAP") ? atoi(getenv("BST_ATTN_SPLIT_CAP")) : 0;
    if (split_cap > 0 && want > split_cap) want = split_cap;
    n_splits = want < 1 ? 1 : want;
  }
  if (n_splits > pages) n_splits = pages;
  int pps = (pages + n_splits - 1) / n_splits;
  pps += pps & 1;  // the default kernel walks 128-key tiles (page pairs)
  n_splits = (pages + pps - 1) / pps;
  if (n_splits > 1) {
    const size_t need = A_WS_CNT_BYTES + (size_t)n_req * n_splits * s * n_q * (A_D + 2) * sizeof(float);
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
  a.cnt = reinterpret_cast<unsigned long long*>(ws);
  a.ws_o = ws ? ws + A_WS_CNT_BYTES / sizeof(float) : nullptr;
  a.ws_ml = ws ? a.ws_o + (size_t)n_req * n_splits * s * n_q * A_D : nullptr;
  a.n_req = n_req;
  a.req_pages = req_pages;
  a.req_state = req_state;
  a.rows_per_block = 128;
  a.row_off = row_off;
  a.row_cnt = row_cnt;
  a.pf = take_prefetch();
  a.seq = bnd_next_seq();
  cudaStream_t st = as_stream(stream);
  if (keymajor) {
    // key-major kernel: row blocks of <= 128 rows balanced over R, one CTA per SM
    const int rbk = (R + 127) / 128;
    const int rpb = (R + rbk - 1) / rbk;
    const int nch = (rpb + 15) / 16;
    a.row_blocks = rbk;
    a.rows_per_block = rpb;
    // split plan.  Global merge (one wave of CTAs over every SM, partials through L2 and
    // a gpu-scope counter barrier) vs cluster merge (the splits of a (head, row block)
    // form one thread-block cluster and merge over DSMEM): per-CTA tile time ~1.2 us,
    // or the HBM share when the grid saturates HBM; the L2 merge chain costs ~6 us,
    // the DSMEM merge ~1 us.  The live context is known on the host only as a bound.
    const int G = n_kv * rbk * n_req;
    const int hint_keys = state ? max_keys : c + keys_after_c;
    const int tiles = ((hint_keys + A_PAGE - 1) / A_PAGE + 1) / 2;
    const double t_tile = 1.2, bw_us = 6.5e6 / 65536.0;  // tiles per us the whole GPU can stream
    auto tile_time = [&](int ctas) { return fmax(t_tile, ctas / bw_us); };
    int splits = 0, merge_mode = 0, cs_best = 0;
    if (n_splits_arg > 0) {
      splits = n_splits_arg;
    } else {
      const int sg = max(1, min(pages, n_sm / G));
      double best = ((tiles + sg - 1) / sg) * tile_time(G * sg) + (sg > 1 ? 6.0 : 0.0);
      splits = sg;
      static int occ[9][4];  // [nch][cs 2, 4, 8] resident clusters (-1: unknown)
      static bool occ_init = false;
      if (!occ_init) {
        for (int i = 0; i < 9; ++i) for (int j = 0; j < 4; ++j) occ[i][j] = -1;
        occ_init = true;
      }
      const int nc8 = nch > 8 ? 8 : nch;
      for (int j = 0; j < 3; ++j) {
        const int cs = 2 << j;
        if (cs > pages) break;
        if (occ[nc8][j] < 0) occ[nc8][j] = kt_cluster_occupancy(nc8, cs);
        if (occ[nc8][j] < G) continue;
        const double tc = ((tiles + cs - 1) / cs) * tile_time(G * cs) + 1.0;
        if (tc < best) { best = tc; splits = cs; cs_best = cs; }
      }
      if (cs_best) merge_mode = 2;
    }
    if (splits > pages) splits = pages;
    if (merge_mode == 2) {
      a.n_splits = cs_best;  // exactly one cluster per (head, row block, request)
      a.pages_per_split = (pages + cs_best - 1) / cs_best;
    } else {
      int pk = (pages + splits - 1) / splits;
      pk += pk & 1;  // 128-key tiles
      a.n_splits = (pages + pk - 1) / pk;
      a.pages_per_split = pk;
    }
    // two workspace banks (counters + partials) alternating with the layer, so back-to-back
    // launches whose CTAs overlap under PDL never share a counter or a partial buffer
    const size_t bank_floats = (size_t)n_req * a.n_splits * s * n_q * (A_D + 2);
    if (a.n_splits > 1 && merge_mode != 2) {
      const size_t need = A_WS_CNT_BYTES + 2 * bank_floats * sizeof(float);
      BST_REQUIRE(ws && ws_bytes >= need, "attention workspace too small: %zu < %zu", ws_bytes, need);
    }
    const int bank = layer & 1;
    if (ws) {
      a.cnt = reinterpret_cast<unsigned long long*>(ws) + bank * (A_WS_CNT_BYTES / 16);
      a.ws_o = ws + A_WS_CNT_BYTES / sizeof(float) + bank * bank_floats;
      a.ws_ml = a.ws_o + (size_t)n_req * a.n_splits * s * n_q * A_D;
    }
    if (merge_mode == 2)
      a.merge = 2;
    else
      a.merge = (a.n_splits > 1 && n_kv * a.n_splits * rbk * n_req <= n_sm &&
                 n_kv * rbk * n_req * sizeof(unsigned long long) <= A_WS_CNT_BYTES / 2) ? 1 : 0;
    static bool kt_attr = false;
    if (!kt_attr) {
#define KT_ATTR(n) BST_CUDA(cudaFuncSetAttribute(attn_kt_kernel<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, kt_smem(n)))
      KT_ATTR(1); KT_ATTR(2); KT_ATTR(3); KT_ATTR(4); KT_ATTR(5); KT_ATTR(6); KT_ATTR(7); KT_ATTR(8);
#undef KT_ATTR
      kt_attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_kv, a.n_splits, rbk * n_req);
    cfg.blockDim = dim3(KT_THREADS);
    cfg.dynamicSmemBytes = kt_smem(nch > 8 ? 8 : nch);
    cfg.stream = st;
    cudaLaunchAttribute lat[2];
    lat[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    lat[0].val.programmaticStreamSerializationAllowed = 1;
    lat[1].id = cudaLaunchAttributeClusterDimension;
    lat[1].val.clusterDim.x = 1;
    lat[1].val.clusterDim.y = a.merge == 2 ? a.n_splits : 1;
    lat[1].val.clusterDim.z = 1;
    cfg.attrs = lat;
    cfg.numAttrs = 2;
    switch (nch) {
      case 1: BST_CUDA(cudaLaunchKernelEx(&cfg, attn_kt_kernel<1>, tm, a)); break;
      case 2: BST_CUDA(cudaLaunchKernelEx(&cfg, attn_kt_kernel<2>, tm, a)); break;
      case 3: BST_CUDA(cudaLaunchKernelEx(&cfg, attn_kt_kernel<3>, tm, a)); break;
      case 4: BST_CUDA(cudaLaunchKernelEx(&cfg, attn_kt_kernel<4>, tm, a)); break;
      case 5: BST_CUDA(cudaLaunchKernelEx(&cfg, attn_kt_kernel<5>, tm, a)); break;
      case 6: BST_CUDA(cudaLaunchKernelEx(&cfg, attn_kt_kernel<6>, tm, a)); break;
      case 7: BST_CUDA(cudaLaunchKernelEx(&cfg, attn_kt_kernel<7>, tm, a)); break;
      default: BST_CUDA(cudaLaunchKernelEx(&cfg, attn_kt_kernel<8>, tm, a)); break;
    }
    if (a.n_splits > 1 && !a.merge)
      BST_CUDA(launch_pdl(attn_combine_kernel, dim3((s * n_q + 7) / 8, n_req), dim3(256), 0, st, a));
    BST_LAUNCH_CHECK();
    return BST_OK;
  }
  static bool attr = false;
  const int smem_tc = T_Q_BYTES + T_STAGES * A_STAGE_BYTES + 1024;
  const int smem_tc2 = T_Q_BYTES + (T2_KS + T2_VS) * A_TILE_BYTES + 2048 + 1024;
  if (!attr) {
    BST_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tc));
    BST_CUDA(cudaFuncSetAttribute(attn_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tc2));
    attr = true;
  }
  if (ws && n_splits > 1) {  // two workspace banks alternating with the layer (see the key-major path)
    const size_t bank_floats = (size_t)n_req * n_splits * s * n_q * (A_D + 2);
    const size_t need = A_WS_CNT_BYTES + 2 * bank_floats * sizeof(float);
    BST_REQUIRE(ws_bytes >= need, "attention workspace too small: %zu < %zu", ws_bytes, need);
    const int bank = layer & 1;
    a.cnt = reinterpret_cast<unsigned long long*>(ws) + bank * (A_WS_CNT_BYTES / 16);
    a.ws_o = ws + A_WS_CNT_BYTES / sizeof(float) + bank * bank_floats;
    a.ws_ml = a.ws_o + (size_t)n_req * n_splits * s * n_q * A_D;
  }
  // row-major kernels, chosen by shape: the single-group kernel for short per-CTA page
  // runs, two alternating softmax groups once a CTA walks >= T2_MIN_PAGES pages (long
  // context; the tc2 kernel on short runs broke the tiny-config exactness)
  bool two_groups = pps >= T2_MIN_PAGES;
  a.merge = (n_splits > 1 && n_kv * n_splits * row_blocks * n_req <= n_sm &&
             n_kv * row_blocks * n_req * sizeof(unsigned long long) <= A_WS_CNT_BYTES / 2) ? 1 : 0;
  // Split merge inside a thread-block cluster over DSMEM when every cluster is co-resident
  // (the largest cluster <= the one-wave split count that fits); taken when it lengthens
  // each CTA's page run by at most 4 pages (~0.65 us each) against the ~3 us it saves.
  // BST_ATTN_CLUSTER=0 disables it (measurement).
#ifndef BST_CLUSTER_SLACK  // measurement builds may override: extra pages per CTA a cluster may cost
#define BST_CLUSTER_SLACK 4
#endif
  static int cl_on = -1;
  if (cl_on < 0) cl_on = getenv("BST_ATTN_CLUSTER") ? atoi(getenv("BST_ATTN_CLUSTER")) : 1;
  if (cl_on && a.merge && n_splits_arg <= 0) {
    const int groups_total = n_kv * row_blocks * n_req;
    for (int ncl = n_splits > T2_CLUSTER_MAX ? T2_CLUSTER_MAX : n_splits; ncl >= 2; --ncl) {
      int pk = (pages + ncl - 1) / ncl;
      pk += pk & 1;
      const int nsc = (pages + pk - 1) / pk;
      const bool tg = pk >= T2_MIN_PAGES;
      if (nsc < 2 || rm_cluster_fits(tg, nsc, tg ? smem_tc2 : smem_tc) < groups_total) continue;
      if (pk - pps <= BST_CLUSTER_SLACK) {
        n_splits = nsc;
        pps = pk;
        two_groups = tg;
        a.n_splits = n_splits;
        a.pages_per_split = pps;
        a.merge = 2;
      }
      break;
    }
  }
  {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_kv, n_splits, row_blocks * n_req);
    cfg.blockDim = dim3(two_groups ? T2_THREADS : T_THREADS);
    cfg.dynamicSmemBytes = two_groups ? smem_tc2 : smem_tc;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 1;
    attr[1].val.clusterDim.y = a.merge == 2 ? n_splits : 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.merge == 2 ? 2 : 1;
    if (two_groups)
      BST_CUDA(cudaLaunchKernelEx(&cfg, attn_tc2_kernel, tm, a));
    else
      BST_CUDA(cudaLaunchKernelEx(&cfg, attn_tc_kernel, tm, a));
  }
  if (n_splits > 1 && !a.merge) {
    const int rows_total = s * n_q;
    BST_CUDA(launch_pdl(attn_combine_kernel, dim3((rows_total + 7) / 8, n_req), dim3(256), 0, st, a));
  }
  BST_LAUNCH_CHECK();
  return BST_OK;
}

}  // namespace bst

extern "C" int bst_attention(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride, const void* kv_cache,
                             int n_layers, int n_pages_total, int layer, const int32_t* page_table, int n_q, int n_kv,
                             int s, int c, int keys_after_c, int max_keys, const int32_t* state, int c_idx, int mode,
                             const uint32_t* anc, int mask_words, int n_splits, float* ws, size_t ws_bytes,
                             bst_stream_t stream) {
  return bst::attention_impl(q, q_tok_stride, out, o_tok_stride, kv_cache, n_layers, n_pages_total, layer, page_table,
                             n_q, n_kv, s, c, keys_after_c, max_keys, state, c_idx, mode, anc, mask_words, n_splits,
                             ws, ws_bytes, 1, 0, 0, false, nullptr, nullptr, stream);
}

extern "C" int bst_attention_keymajor(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride,
                                      const void* kv_cache, int n_layers, int n_pages_total, int layer,
                                      const int32_t* page_table, int n_q, int n_kv, int s, int c, int keys_after_c,
                                      int max_keys, const int32_t* state, int c_idx, int mode, const uint32_t* anc,
                                      int mask_words, int n_splits, float* ws, size_t ws_bytes,
                                      bst_stream_t stream) {
  return bst::attention_impl(q, q_tok_stride, out, o_tok_stride, kv_cache, n_layers, n_pages_total, layer, page_table,
                             n_q, n_kv, s, c, keys_after_c, max_keys, state, c_idx, mode, anc, mask_words, n_splits,
                             ws, ws_bytes, 1, 0, 0, true, nullptr, nullptr, stream);
}

extern "C" int bst_attention_batch(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride,
                                   const void* kv_cache, int n_layers, int n_pages_total, int layer,
                                   const int32_t* page_table, int req_pages, int n_q, int n_kv, int n_req, int s,
                                   int keys_after_c, int max_keys, const int32_t* state, int req_state, int c_idx,
                                   int mode, const uint32_t* anc, int mask_words, int n_splits, float* ws,
                                   size_t ws_bytes, bst_stream_t stream) {
  return bst::attention_impl(q, q_tok_stride, out, o_tok_stride, kv_cache, n_layers, n_pages_total, layer, page_table,
                             n_q, n_kv, s, 0, keys_after_c, max_keys, state, c_idx, mode, anc, mask_words, n_splits,
                             ws, ws_bytes, n_req, req_pages, req_state, false, nullptr, nullptr, stream);
}

extern "C" int bst_attention_ragged(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride,
                                    const void* kv_cache, int n_layers, int n_pages_total, int layer,
                                    const int32_t* page_table, int req_pages, int n_q, int n_kv, int n_req,
                                    int s_max, const int32_t* row_off, const int32_t* row_cnt, int keys_after_c,
                                    int max_keys, const int32_t* state, int req_state, int c_idx, int mode,
                                    const uint32_t* anc, int mask_words, int n_splits, float* ws, size_t ws_bytes,
                                    bst_stream_t stream) {
  BST_REQUIRE(row_off && row_cnt, "null row offsets / counts");
  return bst::attention_impl(q, q_tok_stride, out, o_tok_stride, kv_cache, n_layers, n_pages_total, layer, page_table,
                             n_q, n_kv, s_max, 0, keys_after_c, max_keys, state, c_idx, mode, anc, mask_words, n_splits,
                             ws, ws_bytes, n_req, req_pages, req_state, false, row_off, row_cnt, stream);
}

extern "C" size_t bst_attention_workspace(int n_q, int s, int n_splits) {  // two banks of partials
  return bst::A_WS_CNT_BYTES + 2 * (size_t)(n_splits < 1 ? 1 : n_splits) * s * n_q * (128 + 2) * sizeof(float);
}

extern "C" int bst_debug_attn_trace_cta(int y) {
  BST_CUDA(cudaMemcpyToSymbol(bst::g_attn_trace_y, &y, sizeof(int)));
  return BST_OK;
}

extern "C" int bst_debug_attn_trace(void* buf) {
  BST_CUDA(cudaMemcpyToSymbol(bst::g_attn_trace, &buf, sizeof(void*)));
  return BST_OK;
}

// debug: how many clusters of `cluster` attention CTAs (dynamic smem `smem`) fit at once
extern "C" int bst_debug_cluster_occupancy(int cluster, int smem) {
  using namespace bst;
  BST_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  BST_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(8, cluster, 1);
  cfg.blockDim = dim3(T_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = cluster;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  BST_CUDA(cudaOccupancyMaxActiveClusters(&n, attn_tc_kernel, &cfg));
  return n;
}

// debug: clusters of `cluster` key-major attention CTAs (dynamic smem `smem`) resident at once
extern "C" int bst_debug_cluster_occupancy_kt(int cluster, int smem) {
  using namespace bst;
  BST_CUDA(cudaFuncSetAttribute(attn_kt_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));  // probe only
  BST_CUDA(cudaFuncSetAttribute(attn_kt_kernel<5>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(8, cluster, 1);
  cfg.blockDim = dim3(KT_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = cluster;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  BST_CUDA(cudaOccupancyMaxActiveClusters(&n, attn_kt_kernel<5>, &cfg));
  return n;
}

extern "C" int bst_debug_kt_ablate(int v) {
  BST_CUDA(cudaMemcpyToSymbol(bst::g_kt_ablate, &v, sizeof(int)));
  return BST_OK;
}

extern "C" int bst_debug_bnd_trace_attn(void* buf) {  // BST_TRACE builds only
#ifdef BST_TRACE
  BST_CUDA(cudaMemcpyToSymbol(bst::g_bnd, &buf, sizeof(void*)));
  return BST_OK;
#else
  (void)buf;
  return BST_EINVAL;
#endif
}

// debug: resident clusters of `cs` two-group attention CTAs at the kernel's shared memory
extern "C" int bst_debug_tc2_cluster_fits(int cs) {
  using namespace bst;
  const int smem_tc2 = T_Q_BYTES + (T2_KS + T2_VS) * A_TILE_BYTES + 2048 + 1024;
  return rm_cluster_fits(true, cs, smem_tc2);
}
