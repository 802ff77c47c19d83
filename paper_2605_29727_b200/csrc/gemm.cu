// K4 — weight-streaming bf16 GEMM on tcgen05 (TMA -> smem ring -> UMMA -> TMEM).
//
//   Y[m, n_out] = X[m, K] . W[n_out, K]^T        (nn.Linear, W row-major)
//
// Verify-time GEMMs are skinny (m = s = N+1 <= 256 tokens) and read every
// weight byte exactly once, so the kernel is built around HBM streaming:
// "swap AB" — the weight tile is the 128-row UMMA A operand, the token tile
// the N operand (N = round_up(m, 16) <= 256), the accumulator is 128 lanes x N
// fp32 columns of TMEM.  Work = (m_tile, k_block) units split evenly over one
// persistent CTA per SM (stream-K): a CTA covers a contiguous unit range, so a
// tile is shared by at most a few CTAs; each writes its fp32 partial to its
// own slot and the consumer kernel (residual/norm/SwiGLU/argmax epilogue)
// reduces the slots in fixed order — deterministic, no atomics.
//
// Roles per CTA (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner +
// single-thread UMMA issuer, warps 2-5 = epilogue (TMEM -> registers -> L2).
// The TMEM accumulator is double buffered so the next segment's MMAs overlap
// the previous segment's epilogue.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"

namespace bst {

constexpr int G_THREADS = 192;
constexpr int G_BM = 128;
constexpr int G_BK = 64;
constexpr int G_TILE_W = G_BM * G_BK * 2;  // 16 KiB
constexpr int G_MAX_STAGES = 12;
// one-CTA ring budget by token columns (leaves room for a co-resident epilogue CTA under PDL
// overlap): 160 KiB, except 176 KiB for 49..112 columns and 200 KiB at 128 — measured in the
// verify graph at 32 / 48 / 96 / 128 / 256 rows (BST_GEMM_SMEM_KB sweeps 128..200): 96 rows
// 4.01-4.04 -> 3.96-3.98 ms, 128 rows 4.38-4.42 -> 4.25 ms; 32 / 48 rows and the drafter's
// 17 / 34 rows equal or best at 160, the one-CTA launches at 256 rows slower above 160
constexpr int G_SMEM_BUDGET = 160 * 1024;
__host__ __forceinline__ int gemm_smem_budget(int bn) {
  return bn <= 48 || bn > 128 ? G_SMEM_BUDGET : (bn < 128 ? 176 * 1024 : 200 * 1024);
}
constexpr int G_SMEM_BUDGET_PAIR = 200 * 1024;  // pair mode: 3 stages of 2 weight tiles + a 256-row X block

// ------------------------------------------------------------ tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::mutex g_mu;

static int get_encoder() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_encode) return BST_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable: %s", cudaGetErrorString(e));
    return BST_ECUDA;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return BST_OK;
}

// 2-D bf16 tensor [rows, cols] (row stride in elements), box = box_rows x 64, 128B swizzle.
int make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t row_stride,
                   uint32_t box_rows, uint32_t box_cols) {
  int rc = get_encoder();
  if (rc) return rc;
  BST_REQUIRE(((uintptr_t)ptr & 15) == 0, "TMA base pointer must be 16-byte aligned");
  BST_REQUIRE((row_stride * 2) % 16 == 0, "TMA row stride must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu box=%ux%u", (int)r,
              (unsigned long long)rows, (unsigned long long)cols, box_rows, box_cols);
    return BST_ECUDA;
  }
  return BST_OK;
}

// Tensor-map cache keyed by (ptr, rows, cols, stride, box): weights are encoded once.
struct MapKey {
  uintptr_t ptr;
  uint64_t rows, cols, stride;
  uint32_t br, bc;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && stride == o.stride && br == o.br && bc == o.bc;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<uintptr_t>()(k.ptr) ^ (k.rows * 1315423911u) ^ (k.cols << 7) ^ (k.stride << 13) ^
           ((uint64_t)k.br << 29) ^ ((uint64_t)k.bc << 41);
  }
};
static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

int cached_tmap(CUtensorMap* out, const void* ptr, uint64_t rows, uint64_t cols, uint64_t stride, uint32_t br,
                uint32_t bc) {
  MapKey key{(uintptr_t)ptr, rows, cols, stride, br, bc};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return BST_OK;
    }
  }
  int rc = make_tmap_bf16(out, ptr, rows, cols, stride, br, bc);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps[key] = *out;
  return BST_OK;
}

// ------------------------------------------------------------------ kernel
__device__ long long* g_gemm_trace = nullptr;  // debug: globaltimer stamps of CTA g_trace_cta
__device__ int g_trace_cta = 0;
__device__ __forceinline__ void gtrace(int k) {
#ifdef BST_TRACE  // phase tracing (scripts/gemm_trace.py); compiled out by default
  if (g_gemm_trace && blockIdx.x == g_trace_cta && k < 64) {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_gemm_trace[k] = t;
  }
#else
  (void)k;
#endif
}

BST_BND_TRACE_DEF

struct Seg {
  int tile, kb_lo, kb_hi, slot;  // tile = super-tile index (first weight tile = tile * TP)
};

__device__ __forceinline__ bool next_seg(const bst_gemm_sched_t& s, int64_t& u, int64_t u1, Seg& seg) {
  if (u >= u1) return false;
  seg.tile = (int)(u / s.n_kb);
  seg.kb_lo = (int)(u % s.n_kb);
  { const int64_t lim = (int64_t)seg.kb_lo + (u1 - u); seg.kb_hi = (int)(lim < s.n_kb ? lim : s.n_kb); }
  seg.slot = (int)blockIdx.x - sched_first_st(s, seg.tile);
  u += seg.kb_hi - seg.kb_lo;
  return true;
}

// TP = weight tiles per unit.  TP = 2 (m > 128): each stage holds two 128-row weight
// tiles and one X k-block, and the issuer runs two MMAs into two TMEM accumulators,
// halving the X re-reads from L2 per weight byte (profiles/r1_gemm_m256_tensor.txt).
template <int TP>
__global__ void __launch_bounds__(G_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                     bst_gemm_sched_t s, float* __restrict__ partial, int stages, int trigger) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[G_MAX_STAGES], empty[G_MAX_STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) gtrace(0);
  if (threadIdx.x == 0) BND(s.reserved, 0);
  if (threadIdx.x == 0 && blockIdx.x == 0) BND_KIND(s.reserved, 1000000ull + s.n_out);
  if (trigger) sm100::grid_dep_launch();
  const uint32_t base = (sm100::smem_u32(smem_raw) + 1023) & ~1023u;
  uint8_t* smem = smem_raw + (base - sm100::smem_u32(smem_raw));
  const int bn = s.bn;
  const uint32_t x_bytes = (uint32_t)bn * G_BK * 2;
  const uint32_t stage_bytes = TP * G_TILE_W + x_bytes;
  const uint32_t tcols = s.tmem_cols;
  // accumulator buffers: two when 2 * TP * bn columns fit in the allocation
  const int nacc = (int)tcols >= 2 * TP * bn ? 2 : 1;

  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tmW);
    sm100::prefetch_tmap(&tmX);
    for (int i = 0; i < stages; ++i) { sm100::mbar_init(&full[i], 1); sm100::mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { sm100::mbar_init(&tfull[i], 1); sm100::mbar_init(&tempty[i], 4); }
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc(&tmem_base_sh, tcols);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  if (threadIdx.x == 0) gtrace(1);

  const int64_t u0 = (int64_t)blockIdx.x * s.units / s.grid;
  const int64_t u1 = (int64_t)(blockIdx.x + 1) * s.units / s.grid;

  if (warp == 0) {
    // ---------------- TMA producer
    // PDL: the weight tiles of the first `stages` k-blocks do not depend on the
    // previous kernel, so they are issued before griddepcontrol.wait; the X
    // (activation) tiles are issued only after the dependency resolves.
    if (lane == 0) {
      const uint64_t pol_w = sm100::policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      int64_t u = u0;
      Seg seg;
      int issued = 0;
      // weight tiles of super-tile st present in the matrix (the last one may be short)
      auto ntiles = [&](int st) { return TP == 1 ? 1 : (st * TP + 1 < s.n_mt ? 2 : 1); };
      auto load_w = [&](uint8_t* sw, uint64_t* bar, int kb, int st, int nt) {
        for (int t = 0; t < nt; ++t)
          sm100::tma_load_2d_hint(sw + t * G_TILE_W, &tmW, bar, kb * G_BK, (st * TP + t) * G_BM, pol_w);
      };
      // pass 1: prologue weights
      {
        int64_t uu = u0;
        Seg sg;
        int st = 0;
        while (st < stages && next_seg(s, uu, u1, sg)) {
          const int nt = ntiles(sg.tile);
          for (int kb = sg.kb_lo; kb < sg.kb_hi && st < stages; ++kb, ++st) {
            uint8_t* sw = smem + st * stage_bytes;
            sm100::mbar_add_tx(&full[st], nt * G_TILE_W);
            load_w(sw, &full[st], kb, sg.tile, nt);
          }
        }
        issued = st;
      }
      gtrace(2);
      sm100::grid_dep_wait();
      gtrace(3);
      BND(s.reserved, 2);
      BND(s.reserved, 3);
      int idx = 0;
      while (next_seg(s, u, u1, seg)) {
        const int nt = ntiles(seg.tile);
        for (int kb = seg.kb_lo; kb < seg.kb_hi; ++kb, ++idx) {
          uint8_t* sw = smem + stage * stage_bytes;
          if (idx < issued) {  // weights already in flight: add the X tile and arrive
            sm100::mbar_expect_tx(&full[stage], x_bytes);
          } else {
            sm100::mbar_wait(&empty[stage], phase ^ 1);
            sm100::mbar_expect_tx(&full[stage], nt * G_TILE_W + x_bytes);
            load_w(sw, &full[stage], kb, seg.tile, nt);
          }
          sm100::tma_load_2d(sw + TP * G_TILE_W, &tmX, &full[stage], kb * G_BK, 0);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- UMMA issuer
    const uint32_t idesc = sm100::idesc_bf16(G_BM, bn);
    int stage = 0;
    uint32_t phase = 0;
    int64_t u = u0;
    Seg seg;
    int j = 0;
    while (next_seg(s, u, u1, seg)) {
      const int acc = nacc == 2 ? (j & 1) : 0;
      const int use = nacc == 2 ? (j >> 1) : j;
      const int nt = TP == 1 ? 1 : (seg.tile * TP + 1 < s.n_mt ? 2 : 1);
      sm100::mbar_wait(&tempty[acc], (use & 1) ^ 1);
      sm100::tc_fence_after();
      const uint32_t d = tmem + acc * TP * bn;
      for (int kb = seg.kb_lo; kb < seg.kb_hi; ++kb) {
        sm100::mbar_wait(&full[stage], phase);
        if (lane == 0) gtrace(8 + (kb - seg.kb_lo) + j * 24);
        sm100::tc_fence_after();
        if (sm100::elect_one()) {
          const uint32_t a_addr = base + stage * stage_bytes;
          const uint64_t bdesc = sm100::desc_k_sw128(a_addr + TP * G_TILE_W);
#pragma unroll
          for (int t = 0; t < TP; ++t) {
            if (t < nt) {
              const uint64_t adesc = sm100::desc_k_sw128(a_addr + t * G_TILE_W);
#pragma unroll
              for (int k = 0; k < G_BK / 16; ++k)  // +32 B per K=16 step inside the 128B swizzle atom
                sm100::umma_f16(d + t * bn, adesc + 2 * k, bdesc + 2 * k, idesc,
                                (kb > seg.kb_lo || k > 0) ? 1u : 0u);
            }
          }
          sm100::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
      if (sm100::elect_one()) sm100::umma_commit(&tfull[acc]);
      __syncwarp();
      ++j;
    }
  } else {
    // ---------------- epilogue: TMEM -> fp32 partial slot
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    int64_t u = u0;
    Seg seg;
    int j = 0;
    while (next_seg(s, u, u1, seg)) {
      const int acc = nacc == 2 ? (j & 1) : 0;
      const int use = nacc == 2 ? (j >> 1) : j;
      const int nt = TP == 1 ? 1 : (seg.tile * TP + 1 < s.n_mt ? 2 : 1);
      sm100::mbar_wait(&tfull[acc], use & 1);
      sm100::tc_fence_after();
      for (int t = 0; t < nt; ++t) {
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (acc * TP + t) * bn;
        float* dst = partial + ((int64_t)((seg.tile * TP + t) * s.s_max + seg.slot) * bn) * G_BM + row;
        for (int c0 = 0; c0 < bn; c0 += 16) {
          float v[16];
          sm100::tmem_ld16(taddr + c0, v);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i < s.m) dst[(int64_t)(c0 + i) * G_BM] = v[i];
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (lane == 0 && quad == 0) gtrace(4 + j);
      ++j;
    }
  }
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, tcols);
  }
  if (threadIdx.x == 0) gtrace(7);
  if (threadIdx.x == 0) BND(s.reserved, 1);
}

// CTA-pair variant (s.cta2, m > 128 on even tile counts): a cluster of two CTAs owns
// a 256-row weight super-tile; tcgen05.mma.cta_group::2 (M = 256, N = bn) reads the
// weights split along M (128 rows per CTA) and the X k-block split along N (bn / 2
// token rows per CTA), so each SM ingests 16 KiB of weights + bn / 2 x 128 B of X per
// k-block instead of the full X block: half the L2 -> SM traffic of the one-CTA kernel
// at full tensor rate.  Stream-K runs over pairs (s.grid = number of pairs); each CTA
// writes the partial of its own 128-row tile.  Only rank 0 issues MMAs; both CTAs load.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G_THREADS, 1)
    gemm_bf16_2cta_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                          bst_gemm_sched_t s, float* __restrict__ partial, int stages, int trigger) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[G_MAX_STAGES], empty[G_MAX_STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (trigger) sm100::grid_dep_launch();
  const uint32_t rank = sm100::cluster_ctarank();
  const int pair = (int)blockIdx.x >> 1;
  const uint32_t base = (sm100::smem_u32(smem_raw) + 1023) & ~1023u;
  uint8_t* smem = smem_raw + (base - sm100::smem_u32(smem_raw));
  // bn > 256: two N chunks of bn / 2 token columns; each CTA loads the rank's half of each
  const int bn = s.bn, nch = bn > 256 ? 2 : 1, cn = bn / nch, hn = cn >> 1;
  const uint32_t xh_bytes = (uint32_t)(nch * hn) * G_BK * 2;
  const uint32_t stage_bytes = G_TILE_W + xh_bytes;
  const uint32_t tcols = s.tmem_cols;
  const int nacc = (int)tcols >= 2 * bn ? 2 : 1;

  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tmW);
    sm100::prefetch_tmap(&tmX);
    for (int i = 0; i < stages; ++i) { sm100::mbar_init(&full[i], 1); sm100::mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { sm100::mbar_init(&tfull[i], 1); sm100::mbar_init(&tempty[i], 8); }
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc2(&tmem_base_sh, tcols);
  sm100::tc_fence_before();
  sm100::cluster_sync();  // barriers of both CTAs initialised before any remote arrival
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  const int64_t u0 = (int64_t)pair * s.units / s.grid;
  const int64_t u1 = (int64_t)(pair + 1) * s.units / s.grid;
  auto seg_next = [&](int64_t& u, Seg& seg) {
    if (u >= u1) return false;
    seg.tile = (int)(u / s.n_kb);
    seg.kb_lo = (int)(u % s.n_kb);
    const int64_t lim = (int64_t)seg.kb_lo + (u1 - u);
    seg.kb_hi = (int)(lim < s.n_kb ? lim : s.n_kb);
    seg.slot = pair - sched_first_st(s, seg.tile);
    u += seg.kb_hi - seg.kb_lo;
    return true;
  };

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs): own weight half + own X half
    if (lane == 0) {
      const uint64_t pol_w = sm100::policy_evict_first(), pol_x = sm100::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int64_t u = u0;
      Seg seg;
      int issued = 0;
      {
        int64_t uu = u0;
        Seg sg;
        int st = 0;
        while (st < stages && seg_next(uu, sg)) {
          for (int kb = sg.kb_lo; kb < sg.kb_hi && st < stages; ++kb, ++st) {
            if (rank == 0) sm100::mbar_add_tx(&full[st], 2 * G_TILE_W);
            sm100::tma_load_2d_2cta(smem + st * stage_bytes, &tmW, &full[st], kb * G_BK,
                                    (sg.tile * 2 + (int)rank) * G_BM, pol_w);
          }
        }
        issued = st;
      }
      sm100::grid_dep_wait();
      int idx = 0;
      while (seg_next(u, seg)) {
        for (int kb = seg.kb_lo; kb < seg.kb_hi; ++kb, ++idx) {
          uint8_t* sw = smem + stage * stage_bytes;
          if (idx >= issued) {
            sm100::mbar_wait(&empty[stage], phase ^ 1);
            if (rank == 0) sm100::mbar_add_tx(&full[stage], 2 * G_TILE_W);
            sm100::tma_load_2d_2cta(sw, &tmW, &full[stage], kb * G_BK, (seg.tile * 2 + (int)rank) * G_BM, pol_w);
          }
          if (rank == 0) sm100::mbar_expect_tx(&full[stage], 2 * xh_bytes);  // the leader's arrival
          for (int c = 0; c < nch; ++c)
            sm100::tma_load_2d_2cta(sw + G_TILE_W + c * hn * 128, &tmX, &full[stage], kb * G_BK, c * cn + (int)rank * hn,
                                    pol_x);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- UMMA issuer (leader only)
    if (rank == 0) {
      const uint32_t idesc = sm100::idesc_bf16(2 * G_BM, cn);
      int stage = 0;
      uint32_t phase = 0;
      int64_t u = u0;
      Seg seg;
      int j = 0;
      while (seg_next(u, seg)) {
        const int acc = nacc == 2 ? (j & 1) : 0;
        const int use = nacc == 2 ? (j >> 1) : j;
        sm100::mbar_wait_cluster(&tempty[acc], (use & 1) ^ 1);
        sm100::tc_fence_after();
        const uint32_t d = tmem + acc * bn;
        for (int kb = seg.kb_lo; kb < seg.kb_hi; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          if (sm100::elect_one()) {
            const uint32_t a_addr = base + stage * stage_bytes;
            const uint64_t adesc = sm100::desc_k_sw128(a_addr);
            for (int c = 0; c < nch; ++c) {
              const uint64_t bdesc = sm100::desc_k_sw128(a_addr + G_TILE_W + c * hn * 128);
#pragma unroll
              for (int k = 0; k < G_BK / 16; ++k)
                sm100::umma_f16_2cta(d + c * cn, adesc + 2 * k, bdesc + 2 * k, idesc,
                                     (kb > seg.kb_lo || k > 0) ? 1u : 0u);
            }
            sm100::umma_commit_2cta(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
        if (sm100::elect_one()) sm100::umma_commit_2cta(&tfull[acc], 0x3);
        __syncwarp();
        ++j;
      }
    }
  } else {
    // ---------------- epilogue (both CTAs): TMEM -> fp32 partial slot of the own tile
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    int64_t u = u0;
    Seg seg;
    int j = 0;
    while (seg_next(u, seg)) {
      const int acc = nacc == 2 ? (j & 1) : 0;
      const int use = nacc == 2 ? (j >> 1) : j;
      sm100::mbar_wait(&tfull[acc], use & 1);
      sm100::tc_fence_after();
      const int tile = seg.tile * 2 + (int)rank;
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + acc * bn;
      float* dst = partial + ((int64_t)(tile * s.s_max + seg.slot) * bn) * G_BM + row;
      for (int c0 = 0; c0 < bn; c0 += 16) {
        float v[16];
        sm100::tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c0 + i < s.m) dst[(int64_t)(c0 + i) * G_BM] = v[i];
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_remote(&tempty[acc], 0);
      ++j;
    }
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();  // both CTAs done with TMEM and with remote barriers
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc2(tmem, tcols);
  }
}

// ------------------------------------------------------ reduction kernels
__global__ void gemm_reduce_kernel(const float* __restrict__ partial, bst_gemm_sched_t s, float* y_f32,
                                   __nv_bfloat16* y_bf16, int64_t ldy) {
  pdl_enter();
  const int t = blockIdx.y;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g * 4 < s.n_out; g += gridDim.x * blockDim.x) {
    const int n0 = g * 4;
    if (n0 + 4 <= s.n_out) {
      const float4 v = gemm_load4(partial, s, t, n0);
      const float vv[4] = {v.x, v.y, v.z, v.w};
      for (int e = 0; e < 4; ++e) {
        if (y_f32) y_f32[(int64_t)t * ldy + n0 + e] = vv[e];
        if (y_bf16) y_bf16[(int64_t)t * ldy + n0 + e] = __float2bfloat16(vv[e]);
      }
    } else {
      for (int n = n0; n < s.n_out; ++n) {
        const float v = gemm_load(partial, s, t, n);
        if (y_f32) y_f32[(int64_t)t * ldy + n] = v;
        if (y_bf16) y_bf16[(int64_t)t * ldy + n] = __float2bfloat16(v);
      }
    }
  }
}

// Per-token argmax over the full output width, lowest index on ties (np.argmax).
// vocab_offset: global index of output column 0 (vocab-parallel LM head shards).
__global__ void gemm_argmax_kernel(const float* __restrict__ partial, bst_gemm_sched_t s,
                                   unsigned long long* best, int vocab_offset = 0) {
  pdl_enter();
  const int t = blockIdx.y;
  unsigned long long key = 0;
  auto consider = [&](float v, int n) {
    unsigned int b = __float_as_uint(v);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    const unsigned long long k = ((unsigned long long)b << 32) | (0xFFFFFFFFu - (unsigned)(n + vocab_offset));
    key = k > key ? k : key;
  };
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g * 4 < s.n_out; g += gridDim.x * blockDim.x) {
    const int n0 = g * 4;
    if (n0 + 4 <= s.n_out) {
      const float4 v = gemm_load4(partial, s, t, n0);
      consider(v.x, n0);
      consider(v.y, n0 + 1);
      consider(v.z, n0 + 2);
      consider(v.w, n0 + 3);
    } else {
      for (int n = n0; n < s.n_out; ++n) consider(gemm_load(partial, s, t, n), n);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
    key = ok > key ? ok : key;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(best + t, key);
}

// ---- temperature sampling (T > 0): Gumbel-max over logits / T.  The noise of vocabulary
// entry n at row t is Philox4x32-10 keyed by the request seed with counter (n / 4,
// absolute position c + pos[t]), so a sample is a function of (seed, position, logits):
// the tree row of a node at depth d and the autoregressive step at the same position draw
// the same noise, and tree decode reproduces sampled AR decode exactly (the sampled
// analogue of greedy output preservation, exact-match verification verify_sim.py:111-126).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = c.x * 0xD2511F53u, hi0 = __umulhi(c.x, 0xD2511F53u);
    const uint32_t lo1 = c.z * 0xCD9E8D57u, hi1 = __umulhi(c.z, 0xCD9E8D57u);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
__device__ __forceinline__ float gumbel_of(uint32_t x) {
  const float u = (float)(x >> 8) * 5.9604645e-8f + 2.9802322e-8f;  // (0, 1)
  return -__logf(-__logf(u));
}
__global__ void gemm_sample_kernel(const float* __restrict__ partial, bst_gemm_sched_t s, unsigned long long* best,
                                   const int32_t* __restrict__ pos, const int32_t* __restrict__ state, int c_idx,
                                   float inv_t, uint2 seed) {
  pdl_enter();
  const int t = blockIdx.y;
  const uint32_t apos = (uint32_t)((state ? state[c_idx] : 0) + pos[t]);
  unsigned long long key = 0;
  auto consider = [&](float v, int n) {
    unsigned int b = __float_as_uint(v);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    const unsigned long long k = ((unsigned long long)b << 32) | (0xFFFFFFFFu - (unsigned)n);
    key = k > key ? k : key;
  };
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g * 4 < s.n_out; g += gridDim.x * blockDim.x) {
    const int n0 = g * 4;
    const uint4 r = philox4x32_10(make_uint4((uint32_t)g, apos, 0u, 0u), seed);
    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
    if (n0 + 4 <= s.n_out) {
      const float4 v = gemm_load4(partial, s, t, n0);
      consider(fmaf(v.x, inv_t, gumbel_of(rr[0])), n0);
      consider(fmaf(v.y, inv_t, gumbel_of(rr[1])), n0 + 1);
      consider(fmaf(v.z, inv_t, gumbel_of(rr[2])), n0 + 2);
      consider(fmaf(v.w, inv_t, gumbel_of(rr[3])), n0 + 3);
    } else {
      for (int n = n0; n < s.n_out; ++n) consider(fmaf(gemm_load(partial, s, t, n), inv_t, gumbel_of(rr[n - n0])), n);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
    key = ok > key ? ok : key;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(best + t, key);
}

__global__ void argmax_finalize_kernel(const unsigned long long* best, int m, int32_t* out) {
  pdl_enter();
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) out[t] = (int32_t)(0xFFFFFFFFu - (unsigned)(best[t] & 0xFFFFFFFFull));
}
// packed keys <-> signed int64 (flip the top bit) so a signed MAX all-reduce (NCCL int64)
// orders them exactly as the unsigned comparison above
__global__ void argmax_key_flip_kernel(unsigned long long* keys, int m) {
  pdl_enter();
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) keys[t] ^= 0x8000000000000000ull;
}
__global__ void argmax_from_signed_kernel(const unsigned long long* keys, int m, int32_t* out) {
  pdl_enter();
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) out[t] = (int32_t)(0xFFFFFFFFu - (unsigned)(keys[t] & 0xFFFFFFFFull));
}

}  // namespace bst

// ---------------------------------------------------------------- C ABI
extern "C" int bst_gemm_schedule(int n_out, int k, int m, int grid, bst_gemm_sched_t* out) {
  using namespace bst;
  BST_REQUIRE(out, "null schedule");
  BST_REQUIRE(n_out >= 1 && k >= 1, "bad GEMM shape n_out=%d k=%d", n_out, k);
  BST_REQUIRE(m >= 1 && m <= 512, "m must be in [1, 512] (got %d); chunk larger batches", m);
  BST_REQUIRE(k % 8 == 0, "K must be a multiple of 8 (16-byte TMA rows), got %d", k);
  bst_gemm_sched_t s{};
  s.n_out = n_out;
  s.k = k;
  s.m = m;
  s.bn = m > 256 ? ((m + 31) / 32) * 32 : ((m + 15) / 16) * 16;  // > 256: two N chunks of bn / 2
  s.n_mt = (n_out + G_BM - 1) / G_BM;
  s.n_kb = (k + G_BK - 1) / G_BK;
  if (grid <= 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = sms;
  }
  // two weight tiles per unit above pair_min_bn token columns (BST_GEMM_PAIR_MIN_BN:
  // measurement knob, 0 disables)
  static int pair_min_bn = -1;
  if (pair_min_bn < 0) {
    const char* e = getenv("BST_GEMM_PAIR_MIN_BN");
    pair_min_bn = e ? atoi(e) : 144;
  }
  // pair mode loses TMEM double buffering at bn > 128 and doubles each CTA's partial
  // tile, so it only pays when every CTA streams at least one full tile (n_mt >= grid)
  // (very wide outputs, e.g. the LM head's 1187 tiles, already pay from bn = 96)
  s.pair = (pair_min_bn > 0 && ((s.bn >= pair_min_bn && s.n_mt >= grid) ||
                                (s.bn >= 96 && s.bn >= pair_min_bn / 2 && s.n_mt >= 4 * grid))) ? 2 : 1;
  // CTA-pair mode (cta_group::2) for m > 128 on even tile counts (BST_GEMM_2CTA=0/1)
  static int cta2_on = -1;
  if (cta2_on < 0) cta2_on = getenv("BST_GEMM_2CTA") ? atoi(getenv("BST_GEMM_2CTA")) : 1;
  s.cta2 = (cta2_on && s.bn >= 144 && s.n_mt % 2 == 0 && grid >= 2) ? 1 : 0;
  if (s.cta2) {
    s.pair = 2;
    grid /= 2;  // stream-K over CTA pairs
  }
  BST_REQUIRE(m <= 256 || s.cta2, "m > 256 needs the CTA-pair kernel (even tile count, got n_out=%d m=%d)", n_out, m);
  s.units = (int64_t)((s.n_mt + s.pair - 1) / s.pair) * s.n_kb;
  s.grid = (int)(s.units < grid ? s.units : grid);
  int smax = 1;
  for (int t = 0; t < s.n_mt; ++t) {
    int c = sched_last_cta(s, t) - sched_first_cta(s, t) + 1;
    smax = c > smax ? c : smax;
  }
  s.s_max = smax;
  int tc = 32;
  while (tc < 2 * (s.cta2 ? 1 : s.pair) * s.bn && tc < 512) tc <<= 1;  // double buffered when it fits
  if (tc < s.bn) tc = 512;
  s.tmem_cols = tc;
  const int stage_bytes = s.cta2 ? G_TILE_W + (s.bn / 2) * G_BK * 2 : s.pair * G_TILE_W + s.bn * G_BK * 2;
  static int budget_env = -1, budget_pair = 0;
  if (budget_env < 0) {
    const char* e = getenv("BST_GEMM_SMEM_KB");  // measurement knobs
    budget_env = e ? atoi(e) * 1024 : 0;
    e = getenv("BST_GEMM_PAIR_SMEM_KB");
    budget_pair = e ? atoi(e) * 1024 : G_SMEM_BUDGET_PAIR;
  }
  const int budget = budget_env > 0 ? budget_env : gemm_smem_budget(s.bn);
  // pair and CTA-pair modes (m > 128): deeper weight prefetch, no co-resident epilogue needed
  int stages = ((s.pair == 2 ? budget_pair : budget) - 1024) / stage_bytes;
  BST_REQUIRE(stages >= 2, "GEMM smem budget too small for two stages");
  s.stages = stages > G_MAX_STAGES ? G_MAX_STAGES : stages;
  s.partial_floats = (int64_t)s.n_mt * s.s_max * s.bn * G_BM;
  *out = s;
  return BST_OK;
}

extern "C" int bst_gemm(const void* w, const void* x, int64_t ld_x, const bst_gemm_sched_t* sched, float* partial,
                        size_t partial_bytes, bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(w && x && sched && partial, "null pointer argument");
  bst_gemm_sched_t s = *sched;
  s.reserved = bnd_next_seq();
  BST_REQUIRE(partial_bytes >= (size_t)s.partial_floats * sizeof(float), "partial buffer too small");
  BST_REQUIRE(ld_x >= s.k, "ld_x < K");
  BST_REQUIRE(s.pair == 1 || s.pair == 2, "bad schedule (pair=%d)", s.pair);
  if (s.cta2) {
    CUtensorMap tw2, tx2;
    int rc2 = cached_tmap(&tw2, w, (uint64_t)s.n_out, (uint64_t)s.k, (uint64_t)s.k, G_BM, G_BK);
    if (rc2) return rc2;
    rc2 = make_tmap_bf16(&tx2, x, (uint64_t)s.m, (uint64_t)s.k, (uint64_t)ld_x,
                         (uint32_t)(s.bn > 256 ? s.bn / 4 : s.bn / 2), G_BK);
    if (rc2) return rc2;
    const int smem2 = s.stages * (G_TILE_W + (s.bn / 2) * G_BK * 2) + 1024;
    static int configured2 = 0;
    if (smem2 > configured2) {
      BST_CUDA(cudaFuncSetAttribute(gemm_bf16_2cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
      configured2 = smem2;
    }
    cudaLaunchConfig_t cfg2{};
    cfg2.gridDim = dim3(2 * s.grid);
    cfg2.blockDim = dim3(G_THREADS);
    cfg2.dynamicSmemBytes = smem2;
    cfg2.stream = as_stream(stream);
    cudaLaunchAttribute at2[1];
    at2[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at2[0].val.programmaticStreamSerializationAllowed = 1;
    cfg2.attrs = at2;
    cfg2.numAttrs = 1;
    static int trig2 = -1;
    // No PDL trigger at CTA entry for the CTA-pair kernel: with it, a batched draft phase
    // (CTA-pair GEMMs at 144-256 rows, back to back with their epilogues) deadlocked the
    // GPU within a few cycles (scripts/c3_probe.py, 64 requests); dependents launch when
    // the grid retires.  BST_GEMM2_TRIGGER=1 re-enables it (measurement only).
    if (trig2 < 0) trig2 = getenv("BST_GEMM2_TRIGGER") ? atoi(getenv("BST_GEMM2_TRIGGER")) : 0;
    BST_CUDA(cudaLaunchKernelEx(&cfg2, gemm_bf16_2cta_kernel, tw2, tx2, s, partial, (int)s.stages, trig2));
    return BST_OK;
  }
  CUtensorMap tw, tx;
  int rc = cached_tmap(&tw, w, (uint64_t)s.n_out, (uint64_t)s.k, (uint64_t)s.k, G_BM, G_BK);
  if (rc) return rc;
  rc = make_tmap_bf16(&tx, x, (uint64_t)s.m, (uint64_t)s.k, (uint64_t)ld_x, (uint32_t)s.bn, G_BK);
  if (rc) return rc;
  const int smem = s.stages * (s.pair * G_TILE_W + s.bn * G_BK * 2) + 1024;
  static int configured[3] = {0, 0, 0};
  auto kern = s.pair == 2 ? gemm_bf16_kernel<2> : gemm_bf16_kernel<1>;
  if (smem > configured[s.pair]) {
    BST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured[s.pair] = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(s.grid);
  cfg.blockDim = dim3(G_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // PDL trigger at CTA entry: a PDL-launched successor (the next GEMM, which waits on
  // griddepcontrol.wait before loading X) is scheduled as soon as SMs free up instead of
  // after this grid retires; plain-launched epilogues still wait for completion.
  // BST_GEMM_TRIGGER=0 disables it (measurement).
  static int trigger = -1;
  if (trigger < 0) trigger = getenv("BST_GEMM_TRIGGER") ? atoi(getenv("BST_GEMM_TRIGGER")) : 1;
  BST_CUDA(cudaLaunchKernelEx(&cfg, kern, tw, tx, s, partial, (int)s.stages, trigger));
  return BST_OK;
}

extern "C" int bst_gemm_reduce(const float* partial, const bst_gemm_sched_t* sched, float* y_f32, void* y_bf16,
                               int64_t ldy, bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(partial && sched && (y_f32 || y_bf16), "null pointer argument");
  const bst_gemm_sched_t s = *sched;
  dim3 grid((s.n_out / 4 + 255) / 256 < 148 ? (s.n_out / 4 + 255) / 256 + 1 : 148, s.m);
  BST_CUDA(launch_pdl(gemm_reduce_kernel, dim3(grid), dim3(256), 0, as_stream(stream), partial, s, y_f32,
                                                          static_cast<__nv_bfloat16*>(y_bf16), ldy));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_gemm_argmax(const float* partial, const bst_gemm_sched_t* sched, void* scratch_u64,
                               int32_t* argmax, bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(partial && sched && scratch_u64 && argmax, "null pointer argument");
  const bst_gemm_sched_t s = *sched;
  cudaStream_t st = as_stream(stream);
  BST_CUDA(cudaMemsetAsync(scratch_u64, 0, sizeof(unsigned long long) * s.m, st));
  dim3 grid(s.n_out / 4 / 256 < 74 ? s.n_out / 4 / 256 + 1 : 74, s.m);
  BST_CUDA(launch_pdl(gemm_argmax_kernel, dim3(grid), dim3(256), 0, st, partial, s, static_cast<unsigned long long*>(scratch_u64), 0));
  BST_CUDA(launch_pdl(argmax_finalize_kernel, dim3((s.m + 127) / 128), dim3(128), 0, st, static_cast<unsigned long long*>(scratch_u64), s.m,
                                                            argmax));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

// Temperature sample per row: argmax_n (logit_n / T + Gumbel(seed, c + pos[row], n)).
extern "C" int bst_gemm_sample(const float* partial, const bst_gemm_sched_t* sched, void* scratch_u64,
                               int32_t* out, const int32_t* pos, const int32_t* state, int c_idx, float temperature,
                               uint64_t seed, bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(partial && sched && scratch_u64 && out && pos, "null pointer argument");
  BST_REQUIRE(temperature > 0.f, "temperature must be > 0 (T = 0 is bst_gemm_argmax)");
  const bst_gemm_sched_t s = *sched;
  cudaStream_t st = as_stream(stream);
  BST_CUDA(cudaMemsetAsync(scratch_u64, 0, sizeof(unsigned long long) * s.m, st));
  dim3 grid(s.n_out / 4 / 256 < 74 ? s.n_out / 4 / 256 + 1 : 74, s.m);
  BST_CUDA(launch_pdl(gemm_sample_kernel, dim3(grid), dim3(256), 0, st, partial, s, static_cast<unsigned long long*>(scratch_u64), pos, state,
                                           c_idx, 1.f / temperature,
                                           make_uint2((uint32_t)seed, (uint32_t)(seed >> 32))));
  BST_CUDA(launch_pdl(argmax_finalize_kernel, dim3((s.m + 127) / 128), dim3(128), 0, st, static_cast<unsigned long long*>(scratch_u64), s.m, out));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

// Vocab-parallel LM head: per-row packed argmax keys of this shard (global index =
// vocab_offset + column), as signed int64 ready for a MAX all-reduce across shards.
extern "C" int bst_gemm_argmax_keys(const float* partial, const bst_gemm_sched_t* sched, int64_t* keys,
                                    int vocab_offset, bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(partial && sched && keys, "null pointer argument");
  BST_REQUIRE(vocab_offset >= 0, "vocab_offset must be >= 0");
  const bst_gemm_sched_t s = *sched;
  cudaStream_t st = as_stream(stream);
  BST_CUDA(cudaMemsetAsync(keys, 0, sizeof(int64_t) * s.m, st));
  dim3 grid(s.n_out / 4 / 256 < 74 ? s.n_out / 4 / 256 + 1 : 74, s.m);
  unsigned long long* k = reinterpret_cast<unsigned long long*>(keys);
  BST_CUDA(launch_pdl(gemm_argmax_kernel, dim3(grid), dim3(256), 0, st, partial, s, k, vocab_offset));
  BST_CUDA(launch_pdl(argmax_key_flip_kernel, dim3((s.m + 127) / 128), dim3(128), 0, st, k, s.m));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

// argmax indices from all-reduced signed keys (lowest global index on ties)
extern "C" int bst_argmax_from_keys(const int64_t* keys, int m, int32_t* argmax, bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(keys && argmax && m >= 0, "bad arguments");
  if (m == 0) return BST_OK;
  BST_CUDA(launch_pdl(argmax_from_signed_kernel, dim3((m + 127) / 128), dim3(128), 0, as_stream(stream), 
      reinterpret_cast<const unsigned long long*>(keys), m, argmax));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_debug_gemm_trace(void* buf, int cta) {
  BST_CUDA(cudaMemcpyToSymbol(bst::g_gemm_trace, &buf, sizeof(void*)));
  BST_CUDA(cudaMemcpyToSymbol(bst::g_trace_cta, &cta, sizeof(int)));
  return BST_OK;
}

extern "C" int bst_debug_bnd_trace_gemm(void* buf) {  // BST_TRACE builds only
#ifdef BST_TRACE
  BST_CUDA(cudaMemcpyToSymbol(bst::g_bnd, &buf, sizeof(void*)));
  return BST_OK;
#else
  (void)buf;
  return BST_EINVAL;
#endif
}
