// K5 — fused elementwise epilogues of the Qwen3-style forward (omitted from
// the reference cost model: PAPER.md:1002-1003).  Every kernel
// reads the GEMM's fp32 stream-K partial slots directly (gemm_load), so the
// GEMM output never round-trips through a separate reduction pass.
//
//   embed_rmsnorm     tokens -> residual (fp32) and RMSNorm(x)*w (bf16)
//   qkv_rope          q/k RMSNorm per head + RoPE (theta) at positions pos[],
//                     q -> bf16, k/v -> paged KV cache slot slot[] (append)
//   residual_rmsnorm  residual += Y; x = RMSNorm(residual)*w; optional bf16
//                     copy of the residual (target features for the drafter)
//   swiglu            act = silu(gate) * up  (gate/up = one fused GEMM)
//   gather_rows       rows[path[i]] -> dst[i]  (accepted-path hidden features)
#include <climits>
#include <cstdlib>
#include <utility>
#include <cuda_bf16.h>

#include "common.cuh"
#include "gemm.cuh"
#include "rope.cuh"
#include "sm100.cuh"

namespace bst {

constexpr int E_THREADS = 256;


__device__ __forceinline__ float block_sum(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// ----------------------------------------------------------------- embed
__global__ void embed_rmsnorm_kernel(const int32_t* __restrict__ tokens, const __nv_bfloat16* __restrict__ emb, int h,
                                     const __nv_bfloat16* __restrict__ w, float eps, float* __restrict__ resid,
                                     __nv_bfloat16* __restrict__ x, int64_t ldx) {
  // one row per CTA; 16-byte chunks of 8 columns held in registers (h <= 8192, h % 8 == 0)
  pdl_enter();
  __shared__ float sh[32];
  constexpr int CPT = 4;  // chunks per thread (E_THREADS x 8 x CPT columns)
  const int t = blockIdx.x;
  const int64_t tok = tokens[t];
  const int nc = h >> 3;
  float v[CPT][8];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int c = threadIdx.x + j * E_THREADS;
    if (c < nc) {
      const uint4 raw = reinterpret_cast<const uint4*>(emb + tok * h)[c];
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(b[e]);
        v[j][2 * e] = f.x;
        v[j][2 * e + 1] = f.y;
        ss += f.x * f.x + f.y * f.y;
      }
      float4* rp = reinterpret_cast<float4*>(resid + (int64_t)t * h) + 2 * c;
      rp[0] = make_float4(v[j][0], v[j][1], v[j][2], v[j][3]);
      rp[1] = make_float4(v[j][4], v[j][5], v[j][6], v[j][7]);
    }
  }
  const float inv = rsqrtf(block_sum(ss, sh) / h + eps);
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int c = threadIdx.x + j * E_THREADS;
    if (c < nc) {
      const uint4 wr = reinterpret_cast<const uint4*>(w)[c];
      const __nv_bfloat162* wb = reinterpret_cast<const __nv_bfloat162*>(&wr);
      uint4 o;
      __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 wf = __bfloat1622float2(wb[e]);
        ob[e] = __floats2bfloat162_rn(v[j][2 * e] * inv * wf.x, v[j][2 * e + 1] * inv * wf.y);
      }
      reinterpret_cast<uint4*>(x + (int64_t)t * ldx)[c] = o;
    }
  }
}

// ------------------------------------------------------- residual + norm
// One CTA (1024 threads) per row; each thread owns groups of 4 columns.
// partial == nullptr: only normalise.  resid == nullptr: normalise Y itself.
constexpr int R_THREADS = 1024;
BST_BND_TRACE_DEF

__global__ void __launch_bounds__(R_THREADS) residual_rmsnorm_kernel(
    const float* __restrict__ partial, bst_gemm_sched_t s, float* resid, int h, const __nv_bfloat16* __restrict__ w,
    float eps, __nv_bfloat16* x, int64_t ldx, __nv_bfloat16* feat, int64_t ldf, int rows, bst_prefetch_t pf) {
  sm100::grid_dep_launch();
  if (threadIdx.x == 0) BND(s.reserved, 0);
  if (threadIdx.x == 0 && blockIdx.x == 0) BND_KIND(s.reserved, 2);
  if (threadIdx.x == 0) issue_prefetch(pf, blockIdx.x, gridDim.x);
  const int ng = h >> 2;
  // the norm weights are constant: fetch them while the producer GEMM drains (h <= 8192:
  // at most two 4-column groups per thread)
  uint2 wv[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int g = threadIdx.x + j * R_THREADS;
    if (x && g < ng) wv[j] = reinterpret_cast<const uint2*>(w)[g];
  }
  sm100::grid_dep_wait();  // PDL launch: the producer GEMM's partials are complete past this point
  if (threadIdx.x == 0) BND(s.reserved, 2);
  if (threadIdx.x == 0) BND(s.reserved, 3);
  __shared__ float sh[32];
  __shared__ float4 vals[2048];
  const int t = blockIdx.x;
  if (t >= rows) return;
  float ss = 0.f;
  for (int g = threadIdx.x; g < ng; g += R_THREADS) {
    float4 v = resid ? reinterpret_cast<const float4*>(resid + (int64_t)t * h)[g] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (partial) {
      const float4 y = gemm_load4(partial, s, t, g * 4);
      v.x += y.x; v.y += y.y; v.z += y.z; v.w += y.w;
    }
    if (resid) reinterpret_cast<float4*>(resid + (int64_t)t * h)[g] = v;
    if (feat) {
      __nv_bfloat162* f = reinterpret_cast<__nv_bfloat162*>(feat + (int64_t)t * ldf + g * 4);
      f[0] = __floats2bfloat162_rn(v.x, v.y);
      f[1] = __floats2bfloat162_rn(v.z, v.w);
    }
    vals[g] = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  const float inv = rsqrtf(block_sum(ss, sh) / h + eps);
  if (x) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int g = threadIdx.x + j * R_THREADS;
      if (g >= ng) break;
      const float4 v = vals[g];
      const __nv_bfloat162* wp = reinterpret_cast<const __nv_bfloat162*>(&wv[j]);
      const float2 w01 = __bfloat1622float2(wp[0]), w23 = __bfloat1622float2(wp[1]);
      __nv_bfloat162* xp = reinterpret_cast<__nv_bfloat162*>(x + (int64_t)t * ldx + g * 4);
      xp[0] = __floats2bfloat162_rn(v.x * inv * w01.x, v.y * inv * w01.y);
      xp[1] = __floats2bfloat162_rn(v.z * inv * w23.x, v.w * inv * w23.y);
    }
  }
#ifdef BST_TRACE
  __syncthreads();
  if (threadIdx.x == 0) BND(s.reserved, 1);
#endif
}


// Residual update from a DENSE y (the tensor-parallel all-reduced row-parallel output,
// fp32 or bf16): resid += y; x = RMSNorm(resid) * w; optional bf16 copy of the residual.
// Same arithmetic as residual_rmsnorm_kernel with y in place of the partial slots.
template <typename YT>
__global__ void __launch_bounds__(R_THREADS) residual_dense_kernel(
    const YT* __restrict__ y, int64_t ldy, float* resid, int h, const __nv_bfloat16* __restrict__ w, float eps,
    __nv_bfloat16* x, int64_t ldx, __nv_bfloat16* feat, int64_t ldf) {
  pdl_enter();
  __shared__ float sh[32];
  __shared__ float4 vals[2048];
  const int t = blockIdx.x;
  const int ng = h >> 2;
  float ss = 0.f;
  for (int g = threadIdx.x; g < ng; g += R_THREADS) {
    float4 v = reinterpret_cast<const float4*>(resid + (int64_t)t * h)[g];
    if (y) {
      const YT* yp = y + (int64_t)t * ldy + g * 4;
      v.x += (float)yp[0]; v.y += (float)yp[1]; v.z += (float)yp[2]; v.w += (float)yp[3];
    }
    reinterpret_cast<float4*>(resid + (int64_t)t * h)[g] = v;
    if (feat) {
      __nv_bfloat162* f = reinterpret_cast<__nv_bfloat162*>(feat + (int64_t)t * ldf + g * 4);
      f[0] = __floats2bfloat162_rn(v.x, v.y);
      f[1] = __floats2bfloat162_rn(v.z, v.w);
    }
    vals[g] = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  const float inv = rsqrtf(block_sum(ss, sh) / h + eps);
  for (int g = threadIdx.x; g < ng; g += R_THREADS) {
    const float4 v = vals[g];
    const __nv_bfloat162* wp = reinterpret_cast<const __nv_bfloat162*>(w + g * 4);
    const float2 w01 = __bfloat1622float2(wp[0]), w23 = __bfloat1622float2(wp[1]);
    __nv_bfloat162* xp = reinterpret_cast<__nv_bfloat162*>(x + (int64_t)t * ldx + g * 4);
    xp[0] = __floats2bfloat162_rn(v.x * inv * w01.x, v.y * inv * w01.y);
    xp[1] = __floats2bfloat162_rn(v.z * inv * w23.x, v.w * inv * w23.y);
  }
}

// ------------------------------------------------------------- q/k/v + rope
#ifndef BST_QR_LOAD_BATCH  // measurement builds may override
#define BST_QR_LOAD_BATCH 4
#endif
constexpr int QR_LOAD_BATCH = BST_QR_LOAD_BATCH;
// One CTA per (token row, group of 16 heads); one warp per head (d = 128, 4 values per lane).
__global__ void qkv_rope_kernel(const float* __restrict__ partial, bst_gemm_sched_t s, RopeArgs ra, bst_prefetch_t pf) {
  sm100::grid_dep_launch();
  if (threadIdx.x == 0) BND(s.reserved, 0);
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) BND_KIND(s.reserved, 3);
  if (threadIdx.x == 0 && blockIdx.y == 0) issue_prefetch(pf, blockIdx.x, gridDim.x);
  const int t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const RopeConst rc = rope_const(ra, lane);  // constant weights: fetched while the GEMM drains
  sm100::grid_dep_wait();
  if (threadIdx.x == 0) BND(s.reserved, 2);
  if (threadIdx.x == 0) BND(s.reserved, 3);
  const int nw = blockDim.x >> 5;
  const int h_end = min(ra.n_q + 2 * ra.n_kv, (int)(blockIdx.y + 1) * nw);
  for (int hd = blockIdx.y * nw + warp; hd < h_end; hd += nw) {
    // the qkv tiles span ~4 stream-K slots: their loads in flight together (the next kernel,
    // K3, takes a whole SM, so the extra registers cost no co-residency)
    const float4 y4 = gemm_load4<QR_LOAD_BATCH>(partial, s, t, hd * 128 + lane * 4);
    float v[4] = {y4.x, y4.y, y4.z, y4.w};
    rope_store_head(ra, rc, t, hd, v, lane);
  }
#ifdef BST_TRACE
  __syncthreads();
  if (threadIdx.x == 0) BND(s.reserved, 1);
#endif
}

// ---------------------------------------------------------------- swiglu
// G 4-column groups per thread, G = 1 or 2 chosen by the host (bst_swiglu): 256-thread CTAs,
// at most 7 of them per SM beside the down GEMM's early-launched CTA; G = 2 once one group
// per thread would need a second wave (96 rows: 4.06-4.08 -> 4.02-4.03 ms in the verify
// graph; at 32 rows G = 1 is 45 us faster; four groups slower everywhere)
template <int SW_GROUPS>
__global__ void swiglu_kernel(const float* __restrict__ partial, bst_gemm_sched_t s, int ffn, __nv_bfloat16* act,
                              int64_t lda, bst_prefetch_t pf) {
  if (threadIdx.x == 0) issue_prefetch(pf, blockIdx.y * gridDim.x + blockIdx.x, gridDim.x * gridDim.y);
  const int t = blockIdx.y;
  sm100::grid_dep_launch();
  if (threadIdx.x == 0) BND(s.reserved, 0);
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) BND_KIND(s.reserved, 4);
  sm100::grid_dep_wait();
  if (threadIdx.x == 0) BND(s.reserved, 2);
  if (threadIdx.x == 0) BND(s.reserved, 3);
  const int g0 = blockIdx.x * blockDim.x * SW_GROUPS + threadIdx.x;
  float4 gt[SW_GROUPS], up[SW_GROUPS];
#pragma unroll
  for (int j = 0; j < SW_GROUPS; ++j) {
    const int g = g0 + j * blockDim.x;
    if (g < (ffn >> 2)) {
      gt[j] = gemm_load4(partial, s, t, g * 4);
      up[j] = gemm_load4(partial, s, t, ffn + g * 4);
    }
  }
  auto si = [](float z) { return z / (1.f + __expf(-z)); };
#pragma unroll
  for (int j = 0; j < SW_GROUPS; ++j) {
    const int g = g0 + j * blockDim.x;
    if (g < (ffn >> 2)) {
      __nv_bfloat162* ap = reinterpret_cast<__nv_bfloat162*>(act + (int64_t)t * lda + g * 4);
      ap[0] = __floats2bfloat162_rn(si(gt[j].x) * up[j].x, si(gt[j].y) * up[j].y);
      ap[1] = __floats2bfloat162_rn(si(gt[j].z) * up[j].z, si(gt[j].w) * up[j].w);
    }
  }
#ifdef BST_TRACE
  __syncthreads();
  if (threadIdx.x == 0) BND(s.reserved, 1);
#endif
}

// ------------------------------------------------------------ gather rows
__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ src, int64_t lds, const int32_t* __restrict__ idx,
                                   const int32_t* __restrict__ count, int max_rows, int cols,
                                   __nv_bfloat16* __restrict__ dst, int64_t ldd, const int32_t* __restrict__ row_base) {
  pdl_enter();
  const int r = blockIdx.x;
  const int n = count ? *count : max_rows;
  const int64_t base = row_base ? *row_base : 0;
  const int4* sp = reinterpret_cast<const int4*>(src + (base + (r < n ? idx[r] : 0)) * lds);
  int4* dp = reinterpret_cast<int4*>(dst + (int64_t)r * ldd);
  for (int i = threadIdx.x; i < cols / 8; i += blockDim.x) dp[i] = r < n ? sp[i] : make_int4(0, 0, 0, 0);
}

}  // namespace bst

// ------------------------------------------------------------------ C ABI
using namespace bst;

extern "C" int bst_embed_rmsnorm(const int32_t* tokens, int rows, const void* emb, int h, const void* w, float eps,
                                 float* resid, void* x, int64_t ldx, bst_stream_t stream) {
  BST_REQUIRE(tokens && emb && w && resid && x, "null pointer argument");
  BST_REQUIRE(h % 8 == 0 && h <= 8 * 4 * E_THREADS && ldx % 8 == 0, "embedding width must be a multiple of 8, <= 8192");
  BST_CUDA(launch_pdl(embed_rmsnorm_kernel, dim3(rows), dim3(E_THREADS), 0, as_stream(stream), 
      tokens, static_cast<const __nv_bfloat16*>(emb), h, static_cast<const __nv_bfloat16*>(w), eps, resid,
      static_cast<__nv_bfloat16*>(x), ldx));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_residual_rmsnorm(const float* partial, const bst_gemm_sched_t* sched, float* resid, int rows, int h,
                                    const void* w, float eps, void* x, int64_t ldx, void* feat, int64_t ldf,
                                    bst_stream_t stream) {
  BST_REQUIRE(h <= 8192 && h % 4 == 0, "hidden size must be a multiple of 4 and <= 8192");
  BST_REQUIRE(!partial || sched, "partial without schedule");
  bst_gemm_sched_t s{};
  if (sched) s = *sched;
  s.reserved = bnd_next_seq();
  BST_CUDA(launch_pdl(residual_rmsnorm_kernel, dim3(rows), dim3(R_THREADS), 0, as_stream(stream), partial, s, resid, h,
                      static_cast<const __nv_bfloat16*>(w), eps, static_cast<__nv_bfloat16*>(x), ldx,
                      static_cast<__nv_bfloat16*>(feat), ldf, rows, take_prefetch()));
  BST_LAUNCH_CHECK();
  return BST_OK;
}


extern "C" int bst_residual_dense(const void* y, int y_bf16, int64_t ldy, float* resid, int rows, int h, const void* w,
                                  float eps, void* x, int64_t ldx, void* feat, int64_t ldf, bst_stream_t stream) {
  BST_REQUIRE(resid && w && x, "null pointer argument");
  BST_REQUIRE(h <= 8192 && h % 4 == 0, "hidden size must be a multiple of 4 and <= 8192");
  if (rows <= 0) return BST_OK;
  if (y_bf16)
    BST_CUDA(launch_pdl(residual_dense_kernel<__nv_bfloat16>, dim3(rows), dim3(R_THREADS), 0, as_stream(stream),
                        static_cast<const __nv_bfloat16*>(y), ldy, resid, h, static_cast<const __nv_bfloat16*>(w), eps,
                        static_cast<__nv_bfloat16*>(x), ldx, static_cast<__nv_bfloat16*>(feat), ldf));
  else
    BST_CUDA(launch_pdl(residual_dense_kernel<float>, dim3(rows), dim3(R_THREADS), 0, as_stream(stream),
                        static_cast<const float*>(y), ldy, resid, h, static_cast<const __nv_bfloat16*>(w), eps,
                        static_cast<__nv_bfloat16*>(x), ldx, static_cast<__nv_bfloat16*>(feat), ldf));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

namespace bst {
RopeArgs make_rope_args(int n_q, int n_kv, const void* q_norm, const void* k_norm, float eps, const float* inv_freq,
                        const int32_t* pos, const int32_t* slot, const int32_t* qrow, void* q_out, int64_t q_tok_stride,
                        void* kv, int64_t layer_off_elems, const int32_t* page_table, int page_size,
                        const int32_t* state, int state_c_idx, int req_rows, int req_span, int req_state,
                        int req_slots, const int32_t* row_req) {
  RopeArgs r;
  r.n_q = n_q;
  r.n_kv = n_kv;
  r.qn = static_cast<const __nv_bfloat16*>(q_norm);
  r.kn = static_cast<const __nv_bfloat16*>(k_norm);
  r.eps = eps;
  r.inv_freq = inv_freq;
  r.pos = pos;
  r.slot = slot;
  r.qrow = qrow;
  r.q_out = static_cast<__nv_bfloat16*>(q_out);
  r.q_tok_stride = q_tok_stride;
  r.kv = static_cast<__nv_bfloat16*>(kv);
  r.layer_off = layer_off_elems;
  r.page_table = page_table;
  r.page_size = page_size;
  r.state = state;
  r.c_idx = state_c_idx;
  r.req_rows = req_rows;
  r.req_span = req_span > 0 ? req_span : 1;
  r.req_state = req_state;
  r.req_slots = req_slots;
  r.row_req = row_req;
  return r;
}
}  // namespace bst

extern "C" int bst_qkv_rope_batch(const float* partial, const bst_gemm_sched_t* sched, int rows, int n_q, int n_kv,
                                  const void* q_norm, const void* k_norm, float eps, const float* inv_freq,
                                  const int32_t* pos, const int32_t* slot, const int32_t* qrow, void* q_out,
                                  int64_t q_tok_stride, void* kv, int64_t layer_off_elems, const int32_t* page_table,
                                  int page_size, const int32_t* state, int state_c_idx, int req_rows, int req_span,
                                  int req_state, int req_slots, const int32_t* row_req, bst_stream_t stream) {
  BST_REQUIRE(partial && sched && q_norm && k_norm && inv_freq && pos && slot && q_out && kv && page_table,
              "null pointer argument");
  BST_REQUIRE(sched->n_out == (n_q + 2 * n_kv) * 128, "qkv width mismatch (head_dim must be 128)");
  const RopeArgs ra = make_rope_args(n_q, n_kv, q_norm, k_norm, eps, inv_freq, pos, slot, qrow, q_out, q_tok_stride,
                                     kv, layer_off_elems, page_table, page_size, state, state_c_idx, req_rows,
                                     req_span, req_state, req_slots, row_req);
  bst_gemm_sched_t s = *sched;
  s.reserved = bnd_next_seq();
  BST_CUDA(launch_pdl(qkv_rope_kernel, dim3(rows, (n_q + 2 * n_kv + 15) / 16), dim3(512), 0, as_stream(stream),
                      partial, s, ra, take_prefetch()));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_qkv_rope(const float* partial, const bst_gemm_sched_t* sched, int rows, int n_q, int n_kv,
                            const void* q_norm, const void* k_norm, float eps, const float* inv_freq, const int32_t* pos,
                            const int32_t* slot, const int32_t* qrow, void* q_out, int64_t q_tok_stride, void* kv,
                            int64_t layer_off_elems, const int32_t* page_table, int page_size, const int32_t* state,
                            int state_c_idx, bst_stream_t stream) {
  return bst_qkv_rope_batch(partial, sched, rows, n_q, n_kv, q_norm, k_norm, eps, inv_freq, pos, slot, qrow, q_out,
                            q_tok_stride, kv, layer_off_elems, page_table, page_size, state, state_c_idx, 0, 1, 0, 0,
                            nullptr, stream);
}

extern "C" int bst_swiglu(const float* partial, const bst_gemm_sched_t* sched, int rows, int ffn, void* act,
                          int64_t lda, bst_stream_t stream) {
  BST_REQUIRE(partial && sched && act, "null pointer argument");
  BST_REQUIRE(sched->n_out == 2 * ffn && ffn % 4 == 0, "gate/up width mismatch");
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    BST_CUDA(cudaGetDevice(&dev));
    BST_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  }
  const int ctas1 = (ffn / 4 + 255) / 256;
  const int groups = (int64_t)ctas1 * rows <= 7ll * n_sm ? 1 : 2;
  dim3 grid((ffn / 4 + 256 * groups - 1) / (256 * groups), rows);
  bst_gemm_sched_t s = *sched;
  s.reserved = bnd_next_seq();
  BST_CUDA(launch_pdl(groups == 1 ? swiglu_kernel<1> : swiglu_kernel<2>, grid, dim3(256), 0, as_stream(stream), partial, s, ffn,
                      static_cast<__nv_bfloat16*>(act), lda, take_prefetch()));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_gather_rows(const void* src, int64_t lds, const int32_t* idx, const int32_t* count, int max_rows,
                               int cols, void* dst, int64_t ldd, const int32_t* row_base, bst_stream_t stream) {
  BST_REQUIRE(src && idx && dst, "null pointer argument");
  BST_REQUIRE(cols % 8 == 0 && lds % 8 == 0 && ldd % 8 == 0, "rows must be 16-byte multiples");
  BST_CUDA(launch_pdl(gather_rows_kernel, dim3(max_rows), dim3(256), 0, as_stream(stream), static_cast<const __nv_bfloat16*>(src), lds, idx, count,
                                                              max_rows, cols, static_cast<__nv_bfloat16*>(dst), ldd,
                                                              row_base));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

// ------------------------------------------------------ decode-state plumbing
namespace bst {
__global__ void verify_rows_kernel(const int32_t* state, const int32_t* tree_token, const int32_t* tree_depth,
                                   const int32_t* meta, int rows, int32_t* tokens, int32_t* pos, int32_t* slot) {
  pdl_enter();
  const int n = meta[0];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    const bool real = i <= n;
    tokens[i] = i == 0 ? state[BST_ST_BONUS] : (real ? tree_token[i] : 0);
    pos[i] = real ? tree_depth[i] : 0;
    slot[i] = i;
  }
}
__global__ void drafter_rows_kernel(const int32_t* state, int gamma, int mask_token, int ctx_rows, int32_t* tokens,
                                    int32_t* pos, int32_t* slot, int32_t* qrow) {
  pdl_enter();
  const int n_new = state[BST_ST_NNEW];
  const int i = threadIdx.x;
  if (i <= gamma) {
    tokens[i] = i == 0 ? state[BST_ST_BONUS] : mask_token;
    pos[i] = i;
    slot[i] = i;
    qrow[i] = i;
  } else if (i < gamma + 1 + ctx_rows) {
    const int j = i - gamma - 1;
    tokens[i] = 0;
    pos[i] = j - n_new;
    slot[i] = j < n_new ? j - n_new : INT_MIN;
    qrow[i] = -1;
  }
}
// batched drafter rows: request r's gamma+1 query rows at [r*(gamma+1), ...), its
// ctx_rows context rows at [n_req*(gamma+1) + r*ctx_rows, ...); qrow = the q-buffer row
__global__ void drafter_rows_batch_kernel(const int32_t* state, int req_state, int n_req, int gamma, int mask_token,
                                          int ctx_rows, int32_t* tokens, int32_t* pos, int32_t* slot, int32_t* qrow) {
  pdl_enter();
  const int r = blockIdx.x;
  const int n_new = state[r * req_state + BST_ST_NNEW];
  const int i = threadIdx.x;
  if (i <= gamma) {
    const int t = r * (gamma + 1) + i;
    tokens[t] = i == 0 ? state[r * req_state + BST_ST_BONUS] : mask_token;
    pos[t] = i;
    slot[t] = i;
    qrow[t] = t;
  } else if (i < gamma + 1 + ctx_rows) {
    const int j = i - gamma - 1;
    const int t = n_req * (gamma + 1) + r * ctx_rows + j;
    tokens[t] = 0;
    pos[t] = j - n_new;
    slot[t] = j < n_new ? j - n_new : INT_MIN;
    qrow[t] = -1;
  }
}
__global__ void commit_state_kernel(int32_t* state, const int32_t* meta, const int32_t* committed, int max_path,
                                    int32_t* out_tokens, int out_cap, const int32_t* tree_meta,
                                    const double* surrogate, int32_t* log_i32, double* log_f64, int log_cap) {
  pdl_enter();
  const int len = meta[0];
  const int base = state[BST_ST_COMMITTED];
  for (int i = threadIdx.x; i < len && i < max_path; i += blockDim.x)
    if (base + i < out_cap) out_tokens[base + i] = committed[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int cyc = state[BST_ST_CYCLE];
    if (log_i32 && cyc < log_cap) {
      log_i32[cyc * 8 + 0] = tree_meta ? tree_meta[0] : -1;  // tree size N
      log_i32[cyc * 8 + 1] = tree_meta ? tree_meta[1] : -1;  // nodes expanded
      log_i32[cyc * 8 + 2] = tree_meta ? tree_meta[2] : -1;  // stop reason
      log_i32[cyc * 8 + 3] = len;                            // accepted_len (incl. bonus)
      log_i32[cyc * 8 + 4] = state[BST_ST_C];                // context c of this cycle
      log_i32[cyc * 8 + 5] = meta[1];                        // bonus
      if (log_f64) log_f64[cyc] = surrogate ? surrogate[0] : 0.0;
    }
    state[BST_ST_C] += len;
    state[BST_ST_NNEW] = len;
    state[BST_ST_BONUS] = meta[1];
    state[BST_ST_COMMITTED] = base + len;
    state[BST_ST_CYCLE] = cyc + 1;
  }
}
}  // namespace bst

extern "C" int bst_verify_rows(const int32_t* state, const int32_t* tree_token, const int32_t* tree_depth,
                               const int32_t* meta, int rows, int32_t* tokens, int32_t* pos, int32_t* slot,
                               bst_stream_t stream) {
  BST_REQUIRE(state && tree_token && tree_depth && meta && tokens && pos && slot, "null pointer argument");
  BST_CUDA(launch_pdl(verify_rows_kernel, dim3((rows + 255) / 256), dim3(256), 0, as_stream(stream), state, tree_token, tree_depth, meta, rows,
                                                                        tokens, pos, slot));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_drafter_rows(const int32_t* state, int gamma, int mask_token, int ctx_rows, int32_t* tokens,
                                int32_t* pos, int32_t* slot, int32_t* qrow, bst_stream_t stream) {
  BST_REQUIRE(state && tokens && pos && slot && qrow, "null pointer argument");
  BST_REQUIRE(gamma + 1 + ctx_rows <= 1024, "too many drafter rows");
  BST_CUDA(launch_pdl(drafter_rows_kernel, dim3(1), dim3(1024), 0, as_stream(stream), state, gamma, mask_token, ctx_rows, tokens, pos, slot, qrow));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_drafter_rows_batch(const int32_t* state, int req_state, int n_req, int gamma, int mask_token,
                                      int ctx_rows, int32_t* tokens, int32_t* pos, int32_t* slot, int32_t* qrow,
                                      bst_stream_t stream) {
  BST_REQUIRE(state && tokens && pos && slot && qrow && n_req >= 1, "null pointer argument");
  BST_REQUIRE(gamma + 1 + ctx_rows <= 1024, "too many drafter rows");
  BST_CUDA(launch_pdl(drafter_rows_batch_kernel, dim3(n_req), dim3(1024), 0, as_stream(stream), state, req_state, n_req, gamma, mask_token, ctx_rows,
                                                                   tokens, pos, slot, qrow));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_commit_state(int32_t* state, const int32_t* accept_meta, const int32_t* committed, int max_path,
                                int32_t* out_tokens, int out_cap, const int32_t* tree_meta, const double* surrogate,
                                int32_t* log_i32, double* log_f64, int log_cap, bst_stream_t stream) {
  BST_REQUIRE(state && accept_meta && committed && out_tokens, "null pointer argument");
  BST_CUDA(launch_pdl(commit_state_kernel, dim3(1), dim3(128), 0, as_stream(stream), state, accept_meta, committed, max_path, out_tokens, out_cap,
                                                        tree_meta, surrogate, log_i32, log_f64, log_cap));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_debug_bnd_trace_elem(void* buf) {  // BST_TRACE builds only
#ifdef BST_TRACE
  BST_CUDA(cudaMemcpyToSymbol(bst::g_bnd, &buf, sizeof(void*)));
  return BST_OK;
#else
  (void)buf;
  return BST_EINVAL;
#endif
}
