// q/k RMSNorm + rotary embedding + q / paged-KV store of one (token row, head): shared
// by the qkv_rope epilogue kernel and the qkv GEMM's fused tile fixup (gemm.cu).
#pragma once
#include <climits>
#include <cuda_bf16.h>

#include "common.cuh"

namespace bst {

struct RopeArgs {
  int n_q, n_kv;
  const __nv_bfloat16* qn;  // q_norm weight [128]
  const __nv_bfloat16* kn;  // k_norm weight [128]
  float eps;
  const float* inv_freq;    // [64]
  const int32_t* pos;       // per row, relative to the request's context c
  const int32_t* slot;      // per row KV slot relative to c (INT_MIN: no K/V)
  const int32_t* qrow;      // per row q output row (< 0: no q); nullptr = identity
  __nv_bfloat16* q_out;
  int64_t q_tok_stride;
  __nv_bfloat16* kv;        // paged cache [layer][page][K|V][n_kv][page_size][128]
  int64_t layer_off;
  const int32_t* page_table;
  int page_size;
  const int32_t* state;     // c = state[r * req_state + c_idx] (nullptr: c = 0)
  int c_idx;
  int req_rows, req_span, req_state, req_slots;  // batched requests (req_rows = 0: one request)
  const int32_t* row_req;   // ragged batch: request of each row (< 0: padding row); overrides req_rows
};

// The lane's constant operands: q/k norm weights and RoPE inverse frequencies of dims
// 4 lane .. 4 lane + 3 (loaded before griddepcontrol.wait; they never change).
struct RopeConst {
  float qn[4], kn[4], fr[4];
};
__device__ __forceinline__ RopeConst rope_const(const RopeArgs& a, int lane) {
  RopeConst c;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    c.qn[e] = __bfloat162float(a.qn[lane * 4 + e]);
    c.kn[e] = __bfloat162float(a.kn[lane * 4 + e]);
    c.fr[e] = a.inv_freq[(lane * 4 + e) & 63];
  }
  return c;
}

// This warp's lane holds dims 4 lane .. 4 lane + 3 of head `hd` for token row t in v.
__device__ __forceinline__ void rope_store_head(const RopeArgs& a, const RopeConst& rc, int t, int hd, float (&v)[4],
                                                int lane) {
  int r = a.req_rows > 0 ? (t % a.req_span) / a.req_rows : 0;
  if (a.row_req) {
    r = a.row_req[t];
    if (r < 0) return;  // padding row of a ragged batch: no q, no K/V
  }
  const int c0 = a.state ? a.state[r * a.req_state + a.c_idx] : 0;
  const bool is_q = hd < a.n_q, is_k = !is_q && hd < a.n_q + a.n_kv;
  const int qr = a.qrow ? a.qrow[t] : t;
  const int sl = a.slot[t] == INT_MIN ? -1 : a.slot[t] + c0 + r * a.req_slots;
  if (is_q && qr < 0) return;
  if (!is_q && sl < 0) return;
  if (is_q || is_k) {
    float ss = v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3];
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / 128.f + a.eps);
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = v[e] * inv * (is_q ? rc.qn[e] : rc.kn[e]);
    // rotate_half: lanes 0-15 hold dims 0-63, lanes 16-31 hold 64-127
    const int p = a.pos[t] + c0;
    float o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float sn, cs;
      sincosf((float)p * rc.fr[e], &sn, &cs);
      const float partner = __shfl_xor_sync(0xffffffffu, v[e], 16);
      o[e] = lane < 16 ? v[e] * cs - partner * sn : v[e] * cs + partner * sn;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = o[e];
  }
  const __nv_bfloat162 lo = __floats2bfloat162_rn(v[0], v[1]), hi = __floats2bfloat162_rn(v[2], v[3]);
  __nv_bfloat16* dst;
  if (is_q) {
    dst = a.q_out + (int64_t)qr * a.q_tok_stride + hd * 128 + lane * 4;
  } else {
    const int head = is_k ? hd - a.n_q : hd - a.n_q - a.n_kv;
    const int64_t page = a.page_table[sl / a.page_size];
    const int64_t off = ((page * 2 + (is_k ? 0 : 1)) * a.n_kv + head) * a.page_size + (sl % a.page_size);
    dst = a.kv + a.layer_off + off * 128 + lane * 4;
  }
  *reinterpret_cast<__nv_bfloat162*>(dst) = lo;
  *reinterpret_cast<__nv_bfloat162*>(dst + 2) = hi;
}

}  // namespace bst
