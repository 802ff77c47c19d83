// Ragged batched verify (config 3 with per-request adaptive budgets).
//
// Each request r of a batch has its own Algorithm-1 tree of N*_r nodes, so its
// verify block is s_r = N*_r + 1 rows.  Rows are packed request after request
// (no padding between requests): row_off[r] = sum_{r' < r} s_r', and the GEMMs of
// the target forward run over the packed rows only.  Three small kernels plumb it:
//   * ragged_rows: offsets, counts, total; token / position / KV-slot / request of
//     every packed row (rows past the total up to rows_cap are padding: no K/V);
//   * ragged_unpack: a packed per-row int32 result (the LM-head argmax) back to a
//     per-request [n_req][s_max] layout for the per-request K6 accept walk;
//   * batch_plan: each request's next Algorithm-1 plan against the batch-aware
//     verify cost — the pass costs the weights once plus every request's rows, so
//     request r's curve is the reference LatencyCurve of its own rows shifted by the
//     other requests' flops / bytes (held at their last tree sizes), and S_hat counts
//     the batch's accepted tokens: a_offset = the others' surrogates.
// With one request every shift is 0 and K2 is exactly run_cycle (controller.py:56-107).
#include <climits>

#include "common.cuh"

namespace bst {

constexpr int RG_THREADS = 1024;

__global__ void __launch_bounds__(RG_THREADS) ragged_rows_kernel(const bst_tree_t* __restrict__ trees,
                                                                 const int32_t* __restrict__ state, int req_state,
                                                                 int n_req, int s_max, int rows_cap, int32_t* row_off,
                                                                 int32_t* row_cnt, int32_t* total, int32_t* tokens,
                                                                 int32_t* pos, int32_t* slot, int32_t* row_req) {
  pdl_enter();
  __shared__ int off_s[RG_THREADS + 1];
  __shared__ int warp_sum_s[RG_THREADS / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int cnt = t < n_req ? min(trees[t].meta[0] + 1, s_max) : 0;
  // block exclusive scan of the counts (request order)
  int v = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  if (lane == 31) warp_sum_s[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int w = warp_sum_s[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += u;
    }
    warp_sum_s[lane] = w;
  }
  __syncthreads();
  const int incl = v + (warp > 0 ? warp_sum_s[warp - 1] : 0);
  off_s[t + 1] = incl;
  if (t == 0) off_s[0] = 0;
  if (t < n_req) {
    row_off[t] = incl - cnt;
    row_cnt[t] = cnt;
  }
  __syncthreads();
  const int n_rows = off_s[n_req];
  if (t == 0) *total = n_rows;
  for (int i = t; i < rows_cap; i += RG_THREADS) {
    if (i >= n_rows) {
      tokens[i] = 0;
      pos[i] = 0;
      slot[i] = INT_MIN;
      row_req[i] = -1;
      continue;
    }
    int lo = 0, hi = n_req - 1;  // the request whose [off, off + cnt) holds row i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off_s[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int j = i - off_s[lo];
    const bst_tree_t tr = trees[lo];
    tokens[i] = j == 0 ? state[lo * req_state + BST_ST_BONUS] : tr.token[j];
    pos[i] = tr.depth[j];
    slot[i] = j;
    row_req[i] = lo;
  }
}

__global__ void ragged_unpack_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ row_off,
                                     const int32_t* __restrict__ row_cnt, int s_max, int32_t* __restrict__ dst) {
  pdl_enter();
  const int r = blockIdx.x;
  const int off = row_off[r], cnt = row_cnt[r];
  for (int j = threadIdx.x; j < s_max; j += blockDim.x) dst[(int64_t)r * s_max + j] = j < cnt ? src[off + j] : -1;
}

// One CTA; thread r owns request r.  `first`: no tree yet, the others count as their root row.
__global__ void __launch_bounds__(RG_THREADS) batch_plan_kernel(const bst_plan_t* __restrict__ base,
                                                                bst_plan_t* __restrict__ out,
                                                                const bst_tree_t* __restrict__ trees,
                                                                const int32_t* __restrict__ state, int req_state,
                                                                int n_req, int first) {
  pdl_enter();
  __shared__ long long f_s[RG_THREADS], b_s[RG_THREADS];
  __shared__ double a_s[RG_THREADS];
  __shared__ long long f_tot, b_tot;
  __shared__ double a_tot;
  const int r = threadIdx.x;
  if (r < n_req) {
    const bst_plan_t& p = base[r];
    const long long c = state[r * req_state + p.c_idx];
    const long long s = first ? 1 : (long long)trees[r].meta[0] + 1;
    const long long f1 = p.curve.flops_lin + p.d_flops_lin * c;
    const long long b1 = p.curve.bytes_lin + p.d_bytes_lin * c;
    f_s[r] = (f1 + p.curve.flops_quad * s) * s;
    b_s[r] = p.d_bytes_const * c + (b1 + p.curve.bytes_quad * s) * s;  // KV + activations (weights once)
    a_s[r] = first ? 1.0 : trees[r].surrogate[0];
  }
  __syncthreads();
  if (r == 0) {  // fixed request order: deterministic totals
    long long f = 0, b = 0;
    double a = 0.0;
    for (int i = 0; i < n_req; ++i) {
      f += f_s[i];
      b += b_s[i];
      a += a_s[i];
    }
    f_tot = f;
    b_tot = b;
    a_tot = a;
  }
  __syncthreads();
  if (r < n_req) {
    bst_plan_t p = base[r];
    p.curve.flops_const = f_tot - f_s[r];
    p.curve.bytes_const += b_tot - b_s[r];
    p.a_offset = a_tot - a_s[r];
    out[r] = p;
  }
}

}  // namespace bst

using namespace bst;

extern "C" int bst_ragged_rows(const bst_tree_t* trees_dev, const int32_t* state, int req_state, int n_req, int s_max,
                               int rows_cap, int32_t* row_off, int32_t* row_cnt, int32_t* total, int32_t* tokens,
                               int32_t* pos, int32_t* slot, int32_t* row_req, bst_stream_t stream) {
  BST_REQUIRE(trees_dev && state && row_off && row_cnt && total && tokens && pos && slot && row_req,
              "null pointer argument");
  BST_REQUIRE(n_req >= 1 && n_req <= RG_THREADS, "n_req must be in [1, %d]", RG_THREADS);
  BST_REQUIRE(s_max >= 1 && rows_cap >= 1, "bad sizes");
  BST_CUDA(launch_pdl(ragged_rows_kernel, dim3(1), dim3(RG_THREADS), 0, as_stream(stream), trees_dev, state,
                      req_state, n_req, s_max, rows_cap, row_off, row_cnt, total, tokens, pos, slot, row_req));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_ragged_unpack(const int32_t* src, const int32_t* row_off, const int32_t* row_cnt, int n_req,
                                 int s_max, int32_t* dst, bst_stream_t stream) {
  BST_REQUIRE(src && row_off && row_cnt && dst && n_req >= 1 && s_max >= 1, "bad arguments");
  BST_CUDA(launch_pdl(ragged_unpack_kernel, dim3(n_req), dim3(256), 0, as_stream(stream), src, row_off, row_cnt, s_max,
                      dst));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_batch_plan(const bst_plan_t* base_dev, bst_plan_t* out_dev, const bst_tree_t* trees_dev,
                              const int32_t* state, int req_state, int n_req, int first, bst_stream_t stream) {
  BST_REQUIRE(base_dev && out_dev && trees_dev && state, "null pointer argument");
  BST_REQUIRE(n_req >= 1 && n_req <= RG_THREADS, "n_req must be in [1, %d]", RG_THREADS);
  BST_CUDA(launch_pdl(batch_plan_kernel, dim3(1), dim3(RG_THREADS), 0, as_stream(stream), base_dev, out_dev, trees_dev,
                      state, req_state, n_req, first));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_struct_size(int which) {  // ABI check for bindings: 0 curve, 1 plan, 2 tree, 3 gemm schedule
  switch (which) {
    case 0: return (int)sizeof(bst_curve_t);
    case 1: return (int)sizeof(bst_plan_t);
    case 2: return (int)sizeof(bst_tree_t);
    case 3: return (int)sizeof(bst_gemm_sched_t);
    default: return BST_EINVAL;
  }
}
