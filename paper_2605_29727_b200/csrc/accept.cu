// K6 — greedy acceptance walk, commit and in-place KV compaction; linearize mask.
//
// bst_accept replaces verify_tree (verify_sim.py:358-389) + commit
// (verify_sim.py:392-405) given the target's greedy token for every tree row
// (row i = the target's argmax after the path to node i).  One warp walks from
// the root; each step scans the current node's children (CSR from K2) with a
// ballot.  bst_kv_compact realises the paper's "KV cache reordered and cropped"
// (PAPER.md:911): slot c+path[i] -> c+i.  Sources are strictly increasing and
// >= destinations, but dst(i) can equal src(j) for j < i, so every CTA first
// stages all moved rows of its (layer, K/V, head) slice in shared memory, then
// writes them back — no cross-CTA overlap, no read-after-write hazard.
#include <cuda_bf16.h>

#include "common.cuh"

namespace bst {

__global__ void accept_kernel(const int32_t* __restrict__ token, const int32_t* __restrict__ child_start,
                              const int32_t* __restrict__ child_list, const int32_t* __restrict__ argmax,
                              int max_path, int32_t* path, int32_t* committed, int32_t* meta) {
  pdl_enter();
  const int lane = threadIdx.x;
  int cur = 0, len = 1, bonus = -1;
  if (lane == 0) path[0] = 0;
  while (true) {
    const int want = argmax[cur];
    const int b = child_start[cur], e = child_start[cur + 1];
    int found = -1;
    for (int j = b + lane; j < e && found < 0; j += 32) {
      const int child = child_list[j];
      if (token[child] == want) found = child;
    }
    // reduce: (parent, token) pairs are unique, so at most one lane matched
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) found = max(found, __shfl_xor_sync(0xffffffffu, found, o));
    if (found < 0 || len >= max_path) {
      bonus = want;
      break;
    }
    if (lane == 0) {
      path[len] = found;
      committed[len - 1] = want;
    }
    ++len;
    cur = found;
  }
  if (lane == 0) {
    committed[len - 1] = bonus;  // commit order: accepted draft tokens, then the bonus
    meta[0] = len;
    meta[1] = bonus;
    meta[2] = len;
  }
}

// grid: (n_layers * 2 * n_kv) CTAs; each owns one (layer, K|V, head) slice.
__global__ void kv_compact_kernel(__nv_bfloat16* kv, int n_kv, int head_dim, int page_size, int64_t layer_stride,
                                  const int32_t* __restrict__ page_table, const int32_t* __restrict__ c_dev,
                                  const int32_t* __restrict__ path, const int32_t* __restrict__ meta, int max_path) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char stage_raw[];
  const int len = meta[0];
  if (len <= 1) return;
  const int c = *c_dev;
  const int slice = blockIdx.x;
  const int head = slice % n_kv;
  const int kvsel = (slice / n_kv) & 1;
  const int layer = slice / (2 * n_kv);
  const int64_t page_elems = (int64_t)2 * n_kv * page_size * head_dim;
  __nv_bfloat16* base = kv + layer * layer_stride;
  const int vec = head_dim / 8;  // int4 = 8 bf16
  int4* stage = reinterpret_cast<int4*>(stage_raw);
  auto row_ptr = [&](int slot) {
    const int page = page_table[slot / page_size];
    const int off = slot % page_size;
    return reinterpret_cast<int4*>(base + page * page_elems + ((int64_t)kvsel * n_kv + head) * page_size * head_dim +
                                   (int64_t)off * head_dim);
  };
  const int n = min(len, max_path);
  for (int t = threadIdx.x; t < n * vec; t += blockDim.x) {
    const int i = t / vec, v = t % vec;
    stage[t] = row_ptr(c + path[i])[v];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n * vec; t += blockDim.x) {
    const int i = t / vec, v = t % vec;
    if (path[i] != i) row_ptr(c + i)[v] = stage[t];
  }
}

__global__ void linearize_mask_kernel(const uint32_t* __restrict__ anc, int mask_words, int t, int prefix_len,
                                      uint8_t* mask) {
  pdl_enter();
  const int64_t n = (int64_t)prefix_len + t;
  const int64_t row = blockIdx.x;
  uint8_t* out = mask + row * n;
  const int64_t tree_row = row - prefix_len;
  for (int64_t col = threadIdx.x; col < n; col += blockDim.x) {
    uint8_t v;
    if (col < prefix_len) {
      v = 1;
    } else if (tree_row < 0) {
      v = 0;
    } else {
      const int64_t j = col - prefix_len;
      v = (anc[tree_row * mask_words + (j >> 5)] >> (j & 31)) & 1u;
    }
    out[col] = v;
  }
}

}  // namespace bst

extern "C" int bst_accept(const int32_t* token, const int32_t* child_start, const int32_t* child_list,
                          const int32_t* argmax, int max_path, int32_t* path, int32_t* committed, int32_t* meta,
                          bst_stream_t stream) {
  BST_REQUIRE(token && child_start && child_list && argmax && path && committed && meta, "null pointer argument");
  BST_REQUIRE(max_path >= 1, "max_path must be >= 1");
  BST_CUDA(bst::launch_pdl(bst::accept_kernel, dim3(1), dim3(32), 0, bst::as_stream(stream), token, child_start, child_list, argmax, max_path, path,
                                                            committed, meta));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_kv_compact(void* kv, int n_layers, int n_kv, int head_dim, int page_size, int64_t layer_stride_elems,
                              const int32_t* page_table, const int32_t* c_dev, const int32_t* path,
                              const int32_t* meta, int max_path, bst_stream_t stream) {
  BST_REQUIRE(kv && page_table && c_dev && path && meta, "null pointer argument");
  BST_REQUIRE(head_dim % 8 == 0, "head_dim must be a multiple of 8");
  BST_REQUIRE(n_layers >= 1 && n_kv >= 1 && page_size >= 1 && max_path >= 1, "bad shape");
  const size_t smem = (size_t)max_path * head_dim * 2;
  BST_REQUIRE(smem <= 48 * 1024, "max_path*head_dim too large");
  BST_CUDA(bst::launch_pdl(bst::kv_compact_kernel, dim3(n_layers * 2 * n_kv), dim3(128), smem, bst::as_stream(stream), 
      static_cast<__nv_bfloat16*>(kv), n_kv, head_dim, page_size, layer_stride_elems, page_table, c_dev, path, meta,
      max_path));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_linearize_mask(const uint32_t* anc_mask, int mask_words, int t, int prefix_len, uint8_t* mask,
                                  bst_stream_t stream) {
  BST_REQUIRE(anc_mask && mask, "null pointer argument");
  BST_REQUIRE(t >= 1 && prefix_len >= 0, "bad shape");
  BST_REQUIRE((int64_t)mask_words * 32 >= t, "mask_words too small");
  const int64_t n = (int64_t)prefix_len + t;
  BST_REQUIRE(n < (1ll << 31), "mask too large");
  BST_CUDA(bst::launch_pdl(bst::linearize_mask_kernel, dim3((unsigned)n), dim3(256), 0, bst::as_stream(stream), anc_mask, mask_words, t, prefix_len, mask));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

namespace bst {
__global__ void ancestor_mask_kernel(const int32_t* __restrict__ parent, int t, int mask_words, uint32_t* mask) {
  pdl_enter();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < t; i += gridDim.x * blockDim.x) {
    uint32_t* row = mask + (size_t)i * mask_words;
    for (int w = 0; w < mask_words; ++w) row[w] = 0u;
    for (int j = i; j >= 0; j = j == 0 ? -1 : parent[j]) row[j >> 5] |= 1u << (j & 31);
  }
}
}  // namespace bst

// Ancestor-or-self bitmask of an explicit tree (parent[0] = -1, parent[i] < i).
extern "C" int bst_ancestor_mask(const int32_t* parent, int t, int mask_words, uint32_t* mask, bst_stream_t stream) {
  BST_REQUIRE(parent && mask, "null pointer argument");
  BST_REQUIRE(t >= 1 && (int64_t)mask_words * 32 >= t, "bad shape");
  BST_CUDA(bst::launch_pdl(bst::ancestor_mask_kernel, dim3((t + 255) / 256), dim3(256), 0, bst::as_stream(stream), parent, t, mask_words, mask));
  BST_LAUNCH_CHECK();
  return BST_OK;
}
