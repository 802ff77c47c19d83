/*
 * bastion.h — C ABI of the B200-native BASTION draft→expand→verify→accept engine.
 *
 * Every entry point takes caller-owned DEVICE buffers (plain pointers + sizes)
 * and an explicit CUDA stream, never allocates on the hot path, and returns an
 * int status (0 = ok, <0 = error; text via bst_last_error()).  No torch types.
 *
 * Each function replaces one reference (``specplan``, Python) interface; the
 * reference file:line is cited beside it (paths relative to
 * /root/reference/pkg/src/specplan).  INTEGRATION.md shows the ctypes binding a
 * maintainer adds on the reference side.
 */
#ifndef BASTION_H_
#define BASTION_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* bst_stream_t; /* cudaStream_t; NULL = legacy default stream */

#define BST_OK 0
#define BST_EINVAL (-1) /* argument error   -> ValueError in the Python shim   */
#define BST_ECUDA (-2)  /* CUDA error        -> RuntimeError                    */
#define BST_ECAP (-3)   /* internal capacity exceeded (caller retries bigger)   */

int bst_abi_version(void);
const char* bst_last_error(void);

/* ------------------------------------------------------------------------
 * Latency curve at a fixed context c.
 * Replaces LatencyCurve (cost_model.py:284-309): exact integer coefficients,
 * reciprocal multiplies, variant factors slope/intercept/ratio.
 * ---------------------------------------------------------------------- */
typedef struct {
  int64_t flops_lin, flops_quad;             /* cost_model.py:290-291 */
  int64_t bytes_const, bytes_lin, bytes_quad; /* cost_model.py:292-294 */
  double inv_peak, inv_bw;                   /* cost_model.py:295-296 */
  double slope, intercept, ratio;            /* cost_model.py:297-303 */
  /* Batched verify (extension, 0 for one request): flops of the other requests
   * verified in the same pass; compute = (flops_const + (lin + quad s) s) / peak. */
  int64_t flops_const;
} bst_curve_t;

/* Host-side evaluation of LatencyCurve.latency(s) with the device arithmetic. */
double bst_curve_latency(const bst_curve_t* curve, int64_t s);

/* ------------------------------------------------------------------------
 * K1 — top-K candidate lattice.
 * bst_topk_logits replaces the drafter plugin's softmax + MarginalBlock rows
 * (lattice.py:24-55) fused with top_k_truncate (lattice.py:128-142):
 *   m = max_v l, Z = sum_v exp64(l_v - m), prob_v = exp64(l_v - m) / Z,
 *   keep the k best by (prob desc, token asc).
 * logits: [gamma, row_stride] fp32 (dtype 0) or bf16 (dtype 1).
 * probs_full (nullable): fp64 [gamma, vocab] full rows, bit-identical to the
 * lattice probabilities (the MarginalBlock a reference plugin would return).
 * bst_topk_probs replaces top_k_truncate on an fp64 MarginalBlock.
 * ---------------------------------------------------------------------- */
size_t bst_topk_workspace(int gamma, int vocab, int k);
int bst_topk_logits(const void* logits, int dtype, int gamma, int vocab, int64_t row_stride, int k,
                    int32_t* tok, double* prob, double* probs_full, void* ws, size_t ws_bytes,
                    bst_stream_t stream);
int bst_topk_probs(const double* probs, int gamma, int vocab, int k, int32_t* tok, double* prob,
                   void* ws, size_t ws_bytes, bst_stream_t stream);

/* ------------------------------------------------------------------------
 * K2 — tree expansion.
 * policy ADAPTIVE replaces run_cycle (controller.py:56-107) incl. the
 * LatencyCurve evaluation; FIXED replaces best_first_expand
 * (draft_tree.py:138-155) over ExpansionFrontier/iter_best_first
 * (draft_tree.py:69-135); BEAM replaces beam_expand (draft_tree.py:158-189),
 * greedy chain = BEAM width 1 depth gamma (verify_sim.py:419-420).
 * ---------------------------------------------------------------------- */
enum { BST_POLICY_ADAPTIVE = 0, BST_POLICY_FIXED = 1, BST_POLICY_BEAM = 2 };
enum { BST_STOP_FIRST_DECREASE = 0, BST_STOP_FRONTIER_EXHAUSTED = 1, BST_STOP_BUDGET_CAP = 2 };
enum { BST_ALGO_AUTO = 0, BST_ALGO_SORT = 1, BST_ALGO_HEAP = 2 };

typedef struct {
  int32_t policy;   /* BST_POLICY_* */
  int32_t n_max;    /* ControllerConfig.n_max / best_first n_max */
  int32_t width;    /* beam width */
  int32_t depth;    /* beam depth */
  int32_t algo;     /* BST_ALGO_*: sort-based parallel (default) or sequential heap */
  int32_t _pad;
  bst_curve_t curve; /* adaptive only */
  double fixed_cost; /* t_draft + t_aux, controller.py:73 */
  double l_ar;       /* CycleLatencies.l_ar */
  /* Optional device-resident decode state: when `state` is non-null the
   * context is c = state[c_idx] and the curve coefficients are
   * base + d_* * c (exact integers, LatencyCurve at context c).            */
  const int32_t* state;
  int32_t c_idx;
  int32_t _pad2;
  int64_t d_flops_lin, d_bytes_const, d_bytes_lin;
  /* Batched verify (extension, 0 for one request): surrogate of the other requests
   * of the pass; Algorithm 1 scores S_hat = (a_offset + a_hat) * l_ar / C_hat, the
   * batch's accepted tokens per pass time with the others' trees held fixed.      */
  double a_offset;
} bst_plan_t;

/* Output arrays (device), row 0 = root.  Capacity n_cap+1 rows. */
typedef struct {
  int32_t* parent;      /* [n_cap+1] root -1 */
  int32_t* depth;       /* [n_cap+1] */
  int32_t* token;       /* [n_cap+1] root -1 */
  int32_t* rank;        /* [n_cap+1] lattice rank, root -1 */
  double* rho;          /* [n_cap+1] path scores, root 1.0 */
  double* trace;        /* [n_cap] S_hat per expanded node (adaptive), nullable */
  int32_t* meta;        /* [8]: 0 n_nodes, 1 n_expanded, 2 stop, 3 algo used, 4 enumerated */
  double* surrogate;    /* [1] */
  uint32_t* anc_mask;   /* [(n_cap+1) * mask_words] ancestor-or-self bits, nullable */
  int32_t mask_words;   /* u32 words per mask row (>= ceil((n_cap+1)/32)) */
  int32_t _pad;
  int32_t* child_start; /* [n_cap+2] children CSR offsets, nullable */
  int32_t* child_list;  /* [n_cap] */
} bst_tree_t;

size_t bst_expand_workspace(int gamma, int k, int n_cap);
int bst_expand(const int32_t* tok, const double* prob, int gamma, int k, const bst_plan_t* plan,
               int n_cap, const bst_tree_t* out, void* ws, size_t ws_bytes, bst_stream_t stream);

/* Dense (prefix_len + t)^2 byte mask of linearize (verify_sim.py:336-355) from
 * the ancestor bitmask: prefix columns 1 for every row, tree block = ancestors. */
int bst_linearize_mask(const uint32_t* anc_mask, int mask_words, int t, int prefix_len, uint8_t* mask,
                       bst_stream_t stream);

/* Ancestor-or-self bitmask of an explicit tree (parent[0] = -1, parent[i] < i),
 * for trees built on the host (build_tree, draft_tree.py:204-236).          */
int bst_ancestor_mask(const int32_t* parent, int t, int mask_words, uint32_t* mask, bst_stream_t stream);

/* ------------------------------------------------------------------------
 * K6 — greedy acceptance walk + KV compaction.
 * bst_accept replaces verify_tree (verify_sim.py:358-389) + commit
 * (verify_sim.py:392-405) given the target's greedy token per tree row:
 * out: path[max_path] node ids (root 0 first), meta[0] = accepted_len (incl.
 * root), meta[1] = bonus token, meta[2] = number of committed tokens.
 * committed[] receives accepted draft tokens then the bonus (commit order).
 * ---------------------------------------------------------------------- */
/* Device plan variant: identical to bst_expand but the plan lives in device
 * memory (so a captured CUDA graph can be re-planned by a host->device copy). */
int bst_expand_dev(const int32_t* tok, const double* prob, int gamma, int k, const bst_plan_t* plan_dev,
                   int policy, int n_max, int n_cap, const bst_tree_t* out, void* ws, size_t ws_bytes,
                   bst_stream_t stream);
/* K2 over n_req independent requests in one launch (batched engine, config 3): request r
 * reads lattice rows tok/prob + r * lat_stride, plan_dev[r], writes trees_dev[r] (device
 * array of n_req bst_tree_t); ws: n_req x bst_expand_workspace(gamma, k, n_cap) bytes. */
int bst_expand_dev_batch(const int32_t* tok, const double* prob, int64_t lat_stride, int gamma, int k,
                         const bst_plan_t* plan_dev, int policy, int n_max, int n_cap, const bst_tree_t* trees_dev,
                         int n_req, void* ws, size_t ws_bytes, bst_stream_t stream);

int bst_accept(const int32_t* token, const int32_t* child_start, const int32_t* child_list,
               const int32_t* argmax, int max_path, int32_t* path, int32_t* committed, int32_t* meta,
               bst_stream_t stream);

/* Paged KV cache: layout [layer][page][2 (K,V)][n_kv][page_size][head_dim] bf16.
 * Moves slot c+path[i] -> c+i for i < meta[0] in every layer (race-free:
 * each CTA owns one (layer, K/V, head) slice and stages rows in smem).   */
int bst_kv_compact(void* kv, int n_layers, int n_kv, int head_dim, int page_size, int64_t layer_stride_elems,
                   const int32_t* page_table, const int32_t* c_dev, const int32_t* path, const int32_t* meta,
                   int max_path, bst_stream_t stream);

/* ------------------------------------------------------------------------
 * K4 — bf16 weight-streaming GEMM on tcgen05, Y[m,n_out] = X[m,K] . W[n_out,K]^T.
 * Replaces the dense matmul rows of the Appendix-D cost model
 * (cost_model.py:118-123) — the reference has no GEMM.
 * Output is a set of fp32 partial slots (stream-K over (tile, k-block)
 * units); consumers reduce them in fixed order (bst_gemm_reduce / argmax or
 * the fused epilogue kernels of the model forward).
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t n_out, k, m, bn;      /* bn = round_up(m, 16) token columns (<= 256); m in 257..512 only on
                                   the CTA-pair kernel (even tile counts): bn = round_up(m, 32) */
  int32_t n_mt, n_kb, grid, s_max;
  int64_t units;                /* ceil(n_mt / pair) * n_kb */
  int32_t tmem_cols, stages;
  int64_t partial_floats;       /* size of the partial buffer */
  int32_t pair;                 /* weight tiles per stream-K unit (1, or 2 for m > 128: X k-block shared) */
  int32_t reserved;             /* trace builds: launch sequence number */
  int32_t cta2;                 /* 1: CTA-pair kernel (tcgen05 cta_group::2), grid = number of pairs */
  int32_t pad_;
} bst_gemm_sched_t;

int bst_gemm_schedule(int n_out, int k, int m, int grid, bst_gemm_sched_t* out);
int bst_gemm(const void* w, const void* x, int64_t ld_x, const bst_gemm_sched_t* sched, float* partial,
             size_t partial_bytes, bst_stream_t stream);
int bst_gemm_reduce(const float* partial, const bst_gemm_sched_t* sched, float* y_f32, void* y_bf16, int64_t ldy,
                    bst_stream_t stream);
/* Per-row argmax of Y with numpy tie-break (lowest index), verify_sim.py:107-109. */
int bst_gemm_argmax(const float* partial, const bst_gemm_sched_t* sched, void* scratch_u64, int32_t* argmax,
                    bst_stream_t stream);
/* Temperature-T sample per row (exact-match sampled verification, verify_sim.py:111-126):
 * argmax over n of logit_n / T + Gumbel noise, the noise a Philox4x32-10 function of
 * (seed, absolute position c + pos[row], n) with c = state[c_idx] (state may be NULL:
 * c = 0), so the tree row of a node and the AR step at the same position sample
 * identically.  T must be > 0. */
int bst_gemm_sample(const float* partial, const bst_gemm_sched_t* sched, void* scratch_u64, int32_t* out,
                    const int32_t* pos, const int32_t* state, int c_idx, float temperature, uint64_t seed,
                    bst_stream_t stream);
/* K1 on the GEMM output (replaces the drafter plugin's softmax + top_k_truncate, lattice.py:24-55,
 * 128-142, like bst_topk_logits): the drafter LM head's partial slots are read directly,
 * summed as bst_gemm_reduce sums them, so the lattice is bit-identical to reducing first;
 * rows 0..gamma-1 of the GEMM, sched->n_out == vocab.  No full-row export. */
int bst_topk_gemm_partial(const float* partial, const bst_gemm_sched_t* sched, int gamma, int vocab, int k,
                          int32_t* tok, double* prob, void* ws, size_t ws_bytes, bst_stream_t stream);
/* Vocab-parallel LM head (tensor-parallel target): per-row argmax keys of
 * this shard, key = (order-preserving fp32 bits << 32 | 0xFFFFFFFF - global index),
 * global index = vocab_offset + column, top bit flipped so a signed int64 MAX
 * all-reduce across shards keeps np.argmax's lowest-index tie-break
 * (verify_sim.py:107-109).  bst_argmax_from_keys decodes the reduced keys. */
int bst_gemm_argmax_keys(const float* partial, const bst_gemm_sched_t* sched, int64_t* keys, int vocab_offset,
                         bst_stream_t stream);
int bst_argmax_from_keys(const int64_t* keys, int m, int32_t* argmax, bst_stream_t stream);

/* L2 prefetch hint: DRAM-idle kernels (attention, epilogues) stream the next
 * GEMM's weights into L2 while they run (weights never depend on activations). */
typedef struct {
  const void* ptr[2];
  uint64_t bytes[2];
} bst_prefetch_t;
int bst_set_prefetch(const bst_prefetch_t* pf); /* applies to the next K3/K5 launch on this thread */

/* ------------------------------------------------------------------------
 * K3 — tree-masked attention over the paged KV cache
 * (mask semantics of linearize, verify_sim.py:336-355; cost PAPER.md:1056-1062).
 * mode 0 TREE (prefix + ancestor bitmask), 1 CAUSAL (chunked prefill),
 * 2 FULL (drafter block).  c = state[c_idx] when state is non-null.
 * ws (n_splits > 1): the first 4 KiB hold split-arrival counters and must be
 * zero before the first call (each call leaves them zero); the rest holds the
 * per-split partial rows.  One ws per concurrently running call.
 * ---------------------------------------------------------------------- */
int bst_attention(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride, const void* kv_cache,
                  int n_layers, int n_pages_total, int layer, const int32_t* page_table, int n_q, int n_kv, int s,
                  int c, int keys_after_c, int max_keys, const int32_t* state, int c_idx, int mode,
                  const uint32_t* anc, int mask_words, int n_splits, float* ws, size_t ws_bytes, bst_stream_t stream);
/* Batched K3: n_req requests of s query rows each in one launch (config 3).
 * Request r owns q/out rows [r*s, r*s+s), page_table[r*req_pages ...], state
 * words state[r*req_state ...] (c = state[r*req_state + c_idx]) and ancestor-mask
 * rows anc[(r*s + i) * mask_words ...].  ws: bst_attention_workspace(n_q, s, n_splits)
 * times n_req (plus the shared 4 KiB counter head). */
int bst_attention_batch(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride, const void* kv_cache,
                        int n_layers, int n_pages_total, int layer, const int32_t* page_table, int req_pages, int n_q,
                        int n_kv, int n_req, int s, int keys_after_c, int max_keys, const int32_t* state, int req_state,
                        int c_idx, int mode, const uint32_t* anc, int mask_words, int n_splits, float* ws,
                        size_t ws_bytes, bst_stream_t stream);
size_t bst_attention_workspace(int n_q, int s, int n_splits);
/* Split partials alternate between two workspace banks with the layer index, so the
 * workspace holds 2 x n_splits x s x n_q x 130 floats after the counter head.
 * bst_attention picks its kernel by shape only: the single-softmax-group row-major
 * tcgen05 kernel for short per-CTA page runs, the two-group one from 8 pages on. */
/* Key-major K3 (S^T = K Q^T: one key per TMEM lane, every query row in the columns;
 * reference-max softmax; cluster/DSMEM or L2 split merge).  Same arguments and
 * results as bst_attention; a separate kernel kept for the measurements of DESIGN §5. */
int bst_attention_keymajor(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride, const void* kv_cache,
                           int n_layers, int n_pages_total, int layer, const int32_t* page_table, int n_q, int n_kv,
                           int s, int c, int keys_after_c, int max_keys, const int32_t* state, int c_idx, int mode,
                           const uint32_t* anc, int mask_words, int n_splits, float* ws, size_t ws_bytes,
                           bst_stream_t stream);

/* Ragged batched K3 (config 3, per-request adaptive trees): request r's query rows are
 * q/out rows [row_off[r], row_off[r] + row_cnt[r]) of a packed layout (device arrays,
 * written by bst_ragged_rows earlier in the same stream); its ancestor-mask rows stay at
 * anc[(r*s_max + i) * mask_words].  Same semantics as bst_attention_batch otherwise. */
int bst_attention_ragged(const void* q, int64_t q_tok_stride, void* out, int64_t o_tok_stride, const void* kv_cache,
                         int n_layers, int n_pages_total, int layer, const int32_t* page_table, int req_pages, int n_q,
                         int n_kv, int n_req, int s_max, const int32_t* row_off, const int32_t* row_cnt,
                         int keys_after_c, int max_keys, const int32_t* state, int req_state, int c_idx, int mode,
                         const uint32_t* anc, int mask_words, int n_splits, float* ws, size_t ws_bytes,
                         bst_stream_t stream);

/* ------------------------------------------------------------------------
 * K5 — fused elementwise epilogues of the target/drafter forward.
 * ---------------------------------------------------------------------- */
int bst_embed_rmsnorm(const int32_t* tokens, int rows, const void* emb, int h, const void* w, float eps, float* resid,
                      void* x, int64_t ldx, bst_stream_t stream);
/* Residual update from a dense y (the tensor-parallel all-reduced row-parallel output, fp32
 * or bf16 when y_bf16; NULL: normalise only): resid += y; x = RMSNorm(resid) * w. */
int bst_residual_dense(const void* y, int y_bf16, int64_t ldy, float* resid, int rows, int h, const void* w, float eps,
                       void* x, int64_t ldx, void* feat, int64_t ldf, bst_stream_t stream);
int bst_residual_rmsnorm(const float* partial, const bst_gemm_sched_t* sched, float* resid, int rows, int h,
                         const void* w, float eps, void* x, int64_t ldx, void* feat, int64_t ldf, bst_stream_t stream);
/* pos/slot are relative to c = state[c_idx]; slot == INT32_MIN skips the KV write,
 * qrow < 0 skips the q write. */
int bst_qkv_rope(const float* partial, const bst_gemm_sched_t* sched, int rows, int n_q, int n_kv, const void* q_norm,
                 const void* k_norm, float eps, const float* inv_freq /* [64] */, const int32_t* pos,
                 const int32_t* slot,
                 const int32_t* qrow, void* q_out, int64_t q_tok_stride, void* kv, int64_t layer_off_elems,
                 const int32_t* page_table, int page_size, const int32_t* state, int state_c_idx, bst_stream_t stream);
/* batched requests (req_rows > 0): row t belongs to request r = (t % req_span) / req_rows,
 * positions/slots are relative to c_r = state[r*req_state + c_idx] and slots are offset by
 * r*req_slots (request r's page range in a shared page table). */
int bst_qkv_rope_batch(const float* partial, const bst_gemm_sched_t* sched, int rows, int n_q, int n_kv,
                       const void* q_norm, const void* k_norm, float eps, const float* inv_freq, const int32_t* pos,
                       const int32_t* slot, const int32_t* qrow, void* q_out, int64_t q_tok_stride, void* kv,
                       int64_t layer_off_elems, const int32_t* page_table, int page_size, const int32_t* state,
                       int state_c_idx, int req_rows, int req_span, int req_state, int req_slots,
                       const int32_t* row_req /* ragged batch: request of each row, < 0 = padding; nullable */,
                       bst_stream_t stream);
int bst_swiglu(const float* partial, const bst_gemm_sched_t* sched, int rows, int ffn, void* act, int64_t lda,
               bst_stream_t stream);
/* dst[r] = src[*row_base + idx[r]] for r < *count (row_base nullable: 0), zero rows after. */
int bst_gather_rows(const void* src, int64_t lds, const int32_t* idx, const int32_t* count, int max_rows, int cols,
                    void* dst, int64_t ldd, const int32_t* row_base, bst_stream_t stream);

/* ------------------------------------------------------------------------
 * Decode-state plumbing of the on-device loop (no host round trip):
 * state[0]=c (cached tokens = root slot), [1]=n_new (pending drafter
 * context rows), [2]=bonus (pending root token), [3]=committed count.
 * ---------------------------------------------------------------------- */
enum { BST_ST_C = 0, BST_ST_NNEW = 1, BST_ST_BONUS = 2, BST_ST_COMMITTED = 3, BST_ST_CYCLE = 4 };
/* verify rows from the tree: token (root = bonus), pos = depth, slot = row;
 * rows beyond n_nodes are padding (token 0, pos 0, slot = row). */
int bst_verify_rows(const int32_t* state, const int32_t* tree_token, const int32_t* tree_depth, const int32_t* meta,
                    int rows, int32_t* tokens, int32_t* pos, int32_t* slot, bst_stream_t stream);
/* drafter rows: block rows 0..gamma (bonus, mask x gamma) at pos/slot 0..gamma;
 * ctx rows i < n_new at pos/slot i - n_new, the rest skipped. */
int bst_drafter_rows(const int32_t* state, int gamma, int mask_token, int ctx_rows, int32_t* tokens, int32_t* pos,
                     int32_t* slot, int32_t* qrow, bst_stream_t stream);
/* batched drafter rows: request r's gamma+1 block rows at [r*(gamma+1), ...) (qrow = row),
 * its ctx_rows context rows at [n_req*(gamma+1) + r*ctx_rows, ...); state words of
 * request r at state[r*req_state ...]. */
int bst_drafter_rows_batch(const int32_t* state, int req_state, int n_req, int gamma, int mask_token, int ctx_rows,
                           int32_t* tokens, int32_t* pos, int32_t* slot, int32_t* qrow, bst_stream_t stream);
/* after bst_accept: append committed tokens to out_tokens, c += len,
 * n_new = len, bonus = meta[1]; log this cycle (tree meta, len, c, bonus,
 * surrogate) at log[state[BST_ST_CYCLE]] (8 int32 + 1 f64 per cycle). */
int bst_commit_state(int32_t* state, const int32_t* accept_meta, const int32_t* committed, int max_path,
                     int32_t* out_tokens, int out_cap, const int32_t* tree_meta, const double* surrogate,
                     int32_t* log_i32, double* log_f64, int log_cap, bst_stream_t stream);

/* ------------------------------------------------------------------------
 * Ragged batched verify (extension beyond the reference's batch-1 controller,
 * PAPER.md:686).  Request r verifies s_r = N*_r + 1 rows, packed
 * request after request.
 * bst_ragged_rows: row_off/row_cnt [n_req], *total = sum s_r; tokens/pos/slot/row_req
 *   for rows [0, rows_cap) (root token = state bonus, pos = depth, slot = row in the
 *   tree; rows >= total: token 0, slot INT32_MIN, row_req -1).
 * bst_ragged_unpack: dst[r*s_max + i] = src[row_off[r] + i] (i < row_cnt[r]), else -1.
 * bst_batch_plan: out[r] = base[r] with the batch-aware verify cost: curve.flops_const /
 *   bytes_const += the other requests' flops / KV + activation bytes at their last tree
 *   sizes and contexts (weights counted once), a_offset = their surrogates (first != 0:
 *   no trees yet, every other request counts as its root row, surrogate 1).  One request:
 *   out == base, i.e. exactly run_cycle (controller.py:56-107).
 * ---------------------------------------------------------------------- */
int bst_ragged_rows(const bst_tree_t* trees_dev, const int32_t* state, int req_state, int n_req, int s_max,
                    int rows_cap, int32_t* row_off, int32_t* row_cnt, int32_t* total, int32_t* tokens, int32_t* pos,
                    int32_t* slot, int32_t* row_req, bst_stream_t stream);
int bst_ragged_unpack(const int32_t* src, const int32_t* row_off, const int32_t* row_cnt, int n_req, int s_max,
                      int32_t* dst, bst_stream_t stream);
int bst_batch_plan(const bst_plan_t* base_dev, bst_plan_t* out_dev, const bst_tree_t* trees_dev,
                   const int32_t* state, int req_state, int n_req, int first, bst_stream_t stream);
/* sizeof of the ABI structs (0 curve, 1 plan, 2 tree, 3 GEMM schedule) for binding checks. */
int bst_struct_size(int which);

#ifdef __cplusplus
}
#endif
#endif /* BASTION_H_ */
