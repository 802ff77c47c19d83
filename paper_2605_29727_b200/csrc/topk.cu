// K1 — drafter logits -> fp64 marginals -> top-K candidate lattice.
//
// Replaces the plugin softmax that produces MarginalBlock rows
// (lattice.py:24-55) fused with top_k_truncate (lattice.py:128-142).
// Ordering is (prob desc, token asc) on the FINAL fp64 probabilities, so the
// lattice equals top_k_truncate applied to the fp64 rows this kernel also
// emits (probs_full) — bit for bit.
//
// Logits (hot path): k1_fast_chunk (per chunk: max, fp64 sum, top-(K+1) by
// logit) -> k1_fast_finalize (per row: m, Z, exact fp64 probs of the K
// survivors, (prob desc, token asc) order, boundary check; in-CTA fallback)
// (exact full-row selection, only for rows whose K/K+1 boundary logits are
// distinct but < 1e-12 apart).  fp64 MarginalBlock rows are probs_full.
// fp64 probability input (top_k_truncate): exact chunked selection on the
// probabilities themselves (k1_chunk_select + k1_merge).
// The row is split in CHUNK-element chunks so gamma=16 rows of V=151936 fill
// ~600 CTAs (4 waves of 148 SMs) instead of 16.
#include <cuda_bf16.h>

#include "common.cuh"
#include "gemm.cuh"

namespace bst {

constexpr int TK_THREADS = 256;
constexpr int TK_PER_THREAD = 16;
constexpr int TK_CHUNK = TK_THREADS * TK_PER_THREAD;  // 4096
constexpr int TK_MAX_K = 256;

struct TopkWs {
  float* pmax;     // [gamma][chunks]
  double* psum;    // [gamma][chunks]
  double* cprob;   // [gamma][chunks][k]
  int32_t* ctok;   // [gamma][chunks][k]
  unsigned long long* ckeys;  // [gamma][chunks][k+1] (fast logits path)
  double* stats;   // [gamma][2] (m, Z)
  int* fallback;   // [gamma]
};

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static TopkWs carve(void* ws, int gamma, int chunks, int k, size_t* total) {
  char* p = static_cast<char*>(ws);
  TopkWs w;
  size_t off = 0;
  w.pmax = reinterpret_cast<float*>(p + off);
  off += align_up(sizeof(float) * gamma * chunks);
  w.psum = reinterpret_cast<double*>(p + off);
  off += align_up(sizeof(double) * gamma * chunks);
  w.cprob = reinterpret_cast<double*>(p + off);
  off += align_up(sizeof(double) * gamma * chunks * k);
  w.ctok = reinterpret_cast<int32_t*>(p + off);
  off += align_up(sizeof(int32_t) * gamma * chunks * k);
  w.ckeys = reinterpret_cast<unsigned long long*>(p + off);
  off += align_up(sizeof(unsigned long long) * gamma * chunks * (k + 1));
  w.stats = reinterpret_cast<double*>(p + off);
  off += align_up(sizeof(double) * gamma * 2);
  w.fallback = reinterpret_cast<int*>(p + off);
  off += align_up(sizeof(int) * gamma);
  *total = off;
  return w;
}

__device__ __forceinline__ float load_logit(const void* base, int dtype, int64_t idx) {
  if (dtype == 0) return __ldg(static_cast<const float*>(base) + idx);
  return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx]);
}

// Logit source of the fast path: an fp32/bf16 [gamma, stride] matrix, or the LM head's
// stream-K partial slots (the K4 GEMM output, summed here in the order gemm_reduce uses:
// slot 0, then the higher k ranges), so K1 reads the GEMM output without a reduce pass.
struct LogitSrc {
  const void* logits;
  int dtype;
  int64_t stride;
  const float* partial;  // non-null: partial slots of sched
  bst_gemm_sched_t sched;
};
__device__ __forceinline__ float src_logit(const LogitSrc& src, int row, int v) {
  if (src.partial) {
    const bst_gemm_sched_t& s = src.sched;
    const int tile = v >> 7;
    const int nslot = tile_nslot(s, tile);
    const float* p = src.partial + ((int64_t)tile * s.s_max * s.bn + row) * 128 + (v & 127);
    float acc = __ldg(p);
    for (int k = 1; k < nslot; ++k) acc += __ldg(p + (int64_t)k * s.bn * 128);
    return acc;
  }
  return load_logit(src.logits, src.dtype, (int64_t)row * src.stride + v);
}

__device__ __forceinline__ bool better(double pa, int ta, double pb, int tb) {
  return pa > pb || (pa == pb && ta < tb);
}

// --- A: chunk max ----------------------------------------------------------
__global__ void __launch_bounds__(TK_THREADS) k1_chunk_max(const void* logits, int dtype, int vocab,
                                                           int64_t stride, float* pmax) {
  pdl_enter();
  const int row = blockIdx.y, chunk = blockIdx.x, chunks = gridDim.x;
  const int64_t base = (int64_t)row * stride;
  float m = -INFINITY;
  for (int i = 0; i < TK_PER_THREAD; ++i) {
    int v = chunk * TK_CHUNK + i * TK_THREADS + threadIdx.x;
    if (v < vocab) m = fmaxf(m, load_logit(logits, dtype, base + v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[TK_THREADS / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = red[0];
    for (int w = 1; w < TK_THREADS / 32; ++w) r = fmaxf(r, red[w]);
    pmax[row * chunks + chunk] = r;
  }
}

__device__ __forceinline__ float row_max(const float* pmax, int row, int chunks) {
  // every block reduces the same small array in the same order
  float m = -INFINITY;
  for (int j = 0; j < chunks; ++j) m = fmaxf(m, pmax[row * chunks + j]);
  return m;
}

// --- B: chunk sum of exp(l - m) in fp64 (fixed reduction order) ------------
__global__ void __launch_bounds__(TK_THREADS) k1_chunk_sum(const void* logits, int dtype, int vocab,
                                                           int64_t stride, const float* pmax,
                                                           double* psum) {
  pdl_enter();
  const int row = blockIdx.y, chunk = blockIdx.x, chunks = gridDim.x;
  __shared__ float sm_m;
  if (threadIdx.x == 0) sm_m = row_max(pmax, row, chunks);
  __syncthreads();
  const double m = (double)sm_m;
  const int64_t base = (int64_t)row * stride;
  double s = 0.0;
  for (int i = 0; i < TK_PER_THREAD; ++i) {
    int v = chunk * TK_CHUNK + i * TK_THREADS + threadIdx.x;
    if (v < vocab) s = __dadd_rn(s, exp((double)load_logit(logits, dtype, base + v) - m));
  }
  s = warp_sum(s);
  __shared__ double red[TK_THREADS / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < TK_THREADS / 32; ++w) r = __dadd_rn(r, red[w]);
    psum[row * chunks + chunk] = r;
  }
}

// Block-wide argmax extraction of k winners over per-thread candidate lists.
// cand arrays are in registers (TK_PER_THREAD per thread); taken marks used.
__device__ void block_extract(double (&p)[TK_PER_THREAD], int (&t)[TK_PER_THREAD], int n_valid_per_thread,
                              int k, double* out_p, int32_t* out_t) {
  __shared__ double sp[TK_THREADS / 32];
  __shared__ int st[TK_THREADS / 32];
  __shared__ int sw[TK_THREADS / 32];
  __shared__ int win_thread, win_slot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = 0; r < k; ++r) {
    // local best
    double bp = -1.0;
    int bt = 0x7fffffff, bs = -1;
    for (int i = 0; i < n_valid_per_thread; ++i) {
      if (t[i] >= 0 && better(p[i], t[i], bp, bt)) { bp = p[i]; bt = t[i]; bs = i; }
    }
    int who = threadIdx.x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double op = __shfl_xor_sync(0xffffffffu, bp, o);
      int ot = __shfl_xor_sync(0xffffffffu, bt, o);
      int ow = __shfl_xor_sync(0xffffffffu, who, o);
      if (better(op, ot, bp, bt)) { bp = op; bt = ot; who = ow; }
    }
    if (lane == 0) { sp[warp] = bp; st[warp] = bt; sw[warp] = who; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double gp = sp[0];
      int gt = st[0], gw = sw[0];
      for (int w = 1; w < TK_THREADS / 32; ++w)
        if (better(sp[w], st[w], gp, gt)) { gp = sp[w]; gt = st[w]; gw = sw[w]; }
      out_p[r] = gp;
      out_t[r] = gt;
      win_thread = gw;
    }
    __syncthreads();
    if (threadIdx.x == win_thread) {
      // remove the winner from this thread's list
      int wi = -1;
      double wp = -1.0;
      int wt = 0x7fffffff;
      for (int i = 0; i < n_valid_per_thread; ++i)
        if (t[i] >= 0 && better(p[i], t[i], wp, wt)) { wp = p[i]; wt = t[i]; wi = i; }
      if (wi >= 0) t[wi] = -1;
      (void)win_slot;
    }
    __syncthreads();
  }
}

// --- C: probabilities + per-chunk top-k ------------------------------------
__global__ void __launch_bounds__(TK_THREADS) k1_chunk_select(const void* logits, int dtype,
                                                              const double* probs_in, int vocab,
                                                              int64_t stride, const float* pmax,
                                                              const double* psum, int k,
                                                              double* probs_full, double* cprob,
                                                              int32_t* ctok) {
  pdl_enter();
  const int row = blockIdx.y, chunk = blockIdx.x, chunks = gridDim.x;
  __shared__ double sm_z;
  __shared__ float sm_m;
  if (probs_in == nullptr && threadIdx.x == 0) {
    sm_m = row_max(pmax, row, chunks);
    double z = 0.0;
    for (int j = 0; j < chunks; ++j) z = __dadd_rn(z, psum[row * chunks + j]);
    sm_z = z;
  }
  __syncthreads();
  double p[TK_PER_THREAD];
  int t[TK_PER_THREAD];
  const int64_t base = (int64_t)row * stride;
  for (int i = 0; i < TK_PER_THREAD; ++i) {
    int v = chunk * TK_CHUNK + i * TK_THREADS + threadIdx.x;
    if (v < vocab) {
      double q;
      if (probs_in != nullptr) {
        q = probs_in[base + v];
      } else {
        q = __ddiv_rn(exp((double)load_logit(logits, dtype, base + v) - (double)sm_m), sm_z);
        if (probs_full) probs_full[(int64_t)row * vocab + v] = q;
      }
      p[i] = q;
      t[i] = v;
    } else {
      p[i] = -1.0;
      t[i] = -1;
    }
  }
  const int kk = min(k, min(TK_CHUNK, vocab - chunk * TK_CHUNK));
  double* op = cprob + ((int64_t)row * chunks + chunk) * k;
  int32_t* ot = ctok + ((int64_t)row * chunks + chunk) * k;
  block_extract(p, t, TK_PER_THREAD, kk, op, ot);
  if (threadIdx.x == 0)
    for (int r = kk; r < k; ++r) { op[r] = -1.0; ot[r] = -1; }
}

// --- D: merge chunk candidates of one row ----------------------------------
__global__ void __launch_bounds__(TK_THREADS) k1_merge(const double* cprob, const int32_t* ctok, int chunks,
                                                       int k, int32_t* tok_out, double* prob_out) {
  pdl_enter();
  const int row = blockIdx.x;
  const int n = chunks * k;
  double p[TK_PER_THREAD];
  int t[TK_PER_THREAD];
  for (int i = 0; i < TK_PER_THREAD; ++i) {
    int j = i * TK_THREADS + threadIdx.x;
    if (j < n) {
      p[i] = cprob[(int64_t)row * n + j];
      t[i] = ctok[(int64_t)row * n + j];
    } else {
      p[i] = -1.0;
      t[i] = -1;
    }
  }
  block_extract(p, t, TK_PER_THREAD, k, prob_out + (int64_t)row * k, tok_out + (int64_t)row * k);
}


// ===========================================================================
// Fast path for logits (default): top-(K+1) by (logit desc, token asc) per
// chunk, then exact fp64 probabilities for the survivors only.
// prob_v = exp64(l_v - m) / Z is non-decreasing in l_v, so the top-K by
// (prob desc, token asc) equals the top-K by (logit desc, token asc) unless two
// DISTINCT logits at the K boundary are within 1e-12 (where fp64 rounding could
// tie or swap them) — that row then takes the exact full-row path.
// ===========================================================================
constexpr int TK_KP_MAX = 65;

__device__ __forceinline__ unsigned long long logit_key(float l, int tok) {
  unsigned int b = __float_as_uint(l);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)b << 32) | (0xFFFFFFFFu - (unsigned)tok);
}
__device__ __forceinline__ float key_logit(unsigned long long k) {
  unsigned int b = (unsigned int)(k >> 32);
  b = (b & 0x80000000u) ? (b & 0x7FFFFFFFu) : ~b;
  return __uint_as_float(b);
}
__device__ __forceinline__ int key_tok(unsigned long long k) { return (int)(0xFFFFFFFFu - (unsigned)(k & 0xFFFFFFFFu)); }

// block-wide: top-n keys (descending) of per-thread candidate lists.  Each warp first
// extracts its own top-n with warp shuffles (no block barrier per round), then warp 0
// merges the warps' candidates; keys are unique (token in the low bits).
__device__ void block_top_keys(unsigned long long (&c)[TK_PER_THREAD], int n, unsigned long long* out) {
  constexpr int NW = TK_THREADS / 32;
  constexpr int PL = (NW * TK_KP_MAX + 31) / 32;  // merge candidates per lane of warp 0
  __shared__ unsigned long long cand[NW][TK_KP_MAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = 0; r < n; ++r) {
    unsigned long long b = 0;
#pragma unroll
    for (int i = 0; i < TK_PER_THREAD; ++i) b = c[i] > b ? c[i] : b;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
      b = ob > b ? ob : b;
    }
    if (lane == 0) cand[warp][r] = b;
#pragma unroll
    for (int i = 0; i < TK_PER_THREAD; ++i)
      if (c[i] == b) c[i] = 0;
  }
  __syncthreads();
  if (warp == 0) {
    unsigned long long m[PL];
#pragma unroll
    for (int i = 0; i < PL; ++i) {
      const int j = i * 32 + lane;  // candidate j = (warp j / n, rank j % n)
      m[i] = j < NW * n ? cand[j / n][j % n] : 0ull;
    }
    for (int r = 0; r < n; ++r) {
      unsigned long long b = 0;
#pragma unroll
      for (int i = 0; i < PL; ++i) b = m[i] > b ? m[i] : b;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
        b = ob > b ? ob : b;
      }
      if (lane == 0) out[r] = b;
#pragma unroll
      for (int i = 0; i < PL; ++i)
        if (m[i] == b) m[i] = 0;
    }
  }
  __syncthreads();
}

// A: per (chunk, row): fp32 max m_c, fp64 S_c = sum exp(l - m_c), top-(K+1) keys
__global__ void __launch_bounds__(TK_THREADS) k1_fast_chunk(LogitSrc src, int vocab, int kp, float* pmax, double* psum,
                                                            unsigned long long* ckeys) {
  pdl_enter();
  const int row = blockIdx.y, chunk = blockIdx.x, chunks = gridDim.x;
  float l[TK_PER_THREAD];
  unsigned long long key[TK_PER_THREAD];
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < TK_PER_THREAD; ++i) {
    const int v = chunk * TK_CHUNK + i * TK_THREADS + threadIdx.x;
    if (v < vocab) {
      l[i] = src_logit(src, row, v);
      key[i] = logit_key(l[i], v);
      m = fmaxf(m, l[i]);
    } else {
      l[i] = -INFINITY;
      key[i] = 0;
    }
  }
  __shared__ float wm[TK_THREADS / 32];
  __shared__ double ws_[TK_THREADS / 32];
  __shared__ float sm_m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = wm[0];
    for (int w = 1; w < TK_THREADS / 32; ++w) r = fmaxf(r, wm[w]);
    sm_m = r;
  }
  __syncthreads();
  const double mc = (double)sm_m;
  double sacc = 0.0;
#pragma unroll
  for (int i = 0; i < TK_PER_THREAD; ++i)
    if (key[i]) sacc = __dadd_rn(sacc, exp((double)l[i] - mc));
  sacc = warp_sum(sacc);
  if ((threadIdx.x & 31) == 0) ws_[threadIdx.x >> 5] = sacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < TK_THREADS / 32; ++w) r = __dadd_rn(r, ws_[w]);
    pmax[row * chunks + chunk] = sm_m;
    psum[row * chunks + chunk] = r;
  }
  block_top_keys(key, kp, ckeys + ((int64_t)row * chunks + chunk) * kp);
}

__device__ void k1_fallback_row(const LogitSrc& src, int vocab, int row, double m, double z, int k, int32_t* tok_out,
                                double* prob_out);

// B: per row: m, Z (fixed order), global top-(K+1), exact fp64 probs, boundary check; a
// row whose K-th / (K+1)-th logits are distinct but < 1e-12 apart redoes the selection on
// the exact fp64 probabilities of the whole row in the same CTA (k1_fallback_row)
__global__ void __launch_bounds__(TK_THREADS) k1_fast_finalize(const float* pmax, const double* psum,
                                                               const unsigned long long* ckeys, int chunks, int kp,
                                                               int k, int32_t* tok_out, double* prob_out,
                                                               double* stats, int* fallback, LogitSrc src, int vocab) {
  pdl_enter();
  __shared__ int fb_sh;
  const int row = blockIdx.x;
  const int n = chunks * kp;
  unsigned long long c[TK_PER_THREAD];
#pragma unroll
  for (int i = 0; i < TK_PER_THREAD; ++i) {
    const int j = i * TK_THREADS + threadIdx.x;
    c[i] = j < n ? ckeys[(int64_t)row * n + j] : 0ull;
  }
  __shared__ unsigned long long top[TK_KP_MAX];
  block_top_keys(c, kp, top);
  if (threadIdx.x == 0) {
    float mf = -INFINITY;
    for (int j = 0; j < chunks; ++j) mf = fmaxf(mf, pmax[row * chunks + j]);
    const double m = (double)mf;
    double z = 0.0;
    for (int j = 0; j < chunks; ++j)
      z = __dadd_rn(z, __dmul_rn(exp((double)pmax[row * chunks + j] - m), psum[row * chunks + j]));
    stats[row * 2] = m;
    stats[row * 2 + 1] = z;
    // boundary: the K-th and (K+1)-th by logit must be equal or >= 1e-12 apart
    int fb = 0;
    if (kp > k && top[k] != 0ull) {
      const double gap = (double)key_logit(top[k - 1]) - (double)key_logit(top[k]);
      if (gap > 0.0 && gap < 1e-12) fb = 1;
    }
    fallback[row] = fb;
    fb_sh = fb;
    // exact probabilities, then (prob desc, token asc) insertion sort of the K survivors
    double p[TK_KP_MAX];
    int t[TK_KP_MAX];
    for (int j = 0; j < k; ++j) {
      t[j] = key_tok(top[j]);
      p[j] = __ddiv_rn(exp((double)key_logit(top[j]) - m), z);
    }
    for (int a = 1; a < k; ++a) {
      const double pa = p[a];
      const int ta = t[a];
      int b = a - 1;
      while (b >= 0 && (p[b] < pa || (p[b] == pa && t[b] > ta))) {
        p[b + 1] = p[b];
        t[b + 1] = t[b];
        --b;
      }
      p[b + 1] = pa;
      t[b + 1] = ta;
    }
    for (int j = 0; j < k; ++j) {
      tok_out[row * k + j] = t[j];
      prob_out[row * k + j] = p[j];
    }
  }
  __syncthreads();
  if (fb_sh) k1_fallback_row(src, vocab, row, stats[row * 2], stats[row * 2 + 1], k, tok_out, prob_out);
}

// Full fp64 rows (MarginalBlock export) with the same m and Z.
__global__ void __launch_bounds__(TK_THREADS) k1_full_rows(const void* logits, int dtype, int vocab, int64_t stride,
                                                           const double* stats, double* probs_full) {
  pdl_enter();
  const int row = blockIdx.y;
  const double m = stats[row * 2], z = stats[row * 2 + 1];
  for (int v = blockIdx.x * TK_THREADS + threadIdx.x; v < vocab; v += gridDim.x * TK_THREADS)
    probs_full[(int64_t)row * vocab + v] =
        __ddiv_rn(exp((double)load_logit(logits, dtype, (int64_t)row * stride + v) - m), z);
}

// Exact fallback: rows flagged by the boundary check redo the selection on the
// fp64 probabilities of the whole row (single CTA per flagged row).
__device__ void k1_fallback_row(const LogitSrc& src, int vocab, int row, double m, double z, int k, int32_t* tok_out,
                                double* prob_out) {
  // running top-k over the row: per 4096-element block, merge the block's top-k with the current list
  __shared__ double cur_p[TK_MAX_K];
  __shared__ int cur_t[TK_MAX_K];
  __shared__ double blk_p[TK_MAX_K];
  __shared__ int32_t blk_t[TK_MAX_K];
  if (threadIdx.x == 0)
    for (int j = 0; j < k; ++j) { cur_p[j] = -1.0; cur_t[j] = 0x7fffffff; }
  __syncthreads();
  for (int b0 = 0; b0 < vocab; b0 += TK_CHUNK) {
    double p[TK_PER_THREAD];
    int t[TK_PER_THREAD];
    for (int i = 0; i < TK_PER_THREAD; ++i) {
      const int v = b0 + i * TK_THREADS + threadIdx.x;
      if (v < vocab) {
        p[i] = __ddiv_rn(exp((double)src_logit(src, row, v) - m), z);
        t[i] = v;
      } else {
        p[i] = -1.0;
        t[i] = -1;
      }
    }
    block_extract(p, t, TK_PER_THREAD, min(k, vocab - b0), blk_p, blk_t);
    if (threadIdx.x == 0) {
      const int nb = min(k, vocab - b0);
      double mp[2 * TK_MAX_K];
      int mt[2 * TK_MAX_K];
      int a = 0, b = 0, o = 0;
      while (o < k && (a < k || b < nb)) {
        const bool take_a = b >= nb || (a < k && better(cur_p[a], cur_t[a], blk_p[b], blk_t[b]));
        mp[o] = take_a ? cur_p[a] : blk_p[b];
        mt[o] = take_a ? cur_t[a] : blk_t[b];
        if (take_a) ++a; else ++b;
        ++o;
      }
      for (int j = 0; j < k; ++j) { cur_p[j] = mp[j]; cur_t[j] = mt[j]; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int j = 0; j < k; ++j) { tok_out[row * k + j] = cur_t[j]; prob_out[row * k + j] = cur_p[j]; }
}

static int run_topk(const void* logits, int dtype, const double* probs_in, int gamma, int vocab, int64_t stride,
                    int k, int32_t* tok, double* prob, double* probs_full, void* ws, size_t ws_bytes,
                    cudaStream_t st, const float* partial = nullptr, const bst_gemm_sched_t* sched = nullptr) {
  BST_REQUIRE(gamma >= 1, "gamma must be >= 1, got %d", gamma);
  BST_REQUIRE(vocab >= 2, "vocab_size must be >= 2, got %d", vocab);
  BST_REQUIRE(k >= 1 && k <= vocab, "k must be in [1, %d], got %d", vocab, k);
  BST_REQUIRE(k <= TK_MAX_K, "k=%d exceeds the kernel limit %d", k, TK_MAX_K);
  BST_REQUIRE(stride >= vocab, "row stride %lld < vocab %d", (long long)stride, vocab);
  const int chunks = (vocab + TK_CHUNK - 1) / TK_CHUNK;
  BST_REQUIRE((int64_t)chunks * k <= TK_CHUNK, "vocab*k too large for one merge block");
  size_t need = 0;
  TopkWs w = carve(ws, gamma, chunks, k, &need);
  BST_REQUIRE(ws != nullptr && ws_bytes >= need, "workspace too small: %zu < %zu", ws_bytes, need);
  dim3 grid(chunks, gamma);
  const int kp = k + 1 <= vocab ? k + 1 : k;
  LogitSrc src{logits, dtype, stride, partial, sched ? *sched : bst_gemm_sched_t{}};
  BST_REQUIRE(!partial || (probs_in == nullptr && probs_full == nullptr && kp < TK_KP_MAX &&
                           (int64_t)chunks * kp <= TK_CHUNK),
              "K1 over GEMM partials: fast path only, no full-row export");
  if (probs_in == nullptr && kp < TK_KP_MAX && (int64_t)chunks * kp <= TK_CHUNK) {
    BST_CUDA(launch_pdl(k1_fast_chunk, dim3(grid), dim3(TK_THREADS), 0, st, src, vocab, kp, w.pmax, w.psum, w.ckeys));
    BST_CUDA(launch_pdl(k1_fast_finalize, dim3(gamma), dim3(TK_THREADS), 0, st, w.pmax, w.psum, w.ckeys, chunks, kp, k, tok,
                        prob, w.stats, w.fallback, src, vocab));
    if (probs_full) BST_CUDA(launch_pdl(k1_full_rows, dim3(dim3(chunks, gamma)), dim3(TK_THREADS), 0, st, logits, dtype, vocab, stride, w.stats,
                                                                            probs_full));
    BST_LAUNCH_CHECK();
    return BST_OK;
  }
  if (probs_in == nullptr) {
    BST_CUDA(launch_pdl(k1_chunk_max, dim3(grid), dim3(TK_THREADS), 0, st, logits, dtype, vocab, stride, w.pmax));
    BST_CUDA(launch_pdl(k1_chunk_sum, dim3(grid), dim3(TK_THREADS), 0, st, logits, dtype, vocab, stride, w.pmax, w.psum));
  }
  BST_CUDA(launch_pdl(k1_chunk_select, dim3(grid), dim3(TK_THREADS), 0, st, logits, dtype, probs_in, vocab, stride, w.pmax, w.psum, k,
                                               probs_full, w.cprob, w.ctok));
  BST_CUDA(launch_pdl(k1_merge, dim3(gamma), dim3(TK_THREADS), 0, st, w.cprob, w.ctok, chunks, k, tok, prob));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

}  // namespace bst

extern "C" size_t bst_topk_workspace(int gamma, int vocab, int k) {
  if (gamma < 1 || vocab < 1 || k < 1) return 0;
  size_t need = 0;
  const int chunks = (vocab + bst::TK_CHUNK - 1) / bst::TK_CHUNK;
  bst::carve(nullptr, gamma, chunks, k, &need);
  return need;
}

extern "C" int bst_topk_logits(const void* logits, int dtype, int gamma, int vocab, int64_t row_stride, int k,
                               int32_t* tok, double* prob, double* probs_full, void* ws, size_t ws_bytes,
                               bst_stream_t stream) {
  BST_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 (fp32) or 1 (bf16), got %d", dtype);
  BST_REQUIRE(logits && tok && prob, "null pointer argument");
  return bst::run_topk(logits, dtype, nullptr, gamma, vocab, row_stride, k, tok, prob, probs_full, ws, ws_bytes,
                       bst::as_stream(stream));
}

extern "C" int bst_topk_gemm_partial(const float* partial, const bst_gemm_sched_t* sched, int gamma, int vocab, int k,
                                     int32_t* tok, double* prob, void* ws, size_t ws_bytes, bst_stream_t stream) {
  BST_REQUIRE(partial && sched && tok && prob, "null pointer argument");
  BST_REQUIRE(sched->n_out == vocab && sched->m >= gamma, "schedule (n_out=%d, m=%d) does not cover %d x %d logits",
              sched->n_out, sched->m, gamma, vocab);
  return bst::run_topk(nullptr, 0, nullptr, gamma, vocab, vocab, k, tok, prob, nullptr, ws, ws_bytes,
                       bst::as_stream(stream), partial, sched);
}

extern "C" int bst_topk_probs(const double* probs, int gamma, int vocab, int k, int32_t* tok, double* prob,
                              void* ws, size_t ws_bytes, bst_stream_t stream) {
  BST_REQUIRE(probs && tok && prob, "null pointer argument");
  return bst::run_topk(nullptr, 0, probs, gamma, vocab, vocab, k, tok, prob, nullptr, ws, ws_bytes,
                       bst::as_stream(stream));
}
