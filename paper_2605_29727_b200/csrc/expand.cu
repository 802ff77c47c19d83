// K2 — best-first / adaptive / beam tree expansion on one CTA.
//
// Replaces ExpansionFrontier + iter_best_first + best_first_expand
// (draft_tree.py:69-155), run_cycle (controller.py:56-107, incl.
// LatencyCurve.latency cost_model.py:305-309) and beam_expand
// (draft_tree.py:158-189).
//
// Best-first without a heap.  The reference pops nodes in increasing key
// (-rho, depth, token, parent_pop_index); a node's parent and previous sibling
// always have a strictly smaller key, so the lazy child/sibling heap pops the
// GLOBAL key order of all positive-rho lattice nodes.  We therefore:
//   1. estimate a threshold tau with a log-bin histogram DP over the lattice
//      (conservative: at least min(n_max, reachable) nodes have rho >= tau);
//   2. enumerate {rho >= tau} level by level (prefix-closed, exact fp64 rho =
//      rho_parent * p as in draft_tree.py:102,113);
//   3. bitonic-sort by (-rho, depth, token, enumeration index) and repair the
//      rare exact ties of (rho, depth, token) by the parent's final position,
//      depth by depth;
//   4. run Algorithm 1's S_hat scan: sequential fp64 a_hat (one thread, same
//      addition order as controller.py:85), parallel S_hat, first strict
//      decrease via a block prefix-max.
// If the enumeration would exceed the shared-memory capacity (pathological
// ties / flat rows) the same kernel falls back to the reference's sequential
// lazy heap on thread 0 — still exact, just slower.
// Compiled with -fmad=false; every fp64 op below is also explicitly _rn.
#include "common.cuh"

namespace bst {

constexpr int EX_THREADS = 1024;
constexpr int EX_WARPS = EX_THREADS / 32;
constexpr int EX_CAP = 8192;   // enumerated-node capacity of the sort path
constexpr int EX_BINS = 4096;  // histogram bins of the threshold DP
constexpr int EX_MAXG = 127;
constexpr int EX_MAXK = 128;
constexpr int EX_PASS1 = 256;  // adaptive: nodes planned by the first pass
constexpr unsigned short NO_PARENT = 0xFFFF;

__device__ long long* g_ex_trace = nullptr;
__device__ __forceinline__ void ex_trace(int k) {
#ifdef BST_TRACE  // phase tracing (scripts/expand_trace.py); compiled out by default
  if (g_ex_trace && threadIdx.x == 0 && k < 16) {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_ex_trace[k] = t;
  }
#else
  (void)k;
#endif
}

struct HeapEntry {
  double rho;
  unsigned long long lo;  // depth<<44 | token<<20 | parent
  int rank;
  int _pad;
};

__device__ __forceinline__ bool heap_less(const HeapEntry& a, const HeapEntry& b) {
  // smaller key pops first: rho desc, then (depth, token, parent) asc
  return a.rho > b.rho || (a.rho == b.rho && a.lo < b.lo);
}

// ---------------------------------------------------------------- block scans
__device__ int block_excl_scan(int v, int* sh, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    sh[lane] = t;
  }
  __syncthreads();
  int before = (w > 0) ? sh[w - 1] : 0;
  *total = sh[EX_WARPS - 1];
  __syncthreads();
  return before + x - v;
}

// exclusive prefix-max of doubles (identity -inf)
__device__ double block_excl_max(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = fmax(x, y);
  }
  double excl_in_warp = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) excl_in_warp = -INFINITY;
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    double t = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t = fmax(t, y);
    }
    sh[lane] = t;
  }
  __syncthreads();
  double before = (w > 0) ? sh[w - 1] : -INFINITY;
  __syncthreads();
  return fmax(before, excl_in_warp);
}

// ------------------------------------------------------------ shared layout
struct ExSmem {
  unsigned long long hi[EX_CAP];  // ~rho bits (ascending = rho desc); DP aliases here
  unsigned long long lo[EX_CAP];  // depth<<40 | token<<16 | idx
  unsigned short par[EX_CAP];     // enumeration index of parent (NO_PARENT for depth 1)
  unsigned short pos[EX_CAP];     // sorted position of each enumeration index
  unsigned char rnk[EX_CAP];
  unsigned short runs[EX_CAP / 2];
  int lvl_start[EX_MAXG + 2];
  int scan[EX_WARPS];
  double dscan[EX_WARPS];
  int n_runs, overflow, n_enum, all_enumerated, min_stop, best_idx, max_depth;
  double best_val;
  double tau;
  double lat_p[2048];  // lattice staged in smem when gamma*k <= 2048
  int lat_t[2048];
};

struct ExWs {
  double* ahat;     // [n_cap]
  double* shat;     // [n_cap] (used when out->trace is null)
  int* counts;      // [n_cap + 2]
  HeapEntry* heap;  // [2 * n_cap + 4]
};

static size_t ex_align(size_t x) { return (x + 255) & ~size_t(255); }

static ExWs ex_carve(void* ws, int n_cap, size_t* total) {
  char* p = static_cast<char*>(ws);
  ExWs w;
  size_t off = 0;
  w.ahat = reinterpret_cast<double*>(p + off);
  off += ex_align(sizeof(double) * (n_cap + 1));
  w.shat = reinterpret_cast<double*>(p + off);
  off += ex_align(sizeof(double) * (n_cap + 1));
  w.counts = reinterpret_cast<int*>(p + off);
  off += ex_align(sizeof(int) * (n_cap + 2));
  w.heap = reinterpret_cast<HeapEntry*>(p + off);
  off += ex_align(sizeof(HeapEntry) * (2 * (size_t)n_cap + 4));
  *total = off;
  return w;
}

// --------------------------------------------------- threshold estimate (DP)
// Returns tau such that #{lattice nodes with rho >= tau} >= min(n_max, reachable),
// or 0.0 meaning "enumerate every positive node".
__device__ double estimate_tau(const double* prob, int gamma, int k, int n_max, ExSmem& sm) {
  unsigned int* hprev = reinterpret_cast<unsigned int*>(sm.hi);
  unsigned int* hcur = hprev + EX_BINS;
  unsigned int* tot = hcur + EX_BINS;
  const unsigned int SAT = 1u << 30;
  __shared__ int s_bstar;
  int* cost = reinterpret_cast<int*>(sm.lo);  // [gamma*k] quantized -log2(p), lo is free here
  __shared__ int s_range, s_cross;
  for (int pass = 0; pass < 4; ++pass) {
    // pass 0: 1/16-bit bins up to 2^-16 (the usual crossing: a quarter of the bins, a quarter
    // of the instructions per level); pass 1: up to 2^-64 (typical drafter rows); pass 2: up
    // to 2^-256; pass 3: 1/2-bit bins covering the whole fp64 range.  Bins below a pass's
    // range get the same counts in every pass (the convolution only reads lower bins), so
    // the first crossing — and tau — do not depend on the pass that finds it.
    const double S = pass < 3 ? 16.0 : 2.0;
    const int max_range = pass == 0 ? 256 : (pass == 1 ? 1024 : EX_BINS);
    // est cost = floor(-log2(p) * S) + 1 >= the true scaled cost, so a path's
    // summed est cost never undercounts: est <= B  =>  rho > 2^(-(B+1)/S).
    for (int e = threadIdx.x; e < gamma * k; e += EX_THREADS) {
      double p = __ldg(prob + e);
      double c = p > 0.0 ? floor(-log2(p) * S) + 1.0 : -1.0;
      cost[e] = c < 0.0 ? -1 : (c < EX_BINS ? (int)c : EX_BINS);
    }
    for (int b = threadIdx.x; b < EX_BINS; b += EX_THREADS) { hprev[b] = 0; tot[b] = 0; }
    if (threadIdx.x == 0) { s_range = max_range; s_cross = 0; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int r = 0; r < k; ++r)
        if (cost[r] >= 0 && cost[r] < EX_BINS) hprev[cost[r]] += 1;
    }
    __syncthreads();
    for (int b = threadIdx.x; b < EX_BINS; b += EX_THREADS) tot[b] = hprev[b];
    __syncthreads();
    // first bin whose cumulative count (capped per bin at n_max) reaches n_max
    auto crossing = [&](int range) {
      const int per = (range + EX_THREADS - 1) / EX_THREADS;
      const int b0 = threadIdx.x * per;
      int loc = 0;
      for (int b = b0; b < min(b0 + per, range); ++b) loc += (int)min((unsigned int)n_max, tot[b]);
      int total;
      int run = block_excl_scan(loc, sm.scan, &total);
      if (total >= n_max) {
        for (int b = b0; b < min(b0 + per, range); ++b) {
          run += (int)min((unsigned int)n_max, tot[b]);
          if (run >= n_max) {
            atomicMin(&s_range, b + 1);
            s_cross = 1;
            break;
          }
        }
      }
      __syncthreads();
    };
    // level-by-level convolution of the path-cost histogram over every bin < max_range
    // (one bin per thread for pass 0, ping-pong buffers: one barrier per level); the
    // crossing is located once at the end — tot only grows with the levels, so the first
    // crossing bin is the same as tracking it level by level
    unsigned int* hp = hprev;
    unsigned int* hc = hcur;
    for (int d = 2; d <= gamma; ++d) {
      int cr[8];
      int nk = 0;
      for (int r = 0; r < k && r < 8; ++r) {
        cr[r] = cost[(d - 1) * k + r];
        if (cr[r] >= 0) nk = r + 1;
      }
      for (int b = threadIdx.x; b < max_range; b += EX_THREADS) {
        unsigned long long acc = 0;
        if (k <= 8) {
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (r < nk && cr[r] <= b) acc += hp[b - cr[r]];
        } else {
          for (int r = 0; r < k; ++r) {
            const int ci = cost[(d - 1) * k + r];
            if (ci < 0) break;
            if (ci <= b) acc += hp[b - ci];
          }
        }
        const unsigned int a32 = acc > SAT ? SAT : (unsigned int)acc;
        hc[b] = a32;
        const unsigned long long t = (unsigned long long)tot[b] + a32;
        tot[b] = t > SAT ? SAT : (unsigned int)t;
      }
      __syncthreads();
      unsigned int* tmp = hp;
      hp = hc;
      hc = tmp;
    }
    crossing(max_range);
    if (threadIdx.x == 0) s_bstar = s_cross ? s_range - 1 : -1;
    __syncthreads();
    int bstar = s_bstar;
    __syncthreads();
    if (bstar >= 0) return exp2(-(double)(bstar + 1) / S);
  }
  return 0.0;
}

// ------------------------------------------------------------- enumeration
// Enumerate every node with rho >= tau (rho > 0).  Returns false on overflow.
// Level d's candidates are the (parent at level d-1, lattice rank) pairs; a row's
// probabilities are sorted descending, so the kept children of a parent are a prefix
// (the reference's break at the first child below tau).  Slots inside a level come from
// warp-aggregated atomics: the enumeration order inside a level is arbitrary, which is
// safe because the final order is the sort by (rho, depth, token) with exact ties
// repaired by the parent's sorted position (fix_ties), never by enumeration index.
__device__ bool enumerate_nodes(const int32_t* tok, const double* prob, int gamma, int k, double tau,
                                ExSmem& sm) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { sm.n_enum = 0; sm.overflow = 0; sm.lvl_start[1] = 0; sm.max_depth = 0; }
  __syncthreads();
  int prev_lo = 0, prev_hi = 0;  // enumeration range of the previous level (root for d=1)
  for (int d = 1; d <= gamma; ++d) {
    const double* pr = prob + (size_t)(d - 1) * k;
    const int32_t* tr = tok + (size_t)(d - 1) * k;
    const int n_par = d == 1 ? 1 : prev_hi - prev_lo;
    const int base = sm.lvl_start[d];
    const int n_items = n_par * k;
    for (int i0 = 0; i0 < n_items; i0 += EX_THREADS) {
      const int item = i0 + threadIdx.x;
      int pi = 0, r = 0;
      double v = 0.0;
      bool take = false;
      if (item < n_items) {
        pi = item / k;
        r = item - pi * k;
        const double prho = d == 1 ? 1.0 : bitsd(~sm.hi[prev_lo + pi]);
        v = __dmul_rn(prho, pr[r]);
        take = v > 0.0 && !(v < tau);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      int slot0 = 0;
      if (lane == 0 && bal) slot0 = atomicAdd(&sm.n_enum, __popc(bal));
      slot0 = __shfl_sync(0xffffffffu, slot0, 0);
      if (take) {
        const int w = slot0 + __popc(bal & ((1u << lane) - 1u));
        if (w < EX_CAP) {
          sm.hi[w] = ~dbits(v);
          sm.lo[w] = ((unsigned long long)d << 40) | ((unsigned long long)(unsigned)tr[r] << 16) |
                     (unsigned long long)w;
          sm.par[w] = d == 1 ? NO_PARENT : (unsigned short)(prev_lo + pi);
          sm.rnk[w] = (unsigned char)r;
        } else {
          sm.overflow = 1;
        }
      }
    }
    __syncthreads();
    const int top = sm.n_enum;
    if (sm.overflow || top > EX_CAP) return false;
    const int total = top - base;
    if (threadIdx.x == 0) {
      sm.lvl_start[d + 1] = top;
      if (total > 0) sm.max_depth = d;
    }
    __syncthreads();
    if (total == 0) break;
    prev_lo = base;
    prev_hi = top;
  }
  return true;
}

__device__ __forceinline__ bool key_gt(unsigned long long ah, unsigned long long al, unsigned long long bh,
                                       unsigned long long bl) {
  return ah > bh || (ah == bh && al > bl);
}

// Compare-exchange helpers of the register stages: 128-bit keys (hi, lo), unique except
// the ~0 padding (equal keys never swap).
__device__ __forceinline__ void reg_cas(unsigned long long& ah, unsigned long long& al, unsigned long long& bh,
                                        unsigned long long& bl, bool asc) {
  if (key_gt(ah, al, bh, bl) == asc) {
    unsigned long long th = ah, tl = al;
    ah = bh; al = bl; bh = th; bl = tl;
  }
}
__device__ __forceinline__ void reg_xchg(unsigned long long& h, unsigned long long& l, int j, bool lower, bool asc) {
  const unsigned long long oh = __shfl_xor_sync(0xffffffffu, h, j), ol = __shfl_xor_sync(0xffffffffu, l, j);
  // the lower position keeps the smaller key when ascending, the larger when descending
  const bool other_smaller = key_gt(h, l, oh, ol);
  if (lower == asc ? other_smaller : !other_smaller && !(oh == h && ol == l)) { h = oh; l = ol; }
}

// Bitonic sort of (hi, lo) over p2 = next power of two >= max(n, 64) keys.  Stages with
// j >= 64 compare across warp blocks through shared memory (block / named barrier per
// stage); each run of stages with j <= 32 touches only one aligned block of 64 keys per
// warp and runs in registers (2 keys per lane: block positions lane and lane + 32; j = 32
// inside the lane, j <= 16 by shuffles), so shared memory is read and written once per run.
__device__ void bitonic_sort(ExSmem& sm, int n) {
  int p2 = 64;
  while (p2 < n) p2 <<= 1;
  for (int i = n + threadIdx.x; i < p2; i += EX_THREADS) { sm.hi[i] = ~0ull; sm.lo[i] = ~0ull; }
  __syncthreads();
  const int active = min(EX_THREADS, p2 >> 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = active >> 5;
  auto bar = [&]() {
    if (active == EX_THREADS) __syncthreads();
    else asm volatile("bar.sync 2, %0;" ::"r"(active));
  };
  if (threadIdx.x < active) {
    for (int kk = 2; kk <= p2; kk <<= 1) {
      int j = kk >> 1;
      for (; j >= 64; j >>= 1) {  // cross-block stages
        for (int i = threadIdx.x; i < (p2 >> 1); i += active) {
          const int a = ((i & ~(j - 1)) << 1) | (i & (j - 1));
          const int b = a + j;
          const bool asc = (a & kk) == 0;
          unsigned long long ah = sm.hi[a], al = sm.lo[a], bh = sm.hi[b], bl = sm.lo[b];
          if (key_gt(ah, al, bh, bl) == asc) {
            sm.hi[a] = bh; sm.lo[a] = bl; sm.hi[b] = ah; sm.lo[b] = al;
          }
        }
        bar();
      }
      // register run: stages j .. 1 (j <= 32); for kk <= 64 the runs of kk = 2 .. 64 merge
      if (kk < 64 && kk < p2) continue;  // handled by the kk = 64 run below
      for (int blk = warp; blk < (p2 >> 6); blk += nwarps) {
        const int base = blk << 6;
        const int p0 = base + lane, p1 = p0 + 32;
        unsigned long long h0 = sm.hi[p0], l0 = sm.lo[p0], h1 = sm.hi[p1], l1 = sm.lo[p1];
        const int k_lo = kk <= 64 ? 2 : kk;  // first stage group of this run
        for (int kq = k_lo; kq <= kk; kq <<= 1) {
          for (int jj = (kq == kk ? min(j, 32) : (kq >> 1)); jj > 0; jj >>= 1) {
            if (jj == 32) {
              reg_cas(h0, l0, h1, l1, (p0 & kq) == 0);
            } else {
              reg_xchg(h0, l0, jj, (p0 & jj) == 0, (p0 & kq) == 0);
              reg_xchg(h1, l1, jj, (p1 & jj) == 0, (p1 & kq) == 0);
            }
          }
        }
        sm.hi[p0] = h0; sm.lo[p0] = l0; sm.hi[p1] = h1; sm.lo[p1] = l1;
      }
      bar();
    }
  }
  __syncthreads();
}

// Repair exact (rho, depth, token) ties by the parent's final position.
__device__ void fix_ties(ExSmem& sm, int n) {
  for (int i = threadIdx.x; i < n; i += EX_THREADS) sm.pos[sm.lo[i] & 0xFFFF] = (unsigned short)i;
  if (threadIdx.x == 0) sm.n_runs = 0;
  __syncthreads();
  for (int i = threadIdx.x; i + 1 < n; i += EX_THREADS) {
    bool same_next = sm.hi[i] == sm.hi[i + 1] && (sm.lo[i] >> 16) == (sm.lo[i + 1] >> 16);
    bool same_prev = i > 0 && sm.hi[i] == sm.hi[i - 1] && (sm.lo[i] >> 16) == (sm.lo[i - 1] >> 16);
    if (same_next && !same_prev) {
      int slot = atomicAdd(&sm.n_runs, 1);
      if (slot < EX_CAP / 2) sm.runs[slot] = (unsigned short)i;
    }
  }
  __syncthreads();
  const int n_runs = min(sm.n_runs, EX_CAP / 2);
  if (n_runs == 0) return;
  for (int d = 2; d <= sm.max_depth; ++d) {
    for (int q = threadIdx.x; q < n_runs; q += EX_THREADS) {
      int s = sm.runs[q];
      if ((int)(sm.lo[s] >> 40) != d) continue;
      unsigned long long key = sm.lo[s] >> 16;
      int e = s + 1;
      while (e < n && sm.hi[e] == sm.hi[s] && (sm.lo[e] >> 16) == key) ++e;
      // insertion sort of lo[s..e) by pos[par[idx]]
      for (int a = s + 1; a < e; ++a) {
        unsigned long long x = sm.lo[a];
        int kx = sm.pos[sm.par[x & 0xFFFF]];
        int b = a - 1;
        while (b >= s && (int)sm.pos[sm.par[sm.lo[b] & 0xFFFF]] > kx) { sm.lo[b + 1] = sm.lo[b]; --b; }
        sm.lo[b + 1] = x;
      }
      for (int a = s; a < e; ++a) sm.pos[sm.lo[a] & 0xFFFF] = (unsigned short)a;
    }
    __syncthreads();
  }
}

// ------------------------------------------------- sequential heap fallback
// The reference's lazy frontier verbatim (draft_tree.py:79-135), on thread 0.
__device__ int heap_expand(const int32_t* tok, const double* prob, int gamma, int k, int limit, HeapEntry* heap,
                           const bst_tree_t& out) {
  int n = 0, size = 0;
  auto push = [&](double rho, int depth, int token, int parent, int rank) {
    HeapEntry e;
    e.rho = rho;
    e.lo = ((unsigned long long)depth << 44) | ((unsigned long long)(unsigned)token << 20) | (unsigned)parent;
    e.rank = rank;
    int i = size++;
    while (i > 0) {
      int p = (i - 1) >> 1;
      if (!heap_less(e, heap[p])) break;
      heap[i] = heap[p];
      i = p;
    }
    heap[i] = e;
  };
  if (k > 0 && prob[0] > 0.0) push(prob[0], 1, tok[0], 0, 0);
  while (size > 0 && n < limit) {
    HeapEntry top = heap[0];
    HeapEntry last = heap[--size];
    int i = 0;
    while (true) {
      int c = 2 * i + 1;
      if (c >= size) break;
      if (c + 1 < size && heap_less(heap[c + 1], heap[c])) ++c;
      if (!heap_less(heap[c], last)) break;
      heap[i] = heap[c];
      i = c;
    }
    if (size > 0) heap[i] = last;
    const int depth = (int)(top.lo >> 44);
    const int token = (int)((top.lo >> 20) & 0xFFFFFF);
    const int parent = (int)(top.lo & 0xFFFFF);
    const int node = ++n;
    out.parent[node] = parent;
    out.depth[node] = depth;
    out.token[node] = token;
    out.rank[node] = top.rank;
    out.rho[node] = top.rho;
    if (depth < gamma) {  // rank-0 child, draft_tree.py:96-104
      double c = __dmul_rn(top.rho, prob[(size_t)depth * k]);
      if (c > 0.0) push(c, depth + 1, tok[(size_t)depth * k], node, 0);
    }
    if (top.rank + 1 < k) {  // next sibling, draft_tree.py:106-115
      double prho = parent == 0 ? 1.0 : out.rho[parent];
      double s = __dmul_rn(prho, prob[(size_t)(depth - 1) * k + top.rank + 1]);
      if (s > 0.0) push(s, depth, tok[(size_t)(depth - 1) * k + top.rank + 1], parent, top.rank + 1);
    }
  }
  return n;
}

// -------------------------------------------------------- post-processing
// Writes the root row, Algorithm-1 stop logic (adaptive), surrogate, meta,
// ancestor bitmask and children CSR for the first n_nodes rows.
// Algorithm 1's stop test over the first n_eval nodes of the tree (rho from out.rho): true
// when S_hat strictly decreases inside them (controller.py:85-98; the same a_hat order and
// S_hat arithmetic as finish_tree).  Scratch: the staged lattice in shared memory.
__device__ bool first_decrease_within(int n_eval, const bst_plan_t& plan, const bst_tree_t& out, ExSmem& sm) {
  double* ahat = sm.lat_p;                              // [2048]
  double* shat = reinterpret_cast<double*>(sm.lat_t);   // [1024]
  if (n_eval < 1 || n_eval > 1024) return false;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 1.0;
    for (int i = 0; i < n_eval; ++i) {
      a = __dadd_rn(a, out.rho[i + 1]);
      ahat[i] = a;
    }
    sm.min_stop = 0x7fffffff;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_eval; i += EX_THREADS) {
    double c_hat = __dadd_rn(plan.fixed_cost, curve_latency(plan.curve, (long long)i + 2));
    shat[i] = __ddiv_rn(__dmul_rn(__dadd_rn(ahat[i], plan.a_offset), plan.l_ar), c_hat);
  }
  __syncthreads();
  const int per = (n_eval + EX_THREADS - 1) / EX_THREADS;
  const int s0 = threadIdx.x * per;
  double local = -INFINITY;
  for (int i = s0; i < min(s0 + per, n_eval); ++i) local = fmax(local, shat[i]);
  double run = block_excl_max(local, sm.dscan);
  for (int i = s0; i < min(s0 + per, n_eval); ++i) {
    if (shat[i] < run) { atomicMin(&sm.min_stop, i); break; }
    run = fmax(run, shat[i]);
  }
  __syncthreads();
  const bool found = sm.min_stop != 0x7fffffff;
  __syncthreads();
  return found;
}

__device__ void finish_tree(int n_eval, bool adaptive, bool is_fixed_or_adaptive, int n_max, const bst_plan_t& plan,
                            const bst_tree_t& out, const ExWs& ws, int algo_used, int enumerated, ExSmem& sm) {
  // Stage rho / parent of rows 0..n_eval in shared memory (the sort arrays are free
  // now): every sequential walk below then runs at smem latency, not DRAM latency.
  const bool in_smem = n_eval + 1 <= EX_CAP;
  double* rho_s = reinterpret_cast<double*>(sm.hi);
  int* par_s = reinterpret_cast<int*>(sm.lo);
  int* cnt_s = par_s + EX_CAP;  // [EX_CAP + 2]... lo holds 2*EX_CAP ints
  if (threadIdx.x == 0) {
    out.parent[0] = -1; out.depth[0] = 0; out.token[0] = -1; out.rank[0] = -1; out.rho[0] = 1.0;
  }
  if (in_smem) {
    for (int i = threadIdx.x; i <= n_eval; i += EX_THREADS) {
      rho_s[i] = i == 0 ? 1.0 : out.rho[i];
      par_s[i] = i == 0 ? -1 : out.parent[i];
    }
  }
  __syncthreads();
  // a_hat / S_hat scratch in shared memory when they fit (the staged lattice is dead now)
  const bool ah_smem = in_smem && n_eval <= 2048;
  double* ahat = ah_smem ? sm.lat_p : ws.ahat;
  const bool sh_smem = in_smem && n_eval <= 1024;
  double* shat_s = sh_smem ? reinterpret_cast<double*>(sm.lat_t) : (out.trace ? out.trace : ws.shat);
  if (threadIdx.x == 0) {
    // controller.py:85 / draft_tree.py:153 addition order; 8 loads in flight per step
    double a = 1.0;
    int i = 0;
    if (in_smem) {
      for (; i + 8 <= n_eval; i += 8) {
        double r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = rho_s[i + 1 + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          a = __dadd_rn(a, r[k]);
          ahat[i + k] = a;
        }
      }
      for (; i < n_eval; ++i) {
        a = __dadd_rn(a, rho_s[i + 1]);
        ahat[i] = a;
      }
    } else {
      for (; i < n_eval; ++i) {
        a = __dadd_rn(a, out.rho[i + 1]);
        ahat[i] = a;
      }
    }
  }
  __syncthreads();
  int n_nodes = n_eval, n_expanded = n_eval, stop = -1;
  if (adaptive && n_eval > 0) {
    double* shat = shat_s;
    for (int i = threadIdx.x; i < n_eval; i += EX_THREADS) {
      double c_hat = __dadd_rn(plan.fixed_cost, curve_latency(plan.curve, (long long)i + 2));
      shat[i] = __ddiv_rn(__dmul_rn(__dadd_rn(ahat[i], plan.a_offset), plan.l_ar), c_hat);
      if (sh_smem && out.trace) out.trace[i] = shat[i];
    }
    if (threadIdx.x == 0) { sm.min_stop = 0x7fffffff; }
    __syncthreads();
    // contiguous segment per thread -> exclusive prefix max -> first decrease
    const int per = (n_eval + EX_THREADS - 1) / EX_THREADS;
    const int s0 = threadIdx.x * per;
    double local = -INFINITY;
    for (int i = s0; i < min(s0 + per, n_eval); ++i) local = fmax(local, shat[i]);
    double run = block_excl_max(local, sm.dscan);
    for (int i = s0; i < min(s0 + per, n_eval); ++i) {
      if (shat[i] < run) { atomicMin(&sm.min_stop, i); break; }
      run = fmax(run, shat[i]);
    }
    __syncthreads();
    const int stop_i = sm.min_stop;
    if (stop_i != 0x7fffffff) {
      n_expanded = stop_i + 1;
      stop = BST_STOP_FIRST_DECREASE;
    } else {
      n_expanded = n_eval;
      stop = n_eval >= n_max ? BST_STOP_BUDGET_CAP : BST_STOP_FRONTIER_EXHAUSTED;
    }
    // best_n = first index of the maximum over the considered prefix
    if (threadIdx.x == 0) { sm.best_val = -INFINITY; sm.best_idx = 0x7fffffff; }
    __syncthreads();
    double bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < n_expanded; i += EX_THREADS)
      if (shat[i] > bv) { bv = shat[i]; bi = i; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    __shared__ double wv[EX_WARPS];
    __shared__ int wi[EX_WARPS];
    if ((threadIdx.x & 31) == 0) { wv[threadIdx.x >> 5] = bv; wi[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 0; w < EX_WARPS; ++w)
        if (wv[w] > sm.best_val || (wv[w] == sm.best_val && wi[w] < sm.best_idx)) {
          sm.best_val = wv[w];
          sm.best_idx = wi[w];
        }
    }
    __syncthreads();
    n_nodes = sm.best_idx + 1;
  }
  (void)is_fixed_or_adaptive;
  if (threadIdx.x == 0) {
    out.meta[0] = n_nodes;
    out.meta[1] = n_expanded;
    out.meta[2] = stop;
    out.meta[3] = algo_used;
    out.meta[4] = enumerated;
    out.surrogate[0] = n_nodes > 0 ? ahat[n_nodes - 1] : 1.0;
  }
  // ancestor-or-self bitmask rows 0..n_nodes (walks parents in smem)
  if (out.anc_mask) {
    const int W = out.mask_words;
    // ancestors are visited in decreasing index order, so each word of the row is
    // complete when the walk leaves it: every word is stored once, zeros included
    for (int i = threadIdx.x; i <= n_nodes; i += EX_THREADS) {
      uint32_t* row = out.anc_mask + (size_t)i * W;
      int w_hi = W - 1, cur_w = i >> 5;
      uint32_t bits = 0u;
      int j = i;
      while (true) {
        const int jw = j >= 0 ? (j >> 5) : -1;
        if (jw != cur_w) {
          for (; w_hi > cur_w; --w_hi) row[w_hi] = 0u;
          row[cur_w] = bits;
          w_hi = cur_w - 1;
          bits = 0u;
          cur_w = jw;
          if (j < 0) break;
        }
        bits |= 1u << (j & 31);
        j = j == 0 ? -1 : (in_smem ? par_s[j] : out.parent[j]);
      }
      for (; w_hi >= 0; --w_hi) row[w_hi] = 0u;
    }
  }
  // children CSR: counts in smem, block exclusive scan, stable fill by child id
  if (out.child_start && out.child_list) {
    if (in_smem && n_nodes + 2 <= EX_CAP) {
      for (int i = threadIdx.x; i <= n_nodes + 1; i += EX_THREADS) cnt_s[i] = 0;
      __syncthreads();
      for (int i = 1 + threadIdx.x; i <= n_nodes; i += EX_THREADS) atomicAdd(&cnt_s[par_s[i]], 1);
      __syncthreads();
      const int per = (n_nodes + 1 + EX_THREADS - 1) / EX_THREADS;
      const int b0 = threadIdx.x * per;
      int loc = 0;
      for (int i = b0; i < min(b0 + per, n_nodes + 1); ++i) loc += cnt_s[i];
      int total;
      int off = block_excl_scan(loc, sm.scan, &total);
      for (int i = b0; i < min(b0 + per, n_nodes + 1); ++i) {
        const int c = cnt_s[i];
        out.child_start[i] = off;
        cnt_s[i] = off;
        off += c;
      }
      if (threadIdx.x == 0) out.child_start[n_nodes + 1] = total;
      __syncthreads();
      for (int i = 1 + threadIdx.x; i <= n_nodes; i += EX_THREADS) {
        const int slot = atomicAdd(&cnt_s[par_s[i]], 1);
        out.child_list[slot] = i;
      }
    } else {
      for (int i = threadIdx.x; i <= n_nodes + 1; i += EX_THREADS) ws.counts[i] = 0;
      __syncthreads();
      for (int i = 1 + threadIdx.x; i <= n_nodes; i += EX_THREADS) atomicAdd(&ws.counts[out.parent[i]], 1);
      __syncthreads();
      if (threadIdx.x == 0) {
        int acc = 0;
        for (int i = 0; i <= n_nodes; ++i) {
          int c = ws.counts[i];
          out.child_start[i] = acc;
          ws.counts[i] = acc;
          acc += c;
        }
        out.child_start[n_nodes + 1] = acc;
      }
      __syncthreads();
      for (int i = 1 + threadIdx.x; i <= n_nodes; i += EX_THREADS) {
        int slot = atomicAdd(&ws.counts[out.parent[i]], 1);
        out.child_list[slot] = i;
      }
    }
  }
}

// Effective plan: optionally loaded from device memory and specialised to the
// device-resident context c (LatencyCurve at c: cost_model.py:290-294 are
// affine in c with exact integer slopes).
__device__ __forceinline__ bst_plan_t resolve_plan(bst_plan_t plan, const bst_plan_t* plan_dev) {
  if (plan_dev) {
    const int32_t policy = plan.policy, n_max = plan.n_max;
    plan = *plan_dev;
    plan.policy = policy;
    plan.n_max = n_max;
  }
  if (plan.state) {
    const long long c = plan.state[plan.c_idx];
    plan.curve.flops_lin += plan.d_flops_lin * c;
    plan.curve.bytes_const += plan.d_bytes_const * c;
    plan.curve.bytes_lin += plan.d_bytes_lin * c;
  }
  return plan;
}

// Batched form (trees != nullptr): CTA r expands request r's lattice (tok/prob + r *
// lat_stride) with plan_dev[r] into trees[r], workspace shifted by r * ws_stride bytes.
__global__ void __launch_bounds__(EX_THREADS, 1)
    expand_best_first_kernel(const int32_t* __restrict__ tok_in, const double* __restrict__ prob_in, int gamma, int k,
                             bst_plan_t plan_in, const bst_plan_t* plan_dev_in, int n_cap, bst_tree_t out_in,
                             ExWs ws_in, int heap_in_smem, const bst_tree_t* trees, int64_t lat_stride,
                             int64_t ws_stride) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ExSmem& sm = *reinterpret_cast<ExSmem*>(smem_raw);
  const int req = trees ? (int)blockIdx.x : 0;
  const int32_t* tok = tok_in + req * lat_stride;
  const double* prob = prob_in + req * lat_stride;
  const bst_plan_t* plan_dev = plan_dev_in ? plan_dev_in + req : nullptr;
  const bst_tree_t out = trees ? trees[req] : out_in;
  ExWs ws = ws_in;
  if (trees) {
    const int64_t o = req * ws_stride;
    ws.ahat = reinterpret_cast<double*>(reinterpret_cast<char*>(ws.ahat) + o);
    ws.shat = reinterpret_cast<double*>(reinterpret_cast<char*>(ws.shat) + o);
    ws.counts = reinterpret_cast<int*>(reinterpret_cast<char*>(ws.counts) + o);
    ws.heap = reinterpret_cast<HeapEntry*>(reinterpret_cast<char*>(ws.heap) + o);
  }
  const bst_plan_t plan = resolve_plan(plan_in, plan_dev);
  const bool adaptive = plan.policy == BST_POLICY_ADAPTIVE;
  const int n_max = plan.n_max;
  const int limit_full = min(n_max, n_cap);
  // Adaptive plans usually stop far below n_max (S_hat's first strict decrease), so a first
  // pass plans only the best EX_PASS1 nodes; the full limit is enumerated only when the
  // frontier reaches EX_PASS1 nodes without a decrease.  The first EX_PASS1 nodes of both
  // passes are the same exact pop order, so the result is identical either way.
  const int limit1 = adaptive ? min(limit_full, EX_PASS1) : limit_full;
  int n_eval = 0;
  int algo_used = BST_ALGO_SORT;
  bool ok = false;
  int enumerated = 0;
  ex_trace(0);
  for (int pass = 0;; ++pass) {
  const int limit = pass == 0 ? limit1 : limit_full;
  n_eval = 0;
  algo_used = BST_ALGO_SORT;
  ok = false;
  enumerated = 0;
  if (plan.algo != BST_ALGO_HEAP) {
    double tau = estimate_tau(prob, gamma, k, limit, sm);
    const bool staged = gamma * k <= 2048;
    if (staged)
      for (int e = threadIdx.x; e < gamma * k; e += EX_THREADS) { sm.lat_p[e] = prob[e]; sm.lat_t[e] = tok[e]; }
    __syncthreads();
    ex_trace(1);
    ok = enumerate_nodes(staged ? sm.lat_t : tok, staged ? sm.lat_p : prob, gamma, k,
                         tau > 0.0 ? tau : 4.9406564584124654e-324, sm);
    ex_trace(2);
    if (ok) {
      const int n = sm.n_enum;
      enumerated = n;
      bitonic_sort(sm, n);
      ex_trace(3);
      fix_ties(sm, n);
      ex_trace(4);
      n_eval = min(limit, n);
      for (int i = threadIdx.x; i < n_eval; i += EX_THREADS) {
        unsigned long long lo = sm.lo[i];
        int idx = (int)(lo & 0xFFFF);
        unsigned short pe = sm.par[idx];
        out.parent[i + 1] = pe == NO_PARENT ? 0 : (int)sm.pos[pe] + 1;
        out.depth[i + 1] = (int)(lo >> 40);
        out.token[i + 1] = (int)((lo >> 16) & 0xFFFFFF);
        out.rank[i + 1] = (int)sm.rnk[idx];
        out.rho[i + 1] = bitsd(~sm.hi[i]);
      }
    }
  }
  if (!ok) {
    algo_used = BST_ALGO_HEAP;
    __syncthreads();
    __shared__ int s_n;
    if (threadIdx.x == 0) {
      HeapEntry* heap = heap_in_smem ? reinterpret_cast<HeapEntry*>(smem_raw) : ws.heap;
      s_n = heap_expand(tok, prob, gamma, k, limit, heap, out);
    }
    __syncthreads();
    n_eval = s_n;
  }
  __syncthreads();
  if (pass > 0 || limit1 == limit_full || n_eval < limit1) break;
  if (first_decrease_within(n_eval, plan, out, sm)) break;
  }
  __syncthreads();
  ex_trace(5);
  finish_tree(n_eval, adaptive, true, n_max, plan, out, ws, algo_used, enumerated, sm);
  __syncthreads();
  ex_trace(6);
}

// ------------------------------------------------------------------- beam
// beam_expand (draft_tree.py:158-189): per level, candidates (rho_parent*p,
// token, parent id) for every survivor x every lattice entry with rho > 0,
// sorted by (-rho, token, parent); keep `width`; ids in level order.
__global__ void __launch_bounds__(EX_THREADS, 1)
    expand_beam_kernel(const int32_t* __restrict__ tok, const double* __restrict__ prob, int gamma, int k,
                       bst_plan_t plan, int n_cap, bst_tree_t out, ExWs ws) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ExSmem& sm = *reinterpret_cast<ExSmem*>(smem_raw);
  __shared__ int s_next_id, s_surv_lo, s_surv_hi;
  if (threadIdx.x == 0) {
    s_next_id = 1;
    s_surv_lo = 0;
    s_surv_hi = 1;  // survivors = node ids [lo, hi); root = 0
    out.rho[0] = 1.0;
  }
  __syncthreads();
  for (int level = 1; level <= plan.depth; ++level) {
    const int lo_id = s_surv_lo, hi_id = s_surv_hi;
    const int n_surv = hi_id - lo_id;
    const int n_cand = n_surv * k;
    const double* pr = prob + (size_t)(level - 1) * k;
    const int32_t* tr = tok + (size_t)(level - 1) * k;
    // candidate c = (survivor c / k, rank c % k); invalid -> sentinel
    int valid_local = 0;
    for (int c = threadIdx.x; c < n_cand; c += EX_THREADS) {
      int sid = lo_id + c / k, r = c % k;
      double prho = out.rho[sid];
      double v = __dmul_rn(prho, __ldg(pr + r));
      if (v > 0.0) {
        sm.hi[c] = ~dbits(v);
        sm.lo[c] = ((unsigned long long)(unsigned)__ldg(tr + r) << 40) | ((unsigned long long)sid << 8) |
                   (unsigned long long)r;
        ++valid_local;
      } else {
        sm.hi[c] = ~0ull;
        sm.lo[c] = ~0ull;
      }
    }
    int n_valid;
    block_excl_scan(valid_local, sm.scan, &n_valid);
    if (n_valid == 0) break;
    bitonic_sort(sm, n_cand);
    const int take = min(plan.width, n_valid);
    const int base = s_next_id;
    for (int i = threadIdx.x; i < take; i += EX_THREADS) {
      int id = base + i;
      if (id <= n_cap) {
        unsigned long long lo = sm.lo[i];
        out.parent[id] = (int)((lo >> 8) & 0xFFFFFFFF);
        out.depth[id] = level;
        out.token[id] = (int)(lo >> 40);
        out.rank[id] = (int)(lo & 0xFF);
        out.rho[id] = bitsd(~sm.hi[i]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_surv_lo = base;
      s_surv_hi = base + take;
      s_next_id = base + take;
    }
    __syncthreads();
  }
  const int n_nodes = min(s_next_id - 1, n_cap);
  finish_tree(n_nodes, false, false, n_nodes, plan, out, ws, BST_ALGO_SORT, n_nodes, sm);
  if (threadIdx.x == 0) out.meta[2] = -1;
}

}  // namespace bst

extern "C" size_t bst_expand_workspace(int gamma, int k, int n_cap) {
  (void)gamma;
  (void)k;
  size_t need = 0;
  bst::ex_carve(nullptr, n_cap < 1 ? 1 : n_cap, &need);
  return need;
}

extern "C" int bst_expand(const int32_t* tok, const double* prob, int gamma, int k, const bst_plan_t* plan,
                          int n_cap, const bst_tree_t* out, void* ws, size_t ws_bytes, bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(tok && prob && plan && out, "null pointer argument");
  BST_REQUIRE(gamma >= 1 && gamma <= EX_MAXG, "gamma must be in [1, %d], got %d", EX_MAXG, gamma);
  BST_REQUIRE(k >= 1 && k <= EX_MAXK, "k must be in [1, %d], got %d", EX_MAXK, k);
  BST_REQUIRE((int64_t)gamma * k <= 2 * EX_CAP, "gamma*k exceeds %d", 2 * EX_CAP);
  BST_REQUIRE(n_cap >= 1, "n_cap must be >= 1");
  BST_REQUIRE(out->parent && out->depth && out->token && out->rank && out->rho && out->meta && out->surrogate,
              "tree output arrays must be non-null");
  BST_REQUIRE(!out->anc_mask || (int64_t)out->mask_words * 32 >= (int64_t)n_cap + 1, "mask_words too small");
  const bst_plan_t p = *plan;
  if (p.policy == BST_POLICY_BEAM) {
    BST_REQUIRE(p.width >= 1, "width must be >= 1, got %d", p.width);
    BST_REQUIRE(p.depth >= 1 && p.depth <= gamma, "depth must be in [1, %d], got %d", gamma, p.depth);
    BST_REQUIRE((int64_t)p.width * k <= EX_CAP, "beam width*k exceeds %d", EX_CAP);
    BST_REQUIRE((int64_t)p.width * p.depth <= n_cap, "beam width*depth exceeds n_cap");
  } else {
    BST_REQUIRE(p.policy == BST_POLICY_ADAPTIVE || p.policy == BST_POLICY_FIXED, "unknown policy %d", p.policy);
    BST_REQUIRE(p.n_max >= 1, "n_max must be >= 1, got %d", p.n_max);
    BST_REQUIRE(p.n_max <= n_cap, "n_max %d exceeds n_cap %d", p.n_max, n_cap);
    BST_REQUIRE(n_cap < (1 << 20), "n_cap must be < 2^20");
    if (p.policy == BST_POLICY_ADAPTIVE) {
      // exact int64 curve arithmetic up to s = n_cap + 1 (Python ints are unbounded)
      const long double smax = (long double)n_cap + 1;
      long double f = ((long double)p.curve.flops_lin + (long double)p.curve.flops_quad * smax) * smax;
      long double b = (long double)p.curve.bytes_const +
                      ((long double)p.curve.bytes_lin + (long double)p.curve.bytes_quad * smax) * smax;
      BST_REQUIRE(f < 9.0e18L && b < 9.0e18L, "latency-curve coefficients overflow int64 at s=%d", n_cap + 1);
    }
  }
  size_t need = 0;
  ExWs w = ex_carve(ws, n_cap, &need);
  BST_REQUIRE(ws != nullptr && ws_bytes >= need, "workspace too small: %zu < %zu", ws_bytes, need);
  const size_t smem = sizeof(ExSmem);
  static bool attr_done = false;
  if (!attr_done) {
    BST_CUDA(cudaFuncSetAttribute(expand_best_first_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    BST_CUDA(cudaFuncSetAttribute(expand_beam_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_done = true;
  }
  cudaStream_t st = as_stream(stream);
  if (p.policy == BST_POLICY_BEAM) {
    BST_CUDA(launch_pdl(expand_beam_kernel, dim3(1), dim3(EX_THREADS), smem, st, tok, prob, gamma, k, p, n_cap, *out, w));
  } else {
    const int heap_in_smem = (2 * (size_t)n_cap + 4) * sizeof(HeapEntry) <= sizeof(unsigned long long) * EX_CAP * 2;
    BST_CUDA(launch_pdl(expand_best_first_kernel, dim3(1), dim3(EX_THREADS), smem, st, tok, prob, gamma, k, p, nullptr, n_cap, *out, w,
                                                          heap_in_smem, static_cast<const bst_tree_t*>(nullptr), (int64_t)0, (int64_t)0));
  }
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" double bst_curve_latency(const bst_curve_t* curve, int64_t s) { return bst::curve_latency(*curve, s); }

extern "C" int bst_expand_dev(const int32_t* tok, const double* prob, int gamma, int k, const bst_plan_t* plan_dev,
                              int policy, int n_max, int n_cap, const bst_tree_t* out, void* ws, size_t ws_bytes,
                              bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(tok && prob && plan_dev && out, "null pointer argument");
  BST_REQUIRE(policy == BST_POLICY_ADAPTIVE || policy == BST_POLICY_FIXED, "device plans support adaptive/fixed");
  BST_REQUIRE(gamma >= 1 && gamma <= EX_MAXG && k >= 1 && k <= EX_MAXK, "bad lattice shape");
  BST_REQUIRE(n_max >= 1 && n_max <= n_cap && n_cap < (1 << 20), "bad n_max/n_cap");
  size_t need = 0;
  ExWs w = ex_carve(ws, n_cap, &need);
  BST_REQUIRE(ws != nullptr && ws_bytes >= need, "workspace too small: %zu < %zu", ws_bytes, need);
  const size_t smem = sizeof(ExSmem);
  static bool attr_done = false;
  if (!attr_done) {
    BST_CUDA(cudaFuncSetAttribute(expand_best_first_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_done = true;
  }
  bst_plan_t p{};
  p.policy = policy;
  p.n_max = n_max;
  const int heap_in_smem = (2 * (size_t)n_cap + 4) * sizeof(HeapEntry) <= sizeof(unsigned long long) * EX_CAP * 2;
  BST_CUDA(launch_pdl(expand_best_first_kernel, dim3(1), dim3(EX_THREADS), smem, as_stream(stream), tok, prob, gamma, k, p, plan_dev, n_cap, *out,
                                                                        w, heap_in_smem, static_cast<const bst_tree_t*>(nullptr), (int64_t)0, (int64_t)0));
  BST_LAUNCH_CHECK();
  return BST_OK;
}

extern "C" int bst_debug_expand_trace(void* buf) {
  BST_CUDA(cudaMemcpyToSymbol(bst::g_ex_trace, &buf, sizeof(void*)));
  return BST_OK;
}

// K2 for n_req requests in one launch (config 3's batched engine): request r's lattice
// rows at tok/prob + r * lat_stride, plan plan_dev[r], tree trees[r] (a device array of
// n_req bst_tree_t); ws holds n_req x bst_expand_workspace(gamma, k, n_cap) bytes.
extern "C" int bst_expand_dev_batch(const int32_t* tok, const double* prob, int64_t lat_stride, int gamma, int k,
                                    const bst_plan_t* plan_dev, int policy, int n_max, int n_cap,
                                    const bst_tree_t* trees_dev, int n_req, void* ws, size_t ws_bytes,
                                    bst_stream_t stream) {
  using namespace bst;
  BST_REQUIRE(tok && prob && plan_dev && trees_dev && n_req >= 1, "bad arguments");
  BST_REQUIRE(policy == BST_POLICY_ADAPTIVE || policy == BST_POLICY_FIXED, "device plans support adaptive/fixed");
  BST_REQUIRE(gamma >= 1 && gamma <= EX_MAXG && k >= 1 && k <= EX_MAXK, "bad lattice shape");
  BST_REQUIRE(n_max >= 1 && n_max <= n_cap && n_cap < (1 << 20), "bad n_max/n_cap");
  size_t per = 0;
  ExWs w = ex_carve(ws, n_cap, &per);
  BST_REQUIRE(ws != nullptr && ws_bytes >= per * (size_t)n_req, "workspace too small: %zu < %zu", ws_bytes,
              per * (size_t)n_req);
  const size_t smem = sizeof(ExSmem);
  BST_CUDA(cudaFuncSetAttribute(expand_best_first_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  bst_plan_t p{};
  p.policy = policy;
  p.n_max = n_max;
  const int heap_in_smem = (2 * (size_t)n_cap + 4) * sizeof(HeapEntry) <= sizeof(unsigned long long) * EX_CAP * 2;
  BST_CUDA(launch_pdl(expand_best_first_kernel, dim3(n_req), dim3(EX_THREADS), smem, as_stream(stream), tok, prob,
                      gamma, k, p, plan_dev, n_cap, bst_tree_t{}, w, heap_in_smem, trees_dev, lat_stride,
                      (int64_t)per));
  BST_LAUNCH_CHECK();
  return BST_OK;
}
