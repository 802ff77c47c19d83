// Shared helpers for the bastion C-ABI library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/bastion.h"

namespace bst {

void set_error(const char* fmt, ...);

#define BST_REQUIRE(cond, ...)          \
  do {                                  \
    if (!(cond)) {                      \
      ::bst::set_error(__VA_ARGS__);    \
      return BST_EINVAL;                \
    }                                   \
  } while (0)

#define BST_CUDA(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      ::bst::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_)); \
      return BST_ECUDA;                                                                \
    }                                                                                  \
  } while (0)

#define BST_LAUNCH_CHECK() BST_CUDA(cudaGetLastError())

inline cudaStream_t as_stream(bst_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Positive doubles order like their bit patterns.
__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double bitsd(unsigned long long b) {
  return __longlong_as_double(static_cast<long long>(b));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// LatencyCurve.latency (cost_model.py:305-309) with round-to-nearest and no
// contraction, matching Python's int->float conversion and float arithmetic.
__host__ __device__ inline double curve_latency(const bst_curve_t& c, long long s) {
  long long f = c.flops_const + (c.flops_lin + c.flops_quad * s) * s;
  long long b = c.bytes_const + (c.bytes_lin + c.bytes_quad * s) * s;
#ifdef __CUDA_ARCH__
  double compute = __dmul_rn(__ll2double_rn(f), c.inv_peak);
  double memory = __dmul_rn(__ll2double_rn(b), c.inv_bw);
  double raw = compute > memory ? compute : memory;
  return __dmul_rn(c.ratio, __dadd_rn(__dmul_rn(c.slope, raw), c.intercept));
#else
  volatile double compute = (double)f * c.inv_peak;
  volatile double memory = (double)b * c.inv_bw;
  double raw = compute > memory ? compute : memory;
  volatile double t = c.slope * raw;
  volatile double u = t + c.intercept;
  return c.ratio * u;
#endif
}

// Pending L2-prefetch hint (bst_set_prefetch) consumed by the next K3/K5 launch.
bst_prefetch_t take_prefetch();

// Programmatic dependent launch (PDL) of the small kernels: every such kernel starts
// with pdl_enter() (griddepcontrol.launch_dependents, then griddepcontrol.wait before
// any global access), so its CTAs may become resident while the predecessor drains and
// the next PDL kernel may be scheduled early.  BST_PDL=0 disables it (measurement).

// Boundary tracing (BST_TRACE builds, scripts/boundary_trace.py): per launch sequence
// number, [first CTA entry, first dependency release, last dependency release, last CTA
// end] in globaltimer ns.  Each translation unit has its own buffer pointer.
#ifdef BST_TRACE
#define BST_BND_TRACE_DEF static __device__ unsigned long long* g_bnd = nullptr;
__device__ __forceinline__ unsigned long long bnd_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define BND(seq, k)                                                                              \
  do {                                                                                           \
    if (g_bnd && (seq) > 0 && (seq) < 4096) {                                                   \
      if ((k) & 1) atomicMax(g_bnd + (int64_t)(seq) * 8 + (k), bnd_now());                      \
      else atomicMin(g_bnd + (int64_t)(seq) * 8 + (k), bnd_now());                               \
    }                                                                                            \
  } while (0)
#define BND_KIND(seq, v)                                                                         \
  do {                                                                                           \
    if (g_bnd && (seq) > 0 && (seq) < 4096) g_bnd[(int64_t)(seq) * 8 + 4] = (v);                \
  } while (0)
#else
#define BST_BND_TRACE_DEF
#define BND(seq, k) \
  do {              \
  } while (0)
#define BND_KIND(seq, v) \
  do {                   \
  } while (0)
#endif
int bnd_next_seq();
void bnd_reset_seq();
int pdl_enabled();
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
template <typename... K, typename... A>
inline cudaError_t launch_pdl(void (*kern)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<K>(args)...);
}

}  // namespace bst
