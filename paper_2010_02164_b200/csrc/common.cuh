// Shared device helpers for the VarStream sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>

#include "../../include/varstream.h"

#define VS_LOG2E 1.4426950408889634f
#define VS_LN2 0.6931471805599453f

namespace vs {

// ---- orderable encodings -------------------------------------------------
// fp32 -> uint32 preserving total order (larger float -> larger uint).
__device__ __forceinline__ uint32_t ord_f32(float x) {
  if (x == 0.0f) x = 0.0f;  // canonicalise -0
  uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__device__ __forceinline__ uint64_t ord_f64(double x) {
  if (x == 0.0) x = 0.0;
  uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// 64-bit selection key of a row entry: (logp desc, token asc) == larger key first.
__device__ __forceinline__ uint64_t row_key(float logp, int tok) {
  return ((uint64_t)ord_f32(logp) << 32) | (uint64_t)(0xffffffffu - (uint32_t)tok);
}
__device__ __forceinline__ int key_tok(uint64_t k) { return (int)(0xffffffffu - (uint32_t)k); }
__device__ __forceinline__ float key_logp(uint64_t k) { return unord_f32((uint32_t)(k >> 32)); }

// ---- hashing (bit-identical to oracle/scorers.py) --------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t prefix_init(uint64_t src_seed, int sos) {
  return mix64(src_seed + (uint64_t)(sos + 1) * 0xD6E8FEB86659FD93ull);
}
__host__ __device__ __forceinline__ uint64_t prefix_step(uint64_t h, int tok) {
  return mix64(h ^ ((uint64_t)(tok + 1) * 0xD6E8FEB86659FD93ull));
}
__device__ __forceinline__ uint32_t fmix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  return x;
}

// ---- loads -----------------------------------------------------------------
// Streaming 16-byte load: read-only, do not allocate in L1 (each byte is read once).
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}

// ---- warp helpers ------------------------------------------------------------
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
  uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    uint64_t o = shfl_xor_u64(v, m);
    v = o > v ? o : v;
  }
  return v;
}

// Online log-sum-exp pair merge: (m, s) with s = sum exp(x - m).
__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2) {
  float mn = fmaxf(m, m2);
  if (mn == -INFINITY) return;  // both empty
  float a = (m == -INFINITY) ? 0.0f : s * exp2f((m - mn) * VS_LOG2E);
  float b = (m2 == -INFINITY) ? 0.0f : s2 * exp2f((m2 - mn) * VS_LOG2E);
  m = mn;
  s = a + b;
}

// ---- programmatic dependent launch (PDL) -------------------------------------
// Every kernel starts with VS_PDL_ENTRY(): wait until the preceding kernel in
// the stream has completed (its writes visible), then allow the next one to
// be launched, so launch latency and the next grid's ramp overlap this
// kernel's tail.  Kernels are launched with vs_launch (cudaLaunchKernelEx +
// programmatic stream serialization; VS_PDL=0 disables it).
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t vs_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Cluster launch (cluster_x CTAs per cluster along x) with PDL.
template <typename... KArgs, typename... Args>
cudaError_t vs_launch_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace vs

#define VS_PDL_ENTRY() ::vs::pdl_entry()

// Phase timing probes (profiling builds only: -DVS_PHASE_PROF).  Thread 0
// of the probing CTA keeps SM clock stamps in shared memory (no memory
// traffic on the measured path); VS_PROF_FLUSH adds (stamp - start) per probe
// to global accumulators once per launch.
#ifdef VS_PHASE_PROF
static __device__ unsigned long long g_prof_acc[32];
static __shared__ long long s_prof[32];
#define VS_PROF_T0(cond)                                     \
  if ((cond) && threadIdx.x == 0) {                          \
    for (int _q = 0; _q < 32; ++_q) s_prof[_q] = 0;          \
    s_prof[0] = clock64();                                   \
  }
#define VS_PROF(cond, i) \
  if ((cond) && threadIdx.x == 0) s_prof[i] = clock64()
#define VS_PROF_FLUSH(cond)                                                        \
  if ((cond) && threadIdx.x == 0) {                                                \
    for (int _q = 1; _q < 31; ++_q)                                                \
      if (s_prof[_q]) atomicAdd(&g_prof_acc[_q], (unsigned long long)(s_prof[_q] - s_prof[0])); \
    atomicAdd(&g_prof_acc[31], 1ull);                                              \
  }
// Slowest-CTA view: every probing CTA folds its own stamps 1..7 (cycles since
// its start) into g_prof_max with atomicMax before it counts in; the CTA that
// runs the scheduler moves the per-launch maxima into g_prof_acc[16 + i].
static __device__ unsigned long long g_prof_max[8];
#define VS_PROF_MAX_FOLD()                                                          \
  if (threadIdx.x == 0) {                                                           \
    for (int _q = 1; _q < 8; ++_q)                                                  \
      if (s_prof[_q]) atomicMax(&g_prof_max[_q], (unsigned long long)(s_prof[_q] - s_prof[0])); \
  }
#define VS_PROF_MAX_COLLECT()                                                       \
  if (threadIdx.x == 0) {                                                           \
    for (int _q = 1; _q < 8; ++_q) {                                                \
      atomicAdd(&g_prof_acc[16 + _q], atomicExch(&g_prof_max[_q], 0ull));          \
    }                                                                               \
  }
#else
#define VS_PROF_T0(cond) (void)0
#define VS_PROF(cond, i) (void)0
#define VS_PROF_FLUSH(cond) (void)0
#define VS_PROF_MAX_FOLD() (void)0
#define VS_PROF_MAX_COLLECT() (void)0
#endif

#define VS_CUDA_RET()                                              \
  do {                                                             \
    cudaError_t _e = cudaGetLastError();                           \
    return _e == cudaSuccess ? VS_OK : VS_ERR_CUDA;                \
  } while (0)
