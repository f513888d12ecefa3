// Shared device helpers of the row-selection kernels (K1-split, K5): bulk
// copies and mbarriers, orderable keys, warp selection, the exact radix
// fallback and the tie-aware final selection (see row_topm.cu for the
// exactness argument).
#pragma once
#include "common.cuh"

namespace vs {
namespace tk {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(unsigned long long v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float ex2f(float x) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
  return e;
}
__device__ __forceinline__ uint64_t vkey(float x, int tok) {
  return ((uint64_t)ord_f32(x) << 32) | (uint64_t)(0xffffffffu - (uint32_t)tok);
}

template <typename T>
__device__ __forceinline__ float prev_repr(float x);
template <>
__device__ __forceinline__ float prev_repr<float>(float x) {
  return nextafterf(x, -INFINITY);
}
template <>
__device__ __forceinline__ float prev_repr<__nv_bfloat16>(float x) {
  const uint32_t u = __float_as_uint(x);
  if (x == 0.0f) return __uint_as_float(0x80010000u);
  if (isinf(x)) return x < 0.0f ? x : __uint_as_float(0x7f7f0000u);
  return __uint_as_float((u & 0x80000000u) ? u + 0x10000u : u - 0x10000u);
}

// Top-`keep` keys of buf[0..cnt) into buf[0..keep) (desc) by `keep` warp
// argmax rounds; returns the keep-th key (0 if fewer).
static __device__ __noinline__ uint64_t warp_select(uint64_t* __restrict__ buf, int cnt, int keep,
                                             uint64_t* __restrict__ sel) {
  const int lane = threadIdx.x & 31;
  uint64_t last = 0;
  for (int r = 0; r < keep; ++r) {
    uint64_t lb = 0;
    int li = -1;
    for (int e = lane; e < cnt; e += 32) {
      const uint64_t k = buf[e];
      if (k > lb) {
        lb = k;
        li = e;
      }
    }
    const uint64_t wb = warp_max_u64(lb);
    if (wb != 0 && lb == wb) buf[li] = 0;
    if (lane == 0) sel[r] = wb;
    last = wb;
    __syncwarp();
  }
  for (int r = lane; r < keep; r += 32) buf[r] = sel[r];
  __syncwarp();
  return last;
}

// Exact fallback over one row: M-th largest (logp, token) key by MSB-first
// radix select, then collect + rank (same algorithm as row_topm.cu).
template <typename T>
__device__ __noinline__ void exact_select(const T* __restrict__ row, int V, float lse, int Meff,
                                          unsigned* __restrict__ hist, uint64_t* __restrict__ buf,
                                          uint64_t* __restrict__ sel) {
  const int lane = threadIdx.x & 31;
  uint64_t prefix = 0;
  int want = Meff;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    const uint64_t hi_mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
    for (int i = lane; i < V; i += 32) {
      const uint64_t key = row_key(__fsub_rn(to_f32<T>(row[i]), lse), i);
      if ((key & hi_mask) == (prefix & hi_mask)) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncwarp();
    int digit = 0, above = 0;
    if (lane == 0) {
      unsigned cum = 0;
      for (int d = 255; d >= 0; --d) {
        const unsigned c = hist[d];
        if (cum + c >= (unsigned)want) {
          digit = d;
          above = (int)cum;
          break;
        }
        cum += c;
      }
    }
    digit = __shfl_sync(FULL, digit, 0);
    above = __shfl_sync(FULL, above, 0);
    want -= above;
    prefix |= (uint64_t)digit << shift;
    __syncwarp();
  }
  int cnt = 0;
  for (int i0 = 0; i0 < V; i0 += 32) {
    const int i = i0 + lane;
    uint64_t key = 0;
    bool c = false;
    if (i < V) {
      key = row_key(__fsub_rn(to_f32<T>(row[i]), lse), i);
      c = key >= prefix;
    }
    const unsigned b = __ballot_sync(FULL, c);
    if (c) buf[cnt + __popc(b & ((1u << lane) - 1u))] = key;
    cnt += __popc(b);
  }
  __syncwarp();
  warp_select(buf, cnt, Meff, sel);
}

// Descending bitonic sort of one 64-bit key per lane.
__device__ __forceinline__ uint64_t warp_sort_desc(uint64_t v, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = (uint64_t)__shfl_xor_sync(FULL, (unsigned long long)v, j);
      const bool hi = ((lane & k) == 0) == ((lane & j) == 0);
      v = hi ? (o > v ? o : v) : (o < v ? o : v);
    }
  return v;
}

__device__ __forceinline__ void fold(float& m, float& s, float m2, float s2) {
  // canonical in-order fold of segment (max, sumexp) pairs
  const float mn = fmaxf(m, m2);
  if (mn == -INFINITY) return;
  const float a = (m == -INFINITY) ? 0.0f : s * exp2f((m - mn) * VS_LOG2E);
  const float b = (m2 == -INFINITY) ? 0.0f : s2 * exp2f((m2 - mn) * VS_LOG2E);
  m = mn;
  s = a + b;
}

// Final selection of one row from its candidate keys already re-keyed by
// logp in buf[0..cnt); thetas[] are the pieces' filter thresholds.
template <typename T>
__device__ __forceinline__ void finish_row(const T* __restrict__ row, int V, int M, int Meff, float lse,
                                           int cnt, const uint64_t* thetas, int nth,
                                           uint64_t* __restrict__ buf, uint64_t* __restrict__ sel,
                                           unsigned* __restrict__ hist, int r, int* __restrict__ top_tok,
                                           float* __restrict__ top_logp, float* __restrict__ row_lse,
                                           int* __restrict__ fb_count, bool nofb = false) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const uint64_t kth = cnt >= Meff ? warp_select(buf, cnt, Meff, sel) : 0ull;
  bool ok = kth != 0ull;
  for (int q = 0; q < nth && ok; ++q) {
    const uint64_t th = thetas[q];
    if (th == 0ull) continue;
    const float tx = unord_f32((uint32_t)(th >> 32));
    const uint32_t t_lp = (uint32_t)(kth >> 32);
    const int t_tok = key_tok(kth);
    const int th_tok = (int)(0xffffffffu - (uint32_t)th);
    ok = ord_f32(__fsub_rn(prev_repr<T>(tx), lse)) < t_lp;
    if (ok) {
      const uint32_t lp = ord_f32(__fsub_rn(tx, lse));
      ok = lp < t_lp || (lp == t_lp && (th_tok == -1 || th_tok >= t_tok));
    }
  }
  if (!ok && !nofb) {
    exact_select<T>(row, V, lse, Meff, hist, buf, sel);
    if (lane == 0 && fb_count) atomicAdd(fb_count, 1);
  }
  for (int j = lane; j < M; j += 32) {
    if (j < Meff) {
      const uint64_t kk = sel[j];
      top_tok[(int64_t)r * M + j] = key_tok(kk);
      top_logp[(int64_t)r * M + j] = key_logp(kk);
    } else {
      top_tok[(int64_t)r * M + j] = -1;
      top_logp[(int64_t)r * M + j] = -INFINITY;
    }
  }
  if (lane == 0 && row_lse) row_lse[r] = lse;
}

// Final selection of a whole row from its re-keyed list sorted across lanes
// (lane j holds the j-th key); θ is the piece's filter threshold.
template <typename T>
__device__ __forceinline__ void finish_sorted(const T* __restrict__ row, int V, int M, int Meff, float lse,
                                              uint64_t kk, uint64_t theta, uint64_t* __restrict__ buf,
                                              uint64_t* __restrict__ sel, unsigned* __restrict__ hist, int r,
                                              int* __restrict__ top_tok, float* __restrict__ top_logp,
                                              float* __restrict__ row_lse, int* __restrict__ fb_count,
                                              bool nofb) {
  const int lane = threadIdx.x & 31;
  const uint64_t kth = (uint64_t)__shfl_sync(FULL, (unsigned long long)kk, Meff - 1);
  bool ok = kth != 0ull;
  if (ok && theta != 0ull) {
    const float tx = unord_f32((uint32_t)(theta >> 32));
    const uint32_t t_lp = (uint32_t)(kth >> 32);
    const int t_tok = key_tok(kth);
    const int th_tok = (int)(0xffffffffu - (uint32_t)theta);
    ok = ord_f32(__fsub_rn(prev_repr<T>(tx), lse)) < t_lp;
    if (ok) {
      const uint32_t lp = ord_f32(__fsub_rn(tx, lse));
      ok = lp < t_lp || (lp == t_lp && (th_tok == -1 || th_tok >= t_tok));
    }
  }
  if (!ok && !nofb) {
    exact_select<T>(row, V, lse, Meff, hist, buf, sel);
    if (lane == 0 && fb_count) atomicAdd(fb_count, 1);
    kk = lane < Meff ? sel[lane] : 0ull;
  }
  if (lane < M) {
    top_tok[(int64_t)r * M + lane] = lane < Meff ? key_tok(kk) : -1;
    top_logp[(int64_t)r * M + lane] = lane < Meff ? key_logp(kk) : -INFINITY;
  }
  if (lane == 0 && row_lse) row_lse[r] = lse;
}

}  // namespace tk
}  // namespace vs
