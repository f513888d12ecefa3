// Decode attention over PHYSICAL rows (the decoder scorer's self- and
// cross-attention).
//
// One scored row r attends over `len[r]` cached positions of cache row
// idx[r]: the engine's physical row (self-attention K/V, include/varstream.h)
// or the row's slot (encoder states placed by vs_scatter_rows).  The cache is
// read in place — no gather of K/V into a dense batch — so a step reads each
// live candidate's prefix exactly once: R * len * 2 * H * Dh * 2 bytes.
//
// Three kernels, one warp per (row, head) unit of work (Dh = 64):
//   * row_attention_tiled_kernel (default for vs_row_attention): CTA per (row,
//     4 heads); the row's K/V slices are staged per 32-position tile into
//     shared memory with cp.async (XOR-swizzled chunks), scores with lane =
//     position, online softmax in fp32, V accumulated from shared memory;
//   * row_attention_kernel (VS_ATTN_TILED=0): the same per row, straight from
//     global memory (one 128-byte K line per lane in flight);
//   * row_attention_grouped_kernel (vs_row_attention_grouped, cross-attention):
//     rows of one beam share the slot's encoder states; mma.m16n8k16 tiles.
// With `knew`/`vnew` the row's newest position (len-1) is taken from them and
// also written into the cache (the self-attention append), so the cache
// write and the attention are one launch.
#include "common.cuh"
#include <cstdlib>

namespace vs {
namespace {

constexpr int DH = 64;
constexpr int MAXL = 256;  // positions per row (scores kept in registers, 8 per lane)
constexpr int HPC = 4;     // heads (warps) per CTA

__device__ __forceinline__ float2 bf2(uint32_t w) { return make_float2(bf16lo(w), bf16hi(w)); }

// One (row, head) pair, one warp (see file comment).  KL(t, c) returns the
// 16-byte chunk c (dims 8c..8c+7) of position t's K line, VL(t, c) the V chunk;
// the arithmetic order is the same whatever the source (bit-identical results).
template <typename KL, typename VL>
__device__ __forceinline__ void attend(const __nv_bfloat16* __restrict__ q, int64_t q_ld, int r, int64_t hoff,
                                       int L, float scale, int lane, float* __restrict__ sp, KL kline, VL vline,
                                       __nv_bfloat16* __restrict__ out, int64_t out_ld) {
  // q for this head, in fp32 pairs (64 dims -> 32 registers of bf16x2)
  uint32_t qw[DH / 2];
  {
    const uint4* qp = reinterpret_cast<const uint4*>(q + (int64_t)r * q_ld + hoff);
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      const uint4 v = __ldg(qp + i);
      qw[4 * i] = v.x;
      qw[4 * i + 1] = v.y;
      qw[4 * i + 2] = v.z;
      qw[4 * i + 3] = v.w;
    }
  }
  float sc[MAXL / 32];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < MAXL / 32; ++i) sc[i] = -INFINITY;
#pragma unroll
  for (int i = 0; i < MAXL / 32; ++i) {
    if (32 * i >= L) break;  // warp-uniform
    const int t = lane + 32 * i;
    float s = -INFINITY;
    if (t < L) {
      float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
      for (int c = 0; c < DH / 8; ++c) {
        const uint4 kv = kline(t, c);
        const uint32_t kw[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2 a = bf2(qw[4 * c + u]), b = bf2(kw[u]);
          acc0 = fmaf(a.x, b.x, acc0);
          acc1 = fmaf(a.y, b.y, acc1);
        }
      }
      s = (acc0 + acc1) * scale;
    }
    sc[i] = s;
    mx = fmaxf(mx, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < MAXL / 32; ++i) {
    if (32 * i >= L) break;
    const float p = (lane + 32 * i < L) ? __expf(sc[i] - mx) : 0.f;
    sc[i] = p;
    sum += p;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = sum > 0.f ? 1.f / sum : 0.f;
  // probabilities -> shared memory, then the output with 4 lane groups x 8
  // lanes: group g takes positions t = g (mod 4), lane `sub` of the group owns
  // dims 8*sub..8*sub+7 (one 16-byte V load per position); 16 positions (4 per
  // group) are loaded per iteration, groups are summed by shuffles at the end.
  __syncwarp();
#pragma unroll
  for (int i = 0; i < MAXL / 32; ++i) {
    if (32 * i >= L) break;
    sp[lane + 32 * i] = sc[i] * inv;
  }
  __syncwarp();
  const int g = lane >> 3, sub = lane & 7;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  for (int t0 = 0; t0 < L; t0 += 16) {
    uint4 vv[4];
    float pp[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + 4 * u + g;
      vv[u] = make_uint4(0u, 0u, 0u, 0u);
      pp[u] = 0.f;
      if (t < L) {
        vv[u] = vline(t, sub);
        pp[u] = sp[t];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t w4[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        const float2 v = bf2(w4[q2]);
        acc[2 * q2] = fmaf(pp[u], v.x, acc[2 * q2]);
        acc[2 * q2 + 1] = fmaf(pp[u], v.y, acc[2 * q2 + 1]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 8);
    acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 16);
  }
  if (g == 0) {
    uint4 o;
    __nv_bfloat162 b0 = __floats2bfloat162_rn(acc[0], acc[1]), b1 = __floats2bfloat162_rn(acc[2], acc[3]);
    __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[4], acc[5]), b3 = __floats2bfloat162_rn(acc[6], acc[7]);
    o.x = *reinterpret_cast<uint32_t*>(&b0);
    o.y = *reinterpret_cast<uint32_t*>(&b1);
    o.z = *reinterpret_cast<uint32_t*>(&b2);
    o.w = *reinterpret_cast<uint32_t*>(&b3);
    *reinterpret_cast<uint4*>(out + (int64_t)r * out_ld + hoff + sub * 8) = o;
  }
}

__global__ void __launch_bounds__(HPC * 32, 6) row_attention_kernel(
    const __nv_bfloat16* __restrict__ q, int64_t q_ld, __nv_bfloat16* __restrict__ kc,
    __nv_bfloat16* __restrict__ vc, int64_t row_stride, int64_t pos_stride, const int* __restrict__ idx,
    const int* __restrict__ lens, const __nv_bfloat16* __restrict__ knew, const __nv_bfloat16* __restrict__ vnew,
    int64_t new_ld, __nv_bfloat16* __restrict__ out, int64_t out_ld, int H, float scale, int R_host,
    const int* __restrict__ d_R) {
  VS_PDL_ENTRY();
  __shared__ float sp[HPC][MAXL];
  const int r = blockIdx.x;
  const int R = d_R ? *d_R : R_host;
  if (r >= R) return;
  const int hw = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y * HPC + hw;
  if (h >= H) return;
  const int L = lens[r];
  const int64_t row = idx[r];
  const int64_t hoff = (int64_t)h * DH;
  const bool has_new = knew != nullptr;
  if (has_new && lane < DH / 8) {  // append: write the new K/V line into the cache
    const int64_t dst = row * row_stride + (int64_t)(L - 1) * pos_stride + hoff + lane * 8;
    const int64_t src = (int64_t)r * new_ld + hoff + lane * 8;
    *reinterpret_cast<uint4*>(kc + dst) = *reinterpret_cast<const uint4*>(knew + src);
    *reinterpret_cast<uint4*>(vc + dst) = *reinterpret_cast<const uint4*>(vnew + src);
  }
  const __nv_bfloat16* kb = kc + row * row_stride + hoff;
  const __nv_bfloat16* vb = vc + row * row_stride + hoff;
  const __nv_bfloat16* kn = has_new ? knew + (int64_t)r * new_ld + hoff : nullptr;
  const __nv_bfloat16* vn = has_new ? vnew + (int64_t)r * new_ld + hoff : nullptr;
  auto kline = [&](int t, int c) -> uint4 {
    const __nv_bfloat16* p = (has_new && t == L - 1) ? kn : kb + (int64_t)t * pos_stride;
    return reinterpret_cast<const uint4*>(p)[c];
  };
  auto vline = [&](int t, int c) -> uint4 {
    const __nv_bfloat16* p = (has_new && t == L - 1) ? vn : vb + (int64_t)t * pos_stride;
    return reinterpret_cast<const uint4*>(p)[c];
  };
  attend(q, q_ld, r, hoff, L, scale, lane, sp[hw], kline, vline, out, out_ld);
}

// Grouped rows sharing one cache row (cross-attention: a beam's rows all read
// their slot's encoder states) on the tensor cores.  One CTA (4 warps) per
// (group, head): the slot's K/V lines of that head (<= 256 positions) and up to
// 64 of the group's query rows are staged in shared memory (16-byte chunks
// XOR-swizzled by row for conflict-free ldmatrix), and each warp runs a
// FlashAttention-2 style pass for 16 rows: S = Q·K^T with mma.m16n8k16 (bf16
// in, fp32 accumulate) over 64-position tiles, online softmax in fp32, P
// (bf16) · V with mma.  Per beam the K/V tile is read once for all its rows.
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
               "{%8, %9}, {%0, %1, %2, %3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Tiled per-row attention (the self-attention with append): the CTA's K and V
// slices (HPC heads x 32 positions) are staged into shared memory with
// cp.async, double-buffered, so a whole tile (32 KB) is in flight per CTA
// instead of one 128-byte line per lane; 16-byte chunks are XOR-swizzled by
// position so lanes over positions read conflict-free.  Online softmax per
// tile (lane = position), V accumulated from shared memory.
constexpr int TP = 32;   // positions per tile
constexpr int TBUF = 1;  // tile buffers per CTA (32 KB of smem: 6 CTAs per SM; other CTAs overlap the refill)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(HPC * 32, 6) row_attention_tiled_kernel(
    const __nv_bfloat16* __restrict__ q, int64_t q_ld, __nv_bfloat16* __restrict__ kc,
    __nv_bfloat16* __restrict__ vc, int64_t row_stride, int64_t pos_stride, const int* __restrict__ idx,
    const int* __restrict__ lens, const __nv_bfloat16* __restrict__ knew, const __nv_bfloat16* __restrict__ vnew,
    int64_t new_ld, __nv_bfloat16* __restrict__ out, int64_t out_ld, int H, float scale, int R_host,
    const int* __restrict__ d_R) {
  VS_PDL_ENTRY();
  extern __shared__ __align__(128) uint4 tsm[];  // K [TBUF][TP][HPC][8], V [TBUF][TP][HPC][8]
  __shared__ float sp[HPC][TP];
  __shared__ uint4 qs[HPC][DH / 8];  // this row's q for the CTA's heads (broadcast reads)
  uint4* Kt = tsm;
  uint4* Vt = tsm + TBUF * TP * HPC * 8;
  const int r = blockIdx.x;
  const int R = d_R ? *d_R : R_host;
  if (r >= R) return;
  const int tid = threadIdx.x, hw = tid >> 5, lane = tid & 31;
  const int hb = blockIdx.y * HPC;
  const int h = hb + hw;
  const int L = lens[r];
  const int64_t row = idx[r];
  const bool has_new = knew != nullptr;
  if (has_new && lane < DH / 8 && h < H) {  // append: write the new K/V line into the cache
    const int64_t dst = row * row_stride + (int64_t)(L - 1) * pos_stride + (int64_t)h * DH + lane * 8;
    const int64_t src = (int64_t)r * new_ld + (int64_t)h * DH + lane * 8;
    *reinterpret_cast<uint4*>(kc + dst) = *reinterpret_cast<const uint4*>(knew + src);
    *reinterpret_cast<uint4*>(vc + dst) = *reinterpret_cast<const uint4*>(vnew + src);
  }
  const int ntile = (L + TP - 1) / TP;
  // stage tile `t` into buffer `bf`: TP positions x HPC heads x 8 chunks, K and V
  auto stage = [&](int t, int bf) {
    for (int i = tid; i < TP * HPC * 8; i += HPC * 32) {
      const int c = i & 7, hh = (i >> 3) % HPC, pl = i / (8 * HPC);
      const int pos = t * TP + pl;
      if (pos >= L || hb + hh >= H) continue;
      const int64_t hoff = (int64_t)(hb + hh) * DH;
      const __nv_bfloat16 *ks, *vs;
      if (has_new && pos == L - 1) {  // the newest position from k_new/v_new (not via the cache write)
        ks = knew + (int64_t)r * new_ld + hoff;
        vs = vnew + (int64_t)r * new_ld + hoff;
      } else {
        ks = kc + row * row_stride + (int64_t)pos * pos_stride + hoff;
        vs = vc + row * row_stride + (int64_t)pos * pos_stride + hoff;
      }
      const int d = ((bf * TP + pl) * HPC + hh) * 8 + (c ^ (pl & 7));
      cp_async16(Kt + d, reinterpret_cast<const uint4*>(ks) + c);
      cp_async16(Vt + d, reinterpret_cast<const uint4*>(vs) + c);
    }
  };
  stage(0, 0);
  cp_commit();
  if (TBUF > 1 && ntile > 1) stage(1, 1);
  cp_commit();
  if (h < H && lane < DH / 8)
    qs[hw][lane] = reinterpret_cast<const uint4*>(q + (int64_t)r * q_ld + (int64_t)h * DH)[lane];
  const int g = lane >> 3, sub = lane & 7;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  float m = -INFINITY, l = 0.f;
  for (int t = 0; t < ntile; ++t) {
    const int bf = t % TBUF;
    if (TBUF > 1) cp_wait<1>();
    else cp_wait<0>();
    __syncthreads();
    if (h < H) {
      const int pl = lane, pos = t * TP + pl;
      float sc = -INFINITY;
      if (pos < L) {
        const uint4* kl = Kt + ((bf * TP + pl) * HPC + hw) * 8;
        float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) {
          const uint4 kv = kl[c ^ (pl & 7)];
          const uint4 qv = qs[hw][c];
          const uint32_t kw[4] = {kv.x, kv.y, kv.z, kv.w};
          const uint32_t qc[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 a = bf2(qc[u]), b = bf2(kw[u]);
            acc0 = fmaf(a.x, b.x, acc0);
            acc1 = fmaf(a.y, b.y, acc1);
          }
        }
        sc = (acc0 + acc1) * scale;
      }
      float mx = sc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float mn = fmaxf(m, mx);
      const float cr = m == -INFINITY ? 0.f : __expf(m - mn);
      const float p = pos < L ? __expf(sc - mn) : 0.f;
      float ps = p;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      l = l * cr + ps;
      m = mn;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] *= cr;
      sp[hw][pl] = p;
      __syncwarp();
      const int nt = min(TP, L - t * TP);
      for (int t0 = 0; t0 < nt; t0 += 16) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int pl2 = t0 + 4 * u + g;
          if (pl2 < nt) {
            const uint4 vv = Vt[((bf * TP + pl2) * HPC + hw) * 8 + (sub ^ (pl2 & 7))];
            const float pp = sp[hw][pl2];
            const uint32_t w4[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              const float2 v = bf2(w4[q2]);
              acc[2 * q2] = fmaf(pp, v.x, acc[2 * q2]);
              acc[2 * q2 + 1] = fmaf(pp, v.y, acc[2 * q2 + 1]);
            }
          }
        }
      }
      __syncwarp();
    }
    __syncthreads();  // buffer bf is free again
    if (t + TBUF < ntile) stage(t + TBUF, bf);
    cp_commit();
  }
  if (h >= H) return;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 8);
    acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 16);
  }
  if (g == 0) {
    const float inv = l > 0.f ? 1.f / l : 0.f;
    uint4 o;
    o.x = pack_bf16(acc[0] * inv, acc[1] * inv);
    o.y = pack_bf16(acc[2] * inv, acc[3] * inv);
    o.z = pack_bf16(acc[4] * inv, acc[5] * inv);
    o.w = pack_bf16(acc[6] * inv, acc[7] * inv);
    *reinterpret_cast<uint4*>(out + (int64_t)r * out_ld + (int64_t)h * DH + sub * 8) = o;
  }
}

constexpr int GROWS = 64;  // query rows per CTA pass (4 warps x 16)
__global__ void __launch_bounds__(128) row_attention_grouped_kernel(
    const __nv_bfloat16* __restrict__ q, int64_t q_ld, const __nv_bfloat16* __restrict__ kc,
    const __nv_bfloat16* __restrict__ vc, int64_t row_stride, int64_t pos_stride, const int* __restrict__ idx,
    const int* __restrict__ lens, const int* __restrict__ grp_off, const int* __restrict__ d_ngrp,
    __nv_bfloat16* __restrict__ out, int64_t out_ld, float scale) {
  VS_PDL_ENTRY();
  extern __shared__ __align__(128) uint4 sm[];
  uint4* Ks = sm;                  // [MAXL][8]
  uint4* Vs = sm + MAXL * 8;       // [MAXL][8]
  uint4* Qs = sm + 2 * MAXL * 8;   // [GROWS][8]
  const int gi = blockIdx.x;
  if (gi >= *d_ngrp) return;
  const int r0 = grp_off[gi], nr = grp_off[gi + 1] - r0;
  if (nr <= 0) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t hoff = (int64_t)blockIdx.y * DH;
  const int L = lens[r0];
  const int64_t row = idx[r0];
  const int Lt = (L + 63) & ~63;
  for (int i = tid; i < Lt * 8; i += 128) {  // K/V lines of this (slot, head); zero past L
    const int t = i >> 3, c = i & 7;
    uint4 kv = make_uint4(0u, 0u, 0u, 0u), vv = kv;
    if (t < L) {
      const int64_t off = row * row_stride + (int64_t)t * pos_stride + hoff;
      kv = reinterpret_cast<const uint4*>(kc + off)[c];
      vv = reinterpret_cast<const uint4*>(vc + off)[c];
    }
    Ks[t * 8 + (c ^ (t & 7))] = kv;
    Vs[t * 8 + (c ^ (t & 7))] = vv;
  }
  const float sl2 = scale * 1.4426950408889634f;  // softmax in base 2
  for (int c0 = 0; c0 < nr; c0 += GROWS) {
    const int n = min(GROWS, nr - c0);
    for (int i = tid; i < GROWS * 8; i += 128) {
      const int rr = i >> 3, c = i & 7;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (rr < n) v = reinterpret_cast<const uint4*>(q + (int64_t)(r0 + c0 + rr) * q_ld + hoff)[c];
      Qs[rr * 8 + (c ^ (rr & 7))] = v;
    }
    __syncthreads();
    if (16 * w < n) {
      const int mi = lane >> 3, li = lane & 7;
      uint32_t a[4][4];  // Q fragments, 4 k16 steps over the 64 dims
#pragma unroll
      for (int k16 = 0; k16 < 4; ++k16) {
        const int rr = 16 * w + li + ((mi & 1) ? 8 : 0), c = 2 * k16 + (mi >> 1);
        ldsm_x4(a[k16], smem_addr(Qs + rr * 8 + (c ^ (rr & 7))));
      }
      float o[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
      float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;  // rows lane/4 and lane/4 + 8
      for (int p0 = 0; p0 < Lt; p0 += 64) {
        float sc[8][4];
#pragma unroll
        for (int n8 = 0; n8 < 8; ++n8) {
          sc[n8][0] = sc[n8][1] = sc[n8][2] = sc[n8][3] = 0.f;
          const int pos = p0 + 8 * n8 + li;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            uint32_t b[4];
            const int c = 4 * kk + mi;
            ldsm_x4(b, smem_addr(Ks + pos * 8 + (c ^ (pos & 7))));
            mma_bf16(sc[n8], a[2 * kk], b[0], b[1]);
            mma_bf16(sc[n8], a[2 * kk + 1], b[2], b[3]);
          }
        }
        float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
        for (int n8 = 0; n8 < 8; ++n8)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int pos = p0 + 8 * n8 + 2 * (lane & 3) + (e & 1);
            const float v = pos < L ? sc[n8][e] * sl2 : -INFINITY;
            sc[n8][e] = v;
            if (e < 2) mx_a = fmaxf(mx_a, v);
            else mx_b = fmaxf(mx_b, v);
          }
#pragma unroll
        for (int o2 = 1; o2 <= 2; o2 <<= 1) {
          mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, o2));
          mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, o2));
        }
        const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
        const float cr_a = m_a == -INFINITY ? 0.f : exp2f(m_a - mn_a);  // 0 on the first tile
        const float cr_b = m_b == -INFINITY ? 0.f : exp2f(m_b - mn_b);
        m_a = mn_a;
        m_b = mn_b;
        l_a *= cr_a;
        l_b *= cr_b;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          o[j][0] *= cr_a;
          o[j][1] *= cr_a;
          o[j][2] *= cr_b;
          o[j][3] *= cr_b;
        }
        uint32_t pa[4][4];  // P as A fragments, 4 k16 steps over the tile's 64 positions
#pragma unroll
        for (int n8 = 0; n8 < 8; ++n8) {
          const float p0v = exp2f(sc[n8][0] - mn_a), p1v = exp2f(sc[n8][1] - mn_a);
          const float p2v = exp2f(sc[n8][2] - mn_b), p3v = exp2f(sc[n8][3] - mn_b);
          l_a += p0v + p1v;
          l_b += p2v + p3v;
          pa[n8 >> 1][(n8 & 1) * 2] = pack_bf16(p0v, p1v);
          pa[n8 >> 1][(n8 & 1) * 2 + 1] = pack_bf16(p2v, p3v);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int pos = p0 + 16 * t + li + ((mi & 1) ? 8 : 0);
#pragma unroll
          for (int n8 = 0; n8 < 8; n8 += 2) {
            uint32_t b[4];
            const int c = n8 + (mi >> 1);
            ldsm_x4_t(b, smem_addr(Vs + pos * 8 + (c ^ (pos & 7))));
            mma_bf16(o[n8], pa[t], b[0], b[1]);
            mma_bf16(o[n8 + 1], pa[t], b[2], b[3]);
          }
        }
      }
#pragma unroll
      for (int o2 = 1; o2 <= 2; o2 <<= 1) {
        l_a += __shfl_xor_sync(0xffffffffu, l_a, o2);
        l_b += __shfl_xor_sync(0xffffffffu, l_b, o2);
      }
      const float ia = l_a > 0.f ? 1.f / l_a : 0.f, ib = l_b > 0.f ? 1.f / l_b : 0.f;
      const int ra = 16 * w + (lane >> 2), rb = ra + 8;
#pragma unroll
      for (int n8 = 0; n8 < 8; ++n8) {
        const int d = 8 * n8 + 2 * (lane & 3);
        if (ra < n)
          *reinterpret_cast<uint32_t*>(out + (int64_t)(r0 + c0 + ra) * out_ld + hoff + d) =
              pack_bf16(o[n8][0] * ia, o[n8][1] * ia);
        if (rb < n)
          *reinterpret_cast<uint32_t*>(out + (int64_t)(r0 + c0 + rb) * out_ld + hoff + d) =
              pack_bf16(o[n8][2] * ib, o[n8][3] * ib);
      }
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace vs

extern "C" int vs_row_attention(const void* q, int64_t q_ld, void* k_cache, void* v_cache, int64_t row_stride,
                                int64_t pos_stride, const int32_t* idx, const int32_t* lens, const void* k_new,
                                const void* v_new, int64_t new_ld, void* out, int64_t out_ld, int32_t heads,
                                int32_t head_dim, float scale, int32_t R_host, const int32_t* d_R, int32_t R_grid,
                                void* stream) {
  if (!q || !k_cache || !v_cache || !idx || !lens || !out || head_dim != vs::DH || heads < 1 || heads % vs::HPC ||
      R_grid < 0 || ((k_new == nullptr) != (v_new == nullptr)))
    return VS_ERR_CONFIG;
  if (R_grid == 0) return VS_OK;
  static int tiled = -1;  // VS_ATTN_TILED=0: the register kernel (one K line per lane in flight)
  if (tiled < 0) {
    const char* e = getenv("VS_ATTN_TILED");
    tiled = e ? atoi(e) : 1;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (tiled) {
    const size_t dsm = 2 * vs::TBUF * vs::TP * vs::HPC * 8 * sizeof(uint4);  // K and V tiles
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(vs::row_attention_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
      attr = true;
    }
    vs::vs_launch(vs::row_attention_tiled_kernel, dim3(R_grid, heads / vs::HPC), dim3(32 * vs::HPC), dsm, st,
                  static_cast<const __nv_bfloat16*>(q), q_ld, static_cast<__nv_bfloat16*>(k_cache),
                  static_cast<__nv_bfloat16*>(v_cache), row_stride, pos_stride, idx, lens,
                  static_cast<const __nv_bfloat16*>(k_new), static_cast<const __nv_bfloat16*>(v_new), new_ld,
                  static_cast<__nv_bfloat16*>(out), out_ld, heads, scale, R_host, d_R);
  } else {
    vs::vs_launch(vs::row_attention_kernel, dim3(R_grid, heads / vs::HPC), dim3(32 * vs::HPC), 0, st,
                  static_cast<const __nv_bfloat16*>(q), q_ld, static_cast<__nv_bfloat16*>(k_cache),
                  static_cast<__nv_bfloat16*>(v_cache), row_stride, pos_stride, idx, lens,
                  static_cast<const __nv_bfloat16*>(k_new), static_cast<const __nv_bfloat16*>(v_new), new_ld,
                  static_cast<__nv_bfloat16*>(out), out_ld, heads, scale, R_host, d_R);
  }
  VS_CUDA_RET();
}

extern "C" int vs_row_attention_grouped(const void* q, int64_t q_ld, const void* k_cache, const void* v_cache,
                                        int64_t row_stride, int64_t pos_stride, const int32_t* idx,
                                        const int32_t* lens, const int32_t* grp_off, const int32_t* d_ngroups,
                                        int32_t G_grid, void* out, int64_t out_ld, int32_t heads, int32_t head_dim,
                                        float scale, void* stream) {
  if (!q || !k_cache || !v_cache || !idx || !lens || !grp_off || !d_ngroups || !out || head_dim != vs::DH ||
      heads < 1 || G_grid < 0)
    return VS_ERR_CONFIG;
  if (G_grid == 0) return VS_OK;
  static bool attr = false;
  const size_t dsm = (2 * vs::MAXL + vs::GROWS) * 8 * sizeof(uint4);  // K, V of one (slot, head) + Q rows
  if (!attr) {
    cudaFuncSetAttribute(vs::row_attention_grouped_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
    attr = true;
  }
  vs::vs_launch(vs::row_attention_grouped_kernel, dim3(G_grid, heads), dim3(128), dsm,
                static_cast<cudaStream_t>(stream), static_cast<const __nv_bfloat16*>(q), q_ld,
                static_cast<const __nv_bfloat16*>(k_cache), static_cast<const __nv_bfloat16*>(v_cache), row_stride,
                pos_stride, idx, lens, grp_off, d_ngroups, static_cast<__nv_bfloat16*>(out), out_ld, scale);
  VS_CUDA_RET();
}
