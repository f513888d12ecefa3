// Decode attention over PHYSICAL rows (the decoder scorer's self- and
// cross-attention).
//
// One scored row r attends over `len[r]` cached positions of cache row
// idx[r]: the engine's physical row (self-attention K/V, include/varstream.h)
// or the row's slot (encoder states placed by vs_scatter_rows).  The cache is
// read in place — no gather of K/V into a dense batch — so a step reads each
// live candidate's prefix exactly once: R * len * 2 * H * Dh * 2 bytes.
//
// CTA per row, one warp per head (Dh = 64).  Scores: lane t owns positions
// t, t+32, ... (one 128-byte K line per position, q in registers), softmax by
// warp reductions in fp32, then the output with lanes over head dims (two
// per lane, 128-byte coalesced V lines, probabilities broadcast by shuffle).
// With `knew`/`vnew` the row's newest position (len-1) is taken from them and
// also written into the cache (the self-attention append), so the cache
// write and the attention are one launch.
#include "common.cuh"

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
// their slot's encoder states).  One CTA per (group, head): the slot's K/V
// lines of that head are staged once into shared memory (chunk c of position t
// at c ^ (t & 7): conflict-free 16-byte reads for lanes over positions), then
// the CTA's warps take the group's rows.  Per row the arithmetic is the one of
// row_attention_kernel, so the outputs are bit-identical to it.
constexpr int GW = 8;
__global__ void __launch_bounds__(GW * 32) row_attention_grouped_kernel(
    const __nv_bfloat16* __restrict__ q, int64_t q_ld, const __nv_bfloat16* __restrict__ kc,
    const __nv_bfloat16* __restrict__ vc, int64_t row_stride, int64_t pos_stride, const int* __restrict__ idx,
    const int* __restrict__ lens, const int* __restrict__ grp_off, const int* __restrict__ d_ngrp,
    __nv_bfloat16* __restrict__ out, int64_t out_ld, float scale) {
  VS_PDL_ENTRY();
  extern __shared__ __align__(16) uint4 kvs[];  // [2][MAXL][8] 16-byte chunks
  __shared__ float sp[GW][MAXL];
  const int gi = blockIdx.x;
  if (gi >= *d_ngrp) return;
  const int r0 = grp_off[gi], nr = grp_off[gi + 1] - r0;
  if (nr <= 0) return;
  const int h = blockIdx.y;
  const int64_t hoff = (int64_t)h * DH;
  const int L = lens[r0];
  const int64_t row = idx[r0];
  uint4* ks = kvs;
  uint4* vs = kvs + MAXL * 8;
  for (int i = threadIdx.x; i < L * 8; i += GW * 32) {
    const int t = i >> 3, c = i & 7;
    const int64_t off = row * row_stride + (int64_t)t * pos_stride + hoff;
    ks[t * 8 + (c ^ (t & 7))] = reinterpret_cast<const uint4*>(kc + off)[c];
    vs[t * 8 + (c ^ (t & 7))] = reinterpret_cast<const uint4*>(vc + off)[c];
  }
  __syncthreads();
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto kline = [&](int t, int c) -> uint4 { return ks[t * 8 + (c ^ (t & 7))]; };
  auto vline = [&](int t, int c) -> uint4 { return vs[t * 8 + (c ^ (t & 7))]; };
  for (int rr = wid; rr < nr; rr += GW) attend(q, q_ld, r0 + rr, hoff, L, scale, lane, sp[wid], kline, vline, out, out_ld);
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
  vs::vs_launch(vs::row_attention_kernel, dim3(R_grid, heads / vs::HPC), dim3(32 * vs::HPC), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const __nv_bfloat16*>(q), q_ld, static_cast<__nv_bfloat16*>(k_cache),
      static_cast<__nv_bfloat16*>(v_cache), row_stride, pos_stride, idx, lens,
      static_cast<const __nv_bfloat16*>(k_new), static_cast<const __nv_bfloat16*>(v_new), new_ld,
      static_cast<__nv_bfloat16*>(out), out_ld, heads, scale, R_host, d_R);
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
  const size_t dsm = 2 * vs::MAXL * 8 * sizeof(uint4);  // 64 KB: K and V of one (slot, head)
  if (!attr) {
    cudaFuncSetAttribute(vs::row_attention_grouped_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
    attr = true;
  }
  vs::vs_launch(vs::row_attention_grouped_kernel, dim3(G_grid, heads), dim3(32 * vs::GW), dsm,
                static_cast<cudaStream_t>(stream), static_cast<const __nv_bfloat16*>(q), q_ld,
                static_cast<const __nv_bfloat16*>(k_cache), static_cast<const __nv_bfloat16*>(v_cache), row_stride,
                pos_stride, idx, lens, grp_off, d_ngroups, static_cast<__nv_bfloat16*>(out), out_ld, scale);
  VS_CUDA_RET();
}
