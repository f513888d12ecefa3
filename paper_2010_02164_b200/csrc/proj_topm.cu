// K5 proj_lse_topM: the decoder's vocab projection on the 5th-gen tensor
// cores with the log-softmax / top-M of K1 fused into the GEMM epilogue.
//
//   logits[r, v] = bf16( H[r, :] . W[v, :] )          (+ EOS bias on column eos)
//   lse[r] = log sum_v exp(logits[r, v]),  top-M of logits[r, :] by (logp desc, token asc)
//
// Same contract as K1 (bb/model.py:216-217 + bb/search.py:63-73) on the bf16
// logits this kernel produces; it replaces "cuBLAS GEMM -> logits in HBM -> K1
// re-reads them" by one persistent warp-specialised kernel:
//
//  * warp 0 (one lane): TMA producer — 128x64 tiles of H and 256x64 tiles of W
//    (SWIZZLE_128B, K-major) into a 4-stage shared-memory ring (mbarriers);
//  * warp 1 (one lane): tcgen05.mma.cta_group::1.kind::f16 128x256x16 into a
//    double-buffered fp32 accumulator in TMEM (2 x 256 columns), stages
//    released with tcgen05.commit;
//  * warps 2-5: epilogue.  Thread = one row of the 128-row tile (its TMEM
//    lane): tcgen05.ld 32 columns at a time, bf16 rounding, EOS bias, the
//    tile's (max, sum exp) and the row's top-M keys of the tile, kept in
//    registers; logits are also written (bf16) for the exact fallback.
//  * tiles are walked m-fastest so the CTAs running concurrently share the
//    same W columns through L2 (W is read from HBM about once per step).
//
// A second small kernel (one warp per row) folds the per-tile (max, sumexp)
// pairs in tile order (fixed order -> deterministic lse), merges the per-tile
// top-M lists, re-keys by logp = fp32(x - lse), runs the tie-aware proof of
// row_topm.cu against every tile's threshold and, if unprovable, the exact
// radix select over the written logits row.
#include "select_common.cuh"

#include <cuda.h>
#include <cstdlib>

namespace vs {
namespace pj {

using namespace tk;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, UK = 16;
constexpr int MAXK = 8;  // per-tile candidates (M <= 8)
constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
constexpr int NTHREADS = 320;  // TMA warp, MMA warp, 8 epilogue warps
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);  // bf16 x bf16 -> f32, K-major, 128x256

struct Smem {
  alignas(1024) unsigned char a[STAGES][A_BYTES];
  alignas(1024) unsigned char b[STAGES][B_BYTES];
  uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // K-major SWIZZLE_128B canonical layout: 8-row atoms of 1024 B (SBO), LBO unused
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
// multicast variant: the box lands at the same smem offset in every CTA of
// `mask` and completes bytes on each destination CTA's barrier at `bar`'s offset
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {  // CTA-local -> cluster address
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_expect_tx_cl(uint32_t cbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl(uint32_t cbar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cbar) : "memory");
}
__device__ __forceinline__ void tma_load_2d_cl(void* dst, const CUtensorMap* map, uint32_t cbar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(cbar), "r"(x), "r"(y)
      : "memory");
}
constexpr uint32_t IDESC2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)((2 * BM) >> 4) << 24);  // M = 256 across the CTA pair
__device__ __forceinline__ void umma2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC2), "r"(accum));
}
__device__ __forceinline__ void umma2_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#define VS_TMEM_LD32(taddr, v)                                                                                 \
  asm volatile(                                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                        \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),       \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),            \
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),            \
        "=r"(v[30]), "=r"(v[31])                                                                              \
      : "r"(taddr))

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// 32 fp32 accumulators -> the bf16 logits (EOS bias, vocab end) as floats
__device__ __forceinline__ void load_chunk(const uint32_t (&v)[32], float (&x)[32], uint32_t (&pk)[16], int col0,
                                           int eos, float eb, int V) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk[j]) : "f"(__uint_as_float(v[2 * j + 1])),
        "f"(__uint_as_float(v[2 * j])));
    x[2 * j] = bf16lo(pk[j]);
    x[2 * j + 1] = bf16hi(pk[j]);
  }
  if ((eos >= col0 && eos < col0 + 32) || col0 + 32 > V) {  // rare chunk
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col0 + j == eos) x[j] = bf16r(x[j] + eb);
      if (col0 + j >= V) x[j] = -INFINITY;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      __nv_bfloat162 b2 = __floats2bfloat162_rn(x[2 * j], x[2 * j + 1]);
      pk[j] = *reinterpret_cast<uint32_t*>(&b2);
    }
  }
}

// CL = 1: one CTA per 128x256 tile.  CL = 2: CTA pairs (clusters of 2 along M)
// compute tiles (2mp, n) and (2mp+1, n); each CTA loads half of the shared W
// stage and multicasts it to both.  CL = 3: CTA pairs issuing one
// tcgen05.mma.cta_group::2 (M = 256) from the leader: each CTA holds its 128
// rows of H and 128 of the 256 W rows, all TMA completions land on the
// leader's barriers, the leader's commits release both CTAs' stages and
// accumulators, both epilogues drain their own TMEM.
template <int Mk, int CL>
__global__ void __launch_bounds__(NTHREADS, 1) proj_topm_kernel(
    const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_w, int R_host,
    const int* __restrict__ d_R, int K, int V, int eos, const float* __restrict__ eos_add,
    __nv_bfloat16* __restrict__ logits, int64_t ldo, float2* __restrict__ part_ms, int Nt, int dbg) {
  VS_PDL_ENTRY();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = d_R ? *d_R : R_host;
  const int Mt = (R + BM - 1) / BM;
  constexpr bool SM2 = CL == 3;
  constexpr int CLX = CL == 1 ? 1 : 2;  // CTAs per cluster
  const int Mu = (Mt + CLX - 1) / CLX;  // M units (pairs of M tiles when clustered)
  const int units = Mu * Nt;
  const int u0 = blockIdx.x / CLX, ustep = gridDim.x / CLX;
  const int crank = CLX > 1 ? (int)cluster_rank() : 0;
  const int nk = K / BK;
  constexpr uint16_t CMASK = (uint16_t)((1u << CLX) - 1u);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&S.full[i], SM2 ? 2 : 1);            // SM2: both producers arrive (leader's copy)
      mbar_init(&S.empty[i], CL == 2 ? 2 : 1);       // CL2: every CTA's MMA consumed the stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.tfull[i], 1);
      mbar_init(&S.tempty[i], SM2 ? 16 : 8);  // SM2: both CTAs' epilogue warps (leader's copy)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (wid == 1) {
    if (SM2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(&S.tmem_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(&S.tmem_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CL > 1) cluster_sync();  // peers' barriers initialised before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;

  if (wid == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int u = u0; u < units; u += ustep) {
        const int m = (u % Mu) * CLX + crank, n = u / Mu;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&S.empty[st], ph ^ 1u);
          if (SM2) {  // this CTA's 128 H rows and 128 W rows, completing on the leader's barrier
            const uint32_t lbar = mapa(smem_u32(&S.full[st]), 0);
            mbar_expect_tx_cl(lbar, A_BYTES + B_BYTES / 2);
            tma_load_2d_cl(S.a[st], &tmap_h, lbar, kb * BK, m * BM);
            tma_load_2d_cl(S.b[st], &tmap_w, lbar, kb * BK, n * BN + crank * (BN / 2));
          } else {
            mbar_expect_tx(&S.full[st], A_BYTES + B_BYTES);
            tma_load_2d(S.a[st], &tmap_h, &S.full[st], kb * BK, m * BM);
            if (CL == 1)
              tma_load_2d(S.b[st], &tmap_w, &S.full[st], kb * BK, n * BN);
            else
              tma_load_2d_mc(S.b[st] + crank * (B_BYTES / 2), &tmap_w, &S.full[st], kb * BK,
                             n * BN + crank * (BN / 2), CMASK);
          }
          if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (wid == 1) {
    // ===== MMA issuer (SM2: the leader CTA only) =====
    if (lane == 0 && (!SM2 || crank == 0)) {
      int st = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int u = u0; u < units; u += ustep) {
        mbar_wait(&S.tempty[acc], aph ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&S.full[st], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = sw128_desc(smem_u32(S.a[st])), bd = sw128_desc(smem_u32(S.b[st]));
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {  // advance 16 bf16 = 32 B along K
            if (SM2)
              umma2(d, ad + (uint64_t)((k * UK * 2) >> 4), bd + (uint64_t)((k * UK * 2) >> 4), (kb | k) != 0);
            else
              umma(d, ad + (uint64_t)((k * UK * 2) >> 4), bd + (uint64_t)((k * UK * 2) >> 4), (kb | k) != 0);
          }
          if (SM2)
            umma2_commit_mc(&S.empty[st], CMASK);  // both CTAs' stages are free
          else if (CL == 1)
            umma_commit(&S.empty[st]);
          else
            umma_commit_mc(&S.empty[st], CMASK);  // the stage is free in every CTA's view
          if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
          }
        }
        if (SM2)
          umma2_commit_mc(&S.tfull[acc], CMASK);  // both CTAs' accumulators are ready
        else
          umma_commit(&S.tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          aph ^= 1u;
        }
      }
    }
  } else {
    // ===== epilogue: thread <-> row (its TMEM lane), two warps per lane
    // quadrant, each owning half of the tile's columns (a "sub-tile") =====
    const int ew = wid - 2;
    const int q = wid & 3;       // TMEM lane quadrant this warp may access
    const int half = ew >> 2;    // column half of the tile
    int acc = 0;
    uint32_t aph = 0;
    const unsigned long long L2E2 = pk2(VS_LOG2E, VS_LOG2E);
    for (int u = u0; u < units; u += ustep) {
      const int m = (u % Mu) * CLX + crank, n = u / Mu;
      const int row = m * BM + q * 32 + lane;
      const bool live = row < R;
      const float eb = (live && eos_add) ? eos_add[row] : 0.0f;
      const int sub = 2 * n + half;  // partial-record index (sub-tiles of BN/2 columns)
      mbar_wait(&S.tfull[acc], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (dbg) {  // timing knob: main loop only (results invalid)
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (SM2)
            mbar_arrive_cl(mapa(smem_u32(&S.tempty[acc]), 0));
          else
            mbar_arrive(&S.tempty[acc]);
        }
        if (++acc == 2) {
          acc = 0;
          aph ^= 1u;
        }
        continue;
      }
      float mx = -INFINITY, sm = 0.0f;
      // TMEM -> registers double-buffered: chunk c+1's tcgen05.ld is in flight
      // while chunk c is processed
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + half * (BN / 2));
      uint32_t vb[2][32];
      VS_TMEM_LD32(tbase, vb[0]);  // warp-collective: every lane, every iteration below
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) {
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");  // chunk c has landed
        if (c + 1 < BN / 64) VS_TMEM_LD32(tbase + (uint32_t)((c + 1) * 32), vb[(c + 1) & 1]);
        const uint32_t(&v)[32] = vb[c & 1];
        const int cc = half * (BN / 2) + c * 32;  // column within the tile
        const int col0 = n * BN + cc;
        float x[32];
        uint32_t pk[16];
        load_chunk(v, x, pk, col0, eos, eb, V);
        if (!live) continue;
        __nv_bfloat16* out = logits + (int64_t)row * ldo + col0;
        if (col0 + 32 <= V) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
            reinterpret_cast<uint4*>(out)[g] = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < V) out[j] = __float2bfloat16_rn(x[j]);
        }
        float cm = x[0];
#pragma unroll
        for (int j = 1; j < 32; ++j) cm = fmaxf(cm, x[j]);
        if (cm == -INFINITY) continue;
        const float mn = fmaxf(mx, cm);
        const float nml = -mn * VS_LOG2E;
        const unsigned long long N2 = pk2(nml, nml);
        unsigned long long a2 = pk2(0.0f, 0.0f), b2 = pk2(0.0f, 0.0f);
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float t0, t1, t2, t3;
          up2(fma2(pk2(x[j], x[j + 1]), L2E2, N2), t0, t1);
          up2(fma2(pk2(x[j + 2], x[j + 3]), L2E2, N2), t2, t3);
          a2 = add2(a2, pk2(ex2f(t0), ex2f(t1)));
          b2 = add2(b2, pk2(ex2f(t2), ex2f(t3)));
        }
        a2 = add2(a2, b2);
        float s0, s1;
        up2(a2, s0, s1);
        sm = (mx == -INFINITY ? 0.0f : sm * ex2f((mx - mn) * VS_LOG2E)) + (s0 + s1);
        mx = mn;
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (SM2)
          mbar_arrive_cl(mapa(smem_u32(&S.tempty[acc]), 0));  // the leader's MMA reuses both TMEMs
        else
          mbar_arrive(&S.tempty[acc]);
      }
      // (sub-tile max, sum exp(x - max)): the merge also uses the max to pick
      // the only sub-tiles that can hold the row's top-M
      if (live) part_ms[(int64_t)row * (2 * Nt) + sub] = make_float2(mx, sm);
      if (++acc == 2) {
        acc = 0;
        aph ^= 1u;
      }
    }
  }
  __syncthreads();
  if (CL > 1) cluster_sync();  // no CTA leaves while a peer may still multicast into it
  if (wid == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (SM2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// One warp per row.  lse: in-order fold of the sub-tiles' (max, sumexp).
// Top-M: θ = M-th largest sub-tile maximum is a lower bound of the row's M-th
// largest logit (the M largest sub-tile maxima are M distinct elements), so
// only sub-tiles whose maximum is >= θ (normally exactly M of the 330) can
// hold a top-M element; their logits (written by the GEMM epilogue) are
// scanned, elements >= θ are ranked by (logp desc, token asc), and the
// tie-aware proof of row_topm.cu checks the boundary against θ (every element
// not collected has x < θ).  Unprovable rows take the exact radix select.
constexpr int MAXS = 512;  // sub-tiles per row (V <= 65536)
__global__ void __launch_bounds__(128) proj_merge_kernel(int R_host, const int* __restrict__ d_R, int V, int M,
                                                         int Ns, const float2* __restrict__ part_ms,
                                                         const __nv_bfloat16* __restrict__ logits, int64_t ldo,
                                                         int* __restrict__ top_tok, float* __restrict__ top_logp,
                                                         float* __restrict__ row_lse, int* __restrict__ fb_count) {
  VS_PDL_ENTRY();
  __shared__ uint64_t sbuf[4][192];
  __shared__ uint64_t ssel[4][32];
  __shared__ float smax[4][MAXS];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 4 + wid;
  const int R = d_R ? *d_R : R_host;
  if (r >= R) return;
  const int Meff = M < V ? M : V;
  const int SUBW = BN / 2;
  // fixed-order tree: each lane folds sub-tiles lane, lane+32, ... then a
  // butterfly merge across lanes (deterministic for a given V)
  float m = -INFINITY, s = 0.0f;
  for (int q = lane; q < Ns; q += 32) {
    const float2 v = part_ms[(int64_t)r * Ns + q];
    smax[wid][q] = v.x;
    fold(m, s, v.x, v.y);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float m2 = __shfl_xor_sync(FULL, m, o), s2 = __shfl_xor_sync(FULL, s, o);
    // both partners combine the same ordered pair (lower lane first): identical results
    if (lane & o) {
      float mm = m2, ss = s2;
      fold(mm, ss, m, s);
      m = mm;
      s = ss;
    } else {
      fold(m, s, m2, s2);
    }
  }
  __syncwarp();
  const float lse = (m == -INFINITY || s == 0.0f) ? -INFINITY : m + logf(s);
  // θ: Meff-th largest sub-tile maximum (Meff warp-argmax rounds)
  float thx = -INFINITY;
  for (int rnd = 0; rnd < Meff; ++rnd) {
    float lb = -INFINITY;
    int li = -1;
    for (int q = lane; q < Ns; q += 32)
      if (smax[wid][q] > lb || (li < 0 && smax[wid][q] == lb)) {
        lb = smax[wid][q];
        li = q;
      }
    float wb = lb;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wb = fmaxf(wb, __shfl_xor_sync(FULL, wb, o));
    const unsigned own = __ballot_sync(FULL, li >= 0 && lb == wb);
    if (own && lane == __ffs(own) - 1) smax[wid][li] = -INFINITY;  // consume one maximum
    thx = wb;
    __syncwarp();
  }
  // collect every element >= θ of the sub-tiles whose maximum is >= θ
  const __nv_bfloat16* lrow = logits + (int64_t)r * ldo;
  int cnt = 0;
  for (int q0 = 0; q0 < Ns; q0 += 32) {
    const int q = q0 + lane;
    const float2 v = q < Ns ? part_ms[(int64_t)r * Ns + q] : make_float2(-INFINITY, 0.0f);
    unsigned sel = __ballot_sync(FULL, q < Ns && v.x >= thx && v.x != -INFINITY);
    if (thx == -INFINITY) sel = __ballot_sync(FULL, q < Ns);  // fewer than Meff finite logits
    while (sel) {
      const int sq = q0 + __ffs(sel) - 1;
      sel &= sel - 1;
      // 128 columns of sub-tile sq: 4 per lane
      const int c0 = sq * SUBW + lane * 4;
      float xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = c0 + u < V ? __bfloat162float(lrow[c0 + u]) : -INFINITY;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool c = c0 + u < V && xv[u] >= thx;
        const unsigned b = __ballot_sync(FULL, c);
        if (cnt + __popc(b) > 192) {  // compact exactly (by logit key) before appending
          __syncwarp();
          warp_select(sbuf[wid], cnt, Meff, ssel[wid]);
          cnt = Meff;
        }
        if (c) sbuf[wid][cnt + __popc(b & ((1u << lane) - 1u))] = vkey(xv[u], c0 + u);
        cnt += __popc(b);
        __syncwarp();
      }
    }
  }
  // re-key by logp, select the top-Meff
  for (int e = lane; e < cnt; e += 32) {
    const uint64_t k = sbuf[wid][e];
    sbuf[wid][e] = row_key(__fsub_rn(unord_f32((uint32_t)(k >> 32)), lse), (int)(0xffffffffu - (uint32_t)k));
  }
  __syncwarp();
  const uint64_t kth = cnt >= Meff ? warp_select(sbuf[wid], cnt, Meff, ssel[wid]) : 0ull;
  uint64_t kk = lane < Meff ? ssel[wid][lane] : 0ull;
  bool ok = kth != 0ull;
  if (ok && thx != -INFINITY) {  // every element not collected has x < θ
    const uint32_t t_lp = (uint32_t)(kth >> 32);
    ok = ord_f32(__fsub_rn(prev_repr<__nv_bfloat16>(thx), lse)) < t_lp;
  }
  if (!ok) {
    exact_select<__nv_bfloat16>(lrow, V, lse, Meff, reinterpret_cast<unsigned*>(sbuf[wid] + 64), sbuf[wid],
                                ssel[wid]);
    kk = lane < Meff ? ssel[wid][lane] : 0ull;
    if (lane == 0 && fb_count) atomicAdd(fb_count, 1);
  }
  if (lane < M) {
    top_tok[(int64_t)r * M + lane] = lane < Meff ? key_tok(kk) : -1;
    top_logp[(int64_t)r * M + lane] = lane < Meff ? key_logp(kk) : -INFINITY;
  }
  if (lane == 0 && row_lse) row_lse[r] = lse;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  EncodeTiled enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t ws_bytes(int R_grid, int V) {
  const int Nt = 2 * ((V + BN - 1) / BN);  // sub-tiles of BN/2 columns
  return (size_t)R_grid * Nt * sizeof(float2);
}

}  // namespace pj
}  // namespace vs

extern "C" size_t vs_proj_lse_topm_ws_bytes(int32_t R_grid, int32_t V) { return vs::pj::ws_bytes(R_grid, V); }

extern "C" int vs_proj_lse_topm(const void* H, int64_t ldh, const void* W, int64_t ldw, int32_t R_host,
                                const int32_t* d_R, int32_t R_grid, int32_t K, int32_t V, int32_t M, int32_t eos,
                                const float* eos_add, void* logits, int64_t ldo, int32_t* top_tok, float* top_logp,
                                float* row_lse, int32_t* fallback_count, void* workspace, size_t workspace_bytes,
                                void* stream) {
  using namespace vs::pj;
  if (!H || !W || !logits || !top_tok || !top_logp || K % BK || K < BK || V < 1 || M < 1 || M > MAXK || R_grid < 0 ||
      (ldh * 2) % 16 || (ldw * 2) % 16 || (logits && ((ldo * 2) % 16 || ldo < V)) ||
      (reinterpret_cast<uintptr_t>(H) & 15) || (reinterpret_cast<uintptr_t>(W) & 15))
    return VS_ERR_CONFIG;
  if (R_grid == 0) return VS_OK;
  if (2 * ((V + BN - 1) / BN) > MAXS) return VS_ERR_CONFIG;
  if (!workspace || workspace_bytes < ws_bytes(R_grid, V)) return VS_ERR_CONFIG;
  CUtensorMap mh, mw;
  static int CLn = -1;
  if (CLn < 0) {
    // 1: single CTAs; 2 (default): CTA pairs multicasting W; 3: CTA pairs with cta_group::2 MMA
    const char* c = getenv("VS_K5_CL");
    CLn = c ? atoi(c) : 2;
    if (CLn < 1 || CLn > 3) CLn = 2;
  }
  const int CLX = CLn == 1 ? 1 : 2;
  if (!make_map(&mh, H, R_grid, K, ldh, BM) || !make_map(&mw, W, V, K, ldw, BN / CLX)) return VS_ERR_CUDA;
  const int Nt = (V + BN - 1) / BN;
  float2* pms = static_cast<float2*>(workspace);
  static int sms = 0, dbg = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* d = getenv("VS_K5_DBG");
    dbg = d ? atoi(d) : 0;
  }
  const int units_max = ((R_grid + BM - 1) / BM + CLX - 1) / CLX * Nt;
  int grid = units_max * CLX < sms ? units_max * CLX : sms;
  grid -= grid % CLX;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaErrorInvalidValue;
#define VS_K5_ONE(MK_, CL_)                                                                                   \
  do {                                                                                                        \
    static bool attr = false;                                                                                 \
    if (!attr) {                                                                                              \
      cudaFuncSetAttribute(proj_topm_kernel<MK_, CL_>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                           (int)sizeof(Smem) + 1024);                                                         \
      attr = true;                                                                                            \
    }                                                                                                         \
    e = vs::vs_launch_cluster(proj_topm_kernel<MK_, CL_>, dim3(grid), dim3(NTHREADS), sizeof(Smem) + 1024, st, \
                              CL_ == 1 ? 1 : 2, mh, mw, (int)R_host, d_R, (int)K, (int)V, (int)eos, eos_add,               \
                              static_cast<__nv_bfloat16*>(logits), ldo, pms, Nt, dbg);                        \
  } while (0)
#define VS_K5(MK_)       \
  case MK_:              \
    if (CLn == 3)        \
      VS_K5_ONE(MK_, 3); \
    else if (CLn == 2)   \
      VS_K5_ONE(MK_, 2); \
    else                 \
      VS_K5_ONE(MK_, 1); \
    break;
  switch (M) {
    VS_K5(1) VS_K5(2) VS_K5(3) VS_K5(4) VS_K5(5) VS_K5(6) VS_K5(7) VS_K5(8)
  }
#undef VS_K5
#undef VS_K5_ONE
  if (e != cudaSuccess) return VS_ERR_CUDA;
  e = vs::vs_launch(proj_merge_kernel, dim3((R_grid + 3) / 4), dim3(128), 0, st, (int)R_host, d_R, (int)V, (int)M,
                    2 * Nt, static_cast<const float2*>(pms), static_cast<const __nv_bfloat16*>(logits), ldo, top_tok,
                    top_logp, row_lse, fallback_count);
  return e == cudaSuccess ? VS_OK : VS_ERR_CUDA;
}
