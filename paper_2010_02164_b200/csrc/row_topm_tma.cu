// K1 (TMA-staged, split-row) row_lse_topM for sm_100a.
//
// Same contract as row_topm.cu (bb/model.py:216-217 log-softmax +
// bb/search.py:63-73 per-parent top-M by (row value desc, token asc)), built
// for HBM streaming on B200:
//
//  * Work is the row-major sequence of 4 KB SEGMENTS of all R rows.  A
//    persistent grid (CTAs_per_SM x 148 CTAs of 4 warps) gives every warp one
//    contiguous, equally sized slice of that sequence, so the machine is full
//    whatever R is (573 rows at the WMT step, 6400 at full width, 1 row).
//  * Each warp streams its slice through a private ring of NS 4 KB shared-
//    memory stages filled by cp.async.bulk (the TMA engine, UBLKCP) and
//    completed on per-stage mbarriers: NS-1 segments in flight per warp with
//    no registers held, one elected lane issuing.
//  * Per segment the hot loop is: LDS.128 x 8, a packed bf16x2 max tree (the
//    exact segment max m_seg, warp-uniform after 5 shuffles), then
//    sum exp(x - m_seg) with FFMA2 + MUFU.EX2 + FADD2.  No online rescale is
//    needed inside a segment (m_seg is its exact max).
//  * lse is a PARTITION-INVARIANT function of the row: every segment's
//    (m_seg, s_seg) is computed with a fixed lane<->element mapping and the
//    row's (m, s) is the in-order left fold over segments 0..nseg-1, whether
//    one warp owns the row or its segments are spread over several warps (the
//    fold then runs in the row's finisher from per-segment pairs).
//  * Top-M candidates live in a register-resident sorted list (lane j holds
//    the j-th key) whose M-th key is the warp-uniform threshold θ (bootstrapped
//    from the 32 lane maxima of a piece's first segment); a segment whose
//    maximum is below θ costs one uniform compare.  Row pieces owned by
//    several warps publish their top-M logit keys + θ; the last piece to arrive
//    (per-row counter) merges, re-keys by logp = fp32(x - lse), selects, runs
//    the tie-aware proof and, if unprovable, the exact radix select (counted).
//
// Requirements (else the caller uses row_topm.cu): 16-byte aligned rows
// (logits and ld*sizeof(T)), V*sizeof(T) >= 4096, M <= 32.
#include "select_common.cuh"
#include <cstdlib>

namespace vs {
namespace tk {

constexpr int NW = 4;            // warps per CTA
constexpr int SEGB = 4096;       // bytes per segment == one TMA stage
constexpr int VPL = SEGB / 16 / 32;  // 16-byte vectors per lane per segment (8)
constexpr int CAPW = 192;        // per-warp candidate buffer (keys)
constexpr int MAXM = 32;
constexpr int MAXP = 64;          // segments (hence pieces) per row

struct PartRec {                 // one row piece published for the finisher
  uint64_t theta;
  int32_t cnt;
  int32_t pad;
  uint64_t keys[MAXM];           // top-min(cnt, M) logit keys (value desc, token asc)
};

template <int NS>
struct WarpSmem {
  alignas(128) unsigned char stage[NS][SEGB];
  uint64_t bar[NS];
  uint64_t buf[CAPW];   // candidates; the exact fallback uses buf[64..192) as its histogram
  uint64_t sel[MAXM];
  uint64_t ths[MAXP];   // finisher: the pieces' thresholds
  int pslot[MAXP];      // finisher: first segment of each piece
  int poff[MAXP + 1];   // finisher: prefix of the pieces' key counts
};

// ---- segment decode: per-lane view of one 4 KB stage ------------------------
// Lane l owns 16-byte vectors l + 32*j (j < VPL) of the segment: a fixed
// mapping, so (m_seg, s_seg) depend only on the segment's bytes.
template <typename T>
struct Seg;

template <>
struct Seg<__nv_bfloat16> {
  static constexpr int EPV = 8;  // elements per vector
  uint32_t w[VPL][4];
  uint32_t vmax[VPL];  // packed bf16x2 max of each vector
  __device__ __forceinline__ void load(const unsigned char* st, int nvec, int lane) {
    const uint4* s = reinterpret_cast<const uint4*>(st);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int v = lane + 32 * j;
      uint4 q = make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);  // -inf pairs
      if (v < nvec) q = s[v];
      w[j][0] = q.x;
      w[j][1] = q.y;
      w[j][2] = q.z;
      w[j][3] = q.w;
    }
  }
  __device__ __forceinline__ float lane_max() {
#pragma unroll
    for (int j = 0; j < VPL; ++j) vmax[j] = bmax2(bmax2(w[j][0], w[j][1]), bmax2(w[j][2], w[j][3]));
    uint32_t a = bmax2(bmax2(vmax[0], vmax[1]), bmax2(vmax[2], vmax[3]));
    uint32_t b = bmax2(bmax2(vmax[4], vmax[5]), bmax2(vmax[6], vmax[7]));
    const uint32_t m = bmax2(a, b);
    return fmaxf(bf16lo(m), bf16hi(m));
  }
  __device__ __forceinline__ float vec_max(int j) const { return fmaxf(bf16lo(vmax[j]), bf16hi(vmax[j])); }
  __device__ __forceinline__ void load_full(const unsigned char* st, int lane) {
    const uint4* s = reinterpret_cast<const uint4*>(st);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const uint4 q = s[lane + 32 * j];
      w[j][0] = q.x;
      w[j][1] = q.y;
      w[j][2] = q.z;
      w[j][3] = q.w;
    }
  }
  // bit j set when vector j holds an element >= tx (tx is a bf16 value)
  __device__ __forceinline__ unsigned pass_mask(float tx) const {
    const uint32_t t = __float_as_uint(tx) >> 16;
    const uint32_t t2 = t | (t << 16);
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      uint32_t p;
      asm("{\n.reg .pred a, b;\nsetp.ge.bf16x2 a|b, %1, %2;\nor.pred a, a, b;\nselp.u32 %0, 1, 0, a;\n}"
          : "=r"(p) : "r"(vmax[j]), "r"(t2));
      m |= p << j;
    }
    return m;
  }
  __device__ __forceinline__ float elem(int j, int e) const {
    const uint32_t q = w[j][e >> 1];
    return (e & 1) ? bf16hi(q) : bf16lo(q);
  }
  // sum exp(x - m) over the lane's elements (fixed order)
  __device__ __forceinline__ float lane_sumexp(float nml) {
    const unsigned long long L2E2 = pk2(VS_LOG2E, VS_LOG2E), N2 = pk2(nml, nml);
    unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int j = 0; j < VPL; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float t0, t1;
        up2(fma2(pk2(bf16lo(w[j][q]), bf16hi(w[j][q])), L2E2, N2), t0, t1);
        acc[q] = add2(acc[q], pk2(ex2f(t0), ex2f(t1)));
      }
    acc[0] = add2(acc[0], acc[1]);
    acc[2] = add2(acc[2], acc[3]);
    acc[0] = add2(acc[0], acc[2]);
    float a, b;
    up2(acc[0], a, b);
    return a + b;
  }
};

template <>
struct Seg<float> {
  static constexpr int EPV = 4;
  float x[VPL][4];
  float vm[VPL];
  __device__ __forceinline__ void load(const unsigned char* st, int nvec, int lane) {
    const float4* s = reinterpret_cast<const float4*>(st);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int v = lane + 32 * j;
      float4 q = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      if (v < nvec) q = s[v];
      x[j][0] = q.x;
      x[j][1] = q.y;
      x[j][2] = q.z;
      x[j][3] = q.w;
    }
  }
  __device__ __forceinline__ float lane_max() {
#pragma unroll
    for (int j = 0; j < VPL; ++j) vm[j] = fmaxf(fmaxf(x[j][0], x[j][1]), fmaxf(x[j][2], x[j][3]));
    return fmaxf(fmaxf(fmaxf(vm[0], vm[1]), fmaxf(vm[2], vm[3])), fmaxf(fmaxf(vm[4], vm[5]), fmaxf(vm[6], vm[7])));
  }
  __device__ __forceinline__ float vec_max(int j) const { return vm[j]; }
  __device__ __forceinline__ void load_full(const unsigned char* st, int lane) {
    const float4* s = reinterpret_cast<const float4*>(st);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const float4 q = s[lane + 32 * j];
      x[j][0] = q.x;
      x[j][1] = q.y;
      x[j][2] = q.z;
      x[j][3] = q.w;
    }
  }
  __device__ __forceinline__ unsigned pass_mask(float tx) const {
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < VPL; ++j) m |= (vm[j] >= tx ? 1u : 0u) << j;
    return m;
  }
  __device__ __forceinline__ float elem(int j, int e) const { return x[j][e]; }
  __device__ __forceinline__ float lane_sumexp(float nml) {
    const unsigned long long L2E2 = pk2(VS_LOG2E, VS_LOG2E), N2 = pk2(nml, nml);
    unsigned long long acc[2] = {0ull, 0ull};
#pragma unroll
    for (int j = 0; j < VPL; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float t0, t1;
        up2(fma2(pk2(x[j][2 * q], x[j][2 * q + 1]), L2E2, N2), t0, t1);
        acc[q] = add2(acc[q], pk2(ex2f(t0), ex2f(t1)));
      }
    acc[0] = add2(acc[0], acc[1]);
    float a, b;
    up2(acc[0], a, b);
    return a + b;
  }
};

struct Cand {
  uint64_t theta;  // every element not in buf has key <= theta (0: none filtered)
  float theta_x;
  int cnt;
};

// ---- register-resident top-M list ------------------------------------------
// Lane i < M holds the i-th largest logit key of the piece so far (0 = empty);
// θ = max(bootstrap key, M-th key once the list is full).  Every element not
// in the list has key <= θ.  Insertion is warp-synchronous (one ballot).
struct TopList {
  uint64_t tk;     // this lane's entry
  uint64_t theta;  // warp-uniform
  float theta_x;
};
__device__ __forceinline__ void tl_insert(TopList& t, uint64_t k, int Meff, int lane) {
  const int pos = __popc(__ballot_sync(FULL, t.tk > k));
  if (pos >= Meff) return;  // uniform
  const uint64_t up = (uint64_t)__shfl_up_sync(FULL, (unsigned long long)t.tk, 1);
  t.tk = lane == pos ? k : (lane > pos && lane < Meff ? up : t.tk);
  const uint64_t last = (uint64_t)__shfl_sync(FULL, (unsigned long long)t.tk, Meff - 1);
  if (last > t.theta) {
    t.theta = last;
    t.theta_x = unord_f32((uint32_t)(last >> 32));
  }
}
// Candidates `k` held by lanes with cnd set (keys > θ at test time), in lane order.
__device__ __forceinline__ void tl_insert_ballot(TopList& t, bool cnd, uint64_t k, int Meff, int lane) {
  unsigned b = __ballot_sync(FULL, cnd);
  while (b) {
    const int src = __ffs(b) - 1;
    b &= b - 1;
    const uint64_t kk = (uint64_t)__shfl_sync(FULL, (unsigned long long)k, src);
    if (kk > t.theta) tl_insert(t, kk, Meff, lane);
  }
}
// Insert this lane's elements of the vectors flagged in `pm` (bit j: vector
// lane + 32*j of the segment in shared memory holds an element >= θx).
template <typename T>
__device__ __noinline__ TopList append_vecs(TopList t, unsigned pm, const unsigned char* __restrict__ st,
                                            int nvec, int tok_base, int Meff) {
  constexpr int EPV = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const T* el = reinterpret_cast<const T*>(st);
  // vectors past the end of a partial segment hold stale bytes: never flagged
  for (int j = 0; j < VPL; ++j)
    if (lane + 32 * j >= nvec) pm &= ~(1u << j);
  while (__any_sync(FULL, pm != 0)) {
    const int j = pm ? __ffs(pm) - 1 : 0;
    const int v = lane + 32 * j;
    unsigned em = 0;
    if (pm) {
#pragma unroll
      for (int e = 0; e < EPV; ++e)
        if (to_f32<T>(el[v * EPV + e]) >= t.theta_x) em |= 1u << e;
      pm &= pm - 1;
    }
    while (__any_sync(FULL, em != 0)) {
      const int e = em ? __ffs(em) - 1 : 0;
      const uint64_t k = vkey(to_f32<T>(el[v * EPV + e]), tok_base + v * EPV + e);
      const bool cnd = em != 0 && k > t.theta;
      em &= em - 1;
      tl_insert_ballot(t, cnd, k, Meff, lane);
    }
  }
  return t;
}

// Workspace: one record per row, laid out by (V, dtype) only — the same row
// always finds its counter at the same address whatever R_grid a call uses.
//   int32 cnt; int32 pad[3]; float2 seg_ms[nseg]; PartRec parts[nseg]
__host__ __device__ __forceinline__ int64_t row_stride(int nseg) {
  return 16 + (int64_t)nseg * 8 + (int64_t)nseg * (int64_t)sizeof(PartRec);
}

template <typename T, int NS>
__global__ void __launch_bounds__(NW * 32, 5) row_lse_topm_tma_kernel(
    const T* __restrict__ logits, int64_t ld, int V, int M, int R_host, const int* __restrict__ d_R,
    int* __restrict__ top_tok, float* __restrict__ top_logp, float* __restrict__ row_lse,
    int* __restrict__ fb_count, int normalized, unsigned char* __restrict__ ws, int flush_min, int dbg) {
  VS_PDL_ENTRY();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  WarpSmem<NS>* all = reinterpret_cast<WarpSmem<NS>*>(smem_raw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem<NS>& S = all[wid];
  const int R = d_R ? *d_R : R_host;
  constexpr int EPV = 16 / sizeof(T);
  const int vrow = (int)(((int64_t)V * sizeof(T)) / 16);  // full 16-byte vectors per row
  const int tail0 = vrow * EPV;                             // first scalar-tail element
  const int nseg = (vrow * 16 + SEGB - 1) / SEGB;
  const int last_bytes = vrow * 16 - (nseg - 1) * SEGB;
  const int64_t total = (int64_t)R * nseg;
  const int64_t G = (int64_t)gridDim.x * NW;
  const int64_t w = (int64_t)blockIdx.x * NW + wid;
  const int64_t a = w * total / G, b = (w + 1) * total / G;
  if (a >= b) return;
  const int Meff = M < V ? M : V;
  const int flush_at = max(flush_min, Meff + 8);
  const uint64_t pol = policy_evict_first();
  const unsigned char* base = reinterpret_cast<const unsigned char*>(logits);
  const int64_t ldb = ld * (int64_t)sizeof(T);
  const int64_t rs = row_stride(nseg);

  // issue cursor (lane 0): next segment to fetch, as (row, seg)
  int ir = (int)(a / nseg), isg = (int)(a % nseg);
  int64_t ix = a;
  auto issue = [&](int st) {
    const unsigned nb = (unsigned)(isg == nseg - 1 ? last_bytes : SEGB);
    mbar_expect_tx(&S.bar[st], nb);
    bulk_g2s(S.stage[st], base + ir * ldb + (int64_t)isg * SEGB, nb, &S.bar[st], pol);
    ++ix;
    if (++isg == nseg) {
      isg = 0;
      ++ir;
    }
  };
  if (lane == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&S.bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < NS && ix < b; ++i) issue(i);
  }
  __syncwarp();

  TopList c{0ull, 0ull, -INFINITY};
  float pm = -INFINITY, ps = 0.0f;  // in-order fold of this piece's segments
  bool whole = false, boot = true;
  int r = (int)(a / nseg), sgi = (int)(a % nseg);
  int st = 0;
  unsigned phase = 0;
  int piece0 = sgi;  // first segment of the current piece
  whole = sgi == 0 && (int64_t)r * nseg + nseg <= b;

  for (int64_t x = a; x < b; ++x) {
    mbar_wait(&S.bar[st], phase);
    if (dbg & 2) {  // timing knob: stream only (results invalid)
      __syncwarp();
      if (lane == 0 && ix < b) issue(st);
      if (++st == NS) {
        st = 0;
        phase ^= 1u;
      }
      continue;
    }
    Seg<T> sg;
    const bool last_seg = sgi == nseg - 1;
    const int nvec = (last_seg ? last_bytes : SEGB) >> 4;
    if (nvec == SEGB / 16)
      sg.load_full(S.stage[st], lane);
    else
      sg.load(S.stage[st], nvec, lane);
    float lm = sg.lane_max();
    // scalar tail of the row (V*sizeof(T) not a multiple of 16): last segment
    float tx = -INFINITY;
    if (last_seg && tail0 + lane < V) {
      tx = to_f32<T>(*reinterpret_cast<const T*>(base + r * ldb + (int64_t)(tail0 + lane) * sizeof(T)));
      lm = fmaxf(lm, tx);
    }
    // lane-local sum of exp(x - lm): off the warp-reduction critical path
    float sl = 0.0f;
    if (!(dbg & 8) && lm != -INFINITY) {
      const float nml = -lm * VS_LOG2E;
      sl = sg.lane_sumexp(nml);
      if (last_seg && tail0 + lane < V) sl += ex2f(fmaf(tx, VS_LOG2E, nml));
    }
    float mseg = lm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mseg = fmaxf(mseg, __shfl_xor_sync(FULL, mseg, o));
    if (boot) {  // θ bootstrap on a piece's first segment: M-th largest lane maximum
      boot = false;
      float v = lm;
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const float o = __shfl_xor_sync(FULL, v, j);
          v = (((lane & k) == 0) == ((lane & j) == 0)) ? fmaxf(v, o) : fminf(v, o);
        }
      const float t0 = __shfl_sync(FULL, v, Meff - 1);
      if (t0 != -INFINITY) {
        c.theta = (uint64_t)ord_f32(t0) << 32;
        c.theta_x = t0;
      }
    }
    if (!(dbg & 4) && mseg >= c.theta_x) {  // warp-uniform: this segment may hold candidates
      unsigned pmask = lm >= c.theta_x ? sg.pass_mask(c.theta_x) : 0u;
      if (__any_sync(FULL, pmask != 0))
        c = append_vecs<T>(c, pmask, S.stage[st], nvec, sgi * (SEGB / (int)sizeof(T)), Meff);
      if (last_seg) {
        const uint64_t k = vkey(tx, tail0 + lane);
        tl_insert_ballot(c, tx >= c.theta_x && k > c.theta, k, Meff, lane);
      }
    }
    // segment sum relative to the segment max (fixed lane order -> deterministic)
    float sseg = lm == -INFINITY ? 0.0f : sl * ex2f((lm - mseg) * VS_LOG2E);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sseg += __shfl_xor_sync(FULL, sseg, o);
    __syncwarp();  // every lane is done with the stage -> refill it
    if (lane == 0 && ix < b) issue(st);
    unsigned char* rec = ws + (int64_t)r * rs;
    if (whole) {
      fold(pm, ps, mseg, sseg);
    } else if (lane == 0) {
      reinterpret_cast<float2*>(rec + 16)[sgi] = make_float2(mseg, sseg);
    }
    // advance the consume cursor
    if (++st == NS) {
      st = 0;
      phase ^= 1u;
    }
    const bool piece_end = last_seg || x + 1 == b;
    const int cur_r = r;
    if (++sgi == nseg) {
      sgi = 0;
      ++r;
    }
    if (!piece_end) continue;
    const bool was_whole = whole;
    const int first = piece0;
    // next piece starts at (r, sgi) == (cur_r + 1, 0)
    piece0 = 0;
    whole = (int64_t)r * nseg + nseg <= b;
    boot = true;
    if (was_whole) {
      const float lse = normalized ? 0.0f
                                   : ((pm == -INFINITY || ps == 0.0f) ? -INFINITY : pm + logf(ps));
      // re-key the list by logp (monotone in the logit; ties re-sorted by token)
      uint64_t kk = 0;
      if (c.tk) kk = row_key(__fsub_rn(unord_f32((uint32_t)(c.tk >> 32)), lse), (int)(0xffffffffu - (uint32_t)c.tk));
      kk = warp_sort_desc(kk, lane);
      finish_sorted<T>(reinterpret_cast<const T*>(base + cur_r * ldb), V, M, Meff, lse, kk, c.theta, S.buf,
                       S.sel, reinterpret_cast<unsigned*>(S.buf + 64), cur_r, top_tok, top_logp, row_lse,
                       fb_count, dbg != 0);
    } else {
      // split row: publish this piece; the last one to arrive finishes the row
      __syncwarp();
      const int ccnt = __popc(__ballot_sync(FULL, c.tk != 0));
      const int nmine = (int)(x + 1 - max(a, (int64_t)cur_r * nseg));
      PartRec* parts = reinterpret_cast<PartRec*>(rec + 16 + nseg * 8);
      PartRec* pr = &parts[first];
      if (lane < ccnt) pr->keys[lane] = c.tk;
      if (lane == 0) {
        pr->theta = c.theta;
        pr->cnt = ccnt;
      }
      __threadfence();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(reinterpret_cast<int*>(rec), nmine);
      old = __shfl_sync(FULL, old, 0);
      if (old + nmine == nseg) {
        // ---- finisher: all loads issued lane-parallel ---------------------------
        __threadfence();
        const float2* ms = reinterpret_cast<const float2*>(rec + 16);
        float m = -INFINITY, s = 0.0f;
        for (int q0 = 0; q0 < nseg; q0 += 32) {
          float2 v = make_float2(-INFINITY, 0.0f);
          if (q0 + lane < nseg) v = __ldcg(&ms[q0 + lane]);
          const int nq = min(32, nseg - q0);
          for (int q = 0; q < nq; ++q) fold(m, s, __shfl_sync(FULL, v.x, q), __shfl_sync(FULL, v.y, q));
        }
        const float lse = normalized ? 0.0f : ((m == -INFINITY || s == 0.0f) ? -INFINITY : m + logf(s));
        const int64_t x0 = (int64_t)cur_r * nseg;
        auto owner = [&](int64_t y) { return ((y + 1) * G - 1) / total; };
        // piece headers, lane-parallel: slot, key count, θ
        int np = 0, tot = 0;
        for (int q0 = 0; q0 < nseg; q0 += 32) {
          const int q = q0 + lane;
          const bool starts = q < nseg && (q == 0 || owner(x0 + q) != owner(x0 + q - 1));
          const unsigned bal = __ballot_sync(FULL, starts);
          int nq = 0;
          if (starts) {
            nq = __ldcg(&parts[q].cnt);
            const int i = np + __popc(bal & ((1u << lane) - 1u));
            S.pslot[i] = q;
            S.ths[i] = __ldcg(reinterpret_cast<const unsigned long long*>(&parts[q].theta));
          }
          int off = nq;  // inclusive prefix over the starting lanes
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, off, o);
            if (lane >= o) off += t;
          }
          if (starts) S.poff[np + __popc(bal & ((1u << lane) - 1u)) + 1] = tot + off;
          tot += __shfl_sync(FULL, off, 31);
          np += __popc(bal);
        }
        if (lane == 0) S.poff[0] = 0;
        __syncwarp();
        // keys, 4 loads per lane in flight, re-keyed by logp; compacted exactly
        // to the top-Meff by the final key whenever the buffer would overflow
        int cnt = 0;
        for (int e0 = 0; e0 < tot; e0 += 128) {
          if (cnt + 128 > CAPW) {
            warp_select(S.buf, cnt, Meff, S.sel);
            cnt = Meff;
          }
          uint64_t kk[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = e0 + 32 * u + lane;
            kk[u] = 0;
            if (e < tot) {
              int pi = 0;
              while (S.poff[pi + 1] <= e) ++pi;
              kk[u] = __ldcg(reinterpret_cast<const unsigned long long*>(&parts[S.pslot[pi]].keys[e - S.poff[pi]]));
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = e0 + 32 * u + lane;
            if (e < tot)
              S.buf[cnt + 32 * u + lane] = row_key(__fsub_rn(unord_f32((uint32_t)(kk[u] >> 32)), lse),
                                                   (int)(0xffffffffu - (uint32_t)kk[u]));
          }
          cnt += min(128, tot - e0);
          __syncwarp();
        }
        if (lane == 0) *reinterpret_cast<int*>(rec) = 0;  // ready for the next launch
        __syncwarp();
        finish_row<T>(reinterpret_cast<const T*>(base + cur_r * ldb), V, M, Meff, lse, cnt, S.ths, np, S.buf,
                      S.sel, reinterpret_cast<unsigned*>(S.buf + 64), cur_r, top_tok, top_logp, row_lse, fb_count, dbg != 0);
      }
    }
    c = TopList{0ull, 0ull, -INFINITY};
    pm = -INFINITY;
    ps = 0.0f;
  }
}

}  // namespace tk

// Workspace bytes for R_grid rows of V elements of `esize` bytes.
size_t tma_ws_bytes(int R_grid, int V, int esize) {
  const int vrow = (int)(((int64_t)V * esize) / 16);
  const int nseg = (vrow * 16 + tk::SEGB - 1) / tk::SEGB;
  return (size_t)R_grid * (size_t)tk::row_stride(nseg);
}

template <typename T>
int launch_tma(const void* logits, int64_t ld, int V, int M, int R_host, const int* d_R, int R_grid,
               int* top_tok, float* top_logp, float* row_lse, int* fb, int norm, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  if (tma_ws_bytes(R_grid, V, sizeof(T)) > ws_bytes) return VS_ERR_CONFIG;
  static int sms = 0, ctas = 0, ns = 0, flush_min = 16, dbg = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* e = getenv("VS_K1T_CTAS");  // 0 = as many as fit
    ctas = e ? atoi(e) : 0;
    const char* n = getenv("VS_K1T_NS");
    ns = n ? atoi(n) : 2;
    const char* f = getenv("VS_K1_FLUSH");
    if (f) flush_min = atoi(f);
    const char* d = getenv("VS_K1T_DBG");  // timing knob only: 1 no append, 2 stream only
    if (d) dbg = atoi(d);
  }
  const T* x = static_cast<const T*>(logits);
#define VS_K1T(NS_)                                                                                  \
  do {                                                                                               \
    auto kern = tk::row_lse_topm_tma_kernel<T, NS_>;                                                 \
    const int smem = tk::NW * (int)sizeof(tk::WarpSmem<NS_>);                                        \
    static int fit = 0;                                                                              \
    if (!fit) {                                                                                      \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                 \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kern, tk::NW * 32, smem);                  \
      if (fit < 1) fit = 1;                                                                          \
    }                                                                                                \
    const int grid = sms * (ctas > 0 ? min(ctas, fit) : fit);                                        \
    vs::vs_launch(kern, dim3(grid), dim3(tk::NW * 32), smem, st, x, ld, V, M, R_host, d_R, top_tok, top_logp, row_lse, fb, norm, \
                                          static_cast<unsigned char*>(ws), flush_min, dbg);               \
  } while (0)
  switch (ns) {
    case 3: VS_K1T(3); break;
    case 4: VS_K1T(4); break;
    default: VS_K1T(2); break;
  }
#undef VS_K1T
  VS_CUDA_RET();
}

// Dispatch: the split-row TMA kernel wins for wider per-row selections
// (M = 32: 2.4x the warp-per-row kernel at full width); for M <= 8 the two are
// at parity at full width and the warp-per-row kernel is ~7% faster on the
// small WMT steps, so it stays the default there.  VS_K1_IMPL=tma|legacy
// overrides (A/B measurement).
bool tma_eligible(const void* logits, int64_t ld, int V, int M, int esize, bool pinned) {
  static int impl = -1;  // -1 auto, 0 legacy, 1 tma
  if (impl == -1) {
    const char* e = getenv("VS_K1_IMPL");
    impl = e ? (e[0] == 't' ? 1 : (e[0] == 'l' ? 0 : 2)) : 2;
    if (getenv("VS_K1_LEGACY")) impl = 0;
  }
  if (!pinned && impl == 0) return false;
  if (!pinned && impl == 2 && M <= 8) return false;
  return M <= tk::MAXM && (int64_t)V * esize >= tk::SEGB && (int64_t)V * esize <= (int64_t)tk::MAXP * tk::SEGB &&
         ((uintptr_t)logits & 15) == 0 &&
         ((ld * esize) & 15) == 0;
}

template int launch_tma<float>(const void*, int64_t, int, int, int, const int*, int, int*, float*, float*, int*,
                               int, void*, size_t, cudaStream_t);
template int launch_tma<__nv_bfloat16>(const void*, int64_t, int, int, int, const int*, int, int*, float*,
                                       float*, int*, int, void*, size_t, cudaStream_t);

}  // namespace vs

extern "C" size_t vs_row_lse_topm_ws_bytes(int32_t R_grid, int32_t V, int32_t dtype) {
  dtype &= ~(VS_ROWS_NORMALIZED | VS_K1_SPLIT | VS_K1_WARP);
  return vs::tma_ws_bytes(R_grid, V, dtype == VS_DTYPE_F32 ? 4 : 2);
}
