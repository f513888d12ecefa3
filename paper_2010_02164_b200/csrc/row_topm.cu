// K1 row_lse_topM: fused log-softmax + per-row top-M (sm_100a).
//
// Replaces bb/model.py:216-217 (log-softmax of one |V| row) and
// bb/search.py:63-73 (_candidate_pool: first M of sorted(range(V),
// key=(-row[t], t))), for every scored row of a timestep at once.
//
// W warps per row (W from the device-side row count, 8 warps per CTA).  The row
// is read from HBM exactly once: 16-byte non-allocating vector loads, U vectors
// per lane per batch, double-buffered in registers (or a per-warp shared-memory
// ring filled by cp.async.bulk).  Per element the hot loop does only the online
// log-sum-exp (FFMA2, ex2, FADD2) against a warp-uniform, lazily raised max, and
// per vector one compare of its max against a warp-uniform candidate threshold
// θ (one warp vote guards both rare paths):
//   * M <= 32: candidates live in a register top-list (lane j holds the j-th
//     key; 32-bit keys for bf16 rows with |V| < 65536), seeded from the lane
//     maxima of the first two batches, so θ is always the exact M-th key;
//   * M > 32: passing elements are appended to a per-warp shared-memory buffer
//     (ballot compaction); when it fills, M argmax rounds keep the top-M and
//     raise θ.
// Epilogue: warp-reduce lse, re-key the candidates by the contract value
// logp = fp32(x - lse) with token-ascending ties, M warp-argmax rounds, and an
// exact verification that no element filtered out by θ can reach the M-th
// (logp, token) key — tie-aware, using the next-smaller representable input
// value.  Rows that cannot be proven fall back to an exact warp radix select
// over 64-bit keys.  Every decision is a pure function of the row.
#include "common.cuh"
#include "select_common.cuh"
#include <cstdlib>
#include <type_traits>

namespace vs {
namespace {

constexpr int WPC = 8;                 // warps per CTA (W warps per row, WPC/W rows)
constexpr int NSEG = WPC;              // fixed lse segments per row (any W divides it)
constexpr int CAPW = 416;              // per-warp candidate buffer (keys)
constexpr int FLUSH_MIN = 16;
#ifndef PICKW_C0
#define PICKW_C0 0.5f  // per-task fixed cost relative to streaming one row
#endif          // raise θ once this many candidates are buffered
constexpr unsigned FULL = 0xffffffffu;

template <typename T>
__device__ __forceinline__ void unpack(const uint4& v, float (&x)[16 / sizeof(T)]);
template <>
__device__ __forceinline__ void unpack<float>(const uint4& v, float (&x)[4]) {
  x[0] = __uint_as_float(v.x);
  x[1] = __uint_as_float(v.y);
  x[2] = __uint_as_float(v.z);
  x[3] = __uint_as_float(v.w);
}
template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4& v, float (&x)[8]) {
  x[0] = bf16lo(v.x);
  x[1] = bf16hi(v.x);
  x[2] = bf16lo(v.y);
  x[3] = bf16hi(v.y);
  x[4] = bf16lo(v.z);
  x[5] = bf16hi(v.z);
  x[6] = bf16lo(v.w);
  x[7] = bf16hi(v.w);
}

// Next smaller value representable in the input dtype (for the tie-aware proof).
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

// Packed fp32x2 helpers (sm_100: FFMA2 / FADD2 / FMUL2 issue two lanes of work).
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
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// Bulk L2 prefetch (TMA engine, no registers / smem held while in flight).
__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ float ex2f(float x) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
  return e;
}
// The running max m of the online log-sum-exp is warp-uniform and lazily raised:
// it only moves when some element exceeds m + RESCALE_MARGIN, so exp(x - m) stays
// <= e^16 (sums stay far from fp32 overflow) and the hot loop needs no per-vector
// rescale (an exponential per vector saved).
constexpr float RESCALE_MARGIN = 16.0f;

// logit key: larger = earlier in (value desc, token asc).
__device__ __forceinline__ uint64_t vkey(float x, int tok) {
  return ((uint64_t)ord_f32(x) << 32) | (uint64_t)(0xffffffffu - (uint32_t)tok);
}

// Keep the top-`keep` keys of buf[0..cnt) in buf[0..keep) (sorted desc) using
// `keep` warp-argmax rounds; returns the keep-th key (0 if fewer entries).
__device__ __noinline__ uint64_t warp_select(uint64_t* __restrict__ buf, int cnt, int keep,
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
    if (wb != 0 && lb == wb) buf[li] = 0;  // unique owner (keys are distinct)
    if (lane == 0) sel[r] = wb;
    last = wb;
    __syncwarp();
  }
  for (int r = lane; r < keep; r += 32) buf[r] = sel[r];
  __syncwarp();
  return last;
}

// Exact fallback: M-th largest 64-bit (logp, token) key by MSB-first radix
// select (8 x 8-bit passes over the row), then collect + rank the top-M.
template <typename T>
__device__ __noinline__ void warp_exact_select(const T* __restrict__ row, int V, float lse, int Meff,
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
  int cnt = 0;  // exactly Meff keys are >= prefix (keys are unique)
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

struct Cand {
  uint64_t theta;  // candidate threshold key (warp-uniform); 0 = everything passes
  float theta_x;   // logit part of theta (-inf when theta == 0)
  int cnt;         // buffer fill (warp-uniform)
};

// Candidate append (warp-synchronous, taken only when some lane's vector max
// reaches θ): a per-lane bitmask of elements >= θx, then one ballot round per
// pending element (usually one round), keys compacted into the warp buffer.
template <bool INL>
__device__ __forceinline__ Cand append_fast(Cand c, float x0, float x1, float x2, float x3, float x4,
                                         float x5, float x6, float x7, int n, int tok0,
                                         uint64_t* __restrict__ buf, uint64_t* __restrict__ sel, int Meff,
                                         int flush_at) {
  const float x[8] = {x0, x1, x2, x3, x4, x5, x6, x7};
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  unsigned mask = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < n && x[j] >= c.theta_x) mask |= 1u << j;
  while (__any_sync(FULL, mask != 0)) {
    const int j = mask ? __ffs(mask) - 1 : 0;
    float xj = x[0];
#pragma unroll
    for (int q = 1; q < 8; ++q) xj = (j == q) ? x[q] : xj;
    const uint64_t k = vkey(xj, tok0 + j);
    const bool cnd = mask != 0 && k > c.theta;
    mask &= mask - 1;
    const unsigned b = __ballot_sync(FULL, cnd);
    if (cnd) buf[c.cnt + __popc(b & lt_mask)] = k;
    c.cnt += __popc(b);
  }
  if (c.cnt >= flush_at) {
    __syncwarp();
    const uint64_t th = warp_select(buf, c.cnt, Meff, sel);
    if (th > c.theta) {
      c.theta = th;
      c.theta_x = unord_f32((uint32_t)(th >> 32));
    }
    c.cnt = Meff;
  }
  return c;
}

// Register top-list (Meff <= 32): lane j holds the j-th largest key seen so far
// and θ is always the exact Meff-th key, so no buffer flushes and the fewest
// possible candidate entries (≈ M·ln(V/M) per row).  Keys are 64-bit
// (ord(x) << 32 | ~token) or, for bf16 rows with |V| < 65536, 32-bit
// (ord16(x) << 16 | 0xFFFF - token): same order, half the shuffles/compares.
// A key whose token field is 0 means "token +inf" (x == θx still passes).
template <typename K>
struct KeyOps;
template <>
struct KeyOps<uint64_t> {
  static __device__ __forceinline__ uint64_t key(float x, int tok) { return vkey(x, tok); }
  static __device__ __forceinline__ uint64_t bound(float x) { return (uint64_t)ord_f32(x) << 32; }
  static __device__ __forceinline__ float val(uint64_t k) { return unord_f32((uint32_t)(k >> 32)); }
  static __device__ __forceinline__ uint64_t to64(uint64_t k) { return k; }
};
template <>
struct KeyOps<uint32_t> {
  static __device__ __forceinline__ uint32_t key(float x, int tok) {
    return (ord_f32(x) & 0xFFFF0000u) | (0xFFFFu - (uint32_t)tok);
  }
  static __device__ __forceinline__ uint32_t bound(float x) { return ord_f32(x) & 0xFFFF0000u; }
  static __device__ __forceinline__ float val(uint32_t k) {
    return unord_f32((k & 0xFFFF0000u) | ((k & 0x80000000u) ? 0u : 0xFFFFu));
  }
  static __device__ __forceinline__ uint64_t to64(uint32_t k) {
    if (k == 0u) return 0ull;
    const uint64_t hi = (uint64_t)ord_f32(val(k)) << 32;
    return (k & 0xFFFFu) ? hi | (uint64_t)(0xffffffffu - (0xFFFFu - (k & 0xFFFFu))) : hi;
  }
};
template <typename K>
struct TopList {
  K tk;        // this lane's entry (0 = empty)
  K theta;     // exact Meff-th key (warp-uniform; 0 = everything passes)
  float theta_x;
};
template <typename K>
__device__ __forceinline__ void tl_insert(TopList<K>& t, K k, int Meff, int lane) {
  const int pos = __popc(__ballot_sync(FULL, t.tk > k));
  if (pos >= Meff || __any_sync(FULL, t.tk == k)) return;  // uniform (== : a seeded key seen again)
  const K up = (K)__shfl_up_sync(FULL, t.tk, 1);
  t.tk = lane == pos ? k : (lane > pos && lane < Meff ? up : t.tk);
  const K last = (K)__shfl_sync(FULL, t.tk, Meff - 1);
  if (last > t.theta) {
    t.theta = last;
    t.theta_x = KeyOps<K>::val(last);
  }
}
// Insert this lane's elements >= θx of one vector (warp-synchronous; taken only
// when some lane's vector max reaches θx): one ballot round per pending element.
template <typename K>
__device__ __forceinline__ void tl_append(TopList<K>& t, const float (&x)[8], int n, int tok0, int Meff) {
  const int lane = threadIdx.x & 31;
  unsigned em = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < n && x[j] >= t.theta_x) em |= 1u << j;
  while (__any_sync(FULL, em != 0)) {
    const int j = em ? __ffs(em) - 1 : 0;
    float xj = x[0];
#pragma unroll
    for (int q = 1; q < 8; ++q) xj = (j == q) ? x[q] : xj;
    const K k = KeyOps<K>::key(xj, tok0 + j);
    const bool cnd = em != 0 && k > t.theta;
    em &= em - 1;
    unsigned b = __ballot_sync(FULL, cnd);
    while (b) {
      const int src = __ffs(b) - 1;
      b &= b - 1;
      const K kk = (K)__shfl_sync(FULL, k, src);
      if (kk > t.theta) tl_insert(t, kk, Meff, lane);
    }
  }
}
// Seed the list from the 32 lane maxima (value, first token) of the bootstrap
// window: a bitonic sort leaves the top Meff in lanes 0..Meff-1, i.e. exactly
// the state after inserting them.  Returns the window maximum.
template <typename K>
__device__ __forceinline__ float tl_seed(TopList<K>& t, float lm, int lt, int Meff, int lane) {
  K k = lm == -INFINITY ? (K)0 : KeyOps<K>::key(lm, lt);
#pragma unroll
  for (int s = 2; s <= 32; s <<= 1)
#pragma unroll
    for (int j = s >> 1; j > 0; j >>= 1) {
      const K o = (K)__shfl_xor_sync(FULL, k, j);
      k = (((lane & s) == 0) == ((lane & j) == 0)) ? (k > o ? k : o) : (k < o ? k : o);
    }
  t.tk = lane < Meff ? k : (K)0;
  const K last = (K)__shfl_sync(FULL, k, Meff - 1);
  if (last != (K)0) {
    t.theta = last;
    t.theta_x = KeyOps<K>::val(last);
  }
  const K top = (K)__shfl_sync(FULL, k, 0);
  return top ? KeyOps<K>::val(top) : -INFINITY;
}

// Warps per row from the live row count: minimise the makespan
// ceil(R*W/T) * (c0 + 1/W) over W in {1,2,4,8} (T = resident warps, c0 =
// per-task boot/epilogue cost relative to streaming a whole row) — balances
// wave quantisation against the per-warp fixed cost.
__host__ __device__ __forceinline__ int pick_w(int R, int V, int T, float c0 = PICKW_C0) {
  if (V < 4096 || R <= 0) return 1;
  if (c0 < 0.0f) return min(WPC, (int)(-c0));  // VS_K1_C0=-W pins W (measurement knob)
  int best = 1;
  float bc = 1e30f, inv = 1.0f;  // 32-bit unsigned math: this runs in every warp's prologue
  for (int w = 1; w <= WPC; w <<= 1, inv *= 0.5f) {
    const float waves = (float)(((unsigned)R * (unsigned)w + (unsigned)T - 1u) / (unsigned)T);
    const float cost = waves * (c0 + inv);
    if (cost < bc - 1e-6f) {
      bc = cost;
      best = w;
    }
  }
  return best;
}

struct PartSmem {  // per-warp results exchanged between the W warps of a row
  float m, s;
  uint64_t theta;
  float theta_x;
  int cnt;
};

// W warps per row (W in {1,2,4}; 4/W rows per CTA).  Warp `part` of a row
// streams vectors [part*seg, (part+1)*seg); the row's leader warp combines.
// TLK: 0 = candidates in the flushed shared-memory buffer; 1/2 = register
// top-list (Meff <= 32) with 64/32-bit keys.  NS > 0 (ring): the warp's slice streams through a
// private ring of NS shared-memory chunks of U·512 B filled by cp.async.bulk
// (one lane issues, per-chunk mbarriers) instead of register double-buffering,
// so NS-1 chunks stay in flight while one is reduced and no registers are held
// by loads.
template <typename T, int U, int MINB, int TLK, int NS>
__global__ void __launch_bounds__(WPC * 32, MINB) row_lse_topm_warp_kernel(
    const T* __restrict__ logits, int64_t ld, int V, int M, int R_host, const int* __restrict__ d_R,
    int* __restrict__ top_tok, float* __restrict__ top_logp, float* __restrict__ row_lse,
    int* __restrict__ fb_count, int normalized, int sms, int flush_min, int pf_batches,
    int warps_per_sm, float c0) {
  VS_PDL_ENTRY();
  constexpr int VEC = 16 / sizeof(T);
  constexpr bool TL = TLK > 0;
  using K = typename std::conditional<TLK == 2, uint32_t, uint64_t>::type;
  constexpr int CAP = TL ? 128 : CAPW;  // TL: <= 4 parts x 32 keys at the merge
  __shared__ uint64_t sbuf[WPC][CAP];
  __shared__ uint64_t rbar[WPC][NS > 0 ? NS : 1];
  __shared__ uint64_t ssel[WPC][VS_MAX_M];
  __shared__ unsigned shist[WPC][256];
  __shared__ PartSmem spart[WPC];
  __shared__ float2 segp[WPC][NSEG + 1];  // per row (at its leader): segment (m, s) pairs
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int R = d_R ? *d_R : R_host;
  if ((int)blockIdx.x >= R) return;  // idle for any W (a CTA starts at row >= blockIdx.x)
  const int W = pick_w(R, V, sms * warps_per_sm, c0);
  const int part = wid % W, leader = wid - part;
  const int r = blockIdx.x * (WPC / W) + wid / W;
  if (blockIdx.x * (WPC / W) >= R) return;  // whole CTA idle (uniform)
  const bool active = r < R;
  uint64_t* buf = sbuf[wid];
  uint64_t* sel = ssel[wid];
  const int Meff = M < V ? M : V;
  const int flush_at = max(flush_min, Meff + 8);
  const T* __restrict__ row = logits + (int64_t)(active ? r : 0) * ld;

  // m starts at a finite floor (logits must be > -1e30 or -inf) so the hot loop
  // needs no -inf guards: ex2(x*log2e - m*log2e) is 0 for x = -inf and the
  // branchless rescale ex2((m_old - m_new)*log2e) is 0 on the first vector.
  constexpr float M_FLOOR = -1e30f;
  float m = M_FLOOR, m_thr = M_FLOOR + RESCALE_MARGIN;  // warp-uniform (see RESCALE_MARGIN)
  unsigned long long nml2 = pk2(-M_FLOOR * VS_LOG2E, -M_FLOOR * VS_LOG2E);
  unsigned long long s01 = pk2(0.0f, 0.0f);  // (even, odd) partial sums of exp(x - m)
  const unsigned long long L2E2 = pk2(VS_LOG2E, VS_LOG2E);
  Cand c{0ull, -INFINITY, 0};
  TopList<K> tl{(K)0, (K)0, -INFINITY};
  // one warp vote per vector guards both rare paths: gate = min(θx, m_thr)
  float gate = fminf(TL ? tl.theta_x : c.theta_x, m_thr);
  // Partition-invariant lse: the row is cut into NSEG fixed segments (plus the
  // scalar tail as segment NSEG); each segment's (m, s) pair starts from a fresh
  // m and is streamed with the same lane mapping whichever warp owns it, and the
  // row's lse is the in-order left fold of the NSEG+1 pairs.  So lse (and every
  // logp) of a row is bit-identical whatever W the live row count picks.
  auto seg_flush = [&](int idx) {
    float a, b;
    up2(s01, a, b);
    float sv = a + b;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(FULL, sv, o);
    if (lane == 0) segp[wid - wid % W][idx] = make_float2(m, sv);
    m = M_FLOOR;
    m_thr = M_FLOOR + RESCALE_MARGIN;
    nml2 = pk2(-M_FLOOR * VS_LOG2E, -M_FLOOR * VS_LOG2E);
    s01 = pk2(0.0f, 0.0f);
    gate = fminf(TL ? tl.theta_x : c.theta_x, m_thr);
  };

  // Candidate path of one vector (warp-synchronous).
  auto cand = [&](const float (&x)[VEC], int n, int tok0) {
#ifndef K1_ABL_NOCAND  // ablation build only (tools/k1_ablate.sh)
    if (TL) {
      if constexpr (VEC == 8) {
        tl_append(tl, reinterpret_cast<const float(&)[8]>(x), n, tok0, Meff);
      } else {
        const float x8[8] = {x[0], x[1 % VEC], x[2 % VEC], x[3 % VEC], -INFINITY, -INFINITY, -INFINITY,
                             -INFINITY};
        tl_append(tl, x8, n, tok0, Meff);
      }
    } else if (VEC == 8)
      c = append_fast<true>(c, x[0], x[1], x[2], x[3], x[VEC > 4 ? 4 : 0], x[VEC > 5 ? 5 : 0],
                            x[VEC > 6 ? 6 : 0], x[VEC > 7 ? 7 : 0], n, tok0, buf, sel, Meff, flush_at);
    else
      c = append_fast<true>(c, x[0], x[1 % VEC], x[2 % VEC], x[3 % VEC], -INFINITY, -INFINITY, -INFINITY,
                            -INFINITY, n, tok0, buf, sel, Meff, flush_at);
#endif
  };
  auto consume = [&](const float (&x)[VEC], int n, int tok0) {
    float cm = x[0];
#pragma unroll
    for (int j = 1; j < VEC; ++j) cm = fmaxf(cm, x[j]);
    // One warp vote guards both rare paths: θx <= (warp max so far) <= m_thr, so
    // an element above m_thr also passes the candidate test.
    if (__any_sync(FULL, cm >= gate)) {
      if (__any_sync(FULL, cm > m_thr)) {  // raise the shared max, rescale the sums
        float mw = cm;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(FULL, mw, o));
        const float sc = ex2f((m - mw) * VS_LOG2E);
        s01 = mul2(s01, pk2(sc, sc));
        m = mw;
        m_thr = m + RESCALE_MARGIN;
        nml2 = pk2(-m * VS_LOG2E, -m * VS_LOG2E);
      }
      if (__any_sync(FULL, cm >= (TL ? tl.theta_x : c.theta_x))) cand(x, n, tok0);
      gate = fminf(TL ? tl.theta_x : c.theta_x, m_thr);
    }
#pragma unroll
    for (int j = 0; j < VEC; j += 2) {
      const unsigned long long t = fma2(pk2(x[j], x[j + 1]), L2E2, nml2);  // FFMA2: (x - m)*log2e
#ifdef K1_ABL_NOEXP
      s01 = add2(s01, t);  // ablation build only (tools/k1_ablate.sh)
#else
      float t0, t1;
      up2(t, t0, t1);
      s01 = add2(s01, pk2(ex2f(t0), ex2f(t1)));  // MUFU.EX2 + FADD2
#endif
    }
  };

  // θ bootstrap from the lane maxima (value, first token) of the first two
  // batches: the top-list is seeded with the top Meff of them (buffer mode: θ =
  // the Meff-th largest value), and the shared max m starts at the largest.
  auto boot = [&](float lm, int lt) {
    float m0;
    if constexpr (TL) {
      if (W > 1) {
        // the W parts of a row pool their 32 lane maxima: every part starts with
        // θ = the Meff-th largest of the W·32 (a bound with token "+inf", so every
        // element of that value passes) and an empty list.  The Meff largest maxima
        // are distinct elements >= θ, each inserted by its own part, so the merged
        // top-Meff is exact and the proof holds; a W-times larger window gives a
        // higher θ and fewer insertions per part.
        // the row's parts' candidate buffers (contiguous, unused until the epilogue)
        uint64_t* pool = sbuf[wid - part];
        pool[part * 32 + lane] = lm == -INFINITY ? 0ull : (uint64_t)KeyOps<K>::key(lm, lt);
        asm volatile("bar.sync %0, %1;" ::"r"(1 + wid / W), "r"(W * 32) : "memory");
        K kth = 0, prev = (K)~(K)0;
        for (int j = 0; j < Meff; ++j) {  // Meff rounds: largest key strictly below prev
          K b = 0;
          for (int q = 0; q < W; ++q) {
            const K vq = (K)pool[q * 32 + lane];
            b = (vq < prev && vq > b) ? vq : b;
          }
          if constexpr (sizeof(K) == 4) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const K ob = (K)__shfl_xor_sync(FULL, (uint32_t)b, o);
              b = ob > b ? ob : b;
            }
          } else {
            b = (K)warp_max_u64((uint64_t)b);
          }
          kth = prev = b;
          if (b == 0) break;
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + wid / W), "r"(W * 32) : "memory");  // pool read by all
        tl.tk = (K)0;
        if (kth != 0) {
          const float t0 = KeyOps<K>::val(kth);
          tl.theta = KeyOps<K>::bound(t0);
          tl.theta_x = t0;
        }
        m0 = 0.0f;
      } else {
        m0 = tl_seed(tl, lm, lt, Meff, lane);
      }
    } else {
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const float o = __shfl_xor_sync(FULL, lm, j);
          lm = (((lane & k) == 0) == ((lane & j) == 0)) ? fmaxf(lm, o) : fminf(lm, o);
        }
      const float t0 = __shfl_sync(FULL, lm, Meff - 1);
      m0 = __shfl_sync(FULL, lm, 0);
      if (t0 != -INFINITY) {
        c.theta = (uint64_t)ord_f32(t0) << 32;  // (t0, token = +inf): x == t0 still passes
        c.theta_x = t0;
      }
    }
    (void)m0;  // the running max is per segment (partition-invariant lse)
    gate = fminf(TL ? tl.theta_x : c.theta_x, m_thr);
  };
  // lane max with its first token over one vector (bootstrap only)
  auto lane_argmax = [&](const float (&x)[VEC], int tok0, float& lm, int& lt) {
#pragma unroll
    for (int j = 0; j < VEC; ++j)
      if (x[j] > lm) {
        lm = x[j];
        lt = tok0 + j;
      }
  };

  if (active) {
    const bool vec_ok = (reinterpret_cast<uintptr_t>(row) & 15) == 0;
    const int ntot = vec_ok ? V / VEC : 0;
    // NSEG segments of Qs vectors (a multiple of the double batch), NSEG/W per part
    constexpr int DB = 2 * 32 * U;
    const int Qs = ((ntot + NSEG - 1) / NSEG + DB - 1) / DB * DB;
    const int spp = NSEG / W;
    const int v0 = min(ntot, part * spp * Qs), v1 = min(ntot, v0 + spp * Qs);
    int segi = part * spp, seg_next = v0 + Qs;
    const uint4* __restrict__ vrow = reinterpret_cast<const uint4*>(row);
    if constexpr (NS > 0) {
      constexpr int CH = 32 * U;  // vectors per chunk
      extern __shared__ __align__(128) unsigned char ring_smem[];
      uint4* stg = reinterpret_cast<uint4*>(ring_smem) + (size_t)wid * NS * CH;
      uint64_t* bars = rbar[wid];
      const int nvt = v1 - v0, nch = (nvt + CH - 1) / CH;
      const uint64_t pol = tk::policy_evict_first();
      if (lane == 0) {
        for (int q = 0; q < NS; ++q) tk::mbar_init(&bars[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncwarp();
      auto issue = [&](int ch) {
        const int q = ch % NS;
        const unsigned bytes = (unsigned)min(CH, nvt - ch * CH) * 16u;
        tk::mbar_expect_tx(&bars[q], bytes);
        tk::bulk_g2s(stg + q * CH, vrow + v0 + ch * CH, bytes, &bars[q], pol);
      };
      if (lane == 0)
        for (int ch = 0; ch < min(NS, nch); ++ch) issue(ch);
      if (Meff <= 32) {  // bootstrap θ: M-th largest of 32 lane maxima over 2 chunks
        float lm = -INFINITY;
        int lt = 0;
        for (int ch = 0; ch < min(2, nch); ++ch) {
          tk::mbar_wait(&bars[ch], 0);
          const uint4* sv = stg + ch * CH;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = lane + 32 * u;
            if (ch * CH + i < nvt) {
              float x[VEC];
              unpack<T>(sv[i], x);
              lane_argmax(x, (v0 + ch * CH + i) * VEC, lm, lt);
            }
          }
        }
        boot(lm, lt);
      }
      for (int ch = 0; ch < nch; ++ch) {
        if (v0 + ch * CH == seg_next) {
          seg_flush(segi++);
          seg_next += Qs;
        }
        const int q = ch % NS;
        tk::mbar_wait(&bars[q], (unsigned)(ch / NS) & 1u);
        const uint4* sv = stg + q * CH;
        const int nv = min(CH, nvt - ch * CH), tok = (v0 + ch * CH) * VEC;
        if (nv == CH) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            float x[VEC];
            unpack<T>(sv[lane + 32 * u], x);
            consume(x, VEC, tok + (lane + 32 * u) * VEC);
          }
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = lane + 32 * u;
            if (__any_sync(FULL, i < nv)) {
              float x[VEC];
              if (i < nv) unpack<T>(sv[i], x);
              else
#pragma unroll
                for (int j = 0; j < VEC; ++j) x[j] = -INFINITY;
              consume(x, VEC, tok + i * VEC);
            }
          }
        }
        __syncwarp();
        if (lane == 0 && ch + NS < nch) issue(ch + NS);
      }
    } else {
      constexpr int BATCH = 32 * U;  // vectors per warp per batch
      uint4 cur[U], nxt[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = v0 + lane + 32 * u;
        if (i < v1) cur[u] = ldg_stream(vrow + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = v0 + BATCH + lane + 32 * u;
        if (i < v1) nxt[u] = ldg_stream(vrow + i);
      }
      if (Meff <= 32) {  // bootstrap θ: M-th largest of 32 lane maxima over 2 batches
        float lm = -INFINITY;
        int lt = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float x[VEC];
          if (v0 + lane + 32 * u < v1) {
            unpack<T>(cur[u], x);
            lane_argmax(x, (v0 + lane + 32 * u) * VEC, lm, lt);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float x[VEC];
          if (v0 + BATCH + lane + 32 * u < v1) {
            unpack<T>(nxt[u], x);
            lane_argmax(x, (v0 + BATCH + lane + 32 * u) * VEC, lm, lt);
          }
        }
        boot(lm, lt);
      }
      int base = v0;
      const int pf_dist = 2 * BATCH * pf_batches;  // vectors ahead of the demand loads
      if (lane == 0 && pf_batches > 0) {  // prime the L2 prefetch window
        const int p1 = min(v1, v0 + pf_dist);
        if (p1 > v0 + 2 * BATCH) l2_prefetch(vrow + v0 + 2 * BATCH, (unsigned)(p1 - v0 - 2 * BATCH) * 16u);
      }
      // full double-batches: no per-vector bounds checks
      for (; base + 2 * BATCH <= v1; base += 2 * BATCH) {
        if (base == seg_next) {
          seg_flush(segi++);
          seg_next += Qs;
        }
        if (lane == 0 && pf_batches > 0) {
          const int p0 = base + pf_dist, p1 = min(v1, p0 + 2 * BATCH);
          if (p1 > p0) l2_prefetch(vrow + p0, (unsigned)(p1 - p0) * 16u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float x[VEC];
          unpack<T>(cur[u], x);
          consume(x, VEC, (base + lane + 32 * u) * VEC);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = base + 2 * BATCH + lane + 32 * u;
          if (i < v1) cur[u] = ldg_stream(vrow + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float x[VEC];
          unpack<T>(nxt[u], x);
          consume(x, VEC, (base + BATCH + lane + 32 * u) * VEC);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = base + 3 * BATCH + lane + 32 * u;
          if (i < v1) nxt[u] = ldg_stream(vrow + i);
        }
      }
      // remainder (< 2 batches, already loaded into cur / nxt): checked
      if (base == seg_next && base < v1) {
        seg_flush(segi++);
        seg_next += Qs;
      }
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = base + h * BATCH + lane + 32 * u;
          if (__any_sync(FULL, i < v1)) {
            float x[VEC];
            if (i < v1) unpack<T>(h ? nxt[u] : cur[u], x);
            else
#pragma unroll
              for (int j = 0; j < VEC; ++j) x[j] = -INFINITY;
            consume(x, VEC, i * VEC);
          }
        }
      }
    }
    // close this part's segments (empty ones give (M_FLOOR, 0) pairs)
    while (segi < (part + 1) * spp) seg_flush(segi++);
    if (part == W - 1) {  // tail / unaligned rows: segment NSEG
      for (int i0 = ntot * VEC; i0 < V; i0 += 32) {
        const int i = i0 + lane;
        float x[VEC];
        x[0] = i < V ? to_f32<T>(row[i]) : -INFINITY;
#pragma unroll
        for (int j = 1; j < VEC; ++j) x[j] = -INFINITY;
        consume(x, 1, i);
      }
      seg_flush(NSEG);
    }
  }
  if (TL) {  // hand the list to the common epilogue as a sorted buffer
    const bool has = lane < Meff && tl.tk != (K)0;
    if (has) buf[lane] = KeyOps<K>::to64(tl.tk);
    c.cnt = __popc(__ballot_sync(FULL, has));
    c.theta = KeyOps<K>::to64(tl.theta);
    c.theta_x = tl.theta_x;
    __syncwarp();
  }
  // ---- lse: in-order left fold of the row's segment pairs ----------------------------
  // lane q holds pair q; the max and the rescaled sum are fixed xor trees over
  // the same NSEG+1 pairs in every warp of the row (partition-invariant)
  // the W warps of this row only (named barrier 1 + row-in-CTA): a row never
  // waits for the other rows of its CTA
  if (W > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + wid / W), "r"(W * 32) : "memory");
  else __syncwarp();
  float s;
  {
    const float2 pq = lane <= NSEG ? segp[leader][lane] : make_float2(-INFINITY, 0.0f);
    m = pq.x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
    s = pq.y > 0.0f ? pq.y * ex2f((pq.x - m) * VS_LOG2E) : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  }
  const float lse_raw = (m <= -1e30f || s == 0.0f) ? -INFINITY : m + logf(s);
  const float lse = normalized ? 0.0f : lse_raw;
  // ---- re-key own candidates by (logp, token) ---------------------------------------
  __syncwarp();
  for (int e = lane; e < c.cnt; e += 32) {
    const uint64_t k = buf[e];
    buf[e] = row_key(__fsub_rn(unord_f32((uint32_t)(k >> 32)), lse), (int)(0xffffffffu - (uint32_t)k));
  }
  if (W > 1) {
    if (lane == 0) {
      spart[wid].theta = c.theta;
      spart[wid].theta_x = c.theta_x;
      spart[wid].cnt = c.cnt;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + wid / W), "r"(W * 32) : "memory");
    if (part != 0 || !active) return;
    // leader: gather the other parts' candidates behind its own (CAPW suffices:
    // each part holds < flush_at + 256 entries only transiently; after the
    // stream it holds < flush_at <= 160, and W <= 4 parts -> keep top-Meff each)
    for (int q = 1; q < W; ++q) {
      const int nq = spart[leader + q].cnt;
      const uint64_t* bq = sbuf[leader + q];
      if (c.cnt + nq > CAP) {  // compact own buffer first (exact: by final key)
        __syncwarp();
        warp_select(buf, c.cnt, Meff, sel);
        c.cnt = Meff;
      }
      for (int e = lane; e < nq; e += 32) buf[c.cnt + e] = bq[e];
      c.cnt += nq;
      __syncwarp();
    }
  }
  if (!active) return;
  __syncwarp();
  const uint64_t kth = c.cnt >= Meff ? warp_select(buf, c.cnt, Meff, sel) : 0ull;
  // ---- proof that nothing filtered out by any part's θ precedes the M-th key -----
  bool ok = kth != 0ull;
  for (int q = 0; q < W && ok; ++q) {
    const uint64_t th = W > 1 ? spart[leader + q].theta : c.theta;
    const float tx = W > 1 ? spart[leader + q].theta_x : c.theta_x;
    if (th == 0ull) continue;  // that part kept every element it saw
    const uint32_t t_lp = (uint32_t)(kth >> 32);
    const int t_tok = key_tok(kth);
    const int th_tok = (int)(0xffffffffu - (uint32_t)th);  // -1 encodes "+inf token"
    // (a) values strictly below θ's logit: their logp <= fl(prev(θx) - lse)
    ok = ord_f32(__fsub_rn(prev_repr<T>(tx), lse)) < t_lp;
    // (b) values equal to θ's logit with a larger token than θ's
    if (ok) {
      const uint32_t lp = ord_f32(__fsub_rn(tx, lse));
      ok = lp < t_lp || (lp == t_lp && (th_tok == -1 || th_tok >= t_tok));
    }
  }
#ifdef K1_ABL_NOCAND
  ok = true;
#endif
  if (!ok) {
    warp_exact_select<T>(row, V, lse, Meff, shist[wid], buf, sel);
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

// Opt a kernel in to its dynamic shared memory once (static + dynamic > 48 KB).
void allow_dyn_smem(const void* kern, size_t dsm) {
  static const void* done[64];
  static int n = 0;
  for (int i = 0; i < n; ++i)
    if (done[i] == kern) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (n < 64) done[n++] = kern;
}

template <typename T>
int launch(const void* logits, int64_t ld, int V, int M, int R_host, const int* d_R, int rows, int* top_tok,
           float* top_logp, float* row_lse, int* fb, int norm, cudaStream_t st) {
  // warps per row: enough warps in flight for small steps (>= ~2 rows' worth per
  // SM-quarter), one warp per row once rows alone fill the machine.
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static int variant = -1, flush_min = FLUSH_MIN, pf = 0;  // knobs: VS_K1_VARIANT/_FLUSH/_PF/_C0
  static int tl_mode = 1;  // VS_K1_TL: 0 buffered candidates, 3 top-list with 64-bit keys only
  static float c0 = PICKW_C0;
  if (variant < 0) {
    const char* y = getenv("VS_K1_TL");
    if (y) tl_mode = atoi(y);
    const char* c = getenv("VS_K1_C0");
    if (c) c0 = (float)atof(c);
    const char* q = getenv("VS_K1_PF");
    if (q) pf = atoi(q);
    const char* e = getenv("VS_K1_VARIANT");
    variant = e ? atoi(e) : 3;
    const char* f = getenv("VS_K1_FLUSH");
    if (f) flush_min = atoi(f);
  }
  // variants: 0/1/3 register double-buffering (U, CTAs/SM) = (4,2) (2,4) (3,3);
  // 4/5 shared-memory ring (U, NS, CTAs/SM) = (4,3,3) (2,4,4)
  const int ctas_per_sm = variant == 0 ? 2 : ((variant == 3 || variant == 4) ? 3 : 4);
  const int Tw = sms * ctas_per_sm * WPC;
  // grid covers the worst case over the W the kernel will pick from the live R
  int grid;
  if (d_R) {
    static int cached_rows = -1, cached_grid = 0, cached_T = 0;
    if (rows != cached_rows || Tw != cached_T) {
      int g = 1;
      for (int r = 1; r <= rows; ++r) g = max(g, (r * pick_w(r, V, Tw, c0) + WPC - 1) / WPC);
      cached_rows = rows;
      cached_T = Tw;
      cached_grid = g;
    }
    grid = cached_grid;
  } else {
    grid = (rows * pick_w(rows, V, Tw, c0) + WPC - 1) / WPC;
  }
  const T* p = static_cast<const T*>(logits);
  // candidate mode: register top-list for Meff <= 32, 32-bit keys for bf16 rows with |V| < 65536
  const int TLm = ((M < V ? M : V) <= 32 && tl_mode) ? ((sizeof(T) == 2 && V < 65536 && tl_mode != 3) ? 2 : 1) : 0;
#define VS_K1_LAUNCH(U_, B_, TL_, NS_)                                                                  \
  do {                                                                                                   \
    auto kern = row_lse_topm_warp_kernel<T, U_, B_, TL_, NS_>;                                           \
    const size_t dsm = (size_t)WPC * NS_ * 32 * U_ * 16;                                                \
    if (dsm > 0) allow_dyn_smem((const void*)kern, dsm);                                                  \
    vs::vs_launch(kern, dim3(grid), dim3(WPC * 32), dsm, st, p, ld, V, M, R_host, d_R, top_tok, top_logp,    \
                  row_lse, fb, norm, sms, flush_min, pf, ctas_per_sm * WPC, c0);                         \
  } while (0)
#define VS_K1_LAUNCH3(U_, B_, NS_)  \
  if (TLm == 2)                     \
    VS_K1_LAUNCH(U_, B_, 2, NS_);   \
  else if (TLm == 1)                \
    VS_K1_LAUNCH(U_, B_, 1, NS_);   \
  else                              \
    VS_K1_LAUNCH(U_, B_, 0, NS_);
  switch (variant) {
    case 0: VS_K1_LAUNCH3(4, 2, 0); break;
    case 3: VS_K1_LAUNCH3(3, 3, 0); break;
    case 4: VS_K1_LAUNCH3(4, 3, 3); break;
    case 5: VS_K1_LAUNCH3(2, 4, 4); break;
    default: VS_K1_LAUNCH3(2, 4, 0); break;
  }
#undef VS_K1_LAUNCH3
#undef VS_K1_LAUNCH
  VS_CUDA_RET();
}

}  // namespace

// row_topm_tma.cu
bool tma_eligible(const void* logits, int64_t ld, int V, int M, int esize, bool pinned);
template <typename T>
int launch_tma(const void* logits, int64_t ld, int V, int M, int R_host, const int* d_R, int R_grid,
               int* top_tok, float* top_logp, float* row_lse, int* fb, int norm, void* ws, size_t ws_bytes,
               cudaStream_t st);
}  // namespace vs

namespace vs {
bool pdl_enabled() {
  static int e = -1;
  if (e < 0) {
    const char* v = getenv("VS_PDL");
    e = v ? atoi(v) : 1;
  }
  return e != 0;
}
}  // namespace vs

extern "C" int vs_version(void) { return 3; }

extern "C" int vs_row_lse_topm_ws(const void* logits, int32_t dtype, int64_t ld, int32_t V, int32_t M,
                                  int32_t R_host, const int32_t* d_R, int32_t R_grid, int32_t* top_tok,
                                  float* top_logp, float* row_lse, int32_t* fallback_count, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  if (!logits || !top_tok || !top_logp || V < 1 || M < 1 || M > VS_MAX_M || ld < V || R_grid < 0)
    return VS_ERR_CONFIG;
  if (R_grid == 0) return VS_OK;
  const int norm = (dtype & VS_ROWS_NORMALIZED) ? 1 : 0;
  const int pin = dtype & (VS_K1_SPLIT | VS_K1_WARP);
  const int dt = dtype & ~(VS_ROWS_NORMALIZED | VS_K1_SPLIT | VS_K1_WARP);
  dtype &= ~(VS_K1_SPLIT | VS_K1_WARP);
  const int es = dt == VS_DTYPE_F32 ? 4 : 2;
  if (workspace && (dt == VS_DTYPE_F32 || dt == VS_DTYPE_BF16) && !(pin & VS_K1_WARP) &&
      vs::tma_eligible(logits, ld, V, M, es, (pin & VS_K1_SPLIT) != 0)) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dt == VS_DTYPE_F32)
      return vs::launch_tma<float>(logits, ld, V, M, R_host, d_R, R_grid, top_tok, top_logp, row_lse,
                                   fallback_count, norm, workspace, workspace_bytes, st);
    return vs::launch_tma<__nv_bfloat16>(logits, ld, V, M, R_host, d_R, R_grid, top_tok, top_logp, row_lse,
                                         fallback_count, norm, workspace, workspace_bytes, st);
  }
  return vs_row_lse_topm(logits, dtype, ld, V, M, R_host, d_R, R_grid, top_tok, top_logp, row_lse,
                         fallback_count, stream);
}

extern "C" int vs_row_lse_topm(const void* logits, int32_t dtype, int64_t ld, int32_t V, int32_t M,
                               int32_t R_host, const int32_t* d_R, int32_t R_grid, int32_t* top_tok,
                               float* top_logp, float* row_lse, int32_t* fallback_count,
                               void* stream) {
  if (!logits || !top_tok || !top_logp || V < 1 || M < 1 || M > VS_MAX_M || ld < V || R_grid < 0)
    return VS_ERR_CONFIG;
  if (R_grid == 0) return VS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int norm = (dtype & VS_ROWS_NORMALIZED) ? 1 : 0;
  dtype &= ~VS_ROWS_NORMALIZED;
  if (dtype == VS_DTYPE_F32)
    return vs::launch<float>(logits, ld, V, M, R_host, d_R, R_grid, top_tok, top_logp, row_lse, fallback_count, norm, st);
  if (dtype == VS_DTYPE_BF16)
    return vs::launch<__nv_bfloat16>(logits, ld, V, M, R_host, d_R, R_grid, top_tok, top_logp, row_lse, fallback_count, norm, st);
  return VS_ERR_CONFIG;
}
