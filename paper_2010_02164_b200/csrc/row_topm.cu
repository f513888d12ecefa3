// K1 row_lse_topM: fused log-softmax + per-row top-M (sm_100a).
//
// Replaces bb/model.py:216-217 (log-softmax of one |V| row) and
// bb/search.py:63-73 (_candidate_pool: first M of sorted(range(V),
// key=(-row[t], t))), for every scored row of a timestep at once.
//
// One CTA per row.  The row is streamed from HBM exactly once with 16-byte
// non-allocating vector loads (4 in flight per thread).  While streaming,
// each thread keeps
//   * an online (max, sum exp) pair                  -> lse
//   * a sorted register list of its TL best logits   -> candidate superset
// After a block-wide lse reduction every kept entry is re-keyed by the exact
// contract value logp = fp32(x - lse) with token-ascending ties (a 64-bit
// key), lists are merged by warp-shuffle argmax rounds (partial-sort merge)
// and the block's top-M is verified: if any thread's TL-th kept entry could
// still reach the M-th logp (ties/ambiguity), the row falls back to an exact
// block radix select over 64-bit keys (re-reading the row).  Decisions never
// depend on atomic ordering, so the result is a pure function of the row.
#include "common.cuh"

namespace vs {
namespace {

template <int TL>
__device__ __forceinline__ void list_insert(float (&lv)[TL], int (&lt)[TL], float x, int tok) {
  float cv = x;
  int ct = tok;
#pragma unroll
  for (int q = 0; q < TL; ++q) {
    if (cv > lv[q]) {  // strict: equal logits keep the earlier (lower) token first
      float tv = lv[q];
      int tt = lt[q];
      lv[q] = cv;
      lt[q] = ct;
      cv = tv;
      ct = tt;
    }
  }
}

struct Online {
  float m, s;
};

template <int TL, int N>
__device__ __forceinline__ void consume(Online& o, float (&lv)[TL], int (&lt)[TL], const float (&x)[N],
                                        int tok0) {
  float cm = x[0];
#pragma unroll
  for (int j = 1; j < N; ++j) cm = fmaxf(cm, x[j]);
  if (cm > o.m) {
    o.s = (o.m == -INFINITY) ? 0.0f : o.s * exp2f((o.m - cm) * VS_LOG2E);
    o.m = cm;
  }
  if (o.m != -INFINITY) {
    const float ml = o.m * VS_LOG2E;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      float e;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fmaf(x[j], VS_LOG2E, -ml)));
      o.s += e;
    }
  }
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (x[j] > lv[TL - 1]) list_insert<TL>(lv, lt, x[j], tok0 + j);
}

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

// Exact top-M by 64-bit key via MSB-first radix select (8 x 8-bit passes).
// Rare path: only rows whose fast-path superset could not be proven.
template <typename T, int NT>
__device__ void exact_select(const T* __restrict__ row, int V, float lse, int Meff,
                             uint64_t* __restrict__ out_keys, uint64_t* __restrict__ scratch,
                             unsigned* __restrict__ hist) {
  __shared__ uint64_t s_prefix;
  __shared__ int s_want;
  __shared__ unsigned s_cnt;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_prefix = 0;
    s_want = Meff;
    s_cnt = 0;
  }
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = tid; i < 256; i += NT) hist[i] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    const uint64_t hi_mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
    for (int i = tid; i < V; i += NT) {
      const uint64_t key = row_key(__fsub_rn(to_f32<T>(row[i]), lse), i);
      if ((key & hi_mask) == (prefix & hi_mask)) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int want = s_want;
      unsigned cum = 0;
      for (int d = 255; d >= 0; --d) {
        const unsigned c = hist[d];
        if (cum + c >= (unsigned)want) {
          s_want = want - (int)cum;
          s_prefix = prefix | ((uint64_t)d << shift);
          break;
        }
        cum += c;
      }
    }
    __syncthreads();
  }
  const uint64_t kth = s_prefix;
  for (int i = tid; i < V; i += NT) {
    const uint64_t key = row_key(__fsub_rn(to_f32<T>(row[i]), lse), i);
    if (key >= kth) {
      const unsigned idx = atomicAdd(&s_cnt, 1u);
      if (idx < (unsigned)VS_MAX_M) scratch[idx] = key;
    }
  }
  __syncthreads();
  for (int j = tid; j < Meff; j += NT) {  // keys are unique -> ranks are a permutation
    const uint64_t kj = scratch[j];
    int rank = 0;
    for (int i = 0; i < Meff; ++i) rank += scratch[i] > kj;
    out_keys[rank] = kj;
  }
  __syncthreads();
}

template <typename T, int NT, int TL>
__global__ void __launch_bounds__(NT) row_lse_topm_kernel(
    const T* __restrict__ logits, int64_t ld, int V, int M, int R_host, const int* __restrict__ d_R,
    int* __restrict__ top_tok, float* __restrict__ top_logp, float* __restrict__ row_lse,
    int* __restrict__ fb_count, int normalized) {
  constexpr int NW = NT / 32;
  constexpr int VEC = 16 / sizeof(T);
  constexpr int U = 4;
  __shared__ float red_m[NW], red_s[NW];
  __shared__ uint64_t wkeys[NW][VS_MAX_M];
  __shared__ uint64_t fkeys[VS_MAX_M];
  __shared__ unsigned hist[256];
  __shared__ float s_lse;

  const int R = d_R ? *d_R : R_host;
  const int r = blockIdx.x;
  if (r >= R) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int Meff = M < V ? M : V;
  const T* __restrict__ row = logits + (int64_t)r * ld;

  Online o{-INFINITY, 0.0f};
  float lv[TL];
  int lt[TL];
#pragma unroll
  for (int q = 0; q < TL; ++q) {
    lv[q] = -INFINITY;
    lt[q] = 0x7fffffff;
  }

  // ---- single streaming pass over the row ---------------------------------
  int done = 0;
  if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
    const int nvec = V / VEC;
    const uint4* __restrict__ vrow = reinterpret_cast<const uint4*>(row);
    for (int b = tid; b < nvec; b += NT * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = b + u * NT;
        if (i < nvec) v[u] = ldg_stream(vrow + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = b + u * NT;
        if (i < nvec) {
          float x[VEC];
          unpack<T>(v[u], x);
          consume<TL, VEC>(o, lv, lt, x, i * VEC);
        }
      }
    }
    done = nvec * VEC;
  }
  for (int i = done + tid; i < V; i += NT) {  // tail (or unaligned row)
    float x[1] = {to_f32<T>(row[i])};
    consume<TL, 1>(o, lv, lt, x, i);
  }

  // ---- lse = max + log(sum exp(x - max)) ---------------------------------------
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, o.m, m);
    const float s2 = __shfl_xor_sync(0xffffffffu, o.s, m);
    lse_merge(o.m, o.s, m2, s2);
  }
  if (lane == 0) {
    red_m[wid] = o.m;
    red_s[wid] = o.s;
  }
  __syncthreads();
  if (wid == 0) {
    float mm = lane < NW ? red_m[lane] : -INFINITY;
    float ss = lane < NW ? red_s[lane] : 0.0f;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, mm, m);
      const float s2 = __shfl_xor_sync(0xffffffffu, ss, m);
      lse_merge(mm, ss, m2, s2);
    }
    if (lane == 0) s_lse = (mm == -INFINITY) ? -INFINITY : mm + logf(ss);
  }
  __syncthreads();
  const float lse = normalized ? 0.0f : s_lse;

  // ---- exact keys, per-thread sort ---------------------------------------------
  uint64_t key[TL];
#pragma unroll
  for (int q = 0; q < TL; ++q) key[q] = (lt[q] == 0x7fffffff) ? 0ull : row_key(__fsub_rn(lv[q], lse), lt[q]);
#pragma unroll
  for (int i = 0; i < TL; ++i)
#pragma unroll
    for (int j = 0; j < TL - 1 - i; ++j)
      if (key[j] < key[j + 1]) {
        const uint64_t t = key[j];
        key[j] = key[j + 1];
        key[j + 1] = t;
      }

  // ---- warp merge: Meff argmax rounds over lane heads -------------------------
  for (int j = 0; j < Meff; ++j) {
    const uint64_t best = warp_max_u64(key[0]);
    if (best != 0ull && key[0] == best) {
#pragma unroll
      for (int q = 0; q < TL - 1; ++q) key[q] = key[q + 1];
      key[TL - 1] = 0ull;
    }
    if (lane == 0) wkeys[wid][j] = best;
  }
  __syncthreads();
  // ---- block merge of NW sorted warp lists (warp 0) ---------------------------
  if (wid == 0) {
    int pos = 0;
    uint64_t head = lane < NW ? wkeys[lane][0] : 0ull;
    for (int j = 0; j < Meff; ++j) {
      const uint64_t best = warp_max_u64(head);
      if (best != 0ull && head == best) {
        ++pos;
        head = pos < Meff ? wkeys[lane][pos] : 0ull;
      }
      if (lane == 0) fkeys[j] = best;
    }
  }
  __syncthreads();

  // ---- verification: can a rejected entry reach the M-th logp? ----------------
  const uint64_t kth = fkeys[Meff - 1];
  int fail = (kth == 0ull);
  if (!fail) fail = ord_f32(__fsub_rn(lv[TL - 1], lse)) >= (uint32_t)(kth >> 32);
  if (__syncthreads_or(fail)) {
    exact_select<T, NT>(row, V, lse, Meff, fkeys, &wkeys[0][0], hist);
    if (tid == 0 && fb_count) atomicAdd(fb_count, 1);
  }

  for (int j = tid; j < M; j += NT) {
    if (j < Meff) {
      const uint64_t kk = fkeys[j];
      top_tok[(int64_t)r * M + j] = key_tok(kk);
      top_logp[(int64_t)r * M + j] = key_logp(kk);
    } else {
      top_tok[(int64_t)r * M + j] = -1;
      top_logp[(int64_t)r * M + j] = -INFINITY;
    }
  }
  if (tid == 0 && row_lse) row_lse[r] = lse;
}

template <typename T, int NT>
int launch_tl(const void* logits, int64_t ld, int V, int M, int R_host, const int* d_R, int grid,
              int* top_tok, float* top_logp, float* row_lse, int* fb, int norm, cudaStream_t st) {
  const T* p = static_cast<const T*>(logits);
  const int TLsel = M <= 4 ? M : (M <= 16 ? 4 : 8);
  switch (TLsel) {
    case 1: row_lse_topm_kernel<T, NT, 1><<<grid, NT, 0, st>>>(p, ld, V, M, R_host, d_R, top_tok, top_logp, row_lse, fb, norm); break;
    case 2: row_lse_topm_kernel<T, NT, 2><<<grid, NT, 0, st>>>(p, ld, V, M, R_host, d_R, top_tok, top_logp, row_lse, fb, norm); break;
    case 3: row_lse_topm_kernel<T, NT, 3><<<grid, NT, 0, st>>>(p, ld, V, M, R_host, d_R, top_tok, top_logp, row_lse, fb, norm); break;
    case 4: row_lse_topm_kernel<T, NT, 4><<<grid, NT, 0, st>>>(p, ld, V, M, R_host, d_R, top_tok, top_logp, row_lse, fb, norm); break;
    default: row_lse_topm_kernel<T, NT, 8><<<grid, NT, 0, st>>>(p, ld, V, M, R_host, d_R, top_tok, top_logp, row_lse, fb, norm); break;
  }
  VS_CUDA_RET();
}

template <typename T>
int launch_nt(const void* logits, int64_t ld, int V, int M, int R_host, const int* d_R, int grid,
              int* top_tok, float* top_logp, float* row_lse, int* fb, int norm, cudaStream_t st) {
  if (V >= 8192) return launch_tl<T, 256>(logits, ld, V, M, R_host, d_R, grid, top_tok, top_logp, row_lse, fb, norm, st);
  return launch_tl<T, 128>(logits, ld, V, M, R_host, d_R, grid, top_tok, top_logp, row_lse, fb, norm, st);
}

}  // namespace
}  // namespace vs

extern "C" int vs_version(void) { return 1; }

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
    return vs::launch_nt<float>(logits, ld, V, M, R_host, d_R, R_grid, top_tok, top_logp, row_lse, fallback_count, norm, st);
  if (dtype == VS_DTYPE_BF16)
    return vs::launch_nt<__nv_bfloat16>(logits, ld, V, M, R_host, d_R, R_grid, top_tok, top_logp, row_lse, fallback_count, norm, st);
  return VS_ERR_CONFIG;
}
