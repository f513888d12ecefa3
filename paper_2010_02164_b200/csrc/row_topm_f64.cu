// K1-f64: per-row top-M over already-normalised fp64 log-prob rows.
//
// The reference Scorer protocol returns fp64 log-prob rows (bb/model.py:216-217
// computes them in numpy fp64) and the search adds them to the parent score in
// fp64 (bb/search.py:71, bb/core.py:173).  Rounding those rows to fp32 before
// the row kernel changes the emitted scores and can merge distinct values into
// ties, so reference scorers driven through HostScorerAdapter get this exact
// path instead: the top-M tokens by (row value desc, token asc)
// (bb/search.py:69) with the fp64 values themselves handed to the beam step
// (vs_state.top_logp64).
//
// This is the parity path for host scorers (rows arrive over PCIe from Python),
// not a throughput path: one warp per row runs M rounds of a warp arg-max over
// 64-bit order keys, each round restricted to keys strictly below the previous
// winner.  The row stays in L1/L2 across rounds.
#include "common.cuh"

namespace {

// (value desc, token asc) as one comparable pair; larger = ranked first.
struct Key {
  uint64_t v;  // ord_f64(value)
  uint32_t t;  // 0xffffffff - token
};
__device__ __forceinline__ bool key_gt(Key a, Key b) { return a.v > b.v || (a.v == b.v && a.t > b.t); }

__device__ __forceinline__ double unord_f64(uint64_t u) {
  return __longlong_as_double((long long)((u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u));
}

__global__ void __launch_bounds__(256) row_topm_f64_kernel(const double* __restrict__ rows, int64_t ld, int V, int M,
                                                          int R_host, const int* __restrict__ d_R,
                                                          int* __restrict__ top_tok, float* __restrict__ top_logp,
                                                          double* __restrict__ top_logp64) {
  VS_PDL_ENTRY();
  const int R = d_R ? *d_R : R_host;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += warps) {
    const double* row = rows + (int64_t)r * ld;
    Key prev{~0ull, ~0u};  // above every key
    bool have_prev = false;
    for (int j = 0; j < M; ++j) {
      Key best{0ull, 0u};
      bool found = false;
      for (int t = lane; t < V; t += 32) {
        const double x = row[t];
        if (x != x) continue;  // NaN never ranks
        const Key c{vs::ord_f64(x), 0xffffffffu - (uint32_t)t};
        if (have_prev && !key_gt(prev, c)) continue;
        if (!found || key_gt(c, best)) best = c, found = true;
      }
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) {
        const uint64_t ov = vs::shfl_xor_u64(best.v, m);
        const uint32_t ot = __shfl_xor_sync(0xffffffffu, best.t, m);
        const int of = __shfl_xor_sync(0xffffffffu, (int)found, m);
        const Key o{ov, ot};
        if (of && (!found || key_gt(o, best))) best = o, found = true;
      }
      const int64_t o = (int64_t)r * M + j;
      if (lane == 0) {
        if (found) {
          const double lp = unord_f64(best.v);
          top_tok[o] = (int)(0xffffffffu - best.t);
          top_logp64[o] = lp;
          if (top_logp) top_logp[o] = (float)lp;
        } else {  // V < M (or NaN rows): pad like the fp32 kernels
          top_tok[o] = -1;
          top_logp64[o] = -INFINITY;
          if (top_logp) top_logp[o] = -INFINITY;
        }
      }
      prev = best;
      have_prev = true;
      if (!found) prev = Key{0ull, 0u};
    }
  }
}

}  // namespace

extern "C" int vs_row_topm_f64(const double* rows, int64_t ld, int32_t V, int32_t M, int32_t R_host,
                               const int32_t* d_R, int32_t R_grid, int32_t* top_tok, float* top_logp,
                               double* top_logp64, void* stream) {
  if (!rows || !top_tok || !top_logp64 || V < 1 || M < 1 || M > VS_MAX_M || ld < V || R_grid < 0 || R_host < 0)
    return VS_ERR_CONFIG;
  if (!d_R && R_host > R_grid) return VS_ERR_CONFIG;
  if (R_grid == 0) return VS_OK;
  const int wpc = 8;
  const int grid = (R_grid + wpc - 1) / wpc;
  cudaError_t e = vs::vs_launch(row_topm_f64_kernel, dim3(grid), dim3(32 * wpc), 0, (cudaStream_t)stream, rows, ld,
                                (int)V, (int)M, (int)R_host, d_R, top_tok, top_logp, top_logp64);
  return e == cudaSuccess ? VS_OK : VS_ERR_CUDA;
}
