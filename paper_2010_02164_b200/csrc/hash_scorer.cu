// Synthetic device scorer: deterministic logits for every scored row.
//
// Stands in for the decoder's vocab projection in the search benchmark. It
// mirrors the structure of the reference's SeededHashScorer
// (bb/model.py:177-218): logits are a pure function of (seed, source,
// candidate prefix, token) and the EOS logit is eos_bias * len / src_len,
// but the generator is a counter hash (splitmix64 / murmur3 fmix32) built
// from IEEE-exact operations only, so oracle/scorers.py:HashLogitsCPU
// reproduces every logit bit for bit on the CPU.
#include "common.cuh"

namespace vs {
namespace {

__global__ void hash_encode_kernel(vs_config cfg, vs_state st, uint64_t seed) {
  VS_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int nadm = st.status[VS_ST_NADMIT];
  if (i >= nadm) return;
  const int s = st.status[VS_ST_HDR + 3 * cfg.n + i];
  const int input = st.slot_input[s];
  uint64_t h = mix64(seed ^ 0x9E3779B97F4A7C15ull);
  for (int p = st.src_off[input]; p < st.src_off[input + 1]; ++p)
    h = mix64(h ^ ((uint64_t)st.src_tok[p] + 0x632BE59BD9B4E019ull));
  st.slot_seed[s] = h;
  st.c_hash[s * cfg.k] = prefix_init(h, cfg.sos);
}

__device__ __forceinline__ float hash_logit(uint32_t key, int v, float scale, int power) {
  const uint32_t bits = fmix32(((uint32_t)v * 0x9E3779B9u) ^ key);
  if (power == 0) {  // log-like: -scale * (e + f), u' = ((bits>>8)+1) * 2^-24 = 2^e (1+f)
    // e + f = (bits(u') - bits(1.0)) * 2^-23 exactly up to one rounding, and
    // bits(u') = bits(float(n)) - 24·2^23, so the logit is two conversions, an
    // add and two multiplies (bit-identical to the oracle's e/f formula: float
    // rounding commutes with the power-of-two scalings).
    const uint32_t n = (bits >> 8) + 1u;
    const int X = (int)(__float_as_uint((float)n) - 0x4B800000u);
    return __fmul_rn(__fmul_rn((float)X, 1.1920928955078125e-07f), -scale);
  }
  float u = __fmul_rn((float)(bits >> 8), 5.9604644775390625e-08f);  // * 2^-24, exact
  if (power >= 2) u = __fmul_rn(u, u);
  if (power >= 4) u = __fmul_rn(u, u);
  return __fmul_rn(u, scale);
}

__device__ __forceinline__ unsigned long long pk2f(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}

template <typename T>
__device__ __forceinline__ T cvt(float x);
template <>
__device__ __forceinline__ float cvt<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// Persistent grid-stride over (row, 2048-column chunk) work items with the
// live row count read from device memory; rows of freshly admitted beams
// (length 1) hash their source inline (the encode, fused: one launch per step).
// live row count read from device memory: no empty CTAs are launched for
// rows beyond R_t.  8 consecutive tokens per thread, one 16-byte store (bf16).
// Each thread writes HVPT 16-byte groups of 8 logits per (row, chunk) work item,
// so the per-item row lookups are amortised; the EOS value (a division) is only
// computed in the one group that holds EOS.
constexpr int HVPT = 2;
template <typename T>
__global__ void __launch_bounds__(256) hash_logits_kernel(vs_config cfg, vs_state st, vs_hash_params hp,
                                                          T* __restrict__ logits, int64_t ld, int cols) {
  VS_PDL_ENTRY();
  const int R = st.status[VS_ST_R];
  const int V = cfg.vocab_size;
  for (int w = blockIdx.x; w < R * cols; w += gridDim.x) {
    const int r = w / cols, cchunk = w - r * cols;
    const int s = st.row_slot[r];
    uint64_t h;
    if (st.row_len[r] == 1) {  // a beam admitted by this step's schedule: encode it inline
      const int input = st.slot_input[s];
      uint64_t sh = mix64(hp.seed ^ 0x9E3779B97F4A7C15ull);  // == hash_encode_kernel
      for (int p = st.src_off[input]; p < st.src_off[input + 1]; ++p)
        sh = mix64(sh ^ ((uint64_t)st.src_tok[p] + 0x632BE59BD9B4E019ull));
      h = prefix_init(sh, cfg.sos);
      if (cchunk == 0 && threadIdx.x == 0) {  // the beam step extends c_hash
        st.slot_seed[s] = sh;
        st.c_hash[s * cfg.k] = h;
      }
    } else {
      h = st.c_hash[s * cfg.k + st.row_cand[r]];
    }
    const uint32_t key = (uint32_t)(h ^ (h >> 32));
    T* out = logits + (int64_t)r * ld;
#pragma unroll
    for (int g = 0; g < HVPT; ++g) {
      const int v0 = ((cchunk * HVPT + g) * blockDim.x + threadIdx.x) * 8;
      if (v0 >= V) continue;
      T vals[8];
      if ((unsigned)(cfg.eos - v0) < 8u) {  // the one group holding EOS
        const float eos_val =
            __fdiv_rn(__fmul_rn(hp.eos_bias, (float)st.row_len[r]), (float)st.slot_src_len[s]);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int v = v0 + j;
          vals[j] = cvt<T>((v == cfg.eos) ? eos_val : hash_logit(key, v, hp.scale, hp.power));
        }
      } else if (hp.power == 0) {  // log-like, two elements per packed multiply (same roundings)
        float lg[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t bits = fmix32(((uint32_t)(v0 + j) * 0x9E3779B9u) ^ key);
          lg[j] = (float)(int)(__float_as_uint((float)((bits >> 8) + 1u)) - 0x4B800000u);
        }
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          unsigned long long t;
          asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk2f(lg[j], lg[j + 1])),
              "l"(pk2f(1.1920928955078125e-07f, 1.1920928955078125e-07f)));
          asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(t) : "l"(pk2f(-hp.scale, -hp.scale)));
          float a, b;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(t));
          vals[j] = cvt<T>(a);
          vals[j + 1] = cvt<T>(b);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) vals[j] = cvt<T>(hash_logit(key, v0 + j, hp.scale, hp.power));
      }
      const bool vec_ok = (v0 + 8 <= V) && ((reinterpret_cast<uintptr_t>(out + v0) & 15) == 0);
      if (vec_ok) {
        if (sizeof(T) == 2) {
          *reinterpret_cast<uint4*>(out + v0) = *reinterpret_cast<const uint4*>(vals);
        } else {
          reinterpret_cast<uint4*>(out + v0)[0] = reinterpret_cast<const uint4*>(vals)[0];
          reinterpret_cast<uint4*>(out + v0)[1] = reinterpret_cast<const uint4*>(vals)[1];
        }
      } else {
        for (int j = 0; j < 8 && v0 + j < V; ++j) out[v0 + j] = vals[j];
      }
    }
  }
}

}  // namespace
}  // namespace vs

extern "C" int vs_hash_encode(const vs_config* cfg, const vs_state* st, uint64_t seed, void* stream) {
  if (!cfg || !st) return VS_ERR_CONFIG;
  const int n = cfg->n;
  vs::vs_launch(vs::hash_encode_kernel, dim3((n + 127) / 128), dim3(128), 0, static_cast<cudaStream_t>(stream), *cfg, *st, seed);
  VS_CUDA_RET();
}

extern "C" int vs_hash_logits(const vs_config* cfg, const vs_state* st, const vs_hash_params* hp,
                              void* logits, int64_t ld, int32_t R_grid, void* stream) {
  if (!cfg || !st || !hp || !logits || ld < cfg->vocab_size) return VS_ERR_CONFIG;
  if (hp->power != 0 && hp->power != 1 && hp->power != 2 && hp->power != 4) return VS_ERR_CONFIG;
  if (R_grid <= 0) return VS_OK;
  const int cols = (cfg->vocab_size + 8 * 256 * vs::HVPT - 1) / (8 * 256 * vs::HVPT);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const long need = (long)R_grid * cols;
  const int grid = (int)(need < (long)sms * 8 ? need : (long)sms * 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (hp->dtype == VS_DTYPE_F32)
    vs::vs_launch(vs::hash_logits_kernel<float>, dim3(grid), dim3(256), 0, s, *cfg, *st, *hp, static_cast<float*>(logits), ld, cols);
  else if (hp->dtype == VS_DTYPE_BF16)
    vs::vs_launch(vs::hash_logits_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, s, *cfg, *st, *hp, static_cast<__nv_bfloat16*>(logits), ld, cols);
  else
    return VS_ERR_CONFIG;
  VS_CUDA_RET();
}
