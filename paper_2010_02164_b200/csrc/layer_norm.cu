// Row LayerNorm (no affine) for the decoder scorers' bf16 activations (sm_100a).
//
// The batched decoder step (decoder.GraphedTransformerScorer, §8(f) row 1) runs
// 3 LayerNorms per layer on [R, d] bf16 rows; PyTorch's kernel took 12% of the
// WMT decoder step (profiles/round1/dec_launches_summary.txt: 5.5 us for a
// 2.9 MB row block).  One warp per row: the row is held in registers (d/32
// elements per lane, 16-byte loads), mean and variance are two fp32 passes over
// the registers (xor-tree warp sums), y = (x - mean) * rsqrt(var + eps) rounded
// to bf16 — the same math as F.layer_norm on bf16 input.
#include "common.cuh"

namespace {

template <int VPL>  // 16-byte vectors per lane (d = VPL * 256)
__global__ void __launch_bounds__(256) layer_norm_bf16_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                              __nv_bfloat16* __restrict__ y, int64_t ldy, int R,
                                                              float eps) {
  VS_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= R) return;
  constexpr int D = VPL * 256;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)r * ldx);
  float v[VPL][8];
  float s = 0.0f;
#pragma unroll
  for (int q = 0; q < VPL; ++q) {
    const uint4 w = xr[q * 32 + lane];
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[q][2 * j] = vs::bf16lo(u[j]);
      v[q][2 * j + 1] = vs::bf16hi(u[j]);
      s += v[q][2 * j] + v[q][2 * j + 1];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s * (1.0f / D);
  float ss = 0.0f;
#pragma unroll
  for (int q = 0; q < VPL; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float d = v[q][j] - mean;
      ss += d * d;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float rstd = rsqrtf(ss * (1.0f / D) + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + (int64_t)r * ldy);
#pragma unroll
  for (int q = 0; q < VPL; ++q) {
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 p = __floats2bfloat162_rn((v[q][2 * j] - mean) * rstd, (v[q][2 * j + 1] - mean) * rstd);
      o[j] = *reinterpret_cast<const uint32_t*>(&p);
    }
    yr[q * 32 + lane] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace

extern "C" int vs_layer_norm_bf16(const void* x, int64_t ldx, void* y, int64_t ldy, int32_t R, int32_t d, float eps,
                                  void* stream) {
  if (!x || !y || R < 0 || d < 256 || d % 256 || d > 4096 || ldx < d || ldy < d || (ldx % 8) || (ldy % 8) ||
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15))
    return VS_ERR_CONFIG;
  if (R == 0) return VS_OK;
  const dim3 grid((R + 7) / 8), block(256);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const auto* xp = static_cast<const __nv_bfloat16*>(x);
  auto* yp = static_cast<__nv_bfloat16*>(y);
  switch (d / 256) {
    case 1: vs::vs_launch(layer_norm_bf16_kernel<1>, grid, block, 0, st, xp, ldx, yp, ldy, (int)R, eps); break;
    case 2: vs::vs_launch(layer_norm_bf16_kernel<2>, grid, block, 0, st, xp, ldx, yp, ldy, (int)R, eps); break;
    case 4: vs::vs_launch(layer_norm_bf16_kernel<4>, grid, block, 0, st, xp, ldx, yp, ldy, (int)R, eps); break;
    case 8: vs::vs_launch(layer_norm_bf16_kernel<8>, grid, block, 0, st, xp, ldx, yp, ldy, (int)R, eps); break;
    case 16: vs::vs_launch(layer_norm_bf16_kernel<16>, grid, block, 0, st, xp, ldx, yp, ldy, (int)R, eps); break;
    default: return VS_ERR_CONFIG;
  }
  VS_CUDA_RET();
}
