// K4 row-state reorder and encoder-state placement (sm_100a).
//
// No reference equivalent: the reference scorer is stateless and every
// Candidate carries its whole token tuple (bb/core.py:58,170), every slot its
// Encoding (bb/scheduler.py:48-54).  With an incremental decoder the per-row
// state (self-attention K/V, positions [0, l_t)) must follow the beam's
// parent pointers.  vs_beam_step plans the minimum set of copies (only extra
// children of a parent that stay active); this kernel executes them.  Each
// (src, dst, len) entry copies len*pos_bytes bytes of every plane with
// 16-byte vector loads/stores; destinations are never sources, so no staging.
#include "common.cuh"

namespace vs {
namespace {

// Persistent grid: CTAs stride over the (copy, plane) items of the device-side
// n_copy; each item is copied with 4 independent 16-byte loads in flight per
// thread before their stores (the row of one item is up to max_len·pos_bytes).
__global__ void __launch_bounds__(256) rows_copy_kernel(unsigned char* __restrict__ base,
                                                        int64_t plane_stride, int planes,
                                                        int64_t row_stride, int64_t pos_bytes,
                                                        const int32_t* __restrict__ copy_list,
                                                        const int32_t* __restrict__ n_copy) {
  VS_PDL_ENTRY();
  const int items = *n_copy * planes;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int c = it / planes, plane = it - c * planes;
    const int src = copy_list[3 * c], dst = copy_list[3 * c + 1], len = copy_list[3 * c + 2];
    const int64_t bytes = pos_bytes > 0 ? (int64_t)len * pos_bytes : -pos_bytes;  // < 0: fixed-size record
    const unsigned char* s = base + plane * plane_stride + (int64_t)src * row_stride;
    unsigned char* d = base + plane * plane_stride + (int64_t)dst * row_stride;
    if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | (uintptr_t)bytes) & 15) == 0) {
      const uint4* s4 = reinterpret_cast<const uint4*>(s);
      uint4* d4 = reinterpret_cast<uint4*>(d);
      const int64_t n4 = bytes >> 4;
      int64_t i = threadIdx.x;
      for (; i + 3 * 256 < n4; i += 4 * 256) {
        const uint4 v0 = s4[i], v1 = s4[i + 256], v2 = s4[i + 512], v3 = s4[i + 768];
        d4[i] = v0;
        d4[i + 256] = v1;
        d4[i + 512] = v2;
        d4[i + 768] = v3;
      }
      for (; i < n4; i += 256) d4[i] = s4[i];
    } else {
      for (int64_t i = threadIdx.x; i < bytes; i += blockDim.x) d[i] = s[i];
    }
  }
}

__global__ void __launch_bounds__(256) scatter_rows_kernel(unsigned char* __restrict__ dst,
                                                           int64_t dst_stride,
                                                           const unsigned char* __restrict__ src,
                                                           int64_t src_stride, int64_t bytes,
                                                           const int32_t* __restrict__ slots,
                                                           const int32_t* __restrict__ d_count) {
  VS_PDL_ENTRY();
  const int i = blockIdx.x;
  if (d_count && i >= *d_count) return;
  const unsigned char* s = src + (int64_t)i * src_stride;
  unsigned char* d = dst + (int64_t)slots[i] * dst_stride;
  if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | (uintptr_t)bytes) & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    for (int64_t j = threadIdx.x; j < (bytes >> 4); j += blockDim.x) d4[j] = s4[j];
  } else {
    for (int64_t j = threadIdx.x; j < bytes; j += blockDim.x) d[j] = s[j];
  }
}

}  // namespace
}  // namespace vs

extern "C" int vs_rows_copy(void* base, int64_t plane_stride_bytes, int32_t planes,
                            int64_t row_stride_bytes, int64_t pos_bytes, const int32_t* copy_list,
                            const int32_t* n_copy, int32_t max_copies, void* stream) {
  if (!base || !copy_list || !n_copy || planes < 1 || planes > 65535 || pos_bytes == 0)
    return VS_ERR_CONFIG;
  if (max_copies <= 0) return VS_OK;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const long need = (long)max_copies * planes;
  const int grid = (int)(need < (long)sms * 8 ? need : (long)sms * 8);
  vs::vs_launch(vs::rows_copy_kernel, dim3(grid), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<unsigned char*>(base), plane_stride_bytes, planes, row_stride_bytes, pos_bytes,
      copy_list, n_copy);
  VS_CUDA_RET();
}

extern "C" int vs_scatter_rows(void* dst, int64_t dst_stride_bytes, const void* src,
                               int64_t src_stride_bytes, int64_t bytes, const int32_t* slots,
                               const int32_t* d_count, int32_t count_max, void* stream) {
  if (!dst || !src || !slots || bytes < 0) return VS_ERR_CONFIG;
  if (count_max <= 0 || bytes == 0) return VS_OK;
  vs::vs_launch(vs::scatter_rows_kernel, dim3(count_max), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<unsigned char*>(dst), dst_stride_bytes, static_cast<const unsigned char*>(src),
      src_stride_bytes, bytes, slots, d_count);
  VS_CUDA_RET();
}
