// K3 compact_refill_select, standalone launch (sm_100a): one CTA of 1,024
// threads runs vs::schedule_block (csrc/schedule.cuh).  Used for the first
// schedule of a run and for flush-phase transitions; every other step runs the
// same routine in the last CTA of the fused beam-step kernel
// (vs_beam_step_schedule, csrc/beam_step.cu).
#include "schedule.cuh"

namespace vs {
namespace {

constexpr int NT3 = 1024;

__global__ void __launch_bounds__(NT3) schedule_kernel(vs_config cfg, vs_state st, int N, int first,
                                                       int do_remove, int admit_mode, int select_mode,
                                                       int32_t* mirror) {
  VS_PDL_ENTRY();
  extern __shared__ __align__(16) int sched_smem[];
  schedule_block<NT3>(cfg, st, N, first, do_remove, admit_mode, select_mode, mirror, sched_smem);
}

}  // namespace

// Device view of a host-mapped pinned buffer (nullptr stays nullptr).
int32_t* mapped_ptr(void* host) {
  if (!host) return nullptr;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, host, 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return static_cast<int32_t*>(d);
}

}  // namespace vs

extern "C" int vs_schedule(const vs_config* cfg, const vs_state* st, int32_t N, int32_t first_call,
                           int32_t do_remove, int32_t admit_mode, int32_t select_mode, void* stream) {
  return vs_schedule_mirror(cfg, st, N, first_call, do_remove, admit_mode, select_mode, nullptr, stream);
}

extern "C" int vs_schedule_mirror(const vs_config* cfg, const vs_state* st, int32_t N, int32_t first_call,
                                  int32_t do_remove, int32_t admit_mode, int32_t select_mode,
                                  int32_t* status_mirror, void* stream) {
  if (!cfg || !st || cfg->n < 1 || cfg->n > VS_MAX_SLOTS || cfg->k < 1 || cfg->k > VS_MAX_K ||
      N < 1 || cfg->capacity < cfg->k)
    return VS_ERR_CONFIG;
  int32_t* mirror = vs::mapped_ptr(status_mirror);
  if (status_mirror && !mirror) return VS_ERR_CONFIG;
  vs::vs_launch(vs::schedule_kernel, dim3(1), dim3(vs::NT3), vs::sched_smem_bytes(cfg->n),
                static_cast<cudaStream_t>(stream), *cfg, *st, N, first_call, do_remove, admit_mode,
                select_mode, mirror);
  VS_CUDA_RET();
}
