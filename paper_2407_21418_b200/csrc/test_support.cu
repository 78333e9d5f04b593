// test_support.cu — a TEST hook, not part of the hot path: a grid that holds
// SMs (one CTA per SM: maximal dynamic shared memory) until the host raises a
// flag, so tests can run the executor while another kernel occupies most of
// the GPU (tests/test_split_k_concurrency.py: split-K must not depend on all
// of a tile's splits being resident at once).
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"
#include "status.h"

namespace ftb {
namespace {

// ctl (mapped pinned host memory): [0] flag set by the host, [1] CTAs that
// arrived, [2] CTAs that gave up at the timeout
__global__ void occupy_kernel(volatile int32_t* ctl, long long timeout_ns) {
  extern __shared__ uint8_t smem[];
  if (threadIdx.x == 0) {
    smem[0] = 1;
    atomicAdd_system(const_cast<int32_t*>(ctl) + 1, 1);
    long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ctl[0] == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicAdd_system(const_cast<int32_t*>(ctl) + 2, 1);
        break;
      }
      __nanosleep(2000);
    }
  }
  __syncthreads();
}

}  // namespace
}  // namespace ftb

extern "C" ftb_status ftb_test_occupy_sms(int32_t n_ctas, int32_t* ctl_host, int64_t timeout_ns, void* stream) {
  return ftb::guarded([&] {
    if (n_ctas < 1 || !ctl_host) throw ftb::input_error("occupy: need n_ctas >= 1 and a control block");
    cudaError_t e = ftb::configure_smem_once<ftb::occupy_kernel>(232448);
    if (e == cudaSuccess) {
      ftb::occupy_kernel<<<n_ctas, 32, 232448, static_cast<cudaStream_t>(stream)>>>(ctl_host, timeout_ns);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) throw ftb::cuda_error(std::string("occupy: ") + cudaGetErrorString(e));
  });
}
