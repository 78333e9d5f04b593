// Per-launch floor of a PDL chain on B200: what does a launch cost when the
// kernel does (almost) nothing, as a function of grid size, dynamic smem,
// TMEM allocation and griddepcontrol? 20 launches captured in a CUDA graph
// (as bench.py's per-shape timing runs the executor), time / 20.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_floor launch_floor.cu && ./launch_floor
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int kMode>
__global__ void __launch_bounds__(192, 1) k(int* out) {
  extern __shared__ uint8_t smem[];
  uint32_t& holder = *reinterpret_cast<uint32_t*>(smem);  // >= 16 B of dynamic smem
  if (kMode & 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (kMode & 4) {
    if ((threadIdx.x >> 5) == 2) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(&holder))) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    __syncthreads();
  }
  if (kMode & 2) asm volatile("griddepcontrol.wait;" ::: "memory");
  if ((kMode & 8) && threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(blockIdx.x);
  if (kMode & 4) {
    __syncthreads();
    if ((threadIdx.x >> 5) == 2)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder) : "memory");
  }
}

template <int kMode>
float run(int grid, int smem, bool pdl, bool graph, int* out) {
  cudaFuncSetAttribute(k<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  auto launch = [&] {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(192);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&lc, k<kMode>, out);
  };
  const int n = 20;
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < n; ++i) launch();
    e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess || !g) { printf("capture failed: %s\n", cudaGetErrorString(e)); return -1.f; }
    e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) { printf("instantiate failed: %s\n", cudaGetErrorString(e)); return -1.f; }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, s);
    if (graph) cudaGraphLaunch(ge, s);
    else for (int i = 0; i < n; ++i) launch();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best = ms < best ? ms : best;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return best * 1e3f / n;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int* out;
  cudaMalloc(&out, 4096 * sizeof(int));
  const char* names[16] = {"empty", "+trigger", "+wait", "+trigger+wait", "+tmem", "+tmem+trigger", "+tmem+wait",
                           "+tmem+trigger+wait", "+store", "+store+trigger", "+store+wait", "+store+trigger+wait",
                           "+store+tmem", "", "", "+store+tmem+trigger+wait"};
  for (int grid : {1, 24, 96, 148}) {
    for (int smem : {16, 200 * 1024}) {
      for (int graph : {0, 1}) {
        printf("grid %3d smem %6d %s:", grid, smem, graph ? "graph" : "eager");
        printf(" %s %.2f |", names[0], run<0>(grid, smem, true, graph, out));
        printf(" %s %.2f |", names[3], run<3>(grid, smem, true, graph, out));
        printf(" %s %.2f |", names[11], run<11>(grid, smem, true, graph, out));
        printf(" %s %.2f |", names[15], run<15>(grid, smem, true, graph, out));
        printf(" nopdl %s %.2f\n", names[15], run<15>(grid, smem, false, graph, out));
      }
    }
  }
  return 0;
}
