// Power / data-movement probe for the Dense main loop (DESIGN.md round-2 plan
// item 2): single-CTA tcgen05.mma M=128 N=256 K=16 (4 per 64-wide K block),
// 4-stage TMA ring of 48 KiB, clusters of 2 CTAs in both modes.
//   MODE=0: each CTA loads its A box (128 rows) and the full B box (256 rows)
//   MODE=1: each CTA loads its A box and HALF of the B box (128 rows) with
//           .multicast::cluster to both CTAs; each full barrier expects 48 KiB;
//           the MMA commit arrives on both CTAs' empty barriers (count 2)
// Both CTAs of a cluster use the same B rows, so MODE=1 moves 1/3 fewer bytes
// from L2 for the same MMAs. Run each mode alone for ~2 s while sampling SM
// clocks (nvidia-smi) to compare sustained TF/s under the power cap.
//   MODE=2: one CTA computes a 256x256 tile (two 128-lane accumulators of 256
//           columns): A 256 rows + B 256 rows per 64-wide K block (64 KiB,
//           3 stages), 8 MMAs per K block: 1/3 fewer staged bytes per flop
//   MODE=3: CTA pair (tcgen05 cta_group::2, M=256 N=256 per pair): each CTA
//           stages its 128 A rows + half of B (32 KiB), the leader issues
// Usage: MODE=0|1|2|3 SECS=2 ./mcast_bench
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2407_21418_b200/csrc/ptx.cuh"
using namespace ftb;

struct Maps { CUtensorMap a; CUtensorMap bh; CUtensorMap bf; };  // A box 128 rows, B half 128 rows, B full 256 rows

__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(static_cast<uint16_t>(0x3))
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc1(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_addr(bar)),
               "h"(static_cast<uint16_t>(0x3))
               : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) mcast_kernel(const __grid_constant__ Maps maps, int iters, int R) {
  constexpr int S = MODE == 2 ? 3 : (MODE == 3 ? 6 : 4), kA = (MODE == 2 ? 256 : 128) * 128,
                kB = (MODE == 3 ? 128 : 256) * 128, kStage = kA + kB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kStage);
  uint64_t* empty = full + 8;
  uint64_t* done = full + 16;
  uint32_t* holder = reinterpret_cast<uint32_t*>(full + 24);
  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MODE == 1 ? 2 : 1); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    if (MODE == 3) tmem_alloc_pair<512>(holder);
    else tmem_alloc<512>(holder);
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *holder;
  const int cluster = blockIdx.x >> 1;
  if (warp == 0 && lane == 0) {
    int ps = 0, ph = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&empty[ps], ph ^ 1);
      uint8_t* dst = smem + ps * kStage;
      const int k0 = (it % 64) * 64;
      // L2-resident working set (like a large GEMM's reused tiles): 16 A tiles
      // (1 MiB each over K = 4096) and 8 B tiles (2 MiB each), 32 MiB in all
      const int arow = ((cluster * 2 + rank) % 16) * 128;
      const int brow = 4096 + (cluster % 8) * 256;
      if (MODE == 3) {  // both CTAs' loads signal the leader's full barrier
        const uint32_t fb = smem_addr(&full[ps]) & 0xFEFFFFFFu;
        if (rank == 0) mbar_arrive_expect_tx(&full[ps], 2 * kStage);
        tma_load_3d_pair(dst, &maps.a, fb, k0, arow, 0);
        tma_load_3d_pair(dst + kA, &maps.bh, fb, k0, brow + rank * 128, 0);
        if (++ps == S) { ps = 0; ph ^= 1; }
        continue;
      }
      mbar_arrive_expect_tx(&full[ps], kStage);
      tma_load_3d(dst, &maps.a, &full[ps], k0, arow, 0);
      if (MODE == 2) {
        tma_load_3d(dst + 128 * 128, &maps.a, &full[ps], k0, arow + 2048, 0);
        tma_load_3d(dst + kA, &maps.bf, &full[ps], k0, brow, 0);
      } else if (MODE == 0) {
        tma_load_3d(dst + kA, &maps.bf, &full[ps], k0, brow, 0);
      } else {
        tma_load_3d_mc(dst + kA + rank * (kB / 2), &maps.bh, &full[ps], k0, brow + rank * 128, 0);
      }
      if (++ps == S) { ps = 0; ph ^= 1; }
    }
  } else if (warp == 2 && lane == 0 && MODE == 3) {
    if (rank == 0) {  // the leader issues the pair MMAs
      int cs = 0, ph = 0;
      const uint32_t idesc = idesc_bf16_f32(256, 256, 0, 0);
      for (int it = 0; it < iters; ++it) {
        mbar_wait(&full[cs], ph);
        tc_fence_after();
        const uint32_t la = smem_addr(smem + cs * kStage), ca = la + kA;
        for (int kk = 0; kk < 4; ++kk)
          tc_mma_f16_pair(tmem, umma_desc_sw128(la + kk * 32, 16, 1024), umma_desc_sw128(ca + kk * 32, 16, 1024), idesc,
                          (it | kk) != 0);
        tc_commit_pair_mc(&empty[cs]);
        if (++cs == S) { cs = 0; ph ^= 1; }
      }
      tc_commit_pair_mc(done);
    }
    mbar_wait(done, 0);
  } else if (warp == 2 && lane == 0) {
    int cs = 0, ph = 0;
    const uint32_t idesc = idesc_bf16_f32(128, 256, 0, 0);
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&full[cs], ph);
      tc_fence_after();
      const uint32_t la = smem_addr(smem + cs * kStage), ca = la + kA;
      for (int kk = 0; kk < 4; ++kk) {
        tc_mma_f16(tmem, umma_desc_sw128(la + kk * 32, 16, 1024), umma_desc_sw128(ca + kk * 32, 16, 1024), idesc,
                   (it | kk) != 0);
        if (MODE == 2)  // second 128-lane half of the 256-row A tile into the second accumulator
          tc_mma_f16(tmem + 256, umma_desc_sw128(la + 16384 + kk * 32, 16, 1024),
                     umma_desc_sw128(ca + kk * 32, 16, 1024), idesc, (it | kk) != 0);
      }
      if (MODE == 1) tc_commit_mc1(&empty[cs]); else tc_commit(&empty[cs]);
      if (++cs == S) { cs = 0; ph ^= 1; }
    }
    tc_commit(done);
    mbar_wait(done, 0);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    if (MODE == 3) tmem_dealloc_pair<512>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

// pseudo-random bf16 in [-0.5, 0.5): tensor-core power is data dependent
// (all-zero operands run at full clock with no power cap)
__global__ void fill(uint16_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = static_cast<uint32_t>(i) * 2654435761u;
    h ^= h >> 13;
    const float f = static_cast<float>(h % 1000u) / 1000.f - 0.5f;
    p[i] = static_cast<uint16_t>(__float_as_uint(f) >> 16);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static void make(CUtensorMap* m, void* base, int64_t inner, int64_t rows, uint32_t box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)inner * 2, (cuuint64_t)(inner * rows * 2)};
  cuuint32_t box[3] = {64, box_rows, 1}, es[3] = {1, 1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d\n", r);
}

int main() {
  const int mode = getenv("MODE") ? atoi(getenv("MODE")) : 0;
  const double secs = getenv("SECS") ? atof(getenv("SECS")) : 2.0;
  const int64_t K = 4096, R = 8192;  // 64 MiB operand pool; the kernel touches 32 MiB of it
  void* buf; cudaMalloc(&buf, K * R * 2);
  if (getenv("ZEROS")) cudaMemset(buf, 0, K * R * 2);
  else fill<<<1024, 256>>>(static_cast<uint16_t*>(buf), K * R);
  Maps m;
  make(&m.a, buf, K, R, 128);
  make(&m.bh, buf, K, R, 128);
  make(&m.bf, buf, K, R, 256);
  const int ctas = 148, iters = 4096;  // 64 tiles of K=4096 per CTA per launch
  const int smem = (mode == 2 ? 3 * (256 + 256) : (mode == 3 ? 6 * (128 + 128) : 4 * (128 + 256))) * 128 + 2048;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(ctas); lc.blockDim = dim3(128); lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  lc.attrs = at; lc.numAttrs = 1;
  auto kern = mode == 3 ? mcast_kernel<3> : (mode == 2 ? mcast_kernel<2> : (mode ? mcast_kernel<1> : mcast_kernel<0>));
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, m, 64, (int)R);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int launches = 0;
  float total_ms = 0;
  while (total_ms < secs * 1e3) {
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) e = cudaLaunchKernelEx(&lc, kern, m, iters, (int)R);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    total_ms += ms; launches += 10;
  }
  const double flops = (mode == 2 ? 2.0 : 1.0) * 2.0 * 128 * 256 * 64 * (double)iters * ctas * launches;
  printf("MODE=%d err=%d: %d launches in %.0f ms: %.0f TF/s (%.1f us/launch)\n", mode, (int)e, launches, total_ms,
         flops / (total_ms * 1e-3) / 1e12, total_ms * 1e3 / launches);
  return 0;
}
