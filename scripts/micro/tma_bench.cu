// TMA ingest microbenchmark: per-SM bytes/clk for single-CTA TMA vs 2-CTA
// (cta_group::2) TMA, with a ring of S stages and a consumer that releases
// stages immediately (no MMA). Usage: ./tma_bench
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include "../../paper_2407_21418_b200/csrc/ptx.cuh"

using namespace ftb;

struct Maps { CUtensorMap a; CUtensorMap b; };

template <int MODE, int MASK = 0>  // 0 single-CTA, 1 cluster-2 with cta_group::2 TMA, 2 cluster-2 plain TMA
__global__ void __launch_bounds__(192, 1) tma_kernel(const __grid_constant__ Maps maps_p, int iters, int S,
                                                    int a_rows, int b_rows, unsigned long long* out, const Maps* gmaps, int ndesc, int big, int R_rows) {
  const Maps& maps0 = gmaps ? *gmaps : maps_p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = (a_rows + b_rows) * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + 16;
  uint32_t rank = 0;
  if (MODE != 0) rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MODE == 4 ? 2 : 1); }
    mbar_init(&empty[15], 1);
    fence_barrier_init();
  }
  if (MODE != 0) cluster_sync(); else __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    int ps = 0, ph = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&empty[ps], ph ^ 1);
      uint8_t* dst = smem + ps * stage_bytes;
      int k0 = (it % 64) * 64;
      const Maps& maps = (gmaps && ndesc > 1) ? gmaps[(it + blockIdx.x) % ndesc] : maps0;
      int row = big ? ((blockIdx.x * 64 + it / 64) * 256) % (R_rows - 512) : ((blockIdx.x * 7 + it / 64) % 16) * 256;
      if (MODE == 5) {
        mbar_arrive_expect_tx(&full[ps], (a_rows + b_rows) * 128);
        // a_rows = 256 rows of smem = 128 rows x 2 K blocks in one box
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                     :: "r"(smem_addr(dst)), "l"(reinterpret_cast<uint64_t>(&maps.a)), "r"(smem_addr(&full[ps])),
                        "r"(0), "r"(row), "r"((k0 / 64) % 32) : "memory");
        if (b_rows) tma_load_3d(dst + a_rows * 128, &maps.b, &full[ps], k0, row + 128, 0);
      } else if (MODE == 4) {
        // own lane box (a_rows) + half of a 2*b_rows col tile, multicast to both CTAs
        mbar_arrive_expect_tx(&full[ps], (a_rows + 2 * b_rows) * 128);
        tma_load_3d(dst, &maps.a, &full[ps], k0, row, 0);
        const uint32_t half_dst = smem_addr(dst + a_rows * 128 + rank * b_rows * 128);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
            " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(half_dst),
            "l"(reinterpret_cast<uint64_t>(&maps.b)), "r"(smem_addr(&full[ps])), "r"(k0), "r"(row + 128 + (int)rank * b_rows), "r"(0),
            "h"((uint16_t)0x3)
            : "memory");
      } else if (MODE == 1) {
        uint32_t fb = MASK ? (smem_addr(&full[ps]) & 0xFEFFFFFFu) : mapa_shared(smem_addr(&full[ps]), 0);
        if (rank == 0) mbar_arrive_expect_tx(&full[ps], 2 * stage_bytes);
        tma_load_3d_pair(dst, &maps.a, fb, k0, row, 0);
        if (b_rows) tma_load_3d_pair(dst + a_rows * 128, &maps.b, fb, k0, row + 128, 0);
      } else {
        mbar_arrive_expect_tx(&full[ps], stage_bytes);
        tma_load_3d(dst, &maps.a, &full[ps], k0, row, 0);
        if (b_rows) tma_load_3d(dst + a_rows * 128, &maps.b, &full[ps], k0, row + 128, 0);
      }
      if (++ps == S) { ps = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0 && (MODE != 1 || rank == 0)) {
    int cs = 0, ph = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&full[cs], ph);
      if (MODE == 4) {
        // both CTAs must have consumed stage cs before either re-fills it (multicast writes both)
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(smem_addr(&empty[cs]), 0)) : "memory");
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(smem_addr(&empty[cs]), 1)) : "memory");
      } else if (MODE == 1) {
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(smem_addr(&empty[cs]), 0)) : "memory");
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(smem_addr(&empty[cs]), 1)) : "memory");
      } else {
        mbar_arrive(&empty[cs]);
      }
      if (++cs == S) { cs = 0; ph ^= 1; }
    }
    mbar_arrive(&empty[15]);
  } else if (warp >= 2 && MODE != 1) {
    if (MODE == 0 && rank == 0 && blockDim.x > 64) mbar_wait(&empty[15], 0);
  }
  if (MODE != 0) cluster_sync(); else __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;

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
  const int64_t K = 4096, R = 65536;  // 512 MiB: BIG mode streams from HBM
  void* buf; cudaMalloc(&buf, K * R * 2); cudaMemset(buf, 0, K * R * 2);
  unsigned long long* out; cudaMalloc(&out, 148 * 8);
  int ctas = getenv("CTAS") ? atoi(getenv("CTAS")) : 148, iters = getenv("ITERS") ? atoi(getenv("ITERS")) : 2000;
  Maps* dmaps; cudaMalloc(&dmaps, 512 * sizeof(Maps));
  struct Cfg { int mode, a, b, S; const char* name; int gm = 0; int spin = 0; int big = 0; } cfgs[] = {
      {5, 256, 0, 6, "ONE 3-D box 128x2kb (32KB) S6"}, {0, 128, 128, 6, "TWO boxes 128+128 (32KB) S6"}, {0, 256, 0, 6, "ONE box 256 rows (32KB) S6"}, {5, 256, 256, 4, "3-D box 2kb + 256 box (64KB) S4"}, {1, 128, 128, 6, "BIG pair 128+128 S6", 0, 0, 1}, {2, 128, 128, 6, "BIG cluster2 plain 128+128 S6", 0, 0, 1}, {0, 128, 128, 6, "BIG single 128+128 S6", 0, 0, 1}, {0, 128, 256, 4, "single 128+256 S4 (same ingest)", 0}, {0, 128, 128, 6, "GMEM-desc single 128+128 S6", 1}, {0, 128, 128, 6, "GMEM 8 descs", 8}, {0, 128, 128, 6, "GMEM 64 descs", 64}, {0, 128, 128, 6, "GMEM 512 descs", 512}, {0, 128, 128, 6, "single + 4 spinning warps", 0, 1}, {0, 128, 256, 4, "single 128+256 + 4 spinning warps", 0, 1}, {1, 128, 128, 6, "GMEM-desc pair 128+128 S6", 1},
      {0, 128, 256, 4, "single 128+256 S4"}, {0, 128, 128, 6, "single 128+128 S6"}, {0, 128, 64, 8, "single 128+64 S8"},
      {0, 128, 0, 8, "single 128 only S8"}, {0, 256, 0, 6, "single 256 only S6"},
      {1, 128, 128, 6, "pair(cta_group::2) 128+128 S6"}, {1, 128, 64, 8, "pair 128+64 S8"}, {3, 128, 128, 6, "pair masked-bar 128+128 S6"},
      {2, 128, 128, 6, "cluster2 plain 128+128 S6"}, {2, 128, 256, 4, "cluster2 plain 128+256 S4"},
  };
  for (auto& c : cfgs) {
    Maps m;
    if (c.mode == 5) {  // 3-D view {64 (k inner), rows, K/64 (k outer)} with box {64, 128, 2}
      cuuint64_t dims[3] = {64, (cuuint64_t)R, (cuuint64_t)(K / 64)};
      cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
      cuuint32_t box[3] = {64, 128, 2}, es[3] = {1, 1, 1};
      CUresult r = enc()(&m.a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) printf("encode 3d-k failed %d\n", r);
    } else
    make(&m.a, buf, K, R, c.a > 0 ? (c.a > 256 ? 256 : c.a) : 64);
    make(&m.b, buf, K, R, c.b > 0 ? c.b : 64);
    for (int d = 0; d < 512; ++d) cudaMemcpy(dmaps + d, &m, sizeof(Maps), cudaMemcpyHostToDevice);
    int smem = c.S * (c.a + (c.mode == 4 ? 2 : 1) * c.b) * 128 + 2048;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(ctas); lc.blockDim = dim3(c.spin ? 192 : 64); lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = c.mode ? 2 : 1;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    cudaError_t e;
    auto launch = [&](int it) {
      if (c.mode == 0) { cudaFuncSetAttribute(tma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, tma_kernel<0>, m, it, c.S, c.a, c.b, out, c.gm ? dmaps : nullptr, c.gm, c.big, (int)R); }
      else if (c.mode == 3) { cudaFuncSetAttribute(tma_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, tma_kernel<1, 1>, m, it, c.S, c.a, c.b, out, c.gm ? dmaps : nullptr, c.gm, c.big, (int)R); }
      else if (c.mode == 5) { cudaFuncSetAttribute(tma_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, tma_kernel<5>, m, it, c.S, c.a, c.b, out, c.gm ? dmaps : nullptr, c.gm, c.big, (int)R); }
      else if (c.mode == 4) { cudaFuncSetAttribute(tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, tma_kernel<4>, m, it, c.S, c.a, c.b, out, c.gm ? dmaps : nullptr, c.gm, c.big, (int)R); }
      else if (c.mode == 1) { cudaFuncSetAttribute(tma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, tma_kernel<1>, m, it, c.S, c.a, c.b, out, c.gm ? dmaps : nullptr, c.gm, c.big, (int)R); }
      else { cudaFuncSetAttribute(tma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, tma_kernel<2>, m, it, c.S, c.a, c.b, out, c.gm ? dmaps : nullptr, c.gm, c.big, (int)R); }
    };
    launch(100); cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); launch(iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> cyc(ctas); cudaMemcpy(cyc.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
    double mc = 0; for (auto v : cyc) mc += v; mc /= ctas;
    double bytes_cta = (double)iters * (c.a + c.b) * 128;
    printf("%-34s err=%d  %.3f ms  per-SM %.1f B/clk  chip %.2f TB/s  (%.0f clk/iter)\n", c.name, (int)e, ms,
           bytes_cta / mc, bytes_cta * ctas / (ms * 1e-3) / 1e12, mc / iters);
  }
  return 0;
}
