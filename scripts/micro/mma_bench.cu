// Main-loop microbenchmark: TMA ring + tcgen05.mma consumer (no epilogue).
// Measures clk per K block (64) for single-CTA M=128 x N and 2-CTA M=256 x N.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>
#include <cstdint>
#include <vector>
#include "../../paper_2407_21418_b200/csrc/ptx.cuh"
using namespace ftb;
struct Maps { CUtensorMap a; CUtensorMap b; };

template <int PAIR>
__global__ void __launch_bounds__(128, 1) mma_kernel(const __grid_constant__ Maps maps, int iters, int S, int N,
                                                     unsigned long long* out, int mma_on, int dbg, int big) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int b_rows = PAIR ? N / 2 : N;
  const int a_bytes = 128 * 128, stage_bytes = a_bytes + b_rows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + 16;
  uint64_t* done = full + 32;
  uint32_t* holder = reinterpret_cast<uint32_t*>(full + 40);
  uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) { if (PAIR) tmem_alloc_pair<512>(holder); else tmem_alloc<512>(holder); }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  __shared__ unsigned long long tiss[16], tland[16];
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0 && mma_on < 2) {  // (modes >= 2: no producer)
    int ps = 0, ph = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&empty[ps], ph ^ 1);
      uint8_t* dst = smem + ps * stage_bytes;
      int k0 = (it % 64) * 64;
      int row = big ? (blockIdx.x * 128 + (it / 64) * 148 * 128) % (1 << 20) : ((blockIdx.x * 7 + it / 64) % 14) * 256;
      if (PAIR) {
        uint32_t fb = smem_addr(&full[ps]) & 0xFEFFFFFFu;
        if (rank == 0) mbar_arrive_expect_tx(&full[ps], 2 * stage_bytes);
        tma_load_3d_pair(dst, &maps.a, fb, k0, row, 0);
        tma_load_3d_pair(dst + a_bytes, &maps.b, fb, k0, row + 128, 0);
      } else {
        mbar_arrive_expect_tx(&full[ps], stage_bytes);
        tma_load_3d(dst, &maps.a, &full[ps], k0, row, 0);
        tma_load_3d(dst + a_bytes, &maps.b, &full[ps], k0, row + 128, 0);
      }
      if (it < 16) tiss[it] = clock64() - t0;
      if (++ps == S) { ps = 0; ph ^= 1; }
    }
  } else if (warp == 1 && mma_on >= 7) {  // 7: converged elect.sync issue, one accumulator; 8: two alternating; 9: four
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, N, 0, 0);
    const uint32_t base = smem_addr(smem);
    for (int it = 0; it < iters; ++it) {
      const int cs = it & 3;
      const uint32_t la = base + cs * stage_bytes, ca = la + a_bytes;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = umma_desc_sw128(la + kk * 32, 16, 1024), bd = umma_desc_sw128(ca + kk * 32, 16, 1024);
        const uint32_t acc = mma_on == 7 ? (it | kk) != 0 : it != 0;
        asm volatile(
            "{\n.reg .pred p, q;\n"
            "elect.sync _|p, 0xffffffff;\n"
            "setp.ne.b32 q, %4, 0;\n"
            "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n}\n" ::"r"(tm + (mma_on == 8 ? (kk & 1) * N : (mma_on == 9 ? kk * N : 0))),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
            : "memory");
      }
    }
    asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_addr(done)) : "memory");
  } else if (warp == 1 && lane == 0 && rank == 0) {
    int cs = 0, ph = 0;
    const uint32_t amn = (mma_on >= 5) ? 1u : 0u, bmn = (mma_on == 6) ? 1u : 0u;
    const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, N, amn, bmn);
    for (int it = 0; it < iters; ++it) {
      if (mma_on < 2) mbar_wait(&full[cs], ph);
      if (it < 16) tland[it] = clock64() - t0;
      tc_fence_after();
      const uint32_t la = smem_addr(smem + cs * stage_bytes), ca = la + a_bytes;
      if (mma_on) {
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = amn ? umma_desc_sw128(la + kk * 2048, 8192, 1024) : umma_desc_sw128(la + kk * 32, 16, 1024);
          const uint64_t bd = bmn ? umma_desc_sw128(ca + kk * 2048, 8192, 1024) : umma_desc_sw128(ca + kk * 32, 16, 1024);
          const uint32_t acc = tmem + (mma_on == 3 ? (kk & 1) * N : (mma_on == 4 ? kk * N : 0));
          if (PAIR) tc_mma_f16_pair(acc, ad, bd, idesc, (it | kk) != 0);
          else tc_mma_f16(acc, ad, bd, idesc, (it | kk) != 0);
        }
      }
      if (mma_on < 2) { if (PAIR) tc_commit_pair_mc(&empty[cs]); else tc_commit(&empty[cs]); }
      if (++cs == S) { cs = 0; ph ^= 1; }
    }
    if (PAIR) tc_commit_pair_mc(done); else tc_commit(done);
  }
  if (warp == 2 && lane == 0) mbar_wait(done, 0);
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (threadIdx.x == 0 && blockIdx.x == 0 && dbg) {
    printf("issue:"); for (int i = 0; i < 16; ++i) printf(" %llu", tiss[i]); printf("\n");
    printf("land :"); for (int i = 0; i < 16; ++i) printf(" %llu", tland[i]); printf("\n");
  }
  if (warp == 1) { tc_fence_after(); if (PAIR) tmem_dealloc_pair<512>(tmem); else tmem_dealloc<512>(tmem); }
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
  const int64_t K = 4096, R = 1 << 20;  // 8 GiB: the 'big' mode streams from HBM
  void* buf; cudaMalloc(&buf, K * R * 2); cudaMemset(buf, 0, K * R * 2);
  unsigned long long* out; cudaMalloc(&out, 148 * 8);
  const int ctas = 148, iters = 4000;
  struct Cfg { int pair, N, S, mma, big = 0; };
  std::vector<Cfg> cfgs = {
      {0, 256, 4, 2}, {0, 256, 4, 7}, {0, 128, 4, 2}, {0, 128, 4, 7}, {0, 64, 4, 2}, {0, 64, 4, 7}, {0, 32, 4, 7},
      {0, 64, 8, 1, 1}, {0, 64, 8, 1, 0}, {0, 256, 4, 1, 1},
      {0, 64, 4, 5}, {0, 128, 4, 5}, {0, 256, 4, 5}, {0, 64, 4, 6}, {0, 128, 4, 6}, {1, 128, 4, 5}, {1, 64, 4, 5},
      {0, 128, 4, 2}, {0, 128, 4, 3}, {0, 128, 4, 4}, {0, 64, 4, 2}, {0, 64, 4, 3}, {0, 64, 4, 4}, {0, 32, 4, 4}, {1, 128, 4, 3}, {1, 64, 4, 4},
      {0, 256, 4, 1}, {0, 256, 4, 0}, {0, 128, 6, 1}, {0, 64, 8, 1}, {0, 256, 3, 1},
      {1, 256, 6, 1}, {1, 256, 6, 0}, {1, 256, 4, 1}, {1, 128, 8, 1}, {1, 64, 8, 1}};
  if (const char* env = getenv("CFGS")) {  // "pair,N,S,mma,big;..."
    cfgs.clear();
    std::string all(env);
    size_t p0 = 0;
    while (p0 < all.size()) {
      size_t p1 = all.find(';', p0);
      if (p1 == std::string::npos) p1 = all.size();
      Cfg c{};
      sscanf(all.substr(p0, p1 - p0).c_str(), "%d,%d,%d,%d,%d", &c.pair, &c.N, &c.S, &c.mma, &c.big);
      cfgs.push_back(c);
      p0 = p1 + 1;
    }
  }
  int dbg = 0;
  for (auto& c : cfgs) {
    Maps m;
    make(&m.a, buf, K, R, 128);
    make(&m.b, buf, K, R, c.pair ? c.N / 2 : c.N);
    int b_rows = c.pair ? c.N / 2 : c.N;
    int smem = c.S * (128 + b_rows) * 128 + 2048;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(ctas); lc.blockDim = dim3(128); lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = c.pair ? 2 : 1;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    cudaError_t e;
    auto launch = [&](int it) {
      if (!c.pair) { cudaFuncSetAttribute(mma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, mma_kernel<0>, m, it, c.S, c.N, out, c.mma, dbg, c.big); }
      else { cudaFuncSetAttribute(mma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, mma_kernel<1>, m, it, c.S, c.N, out, c.mma, dbg, c.big); }
    };
    dbg = 0;
    launch(100); cudaDeviceSynchronize();
    dbg = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); launch(iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> cyc(ctas); cudaMemcpy(cyc.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
    double mc = 0; for (auto v : cyc) mc += v; mc /= ctas;
    double flops = 2.0 * 128 * c.N * 64 * iters * ctas;  // per CTA: 128 lanes x N x 64 per K block
    double ideal = 2.0 * c.N;  // clk per K block at 8192 flop/clk/SM
    printf("%s N=%3d S=%d mma=%d err=%d: %.3f ms, %.0f clk/kblock (ideal %.0f) -> %.0f%%  %.0f TF/s  TMA %.1f B/clk\n",
           c.pair ? "pair  " : "single", c.N, c.S, c.mma, (int)e, ms, mc / iters, ideal, 100 * ideal / (mc / iters),
           c.mma ? flops / (ms * 1e-3) / 1e12 : 0.0, (128 + b_rows) * 128.0 / (mc / iters));
  }
  return 0;
}
