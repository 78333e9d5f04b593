// Main loop + epilogue microbenchmark: persistent items of KB K-blocks,
// 2 TMEM accumulator slots, epilogue warps drain TMEM to global (bf16).
// Variants: epi=0 (no epilogue work, just release), 1 (tcgen05.ld + direct
// 16B stores per row), 2 (tcgen05.ld only).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cstdint>
#include <vector>
#include "../../paper_2407_21418_b200/csrc/ptx.cuh"
using namespace ftb;
struct Maps { CUtensorMap a; CUtensorMap b; CUtensorMap c; };

template <int PAIR>
__global__ void __launch_bounds__(192, 1) epi_kernel(const __grid_constant__ Maps maps_p, int items, int KB, int S,
                                                     int N, unsigned long long* out, int epi, __nv_bfloat16* C, int dbg, int real, const Maps* gmaps) {
  const Maps& maps = gmaps ? *gmaps : maps_p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int b_rows = PAIR ? N / 2 : N;
  const int a_bytes = 128 * 128, stage_bytes = a_bytes + b_rows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + 16;
  uint64_t* tfull = full + 32;
  uint64_t* tempty = full + 34;
  uint32_t* holder = reinterpret_cast<uint32_t*>(full + 40);
  uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], PAIR ? 8 : 4); }
    fence_barrier_init();
  }
  if (warp == 1) { if (PAIR) tmem_alloc_pair<512>(holder); else tmem_alloc<512>(holder); }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  uint8_t* epi_smem = smem + S * stage_bytes + 1024;  // 4 warps x 2 x 2 KiB
  unsigned long long t0 = clock64();
  const int cid = PAIR ? blockIdx.x / 2 : blockIdx.x;
  if (warp == 0 && lane == 0) {
    int ps = 0, ph = 0;
    for (int item = 0; item < items; ++item)
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&empty[ps], ph ^ 1);
        uint8_t* dst = smem + ps * stage_bytes;
        int k0 = kb * 64;
        const int wi = (cid + item * (PAIR ? (int)(gridDim.x / 2) : (int)gridDim.x)) % 256;
        int row = real ? (wi / 16 % 16) * 256 + rank * 128 : ((cid * 7 + item) % 14) * 256 + rank * 128;
        const int brow = real ? (wi % 16) * 256 + rank * b_rows : ((cid * 3 + item) % 14) * 256 + rank * b_rows;
        if (PAIR) {
          uint32_t fb = smem_addr(&full[ps]) & 0xFEFFFFFFu;
          if (rank == 0) mbar_arrive_expect_tx(&full[ps], 2 * stage_bytes);
          tma_load_3d_pair(dst, &maps.a, fb, k0, row, 0);
          tma_load_3d_pair(dst + a_bytes, &maps.b, fb, k0, brow, 0);
        } else {
          mbar_arrive_expect_tx(&full[ps], stage_bytes);
          tma_load_3d(dst, &maps.a, &full[ps], k0, row, 0);
          tma_load_3d(dst + a_bytes, &maps.b, &full[ps], k0, real ? (wi % 16) * 256 : ((cid * 3 + item) % 14) * 256, 0);
        }
        if (++ps == S) { ps = 0; ph ^= 1; }
      }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    int cs = 0, ph = 0;
    const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, N, 0, 0);
    for (int item = 0; item < items; ++item) {
      const int slot = item & 1, use = item >> 1;
      mbar_wait(&tempty[slot], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t acc = tmem + slot * 256;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&full[cs], ph);
        tc_fence_after();
        const uint32_t la = smem_addr(smem + cs * stage_bytes), ca = la + a_bytes;
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = umma_desc_sw128(la + kk * 32, 16, 1024), bd = umma_desc_sw128(ca + kk * 32, 16, 1024);
          if (PAIR) tc_mma_f16_pair(acc, ad, bd, idesc, (kb | kk) != 0);
          else tc_mma_f16(acc, ad, bd, idesc, (kb | kk) != 0);
        }
        if (PAIR) tc_commit_pair_mc(&empty[cs]); else tc_commit(&empty[cs]);
        if (++cs == S) { cs = 0; ph ^= 1; }
      }
      if (PAIR) tc_commit_pair_mc(&tfull[slot]); else tc_commit(&tfull[slot]);
    }
  } else if (warp >= 2) {
    unsigned long long t_ld = 0, t_wait = 0, t_all0 = clock64(), n_chunk = 0, t_tf = 0;
    const int quad = warp & 3;
    for (int item = 0; item < items; ++item) {
      const int slot = item & 1, use = item >> 1;
      unsigned long long tw0 = clock64();
      mbar_wait(&tfull[slot], use & 1);
      t_tf += clock64() - tw0;
      tc_fence_after();
      if (epi) {
        const uint32_t taddr = tmem + ((quad * 32) << 16) + slot * 256;
        const int row = blockIdx.x * 128 + quad * 32 + lane;
        for (int c0 = 0; c0 < N; c0 += 32) {
          uint32_t r[32];
          unsigned long long tl0 = clock64();
          tmem_ld_32x32b_x32(taddr + c0, r);
          tmem_ld_wait();
          t_ld += clock64() - tl0; ++n_chunk;
          if (epi == 1) {
            uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * 256 + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 pk; uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[q * 8 + 2 * e]), __uint_as_float(r[q * 8 + 2 * e + 1]));
                pw[e] = *reinterpret_cast<uint32_t*>(&h);
              }
              dst[q] = pk;
            }
          } else if (epi == 3) {
            // stage 32x32 bf16 (64-B rows, 64-B swizzle) and TMA-store it
            const int buf = (c0 >> 5) & 1;
            uint8_t* stg = epi_smem + (quad * 2 + buf) * 2048;
            unsigned long long ta = clock64();
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            t_wait += clock64() - ta;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 pk; uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[q * 8 + 2 * e]), __uint_as_float(r[q * 8 + 2 * e + 1]));
                pw[e] = *reinterpret_cast<uint32_t*>(&h);
              }
              const int chunk = q ^ ((lane >> 1) & 3);
              *reinterpret_cast<uint4*>(stg + lane * 64 + chunk * 16) = pk;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                           :: "l"(reinterpret_cast<uint64_t>(&maps.c)), "r"(smem_addr(stg)), "r"(c0), "r"(blockIdx.x * 128 + quad * 32), "r"(0) : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
          } else if (r[0] == 0x12345678u) C[0] = __float2bfloat16(1.f);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_addr(&tempty[slot]) & 0xFEFFFFFFu) : "memory");
        else mbar_arrive(&tempty[slot]);
      }
    }
    if (lane == 0 && blockIdx.x == 0 && warp == 2 && dbg)
      printf("epi warp: chunks %llu  ld+wait %.0f clk/chunk  wait_read %.0f clk/chunk  total-busy %.0f clk/chunk  tfull-wait %llu of %llu\n", n_chunk,
             (double)t_ld / n_chunk, (double)t_wait / n_chunk, (double)(clock64() - t_all0 - t_tf) / n_chunk, t_tf, clock64() - t_all0);
  }
  if (warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
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
__global__ void fill(__nv_bfloat16* p, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = __float2bfloat16(((i * 2654435761u) % 1000) / 1000.f - 0.5f);
}

int main() {
  const int64_t K = 4096, R = 4096;
  __nv_bfloat16* buf; cudaMalloc(&buf, K * R * 2);
  fill<<<1024, 256>>>(buf, K * R);
  __nv_bfloat16* buf2; cudaMalloc(&buf2, K * R * 2);
  fill<<<1024, 256>>>(buf2, K * R);
  __nv_bfloat16* C; cudaMalloc(&C, 148 * 128 * 256 * 2);
  unsigned long long* out; cudaMalloc(&out, 148 * 8);
  const int ctas = getenv("CTAS") ? atoi(getenv("CTAS")) : 148;
  struct Cfg { int pair, N, S, KB, items, epi, real = 0, gm = 0; };
  std::vector<Cfg> cfgs = {
      {1, 256, 6, 64, 64, 3, 1, 1}, {0, 256, 4, 64, 64, 3, 1, 1}, {1, 256, 6, 64, 64, 3, 1, 1}, {0, 256, 4, 64, 64, 3, 1, 1},
      };
  if (const char* env = getenv("CFGS")) {  // "pair,N,S,KB,items,epi;..." (real=1, gm=1)
    cfgs.clear();
    std::string all(env);
    size_t p0 = 0;
    while (p0 < all.size()) {
      size_t p1 = all.find(';', p0);
      if (p1 == std::string::npos) p1 = all.size();
      Cfg c{};
      c.real = 1; c.gm = 1;
      sscanf(all.substr(p0, p1 - p0).c_str(), "%d,%d,%d,%d,%d,%d", &c.pair, &c.N, &c.S, &c.KB, &c.items, &c.epi);
      cfgs.push_back(c);
      p0 = p1 + 1;
    }
  }
  int dbg = 0;
  Maps* dmaps; cudaMalloc(&dmaps, sizeof(Maps));
  for (auto& c : cfgs) {
    Maps m;
    make(&m.a, buf, K, R, 128);
    make(&m.b, c.real ? buf2 : buf, K, R, c.pair ? c.N / 2 : c.N);
    {
      cuuint64_t dims[3] = {256, 148 * 128, 1};
      cuuint64_t strides[2] = {256 * 2, 148 * 128 * 256 * 2};
      cuuint32_t box[3] = {32, 32, 1}, es[3] = {1, 1, 1};
      CUresult r = enc()(&m.c, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, C, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) printf("encode C failed %d\n", r);
    }
    cudaMemcpy(dmaps, &m, sizeof(Maps), cudaMemcpyHostToDevice);
    int b_rows = c.pair ? c.N / 2 : c.N;
    int smem = c.S * (128 + b_rows) * 128 + 2048 + 16384;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(ctas); lc.blockDim = dim3(192); lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = c.pair ? 2 : 1;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    cudaError_t e;
    auto launch = [&](int items) {
      if (!c.pair) { cudaFuncSetAttribute(epi_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, epi_kernel<0>, m, items, c.KB, c.S, c.N, out, c.epi, C, dbg, c.real, c.gm ? dmaps : nullptr); }
      else { cudaFuncSetAttribute(epi_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&lc, epi_kernel<1>, m, items, c.KB, c.S, c.N, out, c.epi, C, dbg, c.real, c.gm ? dmaps : nullptr); }
    };
    dbg = 0;
    launch(4); cudaDeviceSynchronize();
    dbg = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); launch(c.items); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> cyc(ctas); cudaMemcpy(cyc.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
    double mc = 0; for (auto v : cyc) mc += v; mc /= ctas;
    double kbs = (double)c.items * c.KB;
    double flops = 2.0 * 128 * c.N * 64 * kbs * ctas;
    printf("%s gm=%d N=%d S=%d KB=%d items=%d epi=%d err=%d: %.3f ms, %.0f clk/kblock (ideal %d), %.0f TF/s, clk %.2f GHz\n",
           c.pair ? "pair  " : "single", c.gm, c.N, c.S, c.KB, c.items, c.epi, (int)e, ms, mc / kbs, 2 * c.N,
           flops / (ms * 1e-3) / 1e12, mc / (ms * 1e6));
  }
  return 0;
}
