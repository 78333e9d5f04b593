// TMA-store microbenchmark: what an epilogue's output write costs per SM for
// different store-box shapes, alone and with TMA loads streaming into the same
// SM (the producer's traffic in the real kernel).
//   ./store_bench            (CTAS=148 ITEMS=... env overrides)
// Each CTA = 4 "epilogue" warps (+ optional loader warp). One item = a 128-row
// x 256-column bf16 tile (64 KiB) written to a distinct place of a 1 GiB C.
// Modes:
//   0  per warp: 2 KiB boxes {32 cols, 32 rows} SWIZZLE_64B, 2 per group, double-buffered (the current epilogue)
//   1  per warp: 4 KiB boxes {64 cols, 32 rows} SWIZZLE_128B, 1 per group, double-buffered
//   2  CTA-wide: 16 KiB boxes {64 cols, 128 rows} SWIZZLE_128B, issued by one thread after a named barrier
//   4  per warp direct st.global.v4 of the staged box (LSU path, coalesced 64 B row segments)
// The staged smem contents are written once per group by the warp (STS.128)
// so the smem write cost is included as in the real epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include "../../paper_2407_21418_b200/csrc/ptx.cuh"
#include "../../paper_2407_21418_b200/csrc/epilogue.cuh"
using namespace ftb;

struct Maps { CUtensorMap s64; CUtensorMap s128; CUtensorMap s128w; CUtensorMap ld; };

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void __launch_bounds__(192, 1) store_kernel(const __grid_constant__ Maps maps, int items, int mode, int load,
                                                      __nv_bfloat16* C, int64_t ldc, unsigned long long* out, int wrap) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage = smem;                 // 4 warps x 8 KiB (modes 0, 1, 4) or 2 x 16 KiB (mode 2)
  uint8_t* ring = smem + 32768;          // loader ring: 4 x 48 KiB
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 32768 + 4 * 49152);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  volatile int* stop = reinterpret_cast<volatile int*>(bars + 16);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) mbar_init(&bars[s], 1);
    *stop = 0;
    fence_barrier_init();
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp == 4) {
    // loader: streams 48 KiB K blocks (three 128-row boxes) into a 4-stage ring as fast as TMA allows
    if (load && lane == 0) {
      int it = 0;
      while (!*stop) {
        const int s = it & 3;
        if (it >= 4) mbar_wait(&bars[s], ((it - 4) >> 2) & 1);
        mbar_arrive_expect_tx(&bars[s], 49152);
        const int row = ((blockIdx.x * 7 + it / 64) % 16) * 384;
        const int k0 = (it % 64) * 64;
        tma_load_3d(ring + s * 49152, &maps.ld, &bars[s], k0, row, 0);
        tma_load_3d(ring + s * 49152 + 16384, &maps.ld, &bars[s], k0, row + 128, 0);
        tma_load_3d(ring + s * 49152 + 32768, &maps.ld, &bars[s], k0, row + 256, 0);
        ++it;
      }
      for (int j = it > 4 ? it - 4 : 0; j < it; ++j) mbar_wait(&bars[j & 3], (j >> 2) & 1);
      out[gridDim.x + blockIdx.x] = it;  // K blocks loaded
    }
  } else if (warp < 4) {
    uint8_t* region = stage + warp * 8192;
    uint32_t ngrp = 0;
    for (int item = 0; item < items; ++item) {
      const int64_t row0 = (static_cast<int64_t>(item) * gridDim.x + blockIdx.x) % wrap * 128;  // distinct tiles, wrap x 64 KiB footprint
      const int col0 = 0;
      for (int c0 = 0; c0 < 256; c0 += 64) {
        uint32_t r[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(static_cast<float>(e + lane + c0));
        if (mode == 0) {
          uint8_t* box = region + (ngrp & 1) * 4096;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          stage_box_bf16(box, r, true);
          stage_box_bf16(box + 2048, r, true);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&maps.s64, smem_addr(box), col0 + c0, static_cast<int>(row0) + warp * 32, 0);
            tma_store_3d(&maps.s64, smem_addr(box + 2048), col0 + c0 + 32, static_cast<int>(row0) + warp * 32, 0);
            bulk_commit();
          }
        } else if (mode == 1) {
          uint8_t* box = region + (ngrp & 1) * 4096;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          // 32 rows x 128 B, SWIZZLE_128B: 16-B chunk index ^= row & 7
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint4 pk = make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]);
            *reinterpret_cast<uint4*>(box + lane * 128 + ((q ^ (lane & 7)) * 16)) = pk;
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&maps.s128, smem_addr(box), col0 + c0, static_cast<int>(row0) + warp * 32, 0);
            bulk_commit();
          }
        } else if (mode == 2) {
          // CTA-wide 128 x 64 box in two 16 KiB buffers; warp w owns rows [32w, 32w+32)
          uint8_t* box = stage + (ngrp & 1) * 16384;
          if (warp == 0 && lane == 0) bulk_wait_read<1>();
          named_bar(1, 128);  // the buffer is free for everyone
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int row = warp * 32 + lane;
            uint4 pk = make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]);
            *reinterpret_cast<uint4*>(box + row * 128 + ((q ^ (row & 7)) * 16)) = pk;
          }
          fence_async_smem();
          named_bar(1, 128);  // all rows staged
          if (warp == 0 && lane == 0) {
            tma_store_3d(&maps.s128w, smem_addr(box), col0 + c0, static_cast<int>(row0), 0);
            bulk_commit();
          }
        } else if (mode == 5) {
          // LSU, coalesced: per instruction 4 rows x 128 B (8 lanes per row), 8 instructions per
          // 32 x 64 group (the register contents stand in for a staged-and-reread box)
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int row = q * 4 + (lane >> 3), cc = (lane & 7) * 8;
            __nv_bfloat16* dst = C + (row0 + warp * 32 + row) * ldc + col0 + c0 + cc;
            __stcg(reinterpret_cast<uint4*>(dst), make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]));
          }
        } else {
          // LSU: each lane writes its own row's 64 columns (8 x 16 B) straight from registers
          __nv_bfloat16* dst = C + (row0 + warp * 32 + lane) * ldc + col0 + c0;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            __stcg(reinterpret_cast<uint4*>(dst) + q, make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]));
        }
        ++ngrp;
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  if (warp < 4) {
    named_bar(2, 128);
    if (threadIdx.x == 0) {
      out[blockIdx.x] = clock64() - t0;
      *stop = 1;
    }
  }
  __syncthreads();
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static void make(CUtensorMap* m, void* base, int64_t inner, int64_t rows, uint32_t bx, uint32_t by, CUtensorMapSwizzle sw) {
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)inner * 2, (cuuint64_t)(inner * rows * 2)};
  cuuint32_t box[3] = {bx, by, 1}, es[3] = {1, 1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d\n", (int)r);
}

int main() {
  const int64_t ldc = 256, rows = 4096 * 128;  // C: 512K rows x 256 cols bf16 = 256 MiB
  const int64_t K = 4096, R = 16 * 384 + 512;   // load source: 6.6K rows x 4096 (L2-resident, 54 MB)
  void *c, *a;
  cudaMalloc(&c, rows * ldc * 2);
  cudaMalloc(&a, R * K * 2);
  cudaMemset(a, 0, R * K * 2);
  unsigned long long* out;
  cudaMalloc(&out, 2 * 148 * 8);
  Maps m;
  make(&m.s64, c, ldc, rows, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  make(&m.s128, c, ldc, rows, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  make(&m.s128w, c, ldc, rows, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  make(&m.ld, a, K, R, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  const int ctas = getenv("CTAS") ? atoi(getenv("CTAS")) : 148;
  const int wrap = getenv("WRAP") ? atoi(getenv("WRAP")) : 4096;  // 256: 16 MiB footprint (L2-resident writes)
  const int smem = 32768 + 4 * 49152 + 1024 + 256;
  cudaFuncSetAttribute(store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"2KiB boxes {32x32} SW64 (current)", "4KiB boxes {64x32} SW128 per warp", "16KiB boxes {64x128} SW128 per CTA",
                         "-", "LSU st.global.v4 per-lane rows", "LSU st.global.v4 coalesced 4 rows x 128 B"};
  for (int items : {1, 16}) {
    for (int load : {0, 1}) {
      for (int mode : {0, 1, 2, 4, 5}) {
        store_kernel<<<ctas, 192, smem>>>(m, items, mode, load, (__nv_bfloat16*)c, ldc, out, wrap);
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) store_kernel<<<ctas, 192, smem>>>(m, items, mode, load, (__nv_bfloat16*)c, ldc, out, wrap);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<unsigned long long> h(2 * ctas);
        cudaMemcpy(h.data(), out, 2 * ctas * 8, cudaMemcpyDeviceToHost);
        double clk = 0, kbs = 0;
        for (int i = 0; i < ctas; ++i) { clk += h[i]; kbs += h[ctas + i]; }
        clk /= ctas;
        kbs /= ctas;
        const double bytes = 65536.0 * items;
        printf("wrap %4d items %2d load %d  %-38s err=%d  %7.2f us/launch  per-SM store %6.1f B/clk (%6.0f clk/item)  loads %.0f KB/clk-ish %s\n",
               wrap, items, load, names[mode], (int)e, ms * 1e3 / reps, bytes / clk, clk / items,
               load ? kbs * 49152 / clk : 0.0, load ? "(48 KiB K blocks loaded per clk)" : "");
      }
    }
  }
  return 0;
}
