// kernel_tc.cu — K1: the persistent sm_100a uKernel executor.
//
// One launch runs every work item of a lowered tile-schedule table (any mix of
// problems, uKernel tile sizes and orientations). Each CTA owns one SM and
// walks its share of the table with three warp roles:
//   warp 0      TMA producer: per 64-wide K block, one box for the lane operand
//               (128 rows) and n_mma/16 (K-major) or n_mma/64 (MN-major) boxes
//               for the column operand, into a 4-stage smem ring (SW128).
//   warp 1      MMA issuer: one elected thread issues 4 x tcgen05.mma
//               (M=128, N=n_mma, K=16) per K block into one of two TMEM
//               accumulators (2 x 256 columns) and commits to mbarriers.
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time, bf16/fp32 convert,
//               predicated stores for ragged uKernel edges; releases the
//               accumulator so the next item's MMAs overlap this store.
// The reference has no executor; the semantics it must honour are
// ProgramPlan coverage (combine.py:40-55): each work item writes exactly its
// rectangle of C, and the rectangles of a plan tile C once.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "exec_types.h"
#include "ptx.cuh"

namespace ftb {

struct TcSmem {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

constexpr int kRingBytes = kStages * (kLaneStageBytes + kColStageBytes);
constexpr int kTcSmemBytes = kRingBytes + 1024 /*align slack*/ + 256 /*barriers*/;

__device__ __forceinline__ void store_out(void* C, int64_t off, float v, int out_f32) {
  if (out_f32)
    static_cast<float*>(C)[off] = v;
  else
    static_cast<__nv_bfloat16*>(C)[off] = __float2bfloat16_rn(v);
}

__global__ void __launch_bounds__(kTcThreads, 1)
    ftb_tc_kernel(const DevProblem* __restrict__ problems, const DevWork* __restrict__ work,
                  int32_t n_work) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* lane_buf = smem;                                  // kStages x 16 KiB
  uint8_t* col_buf = smem + kStages * kLaneStageBytes;       // kStages x 32 KiB
  TcSmem* bars = reinterpret_cast<TcSmem*>(smem + kRingBytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bars->tfull[a], 1);
      mbar_init(&bars->tempty[a], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t g = 0;  // global K-block counter (ring position)
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const DevWork it = work[w];
        const DevProblem& P = problems[it.problem];
        const CUtensorMap* tl = &P.tm_lane;
        const CUtensorMap* tc = &P.tm_col;
        const uint32_t col_bytes = static_cast<uint32_t>(it.n_mma) * kBlockK * 2;
        for (int kb = 0; kb < P.num_kb; ++kb, ++g) {
          const uint32_t s = g % kStages;
          const uint32_t round = g / kStages;
          mbar_wait(&bars->empty[s], (round & 1) ^ 1);
          mbar_arrive_expect_tx(&bars->full[s], kLaneStageBytes + col_bytes);
          uint8_t* ldst = lane_buf + s * kLaneStageBytes;
          uint8_t* cdst = col_buf + s * kColStageBytes;
          const int k0 = kb * kBlockK;
          if (!P.lane_mn) {
            tma_load_3d(ldst, tl, &bars->full[s], k0, it.lane0, it.batch);
          } else {
            tma_load_3d(ldst, tl, &bars->full[s], it.lane0, k0, it.batch);
            tma_load_3d(ldst + 8192, tl, &bars->full[s], it.lane0 + 64, k0, it.batch);
          }
          if (!P.col_mn) {
            for (int r = 0; r < it.n_mma; r += kColBoxRows)
              tma_load_3d(cdst + r * 128, tc, &bars->full[s], k0, it.col0 + r, it.batch);
          } else {
            for (int c = 0; c < it.n_mma; c += 64)
              tma_load_3d(cdst + c * 128, tc, &bars->full[s], it.col0 + c, k0, it.batch);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t g = 0;
      uint32_t local = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++local) {
        const DevWork it = work[w];
        const DevProblem& P = problems[it.problem];
        const uint32_t acc = local & 1;
        const uint32_t use = local >> 1;
        mbar_wait(&bars->tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * kMaxN;
        const uint32_t idesc =
            idesc_bf16_f32(kLaneRows, static_cast<uint32_t>(it.n_mma), P.lane_mn, P.col_mn);
        for (int kb = 0; kb < P.num_kb; ++kb, ++g) {
          const uint32_t s = g % kStages;
          const uint32_t round = g / kStages;
          mbar_wait(&bars->full[s], round & 1);
          tc_fence_after();
          const uint32_t la = smem_addr(lane_buf + s * kLaneStageBytes);
          const uint32_t ca = smem_addr(col_buf + s * kColStageBytes);
#pragma unroll
          for (int kk = 0; kk < kBlockK / 16; ++kk) {
            const uint64_t adesc = P.lane_mn ? umma_desc_sw128(la + kk * 2048, 8192, 1024)
                                             : umma_desc_sw128(la + kk * 32, 16, 1024);
            const uint64_t bdesc = P.col_mn ? umma_desc_sw128(ca + kk * 2048, 8192, 1024)
                                            : umma_desc_sw128(ca + kk * 32, 16, 1024);
            tc_mma_f16(tmem_d, adesc, bdesc, idesc, (kb | kk) != 0);
          }
          tc_commit(&bars->empty[s]);  // frees the smem slot when these MMAs finish
        }
        tc_commit(&bars->tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    uint32_t local = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++local) {
      const DevWork it = work[w];
      const DevProblem& P = problems[it.problem];
      const uint32_t acc = local & 1;
      const uint32_t use = local >> 1;
      mbar_wait(&bars->tfull[acc], use & 1);
      tc_fence_after();
      const int my_lane = quad * 32 + lane;
      const bool lane_ok = my_lane < it.lane_len;
      const int64_t cb = static_cast<int64_t>(it.batch) * P.c_bs;
      if (quad * 32 < it.lane_len) {
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * kMaxN;
        for (int c0 = 0; c0 < it.col_len; c0 += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c0, v);
          tmem_ld_wait();
          if (lane_ok) {
            const int ncol = min(32, it.col_len - c0);
            if (!P.swap) {
              // lane = row i of C, columns = consecutive j
              const int64_t row = it.lane0 + my_lane;
              const int64_t base = cb + row * P.ldc + it.col0 + c0;
              if (!P.out_f32 && ncol == 32 && (base & 7) == 0) {
                uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(P.C) + base);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  uint4 pk;
                  uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[q * 8 + 2 * e]),
                                                             __uint_as_float(v[q * 8 + 2 * e + 1]));
                    pw[e] = *reinterpret_cast<uint32_t*>(&h);
                  }
                  dst[q] = pk;
                }
              } else if (P.out_f32 && ncol == 32 && (base & 3) == 0) {
                float4* dst = reinterpret_cast<float4*>(static_cast<float*>(P.C) + base);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                       __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
              } else {
#pragma unroll
                for (int e = 0; e < 32; ++e)
                  if (e < ncol) store_out(P.C, base + e, __uint_as_float(v[e]), P.out_f32);
              }
            } else {
              // lane = column j of C, TMEM columns = consecutive rows i
              const int64_t col = it.lane0 + my_lane;
              const int64_t base = cb + static_cast<int64_t>(it.col0 + c0) * P.ldc + col;
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (e < ncol) store_out(P.C, base + e * P.ldc, __uint_as_float(v[e]), P.out_f32);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

cudaError_t launch_tc(const DevProblem* problems, const DevWork* work, int32_t n_work,
                      int32_t n_ctas, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(ftb_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kTcSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_work == 0) return cudaSuccess;
  ftb_tc_kernel<<<n_ctas, kTcThreads, kTcSmemBytes, stream>>>(problems, work, n_work);
  return cudaGetLastError();
}

}  // namespace ftb
