// kernel_ffma.cu — K2: fp32 FFMA executor for the validation mode (config 0:
// fp32 Dense, N=K=768; any fp32 Dense / BMM). Same tile-schedule table as
// K1: each work item is an output rectangle (<= 64 x 64 after lowering splits
// a uKernel tile). K streams through a 3-stage shared-memory ring of 32-wide
// slices filled by cp.async — only the item's own rows / columns (the
// uKernels the FFMA descriptor picks are small, e.g. 29 x 32, PAPER.md
// Fig. 8), the K tail zero-filled, B [K, N] rows in 16-B copies when aligned —
// so two slices are in flight behind the one being multiplied. Both slices are
// stored k-major, so every thread reads its 4 x 4 register tile's operands
// with two 16-B shared loads per 16 FFMAs. At fp32 the accumulation order is plain
// sequential-K FFMA, which is what the 1e-5 tolerance is set against.
// Orientation is always lanes = i, columns = j.
//
// Round 2 (scripts/c0_time.py, C0 M = 512, L2-cold chain): round 1's kernel
// issued sixteen 4-B load + store round trips per thread and slice for the
// whole 64 x 64 tile whatever the item's size: 164 us (cuBLAS fp32 22 us);
// the inner loop's eight 4-B shared loads per 16 FFMAs capped it as much.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "exec_types.h"
#include "ptx.cuh"

namespace ftb {

constexpr int kFfmaTile = 64;
constexpr int kFfmaK = 32;
constexpr int kFfmaThreads = 256;
constexpr int kFfmaStages = 3;
constexpr int kFfmaPer = kFfmaTile * kFfmaK / kFfmaThreads;  // 8 elements of A (and of B) per thread and slice
constexpr int kFfmaLdN = kFfmaTile + 4;                       // padded row of a [k][n] slice

// 4-B global -> shared copy; src_bytes = 0 writes a zero
__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
// 16-B global -> shared copy of `bytes` (0..16) valid bytes, the rest zeroed
__device__ __forceinline__ void cp_async16(float* dst, const float* src, int bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <bool kVec>
__global__ void __launch_bounds__(kFfmaThreads)
    ftb_ffma_kernel(const DevProblem* __restrict__ problems, const DevWork* __restrict__ work,
                    int32_t n_work) {
  extern __shared__ float ffma_smem[];
  // A and B slices both [stage][k][64 + 4]: the inner loop reads four rows
  // of A and four columns of B with one 16-B load each
  constexpr int kSaStride = kFfmaK * kFfmaLdN, kSbStride = kFfmaK * kFfmaLdN;
  float* sa = ffma_smem;
  float* sb = ffma_smem + kFfmaStages * kSaStride;
  const int tx = threadIdx.x & 15;  // column group
  const int ty = threadIdx.x >> 4;  // row group
  for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
    const DevWork it = work[w];
    const DevProblem& P = problems[it.problem];
    const float* A = static_cast<const float*>(P.A) + static_cast<int64_t>(it.batch) * P.a_bs;
    const float* B = static_cast<const float*>(P.B) + static_cast<int64_t>(it.batch) * P.b_bs;
    const int i0 = it.lane0, j0 = it.col0, ni = it.lane_len, nj = it.col_len;
    const bool bnk = P.b_nk;
    const int K = P.K;
    const int nslices = (K + kFfmaK - 1) / kFfmaK;
    auto issue = [&](int slice) {  // cp.async the slice into its ring stage (or an empty group past the end)
      if (slice < nslices) {
        const int st = slice % kFfmaStages, k0 = slice * kFfmaK;
        float* a = sa + st * kSaStride;
        float* b = sb + st * kSbStride;
        // A -> [k][row] (4-B copies; consecutive threads take consecutive
        // rows, so the shared-memory writes are conflict free), only the
        // item's rows; the K tail is zero-filled
        for (int e = threadIdx.x; e < kFfmaK * kFfmaTile; e += kFfmaThreads) {
          const int r = e & (kFfmaTile - 1), kk = e / kFfmaTile, gk = k0 + kk;
          if (r < ni) cp_async4(a + kk * kFfmaLdN + r, A + static_cast<int64_t>(i0 + r) * P.lda + min(gk, K - 1), gk < K);
        }
        if (!bnk && kVec) {  // B [K, N] -> [k][n] in 16-B chunks (the last may run past nj: discarded columns)
          const int n4 = (nj + 3) >> 2;
          for (int e = threadIdx.x; e < kFfmaK * n4; e += kFfmaThreads) {
            const int kk = e / n4, c = (e % n4) * 4, gk = k0 + kk;
            cp_async16(b + kk * kFfmaLdN + c, B + static_cast<int64_t>(min(gk, K - 1)) * P.ldb + j0 + c,
                       gk < K ? 16 : 0);
          }
        } else {  // 4-B copies into [k][n]
          for (int e = threadIdx.x; e < kFfmaK * kFfmaTile; e += kFfmaThreads) {
            const int c = e & (kFfmaTile - 1), kk = e / kFfmaTile, gk = k0 + kk;
            if (c < nj)
              cp_async4(b + kk * kFfmaLdN + c,
                        bnk ? B + static_cast<int64_t>(j0 + c) * P.ldb + min(gk, K - 1)
                            : B + static_cast<int64_t>(min(gk, K - 1)) * P.ldb + j0 + c,
                        gk < K);
          }
        }
      }
      cp_async_commit();
    };
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
#pragma unroll
    for (int s = 0; s < kFfmaStages - 1; ++s) issue(s);
    for (int slice = 0; slice < nslices; ++slice) {
      cp_async_wait<kFfmaStages - 2>();  // this slice has landed (for this thread) ...
      __syncthreads();                   // ... and for every thread; the stage refilled below is free
      issue(slice + kFfmaStages - 1);
      const int st = slice % kFfmaStages;
      const float* a = sa + st * kSaStride;
      const float* b = sb + st * kSbStride;
#pragma unroll 8
      for (int kk = 0; kk < kFfmaK; ++kk) {
        // two 16-B shared loads per 16 FFMAs (rows ty*4.., columns tx*4..)
        const float4 av = *reinterpret_cast<const float4*>(a + kk * kFfmaLdN + ty * 4);
        const float4 bv = *reinterpret_cast<const float4*>(b + kk * kFfmaLdN + tx * 4);
        const float ax[4] = {av.x, av.y, av.z, av.w}, bx[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(ax[x], bx[y], acc[x][y]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // the next item's first copies must not overwrite stages still being read
    float* C = static_cast<float*>(P.C) + static_cast<int64_t>(it.batch) * P.c_bs;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int r = ty * 4 + x;
      if (r >= ni) continue;
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int c = tx * 4 + y;
        if (c >= nj) continue;
        float v = acc[x][y];
        if (P.bias)
          v += P.bias_f32 ? static_cast<const float*>(P.bias)[j0 + c]
                          : __bfloat162float(static_cast<const __nv_bfloat16*>(P.bias)[j0 + c]);
        if (P.act == 1) v = 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
        C[static_cast<int64_t>(i0 + r) * P.ldc + j0 + c] = v;
      }
    }
  }
}

int ffma_smem_bytes() { return static_cast<int>(sizeof(float)) * kFfmaStages * 2 * kFfmaK * kFfmaLdN; }

// vec: every operand row 16-B aligned (base and leading dimension), so the
// 16-B copy path is legal; the 4-B path gives bit-identical results (same
// FFMA order, only the copy width differs).
cudaError_t launch_ffma(const DevProblem* problems, const DevWork* work, int32_t n_work,
                        int32_t n_ctas, cudaStream_t stream, bool vec) {
  if (n_work == 0) return cudaSuccess;
  const int smem = ffma_smem_bytes();  // 3 x 2 x 32 x 68 floats = 51 KiB: needs the opt-in
  cudaError_t e = vec ? configure_smem_once<ftb_ffma_kernel<true>>(smem) : configure_smem_once<ftb_ffma_kernel<false>>(smem);
  if (e != cudaSuccess) return e;
  if (vec) ftb_ffma_kernel<true><<<n_ctas, kFfmaThreads, smem, stream>>>(problems, work, n_work);
  else ftb_ffma_kernel<false><<<n_ctas, kFfmaThreads, smem, stream>>>(problems, work, n_work);
  return cudaGetLastError();
}

}  // namespace ftb
