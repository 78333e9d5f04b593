// kernel_ffma.cu — K2: fp32 FFMA executor for the validation mode (config 0:
// fp32 Dense, N=K=768). Same tile-schedule table as K1: each work item is an
// output rectangle (<= 64 x 64 after lowering splits a uKernel tile); K is
// staged through shared memory in 32-wide slices and every thread owns a
// 4 x 4 register tile (the uKernel's reg_tile, metrics.py:77-85, is recorded
// in the table's aux field; at fp32 the accumulation order is plain
// sequential-K FFMA, which is what the 1e-5 tolerance is set against).
// Orientation is always lanes = i, columns = j.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "exec_types.h"

namespace ftb {

constexpr int kFfmaTile = 64;
constexpr int kFfmaK = 32;
constexpr int kFfmaThreads = 256;

__global__ void __launch_bounds__(kFfmaThreads)
    ftb_ffma_kernel(const DevProblem* __restrict__ problems, const DevWork* __restrict__ work,
                    int32_t n_work) {
  __shared__ float sa[kFfmaK][kFfmaTile + 4];  // A^T slice: [k][i]
  __shared__ float sb[kFfmaK][kFfmaTile + 4];  // B slice:   [k][j]
  const int tx = threadIdx.x & 15;             // column group
  const int ty = threadIdx.x >> 4;             // row group
  for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
    const DevWork it = work[w];
    const DevProblem& P = problems[it.problem];
    const float* A = static_cast<const float*>(P.A) + static_cast<int64_t>(it.batch) * P.a_bs;
    const float* B = static_cast<const float*>(P.B) + static_cast<int64_t>(it.batch) * P.b_bs;
    const int i0 = it.lane0, j0 = it.col0, ni = it.lane_len, nj = it.col_len;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    for (int k0 = 0; k0 < P.K; k0 += kFfmaK) {
      // cooperative loads: 64 x 32 of A and 32 x 64 of B, zero-filled outside the tile
      for (int e = threadIdx.x; e < kFfmaTile * kFfmaK; e += kFfmaThreads) {
        const int r = e / kFfmaK, kk = e % kFfmaK;  // A: row r, k kk (k contiguous)
        const int gk = k0 + kk;
        sa[kk][r] = (r < ni && gk < P.K) ? A[static_cast<int64_t>(i0 + r) * P.lda + gk] : 0.f;
      }
      for (int e = threadIdx.x; e < kFfmaTile * kFfmaK; e += kFfmaThreads) {
        int kk, c;
        if (P.b_nk) { c = e / kFfmaK; kk = e % kFfmaK; }   // B[N][K]: k contiguous
        else        { kk = e / kFfmaTile; c = e % kFfmaTile; }  // B[K][N]: n contiguous
        const int gk = k0 + kk;
        float v = 0.f;
        if (c < nj && gk < P.K)
          v = P.b_nk ? B[static_cast<int64_t>(j0 + c) * P.ldb + gk]
                     : B[static_cast<int64_t>(gk) * P.ldb + j0 + c];
        sb[kk][c] = v;
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < kFfmaK; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = sa[kk][ty * 4 + a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = sb[kk][tx * 4 + b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
      }
      __syncthreads();
    }
    float* C = static_cast<float*>(P.C) + static_cast<int64_t>(it.batch) * P.c_bs;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = ty * 4 + a;
      if (r >= ni) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int c = tx * 4 + b;
        if (c >= nj) continue;
        float x = acc[a][b];
        if (P.bias)
          x += P.bias_f32 ? static_cast<const float*>(P.bias)[j0 + c]
                          : __bfloat162float(static_cast<const __nv_bfloat16*>(P.bias)[j0 + c]);
        if (P.act == 1) x = 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
        C[static_cast<int64_t>(i0 + r) * P.ldc + j0 + c] = x;
      }
    }
  }
}

cudaError_t launch_ffma(const DevProblem* problems, const DevWork* work, int32_t n_work,
                        int32_t n_ctas, cudaStream_t stream) {
  if (n_work == 0) return cudaSuccess;
  ftb_ffma_kernel<<<n_ctas, kFfmaThreads, 0, stream>>>(problems, work, n_work);
  return cudaGetLastError();
}

}  // namespace ftb
