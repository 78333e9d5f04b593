// kernel_ffma.cu — K2: fp32 FFMA executor for the validation mode (config 0:
// fp32 Dense, N=K=768; any fp32 Dense / BMM). Same tile-schedule table as
// K1: each work item is an output rectangle of at most 64 x 64 — whole plan
// uKernel rectangles merged (exec.cu; the FFMA descriptor's uKernels are
// small, e.g. 3 x 32 ... 30 x 32, Fig. 8). K streams through a
// 6-stage shared-memory ring of 32-wide slices filled by cp.async — only the
// item's own rows / columns, the K tail zero-filled; A rows (K-contiguous)
// and B [K, N] rows in 16-B copies when aligned — so five slices are in
// flight behind the one being multiplied. A is staged [row][k], B [k][n]:
// per four K steps a thread reads its 4 x 4 register tile's operands with
// eight 16-B shared loads for 64 FFMAs. At fp32 the accumulation order is
// plain sequential-K FFMA, which is what the 1e-5 tolerance is set against.
// Orientation is always lanes = i, columns = j.
//
// Round 2 (scripts/c0_time.py, C0 M = 512, L2-cold chain): round 1's kernel
// issued sixteen 4-B load + store round trips per thread and slice for the
// whole 64 x 64 tile whatever the item's size: 164 us; one CTA per uKernel
// rectangle, 4-B A copies: 115 us; merged rectangles + this kernel: 37.7 us
// (cuBLAS fp32 22.4 us; profiles/r2bk_c0_ffma_merge.txt).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "exec_types.h"
#include "ptx.cuh"

namespace ftb {

constexpr int kFfmaTile = 64;
constexpr int kFfmaK = 32;
constexpr int kFfmaThreads = 256;
constexpr int kFfmaStages = 6;
constexpr int kFfmaPer = kFfmaTile * kFfmaK / kFfmaThreads;  // 8 elements of A (and of B) per thread and slice
constexpr int kFfmaLdN = kFfmaTile + 4;                       // padded row of a [k][n] slice
constexpr int kFfmaLdK = kFfmaK + 4;                          // padded row of an A [row][k] slice (144 B)

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
  // A slices [stage][row][32 + 4] (copied with 16-B cp.async straight from
  // A's K-contiguous rows), B slices [stage][k][64 + 4]: per four K steps the
  // inner loop reads four rows x four k of A and four k x four columns of B
  // with eight 16-B loads for 64 FFMAs
  constexpr int kSaStride = kFfmaTile * kFfmaLdK, kSbStride = kFfmaK * kFfmaLdN;
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
        // A -> [row][k], only the item's rows; the K tail is zero-filled
        if (kVec) {  // 16-B copies of 4 consecutive k (8 per row and slice)
          for (int e = threadIdx.x; e < kFfmaTile * (kFfmaK / 4); e += kFfmaThreads) {
            const int r = e >> 3, c = (e & 7) * 4, gk = k0 + c;
            if (r < ni)
              cp_async16(a + r * kFfmaLdK + c, A + static_cast<int64_t>(i0 + r) * P.lda + (gk < K ? gk : 0),
                         gk < K ? min(16, (K - gk) * 4) : 0);
          }
        } else {
          for (int e = threadIdx.x; e < kFfmaK * kFfmaTile; e += kFfmaThreads) {
            const int kk = e & (kFfmaK - 1), r = e / kFfmaK, gk = k0 + kk;
            if (r < ni) cp_async4(a + r * kFfmaLdK + kk, A + static_cast<int64_t>(i0 + r) * P.lda + min(gk, K - 1), gk < K);
          }
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
#pragma unroll 2
      for (int kk = 0; kk < kFfmaK; kk += 4) {
        // eight 16-B shared loads per 64 FFMAs: rows ty*4.. x k kk..kk+3 of A,
        // k kk..kk+3 x columns tx*4.. of B; the k order per element stays sequential
        float ax[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const float4 av = *reinterpret_cast<const float4*>(a + (ty * 4 + x) * kFfmaLdK + kk);
          ax[x][0] = av.x;
          ax[x][1] = av.y;
          ax[x][2] = av.z;
          ax[x][3] = av.w;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 bv = *reinterpret_cast<const float4*>(b + (kk + q) * kFfmaLdN + tx * 4);
          const float bx[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(ax[x][q], bx[y], acc[x][y]);
        }
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

int ffma_smem_bytes() {
  return static_cast<int>(sizeof(float)) * kFfmaStages * (kFfmaTile * kFfmaLdK + kFfmaK * kFfmaLdN);
}

// vec: every operand row 16-B aligned (base and leading dimension), so the
// 16-B copy path is legal; the 4-B path gives bit-identical results (same
// FFMA order, only the copy width differs).
cudaError_t launch_ffma(const DevProblem* problems, const DevWork* work, int32_t n_work,
                        int32_t n_ctas, cudaStream_t stream, bool vec) {
  if (n_work == 0) return cudaSuccess;
  const int smem = ffma_smem_bytes();  // 6 x (64 x 36 + 32 x 68) floats = 105 KiB: needs the opt-in
  cudaError_t e = vec ? configure_smem_once<ftb_ffma_kernel<true>>(smem) : configure_smem_once<ftb_ffma_kernel<false>>(smem);
  if (e != cudaSuccess) return e;
  if (vec) ftb_ffma_kernel<true><<<n_ctas, kFfmaThreads, smem, stream>>>(problems, work, n_work);
  else ftb_ffma_kernel<false><<<n_ctas, kFfmaThreads, smem, stream>>>(problems, work, n_work);
  return cudaGetLastError();
}

}  // namespace ftb
