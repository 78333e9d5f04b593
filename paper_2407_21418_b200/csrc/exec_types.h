// exec_types.h — device-resident tile-schedule table shared by the host
// lowering (lower.cpp) and the persistent kernels (kernel_tc.cu, kernel_ffma.cu).
#pragma once
#include <cstdint>
#include <cuda.h>

namespace ftb {

// One GEMM problem as the kernels see it. TMA descriptors are built on the
// host (cuTensorMapEncodeTiled) and live in global memory next to the table.
//   lane operand: the tensor whose rows map to TMEM lanes (MMA M = 128)
//   col operand : the tensor whose rows map to TMEM columns (MMA N <= 256)
// orientation 0 (normal): lanes = i (A), cols = j (B)
// orientation 1 (swap-AB): lanes = j (B), cols = i (A)
struct alignas(128) DevProblem {
  CUtensorMap tm_lane;   // box {64, 128, 1} (K-major) or {64, 64, 1} (MN-major)
  CUtensorMap tm_col;    // box {64, 16, 1}  (K-major) or {64, 64, 1} (MN-major)
  // Raw views, used by the FFMA kernel and by the epilogue.
  const void* A;
  const void* B;
  void* C;
  int64_t lda, ldb, ldc;
  int64_t a_bs, b_bs, c_bs;   // batch strides (elements)
  int32_t M, N, K, batch;
  int32_t lane_mn;            // lane operand is MN-major (swap + B stored [K,N])
  int32_t col_mn;             // col operand is MN-major (normal + B stored [K,N])
  int32_t swap;               // orientation
  int32_t out_f32;            // C dtype: 0 bf16, 1 fp32
  int32_t b_nk;               // B stored [N,K]
  int32_t num_kb;             // ceil(K / 64)
  int32_t pad_[2];
};

// One work item: an output rectangle of at most 128 lanes x 256 columns.
struct alignas(16) DevWork {
  int32_t problem;
  int32_t batch;
  int32_t lane0;     // first lane-axis index (i for normal, j for swap)
  int32_t col0;      // first column-axis index
  int32_t lane_len;  // valid lanes (<= 128)
  int32_t col_len;   // valid columns (<= 256)
  int32_t n_mma;     // MMA N (multiple of 16; of 64 when col operand is MN-major)
  int32_t aux;       // FFMA: reg tiles (ri | rj << 16); tcgen05: unused
};

constexpr int kBlockK = 64;          // one 128-B swizzle atom of bf16 along K
constexpr int kLaneRows = 128;       // MMA M
constexpr int kMaxN = 256;           // MMA N upper bound
constexpr int kStages = 4;
constexpr int kLaneStageBytes = kLaneRows * kBlockK * 2;   // 16 KiB
constexpr int kColStageBytes = kMaxN * kBlockK * 2;        // 32 KiB
constexpr int kColBoxRows = 16;                            // K-major col operand box rows
constexpr int kTmemCols = 512;                             // 2 accumulators x 256 columns
constexpr int kTcThreads = 192;                            // 6 warps

}  // namespace ftb
