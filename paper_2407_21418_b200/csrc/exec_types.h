// exec_types.h — device-resident tile-schedule table shared by the host
// lowering (exec.cu) and the persistent kernels (kernel_tc.cu, kernel_ffma.cu).
#pragma once
#include <cstdint>
#include <cuda.h>

namespace ftb {

// One GEMM problem as the FFMA kernel and the host see it.
//   lane operand: the tensor whose rows map to TMEM lanes (MMA M = 128)
//   col operand : the tensor whose rows map to TMEM columns (MMA N <= 256)
// orientation 0 (normal): lanes = i (A), cols = j (B)
// orientation 1 (swap-AB): lanes = j (B), cols = i (A)
struct DevProblem {
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
  const void* bias;           // fused epilogue: bias[N] (or null)
  int32_t bias_f32;           // bias dtype: 0 bf16, 1 fp32
  int32_t act;                // FTB_ACT_*
};

// Fused epilogue of one problem (Dense): C = act(acc + bias[col]).
struct EpiOp {
  const void* bias;  // bias[N] or null
  int32_t bias_f32;
  int32_t act;       // 0 none, 1 GELU (erf)
  int32_t n;         // valid columns of C (bias length)
  int32_t pad_;
};

// TMA descriptors of one problem for the tcgen05 kernel (64-B aligned).
//   lane  : box {64, 128} (K-major) or {64 MN, 64 K} (MN-major)
//   col[q]: K-major boxes of 256 >> q rows (q = 0..4: 256, 128, 64, 32, 16);
//           MN-major: col[0] = box {64 MN, 64 K}
//   out   : C store map (bf16 outputs), box {32 cols, 32 rows}, 64-B swizzle;
//           TMA clips stores at the tensor edge
struct alignas(64) DevMaps {
  CUtensorMap lane;
  CUtensorMap col[5];
  CUtensorMap out;
  EpiOp epi;
};
constexpr int kColMaps = 5;

// Which col[] boxes cover n rows (n multiple of 16, <= 256): bit q set = one
// box of 256 >> q rows; boxes are placed widest first.
__host__ __device__ inline uint32_t col_box_mask(int n) {
  if (n >= 256) return 1u;
  return (((n >> 7) & 1u) << 1) | (((n >> 6) & 1u) << 2) | (((n >> 5) & 1u) << 3) | (((n >> 4) & 1u) << 4);
}

// Logical work item (host export format, 8 x int32): an output rectangle of
// at most 128 lanes x 256 columns of one problem.
struct alignas(16) DevWork {
  int32_t problem;
  int32_t batch;
  int32_t lane0;     // first lane-axis index (i for normal, j for swap)
  int32_t col0;      // first column-axis index
  int32_t lane_len;  // valid lanes (<= 128)
  int32_t col_len;   // valid columns (<= 256)
  int32_t n_mma;     // MMA N (multiple of 16; of 64 when col operand is MN-major)
  int32_t aux;       // unused (0)
};

// Self-contained tcgen05 work item (64 B): everything a role needs without a
// dependent load of the problem record.
//   kFlagTmaStore: the item's rectangle is whole 32 x 32 store boxes or ends
//   at the tensor edge, so the epilogue may store through TMA (clipped by the
//   hardware) instead of predicated st.global.
//   kFlagSplitK: the item computes K blocks [kb0, kb0 + num_kb) of a tile split
//   over nsplit items (pack = kb0 | nsplit << 16 | split << 24, c_bs = tile);
//   partials meet in the fp32 workspace chunk by chunk (32 columns of one lane
//   quadrant); the last split to publish a chunk sums it and stores C, so no
//   split ever waits for another (no co-residency assumption; kernel_tc.cu).
//   kFlagBulkStore: no TMA store map fits (C rows not a multiple of 16 B), but
//   the item covers whole rows of a compact C (col0 = 0, col_len = N = ldc),
//   so each epilogue warp's rows are one contiguous byte range: staged in
//   shared memory in C's own layout and written by a 1-D bulk copy (plus
//   element stores for the < 16 B head and tail) instead of scattered
//   predicated stores.
enum : uint32_t {
  kFlagSwap = 1u, kFlagLaneMN = 2u, kFlagColMN = 4u, kFlagOutF32 = 8u, kFlagTmaStore = 16u, kFlagSplitK = 32u,
  kFlagEpiOp = 64u,     // fused bias / activation: maps->epi
  kFlagBulkStore = 128u,
  // kFlagTmaTail: with kFlagTmaStore, C's row length N is not a multiple of 8
  // bf16; the store map ends at N8 = N & ~7 (boxes clip exactly there) and the
  // item, whose columns end at N, writes its last N - N8 columns per row with
  // element stores
  kFlagTmaTail = 256u
};
// Block-diagonal batch packing (short attention BMMs, exec.cu): `pack` holds
// nb (entries in this item, bits 0-7), the TMA box depth (bits 8-15) and the
// lane slot rows (32 or 64, bits 16-31); entry e of the item is batch
// `batch + e`, its A rows sit at lanes [e*slot, (e+1)*slot) and its result in
// TMEM columns [64e, 64e + 64) of those lanes. pack == 0: a plain item.
struct alignas(64) TcWork {
  const DevMaps* maps;
  void* C;            // element 0 of this batch entry's output matrix
  int64_t ldc;
  int32_t lane0, col0;
  int32_t lane_len, col_len;
  int32_t n_mma, num_kb;
  int32_t batch;
  uint32_t flags;
  uint32_t pack;
  int32_t c_bs;       // batch stride of C in elements (packed items)
};
__host__ __device__ inline int pack_nb(uint32_t p) { return p ? static_cast<int>(p & 0xFFu) : 1; }
__host__ __device__ inline int pack_depth(uint32_t p) { return static_cast<int>((p >> 8) & 0xFFu); }
__host__ __device__ inline int pack_lane_rows(uint32_t p) { return static_cast<int>(p >> 16); }
constexpr int kMaxPack = 4;
__host__ __device__ inline int split_kb0(uint32_t p) { return static_cast<int>(p & 0xFFFFu); }
__host__ __device__ inline int split_n(uint32_t p) { return static_cast<int>((p >> 16) & 0xFFu); }
__host__ __device__ inline int split_idx(uint32_t p) { return static_cast<int>(p >> 24); }
constexpr int kMaxSplit = 8;
constexpr int kSplitRowFloats = 256;                          // columns per tile in the workspace
constexpr int kSplitTileFloats = kMaxSplit * 128 * kSplitRowFloats;
constexpr int kSplitChunks = kSplitRowFloats / 32;            // 32-column chunks per tile row
constexpr int kSplitCntPerTile = 4 * kSplitChunks;            // one arrival counter per (lane quadrant, chunk)

// CTA-pair work item (64 B): two 128-lane slabs (one per CTA of a cluster
// pair) that share the column operand; N = n_mma columns, each CTA stages
// N/2 of them. lane_len[r] == 0 marks an empty half (leftover single).
struct alignas(64) TcPair {
  const DevMaps* maps;
  void* C;
  int64_t ldc;
  int32_t lane0[2];
  int32_t lane_len[2];
  int32_t col0, col_len;
  int32_t n_mma, num_kb;
  int32_t batch;
  uint32_t flags;
};

// Per-launch pipeline shape, chosen by the host from the table's widest item.
struct TcConfig {
  int32_t stages;          // smem ring depth (K blocks of 64)
  int32_t col_stage_bytes; // bytes reserved per stage for the column operand
  int32_t n_acc;           // TMEM accumulator slots (2, 4 or 8)
  int32_t acc_cols;        // columns per slot (512 / n_acc)
  unsigned long long* trace;  // optional: per-CTA phase timestamps (debug)
  float* split_ws;            // split-K partials [tile][split][128][256] fp32
  int32_t* split_cnt;         // split-K arrival counters [tile][4 lane quadrants][8 chunks]
  int32_t cluster_split;      // > 1: split-K partials reduced on chip across a cluster of this many CTAs
  int32_t epi8;               // 1: eight epilogue warps (two groups on alternate items), 320 threads
  int32_t l2_prefetch;        // 1: L2-prefetch the first item's operands before griddepcontrol.wait
  int32_t param_maps;         // 1: single-problem table, descriptors in the kernel parameter (see kernel_tc.cu with_maps)
};
constexpr int kTraceItems = 16;   // items traced per CTA
constexpr int kTraceEvents = 6;   // see kernel_tc.cu
constexpr int kTraceKb = 64;      // K blocks traced per CTA (producer issue, MMA sees data)
constexpr int kTracePerCta = kTraceItems * kTraceEvents + 2 * kTraceKb + 2;  // + CTA start / end stamps

constexpr int kBlockK = 64;          // one 128-B swizzle atom of bf16 along K
constexpr int kLaneRows = 128;       // MMA M
constexpr int kMaxN = 256;           // MMA N upper bound
constexpr int kMaxStages = 8;
constexpr int kMmaFloorN = 200;      // an M=128 K=16 tcgen05.mma costs >= ~100 clk: N below this is not cheaper
constexpr int kLaneStageBytes = kLaneRows * kBlockK * 2;   // 16 KiB
constexpr int kTmemCols = 512;
constexpr int kTcThreads = 192;                            // 6 warps
constexpr int kTcThreadsEpi8 = 320;                        // 10 warps: eight epilogue warps
constexpr int kEpiWarpBytes = 8192;   // per epilogue warp: four 2 KiB bf16 TMA store boxes, or (aliased)
                                       // the 32x33 fp32 transpose tile of the predicated path
constexpr int kEpiStageBytes = 4 * kEpiWarpBytes;
constexpr int kTcSmemBudget = 232448 - 1024;               // max dynamic smem minus align slack

}  // namespace ftb
