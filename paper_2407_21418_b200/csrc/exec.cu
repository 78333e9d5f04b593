// exec.cu — host side of the executor: lowers ProgramPlans to the
// tile-schedule table, encodes TMA descriptors, uploads, and launches K1/K2.
//
// Lowering semantics (the reference's plan coverage, combine.py:40-55 and
// timemodel.py:78-96): part q of a plan covers count_q consecutive tau tiles
// of size smem_q[tau] starting at sum_{p<q} count_p*smem_p[tau]; every other
// space axis s is tiled uniformly by smem[s] from 0 with ceil(E_s/t_s) tiles
// (the last one ragged; elements >= E_s are padding and never stored). Each
// uKernel rectangle is then cut into MMA-sized work items (<= 128 lanes x 256
// columns) — an implementation detail below the uKernel abstraction.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "exec_types.h"
#include "status.h"

namespace ftb {

cudaError_t launch_tc(const TcWork*, int32_t, int32_t, TcConfig, const DevMaps*, cudaStream_t);
cudaError_t launch_tc2(const TcPair*, int32_t, int32_t, TcConfig, cudaStream_t);
int tc_smem_bytes(const TcConfig& cfg);
cudaError_t launch_ffma(const DevProblem*, const DevWork*, int32_t, int32_t, cudaStream_t, bool);

namespace {

#define FTB_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      throw ::ftb::cuda_error(std::string(#call) + ": " + cudaGetErrorString(e_));                \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw cuda_error("cuTensorMapEncodeTiled is unavailable (no CUDA driver?)");
  return fn;
}

// 3-D bf16 tensor map: dims {inner, rows, batch}, SWIZZLE_128B, OOB = zeros.
void encode_map(CUtensorMap* m, const void* base, int64_t inner, int64_t rows, int64_t batch,
                int64_t ld_elems, int64_t batch_stride_elems, uint32_t box_inner,
                uint32_t box_rows, uint32_t box_batch = 1) {
  if (reinterpret_cast<uintptr_t>(base) % 16)
    throw input_error("tcgen05 path needs 16-byte aligned operand base pointers", "A/B");
  if ((ld_elems * 2) % 16)
    throw input_error("tcgen05 path needs row strides that are multiples of 8 bf16 elements",
                      "ld");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(batch)};
  int64_t bs = batch > 1 ? batch_stride_elems : rows * ld_elems;
  if ((bs * 2) % 16) throw input_error("batch stride must be a multiple of 8 elements", "batch");
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld_elems * 2), static_cast<cuuint64_t>(bs * 2)};
  cuuint32_t box[3] = {box_inner, box_rows, box_batch};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

// C store map for the TMA-store epilogue (bf16 outputs): dims {N, M, batch},
// box {32, 32}, 64-B swizzle. Returns false (no TMA stores for this problem)
// for fp32 outputs or when C violates TMA's 16-byte alignment rules. Measured
// on B200 (tests/test_exec_gpu.py::test_dense_strided_output_untouched_padding):
// stores clip the inner dimension at 16-byte granularity, so a row length N
// that is not a multiple of 8 bf16 would clobber up to 7 elements past the
// tensor edge. Such problems (normal orientation, rows 16-B aligned, N >= 8)
// get a map that ends at N8 = N rounded down to 8 — every box clips exactly
// there — and the epilogue writes the last N - N8 (< 8) columns of each row
// with element stores (kFlagTmaTail); returns 2 for that form. Otherwise
// they keep the predicated st.global epilogue.
int encode_out_map(CUtensorMap* m, const ftb_gemm_desc& d, bool swap) {
  if (d.out_dtype != FTB_DT_BF16) return 0;
  int64_t n_map = d.N;
  if ((d.N * 2) % 16) {
    const char* env = std::getenv("FTB_TMA_TAIL");
    // measured (profiles/r2be_tma_tail_min.txt): scores T = 39 / 45 5.1 /
    // 5.3 -> 4.5 / 4.6 us, T = 95 / 121 8.8 / 9.6 -> 6.9 / 7.5 us; T < 16
    // even, so those keep the predicated path
    const char* env_min = std::getenv("FTB_TMA_TAIL_MIN");
    if (swap || d.N < (env_min ? std::atoi(env_min) : 16) || (env && env[0] == '0')) return 0;
    n_map = d.N & ~int64_t(7);
  }
  if (reinterpret_cast<uintptr_t>(d.C) % 16 || (d.ldc * 2) % 16) return 0;
  const int64_t bs = d.batch > 1 ? d.c_batch_stride : d.M * d.ldc;
  if ((bs * 2) % 16) return 0;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(n_map), static_cast<cuuint64_t>(d.M), static_cast<cuuint64_t>(d.batch)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(d.ldc * 2), static_cast<cuuint64_t>(bs * 2)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d.C, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 0;
  return n_map == d.N ? 1 : 2;
}

struct Region {
  int64_t lo[3], hi[3];  // per space axis (dense uses 2)
};

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Validate a program against its problem and enumerate the uKernel rectangles.
std::vector<Region> plan_regions(const ftb_gemm_desc& d, const ftb_program& g,
                                 int64_t* covered_out) {
  const int ns = d.op == FTB_OP_BMM ? 3 : 2;
  if (g.n_space != ns || g.n_reduce != 1)
    throw input_error("program axis counts do not match the operator", "program");
  if (g.tau < 0 || g.tau >= ns) throw input_error("program tau axis out of range", "tau");
  if (g.n_parts < 1 || g.n_parts > 2) throw input_error("program needs one or two parts", "parts");
  int64_t ext[3];
  if (ns == 3) {
    ext[0] = d.batch; ext[1] = d.M; ext[2] = d.N;
  } else {
    ext[0] = d.M; ext[1] = d.N;
  }
  for (int p = 0; p < g.n_parts; ++p) {
    for (int a = 0; a < ns + 1; ++a)
      if (g.smem[p][a] < 1) throw input_error("program tiles must be positive", "smem_tile");
    for (int a = 0; a < ns; ++a)
      if (g.reg[p][a] < 1 || g.smem[p][a] % g.reg[p][a])
        throw input_error("register tile does not divide shared-memory tile", "reg_tile");
    if (g.count[p] < 1) throw input_error("part counts must be >= 1", "count");
  }
  if (g.n_parts == 2)
    for (int a = 0; a < ns + 1; ++a)
      if (a != g.tau && g.smem[0][a] != g.smem[1][a])
        throw input_error("parts disagree on a non-tau tile (combine.py:118-123)", "parts");
  int64_t cover = 0;
  for (int p = 0; p < g.n_parts; ++p) cover += g.count[p] * g.smem[p][g.tau];
  if (cover != ext[g.tau])
    throw input_error("program does not cover the main axis exactly (combine.py:189-193)", "tau");

  std::vector<Region> out;
  int64_t covered = 1;
  for (int a = 0; a < ns; ++a)
    if (a != g.tau) covered *= round_up(ext[a], g.smem[0][a]);
  *covered_out = covered * ext[g.tau];

  int64_t off = 0;
  for (int p = 0; p < g.n_parts; ++p) {
    const int64_t t = g.smem[p][g.tau];
    for (int64_t c = 0; c < g.count[p]; ++c, off += t) {
      // odometer over the non-tau axes
      int64_t idx[3] = {0, 0, 0};
      int64_t nt[3];
      for (int a = 0; a < ns; ++a) nt[a] = (a == g.tau) ? 1 : ceil_div(ext[a], g.smem[p][a]);
      while (true) {
        Region r;
        for (int a = 0; a < ns; ++a) {
          if (a == g.tau) {
            r.lo[a] = off;
            r.hi[a] = off + t;
          } else {
            r.lo[a] = idx[a] * g.smem[p][a];
            r.hi[a] = std::min(ext[a], r.lo[a] + g.smem[p][a]);
          }
        }
        out.push_back(r);
        int a = ns - 1;
        for (; a >= 0; --a) {
          if (++idx[a] < nt[a]) break;
          idx[a] = 0;
        }
        if (a < 0) break;
      }
    }
  }
  return out;
}

struct Piece {
  int64_t start, len;
};
// Cut [lo, hi) into n = ceil(len / maxlen) near-equal pieces whose lengths
// are multiples of `align` (except the last). MN-major operands (B given as
// [K, N]) need align = 8: TMA rejects an innermost box coordinate that is not
// a multiple of 16 bytes (an unaligned piece start faults with an illegal
// instruction, tests/test_fuzz_gpu.py); maxlen is a multiple of 8.
void split(int64_t lo, int64_t hi, int64_t maxlen, std::vector<Piece>& out, int64_t align = 1) {
  out.clear();
  const int64_t len = hi - lo;
  const int64_t n = ceil_div(len, maxlen);
  const int64_t base = std::min(maxlen, round_up(ceil_div(len, n), align));
  for (int64_t s = lo; s < hi; s += base) out.push_back({s, std::min(base, hi - s)});
}

}  // namespace

// Per-device resources of the table allocator: tables live in the device's
// stream-ordered memory pool (cudaMallocAsync / cudaFreeAsync, pool kept
// resident), uploaded on a private non-blocking stream and released on
// another one after every launch that used them — no cudaMalloc, no
// synchronous cudaMemcpy and no cudaFree (each of which would synchronise the
// whole device) on the create / destroy path.
struct DeviceRes {
  cudaStream_t upload = nullptr;
  cudaStream_t reclaim = nullptr;
};
static DeviceRes& device_res(int dev) {
  static std::mutex mu;
  static DeviceRes res[64];
  std::lock_guard<std::mutex> g(mu);
  DeviceRes& r = res[dev & 63];
  if (!r.upload) {
    FTB_CUDA(cudaStreamCreateWithFlags(&r.upload, cudaStreamNonBlocking));
    FTB_CUDA(cudaStreamCreateWithFlags(&r.reclaim, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;  // freed tables stay in the pool for the next create
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  return r;
}

// Pinned staging for table uploads (per device): the table is copied into a
// reusable pinned chunk and sent with one cudaMemcpyAsync on the private
// upload stream; create returns without waiting for it (the first launch
// waits on the table's `ready` event on the device side). A chunk is reused
// once the copy that last read it has completed.
class PinnedPool {
 public:
  void upload(void* dst, const void* src, size_t n, cudaStream_t s) {
    Chunk* c = nullptr;
    {
      std::lock_guard<std::mutex> g(mu_);
      for (auto& ch : chunks_)
        if (!ch->busy && ch->cap >= n && (!ch->recorded || cudaEventQuery(ch->ev) == cudaSuccess)) {
          c = ch.get();
          break;
        }
      if (!c) {
        size_t cap = size_t(1) << 20;
        while (cap < n) cap <<= 1;
        auto ch = std::make_unique<Chunk>();
        FTB_CUDA(cudaHostAlloc(&ch->p, cap, cudaHostAllocPortable));
        FTB_CUDA(cudaEventCreateWithFlags(&ch->ev, cudaEventDisableTiming));
        ch->cap = cap;
        chunks_.push_back(std::move(ch));
        c = chunks_.back().get();
      }
      c->busy = true;
    }
    std::memcpy(c->p, src, n);
    cudaError_t e = cudaMemcpyAsync(dst, c->p, n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev, s);
    {
      std::lock_guard<std::mutex> g(mu_);
      c->recorded = c->recorded || e == cudaSuccess;
      c->busy = false;
    }
    if (e != cudaSuccess) throw cuda_error(std::string("table upload: ") + cudaGetErrorString(e));
  }

 private:
  struct Chunk {
    void* p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool busy = false, recorded = false;
  };
  std::mutex mu_;
  std::vector<std::unique_ptr<Chunk>> chunks_;
};
static PinnedPool& pinned_pool(int dev) {
  static PinnedPool pools[64];
  return pools[dev & 63];
}

// Host image of one table allocation: sections appended at 128-B offsets.
struct Blob {
  std::vector<uint8_t> bytes;
  size_t add(const void* src, size_t n) {
    const size_t off = (bytes.size() + 127) & ~static_cast<size_t>(127);
    bytes.resize(off + n);
    if (src && n) std::memcpy(bytes.data() + off, src, n);
    return off;
  }
};

struct ExecImpl {
  std::vector<DevProblem> problems;
  std::vector<DevMaps> maps;          // tcgen05: TMA descriptors per problem
  std::vector<DevWork> work;          // logical table (export format, FFMA input)
  DevProblem* d_problems = nullptr;
  DevWork* d_work = nullptr;
  DevMaps* d_maps = nullptr;
  std::vector<uint8_t> tma_out;       // per problem: C store map usable (1), or up to N8 only (2, kFlagTmaTail)
  std::vector<int32_t> pack_depth;    // per problem: batch entries per TMA box (1 = no packing)
  std::vector<int32_t> pack_rows;     // per problem: lane box rows when packed
  TcWork* d_tcwork = nullptr;
  TcPair* d_tcpairs = nullptr;
  float* d_split_ws = nullptr;        // split-K fp32 partials
  int32_t* d_split_cnt = nullptr;     // split-K chunk counters (self-resetting)
  unsigned long long* d_trace = nullptr;
  void* d_blob = nullptr;             // one pool allocation: every section above but the workspace
  int device = -1;
  double encode_ms = 0.0;             // host time spent encoding TMA descriptors (FTB_PROFILE_CREATE)
  bool ffma_vec = false;              // FFMA kernel: 16-B operand copies
  cudaEvent_t ready = nullptr;        // the table's upload has landed (recorded on the upload stream)
  bool ready_known = false;           // `ready` observed complete: launches need not wait for it
  bool captured = false;              // launched inside a stream capture: never freed (see ~ExecImpl)
  // streams this table was launched on, each with the event recorded after
  // its last launch: destroy frees only after all of them (stream order)
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> launched;
  cudaStream_t last_stream = nullptr;
  std::mutex mu;     // launches may come from several host threads
  TcConfig cfg{};    // single-CTA kernel (K1)
  TcConfig cfg2{};   // CTA-pair kernel (K1b)
  int64_t n_singles = 0, n_pairs = 0, ctas1 = 0, ctas2 = 0;
  ftb_exec_info info{};
  ~ExecImpl() {
    if (device < 0) {
      if (d_trace) cudaFree(d_trace);
      return;
    }
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    cudaStream_t rs = nullptr;
    try {
      rs = device_res(device).reclaim;
    } catch (...) {
    }
    if (ready) {
      if (rs) cudaStreamWaitEvent(rs, ready, 0);  // never free a table whose upload is in flight
      cudaEventDestroy(ready);
    }
    for (auto& se : launched) {
      if (rs) cudaStreamWaitEvent(rs, se.second, 0);
      cudaEventDestroy(se.second);  // the wait above captured its state
    }
    // A table that was launched inside a stream capture may still be replayed
    // by that CUDA graph after this handle is gone: its memory is deliberately
    // kept (not freed) so no graph can ever read a recycled table.
    if (rs && !captured) {
      if (d_blob) cudaFreeAsync(d_blob, rs);
      if (d_split_ws) cudaFreeAsync(d_split_ws, rs);
    }
    if (d_trace) cudaFree(d_trace);  // debug builds only (ftb_exec_set_trace)
    if (cur >= 0 && cur != device) cudaSetDevice(cur);
  }
};

static int device_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

static void build(ExecImpl& ex, const ftb_gemm_desc* probs, const ftb_program* progs, int32_t n,
                  bool encode) {
  if (n < 1) throw input_error("no problems given", "problems");
  const int32_t in_dt = probs[0].in_dtype;
  for (int32_t p = 0; p < n; ++p)
    if (probs[p].in_dtype != in_dt)
      throw input_error("all problems of one table must share the input dtype", "in_dtype");
  const bool ffma = in_dt == FTB_DT_F32;
  ex.info.kernel = ffma ? 1 : 0;
  std::vector<Piece> lp, cp;
  struct Keyed {
    int64_t cost;
    DevWork w;
  };
  std::vector<Keyed> items;
  static const bool prof_lower = std::getenv("FTB_PROFILE_LOWER") != nullptr;
  double t_regions = 0, t_items = 0, t_raster = 0;
  for (int32_t p = 0; p < n; ++p) {
    const ftb_gemm_desc& d = probs[p];
    if (d.M < 1 || d.N < 1 || d.K < 1 || d.batch < 1)
      throw input_error("problem extents must be >= 1", "shape");
    if (d.op == FTB_OP_DENSE && d.batch != 1) throw input_error("dense problems have batch 1", "batch");
    int64_t covered = 0;
    const auto tp0 = std::chrono::steady_clock::now();
    std::vector<Region> regs = plan_regions(d, progs[p], &covered);
    const auto tp1 = std::chrono::steady_clock::now();
    if (prof_lower) t_regions += std::chrono::duration<double, std::micro>(tp1 - tp0).count();
    const int ib = d.op == FTB_OP_BMM ? 1 : 0;  // index of i among space axes
    DevProblem P;
    std::memset(&P, 0, sizeof(P));
    P.A = d.A; P.B = d.B; P.C = d.C;
    P.lda = d.lda; P.ldb = d.ldb; P.ldc = d.ldc;
    P.a_bs = d.a_batch_stride; P.b_bs = d.b_batch_stride; P.c_bs = d.c_batch_stride;
    P.M = static_cast<int32_t>(d.M); P.N = static_cast<int32_t>(d.N);
    P.K = static_cast<int32_t>(d.K); P.batch = d.batch;
    P.out_f32 = d.out_dtype == FTB_DT_F32;
    P.b_nk = d.b_layout == FTB_B_NK;
    if (d.activation != FTB_ACT_NONE && d.activation != FTB_ACT_GELU)
      throw input_error("unknown activation", "activation");
    if ((d.bias || d.activation != FTB_ACT_NONE) && d.op != FTB_OP_DENSE)
      throw input_error("fused bias / activation epilogues are for Dense problems", "bias");
    if (d.bias && d.bias_dtype != FTB_DT_BF16 && d.bias_dtype != FTB_DT_F32)
      throw input_error("unsupported bias dtype", "bias_dtype");
    P.bias = d.bias;
    P.bias_f32 = d.bias_dtype == FTB_DT_F32;
    P.act = d.activation;
    P.num_kb = static_cast<int32_t>(ceil_div(d.K, kBlockK));
    if (ffma && !P.out_f32) throw input_error("FFMA mode writes fp32 outputs", "out_dtype");

    // Orientation: least tensor-pipe time — per 128-lane slab and column piece
    // an M=128 K=16 MMA costs max(kMmaFloorN, n_mma)/2 clk (B200 measurement,
    // scripts/micro/mma_bench.cu); ties to the normal orientation.
    int swap = 0;
    if (!ffma) {
      int64_t cost[2] = {0, 0};
      for (int o = 0; o < 2; ++o) {
        const bool col_mn = (o == 0) && !P.b_nk;
        const int64_t gran = col_mn ? 64 : 16;
        int64_t last_li = -1, last_lj = -1, last_cost = 0;  // consecutive regions usually share extents
        for (const Region& r : regs) {
          const int64_t li = r.hi[ib] - r.lo[ib], lj = r.hi[ib + 1] - r.lo[ib + 1];
          if (li != last_li || lj != last_lj) {
            const int64_t lane = o ? lj : li, col = o ? li : lj;
            split(0, col, kMaxN, cp);
            int64_t cols = 0;
            for (auto& c : cp) cols += std::max<int64_t>(kMmaFloorN, round_up(c.len, gran));
            last_li = li;
            last_lj = lj;
            last_cost = ceil_div(lane, kLaneRows) * cols;
          }
          cost[o] += last_cost;
        }
      }
      swap = d.orientation >= 0 ? d.orientation : (cost[1] < cost[0] ? 1 : 0);
      // A Dense with M <= 16 streams B once and is memory/latency bound, not
      // MMA bound: swap-AB loads 128 B rows + M A rows per K block instead of a
      // mostly out-of-bounds 128-row A box + 256 B rows (measured, C3 N=K=4096:
      // M=1 9.9 vs 11.8 us, M=16 10.1 vs 10.4 us)
      if (d.orientation < 0 && d.op == FTB_OP_DENSE && d.M <= 16) swap = 1;
    }
    P.swap = swap;
    P.lane_mn = swap && !P.b_nk;
    P.col_mn = !swap && !P.b_nk;
    if (!ffma && d.in_dtype != FTB_DT_BF16) throw input_error("unsupported input dtype", "in_dtype");
    // Block-diagonal batch packing for short attention BMMs: when every
    // batch entry is one work piece with M <= 64 rows and N <= 64 columns,
    // `depth` = 128 / lane_slot consecutive entries share one work item. One
    // 3-D TMA box per operand and K block stacks entry e's A rows at lanes
    // [e*lane_slot, ...) and its B rows at MMA columns [e*64, ...); a single
    // M=128, N=depth*64 MMA computes every entry's block (and the unused
    // off-diagonal blocks: a kind::f16 MMA costs ~100 clk whatever N <= 128
    // is, so one N=256 MMA replaces four N=64 ones at a third of the tensor
    // time), and each epilogue warp drains the diagonal block in its TMEM lane
    // quadrant. The box's third dimension is the batch; rows/columns past M,
    // N and past the last batch entry are zero-filled by TMA.
    int32_t depth = 1, lrows = 0;
    if (!ffma && d.op == FTB_OP_BMM && !swap && !P.lane_mn && d.M <= 64 && d.N <= 64) {
      bool one_piece = true;
      for (const Region& r : regs)
        if (r.hi[ib] - r.lo[ib] != d.M || r.hi[ib + 1] - r.lo[ib + 1] != d.N) one_piece = false;
      const int32_t slot_rows = d.M <= 32 ? 32 : 64;
      const int32_t nb = std::min<int32_t>(kLaneRows / slot_rows, d.batch);
      if (one_piece && nb >= 2 && d.c_batch_stride < (int64_t(1) << 31) && !std::getenv("FTB_NO_PACK")) {
        depth = kLaneRows / slot_rows;
        lrows = slot_rows;
      }
    }
    ex.pack_depth.push_back(depth);
    ex.pack_rows.push_back(lrows);
    if (!ffma && encode) {
      const auto te0 = std::chrono::steady_clock::now();
      // A: [batch][M][lda], K contiguous. B: [batch][N][ldb] (NK) or [batch][K][ldb] (KN).
      DevMaps m;
      std::memset(&m, 0, sizeof(m));
      const void* lane_t = swap ? d.B : d.A;
      const void* col_t = swap ? d.A : d.B;
      const int64_t lane_rows = swap ? d.N : d.M, col_rows = swap ? d.M : d.N;
      const int64_t lane_ld = swap ? d.ldb : d.lda, col_ld = swap ? d.lda : d.ldb;
      const int64_t lane_bs = swap ? d.b_batch_stride : d.a_batch_stride;
      const int64_t col_bs = swap ? d.a_batch_stride : d.b_batch_stride;
      if (depth > 1) {  // packed: one box per operand and K block covers `depth` batch entries
        encode_map(&m.lane, lane_t, d.K, lane_rows, d.batch, lane_ld, lane_bs, 64, lrows, depth);
        if (!P.col_mn)
          encode_map(&m.col[0], col_t, d.K, col_rows, d.batch, col_ld, col_bs, 64, 64, depth);
        else
          encode_map(&m.col[0], col_t, col_rows, d.K, d.batch, col_ld, col_bs, 64, 64, depth);
      } else if (!P.lane_mn) {
        encode_map(&m.lane, lane_t, d.K, lane_rows, d.batch, lane_ld, lane_bs, 64, kLaneRows);
      } else {
        encode_map(&m.lane, lane_t, lane_rows, d.K, d.batch, lane_ld, lane_bs, 64, 64);
      }
      if (depth == 1) {
        if (!P.col_mn) {
          for (int q = 0; q < kColMaps; ++q)
            encode_map(&m.col[q], col_t, d.K, col_rows, d.batch, col_ld, col_bs, 64, 256u >> q);
        } else {
          encode_map(&m.col[0], col_t, col_rows, d.K, d.batch, col_ld, col_bs, 64, 64);
        }
      }
      ex.tma_out.push_back(static_cast<uint8_t>(encode_out_map(&m.out, d, swap)));
      m.epi.bias = d.bias;
      m.epi.bias_f32 = d.bias_dtype == FTB_DT_F32;
      m.epi.act = d.activation;
      m.epi.n = static_cast<int32_t>(d.N);
      m.epi.pad_ = 0;
      ex.maps.push_back(m);
      ex.encode_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - te0).count();
    }
    ex.problems.push_back(P);

    const int64_t lane_max = ffma ? 64 : kLaneRows;
    const int64_t col_max = ffma ? 64 : kMaxN;
    const int64_t gran = P.col_mn ? 64 : 16;
    const size_t first_item = items.size();
    if (ffma) {
      // FFMA items are unions of whole uKernel rectangles. The plan's
      // rectangles form a grid (the parts share every non-tau tile,
      // combine.py:118-123): i cells x j cells per batch entry. Consecutive
      // cells are merged along each axis up to the kernel's 64 x 64 CTA tile
      // (a cell larger than 64 is cut as before), so the small uKernels the
      // FFMA descriptor picks (C0: 3 x 32 ... 30 x 32) no longer leave most of
      // a CTA's 256 threads idle; every output element is still one
      // sequential-K FFMA chain, so the result is bit-identical.
      auto cuts = [&](int ax, int64_t extent) {
        std::vector<int64_t> c;
        for (const Region& r : regs) c.push_back(r.lo[ax]);
        c.push_back(extent);
        std::sort(c.begin(), c.end());
        c.erase(std::unique(c.begin(), c.end()), c.end());
        return c;
      };
      auto group = [&](const std::vector<int64_t>& c, int64_t maxlen, std::vector<Piece>& out) {
        out.clear();
        std::vector<Piece> tmp;
        int64_t gs = c.front(), gl = 0;
        for (size_t k = 0; k + 1 < c.size(); ++k) {
          const int64_t len = c[k + 1] - c[k];
          if (len > maxlen) {
            if (gl) out.push_back({gs, gl});
            split(c[k], c[k + 1], maxlen, tmp, 1);
            out.insert(out.end(), tmp.begin(), tmp.end());
            gs = c[k + 1];
            gl = 0;
            continue;
          }
          if (gl + len > maxlen) {
            out.push_back({gs, gl});
            gs = c[k];
            gl = 0;
          }
          gl += len;
        }
        if (gl) out.push_back({gs, gl});
      };
      group(cuts(ib, d.M), lane_max, lp);
      group(cuts(ib + 1, d.N), col_max, cp);
      for (int64_t b = 0; b < (ib ? d.batch : 1); ++b)
        for (auto& L : lp)
          for (auto& Cc : cp) {
            DevWork w;
            w.problem = p;
            w.batch = static_cast<int32_t>(b);
            w.lane0 = static_cast<int32_t>(L.start);
            w.col0 = static_cast<int32_t>(Cc.start);
            w.lane_len = static_cast<int32_t>(L.len);
            w.col_len = static_cast<int32_t>(Cc.len);
            w.n_mma = static_cast<int32_t>(Cc.len);
            w.aux = 0;
            const int64_t cells = static_cast<int64_t>(P.num_kb) * L.len * Cc.len;
            items.push_back({cells, w});
            ex.info.mma_flops += 2 * cells * kBlockK;
          }
    }
    int64_t last_ilo = -1, last_ihi = -1, last_jlo = -1, last_jhi = -1;
    for (const Region& r : regs) {
      if (ffma) break;
      const int64_t b0 = ib ? r.lo[0] : 0, b1 = ib ? r.hi[0] : 1;
      const int64_t ilo = r.lo[ib], ihi = r.hi[ib], jlo = r.lo[ib + 1], jhi = r.hi[ib + 1];
      // j is C's innermost dimension (and B's when B is [K, N]): pieces along
      // j start on multiples of 8 elements so TMA store (and MN-major load)
      // boxes have 16-byte origins
      if (swap) {
        split(jlo, jhi, lane_max, lp, 8);
        split(ilo, ihi, col_max, cp, 1);
      } else if (ilo == last_ilo && ihi == last_ihi && jlo == last_jlo && jhi == last_jhi) {
        // the same rectangle as the previous region (another batch entry): reuse its pieces
      } else {
        split(ilo, ihi, lane_max, lp, 1);
        split(jlo, jhi, col_max, cp, 8);
      }
      if (!swap) {
        last_ilo = ilo;
        last_ihi = ihi;
        last_jlo = jlo;
        last_jhi = jhi;
      }
      if ((P.lane_mn && lp.front().start % 8) || (P.col_mn && cp.front().start % 8))
        throw input_error("B given as [K, N] needs uKernel tiles along N that start on multiples of 8 "
                          "(TMA 16-byte box origin); pass B as [N, K] (b_layout nk)", "smem_tile");
      for (int64_t b = b0; b < b1; ++b)
        for (auto& L : lp)
          for (auto& Cc : cp) {
            DevWork w;
            w.problem = p;
            w.batch = static_cast<int32_t>(b);
            w.lane0 = static_cast<int32_t>(L.start);
            w.col0 = static_cast<int32_t>(Cc.start);
            w.lane_len = static_cast<int32_t>(L.len);
            w.col_len = static_cast<int32_t>(Cc.len);
            w.n_mma = ffma ? static_cast<int32_t>(Cc.len) : static_cast<int32_t>(round_up(Cc.len, gran));
            w.aux = 0;
            const int64_t cells = static_cast<int64_t>(P.num_kb) * (ffma ? L.len : kLaneRows) * w.n_mma;
            const int64_t cost = ffma ? cells : static_cast<int64_t>(P.num_kb) * std::max<int32_t>(kMmaFloorN, w.n_mma);
            items.push_back({cost, w});
            ex.info.mma_flops += 2 * cells * kBlockK;
          }
    }
    // Rasterise this problem's items for L2 locality: the persistent CTAs run a
    // window of ~one item per SM at a time, so order items by column group
    // (about 32 MiB of the column operand over K), then lane range, then
    // column: a group's column tiles stay L2-resident while the lane tiles
    // stream past once per group. Measured on 8192^3: row-major order read
    // 2.05 GB from DRAM for 0.26 GB of inputs; 32 MiB groups: 1.02 GB, sustained
    // 1065 -> 1232 TF/s (the power-capped clock rises with less DRAM traffic).
    if (!ffma) {
      const int64_t kbytes = std::max<int64_t>(1, d.K * 2);
      static const int64_t raster_mb = [] {
        const char* e = std::getenv("FTB_RASTER_MB");
        return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(32);
      }();
      const int64_t group = std::max<int64_t>(kMaxN, (raster_mb << 20) / kbytes / kMaxN * kMaxN);
      auto raster = [group](const Keyed& a, const Keyed& b) {
        if (a.w.batch != b.w.batch) return a.w.batch < b.w.batch;
        const int64_t ga = a.w.col0 / group, gb = b.w.col0 / group;
        if (ga != gb) return ga < gb;
        // snake: odd groups sweep the lanes backwards, starting on the lane
        // tiles the previous group left in L2
        if (a.w.lane0 != b.w.lane0) return (ga & 1) ? a.w.lane0 > b.w.lane0 : a.w.lane0 < b.w.lane0;
        return a.w.col0 < b.w.col0;
      };
      // (batched attention problems are generated in this order already)
      const auto tr0 = std::chrono::steady_clock::now();
      if (prof_lower) t_items += std::chrono::duration<double, std::micro>(tr0 - tp1).count();
      if (!std::is_sorted(items.begin() + first_item, items.end(), raster))
        std::stable_sort(items.begin() + first_item, items.end(), raster);
      if (prof_lower) t_raster += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tr0).count();
    }
    ex.info.true_flops += 2 * d.batch * d.M * d.N * d.K;
    ex.info.covered_out += covered;
    ex.info.true_out += d.batch * d.M * d.N;
  }
  const auto ts0 = std::chrono::steady_clock::now();
  // Longest-first order so the static round-robin over persistent CTAs
  // balances. Costs take few distinct values (K blocks x MMA width), so the
  // stable order is a counting sort over the distinct costs (O(n), the
  // comparison sort of 35k items was the largest host cost of a C1 table).
  {
    std::vector<int64_t> keys;
    keys.reserve(64);
    for (const Keyed& k : items)
      if (keys.empty() || keys.back() != k.cost) keys.push_back(k.cost);  // runs of equal cost collapse
    std::sort(keys.begin(), keys.end(), std::greater<int64_t>());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    std::vector<int64_t> start(keys.size() + 1, 0);
    std::vector<uint32_t> bucket(items.size());
    for (size_t i = 0; i < items.size(); ++i) {
      const size_t b = static_cast<size_t>(
          std::lower_bound(keys.begin(), keys.end(), items[i].cost, std::greater<int64_t>()) - keys.begin());
      bucket[i] = static_cast<uint32_t>(b);
      ++start[b + 1];
    }
    for (size_t b = 0; b < keys.size(); ++b) start[b + 1] += start[b];
    ex.work.resize(items.size());
    for (size_t i = 0; i < items.size(); ++i) ex.work[static_cast<size_t>(start[bucket[i]]++)] = items[i].w;
  }
  if (prof_lower)
    std::fprintf(stderr, "ftb lower: regions %.0f us, items %.0f us, raster %.0f us, cost order %.0f us (%zu items)\n",
                 t_regions, t_items, t_raster,
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - ts0).count(), items.size());
  ex.info.n_work = static_cast<int64_t>(ex.work.size());
  ex.info.n_problems = n;
  int sms = device_sms();
  if (sms <= 0) sms = 148;
  ex.info.n_ctas = std::min<int64_t>(ex.info.n_work, ffma ? 4 * sms : sms);
  if (ffma) {  // the FFMA kernel's 16-B copies need 16-B aligned operand rows (and item column origins)
    bool vec = true;
    for (const DevProblem& P : ex.problems)
      vec = vec && reinterpret_cast<uintptr_t>(P.A) % 16 == 0 && reinterpret_cast<uintptr_t>(P.B) % 16 == 0 &&
            P.lda % 4 == 0 && P.ldb % 4 == 0 && (P.batch == 1 || (P.a_bs % 4 == 0 && P.b_bs % 4 == 0));
    for (const DevWork& w : ex.work) vec = vec && w.col0 % 4 == 0;
    ex.ffma_vec = vec;
  }
  if (ex.info.n_work > INT32_MAX) throw input_error("tile table too large", "work");
}

// Device upload: problems (FFMA) or TMA descriptors + self-contained items
// (tcgen05), and the per-launch pipeline shape from the widest item.
static void upload(ExecImpl& I) {
  FTB_CUDA(cudaGetDevice(&I.device));
  const cudaStream_t us = device_res(I.device).upload;
  // one pool allocation for the whole table, filled by one async copy (from a
  // pinned staging chunk) on the private upload stream; create does not wait
  // for it — the first launch on a stream waits for `ready` on the device
  // the table is ready on the device when `ready` (recorded on the upload
  // stream after its copy) has fired; launches wait for it device-side
  auto send = [&](Blob& b) {
    pinned_pool(I.device).upload(I.d_blob, b.bytes.data(), b.bytes.size(), us);
    FTB_CUDA(cudaEventCreateWithFlags(&I.ready, cudaEventDisableTiming));
    FTB_CUDA(cudaEventRecord(I.ready, us));
  };
  auto commit = [&](Blob& b) {
    FTB_CUDA(cudaMallocAsync(&I.d_blob, std::max<size_t>(b.bytes.size(), 128), us));
    send(b);
  };
  auto at = [&](size_t off) { return static_cast<uint8_t*>(I.d_blob) + off; };
  if (I.work.empty() || I.info.kernel == 1) {
    Blob b;
    const size_t op = b.add(I.problems.data(), sizeof(DevProblem) * I.problems.size());
    const size_t ow = b.add(I.work.data(), sizeof(DevWork) * I.work.size());
    commit(b);
    I.d_problems = reinterpret_cast<DevProblem*>(at(op));
    I.d_work = reinterpret_cast<DevWork*>(at(ow));
    return;
  }
  // work records reference their problem's descriptors by device address;
  // until the allocation exists they carry the problem index (fixed up below)
  auto maps_of = [](int32_t problem) {
    return reinterpret_cast<const DevMaps*>(static_cast<uintptr_t>(problem));
  };
  auto flags_of = [](const DevProblem& P) {
    return (P.swap ? kFlagSwap : 0u) | (P.lane_mn ? kFlagLaneMN : 0u) | (P.col_mn ? kFlagColMN : 0u) |
           (P.out_f32 ? kFlagOutF32 : 0u) | ((P.bias || P.act) ? kFlagEpiOp : 0u);
  };
  auto c_of = [](const DevProblem& P, int32_t batch) {
    const size_t esz = P.out_f32 ? 4 : 2;
    return static_cast<void*>(static_cast<char*>(P.C) + static_cast<int64_t>(batch) * P.c_bs * esz);
  };
  // TMA stores write whole 32 x 32 boxes: legal for a rectangle whose extents
  // are multiples of 32 or that ends at the tensor edge (the hardware clips).
  const char* env_ts = std::getenv("FTB_TMA_STORE");
  const bool tma_store_on = !(env_ts && env_ts[0] == '0');
  auto tma_ok = [&](const DevWork& w) {
    const DevProblem& P = I.problems[w.problem];
    const int32_t lane_ext = P.swap ? P.N : P.M, col_ext = P.swap ? P.M : P.N;
    // ... and the box origin along C's innermost dimension (j) is 16-byte aligned
    const int32_t j0 = P.swap ? w.lane0 : w.col0;
    return tma_store_on && I.tma_out[w.problem] && j0 % 8 == 0 &&
           (w.lane_len % 32 == 0 || w.lane0 + w.lane_len == lane_ext) &&
           (w.col_len % 32 == 0 || w.col0 + w.col_len == col_ext);
  };
  // Contiguous rows (kFlagBulkStore): whole rows of a compact C, normal
  // orientation, where TMA stores are not legal.
  const char* env_bs = std::getenv("FTB_BULK_STORE");
  const bool bulk_store_on = !(env_bs && env_bs[0] == '0');
  auto bulk_ok = [&](const DevWork& w) {
    const DevProblem& P = I.problems[w.problem];
    return bulk_store_on && !P.swap && P.ldc == P.N && w.col0 == 0 && w.col_len == P.N;
  };
  auto store_flag = [&](bool tma, const DevWork& w) {
    if (tma) {
      const DevProblem& P = I.problems[w.problem];
      const bool tail = I.tma_out[w.problem] == 2 && w.col0 + w.col_len == P.N;  // ends in the unmapped columns
      return kFlagTmaStore | (tail ? kFlagTmaTail : 0u);
    }
    return bulk_ok(w) ? kFlagBulkStore : 0u;
  };
  // CTA pairs: logical items of one problem/batch with the same column range
  // share the column operand; group them (in cost order) two by two. Off by
  // default: measured on B200 the pair kernel loses to the single-CTA kernel
  // with TMA-store epilogues on every C1 shape (profiles/r1b_*); FTB_PAIR=1
  // enables it.
  const char* env = std::getenv("FTB_PAIR");
  const bool pairing = env && env[0] == '1';
  std::vector<int8_t> paired(I.work.size(), 0);
  std::vector<TcPair> pairs;
  if (pairing) {
    std::map<std::array<int32_t, 4>, int64_t> open;  // key -> first unpaired item
    for (size_t i = 0; i < I.work.size(); ++i) {
      const DevWork& w = I.work[i];
      const std::array<int32_t, 4> key{w.problem, w.batch, w.col0, w.col_len};
      auto it = open.find(key);
      if (it == open.end()) {
        open.emplace(key, static_cast<int64_t>(i));
        continue;
      }
      const DevWork& a = I.work[it->second];
      const DevProblem& P = I.problems[w.problem];
      TcPair t;
      std::memset(&t, 0, sizeof(t));
      t.maps = maps_of(w.problem);
      t.C = c_of(P, w.batch);
      t.ldc = P.ldc;
      t.lane0[0] = a.lane0;
      t.lane_len[0] = a.lane_len;
      t.lane0[1] = w.lane0;
      t.lane_len[1] = w.lane_len;
      t.col0 = w.col0;
      t.col_len = w.col_len;
      t.n_mma = static_cast<int32_t>(round_up(w.col_len, P.col_mn ? 128 : 32));
      t.num_kb = P.num_kb;
      t.batch = w.batch;
      t.flags = flags_of(P) | (tma_ok(a) && tma_ok(w) && I.tma_out[w.problem] == 1 ? kFlagTmaStore : 0u);
      pairs.push_back(t);
      paired[it->second] = paired[i] = 1;
      open.erase(it);
    }
  }
  std::vector<TcWork> tw;
  int32_t split_tiles = 0;  // tiles whose split-K partials meet in the global workspace
  int max_n = 16;
  for (size_t i = 0; i < I.work.size(); ++i) {
    if (paired[i]) continue;
    const DevWork& w = I.work[i];
    const DevProblem& P = I.problems[w.problem];
    const int32_t depth = I.pack_depth[w.problem];
    if (depth > 1) {
      // consecutive entries of the same piece shape -> one packed item
      size_t j = i + 1;
      while (j < I.work.size() && static_cast<int32_t>(j - i) < depth) {
        const DevWork& u = I.work[j];
        if (paired[j] || u.problem != w.problem || u.batch != w.batch + static_cast<int32_t>(j - i) ||
            u.lane0 != w.lane0 || u.col0 != w.col0 || u.lane_len != w.lane_len || u.col_len != w.col_len)
          break;
        ++j;
      }
      const int32_t nb = static_cast<int32_t>(j - i);
      bool ok = true;
      for (size_t q = i; q < j; ++q) ok = ok && tma_ok(I.work[q]);
      TcWork t;
      std::memset(&t, 0, sizeof(t));
      t.maps = maps_of(w.problem);
      t.C = c_of(P, w.batch);
      t.ldc = P.ldc;
      t.lane0 = w.lane0;
      t.col0 = w.col0;
      t.lane_len = w.lane_len;
      t.col_len = w.col_len;
      t.n_mma = depth * 64;  // the whole stacked MMA (entry e in columns [64e, 64e + 64))
      t.num_kb = P.num_kb;
      t.batch = w.batch;
      t.flags = flags_of(P) | store_flag(ok, w);
      t.pack = static_cast<uint32_t>(nb) | (static_cast<uint32_t>(depth) << 8) |
               (static_cast<uint32_t>(I.pack_rows[w.problem]) << 16);
      t.c_bs = static_cast<int32_t>(P.c_bs);
      max_n = std::max(max_n, t.n_mma);
      tw.push_back(t);
      i = j - 1;
      continue;
    }
    TcWork t;
    std::memset(&t, 0, sizeof(t));
    t.maps = maps_of(w.problem);
    t.C = c_of(P, w.batch);
    t.ldc = P.ldc;
    t.lane0 = w.lane0;
    t.col0 = w.col0;
    t.lane_len = w.lane_len;
    t.col_len = w.col_len;
    t.n_mma = w.n_mma;
    t.num_kb = P.num_kb;
    t.batch = w.batch;
    t.flags = flags_of(P) | store_flag(tma_ok(w), w);
    max_n = std::max(max_n, w.n_mma);
    tw.push_back(t);
  }
  // Split-K: a table too small to occupy the SMs (e.g. one skinny Dense, or a
  // mid-size shape timed alone) splits each plain item's K blocks over up to
  // kMaxSplit items; partials meet in an fp32 workspace and the last split to
  // publish each 32-column chunk reduces and stores it (kernel_tc.cu). Tables that
  // already fill the GPU (the grouped C1 step) are left alone.
  // Wide on-chip split-K: a table that fills at most half the SMs with
  // long-K items (e.g. one C1 Dense timed alone: 15-36 128 x 256 tiles of
  // 12-48 K blocks) runs one wave whose length is one item's whole K loop.
  // Splitting every item's K range 4 (or 2) ways into a cluster of that many
  // CTAs keeps the full 256-column MMA (the cheapest per FLOP) and cuts the
  // wave to a quarter (half) of the K loop; the splits' fp32 partials (up to
  // 128 KiB, parked in each CTA's idle operand ring) are reduced through
  // distributed shared memory (kernel_tc.cu cluster_reduce). Needs every
  // item splittable (>= FTB_SPLIT_CL_MINKB K blocks per split, default 3)
  // and the table within the co-resident clusters (measured: 33 clusters of
  // 4, 74 of 2, scripts/micro/cluster_occ.cu). OPT-IN (FTB_SPLIT_WIDE_CLUSTER=1):
  // measured on B200 it LOSES — C1 out M=608 6.3 -> 11.8 us, FFN2 M=1024
  // 13.5 -> 15.7 us (profiles/r2g_wide_cluster_split_chain_time.txt): parking a 128 x 256 fp32
  // partial in smem takes ~1.5 us and the DSMEM pull reduction ~7 us
  // (scripts/chain_trace.py), far more than the K blocks it parallelises.
  bool wide_split = false;
  {
    int sms_here = device_sms();
    if (sms_here <= 0) sms_here = 148;
    const char* env_w = std::getenv("FTB_SPLIT_WIDE_CLUSTER");
    const char* env_sk = std::getenv("FTB_SPLITK");
    const char* env_cl = std::getenv("FTB_SPLIT_CLUSTER");
    const bool on = (env_w && env_w[0] == '1') && !(env_sk && env_sk[0] == '0') && !(env_cl && env_cl[0] == '0') &&
                    !pairing;
    const char* env_mk = std::getenv("FTB_SPLIT_CL_MINKB");
    const int cl_min = env_mk ? std::max(1, std::atoi(env_mk)) : 3;
    const int64_t n = static_cast<int64_t>(tw.size());
    if (on && n > 0 && n * 2 <= sms_here) {
      for (int cand : {4, 2}) {
        const int64_t cap = std::min<int64_t>(cand == 4 ? 132 : 148, sms_here);
        if (n * cand > cap) continue;
        bool ok = true;
        for (const TcWork& t : tw) ok = ok && !t.pack && t.num_kb >= cand * cl_min;
        if (!ok) continue;
        std::vector<TcWork> split;
        split.reserve(n * cand);
        for (const TcWork& t : tw)
          for (int q = 0; q < cand; ++q) {
            TcWork u = t;
            const int kb0 = static_cast<int>(static_cast<int64_t>(t.num_kb) * q / cand);
            const int kb1 = static_cast<int>(static_cast<int64_t>(t.num_kb) * (q + 1) / cand);
            u.num_kb = kb1 - kb0;
            u.flags |= kFlagSplitK;
            u.pack = static_cast<uint32_t>(kb0) | (static_cast<uint32_t>(cand) << 16) | (static_cast<uint32_t>(q) << 24);
            u.c_bs = 0;
            split.push_back(u);
          }
        I.cfg.cluster_split = cand;
        tw.swap(split);
        wide_split = true;
        break;
      }
    }
  }
  // Split-K decision for a candidate table (used by the column split below to
  // compare lowerings, and by the split-K pass): {split factor, on chip}.
  // On-chip (cluster) mode when every item splits the same way (s = 4 or 2,
  // >= split_min_kb K blocks per split) and the table fits the co-resident
  // clusters (measured: 33 clusters of 4, 74 of 2 at ~200 KiB smem per CTA,
  // scripts/micro/cluster_occ.cu); else the global-workspace path, narrow
  // items only.
  const char* env_sk = std::getenv("FTB_SPLITK");
  const bool split_on = !(env_sk && env_sk[0] == '0') && !pairing;
  const char* env_mk = std::getenv("FTB_SPLIT_MINKB");
  const int split_min_kb = env_mk ? std::max(1, std::atoi(env_mk)) : 8;
  const char* env_sw = std::getenv("FTB_SPLIT_WIDE");
  const bool split_wide = env_sw && env_sw[0] == '1';
  const char* env_scl = std::getenv("FTB_SPLIT_CLUSTER");
  const bool cluster_on = !(env_scl && env_scl[0] == '0');
  const int sms_all = device_sms() > 0 ? device_sms() : 148;
  auto split_choice = [&](const std::vector<TcWork>& v) -> std::pair<int, bool> {
    const int64_t n = static_cast<int64_t>(v.size());
    if (wide_split || !split_on || n == 0 || n * 2 > sms_all) return {1, false};
    const int target = static_cast<int>(std::min<int64_t>(kMaxSplit, sms_all / n));
    if (cluster_on)
      for (int cand : {4, 2}) {
        if (cand > target) continue;
        bool ok = true;
        for (const TcWork& t : v) ok = ok && !t.pack && t.n_mma <= 128 && t.num_kb / split_min_kb >= cand;
        if (ok && n * cand <= std::min(cand == 4 ? 132 : 148, sms_all)) return {cand, true};
      }
    int s_glob = 1;
    for (const TcWork& t : v)
      if (!t.pack && (t.n_mma <= 128 || split_wide)) s_glob = std::max(s_glob, std::min(target, t.num_kb / split_min_kb));
    return {s_glob, false};
  };
  // Column split: a table with fewer than half as many items as SMs runs one
  // wave whose length is one item's K loop; a 256-column item's K block costs
  // ~550 clk (smem-port bound: 48 KiB TMA write + 48 KiB MMA read), a
  // 128-column one ~350 clk. Halving wide items along the column axis
  // shortens the wave without changing any output bit (same per-element
  // K order).
  {
    int sms_here = device_sms();
    if (sms_here <= 0) sms_here = 148;
    const char* env_cs = std::getenv("FTB_COLSPLIT");
    const bool cs_on = !(env_cs && env_cs[0] == '0') && !pairing;
    const char* env_cw = std::getenv("FTB_COLSPLIT_MIN");
    const int min_w = env_cw ? std::max(32, std::atoi(env_cw)) : 32;  // narrowest piece
    // Halve while the table still fits one wave: 256 -> 128 columns, then
    // 128 -> 64 -> 32 (K-major column operands). Narrow pieces cost little MMA time
    // in a one-wave table (a K block's MMA floor is ~400 clk at N = 64 vs
    // ~460 at N = 128) and halve each SM's share of the output, whose TMA
    // stores leave an SM at ~20-30 B/clk (scripts/micro/store_bench.cu):
    // measured C1 out M=608 6.41 -> 6.03 us, qkv M=160 6.69 -> 6.14, FFN2
    // M=768 15.0 -> 12.3 (profiles/r2au_colsplit64.txt). Not when it would
    // lower the table's split-K factor: a K split halves every CTA's K loop,
    // a column split does not (FFN2 M=800: 12.7 -> 15.6 us, M=352: 9.8 ->
    // 10.4, profiles/r2ax_splitk_colsplit.txt).
    for (int level = 0; level < 3 && !wide_split && cs_on; ++level) {
      auto splittable = [&](const TcWork& t) {
        if (t.pack || t.n_mma <= min_w || t.col_len <= min_w) return false;
        return t.n_mma > 128 || !(t.flags & kFlagColMN);  // MN-major operands: 64-column boxes, n_mma >= 128
      };
      int64_t wide = 0;
      bool to32 = false;
      for (const TcWork& t : tw)
        if (splittable(t)) {
          ++wide;
          to32 = to32 || t.n_mma <= 64;
        }
      // 32-column pieces only while the table stays within half the SMs
      // (measured: out M=352 5.95 -> 5.76 us at 72 CTAs, M=608 6.02 -> 6.23
      // at 120; profiles/r2az_colsplit32.txt)
      const int64_t cap = to32 ? sms_here / 2 : sms_here;
      if (wide == 0 || static_cast<int64_t>(tw.size()) + wide > cap) break;
      std::vector<TcWork> cs;
      cs.reserve(tw.size() + wide);
      for (const TcWork& t : tw) {
        if (!splittable(t)) {
          cs.push_back(t);
          continue;
        }
        const bool col_mn = (t.flags & kFlagColMN) != 0;
        const int half = t.n_mma > 128 ? 128 : static_cast<int>(round_up((t.col_len + 1) / 2, 32));
        TcWork a = t, b = t;
        a.flags &= ~(kFlagBulkStore | kFlagTmaTail);  // pieces no longer cover whole rows; only b ends at N
        b.flags &= ~kFlagBulkStore;
        a.col_len = half;
        a.n_mma = t.n_mma > 128 ? 128 : half;
        b.col0 = t.col0 + half;
        b.col_len = t.col_len - half;
        b.n_mma = static_cast<int32_t>(round_up(b.col_len, col_mn ? 128 : 32));
        cs.push_back(a);
        cs.push_back(b);
      }
      const int s_new = split_choice(cs).first;
      if (s_new < split_choice(tw).first) break;
      if (to32 && static_cast<int64_t>(cs.size()) * s_new > cap) break;  // CTAs after split-K (FFN2 M=160: 8.9 -> 9.3 us at 120)
      tw.swap(cs);
      max_n = 16;
      for (const TcWork& t : tw) max_n = std::max(max_n, t.n_mma);
    }
  }
  {
    const int sms_here = sms_all;
    const int64_t n_items = static_cast<int64_t>(tw.size());
    if (!wide_split && split_on && n_items > 0 && n_items * 2 <= sms_here) {
      const int target = static_cast<int>(std::min<int64_t>(kMaxSplit, sms_here / n_items));
      // on chip whenever the table qualifies: round 2 measured the workspace
      // path 3-5 us slower than a cluster split of the same table even at
      // half the split count (FFN2 M=160 cluster-4 9.4 vs workspace 14.2 us,
      // M=768 cluster-2 vs workspace-4, profiles/r2ax_splitk_colsplit.txt)
      const std::pair<int, bool> sc = split_choice(tw);
      const int s_cl = sc.second ? sc.first : 0;
      std::vector<TcWork> split;
      int32_t tiles = 0;
      for (const TcWork& t : tw) {
        // >= 8 K blocks per split, and only narrow tiles: the fp32 partial
        // round trip (128 x n_mma x 8 B) must stay small next to the operand
        // bytes a split saves (measured: C3 M<=127 22 -> 18 us, M=256 n=256
        // tiles 23 -> 28 us when split)
        const int s_t = s_cl ? s_cl : ((t.n_mma <= 128 || split_wide) ? std::min(target, t.num_kb / split_min_kb) : 1);
        if (t.pack || s_t < 2) {
          split.push_back(t);
          continue;
        }
        const int32_t tile = tiles++;
        for (int q = 0; q < s_t; ++q) {
          TcWork u = t;
          const int kb0 = static_cast<int>(static_cast<int64_t>(t.num_kb) * q / s_t);
          const int kb1 = static_cast<int>(static_cast<int64_t>(t.num_kb) * (q + 1) / s_t);
          u.num_kb = kb1 - kb0;
          u.flags |= kFlagSplitK;
          u.pack = static_cast<uint32_t>(kb0) | (static_cast<uint32_t>(s_t) << 16) |
                   (static_cast<uint32_t>(q) << 24);
          u.c_bs = tile;
          split.push_back(u);
        }
      }
      // one wave (<= one item per SM) keeps a tile's splits concurrent so the
      // per-chunk reductions spread over them; correctness does not depend on
      // it (the last split to publish a chunk reduces it, nobody waits)
      if (tiles > 0 && s_cl) {
        I.cfg.cluster_split = s_cl;  // partials stay on chip: no workspace
        tw.swap(split);
      } else if (tiles > 0 && static_cast<int64_t>(split.size()) <= sms_here) {
        FTB_CUDA(cudaMallocAsync(&I.d_split_ws, sizeof(float) * static_cast<size_t>(tiles) * kSplitTileFloats, us));
        split_tiles = tiles;
        tw.swap(split);
      }
    }
  }
  // Overflow split: a table of n > P plain items (P = SMs) whose last round
  // holds only r = n mod P <= P / 2 items runs that round on r CTAs, so a 5 %
  // larger shape can take 40 % longer (C1 qkv M = 2048: 144 items 10.0 us,
  // M = 2144: 153 items 13.8 us). The r cheapest items (the table is
  // cost-sorted, they are last) are cut into 64-column pieces (128 when
  // 4r > P), which the round-robin deals to the first CTAs after their full
  // items: the last round shrinks to a narrow item's K loop (M = 2144: 11.1
  // us; qkv M = 2496 / 2592, FFN1 M = 1728-2144: -11 to -17 %,
  // profiles/r2bh_overflow_split.txt). Same per-element K order: bit-identical.
  {
    const char* env_ov = std::getenv("FTB_OVERFLOW_SPLIT");
    const int64_t n = static_cast<int64_t>(tw.size()), P = sms_all;
    const int64_t r = n > P ? n % P : 0;  // items of the last, partial round
    bool ok = !(env_ov && env_ov[0] == '0') && !wide_split && !pairing && I.cfg.cluster_split <= 1 && r > 0 &&
              2 * r <= P;
    const int w = 4 * r <= P ? 64 : 128;
    for (int64_t i = 0; ok && i < n; ++i) {
      const TcWork& t = tw[static_cast<size_t>(i)];
      if (t.flags & kFlagSplitK) ok = false;  // workspace split-K tables keep their layout
      if (i >= n - r && (t.pack || (t.flags & kFlagColMN) || t.n_mma <= w || t.col_len <= w)) ok = false;
    }
    if (ok) {
      std::vector<TcWork> ov;
      ov.reserve(static_cast<size_t>(n + 3 * r));
      for (int64_t i = 0; i < n - r; ++i) ov.push_back(tw[static_cast<size_t>(i)]);
      for (int64_t i = n - r; i < n; ++i) {
        const TcWork& t = tw[static_cast<size_t>(i)];
        for (int c = 0; c < t.col_len; c += w) {
          TcWork u = t;
          u.col0 = t.col0 + c;
          u.col_len = std::min(w, t.col_len - c);
          u.n_mma = static_cast<int32_t>(round_up(u.col_len, 32));
          u.flags &= ~kFlagBulkStore;
          if (c + w < t.col_len) u.flags &= ~kFlagTmaTail;  // only the last piece ends at N
          ov.push_back(u);
        }
      }
      tw.swap(ov);
    }
  }
  // Interleave long (MMA/TMA-bound, e.g. Dense) and short (latency-bound,
  // e.g. attention BMM) items in rounds of one item per CTA, so each CTA
  // alternates them: a short item's load -> MMA -> epilogue chain then hides
  // behind the neighbouring long items instead of forming a serial tail.
  {
    const char* env_il = std::getenv("FTB_INTERLEAVE");
    int sms_here = device_sms();
    if (sms_here <= 0) sms_here = 148;
    auto cost = [](const TcWork& t) { return static_cast<int64_t>(t.num_kb) * std::max(kMmaFloorN, t.n_mma); };
    std::vector<TcWork> lng, shrt;
    for (const TcWork& t : tw) (cost(t) >= 4 * kMmaFloorN ? lng : shrt).push_back(t);
    if (!(env_il && env_il[0] == '0') && I.cfg.cluster_split <= 1 && !lng.empty() && !shrt.empty()) {
      std::vector<TcWork> mix;
      mix.reserve(tw.size());
      size_t a = 0, b = 0;
      const double ratio = static_cast<double>(shrt.size()) / static_cast<double>(lng.size());
      double owed = 0.0;
      while (a < lng.size() || b < shrt.size()) {
        const size_t na = std::min(lng.size() - a, static_cast<size_t>(sms_here));
        for (size_t q = 0; q < na; ++q) mix.push_back(lng[a++]);
        owed += na ? na * ratio : static_cast<double>(shrt.size() - b);
        size_t nb = std::min(shrt.size() - b, static_cast<size_t>(owed));
        owed -= static_cast<double>(nb);
        for (size_t q = 0; q < nb; ++q) mix.push_back(shrt[b++]);
      }
      tw.swap(mix);
    }
  }
  // Eight epilogue warps for tables of short items (every item <= 8 K blocks,
  // more items than SMs, no split-K): their epilogue (TMEM -> smem ->
  // TMA store) is the bottleneck (C2 attention, scripts/bmm_trace.py); two
  // groups of four warps drain alternate items, with 8 KiB double-buffered
  // staging each (the ring gives up stages: short items need few).
  {
    const char* env_e8 = std::getenv("FTB_EPI8");
    int sms_here = device_sms();
    if (sms_here <= 0) sms_here = 148;
    int64_t kb_max = 0, out_bytes = 0;
    bool split = false;
    for (const TcWork& t : tw) {
      kb_max = std::max<int64_t>(kb_max, t.num_kb);
      const int64_t entries = t.pack ? pack_nb(t.pack) : 1;
      out_bytes += entries * t.lane_len * t.col_len * ((t.flags & kFlagOutF32) ? 4 : 2);
      split = split || (t.flags & kFlagSplitK);
    }
    const int64_t n = static_cast<int64_t>(tw.size());
    // not for tables of near-full output tiles (>= 48 KiB per item on average):
    // those are DRAM-write bound and a second epilogue group only costs ring
    // stages (C2 scores T=512: 112 -> 124 us). Measured gains: C2 scores
    // T=257 121 -> 85 us, T=64 scores / context 5.7 -> 5.0 us, context T=256
    // 36.4 -> 34.5 us, T=512 100 vs 104 us; C1 per-shape scores 0.147 -> 0.163.
    // every item short (a mixed table such as the C1 step keeps its ring
    // stages for the long Dense items: measured 0.80 vs 0.83 ms with eight warps)
    bool e8 = !pairing && !split && n > sms_here && kb_max <= 8 && out_bytes < (int64_t(48) << 10) * n;
    int mode = e8 ? 1 : 0;
    // Column split (mode 2, OPT-IN FTB_EPI8=2): both warp groups drain half
    // of every item's columns. Measured on tables of <= one item per CTA it
    // LOSES (C1 out M=608 6.39 -> 6.65 us, qkv M=1472 9.2 -> 9.7 us,
    // profiles/r2ab_epi8_colsplit.txt): the 320-thread kernel's smaller ring
    // and register budget cost more than the shorter epilogue tail saves.
    if (env_e8) mode = (env_e8[0] == '1' || env_e8[0] == '2') && !pairing && !split ? env_e8[0] - '0' : 0;
    I.cfg.epi8 = mode;
  }
  I.n_singles = static_cast<int64_t>(tw.size());
  I.n_pairs = static_cast<int64_t>(pairs.size());
  {
    Blob b;
    const size_t op = b.add(nullptr, sizeof(DevProblem) * I.problems.size());
    const size_t om = b.add(nullptr, sizeof(DevMaps) * I.maps.size());
    const size_t ot = b.add(nullptr, sizeof(TcWork) * tw.size());
    const size_t oq = b.add(nullptr, sizeof(TcPair) * pairs.size());
    const size_t oc = b.add(nullptr, sizeof(int32_t) * kSplitCntPerTile * static_cast<size_t>(split_tiles));
    FTB_CUDA(cudaMallocAsync(&I.d_blob, std::max<size_t>(b.bytes.size(), 128), us));
    I.d_problems = reinterpret_cast<DevProblem*>(at(op));
    I.d_maps = reinterpret_cast<DevMaps*>(at(om));
    I.d_tcwork = tw.empty() ? nullptr : reinterpret_cast<TcWork*>(at(ot));
    I.d_tcpairs = pairs.empty() ? nullptr : reinterpret_cast<TcPair*>(at(oq));
    I.d_split_cnt = split_tiles ? reinterpret_cast<int32_t*>(at(oc)) : nullptr;
    for (TcWork& t : tw) t.maps = I.d_maps + reinterpret_cast<uintptr_t>(t.maps);
    for (TcPair& t : pairs) t.maps = I.d_maps + reinterpret_cast<uintptr_t>(t.maps);
    std::memcpy(b.bytes.data() + op, I.problems.data(), sizeof(DevProblem) * I.problems.size());
    std::memcpy(b.bytes.data() + om, I.maps.data(), sizeof(DevMaps) * I.maps.size());
    if (!tw.empty()) std::memcpy(b.bytes.data() + ot, tw.data(), sizeof(TcWork) * tw.size());
    if (!pairs.empty()) std::memcpy(b.bytes.data() + oq, pairs.data(), sizeof(TcPair) * pairs.size());
    // split-K counters start at zero (the Blob is zero-filled) and re-arm themselves
    send(b);
  }
  int sms = device_sms();
  if (sms <= 0) sms = 148;
  I.ctas1 = std::min<int64_t>(I.n_singles, sms);
  I.ctas2 = 2 * std::min<int64_t>(I.n_pairs, sms / 2);
  I.info.n_ctas = std::max(I.ctas1, I.ctas2);
  auto shape_cfg = [](TcConfig& c, int max_cols, int col_rows) {
    // accumulator slots: the widest item decides the slot width (64/128/256 columns)
    c.acc_cols = max_cols <= 64 ? 64 : (max_cols <= 128 ? 128 : 256);
    c.n_acc = kTmemCols / c.acc_cols;
    c.col_stage_bytes = col_rows * kBlockK * 2;
    c.stages = 1;
    for (int s = kMaxStages; s >= 2; --s) {
      TcConfig t = c;
      t.stages = s;
      if (tc_smem_bytes(t) <= 232448) {
        c.stages = s;
        break;
      }
    }
    c.trace = nullptr;
  };
  shape_cfg(I.cfg, max_n, max_n);
  {
    const char* env_pf = std::getenv("FTB_L2_PREFETCH");
    I.cfg.l2_prefetch = (env_pf && env_pf[0] == '0') ? 0 : 1;
    const char* env_pm = std::getenv("FTB_PARAM_MAPS");
    I.cfg.param_maps = (I.maps.size() == 1 && !(env_pm && env_pm[0] == '0')) ? 1 : 0;
  }
  I.cfg.split_ws = I.d_split_ws;
  I.cfg.split_cnt = I.d_split_cnt;
  int max_np = 32;
  for (const TcPair& t : pairs) max_np = std::max(max_np, t.n_mma);
  shape_cfg(I.cfg2, max_np, max_np / 2);
  I.cfg.trace = nullptr;
}

}  // namespace ftb

struct ftb_exec {
  ftb::ExecImpl impl;
};

namespace ftb {
// While another stream of the process is being captured in torch's default
// (global) capture mode, CUDA rejects "unsafe" calls from any thread — the
// stream-ordered allocation and private-stream upload of a table created
// mid-capture (e.g. a GEMM on freshly allocated graph-pool outputs inside
// torch.cuda.graph), or the host wait on a table's upload before its launch
// is recorded. Table create / launch / destroy switch this thread to relaxed
// mode for their duration; none of their calls touches the capturing stream
// except the recorded kernel launch itself.
struct RelaxedCapture {
  cudaStreamCaptureMode prev = cudaStreamCaptureModeRelaxed;
  RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&prev); }
  ~RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&prev); }
};
}  // namespace ftb

extern "C" {

int32_t ftb_device_sm_count(void) { return ftb::device_sms(); }

ftb_status ftb_exec_create(const ftb_gemm_desc* problems, const ftb_program* programs, int32_t n,
                           ftb_exec** out) {
  return ftb::guarded([&] {
    if (!out || !problems || !programs) throw ftb::input_error("null argument");
    ftb::RelaxedCapture relaxed;
    auto* ex = new ftb_exec();
    try {
      static const bool prof = std::getenv("FTB_PROFILE_CREATE") != nullptr;
      auto t0 = std::chrono::steady_clock::now();
      ftb::build(ex->impl, problems, programs, n, /*encode=*/true);
      auto t1 = std::chrono::steady_clock::now();
      auto& I = ex->impl;
      ftb::upload(I);
      if (prof) {
        auto t2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "ftb_exec_create: %d problems, %lld items: build %.3f ms (encode %.3f ms), upload %.3f ms\n",
                     n, static_cast<long long>(I.info.n_work),
                     std::chrono::duration<double, std::milli>(t1 - t0).count(), I.encode_ms,
                     std::chrono::duration<double, std::milli>(t2 - t1).count());
      }
    } catch (...) {
      delete ex;
      throw;
    }
    *out = ex;
  });
}

ftb_status ftb_exec_launch(ftb_exec* ex, void* stream) {
  return ftb::guarded([&] {
    if (!ex) throw ftb::input_error("null exec");
    ftb::RelaxedCapture relaxed;
    auto& I = ex->impl;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> g(I.mu);
    int cur = -1;
    FTB_CUDA(cudaGetDevice(&cur));
    if (I.device >= 0 && cur != I.device)
      throw ftb::input_error("the table lives on device " + std::to_string(I.device) + ", the current device is " +
                             std::to_string(cur), "device");
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    FTB_CUDA(cudaStreamIsCapturing(s, &cap));
    const bool capturing = cap != cudaStreamCaptureStatusNone;
    // Launches of one table are stream ordered (they share the split-K
    // workspace): a launch on a new stream first waits for the previous one.
    // A captured launch marks the table as never-to-be-freed: the graph may
    // replay it after the handle is destroyed.
    if (I.ready && !I.ready_known) {  // the table upload (create did not wait for it)
      if (capturing) {
        FTB_CUDA(cudaEventSynchronize(I.ready));  // a graph must not depend on an outside event
        I.ready_known = true;
      } else {
        FTB_CUDA(cudaStreamWaitEvent(s, I.ready, 0));
        I.ready_known = cudaEventQuery(I.ready) == cudaSuccess;
      }
    }
    if (!capturing && I.last_stream && I.last_stream != s)
      for (auto& se : I.launched)
        if (se.first == I.last_stream) FTB_CUDA(cudaStreamWaitEvent(s, se.second, 0));
    cudaError_t e = I.info.kernel == 1
                        ? ftb::launch_ffma(I.d_problems, I.d_work, static_cast<int32_t>(I.info.n_work),
                                           static_cast<int32_t>(I.info.n_ctas), s, I.ffma_vec)
                        : cudaSuccess;
    if (e == cudaSuccess && I.info.kernel == 0 && I.n_pairs)
      e = ftb::launch_tc2(I.d_tcpairs, static_cast<int32_t>(I.n_pairs), static_cast<int32_t>(I.ctas2), I.cfg2, s);
    if (e == cudaSuccess && I.info.kernel == 0 && I.n_singles)
      e = ftb::launch_tc(I.d_tcwork, static_cast<int32_t>(I.n_singles), static_cast<int32_t>(I.ctas1), I.cfg,
                         I.maps.empty() ? nullptr : I.maps.data(), s);
    if (e != cudaSuccess) throw ftb::cuda_error(std::string("kernel launch: ") + cudaGetErrorString(e));
    if (capturing) I.captured = true;
    if (!capturing) {  // destroy frees the table only after this launch (exec.cu ~ExecImpl)
      cudaEvent_t ev = nullptr;
      for (auto& se : I.launched)
        if (se.first == s) ev = se.second;
      if (!ev) {
        FTB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        I.launched.emplace_back(s, ev);
      }
      FTB_CUDA(cudaEventRecord(ev, s));
      I.last_stream = s;
    }
  });
}

ftb_status ftb_exec_get_info(const ftb_exec* ex, ftb_exec_info* info) {
  return ftb::guarded([&] {
    if (!ex || !info) throw ftb::input_error("null argument");
    *info = ex->impl.info;
  });
}

ftb_status ftb_exec_export_table(const ftb_exec* ex, int32_t* out, int64_t cap, int64_t* n_out) {
  return ftb::guarded([&] {
    if (!ex || !n_out) throw ftb::input_error("null argument");
    const auto& W = ex->impl.work;
    *n_out = static_cast<int64_t>(W.size());
    if (out) {
      const int64_t k = std::min<int64_t>(cap, static_cast<int64_t>(W.size()));
      std::memcpy(out, W.data(), sizeof(ftb::DevWork) * k);
    }
  });
}

void ftb_exec_destroy(ftb_exec* ex) {
  ftb::RelaxedCapture relaxed;  // e.g. an LRU eviction while a graph is being captured
  delete ex;
}

ftb_status ftb_exec_set_trace(ftb_exec* ex, int32_t enable) {
  return ftb::guarded([&] {
    if (!ex) throw ftb::input_error("null exec");
    auto& I = ex->impl;
    if (I.info.kernel != 0) throw ftb::input_error("tracing is only available for the tcgen05 kernel");
    if (enable && !I.d_trace) {
      const size_t n = static_cast<size_t>(I.info.n_ctas) * ftb::kTracePerCta;
      FTB_CUDA(cudaMalloc(&I.d_trace, n * sizeof(unsigned long long)));
      FTB_CUDA(cudaMemset(I.d_trace, 0, n * sizeof(unsigned long long)));
    }
    I.cfg.trace = enable ? I.d_trace : nullptr;
    I.cfg2.trace = enable ? I.d_trace : nullptr;
  });
}

ftb_status ftb_exec_read_trace(const ftb_exec* ex, uint64_t* out, int64_t cap, int64_t* n_out) {
  return ftb::guarded([&] {
    if (!ex || !n_out) throw ftb::input_error("null argument");
    const auto& I = ex->impl;
    const int64_t n = I.d_trace ? I.info.n_ctas * ftb::kTracePerCta : 0;
    *n_out = n;
    if (out && n) FTB_CUDA(cudaMemcpy(out, I.d_trace, sizeof(uint64_t) * std::min(cap, n), cudaMemcpyDeviceToHost));
  });
}

ftb_status ftb_exec_get_config(const ftb_exec* ex, int32_t* out4) {
  return ftb::guarded([&] {
    if (!ex || !out4) throw ftb::input_error("null argument");
    const auto& I = ex->impl;
    const ftb::TcConfig* cs[2] = {&I.cfg, &I.cfg2};
    for (int k = 0; k < 2; ++k) {
      out4[4 * k + 0] = cs[k]->stages; out4[4 * k + 1] = cs[k]->col_stage_bytes;
      out4[4 * k + 2] = cs[k]->n_acc; out4[4 * k + 3] = cs[k]->acc_cols;
    }
    out4[8] = static_cast<int32_t>(I.n_singles);
    out4[9] = static_cast<int32_t>(I.n_pairs);
    out4[10] = I.cfg.cluster_split;                      // on-chip split-K factor (0/1: none)
    out4[11] = I.cfg.split_ws != nullptr ? 1 : 0;        // global-workspace split-K in use
  });
}

ftb_status ftb_lower(const ftb_gemm_desc* problems, const ftb_program* programs, int32_t n,
                     int32_t* out, int64_t cap, int64_t* n_out, ftb_exec_info* info) {
  return ftb::guarded([&] {
    if (!problems || !programs || !n_out) throw ftb::input_error("null argument");
    ftb::ExecImpl I;
    ftb::build(I, problems, programs, n, /*encode=*/false);
    *n_out = static_cast<int64_t>(I.work.size());
    if (out) {
      const int64_t k = std::min<int64_t>(cap, static_cast<int64_t>(I.work.size()));
      std::memcpy(out, I.work.data(), sizeof(ftb::DevWork) * k);
    }
    if (info) *info = I.info;
  });
}

}  // extern "C"
