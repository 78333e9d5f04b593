// kernel_tc.cu — K1: the persistent sm_100a uKernel executor.
//
// One launch runs every work item of a lowered tile-schedule table (any mix of
// problems, uKernel tile sizes and orientations). Each CTA owns one SM and
// walks its share of the table (static round-robin over a cost-sorted list)
// with three warp roles that only meet at mbarriers:
//   warp 0      TMA producer: per 64-wide K block, one (K-major) or two
//               (MN-major) boxes for the 128-row lane operand and 1-5 boxes
//               for the n_mma-row column operand, into an S-stage smem ring
//               (128-B swizzle). Items are prefetched one ahead.
//   warp 1      MMA issuer: one thread issues 4 x tcgen05.mma (M=128,
//               N=n_mma, K=16) per K block into one of n_acc TMEM accumulator
//               slots, commits each stage back to the producer and each
//               finished item to the epilogue.
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time; normal orientation
//               stores each lane's row segment with 16-B vector stores;
//               swap-AB orientation transposes 32x32 blocks through shared
//               memory so stores are row-contiguous too. Predication only on
//               ragged uKernel edges; the slot is released to the MMA warp
//               right after its last tcgen05.ld.
// The reference has no executor; what it must honour is the
// ProgramPlan coverage (combine.py:40-55): each work item writes exactly its
// rectangle of C and the rectangles of a plan tile C once.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "exec_types.h"
#include "ptx.cuh"
#include "epilogue.cuh"

namespace ftb {

__device__ __forceinline__ TcWork load_work(const TcWork* __restrict__ work, int w) {
  TcWork it;
  const uint4* src = reinterpret_cast<const uint4*>(work + w);
  uint4* dst = reinterpret_cast<uint4*>(&it);
#pragma unroll
  for (int q = 0; q < 4; ++q) dst[q] = __ldg(src + q);
  return it;
}

// trace layout: [cta][item < kTraceItems][event] with events
//   0 producer picked the item      1 producer issued K block 0
//   2 MMA saw K block 0 land        3 MMA committed the item
//   4 epilogue saw the accumulator  5 epilogue released it
__device__ __forceinline__ void trace_ev(const TcConfig& cfg, uint32_t local, int ev) {
#ifndef FTB_TRACE
  return;  // release build: phase tracing compiled out (it costs ~6 % per launch)
#endif
  if (cfg.trace && local < kTraceItems)
    cfg.trace[static_cast<size_t>(blockIdx.x) * kTracePerCta + local * kTraceEvents + ev] = globaltimer();
}
// per-K-block events of the first kTraceKb K blocks: 0 producer issued, 1 MMA saw data
__device__ __forceinline__ void trace_kb(const TcConfig& cfg, uint32_t g, int ev) {
#ifndef FTB_TRACE
  return;
#endif
  if (cfg.trace && g < kTraceKb)
    cfg.trace[static_cast<size_t>(blockIdx.x) * kTracePerCta + kTraceItems * kTraceEvents + 2 * g + ev] =
        globaltimer();
}

// Work records are fetched one lane per 32-bit word (a coalesced 64-B load
// whose latency overlaps the current item) and later broadcast from those
// lanes with shfl: ptxas treats a shfl from a constant lane as warp-uniform,
// so the loop bodies keep item fields in uniform registers. Warp converged.
__device__ __forceinline__ uint32_t fetch_work_word(const TcWork* __restrict__ work, int w) {
  const int lane = threadIdx.x & 31;
  return lane < 16 ? __ldg(reinterpret_cast<const uint32_t*>(work + w) + lane) : 0u;
}
__device__ __forceinline__ TcWork bcast_work(uint32_t mine) {
  TcWork it;
  uint32_t* dst = reinterpret_cast<uint32_t*>(&it);
#pragma unroll
  for (int q = 0; q < 16; ++q) dst[q] = __shfl_sync(0xffffffffu, mine, q);
  return it;
}

// Single-problem tables pass the problem's TMA descriptors as a
// __grid_constant__ kernel parameter (cfg.param_maps): TMA loads / stores and
// descriptor prefetches then read them from the launch's parameter bank
// instead of fetching the table copy from global memory after the work
// record arrives — one dependent global round trip off every launch's
// critical path.
__device__ __forceinline__ TcWork with_maps(TcWork t, const TcConfig& cfg, const DevMaps* pm) {
  if (cfg.param_maps) t.maps = pm;
  return t;
}

// Split-K epilogue for one warp (lane quadrant): publish the fp32 partial of
// this split to the workspace and count its arrival per 32-column chunk; the
// split completing a chunk sums all partials of it (fixed split order, so the
// sum is deterministic) and stores C through the predicated path, then
// re-arms the chunk's counter for the next launch.
template <bool kCluster, class Release>
__device__ __forceinline__ void split_epilogue(const TcConfig& cfg, const TcWork& it, uint8_t* region, uint32_t taddr,
                                               int lane_base, bool swap, bool f32, Release release, float* csmem) {
  const int lane = threadIdx.x & 31;
  const int quad = lane_base >> 5;
  if (kCluster) {
    // On-chip mode: the splits of a tile are the CTAs of one cluster, one item
    // each. This split's fp32 partial goes to this CTA's (now idle) operand
    // ring: per (chunk, quad) a 4 KiB block laid out [column group g of 4][lane][4],
    // so each v4 store here and each v4 DSMEM load of cluster_reduce moves
    // 512 contiguous bytes per warp (coalesced; a lane-strided layout made
    // every remote load 32 separate 16-B packets and the reduction 2x
    // slower). cluster_reduce sums the cluster's partials after the kernel's
    // closing cluster barrier.
    for (int c0 = 0; c0 < it.col_len; c0 += 64) {
      const bool two = c0 + 32 < it.col_len;
      uint32_t ra[32], rb[32];
      tmem_ld_32x32b_x32(taddr + c0, ra);
      if (two) tmem_ld_32x32b_x32(taddr + c0 + 32, rb);
      tmem_ld_wait();
      float* blk = csmem + (static_cast<size_t>((c0 >> 5) * 4 + quad) << 10) + lane * 4;
#pragma unroll
      for (int g = 0; g < 8; ++g)
        *reinterpret_cast<float4*>(blk + g * 128) =
            make_float4(__uint_as_float(ra[4 * g]), __uint_as_float(ra[4 * g + 1]), __uint_as_float(ra[4 * g + 2]),
                        __uint_as_float(ra[4 * g + 3]));
      if (two) {
        blk += 4 * 1024;  // next chunk, same quad
#pragma unroll
        for (int g = 0; g < 8; ++g)
          *reinterpret_cast<float4*>(blk + g * 128) =
              make_float4(__uint_as_float(rb[4 * g]), __uint_as_float(rb[4 * g + 1]), __uint_as_float(rb[4 * g + 2]),
                          __uint_as_float(rb[4 * g + 3]));
      }
    }
    release();
    return;
  }
  const int nsplit = split_n(it.pack), me = split_idx(it.pack), tile = it.c_bs;
  // workspace: [tile][split][quad][chunk][32 cols][32 lanes] — every access is
  // one coalesced 128-B row per register index
  float* ws = cfg.split_ws + static_cast<size_t>(tile) * kSplitTileFloats;
  auto part = [&](int split, int c0) {
    return ws + ((static_cast<size_t>(split) * 4 + quad) * (kSplitRowFloats / 32) + (c0 >> 5)) * 1024 + lane;
  };
  const bool active = lane_base < it.lane_len;  // the same for every split of the tile
  // pass 1: publish this split's fp32 partial, then hand TMEM back
  for (int c0 = 0; active && c0 < it.col_len; c0 += 32) {
    uint32_t raw[32];
    tmem_ld_32x32b_x32(taddr + c0, raw);
    tmem_ld_wait();
    float* dst = part(me, c0);
#pragma unroll
    for (int e = 0; e < 32; ++e) __stcg(dst + e * 32, __uint_as_float(raw[e]));
  }
  release();  // TMEM no longer needed
  if (!active) return;
  __threadfence();
  __syncwarp();
  // pass 2: count arrivals per 32-column chunk; the split whose arrival
  // completes a chunk reduces it (fixed split order: the sum is bit-identical
  // whoever reduces) and stores C. No split waits for another, so split-K
  // needs no co-residency (a concurrent kernel holding SMs only delays the
  // last arrival). Chunks are visited in an order rotated by the split index
  // so that, when the splits finish together, the reductions spread over
  // them instead of landing on one warp.
  int32_t* cnt = cfg.split_cnt + static_cast<size_t>(tile) * kSplitCntPerTile + quad * kSplitChunks;
  float* tb = reinterpret_cast<float*>(region);
  if (lane == 0) bulk_wait_read<0>();  // the transpose tile aliases this warp's store boxes
  __syncwarp();
  const int nch = (it.col_len + 31) >> 5;
  for (int j = 0; j < nch; ++j) {
    const int ch = (me + j) % nch;
    int prev = 0;
    if (lane == 0) prev = atomicAdd(cnt + ch, 1);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != nsplit - 1) continue;
    __threadfence();  // every other split's partial of this chunk is visible
    const int c0 = ch * 32;
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = 0.f;
    int sp = 0;
    for (; sp + 3 <= nsplit; sp += 3) {  // three partials in flight; fixed order: deterministic sum
      const float* s0 = part(sp, c0);
      const float* s1 = part(sp + 1, c0);
      const float* s2 = part(sp + 2, c0);
      float a[32], b[32], c[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        a[e] = __ldcg(s0 + e * 32);
        b[e] = __ldcg(s1 + e * 32);
        c[e] = __ldcg(s2 + e * 32);
      }
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = ((v[e] + a[e]) + b[e]) + c[e];
    }
    for (; sp < nsplit; ++sp) {
      const float* src = part(sp, c0);
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] += __ldcg(src + e * 32);
    }
    if (lane == 0) cnt[ch] = 0;  // every split has counted: re-arm for the next launch
    if (it.flags & kFlagEpiOp) {
      uint32_t rb[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) rb[e] = __float_as_uint(v[e]);
      apply_epi(rb, it.maps->epi, !swap, swap ? it.lane0 + lane_base : it.col0 + c0);
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(rb[e]);
    }
    const int ncol = min(32, it.col_len - c0);
    const int nlane = min(32, it.lane_len - lane_base);
    if (!swap)
      store_block32(tb, v, true, it.C, it.ldc, it.lane0 + lane_base, it.col0 + c0, nlane, ncol, f32);
    else
      store_block32(tb, v, false, it.C, it.ldc, it.col0 + c0, it.lane0 + lane_base, ncol, nlane, f32);
  }
}

// On-chip split-K reduction (cfg.cluster_split > 1): CTA `rank` of the
// cluster sums chunks rank, rank + s, ... of its lane quadrant over the s
// partials held in the cluster's shared memories (distributed shared memory,
// 16-B loads, only the chunk's column groups, all peers in flight for s = 4;
// fixed split order: deterministic and
// bit-identical to the workspace path at the same split count), applies the
// fused epilogue op and stores C — through TMA store boxes when the item
// allows it, else the coalesced predicated path.
__device__ __forceinline__ void cluster_reduce(const TcConfig& cfg, const TcWork& it, uint8_t* region, float* csmem,
                                               int quad) {
  const int lane = threadIdx.x & 31;
  const int lane_base = quad * 32;
  if (lane_base >= it.lane_len) return;
  const bool swap = it.flags & kFlagSwap, f32 = it.flags & kFlagOutF32;
  const bool tma = (it.flags & kFlagTmaStore) && !(it.flags & kFlagTmaTail) && !f32;
  const int s = cfg.cluster_split;
  const int rank = static_cast<int>(cluster_ctarank());
  float* tb = reinterpret_cast<float*>(region);
  if (lane == 0) bulk_wait_read<0>();  // the transpose tile aliases this warp's store boxes
  __syncwarp();
  const int nch = (it.col_len + 31) >> 5;
  uint32_t nbox = 0;
  for (int ch = rank; ch < nch; ch += s) {
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = 0.f;
    const uint32_t mine = smem_addr(csmem + (static_cast<size_t>(ch * 4 + quad) << 10) + lane * 4);
    const int ng = (min(32, it.col_len - ch * 32) + 3) >> 2;  // 4-column groups the chunk has
    if (s == 4) {
      // all four peers' loads in flight at once (one DSMEM round trip), then
      // the fixed-order sum
      float4 a[4][8];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const uint32_t pa = mapa_shared(mine, static_cast<uint32_t>(p));
#pragma unroll
        for (int g = 0; g < 8; ++g) a[p][g] = g < ng ? ld_dsmem_v4(pa + g * 512) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          v[4 * g] += a[p][g].x;
          v[4 * g + 1] += a[p][g].y;
          v[4 * g + 2] += a[p][g].z;
          v[4 * g + 3] += a[p][g].w;
        }
    } else {
      int p = 0;
      for (; p + 2 <= s; p += 2) {
        const uint32_t pa = mapa_shared(mine, static_cast<uint32_t>(p));
        const uint32_t pb = mapa_shared(mine, static_cast<uint32_t>(p + 1));
        float4 a[8], b[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          a[g] = g < ng ? ld_dsmem_v4(pa + g * 512) : make_float4(0.f, 0.f, 0.f, 0.f);
          b[g] = g < ng ? ld_dsmem_v4(pb + g * 512) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          v[4 * g] = (v[4 * g] + a[g].x) + b[g].x;
          v[4 * g + 1] = (v[4 * g + 1] + a[g].y) + b[g].y;
          v[4 * g + 2] = (v[4 * g + 2] + a[g].z) + b[g].z;
          v[4 * g + 3] = (v[4 * g + 3] + a[g].w) + b[g].w;
        }
      }
      if (p < s) {
        const uint32_t pa = mapa_shared(mine, static_cast<uint32_t>(p));
        float4 a[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) a[g] = g < ng ? ld_dsmem_v4(pa + g * 512) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          v[4 * g] += a[g].x;
          v[4 * g + 1] += a[g].y;
          v[4 * g + 2] += a[g].z;
          v[4 * g + 3] += a[g].w;
        }
      }
    }
    const int c0 = ch * 32;
    uint32_t rb[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) rb[e] = __float_as_uint(v[e]);
    if (it.flags & kFlagEpiOp) apply_epi(rb, it.maps->epi, !swap, swap ? it.lane0 + lane_base : it.col0 + c0);
    if (tma) {
      uint8_t* box = region + (nbox & 3) * 2048;
      if (lane == 0 && nbox >= 4) bulk_wait_read<3>();  // this box's previous store has read it
      __syncwarp();
      stage_box_bf16(box, rb, !swap);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int l0 = it.lane0 + lane_base, k0 = it.col0 + c0;
        if (!swap) tma_store_3d(&it.maps->out, smem_addr(box), k0, l0, it.batch);
        else tma_store_3d(&it.maps->out, smem_addr(box), l0, k0, it.batch);
        bulk_commit();
      }
      ++nbox;
      continue;
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(rb[e]);
    const int ncol = min(32, it.col_len - c0);
    const int nlane = min(32, it.lane_len - lane_base);
    if (!swap)
      store_block32(tb, v, true, it.C, it.ldc, it.lane0 + lane_base, it.col0 + c0, nlane, ncol, f32);
    else
      store_block32(tb, v, false, it.C, it.ldc, it.col0 + c0, it.lane0 + lane_base, ncol, nlane, f32);
  }
  if (lane == 0) bulk_wait_read<0>();
  __syncwarp();
}

// kCluster: the on-chip split-K variant (cluster launch, one item per CTA);
// kEpi8: eight epilogue warps (tables of short items, epilogue bound;
// 320 threads at a 168-register budget). Separate instantiations, so the
// common kernel carries none of their code.
template <int S, bool kCluster, bool kEpi8>
__global__ void __launch_bounds__(kEpi8 ? 384 : kTcThreads, 1)
    ftb_tc_kernel(const TcWork* __restrict__ work, int32_t n_work, TcConfig cfg, const __grid_constant__ DevMaps pmaps) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived by pointer arithmetic on the __shared__ array
  // so the compiler keeps the shared state space: every staging / transpose
  // access below compiles to STS/LDS rather than generic ST.E/LD.E (an
  // integer round trip through uintptr_t made all 1000 of them generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint8_t* lane_buf = smem;                                   // S x 16 KiB
  uint8_t* col_buf = smem + S * kLaneStageBytes;              // S x col_stage_bytes
  float* epi_buf = reinterpret_cast<float*>(col_buf + S * cfg.col_stage_bytes);  // 4 x 32x33
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(epi_buf) + (kEpi8 ? 2 : 1) * kEpiStageBytes);
  uint64_t* full = bars;                      // [S]
  uint64_t* empty = bars + kMaxStages;        // [S]
  uint64_t* tfull = bars + 2 * kMaxStages;    // [n_acc]
  uint64_t* tempty = bars + 3 * kMaxStages;   // [n_acc]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4 * kMaxStages);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < cfg.n_acc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], (kEpi8 && cfg.epi8 == 2) ? 8 : 4);  // one arrive per epilogue warp on the slot
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_holder);
#ifdef FTB_EPI_TRACE
  if (threadIdx.x == 0) ftb_epi_dbg = cfg.trace;  // same value from every CTA
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_holder, 0);  // warp-uniform
  const uint32_t smem_u32 = smem_addr(smem);
  const uint32_t lane_u32 = smem_addr(lane_buf), col_u32 = smem_addr(col_buf);
  // Programmatic dependent launch: everything above (barrier init, TMEM
  // allocation) and the producer's work-record fetch and descriptor prefetch
  // (host-written at executable creation) overlap the previous grid's tail.
  // Only the producer waits for that grid: every operand load is issued after
  // its wait, and every output write is causally after an operand load.
  // Dependents may launch right away — they in turn wait for this grid.
  griddep_launch_dependents();
#ifdef FTB_TRACE
  // CTA start / end stamps (scripts/tail_spread.py). Debug builds only: these
  // two guarded stores alone cost the release kernel ~13 % on the C1 step
  // (register allocation / scheduling of the whole kernel changes).
  if (threadIdx.x == 0 && cfg.trace)
    cfg.trace[static_cast<size_t>(blockIdx.x) * kTracePerCta + kTracePerCta - 2] = globaltimer();
#endif
  const int G = gridDim.x;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // The whole warp walks the loops with warp-uniform values (work records
    // broadcast from lane 0 with shfl, so ptxas keeps them in uniform
    // registers); lane 0 alone arms the barrier and issues the TMA loads.
    // Records are fetched two items ahead so the next item's descriptor
    // prefetch never waits on a global load.
    uint32_t g = 0;
    uint32_t ps = 0, pphase = 0;  // ring slot / phase
    uint32_t local = 0;
#ifdef FTB_PROD_PROFILE
    unsigned long long c_wait = 0, c_issue = 0, c_item = 0, c_t0 = clock64();
#endif
    TcWork cur, nxt;
    uint32_t pend = 0;  // raw word of the record two items ahead
    if (static_cast<int>(blockIdx.x) < n_work) cur = with_maps(bcast_work(fetch_work_word(work, blockIdx.x)), cfg, &pmaps);
    if (static_cast<int>(blockIdx.x) + G < n_work) nxt = with_maps(bcast_work(fetch_work_word(work, blockIdx.x + G)), cfg, &pmaps);
    if (static_cast<int>(blockIdx.x) + 2 * G < n_work) pend = fetch_work_word(work, blockIdx.x + 2 * G);
    if (lane == 0 && static_cast<int>(blockIdx.x) < n_work) {
      tma_prefetch_desc(&cur.maps->lane);
      tma_prefetch_desc(&cur.maps->col[0]);
      // Programmatic dependent launch: this grid runs ahead of its
      // predecessor's tail. Pull the first item's first K block of operand
      // boxes from HBM into L2 now, so the first loads issued after
      // griddep_wait hit L2 instead of paying the DRAM latency on the
      // launch's critical path (1-item chain: 4.08 -> 3.58 us, profiles/r2j_l2_prefetch_ab.txt).
      if (cfg.l2_prefetch && cur.num_kb <= 2) {  // short items only: measured, long-K Dense
                                                 // items lost ~4 % with it (the prefetch's TMA
                                                 // issue sits on their critical path)
        const bool pk = !(cur.flags & kFlagSplitK) && pack_depth(cur.pack);
        const int kb0 = (cur.flags & kFlagSplitK) ? split_kb0(cur.pack) : 0;
        const int nkb = 1;  // the first K block only: later ones stream behind it (a whole
                            // ring's worth cost 96-CTA tables ~1.3 us, profiles/profiles/r2j_l2_prefetch_ab.txt)
        const uint32_t cmask = col_box_mask(cur.n_mma);
        for (int kb = 0; kb < nkb; ++kb) {
          const int k0 = (kb + kb0) * kBlockK;
          if (pk || !(cur.flags & kFlagLaneMN)) {
            tma_prefetch_l2_3d(&cur.maps->lane, k0, cur.lane0, cur.batch);
          } else {
            tma_prefetch_l2_3d(&cur.maps->lane, cur.lane0, k0, cur.batch);
            tma_prefetch_l2_3d(&cur.maps->lane, cur.lane0 + 64, k0, cur.batch);
          }
          if (!(cur.flags & kFlagColMN)) {
            if (pk) {
              tma_prefetch_l2_3d(&cur.maps->col[0], k0, cur.col0, cur.batch);
            } else {
              int r = 0;
              for (int q = 0; q < kColMaps; ++q)
                if (cmask & (1u << q)) {
                  tma_prefetch_l2_3d(&cur.maps->col[q], k0, cur.col0 + r, cur.batch);
                  r += 256 >> q;
                }
            }
          } else {
            const int ncol = pk ? 64 : cur.n_mma;
            for (int c = 0; c < ncol; c += 64) tma_prefetch_l2_3d(&cur.maps->col[0], cur.col0 + c, k0, cur.batch);
          }
        }
      }
    }
    griddep_wait();
    for (int w = blockIdx.x; w < n_work; w += G, ++local) {
      const TcWork it = cur;
      if (lane == 0) {
        trace_ev(cfg, local, 0);
        if (w + G < n_work) {
          tma_prefetch_desc(&nxt.maps->lane);
          tma_prefetch_desc(&nxt.maps->col[0]);
        }
      }
      const CUtensorMap* tl = &it.maps->lane;
      const bool lane_mn = it.flags & kFlagLaneMN, col_mn = it.flags & kFlagColMN;
      const bool splitk = it.flags & kFlagSplitK;
      const int kb_base = splitk ? split_kb0(it.pack) : 0;
      const int depth = splitk ? 0 : pack_depth(it.pack);  // 0: not packed
      const uint32_t bytes =
          depth ? static_cast<uint32_t>(depth * (pack_lane_rows(it.pack) + 64) * kBlockK * 2)
                : kLaneStageBytes + static_cast<uint32_t>(it.n_mma) * kBlockK * 2;
      const uint32_t cmask = col_box_mask(it.n_mma);
      int boff[kColMaps];  // smem row offset of each column box (widest first)
      {
        int r = 0;
#pragma unroll
        for (int q = 0; q < kColMaps; ++q) {
          boff[q] = r;
          if (cmask & (1u << q)) r += 256 >> q;
        }
      }
#ifdef FTB_PROD_PROFILE
      unsigned long long ci = clock64();
#endif
      for (int kb = 0; kb < it.num_kb; ++kb, ++g) {
        const uint32_t s = ps;
#ifdef FTB_PROD_PROFILE
        unsigned long long cw = clock64();
#endif
        mbar_wait(&empty[s], pphase ^ 1);
        if (++ps == S) { ps = 0; pphase ^= 1; }
#ifdef FTB_PROD_PROFILE
        unsigned long long cs = clock64();
        c_wait += cs - cw;
#endif
        if (lane == 0) {
#ifdef FTB_TRACE_PRE
          trace_kb(cfg, g, 0);  // debug: stamp BEFORE the K block's TMA issue
#endif
          // one lane issues: measured faster here than the converged elect form
          // (619 vs 504 clk per K block, scripts/prod_profile.py)
          mbar_arrive_expect_tx(&full[s], bytes);
          uint8_t* ldst = lane_buf + s * kLaneStageBytes;
          uint8_t* cdst = col_buf + s * cfg.col_stage_bytes;
          const int k0 = (kb + kb_base) * kBlockK;
          if (depth) {  // packed batch entries: one 3-D box per operand
            tma_load_3d(ldst, tl, &full[s], k0, it.lane0, it.batch);
            if (!col_mn) tma_load_3d(cdst, &it.maps->col[0], &full[s], k0, it.col0, it.batch);
            else tma_load_3d(cdst, &it.maps->col[0], &full[s], it.col0, k0, it.batch);
          } else {
            if (!lane_mn) {
              tma_load_3d(ldst, tl, &full[s], k0, it.lane0, it.batch);
            } else {
              tma_load_3d(ldst, tl, &full[s], it.lane0, k0, it.batch);
              tma_load_3d(ldst + 8192, tl, &full[s], it.lane0 + 64, k0, it.batch);
            }
            if (!col_mn) {
#pragma unroll
              for (int q = 0; q < kColMaps; ++q)
                if (cmask & (1u << q))
                  tma_load_3d(cdst + boff[q] * 128, &it.maps->col[q], &full[s], k0, it.col0 + boff[q], it.batch);
            } else {
              for (int c = 0; c < it.n_mma; c += 64)
                tma_load_3d(cdst + c * 128, &it.maps->col[0], &full[s], it.col0 + c, k0, it.batch);
            }
          }
          if (kb == 0) trace_ev(cfg, local, 1);
#ifndef FTB_TRACE_PRE
          trace_kb(cfg, g, 0);
#endif
        }
        __syncwarp();
#ifdef FTB_PROD_PROFILE
        c_issue += clock64() - cs;
#endif
      }
#ifdef FTB_PROD_PROFILE
      c_item += clock64() - ci;
#endif
      cur = nxt;
      if (w + 2 * G < n_work) nxt = with_maps(bcast_work(pend), cfg, &pmaps);
      if (w + 3 * G < n_work) pend = fetch_work_word(work, w + 3 * G);
    }
#ifdef FTB_PROD_PROFILE
    if (lane == 0 && cfg.trace) {
      unsigned long long* t = cfg.trace + static_cast<size_t>(blockIdx.x) * kTracePerCta;
      t[0] = c_wait; t[1] = c_issue; t[2] = c_item; t[3] = g; t[4] = local; t[5] = clock64() - c_t0;
    }
#endif
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // whole warp walks the loops (uniform values); lane 0 issues and commits
    uint32_t g = 0;
    uint32_t ms = 0, mphase = 0;  // MMA ring slot / phase
    uint32_t local = 0;
    uint32_t pend = 0;
#ifdef FTB_PROD_PROFILE
    unsigned long long m_te = 0, m_full = 0, m_issue = 0, m_t0 = clock64();
#endif
    if (static_cast<int>(blockIdx.x) < n_work) pend = fetch_work_word(work, blockIdx.x);
    for (int w = blockIdx.x; w < n_work; w += G, ++local) {
      const TcWork it = bcast_work(pend);
      if (w + G < n_work) pend = fetch_work_word(work, w + G);  // lands while this item runs
      const uint32_t lane_mn = (it.flags & kFlagLaneMN) ? 1u : 0u;
      const uint32_t col_mn = (it.flags & kFlagColMN) ? 1u : 0u;
      const uint32_t slot = local % cfg.n_acc;
      const uint32_t use = local / cfg.n_acc;
#ifdef FTB_PROD_PROFILE
      unsigned long long mt0 = clock64();
#endif
      mbar_wait(&tempty[slot], (use & 1) ^ 1);
      tc_fence_after();
#ifdef FTB_PROD_PROFILE
      m_te += clock64() - mt0;
#endif
      const uint32_t tmem_d = tmem_base + slot * cfg.acc_cols;
      const uint32_t idesc = idesc_bf16_f32(kLaneRows, static_cast<uint32_t>(it.n_mma), lane_mn, col_mn);
      for (int kb = 0; kb < it.num_kb; ++kb, ++g) {
        const uint32_t s = ms;
#ifdef FTB_PROD_PROFILE
        unsigned long long mf0 = clock64();
#endif
        mbar_wait(&full[s], mphase);
        if (++ms == S) { ms = 0; mphase ^= 1; }
        tc_fence_after();
#ifdef FTB_PROD_PROFILE
        unsigned long long mf1 = clock64();
        m_full += mf1 - mf0;
#endif
        if (lane == 0) {
          if (kb == 0) trace_ev(cfg, local, 2);
#ifndef FTB_TRACE_ISSUE
          trace_kb(cfg, g, 1);
#endif
        }
        {
          const uint32_t la = lane_u32 + s * kLaneStageBytes;
          const uint32_t ca = col_u32 + s * static_cast<uint32_t>(cfg.col_stage_bytes);
#pragma unroll
          for (int kk = 0; kk < kBlockK / 16; ++kk) {
            const uint64_t adesc = lane_mn ? umma_desc_sw128(la + kk * 2048, 8192, 1024)
                                           : umma_desc_sw128(la + kk * 32, 16, 1024);
            const uint64_t bdesc = col_mn ? umma_desc_sw128(ca + kk * 2048, 8192, 1024)
                                          : umma_desc_sw128(ca + kk * 32, 16, 1024);
            tc_mma_f16_elect(tmem_d, adesc, bdesc, idesc, (kb | kk) != 0);
          }
          tc_commit_elect(smem_u32 + static_cast<uint32_t>(reinterpret_cast<uint8_t*>(&empty[s]) - smem));
        }
        __syncwarp();
#ifdef FTB_PROD_PROFILE
        m_issue += clock64() - mf1;
#endif
      }
      tc_commit_elect(smem_u32 + static_cast<uint32_t>(reinterpret_cast<uint8_t*>(&tfull[slot]) - smem));
      if (lane == 0) trace_ev(cfg, local, 3);  // accumulator ready for the epilogue
      __syncwarp();
    }
#ifdef FTB_PROD_PROFILE
    if (lane == 0 && cfg.trace) {
      unsigned long long* t = cfg.trace + static_cast<size_t>(blockIdx.x) * kTracePerCta;
      t[6] = m_te; t[7] = m_full; t[8] = m_issue; t[9] = clock64() - m_t0;
    }
#endif
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    // per-warp 8 KiB staging region: four 2 KiB TMA store boxes (two groups of
    // two), or — for predicated items — the 32x33 fp32 transpose tile (aliased).
    // kEpi8: two groups of four warps take alternate items (alternate TMEM
    // slots), 8 KiB each (the staging doubles; the ring gives up stages), so
    // two items' epilogues run concurrently.
    // cfg.epi8 == 2 (column split): both groups take EVERY item, each half
    // of its columns — for tables of at most one item per CTA, where the
    // item's epilogue is the launch's tail and halving it shortens the launch.
    const int egrp = kEpi8 ? (warp - 2) >> 2 : 0;
    const bool csplit = kEpi8 && cfg.epi8 == 2;
    uint8_t* region = reinterpret_cast<uint8_t*>(epi_buf) + (kEpi8 ? (warp - 2) : quad) * kEpiWarpBytes;
    const int step = (kEpi8 && !csplit) ? 2 : 1;
    uint32_t local = csplit ? 0 : egrp, ngrp = 0;
#ifdef FTB_PROD_PROFILE
    unsigned long long e_wait = 0, e_t0 = clock64();
#endif
    TcWork nxt;
    const int w0 = static_cast<int>(blockIdx.x) + (csplit ? 0 : egrp * G);
    if (w0 < n_work) nxt = with_maps(load_work(work, w0), cfg, &pmaps);
    for (int w = w0; w < n_work; w += step * G, local += step) {
      const TcWork it = nxt;
      if (w + step * G < n_work) nxt = with_maps(load_work(work, w + step * G), cfg, &pmaps);
      const uint32_t slot = local % cfg.n_acc;
      const uint32_t use = local / cfg.n_acc;
      const bool swap = it.flags & kFlagSwap, f32 = it.flags & kFlagOutF32;
      const bool tma = it.flags & kFlagTmaStore;
#ifdef FTB_PROD_PROFILE
      unsigned long long ew0 = clock64();
#endif
      mbar_wait(&tfull[slot], use & 1);
#ifdef FTB_PROD_PROFILE
      e_wait += clock64() - ew0;
#endif
      tc_fence_after();
      if (quad == 0 && lane == 0) trace_ev(cfg, local, 4);
      const int lane_base = quad * 32;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lane_base) << 16) + slot * cfg.acc_cols;
      auto release = [&] {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[slot]);
      };
      // this warp group's TMEM / C column window (the whole item unless csplit;
      // the cut sits on a 32-column store-box boundary)
      int clo = 0, clen = it.col_len;
      if (csplit) {
        const int half = ((it.col_len + 1) / 2 + 31) & ~31;
        clo = egrp * half;
        clen = min(it.col_len, clo + half) - clo;
      }
      // kFlagTmaTail: window-relative first column past the store map (N8)
      const int tail0 = (it.flags & kFlagTmaTail) && clo + clen == it.col_len
                            ? max(0, ((it.col0 + it.col_len) & ~7) - (it.col0 + clo))
                            : (1 << 30);
      if (it.flags & kFlagSplitK) {
        split_epilogue<kCluster>(cfg, it, region, taddr, lane_base, swap, f32, release, reinterpret_cast<float*>(smem));
      } else if (clen <= 0) {
        release();
      } else if (!it.pack) {
        epilogue_tile(region, ngrp, taddr + clo, lane_base < it.lane_len, tma, swap, f32, &it.maps->out, it.C, it.ldc,
                      it.lane0, it.lane_len, lane_base, it.col0 + clo, clen, it.batch, release,
                      (it.flags & kFlagEpiOp) ? &it.maps->epi : nullptr,
                      (it.flags & kFlagBulkStore) && clen == it.col_len, tail0);
      } else {
        // block-diagonal pack: this warp's lane quadrant belongs to entry e
        const int wpe = pack_lane_rows(it.pack) / 32;  // warps per entry
        const int e = quad / wpe, r0 = (quad % wpe) * 32;
        const bool active = e < pack_nb(it.pack) && r0 < it.lane_len;
        epilogue_tile(region, ngrp, taddr + e * 64 + clo, active, tma, swap, f32, &it.maps->out,
                      static_cast<char*>(it.C) + static_cast<size_t>(e) * it.c_bs * (f32 ? 4 : 2), it.ldc, 0,
                      it.lane_len, r0, clo, clen, it.batch + e, release, nullptr,
                      (it.flags & kFlagBulkStore) && clen == it.col_len, tail0);
      }
      if (quad == 0 && lane == 0) trace_ev(cfg, local, 5);
    }
#ifdef FTB_END_READ
    if (lane == 0) bulk_wait_read<0>();  // experiment: only the smem reads of the stores
#else
    if (lane == 0) bulk_wait_all();  // output stores complete before the CTA retires
#endif
    __syncwarp();
#ifdef FTB_PROD_PROFILE
    if (lane == 0 && warp == 2 && cfg.trace) {
      unsigned long long* t = cfg.trace + static_cast<size_t>(blockIdx.x) * kTracePerCta;
      t[10] = e_wait; t[11] = clock64() - e_t0;
    }
#endif
  }

  tc_fence_before();
  TcWork cl_it;  // the reduce's work record, fetched before the barrier (off the tail)
  if (kCluster && warp >= 2 && static_cast<int>(blockIdx.x) < n_work) cl_it = with_maps(load_work(work, blockIdx.x), cfg, &pmaps);
  __syncthreads();
  if (kCluster) {  // one item per CTA: reduce the cluster's split-K partials on chip
#ifdef FTB_TRACE
    if (threadIdx.x == 64 && cfg.trace) cfg.trace[blockIdx.x * kTracePerCta + kTraceItems * kTraceEvents + 120] = clock64();  // debug (clk): before the first cluster barrier
#endif
    cluster_sync();              // every split's partial written (release / acquire at cluster scope)
#ifdef FTB_TRACE
    if (threadIdx.x == 64 && cfg.trace) cfg.trace[blockIdx.x * kTracePerCta + kTraceItems * kTraceEvents + 121] = clock64();
#endif
    if (warp >= 2 && static_cast<int>(blockIdx.x) < n_work)
      cluster_reduce(cfg, cl_it, reinterpret_cast<uint8_t*>(epi_buf) + (warp & 3) * kEpiWarpBytes,
                     reinterpret_cast<float*>(smem), warp & 3);
#ifdef FTB_TRACE
    if (threadIdx.x == 64 && cfg.trace) cfg.trace[blockIdx.x * kTracePerCta + kTraceItems * kTraceEvents + 122] = clock64();  // debug (clk): warp 2 done reducing
#endif
    cluster_sync();              // peers have read this CTA's partial before it exits
#ifdef FTB_TRACE
    if (threadIdx.x == 64 && cfg.trace) cfg.trace[blockIdx.x * kTracePerCta + kTraceItems * kTraceEvents + 123] = clock64();
#endif
  }
#ifdef FTB_TRACE
  if (threadIdx.x == 0 && cfg.trace)  // CTA end stamp (all epilogue stores issued and complete)
    cfg.trace[static_cast<size_t>(blockIdx.x) * kTracePerCta + kTracePerCta - 1] = globaltimer();
#endif
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

int tc_smem_bytes(const TcConfig& cfg) {
  return 1024 + cfg.stages * (kLaneStageBytes + cfg.col_stage_bytes) + (cfg.epi8 ? 2 : 1) * kEpiStageBytes +
         (4 * kMaxStages + 2) * 8;
}

template <int S, bool kCluster, bool kEpi8>
static cudaError_t launch_tc_sk(const TcWork* work, int32_t n_work, int32_t n_ctas, TcConfig cfg,
                                const DevMaps& pmaps, cudaStream_t stream) {
  cudaError_t e = configure_smem_once<ftb_tc_kernel<S, kCluster, kEpi8>>(232448);
  if (e != cudaSuccess) return e;
  return launch_pdl_cluster(ftb_tc_kernel<S, kCluster, kEpi8>, n_ctas, kEpi8 ? kTcThreadsEpi8 : kTcThreads,
                            tc_smem_bytes(cfg), kCluster ? cfg.cluster_split : 1, stream, work, n_work, cfg, pmaps);
}
template <int S>
static cudaError_t launch_tc_s(const TcWork* work, int32_t n_work, int32_t n_ctas, TcConfig cfg,
                               const DevMaps& pmaps, cudaStream_t stream) {
  if (cfg.cluster_split > 1) return launch_tc_sk<S, true, false>(work, n_work, n_ctas, cfg, pmaps, stream);
  if (cfg.epi8) return launch_tc_sk<S, false, true>(work, n_work, n_ctas, cfg, pmaps, stream);
  return launch_tc_sk<S, false, false>(work, n_work, n_ctas, cfg, pmaps, stream);
}

// param_maps: the descriptors of a single-problem table (host copy), passed
// as a kernel parameter when cfg.param_maps is set; ignored otherwise.
cudaError_t launch_tc(const TcWork* work, int32_t n_work, int32_t n_ctas, TcConfig cfg, const DevMaps* param_maps,
                      cudaStream_t stream) {
  if (n_work == 0) return cudaSuccess;
  static const DevMaps none{};
  const DevMaps& pm = (cfg.param_maps && param_maps) ? *param_maps : none;
  if (cfg.param_maps && !param_maps) return cudaErrorInvalidValue;
  switch (cfg.stages) {
    case 2: return launch_tc_s<2>(work, n_work, n_ctas, cfg, pm, stream);
    case 3: return launch_tc_s<3>(work, n_work, n_ctas, cfg, pm, stream);
    case 4: return launch_tc_s<4>(work, n_work, n_ctas, cfg, pm, stream);
    case 5: return launch_tc_s<5>(work, n_work, n_ctas, cfg, pm, stream);
    case 6: return launch_tc_s<6>(work, n_work, n_ctas, cfg, pm, stream);
    case 7: return launch_tc_s<7>(work, n_work, n_ctas, cfg, pm, stream);
    case 8: return launch_tc_s<8>(work, n_work, n_ctas, cfg, pm, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ftb
