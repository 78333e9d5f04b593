// kernel_tc2.cu — K1b: the CTA-pair (cta_group::2) uKernel executor.
//
// Clusters of two CTAs on a TPC execute "pair items": two 128-lane slabs of
// one problem (the lane operand rows of each CTA can be anywhere) that share
// the same column range. One tcgen05.mma.cta_group::2 (M = 256, N = n_mma,
// K = 16) issued by the leader CTA reads each CTA's 128-row lane tile and each
// CTA's half of the column tile (N/2 rows) from the two shared memories and
// accumulates 128 x N into each CTA's own TMEM. Per CTA and K block the smem
// traffic is 16 KiB + N*64 B instead of 16 KiB + N*128 B, which is what lets
// the dense GEMMs outrun the per-SM operand-delivery limit of K1.
//
// Roles (per CTA, both CTAs unless noted):
//   warp 0      TMA producer: waits its own `empty` slot (released by the
//               leader's multicast commit), loads its lane slab and its half
//               of the column tile with cta_group::2 TMA whose completion
//               bytes land on the LEADER's `full` barrier.
//   warp 1      (leader only) MMA issuer; commits stages and finished items to
//               both CTAs with multicast tcgen05.commit.
//   warps 2..5  epilogue over the CTA's own 128 lanes; releases an
//               accumulator slot by arriving on the leader's `tempty`.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "epilogue.cuh"
#include "exec_types.h"
#include "ptx.cuh"

namespace ftb {

__device__ __forceinline__ TcPair load_pair(const TcPair* __restrict__ work, int w) {
  TcPair it;
  const uint4* src = reinterpret_cast<const uint4*>(work + w);
  uint4* dst = reinterpret_cast<uint4*>(&it);
#pragma unroll
  for (int q = 0; q < 4; ++q) dst[q] = __ldg(src + q);
  return it;
}

__device__ __forceinline__ void trace2_ev(const TcConfig& cfg, uint32_t local, int ev) {
#ifndef FTB_TRACE
  return;  // release build: tracing compiled out (see kernel_tc.cu)
#endif
  if (cfg.trace && local < kTraceItems)
    cfg.trace[static_cast<size_t>(blockIdx.x) * kTracePerCta + local * kTraceEvents + ev] = globaltimer();
}
__device__ __forceinline__ void trace2_kb(const TcConfig& cfg, uint32_t g, int ev) {
#ifndef FTB_TRACE
  return;
#endif
  if (cfg.trace && g < kTraceKb)
    cfg.trace[static_cast<size_t>(blockIdx.x) * kTracePerCta + kTraceItems * kTraceEvents + 2 * g + ev] =
        globaltimer();
}

template <int S>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
    ftb_tc2_kernel(const TcPair* __restrict__ work, int32_t n_work, TcConfig cfg) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived by pointer arithmetic on the __shared__ array
  // so the compiler keeps the shared state space: every staging / transpose
  // access below compiles to STS/LDS rather than generic ST.E/LD.E (an
  // integer round trip through uintptr_t made all 1000 of them generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint8_t* lane_buf = smem;                                   // S x 16 KiB
  uint8_t* col_buf = smem + S * kLaneStageBytes;              // S x col_stage_bytes (N/2 rows)
  float* epi_buf = reinterpret_cast<float*>(col_buf + S * cfg.col_stage_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(epi_buf) + kEpiStageBytes);
  uint64_t* full = bars;                      // [S]     leader: TMA bytes of both CTAs
  uint64_t* empty = bars + kMaxStages;        // [S]     both: multicast commit
  uint64_t* tfull = bars + 2 * kMaxStages;    // [n_acc] both: multicast commit
  uint64_t* tempty = bars + 3 * kMaxStages;   // [n_acc] leader: 8 epilogue-warp arrivals
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4 * kMaxStages);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < cfg.n_acc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_holder);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated on both
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  griddep_wait();  // operands / outputs only after the previous grid (PDL)
  griddep_launch_dependents();
  const int G = gridDim.x >> 1;          // clusters
  const int cid = blockIdx.x >> 1;       // this cluster

  if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    // whole warp walks the loops (records fetched ahead, broadcast with shfl);
    // lane 0 arms the leader's barrier (leader CTA) and issues the 2-SM loads
    uint32_t g = 0;
    uint32_t ps = 0, pphase = 0;  // producer ring slot / phase
    uint32_t local = 0;
#ifdef FTB_PROD_PROFILE
    unsigned long long c_wait = 0, c_issue = 0, c_item = 0, c_t0 = clock64();
#endif
    TcPair cur, nxt;
    uint32_t pend = 0;
    if (cid < n_work) cur = bcast_record<TcPair>(fetch_record_word(work, cid));
    if (cid + G < n_work) nxt = bcast_record<TcPair>(fetch_record_word(work, cid + G));
    if (cid + 2 * G < n_work) pend = fetch_record_word(work, cid + 2 * G);
    for (int w = cid; w < n_work; w += G, ++local) {
      const TcPair it = cur;
      if (lane == 0) {
        trace2_ev(cfg, local, 0);
        if (w + G < n_work) {
          tma_prefetch_desc(&nxt.maps->lane);
          tma_prefetch_desc(&nxt.maps->col[1]);
        }
      }
#ifdef FTB_PROD_PROFILE
      unsigned long long ci = clock64();
#endif
      const bool lane_mn = it.flags & kFlagLaneMN, col_mn = it.flags & kFlagColMN;
      const int half = it.n_mma >> 1;
      const int lane0 = rank ? it.lane0[1] : it.lane0[0];
      const int colr = it.col0 + static_cast<int>(rank) * half;
      const uint32_t bytes_cta = kLaneStageBytes + static_cast<uint32_t>(half) * kBlockK * 2;
      const uint32_t cmask = col_box_mask(half);
      int boff[kColMaps];  // smem row offset of each column box (widest first)
      {
        int r = 0;
#pragma unroll
        for (int q = 0; q < kColMaps; ++q) {
          boff[q] = r;
          if (cmask & (1u << q)) r += 256 >> q;
        }
      }
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
          const uint32_t fb = smem_addr(&full[s]) & kPeerBitMask;  // leader's barrier
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * bytes_cta);
          uint8_t* ldst = lane_buf + s * kLaneStageBytes;
          uint8_t* cdst = col_buf + s * cfg.col_stage_bytes;
          const int k0 = kb * kBlockK;
          if (!lane_mn) {
            tma_load_3d_pair(ldst, &it.maps->lane, fb, k0, lane0, it.batch);
          } else {
            tma_load_3d_pair(ldst, &it.maps->lane, fb, lane0, k0, it.batch);
            tma_load_3d_pair(ldst + 8192, &it.maps->lane, fb, lane0 + 64, k0, it.batch);
          }
          if (!col_mn) {
#pragma unroll
            for (int q = 0; q < kColMaps; ++q)
              if (cmask & (1u << q))
                tma_load_3d_pair(cdst + boff[q] * 128, &it.maps->col[q], fb, k0, colr + boff[q], it.batch);
          } else {
            for (int c = 0; c < half; c += 64)
              tma_load_3d_pair(cdst + c * 128, &it.maps->col[0], fb, colr + c, k0, it.batch);
          }
          if (kb == 0) trace2_ev(cfg, local, 1);
          trace2_kb(cfg, g, 0);
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
      if (w + 2 * G < n_work) nxt = bcast_record<TcPair>(pend);
      if (w + 3 * G < n_work) pend = fetch_record_word(work, w + 3 * G);
    }
#ifdef FTB_PROD_PROFILE
    if (lane == 0 && cfg.trace) {
      unsigned long long* t = cfg.trace + static_cast<size_t>(blockIdx.x) * kTracePerCta;
      t[0] = c_wait; t[1] = c_issue; t[2] = c_item; t[3] = g; t[4] = local; t[5] = clock64() - c_t0;
    }
#endif
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    // whole warp walks the loops; tcgen05.mma / commits issued converged with elect.sync
    if (leader) {
      uint32_t g = 0;
      uint32_t ms = 0, mphase = 0;  // MMA ring slot / phase
      uint32_t local = 0;
      uint32_t pend = 0;
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t lane_u32 = smem_addr(lane_buf), col_u32 = smem_addr(col_buf);
#ifdef FTB_PROD_PROFILE
      unsigned long long m_te = 0, m_full = 0, m_issue = 0, m_t0 = clock64();
#endif
      if (cid < n_work) pend = fetch_record_word(work, cid);
      for (int w = cid; w < n_work; w += G, ++local) {
        const TcPair it = bcast_record<TcPair>(pend);
        if (w + G < n_work) pend = fetch_record_word(work, w + G);
        const uint32_t slot = local % cfg.n_acc;
        const uint32_t use = local / cfg.n_acc;
        const uint32_t lane_mn = (it.flags & kFlagLaneMN) ? 1u : 0u;
        const uint32_t col_mn = (it.flags & kFlagColMN) ? 1u : 0u;
#ifdef FTB_PROD_PROFILE
        unsigned long long mt0 = clock64();
#endif
        mbar_wait(&tempty[slot], (use & 1) ^ 1);
        tc_fence_after();
#ifdef FTB_PROD_PROFILE
        m_te += clock64() - mt0;
#endif
        const uint32_t tmem_d = tmem_u + slot * cfg.acc_cols;
        const uint32_t idesc = idesc_bf16_f32(2 * kLaneRows, static_cast<uint32_t>(it.n_mma), lane_mn, col_mn);
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
            if (kb == 0) trace2_ev(cfg, local, 2);
            trace2_kb(cfg, g, 1);
          }
          const uint32_t la = lane_u32 + s * kLaneStageBytes;
          const uint32_t ca = col_u32 + s * static_cast<uint32_t>(cfg.col_stage_bytes);
#pragma unroll
          for (int kk = 0; kk < kBlockK / 16; ++kk) {
            const uint64_t adesc = lane_mn ? umma_desc_sw128(la + kk * 2048, 8192, 1024)
                                           : umma_desc_sw128(la + kk * 32, 16, 1024);
            const uint64_t bdesc = col_mn ? umma_desc_sw128(ca + kk * 2048, 8192, 1024)
                                          : umma_desc_sw128(ca + kk * 32, 16, 1024);
            tc_mma_f16_pair_elect(tmem_d, adesc, bdesc, idesc, (kb | kk) != 0);
          }
          tc_commit_pair_mc_elect(smem_addr(&empty[s]));
          __syncwarp();
#ifdef FTB_PROD_PROFILE
          m_issue += clock64() - mf1;
#endif
        }
        tc_commit_pair_mc_elect(smem_addr(&tfull[slot]));
        if (lane == 0) trace2_ev(cfg, local, 3);
        __syncwarp();
      }
#ifdef FTB_PROD_PROFILE
      if (lane == 0 && cfg.trace) {
        unsigned long long* t = cfg.trace + static_cast<size_t>(blockIdx.x) * kTracePerCta;
        t[6] = m_te; t[7] = m_full; t[8] = m_issue; t[9] = clock64() - m_t0;
      }
#endif
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int quad = warp & 3;
    uint8_t* region = reinterpret_cast<uint8_t*>(epi_buf) + quad * kEpiWarpBytes;
    uint32_t local = 0, ngrp = 0;
#ifdef FTB_PROD_PROFILE
    unsigned long long e_wait = 0, e_t0 = clock64();
#endif
    TcPair nxt;
    if (cid < n_work) nxt = load_pair(work, cid);
    for (int w = cid; w < n_work; w += G, ++local) {
      const TcPair it = nxt;
      if (w + G < n_work) nxt = load_pair(work, w + G);  // lands while this item runs
      const uint32_t slot = local % cfg.n_acc;
      const uint32_t use = local / cfg.n_acc;
      const bool swap = it.flags & kFlagSwap, f32 = it.flags & kFlagOutF32;
      const bool tma = it.flags & kFlagTmaStore;
      const int lane_len = rank ? it.lane_len[1] : it.lane_len[0];
      const int lane0 = rank ? it.lane0[1] : it.lane0[0];
#ifdef FTB_PROD_PROFILE
      unsigned long long ew0 = clock64();
#endif
      mbar_wait(&tfull[slot], use & 1);
#ifdef FTB_PROD_PROFILE
      e_wait += clock64() - ew0;
#endif
      tc_fence_after();
      if (quad == 0 && lane == 0) trace2_ev(cfg, local, 4);
      const int lane_base = quad * 32;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lane_base) << 16) + slot * cfg.acc_cols;
      epilogue_tile(
          region, ngrp, taddr, lane_base < lane_len, tma, swap, f32, &it.maps->out, it.C, it.ldc, lane0, lane_len,
          lane_base, it.col0, it.col_len, it.batch,
          [&] {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(smem_addr(&tempty[slot]) & kPeerBitMask);
          },
          (it.flags & kFlagEpiOp) ? &it.maps->epi : nullptr);
      if (quad == 0 && lane == 0) trace2_ev(cfg, local, 5);
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
  cluster_sync();  // no CTA leaves while its peer may still touch its smem / barriers
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<kTmemCols>(tmem_base);
  }
}

int tc_smem_bytes(const TcConfig& cfg);

template <int S>
static cudaError_t launch_tc2_s(const TcPair* work, int32_t n_work, int32_t n_ctas, TcConfig cfg,
                                cudaStream_t stream) {
  cudaError_t e = configure_smem_once<ftb_tc2_kernel<S>>(232448);
  if (e != cudaSuccess) return e;
  return launch_pdl(ftb_tc2_kernel<S>, n_ctas, kTcThreads, tc_smem_bytes(cfg), stream, work, n_work, cfg);
}

cudaError_t launch_tc2(const TcPair* work, int32_t n_work, int32_t n_ctas, TcConfig cfg,
                       cudaStream_t stream) {
  if (n_work == 0) return cudaSuccess;
  switch (cfg.stages) {
    case 2: return launch_tc2_s<2>(work, n_work, n_ctas, cfg, stream);
    case 3: return launch_tc2_s<3>(work, n_work, n_ctas, cfg, stream);
    case 4: return launch_tc2_s<4>(work, n_work, n_ctas, cfg, stream);
    case 5: return launch_tc2_s<5>(work, n_work, n_ctas, cfg, stream);
    case 6: return launch_tc2_s<6>(work, n_work, n_ctas, cfg, stream);
    case 7: return launch_tc2_s<7>(work, n_work, n_ctas, cfg, stream);
    case 8: return launch_tc2_s<8>(work, n_work, n_ctas, cfg, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ftb
