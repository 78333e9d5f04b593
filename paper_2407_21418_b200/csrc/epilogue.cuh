// epilogue.cuh — shared epilogue helpers of the tcgen05 kernels: row-segment
// stores (16-B vectorised when the destination is aligned and the segment is
// full, element-predicated on ragged uKernel edges) and %globaltimer.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "exec_types.h"
#include "ptx.cuh"

namespace ftb {

__device__ __forceinline__ bool aligned16(const void* C, int64_t off, bool f32) {
  return ((reinterpret_cast<uintptr_t>(C) + static_cast<uintptr_t>(off) * (f32 ? 4u : 2u)) & 15u) == 0;
}

__device__ __forceinline__ void store_row32(void* C, int64_t off, const float* v, int n, bool f32,
                                            bool vec_ok) {
  if (f32) {
    float* dst = static_cast<float*>(C) + off;
    if (vec_ok && n == 32) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        __stcg(reinterpret_cast<float4*>(dst) + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (e < n) __stcg(dst + e, v[e]);
    }
  } else {
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(C) + off;
    if (vec_ok && n == 32) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 pk;
        uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
          pw[e] = *reinterpret_cast<uint32_t*>(&h);
        }
        __stcg(reinterpret_cast<uint4*>(dst) + q, pk);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (e < n) __stcg(reinterpret_cast<unsigned short*>(dst) + e, __bfloat16_as_ushort(__float2bfloat16_rn(v[e])));
    }
  }
}

// Store a 32 x 32 fp32 block that a warp holds in registers — one ROW of C
// per lane (lane_is_row) or one COLUMN of C per lane — to C[row0.., col0..]
// (clipped to nrows x ncols). The block goes through a padded smem tile
// (32 x 33 fp32, conflict-free both ways); each lane then writes 8
// consecutive elements of one row per pass, so one warp store instruction
// covers 8 rows x 8 elements x 4 lanes = 8 full 64-B (bf16) row segments
// instead of 32 scattered 16-B pieces.
__device__ __forceinline__ void store_rows8(const float* tb, int rl, int r, int cq, void* C, int64_t ldc,
                                           int64_t row0, int64_t col0, int nrows, int ncols, bool f32) {
  if (r < nrows && cq < ncols) {
    float e[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) e[q] = tb[rl * 33 + cq + q];
    const int64_t off = (row0 + r) * ldc + col0 + cq;
    const int n = min(8, ncols - cq);
    if (f32) {
      float* dst = static_cast<float*>(C) + off;
      if (n == 8 && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
        __stcg(reinterpret_cast<float4*>(dst), make_float4(e[0], e[1], e[2], e[3]));  // st.global: C is device memory
        __stcg(reinterpret_cast<float4*>(dst) + 1, make_float4(e[4], e[5], e[6], e[7]));
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < n) __stcg(dst + q, e[q]);
      }
    } else {
      __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(C) + off;
      if (n == 8 && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
        uint4 pk;
        uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          __nv_bfloat162 h = __floats2bfloat162_rn(e[2 * q], e[2 * q + 1]);
          pw[q] = *reinterpret_cast<uint32_t*>(&h);
        }
        __stcg(reinterpret_cast<uint4*>(dst), pk);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < n) __stcg(reinterpret_cast<unsigned short*>(dst) + q, __bfloat16_as_ushort(__float2bfloat16_rn(e[q])));
      }
    }
  }
}

__device__ __forceinline__ void store_block32(float* tb, const float (&v)[32], bool lane_is_row, void* C,
                                              int64_t ldc, int64_t row0, int64_t col0, int nrows, int ncols,
                                              bool f32) {
  const int lane = threadIdx.x & 31;
  const int cq = (lane & 3) * 8;
  if (lane_is_row) {
#pragma unroll
    for (int x = 0; x < 32; ++x) tb[lane * 33 + x] = v[x];
  } else {
#pragma unroll
    for (int x = 0; x < 32; ++x) tb[x * 33 + lane] = v[x];
  }
  __syncwarp();
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int r = (lane >> 2) + 8 * p;
    store_rows8(tb, r, r, cq, C, ldc, row0, col0, nrows, ncols, f32);
  }
  __syncwarp();
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

}  // namespace ftb

namespace ftb {
// ---------------------------------------------------------------- TMA store epilogue
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, uint32_t src, int32_t c0, int32_t c1,
                                             int32_t c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// 1-D bulk copy shared -> global (16-B aligned addresses, size a multiple of 16)
__device__ __forceinline__ void bulk_store_1d(void* gdst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(gdst)),
               "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Write a warp's 32 x 32 fp32 accumulator block as bf16 into a TMA store box
// (32 C rows x 64 B, SWIZZLE_64B: 16-B chunk index ^= row bits [1,3)); the box
// must be 512-B aligned. lane_is_row: lane l holds C row l (normal
// orientation); otherwise lane l holds C column l and register e is C row e.
__device__ __forceinline__ void stage_box_bf16(uint8_t* box, const uint32_t (&r)[32], bool lane_is_row) {
  const int l = threadIdx.x & 31;
  if (lane_is_row) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 pk;
      uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[q * 8 + 2 * e]), __uint_as_float(r[q * 8 + 2 * e + 1]));
        pw[e] = *reinterpret_cast<uint32_t*>(&h);
      }
      *reinterpret_cast<uint4*>(box + l * 64 + ((q ^ ((l >> 1) & 3)) * 16)) = pk;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 32; ++e)
      *reinterpret_cast<__nv_bfloat16*>(box + e * 64 + (((l >> 3) ^ ((e >> 1) & 3)) * 16) + (l & 7) * 2) =
          __float2bfloat16_rn(__uint_as_float(r[e]));
  }
}

// ---------------------------------------------------------------- fused epilogue op
__device__ __forceinline__ float gelu_erf(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float load_bias(const EpiOp& op, int c) {
  if (!op.bias || c < 0 || c >= op.n) return 0.f;
  return op.bias_f32 ? __ldg(static_cast<const float*>(op.bias) + c)
                     : __bfloat162float(static_cast<const __nv_bfloat16*>(op.bias)[c]);
}
// acc + bias[column], then the activation, on a warp's 32 x 32 chunk (fp32 bits
// in `r`). lane_is_row: lane l is a C row and register e is C column
// col_base + e; otherwise lane l is C column col_base + l (every register).
__device__ __forceinline__ void apply_epi(uint32_t (&r)[32], const EpiOp& op, bool lane_is_row, int col_base) {
  const int l = threadIdx.x & 31;
  const float bl = load_bias(op, col_base + l);
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    float x = __uint_as_float(r[e]) + (lane_is_row ? __shfl_sync(0xffffffffu, bl, e) : bl);
    if (op.act == 1) x = gelu_erf(x);
    r[e] = __float_as_uint(x);
  }
}

// One epilogue warp's share of a finished work item: TMEM lanes
// [lane_base, lane_base + 32) of the accumulator at `taddr`, columns
// [0, col_len). C-side coordinates: normal orientation (swap = false) stores
// lane l as C row lane0 + lane_base + l; swap-AB stores it as C column.
// `release()` hands the accumulator back to the MMA warp right after the
// last TMEM read. `region` is the warp's 8 KiB staging area (four 2 KiB TMA
// boxes or the 32x33 fp32 transpose tile), `ngrp` its running box-group count.
// `op` (or null): fused bias + activation applied before rounding.
#ifdef FTB_EPI_TRACE
// debug: per-CTA epilogue timestamps of warp 4 (lane quadrant 0), first item
// (a device global, not __shared__: static smem would overflow the 227 KiB opt-in)
__device__ unsigned long long* ftb_epi_dbg;
#define FTB_EPI_EV(i)                                                                                   \
  do {                                                                                                  \
    unsigned long long* d_ = ftb_epi_dbg ? ftb_epi_dbg + static_cast<size_t>(blockIdx.x) * kTracePerCta \
                                                + kTraceItems * kTraceEvents + 2 * 40                    \
                                         : nullptr;                                                      \
    if (d_ && (threadIdx.x >> 5) == 4 && (threadIdx.x & 31) == 0) d_[i] = clock64();  \
  } while (0)
#else
#define FTB_EPI_EV(i) \
  do {                \
  } while (0)
#endif

// kFlagBulkStore: this warp's C rows [lane0 + lane_base, + nrows) are whole
// rows of a compact C (col_len == ldc), i.e. one contiguous byte range. Rows
// are staged in the warp's 8 KiB region in C's own layout, at the same
// address phase mod 16 as their destination, so one 1-D bulk copy writes the
// 16-B aligned interior; the < 16 B head and tail go out as element stores.
// (Scores BMMs with T % 8 != 0: their rows are not a multiple of 16 B, which
// no TMA tensor map can describe.)
template <class Release>
__device__ __forceinline__ bool bulk_rows(uint8_t* region, uint32_t taddr, bool f32, void* C, int64_t ldc, int row0,
                                          int nrows, int col_len, int col0, Release& release, const EpiOp* op) {
  const int lane = threadIdx.x & 31;
  const int esz = f32 ? 4 : 2;
  const int rowb = col_len * esz;
  const int rows_per = min(nrows, (8192 - 16) / rowb);
  if (rows_per <= 0) return false;
  char* gbase = static_cast<char*>(C) + static_cast<int64_t>(row0) * ldc * esz;
  bool released = false;
  for (int ra = 0; ra < nrows; ra += rows_per) {
    const int rb = min(nrows, ra + rows_per);
    char* g0 = gbase + static_cast<int64_t>(ra) * rowb;
    const int nbytes = (rb - ra) * rowb;
    const uintptr_t ga = reinterpret_cast<uintptr_t>(g0);
    uint8_t* sb = region + (ga & 15u);
    if (lane == 0) bulk_wait_read<0>();  // the region's previous bulk / TMA stores have read it
    __syncwarp();
    for (int c0 = 0; c0 < col_len; c0 += 32) {
      uint32_t raw[32];
      tmem_ld_32x32b_x32(taddr + c0, raw);
      tmem_ld_wait();
      if (rb >= nrows && c0 + 32 >= col_len) {  // last TMEM read of the item
        release();
        released = true;
      }
      if (op) apply_epi(raw, *op, true, col0 + c0);
      if (lane >= ra && lane < rb) {
        uint8_t* dst = sb + (lane - ra) * rowb + c0 * esz;
        const int n = min(32, col_len - c0);
        if (f32) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e < n) reinterpret_cast<float*>(dst)[e] = __uint_as_float(raw[e]);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e < n) reinterpret_cast<__nv_bfloat16*>(dst)[e] = __float2bfloat16_rn(__uint_as_float(raw[e]));
        }
      }
    }
    fence_async_smem();
    __syncwarp();
    const uintptr_t a0 = (ga + 15) & ~uintptr_t(15), a1 = (ga + nbytes) & ~uintptr_t(15);
    if (a1 > a0) {
      if (lane == 0) {
        bulk_store_1d(reinterpret_cast<void*>(a0), smem_addr(sb + (a0 - ga)), static_cast<uint32_t>(a1 - a0));
        bulk_commit();
      }
      const int nh = static_cast<int>(a0 - ga) / esz, nt = static_cast<int>(ga + nbytes - a1) / esz;
      int off = -1;
      if (lane < nh) off = lane * esz;
      else if (lane >= 16 && lane - 16 < nt) off = static_cast<int>(a1 - ga) + (lane - 16) * esz;
      if (off >= 0) {
        if (f32) __stcg(reinterpret_cast<float*>(g0 + off), *reinterpret_cast<const float*>(sb + off));
        else __stcg(reinterpret_cast<unsigned short*>(g0 + off), *reinterpret_cast<const unsigned short*>(sb + off));
      }
    } else {
      for (int off = lane * esz; off < nbytes; off += 32 * esz) {
        if (f32) __stcg(reinterpret_cast<float*>(g0 + off), *reinterpret_cast<const float*>(sb + off));
        else __stcg(reinterpret_cast<unsigned short*>(g0 + off), *reinterpret_cast<const unsigned short*>(sb + off));
      }
    }
  }
  if (!released) release();
  return true;
}

template <class Release>
__device__ __forceinline__ void epilogue_tile(uint8_t* region, uint32_t& ngrp, uint32_t taddr, bool active, bool tma,
                                              bool swap, bool f32, const CUtensorMap* out_map, void* C, int64_t ldc,
                                              int lane0, int lane_len, int lane_base, int col0, int col_len, int batch,
                                              Release release, const EpiOp* op = nullptr, bool bulk = false,
                                              int tail0 = 1 << 30) {
  const int lane = threadIdx.x & 31;
  bool released = false;
  if (active && bulk && !tma && !swap &&
      bulk_rows(region, taddr, f32, C, ldc, lane0 + lane_base, min(32, lane_len - lane_base), col_len, col0, release, op)) {
    ngrp |= 0x80000000u;  // the last bulk copy may still read any part of the region (see below)
    return;
  }
  if (active) {
    if (tma) {
      // groups of two 32-column chunks: both tcgen05.ld in flight, one proxy
      // fence and one bulk group per pair of TMA stores
      for (int c0 = 0; c0 < col_len; c0 += 64) {
        const bool two = c0 + 32 < col_len;
        uint32_t ra[32], rb[32];
        tmem_ld_32x32b_x32(taddr + c0, ra);
        if (two) tmem_ld_32x32b_x32(taddr + c0 + 32, rb);
        tmem_ld_wait();
        FTB_EPI_EV((c0 >> 6) * 6 + 0);
        if (c0 + 64 >= col_len) {  // last TMEM read of the item
          release();
          released = true;
        }
#ifdef FTB_NULL_EPI
        continue;  // experiment build: accumulators drained, nothing staged or stored
#endif
        if (op) {  // normal: TMEM columns are C columns; swap-AB: lanes are
          apply_epi(ra, *op, !swap, swap ? lane0 + lane_base : col0 + c0);
          if (two) apply_epi(rb, *op, !swap, swap ? lane0 + lane_base : col0 + c0 + 32);
        }
        uint8_t* box = region + (ngrp & 1) * 4096;
        if (ngrp >> 31) {  // a bulk copy of a previous item spans both boxes
          if (lane == 0) bulk_wait_read<0>();
          ngrp &= 0x7fffffffu;
        } else if (lane == 0) {
          bulk_wait_read<1>();  // the group that last used these boxes has read them
        }
        __syncwarp();
        FTB_EPI_EV((c0 >> 6) * 6 + 1);
        stage_box_bf16(box, ra, !swap);
        if (two) stage_box_bf16(box + 2048, rb, !swap);
        FTB_EPI_EV((c0 >> 6) * 6 + 2);
        fence_async_smem();
        __syncwarp();
        FTB_EPI_EV((c0 >> 6) * 6 + 3);
        if (c0 + 64 > tail0 && lane < lane_len - lane_base) {
          // kFlagTmaTail: columns [tail0, col_len) (< 8, starting on a
          // multiple of 8, so inside one 16-B chunk of a staged box and at a
          // 16-B aligned address of C) lie past the store map's end (N
          // rounded down to 8); this lane's row writes them as 8 + 4 + 2 B
          // pieces of that chunk (row `lane` of a box: chunk q at (q ^ ((lane >> 1) & 3)) * 16)
          const int cc = (tail0 - c0) & 31;
          const uint4 v = *reinterpret_cast<const uint4*>(box + ((tail0 - c0) >> 5) * 2048 + lane * 64 +
                                                          (((cc >> 3) ^ ((lane >> 1) & 3)) * 16));
          char* dst = reinterpret_cast<char*>(static_cast<__nv_bfloat16*>(C) +
                                              static_cast<int64_t>(lane0 + lane_base + lane) * ldc + col0 + tail0);
          const int n = col_len - tail0;
          uint32_t w[4] = {v.x, v.y, v.z, v.w};
          int at = 0;
          if (n >= 4) {
            *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
            at = 2;
          }
          if (n & 2) {
            *reinterpret_cast<uint32_t*>(dst + at * 4) = at ? w[2] : w[0];
            ++at;
          }
          if (n & 1) {
            const uint32_t last = at == 0 ? w[0] : (at == 1 ? w[1] : (at == 2 ? w[2] : w[3]));
            *reinterpret_cast<unsigned short*>(dst + at * 4) = static_cast<unsigned short>(last & 0xffffu);
          }
        }
#ifdef FTB_EPI_NOSTORE
        if (false) {  // experiment build: staged but never stored
#else
        if (lane == 0) {
#endif
          const int l0 = lane0 + lane_base, k0 = col0 + c0;
          if (!swap) {
            tma_store_3d(out_map, smem_addr(box), k0, l0, batch);
            FTB_EPI_EV((c0 >> 6) * 6 + 4);
            if (two) tma_store_3d(out_map, smem_addr(box + 2048), k0 + 32, l0, batch);
          } else {
            tma_store_3d(out_map, smem_addr(box), l0, k0, batch);
            if (two) tma_store_3d(out_map, smem_addr(box + 2048), l0, k0 + 32, batch);
          }
          bulk_commit();
        }
        FTB_EPI_EV((c0 >> 6) * 6 + 5);
        ++ngrp;
      }
    } else {
      float* tb = reinterpret_cast<float*>(region);
      if (lane == 0) bulk_wait_read<0>();  // the transpose tile aliases this warp's store boxes
      __syncwarp();
      for (int c0 = 0; c0 < col_len; c0 += 32) {
        uint32_t raw[32];
        tmem_ld_32x32b_x32(taddr + c0, raw);
        tmem_ld_wait();
        if (op) apply_epi(raw, *op, !swap, swap ? lane0 + lane_base : col0 + c0);
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(raw[e]);
        const int ncol = min(32, col_len - c0);
        const int nlane = min(32, lane_len - lane_base);
        // the 32 x 32 block goes through the smem transpose so every store
        // writes 8 rows x 64 B (measured: each lane storing its own row
        // straight from registers is 2x slower on C2 scores T = 100 / 257)
        if (!swap)  // lanes = rows of C, TMEM columns = output columns
          store_block32(tb, v, true, C, ldc, lane0 + lane_base, col0 + c0, nlane, ncol, f32);
        else        // lanes = columns of C, TMEM columns = output rows
          store_block32(tb, v, false, C, ldc, col0 + c0, lane0 + lane_base, ncol, nlane, f32);
      }
    }
  }
  if (!released) release();
}

}  // namespace ftb
