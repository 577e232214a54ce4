// Stages S3 (emit) and S4 (table) of the WAH build on sm_100a.
//
// S3 replaces, in ONE streaming pass over the sorted (value,row) pairs, the
// reference's run_head / scan / read_total / run_start / run_fold /
// value_head / scan / read_total / value_start / emit_words / count_words /
// scan kernels and the three compaction actors
// (p/core/src/wah_builder.cpp:65-285, p/core/src/wah_stages.cpp:29-163).
//
// Per element i of the sorted stream (value v, row r, chunk c = r/31):
//   run head   i==0 or v/c differ from element i-1          (wah_builder.cpp:74-75)
//   literal    OR of 1<<(row%31) over the run (<= 31 elems) (wah_builder.cpp:120-123)
//   gap        c - c_prev - 1 inside a value, c at a value head (wah_builder.cpp:190-192)
//   body       literal, or ONE ones-fill for a maximal stretch of all-ones
//              runs (later runs of the stretch are swallowed) (wah_builder.cpp:193-205)
// All of it is local to a +-31-element window, except a ones-stretch length,
// found by galloping over the sorted pairs: pair[i+t] == (v, r+t) is
// monotone in t because rows are strictly increasing inside a value.
// Word and value counts are scanned inside the tile and across tiles with a
// decoupled look-back, and the compacted words are written straight to their
// final position -- no zero-padded fill/body arrays, no host round trip.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../../include/ndx.h"
#include "common.cuh"
#include "wah_internal.cuh"

namespace ndx {

constexpr int kEmitThreads = 512;
constexpr int kEmitWarps = kEmitThreads / 32;
constexpr int kEmitIPT = 8;
constexpr int kEmitWarpItems = 32 * kEmitIPT;        // 256
constexpr int kEmitTile = kEmitThreads * kEmitIPT;   // 4096
constexpr int kHalo = 32;                            // >= 31 on each side

__device__ __forceinline__ uint32_t pkey(uint64_t e) { return uint32_t(e); }
__device__ __forceinline__ uint32_t prow(uint64_t e) { return uint32_t(e >> 32); }

// Largest t with pairs[g+t] == (v, row+t), given that it holds for t = 30.
__device__ uint32_t stretch_end(const uint64_t* __restrict__ pairs, uint64_t n, uint64_t g,
                                uint32_t v, uint32_t row) {
  auto P = [&](uint64_t t) -> bool {
    if (g + t >= n) return false;
    uint64_t rr = uint64_t(row) + t;
    if (rr > 0xffffffffull) return false;
    uint64_t e = pairs[g + t];
    return pkey(e) == v && prow(e) == uint32_t(rr);
  };
  uint64_t lo = 30, hi, step = 32;
  for (;;) {
    uint64_t cand = lo + step;
    if (!P(cand)) {
      hi = cand;
      break;
    }
    lo = cand;
    step <<= 1;
  }
  while (hi - lo > 1) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (P(mid))
      lo = mid;
    else
      hi = mid;
  }
  return uint32_t(lo);
}

struct EmitScratch {
  uint64_t* val_agg;
  uint64_t* val_pre;
  uint32_t* status;
};

__global__ __launch_bounds__(kEmitThreads) void k_emit(const uint64_t* __restrict__ pairs,
                                                       uint64_t n, Ctl* ctl,
                                                       uint32_t* __restrict__ words,
                                                       uint32_t* __restrict__ vstart,
                                                       uint32_t* __restrict__ values,
                                                       EmitScratch sc, uint32_t epoch_in) {
  extern __shared__ __align__(16) unsigned char emit_smem[];
  uint64_t* win = reinterpret_cast<uint64_t*>(emit_smem);       // [kEmitTile + 2 kHalo]
  uint32_t* ow = reinterpret_cast<uint32_t*>(win + kEmitTile + 2 * kHalo);  // [2 kEmitTile]
  __shared__ uint32_t warp_tot[kEmitWarps];
  __shared__ uint32_t s_tile, s_w0, s_d0, s_tot;

  const uint32_t epoch = (epoch_in + 6u) & 0xffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (n + kEmitTile - 1) / kEmitTile;

  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&ctl->tile_ctr[0], 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint64_t tile_start = tile * kEmitTile;
    const uint32_t m = uint32_t(umin<uint64_t>(kEmitTile, n - tile_start));

    // ---- window [tile_start - 32, tile_start + m + 32)
    for (uint32_t j = threadIdx.x; j < m + 2 * kHalo; j += kEmitThreads) {
      const int64_t g = int64_t(tile_start) - kHalo + j;
      win[j] = (g >= 0 && uint64_t(g) < n) ? ldg_stream(pairs + g) : 0ull;
    }
    __syncthreads();

    // ---- per element: words and value heads (warp-contiguous rounds)
    uint32_t body[kEmitIPT], gapw[kEmitIPT], exw[kEmitIPT];
    uint32_t carry = 0;
#pragma unroll
    for (int r = 0; r < kEmitIPT; ++r) {
      const uint32_t li = uint32_t(warp) * kEmitWarpItems + r * 32 + lane;
      const uint64_t g = tile_start + li;
      uint32_t cnt = 0;
      body[r] = 0;
      gapw[r] = 0;
      if (li < m) {
        const uint64_t cur = win[li + kHalo];
        const uint32_t v = pkey(cur), row = prow(cur), c = row / kChunkBits;
        bool head = true, vhead = true;
        uint32_t pc = 0;
        if (g > 0) {
          const uint64_t pe = win[li + kHalo - 1];
          pc = prow(pe) / kChunkBits;
          vhead = pkey(pe) != v;
          head = vhead || pc != c;
        }
        if (head) {
          uint32_t lit = 0;
          for (uint32_t j = li; j < li + kChunkBits; ++j) {
            if (tile_start + j >= n) break;
            const uint64_t e = win[j + kHalo];
            if (pkey(e) != v || prow(e) / kChunkBits != c) break;
            lit |= 1u << (prow(e) % kChunkBits);
          }
          const uint32_t gap = vhead ? c : c - pc - 1;
          uint32_t b = lit;
          if (lit == kLiteralMask) {
            // swallowed when the previous run is the all-ones chunk c-1
            const bool prev_ones = !vhead && gap == 0 && g >= kChunkBits &&
                                   win[li + kHalo - kChunkBits] ==
                                       (uint64_t(v) | (uint64_t(row - kChunkBits) << 32));
            if (prev_ones) {
              b = 0;
            } else {
              const uint32_t t = stretch_end(pairs, n, g, v, row);
              const uint32_t len = (row + t + 1) / kChunkBits - c;
              b = make_fill(true, len);
            }
          }
          body[r] = b;
          gapw[r] = gap ? make_fill(false, gap) : 0u;
          cnt = ((uint32_t(gap != 0) + uint32_t(b != 0)) << 16) | uint32_t(vhead);
        }
      }
      const uint32_t incl = warp_incl_sum(cnt);
      exw[r] = carry + incl - cnt;
      carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) warp_tot[warp] = carry;
    __syncthreads();

    // ---- tile scan over warps; publish the tile aggregate right away
    if (warp == 0) {
      const uint32_t t = lane < kEmitWarps ? warp_tot[lane] : 0;
      const uint32_t ti = warp_incl_sum(t);
      if (lane < kEmitWarps) warp_tot[lane] = ti - t;
      const uint32_t tot = __shfl_sync(kFull, ti, 31);
      if (lane == 0) {
        s_tot = tot;
        const uint64_t agg = uint64_t(tot >> 16) | (uint64_t(tot & 0xffffu) << 32);
        if (tile == 0) {
          st_relaxed_u64(&sc.val_pre[0], agg);
          st_release_u32(&sc.status[0], (epoch << 16) | 2u);
        } else {
          st_relaxed_u64(&sc.val_agg[tile], agg);
          st_release_u32(&sc.status[tile], (epoch << 16) | 1u);
        }
      }
    }
    __syncthreads();

    // ---- stage the tile's words at tile-local offsets (no global offset needed)
    const uint32_t woff = warp_tot[warp];
#pragma unroll
    for (int r = 0; r < kEmitIPT; ++r) {
      const uint32_t li = uint32_t(warp) * kEmitWarpItems + r * 32 + lane;
      if (li >= m) continue;
      uint32_t o = (woff + exw[r]) >> 16;
      if (gapw[r]) ow[o++] = gapw[r];
      if (body[r]) ow[o] = body[r];
    }

    // ---- decoupled look-back (warp 0) for the tile's global offsets
    if (warp == 0) {
      const uint32_t tot = s_tot;
      const uint64_t agg = uint64_t(tot >> 16) | (uint64_t(tot & 0xffffu) << 32);
      uint64_t excl = 0;
      if (tile > 0) {
        int64_t base = int64_t(tile) - 1;
        for (;;) {
          const int64_t tt = base - lane;
          uint64_t val = 0;
          bool pre = true;
          if (tt >= 0) {
            uint32_t s = ld_acquire_u32(&sc.status[tt]);
            while ((s >> 16) != epoch || (s & 3u) == 0) {
              __nanosleep(20);
              s = ld_acquire_u32(&sc.status[tt]);
            }
            pre = (s & 3u) == 2u;
            val = pre ? ld_relaxed_u64(&sc.val_pre[tt]) : ld_relaxed_u64(&sc.val_agg[tt]);
          }
          const unsigned pm = __ballot_sync(kFull, pre);
          if (pm && lane > __ffs(pm) - 1) val = 0;
          excl += __shfl_sync(kFull, warp_incl_sum64(val), 31);
          if (pm) break;
          base -= 32;
        }
        if (lane == 0) {
          st_relaxed_u64(&sc.val_pre[tile], excl + agg);
          st_release_u32(&sc.status[tile], (epoch << 16) | 2u);
        }
      }
      if (lane == 0) {
        s_w0 = uint32_t(excl);
        s_d0 = uint32_t(excl >> 32);
        if (tile == ntiles - 1) {
          ctl->words = uint64_t(uint32_t(excl)) + (tot >> 16);
          ctl->distinct = uint64_t(uint32_t(excl >> 32)) + (tot & 0xffffu);
        }
      }
    }
    __syncthreads();

    // ---- table rows (value heads) straight to HBM
    const uint32_t w0 = s_w0, d0 = s_d0;
#pragma unroll
    for (int r = 0; r < kEmitIPT; ++r) {
      const uint32_t li = uint32_t(warp) * kEmitWarpItems + r * 32 + lane;
      if (li >= m) continue;
      const uint64_t g = tile_start + li;
      const uint64_t cur = win[li + kHalo];
      const bool vhead = g == 0 || pkey(win[li + kHalo - 1]) != pkey(cur);
      if (vhead) {
        const uint32_t ex = woff + exw[r];
        const uint32_t dd = d0 + (ex & 0xffffu);
        vstart[dd] = w0 + (ex >> 16);
        values[dd] = pkey(cur);
      }
    }
    const uint32_t tw = s_tot >> 16;
    for (uint32_t j = threadIdx.x; j < tw; j += kEmitThreads) words[uint64_t(w0) + j] = ow[j];
    __syncthreads();
  }
}

// S4: (value, offset, length) rows (wah_builder.cpp:238-257).
__global__ void k_table(const uint32_t* __restrict__ values, const uint32_t* __restrict__ vstart,
                        const Ctl* ctl, uint32_t* __restrict__ entries) {
  const uint64_t D = ctl->distinct, W = ctl->words;
  for (uint64_t d = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t lo = vstart[d];
    const uint32_t hi = d + 1 < D ? vstart[d + 1] : uint32_t(W);
    entries[3 * d] = values[d];
    entries[3 * d + 1] = lo;
    entries[3 * d + 2] = hi - lo;
  }
}

constexpr size_t kEmitSmem = size_t(kEmitTile + 2 * kHalo) * 8 + size_t(2 * kEmitTile) * 4;

static uint64_t emit_tiles(uint64_t n) { return (n + kEmitTile - 1) / kEmitTile; }

static int sm_count(int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  return cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
}

}  // namespace ndx

using namespace ndx;

extern "C" {

size_t ndx_wah_emit_scratch_bytes(uint64_t n) {
  const uint64_t t = emit_tiles(n) + 1;
  return size_t(t) * (8 + 8 + 4) + 1024;
}

int ndx_wah_emit(const uint64_t* d_pairs, uint64_t n, void* d_ctl, uint32_t* d_words,
                 uint32_t* d_vstart, uint32_t* d_values, void* d_scratch, uint32_t epoch,
                 void* stream) {
  if (!d_pairs || !d_ctl || !d_words || !d_vstart || !d_values || !d_scratch || n == 0)
    return NDX_E_INVALID;
  if (n >= (1ull << 31)) return NDX_E_TOO_LARGE;
  int sms = 0;
  int rc = sm_count(&sms);
  if (rc) return rc;
  const uint64_t t = emit_tiles(n) + 1;
  EmitScratch sc;
  sc.val_agg = static_cast<uint64_t*>(d_scratch);
  sc.val_pre = sc.val_agg + t;
  sc.status = reinterpret_cast<uint32_t*>(sc.val_pre + t);
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kEmitSmem));
    if (e) return e;
    attr_set[dev & 63] = true;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_emit, kEmitThreads, kEmitSmem);
  if (occ < 1) occ = 1;
  const int grid = int(umin<uint64_t>(emit_tiles(n), uint64_t(sms) * occ));
  k_emit<<<grid, kEmitThreads, kEmitSmem, static_cast<cudaStream_t>(stream)>>>(
      d_pairs, n, static_cast<Ctl*>(d_ctl), d_words, d_vstart, d_values, sc, epoch);
  return cudaGetLastError();
}

int ndx_wah_table(const uint32_t* d_values, const uint32_t* d_vstart, uint64_t n,
                  const void* d_ctl, uint32_t* d_entries, void* stream) {
  if (!d_values || !d_vstart || !d_ctl || !d_entries) return NDX_E_INVALID;
  int sms = 0;
  int rc = sm_count(&sms);
  if (rc) return rc;
  const int grid = int(umin<uint64_t>((n + 255) / 256 + 1, uint64_t(sms) * 4));
  k_table<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_values, d_vstart, static_cast<const Ctl*>(d_ctl), d_entries);
  return cudaGetLastError();
}

}  // extern "C"
