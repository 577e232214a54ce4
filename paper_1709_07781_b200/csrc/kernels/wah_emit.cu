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
    return pairs[g + t] == (uint64_t(v) | (rr << 32));
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

// Static round-robin tiles: CTA c takes tiles c, c+G, c+2G, ...  A tile's
// global offsets are the CTA's own previous tile's offsets plus the
// aggregates of the G tiles in between -- one block-wide read of G
// published aggregates, never a chain of look-backs.  All G CTAs must be
// co-resident (cooperative launch); every dependency is on a smaller tile
// index and aggregates are published before waiting, so it cannot deadlock.
constexpr uint64_t kAggReady = 1ull << 63;

__global__ __launch_bounds__(kEmitThreads) void k_emit(const uint64_t* __restrict__ pairs,
                                                       uint64_t n, Ctl* ctl,
                                                       uint32_t* __restrict__ words,
                                                       uint32_t* __restrict__ vstart,
                                                       uint32_t* __restrict__ values,
                                                       uint64_t* agg) {
  extern __shared__ __align__(16) unsigned char emit_smem[];
  uint64_t* win = reinterpret_cast<uint64_t*>(emit_smem);                   // [kEmitTile + 2 kHalo]
  uint32_t* ow = reinterpret_cast<uint32_t*>(win + kEmitTile + 2 * kHalo);  // [2 kEmitTile]
  __shared__ uint32_t warp_tot[kEmitWarps];
  __shared__ uint32_t red_w[kEmitWarps], red_d[kEmitWarps];
  __shared__ uint32_t s_tot;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (n + kEmitTile - 1) / kEmitTile;
  const uint64_t G = gridDim.x;
  uint64_t prev_w = 0, prev_d = 0;  // this CTA's previous tile's exclusive offsets
  int64_t prev_tile = -1;

  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += G) {
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
      if (lane == 31) {
        s_tot = ti;
        st_relaxed_u64(&agg[tile], kAggReady | uint64_t(ti >> 16) | (uint64_t(ti & 0xffffu) << 32));
      }
    }
    __syncthreads();

    // ---- stage the tile's words at tile-local offsets
    const uint32_t woff = warp_tot[warp];
#pragma unroll
    for (int r = 0; r < kEmitIPT; ++r) {
      const uint32_t li = uint32_t(warp) * kEmitWarpItems + r * 32 + lane;
      if (li >= m) continue;
      uint32_t o = (woff + exw[r]) >> 16;
      if (gapw[r]) ow[o++] = gapw[r];
      if (body[r]) ow[o] = body[r];
    }

    // ---- global offsets: previous tile of this CTA + aggregates in between
    const uint64_t lo = prev_tile < 0 ? 0 : uint64_t(prev_tile);
    uint32_t sw = 0, sd = 0;
    for (uint64_t j = lo + threadIdx.x; j < tile; j += kEmitThreads) {
      uint64_t s = ld_relaxed_u64(&agg[j]);
      while (!(s & kAggReady)) {
        __nanosleep(32);
        s = ld_relaxed_u64(&agg[j]);
      }
      sw += uint32_t(s);
      sd += uint32_t(s >> 32) & 0x7fffffffu;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sw += __shfl_xor_sync(kFull, sw, o);
      sd += __shfl_xor_sync(kFull, sd, o);
    }
    if (lane == 0) {
      red_w[warp] = sw;
      red_d[warp] = sd;
    }
    __syncthreads();
    uint64_t w_add = 0, d_add = 0;
#pragma unroll
    for (int w = 0; w < kEmitWarps; ++w) {
      w_add += red_w[w];
      d_add += red_d[w];
    }
    const uint64_t W0 = prev_w + w_add, D0 = prev_d + d_add;
    prev_w = W0;
    prev_d = D0;
    prev_tile = int64_t(tile);
    const uint32_t tot = s_tot;
    if (threadIdx.x == 0 && tile == ntiles - 1) {
      ctl->words = W0 + (tot >> 16);
      ctl->distinct = D0 + (tot & 0xffffu);
    }

    // ---- table rows (value heads) straight to HBM
#pragma unroll
    for (int r = 0; r < kEmitIPT; ++r) {
      const uint32_t li = uint32_t(warp) * kEmitWarpItems + r * 32 + lane;
      if (li >= m) continue;
      const uint64_t g = tile_start + li;
      const uint64_t cur = win[li + kHalo];
      const bool vhead = g == 0 || pkey(win[li + kHalo - 1]) != pkey(cur);
      if (vhead) {
        const uint32_t ex = woff + exw[r];
        const uint64_t dd = D0 + (ex & 0xffffu);
        vstart[dd] = uint32_t(W0 + (ex >> 16));
        values[dd] = pkey(cur);
      }
    }
    const uint32_t tw = tot >> 16;
    for (uint32_t j = threadIdx.x; j < tw; j += kEmitThreads) words[W0 + j] = ow[j];
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

size_t ndx_wah_emit_scratch_bytes(uint64_t n) { return size_t(emit_tiles(n) + 1) * 8 + 256; }

int ndx_wah_emit(const uint64_t* d_pairs, uint64_t n, void* d_ctl, uint32_t* d_words,
                 uint32_t* d_vstart, uint32_t* d_values, void* d_scratch, void* stream) {
  if (!d_pairs || !d_ctl || !d_words || !d_vstart || !d_values || !d_scratch || n == 0)
    return NDX_E_INVALID;
  if (n >= (1ull << 31)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  static int grid_for[64] = {};
  if (!grid_for[dev & 63]) {
    if ((e = cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kEmitSmem))))
      return e;
    int sms = 0, occ = 0;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_emit, kEmitThreads,
                                                           kEmitSmem)))
      return e;
    grid_for[dev & 63] = sms * (occ > 0 ? occ : 1);
  }
  const uint64_t tiles = emit_tiles(n);
  uint64_t* agg = static_cast<uint64_t*>(d_scratch);
  if ((e = cudaMemsetAsync(agg, 0, tiles * 8, s))) return e;
  int grid = int(umin<uint64_t>(tiles, uint64_t(grid_for[dev & 63])));
  Ctl* ctl = static_cast<Ctl*>(d_ctl);
  void* args[] = {(void*)&d_pairs, (void*)&n, (void*)&ctl,
                  (void*)&d_words, (void*)&d_vstart, (void*)&d_values, (void*)&agg};
  return cudaLaunchCooperativeKernel((const void*)k_emit, dim3(grid), dim3(kEmitThreads), args,
                                     kEmitSmem, s);
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
