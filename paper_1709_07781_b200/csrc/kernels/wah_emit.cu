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
// Words are owned by elements: a run's gap fill by its head element, its
// body word by its tail element, so word order is element order.  A run's
// literal is a segmented warp OR-scan; a ones-stretch length is found by
// galloping over the sorted pairs (pair[i+t] == (v, r+t) is monotone in t
// because rows strictly increase inside a value).  Word and value counts
// are scanned inside the tile and across tiles, and the compacted words are
// written to their final position -- no zero-padded fill/body arrays, no
// host round trip.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../../include/ndx.h"
#include "common.cuh"
#include "wah_internal.cuh"

namespace ndx {

constexpr int kEmitThreads = 256;
constexpr int kEmitWarps = kEmitThreads / 32;
constexpr int kEmitIPT = 4;                             // 32-element rounds per warp per tile
constexpr int kEmitWarpItems = 32 * kEmitIPT;           // 128
constexpr int kEmitTile = kEmitWarps * kEmitWarpItems;  // 1024
constexpr int kHaloL = 32;                              // elements before the tile (carry, prev)
constexpr int kHaloR = 2;                               // elements after it (next; 16 B multiple)
constexpr int kEmitBuf = kHaloL + kEmitTile + kHaloR;
// staging of one tile: per warp 2*kEmitWarpItems words + kEmitWarpItems
// (value, word offset) table heads
constexpr int kStageWarp = 4 * kEmitWarpItems;
constexpr int kStageTile = kEmitWarps * kStageWarp;
constexpr size_t kEmitSmem = size_t(2 * kEmitBuf) * 8 + size_t(2 * kStageTile) * 4;

__device__ __forceinline__ uint32_t pkey(uint64_t e) { return uint32_t(e); }
__device__ __forceinline__ uint32_t prow(uint64_t e) { return uint32_t(e >> 32); }
__device__ __forceinline__ uint64_t mkpair(uint32_t v, uint32_t row) {
  return uint64_t(v) | (uint64_t(row) << 32);
}

// Largest t with pairs[g+t] == (v, row+t), given that it holds for t = 30.
// Monotone in t because rows strictly increase inside a value.
__device__ __noinline__ uint32_t stretch_end(const uint64_t* __restrict__ pairs, uint64_t n,
                                             uint64_t g, uint32_t v, uint32_t row) {
  auto P = [&](uint64_t t) -> bool {
    if (g + t >= n) return false;
    uint64_t rr = uint64_t(row) + t;
    if (rr > 0xffffffffull) return false;
    return __ldg(pairs + g + t) == (uint64_t(v) | (rr << 32));
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

// Body word of an all-ones run whose LAST element is e (row = 31c+30): zero
// when chunk c-1 of the same value is all-ones too (the run is swallowed by
// the stretch's single ones-fill, wah_builder.cpp:193-205), else the
// ones-fill covering the maximal stretch that starts at chunk c.
__device__ __noinline__ uint32_t ones_body(const uint64_t* __restrict__ pairs, uint64_t n,
                                           uint64_t e, uint32_t v, uint32_t row) {
  if (e >= 61 && row >= 61 && __ldg(pairs + e - 61) == mkpair(v, row - 61)) return 0;
  const uint32_t t = stretch_end(pairs, n, e - 30, v, row - 30);
  return make_fill(true, (t + 1) / kChunkBits);
}

// floor(x / 31): two instructions, exact for x < kDiv31FastLimit.
constexpr uint32_t kDiv31FastLimit = 0x8D3DCB08u;
template <bool SMALL>
__device__ __forceinline__ uint32_t div31(uint32_t x) {
  if (SMALL) return __umulhi(x, 2216757315u) >> 4;
  return x / kChunkBits;
}

// One warp's kEmitWarpItems consecutive elements (tile-local from wl), as
// kEmitIPT rounds of 32, into the warp's staging area: its words compacted
// at warp-local offsets (ow) and one (value, warp-local word offset) row per
// value head (hv, ho).  Returns (words << 16) | value heads.  B[li] is
// element ts + li, with 32 elements of left halo and 2 of right halo.
template <bool SMALL>
__device__ __forceinline__ uint32_t warp_tile(const uint64_t* B, const uint64_t* __restrict__ pairs,
                                              uint32_t n, uint32_t ts, uint32_t wl, uint32_t* ow,
                                              uint32_t* hv, uint32_t* ho) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t wb = ts + wl;
  if (wb >= n) return 0;
  // open run carried into the first round: OR over the preceding elements
  // with the same (value, chunk) as element wb (all of them are among the
  // 32 before it: a run has at most 31 elements)
  uint32_t carry;
  {
    const uint64_t e0 = B[wl];
    const uint32_t v0 = pkey(e0), c0 = div31<SMALL>(prow(e0));
    const uint64_t q = B[int(wl) - 32 + int(lane)];
    const uint32_t qrow = prow(q), qc = div31<SMALL>(qrow);
    const bool m = (wb + lane >= 32) & (pkey(q) == v0) & (qc == c0);
    carry = __reduce_or_sync(kFull, m ? 1u << (qrow - qc * kChunkBits) : 0u);
  }
  const unsigned le = lanemask_le(), lt = lanemask_lt();
  uint32_t wc = 0, dc = 0;
#pragma unroll
  for (int r = 0; r < kEmitIPT; ++r) {
    const uint32_t li = wl + r * 32 + lane;
    const uint32_t e = ts + li;
    const bool valid = e < n;
    const uint64_t cur = B[li], prv = B[int(li) - 1], nxt = B[li + 1];
    const uint32_t v = pkey(cur), row = prow(cur), c = div31<SMALL>(row);
    const uint32_t pc = div31<SMALL>(prow(prv)), nc = div31<SMALL>(prow(nxt));
    const bool vhead = valid & ((e == 0) | (pkey(prv) != v));
    const bool head = vhead | (valid & (pc != c));
    const bool tail = valid & ((e + 1 == n) | (pkey(nxt) != v) | (nc != c));
    // run literal: segmented OR-scan over [head lane, lane], plus the open
    // run's carry when the run began in an earlier round; the scan depth is
    // the longest run piece ending in this round
    const unsigned hm = __ballot_sync(kFull, head) & le;
    const uint32_t hl = 31u - __clz(hm | 1u);
    const uint32_t span = __reduce_max_sync(kFull, (tail | (lane == 31)) ? lane - hl + 1 : 0u);
    uint32_t lit = valid ? 1u << (row - c * kChunkBits) : 0u;
    for (uint32_t d = 1; d < span; d <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, lit, d);
      if (lane >= hl + d) lit |= y;
    }
    if (hm == 0) lit |= carry;
    carry = __shfl_sync(kFull, lit, 31);
    const uint32_t gap = vhead ? c : c - pc - 1;
    const uint32_t gapw = (head & (gap != 0)) ? (kFillFlag | gap) : 0u;
    uint32_t body = tail ? lit : 0u;
    if (body == kLiteralMask) body = ones_body(pairs, n, e, v, row);
    const unsigned B0 = __ballot_sync(kFull, gapw != 0);
    const unsigned B1 = __ballot_sync(kFull, body != 0);
    const unsigned BV = __ballot_sync(kFull, vhead);
    uint32_t o = wc + __popc(B0 & lt) + __popc(B1 & lt);
    if (vhead) {
      const uint32_t h = dc + __popc(BV & lt);
      hv[h] = v;
      ho[h] = o;
    }
    if (gapw) ow[o++] = gapw;
    if (body) ow[o] = body;
    wc += __popc(B0) + __popc(B1);
    dc += __popc(BV);
  }
  return (wc << 16) | dc;
}

// Tile schedule: static round-robin (CTA c takes tiles c, c+G, ...).  A
// tile's global offsets are the CTA's own previous tile's offsets plus the
// published aggregates of the G tiles in between -- one block-wide read,
// never a serial look-back chain.  The CTA computes tile k (publishing its
// aggregate) BEFORE it writes tile k-1 out, so by the time it needs the
// aggregates below tile k-1 the other CTAs have had a whole tile's worth of
// time to publish them.  All G CTAs are co-resident (cooperative launch); a
// tile only waits on smaller tiles, whose owners publish before they wait,
// so the schedule cannot deadlock.
//
// The next tile's pairs arrive by one bulk async copy (TMA, mbarrier
// completion) into the other shared buffer while this tile is processed.
constexpr uint64_t kAggReady = 1ull << 63;

__global__ __launch_bounds__(kEmitThreads, 4) void k_emit(const uint64_t* __restrict__ pairs,
                                                          uint64_t n, Ctl* ctl,
                                                          uint32_t* __restrict__ words,
                                                          uint32_t* __restrict__ vstart,
                                                          uint32_t* __restrict__ values,
                                                          uint64_t* agg, int bulk_ok) {
  extern __shared__ __align__(16) unsigned char emit_smem[];
  uint64_t* buf0 = reinterpret_cast<uint64_t*>(emit_smem);
  uint32_t* stage0 = reinterpret_cast<uint32_t*>(buf0 + 2 * kEmitBuf);
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t s_wt[2][kEmitWarps];
  __shared__ uint32_t s_rw[kEmitWarps], s_rd[kEmitWarps];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (n + kEmitTile - 1) / kEmitTile;
  const uint64_t G = gridDim.x;
  const uint32_t n32 = uint32_t(n);  // n < 2^31 (checked by the launcher)
  const bool small_rows = ctl->row_hi < kDiv31FastLimit;

  // Tiles whose halo range lies inside [0, n) arrive by bulk copy; the
  // first and the last ones are gathered by the threads.
  auto by_bulk = [&](uint64_t t) -> bool {
    return bulk_ok && t > 0 && (t + 1) * kEmitTile + kHaloR <= n;
  };
  auto fill = [&](uint64_t t, int b) {
    uint64_t* dst = buf0 + b * kEmitBuf;
    const int64_t g0 = int64_t(t * kEmitTile) - kHaloL;
    if (by_bulk(t)) {
      if (threadIdx.x == 0) {
        fence_proxy_async_smem();
        mbar_expect_tx(&bar[b], kEmitBuf * 8);
        bulk_g2s(dst, pairs + g0, kEmitBuf * 8, &bar[b]);
      }
    } else {
      for (int j = threadIdx.x; j < kEmitBuf; j += kEmitThreads) {
        const int64_t g = g0 + j;
        dst[j] = (g >= 0 && uint64_t(g) < n) ? __ldg(pairs + g) : 0ull;
      }
    }
  };

  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  uint64_t prev_w = 0, prev_d = 0;  // exclusive offsets of this CTA's last written tile
  int64_t prev_tile = -1;
  int64_t pending = -1;             // computed, not yet written
  uint32_t phase = 0;
  uint64_t tile = blockIdx.x;
  if (tile < ntiles) fill(tile, 0);
  __syncthreads();

  for (int it = 0;; tile += G, ++it) {
    const bool has = tile < ntiles;
    if (!has && pending < 0) break;
    const int b = it & 1;
    if (has) {
      if (tile + G < ntiles) fill(tile + G, b ^ 1);
      if (by_bulk(tile)) {
        mbar_wait(&bar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
      }
      const uint64_t* B = buf0 + b * kEmitBuf + kHaloL;  // B[li] = pairs[tile * kEmitTile + li]
      uint32_t* st = stage0 + b * kStageTile + warp * kStageWarp;
      const uint32_t ts = uint32_t(tile * kEmitTile), wl = uint32_t(warp) * kEmitWarpItems;
      const uint32_t tot =
          small_rows
              ? warp_tile<true>(B, pairs, n32, ts, wl, st, st + 2 * kEmitWarpItems,
                                st + 3 * kEmitWarpItems)
              : warp_tile<false>(B, pairs, n32, ts, wl, st, st + 2 * kEmitWarpItems,
                                 st + 3 * kEmitWarpItems);
      if (lane == 0) s_wt[b][warp] = tot;
    }
    __syncthreads();
    if (has && threadIdx.x == 0) {
      uint32_t tw = 0, td = 0;
#pragma unroll
      for (int w = 0; w < kEmitWarps; ++w) {
        tw += s_wt[b][w] >> 16;
        td += s_wt[b][w] & 0xffffu;
      }
      st_relaxed_u64(&agg[tile], kAggReady | uint64_t(tw) | (uint64_t(td) << 32));
    }

    if (pending >= 0) {
      // ---- write the previous tile: global offsets first
      const int pb = b ^ 1;
      const uint64_t pt = uint64_t(pending);
      const uint64_t lo = prev_tile < 0 ? 0 : uint64_t(prev_tile);
      uint32_t sw = 0, sd = 0;
      for (uint64_t j = lo + threadIdx.x; j < pt; j += kEmitThreads) {
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
        s_rw[warp] = sw;
        s_rd[warp] = sd;
      }
      __syncthreads();
      uint64_t W0 = prev_w, D0 = prev_d;
      uint32_t wbw = 0, wbd = 0, tw = 0, td = 0;
#pragma unroll
      for (int w = 0; w < kEmitWarps; ++w) {
        W0 += s_rw[w];
        D0 += s_rd[w];
        const uint32_t t = s_wt[pb][w];
        if (w < warp) {
          wbw += t >> 16;
          wbd += t & 0xffffu;
        }
        tw += t >> 16;
        td += t & 0xffffu;
      }
      prev_w = W0;
      prev_d = D0;
      prev_tile = int64_t(pt);
      if (threadIdx.x == 0 && pt == ntiles - 1) {
        ctl->words = W0 + tw;
        ctl->distinct = D0 + td;
      }
      // ---- copy the warp's staged words and table heads out
      const uint32_t* st = stage0 + pb * kStageTile + warp * kStageWarp;
      const uint32_t mine = s_wt[pb][warp];
      const uint32_t nw = mine >> 16, nd = mine & 0xffffu;
      const uint64_t Ww = W0 + wbw, Dw = D0 + wbd;
      for (uint32_t j = lane; j < nw; j += 32) words[Ww + j] = st[j];
      for (uint32_t j = lane; j < nd; j += 32) {
        values[Dw + j] = st[2 * kEmitWarpItems + j];
        vstart[Dw + j] = uint32_t(Ww + st[3 * kEmitWarpItems + j]);
      }
    }
    pending = has ? int64_t(tile) : -1;
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
  int bulk_ok = (reinterpret_cast<uintptr_t>(d_pairs) & 15) == 0;
  void* args[] = {(void*)&d_pairs, (void*)&n,        (void*)&ctl, (void*)&d_words,
                  (void*)&d_vstart, (void*)&d_values, (void*)&agg, (void*)&bulk_ok};
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
