// Pieces shared by the scatter passes of the WAH sort (wah_sort.cu: plan,
// legacy byte passes, dispatch; wah_pass.cu: the TMA-staged passes).
//
// The sort is the reference's stable LSD radix sort of (value, row) pairs
// (p/core/src/wah_radix.cpp:16-127), done as onesweep-style passes: every
// tile publishes its digit counts, resolves its global digit bases by a
// decoupled look-back over its predecessors' statuses, and scatters.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "wah_internal.cuh"

namespace ndx {

// ---- look-back status word: [63:40] epoch | [39:38] flag | [37:0] count ----
constexpr uint64_t kStAgg = 1ull << 38;
constexpr uint64_t kStPrefix = 2ull << 38;
constexpr uint64_t kStValue = (1ull << 38) - 1;

__device__ __forceinline__ uint64_t st_word(uint32_t epoch, uint64_t flag, uint64_t v) {
  return (uint64_t(epoch & 0xffffffu) << 40) | flag | v;
}
__device__ __forceinline__ bool st_ready(uint64_t s, uint32_t epoch) {
  return uint32_t(s >> 40) == (epoch & 0xffffffu) && (s & (3ull << 38)) != 0;
}

// Exclusive count of digit d over all tiles before `tile`, kLookbackWidth
// predecessor statuses in flight per round trip.
#ifndef NDX_LOOKBACK_WIDTH
#define NDX_LOOKBACK_WIDTH 4
#endif
constexpr int kLookbackWidth = NDX_LOOKBACK_WIDTH;
__device__ __forceinline__ uint64_t lookback(const uint64_t* st, uint64_t tile, uint32_t nb,
                                             uint32_t d, uint32_t epoch) {
  uint64_t excl = 0;
  int64_t t0 = int64_t(tile) - 1;
  while (t0 >= 0) {
    uint64_t s[kLookbackWidth];
#pragma unroll
    for (int j = 0; j < kLookbackWidth; ++j)
      s[j] = t0 - j >= 0 ? ld_relaxed_u64(&st[uint64_t(t0 - j) * nb + d]) : 0ull;
#pragma unroll
    for (int j = 0; j < kLookbackWidth; ++j) {
      if (t0 - j < 0) return excl;
      while (!st_ready(s[j], epoch)) {
        __nanosleep(64);
        s[j] = ld_relaxed_u64(&st[uint64_t(t0 - j) * nb + d]);
      }
      excl += s[j] & kStValue;
      if ((s[j] & (3ull << 38)) == kStPrefix) return excl;
    }
    t0 -= kLookbackWidth;
  }
  return excl;
}

// The same, with the status of tile-1 already loaded (`s0`).
__device__ __forceinline__ uint64_t lookback_from(const uint64_t* st, uint64_t tile, uint32_t nb,
                                                  uint32_t d, uint32_t epoch, uint64_t s0) {
  const uint64_t* p0 = &st[(tile - 1) * nb + d];
  while (!st_ready(s0, epoch)) {
    __nanosleep(64);
    s0 = ld_relaxed_u64(p0);
  }
  uint64_t excl = s0 & kStValue;
  if ((s0 & (3ull << 38)) == kStPrefix || tile == 1) return excl;
  return excl + lookback(st, tile - 1, nb, d, epoch);
}

// Lanes of the warp whose BITS-wide digit equals mine: per bit one ballot
// and a select of it or its complement.
template <int BITS>
__device__ __forceinline__ unsigned warp_match(uint32_t d) {
  unsigned peers = kFull;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t, m;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "vote.sync.ballot.b32 t, p, 0xffffffff;\n\t"
        "selp.b32 m, 0, 0xffffffff, p;\n\t"
        "xor.b32 t, t, m;\n\t"
        "and.b32 %0, %0, t;\n\t}"
        : "+r"(peers)
        : "r"(d), "r"(1u << b));
  }
  return peers;
}

// Exclusive scan of cnt[0..len) into out[], one CTA (len <= 2048).
__device__ __forceinline__ void block_excl_scan(const uint32_t* cnt, uint32_t* out, int len) {
  __shared__ uint32_t warp_tot[32];
  const int per = (len + blockDim.x - 1) / blockDim.x;  // items per thread
  const int lo = threadIdx.x * per;
  uint32_t local = 0;
  for (int i = 0; i < per && lo + i < len; ++i) local += cnt[lo + i];
  uint32_t incl = warp_incl_sum(local);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t t = lane < nw ? warp_tot[lane] : 0;
    uint32_t ti = warp_incl_sum(t);
    if (lane < nw) warp_tot[lane] = ti - t;
  }
  __syncthreads();
  uint32_t run = warp_tot[warp] + incl - local;
  for (int i = 0; i < per && lo + i < len; ++i) {
    uint32_t c = cnt[lo + i];
    out[lo + i] = run;
    run += c;
  }
  __syncthreads();
}

// ---- tile shapes --------------------------------------------------------
// Legacy byte / wide passes (wah_sort.cu, also the sort_pairs primitive).
constexpr int kLegacyByteTile = 256 * 32;
constexpr int kLegacyWideTile = 512 * 32;
// TMA-staged passes (wah_pass.cu).
#ifndef NDX_WIDE_THREADS
#define NDX_WIDE_THREADS 512
#endif
#ifndef NDX_WIDE_IPT
#define NDX_WIDE_IPT 32
#endif
#ifndef NDX_AB_THREADS
#define NDX_AB_THREADS 256
#endif
#ifndef NDX_A_IPT
#define NDX_A_IPT 32
#endif
#ifndef NDX_B_IPT
#define NDX_B_IPT 32
#endif
constexpr int kWideTile = NDX_WIDE_THREADS * NDX_WIDE_IPT;
constexpr int kATile = NDX_AB_THREADS * NDX_A_IPT;
constexpr int kBTile = NDX_AB_THREADS * NDX_B_IPT;
// compact two-pass mode: pass A carries the low 24 bits of the local row
// index; the rest comes from the row segment (2^24 rows) of the element
constexpr int kSegBits = 24;
static_assert((1 << kSegBits) % kATile == 0, "a pass-A tile never straddles a row segment");

// ---- chunks of the first pass ------------------------------------------
// The first pass (wide or A) reads the keys in their original order, so its
// digit counts per stretch of keys are known before it runs: the plan stage
// counts each chunk (a contiguous range of whole kChunkBlock-key blocks),
// scans the counts into per-chunk digit offsets, and the pass walks its
// chunks in order with running offsets -- no look-back, no waiting.
constexpr uint64_t kChunkBlock = 16384;
#ifndef NDX_MAX_CHUNKS
#define NDX_MAX_CHUNKS 1024
#endif
constexpr uint32_t kMaxChunks = NDX_MAX_CHUNKS;
static_assert(kChunkBlock % kWideTile == 0 && kChunkBlock % kATile == 0, "tiles nest in chunk blocks");
__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
// [first, last) element of chunk c of k over n keys
__host__ __device__ inline uint64_t chunk_begin(uint64_t n, uint32_t k, uint32_t c) {
  const uint64_t blocks = ceil_div(n, kChunkBlock);
  const uint64_t b = blocks * c / k;
  return b * kChunkBlock < n ? b * kChunkBlock : n;
}
// the chunk count for n keys: `want` (the first pass's CTA count), at most
// one per block and kMaxChunks
__host__ __device__ inline uint32_t chunk_count(uint64_t n, uint32_t want) {
  const uint64_t blocks = ceil_div(n, kChunkBlock);
  uint64_t k = want < blocks ? want : blocks;
  k = k < kMaxChunks ? k : kMaxChunks;
  return uint32_t(k < 1 ? 1 : k);
}

// ---- status buffer layout ----------------------------------------------
// Fixed offsets, independent of n (a region never holds another region's
// data from an earlier build of a different size):
// [256 B header: u32 epoch counter, u32 pad, u64 high-water mark]
// [GB: segment starts of the compact mode, 256 x kMaxSeg u32]
// [tile_group: pass-B tile -> group of its first element, kMaxTilesB + 1 u32]
// [chunk counts: kMaxChunks x (2048 + 256) u32: the low 11 bits of the key,
//  then byte 0 (the 11 bits folded)]
// [chunk offsets: kMaxChunks x 2048 u32 (first-pass digit)]
// [statuses: the pass with the most (tiles x digits), u64 each]
constexpr uint64_t kMaxValues = 1ull << 31;  // a build takes n < 2^31
constexpr uint64_t kMaxSeg = kMaxValues >> kSegBits;
constexpr uint64_t kMaxTilesB = kMaxValues / kBTile;
constexpr uint64_t kGbOffset = 256;
constexpr uint64_t kTgOffset = kGbOffset + 256 * kMaxSeg * 4;
constexpr uint64_t kChunkHistOffset = (kTgOffset + (kMaxTilesB + 1) * 4 + 255) & ~uint64_t(255);
constexpr uint64_t kChunkHistWords = kWideBuckets + 256;
constexpr uint64_t kChunkOffOffset = kChunkHistOffset + uint64_t(kMaxChunks) * kChunkHistWords * 4;
constexpr uint64_t kStatusOffset = kChunkOffOffset + uint64_t(kMaxChunks) * kWideBuckets * 4;
__host__ __device__ inline uint64_t status_words(uint64_t n) {
  uint64_t w = ceil_div(n, kLegacyWideTile) * kWideBuckets;
  w = umax(w, ceil_div(n, kLegacyByteTile) * 256);
  w = umax(w, ceil_div(n, kWideTile) * kWideBuckets);
  w = umax(w, ceil_div(n, kATile) * 256);
  w = umax(w, ceil_div(n, kBTile) * 256);
  return w;
}
__host__ __device__ inline uint64_t n_segments(uint64_t n) {
  return umax<uint64_t>(1, ceil_div(n, 1ull << kSegBits));
}
__host__ __device__ inline uint64_t status_bytes(uint64_t n) { return kStatusOffset + status_words(n) * 8; }
// legacy passes: dynamic shared memory of k_pass<8> and k_pass<11>
constexpr size_t kLegacyByteSmem = size_t(256) * 32 * 8 + 2 * 256 * 4 + 16;
constexpr size_t kLegacyWideSmem = size_t(512) * 32 * 8 + 2 * kWideBuckets * 4 + 16;
constexpr uint32_t kEpochStep = 8, kEpochMax = 0xfffff8u;  // 24-bit tags, 8 per build

// pass epochs within a build (ctl->epoch + offset): wide 1, bytes 2..5, A 6, B 7
constexpr uint32_t kEpochWide = 1, kEpochA = 6, kEpochB = 7;
// tile counters in ctl->tile_ctr: [0] emit, [1] wide, [2..5] bytes, [6] A, [7] B
constexpr int kCtrWide = 1, kCtrA = 6, kCtrB = 7;

struct SortArgs {
  const uint32_t* in_keys;      // first pass: keys
  const uint32_t* in_payloads;  // first pass: payloads, or null -> row ids synthesised
  uint64_t* X;                  // final output pairs (the last pass writes X) ...
  uint64_t* Y;                  // ... and the ping-pong buffer
  uint32_t* out_keys;           // non-null: the last pass writes SoA here instead of X
  uint32_t* out_payloads;
  uint64_t n;
  uint32_t row_base;
  Ctl* ctl;
  uint64_t* status;             // look-back statuses (status buffer + 256)
  uint32_t* gb;                 // compact mode: segment starts (256 x nseg)
  uint32_t* tile_group;         // compact mode: group of each pass-B tile's first element
  const uint32_t* chunk_off;    // first pass: per-chunk digit offsets (kMaxChunks x 2048)
  uint32_t nchunk;              // chunks of the first pass
};

// wah_pass.cu: the sort stage's dispatcher.  legacy = 1 (sort_pairs, which
// carries caller payloads) runs the legacy passes of wah_sort.cu only.
int launch_sort_dispatch(const SortArgs& a, int legacy, int byte_grid, int legacy_wide_grid, cudaStream_t s);

}  // namespace ndx
