// TMA-staged scatter passes of the WAH sort (stage S2) on sm_100a.
//
// Replaces the reference's stable LSD radix sort of (value, row) pairs
// (p/core/src/wah_radix.cpp:16-127, row_iota at wah_builder.cpp:54-60) for
// the two key shapes of the BASELINE workloads, each in as few HBM bytes as
// the shape allows:
//
//   wide   key range < 2^11 (C1, C3): ONE pass on digit = key - min.
//          keys (4 B) in, row ids (4 B) out, synthesised: the rows form
//          of the sorted stream (the values are the plan's bucket starts,
//          k_vs in wah_sort.cu).
//   A, B   key range < 2^16 with both low bytes varying (C4, C5): two
//          passes whose intermediate is a packed u32 instead of a pair.
//     A    digit = key & 0xff.  Out: hb << 24 | (i & 0xffffff), where hb is
//          the key's second byte and i the element's index in the column.
//          The index bits above 24 ("row segment") are not stored: a pass-A
//          tile lies inside one segment (2^24 / tile), so the first tile of
//          each segment records the global start of every digit there
//          (GB[lo][seg]), and every pass-A run marks the pass-B tiles that
//          begin inside it (tile_group).
//     B    digit = hb.  The element's low byte and row segment are its
//          "group" (lo, seg) -- the pass-A run it came from -- found from
//          tile_group and GB by position.  Out: row ids (rows form); the
//          tile holding the start of low byte lo in pass A's order writes
//          where each key (hb, lo) starts (vs16).
//   Bytes per element: wide 8; A + B 8 + 8 = 16 (the u64 ping-pong of
//   the legacy byte passes, wah_sort.cu, moves 12 + 16 = 28).
//
// The first pass (wide or A) reads the keys in their original order, so
// its digit offsets per chunk of keys come from the plan stage (k_hist
// counts every chunk, k_plan_scan scans the counts): each CTA walks its
// chunks' tiles in order with running digit offsets in shared memory -- no
// look-back and no waiting on other CTAs -- and copies its next tile in by
// TMA while it works on the current one.  Pass B reads pass A's output, so
// its tiles resolve their digit offsets by a decoupled look-back.
//
// Per tile:
//   1. the tile arrives in shared memory by one TMA bulk copy
//      (cp.async.bulk + mbarrier); every thread reads its elements with
//      conflict-free LDS
//   2. warp ballot-match ranking (lane order == row order: stable), per-warp
//      digit counters in shared memory
//   3. tile digit counts, local scan; global digit bases from the running
//      chunk offsets (wide, A) or the look-back (B)
//   4. staging in shared memory in digit order (u32: wide digit | local,
//      A hb | lo | local, B the packed word plus its group when the tile
//      crosses groups)
//   5. coalesced scatter of the staged runs
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <type_traits>

#include "../../../include/ndx.h"
#include "wah_sort_common.cuh"

namespace ndx {

enum PassKind : int { kPassWide = 0, kPassA = 1, kPassB = 2 };

#ifndef NDX_WIDE_MINB
#define NDX_WIDE_MINB 1
#endif
#ifndef NDX_A_MINB
#define NDX_A_MINB 3
#endif
#ifndef NDX_B_MINB
#define NDX_B_MINB 3  // with NDX_B_ALIAS: 3 CTAs per SM (C4 sort 2.307 vs 2.420 ms at 2)
#endif
// input buffer aliased with the staging area (the next tile's copy waits for
// the end of this one; half the shared memory, so more CTAs per SM)
#ifndef NDX_WIDE_ALIAS
#define NDX_WIDE_ALIAS 0
#endif
#ifndef NDX_A_ALIAS
#define NDX_A_ALIAS 0
#endif
#ifndef NDX_B_ALIAS
#define NDX_B_ALIAS 1
#endif
// every lane reads its digit's counter (broadcast) instead of leader + shfl
#ifndef NDX_WIDE_BCAST
#define NDX_WIDE_BCAST 1
#endif
#ifndef NDX_AB_BCAST
#define NDX_AB_BCAST 1  // C4 sort 2.451 vs 2.511 ms with leader read + shuffle
#endif

constexpr int ceil_log2(int v) { return v <= 1 ? 0 : 1 + ceil_log2((v + 1) / 2); }

template <int KIND>
struct PassShape {
  static constexpr int THREADS = KIND == kPassWide ? NDX_WIDE_THREADS : NDX_AB_THREADS;
  static constexpr int IPT = KIND == kPassWide ? NDX_WIDE_IPT : (KIND == kPassA ? NDX_A_IPT : NDX_B_IPT);
  static constexpr int MINB = KIND == kPassWide ? NDX_WIDE_MINB : (KIND == kPassA ? NDX_A_MINB : NDX_B_MINB);
  static constexpr bool ALIAS = KIND == kPassWide ? NDX_WIDE_ALIAS : (KIND == kPassA ? NDX_A_ALIAS : NDX_B_ALIAS);
  static constexpr bool BCAST = KIND == kPassWide ? NDX_WIDE_BCAST : NDX_AB_BCAST;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int WI = 32 * IPT;  // elements per warp
  static constexpr int TILE = THREADS * IPT;
  static constexpr int LOCAL_BITS = ceil_log2(TILE);
  using Stage = uint32_t;  // wide/A: digit | local; B: the packed word (its group in a u16 array beside)
  static_assert(TILE <= 65536 && (TILE & (TILE - 1)) == 0, "ranks ride in 16 bits; tiles are powers of two");
  static_assert(KIND != kPassWide || LOCAL_BITS + kWideMaxBits <= 32, "wide staging packs digit | local");
  static_assert(KIND != kPassA || LOCAL_BITS <= 16, "pass-A staging packs hb | lo | local");
};

struct PassMisc {
  uint32_t lo_start[256];  // pass B: pass A's bucket start of each low byte (16-byte aligned)
  uint64_t bar;            // mbarrier of the input bulk copy
  uint32_t tile[2];        // pass B: tile taken for iteration parity 0/1
  uint32_t tg[2][2];       // pass B: tile_group[t], tile_group[t+1] per parity
  uint32_t sgb[2][32];     // pass B: group starts inside the tile per parity
  uint32_t kbg[33];        // pass B: key base (top bits | lo) of the tile's groups
  uint32_t rbg[33];        // pass B: row base (row_base + seg << 24) of the tile's groups
  uint32_t own[2];         // pass B: low bytes whose starts the tile holds, first | count << 16, per parity
};

// Shared memory of one CTA: [in: TILE u32][R: H | S][cnt NB][gbase NB][run NB][Misc]
template <int KIND, int BITS>
struct PassSmem {
  using SH = PassShape<KIND>;
  static constexpr int NB = 1 << BITS;
  static constexpr size_t kIn = size_t(SH::TILE) * 4;
  static constexpr size_t kH = size_t(SH::WARPS) * NB * 2;
  static constexpr size_t kS = size_t(SH::TILE) * (sizeof(typename SH::Stage) + (KIND == kPassB ? 2 : 0));
  static constexpr size_t kR0 = kH > kS ? kH : kS;
  static constexpr size_t kR = SH::ALIAS ? (kR0 > kIn ? kR0 : kIn) : kR0;
  static constexpr size_t kInOfs = 0;
  static constexpr size_t kROfs = SH::ALIAS ? 0 : kIn;
  static constexpr size_t kCntOfs = kROfs + kR;
  static constexpr size_t kMiscOfs = kCntOfs + 3 * NB * 4;
  static constexpr size_t kBytes = kMiscOfs + sizeof(PassMisc);
};

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// lo16(a) | lo16(b) << 16 in one register.  Opaque to the compiler on
// purpose: with plain shifts and ors it sees through the packing and keeps
// the two halves in separate registers again (spilling the tile).
__device__ __forceinline__ uint32_t pack16(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// Everything a tile needs besides its index (one per CTA, built once).
struct PassCtx {
  SortArgs a;
  const uint32_t* src;     // tile input (keys, or pass A's packed words)
  const uint32_t* bstart;  // pass B: global bucket starts of its digits
  uint64_t n;
  uint32_t tiles, epoch;
  uint32_t kbase;          // wide: digit = key - kbase; A/B: the keys' top 16 bits
  uint32_t nseg;           // A/B: row segments
  bool bulk;               // input 16-byte aligned: tiles arrive by TMA
  uint32_t* inbuf;
  unsigned char* R;
  uint32_t* cnt;
  uint32_t* gbase;
  uint32_t* run;           // wide/A: running global digit offsets of the chunk
  PassMisc* m;
};

template <int KIND>
__device__ __forceinline__ void issue_tile_copy(const PassCtx& c, uint64_t t) {  // one thread
  fence_proxy_async_smem();
  mbar_expect_tx(&c.m->bar, PassShape<KIND>::TILE * 4);
  bulk_g2s(c.inbuf, c.src + t * PassShape<KIND>::TILE, PassShape<KIND>::TILE * 4, &c.m->bar);
}

// ---- steps shared by the three pass kinds -----------------------------------

// 1. the tile's elements into registers (wide: digit; A: the key's low 16
//    bits; B: the packed word)
template <int KIND, int BITS, bool FULL>
__device__ __forceinline__ void load_tile(const PassCtx& c, uint64_t ts, uint32_t tn, uint32_t wofs,
                                          uint32_t& phase, uint32_t (&x)[PassShape<KIND>::IPT]) {
  constexpr int IPT = PassShape<KIND>::IPT;
  if (FULL && c.bulk) {
    mbar_wait(&c.m->bar, phase);
    phase ^= 1u;
#pragma unroll
    for (int r = 0; r < IPT; ++r) x[r] = c.inbuf[wofs + r * 32];
  } else {
#pragma unroll
    for (int r = 0; r < IPT; ++r) x[r] = (FULL || wofs + r * 32 < tn) ? __ldg(c.src + ts + wofs + r * 32) : 0u;
  }
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    if (KIND == kPassWide) x[r] = (x[r] - c.kbase) & ((1u << BITS) - 1);  // the rank goes above bit 16
    if (KIND == kPassA) x[r] &= 0xffffu;                                  // lo | hb << 8, rank above
  }
}

template <int KIND, int BITS>
__device__ __forceinline__ uint32_t digit_of(uint32_t v) {
  if (KIND == kPassB) return v >> 24;
  return v & ((1u << BITS) - 1);
}

// 2. stable rank of every element among its warp's elements of the same
//    digit (wide/A: into bits 16..31 of x; B: two per rk2 register); the
//    per-warp digit counters end in H
template <int KIND, int BITS, bool FULL>
__device__ __forceinline__ void rank_tile(uint16_t* H, uint32_t wofs, uint32_t tn,
                                          uint32_t (&x)[PassShape<KIND>::IPT],
                                          uint32_t (&rk2)[PassShape<KIND>::IPT / 2]) {
  using SH = PassShape<KIND>;
  constexpr uint32_t NB = 1u << BITS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint16_t* Hw = H + warp * NB;
  if constexpr (KIND == kPassWide && NB >= 8) {  // 8 counters per 16-byte store
    uint4* Hw4 = reinterpret_cast<uint4*>(Hw);
    for (uint32_t i = lane; i < NB / 8; i += 32) Hw4[i] = make_uint4(0, 0, 0, 0);
  } else {
    for (uint32_t d = lane; d < NB; d += 32) Hw[d] = 0;
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < SH::IPT; ++r) {
    const uint32_t d = digit_of<KIND, BITS>(x[r]);
    unsigned peers = warp_match<BITS>(d);
    bool valid = true;
    if (!FULL) {
      valid = wofs + r * 32 < tn;
      peers &= __ballot_sync(kFull, valid);
    }
    const int leader = valid ? __ffs(peers) - 1 : lane;
    uint32_t old = 0;
    if constexpr (SH::BCAST) {
      old = Hw[d];
      __syncwarp();
    } else {
      if (lane == leader) old = Hw[d];
      old = __shfl_sync(kFull, old, leader);
    }
    if (valid && lane == leader) Hw[d] = uint16_t(old + __popc(peers));
    const uint32_t rk = old + __popc(peers & lanemask_lt());
    __syncwarp();
    if constexpr (KIND == kPassB) {
      if ((r & 1) == 0)
        rk2[r >> 1] = rk;
      else
        rk2[r >> 1] = pack16(rk2[r >> 1], rk);
    } else {
      x[r] = pack16(x[r], rk);
    }
  }
}

// 3a. per digit: warp offsets in place in H, the tile's count returned
template <int KIND, int BITS>
__device__ __forceinline__ uint32_t warp_offsets(uint16_t* H, uint32_t d) {
  constexpr uint32_t NB = 1u << BITS;
  uint32_t sum = 0;
#pragma unroll
  for (int w = 0; w < PassShape<KIND>::WARPS; ++w) {
    const uint32_t cw = H[w * NB + d];
    H[w * NB + d] = uint16_t(sum);
    sum += cw;
  }
  return sum;
}

// 3a, eight digits at a time (digits 8g .. 8g+7, sixteen-bit lanes: a tile's
//     counts stay below 2^16): warp offsets in place, the counts into cnt
template <int KIND, int BITS>
__device__ __forceinline__ void warp_offsets8(uint16_t* H, uint32_t g, uint32_t* cnt) {
  constexpr uint32_t NG = (1u << BITS) / 8;
  uint4* H4 = reinterpret_cast<uint4*>(H);
  uint4 sum = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int w = 0; w < PassShape<KIND>::WARPS; ++w) {
    const uint4 cw = H4[w * NG + g];
    H4[w * NG + g] = sum;
    sum.x = __vadd2(sum.x, cw.x);
    sum.y = __vadd2(sum.y, cw.y);
    sum.z = __vadd2(sum.z, cw.z);
    sum.w = __vadd2(sum.w, cw.w);
  }
  uint4* c4 = reinterpret_cast<uint4*>(cnt + 8 * g);
  c4[0] = make_uint4(sum.x & 0xffffu, sum.x >> 16, sum.y & 0xffffu, sum.y >> 16);
  c4[1] = make_uint4(sum.z & 0xffffu, sum.z >> 16, sum.w & 0xffffu, sum.w >> 16);
}
// 3b, eight digits at a time: the tile-local starts lc[0..7] into every
//     warp's offsets
template <int KIND, int BITS>
__device__ __forceinline__ void add_local8(uint16_t* H, uint32_t g, const uint32_t (&lc)[8]) {
  constexpr uint32_t NG = (1u << BITS) / 8;
  uint4* H4 = reinterpret_cast<uint4*>(H);
  const uint4 p = make_uint4(lc[0] | (lc[1] << 16), lc[2] | (lc[3] << 16), lc[4] | (lc[5] << 16),
                             lc[6] | (lc[7] << 16));
#pragma unroll
  for (int w = 0; w < PassShape<KIND>::WARPS; ++w) {
    uint4 h = H4[w * NG + g];
    h.x = __vadd2(h.x, p.x);
    h.y = __vadd2(h.y, p.y);
    h.z = __vadd2(h.z, p.z);
    h.w = __vadd2(h.w, p.w);
    H4[w * NG + g] = h;
  }
}

// 3b. the tile-local digit start folded into every warp's offsets, then
//     each element's rank made tile-wide
template <int KIND, int BITS>
__device__ __forceinline__ void add_local(uint16_t* H, uint32_t d, uint32_t local) {
  constexpr uint32_t NB = 1u << BITS;
#pragma unroll
  for (int w = 0; w < PassShape<KIND>::WARPS; ++w) H[w * NB + d] += uint16_t(local);
}
template <int KIND, int BITS>
__device__ __forceinline__ void rank_to_tile(const uint16_t* H, uint32_t (&x)[PassShape<KIND>::IPT],
                                             uint32_t (&rk2)[PassShape<KIND>::IPT / 2]) {
  constexpr uint32_t NB = 1u << BITS;
  const uint16_t* Hw = H + (threadIdx.x >> 5) * NB;
#pragma unroll
  for (int r = 0; r < PassShape<KIND>::IPT; ++r) {
    const uint32_t add = Hw[digit_of<KIND, BITS>(x[r])];
    if constexpr (KIND == kPassB)
      rk2[r >> 1] += add << (16 * (r & 1));
    else
      x[r] += add << 16;
  }
}

// ---- wide / A: chunked, running offsets ---------------------------------------

template <int KIND, int BITS, bool FULL>
__device__ __forceinline__ void chunk_tile(const PassCtx& c, uint64_t tile, int64_t next, uint32_t& phase) {
  using SH = PassShape<KIND>;
  constexpr uint32_t NB = 1u << BITS;
  constexpr uint32_t DMASK = NB - 1;
  constexpr int IPT = SH::IPT;
  constexpr uint32_t TILE = SH::TILE;
  constexpr uint32_t LB = SH::LOCAL_BITS;
  const SortArgs& a = c.a;
  uint16_t* H = reinterpret_cast<uint16_t*>(c.R);
  uint32_t* S = reinterpret_cast<uint32_t*>(c.R);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ts = tile * TILE;
  const uint32_t tn = FULL ? TILE : uint32_t(c.n - ts);
  const uint32_t wofs = uint32_t(warp) * SH::WI + lane;

  uint32_t x[IPT], rk2[IPT / 2];
  load_tile<KIND, BITS, FULL>(c, ts, tn, wofs, phase, x);
  __syncthreads();  // inbuf consumed; R free (previous scatter done)
  // the next tile of this CTA's chunks is known: copy it in now
  if (!SH::ALIAS && threadIdx.x == 0 && next >= 0 && c.bulk && uint64_t(next + 1) * TILE <= c.n)
    issue_tile_copy<KIND>(c, uint64_t(next));

  rank_tile<KIND, BITS, FULL>(H, wofs, tn, x, rk2);
  __syncthreads();
  if constexpr (KIND == kPassWide) {
    // up to 2^11 digits x 16 warps: eight digits per thread and 16-byte
    // shared accesses (C3's pass 374 -> 356 us); pass A's 256 digits keep one
    // thread per digit (eight per thread there measured 94 us slower on C4)
    static_assert(NB >= 8, "eight digits per thread");
    for (uint32_t g = threadIdx.x; g < NB / 8; g += SH::THREADS) warp_offsets8<KIND, BITS>(H, g, c.cnt);
    __syncthreads();
    block_excl_scan(c.cnt, c.gbase, int(NB));  // gbase <- tile-local digit starts (syncs)
    for (uint32_t g = threadIdx.x; g < NB / 8; g += SH::THREADS) {
      uint32_t lc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t d = 8 * g + i;
        const uint32_t local = c.gbase[d], cd = c.cnt[d];
        const uint32_t gstart = c.run[d];  // where this tile's run of d begins in the output
        lc[i] = local;
        c.run[d] = gstart + cd;
        c.gbase[d] = gstart - local;
      }
      add_local8<KIND, BITS>(H, g, lc);
    }
  } else {
    for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS) c.cnt[d] = warp_offsets<KIND, BITS>(H, d);
    __syncthreads();
    block_excl_scan(c.cnt, c.gbase, int(NB));  // gbase <- tile-local digit starts (syncs)
    for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS) {
      const uint32_t local = c.gbase[d], cd = c.cnt[d];
      const uint32_t gstart = c.run[d];  // where this tile's run of d begins in the output
      c.run[d] = gstart + cd;
      c.gbase[d] = gstart - local;
      add_local<KIND, BITS>(H, d, local);
      // segment starts, and the pass-B tiles that begin inside this run
      const uint32_t seg = uint32_t(ts >> kSegBits);
      if ((ts & ((1ull << kSegBits) - 1)) == 0) a.gb[d * c.nseg + seg] = gstart;
      for (uint32_t mt = uint32_t(ceil_div(gstart, kBTile)); uint64_t(mt) * kBTile < uint64_t(gstart) + cd; ++mt)
        a.tile_group[mt] = d * c.nseg + seg;
    }
  }
  __syncthreads();
  rank_to_tile<KIND, BITS>(H, x, rk2);
  __syncthreads();  // H dead: S may overwrite it

  // ---- staging in digit order
#pragma unroll
  for (int r = 0; r < IPT; ++r)
    if (FULL || wofs + r * 32 < tn) {
      const uint32_t v = x[r], local = wofs + r * 32;
      if (KIND == kPassWide)
        S[v >> 16] = ((v & DMASK) << LB) | local;
      else  // hb << 24 | lo << 16 | local (v << 16 drops the rank)
        S[v >> 16] = (v << 16) | local;
    }
  __syncthreads();

  // ---- scatter: consecutive slots of one digit are consecutive globally
  if constexpr (KIND == kPassA) {
    uint32_t* out = reinterpret_cast<uint32_t*>(a.Y);
    const uint32_t segofs = uint32_t(ts) & ((1u << kSegBits) - 1);
#pragma unroll 4
    for (uint32_t jj = threadIdx.x; jj < tn; jj += SH::THREADS) {
      const uint32_t e = S[jj];
      out[c.gbase[(e >> 16) & 0xffu] + jj] = (e & 0xff000000u) | (segofs + (e & 0xffffu));
    }
  } else {
    // rows form: the row ids only (the values are the plan's bucket starts, k_vs)
    uint32_t* out = reinterpret_cast<uint32_t*>(a.X);
    const uint32_t rbase = a.row_base + uint32_t(ts);
#pragma unroll 4
    for (uint32_t jj = threadIdx.x; jj < tn; jj += SH::THREADS) {
      const uint32_t e = S[jj];
      out[c.gbase[e >> LB] + jj] = rbase + (e & ((1u << LB) - 1));
    }
  }
  __syncthreads();
  if (SH::ALIAS && threadIdx.x == 0 && next >= 0 && c.bulk && uint64_t(next + 1) * TILE <= c.n)
    issue_tile_copy<KIND>(c, uint64_t(next));
}

// The chunks of this CTA (blockIdx.x, + gridDim.x, ...), their tiles in
// order, each chunk starting from its scanned digit offsets.
template <int KIND, int BITS>
__device__ __forceinline__ void run_chunked(PassCtx& c) {
  using SH = PassShape<KIND>;
  constexpr uint32_t NB = 1u << BITS;
  const uint32_t K = c.a.nchunk;
  auto first_tile = [&](uint32_t ch) -> int64_t {
    if (ch >= K) return -1;
    const uint64_t e0 = chunk_begin(c.n, K, ch), e1 = chunk_begin(c.n, K, ch + 1);
    return e1 > e0 ? int64_t(e0 / SH::TILE) : -1;
  };
  uint32_t ch = blockIdx.x;
  while (ch < K && first_tile(ch) < 0) ch += gridDim.x;
  if (ch >= K) return;
  if (threadIdx.x == 0) {
    mbar_init(&c.m->bar, 1);
    fence_mbar_init();
    const int64_t t = first_tile(ch);
    if (c.bulk && uint64_t(t + 1) * SH::TILE <= c.n) issue_tile_copy<KIND>(c, uint64_t(t));
  }
  __syncthreads();
  uint32_t phase = 0;
  while (ch < K) {
    const uint64_t t0 = chunk_begin(c.n, K, ch) / SH::TILE;
    const uint64_t t1 = ceil_div(chunk_begin(c.n, K, ch + 1), SH::TILE);
    uint32_t nch = ch + gridDim.x;
    while (nch < K && first_tile(nch) < 0) nch += gridDim.x;
    const uint32_t* off = c.a.chunk_off + uint64_t(ch) * kWideBuckets;
    for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS) c.run[d] = off[d];
    // (visible after the first barrier of the chunk's first tile)
    for (uint64_t t = t0; t < t1; ++t) {
      const int64_t next = t + 1 < t1 ? int64_t(t + 1) : first_tile(nch);
      if ((t + 1) * SH::TILE <= c.n)
        chunk_tile<KIND, BITS, true>(c, t, next, phase);
      else
        chunk_tile<KIND, BITS, false>(c, t, next, phase);
    }
    ch = nch;
  }
}

// ---- B: look-back ---------------------------------------------------------------

// pass B: the groups a tile crosses, staged by cp.async
__device__ __forceinline__ void group_words(const PassCtx& c, uint32_t t, int par) {  // thread 0
  cp_async4(&c.m->tg[par][0], c.a.tile_group + t);
  cp_async4(&c.m->tg[par][1], c.a.tile_group + t + 1);
}
__device__ __forceinline__ void group_starts(const PassCtx& c, int par) {  // warp 0, after tg[par] landed
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t g0 = c.m->tg[par][0], k = c.m->tg[par][1] - g0;
  if (k <= 32 && lane < k) cp_async4(&c.m->sgb[par][lane], c.a.gb + g0 + 1 + lane);
}
// The low bytes lo whose start P_lo (in pass A's order) lies in the tile --
// a contiguous range, P_lo grows with lo; the last tile also takes P_lo == n.
__device__ __forceinline__ void own_range(const PassCtx& c, uint32_t tile, int par) {  // warp 0
  using SH = PassShape<kPassB>;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t a = tile * uint32_t(SH::TILE);
  const uint32_t b = tile + 1 == c.tiles ? uint32_t(c.n) + 1u : a + uint32_t(SH::TILE);
  const uint4* p = reinterpret_cast<const uint4*>(c.m->lo_start) + 2 * lane;
  const uint4 u = p[0], v = p[1];
  uint32_t ca = (u.x < a) + (u.y < a) + (u.z < a) + (u.w < a) + (v.x < a) + (v.y < a) + (v.z < a) + (v.w < a);
  uint32_t cb = (u.x < b) + (u.y < b) + (u.z < b) + (u.w < b) + (v.x < b) + (v.y < b) + (v.z < b) + (v.w < b);
  ca = __reduce_add_sync(kFull, ca);
  cb = __reduce_add_sync(kFull, cb);
  if (lane == 0) c.m->own[par] = ca | ((cb - ca) << 16);
}

// Takes the next tile at the end of this one (claim order == processing
// order, so a tile's predecessors are ahead of it when it looks back),
// copies it in, requests its group words, and prefetches the tile one CTA
// round further on into L2.
__device__ __forceinline__ void claim_next_b(const PassCtx& c, uint32_t* ctr, int par) {  // thread 0
  using SH = PassShape<kPassB>;
  const uint32_t nt = atomicAdd(ctr, 1u);
  c.m->tile[par ^ 1] = nt;
  if (nt >= c.tiles) return;
  if (!SH::ALIAS && uint64_t(nt + 1) * SH::TILE <= c.n) issue_tile_copy<kPassB>(c, nt);
  group_words(c, nt, par ^ 1);
  const uint64_t pf = uint64_t(nt) + gridDim.x;
  if ((pf + 1) * SH::TILE <= c.n)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c.src + pf * SH::TILE), "r"(SH::TILE * 4u)
                 : "memory");
}

template <bool FULL>
__device__ __forceinline__ void lookback_tile(const PassCtx& c, uint32_t* ctr, uint32_t tile, int par,
                                              uint32_t& phase, bool later) {
  constexpr int KIND = kPassB;
  constexpr int BITS = 8;
  using SH = PassShape<KIND>;
  constexpr uint32_t NB = 256;
  constexpr int IPT = SH::IPT;
  constexpr uint32_t TILE = SH::TILE;
  const SortArgs& a = c.a;
  uint16_t* H = reinterpret_cast<uint16_t*>(c.R);
  PassMisc* m = c.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ts = uint64_t(tile) * TILE;
  const uint32_t tn = FULL ? TILE : uint32_t(c.n - ts);
  const uint32_t wofs = uint32_t(warp) * SH::WI + lane;

  uint32_t x[IPT], rk2[IPT / 2];
  load_tile<KIND, BITS, FULL>(c, ts, tn, wofs, phase, x);
  if (later && warp == 0) {
    // this tile's group words were requested at its claim: now its group starts
    if (lane == 0) cp_async_wait_all();
    __syncwarp();
    group_starts(c, par);
    own_range(c, tile, par);
  }
  __syncthreads();  // inbuf consumed; R free (previous scatter done)

  rank_tile<KIND, BITS, FULL>(H, wofs, tn, x, rk2);
  if (warp == 0) cp_async_wait_all();  // this tile's group starts
  __syncthreads();

  // counts published (decoupled look-back status), local starts
  uint64_t* st = a.status + uint64_t(tile) * NB;
  for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS) {
    const uint32_t sum = warp_offsets<KIND, BITS>(H, d);
    c.cnt[d] = sum;
    st_relaxed_u64(&st[d], st_word(c.epoch, tile == 0 ? kStPrefix : kStAgg, sum));
  }
  __syncthreads();
  block_excl_scan(c.cnt, c.gbase, int(NB));  // gbase <- tile-local digit starts (syncs)
  // the first predecessor status of this thread's digit is requested now;
  // its round trip overlaps the rank adjustment and the staging
  static_assert(SH::THREADS == int(NB), "one digit per thread");
  const uint32_t dme = threadIdx.x;
  const uint64_t first = tile > 0 ? ld_relaxed_u64(&a.status[uint64_t(tile - 1) * NB + dme]) : 0ull;
  add_local<KIND, BITS>(H, dme, c.gbase[dme]);
  __syncthreads();
  rank_to_tile<KIND, BITS>(H, x, rk2);
  __syncthreads();  // H dead: S may overwrite it

  // ---- staging: the packed word in digit order, and when the tile crosses
  // groups, each element's group (lo, seg) beside it -- found by walking the
  // group starts inside the tile (positions grow with r)
  uint32_t* S32 = reinterpret_cast<uint32_t*>(c.R);
  uint16_t* G16 = reinterpret_cast<uint16_t*>(S32 + TILE);
  const uint32_t g0 = m->tg[par][0], k = m->tg[par][1] - g0;
  if (k <= 32 && threadIdx.x <= k) {  // key and row base of every group of the tile
    const uint32_t g = g0 + threadIdx.x, lo = g / c.nseg, seg = g - lo * c.nseg;
    m->kbg[threadIdx.x] = c.kbase | lo;
    m->rbg[threadIdx.x] = a.row_base + (seg << kSegBits);
  }
  if (k == 0) {
#pragma unroll
    for (int r = 0; r < IPT; ++r)
      if (FULL || wofs + r * 32 < tn) S32[(rk2[r >> 1] >> (16 * (r & 1))) & 0xffffu] = x[r];
  } else {
    const uint32_t* sg = m->sgb[par];
    const uint32_t p0 = uint32_t(ts) + wofs;
    uint32_t j = 0, nb = k <= 32 ? sg[0] : 0u;
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
      const uint32_t p = p0 + uint32_t(r) * 32;
      if (k <= 32) {
        if (p >= nb) {
          while (j < k && p >= sg[j]) ++j;
          nb = j < k ? sg[j] : 0xffffffffu;
        }
      } else {
        // pathological tile (more than 32 groups start inside it): count
        // the group starts GB[g0+1 .. g0+k] <= p by binary search
        uint32_t lo_i = 0, hi_i = k;
        while (lo_i < hi_i) {
          const uint32_t mid = (lo_i + hi_i) >> 1;
          if (__ldg(a.gb + g0 + 1 + mid) <= p)
            lo_i = mid + 1;
          else
            hi_i = mid;
        }
        j = lo_i;
      }
      if (FULL || wofs + r * 32 < tn) {
        const uint32_t slot = (rk2[r >> 1] >> (16 * (r & 1))) & 0xffffu;
        S32[slot] = x[r];
        G16[slot] = uint16_t(j);
      }
    }
  }

  // ---- look-back: this tile's global base for my digit
  const uint32_t dlocal = c.gbase[dme];
  uint32_t vbase;
  {
    const uint32_t cd = c.cnt[dme], local = dlocal;
    uint64_t excl = 0;
    if (tile > 0) {
      excl = lookback_from(a.status, tile, NB, dme, c.epoch, first);
      st_relaxed_u64(&st[dme], st_word(c.epoch, kStPrefix, excl + cd));
    }
    c.gbase[dme] = c.bstart[dme] + uint32_t(excl) - local;
    vbase = c.bstart[dme] + uint32_t(excl);
  }
  __syncthreads();
  // ---- value starts of the rows form: for each low byte lo whose first
  // group begins in this tile (at pass-A position P_lo), key (dme, lo)
  // starts after this digit's elements of the tile that lie before P_lo
  // (those of groups < lo * nseg; the digit's run is in group order)
  const uint32_t ownw = m->own[par], nown = ownw >> 16;
  if (nown) {
    const uint32_t lo0 = ownw & 0xffffu, cd = c.cnt[dme];
    for (uint32_t lo = lo0; lo < lo0 + nown; ++lo) {
      const uint32_t gl = lo * c.nseg;
      uint32_t before;
      if (k == 0) {
        before = g0 < gl ? cd : 0u;
      } else {
        uint32_t lo_i = 0, hi_i = cd;
        while (lo_i < hi_i) {
          const uint32_t mid = (lo_i + hi_i) >> 1;
          if (g0 + G16[dlocal + mid] < gl)
            lo_i = mid + 1;
          else
            hi_i = mid;
        }
        before = lo_i;
      }
      a.ctl->vs16[(dme << 8) | lo] = vbase + before;
    }
  }

  // ---- scatter, rows form: the row id rebuilt from the packed word (the
  // keys are the value starts above)
  uint32_t* out = reinterpret_cast<uint32_t*>(a.X);
  if (k == 0) {
    const uint32_t rb = m->rbg[0];
#pragma unroll 4
    for (uint32_t jj = threadIdx.x; jj < tn; jj += SH::THREADS) {
      const uint32_t e = S32[jj];
      out[c.gbase[e >> 24] + jj] = rb + (e & 0xffffffu);
    }
  } else {
    for (uint32_t jj = threadIdx.x; jj < tn; jj += SH::THREADS) {
      const uint32_t e = S32[jj], d = e >> 24, gi = G16[jj];
      uint32_t kb, rb;
      if (k <= 32) {
        kb = m->kbg[gi];
        rb = m->rbg[gi];
      } else {
        const uint32_t g = g0 + gi, lo = g / c.nseg, seg = g - lo * c.nseg;
        kb = c.kbase | lo;
        rb = a.row_base + (seg << kSegBits);
      }
      (void)kb;
      out[c.gbase[d] + jj] = rb + (e & 0xffffffu);
    }
  }
  if (threadIdx.x == 0) claim_next_b(c, ctr, par);
  __syncthreads();
  if (SH::ALIAS && threadIdx.x == 0) {
    const uint32_t nt = m->tile[par ^ 1];
    if (nt < c.tiles && uint64_t(nt + 1) * TILE <= c.n) issue_tile_copy<KIND>(c, nt);
  }
}

__device__ __forceinline__ void run_lookback_b(PassCtx& c) {
  using SH = PassShape<kPassB>;
  uint32_t* ctr = &c.a.ctl->tile_ctr[kCtrB];
  PassMisc* m = c.m;
  static_assert(SH::THREADS == 256, "one low byte per thread");
  m->lo_start[threadIdx.x] = c.a.ctl->plan.bucket_start_byte[0][threadIdx.x];
  if (threadIdx.x == 0) {
    mbar_init(&m->bar, 1);
    fence_mbar_init();
    const uint32_t t = atomicAdd(ctr, 1u);
    m->tile[0] = t;
    if (t < c.tiles && uint64_t(t + 1) * SH::TILE <= c.n) issue_tile_copy<kPassB>(c, t);
    if (t < c.tiles) {
      group_words(c, t, 0);
      cp_async_wait_all();
    }
  }
  __syncthreads();
  if (threadIdx.x < 32 && m->tile[0] < c.tiles) {
    group_starts(c, 0);
    own_range(c, m->tile[0], 0);
    cp_async_wait_all();
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int it = 0;; ++it) {
    const int par = it & 1;
    const uint32_t tile = m->tile[par];
    if (tile >= c.tiles) break;
    if (uint64_t(tile + 1) * SH::TILE <= c.n)
      lookback_tile<true>(c, ctr, tile, par, phase, it > 0);
    else
      lookback_tile<false>(c, ctr, tile, par, phase, it > 0);
  }
}

// ---- kernels ------------------------------------------------------------------

// digit width class of the wide pass (the instantiation that runs it)
__host__ __device__ inline int wide_class(uint32_t bits) { return bits <= 4 ? 4 : bits <= 8 ? 8 : bits <= 9 ? 9 : bits <= 10 ? 10 : 11; }

template <int KIND, int BITS>
__device__ __forceinline__ void run_pass(const SortArgs& a, int bulk_ok, unsigned char* smem) {
  using SH = PassShape<KIND>;
  using SM = PassSmem<KIND, BITS>;
  PassCtx c;
  c.a = a;
  c.inbuf = reinterpret_cast<uint32_t*>(smem + SM::kInOfs);
  c.R = smem + SM::kROfs;
  c.cnt = reinterpret_cast<uint32_t*>(smem + SM::kCntOfs);
  c.gbase = c.cnt + SM::NB;
  c.run = c.gbase + SM::NB;
  c.m = reinterpret_cast<PassMisc*>(smem + SM::kMiscOfs);
  const SortPlan& pl = a.ctl->plan;
  c.n = a.n;
  c.tiles = uint32_t(ceil_div(a.n, SH::TILE));
  c.epoch = a.ctl->epoch + kEpochB;
  c.src = KIND == kPassB ? reinterpret_cast<const uint32_t*>(a.Y) : a.in_keys;
  c.bstart = pl.bucket_start_byte[1];
  c.kbase = pl.base;
  c.nseg = pl.nseg;
  c.bulk = bulk_ok != 0;
  if constexpr (KIND == kPassB)
    run_lookback_b(c);
  else
    run_chunked<KIND, BITS>(c);
}

// One kernel per pass kind; the wide pass picks its digit width at run
// time.  A kernel the plan did not pick returns at once: the host launches
// the candidates in stream order and never waits for the plan.
template <int KIND>
__global__ __launch_bounds__(PassShape<KIND>::THREADS, PassShape<KIND>::MINB) void k_tma_pass(SortArgs a,
                                                                                               int bulk_ok) {
  extern __shared__ __align__(128) unsigned char smem[];
  const SortPlan& pl = a.ctl->plan;
  if constexpr (KIND == kPassWide) {
    if (pl.mode != kModeWide) return;
    switch (wide_class(pl.wide_bits)) {
      case 4: return run_pass<kPassWide, 4>(a, bulk_ok, smem);
      case 8: return run_pass<kPassWide, 8>(a, bulk_ok, smem);
      case 9: return run_pass<kPassWide, 9>(a, bulk_ok, smem);
      case 10: return run_pass<kPassWide, 10>(a, bulk_ok, smem);
      default: return run_pass<kPassWide, 11>(a, bulk_ok, smem);
    }
  } else {
    if (pl.mode != kModeAB) return;
    run_pass<KIND, 8>(a, bulk_ok, smem);
  }
}

template <int KIND>
constexpr size_t pass_smem() {
  return PassSmem<KIND, KIND == kPassWide ? kWideMaxBits : 8>::kBytes;  // the widest digit
}

template <int MAXB, int V>
__global__ void k_pass(SortArgs a, int which);  // legacy wide pass (wah_sort.cu)
__global__ void k_pass_bytes(SortArgs a);        // legacy byte passes, one cooperative launch (wah_sort.cu)


// ---------------------------------------------------------------- host ----

struct PassCfg {
  int sms = 0;
  int occ_wide = 1, occ_a = 1, occ_b = 1;
};

template <int KIND>
static int pass_attr(int* occ) {
  const void* f = reinterpret_cast<const void*>(k_tma_pass<KIND>);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pass_smem<KIND>()));
  if (e) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, f, PassShape<KIND>::THREADS, pass_smem<KIND>());
  if (!e && *occ < 1) *occ = 1;
  return e;
}

static int pass_cfg(const PassCfg** out) {
  static PassCfg cfg[64];
  static std::once_flag once[64];
  static int rc_of[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  std::call_once(once[dev & 63], [dev] {
    PassCfg& c = cfg[dev & 63];
    int& rc = rc_of[dev & 63];
    if ((rc = cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev))) return;
    if ((rc = pass_attr<kPassWide>(&c.occ_wide))) return;
    if ((rc = pass_attr<kPassA>(&c.occ_a))) return;
    rc = pass_attr<kPassB>(&c.occ_b);
  });
  if (rc_of[dev & 63]) return rc_of[dev & 63];
  *out = &cfg[dev & 63];
  return 0;
}

// The first pass's chunk count for n keys on this device: one chunk per
// resident pass-A CTA (the wide pass walks several per CTA).
int first_pass_chunks(uint64_t n, uint32_t* k) {
  const PassCfg* c;
  int rc = pass_cfg(&c);
  if (rc) return rc;
  // one chunk per resident pass-A CTA, or two when each still holds at
  // least 16 blocks (2^18 keys): C4 -- 2^28 keys -- sorts 23 us faster in 888
  // chunks than in 444; below that the per-chunk counts cost more than the
  // smaller chunks gain (C3 +8 us in 888)
#ifndef NDX_CHUNK_WAVES
#define NDX_CHUNK_WAVES 2
#endif
#ifndef NDX_CHUNK_MIN_BLOCKS
#define NDX_CHUNK_MIN_BLOCKS 16
#endif
  const uint64_t resident = uint64_t(c->sms) * c->occ_a;
  const uint64_t blocks = ceil_div(n, kChunkBlock);
  const uint64_t waves = blocks >= NDX_CHUNK_WAVES * resident * NDX_CHUNK_MIN_BLOCKS ? NDX_CHUNK_WAVES : 1;
  *k = chunk_count(n, uint32_t(waves * resident));
  return 0;
}

// The sort stage: the candidate passes in stream order, each returning at
// once unless the plan picked it.  (Launching exactly the picked passes from
// the device -- CUDA dynamic parallelism tail launches -- was measured 1.45
// ms slower on C4: device-launched grids of the compact passes ran at about
// two thirds of their host-launched speed; ncu does not profile them either.)
int launch_sort_dispatch(const SortArgs& a, int legacy, int byte_grid, int legacy_wide_grid, cudaStream_t s) {
  const PassCfg* c;
  int rc = pass_cfg(&c);
  if (rc) return rc;
  const int bulk_keys = (reinterpret_cast<uintptr_t>(a.in_keys) & 15u) == 0;
  if (legacy) {
    k_pass<kWideMaxBits, 0><<<legacy_wide_grid, 512, kLegacyWideSmem, s>>>(a, -1);
  } else {
    const int gw = int(umin<uint64_t>(a.nchunk, uint64_t(c->sms) * c->occ_wide));
    const int gb = int(umin<uint64_t>(ceil_div(a.n, kBTile), uint64_t(c->sms) * c->occ_b));
    k_tma_pass<kPassWide><<<gw, PassShape<kPassWide>::THREADS, pass_smem<kPassWide>(), s>>>(a, bulk_keys);
    k_tma_pass<kPassA><<<a.nchunk, PassShape<kPassA>::THREADS, pass_smem<kPassA>(), s>>>(a, bulk_keys);
    k_tma_pass<kPassB><<<gb, PassShape<kPassB>::THREADS, pass_smem<kPassB>(), s>>>(a, 1);
  }
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  // general keys: every byte pass in one cooperative launch (grid barriers)
  SortArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_pass_bytes), dim3(byte_grid), dim3(256),
                                     params, kLegacyByteSmem, s);
}

}  // namespace ndx
