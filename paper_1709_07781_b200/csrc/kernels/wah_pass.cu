// TMA-staged scatter passes of the WAH sort (stage S2) on sm_100a.
//
// Replaces the reference's stable LSD radix sort of (value, row) pairs
// (p/core/src/wah_radix.cpp:16-127, row_iota at wah_builder.cpp:54-60) for
// the two key shapes of the BASELINE workloads, each in as few HBM bytes as
// the shape allows:
//
//   wide   key range < 2^11 (C1, C3): ONE pass on digit = key - min.
//          keys (4 B) in, (key, row) pairs (8 B) out; rows synthesised.
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
//          tile_group and GB by position.  Out: (key, row) pairs.
//   Bytes per element: wide 12; A + B 8 + 12 = 20 (the u64 ping-pong of
//   the legacy byte passes, wah_sort.cu, moves 12 + 16 = 28).
//
// Per tile (persistent CTAs, tiles taken in order from an atomic counter):
//   1. the tile arrives in shared memory by one TMA bulk copy
//      (cp.async.bulk + mbarrier), issued while the previous tile was being
//      ranked; every thread then reads its elements with conflict-free LDS
//   2. warp ballot-match ranking (lane order == row order: stable), per-warp
//      digit counters in shared memory
//   3. digit counts published (decoupled look-back status), local scan
//   4. staging in shared memory in digit order (u32 for wide/A, the final
//      pair for B) while the look-back resolves the tile's global bases
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
// input buffer aliased with the staging area (no TMA overlap inside a CTA,
// half the shared memory, so more CTAs per SM)
#ifndef NDX_WIDE_ALIAS
#define NDX_WIDE_ALIAS 0
#endif
#ifndef NDX_A_ALIAS
#define NDX_A_ALIAS 0
#endif
#ifndef NDX_B_ALIAS
#define NDX_B_ALIAS 1
#endif
// claim the next tile at the end of this one (claim order == processing
// order, so a tile's predecessors are ahead of it when it looks back), its
// TMA copy then, and an L2 prefetch of the tile one CTA round further on;
// 0: claim (and copy) at the start of this tile, a whole tile ahead
#ifndef NDX_CLAIM_LATE
#define NDX_CLAIM_LATE 1
#endif
// every lane reads its digit's counter (broadcast) instead of leader + shfl
#ifndef NDX_WIDE_BCAST
#define NDX_WIDE_BCAST 1
#endif
#ifndef NDX_AB_BCAST
#define NDX_AB_BCAST 1  // C4 sort 2.451 vs 2.511 ms with leader read + shuffle
#endif
// warps that resolve the look-back of a compact-pass tile (each lane takes
// 256 / (32 x warps) digits, their first status reads in flight together);
// 0: every thread resolves its own digit, first read before the staging
#ifndef NDX_AB_LB_WARPS
#define NDX_AB_LB_WARPS 0  // 1 warp: 6.94 ms C4 sort, 2 warps: 4.51 ms, every thread: 2.50 ms
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
  using Stage = typename std::conditional<KIND == kPassB, uint64_t, uint32_t>::type;
  static_assert(TILE <= 65536 && (TILE & (TILE - 1)) == 0, "ranks ride in 16 bits; tiles are powers of two");
  static_assert(KIND != kPassWide || LOCAL_BITS + kWideMaxBits <= 32, "wide staging packs digit | local");
  static_assert(KIND != kPassA || LOCAL_BITS <= 16, "pass-A staging packs lo | hb | local");
};

// Shared memory of one CTA: [in: TILE u32][R: H | S][cnt NB][gbase NB][Misc]
struct PassMisc {
  uint64_t bar;            // mbarrier of the input bulk copy
  uint32_t tile[2];        // tile taken for iteration parity 0/1
  uint32_t tg[2][2];       // pass B: tile_group[t], tile_group[t+1] per parity
  uint32_t sgb[2][32];     // pass B: group starts inside the tile per parity
};

template <int KIND, int BITS>
struct PassSmem {
  using SH = PassShape<KIND>;
  static constexpr int NB = 1 << BITS;
  static constexpr size_t kIn = size_t(SH::TILE) * 4;
  static constexpr size_t kH = size_t(SH::WARPS) * NB * 2;
  static constexpr size_t kS = size_t(SH::TILE) * sizeof(typename SH::Stage);
  static constexpr size_t kR0 = kH > kS ? kH : kS;
  static constexpr size_t kR = SH::ALIAS ? (kR0 > kIn ? kR0 : kIn) : kR0;
  static constexpr size_t kInOfs = 0;
  static constexpr size_t kROfs = SH::ALIAS ? 0 : kIn;
  static constexpr size_t kCntOfs = kROfs + kR;
  static constexpr size_t kMiscOfs = kCntOfs + 2 * NB * 4;
  static constexpr size_t kBytes = kMiscOfs + sizeof(PassMisc);
};

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(smem_dst)), "l"(gsrc) : "memory");
}
// lo16(a) | lo16(b) << 16 in one register.  Opaque to the compiler on
// purpose: with plain shifts and ors it sees through the packing and keeps
// the two halves in separate registers again (spilling the tile).
__device__ __forceinline__ uint32_t pack16(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// (lo, hi) to shared memory, in program order (volatile: keeps the
// scheduler from hoisting a whole unrolled tile's values into registers)
__device__ __forceinline__ void sts_pair(uint32_t addr, uint32_t lo, uint32_t hi) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(lo), "r"(hi) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Everything a tile needs besides its index (one per CTA, built once).
struct PassCtx {
  SortArgs a;
  const uint32_t* src;     // tile input (keys, or pass A's packed words)
  const uint32_t* bstart;  // global bucket starts of this pass's digits
  uint32_t* ctr;           // tile counter
  uint64_t n;
  uint32_t tiles, epoch;
  uint32_t kbase;          // wide: digit = key - kbase; A/B: the keys' top 16 bits
  uint32_t nseg;           // A/B: row segments
  bool bulk;               // input 16-byte aligned: tiles arrive by TMA
  uint32_t* inbuf;
  unsigned char* R;
  uint32_t* cnt;
  uint32_t* gbase;
  PassMisc* m;
};

template <int KIND, int BITS>
__device__ __forceinline__ void issue_tile_copy(const PassCtx& c, uint32_t t) {  // one thread
  fence_proxy_async_smem();
  mbar_expect_tx(&c.m->bar, PassShape<KIND>::TILE * 4);
  bulk_g2s(c.inbuf, c.src + uint64_t(t) * PassShape<KIND>::TILE, PassShape<KIND>::TILE * 4, &c.m->bar);
}

// pass B: the groups a tile crosses, staged by cp.async a tile ahead
__device__ __forceinline__ void group_words(const PassCtx& c, uint32_t t, int par) {  // thread 0
  cp_async4(&c.m->tg[par][0], c.a.tile_group + t);
  cp_async4(&c.m->tg[par][1], c.a.tile_group + t + 1);
}
__device__ __forceinline__ void group_starts(const PassCtx& c, int par) {  // warp 0, after tg[par] landed
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t g0 = c.m->tg[par][0], k = c.m->tg[par][1] - g0;
  if (k <= 32 && lane < k) cp_async4(&c.m->sgb[par][lane], c.a.gb + g0 + 1 + lane);
}

// One tile.  FULL: all TILE elements exist (every tile but the last).
template <int KIND, int BITS>
__device__ __forceinline__ void claim_next(const PassCtx& c, int par) {  // thread 0
  constexpr uint32_t TILE = PassShape<KIND>::TILE;
  const uint32_t nt = atomicAdd(c.ctr, 1u);
  c.m->tile[par ^ 1] = nt;
  if (nt >= c.tiles) return;
  if (!PassShape<KIND>::ALIAS && c.bulk && uint64_t(nt + 1) * TILE <= c.n) issue_tile_copy<KIND, BITS>(c, nt);
  if (KIND == kPassB) group_words(c, nt, par ^ 1);
  if (NDX_CLAIM_LATE && c.bulk) {
    const uint64_t pf = uint64_t(nt) + gridDim.x;  // about one CTA round ahead
    if ((pf + 1) * TILE <= c.n)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c.src + pf * TILE), "r"(TILE * 4u) : "memory");
  }
}

template <int KIND, int BITS, bool FULL>
__device__ __forceinline__ void tma_tile(const PassCtx& c, uint32_t tile, int par, uint32_t& phase, bool later) {
  using SH = PassShape<KIND>;
  using Stage = typename SH::Stage;
  constexpr uint32_t NB = 1u << BITS;
  constexpr uint32_t DMASK = NB - 1;
  constexpr int IPT = SH::IPT;
  constexpr uint32_t TILE = SH::TILE;
  constexpr uint32_t LB = SH::LOCAL_BITS;
  constexpr bool kEarly = KIND != kPassWide && NDX_AB_LB_WARPS == 0;  // first look-back read before the staging
  constexpr int LBW = KIND != kPassWide ? NDX_AB_LB_WARPS : 0;  // look-back warps (0: all threads)
  const SortArgs& a = c.a;
  uint16_t* H = reinterpret_cast<uint16_t*>(c.R);
  Stage* S = reinterpret_cast<Stage*>(c.R);
  uint32_t* cnt = c.cnt;
  uint32_t* gbase = c.gbase;
  PassMisc* m = c.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ts = uint64_t(tile) * TILE;
  const uint32_t tn = FULL ? TILE : uint32_t(c.n - ts);
  const uint32_t wofs = uint32_t(warp) * SH::WI + lane;

  // ---- 1. elements into registers
  uint32_t x[IPT];
  if (FULL && c.bulk) {
    mbar_wait(&m->bar, phase);
    phase ^= 1u;
#pragma unroll
    for (int r = 0; r < IPT; ++r) x[r] = c.inbuf[wofs + r * 32];
  } else {
#pragma unroll
    for (int r = 0; r < IPT; ++r) x[r] = (FULL || wofs + r * 32 < tn) ? __ldg(c.src + ts + wofs + r * 32) : 0u;
  }
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    if (KIND == kPassWide) x[r] = (x[r] - c.kbase) & DMASK;  // digit < 2^11; the rank goes above bit 16
    if (KIND == kPassA) x[r] &= 0xffffu;                     // lo | hb << 8; the rank goes above bit 16
  }
  if (NDX_CLAIM_LATE && KIND == kPassB && later && warp == 0) {
    // this tile's group words were requested at its claim: now its group starts
    if (lane == 0) cp_async_wait_all();
    __syncwarp();
    group_starts(c, par);
  }
  __syncthreads();  // inbuf consumed; R free (previous scatter done)
  if (!NDX_CLAIM_LATE && threadIdx.x == 0) claim_next<KIND, BITS>(c, par);

  // ---- 2. rank
  uint16_t* Hw = H + warp * NB;
  for (uint32_t d = lane; d < NB; d += 32) Hw[d] = 0;
  __syncwarp();
  auto digit = [&](uint32_t v) -> uint32_t {
    if (KIND == kPassB) return v >> 24;
    return v & DMASK;
  };
  constexpr bool kPackRank = KIND == kPassB;  // wide/A: the rank sits in bits 16..31 of x
  uint32_t rk2[kPackRank ? IPT / 2 : 1];
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t d = digit(x[r]);
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
    if constexpr (kPackRank) {
      if ((r & 1) == 0)
        rk2[r >> 1] = rk;
      else
        rk2[r >> 1] = pack16(rk2[r >> 1], rk);
    } else {
      x[r] = pack16(x[r], rk);
    }
  }
  if (KIND == kPassB && warp == 0) cp_async_wait_all();  // this tile's group starts (issued a tile ago)
  __syncthreads();

  // ---- 3. counts: warp offsets in place, tile counts published, local starts
  uint64_t* st = a.status + uint64_t(tile) * NB;
  for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS) {
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < SH::WARPS; ++w) {
      const uint32_t cw = H[w * NB + d];
      H[w * NB + d] = uint16_t(sum);
      sum += cw;
    }
    cnt[d] = sum;
    st_relaxed_u64(&st[d], st_word(c.epoch, tile == 0 ? kStPrefix : kStAgg, sum));
  }
  __syncthreads();
  block_excl_scan(cnt, gbase, int(NB));  // gbase <- tile-local digit starts (syncs)

  constexpr int ND = int((NB + SH::THREADS - 1) / SH::THREADS);
  uint64_t first[kEarly ? ND : 1] = {};
  // global base of digit d for this tile; s0 = the status of tile-1 for d
  // when already read (from_s0), else the look-back reads it
  auto resolve_with = [&](uint32_t d, bool from_s0, uint64_t s0) {
    const uint32_t cd = cnt[d], local = gbase[d];
    uint64_t excl = 0;
    if (tile > 0) {
      excl = from_s0 ? lookback_from(a.status, tile, NB, d, c.epoch, s0) : lookback(a.status, tile, NB, d, c.epoch);
      st_relaxed_u64(&st[d], st_word(c.epoch, kStPrefix, excl + cd));
    }
    const uint32_t gstart = c.bstart[d] + uint32_t(excl);
    gbase[d] = gstart - local;
    if constexpr (KIND == kPassA) {
      // segment starts, and the pass-B tiles that begin inside this run
      const uint32_t seg = uint32_t(ts >> kSegBits);
      if ((ts & ((1ull << kSegBits) - 1)) == 0) a.gb[d * c.nseg + seg] = gstart;
      for (uint32_t mt = uint32_t(ceil_div(gstart, kBTile)); uint64_t(mt) * kBTile < uint64_t(gstart) + cd; ++mt)
        a.tile_group[mt] = d * c.nseg + seg;
    }
  };
  auto resolve = [&](int k, uint32_t d) {
    if constexpr (kEarly)
      resolve_with(d, true, first[k]);
    else
      resolve_with(d, false, 0ull);
    (void)k;
  };
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    const uint32_t d = threadIdx.x + uint32_t(k) * SH::THREADS;
    if (d < NB) {
      const uint32_t local = gbase[d];
      if constexpr (kEarly)
        first[k] = tile > 0 ? ld_relaxed_u64(&a.status[uint64_t(tile - 1) * NB + d]) : 0ull;
      else if constexpr (LBW == 0)
        resolve(k, d);  // look-back first; the local starts go into the counters after it
#pragma unroll
      for (int w = 0; w < SH::WARPS; ++w) H[w * NB + d] += uint16_t(local);
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t add = Hw[digit(x[r])];
    if constexpr (kPackRank)
      rk2[r >> 1] += add << (16 * (r & 1));
    else
      x[r] += add << 16;
  }
  __syncthreads();  // H dead: S may overwrite it

  // ---- 4. staging in digit order
  if constexpr (KIND == kPassB) {
    // group (lo, seg) of each element: walk the group starts inside the
    // tile (positions increase with r)
    const uint32_t g0 = m->tg[par][0], k = m->tg[par][1] - g0;
    const uint32_t* sg = m->sgb[par];
    const uint32_t p0 = uint32_t(ts) + wofs;
    uint32_t j = 0, nb = 0xffffffffu, kb = 0, rb = 0;
    auto set_group = [&](uint32_t g) {
      const uint32_t lo = g / c.nseg, seg = g - lo * c.nseg;
      kb = c.kbase | lo;
      rb = a.row_base + (seg << kSegBits);
    };
    if (k <= 32) {
      set_group(g0);
      if (k > 0) nb = sg[0];
    }
    const uint32_t s_base = smem_addr(S);
    if (k == 0) {  // the whole tile inside one group: (key, row) bases fixed
#pragma unroll
      for (int r = 0; r < IPT; ++r)
        if (FULL || wofs + r * 32 < tn) {
          const uint32_t v = x[r];
          sts_pair(s_base + 8u * ((rk2[r >> 1] >> (16 * (r & 1))) & 0xffffu), kb | ((v >> 24) << 8),
                   rb + (v & 0xffffffu));
        }
    } else {
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
      const uint32_t p = p0 + uint32_t(r) * 32;
      if (k <= 32) {
        if (p >= nb) {
          while (j < k && p >= sg[j]) ++j;
          nb = j < k ? sg[j] : 0xffffffffu;
          set_group(g0 + j);
        }
      } else {
        // pathological tile (more than 32 groups start inside it): count the
        // group starts GB[g0+1 .. g0+k] <= p by binary search
        uint32_t lo_i = 0, hi_i = k;
        while (lo_i < hi_i) {
          const uint32_t mid = (lo_i + hi_i) >> 1;
          if (__ldg(a.gb + g0 + 1 + mid) <= p)
            lo_i = mid + 1;
          else
            hi_i = mid;
        }
        set_group(g0 + lo_i);
      }
      if (FULL || wofs + r * 32 < tn) {
        const uint32_t v = x[r];
        sts_pair(s_base + 8u * ((rk2[r >> 1] >> (16 * (r & 1))) & 0xffffu), kb | ((v >> 24) << 8),
                 rb + (v & 0xffffffu));
      }
    }
    }
  } else {
#pragma unroll
    for (int r = 0; r < IPT; ++r)
      if (FULL || wofs + r * 32 < tn) {
        const uint32_t v = x[r], local = wofs + r * 32;
        if (KIND == kPassWide)
          S[v >> 16] = ((v & DMASK) << LB) | local;
        else  // hb << 24 | lo << 16 | local (v << 16 drops the rank)
          S[v >> 16] = (v << 16) | local;
      }
  }
  if constexpr (kEarly) {
    // look-back, part 2: finish from the status already in hand
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const uint32_t d = threadIdx.x + uint32_t(k) * SH::THREADS;
      if (d < NB) resolve(k, d);
    }
  } else if constexpr (LBW > 0) {
    // LBW warps resolve every digit: the first status of each of a lane's
    // digits is requested at once, the rest of the CTA does not spin
    if (warp < LBW) {
      constexpr int DPL = int(NB) / (32 * LBW);
      static_assert(DPL * 32 * LBW == int(NB), "digits per look-back lane");
      uint64_t s0[DPL];
#pragma unroll
      for (int j = 0; j < DPL; ++j) {
        const uint32_t d = uint32_t(lane + 32 * (warp + LBW * j));
        s0[j] = tile > 0 ? ld_relaxed_u64(&a.status[uint64_t(tile - 1) * NB + d]) : 0ull;
      }
#pragma unroll
      for (int j = 0; j < DPL; ++j) resolve_with(uint32_t(lane + 32 * (warp + LBW * j)), true, s0[j]);
    }
  }
  __syncthreads();

  // ---- 5. scatter: consecutive slots of one digit are consecutive globally
  if constexpr (KIND == kPassA) {
    uint32_t* out = reinterpret_cast<uint32_t*>(a.Y);
    const uint32_t segofs = uint32_t(ts) & ((1u << kSegBits) - 1);
#pragma unroll 4
    for (uint32_t jj = threadIdx.x; jj < tn; jj += SH::THREADS) {
      const uint32_t e = S[jj];
      out[gbase[(e >> 16) & 0xffu] + jj] = (e & 0xff000000u) | (segofs + (e & 0xffffu));
    }
  } else if constexpr (KIND == kPassWide) {
    const uint32_t rbase = a.row_base + uint32_t(ts);
#pragma unroll 4
    for (uint32_t jj = threadIdx.x; jj < tn; jj += SH::THREADS) {
      const uint32_t e = S[jj], d = e >> LB;
      a.X[gbase[d] + jj] = uint64_t(c.kbase + d) | (uint64_t(rbase + (e & ((1u << LB) - 1))) << 32);
    }
  } else {
#pragma unroll 4
    for (uint32_t jj = threadIdx.x; jj < tn; jj += SH::THREADS) {
      const uint64_t e = S[jj];
      a.X[gbase[(uint32_t(e) >> 8) & 0xffu] + jj] = e;
    }
  }
  if (NDX_CLAIM_LATE) {
    if (threadIdx.x == 0) claim_next<KIND, BITS>(c, par);
  } else if (KIND == kPassB && warp == 0 && m->tile[par ^ 1] < c.tiles) {
    if (lane == 0) cp_async_wait_all();  // tile_group words of the next tile
    __syncwarp();
    group_starts(c, par ^ 1);
  }
  __syncthreads();
  if (SH::ALIAS && threadIdx.x == 0) {
    const uint32_t nt = m->tile[par ^ 1];
    if (nt < c.tiles && c.bulk && uint64_t(nt + 1) * TILE <= c.n) issue_tile_copy<KIND, BITS>(c, nt);
  }
}

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
  c.m = reinterpret_cast<PassMisc*>(smem + SM::kMiscOfs);
  const SortPlan& pl = a.ctl->plan;
  c.n = a.n;
  c.tiles = uint32_t(ceil_div(a.n, SH::TILE));
  c.ctr = &a.ctl->tile_ctr[KIND == kPassWide ? kCtrWide : (KIND == kPassA ? kCtrA : kCtrB)];
  c.epoch = a.ctl->epoch + (KIND == kPassWide ? kEpochWide : (KIND == kPassA ? kEpochA : kEpochB));
  c.src = KIND == kPassB ? reinterpret_cast<const uint32_t*>(a.Y) : a.in_keys;
  c.bstart = KIND == kPassWide ? pl.bucket_start_wide : (KIND == kPassA ? pl.bucket_start_byte[0] : pl.bucket_start_byte[1]);
  c.kbase = pl.base;
  c.nseg = pl.nseg;
  c.bulk = bulk_ok != 0;
  PassMisc* m = c.m;

  if (threadIdx.x == 0) {
    mbar_init(&m->bar, 1);
    fence_mbar_init();
    const uint32_t t = atomicAdd(c.ctr, 1u);
    m->tile[0] = t;
    if (t < c.tiles && c.bulk && uint64_t(t + 1) * SH::TILE <= c.n) issue_tile_copy<KIND, BITS>(c, t);
    if (KIND == kPassB && t < c.tiles) {
      group_words(c, t, 0);
      cp_async_wait_all();
    }
  }
  __syncthreads();
  if (KIND == kPassB && threadIdx.x < 32 && m->tile[0] < c.tiles) {
    group_starts(c, 0);
    cp_async_wait_all();
  }
  __syncthreads();

  uint32_t phase = 0;
  for (int it = 0;; ++it) {
    const int par = it & 1;
    const uint32_t tile = m->tile[par];
    if (tile >= c.tiles) break;
    if (uint64_t(tile + 1) * SH::TILE <= c.n)
      tma_tile<KIND, BITS, true>(c, tile, par, phase, it > 0);
    else
      tma_tile<KIND, BITS, false>(c, tile, par, phase, it > 0);
  }
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

__global__ void k_set_row_hi(SortArgs a) { a.ctl->row_hi = a.row_base + uint32_t(a.n - 1); }  // read by emit

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

static int pass_cfg_init(PassCfg& c, int dev) {
  int e;
  if ((e = cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev))) return e;
  if ((e = pass_attr<kPassWide>(&c.occ_wide))) return e;
  if ((e = pass_attr<kPassA>(&c.occ_a))) return e;
  if ((e = pass_attr<kPassB>(&c.occ_b))) return e;
  return 0;
}

// The sort stage: the candidate passes in stream order, each returning at
// once unless the plan picked it.  (Launching exactly the picked passes from
// the device -- CUDA dynamic parallelism tail launches -- was measured 1.45
// ms slower on C4: device-launched grids of the compact passes ran at about
// two thirds of their host-launched speed; ncu does not profile them either.)
int launch_sort_dispatch(const SortArgs& a, int legacy, int byte_grid, int legacy_wide_grid, cudaStream_t s) {
  static PassCfg cfg[64];
  static std::once_flag once[64];
  static int rc_of[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  std::call_once(once[dev & 63], [dev] { rc_of[dev & 63] = pass_cfg_init(cfg[dev & 63], dev); });
  if (rc_of[dev & 63]) return rc_of[dev & 63];
  const PassCfg& c = cfg[dev & 63];
  const int bulk_keys = (reinterpret_cast<uintptr_t>(a.in_keys) & 15u) == 0;
  k_set_row_hi<<<1, 1, 0, s>>>(a);
  if (legacy) {
    k_pass<kWideMaxBits, 0><<<legacy_wide_grid, 512, kLegacyWideSmem, s>>>(a, -1);
  } else {
    const int gw = int(umin<uint64_t>(ceil_div(a.n, kWideTile), uint64_t(c.sms) * c.occ_wide));
    const int ga = int(umin<uint64_t>(ceil_div(a.n, kATile), uint64_t(c.sms) * c.occ_a));
    const int gb = int(umin<uint64_t>(ceil_div(a.n, kBTile), uint64_t(c.sms) * c.occ_b));
    k_tma_pass<kPassWide><<<gw, PassShape<kPassWide>::THREADS, pass_smem<kPassWide>(), s>>>(a, bulk_keys);
    k_tma_pass<kPassA><<<ga, PassShape<kPassA>::THREADS, pass_smem<kPassA>(), s>>>(a, bulk_keys);
    k_tma_pass<kPassB><<<gb, PassShape<kPassB>::THREADS, pass_smem<kPassB>(), s>>>(a, 1);
  }
  if ((e = cudaGetLastError())) return e;
  // general keys: every byte pass in one cooperative launch (grid barriers)
  SortArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_pass_bytes), dim3(byte_grid), dim3(256),
                                     params, kLegacyByteSmem, s);
}

}  // namespace ndx
