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
//
// Two kernels, one per form of the sorted stream (wah_sort.cu): k_emit_rows
// for the rows form (u32 row ids, the value heads from ctl->vs; the wide and
// compact sorts) and k_emit for the pairs form (u64 (key, row); general
// keys).  Both are launched; the one that does not apply returns at once.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "../../../include/ndx.h"
#include "common.cuh"
#include "wah_internal.cuh"

namespace ndx {

#ifndef NDX_EMIT_THREADS
#define NDX_EMIT_THREADS 256
#endif
#ifndef NDX_EMIT_MINB
#define NDX_EMIT_MINB 1
#endif
constexpr int kEmitThreads = NDX_EMIT_THREADS;
constexpr int kEmitWarps = kEmitThreads / 32;
// 14 pairs per thread: 112-byte thread stride, so the 16-byte shared loads
// of a quarter warp hit 8 distinct bank groups (8 pairs -> 64 B stride was a
// 4-way conflict; measured C4 emit 1.49 -> 1.00 ms).  Must be even and < 31.
#ifndef NDX_EMIT_L2PF
#define NDX_EMIT_L2PF 0
#endif
#ifndef NDX_EMIT_K
#define NDX_EMIT_K 14
#endif
#ifndef NDX_EMIT_ROWS_MINB
#define NDX_EMIT_ROWS_MINB 3
#endif
#ifndef NDX_EMIT_AGGPRE
#define NDX_EMIT_AGGPRE 2
#endif
static_assert(NDX_EMIT_K % 2 == 0 && NDX_EMIT_K < 31, "span length");
constexpr int kEmitK = NDX_EMIT_K;                      // consecutive elements per thread
constexpr int kEmitTile = kEmitThreads * kEmitK;        // 1024
constexpr int kHaloL = 32;                              // elements before the tile (carry, prev)
constexpr int kHaloR = 2;                               // elements after it (next; 16 B multiple)
constexpr int kEmitBuf = kHaloL + kEmitTile + kHaloR;
// staging of one tile: 2*kEmitTile words, then kEmitTile table-head values
// and kEmitTile table-head word offsets (tile-local)
// words (2 per pair at most), head values (u32) and head word offsets (u16:
// below 2 * kEmitTile) -- u16 offsets keep two CTAs' worth of buffers in an SM
constexpr int kStageTile = 3 * kEmitTile + kEmitTile / 2;
static_assert(2 * kEmitTile < 65536, "head offsets are u16");
constexpr size_t kEmitSmem = size_t(2 * kEmitBuf) * 8 + size_t(kStageTile) * 4;

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

// Phase-1 summary of one thread's kEmitK consecutive elements ("span").
struct Span {
  uint32_t pk[kEmitK];  // per element: gap-fill length (0: no gap word), << 5 | row % 31 when SMALL
  uint32_t hmask;       // run heads
  uint32_t vmask;       // value heads (first element of a value)
  uint32_t tmask;       // run tails
  uint32_t acc;         // OR of the bits since the last head (or the span start)
  uint32_t nwords;      // words this span emits
  uint32_t first_body;  // 1: literal; 0: swallowed; else the ones-fill word (first run only)
};

// All-ones check of the span's first run when it began before the span
// (the only run of a span that can be all-ones: one that starts inside the
// span either ends inside it with at most kEmitK < 31 elements, or continues
// into a later span where it is that span's first run).
template <bool SMALL>
__device__ __forceinline__ void first_run_check(const uint64_t* B, const uint64_t* __restrict__ pairs,
                                                uint32_t n, uint32_t g0, uint32_t li0, Span& s) {
  s.first_body = 1;
  const uint32_t tm = s.tmask, hm = s.hmask;
  if (tm != 0 && (hm == 0 || __ffs(tm) < __ffs(hm))) {
    const uint32_t j = __ffs(tm) - 1;
    const uint64_t te = B[li0 + j];
    const uint32_t v = pkey(te), row = prow(te);
    if (row - div31<SMALL>(row) * kChunkBits == kChunkBits - 1 && g0 + j >= 30 &&
        B[int(li0 + j) - 30] == mkpair(v, row - 30)) {
      s.first_body = ones_body(pairs, n, g0 + j, v, row);
      if (s.first_body == 0) s.nwords -= 1;
    }
  }
}

// Phase 1: flags, gap lengths and word count of elements ts+li0 ..
// ts+li0+kEmitK-1.  FULL: the span and the element after it exist and the
// span does not start at element 0 (every tile that arrives by bulk copy).
template <bool SMALL, bool FULL>
__device__ __forceinline__ void span_scan(const uint64_t* B, const uint64_t* __restrict__ pairs,
                                          uint32_t n, uint32_t ts, uint32_t li0, Span& s) {
  // 4 x 16 B per thread (the 64 B stride costs 4-way bank conflicts, well
  // inside the shared-memory budget of ~0.25 wavefronts per element)
  uint64_t P[kEmitK];
  const uint4* B4 = reinterpret_cast<const uint4*>(B + li0);
#pragma unroll
  for (int p = 0; p < kEmitK / 2; ++p) {
    const uint4 u = B4[p];
    P[2 * p] = uint64_t(u.x) | (uint64_t(u.y) << 32);
    P[2 * p + 1] = uint64_t(u.z) | (uint64_t(u.w) << 32);
  }
  const uint64_t prv = B[int(li0) - 1], nxt = B[li0 + kEmitK];
  const uint32_t g0 = ts + li0;
  uint32_t pv = pkey(prv), pc = div31<SMALL>(prow(prv));
  uint32_t hm = 0, vm = 0, gaps = 0, acc = 0;
#pragma unroll
  for (int j = 0; j < kEmitK; ++j) {
    const uint32_t v = pkey(P[j]), row = prow(P[j]), c = div31<SMALL>(row);
    const uint32_t bp = row - c * kChunkBits;
    bool vh = v != pv, h = vh | (c != pc);
    if (!FULL) {
      const uint32_t g = g0 + j;
      const bool valid = g < n;
      vh = valid & (vh | (g == 0));
      h = valid & (h | (g == 0));
    }
    const uint32_t gap = h ? (vh ? c : c - pc - 1) : 0u;
    gaps += gap != 0;
    s.pk[j] = SMALL ? (gap << 5) | bp : gap;  // SMALL: chunks < 2^27
    hm |= uint32_t(h) << j;
    vm |= uint32_t(vh) << j;
    acc = (h ? 0u : acc) | (1u << bp);
    pv = v;
    pc = c;
  }
  const bool hN = (pkey(nxt) != pv) | (div31<SMALL>(prow(nxt)) != pc);
  uint32_t tm;
  if (FULL) {
    tm = (hm >> 1) | (uint32_t(hN) << (kEmitK - 1));
  } else {
    const uint32_t nvalid = g0 >= n ? 0u : umin(n - g0, uint32_t(kEmitK + 1));
    const uint32_t valid9 = (1u << nvalid) - 1u;
    const uint32_t h9 = hm | (uint32_t(hN) << kEmitK);
    tm = valid9 & ((1u << kEmitK) - 1u) & ((h9 >> 1) | (~valid9 >> 1));
  }
  s.hmask = hm;
  s.vmask = vm;
  s.tmask = tm;
  s.acc = acc;
  s.nwords = gaps + __popc(tm);
  first_run_check<SMALL>(B, pairs, n, g0, li0, s);
}

// Phase 2: write the span's words at tile-local offset o of `stage` and its
// value heads at h (hv: value, ho: tile-local offset of the value's first
// word).  `carry` is the OR of the span's first run before the span, so the
// running literal simply starts from it.
template <bool SMALL>
__device__ __forceinline__ uint32_t gap_of(uint32_t pk) {
  return SMALL ? pk >> 5 : pk;
}
template <bool SMALL>
__device__ __forceinline__ uint32_t bit_of(uint32_t pk, uint64_t e) {
  if (SMALL) return 1u << (pk & 31u);
  const uint32_t row = prow(e);
  return 1u << (row - (row / kChunkBits) * kChunkBits);
}

template <bool SMALL>
__device__ __forceinline__ void span_emit(const Span& s, const uint64_t* Bs, uint32_t carry,
                                          uint32_t o, uint32_t h, uint32_t* stage, uint32_t* hv,
                                          uint16_t* ho) {
  // shared-space addresses, bumped per word: one STS per word, no generic
  // address arithmetic
  uint32_t sa = smem_addr(stage) + 4u * o;
  uint32_t acc = carry;
  if (s.vmask == 0 && s.first_body == 1) {
#pragma unroll
    for (int j = 0; j < kEmitK; ++j) {
      const uint32_t gap = gap_of<SMALL>(s.pk[j]), bit = bit_of<SMALL>(s.pk[j], Bs[j]);
      if (gap) {
        sts_u32(sa, kFillFlag | gap);
        sa += 4;
      }
      acc = ((s.hmask >> j) & 1u) ? bit : (acc | bit);
      if ((s.tmask >> j) & 1u) {
        sts_u32(sa, acc);
        sa += 4;
      }
    }
    return;
  }
  const uint32_t sbase = smem_addr(stage);
#pragma unroll
  for (int j = 0; j < kEmitK; ++j) {
    const uint32_t gap = gap_of<SMALL>(s.pk[j]), bit = bit_of<SMALL>(s.pk[j], Bs[j]);
    if ((s.vmask >> j) & 1u) {
      hv[h] = pkey(Bs[j]);
      ho[h] = uint16_t((sa - sbase) >> 2);
      ++h;
    }
    if (gap) {
      sts_u32(sa, kFillFlag | gap);
      sa += 4;
    }
    acc = ((s.hmask >> j) & 1u) ? bit : (acc | bit);
    if ((s.tmask >> j) & 1u) {
      const bool first = (s.hmask & ((2u << j) - 1u)) == 0;
      const uint32_t body = (first && s.first_body != 1) ? s.first_body : acc;
      if (body) {
        sts_u32(sa, body);
        sa += 4;
      }
    }
  }
}

// OR of the bits of the elements before tile-local element wl that share
// its (value, chunk): the part of wl's run that lies before the warp (at
// most 30 elements, all inside the 32-element window read here).
template <bool SMALL>
__device__ __forceinline__ uint32_t warp_carry(const uint64_t* B, uint32_t ts, uint32_t wl) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t e0 = B[wl];
  const uint32_t v0 = pkey(e0), c0 = div31<SMALL>(prow(e0));
  const uint64_t q = B[int(wl) - 32 + int(lane)];
  const uint32_t qrow = prow(q), qc = div31<SMALL>(qrow);
  const bool m = (ts + wl + lane >= 32) & (pkey(q) == v0) & (qc == c0);
  return __reduce_or_sync(kFull, m ? 1u << (qrow - qc * kChunkBits) : 0u);
}

// Tile schedule: tiles are handed out in order by an atomic counter.  A
// tile's global offsets are the offsets of this CTA's previous tile plus the
// published aggregates of the tiles in between (about one per CTA) -- a
// block-wide read, never a serial look-back chain.  The CTA computes tile
// k's counts (publishing its aggregate) BEFORE it writes tile k-1 out, so by
// the time it needs the aggregates below tile k-1 the CTAs that took them
// have had a whole phase to publish.  All CTAs are co-resident (cooperative
// launch); a tile waits only on smaller tiles, taken earlier by CTAs that
// publish before they wait, so the schedule cannot deadlock.
//
// Tiles whose halo lies inside [0, n) arrive by one bulk async copy (TMA,
// mbarrier completion) issued a phase ahead; the first and last ones are
// gathered by the threads.

constexpr uint64_t kAggReady = 1ull << 63;

// Phase 1's scans across a warp's spans: the literal carried into each span
// (a segmented OR-scan over the spans' trailing ORs, bit 31 = the span holds
// a run head; the warp's first span gets wcarry) and, interleaved with it
// (two independent shuffle chains), the sum of the spans' (words << 16 |
// value heads).  Returns the inclusive sum; excl = the exclusive one.
__device__ __forceinline__ uint32_t span_scans(const Span& sp, uint32_t wcarry, uint32_t& carry_in,
                                               uint32_t& excl) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t x = (sp.hmask ? 0x80000000u : 0u) | sp.acc;
  const uint32_t cnt = (sp.nwords << 16) | uint32_t(__popc(sp.vmask));
  uint32_t incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, d);
    const uint32_t z = __shfl_up_sync(kFull, incl, d);
    if (lane >= uint32_t(d)) {
      if (!(x >> 31)) x |= y;
      incl += z;
    }
  }
  const uint32_t incl_lit = (x & kLiteralMask) | ((x >> 31) ? 0u : wcarry);
  carry_in = __shfl_up_sync(kFull, incl_lit, 1);
  if (lane == 0) carry_in = wcarry;
  excl = incl - cnt;
  return incl;
}

// The published (words, heads) aggregates of tiles [lo, hi): the first PRE
// per thread are requested a phase early (agg_request), the rest and any
// not yet published are read (waiting) when summed (agg_sum: this thread's
// share, words and heads).
template <int PRE>
__device__ __forceinline__ void agg_request(const uint64_t* agg, uint64_t lo, uint64_t hi, uint64_t (&pre)[PRE]) {
#pragma unroll
  for (int j = 0; j < PRE; ++j) {
    const uint64_t a = lo + threadIdx.x + uint64_t(j) * kEmitThreads;
    pre[j] = a < hi ? ld_relaxed_u64(&agg[a]) : kAggReady;
  }
}
template <int PRE>
__device__ __forceinline__ void agg_sum(const uint64_t* agg, uint64_t lo, uint64_t hi, const uint64_t (&pre)[PRE],
                                        uint32_t& sw, uint32_t& sd) {
  sw = sd = 0;
#pragma unroll
  for (int j = 0; j < PRE; ++j) {
    const uint64_t a = lo + threadIdx.x + uint64_t(j) * kEmitThreads;
    if (a >= hi) break;
    uint64_t s = pre[j];
    while (!(s & kAggReady)) {
      __nanosleep(32);
      s = ld_relaxed_u64(&agg[a]);
    }
    sw += uint32_t(s);
    sd += uint32_t(s >> 32) & 0x7fffffffu;
  }
  for (uint64_t j = lo + threadIdx.x + uint64_t(PRE) * kEmitThreads; j < hi; j += kEmitThreads) {
    uint64_t s = ld_relaxed_u64(&agg[j]);
    while (!(s & kAggReady)) {
      __nanosleep(32);
      s = ld_relaxed_u64(&agg[j]);
    }
    sw += uint32_t(s);
    sd += uint32_t(s >> 32) & 0x7fffffffu;
  }
}

template <bool SMALL>
__device__ __forceinline__ void tile_phase1(bool full, const uint64_t* B,
                                            const uint64_t* __restrict__ pairs, uint32_t n,
                                            uint32_t ts, uint32_t li0, Span& sp) {
  if (full)
    span_scan<SMALL, true>(B, pairs, n, ts, li0, sp);
  else
    span_scan<SMALL, false>(B, pairs, n, ts, li0, sp);
}

__global__ __launch_bounds__(kEmitThreads, NDX_EMIT_MINB) void k_emit(const uint64_t* __restrict__ pairs,
                                                          uint64_t n, Ctl* ctl,
                                                          uint32_t* __restrict__ words,
                                                          uint32_t* __restrict__ vstart,
                                                          uint32_t* __restrict__ values,
                                                          uint64_t* agg, int bulk_ok) {
  if (ctl->rows_form) return;  // k_emit_rows
  extern __shared__ __align__(16) unsigned char emit_smem[];
  uint64_t* buf0 = reinterpret_cast<uint64_t*>(emit_smem);
  uint32_t* stage = reinterpret_cast<uint32_t*>(buf0 + 2 * kEmitBuf);
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t s_wt[2][kEmitWarps];
  __shared__ uint32_t s_wx[2][kEmitWarps];    // exclusive prefix of s_wt over the warps
  __shared__ uint32_t s_tot[2];               // the tile's (words << 16 | value heads)
  __shared__ uint32_t s_accw[2], s_accd[2];   // aggregates below the pending tile: words, heads
  __shared__ uint32_t s_tile[2];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ntiles = uint32_t((n + kEmitTile - 1) / kEmitTile);
  const uint32_t n32 = uint32_t(n);  // n < 2^31 (checked by the launcher)
  const bool small_rows = ctl->row_hi < kDiv31FastLimit;
  uint32_t* ctr = &ctl->tile_ctr[0];

  auto by_bulk = [&](uint32_t t) -> bool {
    return bulk_ok && t > 0 && uint64_t(t + 1) * kEmitTile + kHaloR <= n;
  };
  auto bulk_fill = [&](uint32_t t, int b) {  // one thread
    fence_proxy_async_smem();
    mbar_expect_tx(&bar[b], kEmitBuf * 8);
    bulk_g2s(buf0 + b * kEmitBuf, pairs + (int64_t(t) * kEmitTile - kHaloL), kEmitBuf * 8, &bar[b]);
  };
  auto manual_fill = [&](uint32_t t, int b) {  // all threads
    uint64_t* dst = buf0 + b * kEmitBuf;
    const int64_t g0 = int64_t(t) * kEmitTile - kHaloL;
    for (int j = threadIdx.x; j < kEmitBuf; j += kEmitThreads) {
      const int64_t g = g0 + j;
      dst[j] = (g >= 0 && uint64_t(g) < n) ? __ldg(pairs + g) : 0ull;
    }
  };

  if (threadIdx.x == 0) {
    s_accw[0] = s_accw[1] = s_accd[0] = s_accd[1] = 0;
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    const uint32_t t = atomicAdd(ctr, 1u);
    s_tile[0] = t;
    if (t < ntiles && by_bulk(t)) bulk_fill(t, 0);
  }
  __syncthreads();

  uint64_t prev_w = 0, prev_d = 0;  // exclusive offsets of this CTA's last written tile
  int64_t prev_tile = -1;
  int64_t pending = -1;             // counted, not yet written
  uint32_t phase = 0;
  Span sp;
  uint32_t carry_in = 0, excl = 0;
  for (int it = 0;; ++it) {
    const int b = it & 1;
    const uint32_t tile = s_tile[b];
    const bool has = tile < ntiles;
    if (!has && pending < 0) break;
    const bool full = has && by_bulk(tile);
    const uint64_t* B = buf0 + b * kEmitBuf + kHaloL;  // B[li] = pairs[tile * kEmitTile + li]
    const uint32_t ts = tile * kEmitTile, li0 = threadIdx.x * kEmitK;
    // Start the reads of the aggregates the previous tile's write-out needs
    // now, so their latency hides behind phase 1 (most are published by now;
    // the few that are not get re-read after phase 1).
    constexpr int kAggPre = 4;
    uint64_t pre[kAggPre];
    const uint64_t agg_lo = prev_tile < 0 ? 0 : uint64_t(prev_tile);
    const uint64_t agg_hi = pending < 0 ? agg_lo : uint64_t(pending);
    agg_request(agg, agg_lo, agg_hi, pre);
    if (has) {
      if (full) {
        mbar_wait(&bar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
      } else {
        manual_fill(tile, b);
        __syncthreads();
      }
      // ---- phase 1: counts and carries
      uint32_t wcarry;
      if (small_rows) {
        tile_phase1<true>(full, B, pairs, n32, ts, li0, sp);
        wcarry = warp_carry<true>(B, ts, uint32_t(warp) * 32 * kEmitK);
      } else {
        tile_phase1<false>(full, B, pairs, n32, ts, li0, sp);
        wcarry = warp_carry<false>(B, ts, uint32_t(warp) * 32 * kEmitK);
      }
      const uint32_t incl = span_scans(sp, wcarry, carry_in, excl);
      if (lane == 31) s_wt[b][warp] = incl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (has) {
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kEmitWarps; ++w) {
          s_wx[b][w] = tot;
          tot += s_wt[b][w];
        }
        s_tot[b] = tot;
        st_relaxed_u64(&agg[tile], kAggReady | uint64_t(tot >> 16) | (uint64_t(tot & 0xffffu) << 32));
      }
      // take the next tile; its bulk copy overlaps the rest of this one
      const uint32_t nt = has ? atomicAdd(ctr, 1u) : ntiles;
      s_tile[b ^ 1] = nt;
      if (nt < ntiles && by_bulk(nt)) bulk_fill(nt, b ^ 1);
#if NDX_EMIT_L2PF
      // the tile one CTA round ahead into L2 (as in the sort's tile loop)
      const uint64_t pf = uint64_t(nt) + gridDim.x;
      if (nt < ntiles && (pf + 1) * kEmitTile <= n)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pairs + pf * kEmitTile),
                     "r"(uint32_t(kEmitTile * 8)) : "memory");
#endif
    }

    if (pending >= 0) {
      // ---- write the previous tile out: global offsets first
      const int pb = b ^ 1;
      const uint64_t pt = uint64_t(pending);
      uint32_t sw, sd;
      agg_sum(agg, agg_lo, pt, pre, sw, sd);
      sw = __reduce_add_sync(kFull, sw);
      sd = __reduce_add_sync(kFull, sd);
      if (lane == 0) {
        atomicAdd(&s_accw[pb], sw);
        atomicAdd(&s_accd[pb], sd);
      }
      __syncthreads();
      const uint64_t W0 = prev_w + s_accw[pb], D0 = prev_d + s_accd[pb];
      const uint32_t tw = s_tot[pb] >> 16, td = s_tot[pb] & 0xffffu;
      prev_w = W0;
      prev_d = D0;
      prev_tile = int64_t(pt);
      if (threadIdx.x == 0 && pt == ntiles - 1) {
        ctl->words = W0 + tw;
        ctl->distinct = D0 + td;
      }
      {
        // from a base pointer: one wide multiply-add per address instead
        // of 64-bit index arithmetic (16-byte funnel-shifted stores measured
        // slower: 1.035 ms against 0.987 ms on C4)
        uint32_t* const wd = words + W0;
#pragma unroll 4
        for (uint32_t j = threadIdx.x; j < tw; j += kEmitThreads) wd[j] = stage[j];
      }
      for (uint32_t j = threadIdx.x; j < td; j += kEmitThreads) {
        values[D0 + j] = stage[2 * kEmitTile + j];
        vstart[D0 + j] = uint32_t(W0 + reinterpret_cast<const uint16_t*>(stage + 3 * kEmitTile)[j]);
      }
    }
    __syncthreads();  // the staging area is free again; s_tile[b^1] visible
    if (threadIdx.x == 0) s_accw[b] = s_accd[b] = 0;  // last read the iteration before; next added to the iteration after

    if (has) {
      // ---- phase 2: this tile's words into the staging area
      const uint32_t wbase = s_wx[b][warp];
      const uint32_t o = (wbase >> 16) + (excl >> 16), h = (wbase & 0xffffu) + (excl & 0xffffu);
      if (small_rows)
        span_emit<true>(sp, B + li0, carry_in, o, h, stage, stage + 2 * kEmitTile,
                        reinterpret_cast<uint16_t*>(stage + 3 * kEmitTile));
      else
        span_emit<false>(sp, B + li0, carry_in, o, h, stage, stage + 2 * kEmitTile,
                         reinterpret_cast<uint16_t*>(stage + 3 * kEmitTile));
    }
    pending = has ? int64_t(tile) : -1;
  }
}

// ---- rows form -----------------------------------------------------------------
// The wide pass and pass B write the sorted stream as row ids only; the
// values are the present keys in order with the stream position where each
// begins (ctl->pk / ctl->vs, k_vs).  The emit then reads 4 bytes per element
// instead of 8, and a tile learns its value heads from a 128-byte record
// (k_tile_heads) that arrives with its rows by the same bulk copy.  A value
// head is the only thing the key contributed (wah_builder.cpp:74-75: v
// differs from the element before); the table's values are pk itself.

constexpr int kRowsHaloR = 4;                              // 16-byte multiple of u32 rows
constexpr int kRowsBuf = kHaloL + kEmitTile + kRowsHaloR;  // rows per tile buffer
constexpr int kRecHeads = 60;
struct __align__(16) TileRec {
  uint32_t ib, ie;          // the value heads inside the buffer: vs[ib .. ie) (ib == ie: none)
  uint16_t hp[kRecHeads];   // buffer positions of the first kRecHeads of them
};
static_assert(sizeof(TileRec) == 128, "one bulk copy per record");
// two row buffers, two records, then the words of one tile and the
// tile-local word offsets of its value heads
constexpr size_t kEmitRowsSmem =
    size_t(2 * kRowsBuf) * 4 + 2 * sizeof(TileRec) + size_t(2 * kEmitTile) * 4 + size_t(kEmitTile) * 2;

// The value heads of one tile buffer (positions relative to the buffer's
// first element, ascending): from the record, or -- a tile with more than
// kRecHeads heads -- from vs itself.
struct Heads {
  const uint16_t* hp;
  const uint32_t* vs;
  uint32_t m, ib;
  int64_t p0;  // stream position of buffer element 0
  __device__ __forceinline__ uint32_t at(uint32_t k) const {
    return m <= uint32_t(kRecHeads) ? uint32_t(hp[k]) : uint32_t(int64_t(__ldg(vs + ib + k)) - p0);
  }
  // heads at buffer positions < q
  __device__ __forceinline__ uint32_t below(uint32_t q) const {
    uint32_t lo = 0, hi = m;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (at(mid) < q)
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  }
};

// Largest t with rows[g+t] == row+t inside the value (g+t < end), given that
// it holds for t = 30 (stretch_end of the pairs form).
__device__ __noinline__ uint32_t stretch_end_r(const uint32_t* __restrict__ rows, uint64_t end, uint64_t g,
                                               uint32_t row) {
  auto P = [&](uint64_t t) -> bool {
    if (g + t >= end) return false;
    const uint64_t rr = uint64_t(row) + t;
    if (rr > 0xffffffffull) return false;
    return __ldg(rows + g + t) == uint32_t(rr);
  };
  uint64_t lo = 30, hi, step = 32;
  for (;;) {
    const uint64_t cand = lo + step;
    if (!P(cand)) {
      hi = cand;
      break;
    }
    lo = cand;
    step <<= 1;
  }
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (P(mid))
      lo = mid;
    else
      hi = mid;
  }
  return uint32_t(lo);
}

// ones_body of the pairs form: the value's extent [vs[i], vs[i+1]) replaces
// the key comparisons.
__device__ __noinline__ uint32_t ones_body_r(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ vs,
                                             uint32_t nvals, uint64_t e, uint32_t row) {
  uint32_t lo = 0, hi = nvals;  // vs[lo] <= e < vs[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(vs + mid) <= e)
      lo = mid;
    else
      hi = mid;
  }
  const uint64_t vb = __ldg(vs + lo), ve = __ldg(vs + lo + 1);
  if (e >= 61 && row >= 61 && e - 61 >= vb && __ldg(rows + e - 61) == row - 61) return 0;
  const uint32_t t = stretch_end_r(rows, ve, e - 30, row - 30);
  return make_fill(true, (t + 1) / kChunkBits);
}

// Phase 1 of the rows form (span_scan): the value-head bits come from the
// tile's head list instead of key comparisons.
template <bool SMALL, bool FULL>
__device__ __forceinline__ void span_scan_r(const uint32_t* R, const Heads& H, const uint32_t* __restrict__ rows,
                                            const uint32_t* __restrict__ vs, uint32_t nvals, uint32_t n,
                                            uint32_t ts, uint32_t li0, Span& s) {
  const uint32_t q0 = kHaloL + li0;
  // 7 x 8 B per thread: a 56-byte stride hits distinct bank pairs
  uint32_t r[kEmitK];
  const uint2* R2 = reinterpret_cast<const uint2*>(R + q0);
#pragma unroll
  for (int p = 0; p < kEmitK / 2; ++p) {
    const uint2 u = R2[p];
    r[2 * p] = u.x;
    r[2 * p + 1] = u.y;
  }
  const uint32_t prv = R[q0 - 1], nxt = R[q0 + kEmitK];
  // value heads at q0 .. q0 + kEmitK (bit kEmitK: the element after the span)
  uint32_t vb = 0;
  if (H.m) {
    for (uint32_t k = H.below(q0); k < H.m; ++k) {
      const uint32_t h = H.at(k);
      if (h > q0 + kEmitK) break;
      vb |= 1u << (h - q0);
    }
  }
  const uint32_t g0 = ts + li0;
  uint32_t pc = div31<SMALL>(prv);
  uint32_t hm = 0, vm = 0, gaps = 0, acc = 0;
  if (FULL && vb == 0) {
    // no value head in the span (nearly every span): runs split at chunks only
#pragma unroll
    for (int j = 0; j < kEmitK; ++j) {
      const uint32_t row = r[j], c = div31<SMALL>(row);
      const uint32_t bp = row - c * kChunkBits;
      const bool h = c != pc;
      const uint32_t gap = h ? c - pc - 1 : 0u;
      gaps += gap != 0;
      s.pk[j] = SMALL ? (gap << 5) | bp : gap;
      hm |= uint32_t(h) << j;
      acc = (h ? 0u : acc) | (1u << bp);
      pc = c;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kEmitK; ++j) {
      const uint32_t row = r[j], c = div31<SMALL>(row);
      const uint32_t bp = row - c * kChunkBits;
      bool vh = (vb >> j) & 1u, h = vh | (c != pc);
      if (!FULL) {
        const uint32_t g = g0 + j;
        const bool valid = g < n;
        vh = valid & (vh | (g == 0));
        h = valid & (h | (g == 0));
      }
      const uint32_t gap = h ? (vh ? c : c - pc - 1) : 0u;
      gaps += gap != 0;
      s.pk[j] = SMALL ? (gap << 5) | bp : gap;
      hm |= uint32_t(h) << j;
      vm |= uint32_t(vh) << j;
      acc = (h ? 0u : acc) | (1u << bp);
      pc = c;
    }
  }
  const bool hN = ((vb >> kEmitK) & 1u) | (div31<SMALL>(nxt) != pc);
  uint32_t tm;
  if (FULL) {
    tm = (hm >> 1) | (uint32_t(hN) << (kEmitK - 1));
  } else {
    const uint32_t nvalid = g0 >= n ? 0u : umin(n - g0, uint32_t(kEmitK + 1));
    const uint32_t valid9 = (1u << nvalid) - 1u;
    const uint32_t h9 = hm | (uint32_t(hN) << kEmitK);
    tm = valid9 & ((1u << kEmitK) - 1u) & ((h9 >> 1) | (~valid9 >> 1));
  }
  s.hmask = hm;
  s.vmask = vm;
  s.tmask = tm;
  s.acc = acc;
  s.nwords = gaps + __popc(tm);
  // first_run_check: the span's first run, begun before the span, all-ones?
  s.first_body = 1;
  if (tm != 0 && (hm == 0 || __ffs(tm) < __ffs(hm))) {
    const uint32_t j = __ffs(tm) - 1, q = q0 + j;
    const uint32_t row = R[q];
    if (row - div31<SMALL>(row) * kChunkBits == kChunkBits - 1 && g0 + j >= 30 && R[q - 30] == row - 30) {
      // same value: no head in [q0, q] (the run has none there), and the
      // last one before the span at or before q - 30
      const uint32_t k = H.below(q0);
      if (k == 0 || H.at(k - 1) <= q - 30) {
        s.first_body = ones_body_r(rows, vs, nvals, g0 + j, row);
        if (s.first_body == 0) s.nwords -= 1;
      }
    }
  }
}

// warp_carry of the rows form: "same value as element wl" is "no value head
// after q up to wl".
template <bool SMALL>
__device__ __forceinline__ uint32_t warp_carry_r(const uint32_t* R, const Heads& H, uint32_t ts, uint32_t wl) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t wq = kHaloL + wl;
  const uint32_t c0 = div31<SMALL>(R[wq]);
  const uint32_t q = wq - 32 + lane;
  const uint32_t qrow = R[q], qc = div31<SMALL>(qrow);
  uint32_t lh = 0;
  if (H.m) {
    const uint32_t k = H.below(wq + 1);
    if (k) lh = H.at(k - 1);
  }
  const bool m = (ts + wl + lane >= 32) & (q >= lh) & (qc == c0);
  return __reduce_or_sync(kFull, m ? 1u << (qrow - qc * kChunkBits) : 0u);
}

// Phase 2 of the rows form (span_emit): only the heads' word offsets are
// staged (the values are pk).
template <bool SMALL>
__device__ __forceinline__ void span_emit_r(const Span& s, const uint32_t* Rs, uint32_t carry, uint32_t o,
                                            uint32_t h, uint32_t* stage, uint16_t* ho) {
  uint32_t sa = smem_addr(stage) + 4u * o;
  uint32_t acc = carry;
  auto bit = [&](int j) -> uint32_t {
    if (SMALL) return 1u << (s.pk[j] & 31u);
    const uint32_t row = Rs[j];
    return 1u << (row - (row / kChunkBits) * kChunkBits);
  };
  if (s.vmask == 0 && s.first_body == 1) {
#pragma unroll
    for (int j = 0; j < kEmitK; ++j) {
      const uint32_t gap = gap_of<SMALL>(s.pk[j]), b = bit(j);
      if (gap) {
        sts_u32(sa, kFillFlag | gap);
        sa += 4;
      }
      acc = ((s.hmask >> j) & 1u) ? b : (acc | b);
      if ((s.tmask >> j) & 1u) {
        sts_u32(sa, acc);
        sa += 4;
      }
    }
    return;
  }
  const uint32_t sbase = smem_addr(stage);
#pragma unroll
  for (int j = 0; j < kEmitK; ++j) {
    const uint32_t gap = gap_of<SMALL>(s.pk[j]), b = bit(j);
    if ((s.vmask >> j) & 1u) {
      ho[h] = uint16_t((sa - sbase) >> 2);
      ++h;
    }
    if (gap) {
      sts_u32(sa, kFillFlag | gap);
      sa += 4;
    }
    acc = ((s.hmask >> j) & 1u) ? b : (acc | b);
    if ((s.tmask >> j) & 1u) {
      const bool first = (s.hmask & ((2u << j) - 1u)) == 0;
      const uint32_t body = (first && s.first_body != 1) ? s.first_body : acc;
      if (body) {
        sts_u32(sa, body);
        sa += 4;
      }
    }
  }
}

// Per emit tile: the aggregate word and the head record's range cleared.
__global__ void k_tile_prep(uint64_t* agg, TileRec* __restrict__ recs, uint32_t ntiles) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
    agg[t] = 0;
    *reinterpret_cast<uint2*>(recs + t) = make_uint2(0, 0);
  }
}

// The head records, from the heads' side: value head i (stream position P)
// lies in the buffers of one or two tiles; for each it writes the record's
// range ends it is (first: ib, last: ie) and its slot among the first
// kRecHeads (the heads of the buffer before it, counted backwards).  The
// table's values are the present keys (pk) in order.
constexpr int kHeadsThreads = 1024;
__global__ __launch_bounds__(kHeadsThreads) void k_tile_heads(const Ctl* __restrict__ ctl,
                                                              TileRec* __restrict__ recs, uint32_t ntiles,
                                                              uint32_t* __restrict__ values) {
  if (!ctl->rows_form) return;
  const uint32_t nv = ctl->nvals;
  const uint32_t i = blockIdx.x * kHeadsThreads + threadIdx.x;
  if (i >= nv) return;
  const uint32_t* vs = ctl->vs;
  values[i] = ctl->pk[i];
  const int64_t P = vs[i];
  const int64_t prv = i ? int64_t(vs[i - 1]) : -1;
  const int64_t nxt = i + 1 < nv ? int64_t(vs[i + 1]) : INT64_MAX;
  const uint32_t th = uint32_t((P + kHaloL) / kEmitTile);  // the last tile whose buffer starts at or before P
  for (uint32_t t = th > 0 ? th - 1 : 0; t <= th && t < ntiles; ++t) {
    const int64_t p0 = int64_t(t) * kEmitTile - kHaloL;
    if (P < p0 || P >= p0 + kRowsBuf) continue;
    TileRec* r = recs + t;
    if (prv < p0) r->ib = i;
    if (nxt >= p0 + kRowsBuf) r->ie = i + 1;
    uint32_t k = 0;
    for (uint32_t j = i; k < uint32_t(kRecHeads) && j > 0 && int64_t(vs[j - 1]) >= p0; --j) ++k;
    if (k < uint32_t(kRecHeads)) r->hp[k] = uint16_t(P - p0);
  }
}

// S3 over the rows form: k_emit's tile schedule, aggregates and write-out
// (see there); three CTAs per SM fit beside the half-size buffers.
__global__ __launch_bounds__(kEmitThreads, NDX_EMIT_ROWS_MINB) void k_emit_rows(const uint32_t* __restrict__ rows, uint64_t n,
                                                               Ctl* ctl, uint32_t* __restrict__ words,
                                                               uint32_t* __restrict__ vstart,
                                                               const TileRec* __restrict__ recs, uint64_t* agg,
                                                               int bulk_ok) {
  if (!ctl->rows_form) return;
  extern __shared__ __align__(16) unsigned char emit_smem[];
  uint32_t* buf0 = reinterpret_cast<uint32_t*>(emit_smem);
  TileRec* srec = reinterpret_cast<TileRec*>(buf0 + 2 * kRowsBuf);
  uint32_t* stage = reinterpret_cast<uint32_t*>(srec + 2);
  uint16_t* ho = reinterpret_cast<uint16_t*>(stage + 2 * kEmitTile);
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t s_wt[2][kEmitWarps];
  __shared__ uint32_t s_wx[2][kEmitWarps];  // exclusive prefix of s_wt over the warps
  __shared__ uint32_t s_tot[2];             // the tile's (words << 16 | value heads)
  __shared__ uint32_t s_accw[2], s_accd[2];  // aggregates below the pending tile: words, heads
  __shared__ uint32_t s_full[2];             // the tile arrives by bulk copy (thread 0 decides)
  __shared__ uint32_t s_tile[2];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ntiles = uint32_t((n + kEmitTile - 1) / kEmitTile);
  const uint32_t n32 = uint32_t(n);
  const bool small_rows = ctl->row_hi < kDiv31FastLimit;
  const uint32_t* vs = ctl->vs;
  const uint32_t nvals = ctl->nvals;
  uint32_t* ctr = &ctl->tile_ctr[0];

  auto by_bulk = [&](uint32_t t) -> bool {
    return bulk_ok && t > 0 && uint64_t(t + 1) * kEmitTile + kRowsHaloR <= n;
  };
  auto bulk_fill = [&](uint32_t t, int b) {  // one thread
    fence_proxy_async_smem();
    mbar_expect_tx(&bar[b], kRowsBuf * 4 + uint32_t(sizeof(TileRec)));
    bulk_g2s(buf0 + b * kRowsBuf, rows + (int64_t(t) * kEmitTile - kHaloL), kRowsBuf * 4, &bar[b]);
    bulk_g2s(srec + b, recs + t, uint32_t(sizeof(TileRec)), &bar[b]);
  };
  auto manual_fill = [&](uint32_t t, int b) {  // all threads
    uint32_t* dst = buf0 + b * kRowsBuf;
    const int64_t g0 = int64_t(t) * kEmitTile - kHaloL;
    for (int j = threadIdx.x; j < kRowsBuf; j += kEmitThreads) {
      const int64_t g = g0 + j;
      dst[j] = (g >= 0 && uint64_t(g) < n) ? __ldg(rows + g) : 0u;
    }
    if (threadIdx.x < sizeof(TileRec) / 4)
      reinterpret_cast<uint32_t*>(srec + b)[threadIdx.x] = reinterpret_cast<const uint32_t*>(recs + t)[threadIdx.x];
  };

  if (threadIdx.x == 0) {
    s_accw[0] = s_accw[1] = s_accd[0] = s_accd[1] = 0;
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    const uint32_t t = atomicAdd(ctr, 1u);
    s_tile[0] = t;
    s_full[0] = t < ntiles && by_bulk(t);
    if (s_full[0]) bulk_fill(t, 0);
  }
  __syncthreads();

  uint64_t prev_w = 0, prev_d = 0;
  int64_t prev_tile = -1;
  int64_t pending = -1;
  uint32_t phase = 0;
  Span sp;
  uint32_t carry_in = 0, excl = 0;
  for (int it = 0;; ++it) {
    const int b = it & 1;
    const uint32_t tile = s_tile[b];
    const bool has = tile < ntiles;
    if (!has && pending < 0) break;
    const bool full = s_full[b];
    const uint32_t* R = buf0 + b * kRowsBuf;  // R[kHaloL + li] = rows[tile * kEmitTile + li]
    const uint32_t ts = tile * kEmitTile, li0 = threadIdx.x * kEmitK;
    constexpr int kAggPre = NDX_EMIT_AGGPRE;  // aggregates read ahead per thread (about one per CTA in all)
    uint64_t pre[kAggPre];
    const uint64_t agg_lo = prev_tile < 0 ? 0 : uint64_t(prev_tile);
    const uint64_t agg_hi = pending < 0 ? agg_lo : uint64_t(pending);
    agg_request(agg, agg_lo, agg_hi, pre);
    if (has) {
      if (full) {
        mbar_wait(&bar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
      } else {
        manual_fill(tile, b);
        __syncthreads();
      }
      Heads H;
      H.hp = srec[b].hp;
      H.vs = vs;
      H.m = srec[b].ie - srec[b].ib;
      H.ib = srec[b].ib;
      H.p0 = int64_t(ts) - kHaloL;
      // ---- phase 1: counts and carries
      uint32_t wcarry;
      if (small_rows) {
        if (full)
          span_scan_r<true, true>(R, H, rows, vs, nvals, n32, ts, li0, sp);
        else
          span_scan_r<true, false>(R, H, rows, vs, nvals, n32, ts, li0, sp);
        wcarry = warp_carry_r<true>(R, H, ts, uint32_t(warp) * 32 * kEmitK);
      } else {
        if (full)
          span_scan_r<false, true>(R, H, rows, vs, nvals, n32, ts, li0, sp);
        else
          span_scan_r<false, false>(R, H, rows, vs, nvals, n32, ts, li0, sp);
        wcarry = warp_carry_r<false>(R, H, ts, uint32_t(warp) * 32 * kEmitK);
      }
      const uint32_t incl = span_scans(sp, wcarry, carry_in, excl);
      if (lane == 31) s_wt[b][warp] = incl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (has) {
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kEmitWarps; ++w) {
          s_wx[b][w] = tot;
          tot += s_wt[b][w];
        }
        s_tot[b] = tot;
        st_relaxed_u64(&agg[tile], kAggReady | uint64_t(tot >> 16) | (uint64_t(tot & 0xffffu) << 32));
      }
      const uint32_t nt = has ? atomicAdd(ctr, 1u) : ntiles;
      const bool nfull = nt < ntiles && by_bulk(nt);
      s_tile[b ^ 1] = nt;
      s_full[b ^ 1] = nfull;
      if (nfull) bulk_fill(nt, b ^ 1);
    }

    if (pending >= 0) {
      const int pb = b ^ 1;
      const uint64_t pt = uint64_t(pending);
      uint32_t sw, sd;
      agg_sum(agg, agg_lo, pt, pre, sw, sd);
      sw = __reduce_add_sync(kFull, sw);
      sd = __reduce_add_sync(kFull, sd);
      if (lane == 0) {
        atomicAdd(&s_accw[pb], sw);
        atomicAdd(&s_accd[pb], sd);
      }
      __syncthreads();
      const uint64_t W0 = prev_w + s_accw[pb], D0 = prev_d + s_accd[pb];
      const uint32_t tw = s_tot[pb] >> 16, td = s_tot[pb] & 0xffffu;
      prev_w = W0;
      prev_d = D0;
      prev_tile = int64_t(pt);
      if (threadIdx.x == 0 && pt == ntiles - 1) {
        ctl->words = W0 + tw;
        ctl->distinct = D0 + td;
      }
      {
        uint32_t* const wd = words + W0;
#pragma unroll 4
        for (uint32_t j = threadIdx.x; j < tw; j += kEmitThreads) wd[j] = stage[j];
      }
      for (uint32_t j = threadIdx.x; j < td; j += kEmitThreads) vstart[D0 + j] = uint32_t(W0 + ho[j]);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_accw[b] = s_accd[b] = 0;  // last read the iteration before; next added to the iteration after

    if (has) {
      const uint32_t wbase = s_wx[b][warp];
      const uint32_t o = (wbase >> 16) + (excl >> 16), h = (wbase & 0xffffu) + (excl & 0xffffu);
      const uint32_t* Rs = R + kHaloL + li0;
      if (small_rows)
        span_emit_r<true>(sp, Rs, carry_in, o, h, stage, ho);
      else
        span_emit_r<false>(sp, Rs, carry_in, o, h, stage, ho);
    }
    pending = has ? int64_t(tile) : -1;
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

// scratch: the tiles' aggregate words, then (128-byte aligned) their head records
static size_t rec_offset(uint64_t n) { return (size_t(emit_tiles(n) + 1) * 8 + 127) & ~size_t(127); }

size_t ndx_wah_emit_scratch_bytes(uint64_t n) {
  return rec_offset(n) + size_t(emit_tiles(n)) * sizeof(TileRec) + 256;
}

int ndx_wah_emit(const uint64_t* d_pairs, uint64_t n, void* d_ctl, uint32_t* d_words,
                 uint32_t* d_vstart, uint32_t* d_values, void* d_scratch, void* stream) {
  if (!d_pairs || !d_ctl || !d_words || !d_vstart || !d_values || !d_scratch || n == 0)
    return NDX_E_INVALID;
  if (n >= (1ull << 31)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  // per-device launch shapes, computed once per device (thread-safe)
  static int grid_for[64], grid_rows_for[64], rc_for[64];
  static std::once_flag once[64];
  std::call_once(once[dev & 63], [dev] {
    int& rc = rc_for[dev & 63];
    if ((rc = cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kEmitSmem)))) return;
    if ((rc = cudaFuncSetAttribute(k_emit_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(kEmitRowsSmem))))
      return;
    int sms = 0, occ = 0, occ_rows = 0;
    if ((rc = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev))) return;
    if ((rc = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_emit, kEmitThreads, kEmitSmem))) return;
    if ((rc = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_rows, k_emit_rows, kEmitThreads, kEmitRowsSmem)))
      return;
    grid_for[dev & 63] = sms * (occ > 0 ? occ : 1);
    grid_rows_for[dev & 63] = sms * (occ_rows > 0 ? occ_rows : 1);
  });
  if (rc_for[dev & 63]) return rc_for[dev & 63];
  const uint64_t tiles = emit_tiles(n);
  uint64_t* agg = static_cast<uint64_t*>(d_scratch);
  TileRec* recs = reinterpret_cast<TileRec*>(static_cast<char*>(d_scratch) + rec_offset(n));
  Ctl* ctl = static_cast<Ctl*>(d_ctl);
  k_tile_prep<<<unsigned(umin<uint64_t>((tiles + 255) / 256, 1184)), 256, 0, s>>>(agg, recs, uint32_t(tiles));
  k_tile_heads<<<unsigned(kMaxRowsValues / kHeadsThreads), kHeadsThreads, 0, s>>>(ctl, recs, uint32_t(tiles),
                                                                                  d_values);
  if ((e = cudaGetLastError())) return e;
  int bulk_ok = (reinterpret_cast<uintptr_t>(d_pairs) & 15) == 0;
  // the sorted stream's form is known on the device only: both emit kernels
  // are launched, the one that does not apply returns at once
  {
    const uint32_t* rows = reinterpret_cast<const uint32_t*>(d_pairs);
    int grid = int(umin<uint64_t>(tiles, uint64_t(grid_rows_for[dev & 63])));
    void* args[] = {(void*)&rows,     (void*)&n,    (void*)&ctl, (void*)&d_words,
                    (void*)&d_vstart, (void*)&recs, (void*)&agg, (void*)&bulk_ok};
    if ((e = cudaLaunchCooperativeKernel((const void*)k_emit_rows, dim3(grid), dim3(kEmitThreads), args,
                                         kEmitRowsSmem, s)))
      return e;
  }
  int grid = int(umin<uint64_t>(tiles, uint64_t(grid_for[dev & 63])));
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

// ---------------------------------------------------------------------------
// Result copy-out without a host round trip for the sizes: one kernel reads
// W and D from ctl and writes the counts, the words and the table straight
// into pinned (device-accessible) host memory over PCIe.

namespace ndx {

__global__ void k_copy_out(const Ctl* __restrict__ ctl, const uint32_t* __restrict__ words,
                           const uint32_t* __restrict__ entries, ndx_wah_counts* h_counts,
                           uint32_t* h_words, uint64_t words_cap, uint32_t* h_entries,
                           uint64_t entries_cap) {
  const uint64_t W = ctl->words, D = ctl->distinct;
  const uint64_t nw = umin(W, words_cap), ne = umin(3 * D, entries_cap);
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(h_words) & 15) == 0) {
    const uint64_t n4 = nw / 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(words);
    uint4* d4 = reinterpret_cast<uint4*>(h_words);
    for (uint64_t i = tid; i < n4; i += stride) d4[i] = ldg_stream4(s4 + i);
    for (uint64_t i = 4 * n4 + tid; i < nw; i += stride) h_words[i] = words[i];
  } else {
    for (uint64_t i = tid; i < nw; i += stride) h_words[i] = words[i];
  }
  for (uint64_t i = tid; i < ne; i += stride) h_entries[i] = entries[i];
  if (tid == 0) {
    ndx_wah_counts c;
    c.words = W;
    c.distinct = D;
    c.min_key = ctl->min_key;
    c.max_key = ctl->max_key;
    *h_counts = c;
  }
}

}  // namespace ndx

extern "C" int ndx_wah_copy_out(const void* d_ctl, const uint32_t* d_words,
                                const uint32_t* d_entries, ndx_wah_counts* h_counts,
                                uint32_t* h_words, uint64_t words_cap, uint32_t* h_entries,
                                uint64_t entries_cap, void* stream) {
  if (!d_ctl || !d_words || !d_entries || !h_counts || (!h_words && words_cap) ||
      (!h_entries && entries_cap))
    return NDX_E_INVALID;
  int sms = 0;
  int rc = ndx::sm_count(&sms);
  if (rc) return rc;
  ndx::k_copy_out<<<sms * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const ndx::Ctl*>(d_ctl), d_words, d_entries, h_counts, h_words, words_cap,
      h_entries, entries_cap);
  return cudaGetLastError();
}
