// Stages S1 (plan) and S2 (sort) of the WAH build on sm_100a.
//
// Replaces the reference's row_iota + sort_pairs (p/core/src/wah_builder.cpp:54-63,
// p/core/src/wah_radix.cpp:16-127) and the histogram scans it runs
// (wah_scan.cpp:14-95).  Design:
//
//   S1  k_hist    one streaming read of the keys: key range (min/max) and the
//                 digit histograms (bytes 0,1 and the low 11 bits) in smem,
//                 flushed with one global atomic per bin per CTA.
//       k_plan    picks the pass structure without a host round trip:
//                   range < 2048   -> ONE stable pass on digit = key - min
//                   otherwise      -> byte-wise LSD passes over the bytes
//                                     that vary (constant bytes skipped)
//                 and turns the histograms into bucket start offsets.
//   S2  k_pass<BITS>  persistent onesweep-style stable scatter: tiles are
//                 taken in global order from an atomic counter, the tile's
//                 digit histogram is published before the ranking ("early
//                 counts"), warp ballot-match ranking (lane order == row
//                 order, so it is stable), a decoupled look-back per digit,
//                 smem staging in digit order and a coalesced scatter of
//                 runs.  Consecutive tiles in flight write adjacent parts of
//                 every digit bucket, so partial sectors merge in L2.
//                 The first pass synthesises row ids (no iota buffer).
//   Every kernel is launched unconditionally and exits at once when the plan
//   does not need it (no host synchronisation anywhere).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../../include/ndx.h"
#include "common.cuh"
#include "wah_internal.cuh"

namespace ndx {

// Tile shape of the scatter passes (measured on B200, tools/var_run.sh):
// bigger tiles amortise the per-tile look-back over more pairs, so the
// byte passes run 256 threads x 32 pairs (8192-pair tiles, 2 CTAs/SM) and
// the wide pass -- whose look-back covers up to 2048 digits per tile --
// 512 threads x 32 pairs (16384-pair tiles, 1 CTA/SM).
#ifndef NDX_SORT_THREADS_B
#define NDX_SORT_THREADS_B 256
#endif
#ifndef NDX_SORT_IPT_B
#define NDX_SORT_IPT_B 32
#endif
#ifndef NDX_SORT_MINB_B
#define NDX_SORT_MINB_B 2
#endif
#ifndef NDX_SORT_THREADS_W
#define NDX_SORT_THREADS_W 512
#endif
#ifndef NDX_SORT_IPT_W
#define NDX_SORT_IPT_W 32
#endif
#ifndef NDX_SORT_MINB_W
#define NDX_SORT_MINB_W 1
#endif
#ifndef NDX_SORT_LATE_COUNT
#define NDX_SORT_LATE_COUNT 1
#endif
// narrow-key register packing: measured to help the wide pass (C3 558 ->
// 546 us) and to hurt the byte passes (C4 3.05 -> 3.14 ms)
#ifndef NDX_SORT_NARROW_W
#define NDX_SORT_NARROW_W 1
#endif
#ifndef NDX_SORT_NARROW_B
#define NDX_SORT_NARROW_B 0
#endif
// issue the first look-back read before the staging: measured -1% on the
// byte passes, +2% on the wide pass (more spills there)
#ifndef NDX_SORT_EARLY_LB_B
#define NDX_SORT_EARLY_LB_B 1
#endif
#ifndef NDX_SORT_EARLY_LB_W
#define NDX_SORT_EARLY_LB_W 0
#endif
#ifndef NDX_SORT_ATOMRANK
#define NDX_SORT_ATOMRANK 0
#endif
// wide keys: two ranks (< 2^16) per register, 16 fewer live registers
#ifndef NDX_SORT_L2PF
#define NDX_SORT_L2PF 2  // >0: prefetch the tile NDX_SORT_L2PF/2 CTA rounds ahead into L2
                         // (C4 sort 2.755 -> 2.681 ms, C3 534 -> 515 us; 2 rounds: 2.707 ms)
#endif
#ifndef NDX_SORT_RANK_BCAST
#define NDX_SORT_RANK_BCAST 2  // 0 never, 1 every pass, 2 the wide pass only
#endif
#ifndef NDX_SORT_PACK_RANK
#define NDX_SORT_PACK_RANK 1
#endif
#ifndef NDX_SORT_MATCH_TREE
#define NDX_SORT_MATCH_TREE 0
#endif
// V = 1: the first byte pass (keys in, row ids synthesised) as its own
// kernel -- with narrow keys its ranking needs no row registers, so it can
// run more CTAs per SM than the later passes.
#ifndef NDX_SORT_PROF
#define NDX_SORT_PROF 0
#endif
#ifndef NDX_SORT_SPLIT_FIRST
#define NDX_SORT_SPLIT_FIRST 0
#endif
#ifndef NDX_SORT_MINB_F
#define NDX_SORT_MINB_F 3
#endif
#ifndef NDX_SORT_NARROW_F
#define NDX_SORT_NARROW_F 1
#endif
template <int MAXB, int V = 0>
struct Shape {
  static constexpr bool kWide = MAXB > 8;
  static constexpr bool kFirst = V == 1;
  static constexpr int THREADS = kWide ? NDX_SORT_THREADS_W : NDX_SORT_THREADS_B;
  static constexpr int IPT = kWide ? NDX_SORT_IPT_W : NDX_SORT_IPT_B;  // pairs per thread
  static constexpr int MINB = kWide ? NDX_SORT_MINB_W : (kFirst ? NDX_SORT_MINB_F : NDX_SORT_MINB_B);
  static constexpr bool kNarrowOk = kWide ? NDX_SORT_NARROW_W : (kFirst ? NDX_SORT_NARROW_F : NDX_SORT_NARROW_B);
  static constexpr int WARPS = THREADS / 32;
  static constexpr int WARP_ITEMS = 32 * IPT;
  static constexpr int TILE = THREADS * IPT;
};

// ------------------------------------------------------------------ S1 ----

constexpr int kHistThreads = 512;

// Key range, low-11-bit histogram and byte-1 histogram in one read of the
// keys.  The byte-0 histogram is the low-11 one folded (2 shared atomics per
// key, not 3), and every group of four warps counts into its own copy so a
// skewed column's hot bins are not one shared-memory hot spot.
constexpr int kHistCopies = 4;
#ifndef NDX_HIST_PIPE
#define NDX_HIST_PIPE 1
#endif
#ifndef NDX_HIST_MINB
#define NDX_HIST_MINB 1
#endif
__global__ __launch_bounds__(kHistThreads, NDX_HIST_MINB) void k_hist(const uint32_t* __restrict__ keys,
                                                       uint64_t n, Ctl* ctl) {
  __shared__ uint32_t hws[kHistCopies][kWideBuckets], h1s[kHistCopies][256];
  for (int i = threadIdx.x; i < kHistCopies * kWideBuckets; i += blockDim.x) (&hws[0][0])[i] = 0;
  for (int i = threadIdx.x; i < kHistCopies * 256; i += blockDim.x) (&h1s[0][0])[i] = 0;
  __syncthreads();
  const int copy = (threadIdx.x >> 5) & (kHistCopies - 1);
  uint32_t* hw = hws[copy];
  uint32_t* h1 = h1s[copy];
  uint32_t mx = 0, mxn = 0;
  auto one = [&](uint32_t k) {
    mx = max(mx, k);
    mxn = max(mxn, ~k);
    atomicAdd(&hw[k & (kWideBuckets - 1)], 1u);
    atomicAdd(&h1[(k >> 8) & 255u], 1u);
  };
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(keys) & 15u) == 0) {
    const uint4* q = reinterpret_cast<const uint4*>(keys);
    const uint64_t nq = n / 4;
    uint64_t i = tid;
#if NDX_HIST_PIPE
    // 4 loads in flight, and the next 4 issued before this batch's atomics
    if (i + 3 * stride < nq) {
      uint4 v0 = ldg_stream4(q + i), v1 = ldg_stream4(q + i + stride);
      uint4 v2 = ldg_stream4(q + i + 2 * stride), v3 = ldg_stream4(q + i + 3 * stride);
      for (;;) {
        const uint64_t nx = i + 4 * stride;
        const bool more = nx + 3 * stride < nq;
        uint4 w0 = v0, w1 = v1, w2 = v2, w3 = v3;
        if (more) {
          w0 = ldg_stream4(q + nx);
          w1 = ldg_stream4(q + nx + stride);
          w2 = ldg_stream4(q + nx + 2 * stride);
          w3 = ldg_stream4(q + nx + 3 * stride);
        }
        one(v0.x); one(v0.y); one(v0.z); one(v0.w);
        one(v1.x); one(v1.y); one(v1.z); one(v1.w);
        one(v2.x); one(v2.y); one(v2.z); one(v2.w);
        one(v3.x); one(v3.y); one(v3.z); one(v3.w);
        i = nx;
        if (!more) break;
        v0 = w0; v1 = w1; v2 = w2; v3 = w3;
      }
    }
#else
    for (; i + 3 * stride < nq; i += 4 * stride) {  // 4 loads in flight
      const uint4 v0 = ldg_stream4(q + i), v1 = ldg_stream4(q + i + stride);
      const uint4 v2 = ldg_stream4(q + i + 2 * stride), v3 = ldg_stream4(q + i + 3 * stride);
      one(v0.x); one(v0.y); one(v0.z); one(v0.w);
      one(v1.x); one(v1.y); one(v1.z); one(v1.w);
      one(v2.x); one(v2.y); one(v2.z); one(v2.w);
      one(v3.x); one(v3.y); one(v3.z); one(v3.w);
    }
#endif
    for (; i < nq; i += stride) {
      const uint4 v = ldg_stream4(q + i);
      one(v.x); one(v.y); one(v.z); one(v.w);
    }
    for (uint64_t j = nq * 4 + tid; j < n; j += stride) one(keys[j]);
  } else {
    for (uint64_t j = tid; j < n; j += stride) one(keys[j]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    mxn = max(mxn, __shfl_xor_sync(kFull, mxn, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&ctl->max_seen, mx);
    atomicMax(&ctl->max_not, mxn);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kWideBuckets; i += blockDim.x) {
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < kHistCopies; ++k) c += hws[k][i];
    hws[0][i] = c;
    if (c) atomicAdd(&ctl->hist_wide[i], c);
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < kHistCopies; ++k) c += h1s[k][i];
    if (c) atomicAdd(&ctl->hist_byte[1][i], c);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < kWideBuckets / 256; ++j) c += hws[0][i + 256 * j];
    if (c) atomicAdd(&ctl->hist_byte[0][i], c);
  }
}

// Histograms of bytes 2 and 3, only when the plan found them varying.
__global__ __launch_bounds__(kHistThreads) void k_hist_hi(const uint32_t* __restrict__ keys,
                                                          uint64_t n, Ctl* ctl) {
  if (!ctl->plan.need_hi) return;
  __shared__ uint32_t h2[256], h3[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h2[i] = h3[i] = 0;
  __syncthreads();
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = tid; i < n; i += stride) {
    uint32_t k = ldg_stream(keys + i);
    atomicAdd(&h2[(k >> 16) & 255u], 1u);
    atomicAdd(&h3[k >> 24], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    if (h2[i]) atomicAdd(&ctl->hist_byte[2][i], h2[i]);
    if (h3[i]) atomicAdd(&ctl->hist_byte[3][i], h3[i]);
  }
}

// Exclusive scan of cnt[0..len) into out[], one CTA (len <= 2048).
__device__ void block_excl_scan(const uint32_t* cnt, uint32_t* out, int len) {
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

__device__ void plan_bytes(Ctl* ctl, uint64_t n, int nbytes) {
  SortPlan& p = ctl->plan;
  __shared__ uint32_t s_active[4];
  if (threadIdx.x == 0) {
    uint32_t mn = ctl->min_key;
    uint32_t order = 0;
    for (int k = 0; k < 4; ++k) {
      bool act = k < nbytes && uint64_t(ctl->hist_byte[k][(mn >> (8 * k)) & 255u]) != n;
      p.byte_active[k] = act;
      p.byte_order[k] = act ? order : 0;
      s_active[k] = act;
      if (act) ++order;
    }
    p.npasses = order;
    p.mode = kModeBytes;
    p.complete = 1;
  }
  __syncthreads();
  for (int k = 0; k < 4; ++k)
    if (s_active[k]) block_excl_scan(ctl->hist_byte[k], p.bucket_start_byte[k], 256);
}

// Status buffer: [256 B header: u32 epoch counter, u32 pad, u64 high-water
// mark][statuses of the pass with the most: wide tiles x 2048 digits or byte
// tiles x 256 digits]
__host__ __device__ inline uint64_t status_bytes(uint64_t n) {
  const uint64_t tw = (n + Shape<kWideMaxBits>::TILE - 1) / Shape<kWideMaxBits>::TILE;
  const uint64_t tb = (n + Shape<8>::TILE - 1) / Shape<8>::TILE;
  const uint64_t w = tw * kWideBuckets, b = tb * 256;
  return 256 + (w > b ? w : b) * sizeof(uint64_t);
}
constexpr uint32_t kEpochStep = 8, kEpochMax = 0xfffff8u;  // 24-bit tags, 8 per build

// stage 0: after k_hist; stage 1: after k_hist_hi (no-op unless pending).
// `epoch_counter` lives in the status buffer's header; every build takes a
// fresh tag so statuses of earlier builds never read as ready.
__global__ __launch_bounds__(1024) void k_plan(Ctl* ctl, uint64_t n, int stage,
                                               uint32_t* epoch_counter) {
  SortPlan& p = ctl->plan;
  if (stage == 1) {
    if (p.complete) return;
    plan_bytes(ctl, n, 4);
    return;
  }
  __shared__ uint32_t s_mode, s_wrap;
  __shared__ uint32_t rot[kWideBuckets];
  const uint32_t mn = ~ctl->max_not, mx = ctl->max_seen;
  // The tags are 24 bits: after 2^21 builds they come round again, and a
  // status left by a build one cycle ago (at tiles no build since has
  // reached) would read as ready.  So on the wrap every status ever written
  // -- below the high-water mark kept in the header -- is cleared first.
  uint64_t* hwm = reinterpret_cast<uint64_t*>(epoch_counter) + 1;
  if (threadIdx.x == 0) {
    *hwm = umax(*hwm, status_bytes(n));
    const uint32_t old = *epoch_counter;
    s_wrap = old >= kEpochMax;
    const uint32_t ep = old >= kEpochMax ? kEpochStep : old + kEpochStep;
    *epoch_counter = ep;
    ctl->epoch = ep;
    ctl->min_key = mn;
    ctl->max_key = mx;
    ctl->n_lo = uint32_t(n);
    ctl->n_hi = uint32_t(n >> 32);
    const uint32_t range = mx - mn;
    if (range < uint32_t(kWideBuckets)) {
      p.mode = kModeWide;
      p.base = mn;
      p.wide_bits = range == 0 ? 0 : 32 - __clz(range);
      p.npasses = 1;
      p.complete = 1;
      p.need_hi = 0;
      for (int k = 0; k < 4; ++k) p.byte_active[k] = 0;
    } else {
      p.mode = kModeBytes;
      p.need_hi = (mn >> 16) != (mx >> 16);
      p.complete = !p.need_hi;
    }
    s_mode = p.mode;
  }
  __syncthreads();
  if (s_wrap) {  // once per 2^21 builds: every status ever written, cleared
    uint4* q = reinterpret_cast<uint4*>(reinterpret_cast<char*>(epoch_counter) + 256);
    const uint64_t nq = (*hwm - 256) / sizeof(uint4);
    for (uint64_t i = threadIdx.x; i < nq; i += blockDim.x) q[i] = make_uint4(0, 0, 0, 0);
  }
  if (s_mode == kModeWide) {
    const uint32_t nb = 1u << p.wide_bits;
    for (uint32_t d = threadIdx.x; d < uint32_t(kWideBuckets); d += blockDim.x)
      rot[d] = d < nb ? ctl->hist_wide[(d + mn) & (kWideBuckets - 1)] : 0;
    __syncthreads();
    block_excl_scan(rot, p.bucket_start_wide, kWideBuckets);
  } else if (!p.need_hi) {
    plan_bytes(ctl, n, 2);
  }
}

// ------------------------------------------------------------------ S2 ----

// Look-back status word: [63:40] epoch | [39:38] flag | [37:0] count.
constexpr uint64_t kStAgg = 1ull << 38;
constexpr uint64_t kStPrefix = 2ull << 38;
constexpr uint64_t kStValue = (1ull << 38) - 1;

__device__ __forceinline__ uint64_t st_word(uint32_t epoch, uint64_t flag, uint64_t v) {
  return (uint64_t(epoch & 0xffffffu) << 40) | flag | v;
}
__device__ __forceinline__ bool st_ready(uint64_t s, uint32_t epoch) {
  return uint32_t(s >> 40) == (epoch & 0xffffffu) && (s & (3ull << 38)) != 0;
}

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
  uint64_t* status;             // look-back statuses, tiles x 2048 words (own buffer)
};

struct PassInfo {
  uint32_t shift, bits, base, epoch;
  int p, P;
  const uint32_t* bstart;
};

// The digit of pass `which` (-1 = wide); false if the pass does not run.
__device__ __forceinline__ bool pass_info(const SortArgs& a, int which, PassInfo& pi) {
  const SortPlan& pl = a.ctl->plan;
  if (which < 0) {
    if (pl.mode != kModeWide) return false;
    pi.p = 0;
    pi.P = 1;
    pi.shift = 0;
    pi.bits = pl.wide_bits;
    pi.base = pl.base;
    pi.bstart = pl.bucket_start_wide;
  } else {
    if (pl.mode != kModeBytes || !pl.byte_active[which]) return false;
    pi.p = pl.byte_order[which];
    pi.P = pl.npasses;
    pi.shift = 8u * which;
    pi.bits = 8;
    pi.base = 0;
    pi.bstart = pl.bucket_start_byte[which];
  }
  pi.epoch = a.ctl->epoch + uint32_t(which + 2);
  return true;
}

template <int MAXB>
struct SortSmem {
  static constexpr int NB = 1 << MAXB;
  using SH = Shape<MAXB>;
  static constexpr size_t kHBytes = size_t(SH::WARPS) * NB * sizeof(uint16_t);
  static constexpr size_t kSBytes = size_t(SH::TILE) * sizeof(uint64_t);
  static constexpr size_t kUnion = kHBytes > kSBytes ? kHBytes : kSBytes;
  static constexpr size_t kBytes = kUnion + 2 * NB * sizeof(uint32_t) + 16;
};

// Lanes of the warp whose `BITS`-wide digit equals mine: per bit one
// ballot and one select of it or its complement, then a 3-input AND tree
// (depth 2-3 instead of a chain of BITS dependent ANDs).
template <int BITS>
__device__ __forceinline__ unsigned warp_match(uint32_t d) {
#if NDX_SORT_MATCH_TREE
  unsigned e[BITS];
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool p = (d >> b) & 1u;
    const unsigned v = __ballot_sync(kFull, p);
    e[b] = p ? v : ~v;
  }
  unsigned acc[(BITS + 2) / 3];
#pragma unroll
  for (int i = 0; i < (BITS + 2) / 3; ++i) {
    unsigned x = e[3 * i];
    if (3 * i + 1 < BITS) x &= e[3 * i + 1];
    if (3 * i + 2 < BITS) x &= e[3 * i + 2];
    acc[i] = x;
  }
  unsigned peers = acc[0];
#pragma unroll
  for (int i = 1; i < (BITS + 2) / 3; ++i) peers &= acc[i];
  return peers;
#else
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
#endif
}

struct TileCtx {
  const uint32_t* in_keys;   // first pass (SoA) ...
  const uint32_t* in_pays;   // ... payloads or null (row ids synthesised)
  const uint64_t* in_pairs;  // later passes (AoS)
  uint64_t* out_pairs;
  uint32_t* out_keys;        // SoA output of the last pass (sort_pairs API)
  uint32_t* out_pays;
  uint32_t shift, base, row_base, epoch;
  const uint32_t* bstart;
  uint64_t* status;
  uint16_t* H;               // [warps][NB] per-warp digit counters (aliases S)
  uint64_t* S;               // [tile] staging
  uint32_t* cnt;             // [NB] tile count per digit
  uint32_t* gbase;           // [NB] tile-local start, then global base - local start
  bool narrow;               // every key < 2^16
};

// Exclusive count of digit d over all tiles before `tile` (decoupled
// look-back, kLookbackWidth predecessor statuses in flight at a time: the
// look-back depth grows with the number of tiles in flight, so each step
// covers several predecessors with one round trip).
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

// One tile of a stable scatter pass.  BITS is the digit width (compile
// time, so the ballot match unrolls straight); FULL tiles skip every bounds
// check.  Element order within a warp is round-major / lane-minor, which is
// row order, so ranks taken round by round are stable.
// NARROW: every key is below 2^16 (known from the plan), so a pair's rank
// rides in the upper half of its key register -- 32 fewer live registers in
// the ranking, no spills.
#if NDX_SORT_PROF
// experiment build only: cycles per tile phase, summed over tiles by thread 0
// of each CTA (load, rank, counts+scan, staging, look-back, scatter)
__device__ unsigned long long g_sort_prof[8];
#define PROF_MARK(i)                                                     \
  do {                                                                   \
    if (threadIdx.x == 0) {                                              \
      const long long now_ = clock64();                                  \
      atomicAdd(&g_sort_prof[i], (unsigned long long)(now_ - prof_t_));  \
      prof_t_ = now_;                                                    \
    }                                                                    \
  } while (0)
#else
#define PROF_MARK(i) \
  do {               \
  } while (0)
#endif

template <class SH, int BITS, int NBMAX, bool FULL, bool NARROW>
__device__ __forceinline__ void tile_pass(const TileCtx& t, uint64_t tile, uint32_t tile_n) {
#if NDX_SORT_PROF
  long long prof_t_ = clock64();
  if (threadIdx.x == 0) atomicAdd(&g_sort_prof[7], 1ull);
#endif
  constexpr uint32_t NB = 1u << BITS;
  constexpr uint32_t DMASK = NB - 1;
  auto digit = [&](uint32_t k) -> uint32_t {
    return (((NARROW ? (k & 0xffffu) : k) - t.base) >> t.shift) & DMASK;
  };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t tile_start = tile * SH::TILE;
  uint16_t* Hw = t.H + warp * NBMAX;
  for (uint32_t d = lane; d < NB; d += 32) Hw[d] = 0;
  for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS) t.cnt[d] = 0;

  const uint32_t wofs = uint32_t(warp) * SH::WARP_ITEMS + lane;
  // kFirst (the split-off first byte pass): keys in, row ids synthesised at
  // staging time -- no row registers at all
  constexpr bool kOnlyKeys = SH::kFirst;
  uint32_t key[SH::IPT], pay[kOnlyKeys ? 1 : SH::IPT];
  const uint32_t r0 = t.row_base + uint32_t(tile_start) + wofs;
  auto pay_at = [&](int r) -> uint32_t { return kOnlyKeys ? r0 + uint32_t(r) * 32u : pay[r]; };
  if (!kOnlyKeys && t.in_pairs) {
    const uint64_t* pp = t.in_pairs + tile_start + wofs;
#pragma unroll
    for (int r = 0; r < SH::IPT; ++r) {
      const uint64_t e = (FULL || wofs + r * 32 < tile_n) ? ldg_stream(pp + r * 32) : 0ull;
      key[r] = uint32_t(e);
      pay[r] = uint32_t(e >> 32);
    }
  } else {
    const uint32_t* kp = t.in_keys + tile_start + wofs;
#pragma unroll
    for (int r = 0; r < SH::IPT; ++r)
      key[r] = (FULL || wofs + r * 32 < tile_n) ? ldg_stream(kp + r * 32) : 0u;
    if (!kOnlyKeys) {
      if (t.in_pays) {
        const uint32_t* rp = t.in_pays + tile_start + wofs;
#pragma unroll
        for (int r = 0; r < SH::IPT; ++r)
          pay[r] = (FULL || wofs + r * 32 < tile_n) ? ldg_stream(rp + r * 32) : 0u;
      } else {
#pragma unroll
        for (int r = 0; r < SH::IPT; ++r) pay[r] = r0 + r * 32;
      }
    }
  }
  __syncthreads();
  PROF_MARK(0);

  uint64_t* st = t.status + tile * NB;
#if !NDX_SORT_LATE_COUNT
  // ---- early counts: tile histogram, published before the heavy ranking
#pragma unroll
  for (int r = 0; r < SH::IPT; ++r)
    if (FULL || wofs + r * 32 < tile_n) atomicAdd(&t.cnt[digit(key[r])], 1u);
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS)
    st_relaxed_u64(&st[d], st_word(t.epoch, tile == 0 ? kStPrefix : kStAgg, t.cnt[d]));
#endif

  // ---- rank
  static_assert(SH::TILE <= 65536 && SH::IPT % 2 == 0, "packed ranks need 16-bit tile slots");
  constexpr bool PACK = NDX_SORT_PACK_RANK && !NARROW;
  uint32_t rank[NARROW ? 1 : (PACK ? SH::IPT / 2 : SH::IPT)] = {};
  // rank of round r: in rank[r] or, packed, in half (r & 1) of rank[r / 2]
  auto rank_add = [&](int r, uint32_t v) {
    if (PACK)
      rank[r >> 1] += v << (16 * (r & 1));
    else
      rank[r] += v;
  };
  auto rank_get = [&](int r) -> uint32_t { return PACK ? (rank[r >> 1] >> (16 * (r & 1))) & 0xffffu : rank[r]; };
#pragma unroll
  for (int r = 0; r < SH::IPT; ++r) {
    const uint32_t d = digit(key[r]);
    unsigned peers = warp_match<BITS>(d);
    bool valid = true;
    if (!FULL) {
      valid = wofs + r * 32 < tile_n;
      peers &= __ballot_sync(kFull, valid);
    }
    const int leader = valid ? __ffs(peers) - 1 : lane;
#if NDX_SORT_ATOMRANK
    // one shared atomic per digit group: the counters are u16 pairs packed
    // in u32 words (a warp counts at most 32*IPT < 2^16 per digit), and a
    // warp's atomics to one word apply in program order, so round r+1 sees
    // round r without a load/store chain between rounds
    uint32_t old = 0;
    if (valid && lane == leader) {
      const uint32_t sh = (d & 1u) * 16u;
      old = (atomicAdd(reinterpret_cast<uint32_t*>(Hw) + (d >> 1), uint32_t(__popc(peers)) << sh) >> sh) &
            0xffffu;
    }
    old = __shfl_sync(kFull, old, leader);
    const uint32_t rk = old + __popc(peers & lanemask_lt());
#else
    // wide pass: every lane reads its digit's counter (peers read one
    // address: a broadcast), so no shuffle sits in the round-to-round chain
    // (C3 sort 541 -> 534 us); byte passes keep the leader read + shuffle,
    // which measured faster there (C4 sort 2.755 vs 2.790 ms)
    constexpr bool kBcast = NDX_SORT_RANK_BCAST == 1 || (NDX_SORT_RANK_BCAST == 2 && SH::kWide);
    uint32_t old = 0;
    if constexpr (kBcast) {
      old = Hw[d];
      __syncwarp();
    } else {
      if (lane == leader) old = Hw[d];
      old = __shfl_sync(kFull, old, leader);
    }
    if (valid && lane == leader) Hw[d] = uint16_t(old + __popc(peers));
    const uint32_t rk = old + __popc(peers & lanemask_lt());
    __syncwarp();
#endif
    if (NARROW)
      key[r] |= rk << 16;
    else if (PACK && (r & 1) == 0)
      rank[r >> 1] = rk;
    else if (PACK)
      rank[r >> 1] |= rk << 16;
    else
      rank[r] = rk;
  }
  __syncthreads();
  PROF_MARK(1);

  // ---- per digit: warp offsets (in place); tile-local digit starts
  for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS) {
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < SH::WARPS; ++w) {
      const uint32_t c = t.H[w * NBMAX + d];
      t.H[w * NBMAX + d] = uint16_t(sum);
      sum += c;
    }
#if NDX_SORT_LATE_COUNT
    // the tile's digit counts fall out of the warp counters: published here
    t.cnt[d] = sum;
    st_relaxed_u64(&st[d], st_word(t.epoch, tile == 0 ? kStPrefix : kStAgg, sum));
#endif
  }
#if NDX_SORT_LATE_COUNT
  __syncthreads();  // the scan reads other threads' counts
#endif
  block_excl_scan(t.cnt, t.gbase, int(NB));  // gbase <- tile-local digit starts (syncs)
  PROF_MARK(2);

  if constexpr (SH::kWide ? NDX_SORT_EARLY_LB_W : NDX_SORT_EARLY_LB_B) {
  // ---- look-back, part 1: the first predecessor status of each of this
  // thread's digits is requested now; its round trip overlaps the rank
  // adjustment and the staging, which only need tile-local offsets
  constexpr int ND = int((NB + SH::THREADS - 1) / SH::THREADS);
  uint64_t first[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    const uint32_t d = threadIdx.x + uint32_t(k) * SH::THREADS;
    first[k] = (tile > 0 && d < NB) ? ld_relaxed_u64(&t.status[(tile - 1) * NB + d]) : 0ull;
    if (d < NB) {
      const uint32_t local = t.gbase[d];
#pragma unroll
      for (int w = 0; w < SH::WARPS; ++w) t.H[w * NBMAX + d] += uint16_t(local);
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < SH::IPT; ++r) {
    const uint32_t d = digit(key[r]);
    if (NARROW)
      key[r] += uint32_t(Hw[d]) << 16;
    else
      rank_add(r, Hw[d]);
  }
  __syncthreads();  // H no longer read: S may overwrite it
#pragma unroll
  for (int r = 0; r < SH::IPT; ++r)
    if (FULL || wofs + r * 32 < tile_n) {
      if (NARROW)
        t.S[key[r] >> 16] = uint64_t(key[r] & 0xffffu) | (uint64_t(pay_at(r)) << 32);
      else
        t.S[rank_get(r)] = uint64_t(key[r]) | (uint64_t(pay_at(r)) << 32);
    }
  PROF_MARK(3);
  // ---- look-back, part 2: finish from the status already in hand
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    const uint32_t d = threadIdx.x + uint32_t(k) * SH::THREADS;
    if (d >= NB) break;
    const uint32_t c = t.cnt[d], local = t.gbase[d];
    uint64_t excl = 0;
    if (tile > 0) {
      excl = lookback_from(t.status, tile, NB, d, t.epoch, first[k]);
      st_relaxed_u64(&st[d], st_word(t.epoch, kStPrefix, excl + c));
    }
    t.gbase[d] = t.bstart[d] + uint32_t(excl) - local;
  }
  __syncthreads();
  PROF_MARK(4);
  } else {
  // ---- look-back: global base of each digit for this tile
  for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS) {
    const uint32_t c = t.cnt[d], local = t.gbase[d];
    uint64_t excl = 0;
    if (tile > 0) {
#ifndef NDX_EXP_NOLOOKBACK
      excl = lookback(t.status, tile, NB, d, t.epoch);
#endif
      st_relaxed_u64(&st[d], st_word(t.epoch, kStPrefix, excl + c));
    }
#pragma unroll
    for (int w = 0; w < SH::WARPS; ++w) t.H[w * NBMAX + d] += uint16_t(local);
    t.gbase[d] = t.bstart[d] + uint32_t(excl) - local;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < SH::IPT; ++r) {
    const uint32_t d = digit(key[r]);
    if (NARROW)
      key[r] += uint32_t(Hw[d]) << 16;
    else
      rank_add(r, Hw[d]);
  }
  __syncthreads();  // H no longer read: S may overwrite it
#pragma unroll
  for (int r = 0; r < SH::IPT; ++r)
    if (FULL || wofs + r * 32 < tile_n) {
      if (NARROW)
        t.S[key[r] >> 16] = uint64_t(key[r] & 0xffffu) | (uint64_t(pay_at(r)) << 32);
      else
        t.S[rank_get(r)] = uint64_t(key[r]) | (uint64_t(pay_at(r)) << 32);
    }
  __syncthreads();
  }

  // ---- scatter: consecutive local slots of one digit are consecutive globally
  const uint32_t lim = FULL ? uint32_t(SH::TILE) : tile_n;
  if (t.out_keys) {
    for (uint32_t j = threadIdx.x; j < lim; j += SH::THREADS) {
      const uint64_t e = t.S[j];
      const uint32_t pos = t.gbase[((uint32_t(e) - t.base) >> t.shift) & DMASK] + j;
      t.out_keys[pos] = uint32_t(e);
      t.out_pays[pos] = uint32_t(e >> 32);
    }
  } else {
#pragma unroll 4
    for (uint32_t j = threadIdx.x; j < lim; j += SH::THREADS) {
      const uint64_t e = t.S[j];
      const uint32_t pos = t.gbase[((uint32_t(e) - t.base) >> t.shift) & DMASK] + j;
      t.out_pairs[pos] = e;
    }
  }
  __syncthreads();
  PROF_MARK(5);
}

template <class SH, int BITS, int NBMAX>
__device__ __forceinline__ void tile_loop(const TileCtx& t, uint32_t* ctr, uint32_t* s_tile,
                                          uint64_t n) {
  const uint64_t tiles = (n + SH::TILE - 1) / SH::TILE;
  for (;;) {
    if (threadIdx.x == 0) *s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint64_t tile = *s_tile;
    if (tile >= tiles) return;
#if NDX_SORT_L2PF
    // bulk L2 prefetch of the tile about one round of CTAs ahead (tiles are
    // taken in counter order, so that tile is about one tile-time away):
    // whichever CTA takes it finds its input in L2, and the ranking's loads
    // wait on L2 instead of HBM latency
    if (threadIdx.x == 0) {
      const uint64_t pf = tile + uint64_t(gridDim.x) * NDX_SORT_L2PF / 2;
      if ((pf + 1) * SH::TILE <= n) {
        const void* src = t.in_pairs ? static_cast<const void*>(t.in_pairs + pf * SH::TILE)
                                     : static_cast<const void*>(t.in_keys + pf * SH::TILE);
        const uint32_t bytes = uint32_t(SH::TILE) * (t.in_pairs ? 8u : 4u);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
        if (!t.in_pairs && t.in_pays)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(t.in_pays + pf * SH::TILE),
                       "r"(uint32_t(SH::TILE) * 4u) : "memory");
      }
    }
#endif
    const uint32_t tn = uint32_t(umin<uint64_t>(SH::TILE, n - tile * SH::TILE));
    constexpr bool kNarrowOk = SH::kNarrowOk;
    if (tn == uint32_t(SH::TILE)) {
      if (kNarrowOk && t.narrow)
        tile_pass<SH, BITS, NBMAX, true, true>(t, tile, tn);
      else
        tile_pass<SH, BITS, NBMAX, true, false>(t, tile, tn);
    } else {
      if (kNarrowOk && t.narrow)
        tile_pass<SH, BITS, NBMAX, false, true>(t, tile, tn);
      else
        tile_pass<SH, BITS, NBMAX, false, false>(t, tile, tn);
    }
  }
}

// One stable scatter pass over persistent CTAs.  Pass q writes X iff
// (P-1-q) is even, so the last pass lands in X.
template <int MAXB, int V = 0>
__global__ __launch_bounds__(Shape<MAXB, V>::THREADS, Shape<MAXB, V>::MINB) void k_pass(SortArgs a, int which) {
  if (which < 0 && blockIdx.x == 0 && threadIdx.x == 0)
    a.ctl->row_hi = a.row_base + uint32_t(a.n - 1);  // read by the emit stage
  PassInfo pi;
  if (!pass_info(a, which, pi)) return;
  // the split-off first pass takes pass 0 of a row-id sort (no payload input)
  const bool split0 = NDX_SORT_SPLIT_FIRST && a.in_payloads == nullptr;
  if (V == 1 && !(split0 && pi.p == 0)) return;
  if (MAXB == 8 && V == 0 && split0 && pi.p == 0) return;  // the other kernel's pass
  extern __shared__ __align__(16) unsigned char smem[];
  using SM = SortSmem<MAXB>;
  TileCtx t;
  const bool first = pi.p == 0, last = pi.p == pi.P - 1;
  t.in_keys = first ? a.in_keys : nullptr;
  t.in_pays = first ? a.in_payloads : nullptr;
  t.in_pairs = first ? nullptr : ((((pi.P - 1 - (pi.p - 1)) & 1) == 0) ? a.X : a.Y);
  t.out_pairs = (((pi.P - 1 - pi.p) & 1) == 0) ? a.X : a.Y;
  t.out_keys = last ? a.out_keys : nullptr;
  t.out_pays = last ? a.out_payloads : nullptr;
  t.shift = pi.shift;
  t.base = pi.base;
  t.row_base = a.row_base;
  t.epoch = pi.epoch;
  t.bstart = pi.bstart;
  t.status = a.status;
  t.narrow = Shape<MAXB, V>::kNarrowOk && a.ctl->max_key < 65536u;
  t.H = reinterpret_cast<uint16_t*>(smem);
  t.S = reinterpret_cast<uint64_t*>(smem);
  t.cnt = reinterpret_cast<uint32_t*>(smem + SM::kUnion);
  t.gbase = t.cnt + SM::NB;
  uint32_t* s_tile = t.gbase + SM::NB;
  uint32_t* ctr = &a.ctl->tile_ctr[which + 2];  // [0] emit, [1] wide, [2..5] bytes
  if (MAXB == 8) {
    tile_loop<Shape<MAXB, V>, 8, SM::NB>(t, ctr, s_tile, a.n);
  } else {
    // digits above `bits` are zero for every key, so a wider match is exact
    if (pi.bits <= 4)
      tile_loop<Shape<MAXB, V>, 4, SM::NB>(t, ctr, s_tile, a.n);
    else if (pi.bits <= 8)
      tile_loop<Shape<MAXB, V>, 8, SM::NB>(t, ctr, s_tile, a.n);
    else if (pi.bits <= 9)
      tile_loop<Shape<MAXB, V>, 9, SM::NB>(t, ctr, s_tile, a.n);
    else if (pi.bits <= 10)
      tile_loop<Shape<MAXB, V>, 10, SM::NB>(t, ctr, s_tile, a.n);
    else
      tile_loop<Shape<MAXB, V>, (MAXB > 10 ? 11 : 10), SM::NB>(t, ctr, s_tile, a.n);
  }
}

// ------------------------------------------------------------------ host --

struct LaunchCfg {
  int sms = 0;
  int occ_wide = 1, occ_byte = 1, occ_first = 1;
  bool ready = false;
};
static LaunchCfg g_cfg[64];

static int launch_cfg(LaunchCfg** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  LaunchCfg& c = g_cfg[dev & 63];
  if (!c.ready) {
    if ((e = cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev))) return e;
    const size_t sw = SortSmem<kWideMaxBits>::kBytes, sb = SortSmem<8>::kBytes;
    if ((e = cudaFuncSetAttribute(k_pass<kWideMaxBits>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(sw))))
      return e;
    if ((e = cudaFuncSetAttribute(k_pass<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sb))))
      return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
             &c.occ_wide, k_pass<kWideMaxBits>, Shape<kWideMaxBits>::THREADS, sw)))
      return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_byte, k_pass<8>,
                                                           Shape<8>::THREADS, sb)))
      return e;
#if NDX_SORT_SPLIT_FIRST
    if ((e = cudaFuncSetAttribute(k_pass<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sb))))
      return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_first, k_pass<8, 1>,
                                                           Shape<8, 1>::THREADS, sb)))
      return e;
    if (c.occ_first < 1) c.occ_first = 1;
#endif
#ifdef NDX_SORT_OCC_CAP
    c.occ_wide = umin(c.occ_wide, NDX_SORT_OCC_CAP);
    c.occ_byte = umin(c.occ_byte, NDX_SORT_OCC_CAP);
#endif
    if (c.occ_wide < 1) c.occ_wide = 1;
    if (c.occ_byte < 1) c.occ_byte = 1;
    c.ready = true;
  }
  *out = &c;
  return 0;
}

template <int MAXB>
static uint64_t sort_tiles(uint64_t n) {
  return (n + Shape<MAXB>::TILE - 1) / Shape<MAXB>::TILE;
}

static int launch_sort(SortArgs a, cudaStream_t s, LaunchCfg* c) {
  const int gw = int(umin<uint64_t>(sort_tiles<kWideMaxBits>(a.n), uint64_t(c->sms) * c->occ_wide));
  const int gb = int(umin<uint64_t>(sort_tiles<8>(a.n), uint64_t(c->sms) * c->occ_byte));
  k_pass<kWideMaxBits>
      <<<gw, Shape<kWideMaxBits>::THREADS, SortSmem<kWideMaxBits>::kBytes, s>>>(a, -1);
  for (int k = 0; k < 4; ++k) {
#if NDX_SORT_SPLIT_FIRST
    const int gf = int(umin<uint64_t>(sort_tiles<8>(a.n), uint64_t(c->sms) * c->occ_first));
    k_pass<8, 1><<<gf, Shape<8, 1>::THREADS, SortSmem<8>::kBytes, s>>>(a, k);
#endif
    k_pass<8><<<gb, Shape<8>::THREADS, SortSmem<8>::kBytes, s>>>(a, k);
  }
  return cudaGetLastError();
}

static int launch_plan(const uint32_t* keys, uint64_t n, Ctl* ctl, uint32_t* epoch_counter,
                       cudaStream_t s, LaunchCfg* c) {
  cudaError_t e = cudaMemsetAsync(ctl, 0, offsetof(Ctl, zero_end), s);
  if (e) return e;
  // one wave: every CTA resident (a second partial wave would run alone)
  static int hist_occ = 0;
  if (!hist_occ && (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hist_occ, k_hist, kHistThreads, 0)))
    return e;
  const int grid = int(umax<uint64_t>(1, umin<uint64_t>(uint64_t(c->sms) * umax(hist_occ, 1), (n + 65535) / 65536)));
  k_hist<<<grid, kHistThreads, 0, s>>>(keys, n, ctl);
  k_plan<<<1, 1024, 0, s>>>(ctl, n, 0, epoch_counter);
  k_hist_hi<<<c->sms * 2, kHistThreads, 0, s>>>(keys, n, ctl);
  k_plan<<<1, 1024, 0, s>>>(ctl, n, 1, epoch_counter);
  return cudaGetLastError();
}


}  // namespace ndx

using namespace ndx;

extern "C" {

size_t ndx_wah_ctl_bytes(void) { return (sizeof(Ctl) + 255) & ~size_t(255); }

size_t ndx_wah_status_bytes(uint64_t n) { return status_bytes(n); }

int ndx_wah_plan(const uint32_t* d_keys, uint64_t n, void* d_ctl, void* d_status,
                 void* stream) {
  if (!d_keys || !d_ctl || !d_status || n == 0) return NDX_E_INVALID;
  if (n >= (1ull << 31)) return NDX_E_TOO_LARGE;
  LaunchCfg* c;
  int rc = launch_cfg(&c);
  if (rc) return rc;
  return launch_plan(d_keys, n, static_cast<Ctl*>(d_ctl), static_cast<uint32_t*>(d_status),
                     static_cast<cudaStream_t>(stream), c);
}

int ndx_wah_sort(const uint32_t* d_keys, uint64_t n, uint32_t row_base, void* d_ctl,
                 uint64_t* d_pairs, uint64_t* d_tmp_pairs, void* d_status, void* stream) {
  if (!d_keys || !d_ctl || !d_pairs || !d_tmp_pairs || !d_status || n == 0)
    return NDX_E_INVALID;
  if (n >= (1ull << 31)) return NDX_E_TOO_LARGE;
  LaunchCfg* c;
  int rc = launch_cfg(&c);
  if (rc) return rc;
  SortArgs a{};
  a.in_keys = d_keys;
  a.X = d_pairs;
  a.Y = d_tmp_pairs;
  a.n = n;
  a.row_base = row_base;
  a.ctl = static_cast<Ctl*>(d_ctl);
  a.status = reinterpret_cast<uint64_t*>(static_cast<char*>(d_status) + 256);
  return launch_sort(a, static_cast<cudaStream_t>(stream), c);
}

size_t ndx_sort_pairs_scratch_bytes(uint64_t n) {
  // ctl | X pairs | Y pairs | copies of the input | statuses
  return ndx_wah_ctl_bytes() + size_t(n) * 24 + status_bytes(n) + 1024;
}

// sort_pairs: stable sort of SoA (keys, payloads) in place.  The input is
// copied aside so the last pass can scatter into the caller's buffers; the
// status region is cleared per call (this entry point is not the hot path).
int ndx_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_payloads, uint64_t n, void* d_scratch,
                       void* stream) {
  if (n == 0) return 0;
  if (!d_keys || !d_payloads || !d_scratch) return NDX_E_INVALID;
  if (n >= (1ull << 31)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LaunchCfg* c;
  int rc = launch_cfg(&c);
  if (rc) return rc;
  char* base = static_cast<char*>(d_scratch);
  Ctl* ctl = reinterpret_cast<Ctl*>(base);
  uint64_t* X = reinterpret_cast<uint64_t*>(base + ndx_wah_ctl_bytes());
  uint64_t* Y = X + n;
  uint32_t* ck = reinterpret_cast<uint32_t*>(Y + n);
  uint32_t* cp = ck + n;
  char* status = reinterpret_cast<char*>(((reinterpret_cast<uintptr_t>(cp + n)) + 255) & ~uintptr_t(255));
  cudaError_t e;
  if ((e = cudaMemsetAsync(status, 0, status_bytes(n), s))) return e;
  if ((e = cudaMemcpyAsync(ck, d_keys, n * 4, cudaMemcpyDeviceToDevice, s))) return e;
  if ((e = cudaMemcpyAsync(cp, d_payloads, n * 4, cudaMemcpyDeviceToDevice, s))) return e;
  if ((rc = launch_plan(ck, n, ctl, reinterpret_cast<uint32_t*>(status), s, c))) return rc;
  SortArgs a{};
  a.in_keys = ck;
  a.in_payloads = cp;
  a.X = X;
  a.Y = Y;
  a.out_keys = d_keys;
  a.out_payloads = d_payloads;
  a.n = n;
  a.ctl = ctl;
  a.status = reinterpret_cast<uint64_t*>(status + 256);
  return launch_sort(a, s, c);
}

}  // extern "C"

#if NDX_SORT_PROF
extern "C" int ndx_sort_prof_read(unsigned long long* h, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(h, ndx::g_sort_prof, sizeof(ndx::g_sort_prof));
  if (!e && reset) {
    unsigned long long z[8] = {};
    e = cudaMemcpyToSymbol(ndx::g_sort_prof, z, sizeof(z));
  }
  return e;
}
#endif
