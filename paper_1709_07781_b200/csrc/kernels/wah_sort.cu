// Stages S1 (plan) and S2 (sort) of the WAH build on sm_100a.
//
// Replaces the reference's row_iota + sort_pairs (p/core/src/wah_builder.cpp:54-63,
// p/core/src/wah_radix.cpp:16-127) and the histogram scans it runs
// (wah_scan.cpp:14-95).  Design:
//
//   S1  k_hist    one streaming read of the keys: key range (min/max) and the
//                 digit histograms (bytes 0,1 and the low 11 bits) in smem,
//                 flushed with one global atomic per bin per CTA.
//       k_plan_scan picks the pass structure without a host round trip
//                 (and scans the first pass's per-chunk digit offsets):
//                   range < 2048            -> wide: ONE pass on key - min
//                   bytes 2,3 constant and
//                   bytes 0,1 both varying  -> compact: passes A, B with a
//                                              packed u32 intermediate
//                   otherwise               -> byte-wise LSD passes over the
//                                              bytes that vary
//                 and turns the histograms into bucket start offsets.  Only
//                 when bytes 2/3 vary does it launch (in its own tail, CUDA
//                 dynamic parallelism) their histogram and k_plan_hi.
//       k_vs      (after the passes) the rows form's value starts.
//   S2  the sort stage (launch_sort_dispatch, wah_pass.cu) launches one
//                 kernel per pass kind; each returns at once unless the plan
//                 picked it, so the host never waits for the plan.  The wide
//                 and compact passes are in wah_pass.cu; here are the legacy
//                 passes: k_pass_bytes (every byte pass of general keys in
//                 one cooperative launch) and k_pass<11> (the wide pass of
//                 sort_pairs, which carries caller payloads) -- persistent
//                 onesweep-style stable scatters: warp ballot-match ranking,
//                 the tile's digit counts published after the ranking,
//                 decoupled look-back per digit, smem staging in digit
//                 order, coalesced scatter.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "../../../include/ndx.h"
#include "wah_sort_common.cuh"

namespace ndx {

// Legacy pass shapes (measured on B200 in round 1): byte passes 256 threads
// x 32 pairs (8192-pair tiles, 2 CTAs/SM), the wide pass 512 x 32 (16384,
// 1 CTA/SM: its look-back covers up to 2048 digits per tile).
template <int MAXB>
struct Shape {
  static constexpr bool kWide = MAXB > 8;
  static constexpr int THREADS = kWide ? 512 : 256;
  static constexpr int IPT = 32;  // pairs per thread
  static constexpr int MINB = kWide ? 1 : 2;
  // wide pass: keys < 2^16 there, so a pair's rank rides in the upper half of
  // its key register (measured: helps the wide pass, hurts the byte passes)
  static constexpr bool kNarrowOk = kWide;
  // byte passes: the first look-back read is issued before the staging
  static constexpr bool kEarlyLookback = !kWide;
  // wide pass: every lane reads its digit counter (broadcast) rather than
  // leader read + shuffle (C3 541 -> 534 us; the byte passes measured the
  // other way round, 2.755 vs 2.790 ms on C4)
  static constexpr bool kBcast = kWide;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int WARP_ITEMS = 32 * IPT;
  static constexpr int TILE = THREADS * IPT;
};
static_assert(Shape<8>::TILE == kLegacyByteTile && Shape<kWideMaxBits>::TILE == kLegacyWideTile, "tiles");

// ------------------------------------------------------------------ S1 ----

constexpr int kHistThreads = 512;  // k_hist_hi
#ifndef NDX_HIST_THREADS
#define NDX_HIST_THREADS 256
#endif
#ifndef NDX_HIST_MINB
#define NDX_HIST_MINB 4
#endif
// k_hist: every CTA resident at once, each with the same number of chunks,
// so no SM runs a last round of chunks alone
constexpr int kHistCtaThreads = NDX_HIST_THREADS;

// Key range, low-11-bit histogram and byte-1 histogram in one read of the
// keys, counted per chunk of the first pass (chunk_begin): each CTA takes
// whole chunks, writes every chunk's 11-bit counts (the plan scans them into
// the first pass's per-chunk offsets) and adds them to the column's.  Every
// group of four warps counts into its own copy so a skewed column's hot bins
// are not one shared-memory hot spot.
constexpr int kHistCopies = 4;
__global__ __launch_bounds__(kHistCtaThreads, NDX_HIST_MINB) void k_hist(const uint32_t* __restrict__ keys, uint64_t n,
                                                          Ctl* ctl, uint32_t* __restrict__ chunk_hist,
                                                          uint32_t nchunk) {
  __shared__ uint32_t hws[kHistCopies][kWideBuckets], h1s[kHistCopies][256];
  for (int i = threadIdx.x; i < kHistCopies * 256; i += blockDim.x) (&h1s[0][0])[i] = 0;
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
  const bool vec = (reinterpret_cast<uintptr_t>(keys) & 15u) == 0;  // chunk bounds are 16-key multiples
  for (uint32_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
    for (int i = threadIdx.x; i < kHistCopies * kWideBuckets; i += blockDim.x) (&hws[0][0])[i] = 0;
    __syncthreads();
    const uint64_t e0 = chunk_begin(n, nchunk, c), e1 = chunk_begin(n, nchunk, c + 1);
    if (vec) {
      const uint4* q = reinterpret_cast<const uint4*>(keys + e0);
      const uint64_t nq = (e1 - e0) / 4;
      const uint64_t stride = blockDim.x;
      uint64_t i = threadIdx.x;
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
      for (; i < nq; i += stride) {
        const uint4 v = ldg_stream4(q + i);
        one(v.x); one(v.y); one(v.z); one(v.w);
      }
      for (uint64_t j = e0 + nq * 4 + threadIdx.x; j < e1; j += stride) one(keys[j]);
    } else {
      for (uint64_t j = e0 + threadIdx.x; j < e1; j += blockDim.x) one(keys[j]);
    }
    __syncthreads();
    uint32_t* out = chunk_hist + uint64_t(c) * kChunkHistWords;
    for (int i = threadIdx.x; i < kWideBuckets; i += blockDim.x) {
      uint32_t cnt = 0;
#pragma unroll
      for (int k = 0; k < kHistCopies; ++k) cnt += hws[k][i];
      out[i] = cnt;
      hws[0][i] = cnt;
      if (cnt) atomicAdd(&ctl->hist_wide[i], cnt);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {  // byte 0: the 11 bits folded
      uint32_t cnt = 0;
#pragma unroll
      for (int j = 0; j < kWideBuckets / 256; ++j) cnt += hws[0][i + 256 * j];
      out[kWideBuckets + i] = cnt;
    }
    __syncthreads();
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
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kHistCopies; ++k) cnt += h1s[k][i];
    if (cnt) atomicAdd(&ctl->hist_byte[1][i], cnt);
  }
}

// Histograms of bytes 2 and 3 (launched by the plan only when they vary).
__global__ __launch_bounds__(kHistThreads) void k_hist_hi(const uint32_t* __restrict__ keys, uint64_t n,
                                                          Ctl* ctl) {
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

struct PlanArgs {
  const uint32_t* keys;
  uint64_t n;
  Ctl* ctl;
  uint32_t* epoch_counter;  // status buffer header
  uint32_t* tile_group;     // compact mode: sentinel slot written here
  int allow_compact;        // the WAH build (row ids synthesised); not sort_pairs
  int hist_hi_grid;
};

// The plan once bytes 2/3 were counted (tail-launched by k_plan_scan only
// when they vary; general keys, pairs form).
__global__ __launch_bounds__(1024) void k_plan_hi(PlanArgs a) { plan_bytes(a.ctl, a.n, 4); }

// S1's plan and the first pass's per-chunk digit offsets, one launch.  Every
// CTA makes the (small) plan in shared memory from the key range and the
// histograms -- the same plan in every CTA -- and CTA 0 publishes it, taking
// the build's look-back tag from the counter in the status buffer's header
// (statuses of earlier builds never read as ready).  Then, for the wide and
// compact modes, each CTA takes 32 digits: chunk c's run of digit d starts at
// bucket_start[d] + the count of d in chunks < c (warp g sums its slice of
// the chunks for every digit, the slices are scanned, each warp writes its
// chunks' offsets).
__global__ __launch_bounds__(1024) void k_plan_scan(PlanArgs a, const uint32_t* __restrict__ chunk_hist,
                                                    uint32_t* __restrict__ chunk_off, uint32_t nchunk) {
  Ctl* ctl = a.ctl;
  const uint64_t n = a.n;
  SortPlan& p = ctl->plan;
  __shared__ uint32_t s_h[kWideBuckets], s_bs[kWideBuckets], s_h1[256], s_bs1[256];
  __shared__ uint32_t s_wrap;
  const uint32_t mn = ~ctl->max_not, mx = ctl->max_seen, range = mx - mn;
  const bool wide = range < uint32_t(kWideBuckets);
  const uint32_t wide_bits = range == 0 ? 0u : 32u - __clz(range);
  const bool need_hi = !wide && (mn >> 16) != (mx >> 16);
  bool b0 = false, b1 = false;
  if (wide) {
    const uint32_t nb = 1u << wide_bits;
    for (uint32_t d = threadIdx.x; d < uint32_t(kWideBuckets); d += blockDim.x)
      s_h[d] = d < nb ? ctl->hist_wide[(d + mn) & (kWideBuckets - 1)] : 0u;
    __syncthreads();
    block_excl_scan(s_h, s_bs, kWideBuckets);
  } else {
    // byte 0's histogram is the low-11-bit one folded; byte 1's from k_hist
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
      uint32_t c = 0;
      for (int j = 0; j < kWideBuckets / 256; ++j) c += ctl->hist_wide[i + 256 * j];
      s_h[i] = c;
      s_h1[i] = ctl->hist_byte[1][i];
    }
    __syncthreads();
    b0 = s_h[mn & 255u] != n;
    b1 = s_h1[(mn >> 8) & 255u] != n;
    if (!need_hi) {
      if (b0) block_excl_scan(s_h, s_bs, 256);
      if (b1) block_excl_scan(s_h1, s_bs1, 256);
    }
  }
  const bool ab = !wide && !need_hi && a.allow_compact && b0 && b1;

  if (blockIdx.x == 0) {
    // The tags are 24 bits: after 2^21 builds they come round again, and a
    // status left by a build one cycle ago (at tiles no build since has
    // reached) would read as ready.  So on the wrap every status ever written
    // -- below the high-water mark kept in the header -- is cleared first.
    uint64_t* hwm = reinterpret_cast<uint64_t*>(a.epoch_counter) + 1;
    if (threadIdx.x == 0) {
      *hwm = umax(*hwm, status_bytes(n));
      const uint32_t old = *a.epoch_counter;
      s_wrap = old >= kEpochMax;
      const uint32_t ep = old >= kEpochMax ? kEpochStep : old + kEpochStep;
      *a.epoch_counter = ep;
      ctl->epoch = ep;
      ctl->min_key = mn;
      ctl->max_key = mx;
      ctl->n_lo = uint32_t(n);
      ctl->n_hi = uint32_t(n >> 32);
      p.need_hi = need_hi;
      if (wide) {
        p.mode = kModeWide;
        p.base = mn;
        p.wide_bits = wide_bits;
        p.npasses = 1;
        p.complete = 1;
        for (int k = 0; k < 4; ++k) p.byte_active[k] = 0;
      } else if (need_hi) {
        p.mode = kModeBytes;
        p.complete = 0;
        k_hist_hi<<<a.hist_hi_grid, kHistThreads, 0, cudaStreamTailLaunch>>>(a.keys, n, ctl);
        k_plan_hi<<<1, 1024, 0, cudaStreamTailLaunch>>>(a);
      } else {  // plan_bytes over bytes 0/1, then the compact mode when both vary
        p.byte_active[0] = b0;
        p.byte_active[1] = b1;
        p.byte_active[2] = p.byte_active[3] = 0;
        p.byte_order[0] = 0;
        p.byte_order[1] = b0 ? 1u : 0u;
        p.byte_order[2] = p.byte_order[3] = 0;
        p.npasses = uint32_t(b0) + uint32_t(b1);
        p.mode = kModeBytes;
        p.complete = 1;
        if (ab) {
          p.mode = kModeAB;
          p.base = mn & 0xffff0000u;
          p.nseg = uint32_t(n_segments(n));
          a.tile_group[ceil_div(n, kBTile)] = 256u * p.nseg - 1u;  // group of the position past the end
        }
      }
    }
    if (wide) {
      for (int d = threadIdx.x; d < kWideBuckets; d += blockDim.x) p.bucket_start_wide[d] = s_bs[d];
    } else {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        ctl->hist_byte[0][i] = s_h[i];
        if (!need_hi && b0) p.bucket_start_byte[0][i] = s_bs[i];
        if (!need_hi && b1) p.bucket_start_byte[1][i] = s_bs1[i];
      }
    }
    __syncthreads();
    if (s_wrap) {  // once per 2^21 builds: every status ever written, cleared
      uint4* q = reinterpret_cast<uint4*>(reinterpret_cast<char*>(a.epoch_counter) + kStatusOffset);
      const uint64_t nq = (*hwm - kStatusOffset) / sizeof(uint4);
      for (uint64_t i = threadIdx.x; i < nq; i += blockDim.x) q[i] = make_uint4(0, 0, 0, 0);
    }
  }

  // ---- the first pass's per-chunk digit offsets
  if (!wide && !ab) return;
  const uint32_t nb = wide ? (1u << wide_bits) : 256u;
  if (blockIdx.x * 32 >= nb) return;
  __shared__ uint32_t part[32][33];
  const uint32_t lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const uint32_t d = blockIdx.x * 32 + lane;
  auto count = [&](uint32_t c) -> uint32_t {
    const uint32_t* h = chunk_hist + uint64_t(c) * kChunkHistWords;
    return __ldg(h + (wide ? ((d + mn) & (kWideBuckets - 1)) : kWideBuckets + d));
  };
  // at most kMaxChunks / 32 chunks per warp: every load of the slice in
  // flight at once
  constexpr int kPer = int(kMaxChunks / 32);
  const uint32_t c0 = uint32_t(uint64_t(nchunk) * g / 32), c1 = uint32_t(uint64_t(nchunk) * (g + 1) / 32);
  uint32_t cnt[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) cnt[k] = (d < nb && c0 + k < c1) ? count(c0 + k) : 0u;
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) sum += cnt[k];
  part[g][lane] = sum;
  __syncthreads();
  if (g == 0) {
    uint32_t run = 0;
    for (int k = 0; k < 32; ++k) {
      const uint32_t t = part[k][lane];
      part[k][lane] = run;
      run += t;
    }
  }
  __syncthreads();
  if (d < nb) {
    uint32_t run = s_bs[d] + part[g][lane];
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (c0 + k < c1) {
        chunk_off[uint64_t(c0 + k) * kWideBuckets + d] = run;
        run += cnt[k];
      }
  }
}

// Rows form of the sorted stream (wide and compact modes): the present keys
// in order and the stream position where each one's rows begin -- the value
// heads the emit stage needs, so the passes write 4-byte row ids instead of
// 8-byte (key, row) pairs.  Every key's start is known already (wide: the
// plan's bucket starts; compact: pass B's vs16); a key is present when the
// next one starts later.  One thread per key, 64 CTAs: ballot ranks inside
// the CTA, the CTA's base from its predecessors' published counts (all CTAs
// are resident, each waits on lower ones only).
constexpr int kVsThreads = 1024;
constexpr int kVsBlocks = kMaxRowsValues / kVsThreads;
__global__ __launch_bounds__(kVsThreads) void k_vs(Ctl* ctl, uint64_t n, uint32_t row_base) {
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->row_hi = row_base + uint32_t(n - 1);  // read by the emit
  const SortPlan& p = ctl->plan;
  const uint32_t mode = p.mode;
  if (mode != kModeWide && mode != kModeAB) return;  // bytes mode: pairs (rows_form stays 0)
  const bool wide = mode == kModeWide;
  const uint32_t nb = wide ? (1u << p.wide_bits) : uint32_t(kMaxRowsValues);
  if (blockIdx.x * kVsThreads >= nb) return;
  const uint32_t* start = wide ? p.bucket_start_wide : ctl->vs16;
  const uint32_t k = blockIdx.x * kVsThreads + threadIdx.x;
  const uint32_t pk = k < nb ? start[k] : 0u;
  const uint32_t pn = k + 1 < nb ? start[k + 1] : uint32_t(n);
  const bool present = k < nb && pn > pk;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t bal = __ballot_sync(kFull, present);
  __shared__ uint32_t s_w[32], s_base;
  if (lane == 0) s_w[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = s_w[lane];
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, d);
      if (lane >= uint32_t(d)) x += y;
    }
    s_w[lane] = x - v;
    const uint32_t total = __shfl_sync(kFull, x, 31);
    constexpr uint64_t kReady = 1ull << 63;  // vs_agg is cleared with the control block
    if (lane == 0) st_relaxed_u64(&ctl->vs_agg[blockIdx.x], kReady | total);
    uint32_t before = 0;
    for (uint32_t b = lane; b < blockIdx.x; b += 32) {
      uint64_t w;
      while (!((w = ld_relaxed_u64(&ctl->vs_agg[b])) & kReady)) __nanosleep(20);
      before += uint32_t(w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(kFull, before, o);
    if (lane == 0) {
      s_base = before;
      if ((blockIdx.x + 1) * kVsThreads >= nb) {  // the last block: the totals
        ctl->nvals = before + total;
        ctl->vs[before + total] = uint32_t(n);
        ctl->rows_form = 1;
      }
    }
  }
  __syncthreads();
  if (present) {
    const uint32_t j = s_base + s_w[warp] + __popc(bal & ((1u << lane) - 1u));
    ctl->vs[j] = pk;
    ctl->pk[j] = wide ? p.base + k : (p.base | k);
  }
}


// ------------------------------------------------------------------ S2 ----

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
static_assert(SortSmem<8>::kBytes == kLegacyByteSmem && SortSmem<kWideMaxBits>::kBytes == kLegacyWideSmem,
              "the dispatcher launches the legacy passes with these sizes");

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
  bool pf_ok;                // inputs 16-byte aligned: bulk L2 prefetch allowed
};

// One tile of a stable scatter pass.  BITS is the digit width (compile time,
// so the ballot match unrolls straight); FULL tiles skip every bounds check.
// Element order within a warp is round-major / lane-minor, which is row
// order, so ranks taken round by round are stable.  NARROW: every key is
// below 2^16, so a pair's rank rides in the upper half of its key register.
template <class SH, int BITS, int NBMAX, bool FULL, bool NARROW>
__device__ __forceinline__ void tile_pass(const TileCtx& t, uint64_t tile, uint32_t tile_n) {
  constexpr uint32_t NB = 1u << BITS;
  constexpr uint32_t DMASK = NB - 1;
  auto digit = [&](uint32_t k) -> uint32_t {
    return (((NARROW ? (k & 0xffffu) : k) - t.base) >> t.shift) & DMASK;
  };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t tile_start = tile * SH::TILE;
  uint16_t* Hw = t.H + warp * NBMAX;
  for (uint32_t d = lane; d < NB; d += 32) Hw[d] = 0;

  const uint32_t wofs = uint32_t(warp) * SH::WARP_ITEMS + lane;
  uint32_t key[SH::IPT], pay[SH::IPT];
  const uint32_t r0 = t.row_base + uint32_t(tile_start) + wofs;
  if (t.in_pairs) {
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
    for (int r = 0; r < SH::IPT; ++r) key[r] = (FULL || wofs + r * 32 < tile_n) ? ldg_stream(kp + r * 32) : 0u;
    if (t.in_pays) {
      const uint32_t* rp = t.in_pays + tile_start + wofs;
#pragma unroll
      for (int r = 0; r < SH::IPT; ++r) pay[r] = (FULL || wofs + r * 32 < tile_n) ? ldg_stream(rp + r * 32) : 0u;
    } else {
#pragma unroll
      for (int r = 0; r < SH::IPT; ++r) pay[r] = r0 + r * 32;
    }
  }
  __syncthreads();

  // ---- rank
  static_assert(SH::TILE <= 65536 && SH::IPT % 2 == 0, "packed ranks need 16-bit tile slots");
  uint32_t rank[NARROW ? 1 : SH::IPT / 2] = {};  // two ranks (< 2^16) per register
  auto rank_add = [&](int r, uint32_t v) { rank[r >> 1] += v << (16 * (r & 1)); };
  auto rank_get = [&](int r) -> uint32_t { return (rank[r >> 1] >> (16 * (r & 1))) & 0xffffu; };
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
    uint32_t old = 0;
    if constexpr (SH::kBcast) {
      old = Hw[d];
      __syncwarp();
    } else {
      if (lane == leader) old = Hw[d];
      old = __shfl_sync(kFull, old, leader);
    }
    if (valid && lane == leader) Hw[d] = uint16_t(old + __popc(peers));
    const uint32_t rk = old + __popc(peers & lanemask_lt());
    __syncwarp();
    if (NARROW)
      key[r] |= rk << 16;
    else if ((r & 1) == 0)
      rank[r >> 1] = rk;
    else
      rank[r >> 1] |= rk << 16;
  }
  __syncthreads();

  // ---- per digit: warp offsets (in place); tile counts published
  uint64_t* st = t.status + tile * NB;
  for (uint32_t d = threadIdx.x; d < NB; d += SH::THREADS) {
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < SH::WARPS; ++w) {
      const uint32_t c = t.H[w * NBMAX + d];
      t.H[w * NBMAX + d] = uint16_t(sum);
      sum += c;
    }
    t.cnt[d] = sum;
    st_relaxed_u64(&st[d], st_word(t.epoch, tile == 0 ? kStPrefix : kStAgg, sum));
  }
  __syncthreads();  // the scan reads other threads' counts
  block_excl_scan(t.cnt, t.gbase, int(NB));  // gbase <- tile-local digit starts (syncs)

  constexpr int ND = int((NB + SH::THREADS - 1) / SH::THREADS);
  uint64_t first[ND];
  if constexpr (SH::kEarlyLookback) {
    // the first predecessor status of each of this thread's digits is
    // requested now; its round trip overlaps the rank adjustment and staging
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const uint32_t d = threadIdx.x + uint32_t(k) * SH::THREADS;
      first[k] = (tile > 0 && d < NB) ? ld_relaxed_u64(&t.status[(tile - 1) * NB + d]) : 0ull;
    }
  }
  auto resolve = [&](int k, uint32_t d) {
    const uint32_t c = t.cnt[d], local = t.gbase[d];
    uint64_t excl = 0;
    if (tile > 0) {
      if constexpr (SH::kEarlyLookback)
        excl = lookback_from(t.status, tile, NB, d, t.epoch, first[k]);
      else
        excl = lookback(t.status, tile, NB, d, t.epoch);
      st_relaxed_u64(&st[d], st_word(t.epoch, kStPrefix, excl + c));
    }
    t.gbase[d] = t.bstart[d] + uint32_t(excl) - local;
  };
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    const uint32_t d = threadIdx.x + uint32_t(k) * SH::THREADS;
    if (d >= NB) break;
    const uint32_t local = t.gbase[d];
    if constexpr (!SH::kEarlyLookback) resolve(k, d);  // look-back first, then the local starts
#pragma unroll
    for (int w = 0; w < SH::WARPS; ++w) t.H[w * NBMAX + d] += uint16_t(local);
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
        t.S[key[r] >> 16] = uint64_t(key[r] & 0xffffu) | (uint64_t(pay[r]) << 32);
      else
        t.S[rank_get(r)] = uint64_t(key[r]) | (uint64_t(pay[r]) << 32);
    }
  if constexpr (SH::kEarlyLookback) {
    // look-back, part 2: finish from the status already in hand
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const uint32_t d = threadIdx.x + uint32_t(k) * SH::THREADS;
      if (d >= NB) break;
      resolve(k, d);
    }
  }
  __syncthreads();

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
}

template <class SH, int BITS, int NBMAX>
__device__ __forceinline__ void tile_loop(const TileCtx& t, uint32_t* ctr, uint32_t* s_tile, uint64_t n) {
  const uint64_t tiles = (n + SH::TILE - 1) / SH::TILE;
  for (;;) {
    if (threadIdx.x == 0) *s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint64_t tile = *s_tile;
    if (tile >= tiles) return;
    // bulk L2 prefetch of the tile one round of CTAs ahead (tiles are taken
    // in counter order, so that tile is about one tile-time away): whichever
    // CTA takes it finds its input in L2 (C4 sort 2.755 -> 2.681 ms in r1).
    // Bulk operations need 16-byte aligned addresses: tile offsets are, the
    // input bases are checked (pf_ok).
    if (threadIdx.x == 0 && t.pf_ok) {
      const uint64_t pf = tile + uint64_t(gridDim.x);
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
    const uint32_t tn = uint32_t(umin<uint64_t>(SH::TILE, n - tile * SH::TILE));
    if (tn == uint32_t(SH::TILE)) {
      if (SH::kNarrowOk && t.narrow)
        tile_pass<SH, BITS, NBMAX, true, true>(t, tile, tn);
      else
        tile_pass<SH, BITS, NBMAX, true, false>(t, tile, tn);
    } else {
      if (SH::kNarrowOk && t.narrow)
        tile_pass<SH, BITS, NBMAX, false, true>(t, tile, tn);
      else
        tile_pass<SH, BITS, NBMAX, false, false>(t, tile, tn);
    }
  }
}

// One stable scatter pass over persistent CTAs.  Pass q writes X iff
// (P-1-q) is even, so the last pass lands in X.
template <int MAXB>
__device__ __forceinline__ void legacy_pass(const SortArgs& a, int which, unsigned char* smem) {
  PassInfo pi;
  if (!pass_info(a, which, pi)) return;
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
  t.narrow = Shape<MAXB>::kNarrowOk && a.ctl->max_key < 65536u;
  const void* in = t.in_pairs ? static_cast<const void*>(t.in_pairs) : static_cast<const void*>(t.in_keys);
  t.pf_ok = (reinterpret_cast<uintptr_t>(in) & 15u) == 0 &&
            (!t.in_pays || (reinterpret_cast<uintptr_t>(t.in_pays) & 15u) == 0);
  t.H = reinterpret_cast<uint16_t*>(smem);
  t.S = reinterpret_cast<uint64_t*>(smem);
  t.cnt = reinterpret_cast<uint32_t*>(smem + SM::kUnion);
  t.gbase = t.cnt + SM::NB;
  uint32_t* s_tile = t.gbase + SM::NB;
  uint32_t* ctr = &a.ctl->tile_ctr[which + 2];  // [0] emit, [1] wide, [2..5] bytes
  if (MAXB == 8) {
    tile_loop<Shape<MAXB>, 8, SM::NB>(t, ctr, s_tile, a.n);
  } else {
    // digits above `bits` are zero for every key, so a wider match is exact
    if (pi.bits <= 4)
      tile_loop<Shape<MAXB>, 4, SM::NB>(t, ctr, s_tile, a.n);
    else if (pi.bits <= 8)
      tile_loop<Shape<MAXB>, 8, SM::NB>(t, ctr, s_tile, a.n);
    else if (pi.bits <= 9)
      tile_loop<Shape<MAXB>, 9, SM::NB>(t, ctr, s_tile, a.n);
    else if (pi.bits <= 10)
      tile_loop<Shape<MAXB>, 10, SM::NB>(t, ctr, s_tile, a.n);
    else
      tile_loop<Shape<MAXB>, (MAXB > 10 ? 11 : 10), SM::NB>(t, ctr, s_tile, a.n);
  }
}

template <int MAXB, int V>
__global__ __launch_bounds__(Shape<MAXB>::THREADS, Shape<MAXB>::MINB) void k_pass(SortArgs a, int which) {
  extern __shared__ __align__(16) unsigned char smem[];
  legacy_pass<MAXB>(a, which, smem);
}
// the sort stage (wah_pass.cu) launches the legacy wide pass (sort_pairs)
template __global__ void k_pass<kWideMaxBits, 0>(SortArgs, int);

// Grid-wide barrier of a cooperative launch (every CTA co-resident): a
// counter that the last arriving CTA resets, and a generation it bumps.
__device__ __forceinline__ void grid_barrier(uint32_t* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = ld_acquire_u32(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      st_release_u32(bar + 1, gen + 1);
    } else {
      while (ld_acquire_u32(bar + 1) == gen) __nanosleep(100);
    }
  }
  __syncthreads();
}

// Every byte pass of general keys in one cooperative launch: the active
// bytes in plan order, a grid barrier between passes (no empty launches for
// the bytes that do not vary).
__global__ __launch_bounds__(Shape<8>::THREADS, Shape<8>::MINB) void k_pass_bytes(SortArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SortPlan& pl = a.ctl->plan;
  if (pl.mode != kModeBytes) return;
  const uint32_t P = pl.npasses;
  for (uint32_t p = 0; p < P; ++p) {
    int which = -1;
    for (int k = 0; k < 4; ++k)
      if (pl.byte_active[k] && pl.byte_order[k] == p) which = k;
    if (p > 0) grid_barrier(&a.ctl->grid_bar[0]);
    legacy_pass<8>(a, which, smem);
  }
}

// ------------------------------------------------------------------ host --

int first_pass_chunks(uint64_t n, uint32_t* k);  // wah_pass.cu

struct LegacyCfg {
  int sms = 0;
  int occ_wide = 1, occ_byte = 1, occ_hist = 1;
};

// per-device launch configuration, computed once per device (thread-safe)
static int legacy_cfg(const LegacyCfg** out) {
  static LegacyCfg cfg[64];
  static std::once_flag once[64];
  static int rc_of[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  std::call_once(once[dev & 63], [dev] {
    LegacyCfg& c = cfg[dev & 63];
    int& rc = rc_of[dev & 63];
    const size_t sw = SortSmem<kWideMaxBits>::kBytes, sb = SortSmem<8>::kBytes;
    if ((rc = cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev))) return;
    if ((rc = cudaFuncSetAttribute(k_pass<kWideMaxBits, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sw))))
      return;
    if ((rc = cudaFuncSetAttribute(k_pass_bytes, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sb)))) return;
    if ((rc = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_wide, k_pass<kWideMaxBits, 0>,
                                                            Shape<kWideMaxBits>::THREADS, sw)))
      return;
    if ((rc = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_byte, k_pass_bytes, Shape<8>::THREADS, sb)))
      return;
    if ((rc = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_hist, k_hist, kHistCtaThreads, 0))) return;
    c.occ_wide = umax(c.occ_wide, 1);
    c.occ_byte = umax(c.occ_byte, 1);
    c.occ_hist = umax(c.occ_hist, 1);
  });
  if (rc_of[dev & 63]) return rc_of[dev & 63];
  *out = &cfg[dev & 63];
  return 0;
}

static int launch_plan(const uint32_t* keys, uint64_t n, Ctl* ctl, char* status_buf, int allow_compact,
                       cudaStream_t s) {
  const LegacyCfg* c;
  int rc = legacy_cfg(&c);
  if (rc) return rc;
  cudaError_t e = cudaMemsetAsync(ctl, 0, offsetof(Ctl, zero_end), s);
  if (e) return e;
  uint32_t nchunk = 0;
  if ((rc = first_pass_chunks(n, &nchunk))) return rc;
  uint32_t* chunk_hist = reinterpret_cast<uint32_t*>(status_buf + kChunkHistOffset);
  // one wave: every CTA resident (a second partial wave would run alone)
  // the same number of chunks per CTA everywhere (every CTA resident)
  const uint64_t per = ceil_div(nchunk, uint64_t(c->sms) * c->occ_hist);
  const int grid = int(umax<uint64_t>(1, ceil_div(nchunk, per)));
  k_hist<<<grid, kHistCtaThreads, 0, s>>>(keys, n, ctl, chunk_hist, nchunk);
  PlanArgs pa;
  pa.keys = keys;
  pa.n = n;
  pa.ctl = ctl;
  pa.epoch_counter = reinterpret_cast<uint32_t*>(status_buf);
  pa.tile_group = reinterpret_cast<uint32_t*>(status_buf + kTgOffset);
  pa.allow_compact = allow_compact;
  pa.hist_hi_grid = c->sms * 2;
  k_plan_scan<<<kWideBuckets / 32, 1024, 0, s>>>(pa, chunk_hist,
                                                  reinterpret_cast<uint32_t*>(status_buf + kChunkOffOffset), nchunk);
  return cudaGetLastError();
}

static SortArgs sort_args(uint64_t n, Ctl* ctl, char* status_buf) {
  SortArgs a{};
  a.n = n;
  a.ctl = ctl;
  a.chunk_off = reinterpret_cast<const uint32_t*>(status_buf + kChunkOffOffset);
  first_pass_chunks(n, &a.nchunk);
  a.status = reinterpret_cast<uint64_t*>(status_buf + kStatusOffset);
  a.gb = reinterpret_cast<uint32_t*>(status_buf + kGbOffset);
  a.tile_group = reinterpret_cast<uint32_t*>(status_buf + kTgOffset);
  return a;
}

static int launch_sort(const SortArgs& a, int legacy, cudaStream_t s) {
  const LegacyCfg* c;
  int rc = legacy_cfg(&c);
  if (rc) return rc;
  const int gb = int(umin<uint64_t>(ceil_div(a.n, kLegacyByteTile), uint64_t(c->sms) * c->occ_byte));
  const int gw = int(umin<uint64_t>(ceil_div(a.n, kLegacyWideTile), uint64_t(c->sms) * c->occ_wide));
  return launch_sort_dispatch(a, legacy, gb, gw, s);
}

}  // namespace ndx

using namespace ndx;

extern "C" {

size_t ndx_wah_ctl_bytes(void) { return (sizeof(Ctl) + 255) & ~size_t(255); }

size_t ndx_wah_status_bytes(uint64_t n) { return status_bytes(n); }

int ndx_wah_plan(const uint32_t* d_keys, uint64_t n, void* d_ctl, void* d_status, void* stream) {
  if (!d_keys || !d_ctl || !d_status || n == 0) return NDX_E_INVALID;
  if (n >= kMaxValues) return NDX_E_TOO_LARGE;
  return launch_plan(d_keys, n, static_cast<Ctl*>(d_ctl), static_cast<char*>(d_status), 1,
                     static_cast<cudaStream_t>(stream));
}

int ndx_wah_sort(const uint32_t* d_keys, uint64_t n, uint32_t row_base, void* d_ctl, uint64_t* d_pairs,
                 uint64_t* d_tmp_pairs, void* d_status, void* stream) {
  if (!d_keys || !d_ctl || !d_pairs || !d_tmp_pairs || !d_status || n == 0) return NDX_E_INVALID;
  if (n >= kMaxValues) return NDX_E_TOO_LARGE;
  if (uint64_t(row_base) + n > (1ull << 32)) return NDX_E_TOO_LARGE;  // row ids are u32
  SortArgs a = sort_args(n, static_cast<Ctl*>(d_ctl), static_cast<char*>(d_status));
  a.in_keys = d_keys;
  a.X = d_pairs;
  a.Y = d_tmp_pairs;
  a.row_base = row_base;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int rc = launch_sort(a, 0, s);
  if (rc) return rc;
  k_vs<<<kVsBlocks, kVsThreads, 0, s>>>(a.ctl, n, row_base);
  return cudaGetLastError();
}

static size_t round256(size_t b) { return (b + 255) & ~size_t(255); }

size_t ndx_sort_pairs_scratch_bytes(uint64_t n) {
  // ctl | X pairs | Y pairs | copies of the input | statuses, each 256-aligned
  return ndx_wah_ctl_bytes() + 2 * round256(size_t(n) * 8) + 2 * round256(size_t(n) * 4) + status_bytes(n) + 256;
}

// sort_pairs: stable sort of SoA (keys, payloads) in place.  The input is
// copied aside so the last pass can scatter into the caller's buffers; the
// status region is cleared per call (this entry point is not the hot path).
int ndx_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_payloads, uint64_t n, void* d_scratch, void* stream) {
  if (n == 0) return 0;
  if (!d_keys || !d_payloads || !d_scratch) return NDX_E_INVALID;
  if (n >= kMaxValues) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(d_scratch) + 255) & ~uintptr_t(255));
  Ctl* ctl = reinterpret_cast<Ctl*>(p);
  p += ndx_wah_ctl_bytes();
  uint64_t* X = reinterpret_cast<uint64_t*>(p);
  p += round256(size_t(n) * 8);
  uint64_t* Y = reinterpret_cast<uint64_t*>(p);
  p += round256(size_t(n) * 8);
  uint32_t* ck = reinterpret_cast<uint32_t*>(p);
  p += round256(size_t(n) * 4);
  uint32_t* cp = reinterpret_cast<uint32_t*>(p);
  p += round256(size_t(n) * 4);
  char* status = p;
  cudaError_t e;
  if ((e = cudaMemsetAsync(status, 0, status_bytes(n), s))) return e;
  if ((e = cudaMemcpyAsync(ck, d_keys, n * 4, cudaMemcpyDeviceToDevice, s))) return e;
  if ((e = cudaMemcpyAsync(cp, d_payloads, n * 4, cudaMemcpyDeviceToDevice, s))) return e;
  int rc = launch_plan(ck, n, ctl, status, 0, s);
  if (rc) return rc;
  SortArgs a = sort_args(n, ctl, status);
  a.in_keys = ck;
  a.in_payloads = cp;
  a.X = X;
  a.Y = Y;
  a.out_keys = d_keys;
  a.out_payloads = d_payloads;
  return launch_sort(a, 1, s);
}

}  // extern "C"
