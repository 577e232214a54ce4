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
//   S2  k_onesweep<BITS>  persistent onesweep-style stable scatter: warp
//                 ballot-match ranking, per-warp smem digit counters, a
//                 decoupled look-back across tiles per digit, smem-staged
//                 reordering so global stores are runs of consecutive pairs.
//                 The first pass synthesises row ids (no iota buffer).
//                 Every pass kernel is launched unconditionally and exits at
//                 once when the plan does not need it (no host sync).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../../include/ndx.h"
#include "common.cuh"
#include "wah_internal.cuh"

namespace ndx {

// ------------------------------------------------------------------ S1 ----

constexpr int kHistThreads = 1024;

__device__ __forceinline__ void hist_one(uint32_t k, uint32_t* h0, uint32_t* h1,
                                         uint32_t* hw, uint32_t& mx,
                                         uint32_t& mxn) {
  mx = max(mx, k);
  mxn = max(mxn, ~k);
  atomicAdd(&h0[k & 255u], 1u);
  atomicAdd(&h1[(k >> 8) & 255u], 1u);
  atomicAdd(&hw[k & (kWideBuckets - 1)], 1u);
}

__global__ __launch_bounds__(kHistThreads) void k_hist(const uint32_t* __restrict__ keys,
                                                       uint64_t n, Ctl* ctl) {
  __shared__ uint32_t h0[256], h1[256], hw[kWideBuckets];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h0[i] = h1[i] = 0;
  for (int i = threadIdx.x; i < kWideBuckets; i += blockDim.x) hw[i] = 0;
  __syncthreads();

  uint32_t mx = 0, mxn = 0;
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(keys) & 15u) == 0) {
    const uint64_t nq = n / 4;
    const uint4* q = reinterpret_cast<const uint4*>(keys);
    for (uint64_t i = tid; i < nq; i += stride) {
      uint4 v = ldg_stream4(q + i);
      hist_one(v.x, h0, h1, hw, mx, mxn);
      hist_one(v.y, h0, h1, hw, mx, mxn);
      hist_one(v.z, h0, h1, hw, mx, mxn);
      hist_one(v.w, h0, h1, hw, mx, mxn);
    }
    for (uint64_t i = nq * 4 + tid; i < n; i += stride)
      hist_one(keys[i], h0, h1, hw, mx, mxn);
  } else {
    for (uint64_t i = tid; i < n; i += stride) hist_one(keys[i], h0, h1, hw, mx, mxn);
  }
  // warp-reduce the range, one atomic per warp
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
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    if (h0[i]) atomicAdd(&ctl->hist_byte[0][i], h0[i]);
    if (h1[i]) atomicAdd(&ctl->hist_byte[1][i], h1[i]);
  }
  for (int i = threadIdx.x; i < kWideBuckets; i += blockDim.x)
    if (hw[i]) atomicAdd(&ctl->hist_wide[i], hw[i]);
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

// stage 0: after k_hist; stage 1: after k_hist_hi (no-op unless pending).
__global__ __launch_bounds__(1024) void k_plan(Ctl* ctl, uint64_t n, int stage) {
  SortPlan& p = ctl->plan;
  if (stage == 1) {
    if (p.complete) return;
    plan_bytes(ctl, n, 4);
    return;
  }
  __shared__ uint32_t s_mode;
  __shared__ uint32_t rot[kWideBuckets];
  const uint32_t mn = ~ctl->max_not, mx = ctl->max_seen;
  if (threadIdx.x == 0) {
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
    } else {
      p.mode = kModeBytes;
      p.need_hi = (mn >> 16) != (mx >> 16);
      p.complete = !p.need_hi;
    }
    s_mode = p.mode;
  }
  __syncthreads();
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

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortIPT = 16;                          // items per thread
constexpr int kSortWarpItems = 32 * kSortIPT;         // 512
constexpr int kSortTile = kSortThreads * kSortIPT;    // 4096 pairs

template <int MAXB>
struct SortSmem {
  static constexpr int NB = 1 << MAXB;
  static constexpr size_t kHBytes = size_t(kSortWarps) * NB * sizeof(uint16_t);
  static constexpr size_t kSBytes = size_t(kSortTile) * sizeof(uint64_t);
  static constexpr size_t kUnion = kHBytes > kSBytes ? kHBytes : kSBytes;
  static constexpr size_t kBytes = kUnion + 3 * NB * sizeof(uint32_t) + 16;
};

struct SortArgs {
  const uint32_t* in_keys;      // first pass: keys (SoA)
  const uint32_t* in_payloads;  // first pass: payloads, or null -> rows synthesised
  uint64_t* X;                  // final AoS output (or ping buffer)
  uint64_t* Y;                  // pong buffer
  uint32_t* out_keys;           // non-null: last pass writes SoA here
  uint32_t* out_payloads;
  uint64_t n;
  uint32_t row_base;
  Ctl* ctl;
  uint64_t* status;             // look-back statuses, >= tiles * 2048 words
  uint32_t epoch;
};

__device__ __forceinline__ uint64_t pack_pair(uint32_t key, uint32_t payload) {
  return uint64_t(key) | (uint64_t(payload) << 32);
}

// which = -1: the wide single pass; which = 0..3: the byte-k pass.
//
// Per tile: load -> tile histogram (smem atomics) -> publish the per-digit
// aggregates ("early counts", so successors rarely wait) -> stable warp
// ranking -> look-back per digit -> stage the tile in digit order in smem ->
// scatter runs of consecutive pairs.
template <int MAXB>
__global__ __launch_bounds__(kSortThreads, 3) void k_onesweep(SortArgs a, int which) {
  const SortPlan& pl = a.ctl->plan;
  uint32_t shift, bits, base;
  int p, P;
  const uint32_t* bstart;
  if (which < 0) {
    if (pl.mode != kModeWide) return;
    p = 0;
    P = 1;
    shift = 0;
    bits = pl.wide_bits;
    base = pl.base;
    bstart = pl.bucket_start_wide;
  } else {
    if (pl.mode != kModeBytes || !pl.byte_active[which]) return;
    p = pl.byte_order[which];
    P = pl.npasses;
    shift = 8u * which;
    bits = 8;
    base = 0;
    bstart = pl.bucket_start_byte[which];
  }
  const uint32_t nb = 1u << bits;
  const uint32_t dmask = nb - 1;
  const uint32_t epoch = a.epoch + uint32_t(which + 2);

  // buffer roles: pass q writes X iff (P-1-q) is even
  const bool first = p == 0, last = p == P - 1;
  const uint64_t* in_pairs = first ? nullptr : (((P - 1 - (p - 1)) & 1) == 0 ? a.X : a.Y);
  uint64_t* out_pairs = ((P - 1 - p) & 1) == 0 ? a.X : a.Y;
  const bool out_soa = last && a.out_keys != nullptr;

  extern __shared__ __align__(16) unsigned char smem[];
  using SM = SortSmem<MAXB>;
  uint16_t* H = reinterpret_cast<uint16_t*>(smem);       // [warps][NB]
  uint64_t* S = reinterpret_cast<uint64_t*>(smem);       // [tile] (aliases H)
  uint32_t* bh = reinterpret_cast<uint32_t*>(smem + SM::kUnion);  // tile histogram
  uint32_t* tile_excl = bh + SM::NB;
  uint32_t* gbase = tile_excl + SM::NB;
  uint32_t* s_tile = gbase + SM::NB;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t n = a.n;
  const uint64_t ntiles = (n + kSortTile - 1) / kSortTile;
  uint32_t* ctr = &a.ctl->tile_ctr[which + 2];  // [0] emit, [1] wide, [2..5] bytes
  uint16_t* Hw = H + warp * SM::NB;

  for (;;) {
    if (threadIdx.x == 0) *s_tile = atomicAdd(ctr, 1u);
    for (uint32_t d = lane; d < nb; d += 32) Hw[d] = 0;
    for (uint32_t d = threadIdx.x; d < nb; d += kSortThreads) bh[d] = 0;
    __syncthreads();
    const uint64_t tile = *s_tile;
    if (tile >= ntiles) break;
    const uint64_t tile_start = tile * kSortTile;
    const uint32_t tile_n = uint32_t(umin<uint64_t>(kSortTile, n - tile_start));
    const uint64_t wbase = tile_start + uint64_t(warp) * kSortWarpItems;

    // ---- load (warp-striped: round r, lane l -> element wbase + 32 r + l)
    uint32_t key[kSortIPT], pay[kSortIPT];
#pragma unroll
    for (int r = 0; r < kSortIPT; ++r) {
      const uint64_t i = wbase + uint64_t(r) * 32 + lane;
      if (i < n) {
        if (first) {
          key[r] = ldg_stream(a.in_keys + i);
          pay[r] = a.in_payloads ? ldg_stream(a.in_payloads + i) : a.row_base + uint32_t(i);
        } else {
          uint64_t e = ldg_stream(in_pairs + i);
          key[r] = uint32_t(e);
          pay[r] = uint32_t(e >> 32);
        }
      } else {
        key[r] = 0;
        pay[r] = 0;
      }
    }

    // ---- early counts: tile histogram, published before the heavy ranking
#pragma unroll
    for (int r = 0; r < kSortIPT; ++r) {
      const uint64_t i = wbase + uint64_t(r) * 32 + lane;
      if (i < n) atomicAdd(&bh[((key[r] - base) >> shift) & dmask], 1u);
    }
    __syncthreads();
    uint64_t* st = a.status + tile * nb;
    for (uint32_t d = threadIdx.x; d < nb; d += kSortThreads)
      st_relaxed_u64(&st[d], status_word(epoch, tile == 0 ? kFlagPrefix : kFlagAgg, bh[d]));

    // ---- rank: stable within the warp (lane order == row order per round)
    uint32_t rank[kSortIPT];
#pragma unroll
    for (int r = 0; r < kSortIPT; ++r) {
      const uint64_t i = wbase + uint64_t(r) * 32 + lane;
      const bool valid = i < n;
      const unsigned vmask = __ballot_sync(kFull, valid);
      const uint32_t d = ((key[r] - base) >> shift) & dmask;
      unsigned peers = vmask;
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        if (b < int(bits)) {
          unsigned bit = (d >> b) & 1u;
          unsigned bal = __ballot_sync(kFull, bit);
          peers &= bit ? bal : ~bal;
        }
      }
      const int leader = valid ? __ffs(peers) - 1 : lane;
      uint32_t old = 0;
      if (valid && lane == leader) old = Hw[d];
      old = __shfl_sync(kFull, old, leader);
      if (valid && lane == leader) Hw[d] = uint16_t(old + __popc(peers));
      rank[r] = old + __popc(peers & lanemask_lt());
      __syncwarp();
    }
    __syncthreads();

    // ---- per digit: warp offsets; tile-local digit offsets
    for (uint32_t d = threadIdx.x; d < nb; d += kSortThreads) {
      uint32_t sum = 0;
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        uint32_t c = H[w * SM::NB + d];
        H[w * SM::NB + d] = uint16_t(sum);
        sum += c;
      }
    }
    block_excl_scan(bh, tile_excl, int(nb));  // ends with __syncthreads

    // ---- decoupled look-back per digit
    for (uint32_t d = threadIdx.x; d < nb; d += kSortThreads) {
      const uint32_t cnt = bh[d];
      uint64_t excl = 0;
      if (tile > 0) {
        int64_t t = int64_t(tile) - 1;
        for (;;) {
          uint64_t s = ld_relaxed_u64(&a.status[uint64_t(t) * nb + d]);
          while (!status_ready(s, epoch)) {
            __nanosleep(20);
            s = ld_relaxed_u64(&a.status[uint64_t(t) * nb + d]);
          }
          excl += s & kValueMask;
          if (status_is_prefix(s)) break;
          --t;
        }
        st_relaxed_u64(&st[d], status_word(epoch, kFlagPrefix, excl + cnt));
      }
      gbase[d] = bstart[d] + uint32_t(excl) - tile_excl[d];
    }
    __syncthreads();

    // ---- local (in-tile) positions, then stage the tile in smem
#pragma unroll
    for (int r = 0; r < kSortIPT; ++r) {
      const uint32_t d = ((key[r] - base) >> shift) & dmask;
      rank[r] += tile_excl[d] + Hw[d];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortIPT; ++r) {
      const uint64_t i = wbase + uint64_t(r) * 32 + lane;
      if (i < n) S[rank[r]] = pack_pair(key[r], pay[r]);
    }
    __syncthreads();

    // ---- scatter: consecutive local slots of one digit are consecutive globally
    for (uint32_t j = threadIdx.x; j < tile_n; j += kSortThreads) {
      const uint64_t e = S[j];
      const uint32_t k = uint32_t(e);
      const uint32_t d = ((k - base) >> shift) & dmask;
      const uint32_t pos = gbase[d] + j;
      if (out_soa) {
        a.out_keys[pos] = k;
        a.out_payloads[pos] = uint32_t(e >> 32);
      } else {
        out_pairs[pos] = e;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host --

struct LaunchCfg {
  int sms = 0;
  int occ_wide = 1, occ_byte = 1;
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
    size_t sw = SortSmem<kWideMaxBits>::kBytes, sb = SortSmem<8>::kBytes;
    if ((e = cudaFuncSetAttribute(k_onesweep<kWideMaxBits>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(sw))))
      return e;
    if ((e = cudaFuncSetAttribute(k_onesweep<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sb))))
      return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_wide, k_onesweep<kWideMaxBits>,
                                                           kSortThreads, sw)))
      return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_byte, k_onesweep<8>,
                                                           kSortThreads, sb)))
      return e;
    if (c.occ_wide < 1) c.occ_wide = 1;
    if (c.occ_byte < 1) c.occ_byte = 1;
    c.ready = true;
  }
  *out = &c;
  return 0;
}

static uint64_t sort_tiles(uint64_t n) { return (n + kSortTile - 1) / kSortTile; }

}  // namespace ndx

using namespace ndx;

extern "C" {

size_t ndx_wah_ctl_bytes(void) { return (sizeof(Ctl) + 255) & ~size_t(255); }

size_t ndx_wah_sort_scratch_bytes(uint64_t n) {
  // look-back statuses (tiles x 2048 u64) + one pong buffer of pairs
  size_t st = size_t(sort_tiles(n)) * kWideBuckets * sizeof(uint64_t);
  st = (st + 255) & ~size_t(255);
  return st + size_t(n) * sizeof(uint64_t) + 256;
}

int ndx_wah_plan(const uint32_t* d_keys, uint64_t n, void* d_ctl, void* stream) {
  if (!d_keys || !d_ctl || n == 0) return NDX_E_INVALID;
  if (n >= (1ull << 31)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LaunchCfg* c;
  int rc = launch_cfg(&c);
  if (rc) return rc;
  Ctl* ctl = static_cast<Ctl*>(d_ctl);
  cudaError_t e = cudaMemsetAsync(ctl, 0, offsetof(Ctl, zero_end), s);
  if (e) return e;
  const uint64_t want = (n + 4ull * kHistThreads * 8 - 1) / (4ull * kHistThreads * 8);
  const int grid = int(umin<uint64_t>(uint64_t(c->sms) * 2, umax<uint64_t>(want, 1)));
  k_hist<<<grid, kHistThreads, 0, s>>>(d_keys, n, ctl);
  k_plan<<<1, 1024, 0, s>>>(ctl, n, 0);
  k_hist_hi<<<grid, kHistThreads, 0, s>>>(d_keys, n, ctl);
  k_plan<<<1, 1024, 0, s>>>(ctl, n, 1);
  return cudaGetLastError();
}

int ndx_wah_sort(const uint32_t* d_keys, uint64_t n, uint32_t row_base, void* d_ctl,
                 uint64_t* d_pairs, void* d_scratch, uint32_t epoch, void* stream) {
  if (!d_keys || !d_ctl || !d_pairs || !d_scratch || n == 0) return NDX_E_INVALID;
  if (n >= (1ull << 31)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LaunchCfg* c;
  int rc = launch_cfg(&c);
  if (rc) return rc;
  const uint64_t tiles = sort_tiles(n);
  size_t st = (size_t(tiles) * kWideBuckets * sizeof(uint64_t) + 255) & ~size_t(255);
  SortArgs a{};
  a.in_keys = d_keys;
  a.in_payloads = nullptr;
  a.X = d_pairs;
  a.Y = reinterpret_cast<uint64_t*>(static_cast<char*>(d_scratch) + st);
  a.n = n;
  a.row_base = row_base;
  a.ctl = static_cast<Ctl*>(d_ctl);
  a.status = static_cast<uint64_t*>(d_scratch);
  a.epoch = epoch;
  const int gw = int(umin<uint64_t>(tiles, uint64_t(c->sms) * c->occ_wide));
  const int gb = int(umin<uint64_t>(tiles, uint64_t(c->sms) * c->occ_byte));
  k_onesweep<kWideMaxBits><<<gw, kSortThreads, SortSmem<kWideMaxBits>::kBytes, s>>>(a, -1);
  for (int k = 0; k < 4; ++k)
    k_onesweep<8><<<gb, kSortThreads, SortSmem<8>::kBytes, s>>>(a, k);
  return cudaGetLastError();
}

size_t ndx_sort_pairs_scratch_bytes(uint64_t n) {
  // ctl + statuses + pong pairs + ping pairs + SoA copies of the input
  return ndx_wah_ctl_bytes() + ndx_wah_sort_scratch_bytes(n) + size_t(n) * 16 + 512;
}

// sort_pairs: stable sort of SoA (keys, payloads) in place.  The input is
// copied aside first so the last pass can scatter into the caller's buffers.
int ndx_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_payloads, uint64_t n, void* d_scratch,
                       uint32_t epoch, void* stream) {
  if (n == 0) return 0;
  if (!d_keys || !d_payloads || !d_scratch) return NDX_E_INVALID;
  if (n >= (1ull << 31)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LaunchCfg* c;
  int rc = launch_cfg(&c);
  if (rc) return rc;
  char* base = static_cast<char*>(d_scratch);
  Ctl* ctl = reinterpret_cast<Ctl*>(base);
  char* sort_scr = base + ndx_wah_ctl_bytes();
  const uint64_t tiles = sort_tiles(n);
  size_t st = (size_t(tiles) * kWideBuckets * sizeof(uint64_t) + 255) & ~size_t(255);
  uint64_t* Y = reinterpret_cast<uint64_t*>(sort_scr + st);
  uint64_t* X = Y + n;
  uint32_t* ck = reinterpret_cast<uint32_t*>(X + n);
  uint32_t* cp = ck + n;
  cudaError_t e;
  if ((e = cudaMemcpyAsync(ck, d_keys, n * 4, cudaMemcpyDeviceToDevice, s))) return e;
  if ((e = cudaMemcpyAsync(cp, d_payloads, n * 4, cudaMemcpyDeviceToDevice, s))) return e;
  if ((rc = ndx_wah_plan(ck, n, ctl, stream))) return rc;
  SortArgs a{};
  a.in_keys = ck;
  a.in_payloads = cp;
  a.X = X;
  a.Y = Y;
  a.out_keys = d_keys;
  a.out_payloads = d_payloads;
  a.n = n;
  a.ctl = ctl;
  a.status = reinterpret_cast<uint64_t*>(sort_scr);
  a.epoch = epoch;
  const int gw = int(umin<uint64_t>(tiles, uint64_t(c->sms) * c->occ_wide));
  const int gb = int(umin<uint64_t>(tiles, uint64_t(c->sms) * c->occ_byte));
  k_onesweep<kWideMaxBits><<<gw, kSortThreads, SortSmem<kWideMaxBits>::kBytes, s>>>(a, -1);
  for (int k = 0; k < 4; ++k)
    k_onesweep<8><<<gb, kSortThreads, SortSmem<8>::kBytes, s>>>(a, k);
  return cudaGetLastError();
}

}  // extern "C"
