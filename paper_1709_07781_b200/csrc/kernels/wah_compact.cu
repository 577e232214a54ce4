// The reference's device primitives behind its public WAH API, on sm_100a:
//   * the three compaction stages of the paper's Listing 5
//     (p/core/src/wah_stages.cpp:29-163): prepare / count / move,
//   * scan_exclusive (p/core/src/wah_scan.cpp:14-95),
//   * the one-warp increment used by the dispatch-overhead probe.
//
// move and scan are single-pass decoupled look-back kernels: the reference's
// move sums all earlier tile counts serially in every tile (O(T^2),
// wah_stages.cpp:117) and its scan recurses over block totals.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../../include/ndx.h"
#include "common.cuh"

namespace ndx {

constexpr uint32_t kStageTile = 4096;  // wah_stages.cpp:11 (counts are per tile)
constexpr int kCThreads = 256;
constexpr int kCWarps = kCThreads / 32;

// prepare: out[2i] = a[i], out[2i+1] = b[i]; cfg[1] = 2k (wah_stages.cpp:36-46).
__global__ void k_prepare(uint32_t* __restrict__ cfg, const uint32_t* __restrict__ a,
                          const uint32_t* __restrict__ b, uint64_t k,
                          uint32_t* __restrict__ out) {
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  if (tid == 0) cfg[1] = uint32_t(2 * k);
  const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                     reinterpret_cast<uintptr_t>(out)) & 15u) == 0;
  uint64_t done = 0;
  if (vec) {
    const uint64_t kq = k / 4;
    for (uint64_t q = tid; q < kq; q += stride) {
      const uint4 x = ldg_stream4(reinterpret_cast<const uint4*>(a) + q);
      const uint4 y = ldg_stream4(reinterpret_cast<const uint4*>(b) + q);
      uint4* o = reinterpret_cast<uint4*>(out) + 2 * q;
      o[0] = make_uint4(x.x, y.x, x.y, y.y);
      o[1] = make_uint4(x.z, y.z, x.w, y.w);
    }
    done = kq * 4;
  }
  for (uint64_t i = done + tid; i < k; i += stride) {
    out[2 * i] = a[i];
    out[2 * i + 1] = b[i];
  }
}

// count: nonzeros per 4096-element tile (wah_stages.cpp:61-80).
__global__ __launch_bounds__(kCThreads) void k_count(const uint32_t* __restrict__ data,
                                                     uint64_t n, uint32_t* __restrict__ counts,
                                                     uint64_t tiles) {
  __shared__ uint32_t wsum[kCWarps];
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint64_t base = t * kStageTile;
    uint32_t c = 0;
    for (uint32_t j = threadIdx.x; j < kStageTile; j += kCThreads) {
      const uint64_t i = base + j;
      if (i < n && ldg_stream(data + i) != 0) ++c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int w = 0; w < kCWarps; ++w) s += wsum[w];
      counts[t] = s;
    }
    __syncthreads();
  }
}

// Decoupled look-back over per-tile u32 sums (mod 2^32); returns the
// exclusive prefix of `tile` to every thread of warp 0.
__device__ uint32_t lookback_u32(uint64_t* status, uint64_t tile, uint32_t agg,
                                 uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  uint32_t excl = 0;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(&status[0], status_word(epoch, kFlagPrefix, agg));
    return 0;
  }
  if (lane == 0) st_relaxed_u64(&status[tile], status_word(epoch, kFlagAgg, agg));
  int64_t base = int64_t(tile) - 1;
  for (;;) {
    const int64_t tt = base - lane;
    uint32_t val = 0;
    bool pre = true;
    if (tt >= 0) {
      uint64_t s;
      do {
        s = ld_relaxed_u64(&status[tt]);
      } while (!status_ready(s, epoch));
      pre = status_is_prefix(s);
      val = uint32_t(s & 0xffffffffull);
    }
    const unsigned pm = __ballot_sync(kFull, pre);
    if (pm && lane > __ffs(pm) - 1) val = 0;
    excl += __shfl_sync(kFull, warp_incl_sum(val), 31);
    if (pm) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed_u64(&status[tile], status_word(epoch, kFlagPrefix, excl + agg));
  return excl;
}

// move: order-preserving scatter of the nonzeros; cfg[1] = total
// (wah_stages.cpp:97-156).  Tile aggregates come from `counts`.
__global__ __launch_bounds__(kCThreads) void k_move(uint32_t* __restrict__ cfg,
                                                    const uint32_t* __restrict__ data, uint64_t n,
                                                    const uint32_t* __restrict__ counts,
                                                    uint32_t* __restrict__ out, uint64_t tiles,
                                                    uint64_t* status, uint32_t* tile_ctr,
                                                    uint32_t epoch) {
  __shared__ uint32_t wtot[kCWarps];
  __shared__ uint32_t s_tile, s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= tiles) break;
    const uint64_t wb = tile * kStageTile + uint64_t(warp) * (kStageTile / kCWarps);
    uint32_t v[kStageTile / kCThreads];
    uint32_t ex[kStageTile / kCThreads];
    uint32_t run = 0;
#pragma unroll
    for (int r = 0; r < int(kStageTile / kCThreads); ++r) {
      const uint64_t i = wb + uint64_t(r) * 32 + lane;
      v[r] = i < n ? ldg_stream(data + i) : 0u;
      const unsigned m = __ballot_sync(kFull, v[r] != 0);
      ex[r] = run + __popc(m & lanemask_lt());
      run += __popc(m);
    }
    if (lane == 0) wtot[warp] = run;
    __syncthreads();
    if (warp == 0) {
      const uint32_t t = lane < kCWarps ? wtot[lane] : 0;
      const uint32_t ti = warp_incl_sum(t);
      if (lane < kCWarps) wtot[lane] = ti - t;
      const uint32_t agg = counts[tile];
      const uint32_t excl = lookback_u32(status, tile, agg, epoch);
      if (lane == 0) {
        s_base = excl;
        if (tile == tiles - 1) cfg[1] = excl + agg;
      }
    }
    __syncthreads();
    const uint32_t b = s_base + wtot[warp];
#pragma unroll
    for (int r = 0; r < int(kStageTile / kCThreads); ++r)
      if (v[r] != 0) out[b + ex[r]] = v[r];
    __syncthreads();
  }
}

// scan_exclusive over u32 with wrap-around (wah_scan.cpp:14-95).
__global__ __launch_bounds__(kCThreads) void k_scan(const uint32_t* __restrict__ in,
                                                    uint32_t* __restrict__ out, uint64_t n,
                                                    uint64_t tiles, uint64_t* status,
                                                    uint32_t* tile_ctr, uint32_t epoch) {
  __shared__ uint32_t wtot[kCWarps];
  __shared__ uint32_t s_tile, s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= tiles) break;
    const uint64_t wb = tile * kStageTile + uint64_t(warp) * (kStageTile / kCWarps);
    uint32_t ex[kStageTile / kCThreads];
    uint32_t run = 0;
#pragma unroll
    for (int r = 0; r < int(kStageTile / kCThreads); ++r) {
      const uint64_t i = wb + uint64_t(r) * 32 + lane;
      const uint32_t x = i < n ? ldg_stream(in + i) : 0u;
      const uint32_t incl = warp_incl_sum(x);
      ex[r] = run + incl - x;
      run += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) wtot[warp] = run;
    __syncthreads();
    if (warp == 0) {
      const uint32_t t = lane < kCWarps ? wtot[lane] : 0;
      const uint32_t ti = warp_incl_sum(t);
      if (lane < kCWarps) wtot[lane] = ti - t;
      const uint32_t agg = __shfl_sync(kFull, ti, 31);
      const uint32_t excl = lookback_u32(status, tile, agg, epoch);
      if (lane == 0) s_base = excl;
    }
    __syncthreads();
    const uint32_t b = s_base + wtot[warp];
#pragma unroll
    for (int r = 0; r < int(kStageTile / kCThreads); ++r) {
      const uint64_t i = wb + uint64_t(r) * 32 + lane;
      if (i < n) out[i] = b + ex[r];
    }
    __syncthreads();
  }
}

__global__ void k_tiny_increment(uint32_t* p) {
  if (threadIdx.x == 0) p[0] += 1u;
}

static int sms_now(int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  return cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
}

static uint64_t stage_tiles(uint64_t n) { return (n + kStageTile - 1) / kStageTile; }

}  // namespace ndx

using namespace ndx;

extern "C" {

int ndx_compact_prepare(uint32_t* d_cfg, const uint32_t* d_a, const uint32_t* d_b, uint64_t k,
                        uint32_t* d_out, void* stream) {
  if (!d_cfg || (k && (!d_a || !d_b || !d_out))) return NDX_E_INVALID;
  int sms = 0;
  int rc = sms_now(&sms);
  if (rc) return rc;
  const int grid = int(umin<uint64_t>((k / 4 + 255) / 256 + 1, uint64_t(sms) * 8));
  k_prepare<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_cfg, d_a, d_b, k, d_out);
  return cudaGetLastError();
}

int ndx_compact_count(const uint32_t* d_data, uint64_t n, uint32_t* d_counts, void* stream) {
  if (!d_counts || (n && !d_data)) return NDX_E_INVALID;
  int sms = 0;
  int rc = sms_now(&sms);
  if (rc) return rc;
  const uint64_t tiles = stage_tiles(n > 0 ? n : 1);
  const int grid = int(umin<uint64_t>(tiles, uint64_t(sms) * 8));
  k_count<<<grid, kCThreads, 0, static_cast<cudaStream_t>(stream)>>>(d_data, n, d_counts, tiles);
  return cudaGetLastError();
}

size_t ndx_compact_move_scratch_bytes(uint64_t n) {
  return size_t(stage_tiles(n > 0 ? n : 1) + 1) * 8 + 256;
}

int ndx_compact_move(uint32_t* d_cfg, const uint32_t* d_data, uint64_t n,
                     const uint32_t* d_counts, uint32_t* d_out, void* d_scratch, void* stream) {
  if (!d_cfg || !d_counts || !d_scratch || (n && (!d_data || !d_out))) return NDX_E_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int sms = 0;
  int rc = sms_now(&sms);
  if (rc) return rc;
  const uint64_t tiles = stage_tiles(n > 0 ? n : 1);
  uint32_t* ctr = reinterpret_cast<uint32_t*>(static_cast<char*>(d_scratch));
  uint64_t* status = reinterpret_cast<uint64_t*>(static_cast<char*>(d_scratch) + 256);
  // counter + statuses cleared per call (status epoch 1 then means "this call")
  cudaError_t e = cudaMemsetAsync(ctr, 0, 256 + tiles * 8, s);
  if (e) return e;
  const int grid = int(umin<uint64_t>(tiles, uint64_t(sms) * 8));
  k_move<<<grid, kCThreads, 0, s>>>(d_cfg, d_data, n, d_counts, d_out, tiles, status, ctr, 1u);
  return cudaGetLastError();
}

size_t ndx_scan_scratch_bytes(uint64_t n) { return size_t(stage_tiles(n) + 1) * 8 + 256; }

int ndx_scan_exclusive_u32(const uint32_t* d_in, uint32_t* d_out, uint64_t n, void* d_scratch,
                           void* stream) {
  if (n == 0) return 0;
  if (!d_in || !d_out || !d_scratch) return NDX_E_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int sms = 0;
  int rc = sms_now(&sms);
  if (rc) return rc;
  const uint64_t tiles = stage_tiles(n);
  uint32_t* ctr = reinterpret_cast<uint32_t*>(static_cast<char*>(d_scratch));
  uint64_t* status = reinterpret_cast<uint64_t*>(static_cast<char*>(d_scratch) + 256);
  cudaError_t e = cudaMemsetAsync(ctr, 0, 256 + tiles * 8, s);
  if (e) return e;
  const int grid = int(umin<uint64_t>(tiles, uint64_t(sms) * 8));
  k_scan<<<grid, kCThreads, 0, s>>>(d_in, d_out, n, tiles, status, ctr, 1u);
  return cudaGetLastError();
}

int ndx_tiny_increment(uint32_t* d_p, void* stream) {
  if (!d_p) return NDX_E_INVALID;
  k_tiny_increment<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(d_p);
  return cudaGetLastError();
}

}  // extern "C"
