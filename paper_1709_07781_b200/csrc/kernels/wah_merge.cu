// Multi-GPU build: per-shard metadata and the final word assembly
// (SURVEY.md section 8(e), Appendix B).
//
// Shard g builds rows [S_g, S_{g+1}) with S_g = 0 (mod 31) and global row
// ids (row_base = S_g), so no 31-row chunk straddles two shards and each
// local index is canonical except for its leading zero-fill.  The merge only
// touches the ends of each value's piece:
//   * the local leading zero-fill is replaced by the cross-shard gap fill
//     (or dropped / kept for the first piece),
//   * ones-fills that meet at gap 0 are fused into one.
// The planning over the (small) metadata runs on the device (wah_plan.cu)
// or on the host (csrc/runtime/wah_shard.cpp); these kernels do the
// per-value metadata and the copy of every piece to its final position.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../../include/ndx.h"
#include "common.cuh"
#include "wah_internal.cuh"

namespace ndx {

__device__ __forceinline__ uint32_t fill_chunks(uint32_t w) { return w & kLenMask; }
__device__ __forceinline__ bool is_zero_fill(uint32_t w) { return (w & 0xC0000000u) == kFillFlag; }
__device__ __forceinline__ bool is_ones_fill(uint32_t w) { return (w & 0xC0000000u) == 0xC0000000u; }

// First index in pairs[0, n) whose key is >= v (keys ascending).
__device__ __forceinline__ uint64_t lower_key(const uint64_t* pairs, uint64_t n, uint32_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (uint32_t(__ldg(pairs + mid)) < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Metadata of entry d: first / last chunk of the value (from the sorted
// stream: rows form -- the value's rows are [vs[d], vs[d+1]) -- or pairs),
// leading and trailing ones-fill of the body, and the body range (the words
// after the local leading zero-fill).
__device__ __forceinline__ ndx_shard_meta meta_of(const Ctl* ctl, const uint64_t* stream, uint64_t n,
                                                  const uint32_t* __restrict__ entries,
                                                  const uint32_t* __restrict__ words, uint64_t d) {
  const uint32_t v = entries[3 * d], off = entries[3 * d + 1], len = entries[3 * d + 2];
  ndx_shard_meta m;
  m.value = v;
  if (ctl->rows_form) {
    const uint32_t* rows = reinterpret_cast<const uint32_t*>(stream);
    m.f = __ldg(rows + ctl->vs[d]) / kChunkBits;
    m.l = __ldg(rows + ctl->vs[d + 1] - 1) / kChunkBits;
  } else {
    const uint64_t lo = lower_key(stream, n, v);
    const uint64_t hi = v == 0xffffffffu ? n : lower_key(stream, n, v + 1);
    m.f = uint32_t(__ldg(stream + lo) >> 32) / kChunkBits;
    m.l = uint32_t(__ldg(stream + hi - 1) >> 32) / kChunkBits;
  }
  m.skip = is_zero_fill(words[off]) ? 1u : 0u;
  m.body_off = off + m.skip;
  m.body_len = len - m.skip;
  const uint32_t first = words[m.body_off], last = words[m.body_off + m.body_len - 1];
  m.a = is_ones_fill(first) ? fill_chunks(first) : 0u;
  m.z = is_ones_fill(last) ? fill_chunks(last) : 0u;
  return m;
}

// One thread per value of the local index.
__global__ void k_shard_meta(const uint64_t* __restrict__ stream, uint64_t n, const Ctl* ctl,
                             const uint32_t* __restrict__ entries, uint64_t D,
                             const uint32_t* __restrict__ words, ndx_shard_meta* __restrict__ meta) {
  for (uint64_t d = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x)
    meta[d] = meta_of(ctl, stream, n, entries, words, d);
}

// The same with the value count on the device (ctl's ndx_wah_counts) and a
// capacity: at most `cap` records are written (the plan flags a shard whose
// count exceeds it).
__global__ void k_shard_meta_dev(const uint64_t* __restrict__ stream, uint64_t n,
                                 const uint32_t* __restrict__ entries, const Ctl* ctl, uint64_t cap,
                                 const uint32_t* __restrict__ words, ndx_shard_meta* __restrict__ meta) {
  const uint64_t D = umin<uint64_t>(ctl->distinct, cap);
  for (uint64_t d = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x)
    meta[d] = meta_of(ctl, stream, n, entries, words, d);
}

// One warp per piece: the optional lead word, then src_len words copied from
// the piece's shard words (already offset into the staging buffer).
__global__ void k_assemble(const uint32_t* __restrict__ src, const ndx_piece* __restrict__ pieces,
                           uint64_t npieces, uint32_t* __restrict__ out) {
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t p = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; p < npieces; p += warps) {
    const ndx_piece pc = pieces[p];
    uint32_t* dst = out + pc.dst;
    if (pc.lead) {
      if (lane == 0) dst[0] = pc.lead;
      ++dst;
    }
    const uint32_t* s = src + pc.src_off;
    for (uint32_t j = lane; j < pc.src_len; j += 32) dst[j] = __ldg(s + j);
  }
}

}  // namespace ndx

using namespace ndx;

extern "C" {

int ndx_wah_shard_meta(const uint64_t* d_pairs, uint64_t n, const void* d_ctl, const uint32_t* d_entries,
                       uint64_t n_entries, const uint32_t* d_words, ndx_shard_meta* d_meta,
                       void* stream) {
  if (n_entries == 0) return 0;
  if (!d_pairs || !d_ctl || !d_entries || !d_words || !d_meta || n == 0) return NDX_E_INVALID;
  const int grid = int(umin<uint64_t>((n_entries + 255) / 256, 4096));
  k_shard_meta<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_pairs, n, static_cast<const Ctl*>(d_ctl), d_entries, n_entries, d_words, d_meta);
  return cudaGetLastError();
}

int ndx_wah_shard_meta_dev(const uint64_t* d_pairs, uint64_t n, const uint32_t* d_entries,
                           const void* d_ctl, uint64_t cap, const uint32_t* d_words, ndx_shard_meta* d_meta,
                           void* stream) {
  if (!d_pairs || !d_entries || !d_ctl || !d_words || !d_meta || n == 0 || cap == 0) return NDX_E_INVALID;
  const int grid = int(umin<uint64_t>((cap + 255) / 256, 148 * 8));
  k_shard_meta_dev<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_pairs, n, d_entries, static_cast<const Ctl*>(d_ctl), cap, d_words, d_meta);
  return cudaGetLastError();
}

int ndx_wah_assemble(const uint32_t* d_src, const ndx_piece* d_pieces, uint64_t n_pieces,
                     uint32_t* d_out, void* stream) {
  if (n_pieces == 0) return 0;
  if (!d_src || !d_pieces || !d_out) return NDX_E_INVALID;
  const int grid = int(umin<uint64_t>((n_pieces + 7) / 8, 148 * 16));
  k_assemble<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_src, d_pieces, n_pieces, d_out);
  return cudaGetLastError();
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Assembly straight from the device plan: pieces in their plan slots
// (g * stride + i), every shard's words in its own buffer.  One CTA per
// piece, the CTA striding over the piece's words (a hot value's piece spans
// millions of words).
namespace ndx {
namespace {
constexpr int kAsmShards = 64;
struct ShardSrc {
  const uint32_t* src[kAsmShards];
  uint32_t count[kAsmShards];
};
__global__ void __launch_bounds__(512) k_assemble_slots(ShardSrc ss, uint32_t shards, uint32_t stride,
                                                        const ndx_piece* __restrict__ pieces,
                                                        uint32_t* __restrict__ out) {
  const uint64_t slots = uint64_t(shards) * stride;
  for (uint64_t x = blockIdx.x; x < slots; x += gridDim.x) {
    const uint32_t g = uint32_t(x / stride), i = uint32_t(x % stride);
    if (i >= ss.count[g]) continue;
    const ndx_piece pc = pieces[x];
    uint32_t* dst = out + pc.dst;
    if (pc.lead) {
      if (threadIdx.x == 0) dst[0] = pc.lead;
      ++dst;
    }
    const uint32_t* s = ss.src[g] + pc.src_off;
    for (uint32_t j = threadIdx.x; j < pc.src_len; j += blockDim.x) dst[j] = __ldg(s + j);
  }
}
}  // namespace
}  // namespace ndx

extern "C" int ndx_wah_assemble_slots(const uint32_t* const* h_src, uint32_t shards,
                                      const ndx_piece* d_pieces, uint64_t stride,
                                      const uint64_t* h_counts, uint32_t* d_out, void* stream) {
  if (!h_src || !d_pieces || !h_counts || !d_out || shards == 0 || shards > 64) return NDX_E_INVALID;
  ndx::ShardSrc ss{};
  uint64_t total = 0;
  for (uint32_t g = 0; g < shards; ++g) {
    ss.src[g] = h_src[g];
    ss.count[g] = uint32_t(h_counts[g]);
    total += h_counts[g];
  }
  if (total == 0) return 0;
  const int grid = int(umin<uint64_t>(uint64_t(shards) * stride, 148ull * 32));
  ndx::k_assemble_slots<<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(ss, shards, uint32_t(stride),
                                                                             d_pieces, d_out);
  return cudaGetLastError();
}
