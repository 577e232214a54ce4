// The multi-GPU merge plan on the device: the same
// result as the host planner (csrc/runtime/wah_shard.cpp plan_merge_into),
// computed where the all-gathered metadata already is.
//
//   1. flatten the shards' records (shard-major) and stable-sort them by
//      value: records of one value end up adjacent, in shard order;
//   2. one thread per value walks its (at most G) pieces in shard order and
//      applies the merge rules: the first piece keeps a zero-fill of f
//      chunks, later pieces get the zero-fill of the gap, and ones-fills that
//      meet at gap 0 are fused into one word;
//   3. an exclusive scan of the per-value lengths gives the table and every
//      piece's absolute destination.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../../include/ndx.h"
#include "common.cuh"

namespace ndx {
namespace {

constexpr int kPThreads = 256;

int pgrid(uint64_t n) {
  return int(umax<uint64_t>(1, umin<uint64_t>((n + kPThreads - 1) / kPThreads, 148ull * 16)));
}

constexpr int kMaxShards = 64;
struct ShardTab {
  uint32_t base[kMaxShards + 1];  // record index of each shard's first record
  uint32_t count[kMaxShards];
};

// flat record r <- (value, slot) with slot = g * stride + i, shard-major
__global__ void k_flatten(const ndx_shard_meta* metas, ShardTab tab, uint32_t G, uint32_t stride,
                          uint32_t* keys, uint32_t* slots) {
  const uint64_t total = uint64_t(G) * stride;
  for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < total;
       x += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t g = uint32_t(x / stride), i = uint32_t(x % stride);
    if (i >= tab.count[g]) continue;
    const uint32_t r = tab.base[g] + i;
    keys[r] = metas[x].value;
    slots[r] = uint32_t(x);
  }
}

__global__ void k_vheads(const uint32_t* keys, uint32_t R, uint32_t* head) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < R; j += gridDim.x * blockDim.x)
    head[j] = (j == 0 || keys[j] != keys[j - 1]) ? 1u : 0u;
}

// One thread per value: its pieces in shard order (appendix B), lengths
// relative to the value's start; len[v] = the value's word count.
__global__ void k_values(const ndx_shard_meta* metas, const uint32_t* keys, const uint32_t* slots,
                         const uint32_t* head, const uint32_t* vid, uint32_t R,
                         ndx_piece* pieces, uint32_t* len, uint32_t* err) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < R; j += gridDim.x * blockDim.x) {
    if (!head[j]) continue;
    const uint32_t v = keys[j];
    uint32_t l = 0;       // words so far
    uint32_t prev_l = 0;  // last chunk of the previous piece
    // the value's current last word: owning piece, lead or not, ones length
    ndx_piece* last_piece = nullptr;
    bool last_is_lead = false;
    uint32_t last_ones = 0;
    for (uint32_t k = j; k < R && keys[k] == v; ++k) {
      const ndx_shard_meta m = metas[slots[k]];
      ndx_piece p{0, m.body_off, m.body_len, 0, 0};
      if (m.body_len == 0) atomicOr(err, 1u);
      if (k == j) {
        if (m.f > 0) p.lead = make_fill(false, m.f);
      } else {
        if (m.f <= prev_l) atomicOr(err, 2u);
        const uint32_t gap = m.f - prev_l - 1;
        if (gap > 0) {
          p.lead = make_fill(false, gap);
        } else if (last_ones > 0 && m.a > 0) {
          if (last_is_lead)
            last_piece->lead = 0;
          else
            last_piece->src_len -= 1;
          --l;
          p.lead = make_fill(true, last_ones + m.a);
          p.src_off += 1;
          p.src_len -= 1;
        }
      }
      p.dst = l;  // relative; made absolute once the value offsets are known
      l += (p.lead ? 1u : 0u) + p.src_len;
      ndx_piece* out = &pieces[slots[k]];
      *out = p;
      last_piece = out;
      if (p.src_len > 0) {
        last_is_lead = false;
        last_ones = m.z;
      } else {
        last_is_lead = true;
        last_ones = (p.lead & 0xC0000000u) == 0xC0000000u ? (p.lead & kLenMask) : 0u;
      }
      prev_l = m.l;
    }
    len[vid[j]] = l;
  }
}

__global__ void k_finalize(const uint32_t* keys, const uint32_t* slots, const uint32_t* head,
                           const uint32_t* vid, const uint32_t* off, const uint32_t* len,
                           uint32_t R, ndx_piece* pieces, uint32_t* entries) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < R; j += gridDim.x * blockDim.x) {
    const uint32_t d = vid[j];
    pieces[slots[j]].dst += off[d];
    if (head[j]) {
      entries[3 * d] = keys[j];
      entries[3 * d + 1] = off[d];
      entries[3 * d + 2] = len[d];
    }
  }
}

// vid[j] = index of record j's value: inclusive scan of heads minus one
__global__ void k_vid(const uint32_t* head_excl, const uint32_t* head, uint32_t R, uint32_t* vid,
                      uint64_t* totals) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < R; j += gridDim.x * blockDim.x)
    vid[j] = head_excl[j] + head[j] - 1u;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    totals[0] = R ? uint64_t(head_excl[R - 1]) + head[R - 1] : 0ull;
}

__global__ void k_words_total(const uint32_t* off, const uint32_t* len, const uint64_t* totals_in,
                              uint64_t* totals) {
  const uint64_t D = totals_in[0];
  totals[1] = D ? uint64_t(off[D - 1]) + len[D - 1] : 0ull;
}

}  // namespace
}  // namespace ndx

using namespace ndx;

extern "C" {

size_t ndx_merge_plan_scratch_bytes(uint64_t records) {
  const uint64_t R1 = records + 1;
  return size_t(R1) * 4 * 7 + ndx_sort_pairs_scratch_bytes(R1) + ndx_scan_scratch_bytes(R1) + 8 * 256;
}

int ndx_merge_plan(const ndx_shard_meta* d_metas, uint64_t stride, const uint64_t* h_counts,
                   uint32_t shards, uint32_t* d_entries, ndx_piece* d_pieces, uint64_t* d_totals,
                   void* d_scratch, void* stream) {
  if (!d_metas || !h_counts || !d_entries || !d_pieces || !d_totals || !d_scratch)
    return NDX_E_INVALID;
  if (shards == 0 || shards > uint32_t(kMaxShards)) return NDX_E_INVALID;
  ShardTab tab{};
  uint64_t R = 0;
  for (uint32_t g = 0; g < shards; ++g) {
    if (h_counts[g] > stride) return NDX_E_INVALID;
    tab.base[g] = uint32_t(R);
    tab.count[g] = uint32_t(h_counts[g]);
    R += h_counts[g];
  }
  tab.base[shards] = uint32_t(R);
  if (uint64_t(shards) * stride >= (1ull << 31)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if ((e = cudaMemsetAsync(d_totals, 0, 3 * sizeof(uint64_t), s))) return e;
  if (R == 0) return 0;
  auto align = [](char* q) {
    return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(q) + 255) & ~uintptr_t(255));
  };
  const uint64_t R1 = R + 1;
  char* p = align(static_cast<char*>(d_scratch));
  uint32_t* keys = reinterpret_cast<uint32_t*>(p);
  p = align(p + R1 * 4);
  uint32_t* slots = reinterpret_cast<uint32_t*>(p);
  p = align(p + R1 * 4);
  uint32_t* head = reinterpret_cast<uint32_t*>(p);
  p = align(p + R1 * 4);
  uint32_t* hscan = reinterpret_cast<uint32_t*>(p);
  p = align(p + R1 * 4);
  uint32_t* vid = reinterpret_cast<uint32_t*>(p);
  p = align(p + R1 * 4);
  uint32_t* len = reinterpret_cast<uint32_t*>(p);
  p = align(p + R1 * 4);
  uint32_t* off = reinterpret_cast<uint32_t*>(p);
  p = align(p + R1 * 4);
  void* sort_scr = p;
  p = align(p + ndx_sort_pairs_scratch_bytes(R1));
  void* scan_scr = p;
  uint32_t* err = reinterpret_cast<uint32_t*>(d_totals + 2);
  k_flatten<<<pgrid(uint64_t(shards) * stride), kPThreads, 0, s>>>(d_metas, tab, shards, uint32_t(stride),
                                                                  keys, slots);
  int rc = ndx_sort_pairs_u32(keys, slots, R, sort_scr, stream);  // stable: shard order kept
  if (rc) return rc;
  const uint32_t R32 = uint32_t(R);
  k_vheads<<<pgrid(R), kPThreads, 0, s>>>(keys, R32, head);
  if ((rc = ndx_scan_exclusive_u32(head, hscan, R, scan_scr, stream))) return rc;
  k_vid<<<pgrid(R), kPThreads, 0, s>>>(hscan, head, R32, vid, d_totals);
  if ((e = cudaMemsetAsync(len, 0, R * 4, s))) return e;
  k_values<<<pgrid(R), kPThreads, 0, s>>>(d_metas, keys, slots, head, vid, R32, d_pieces, len, err);
  if ((rc = ndx_scan_exclusive_u32(len, off, R, scan_scr, stream))) return rc;
  k_finalize<<<pgrid(R), kPThreads, 0, s>>>(keys, slots, head, vid, off, len, R32, d_pieces, d_entries);
  k_words_total<<<1, 1, 0, s>>>(off, len, d_totals, d_totals);
  return cudaGetLastError();
}

}  // extern "C"
