// Multi-GPU build, the per-step device work after the metadata all-gather
// (SURVEY.md section 8(e), Appendix B): the merge plan from device-resident
// shard counts (no host round trip), and the exchange of the words as one
// kernel over NVLink peer memory.
//
// Every rank holds the all-gathered per-value metadata of every shard
// (ndx_shard_meta, shard g's records in slots [g*cap, g*cap + count_g),
// ascending values, at most one record per value and shard).  Then:
//
//   k_dp_rank     global merge rank of every record: its index in its shard
//                 plus, per other shard, the records with a smaller value
//                 (and, for lower shards, the equal one) -- binary searches,
//                 so records of one value end adjacent, in shard order
//   k_dp_heads    value heads over the merged order  (+ exclusive scan)
//   k_dp_values   one thread per value: its pieces in shard order with the
//                 Appendix B rules (first piece keeps a zero-fill of f
//                 chunks, later ones get the gap fill, ones-fills meeting at
//                 gap 0 fuse into one word); the value's word count
//                 (+ exclusive scan: the value offsets)
//   k_dp_finalize the merged table, every piece's absolute destination, and
//                 the pieces in merged (= destination) order
//   k_dp_totals   D, W, and the owner bounds: rank h owns the words
//                 [b_h, b_h+1), cut at the first value at or after h*W/G
//   k_dp_pull     rank h's slice: every output chunk of 4096 words finds its
//                 pieces by binary search and copies them from the owning
//                 shard's words -- read straight from that GPU's memory over
//                 NVLink (IPC-mapped peer pointers), so there is no separate
//                 send/receive and no host-sized all-to-all
#include <cuda_runtime.h>

#include <cstdint>

#include "../../../include/ndx.h"
#include "common.cuh"

namespace ndx {
namespace {

constexpr int kDThreads = 256;
constexpr uint32_t kPullChunk = 4096;
constexpr uint32_t kErrBody = 1, kErrOverlap = 2, kErrOverflow = 4, kErrSlice = 8;

int dgrid(uint64_t n) {
  return int(umax<uint64_t>(1, umin<uint64_t>((n + kDThreads - 1) / kDThreads, 148ull * 16)));
}

struct DPlan {
  const ndx_shard_meta* metas;  // G x cap slots
  const ndx_wah_counts* counts; // G shard counts (distinct = records of the shard)
  uint32_t G, cap;
  uint32_t* order;              // merged rank -> slot
  uint32_t* head;               // merged rank: first record of its value
  uint32_t* hscan;              // exclusive scan of head
  uint32_t* len;                // value -> words
  uint32_t* off;                // value -> offset (exclusive scan of len)
  ndx_piece* pieces;            // slot -> piece (dst relative, then absolute)
  ndx_piece* merged;            // merged rank -> piece (pad = source shard)
  uint32_t* entries;            // merged (value, offset, length) table
  uint64_t* totals;             // [0] D, [1] W, [2] error flags, [3] records
  uint64_t* bounds;             // G + 1 owner bounds
};

__device__ __forceinline__ uint32_t shard_count(const DPlan& p, uint32_t g) {
  const uint64_t c = p.counts[g].distinct;
  return uint32_t(c < p.cap ? c : p.cap);
}

// records of shard g with value < v (strict) or <= v
__device__ __forceinline__ uint32_t count_below(const DPlan& p, uint32_t g, uint32_t v, bool inclusive) {
  const ndx_shard_meta* m = p.metas + uint64_t(g) * p.cap;
  uint32_t lo = 0, hi = shard_count(p, g);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint32_t x = __ldg(&m[mid].value);
    if (x < v || (inclusive && x == v))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void k_dp_rank(DPlan p) {
  const uint64_t slots = uint64_t(p.G) * p.cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t r = 0;
    uint32_t flags = 0;
    for (uint32_t g = 0; g < p.G; ++g) {
      r += shard_count(p, g);
      if (p.counts[g].distinct > p.cap) flags |= kErrOverflow;  // metadata capacity exceeded
    }
    p.totals[3] = r;
    if (flags) atomicOr(reinterpret_cast<unsigned long long*>(p.totals + 2), flags);
  }
  for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < slots; s += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t g = uint32_t(s / p.cap), i = uint32_t(s % p.cap);
    if (i >= shard_count(p, g)) continue;
    const uint32_t v = p.metas[s].value;
    uint32_t rank = i;
    for (uint32_t h = 0; h < p.G; ++h)
      if (h != g) rank += count_below(p, h, v, h < g);
    p.order[rank] = uint32_t(s);
  }
}

__global__ void k_dp_heads(DPlan p, uint64_t rpad) {
  const uint64_t R = p.totals[3];
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < rpad; j += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t h = 0;
    if (j < R) h = j == 0 || p.metas[p.order[j]].value != p.metas[p.order[j - 1]].value;
    p.head[j] = h;
    p.len[j] = 0;
  }
}

__global__ void k_dp_values(DPlan p) {
  const uint64_t R = p.totals[3];
  unsigned long long* err = reinterpret_cast<unsigned long long*>(p.totals + 2);
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < R; j += uint64_t(gridDim.x) * blockDim.x) {
    if (!p.head[j]) continue;
    const uint32_t v = p.metas[p.order[j]].value;
    uint32_t l = 0;       // words so far
    uint32_t prev_l = 0;  // last chunk of the previous piece
    ndx_piece* last_piece = nullptr;  // the value's current last word: its piece,
    bool last_is_lead = false;        // whether it is that piece's lead,
    uint32_t last_ones = 0;           // and its ones-fill length (0: not a ones-fill)
    for (uint64_t k = j; k < R; ++k) {
      const uint32_t slot = p.order[k];
      const ndx_shard_meta m = p.metas[slot];
      if (m.value != v) break;
      ndx_piece pc{0, m.body_off, m.body_len, 0, 0};
      if (m.body_len == 0) atomicOr(err, kErrBody);
      if (k == j) {
        if (m.f > 0) pc.lead = make_fill(false, m.f);
      } else {
        if (m.f <= prev_l) atomicOr(err, kErrOverlap);
        const uint32_t gap = m.f - prev_l - 1;
        if (gap > 0) {
          pc.lead = make_fill(false, gap);
        } else if (last_ones > 0 && m.a > 0) {  // ones + ones at gap 0: one fused fill
          if (last_is_lead)
            last_piece->lead = 0;
          else
            last_piece->src_len -= 1;
          --l;
          pc.lead = make_fill(true, last_ones + m.a);
          pc.src_off += 1;
          pc.src_len -= 1;
        }
      }
      pc.dst = l;  // relative; made absolute once the value offsets are known
      l += (pc.lead ? 1u : 0u) + pc.src_len;
      ndx_piece* out = &p.pieces[slot];
      *out = pc;
      last_piece = out;
      if (pc.src_len > 0) {
        last_is_lead = false;
        last_ones = m.z;
      } else {
        last_is_lead = true;
        last_ones = (pc.lead & 0xC0000000u) == 0xC0000000u ? (pc.lead & kLenMask) : 0u;
      }
      prev_l = m.l;
    }
    p.len[p.hscan[j]] = l;
  }
}

__global__ void k_dp_finalize(DPlan p) {
  const uint64_t R = p.totals[3];
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < R; j += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t slot = p.order[j];
    const uint32_t d = p.hscan[j] + p.head[j] - 1u;
    ndx_piece pc = p.pieces[slot];
    pc.dst += p.off[d];
    pc.pad = slot / p.cap;  // the source shard
    p.pieces[slot] = pc;
    p.merged[j] = pc;
    if (p.head[j]) {
      p.entries[3 * uint64_t(d)] = p.metas[slot].value;
      p.entries[3 * uint64_t(d) + 1] = p.off[d];
      p.entries[3 * uint64_t(d) + 2] = p.len[d];
    }
  }
}

__global__ void k_dp_totals(DPlan p) {
  if (threadIdx.x != 0) return;
  const uint64_t R = p.totals[3];
  const uint64_t D = R ? uint64_t(p.hscan[R - 1]) + p.head[R - 1] : 0;
  const uint64_t W = D ? uint64_t(p.off[D - 1]) + p.len[D - 1] : 0;
  p.totals[0] = D;
  p.totals[1] = W;
  p.bounds[0] = 0;
  for (uint32_t h = 1; h < p.G; ++h) {
    const uint64_t want = W * h / p.G;
    uint64_t lo = 0, hi = D;  // first value whose offset >= want
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (p.off[mid] < want)
        lo = mid + 1;
      else
        hi = mid;
    }
    p.bounds[h] = lo < D ? p.off[lo] : W;
  }
  p.bounds[p.G] = W;
}

struct Peers {
  const uint32_t* words[64];  // shard g's local words (peer memory for g != rank)
};

// Rank `rank`'s owned slice [bounds[rank], bounds[rank+1]) (or, all_words,
// the whole merged array) assembled from every shard's words.  One CTA per
// 4096-word output chunk, its threads striding over the chunk's words.
__global__ __launch_bounds__(256, 4) void k_dp_pull(Peers peers, const ndx_piece* __restrict__ merged,
                                                 const uint64_t* __restrict__ totals,
                                                 const uint64_t* __restrict__ bounds, uint32_t rank, int all_words,
                                                 uint32_t* __restrict__ out, uint64_t out_cap,
                                                 uint64_t* __restrict__ err_out) {
  __shared__ uint64_t s_k0, s_k1;
  const uint64_t R = totals[3];
  const uint64_t b0 = all_words ? 0 : bounds[rank], b1 = all_words ? totals[1] : bounds[rank + 1];
  if (b1 - b0 > out_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(reinterpret_cast<unsigned long long*>(err_out), kErrSlice);
    return;
  }
  const uint64_t chunks = (b1 - b0 + kPullChunk - 1) / kPullChunk;
  auto plen = [](const ndx_piece& pc) -> uint64_t { return (pc.lead ? 1u : 0u) + uint64_t(pc.src_len); };
  for (uint64_t q = blockIdx.x; q < chunks; q += gridDim.x) {
    const uint64_t c0 = b0 + q * kPullChunk, c1 = umin<uint64_t>(c0 + kPullChunk, b1);
    if (threadIdx.x == 0) {
      // last piece starting at or before c0 (pieces are in destination order;
      // empty pieces -- a fused lead dropped -- may share a dst)
      uint64_t lo = 0, hi = R;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (merged[mid].dst <= c0)
          lo = mid + 1;
        else
          hi = mid;
      }
      uint64_t k0 = lo ? lo - 1 : 0;
      while (k0 + 1 < R && merged[k0].dst + plen(merged[k0]) <= c0) ++k0;
      lo = k0;
      hi = R;  // first piece starting at or after c1
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (merged[mid].dst < c1)
          lo = mid + 1;
        else
          hi = mid;
      }
      s_k0 = k0;
      s_k1 = lo;
    }
    __syncthreads();
    // every thread walks its positions of the chunk (stride blockDim) and the
    // pieces under them: a hot value's single piece spreads over the whole
    // CTA, a run of tiny pieces costs one step per piece
    uint64_t k = s_k0;
    const uint64_t k1 = s_k1;
    ndx_piece pc = merged[k];
    uint64_t d1 = pc.dst + plen(pc), body = pc.dst + (pc.lead ? 1u : 0u);
    const uint32_t* src = peers.words[pc.pad] + pc.src_off;  // word `body` of the output
    // all of the thread's words of the chunk are loaded before any is
    // stored: kPullChunk / 256 loads in flight per thread
    constexpr int kPer = kPullChunk / 256;
    uint32_t w[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const uint64_t x = c0 + threadIdx.x + uint64_t(j) * 256;
      if (x < c1) {
        while (x >= d1 && k + 1 < k1) {
          pc = merged[++k];
          d1 = pc.dst + plen(pc);
          body = pc.dst + (pc.lead ? 1u : 0u);
          src = peers.words[pc.pad] + pc.src_off;
        }
        w[j] = x < body ? pc.lead : __ldg(src + (x - body));
      }
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const uint64_t x = c0 + threadIdx.x + uint64_t(j) * 256;
      if (x < c1) out[x - b0] = w[j];
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace ndx

using namespace ndx;

extern "C" {

size_t ndx_dist_plan_scratch_bytes(uint32_t shards, uint64_t cap) {
  const uint64_t rpad = uint64_t(shards) * cap + 1;
  return size_t(rpad) * (4 * 5 + 2 * sizeof(ndx_piece)) + ndx_scan_scratch_bytes(rpad) * 2 + 8 * 256;
}

int ndx_dist_plan(const ndx_shard_meta* d_metas, uint64_t cap, const ndx_wah_counts* d_counts, uint32_t shards,
                  uint32_t* d_entries, ndx_piece* d_merged, uint64_t* d_totals, uint64_t* d_bounds,
                  void* d_scratch, void* stream) {
  if (!d_metas || !d_counts || !d_entries || !d_merged || !d_totals || !d_bounds || !d_scratch)
    return NDX_E_INVALID;
  if (shards == 0 || shards > 64 || cap == 0) return NDX_E_INVALID;
  const uint64_t rpad = uint64_t(shards) * cap;
  if (rpad >= (1ull << 31)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto align = [](char* q) {
    return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(q) + 255) & ~uintptr_t(255));
  };
  const uint64_t R1 = rpad + 1;
  char* q = align(static_cast<char*>(d_scratch));
  DPlan p{};
  p.metas = d_metas;
  p.counts = d_counts;
  p.G = shards;
  p.cap = uint32_t(cap);
  auto take = [&](size_t bytes) {
    char* r = q;
    q = align(q + bytes);
    return r;
  };
  p.order = reinterpret_cast<uint32_t*>(take(R1 * 4));
  p.head = reinterpret_cast<uint32_t*>(take(R1 * 4));
  p.hscan = reinterpret_cast<uint32_t*>(take(R1 * 4));
  p.len = reinterpret_cast<uint32_t*>(take(R1 * 4));
  p.off = reinterpret_cast<uint32_t*>(take(R1 * 4));
  p.pieces = reinterpret_cast<ndx_piece*>(take(R1 * sizeof(ndx_piece)));
  void* scan1 = take(ndx_scan_scratch_bytes(R1));
  void* scan2 = take(ndx_scan_scratch_bytes(R1));
  p.merged = d_merged;
  p.entries = d_entries;
  p.totals = d_totals;
  p.bounds = d_bounds;
  cudaError_t e;
  if ((e = cudaMemsetAsync(d_totals, 0, 4 * sizeof(uint64_t), s))) return e;
  k_dp_rank<<<dgrid(rpad), kDThreads, 0, s>>>(p);
  k_dp_heads<<<dgrid(rpad), kDThreads, 0, s>>>(p, rpad);
  int rc = ndx_scan_exclusive_u32(p.head, p.hscan, rpad, scan1, stream);
  if (rc) return rc;
  k_dp_values<<<dgrid(rpad), kDThreads, 0, s>>>(p);
  if ((rc = ndx_scan_exclusive_u32(p.len, p.off, rpad, scan2, stream))) return rc;
  k_dp_finalize<<<dgrid(rpad), kDThreads, 0, s>>>(p);
  k_dp_totals<<<1, 32, 0, s>>>(p);
  return cudaGetLastError();
}

int ndx_dist_pull(const uint32_t* const* h_shard_words, uint32_t shards, const ndx_piece* d_merged,
                  uint64_t max_records, uint64_t* d_totals, const uint64_t* d_bounds, uint32_t rank, int all_words,
                  uint32_t* d_out, uint64_t out_cap, uint64_t out_hint, void* stream) {
  if (!h_shard_words || !d_merged || !d_totals || !d_bounds || !d_out || shards == 0 || shards > 64 ||
      rank >= shards)
    return NDX_E_INVALID;
  (void)max_records;
  Peers pr{};
  for (uint32_t g = 0; g < shards; ++g) pr.words[g] = h_shard_words[g];
  // about 2 CTAs per SM of chunks, every chunk visited (grid-stride)
  const uint64_t chunks = umax<uint64_t>(1, (out_hint + kPullChunk - 1) / kPullChunk);
  const int grid = int(umin<uint64_t>(chunks, 148ull * 8));
  k_dp_pull<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(pr, d_merged, d_totals, d_bounds, rank, all_words,
                                                                 d_out, out_cap, d_totals + 2);
  return cudaGetLastError();
}

}  // extern "C"
