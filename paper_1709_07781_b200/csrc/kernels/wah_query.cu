// Query side of the index on the GPU: decode a WAH
// bitmap, bitwise AND / OR / AND-NOT of decoded bitmaps, the rows of a
// bitmap, and canonical re-encoding.
//
// Decoded bitmaps are "chunk arrays": one u32 per 31-row chunk holding that
// chunk's literal (bit i = row 31c + i), the unit the WAH words are made of,
// so decoding and encoding never shift bits across words.
//
// Reference: decode (p/core/src/wah_words.cpp:21-34), rows_for
// (wah_words.cpp:93-103), encode + CanonicalWriter (wah_words.cpp:7-19,
// p/core/include/ndactor/wah.hpp:36-74).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../../include/ndx.h"
#include "common.cuh"

namespace ndx {

namespace {

constexpr int kQThreads = 256;

int grid_for(uint64_t n, int per_thread = 1) {
  uint64_t g = (n + uint64_t(kQThreads) * per_thread - 1) / (uint64_t(kQThreads) * per_thread);
  return int(umax<uint64_t>(1, umin<uint64_t>(g, 148ull * 32)));
}

__device__ __forceinline__ uint32_t chunks_of(uint32_t w) {
  return (w & kFillFlag) ? (w & kLenMask) : 1u;
}

// cc[i] = chunks covered by word i; a zero-length fill raises the error flag.
__global__ void k_word_chunks(const uint32_t* __restrict__ words, uint64_t n, uint32_t* cc,
                              uint32_t* err) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t w = words[i];
    const uint32_t c = chunks_of(w);
    if (c == 0) atomicOr(err, 1u);
    cc[i] = c;
  }
}

// One thread per output chunk: the covering word by binary search over the
// words' exclusive chunk starts; chunks past the stream are zero.
__global__ void k_expand(const uint32_t* __restrict__ words, const uint32_t* __restrict__ start,
                         uint64_t n_words, const uint32_t* covered_p, uint32_t* __restrict__ chunks,
                         uint64_t n_chunks) {
  const uint32_t covered = n_words ? *covered_p : 0u;
  for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n_chunks;
       c += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t v = 0;
    if (c < covered) {
      uint64_t lo = 0, hi = n_words;  // last word with start <= c
      while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (start[mid] <= c)
          lo = mid;
        else
          hi = mid;
      }
      const uint32_t w = words[lo];
      v = (w & kFillFlag) ? ((w & kOnesFlag) ? kLiteralMask : 0u) : w;
    }
    chunks[c] = v;
  }
}

__global__ void k_set(uint32_t* p, uint32_t v) { *p = v; }

__global__ void k_total(const uint32_t* last_excl, const uint32_t* last_val, uint32_t* total) {
  *total = *last_excl + *last_val;
}

template <int OP>
__global__ void k_bitop(const uint4* __restrict__ a, const uint4* __restrict__ b, uint4* out,
                        uint64_t n4) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 x = a[i], y = b[i];
    uint4 r;
    if (OP == 0) r = make_uint4(x.x & y.x, x.y & y.y, x.z & y.z, x.w & y.w);
    if (OP == 1) r = make_uint4(x.x | y.x, x.y | y.y, x.z | y.z, x.w | y.w);
    if (OP == 2) r = make_uint4(x.x & ~y.x, x.y & ~y.y, x.z & ~y.z, x.w & ~y.w);
    out[i] = r;
  }
}
template <int OP>
__global__ void k_bitop_tail(const uint32_t* a, const uint32_t* b, uint32_t* out, uint64_t from,
                             uint64_t n) {
  const uint64_t i = from + threadIdx.x;
  if (i < n) out[i] = OP == 0 ? (a[i] & b[i]) : OP == 1 ? (a[i] | b[i]) : (a[i] & ~b[i]);
}

__global__ void k_popc(const uint32_t* __restrict__ chunks, uint64_t n, uint32_t* cnt) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    cnt[i] = __popc(chunks[i] & kLiteralMask);
}

__global__ void k_rows(const uint32_t* __restrict__ chunks, const uint32_t* __restrict__ off,
                       uint64_t n, uint32_t row_limit, uint32_t* rows) {
  for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
       c += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t bits = chunks[c] & kLiteralMask;
    uint32_t o = off[c];
    while (bits) {
      const uint32_t i = __ffs(bits) - 1;
      bits &= bits - 1;
      const uint64_t row = uint64_t(c) * kChunkBits + i;
      if (row < row_limit) rows[o] = uint32_t(row);
      ++o;
    }
  }
}

// Encode: chunk type 0 zero / 1 ones / 2 mixed; a word starts at every
// mixed chunk and wherever a uniform run begins.
__device__ __forceinline__ uint32_t ctype(uint32_t v) {
  v &= kLiteralMask;
  return v == 0 ? 0u : (v == kLiteralMask ? 1u : 2u);
}

__global__ void k_last_set(const uint32_t* __restrict__ chunks, uint64_t n, uint32_t* last1) {
  uint32_t best = 0;
  for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
       c += uint64_t(gridDim.x) * blockDim.x)
    if (chunks[c] & kLiteralMask) best = umax(best, uint32_t(c) + 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = umax(best, __shfl_xor_sync(kFull, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(last1, best);
}

__global__ void k_heads(const uint32_t* __restrict__ chunks, const uint32_t* n_eff_p, uint64_t n,
                        uint32_t* head) {
  const uint32_t n_eff = n_eff_p ? *n_eff_p : uint32_t(n);
  for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
       c += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t h = 0;
    if (c < n_eff) {
      const uint32_t t = ctype(chunks[c]);
      h = (c == 0 || t == 2 || t != ctype(chunks[c - 1])) ? 1u : 0u;
    }
    head[c] = h;
  }
}

__global__ void k_positions(const uint32_t* __restrict__ head, const uint32_t* __restrict__ idx,
                            uint64_t n, uint32_t* pos) {
  for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
       c += uint64_t(gridDim.x) * blockDim.x)
    if (head[c]) pos[idx[c]] = uint32_t(c);
}

__global__ void k_words(const uint32_t* __restrict__ chunks, const uint32_t* __restrict__ pos,
                        const uint32_t* n_words_p, const uint32_t* n_eff_p, uint64_t n,
                        uint32_t* words, uint32_t* err) {
  const uint32_t K = *n_words_p;
  const uint32_t n_eff = n_eff_p ? *n_eff_p : uint32_t(n);
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < K;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = pos[k];
    const uint32_t v = chunks[c] & kLiteralMask;
    const uint32_t t = ctype(v);
    if (t == 2) {
      words[k] = v;
    } else {
      const uint32_t end = k + 1 < K ? pos[k + 1] : n_eff;
      const uint32_t len = end - c;
      if (len > kLenMask) atomicOr(err, 2u);
      words[k] = make_fill(t == 1, len);
    }
  }
}

}  // namespace

}  // namespace ndx

using namespace ndx;

extern "C" {

size_t ndx_wah_decode_scratch_bytes(uint64_t n_words) {
  return size_t(n_words + 1) * 8 + ndx_scan_scratch_bytes(n_words + 1) + 1024;
}

int ndx_wah_decode(const uint32_t* d_words, uint64_t n_words, uint32_t* d_chunks,
                   uint64_t n_chunks, void* d_scratch, uint32_t* d_info, void* stream) {
  if ((!d_words && n_words) || (!d_chunks && n_chunks) || !d_scratch || !d_info)
    return NDX_E_INVALID;
  if (n_words >= (1ull << 31) || n_chunks >= (1ull << 32)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  uint32_t* cc = static_cast<uint32_t*>(d_scratch);
  uint32_t* start = cc + (n_words + 1);
  void* scan_scr = reinterpret_cast<void*>(
      (reinterpret_cast<uintptr_t>(start + n_words + 1) + 255) & ~uintptr_t(255));
  if ((e = cudaMemsetAsync(d_info, 0, 8, s))) return e;
  if (n_words) {
    k_word_chunks<<<grid_for(n_words), kQThreads, 0, s>>>(d_words, n_words, cc, d_info + 1);
    int rc = ndx_scan_exclusive_u32(cc, start, n_words, scan_scr, stream);
    if (rc) return rc;
    k_total<<<1, 1, 0, s>>>(start + n_words - 1, cc + n_words - 1, d_info);
  }
  if (n_chunks)
    k_expand<<<grid_for(n_chunks), kQThreads, 0, s>>>(d_words, start, n_words, d_info, d_chunks,
                                                       n_chunks);
  return cudaGetLastError();
}

static int bitop(int op, const uint32_t* a, const uint32_t* b, uint32_t* out, uint64_t n,
                 void* stream) {
  if (n == 0) return 0;
  if (!a || !b || !out) return NDX_E_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                         reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const uint64_t n4 = aligned ? n / 4 : 0;
  const uint4 *a4 = reinterpret_cast<const uint4*>(a), *b4 = reinterpret_cast<const uint4*>(b);
  uint4* o4 = reinterpret_cast<uint4*>(out);
  const uint64_t from = n4 * 4;
  const int tail_blocks = int((n - from + kQThreads - 1) / kQThreads);
  switch (op) {
    case 0:
      if (n4) k_bitop<0><<<grid_for(n4), kQThreads, 0, s>>>(a4, b4, o4, n4);
      for (int k = 0; k < tail_blocks; ++k)
        k_bitop_tail<0><<<1, kQThreads, 0, s>>>(a, b, out, from + uint64_t(k) * kQThreads, n);
      break;
    case 1:
      if (n4) k_bitop<1><<<grid_for(n4), kQThreads, 0, s>>>(a4, b4, o4, n4);
      for (int k = 0; k < tail_blocks; ++k)
        k_bitop_tail<1><<<1, kQThreads, 0, s>>>(a, b, out, from + uint64_t(k) * kQThreads, n);
      break;
    default:
      if (n4) k_bitop<2><<<grid_for(n4), kQThreads, 0, s>>>(a4, b4, o4, n4);
      for (int k = 0; k < tail_blocks; ++k)
        k_bitop_tail<2><<<1, kQThreads, 0, s>>>(a, b, out, from + uint64_t(k) * kQThreads, n);
  }
  return cudaGetLastError();
}

int ndx_chunks_and(const uint32_t* a, const uint32_t* b, uint32_t* out, uint64_t n, void* stream) {
  return bitop(0, a, b, out, n, stream);
}
int ndx_chunks_or(const uint32_t* a, const uint32_t* b, uint32_t* out, uint64_t n, void* stream) {
  return bitop(1, a, b, out, n, stream);
}
int ndx_chunks_andnot(const uint32_t* a, const uint32_t* b, uint32_t* out, uint64_t n,
                      void* stream) {
  return bitop(2, a, b, out, n, stream);
}

size_t ndx_chunks_rows_scratch_bytes(uint64_t n_chunks) {
  return size_t(n_chunks + 1) * 8 + ndx_scan_scratch_bytes(n_chunks + 1) + 1024;
}

int ndx_chunks_rows(const uint32_t* d_chunks, uint64_t n_chunks, uint32_t row_limit,
                    uint32_t* d_rows, void* d_scratch, uint32_t* d_count, void* stream) {
  if (!d_count || (n_chunks && (!d_chunks || !d_rows || !d_scratch))) return NDX_E_INVALID;
  if (n_chunks >= (1ull << 32) / kChunkBits) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if ((e = cudaMemsetAsync(d_count, 0, 4, s))) return e;
  if (n_chunks == 0) return 0;
  uint32_t* cnt = static_cast<uint32_t*>(d_scratch);
  uint32_t* off = cnt + (n_chunks + 1);
  void* scan_scr = reinterpret_cast<void*>(
      (reinterpret_cast<uintptr_t>(off + n_chunks + 1) + 255) & ~uintptr_t(255));
  k_popc<<<grid_for(n_chunks), kQThreads, 0, s>>>(d_chunks, n_chunks, cnt);
  int rc = ndx_scan_exclusive_u32(cnt, off, n_chunks, scan_scr, stream);
  if (rc) return rc;
  k_rows<<<grid_for(n_chunks), kQThreads, 0, s>>>(d_chunks, off, n_chunks, row_limit, d_rows);
  k_total<<<1, 1, 0, s>>>(off + n_chunks - 1, cnt + n_chunks - 1, d_count);
  return cudaGetLastError();
}

size_t ndx_wah_encode_scratch_bytes(uint64_t n_chunks) {
  return size_t(n_chunks + 1) * 12 + ndx_scan_scratch_bytes(n_chunks + 1) + 1024;
}

int ndx_wah_encode(const uint32_t* d_chunks, uint64_t n_chunks, int trim_trailing,
                   uint32_t* d_words, void* d_scratch, uint32_t* d_info, void* stream) {
  if (!d_info || (n_chunks && (!d_chunks || !d_words || !d_scratch))) return NDX_E_INVALID;
  if (n_chunks >= (1ull << 32)) return NDX_E_TOO_LARGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  // d_info: [0] words, [1] error flags, [2] chunks encoded
  if ((e = cudaMemsetAsync(d_info, 0, 12, s))) return e;
  if (n_chunks == 0) return 0;
  uint32_t* head = static_cast<uint32_t*>(d_scratch);
  uint32_t* idx = head + (n_chunks + 1);
  uint32_t* pos = idx + (n_chunks + 1);
  void* scan_scr = reinterpret_cast<void*>(
      (reinterpret_cast<uintptr_t>(pos + n_chunks + 1) + 255) & ~uintptr_t(255));
  const uint32_t* n_eff = nullptr;  // null: every chunk is encoded
  if (trim_trailing) {
    k_last_set<<<grid_for(n_chunks), kQThreads, 0, s>>>(d_chunks, n_chunks, d_info + 2);
    n_eff = d_info + 2;
  } else {
    k_set<<<1, 1, 0, s>>>(d_info + 2, uint32_t(n_chunks));
  }
  k_heads<<<grid_for(n_chunks), kQThreads, 0, s>>>(d_chunks, n_eff, n_chunks, head);
  int rc = ndx_scan_exclusive_u32(head, idx, n_chunks, scan_scr, stream);
  if (rc) return rc;
  k_total<<<1, 1, 0, s>>>(idx + n_chunks - 1, head + n_chunks - 1, d_info);
  k_positions<<<grid_for(n_chunks), kQThreads, 0, s>>>(head, idx, n_chunks, pos);
  k_words<<<grid_for(n_chunks), kQThreads, 0, s>>>(d_chunks, pos, d_info, n_eff, n_chunks, d_words,
                                                    d_info + 1);
  return cudaGetLastError();
}

}  // extern "C"

// ---------------------------------------------------------------------------
// fp32 square matrix product for the paper's facade-overhead protocol
// (p/core/src/bench_protocols.cpp spawn_matmul / enqueue_matmul): one output
// per thread, the k sum in ascending order with separately rounded multiply
// and add, so the result is bit-identical to the triple-loop oracle.  It is
// a dispatch-overhead probe at n <= 256, not a GEMM workload.
namespace ndx {
namespace {
constexpr int kMmTile = 16;
__global__ void k_matmul(const float* __restrict__ a, const float* __restrict__ b,
                         float* __restrict__ out, uint32_t n) {
  __shared__ float ta[kMmTile][kMmTile], tb[kMmTile][kMmTile + 1];
  const uint32_t x = blockIdx.x * kMmTile + threadIdx.x, y = blockIdx.y * kMmTile + threadIdx.y;
  float acc = 0.f;
  for (uint32_t k0 = 0; k0 < n; k0 += kMmTile) {
    const uint32_t ka = k0 + threadIdx.x, kb = k0 + threadIdx.y;
    ta[threadIdx.y][threadIdx.x] = (y < n && ka < n) ? a[uint64_t(y) * n + ka] : 0.f;
    tb[threadIdx.y][threadIdx.x] = (kb < n && x < n) ? b[uint64_t(kb) * n + x] : 0.f;
    __syncthreads();
    const uint32_t kmax = umin<uint32_t>(kMmTile, n - k0);
    for (uint32_t k = 0; k < kmax; ++k) acc = __fadd_rn(acc, __fmul_rn(ta[threadIdx.y][k], tb[k][threadIdx.x]));
    __syncthreads();
  }
  if (x < n && y < n) out[uint64_t(y) * n + x] = acc;
}
}  // namespace
}  // namespace ndx

extern "C" int ndx_matmul_f32(const float* d_a, const float* d_b, float* d_out, uint64_t n,
                              void* stream) {
  if (n == 0) return 0;
  if (!d_a || !d_b || !d_out) return NDX_E_INVALID;
  if (n > 65536) return NDX_E_TOO_LARGE;
  const dim3 block(ndx::kMmTile, ndx::kMmTile);
  const dim3 grid(unsigned((n + ndx::kMmTile - 1) / ndx::kMmTile), unsigned((n + ndx::kMmTile - 1) / ndx::kMmTile));
  ndx::k_matmul<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(d_a, d_b, d_out, uint32_t(n));
  return cudaGetLastError();
}
