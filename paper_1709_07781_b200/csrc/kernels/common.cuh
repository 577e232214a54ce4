// Shared device helpers for the WAH build kernels (sm_100a).
//
// Decoupled look-back statuses carry an epoch so the status arrays never need
// clearing between builds: a status whose epoch differs from the running
// pass's epoch reads as "not ready".
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ndx {

constexpr uint32_t kChunkBits = 31;           // wah.hpp:15-21
constexpr uint32_t kFillFlag = 0x80000000u;
constexpr uint32_t kOnesFlag = 0x40000000u;
constexpr uint32_t kLenMask = 0x3fffffffu;
constexpr uint32_t kLiteralMask = 0x7fffffffu;

__host__ __device__ constexpr uint32_t make_fill(bool ones, uint32_t len) {
  return kFillFlag | (ones ? kOnesFlag : 0u) | len;
}

constexpr unsigned kFull = 0xffffffffu;

template <class T>
__host__ __device__ __forceinline__ T umin(T a, T b) { return a < b ? a : b; }
template <class T>
__host__ __device__ __forceinline__ T umax(T a, T b) { return a < b ? b : a; }

// ---- look-back status word: [63:48] epoch | [47:46] flag | [45:0] value ----
constexpr uint64_t kFlagAgg = 1ull << 46;
constexpr uint64_t kFlagPrefix = 2ull << 46;
constexpr uint64_t kValueMask = (1ull << 46) - 1;

__device__ __forceinline__ uint64_t status_word(uint32_t epoch, uint64_t flag,
                                                uint64_t value) {
  return (uint64_t(epoch & 0xffffu) << 48) | flag | (value & kValueMask);
}
__device__ __forceinline__ bool status_ready(uint64_t s, uint32_t epoch) {
  return (s >> 48) == (epoch & 0xffffu) && (s & (3ull << 46)) != 0;
}
__device__ __forceinline__ bool status_is_prefix(uint64_t s) {
  return (s & (3ull << 46)) == kFlagPrefix;
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streaming loads: the inputs are read exactly once per kernel.
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ldg_stream(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cs.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ldg_stream4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// ---- bulk async copy global -> shared (TMA 1-D) completing on an mbarrier ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Orders this thread's earlier generic-proxy shared accesses before later
// async-proxy (bulk copy) writes to the same shared memory.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
// bytes and both addresses must be multiples of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned lanemask_le() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}

// Lanes of the warp holding the same `bits`-wide label (ballot-based match;
// valid-lane masking is the caller's).
template <int BITS>
__device__ __forceinline__ unsigned match_label(uint32_t label) {
  unsigned peers = kFull;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    unsigned bit = (label >> b) & 1u;
    unsigned bal = __ballot_sync(kFull, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}

__device__ __forceinline__ uint32_t warp_incl_sum(uint32_t v) {
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(kFull, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_incl_sum64(uint64_t v) {
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t t = __shfl_up_sync(kFull, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}

}  // namespace ndx
