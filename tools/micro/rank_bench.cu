// Microbenchmark: cost of stable warp ranking variants (no global memory in
// the timed loop).  Elements per second per variant and digit width.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned lanemask_lt() { unsigned m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

template <int BITS>
__device__ __forceinline__ unsigned match_ballot(uint32_t d) {
  unsigned peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t, m;\n\tand.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t"
        "vote.sync.ballot.b32 t, p, 0xffffffff;\n\tselp.b32 m, 0, 0xffffffff, p;\n\txor.b32 t, t, m;\n\t"
        "and.b32 %0, %0, t;\n\t}" : "+r"(peers) : "r"(d), "r"(1u << b));
  }
  return peers;
}

template <int BITS, int MODE>
__global__ void k_rank(uint32_t seed, int iters, uint32_t* sink) {
  constexpr int NB = 1 << BITS;
  __shared__ uint32_t M[8][NB];
  __shared__ uint16_t H[8][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = lane; i < NB; i += 32) { M[warp][i] = 0; H[warp][i] = 0; }
  __syncwarp();
  uint32_t x = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 40503u);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    const uint32_t d = (x >> 8) & (NB - 1);
    unsigned peers;
    if (MODE == 0) {
      peers = match_ballot<BITS>(d);
    } else if (MODE == 1) {
      atomicOr(&M[warp][d], 1u << lane);
      __syncwarp();
      peers = M[warp][d];
      __syncwarp();
    } else {
      peers = __match_any_sync(0xffffffffu, d);
    }
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == leader) {
      old = H[warp][d];
      H[warp][d] = uint16_t(old + __popc(peers));
      if (MODE == 1) M[warp][d] = 0;
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    acc += old + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <int BITS, int MODE>
void run(const char* name) {
  uint32_t* sink;
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  k_rank<BITS, MODE><<<blocks, threads>>>(1, iters, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_rank<BITS, MODE><<<blocks, threads>>>(2, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double elems = double(blocks) * threads * iters;
  printf("%-12s bits=%2d  %7.1f G elem/s  (%.2f elem/SM-cycle at 1.92 GHz)\n", name, BITS, elems / ms / 1e6,
         elems / (ms * 1e-3) / (sms * 1.92e9));
  cudaFree(sink);
}

int main() {
  run<8, 0>("ballot"); run<8, 1>("atomic-or"); run<8, 2>("match_any");
  run<10, 0>("ballot"); run<10, 2>("match_any");
  run<9, 0>("ballot"); run<9, 1>("atomic-or"); run<9, 2>("match_any");
  return 0;
}
