// Warp ranking microbenchmark (diagnostic, not product): the stable rank of
// 32 lanes' keys among equal keys in a warp — what the sort's scatter and
// in-bucket passes do per 32 lookups — via (a) a shared-memory OR of lane
// bits into a per-key mask word (what sort.cu does), (b) match.any.sync.
// 1024 distinct keys per warp (10-bit buckets), keys from a hash.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 warp_rank.cu -o wr && ./wr
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int MODE, int KB>
__global__ void rank_kernel(int iters, uint32_t* out, int hot) {
  extern __shared__ uint32_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = 1 << KB;
  uint32_t* cur = sm + warp * (2 * nk);
  uint32_t* msk = cur + nk;
  for (int k = lane; k < nk; k += 32) { cur[k] = 0; msk[k] = 0; }
  __syncwarp();
  const unsigned me = 1u << lane, lt = me - 1u;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t key = hsh(blockIdx.x * 7919u + threadIdx.x * 131u + it * 31337u);
    key = (hot && (key >> 28) < 6) ? (key & 7u) : (key & (nk - 1));  // ~38 % on 8 hot keys
    unsigned peers;
    if (MODE == 0) {
      atomicOr(&msk[key], me);
      __syncwarp();
      peers = msk[key];
    } else {
      peers = __match_any_sync(0xffffffffu, key);
    }
    const uint32_t s0 = cur[key];
    __syncwarp();
    if ((peers & lt) == 0) {
      if (MODE == 0) msk[key] = 0;
      cur[key] = s0 + __popc(peers);
    }
    __syncwarp();
    acc += s0 + __popc(peers & lt);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE, int KB>
void run(uint32_t* out, int hot) {
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  const size_t smem = 8 * 2 * (1 << KB) * 4;
  cudaFuncSetAttribute(rank_kernel<MODE, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    rank_kernel<MODE, KB><<<blocks, threads, smem>>>(iters, out, hot);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double chunks = (double)blocks * (threads / 32) * iters;
  printf("%s keys=%4d hot=%d: %6.2f G chunk-ranks/s (%.1f G items/s)  err=%s\n",
         MODE == 0 ? "shared-OR " : "match.any ", 1 << KB, hot, chunks / (best * 1e6),
         32 * chunks / (best * 1e6), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  for (int hot = 0; hot < 2; ++hot) {
    run<0, 10>(out, hot);
    run<1, 10>(out, hot);
    run<0, 6>(out, hot);
    run<1, 6>(out, hot);
  }
  return 0;
}
