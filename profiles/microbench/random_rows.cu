// Random-row HBM microbenchmark (diagnostic, not product): what a B200
// sustains for random row gathers / read-modify-writes of 64-512 B rows over
// a 9 GB table — the access pattern of K1 (gather) and K4 (row RMW).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 random_rows.cu -o rr && ./rr
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// each group of L lanes (L = row_bytes/16) handles one random row per step
template <int MODE>  // 0 gather (sum into out), 1 RMW, 2 write-only
__global__ void rows_kernel(float4* w, int64_t nrows, int L, int64_t steps, float4* out) {
  const int lane = threadIdx.x & 31;
  const int g = lane / L, s = lane % L, G = 32 / L;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t it = 0; it < steps; it += 8) {
    float4 v[8];
    int64_t r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      r[u] = mix((gw * steps + it + u) * G + g) & (nrows - 1);  // nrows is a power of two
      if (MODE != 2) v[u] = w[r[u] * L + s];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
      if (MODE == 1) { v[u].x += 1.f; w[r[u] * L + s] = v[u]; }
      if (MODE == 2) w[r[u] * L + s] = make_float4(1, 2, 3, 4);
    }
  }
  if (MODE == 0) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const size_t bytes = 8ull << 30;
  float4* w;
  cudaMalloc(&w, bytes);
  cudaMemset(w, 0, bytes);
  float4* out;
  cudaMalloc(&out, 148 * 64 * 32 * 16 * 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[3] = {"gather", "rmw", "write"};
  for (int mode = 0; mode < 3; ++mode)
    for (int rb = 64; rb <= 512; rb *= 2) {
      const int L = rb / 16;
      const int64_t nrows = bytes / rb;
      const int blocks = 148 * 8, threads = 256;
      const int64_t steps = 1024;
      const double nrow_total = (double)blocks * threads / 32 * (32 / L) * steps;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) rows_kernel<0><<<blocks, threads>>>(w, nrows, L, steps, out);
        if (mode == 1) rows_kernel<1><<<blocks, threads>>>(w, nrows, L, steps, out);
        if (mode == 2) rows_kernel<2><<<blocks, threads>>>(w, nrows, L, steps, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double traffic = nrow_total * rb * (mode == 1 ? 2 : 1);
        if (rep) printf("%-6s row %4d B: %7.1f GB/s (%.3f ms)\n", names[mode], rb, traffic / ms / 1e6, ms);
      }
    }
  return 0;
}
