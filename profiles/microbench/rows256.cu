// Random-row gather microbenchmark (diagnostic, not product): 16-byte lane
// slices (LDG.128, what K1 issues) against 32-byte slices (LDG.256,
// ld.global.nc.v8.f32, new on sm_100) for random 64-512 B rows of an 8 GB
// table, U rows in flight per lane group.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 rows256.cu -o r256 && ./r256
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct F8 { float v[8]; };
template <int SB>  // slice bytes: 16 or 32
__device__ __forceinline__ void ld(const float* p, float (&v)[8]) {
  if (SB == 16) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                   "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
  }
}

template <int SB, int U>
__global__ void gather(const float* w, int64_t nrows, int rb, int64_t steps, float* out) {
  const int L = rb / SB;  // lanes per row
  const int lane = threadIdx.x & 31;
  const int g = lane / L, s = lane % L, G = 32 / L;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int E = SB / 4;
  float acc = 0.f;
  for (int64_t it = 0; it < steps; it += U) {
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = mix((gw * steps + it + u) * G + g) & (nrows - 1);
      ld<SB>(w + r * (rb / 4) + s * E, v[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e < E) acc += v[u][e];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int SB, int U>
void run(const float* w, size_t bytes, float* out, cudaEvent_t a, cudaEvent_t b) {
  for (int rb = 64; rb <= 512; rb *= 2) {
    if (rb < SB * 1) continue;
    const int L = rb / SB;
    if (L > 32) continue;
    const int64_t nrows = bytes / rb;
    const int blocks = 148 * 8, threads = 256;
    const int64_t steps = 512;
    const double rows = (double)blocks * threads / 32 * (32 / L) * steps;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      gather<SB, U><<<blocks, threads>>>(w, nrows, rb, steps, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("slice %2d B  U=%d  row %3d B: %7.1f GB/s  %6.2f G rows/s\n", SB, U, rb,
           rows * rb / (best * 1e6), rows / (best * 1e6));
  }
}

int main() {
  const size_t bytes = 8ull << 30;
  float* w;
  cudaMalloc(&w, bytes);
  cudaMemset(w, 0, bytes);
  float* out;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  run<16, 4>(w, bytes, out, a, b);
  run<16, 8>(w, bytes, out, a, b);
  run<32, 2>(w, bytes, out, a, b);
  run<32, 4>(w, bytes, out, a, b);
  run<32, 8>(w, bytes, out, a, b);
  return 0;
}
