// Row-update microbenchmark (diagnostic, not product): the candidate ways a
// B200 can apply K4's per-unique-row update W[r] -= lr * g and gather K1's
// rows, over random 64-512 B rows of an 8 GiB table.
//   rmw   LDG row -> add -> STG row (what sgd_kernel does today)
//   red   red.global.add.v4.f32 of the delta (no load on the SM; the L2 does
//         the read-modify-write, fire-and-forget)
//   bulk  cp.async.bulk (TMA) gather of rows into a shared-memory ring with
//         mbarrier completion, summed from smem (K1 / gradient gather shape)
//   ldg   plain LDG gather (reference for bulk)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 row_update.cu -o ru && ./ru
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ void red_v4(float4* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// MODE 0 ldg gather, 1 rmw, 2 red
template <int MODE>
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
      r[u] = mix((gw * steps + it + u) * G + g) & (nrows - 1);
      if (MODE <= 1) v[u] = w[r[u] * L + s];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
      if (MODE == 1) { v[u].x += 1.f; w[r[u] * L + s] = v[u]; }
      if (MODE == 2) red_v4(w + r[u] * L + s, make_float4(1e-7f, 0.f, 0.f, 0.f));
    }
  }
  if (MODE == 0) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// TMA bulk gather: each warp owns a 2-stage ring of kStageBytes per stage.
constexpr int kStageBytes = 4096;
constexpr int kWarps = 8;

__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(m))), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(m))), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W;\n}" ::"r"(a), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* m) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(static_cast<unsigned>(__cvta_generic_to_shared(m)))
      : "memory");
}

__global__ void __launch_bounds__(kWarps * 32) bulk_kernel(const float4* w, int64_t nrows, int rb,
                                                          int64_t steps, float4* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar[kWarps][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = smem + warp * 2 * kStageBytes;
  const int per_stage = kStageBytes / rb;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (lane == 0) {
    mbar_init(&bar[warp][0], 1);
    mbar_init(&bar[warp][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t n_stages = steps * 32 / per_stage;  // rows = steps*32 per warp
  auto issue = [&](int64_t st) {
    const int b = st & 1;
    if (lane == 0) mbar_expect(&bar[warp][b], per_stage * rb);
    __syncwarp();
    for (int i = lane; i < per_stage; i += 32) {
      const int64_t r = mix(gw * steps * 32 + st * per_stage + i) & (nrows - 1);
      bulk_g2s(ring + b * kStageBytes + i * rb, reinterpret_cast<const char*>(w) + r * rb, rb,
               &bar[warp][b]);
    }
  };
  float4 acc = make_float4(0, 0, 0, 0);
  issue(0);
  for (int64_t st = 0; st < n_stages; ++st) {
    if (st + 1 < n_stages) issue(st + 1);
    mbar_wait(&bar[warp][st & 1], (st >> 1) & 1);
    const float4* p = reinterpret_cast<const float4*>(ring + (st & 1) * kStageBytes);
    for (int i = lane; i < kStageBytes / 16; i += 32) {
      const float4 v = p[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
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
  const char* names[3] = {"ldg", "rmw", "red"};
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
        const double traffic = nrow_total * rb * (mode >= 1 ? 2 : 1);
        if (rep)
          printf("%-5s row %4d B: %7.1f GB/s DRAM-equiv (%.3f ms, %.0f Mrows/s)\n", names[mode], rb,
                 traffic / ms / 1e6, ms, nrow_total / ms / 1e3);
      }
    }
  const int smem = kWarps * 2 * kStageBytes;
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int blocks_per_sm = 1; blocks_per_sm <= 3; ++blocks_per_sm)
    for (int rb = 64; rb <= 512; rb *= 2) {
      const int64_t nrows = bytes / rb;
      const int blocks = 148 * blocks_per_sm;
      const int64_t steps = 256;
      const double nrow_total = (double)blocks * kWarps * steps * 32;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        bulk_kernel<<<blocks, kWarps * 32, smem>>>(w, nrows, rb, steps, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { printf("bulk error %s\n", cudaGetErrorString(e)); return 1; }
        if (rep)
          printf("bulk  row %4d B, %d CTA/SM: %7.1f GB/s (%.3f ms, %.0f Mrows/s)\n", rb,
                 blocks_per_sm, nrow_total * rb / ms / 1e6, ms, nrow_total / ms / 1e3);
      }
    }
  return 0;
}
