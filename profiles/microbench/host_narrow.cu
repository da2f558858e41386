// host_narrow.cu — can the host narrow an int64 LookupBatch to int32 faster
// than PCIe moves the int64 bytes? (e2e path design question.)
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a host_narrow.cu -o host_narrow
// Measures: (a) pinned int64 H2D rate; (b) host narrowing rate with N
// threads (pinned int64 -> pinned int32); (c) narrowing pipelined with the
// int32 H2D (chunks of 8 MB int32, 4 slots, N threads).
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

static void narrow_range(const int64_t* in, int32_t* out, int64_t n, int* bad) {
  int b = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t v = in[i];
    b |= (v >> 31) != 0;
    out[i] = static_cast<int32_t>(v);
  }
  *bad |= b;
}

static void narrow_mt(const int64_t* in, int32_t* out, int64_t n, int nt) {
  std::vector<std::thread> th;
  std::vector<int> bad(nt, 0);
  const int64_t per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int64_t a = t * per, e = std::min(n, a + per);
    if (a < e) th.emplace_back(narrow_range, in + a, out + a, e - a, &bad[t]);
  }
  for (auto& x : th) x.join();
}

int main() {
  const int64_t n = 50'000'000;  // ~ cfg3's 45 M indices + 6.5 M offsets
  int64_t* in = nullptr;
  int32_t* out = nullptr;
  cudaMallocHost(&in, n * 8);
  cudaMallocHost(&out, n * 4);
  for (int64_t i = 0; i < n; ++i) in[i] = (i * 2654435761ll) & 0xfffff;
  int64_t* d64 = nullptr;
  cudaMalloc(&d64, n * 8);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0, st);
    cudaMemcpyAsync(d64, in, n * 8, cudaMemcpyHostToDevice, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("H2D int64 %.0f MB: %.2f ms = %.1f GB/s\n", n * 8 / 1e6, ms, n * 8 / ms / 1e6);
  }
  const unsigned hw = std::thread::hardware_concurrency();
  std::printf("hardware_concurrency %u\n", hw);
  for (int nt : {1, 2, 4, 8, 16, 32}) {
    if (nt > static_cast<int>(hw) * 2) break;
    narrow_mt(in, out, n, nt);
    const double t0 = now();
    for (int r = 0; r < 3; ++r) narrow_mt(in, out, n, nt);
    const double dt = (now() - t0) / 3;
    std::printf("narrow %2d threads: %.2f ms = %.1f GB/s of int64 input\n", nt, dt * 1e3,
                n * 8 / dt / 1e9);
  }
  // (c) pipelined: chunks narrowed by nt threads into 4 pinned int32 slots,
  // each slot's H2D queued as soon as it is narrowed
  int32_t* d32 = reinterpret_cast<int32_t*>(d64);
  const int64_t chunk = int64_t(4) << 20;  // int32 elements per slot (16 MB)
  int32_t* slots = nullptr;
  cudaMallocHost(&slots, 4 * chunk * 4);
  cudaEvent_t sev[4];
  for (auto& e : sev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (int nt : {4, 8, 16}) {
    if (nt > static_cast<int>(hw)) break;
    for (int r = 0; r < 3; ++r) {
      bool used[4] = {};
      const double t0 = now();
      int k = 0;
      for (int64_t a = 0; a < n; a += chunk, k = (k + 1) % 4) {
        const int64_t m = std::min(chunk, n - a);
        if (used[k]) cudaEventSynchronize(sev[k]);
        narrow_mt(in + a, slots + k * chunk, m, nt);
        cudaMemcpyAsync(d32 + a, slots + k * chunk, m * 4, cudaMemcpyHostToDevice, st);
        cudaEventRecord(sev[k], st);
        used[k] = true;
      }
      cudaStreamSynchronize(st);
      const double dt = now() - t0;
      std::printf("pipelined narrow+H2D %2d threads: %.2f ms (int64 H2D would take %.2f ms)\n",
                  nt, dt * 1e3, n * 8 / 55e9 * 1e3);
    }
  }
  return 0;
}
