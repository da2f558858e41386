// tbe.cu — hot kernels of the embedding stage on sm_100a.
//
//   K1 tbe_forward_kernel  — fused multi-table sum-pooled EmbeddingBag
//                            forward (the reference's fused_kernel stage,
//                            oracle.hpp:163-174, executed for real);
//   K4 build_keys / CUB radix sort / head select / sgd_kernel — the
//                            backward (oracle.hpp:149 bwd_comp): duplicate
//                            rows are reduced in a fixed order before one
//                            coalesced row-wise SGD write-back.
//
// Both gathers are HBM-bound random row reads. A warp is split into P
// spans (one bag / one unique row each); a span splits into GB row groups
// of L = dim/4 lanes, each lane moving one 16-byte float4 slice. Every
// group keeps U independent row loads in flight. Partial sums combine with
// a fixed xor-shuffle tree, so results are bitwise reproducible run to run.
#include <cub/cub.cuh>

#include "common.h"
#include "synth.cuh"
#include "tbe.h"

namespace sp {
namespace {

__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

__device__ __forceinline__ float4 ldg_f4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

__device__ __forceinline__ float4 shfl_xor_f4(float4 v, int m) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, m);
  v.z = __shfl_xor_sync(0xffffffffu, v.z, m);
  v.w = __shfl_xor_sync(0xffffffffu, v.w, m);
  return v;
}

// Config per dim class: L lanes per row, P spans per warp, U unroll.
template <int CLS>
struct Cfg;
template <> struct Cfg<0> { static constexpr int L = 1, P = 8, U = 4; };
template <> struct Cfg<1> { static constexpr int L = 2, P = 8, U = 4; };
template <> struct Cfg<2> { static constexpr int L = 4, P = 4, U = 4; };
template <> struct Cfg<3> { static constexpr int L = 8, P = 2, U = 4; };
template <> struct Cfg<4> { static constexpr int L = 16, P = 2, U = 8; };
template <> struct Cfg<5> { static constexpr int L = 32, P = 1, U = 8; };

// ---------------------------------------------------------------------------
// K1

// One warp: P consecutive bags [b0, b0+P) of table m.
template <int CLS>
__device__ __forceinline__ void fwd_warp(const TableMeta& m, int batch,
                                         int b0, int lane,
                                         const int32_t* __restrict__ off,
                                         const int32_t* __restrict__ idx,
                                         const float* __restrict__ w,
                                         float* __restrict__ out,
                                         int64_t ldo) {
  constexpr int L = Cfg<CLS>::L, P = Cfg<CLS>::P, U = Cfg<CLS>::U;
  constexpr int S = 32 / P, GB = S / L;
  const int span = lane / S, ls = lane % S, g = ls / L, s = ls % L;
  const int b = b0 + span;
  const bool ok = b < batch;
  int beg = 0, end = 0;
  if (ok) {
    const int64_t k = static_cast<int64_t>(m.local) * batch + b;
    beg = off[k];
    end = off[k + 1];
  }
  const float* wt = w + m.woff + 4 * s;
  const int dim = m.dim;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = beg + g; k < end; k += GB * U) {
    int r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = k + u * GB;
      r[u] = kk < end ? __ldg(idx + kk) : -1;
    }
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      v[u] = r[u] >= 0 ? ldg_f4(wt + static_cast<int64_t>(r[u]) * dim)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < U; ++u) acc = f4_add(acc, v[u]);
  }
#pragma unroll
  for (int o = L; o < S; o <<= 1) acc = f4_add(acc, shfl_xor_f4(acc, o));
  if (ok && g == 0)
    *reinterpret_cast<float4*>(out + static_cast<int64_t>(b) * ldo + m.lcol +
                               4 * s) = acc;
}

// Any dim: one warp per bag, 32 scalar columns at a time.
__device__ __forceinline__ void fwd_warp_generic(
    const TableMeta& m, int batch, int b, int lane,
    const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
    const float* __restrict__ w, float* __restrict__ out, int64_t ldo) {
  if (b >= batch) return;
  const int64_t k = static_cast<int64_t>(m.local) * batch + b;
  const int beg = off[k], end = off[k + 1];
  for (int c0 = 0; c0 < m.dim; c0 += 32) {
    const int c = c0 + lane;
    float acc = 0.f;
    for (int p = beg; p < end; ++p) {
      const int r = __ldg(idx + p);
      if (c < m.dim) acc += __ldg(w + m.woff + static_cast<int64_t>(r) * m.dim + c);
    }
    if (c < m.dim) out[static_cast<int64_t>(b) * ldo + m.lcol + c] = acc;
  }
}

__global__ void __launch_bounds__(kBlockThreads)
    tbe_forward_kernel(const TableMeta* __restrict__ meta, int n_tables,
                       int batch, const int32_t* __restrict__ off,
                       const int32_t* __restrict__ idx,
                       const float* __restrict__ w, float* __restrict__ out,
                       int64_t ldo) {
  // block -> table (meta is in grid order; block_start ascending)
  __shared__ int s_t;
  if (threadIdx.x == 0) {
    int lo = 0, hi = n_tables - 1;
    const int64_t blk = blockIdx.x;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (meta[mid].block_start <= blk) lo = mid; else hi = mid - 1;
    }
    s_t = lo;
  }
  __syncthreads();
  const TableMeta m = meta[s_t];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t blk_in_table = blockIdx.x - m.block_start;
  switch (m.cls) {
#define SP_FWD_CASE(C)                                                     \
  case C: {                                                                \
    const int b0 = static_cast<int>((blk_in_table * kWarpsPerBlock + warp) * \
                                    Cfg<C>::P);                            \
    fwd_warp<C>(m, batch, b0, lane, off, idx, w, out, ldo);                \
  } break;
    SP_FWD_CASE(0)
    SP_FWD_CASE(1)
    SP_FWD_CASE(2)
    SP_FWD_CASE(3)
    SP_FWD_CASE(4)
    SP_FWD_CASE(5)
#undef SP_FWD_CASE
    default:
      fwd_warp_generic(m, batch,
                       static_cast<int>(blk_in_table * kWarpsPerBlock + warp),
                       lane, off, idx, w, out, ldo);
  }
}

// ---------------------------------------------------------------------------
// K4 step 1: keys. A block takes 256 bags of one table, stages their
// offsets in shared memory and walks the positions coalesced.

constexpr int kKeyBags = 256;

__global__ void __launch_bounds__(kKeyBags)
    build_keys_kernel(const TableMeta* __restrict__ meta, int batch,
                      int tiles_per_table, const int32_t* __restrict__ off,
                      const int32_t* __restrict__ idx,
                      uint32_t* __restrict__ keys, uint32_t* __restrict__ bags) {
  __shared__ int32_t s_off[kKeyBags + 1];
  const int t = blockIdx.x / tiles_per_table;
  const int tile = blockIdx.x % tiles_per_table;
  const int b0 = tile * kKeyBags;
  const int nb = min(kKeyBags, batch - b0);
  const TableMeta m = meta[t];
  const int64_t base = static_cast<int64_t>(m.local) * batch + b0;
  for (int i = threadIdx.x; i <= nb; i += blockDim.x) s_off[i] = off[base + i];
  __syncthreads();
  const int p0 = s_off[0], p1 = s_off[nb];
  for (int p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    // bag = last j with s_off[j] <= p (j < nb)
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= p) lo = mid; else hi = mid - 1;
    }
    keys[p] = m.rowbase + static_cast<uint32_t>(__ldg(idx + p));
    bags[p] = static_cast<uint32_t>(b0 + lo);
  }
}

struct HeadFlag {
  const uint32_t* keys;
  __device__ __forceinline__ bool operator()(const uint32_t& k) const {
    return k == 0 || keys[k] != keys[k - 1];
  }
};

// ---------------------------------------------------------------------------
// K4 step 4: SGD. Persistent warps walk units of kSegUnit consecutive
// segments; a unit is processed in rounds of up to P segments of one table.

constexpr int kSegUnit = 32;

__device__ __forceinline__ int table_of_key(const uint32_t* __restrict__ rb_end,
                                            int n_tables, uint32_t key) {
  // first t with rowbase_end[t] > key
  int lo = 0, hi = n_tables - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rb_end[mid] > key) hi = mid; else lo = mid + 1;
  }
  return lo;
}

template <int CLS>
__device__ __forceinline__ int sgd_round(
    const TableMeta& m, uint32_t rb_end, int s, int uend, int nseg, int64_t n,
    int lane, const uint32_t* __restrict__ keys,
    const uint32_t* __restrict__ bags, const uint32_t* __restrict__ seg,
    const float* __restrict__ grad, int64_t ldg, float lr,
    float* __restrict__ w) {
  constexpr int L = Cfg<CLS>::L, P = Cfg<CLS>::P, U = Cfg<CLS>::U;
  constexpr int S = 32 / P, GB = S / L;
  const int span = lane / S, ls = lane % S, g = ls / L, sub = ls % L;
  const int u = s + span;
  bool valid = u < uend;
  int beg = 0, end = 0;
  uint32_t key = 0;
  if (valid) {
    beg = static_cast<int>(seg[u]);
    end = u + 1 < nseg ? static_cast<int>(seg[u + 1]) : static_cast<int>(n);
    key = keys[beg];
    valid = key < rb_end;
  }
  // spans must be a contiguous prefix of valid segments
  const unsigned bal = __ballot_sync(0xffffffffu, valid && ls == 0);
  int nvalid = 0;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    if (!(bal & (1u << (j * S)))) break;
    ++nvalid;
  }
  const bool active = span < nvalid;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float* wrow = nullptr;
  float4 wold = make_float4(0.f, 0.f, 0.f, 0.f);
  if (active) {
    const int64_t row = static_cast<int64_t>(key - m.rowbase);
    wrow = w + m.woff + row * m.dim + 4 * sub;
    if (g == 0) wold = *reinterpret_cast<const float4*>(wrow);
    const float* gcol = grad + m.lcol + 4 * sub;
    for (int k = beg + g; k < end; k += GB * U) {
      uint32_t bg[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int kk = k + q * GB;
        bg[q] = kk < end ? __ldg(bags + kk) : 0xffffffffu;
      }
      float4 v[U];
#pragma unroll
      for (int q = 0; q < U; ++q)
        v[q] = bg[q] != 0xffffffffu
                   ? ldg_f4(gcol + static_cast<int64_t>(bg[q]) * ldg)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < U; ++q) acc = f4_add(acc, v[q]);
    }
  }
#pragma unroll
  for (int o = L; o < S; o <<= 1) acc = f4_add(acc, shfl_xor_f4(acc, o));
  if (active && g == 0) {
    float4 r;
    r.x = fmaf(-lr, acc.x, wold.x);
    r.y = fmaf(-lr, acc.y, wold.y);
    r.z = fmaf(-lr, acc.z, wold.z);
    r.w = fmaf(-lr, acc.w, wold.w);
    *reinterpret_cast<float4*>(wrow) = r;
  }
  return nvalid;
}

__device__ __forceinline__ int sgd_round_generic(
    const TableMeta& m, int s, int nseg, int64_t n, int lane,
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ bags,
    const uint32_t* __restrict__ seg, const float* __restrict__ grad,
    int64_t ldg, float lr, float* __restrict__ w) {
  const int beg = static_cast<int>(seg[s]);
  const int end = s + 1 < nseg ? static_cast<int>(seg[s + 1]) : static_cast<int>(n);
  const int64_t row = static_cast<int64_t>(keys[beg] - m.rowbase);
  for (int c0 = 0; c0 < m.dim; c0 += 32) {
    const int c = c0 + lane;
    float acc = 0.f;
    for (int k = beg; k < end; ++k) {
      const uint32_t bg = __ldg(bags + k);
      if (c < m.dim) acc += __ldg(grad + static_cast<int64_t>(bg) * ldg + m.lcol + c);
    }
    if (c < m.dim) {
      float* p = w + m.woff + row * m.dim + c;
      *p = fmaf(-lr, acc, *p);
    }
  }
  return 1;
}

__global__ void __launch_bounds__(kBlockThreads)
    sgd_kernel(const TableMeta* __restrict__ meta,
               const uint32_t* __restrict__ rb_end, int n_tables,
               const uint32_t* __restrict__ keys,
               const uint32_t* __restrict__ bags,
               const uint32_t* __restrict__ seg,
               const int32_t* __restrict__ d_nseg, int64_t n,
               const float* __restrict__ grad, int64_t ldg, float lr,
               float* __restrict__ w) {
  const int nseg = *d_nseg;
  const int units = (nseg + kSegUnit - 1) / kSegUnit;
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int unit = gwarp; unit < units; unit += nwarps) {
    int s = unit * kSegUnit;
    const int uend = min(s + kSegUnit, nseg);
    while (s < uend) {
      const uint32_t key0 = keys[seg[s]];
      const int t = table_of_key(rb_end, n_tables, key0);
      const TableMeta m = meta[t];
      const uint32_t re = rb_end[t];
      switch (m.cls) {
#define SP_SGD_CASE(C)                                                        \
  case C:                                                                     \
    s += sgd_round<C>(m, re, s, uend, nseg, n, lane, keys, bags, seg, grad,   \
                      ldg, lr, w);                                            \
    break;
        SP_SGD_CASE(0)
        SP_SGD_CASE(1)
        SP_SGD_CASE(2)
        SP_SGD_CASE(3)
        SP_SGD_CASE(4)
        SP_SGD_CASE(5)
#undef SP_SGD_CASE
        default:
          s += sgd_round_generic(m, s, nseg, n, lane, keys, bags, seg, grad,
                                 ldg, lr, w);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Generator / layout kernels

__global__ void init_weights_kernel(float* __restrict__ w, int64_t rows,
                                    int dim, int32_t gid, uint64_t seed) {
  const int64_t n = rows * dim;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       e < n; e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / dim;
    const int c = static_cast<int>(e - r * dim);
    w[e] = weight_from_base(
        h3(seed, kTagW, static_cast<uint64_t>(gid), static_cast<uint64_t>(r)), c);
  }
}

__global__ void synth_lengths_kernel(const int32_t* __restrict__ gid,
                                     const int64_t* __restrict__ lmax,
                                     int n_tables, int batch, uint64_t seed,
                                     int32_t* __restrict__ len) {
  const int64_t n = static_cast<int64_t>(n_tables) * batch;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       k < n; k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(k / batch);
    const int64_t b = k - static_cast<int64_t>(i) * batch;
    len[k] = static_cast<int32_t>(bag_len(seed, gid[i], b, lmax[i]));
  }
}

__global__ void synth_indices_kernel(const int32_t* __restrict__ gid,
                                     const int64_t* __restrict__ rows,
                                     const uint64_t* __restrict__ thr,
                                     int n_tables, int batch, uint64_t seed,
                                     const int32_t* __restrict__ off,
                                     int32_t* __restrict__ idx) {
  const int64_t n = static_cast<int64_t>(n_tables) * batch;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       k < n; k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(k / batch);
    const int64_t b = k - static_cast<int64_t>(i) * batch;
    const uint64_t base = h3(seed, kTagIdx, static_cast<uint64_t>(gid[i]),
                             static_cast<uint64_t>(b));
    const int beg = off[k], end = off[k + 1];
    for (int p = beg; p < end; ++p)
      idx[p] = static_cast<int32_t>(bag_index(base, p - beg, rows[i], thr[i]));
  }
}

// flag bits: 1 = offsets decrease, 2 = index out of [0, rows)
__global__ void narrow_table_kernel(const int64_t* __restrict__ off64,
                                    const int64_t* __restrict__ idx64,
                                    int batch, int64_t nnz, int64_t rows,
                                    int32_t base, int32_t* __restrict__ off,
                                    int32_t* __restrict__ idx,
                                    int32_t* __restrict__ flag) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t o0 = off64[0];
  int bad = 0;
  for (int64_t b = t0; b <= batch; b += stride) {
    const int64_t a = off64[b];
    if (b < batch && off64[b + 1] < a) bad |= 1;
    off[b] = static_cast<int32_t>(a - o0) + base;
  }
  for (int64_t p = t0; p < nnz; p += stride) {
    const int64_t r = idx64[p];
    if (r < 0 || r >= rows) bad |= 2;
    idx[p] = static_cast<int32_t>(r);
  }
  if (bad) atomicOr(flag, bad);
}

__global__ void synth_grad_kernel(float* __restrict__ g, int64_t n_rows,
                                  int64_t bag0,
                                  const int32_t* __restrict__ colmap,
                                  int64_t width, uint64_t seed) {
  const int64_t n = n_rows * width;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       e < n; e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / width;
    const int64_t c = e - r * width;
    g[e] = grad_value(seed, bag0 + r, colmap[c]);
  }
}

int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 148 * 64 ? (b > 0 ? b : 1) : 148 * 64);
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers

void launch_tbe_forward(const TableMeta* d_meta, int n_tables, int64_t n_blocks,
                        int batch, const int32_t* d_off, const int32_t* d_idx,
                        const float* d_w, float* d_out, int64_t ldo,
                        cudaStream_t st) {
  if (n_blocks <= 0) return;
  tbe_forward_kernel<<<static_cast<unsigned>(n_blocks), kBlockThreads, 0, st>>>(
      d_meta, n_tables, batch, d_off, d_idx, d_w, d_out, ldo);
  SP_LAUNCHED();
}

void launch_build_keys(const TableMeta* d_meta_canon, int n_tables, int batch,
                       const int32_t* d_off, const int32_t* d_idx,
                       uint32_t* d_keys, uint32_t* d_bags, cudaStream_t st) {
  if (n_tables <= 0) return;
  const int tiles = (batch + kKeyBags - 1) / kKeyBags;
  build_keys_kernel<<<n_tables * tiles, kKeyBags, 0, st>>>(
      d_meta_canon, batch, tiles, d_off, d_idx, d_keys, d_bags);
  SP_LAUNCHED();
}

size_t sort_pairs(void* temp, size_t temp_bytes, uint32_t* keys_in,
                  uint32_t* keys_out, uint32_t* vals_in, uint32_t* vals_out,
                  int64_t n, int end_bit, cudaStream_t st) {
  size_t bytes = temp_bytes;
  SP_CUDA(cub::DeviceRadixSort::SortPairs(temp, bytes, keys_in, keys_out,
                                          vals_in, vals_out, n, 0, end_bit, st));
  return bytes;
}

size_t select_heads(void* temp, size_t temp_bytes, const uint32_t* d_keys,
                    int64_t n, uint32_t* d_seg, int32_t* d_nseg,
                    cudaStream_t st) {
  size_t bytes = temp_bytes;
  cub::CountingInputIterator<uint32_t> it(0);
  SP_CUDA(cub::DeviceSelect::If(temp, bytes, it, d_seg, d_nseg, n,
                                HeadFlag{d_keys}, st));
  return bytes;
}

size_t exclusive_scan_i32(void* temp, size_t temp_bytes, const int32_t* in,
                          int32_t* out, int64_t n, cudaStream_t st) {
  size_t bytes = temp_bytes;
  SP_CUDA(cub::DeviceScan::ExclusiveSum(temp, bytes, in, out, n, st));
  return bytes;
}

int sgd_grid(int device) {
  int sms = 148, per_sm = 1;
  SP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sgd_kernel,
                                                        kBlockThreads, 0));
  return sms * (per_sm > 0 ? per_sm : 1);
}

void launch_sgd(const TableMeta* d_meta_canon, const uint32_t* d_rowbase_end,
                int n_tables, const uint32_t* d_keys, const uint32_t* d_bags,
                const uint32_t* d_seg, const int32_t* d_nseg, int64_t n,
                const float* d_grad, int64_t ldg, float lr, float* d_w,
                int grid, cudaStream_t st) {
  if (n <= 0 || n_tables <= 0) return;
  sgd_kernel<<<grid, kBlockThreads, 0, st>>>(d_meta_canon, d_rowbase_end,
                                             n_tables, d_keys, d_bags, d_seg,
                                             d_nseg, n, d_grad, ldg, lr, d_w);
  SP_LAUNCHED();
}

void launch_init_weights(float* d_w, int64_t rows, int dim, int32_t gid,
                         uint64_t seed, cudaStream_t st) {
  init_weights_kernel<<<grid_for(rows * dim, 256), 256, 0, st>>>(d_w, rows, dim,
                                                                  gid, seed);
  SP_LAUNCHED();
}

void launch_synth_lengths(const int32_t* d_gid, const int64_t* d_lmax,
                          int n_tables, int batch, uint64_t seed,
                          int32_t* d_len, cudaStream_t st) {
  synth_lengths_kernel<<<grid_for(static_cast<int64_t>(n_tables) * batch, 256),
                         256, 0, st>>>(d_gid, d_lmax, n_tables, batch, seed,
                                       d_len);
  SP_LAUNCHED();
}

void launch_synth_indices(const int32_t* d_gid, const int64_t* d_rows,
                          const uint64_t* d_thr, int n_tables, int batch,
                          uint64_t seed, const int32_t* d_off, int32_t* d_idx,
                          cudaStream_t st) {
  synth_indices_kernel<<<grid_for(static_cast<int64_t>(n_tables) * batch, 256),
                         256, 0, st>>>(d_gid, d_rows, d_thr, n_tables, batch,
                                       seed, d_off, d_idx);
  SP_LAUNCHED();
}

void launch_narrow_table(const int64_t* d_off64, const int64_t* d_idx64,
                         int batch, int64_t nnz, int64_t rows, int32_t base,
                         int32_t* d_off, int32_t* d_idx, int32_t* d_flag,
                         cudaStream_t st) {
  const int64_t n = nnz > batch ? nnz : batch;
  narrow_table_kernel<<<grid_for(n, 256), 256, 0, st>>>(
      d_off64, d_idx64, batch, nnz, rows, base, d_off, d_idx, d_flag);
  SP_LAUNCHED();
}

void launch_synth_grad(float* d_grad, int64_t n_rows, int64_t bag0,
                       const int32_t* d_colmap, int64_t width, uint64_t seed,
                       cudaStream_t st) {
  if (n_rows * width <= 0) return;
  synth_grad_kernel<<<grid_for(n_rows * width, 256), 256, 0, st>>>(
      d_grad, n_rows, bag0, d_colmap, width, seed);
  SP_LAUNCHED();
}

}  // namespace sp
