// tbe.cu — hot kernels of the embedding stage on sm_100a.
//
//   K1 tbe_forward_kernel — fused multi-table sum-pooled EmbeddingBag
//      forward (the reference's fused_kernel stage, oracle.hpp:163-174,
//      executed for real). Optionally emits the backward's sort keys.
//   K4 build_keys (when K1 did not emit them) -> CUB stable radix sort ->
//      sgd_kernel — the backward (oracle.hpp:149 bwd_comp): duplicate rows
//      are reduced in the sorted (= original) order before one coalesced
//      row-wise SGD write-back.
//
// Both are HBM-bound random row gathers. Each block owns a tile: K1 a run
// of consecutive bags of one table, K4 a run of sorted positions. The tile's
// offsets/indices (K1) or keys/bags (K4) are staged in shared memory with
// coalesced loads, so the only long-latency dependency left per bag/row is
// the row gather itself. A warp is split into P spans (one bag / one unique
// row each); a span splits into GB groups of L = dim/4 lanes, each lane
// moving one 16-byte float4 slice, U rows in flight per group. Partial
// sums combine with a fixed xor-shuffle tree: bitwise reproducible.
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

// L2 eviction-priority policies (createpolicy) for loads that should stay
// resident (the per-table gradient slice in K4) or stream through.
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ float4 ldg_f4_policy(const float* ptr, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(ptr), "l"(pol));
  return v;
}

#ifndef SP_SGD_RED  // 1: apply the row update as red.global.add.v4.f32 (no W load)
#define SP_SGD_RED 1
#endif
// Vector reduction at L2: fire-and-forget, the SM never waits for the row
// (each unique row has exactly one update per launch, so the result is
// deterministic: W + fp32(-lr * sum), round-to-nearest at L2). Measured on
// B200 at cfg3: SGD 2.51 -> 2.33 ms with the old geometry, and it frees the
// registers that held the old row for more rows/positions in flight.
__device__ __forceinline__ void red_add_f4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ float4 shfl_xor_f4(float4 v, int m) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, m);
  v.z = __shfl_xor_sync(0xffffffffu, v.z, m);
  v.w = __shfl_xor_sync(0xffffffffu, v.w, m);
  return v;
}

// Geometry per dim class (dim = 4, 8, 16, 32, 64, 128 for class 0..5):
// a row is split over L lanes, each lane moving V float4 (16V bytes); a
// warp holds P spans (one bag / one unique row each) of 32/P lanes; a span
// holds GB = (32/P)/L row groups, each keeping U rows in flight.
template <int L_, int V_, int P_, int U_>
struct Geo {
  static constexpr int L = L_, V = V_, P = P_, U = U_;
  static constexpr int S = 32 / P, GB = S / L;
  static_assert(S % L == 0 && GB >= 1, "bad geometry");
};
// K1: bags are ~2*pf long; GB*U rows of a bag in flight.
template <int CLS> struct FwdGeo;
template <> struct FwdGeo<0> : Geo<1, 1, 8, 4> {};
template <> struct FwdGeo<1> : Geo<2, 1, 8, 4> {};
template <> struct FwdGeo<2> : Geo<4, 1, 4, 4> {};
template <> struct FwdGeo<3> : Geo<8, 1, 2, 4> {};
template <> struct FwdGeo<4> : Geo<16, 1, 2, 8> {};
template <> struct FwdGeo<5> : Geo<32, 1, 1, 8> {};
// K4 SGD: most runs hold 1-2 positions, so more runs per warp (P) matter
// more than rows per run; lanes move up to 64 B of a row.
template <int CLS> struct SgdGeo;
#ifdef SP_GEO_HEADER  // A/B builds: -DSP_GEO_HEADER=\"geo.h\" overriding the knobs below
#include SP_GEO_HEADER
#endif
#ifndef SP_SGD_G0
// (L, V, P, U) per dim class; tuned on B200 at cfg3 (profiles/r01_notes.md).
// With the L2 reduction update no register holds the old row, so lanes take
// 64 B of a row (V = 4) for dims >= 64 and every group keeps U = 2
// positions in flight: SGD 2.33 -> 2.09 ms.
#define SP_SGD_G0 1, 1, 16, 2
#define SP_SGD_G1 2, 1, 16, 1
#define SP_SGD_G2 2, 2, 16, 2
#define SP_SGD_G3 4, 2, 8, 2
#define SP_SGD_G4 4, 4, 8, 2
#define SP_SGD_G5 8, 4, 4, 2
#endif
#ifndef SP_SGD_INTERLEAVE  // lane float4 slices: 1 interleaved (s, s+L, ..), 0 blocked
#define SP_SGD_INTERLEAVE 1
#endif
template <> struct SgdGeo<0> : Geo<SP_SGD_G0> {};
template <> struct SgdGeo<1> : Geo<SP_SGD_G1> {};
template <> struct SgdGeo<2> : Geo<SP_SGD_G2> {};
template <> struct SgdGeo<3> : Geo<SP_SGD_G3> {};
template <> struct SgdGeo<4> : Geo<SP_SGD_G4> {};
template <> struct SgdGeo<5> : Geo<SP_SGD_G5> {};
// K4 SGD, long runs (hot rows): the whole warp on one run.
template <int CLS> struct LongGeo;
template <> struct LongGeo<0> : Geo<1, 1, 1, 4> {};
template <> struct LongGeo<1> : Geo<2, 1, 1, 4> {};
template <> struct LongGeo<2> : Geo<4, 1, 1, 4> {};
template <> struct LongGeo<3> : Geo<8, 1, 1, 4> {};
template <> struct LongGeo<4> : Geo<16, 1, 1, 8> {};
template <> struct LongGeo<5> : Geo<32, 1, 1, 8> {};

// ---------------------------------------------------------------------------
// K1

struct FwdTile {
  int32_t t;   // canonical local table index
  int32_t b0;  // first bag
  int32_t nb;  // bags in the tile
  int32_t pad;
};

constexpr int kTileBags = 256;
constexpr int kIdxCap = 4096;  // staged indices per tile (16 KB)

template <class G>
__device__ __forceinline__ void fwd_tile_warp(const TableMeta& m, int b0, int nb,
                                              int p0, int warp, int lane,
                                              const int32_t* s_off,
                                              const int32_t* s_idx,
                                              const int32_t* __restrict__ idx,
                                              const float* __restrict__ w,
                                              float* __restrict__ out,
                                              int64_t ldo) {
  constexpr int L = G::L, V = G::V, P = G::P, U = G::U, S = G::S, GB = G::GB;
  const int span = lane / S, ls = lane % S, g = ls / L, s = ls % L;
  const float* wt = w + m.woff + 4 * s;  // lane s moves float4 s, s+L, s+2L, ... (coalesced)
  const int dim = m.dim;
  for (int bg = warp * P; bg < nb; bg += kWarpsPerBlock * P) {
    const int bag = bg + span;
    const bool ok = bag < nb;
    int beg = 0, end = 0;
    if (ok) {
      beg = s_off[bag] - p0;
      end = s_off[bag + 1] - p0;
    }
    float4 acc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = beg + g; k < end; k += GB * U) {
      int r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k + u * GB;
        r[u] = kk < end ? (kk < kIdxCap ? s_idx[kk] : __ldg(idx + p0 + kk)) : -1;
      }
      float4 v[U][V];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j)
          v[u][j] = r[u] >= 0 ? ldg_f4(wt + static_cast<int64_t>(r[u]) * dim + 4 * L * j)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = f4_add(acc[j], v[u][j]);
    }
#pragma unroll
    for (int o = L; o < S; o <<= 1)
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = f4_add(acc[j], shfl_xor_f4(acc[j], o));
    if (ok && g == 0) {
      float* o = out + static_cast<int64_t>(b0 + bag) * ldo + m.lcol + 4 * s;
#pragma unroll
      for (int j = 0; j < V; ++j) __stcs(reinterpret_cast<float4*>(o + 4 * L * j), acc[j]);
    }
  }
}

// Any dim: one warp per bag, 32 scalar columns at a time.
__device__ __forceinline__ void fwd_tile_warp_generic(
    const TableMeta& m, int b0, int nb, int p0, int warp, int lane,
    const int32_t* s_off, const int32_t* s_idx, const int32_t* __restrict__ idx,
    const float* __restrict__ w, float* __restrict__ out, int64_t ldo) {
  for (int bag = warp; bag < nb; bag += kWarpsPerBlock) {
    const int beg = s_off[bag] - p0, end = s_off[bag + 1] - p0;
    for (int c0 = 0; c0 < m.dim; c0 += 32) {
      const int c = c0 + lane;
      float acc = 0.f;
      for (int k = beg; k < end; ++k) {
        const int r = k < kIdxCap ? s_idx[k] : __ldg(idx + p0 + k);
        if (c < m.dim) acc += __ldg(w + m.woff + static_cast<int64_t>(r) * m.dim + c);
      }
      if (c < m.dim) out[static_cast<int64_t>(b0 + bag) * ldo + m.lcol + c] = acc;
    }
  }
}

// BagT: the sort payload — uint16_t when the batch fits 16 bits (6-byte
// pairs through the radix sort instead of 8), else uint32_t.
template <bool kEmitKeys, class BagT>
__global__ void __launch_bounds__(kBlockThreads)
    tbe_forward_kernel(const TableMeta* __restrict__ meta,
                       const FwdTile* __restrict__ tiles, int batch,
                       const int32_t* __restrict__ off,
                       const int32_t* __restrict__ idx,
                       const float* __restrict__ w, float* __restrict__ out,
                       int64_t ldo, uint32_t* __restrict__ keys,
                       BagT* __restrict__ bags) {
  __shared__ int32_t s_off[kTileBags + 1];
  __shared__ int32_t s_idx[kIdxCap];
  const FwdTile tile = tiles[blockIdx.x];
  const TableMeta m = meta[tile.t];
  const int64_t base = static_cast<int64_t>(tile.t) * batch + tile.b0;
  for (int i = threadIdx.x; i <= tile.nb; i += kBlockThreads) s_off[i] = off[base + i];
  __syncthreads();
  const int p0 = s_off[0];
  const int np = s_off[tile.nb] - p0;
  for (int i = threadIdx.x; i < np; i += kBlockThreads) {
    const int32_t v = __ldg(idx + p0 + i);
    if (i < kIdxCap) s_idx[i] = v;
    if (kEmitKeys) {
      // bag of position i: last j with s_off[j] <= p0 + i
      int lo = 0, hi = tile.nb - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_off[mid] <= p0 + i) lo = mid; else hi = mid - 1;
      }
      __stcs(keys + p0 + i, m.rowbase + static_cast<uint32_t>(v));
      bags[p0 + i] = static_cast<BagT>(tile.b0 + lo);
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  switch (m.cls) {
#define SP_FWD_CASE(C)                                                         \
  case C:                                                                      \
    fwd_tile_warp<FwdGeo<C>>(m, tile.b0, tile.nb, p0, warp, lane, s_off, s_idx, \
                             idx, w, out, ldo);                                \
    break;
    SP_FWD_CASE(0)
    SP_FWD_CASE(1)
    SP_FWD_CASE(2)
    SP_FWD_CASE(3)
    SP_FWD_CASE(4)
    SP_FWD_CASE(5)
#undef SP_FWD_CASE
    default:
      fwd_tile_warp_generic(m, tile.b0, tile.nb, p0, warp, lane, s_off, s_idx, idx,
                            w, out, ldo);
  }
}

// ---------------------------------------------------------------------------
// K4 step 1 (only when K1 did not emit them): keys[p] = rowbase + idx[p],
// bags[p] = bag of p. A block takes 256 bags of one table.

template <class BagT>
__global__ void __launch_bounds__(kTileBags)
    build_keys_kernel(const TableMeta* __restrict__ meta, int batch,
                      int tiles_per_table, const int32_t* __restrict__ off,
                      const int32_t* __restrict__ idx,
                      uint32_t* __restrict__ keys, BagT* __restrict__ bags) {
  __shared__ int32_t s_off[kTileBags + 1];
  const int t = blockIdx.x / tiles_per_table;
  const int tile = blockIdx.x % tiles_per_table;
  const int b0 = tile * kTileBags;
  const int nb = min(kTileBags, batch - b0);
  const TableMeta m = meta[t];
  const int64_t base = static_cast<int64_t>(m.local) * batch + b0;
  for (int i = threadIdx.x; i <= nb; i += blockDim.x) s_off[i] = off[base + i];
  __syncthreads();
  const int p0 = s_off[0], p1 = s_off[nb];
  for (int p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= p) lo = mid; else hi = mid - 1;
    }
    keys[p] = m.rowbase + static_cast<uint32_t>(__ldg(idx + p));
    bags[p] = static_cast<BagT>(b0 + lo);
  }
}

struct HeadFlag {
  const uint32_t* keys;
  __device__ __forceinline__ bool operator()(const uint32_t& k) const {
    return k == 0 || keys[k] != keys[k - 1];
  }
};

// ---------------------------------------------------------------------------
// K4 step 3: SGD over the sorted (key, bag) pairs. A block owns the run
// heads inside its tile of kTilePos sorted positions (a run that starts in
// the tile is finished by the tile's block even past the tile end; a run
// that started earlier belongs to the previous tile). Keys/bags/heads are
// staged in shared memory; warps take contiguous slices of the tile's runs
// and process them in rounds of up to P runs of the same table.

constexpr int kTilePos = 2048;
constexpr int kPosPerThread = kTilePos / kBlockThreads;
constexpr int kMaxSmemTables = 512;

constexpr int kRunChunk = 16;  // runs claimed per warp at a time (>= max P)
constexpr int kLongRun = 32;   // runs at least this long get the whole warp

struct SgdShared {
  uint32_t key[kTilePos];
  uint32_t bag[kTilePos];
  uint16_t head[kTilePos + 1];
  uint32_t rb_end[kMaxSmemTables];
  int64_t gstart[kMaxSortGroups + 1];  // sort groups: first position
  int32_t gt0[kMaxSortGroups + 1];     //              first local table
  int ngroups;
  int nhead;
  int last_end;  // end (tile-relative) of the last run
  int next;      // next unclaimed run
};

// Keys are relative to their sort group; a group start always begins a run.
__device__ __forceinline__ bool is_group_start(const SgdShared& sh, int64_t p) {
  for (int g = 1; g < sh.ngroups; ++g)
    if (sh.gstart[g] == p) return true;
  return false;
}

__device__ __forceinline__ int group_of(const SgdShared& sh, int64_t p) {
  int g = 0;
  while (g + 1 < sh.ngroups && sh.gstart[g + 1] <= p) ++g;
  return g;
}

__device__ __forceinline__ int table_of_key(const uint32_t* rb_end, int n_tables,
                                            uint32_t key) {
  int lo = 0, hi = n_tables - 1;  // first t with rb_end[t] > key
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rb_end[mid] > key) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t pos_key(const SgdShared& sh, int i, int np,
                                            int64_t p0,
                                            const uint32_t* __restrict__ keys) {
  return i < np ? sh.key[i] : __ldg(keys + p0 + i);
}

template <class BagT>
__device__ __forceinline__ uint32_t pos_bag(const SgdShared& sh, int i, int np,
                                            int64_t p0,
                                            const BagT* __restrict__ bags) {
  return i < np ? sh.bag[i] : static_cast<uint32_t>(__ldg(bags + p0 + i));
}

// One round: runs [j, j+P) of the tile's head list that belong to table m.
template <class G, class BagT>
__device__ __forceinline__ int sgd_round(const TableMeta& m, uint32_t rb_end, int gend,
                                         int j, int jend, int np, int64_t p0,
                                         int lane, const SgdShared& sh,
                                         const BagT* __restrict__ bags,
                                         const float* __restrict__ grad,
                                         int64_t ldg, float lr,
                                         float* __restrict__ w) {
  constexpr int L = G::L, V = G::V, P = G::P, U = G::U, S = G::S, GB = G::GB;
  const int span = lane / S, ls = lane % S, g = ls / L, sub = ls % L;
  constexpr int kLane = SP_SGD_INTERLEAVE ? 1 : V, kStep = SP_SGD_INTERLEAVE ? L : 1;
  const int u = j + span;
  bool valid = u < jend;
  int beg = 0, end = 0;
  uint32_t key = 0;
  if (valid) {
    beg = sh.head[u];
    end = u + 1 < sh.nhead ? sh.head[u + 1] : sh.last_end;
    key = sh.key[beg];
    // same table (and sort group); a long run (other than the first) gets
    // its own round
    valid = key < rb_end && beg < gend && (span == 0 || end - beg < kLongRun);
  }
  const unsigned bal = __ballot_sync(0xffffffffu, valid && ls == 0);
  // spans must be a contiguous prefix of valid runs
  int nvalid = 0;
#pragma unroll
  for (int q = 0; q < P; ++q) {
    if (!(bal & (1u << (q * S)))) break;
    ++nvalid;
  }
  const bool active = span < nvalid;
  float4 acc[V], wold[V];
#pragma unroll
  for (int q = 0; q < V; ++q) {
    acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    wold[q] = acc[q];
  }
  float* wrow = nullptr;
  if (active) {
    const int64_t row = static_cast<int64_t>(key - m.rowbase);
    wrow = w + m.woff + row * m.dim + 4 * kLane * sub;
    if (g == 0 && !SP_SGD_RED)
#pragma unroll
      for (int q = 0; q < V; ++q) wold[q] = *reinterpret_cast<const float4*>(wrow + 4 * kStep * q);
    const float* gcol = grad + m.lcol + 4 * kLane * sub;
    for (int k = beg + g; k < end; k += GB * U) {
      uint32_t bg[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int kk = k + q * GB;
        bg[q] = kk < end ? pos_bag(sh, kk, np, p0, bags) : 0xffffffffu;
      }
      float4 v[U][V];
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int c = 0; c < V; ++c)
          v[q][c] = bg[q] != 0xffffffffu
                        ? ldg_f4(gcol + static_cast<int64_t>(bg[q]) * ldg + 4 * kStep * c)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int c = 0; c < V; ++c) acc[c] = f4_add(acc[c], v[q][c]);
    }
  }
#pragma unroll
  for (int o = L; o < S; o <<= 1)
#pragma unroll
    for (int c = 0; c < V; ++c) acc[c] = f4_add(acc[c], shfl_xor_f4(acc[c], o));
  if (active && g == 0) {
#pragma unroll
    for (int c = 0; c < V; ++c) {
      float4 r;
      if (SP_SGD_RED) {
        r = make_float4(-lr * acc[c].x, -lr * acc[c].y, -lr * acc[c].z, -lr * acc[c].w);
        red_add_f4(wrow + 4 * kStep * c, r);
        continue;
      }
      r.x = fmaf(-lr, acc[c].x, wold[c].x);
      r.y = fmaf(-lr, acc[c].y, wold[c].y);
      r.z = fmaf(-lr, acc[c].z, wold[c].z);
      r.w = fmaf(-lr, acc[c].w, wold[c].w);
      *reinterpret_cast<float4*>(wrow + 4 * kStep * c) = r;
    }
  }
  return nvalid;
}

template <class BagT>
__device__ __forceinline__ int sgd_round_generic(
    const TableMeta& m, int j, int np, int64_t p0, int lane, const SgdShared& sh,
    const BagT* __restrict__ bags, const float* __restrict__ grad, int64_t ldg,
    float lr, float* __restrict__ w) {
  const int beg = sh.head[j];
  const int end = j + 1 < sh.nhead ? sh.head[j + 1] : sh.last_end;
  const int64_t row = static_cast<int64_t>(sh.key[beg] - m.rowbase);
  for (int c0 = 0; c0 < m.dim; c0 += 32) {
    const int c = c0 + lane;
    float acc = 0.f;
    for (int k = beg; k < end; ++k) {
      const uint32_t bg = pos_bag(sh, k, np, p0, bags);
      if (c < m.dim) acc += __ldg(grad + static_cast<int64_t>(bg) * ldg + m.lcol + c);
    }
    if (c < m.dim) {
      float* p = w + m.woff + row * m.dim + c;
      *p = fmaf(-lr, acc, *p);
    }
  }
  return 1;
}

#ifndef SP_SGD_MIN_BLOCKS
#define SP_SGD_MIN_BLOCKS 4  // 4 x 256 threads per SM: <= 64 registers
#endif
template <class BagT>
__global__ void __launch_bounds__(kBlockThreads, SP_SGD_MIN_BLOCKS)
    sgd_kernel(const TableMeta* __restrict__ meta,
               const uint32_t* __restrict__ rb_end_g, int n_tables,
               const int64_t* __restrict__ gstart_g, const int32_t* __restrict__ gt0_g,
               int n_groups, const uint32_t* __restrict__ keys,
               const BagT* __restrict__ bags, int64_t n,
               const float* __restrict__ grad, int64_t ldg, float lr,
               float* __restrict__ w) {
  __shared__ SgdShared sh;
  using BlockScan = cub::BlockScan<int, kBlockThreads>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * kTilePos;
  const int np = n - p0 < kTilePos ? static_cast<int>(n - p0) : kTilePos;
  const int tid = threadIdx.x;
  for (int i = tid; i < np; i += kBlockThreads) {
    sh.key[i] = __ldg(keys + p0 + i);
    sh.bag[i] = __ldg(bags + p0 + i);
  }
  const bool rb_in_smem = n_tables <= kMaxSmemTables;
  if (rb_in_smem)
    for (int i = tid; i < n_tables; i += kBlockThreads) sh.rb_end[i] = rb_end_g[i];
  if (tid <= n_groups) {
    sh.gstart[tid] = gstart_g[tid];
    sh.gt0[tid] = gt0_g[tid];
  }
  if (tid == 0) sh.ngroups = n_groups;
  const uint32_t prev = p0 > 0 ? __ldg(keys + p0 - 1) : 0xffffffffu;
  __syncthreads();
  // run heads of the tile (tile-relative positions), in order
  int flags[kPosPerThread];
  int cnt = 0;
#pragma unroll
  for (int q = 0; q < kPosPerThread; ++q) {
    const int i = tid * kPosPerThread + q;
    const uint32_t before = i == 0 ? prev : sh.key[i - 1];
    flags[q] = (i < np && (sh.key[i] != before || (p0 == 0 && i == 0) ||
                           is_group_start(sh, p0 + i)))
                   ? 1 : 0;
    cnt += flags[q];
  }
  int first = 0, total = 0;
  BlockScan(scan_tmp).ExclusiveSum(cnt, first, total);
#pragma unroll
  for (int q = 0; q < kPosPerThread; ++q)
    if (flags[q]) sh.head[first++] = static_cast<uint16_t>(tid * kPosPerThread + q);
  if (tid == 0) {
    sh.nhead = total;
    sh.next = 0;
  }
  // end of the last run: it may continue past the tile
  if (tid < 32) {
    int end = np;
    if (total > 0 && p0 + np < n) {
      // all lanes: scan forward until the key changes
      const uint32_t last_key = sh.key[np - 1];
      for (int64_t base = p0 + np;; base += 32) {
        const int64_t p = base + tid;
        const bool diff = p >= n || __ldg(keys + p) != last_key || is_group_start(sh, p);
        const unsigned bal = __ballot_sync(0xffffffffu, diff);
        if (bal) {
          end = static_cast<int>(base - p0) + __ffs(bal) - 1;
          break;
        }
      }
    }
    if (tid == 0) sh.last_end = end;
  }
  __syncthreads();
  const int nh = sh.nhead;
  if (nh == 0) return;
  const int lane = tid & 31;
  const uint32_t* rb = rb_in_smem ? sh.rb_end : rb_end_g;
  // Warps claim chunks of kRunChunk runs dynamically (hot rows make run
  // lengths very uneven). Inside a chunk: short runs go P at a time, a long
  // run gets the whole warp (all row groups, U rows each in flight).
  for (;;) {
    int j0 = 0;
    if (lane == 0) j0 = atomicAdd(&sh.next, kRunChunk);
    j0 = __shfl_sync(0xffffffffu, j0, 0);
    if (j0 >= nh) break;
    const int jend = min(nh, j0 + kRunChunk);
    int j = j0;
    while (j < jend) {
      const int beg = sh.head[j];
      const int len = (j + 1 < nh ? sh.head[j + 1] : sh.last_end) - beg;
      const uint32_t key0 = sh.key[beg];
      const int grp = group_of(sh, p0 + beg);
      const int gt = sh.gt0[grp];
      const int t = gt + table_of_key(rb + gt, sh.gt0[grp + 1] - gt, key0);
      const TableMeta m = meta[t];
      const uint32_t re = rb[t];
      // runs of this round stay in the group (keys restart at a group start)
      const int gend = sh.gstart[grp + 1] - p0 < kTilePos + 1
                           ? static_cast<int>(sh.gstart[grp + 1] - p0) : kTilePos + 1;
      const bool lng = len >= kLongRun;
      switch (m.cls) {
#define SP_SGD_CASE(C)                                                           \
  case C:                                                                        \
    j += lng ? sgd_round<LongGeo<C>, BagT>(m, re, gend, j, j + 1, np, p0, lane,  \
                                           sh, bags, grad, ldg, lr, w)           \
             : sgd_round<SgdGeo<C>, BagT>(m, re, gend, j, jend, np, p0, lane, sh, \
                                          bags, grad, ldg, lr, w);               \
    break;
        SP_SGD_CASE(0)
        SP_SGD_CASE(1)
        SP_SGD_CASE(2)
        SP_SGD_CASE(3)
        SP_SGD_CASE(4)
        SP_SGD_CASE(5)
#undef SP_SGD_CASE
        default:
          j += sgd_round_generic(m, j, np, p0, lane, sh, bags, grad, ldg, lr, w);
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

std::vector<int4> make_fwd_tiles(const std::vector<TableMeta>& canon,
                                 const std::vector<int>& order, int batch) {
  std::vector<int4> tiles;
  for (int li : order)
    for (int b0 = 0; b0 < batch; b0 += kTileBags)
      tiles.push_back(make_int4(canon[li].local, b0, std::min(kTileBags, batch - b0), 0));
  return tiles;
}

void launch_tbe_forward(const TableMeta* d_meta_canon, const int4* d_tiles,
                        int64_t n_tiles, int batch, const int32_t* d_off,
                        const int32_t* d_idx, const float* d_w, float* d_out,
                        int64_t ldo, uint32_t* d_keys, void* d_bags, bool bags16,
                        cudaStream_t st) {
  if (n_tiles <= 0) return;
  const FwdTile* tiles = reinterpret_cast<const FwdTile*>(d_tiles);
  const unsigned g = static_cast<unsigned>(n_tiles);
  if (!d_keys)
    tbe_forward_kernel<false, uint32_t><<<g, kBlockThreads, 0, st>>>(
        d_meta_canon, tiles, batch, d_off, d_idx, d_w, d_out, ldo, nullptr, nullptr);
  else if (bags16)
    tbe_forward_kernel<true, uint16_t><<<g, kBlockThreads, 0, st>>>(
        d_meta_canon, tiles, batch, d_off, d_idx, d_w, d_out, ldo, d_keys,
        static_cast<uint16_t*>(d_bags));
  else
    tbe_forward_kernel<true, uint32_t><<<g, kBlockThreads, 0, st>>>(
        d_meta_canon, tiles, batch, d_off, d_idx, d_w, d_out, ldo, d_keys,
        static_cast<uint32_t*>(d_bags));
  SP_LAUNCHED();
}

void launch_build_keys(const TableMeta* d_meta_canon, int n_tables, int batch,
                       const int32_t* d_off, const int32_t* d_idx,
                       uint32_t* d_keys, void* d_bags, bool bags16, cudaStream_t st) {
  if (n_tables <= 0) return;
  const int tiles = (batch + kTileBags - 1) / kTileBags;
  if (bags16)
    build_keys_kernel<uint16_t><<<n_tables * tiles, kTileBags, 0, st>>>(
        d_meta_canon, batch, tiles, d_off, d_idx, d_keys, static_cast<uint16_t*>(d_bags));
  else
    build_keys_kernel<uint32_t><<<n_tables * tiles, kTileBags, 0, st>>>(
        d_meta_canon, batch, tiles, d_off, d_idx, d_keys, static_cast<uint32_t*>(d_bags));
  SP_LAUNCHED();
}

size_t sort_pairs(void* temp, size_t temp_bytes, const uint32_t* keys_in,
                  uint32_t* keys_out, const void* vals_in, void* vals_out, bool bags16,
                  int64_t n, int end_bit, cudaStream_t st) {
  size_t bytes = temp_bytes;
  if (bags16)
    SP_CUDA(cub::DeviceRadixSort::SortPairs(temp, bytes, keys_in, keys_out,
                                            static_cast<const uint16_t*>(vals_in),
                                            static_cast<uint16_t*>(vals_out), n, 0, end_bit, st));
  else
    SP_CUDA(cub::DeviceRadixSort::SortPairs(temp, bytes, keys_in, keys_out,
                                            static_cast<const uint32_t*>(vals_in),
                                            static_cast<uint32_t*>(vals_out), n, 0, end_bit, st));
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

void launch_sgd(const TableMeta* d_meta_canon, const uint32_t* d_rowbase_end,
                int n_tables, const int64_t* d_gstart, const int32_t* d_gt0, int n_groups,
                const uint32_t* d_keys, const void* d_bags, bool bags16,
                int64_t n, const float* d_grad, int64_t ldg, float lr, float* d_w,
                cudaStream_t st) {
  if (n <= 0 || n_tables <= 0) return;
  if (n_groups > kMaxSortGroups) raise(SP_ERR_BAD_INPUT, "too many sort groups");
  const unsigned blocks = static_cast<unsigned>((n + kTilePos - 1) / kTilePos);
  if (bags16)
    sgd_kernel<uint16_t><<<blocks, kBlockThreads, 0, st>>>(
        d_meta_canon, d_rowbase_end, n_tables, d_gstart, d_gt0, n_groups, d_keys,
        static_cast<const uint16_t*>(d_bags), n, d_grad, ldg, lr, d_w);
  else
    sgd_kernel<uint32_t><<<blocks, kBlockThreads, 0, st>>>(
        d_meta_canon, d_rowbase_end, n_tables, d_gstart, d_gt0, n_groups, d_keys,
        static_cast<const uint32_t*>(d_bags), n, d_grad, ldg, lr, d_w);
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
