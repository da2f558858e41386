// tbe.cu — hot kernels of the embedding stage on sm_100a.
//
//   K1 tbe_forward_kernel — fused multi-table sum-pooled EmbeddingBag
//      forward (the reference's fused_kernel stage, oracle.hpp:163-174,
//      executed for real). With peer memory its stores land at the
//      receiving ranks (the forward all-to-all fused into the lookup).
//   K4 the backward (oracle.hpp:149 bwd_comp): the stable sort of sort.cu
//      (K4a), then sgd_seg_kernel / sgd_kernel (K4b): duplicate rows are
//      reduced in the sorted (= original) order and every unique row gets
//      one L2 vector-reduction update.
//
// Both are HBM-bound random row gathers / updates over fp32, fp16 or bf16
// tables (16-byte row slices, Slice<T>; 32-byte for K1's fp32 64 B rows,
// Slice256F). K1: a block owns a tile of consecutive bags
// of one table, its offsets/indices staged in shared memory with coalesced
// loads; a warp is split into P spans (one bag each), a span into GB groups
// of L lanes, each lane moving one 16-byte slice with U rows in flight.
// K4: a block owns a tile of sorted positions of one table; short runs go P
// per warp round, hot runs are block-cooperative. Partial sums combine in
// fixed trees: bitwise reproducible.
#include <cub/cub.cuh>

#include <type_traits>

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
#ifdef SP_GEO_HEADER  // A/B builds: -DSP_GEO_HEADER=\"geo.h\" overriding the knobs below
#include SP_GEO_HEADER
#endif
// K1: bags are ~2*pf long; GB*U rows of a bag in flight.
#ifndef SP_FWD_G0
#define SP_FWD_G0 1, 1, 8, 4
#define SP_FWD_G1 2, 1, 8, 4
#define SP_FWD_G2 4, 1, 4, 4
#define SP_FWD_G3 8, 1, 2, 4
#define SP_FWD_G4 16, 1, 2, 8
#define SP_FWD_G5 32, 1, 1, 8
#endif
// K1 fp32 with 32-byte slices (Slice256F): half the lanes per row of the
// 16-byte geometry and half the rows in flight (the same bytes per lane).
// Only the 64 B class (dim 16) gains at cfg3 (K1 1.418 -> 1.405 ms); the
// 128 B class alone -0.8 %, both together 0, and the 256 / 512 B classes
// raise K1 to 43-48 registers (40 warps/SM) and lose 6-19 %.
constexpr unsigned kFwd256Classes = 1u << 2;
template <int CLS> struct FwdGeo256 : Geo<1, 1, 8, 4> {};  // classes not in kFwd256Classes
template <> struct FwdGeo256<2> : Geo<2, 1, 4, 2> {};
template <int CLS> struct FwdGeo;
template <> struct FwdGeo<0> : Geo<SP_FWD_G0> {};
template <> struct FwdGeo<1> : Geo<SP_FWD_G1> {};
template <> struct FwdGeo<2> : Geo<SP_FWD_G2> {};
template <> struct FwdGeo<3> : Geo<SP_FWD_G3> {};
template <> struct FwdGeo<4> : Geo<SP_FWD_G4> {};
template <> struct FwdGeo<5> : Geo<SP_FWD_G5> {};
// K4 SGD: most runs hold 1-2 positions, so more runs per warp (P) matter
// more than rows per run; lanes move up to 64 B of a row.
template <int CLS> struct SgdGeo;
#ifndef SP_SGD_G0
// (L, V, P, U) per dim class; tuned on B200 at cfg3 (profiles/r01_notes.md).
// With the L2 reduction update no register holds the old row, so lanes take
// 64 B of a row (V = 4) for dims >= 64; runs of >= 32 positions go to the
// block-cooperative path, so the short rounds keep U = 1.
#define SP_SGD_G0 1, 1, 16, 2
#define SP_SGD_G1 2, 1, 16, 1
#define SP_SGD_G2 2, 2, 16, 1
#define SP_SGD_G3 4, 2, 8, 1
#define SP_SGD_G4 4, 4, 8, 1
#define SP_SGD_G5 8, 4, 4, 1
#endif
template <> struct SgdGeo<0> : Geo<SP_SGD_G0> {};
template <> struct SgdGeo<1> : Geo<SP_SGD_G1> {};
template <> struct SgdGeo<2> : Geo<SP_SGD_G2> {};
template <> struct SgdGeo<3> : Geo<SP_SGD_G3> {};
template <> struct SgdGeo<4> : Geo<SP_SGD_G4> {};
template <> struct SgdGeo<5> : Geo<SP_SGD_G5> {};
// K4 SGD, long runs (hot rows): each warp of the block sums one slice of
// the run with the whole warp.
#ifndef SP_LONG_G0
#define SP_LONG_G0 1, 1, 1, 4
#define SP_LONG_G1 2, 1, 1, 4
#define SP_LONG_G2 4, 1, 1, 4
#define SP_LONG_G3 8, 1, 1, 4
#define SP_LONG_G4 16, 1, 1, 8
#define SP_LONG_G5 32, 1, 1, 8
#endif
template <int CLS> struct LongGeo;
template <> struct LongGeo<0> : Geo<SP_LONG_G0> {};
template <> struct LongGeo<1> : Geo<SP_LONG_G1> {};
template <> struct LongGeo<2> : Geo<SP_LONG_G2> {};
template <> struct LongGeo<3> : Geo<SP_LONG_G3> {};
template <> struct LongGeo<4> : Geo<SP_LONG_G4> {};
template <> struct LongGeo<5> : Geo<SP_LONG_G5> {};
// K4 on 2-byte rows: a 16-byte slice of the update is 8 fp32 sums (twice
// the registers of an fp32 slice), so fewer slices per lane / rows per warp.
template <int CLS> struct SgdGeoH;
template <> struct SgdGeoH<0> : Geo<1, 1, 16, 1> {};
template <> struct SgdGeoH<1> : Geo<2, 1, 16, 1> {};
template <> struct SgdGeoH<2> : Geo<4, 1, 8, 1> {};
template <> struct SgdGeoH<3> : Geo<8, 1, 4, 1> {};
template <> struct SgdGeoH<4> : Geo<8, 2, 4, 1> {};
template <> struct SgdGeoH<5> : Geo<16, 2, 2, 1> {};
template <int CLS> struct LongGeoH;
template <> struct LongGeoH<0> : Geo<1, 1, 1, 2> {};
template <> struct LongGeoH<1> : Geo<2, 1, 1, 2> {};
template <> struct LongGeoH<2> : Geo<4, 1, 1, 2> {};
template <> struct LongGeoH<3> : Geo<8, 1, 1, 2> {};
template <> struct LongGeoH<4> : Geo<16, 1, 1, 4> {};
template <> struct LongGeoH<5> : Geo<32, 1, 1, 4> {};
// 2-byte tables use the fp32 geometry: K1 keeps slices raw until it sums
// them (Slice<T>::Raw), so a 16-byte slice in flight costs 4 registers for
// every type; fp16 K1 at cfg3 1.241 ms (half the rows in flight, widened at
// load) -> 1.135 ms.
template <int C, class T>
using FwdG = FwdGeo<C>;
template <int C, class T>
using SgdG = std::conditional_t<std::is_same<T, float>::value, SgdGeo<C>, SgdGeoH<C>>;
template <int C, class T>
using LongG = std::conditional_t<std::is_same<T, float>::value, LongGeo<C>, LongGeoH<C>>;

// ---------------------------------------------------------------------------
// K1

struct FwdTile {
  int32_t t;   // canonical local table index
  int32_t b0;  // first bag
  int32_t nb;  // bags in the tile
  int32_t pad;
};

// K1 tile (bags per block): 256: 1.634 ms, 128: 1.607, 64: 1.630 (K1 at cfg3)
constexpr int kFwdTileBags = 128;
constexpr int kIdxCap = 4096;  // staged indices per tile (16 KB)

// 16-byte slices of a table row of element type T, widened to fp32 (K1) and
// the matching L2 vector reduction for the row update (K4): fp32 tables
// (the bench's 4 B/param pools) and fp16 tables (the paper's, PAPER.md:709,
// and the reference's default 2 B/param sizing, table.hpp:30).
template <class T> struct TypeTag { using type = T; };
template <class T> struct Slice;
// K1 keeps each gathered slice raw (Raw: 4 registers for 16 bytes) until
// it is summed, so 2-byte tables hold as many rows in flight per register
// as fp32 ones; load() widens at once (the SGD's gradient path).
template <> struct Slice<float> {
  static constexpr int E = 4;
  using Raw = float4;
  __device__ static __forceinline__ Raw load_raw(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
  }
  __device__ static __forceinline__ Raw zero_raw() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ static __forceinline__ void accum(float (&a)[4], const Raw& x) {
    a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
  }
  __device__ static __forceinline__ void load(const float* p, float (&v)[4]) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
  __device__ static __forceinline__ void red_add(float* p, const float (&d)[4]) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(d[0]),
                 "f"(d[1]), "f"(d[2]), "f"(d[3])
                 : "memory");
  }
  __device__ static __forceinline__ float to_f(float x) { return x; }
  __device__ static __forceinline__ void red_add1(float* p, float d) { atomicAdd(p, d); }
};
template <> struct Slice<__half> {
  static constexpr int E = 8;
  using Raw = uint4;
  __device__ static __forceinline__ Raw load_raw(const __half* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
  }
  __device__ static __forceinline__ Raw zero_raw() { return make_uint4(0u, 0u, 0u, 0u); }
  __device__ static __forceinline__ void accum(float (&a)[8], const Raw& x) {
    const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[k]));
      a[2 * k] += f.x;
      a[2 * k + 1] += f.y;
    }
  }
  __device__ static __forceinline__ void load(const __half* p, float (&v)[8]) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[k]));
      v[2 * k] = f.x;
      v[2 * k + 1] = f.y;
    }
  }
  // W += fp16(d), round-to-nearest at L2 (REDG.ADD.F16x8)
  __device__ static __forceinline__ void red_add(__half* p, const float (&d)[8]) {
    uint32_t u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const __half2 h = __floats2half2_rn(d[2 * k], d[2 * k + 1]);
      u[k] = *reinterpret_cast<const uint32_t*>(&h);
    }
    asm volatile("red.global.add.noftz.v4.f16x2 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(u[0]),
                 "r"(u[1]), "r"(u[2]), "r"(u[3])
                 : "memory");
  }
  __device__ static __forceinline__ float to_f(__half x) { return __half2float(x); }
  __device__ static __forceinline__ void red_add1(__half* p, float d) {
    atomicAdd(p, __float2half_rn(d));
  }
};
// bf16 tables (2 B/param like fp16, fp32's exponent range): widening is a
// 16-bit shift; the update is REDG.ADD.BF16x8 (round-to-nearest at L2)
template <> struct Slice<__nv_bfloat16> {
  static constexpr int E = 8;
  using Raw = uint4;
  __device__ static __forceinline__ Raw load_raw(const __nv_bfloat16* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
  }
  __device__ static __forceinline__ Raw zero_raw() { return make_uint4(0u, 0u, 0u, 0u); }
  __device__ static __forceinline__ void accum(float (&a)[8], const Raw& x) {
    const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[2 * k] += __uint_as_float(w4[k] << 16);
      a[2 * k + 1] += __uint_as_float(w4[k] & 0xffff0000u);
    }
  }
  __device__ static __forceinline__ void load(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[2 * k] = __uint_as_float(w4[k] << 16);
      v[2 * k + 1] = __uint_as_float(w4[k] & 0xffff0000u);
    }
  }
  __device__ static __forceinline__ void red_add(__nv_bfloat16* p, const float (&d)[8]) {
    uint32_t u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(d[2 * k], d[2 * k + 1]);
      u[k] = *reinterpret_cast<const uint32_t*>(&h);
    }
    asm volatile("red.global.add.noftz.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(u[0]),
                 "r"(u[1]), "r"(u[2]), "r"(u[3])
                 : "memory");
  }
  __device__ static __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ static __forceinline__ void red_add1(__nv_bfloat16* p, float d) {
    atomicAdd(p, __float2bfloat16_rn(d));
  }
};

// fp32 rows gathered in 32-byte lane slices (LDG.E.256, new on sm_100):
// the same bytes in flight with half the load instructions. Isolated random
// rows (profiles/microbench/rows256.cu): 128 B 4.65 -> 5.56 TB/s, 256-512 B
// +2-4 %, 64 B +4 %; inside K1 see kFwd256Classes. K1 only: vector
// reductions stop at 128 bits.
struct Slice256F {
  static constexpr int E = 8;
  struct Raw { float v[8]; };
  __device__ static __forceinline__ Raw load_raw(const float* p) {
    Raw r;
    load(p, r.v);
    return r;
  }
  __device__ static __forceinline__ Raw zero_raw() { return Raw{}; }
  __device__ static __forceinline__ void accum(float (&a)[8], const Raw& x) {
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] += x.v[e];
  }
  __device__ static __forceinline__ void load(const float* p, float (&v)[8]) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
          "=f"(v[7])
        : "l"(p));
  }
};

// kPeer: a compile-time path, so the local store path stays exactly the
// plain `out + b * ld` (a runtime branch on a by-value row-map parameter cost
// K1 6% at cfg3). The peer map lives in device memory.
template <bool kPeer>
__device__ __forceinline__ float* out_row(float* out, const RowMap* __restrict__ peer,
                                          int64_t b, int64_t ld) {
  if (!kPeer) return out + b * ld;
  const int64_t j = b / peer->rows_per_part;
  return peer->base[j] + (b - j * peer->rows_per_part) * ld;
}

// kStaged: every position of the tile is in s_idx (np <= kIdxCap), so the
// index fetch has no per-slot bound check against the staging capacity.
template <class G, bool kPeer, class T, bool kStaged = false, class SL = Slice<T>>
__device__ __forceinline__ void fwd_tile_warp(const TableMeta& m, int b0, int nb,
                                              int p0, int warp, int lane,
                                              const int32_t* s_off,
                                              const int32_t* s_idx,
                                              const int32_t* __restrict__ idx,
                                              const T* __restrict__ w,
                                              float* __restrict__ out,
                                              const RowMap* __restrict__ peer,
                                              int64_t ldo) {
  constexpr int L = G::L, V = G::V, P = G::P, U = G::U, S = G::S, GB = G::GB;
  constexpr int E = SL::E;
  const int span = lane / S, ls = lane % S, g = ls / L, s = ls % L;
  const T* wt = w + m.woff + E * s;  // lane s moves slices s, s+L, s+2L, ... (coalesced)
  const int dim = m.dim;
  for (int bg = warp * P; bg < nb; bg += kWarpsPerBlock * P) {
    const int bag = bg + span;
    const bool ok = bag < nb;
    int beg = 0, end = 0;
    if (ok) {
      beg = s_off[bag] - p0;
      end = s_off[bag + 1] - p0;
    }
    float acc[V][E];
#pragma unroll
    for (int j = 0; j < V; ++j)
#pragma unroll
      for (int e = 0; e < E; ++e) acc[j][e] = 0.f;
    for (int k = beg + g; k < end; k += GB * U) {
      int r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k + u * GB;
        if (kStaged)
          r[u] = kk < end ? s_idx[kk] : -1;
        else
          r[u] = kk < end ? (kk < kIdxCap ? s_idx[kk] : __ldg(idx + p0 + kk)) : -1;
      }
      typename SL::Raw v[U][V];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j)
          v[u][j] = r[u] >= 0 ? SL::load_raw(wt + static_cast<int64_t>(r[u]) * dim + E * L * j)
                              : SL::zero_raw();
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) SL::accum(acc[j], v[u][j]);
    }
#pragma unroll
    for (int o = L; o < S; o <<= 1)
#pragma unroll
      for (int j = 0; j < V; ++j)
#pragma unroll
        for (int e = 0; e < E; ++e) acc[j][e] += __shfl_xor_sync(0xffffffffu, acc[j][e], o);
    if (ok && g == 0) {
      float* o = out_row<kPeer>(out, peer, b0 + bag, ldo) + m.lcol + E * s;
#pragma unroll
      for (int j = 0; j < V; ++j)
#pragma unroll
        for (int e = 0; e < E; e += 4)
          __stcs(reinterpret_cast<float4*>(o + E * L * j + e),
                 make_float4(acc[j][e], acc[j][e + 1], acc[j][e + 2], acc[j][e + 3]));
    }
  }
}

// Any dim: one warp per bag, 32 scalar columns at a time.
template <bool kPeer, class T>
__device__ __forceinline__ void fwd_tile_warp_generic(
    const TableMeta& m, int b0, int nb, int p0, int warp, int lane,
    const int32_t* s_off, const int32_t* s_idx, const int32_t* __restrict__ idx,
    const T* __restrict__ w, float* __restrict__ out, const RowMap* __restrict__ peer,
    int64_t ldo) {
  for (int bag = warp; bag < nb; bag += kWarpsPerBlock) {
    const int beg = s_off[bag] - p0, end = s_off[bag + 1] - p0;
    for (int c0 = 0; c0 < m.dim; c0 += 32) {
      const int c = c0 + lane;
      float acc = 0.f;
      for (int k = beg; k < end; ++k) {
        const int r = k < kIdxCap ? s_idx[k] : __ldg(idx + p0 + k);
        if (c < m.dim) acc += Slice<T>::to_f(w[m.woff + static_cast<int64_t>(r) * m.dim + c]);
      }
      if (c < m.dim) out_row<kPeer>(out, peer, b0 + bag, ldo)[m.lcol + c] = acc;
    }
  }
}

template <bool kPeer, class T>
__global__ void __launch_bounds__(kBlockThreads)
    tbe_forward_kernel(const TableMeta* __restrict__ meta,
                       const FwdTile* __restrict__ tiles, int batch,
                       const int32_t* __restrict__ off,
                       const int32_t* __restrict__ idx,
                       const T* __restrict__ w, float* __restrict__ out,
                       const RowMap* __restrict__ peer, int64_t ldo) {
  __shared__ int32_t s_off[kFwdTileBags + 1];
  __shared__ int32_t s_idx[kIdxCap];
  const FwdTile tile = tiles[blockIdx.x];
  const TableMeta m = meta[tile.t];
  const int64_t base = static_cast<int64_t>(tile.t) * batch + tile.b0;
  for (int i = threadIdx.x; i <= tile.nb; i += kBlockThreads) s_off[i] = off[base + i];
  __syncthreads();
  const int p0 = s_off[0];
  const int np = s_off[tile.nb] - p0;
  for (int i = threadIdx.x; i < min(np, kIdxCap); i += kBlockThreads) s_idx[i] = __ldg(idx + p0 + i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  switch (m.cls) {
#define SP_FWD_CASE(C)                                                                    \
  case C:                                                                                 \
    if constexpr (std::is_same<T, float>::value && ((kFwd256Classes >> C) & 1)) {        \
      if (np <= kIdxCap)                                                                  \
        fwd_tile_warp<FwdGeo256<C>, kPeer, T, true, Slice256F>(                           \
            m, tile.b0, tile.nb, p0, warp, lane, s_off, s_idx, idx, w, out, peer, ldo);   \
      else                                                                                \
        fwd_tile_warp<FwdGeo256<C>, kPeer, T, false, Slice256F>(                          \
            m, tile.b0, tile.nb, p0, warp, lane, s_off, s_idx, idx, w, out, peer, ldo);   \
    } else {                                                                              \
      if (np <= kIdxCap)                                                                  \
        fwd_tile_warp<FwdG<C, T>, kPeer, T, true>(m, tile.b0, tile.nb, p0, warp, lane,      \
                                                  s_off, s_idx, idx, w, out, peer, ldo);  \
      else                                                                                \
        fwd_tile_warp<FwdG<C, T>, kPeer, T>(m, tile.b0, tile.nb, p0, warp, lane, s_off,    \
                                            s_idx, idx, w, out, peer, ldo);               \
    }                                                                                     \
    break;
    SP_FWD_CASE(0)
    SP_FWD_CASE(1)
    SP_FWD_CASE(2)
    SP_FWD_CASE(3)
    SP_FWD_CASE(4)
    SP_FWD_CASE(5)
#undef SP_FWD_CASE
    default:
      fwd_tile_warp_generic<kPeer, T>(m, tile.b0, tile.nb, p0, warp, lane, s_off, s_idx, idx,
                                   w, out, peer, ldo);
  }
  // peer stores (the fused forward all-to-all) are made visible system-wide
  // before the block retires; the host/NCCL barrier after K1 orders them
  // against the receivers' reads
  if (kPeer) __threadfence_system();
}

// ---------------------------------------------------------------------------
// K4 step 3: row-wise SGD over the sorted (key, bag) pairs.
//
// The sorted array keeps every table's lookups at the table's CSR position
// range (the key = table row base + row, tables in order), so tiles of at
// most kTilePos positions are cut per table on the host (SgdTile) and a
// block is specialised once on its table's dim class. A block owns the runs
// (unique rows) whose head lies in its tile; a run that reaches the tile end
// is finished by the same block. Prologue: the tile's rows/bags are staged in
// shared memory and one block scan splits the heads into
//   short runs (< kLongRun positions): packed (beg, len) in 16 bits; warps
//     claim chunks of them dynamically and take P at a time (one span each);
//   long runs (hot rows): every warp of the block sums a fixed slice of the
//     run, partial sums meet in shared memory in warp order (deterministic)
//     and one warp applies the row update.
// The update W[row] += -lr * sum is one L2 vector reduction per 16 B
// (red.global.add.v4.f32): each unique row has exactly one writer per
// launch, so it is deterministic, and no SM register waits for the old row.

constexpr int kTilePos = 2048;  // run-based SGD tile (positions, <= 2048: 11-bit run starts)
constexpr int kSegTilePos = 1024;  // segmented SGD tile (positions; 2048 re-read more gradient)
constexpr int kPosPerThread = kTilePos / kBlockThreads;
constexpr int kLongRun = 32;  // runs at least this long are block-cooperative
constexpr int kRunChunk = 16;  // short runs claimed per warp at a time (>= max P)
constexpr int kMaxLong = kTilePos / kLongRun + 1;

struct SgdTile {
  int32_t t;       // canonical local table
  int32_t p0;      // first sorted position of the tile
  int32_t np;      // positions in the tile
  int32_t tstart;  // first position of the table
  int32_t pend;    // one past the table's last position
  int32_t pad[3];
};

template <class BagT>
struct SgdShared {
  uint32_t row[kTilePos];
  BagT bag[kTilePos];
  uint16_t srun[kTilePos];      // short runs: beg | len << 11
  uint16_t lbeg[kMaxLong];      // long runs: first position (tile-relative)
  int32_t lend[kMaxLong];       //            one past the last (may pass np)
  alignas(16) float part[kWarpsPerBlock][256];  // one row: <= 512 B of fp32 or fp16
  int nshort, nlong, next;
};

template <class BagT>
__device__ __forceinline__ uint32_t sgd_bag(const SgdShared<BagT>& sh, int i, int np, int p0,
                                            const BagT* __restrict__ bags) {
  return i < np ? static_cast<uint32_t>(sh.bag[i]) : static_cast<uint32_t>(__ldg(bags + p0 + i));
}

// Gradient columns of one 16-byte weight slice (E fp32 values, E/4 float4).
template <int E>
__device__ __forceinline__ void load_grad(const float* p, float (&v)[E]) {
#pragma unroll
  for (int e = 0; e < E; e += 4) {
    const float4 x = ldg_f4(p + e);
    v[e] = x.x; v[e + 1] = x.y; v[e + 2] = x.z; v[e + 3] = x.w;
  }
}
// 8 gradient values in one 32-byte load (p 32-byte aligned)
__device__ __forceinline__ void load_grad32(const float* p, float (&v)[8]) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7])
      : "l"(p));
}

// One round of up to P short runs [j, jend) of the tile (span s: run j+s).
template <class G, class BagT, class T>
__device__ __forceinline__ void sgd_short_round(const TableMeta& m, int j, int jend, int np,
                                                int p0, int lane, const SgdShared<BagT>& sh,
                                                const BagT* __restrict__ bags,
                                                const float* __restrict__ grad, int64_t ldg,
                                                float lr, T* __restrict__ w) {
  constexpr int L = G::L, V = G::V, U = G::U, S = G::S, GB = G::GB;
  constexpr int E = Slice<T>::E;
  const int span = lane / S, ls = lane % S, g = ls / L, sub = ls % L;
  const int u = j + span;
  const bool active = u < jend;
  float acc[V][E];
#pragma unroll
  for (int c = 0; c < V; ++c)
#pragma unroll
    for (int e = 0; e < E; ++e) acc[c][e] = 0.f;
  int beg = 0;
  if (active) {
    const uint32_t pk = sh.srun[u];
    beg = static_cast<int>(pk & 2047u);
    const int end = beg + static_cast<int>(pk >> 11);
    const float* gcol = grad + m.lcol + E * sub;
    for (int k = beg + g; k < end; k += GB * U) {
      uint32_t bg[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int kk = k + q * GB;
        bg[q] = kk < end ? sgd_bag(sh, kk, np, p0, bags) : 0xffffffffu;
      }
      float v[U][V][E];
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int c = 0; c < V; ++c) {
          if (bg[q] != 0xffffffffu) {
            load_grad<E>(gcol + static_cast<int64_t>(bg[q]) * ldg + E * L * c, v[q][c]);
          } else {
#pragma unroll
            for (int e = 0; e < E; ++e) v[q][c][e] = 0.f;
          }
        }
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int c = 0; c < V; ++c)
#pragma unroll
          for (int e = 0; e < E; ++e) acc[c][e] += v[q][c][e];
    }
  }
#pragma unroll
  for (int o = L; o < S; o <<= 1)
#pragma unroll
    for (int c = 0; c < V; ++c)
#pragma unroll
      for (int e = 0; e < E; ++e) acc[c][e] += __shfl_xor_sync(0xffffffffu, acc[c][e], o);
  if (active && g == 0) {
    T* wrow = w + m.woff + static_cast<int64_t>(sh.row[beg]) * m.dim + E * sub;
#pragma unroll
    for (int c = 0; c < V; ++c) {
      float d[E];
#pragma unroll
      for (int e = 0; e < E; ++e) d[e] = -lr * acc[c][e];
      Slice<T>::red_add(wrow + E * L * c, d);
    }
  }
}

// Long run [beg, end): warp `warp` sums its fixed slice into part[warp].
template <class G, class BagT, class T>
__device__ __forceinline__ void sgd_long_slice(const TableMeta& m, int beg, int end, int np,
                                               int p0, int warp, int lane,
                                               SgdShared<BagT>& sh,
                                               const BagT* __restrict__ bags,
                                               const float* __restrict__ grad, int64_t ldg) {
  constexpr int L = G::L, V = G::V, U = G::U, GB = G::GB;
  constexpr int E = Slice<T>::E;
  const int g = lane / L, sub = lane % L;
  const int len = end - beg;
  const int per = (len + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int s0 = beg + min(len, warp * per), s1 = beg + min(len, (warp + 1) * per);
  float acc[V][E];
#pragma unroll
  for (int c = 0; c < V; ++c)
#pragma unroll
    for (int e = 0; e < E; ++e) acc[c][e] = 0.f;
  const float* gcol = grad + m.lcol + E * sub;
  for (int k = s0 + g; k < s1; k += GB * U) {
    uint32_t bg[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int kk = k + q * GB;
      bg[q] = kk < s1 ? sgd_bag(sh, kk, np, p0, bags) : 0xffffffffu;
    }
    float v[U][V][E];
#pragma unroll
    for (int q = 0; q < U; ++q)
#pragma unroll
      for (int c = 0; c < V; ++c) {
        if (bg[q] != 0xffffffffu) {
          load_grad<E>(gcol + static_cast<int64_t>(bg[q]) * ldg + E * L * c, v[q][c]);
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) v[q][c][e] = 0.f;
        }
      }
#pragma unroll
    for (int q = 0; q < U; ++q)
#pragma unroll
      for (int c = 0; c < V; ++c)
#pragma unroll
        for (int e = 0; e < E; ++e) acc[c][e] += v[q][c][e];
  }
#pragma unroll
  for (int o = L; o < 32; o <<= 1)
#pragma unroll
    for (int c = 0; c < V; ++c)
#pragma unroll
      for (int e = 0; e < E; ++e) acc[c][e] += __shfl_xor_sync(0xffffffffu, acc[c][e], o);
  if (g == 0)
#pragma unroll
    for (int c = 0; c < V; ++c)
#pragma unroll
      for (int e = 0; e < E; e += 4)
        *reinterpret_cast<float4*>(&sh.part[warp][E * sub + E * L * c + e]) =
            make_float4(acc[c][e], acc[c][e + 1], acc[c][e + 2], acc[c][e + 3]);
}

// Short-run (SG) and long-run (LG) geometries of one row class.
template <class SG, class LG, class BagT, class T>
__device__ __forceinline__ void sgd_tile(const TableMeta& m, const SgdTile& tile,
                                         SgdShared<BagT>& sh,
                                         const BagT* __restrict__ bags,
                                         const float* __restrict__ grad, int64_t ldg,
                                         float lr, T* __restrict__ w) {
  constexpr int E = Slice<T>::E;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = tile.np, p0 = tile.p0;
  // long runs first: all warps cooperate, two barriers per run
  for (int r = 0; r < sh.nlong; ++r) {
    const int beg = sh.lbeg[r], end = sh.lend[r];
    sgd_long_slice<LG, BagT, T>(m, beg, end, np, p0, warp, lane, sh, bags, grad, ldg);
    __syncthreads();
    if (warp == 0) {
      T* wrow = w + m.woff + static_cast<int64_t>(sh.row[beg]) * m.dim;
      for (int c = E * lane; c < m.dim; c += 32 * E) {
        float d[E];
#pragma unroll
        for (int e = 0; e < E; e += 4) {
          float4 sum = *reinterpret_cast<const float4*>(&sh.part[0][c + e]);
#pragma unroll
          for (int q = 1; q < kWarpsPerBlock; ++q)
            sum = f4_add(sum, *reinterpret_cast<const float4*>(&sh.part[q][c + e]));
          d[e] = -lr * sum.x;
          d[e + 1] = -lr * sum.y;
          d[e + 2] = -lr * sum.z;
          d[e + 3] = -lr * sum.w;
        }
        Slice<T>::red_add(wrow + c, d);
      }
    }
    __syncthreads();
  }
  // short runs: dynamic chunks, P per round
  const int ns = sh.nshort;
  for (;;) {
    int j0 = 0;
    if (lane == 0) j0 = atomicAdd(&sh.next, kRunChunk);
    j0 = __shfl_sync(0xffffffffu, j0, 0);
    if (j0 >= ns) break;
    const int jend = min(ns, j0 + kRunChunk);
    for (int j = j0; j < jend; j += SG::P)
      sgd_short_round<SG, BagT, T>(m, j, jend, np, p0, lane, sh, bags, grad, ldg, lr, w);
  }
}

// Any other row size: a warp per run, 32 columns at a time, positions in
// sorted order.
template <class BagT, class T>
__device__ void sgd_tile_generic(const TableMeta& m, const SgdTile& tile, SgdShared<BagT>& sh,
                                 const BagT* __restrict__ bags, const float* __restrict__ grad,
                                 int64_t ldg, float lr, T* __restrict__ w) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nrun = sh.nshort + sh.nlong;
  for (int r = warp; r < nrun; r += kWarpsPerBlock) {
    int beg, end;
    if (r < sh.nshort) {
      beg = sh.srun[r] & 2047;
      end = beg + (sh.srun[r] >> 11);
    } else {
      beg = sh.lbeg[r - sh.nshort];
      end = sh.lend[r - sh.nshort];
    }
    T* wrow = w + m.woff + static_cast<int64_t>(sh.row[beg]) * m.dim;
    for (int c = lane; c < m.dim; c += 32) {
      float acc = 0.f;
      for (int k = beg; k < end; ++k)
        acc += __ldg(grad + static_cast<int64_t>(sgd_bag(sh, k, tile.np, tile.p0, bags)) * ldg +
                     m.lcol + c);
      Slice<T>::red_add1(wrow + c, -lr * acc);
    }
  }
}

constexpr int kSgdMinBlocks = 4;  // 4 x 256 threads per SM: <= 64 registers
template <class BagT, class T>
__global__ void __launch_bounds__(kBlockThreads, kSgdMinBlocks)
    sgd_kernel(const TableMeta* __restrict__ meta, const SgdTile* __restrict__ tiles,
               const uint32_t* __restrict__ keys, const BagT* __restrict__ bags,
               const float* __restrict__ grad, int64_t ldg, float lr,
               T* __restrict__ w, const int32_t* __restrict__ abort_flag) {
  if (abort_flag != nullptr && *abort_flag != 0) return;  // invalid batch: no update
  __shared__ SgdShared<BagT> sh;
  using BlockScan = cub::BlockScan<int, kBlockThreads>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  const SgdTile tile = tiles[blockIdx.x];
  const TableMeta m = meta[tile.t];
  const int np = tile.np, p0 = tile.p0, tid = threadIdx.x;
  for (int i = tid; i < np; i += kBlockThreads) {
    sh.row[i] = __ldg(keys + p0 + i) - m.rowbase;
    sh.bag[i] = __ldg(bags + p0 + i);
  }
  const uint32_t prev = p0 > tile.tstart ? __ldg(keys + p0 - 1) - m.rowbase : 0xffffffffu;
  __syncthreads();
  // heads; a run is long iff the position kLongRun-1 ahead has the same row
  // (sorted). Ends: short runs by a short scan, long runs by binary search.
  int sbeg[kPosPerThread], send[kPosPerThread];
  int ns = 0, nl = 0;
#pragma unroll
  for (int q = 0; q < kPosPerThread; ++q) {
    const int i = tid * kPosPerThread + q;
    sbeg[q] = -1;
    send[q] = 0;
    if (i >= np) continue;
    const uint32_t r = sh.row[i];
    if (r == (i == 0 ? prev : sh.row[i - 1])) continue;
    const int la = i + kLongRun - 1;
    const bool lng = la < np ? sh.row[la] == r
                             : (p0 + la < tile.pend && __ldg(keys + p0 + la) - m.rowbase == r);
    int e;
    if (!lng) {
      e = i + 1;
      while (e < np && sh.row[e] == r) ++e;
      if (e == np)  // the run may continue past the tile (still short)
        while (p0 + e < tile.pend && __ldg(keys + p0 + e) - m.rowbase == r) ++e;
      ++ns;
    } else {
      // first position past i + kLongRun - 1 whose row differs
      int lo = la + 1, hi = la + 1;
      int64_t stepw = 1;
      auto same = [&](int x) {
        return x < np ? sh.row[x] == r
                      : (p0 + x < tile.pend && __ldg(keys + p0 + x) - m.rowbase == r);
      };
      while (same(hi)) {  // gallop
        lo = hi + 1;
        hi = static_cast<int>(hi + stepw < tile.pend - p0 ? hi + stepw : tile.pend - p0);
        stepw <<= 1;
      }
      while (lo < hi) {  // first x in [lo, hi] with !same(x)
        const int mid = (lo + hi) >> 1;
        if (same(mid)) lo = mid + 1; else hi = mid;
      }
      e = lo;
      ++nl;
    }
    sbeg[q] = lng ? -2 - i : i;  // long marked negative
    send[q] = e;
  }
  int first = 0, total = 0;
  BlockScan(scan_tmp).ExclusiveSum(ns | (nl << 16), first, total);
  int fs = first & 0xffff, fl = first >> 16;
#pragma unroll
  for (int q = 0; q < kPosPerThread; ++q) {
    if (sbeg[q] >= 0) {
      sh.srun[fs++] = static_cast<uint16_t>(sbeg[q] | ((send[q] - sbeg[q]) << 11));
    } else if (sbeg[q] <= -2) {
      sh.lbeg[fl] = static_cast<uint16_t>(-2 - sbeg[q]);
      sh.lend[fl++] = send[q];
    }
  }
  if (tid == 0) {
    sh.nshort = total & 0xffff;
    sh.nlong = total >> 16;
    sh.next = 0;
  }
  __syncthreads();
  switch (m.cls) {
#define SP_SGD_CASE(C)                                                          \
  case C:                                                                       \
    sgd_tile<SgdG<C, T>, LongG<C, T>, BagT, T>(m, tile, sh, bags, grad, ldg, lr, w); \
    break;
    SP_SGD_CASE(0)
    SP_SGD_CASE(1)
    SP_SGD_CASE(2)
    SP_SGD_CASE(3)
    SP_SGD_CASE(4)
    SP_SGD_CASE(5)
#undef SP_SGD_CASE
    default:
      sgd_tile_generic<BagT, T>(m, tile, sh, bags, grad, ldg, lr, w);
  }
}

// ---------------------------------------------------------------------------
// K4 SGD for wide rows (256- and 512-byte rows: fp32 dims 64/128, fp16
// dims 128/256): a segmented reduction over the sorted positions instead of
// runs. A row of R 16-byte slices is one lane group (R = 32: the warp; R =
// 16: a half warp); the tile's positions are cut into one contiguous chunk
// per group and every group walks its chunk in position order with U
// gradient rows in flight: all lanes of a group see the same row sequence,
// so run boundaries are uniform, hot runs need no special path and there is
// no per-run bookkeeping. A run inside one chunk is applied at its end (one
// L2 vector reduction per slice); a run crossing chunk boundaries leaves its
// partial sums in shared memory and is combined in chunk order after the
// walk; one crossing the tile boundary leaves them in a per-tile carry,
// combined in tile order by sgd_carry_kernel. Every sum is in position
// order up to that fixed chunking: deterministic.

constexpr int kCarryF = 256;  // floats per carry row (<= 512-byte rows of fp32 or fp16)
enum { kNone = 0, kPart = 1, kWhole = 2 };

constexpr int kSegChunksMax = kWarpsPerBlock * 32;  // R = 1: 32 groups per warp

template <class BagT, class T>
struct SegShared {
  uint32_t row[kSegTilePos];
  BagT bag[kSegTilePos];
  alignas(16) float part[512 * Slice<T>::E];  // [C][2][R*E] with C*R = 256
  int kind[kSegChunksMax][2];
  uint32_t prow[kSegChunksMax][2];
};

// One tile of rows of R 16-byte slices (R = 1..32).
template <int R, class BagT, class T>
__device__ __forceinline__ void sgd_seg_tile(const TableMeta& m, const SgdTile& tile,
                                             SegShared<BagT, T>& sh, bool cont_prev,
                                             bool cont_next, const float* __restrict__ grad,
                                             int64_t ldg, float lr, T* __restrict__ w,
                                             float* __restrict__ carry_f,
                                             int32_t* __restrict__ carry_i, int64_t slot) {
  constexpr int E = Slice<T>::E;     // fp32 values per slice
  constexpr int kSegU = 32 / E;  // gradient rows in flight per group (32 fp32 values per lane)
  constexpr int G = 32 / R;          // groups per warp
  constexpr int C = kWarpsPerBlock * G;
  constexpr int W = R * E;           // floats per partial row
  const int np = tile.np, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int c = warp * G + lane / R, sub = lane % R;
  const int cs = static_cast<int>(static_cast<int64_t>(np) * c / C);
  const int ce = static_cast<int>(static_cast<int64_t>(np) * (c + 1) / C);
  const float* gcol = grad + m.lcol + E * sub;
  T* wbase = w + m.woff + E * sub;
  float* part = sh.part;  // [C][2][W]
  if (sub == 0) {
    sh.kind[c][0] = kNone;
    sh.kind[c][1] = kNone;
  }
  if (cs < ce) {
    uint32_t run = sh.row[cs];
    // the chunk's first run began earlier (previous chunk or tile)
    bool head_open = cs > 0 ? sh.row[cs - 1] == run : cont_prev;
    float acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.f;
    auto flush = [&](uint32_t row, bool open_before) {
      if (open_before) {  // the chunk's head partial, combined after the walk
#pragma unroll
        for (int e = 0; e < E; ++e) part[(c * 2) * W + sub * E + e] = acc[e];
        if (sub == 0) {
          sh.kind[c][0] = kPart;
          sh.prow[c][0] = row;
        }
      } else {
        float d[E];
#pragma unroll
        for (int e = 0; e < E; ++e) d[e] = -lr * acc[e];
        Slice<T>::red_add(wbase + static_cast<int64_t>(row) * m.dim, d);
      }
    };
    // 2-byte rows: a lane's 8 gradient columns are one 32-byte load when
    // the table's columns and the gradient's row stride are 32-byte aligned
    // (fp16 SGD at cfg3 1.609 -> 1.524 ms)
    const bool g32 = E == 8 && ((m.lcol | ldg) & 7) == 0;
    for (int k = cs; k < ce; k += kSegU) {
      float v[kSegU][E];
#pragma unroll
      for (int u = 0; u < kSegU; ++u) {
        if (k + u < ce) {
          const float* gp = gcol + static_cast<int64_t>(sh.bag[k + u]) * ldg;
          if constexpr (E == 8) {
            if (g32) load_grad32(gp, v[u]);
            else load_grad<E>(gp, v[u]);
          } else {
            load_grad<E>(gp, v[u]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) v[u][e] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < kSegU; ++u) {
        if (k + u >= ce) break;
        const uint32_t r = sh.row[k + u];
        if (r != run) {
          flush(run, head_open);
          head_open = false;
          run = r;
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] += v[u][e];
      }
    }
    // the chunk's last run: does it continue past the chunk?
    const bool tail_open = ce < np ? sh.row[ce] == run : cont_next;
    if (!tail_open) {
      flush(run, head_open);
    } else {
      const int sl = head_open ? 0 : 1;  // whole chunk in one run : tail partial
#pragma unroll
      for (int e = 0; e < E; ++e) part[(c * 2 + sl) * W + sub * E + e] = acc[e];
      if (sub == 0) {
        sh.kind[c][sl] = head_open ? kWhole : kPart;
        sh.prow[c][sl] = run;
      }
    }
  }
  __syncthreads();
  // chains across chunks, in chunk order (lanes 0..R-1 of warp 0)
  if (warp != 0 || lane >= R) return;
  float acc[E];
  bool open = false, from_prev = false;
  uint32_t row = 0;
  float* gh = carry_f + (slot * 2) * kCarryF;
  float* gt = gh + kCarryF;
  int head_kind = kNone, tail_kind = kNone;
  for (int q = 0; q < C; ++q) {
    const int kh = sh.kind[q][0];
    if (kh != kNone) {
      if (!open) {  // only the tile's first chunk can continue the previous tile
        open = true;
        from_prev = true;
        row = sh.prow[q][0];
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.f;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] += part[(q * 2) * W + lane * E + e];
      if (kh == kPart) {  // the chain ends in chunk q
        if (from_prev) {
#pragma unroll
          for (int e = 0; e < E; ++e) gh[lane * E + e] = acc[e];
          head_kind = kPart;
        } else {
          float d[E];
#pragma unroll
          for (int e = 0; e < E; ++e) d[e] = -lr * acc[e];
          Slice<T>::red_add(wbase + static_cast<int64_t>(row) * m.dim, d);
        }
        open = false;
      }
    }
    if (sh.kind[q][1] == kPart) {  // a chain starts in chunk q
      open = true;
      from_prev = false;
      row = sh.prow[q][1];
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = part[(q * 2 + 1) * W + lane * E + e];
    }
  }
  if (open) {
    if (from_prev) {  // the whole tile is one run
#pragma unroll
      for (int e = 0; e < E; ++e) gh[lane * E + e] = acc[e];
      head_kind = kWhole;
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) gt[lane * E + e] = acc[e];
      tail_kind = kPart;
    }
  }
  if (lane == 0) {
    int32_t* ci = carry_i + slot * 4;
    ci[0] = head_kind;
    ci[1] = tail_kind;
    ci[2] = static_cast<int32_t>(row);
  }
}

constexpr int kSegMinBlocks = 4;  // <= 64 registers; 3 or 5 blocks per SM measured slower
template <class BagT, class T>
__global__ void __launch_bounds__(kBlockThreads, kSegMinBlocks)
    sgd_seg_kernel(const TableMeta* __restrict__ meta, const SgdTile* __restrict__ tiles,
                   const uint32_t* __restrict__ keys, const BagT* __restrict__ bags,
                   const float* __restrict__ grad, int64_t ldg, float lr, T* __restrict__ w,
                   float* __restrict__ carry_f, int32_t* __restrict__ carry_i,
                   const int32_t* __restrict__ abort_flag) {
  if (abort_flag != nullptr && *abort_flag != 0) return;
  __shared__ SegShared<BagT, T> sh;
  const SgdTile tile = tiles[blockIdx.x];
  const TableMeta m = meta[tile.t];
  const int np = tile.np, p0 = tile.p0, tid = threadIdx.x;
  for (int i = tid; i < np; i += kBlockThreads) {
    sh.row[i] = __ldg(keys + p0 + i) - m.rowbase;
    sh.bag[i] = __ldg(bags + p0 + i);
  }
  const bool cont_prev = p0 > tile.tstart && __ldg(keys + p0 - 1) == __ldg(keys + p0);
  const bool cont_next = p0 + np < tile.pend && __ldg(keys + p0 + np) == __ldg(keys + p0 + np - 1);
  __syncthreads();
  switch (m.cls) {
#define SP_SEG_CASE(C)                                                                    \
  case C:                                                                                 \
    sgd_seg_tile<(1 << C), BagT, T>(m, tile, sh, cont_prev, cont_next, grad, ldg, lr, w, \
                                    carry_f, carry_i, blockIdx.x);                        \
    break;
    SP_SEG_CASE(0)
    SP_SEG_CASE(1)
    SP_SEG_CASE(2)
    SP_SEG_CASE(3)
    SP_SEG_CASE(4)
    SP_SEG_CASE(5)
#undef SP_SEG_CASE
    default:
      break;
  }
}

// Runs crossing tiles: tile i's tail + the whole tiles after it + the head
// of the tile where the run ends, in tile order; one warp per tile.
template <int R, class T>
__device__ __forceinline__ void sgd_carry_tile(const TableMeta& m, int i, int n_tiles, int lane,
                                               float lr, T* __restrict__ w,
                                               const float* __restrict__ carry_f,
                                               const int32_t* __restrict__ carry_i) {
  constexpr int E = Slice<T>::E;
  if (lane >= R) return;
  const uint32_t row = static_cast<uint32_t>(carry_i[static_cast<size_t>(i) * 4 + 2]);
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e)
    acc[e] = carry_f[(static_cast<size_t>(i) * 2 + 1) * kCarryF + lane * E + e];
  for (int j = i + 1; j < n_tiles; ++j) {
    const int hk = carry_i[static_cast<size_t>(j) * 4];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] += carry_f[(static_cast<size_t>(j) * 2) * kCarryF + lane * E + e];
    if (hk != kWhole) break;
  }
  float d[E];
#pragma unroll
  for (int e = 0; e < E; ++e) d[e] = -lr * acc[e];
  Slice<T>::red_add(w + m.woff + static_cast<int64_t>(row) * m.dim + E * lane, d);
}

template <class T>
__global__ void sgd_carry_kernel(const TableMeta* __restrict__ meta,
                                 const SgdTile* __restrict__ tiles, int n_tiles, float lr,
                                 T* __restrict__ w, const float* __restrict__ carry_f,
                                 const int32_t* __restrict__ carry_i,
                                 const int32_t* __restrict__ abort_flag) {
  pdl_wait();  // a programmatic dependent of sgd_seg_kernel (launch_sgd)
  if (abort_flag != nullptr && *abort_flag != 0) return;
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n_tiles || carry_i[static_cast<size_t>(i) * 4 + 1] != kPart) return;
  const TableMeta m = meta[tiles[i].t];
  switch (m.cls) {
#define SP_CARRY_CASE(C)                                                      \
  case C:                                                                     \
    sgd_carry_tile<(1 << C), T>(m, i, n_tiles, lane, lr, w, carry_f, carry_i); \
    break;
    SP_CARRY_CASE(0)
    SP_CARRY_CASE(1)
    SP_CARRY_CASE(2)
    SP_CARRY_CASE(3)
    SP_CARRY_CASE(4)
    SP_CARRY_CASE(5)
#undef SP_CARRY_CASE
    default:
      break;
  }
}

// ---------------------------------------------------------------------------
// Generator / layout kernels

__device__ __forceinline__ void store_w(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_w(__half* p, float v) { *p = __float2half_rn(v); }
__device__ __forceinline__ void store_w(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ float load_w(float x) { return x; }
__device__ __forceinline__ float load_w(__half x) { return __half2float(x); }
__device__ __forceinline__ float load_w(__nv_bfloat16 x) { return __bfloat162float(x); }

template <class T>
__global__ void init_weights_kernel(T* __restrict__ w, int64_t rows,
                                    int dim, int32_t gid, uint64_t seed) {
  const int64_t n = rows * dim;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       e < n; e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / dim;
    const int c = static_cast<int>(e - r * dim);
    store_w(w + e, weight_from_base(
                       h3(seed, kTagW, static_cast<uint64_t>(gid), static_cast<uint64_t>(r)), c));
  }
}

// fp32 host rows <-> 2-byte device rows (set_table / get_table)
template <class T>
__global__ void f32_to_w_kernel(const float* __restrict__ src, T* __restrict__ dst, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    store_w(dst + e, src[e]);
}
template <class T>
__global__ void w_to_f32_kernel(const T* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[e] = load_w(src[e]);
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

// flag bits: 1 = offsets decrease, 2 = index out of [0, rows). Bad data is
// clamped (offsets into [0, nnz], indices to row 0) so every later kernel
// stays in bounds even before the host has seen the flag.
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
    const int64_t rel = a - o0;
    off[b] = static_cast<int32_t>(rel < 0 ? 0 : (rel > nnz ? nnz : rel)) + base;
  }
  for (int64_t p = t0; p < nnz; p += stride) {
    const int64_t r = idx64[p];
    const bool out = r < 0 || r >= rows;
    if (out) bad |= 2;
    idx[p] = out ? 0 : static_cast<int32_t>(r);
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
    for (int b0 = 0; b0 < batch; b0 += kFwdTileBags)
      tiles.push_back(make_int4(canon[li].local, b0, std::min(kFwdTileBags, batch - b0), 0));
  return tiles;
}

void launch_tbe_forward(const TableMeta* d_meta_canon, const int4* d_tiles,
                        int64_t n_tiles, int batch, const int32_t* d_off,
                        const int32_t* d_idx, const void* d_w, WeightType wt, float* d_out,
                        const RowMap* d_peer, int64_t ldo, cudaStream_t st) {
  if (n_tiles <= 0) return;
  const FwdTile* tiles = reinterpret_cast<const FwdTile*>(d_tiles);
  const unsigned g = static_cast<unsigned>(n_tiles);
  auto go = [&](auto peer, auto elem) {
    constexpr bool kPeer = decltype(peer)::value;
    using T = typename decltype(elem)::type;
    tbe_forward_kernel<kPeer, T><<<g, kBlockThreads, 0, st>>>(
        d_meta_canon, tiles, batch, d_off, d_idx, static_cast<const T*>(d_w), d_out, d_peer, ldo);
  };
  using F32 = TypeTag<float>;
  using F16 = TypeTag<__half>;
  using BF16 = TypeTag<__nv_bfloat16>;
  if (wt == WeightType::kF16) {
    if (d_peer) go(std::true_type{}, F16{});
    else go(std::false_type{}, F16{});
  } else if (wt == WeightType::kBF16) {
    if (d_peer) go(std::true_type{}, BF16{});
    else go(std::false_type{}, BF16{});
  } else {
    if (d_peer) go(std::true_type{}, F32{});
    else go(std::false_type{}, F32{});
  }
  SP_LAUNCHED();
}

size_t exclusive_scan_i32(void* temp, size_t temp_bytes, const int32_t* in,
                          int32_t* out, int64_t n, cudaStream_t st) {
  size_t bytes = temp_bytes;
  SP_CUDA(cub::DeviceScan::ExclusiveSum(temp, bytes, in, out, n, st));
  return bytes;
}

std::vector<int> make_sgd_tiles(const std::vector<int64_t>& table_nnz,
                                const std::vector<TableMeta>& canon, int64_t counts[2]) {
  // tiles of the generic-dim tables (run-based sgd_kernel), then the tiles
  // of every other table (segmented sgd_seg_kernel), tables in order
  std::vector<int> out;
  for (int part = 0; part < 2; ++part) {
    counts[part] = 0;
    int64_t p = 0;
    for (size_t t = 0; t < table_nnz.size(); ++t) {
      const int64_t e = p + table_nnz[t];
      const int cls = t < canon.size() ? canon[t].cls : -1;
      const int64_t tp = part == 0 ? kTilePos : kSegTilePos;
      if ((cls >= 0 ? 1 : 0) == part)
        for (int64_t q = p; q < e; q += tp) {
          SgdTile tl{};
          tl.t = static_cast<int32_t>(t);
          tl.p0 = static_cast<int32_t>(q);
          tl.np = static_cast<int32_t>(std::min<int64_t>(tp, e - q));
          tl.tstart = static_cast<int32_t>(p);
          tl.pend = static_cast<int32_t>(e);
          const int* raw = reinterpret_cast<const int*>(&tl);
          out.insert(out.end(), raw, raw + kSgdTileInts);
          ++counts[part];
        }
      p = e;
    }
  }
  return out;
}

void launch_sgd(const TableMeta* d_meta_canon, const int* d_tiles, const int64_t counts[2],
                const uint32_t* d_keys, const void* d_bags, bool bags16, const float* d_grad,
                int64_t ldg, float lr, void* d_w, WeightType wt, float* d_carry_f,
                int32_t* d_carry_i, const int32_t* d_abort, cudaStream_t st) {
  static_assert(sizeof(SgdTile) == kSgdTileInts * sizeof(int), "tile layout");
  const SgdTile* tiles = reinterpret_cast<const SgdTile*>(d_tiles);
  auto go = [&](auto elem, auto bag) {
    using T = typename decltype(elem)::type;
    using BagT = typename decltype(bag)::type;
    T* w = static_cast<T*>(d_w);
    const BagT* bags = static_cast<const BagT*>(d_bags);
    if (counts[1] > 0) {
      sgd_seg_kernel<BagT, T><<<static_cast<unsigned>(counts[1]), kBlockThreads, 0, st>>>(
          d_meta_canon, tiles + counts[0], d_keys, bags, d_grad, ldg, lr, w, d_carry_f,
          d_carry_i, d_abort);
      SP_LAUNCHED();
      launch_pdl(sgd_carry_kernel<T>, dim3(static_cast<unsigned>((counts[1] + 7) / 8)),
                 dim3(256), 0, st, d_meta_canon, tiles + counts[0],
                 static_cast<int>(counts[1]), lr, w, d_carry_f, d_carry_i, d_abort);
    }
    if (counts[0] > 0) {
      sgd_kernel<BagT, T><<<static_cast<unsigned>(counts[0]), kBlockThreads, 0, st>>>(
          d_meta_canon, tiles, d_keys, bags, d_grad, ldg, lr, w, d_abort);
      SP_LAUNCHED();
    }
  };
  if (wt == WeightType::kF16) {
    if (bags16) go(TypeTag<__half>{}, TypeTag<uint16_t>{});
    else go(TypeTag<__half>{}, TypeTag<uint32_t>{});
  } else if (wt == WeightType::kBF16) {
    if (bags16) go(TypeTag<__nv_bfloat16>{}, TypeTag<uint16_t>{});
    else go(TypeTag<__nv_bfloat16>{}, TypeTag<uint32_t>{});
  } else {
    if (bags16) go(TypeTag<float>{}, TypeTag<uint16_t>{});
    else go(TypeTag<float>{}, TypeTag<uint32_t>{});
  }
}

size_t sgd_carry_floats(int64_t n_wide_tiles) { return static_cast<size_t>(n_wide_tiles) * 2 * kCarryF; }

void launch_init_weights(void* d_w, WeightType wt, int64_t rows, int dim, int32_t gid,
                         uint64_t seed, cudaStream_t st) {
  if (wt == WeightType::kF16)
    init_weights_kernel<__half><<<grid_for(rows * dim, 256), 256, 0, st>>>(
        static_cast<__half*>(d_w), rows, dim, gid, seed);
  else if (wt == WeightType::kBF16)
    init_weights_kernel<__nv_bfloat16><<<grid_for(rows * dim, 256), 256, 0, st>>>(
        static_cast<__nv_bfloat16*>(d_w), rows, dim, gid, seed);
  else
    init_weights_kernel<float><<<grid_for(rows * dim, 256), 256, 0, st>>>(
        static_cast<float*>(d_w), rows, dim, gid, seed);
  SP_LAUNCHED();
}

void launch_f32_to_weights(const float* d_src, void* d_dst, WeightType wt, int64_t n,
                           cudaStream_t st) {
  if (n <= 0) return;
  if (wt == WeightType::kF16) {
    f32_to_w_kernel<<<grid_for(n, 256), 256, 0, st>>>(d_src, static_cast<__half*>(d_dst), n);
    SP_LAUNCHED();
  } else if (wt == WeightType::kBF16) {
    f32_to_w_kernel<<<grid_for(n, 256), 256, 0, st>>>(d_src, static_cast<__nv_bfloat16*>(d_dst),
                                                      n);
    SP_LAUNCHED();
  } else {
    SP_CUDA(cudaMemcpyAsync(d_dst, d_src, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
}

void launch_weights_to_f32(const void* d_src, WeightType wt, float* d_dst, int64_t n,
                           cudaStream_t st) {
  if (n <= 0) return;
  if (wt == WeightType::kF16) {
    w_to_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(static_cast<const __half*>(d_src), d_dst, n);
    SP_LAUNCHED();
  } else if (wt == WeightType::kBF16) {
    w_to_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(d_src),
                                                      d_dst, n);
    SP_LAUNCHED();
  } else {
    SP_CUDA(cudaMemcpyAsync(d_dst, d_src, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
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
