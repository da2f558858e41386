// bwd.cu — K4 v2: the backward as a two-level stable counting sort fused
// with the row-wise SGD (replaces the device-wide CUB radix sort + tiled
// SGD of tbe.cu for every table of <= 2^25 rows).
//
// The sort groups the lookups of a (virtual) device by (table, row) keeping
// the CSR order among equal rows (== std::stable_sort by key). Rows of a
// table are cut into buckets of 2^shift consecutive rows:
//
//   bwd_hist    per scatter tile (2048 bags of one table): bucket histogram
//   ExclusiveSum over cnt[table][bucket][tile] -> each tile's slot in each
//               bucket (bucket-major, tile-minor == sorted order)
//   bwd_scatter per tile: stable in-tile ranking by bucket (block radix
//               sort of 2048-position chunks), write (row, bag) pairs
//   bwd_bucket  one block per bucket: row histogram -> stable placement of
//               the bags in row order (block radix sort by row, chunked) ->
//               every nonzero row bin is one run: W[row] -= lr * sum of its
//               gradient rows in sorted order (fixed reduction tree)
//
// Traffic per lookup: CSR read (twice, 8 B) + pair write (8 B) + pair read
// (8-12 B) versus ~68 B for a 26-bit 4-pass radix sort of (key, bag) pairs
// plus 8 B for the SGD pass over it. Runs never straddle buckets, so the
// SGD needs no run-boundary bookkeeping across blocks.
#include <cub/cub.cuh>

#include <atomic>

#include "bwd.h"
#include "common.h"
#include "tbe.h"

namespace sp {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kChunk = kThreads * kItems;  // positions per ranking chunk
constexpr int kLocalCap = 4096;            // bags of a bucket kept in smem

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

// table of tile / bucket ids: last t with base[t] <= x
template <class F>
__device__ __forceinline__ int find_table(int n, int64_t x, F base) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (base(mid) <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// histogram per scatter tile

__global__ void __launch_bounds__(kThreads)
    bwd_hist_kernel(const BucketMeta* __restrict__ bm, int n_tables, int batch,
                    const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                    int32_t* __restrict__ cnt) {
  __shared__ int32_t s_hist[kMaxBucketsPerTable];
  const int t = find_table(n_tables, blockIdx.x, [&](int i) { return bm[i].tbase; });
  const BucketMeta m = bm[t];
  const int j = blockIdx.x - m.tbase;
  for (int k = threadIdx.x; k < m.nb; k += kThreads) s_hist[k] = 0;
  __syncthreads();
  const int b0 = j * kScatterBags;
  const int b1 = min(batch, b0 + kScatterBags);
  const int64_t base = static_cast<int64_t>(t) * batch;
  const int p0 = off[base + b0], p1 = off[base + b1];
  for (int p = p0 + threadIdx.x; p < p1; p += kThreads)
    atomicAdd(&s_hist[__ldg(idx + p) >> m.shift], 1);
  __syncthreads();
  for (int k = threadIdx.x; k < m.nb; k += kThreads)
    cnt[m.cbase + static_cast<int64_t>(k) * m.tiles + j] = s_hist[k];
}

// ---------------------------------------------------------------------------
// stable scatter of (row, bag) pairs into bucket order

using ChunkSort = cub::BlockRadixSort<uint16_t, kThreads, kItems, uint16_t>;
using ChunkScan = cub::BlockScan<int, kThreads>;

struct ScatterShared {
  int32_t off[kScatterBags + 1];
  int32_t ctr[kMaxBucketsPerTable];
  int32_t row[kChunk];
  int32_t bag[kChunk];
  uint16_t sk[kChunk];
  union {
    typename ChunkSort::TempStorage sort;
    typename ChunkScan::TempStorage scan;
  } tmp;
};

// Ranks the chunk's items stably by key (key == sentinel for padding):
// after the call item q of this thread has sorted rank r = tid*kItems + q,
// key keys[q], original index vals[q], and run start rs[q] (first rank of
// its key). sk receives the sorted keys.
__device__ __forceinline__ void rank_chunk(uint16_t (&keys)[kItems], uint16_t (&vals)[kItems],
                                           int (&rs)[kItems], int end_bit, uint16_t* sk,
                                           typename ChunkSort::TempStorage& ts,
                                           typename ChunkScan::TempStorage& tsc) {
  ChunkSort(ts).Sort(keys, vals, 0, end_bit);
  const int tid = threadIdx.x;
#pragma unroll
  for (int q = 0; q < kItems; ++q) sk[tid * kItems + q] = keys[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kItems; ++q) {
    const int r = tid * kItems + q;
    rs[q] = (r == 0 || sk[r - 1] != keys[q]) ? r : 0;
  }
  ChunkScan(tsc).InclusiveScan(rs, rs, cub::Max());
}

__global__ void __launch_bounds__(kThreads)
    bwd_scatter_kernel(const BucketMeta* __restrict__ bm, int n_tables, int batch,
                       const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                       const int32_t* __restrict__ cpos, int32_t* __restrict__ prow,
                       int32_t* __restrict__ pbag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ScatterShared& sh = *reinterpret_cast<ScatterShared*>(smem_raw);
  const int t = find_table(n_tables, blockIdx.x, [&](int i) { return bm[i].tbase; });
  const BucketMeta m = bm[t];
  const int j = blockIdx.x - m.tbase;
  const int tid = threadIdx.x;
  const int b0 = j * kScatterBags;
  const int nbag = min(batch - b0, kScatterBags);
  const int64_t base = static_cast<int64_t>(t) * batch + b0;
  for (int i = tid; i <= nbag; i += kThreads) sh.off[i] = off[base + i];
  for (int k = tid; k < m.nb; k += kThreads)
    sh.ctr[k] = cpos[m.cbase + static_cast<int64_t>(k) * m.tiles + j];
  __syncthreads();
  const int p0 = sh.off[0], p1 = sh.off[nbag];
  const uint16_t sentinel = static_cast<uint16_t>(m.nb);
  for (int c0 = p0; c0 < p1; c0 += kChunk) {
    uint16_t keys[kItems], vals[kItems];
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const int i = tid * kItems + q;
      const int p = c0 + i;
      vals[q] = static_cast<uint16_t>(i);
      if (p < p1) {
        const int row = __ldg(idx + p);
        int lo = 0, hi = nbag - 1;  // bag: last b with off[b] <= p
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sh.off[mid] <= p) lo = mid; else hi = mid - 1;
        }
        sh.row[i] = row;
        sh.bag[i] = b0 + lo;
        keys[q] = static_cast<uint16_t>(row >> m.shift);
      } else {
        keys[q] = sentinel;
      }
    }
    __syncthreads();
    int rs[kItems];
    rank_chunk(keys, vals, rs, m.key_bits, sh.sk, sh.tmp.sort, sh.tmp.scan);
    int last[kItems];
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const int r = tid * kItems + q;
      last[q] = 0;
      if (keys[q] == sentinel) continue;
      const int dest = sh.ctr[keys[q]] + (r - rs[q]);
      prow[dest] = sh.row[vals[q]];
      pbag[dest] = sh.bag[vals[q]];
      last[q] = (r == kChunk - 1 || sh.sk[r + 1] != keys[q]) ? r - rs[q] + 1 : 0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kItems; ++q)
      if (last[q]) sh.ctr[keys[q]] += last[q];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// per bucket: row histogram -> stable placement -> SGD over the row runs

template <int L_, int V_, int P_, int U_>
struct Geo {
  static constexpr int L = L_, V = V_, P = P_, U = U_;
  static constexpr int S = 32 / P, GB = S / L;
};
template <int CLS> struct ShortGeo;  // runs of < kLong lookups, P runs per warp
template <> struct ShortGeo<0> : Geo<1, 1, 16, 2> {};
template <> struct ShortGeo<1> : Geo<2, 1, 16, 1> {};
template <> struct ShortGeo<2> : Geo<2, 2, 16, 1> {};
template <> struct ShortGeo<3> : Geo<4, 2, 8, 1> {};
template <> struct ShortGeo<4> : Geo<8, 2, 4, 1> {};
template <> struct ShortGeo<5> : Geo<16, 2, 2, 1> {};
template <int CLS> struct LongGeo;  // one long run per warp
template <> struct LongGeo<0> : Geo<1, 1, 1, 4> {};
template <> struct LongGeo<1> : Geo<2, 1, 1, 4> {};
template <> struct LongGeo<2> : Geo<4, 1, 1, 4> {};
template <> struct LongGeo<3> : Geo<8, 1, 1, 4> {};
template <> struct LongGeo<4> : Geo<16, 1, 1, 8> {};
template <> struct LongGeo<5> : Geo<32, 1, 1, 8> {};

constexpr int kLong = 32;

struct BucketShared {
  int32_t cnt[kMaxBins];    // row histogram, then run starts (+ count)
  int32_t run[kMaxBins];    // compacted nonzero bins
  int32_t bag[kLocalCap];   // bags in sorted order (n <= kLocalCap)
  int32_t row[kChunk];      // chunk staging
  int32_t cbag[kChunk];
  uint16_t sk[kChunk];
  int nrun;
  int next;
  union {
    typename ChunkSort::TempStorage sort;
    typename ChunkScan::TempStorage scan;
  } tmp;
};

// SGD of runs [j, j+P) (P spans; short) or run j alone (P == 1, long).
template <class G>
__device__ __forceinline__ int bucket_round(const TableMeta& m, int64_t row0, int j, int jend,
                                           int lane, const BucketShared& sh,
                                           const int32_t* __restrict__ gbag,
                                           const float* __restrict__ grad, int64_t ldg,
                                           float lr, float* __restrict__ w) {
  constexpr int L = G::L, V = G::V, P = G::P, U = G::U, S = G::S, GB = G::GB;
  const int span = lane / S, ls = lane % S, g = ls / L, sub = ls % L;
  const int u = j + span;
  bool valid = u < jend;
  int beg = 0, end = 0, bin = 0;
  if (valid) {
    // after placement cnt[bin] is the run's end; runs are the nonzero bins
    // in order, so a run begins where the previous one ends
    bin = sh.run[u];
    end = sh.cnt[bin];
    beg = u == 0 ? 0 : sh.cnt[sh.run[u - 1]];
    valid = P == 1 || span == 0 || end - beg < kLong;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, valid && ls == 0);
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
    wrow = w + m.woff + (row0 + bin) * m.dim + 4 * sub;
    if (g == 0)
#pragma unroll
      for (int q = 0; q < V; ++q) wold[q] = *reinterpret_cast<const float4*>(wrow + 4 * L * q);
    const float* gcol = grad + m.lcol + 4 * sub;
    for (int k = beg + g; k < end; k += GB * U) {
      int bg[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int kk = k + q * GB;
        bg[q] = kk < end ? (gbag ? __ldcg(gbag + kk) : sh.bag[kk]) : -1;  // written by this block
      }
      float4 v[U][V];
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int c = 0; c < V; ++c)
          v[q][c] = bg[q] >= 0 ? ldg_f4(gcol + static_cast<int64_t>(bg[q]) * ldg + 4 * L * c)
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
      r.x = fmaf(-lr, acc[c].x, wold[c].x);
      r.y = fmaf(-lr, acc[c].y, wold[c].y);
      r.z = fmaf(-lr, acc[c].z, wold[c].z);
      r.w = fmaf(-lr, acc[c].w, wold[c].w);
      *reinterpret_cast<float4*>(wrow + 4 * L * c) = r;
    }
  }
  return nvalid;
}

__device__ __forceinline__ int bucket_round_generic(const TableMeta& m, int64_t row0, int j,
                                                   int lane, const BucketShared& sh,
                                                   const int32_t* __restrict__ gbag,
                                                   const float* __restrict__ grad,
                                                   int64_t ldg, float lr,
                                                   float* __restrict__ w) {
  const int bin = sh.run[j];
  const int end = sh.cnt[bin];
  const int beg = j == 0 ? 0 : sh.cnt[sh.run[j - 1]];
  for (int c0 = 0; c0 < m.dim; c0 += 32) {
    const int c = c0 + lane;
    float acc = 0.f;
    for (int k = beg; k < end; ++k) {
      const int bg = gbag ? __ldcg(gbag + k) : sh.bag[k];
      if (c < m.dim) acc += __ldg(grad + static_cast<int64_t>(bg) * ldg + m.lcol + c);
    }
    if (c < m.dim) {
      float* p = w + m.woff + (row0 + bin) * m.dim + c;
      *p = fmaf(-lr, acc, *p);
    }
  }
  return 1;
}

__global__ void __launch_bounds__(kThreads)
    bwd_bucket_kernel(const TableMeta* __restrict__ meta, const BucketMeta* __restrict__ bm,
                      int n_tables, const int32_t* __restrict__ cpos, int64_t total,
                      const int32_t* __restrict__ prow, const int32_t* __restrict__ pbag,
                      int32_t* __restrict__ scratch, const float* __restrict__ grad,
                      int64_t ldg, float lr, float* __restrict__ w,
                      uint32_t* __restrict__ sorted_keys, uint32_t* __restrict__ sorted_bags,
                      int do_sgd) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BucketShared& sh = *reinterpret_cast<BucketShared*>(smem_raw);
  const int t = find_table(n_tables, blockIdx.x, [&](int i) { return bm[i].bbase; });
  const BucketMeta b = bm[t];
  const int k = blockIdx.x - b.bbase;
  const int64_t s = cpos[b.cbase + static_cast<int64_t>(k) * b.tiles];
  const int64_t e = k + 1 < b.nb ? cpos[b.cbase + static_cast<int64_t>(k + 1) * b.tiles]
                    : (t + 1 < n_tables ? cpos[bm[t + 1].cbase] : total);
  const int n = static_cast<int>(e - s);
  if (n == 0) return;
  const TableMeta m = meta[t];
  const int tid = threadIdx.x;
  const int64_t row0 = static_cast<int64_t>(k) << b.shift;
  const int64_t span_rows = int64_t(1) << b.shift;
  const int bins = static_cast<int>(m.rows - row0 < span_rows ? m.rows - row0 : span_rows);
  const int mask = (1 << b.shift) - 1;
  // 1. row histogram of the bucket
  for (int i = tid; i < bins; i += kThreads) sh.cnt[i] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += kThreads) atomicAdd(&sh.cnt[__ldg(prow + s + i) & mask], 1);
  __syncthreads();
  // 2. exclusive scan of the bins (run starts) and the run list
  {
    constexpr int kPer = kMaxBins / kThreads;
    static_assert(kPer * kThreads == kMaxBins, "bins per thread");
    int sum = 0, nz = 0;
    int cv[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int i = tid * kPer + q;
      cv[q] = i < bins ? sh.cnt[i] : 0;
      sum += cv[q];
      nz += cv[q] > 0;
    }
    int start = 0, rstart = 0, nrun = 0, tot = 0;
    ChunkScan(sh.tmp.scan).ExclusiveSum(sum, start, tot);
    __syncthreads();
    ChunkScan(sh.tmp.scan).ExclusiveSum(nz, rstart, nrun);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int i = tid * kPer + q;
      if (i < bins) sh.cnt[i] = start;  // run start (advanced to run end below)
      if (cv[q] > 0) sh.run[rstart++] = i;
      start += cv[q];
    }
    if (tid == 0) {
      sh.nrun = nrun;
      sh.next = 0;
    }
  }
  __syncthreads();
  // 3. stable placement of the bags in row order (chunks of kChunk)
  int32_t* gbag = n > kLocalCap ? scratch + s : nullptr;
  const uint16_t sentinel = static_cast<uint16_t>(mask + 1);  // > any bin
  for (int c0 = 0; c0 < n; c0 += kChunk) {
    uint16_t keys[kItems], vals[kItems];
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const int i = tid * kItems + q;
      const int p = c0 + i;
      vals[q] = static_cast<uint16_t>(i);
      if (p < n) {
        const int row = __ldg(prow + s + p);
        sh.row[i] = row;
        sh.cbag[i] = __ldg(pbag + s + p);
        keys[q] = static_cast<uint16_t>(row & mask);
      } else {
        keys[q] = sentinel;
      }
    }
    __syncthreads();
    int rs[kItems];
    rank_chunk(keys, vals, rs, b.shift + 1, sh.sk, sh.tmp.sort, sh.tmp.scan);
    int adv[kItems];
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const int r = tid * kItems + q;
      adv[q] = 0;
      if (keys[q] == sentinel) continue;
      const int dest = sh.cnt[keys[q]] + (r - rs[q]);
      const int bag = sh.cbag[vals[q]];
      if (gbag) gbag[dest] = bag; else sh.bag[dest] = bag;
      if (sorted_keys) {
        sorted_keys[s + dest] = m.rowbase + static_cast<uint32_t>(sh.row[vals[q]]);
        sorted_bags[s + dest] = static_cast<uint32_t>(bag);
      }
      adv[q] = (r == kChunk - 1 || sh.sk[r + 1] != keys[q]) ? r - rs[q] + 1 : 0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kItems; ++q)
      if (adv[q]) sh.cnt[keys[q]] += adv[q];  // -> run end once all chunks are placed
    __syncthreads();
  }
  if (!do_sgd) return;  // sort-only (diagnostics)
  // 4. SGD: runs are the nonzero bins in order; warps claim chunks of runs
  const int lane = tid & 31;
  const int nrun = sh.nrun;
  for (;;) {
    int j0 = 0;
    if (lane == 0) j0 = atomicAdd(&sh.next, 16);
    j0 = __shfl_sync(0xffffffffu, j0, 0);
    if (j0 >= nrun) break;
    const int jend = min(nrun, j0 + 16);
    int j = j0;
    while (j < jend) {
      const int bin = sh.run[j];
      const int len = sh.cnt[bin] - (j == 0 ? 0 : sh.cnt[sh.run[j - 1]]);
      const bool lng = len >= kLong;
      switch (m.cls) {
#define SP_BUCKET_CASE(C)                                                              \
  case C:                                                                              \
    j += lng ? bucket_round<LongGeo<C>>(m, row0, j, j + 1, lane, sh, gbag, grad, ldg, lr, w) \
             : bucket_round<ShortGeo<C>>(m, row0, j, jend, lane, sh, gbag, grad, ldg, lr, w); \
    break;
        SP_BUCKET_CASE(0)
        SP_BUCKET_CASE(1)
        SP_BUCKET_CASE(2)
        SP_BUCKET_CASE(3)
        SP_BUCKET_CASE(4)
        SP_BUCKET_CASE(5)
#undef SP_BUCKET_CASE
        default:
          j += bucket_round_generic(m, row0, j, lane, sh, gbag, grad, ldg, lr, w);
      }
    }
  }
}

int grid_of(int64_t n) { return static_cast<int>(n); }

}  // namespace

bool bucket_plan(const std::vector<TableMeta>& canon, const std::vector<int64_t>& table_nnz,
                 int batch, std::vector<BucketMeta>& out, int64_t& n_cnt, int& n_tiles,
                 int& n_buckets) {
  out.clear();
  int64_t cbase = 0;
  int tbase = 0, bbase = 0;
  for (size_t i = 0; i < canon.size(); ++i) {
    const TableMeta& m = canon[i];
    int rowbits = 1;
    while (rowbits < 40 && (int64_t(1) << rowbits) < m.rows) ++rowbits;
    // buckets of ~kTargetBucket lookups, bins <= kMaxBins, buckets <= kMaxBucketsPerTable
    const int64_t nnz = i < table_nnz.size() ? table_nnz[i] : 0;
    int b = 0;
    while ((int64_t(kTargetBucket) << b) < nnz && b < rowbits) ++b;
    int min_b = 0;
    while ((int64_t(kMaxBins) << min_b) < (int64_t(1) << rowbits)) ++min_b;
    b = std::max(b, min_b);
    b = std::min(b, rowbits);
    const int shift = rowbits - b;
    const int64_t nb = ((m.rows - 1) >> shift) + 1;
    if (nb > kMaxBucketsPerTable || (int64_t(1) << shift) > kMaxBins) return false;
    BucketMeta bmeta{};
    bmeta.shift = shift;
    bmeta.nb = static_cast<int32_t>(nb);
    int kb = 1;
    while ((int64_t(1) << kb) <= nb) ++kb;  // bits for 0..nb (sentinel nb)
    bmeta.key_bits = kb;
    bmeta.tiles = (batch + kScatterBags - 1) / kScatterBags;
    bmeta.cbase = cbase;
    bmeta.tbase = tbase;
    bmeta.bbase = bbase;
    cbase += nb * bmeta.tiles;
    tbase += bmeta.tiles;
    bbase += static_cast<int32_t>(nb);
    out.push_back(bmeta);
  }
  n_cnt = cbase;
  n_tiles = tbase;
  n_buckets = bbase;
  return true;
}

void set_bwd_attributes() {
  // function attributes are per device: once per device of this process
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  SP_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (done.load() & bit) return;
  SP_CUDA(cudaFuncSetAttribute(bwd_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sizeof(ScatterShared))));
  SP_CUDA(cudaFuncSetAttribute(bwd_bucket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sizeof(BucketShared))));
  done.fetch_or(bit);
}

void launch_bwd_partition(const BucketMeta* d_bm, int n_tables, int n_tiles, int64_t n_cnt,
                          int batch, const int32_t* d_off, const int32_t* d_idx,
                          int32_t* d_cnt, int32_t* d_cpos, void* d_temp, size_t temp_bytes,
                          int32_t* d_prow, int32_t* d_pbag, cudaStream_t st) {
  if (n_tables <= 0 || n_tiles <= 0) return;
  set_bwd_attributes();
  bwd_hist_kernel<<<grid_of(n_tiles), kThreads, 0, st>>>(d_bm, n_tables, batch, d_off, d_idx,
                                                          d_cnt);
  SP_LAUNCHED();
  size_t tb = temp_bytes;
  SP_CUDA(cub::DeviceScan::ExclusiveSum(d_temp, tb, d_cnt, d_cpos, n_cnt, st));
  bwd_scatter_kernel<<<grid_of(n_tiles), kThreads, sizeof(ScatterShared), st>>>(
      d_bm, n_tables, batch, d_off, d_idx, d_cpos, d_prow, d_pbag);
  SP_LAUNCHED();
}

void launch_bwd_buckets(const TableMeta* d_meta, const BucketMeta* d_bm, int n_tables,
                        int n_buckets, const int32_t* d_cpos, int64_t nnz,
                        const int32_t* d_prow, const int32_t* d_pbag, int32_t* d_scratch,
                        const float* d_grad, int64_t ldg, float lr, float* d_w,
                        uint32_t* d_sorted_keys, uint32_t* d_sorted_bags, bool do_sgd,
                        cudaStream_t st) {
  if (n_tables <= 0 || n_buckets <= 0 || nnz <= 0) return;
  set_bwd_attributes();
  bwd_bucket_kernel<<<grid_of(n_buckets), kThreads, sizeof(BucketShared), st>>>(
      d_meta, d_bm, n_tables, d_cpos, nnz, d_prow, d_pbag, d_scratch, d_grad, ldg, lr, d_w,
      d_sorted_keys, d_sorted_bags, do_sgd ? 1 : 0);
  SP_LAUNCHED();
}

size_t bwd_scan_temp_bytes(int64_t n_cnt, cudaStream_t st) {
  size_t tb = 0;
  SP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, static_cast<const int32_t*>(nullptr),
                                        static_cast<int32_t*>(nullptr), n_cnt, st));
  return tb;
}

}  // namespace sp
