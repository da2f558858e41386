// sort.cu — K4a: the backward's stable sort of one device's lookups by
// (table, row), hand-written for sm_100a. It replaces the device-wide CUB
// onesweep radix sort (three 8-bit passes over 6-byte pairs with a decoupled
// look-back per pass, latency-bound at ~22 warps/SM on B200).
//
// The sorted order is the one oracle.hpp:149's bwd stage needs for a
// deterministic duplicate-row reduction: std::stable_sort of the
// lookups by key = rowbase_t + row, ties in CSR position order. It uses what
// the CSR already gives: the lookups of a table are contiguous and in bag
// order, so each table sorts independently into its own CSR position range,
// and the bag payload never needs sorting (it is the position order).
//
// One MSD bucketing pass, then warp-local LSD passes, no look-back:
//   P1 sort_count    a block per tile (wb consecutive bags of one table):
//                    histogram of the tile's lookups over the table's nb row
//                    buckets (row >> lo) -> cnt[tile][bucket]
//   P2 sort_scan     a block per table: bucket-major / tile-minor exclusive
//                    scan from the table's CSR start -> each (tile, bucket)
//                    slot's first sorted position, and the bucket starts
//   P3 sort_scatter  a block per tile, 8192 positions at a time in shared
//                    memory: bag of every position (filled bag by bag from
//                    the offsets), per-warp bucket histograms of contiguous
//                    sub-ranges, their bucket-major scan, then each warp
//                    ranks its sub-range in order with match.any (stable) and
//                    writes (row & (2^lo - 1), bag) packed into the bucket slot
//   P4 sort_bucket   a warp per bucket: stable LSD counting sort of its
//                    lookups by the low row bits, <= 10-bit digits (one pass
//                    when lo <= 10), the same match.any ranking; the last
//                    pass writes the final key = rowbase + row and bag
//
// Traffic per lookup: ids read twice (8 B), packed pair written and read
// (4 + 4 B with 16-bit bags), key + bag written (6 B) = 22 B (+ the offsets
// twice, + the count matrix), against 3 x 12 B for CUB's passes plus 10 B
// for its key build. sort_plan(): <= 1024 buckets per table (a warp's
// histogram of them fits shared memory), enough of them for <= 10 low bits
// and ~4096 lookups per bucket; tiles of 4096-32768 lookups.
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <climits>
#include <cmath>

#include "common.h"
#include "tbe.h"

namespace sp {
namespace {

constexpr int kWarps = 8;                  // warps per block (P1, P3, P4)
constexpr int kThreads = 32 * kWarps;
constexpr int kScanThreads = 1024;         // P2 block
constexpr int kMaxBuckets = 1024;          // buckets per table
// P3 positions staged at a time, lookups per P4 bucket (sort_plan): 8192 /
// 4096 measured 6 % faster than 4096 / 2048 at cfg3 (fewer histogram
// zero / scan rounds per lookup in both passes)
constexpr int kCap3 = 8192;
constexpr double kBucketTarget = 4096.0;
// P4's warp-per-bucket kernel (buckets of <= 512 lookups): digits of <= 6
// bits whatever the table's db (which suits its average bucket), so the
// warp's histogram is 96 words instead of 1056: sort 0.820 -> 0.800 ms at
// cfg3 (5 and 7 bits the same within 0.3 %)
constexpr int kSmallDigitBits = 6;
constexpr int kMaxDigitBits = 10;          // <= 10-bit digits (sort_plan picks per table)
constexpr int kSmallCapScan = 512;         // = kSmallCap: buckets above go to sort_big_kernel          // P4 digit (a warp's histogram: 4 KB)
// a warp histogram of 2^db bins takes hist_words(db) words (+ one pad word
// per lane segment); kernels get the launch's widest as `hw`
__host__ __device__ constexpr int hist_words(int db) { return (1 << db) + 32; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Shared memory through 32-bit shared-window addresses (a generic pointer
// into dynamic shared memory is re-translated at every access).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void atoms_inc(uint32_t a) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a) : "memory");
}

// Packed intermediate: low row bits and the bag id.
struct Mid32 {  // lo <= 16 bits, 16-bit bags
  using type = uint32_t;
  __device__ static __forceinline__ type pack(uint32_t lo, uint32_t bag) { return (lo << 16) | bag; }
  __device__ static __forceinline__ uint32_t lo(type m) { return m >> 16; }
  __device__ static __forceinline__ uint32_t bag(type m) { return m & 0xffffu; }
};
struct Mid64 {
  using type = unsigned long long;
  __device__ static __forceinline__ type pack(uint32_t lo, uint32_t bag) {
    return (static_cast<type>(lo) << 32) | bag;
  }
  __device__ static __forceinline__ uint32_t lo(type m) { return static_cast<uint32_t>(m >> 32); }
  __device__ static __forceinline__ uint32_t bag(type m) { return static_cast<uint32_t>(m); }
};

__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory");
}
template <class BagT>
__device__ __forceinline__ uint32_t lds_bag(uint32_t a) {
  if constexpr (sizeof(BagT) == 2) return lds_u16(a);
  else return lds(a);
}
template <class BagT>
__device__ __forceinline__ void sts_bag(uint32_t a, uint32_t v) {
  if constexpr (sizeof(BagT) == 2) sts_u16(a, static_cast<uint16_t>(v));
  else sts(a, v);
}

__device__ __forceinline__ void atoms_or(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Stable warp ranking of R chunks of 32 consecutive items (chunk r = items
// [32 r, 32 r + 32), lane order = item order). cur(r) is the shared address
// of the item's cursor (invalid lanes: a spare word); the word at
// cur(r) + moff is its peer mask, zero between uses. Each lane ORs its bit
// into its key's mask, reads back the group of lanes with the same key, the
// group's lowest lane advances the cursor and clears the mask, and emit(r,
// slot) gets slot = cursor + rank among the lower lanes of the group. (A
// shared-memory OR is far cheaper than match.any on 32 distinct keys.)
template <int R, class CurF, class EmitF>
__device__ __forceinline__ void warp_rank(int nchunks, unsigned lt, unsigned me, uint32_t moff,
                                          CurF&& cur, EmitF&& emit) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r >= nchunks) break;
    const uint32_t c = cur(r);
    atoms_or(c + moff, me);
    __syncwarp();
    const unsigned peers = lds(c + moff);
    const uint32_t s0 = lds(c);
    __syncwarp();
    // the group's lowest lane clears the mask and advances the cursor
    // (predicated stores: no divergent branch)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.eq.u32 p, %2, 0;\n\t"
        "@p st.shared.u32 [%0], 0;\n\t"
        "@p st.shared.u32 [%1], %3;\n\t}" ::"r"(c + moff),
        "r"(c), "r"(peers & (me - 1u)), "r"(s0 + __popc(peers))
        : "memory");
    __syncwarp();
    emit(r, s0 + __popc(peers & lt));
  }
}

// ---------------------------------------------------------------------------
// P1: per tile bucket histogram.

__global__ void __launch_bounds__(kThreads)
    sort_count_kernel(const SortTable* __restrict__ tabs, const int2* __restrict__ tiles,
                      int batch, const int32_t* __restrict__ off,
                      const int32_t* __restrict__ idx, int* __restrict__ cnt) {
  __shared__ uint32_t h[kMaxBuckets];
  const int2 tl = tiles[blockIdx.x];
  const SortTable s = tabs[tl.x];
  const int b0 = tl.y * s.wb, b1 = min(batch, b0 + s.wb);
  const int64_t ob = static_cast<int64_t>(tl.x) * batch;
  const int q0 = __ldg(off + ob + b0), q1 = __ldg(off + ob + b1);
  for (int k = threadIdx.x; k < s.nb; k += kThreads) h[k] = 0;
  __syncthreads();
  const int lo = s.lo;
  const uint32_t hb = smem_addr(h);
  int p = q0 + threadIdx.x;
  for (; p + 3 * kThreads < q1; p += 4 * kThreads) {  // four ids in flight per thread
    const int r0 = __ldg(idx + p), r1 = __ldg(idx + p + kThreads);
    const int r2 = __ldg(idx + p + 2 * kThreads), r3 = __ldg(idx + p + 3 * kThreads);
    atoms_inc(hb + 4u * (r0 >> lo));
    atoms_inc(hb + 4u * (r1 >> lo));
    atoms_inc(hb + 4u * (r2 >> lo));
    atoms_inc(hb + 4u * (r3 >> lo));
  }
  for (; p < q1; p += kThreads) atoms_inc(hb + 4u * (__ldg(idx + p) >> lo));
  __syncthreads();
  int* out = cnt + s.cbase + static_cast<int64_t>(tl.y) * s.nb;
  for (int k = threadIdx.x; k < s.nb; k += kThreads) out[k] = h[k];
}

// ---------------------------------------------------------------------------
// P2: per table, bucket-major exclusive scan of the count matrix from the
// table's CSR start: cnt[tile][bucket] becomes the slot's first position,
// bstart[bucket] the bucket's (bstart[nb] = the table end).

__global__ void __launch_bounds__(kScanThreads)
    sort_scan_kernel(const SortTable* __restrict__ tabs, int t0, int batch,
                     const int32_t* __restrict__ off, int* __restrict__ cnt,
                     int* __restrict__ bstart, int2* __restrict__ big, int* __restrict__ n_big) {
  pdl_wait();  // launched as a programmatic dependent (launch_sort_t)
  using BlockScan = cub::BlockScan<int, kScanThreads>;
  __shared__ typename BlockScan::TempStorage tmp;
  const int t = t0 + blockIdx.x;
  const SortTable s = tabs[t];
  int* c = cnt + s.cbase;
  int* bs = bstart + s.bkbase;
  const int nb = s.nb, nt = s.nwt;
  const int k = threadIdx.x;  // nb <= kMaxBuckets <= kScanThreads
  int tot = 0;
  if (k < nb) {
    int col = 0;
    for (; col + 8 <= nt; col += 8) {
      int v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = c[static_cast<int64_t>(col + u) * nb + k];
#pragma unroll
      for (int u = 0; u < 8; ++u) tot += v[u];
    }
    for (; col < nt; ++col) tot += c[static_cast<int64_t>(col) * nb + k];
  }
  int ex, agg;
  BlockScan(tmp).ExclusiveSum(tot, ex, agg);
  const int base = __ldg(off + static_cast<int64_t>(t) * batch);
  if (k < nb) {
    int run = base + ex;
    bs[k] = run;
    int col = 0;
    for (; col + 8 <= nt; col += 8) {
      int v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = c[static_cast<int64_t>(col + u) * nb + k];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        c[static_cast<int64_t>(col + u) * nb + k] = run;
        run += v[u];
      }
    }
    for (; col < nt; ++col) {
      int* e = c + static_cast<int64_t>(col) * nb + k;
      const int v = *e;
      *e = run;
      run += v;
    }
  }
  if (k == 0) bs[nb] = base + agg;
  if (k < nb && tot > kSmallCapScan) big[atomicAdd(n_big, 1)] = make_int2(t, k);
}

// ---------------------------------------------------------------------------
// P3: stable scatter of a tile's lookups into their (tile, bucket) slots,
// kCap3 positions at a time: warp w takes the contiguous sub-range
// [w m / 8, (w + 1) m / 8) (<= kItems3 ids, kept in registers).
// Shared memory: whist[kWarps][nb_max + 1] | masks[kWarps][nb_max + 1] |
// run[nb_max] | s_bag[kCap3].

constexpr int kR3 = kCap3 / kWarps / 32;  // chunks of 32 per warp and stage
constexpr int kOffWin = 2048;              // bag offsets staged at a time

template <class BagT, class M>
__global__ void __launch_bounds__(kThreads, 4)
    sort_scatter_kernel(const SortTable* __restrict__ tabs, const int2* __restrict__ tiles,
                        int batch, const int32_t* __restrict__ off,
                        const int32_t* __restrict__ idx, const int* __restrict__ cnt,
                        typename M::type* __restrict__ mid, int nb_max) {
  pdl_wait();  // launched as a programmatic dependent (launch_sort_t)
  extern __shared__ __align__(16) unsigned char smem[];
  const int wstride = nb_max + 1;  // + the spare cursor of invalid lanes
  uint32_t* whist = reinterpret_cast<uint32_t*>(smem);
  uint32_t* run = whist + 2 * kWarps * wstride;  // after the cursors and the peer masks
  const uint32_t a_bag = smem_addr(run + nb_max);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int2 tl = tiles[blockIdx.x];
  const SortTable s = tabs[tl.x];
  const int nb = s.nb, lo = s.lo;
  const int b0 = tl.y * s.wb, b1 = min(batch, b0 + s.wb);
  const int32_t* o = off + static_cast<int64_t>(tl.x) * batch;
  const int q0 = __ldg(o + b0), q1 = __ldg(o + b1);
  const int* slots = cnt + s.cbase + static_cast<int64_t>(tl.y) * nb;
  for (int k = threadIdx.x; k < nb; k += kThreads) run[k] = slots[k];
  const uint32_t lmask = (1u << lo) - 1u;
  const unsigned lt = lanemask_lt(), me = 1u << lane;
  const uint32_t wh = smem_addr(whist + warp * wstride);
  const uint32_t mofs = 4u * kWarps * wstride;  // cursor -> its peer mask
  for (int k = lane; k < wstride; k += 32) sts(wh + mofs + 4u * k, 0u);
  __shared__ int s_off[kOffWin + 1];
  __shared__ int s_next;
  int bs = b0;  // a bag that begins at or before the stage start
  for (int c0 = q0; c0 < q1; c0 += kCap3) {
    const int m = min(kCap3, q1 - c0);
    const int i0 = m * warp / kWarps, i1 = m * (warp + 1) / kWarps;
    const int nch = (i1 - i0 + 31) >> 5;
    uint32_t row[kR3];
#pragma unroll
    for (int r = 0; r < kR3; ++r) {
      if (r >= nch) break;
      const int i = i0 + 32 * r + lane;
      row[r] = i < i1 ? static_cast<uint32_t>(__ldg(idx + c0 + i)) : 0u;
    }
    // bag of every staged position: the offsets of bags [bs, ...) come in
    // windows of kOffWin (coalesced), each thread fills its bags' positions
    const int c1 = c0 + m;
    for (int w0 = bs;; w0 += kOffWin) {
      const int nw = min(kOffWin, b1 - w0);
      for (int j = threadIdx.x; j <= nw; j += kThreads) s_off[j] = __ldg(o + w0 + j);
      __syncthreads();
      for (int j = threadIdx.x; j < nw; j += kThreads) {
        const int pb = max(s_off[j], c0), pe = min(s_off[j + 1], c1);
        for (int p = pb; p < pe; ++p) sts_bag<BagT>(a_bag + sizeof(BagT) * (p - c0), w0 + j);
      }
      const bool more = nw == kOffWin && s_off[nw] < c1;
      __syncthreads();  // s_off is reloaded
      if (!more) {
        // the next stage starts in the last bag that began at or before c1
        if (threadIdx.x == 0) {
          int lo = 0, hi = nw;  // last j with s_off[j] <= c1 (s_off[0] <= c0 < c1)
          while (lo < hi) {
            const int mid_j = (lo + hi + 1) >> 1;
            if (s_off[mid_j] <= c1) lo = mid_j; else hi = mid_j - 1;
          }
          s_next = w0 + lo;
        }
        break;
      }
    }
    for (int k = lane; k < wstride; k += 32) sts(wh + 4u * k, 0u);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kR3; ++r) {
      if (r >= nch) break;
      if (i0 + 32 * r + lane < i1) atoms_inc(wh + 4u * (row[r] >> lo));
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nb; k += kThreads) {  // bucket-major, warp-minor
      uint32_t r = run[k];
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t v = whist[w * wstride + k];
        whist[w * wstride + k] = r;
        r += v;
      }
      run[k] = r;
    }
    __syncthreads();
    auto valid = [&](int r) { return i0 + 32 * r + lane < i1; };
    warp_rank<kR3>(
        nch, lt, me, mofs,
        [&](int r) { return wh + 4u * (valid(r) ? row[r] >> lo : static_cast<uint32_t>(nb_max)); },
        [&](int r, uint32_t slot) {
          const int i = i0 + 32 * r + lane;
          if (i < i1)
            mid[slot] = M::pack(row[r] & lmask, lds_bag<BagT>(a_bag + sizeof(BagT) * i));
        });
    __syncthreads();  // s_bag is refilled for the next stage
    bs = s_next;
  }
}

// ---------------------------------------------------------------------------
// P4: stable LSD counting sort of every bucket by its low row bits, in passes
// of <= 10-bit digits, through shared memory: a bucket is read from d_mid
// once (all loads in flight), every pass ranks it into a shared stage, and
// the sorted bucket is written out in order (coalesced keys and bags; a
// scattered 4-byte store per item would cost a whole L2 sector request).
//   sort_bucket_kernel  a warp per bucket of <= kSmallCap lookups (the
//                       bucket lives in the warp's registers, kR4 chunks)
//   sort_big_kernel     a block per larger bucket (P2 listed them): warp w
//                       holds the contiguous sub-range [w n / 8, (w+1) n / 8)
//                       in registers, digits scanned digit-major / warp-minor
//                       across the block; buckets above kBigCap (or 8-byte
//                       pairs) take an unstaged warp path through the
//                       scratch half of d_mid
// A warp histogram has one pad word per lane segment (bin d at d + d / seg),
// so the segment scan is free of bank conflicts.

constexpr int kR4 = 16;           // chunks of 32 items per warp in registers
constexpr int kSmallCap = 32 * kR4;
constexpr int kBigCap = 8192;
constexpr int kRB = kBigCap / kWarps / 32;  // chunks per warp in sort_big_kernel

struct DigitPass {
  int shift, seg_shift;
  int nbin;
  uint32_t dmask;
  __device__ DigitPass(int lo, int pass, int db) {
    shift = pass * db;
    const int bits = min(db, lo - shift);
    nbin = 1 << bits;
    seg_shift = bits > 5 ? bits - 5 : 0;  // bins per lane segment = 2^seg_shift
    dmask = static_cast<uint32_t>(nbin - 1);
  }
  __device__ uint32_t digit(uint32_t lo_bits) const { return (lo_bits >> shift) & dmask; }
  __device__ uint32_t at(uint32_t h, uint32_t d) const { return h + 4u * (d + (d >> seg_shift)); }
  __device__ int words() const { return nbin + (nbin >> seg_shift); }
};

// Exclusive scan of a warp's histogram (lane l owns bins [l seg, (l+1) seg)).
__device__ __forceinline__ void warp_hist_scan(const DigitPass& dp, uint32_t h, uint32_t origin,
                                               int lane) {
  const int seg = 1 << dp.seg_shift;
  const bool own = lane * seg < dp.nbin;
  const uint32_t hs = h + 4u * lane * (seg + 1);
  uint32_t sum = 0;
  if (own)
    for (int k = 0; k < seg; ++k) sum += lds(hs + 4u * k);
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  uint32_t r = origin + incl - sum;
  if (own)
    for (int k = 0; k < seg; ++k) {
      const uint32_t x = lds(hs + 4u * k);
      sts(hs + 4u * k, r);
      r += x;
    }
}

// Unstaged warp path (large buckets with no stage, 8-byte pairs): passes
// ping-pong through scratch, the last one stores keys / bags in place.
template <class BagT, class M>
__device__ void sort_bucket_unstaged(const SortTable& s, int bk, int beg, int end, uint32_t h,
                                     uint32_t mofs, int hw, typename M::type* __restrict__ mid,
                                     typename M::type* __restrict__ scratch,
                                     uint32_t* __restrict__ keys, BagT* __restrict__ bags,
                                     int lane) {
  using V = typename M::type;
  const uint32_t kbase = s.rowbase + (static_cast<uint32_t>(bk) << s.lo);
  const int db = s.db;
  const int passes = (s.lo + db - 1) / db;
  const unsigned lt = lanemask_lt(), me = 1u << lane;
  const uint32_t spare = h + 4u * hw;
  const V* src = mid;
  V v[kR4];
  for (int pass = 0; pass < passes; ++pass) {
    const DigitPass dp(s.lo, pass, db);
    const bool last = pass + 1 == passes;
    V* dst = (pass & 1) ? mid : scratch;
    for (int k = lane; k < dp.words(); k += 32) sts(h + 4u * k, 0u);
    __syncwarp();
    int p = beg + lane;
    for (; p + 96 < end; p += 128) {
      const V v0 = src[p], v1 = src[p + 32], v2 = src[p + 64], v3 = src[p + 96];
      atoms_inc(dp.at(h, dp.digit(M::lo(v0))));
      atoms_inc(dp.at(h, dp.digit(M::lo(v1))));
      atoms_inc(dp.at(h, dp.digit(M::lo(v2))));
      atoms_inc(dp.at(h, dp.digit(M::lo(v3))));
    }
    for (; p < end; p += 32) atoms_inc(dp.at(h, dp.digit(M::lo(src[p]))));
    __syncwarp();
    warp_hist_scan(dp, h, static_cast<uint32_t>(beg), lane);
    __syncwarp();
    for (int g = beg; g < end; g += 32 * kR4) {
      const int nch = min(kR4, (end - g + 31) >> 5);
#pragma unroll
      for (int r = 0; r < kR4; ++r) {
        const int q = g + 32 * r + lane;
        v[r] = (r < nch && q < end) ? src[q] : V(0);
      }
      auto valid = [&](int r) { return g + 32 * r + lane < end; };
      warp_rank<kR4>(
          nch, lt, me, mofs, [&](int r) { return valid(r) ? dp.at(h, dp.digit(M::lo(v[r]))) : spare; },
          [&](int r, uint32_t slot) {
            if (!valid(r)) return;
            if (last) {
              keys[slot] = kbase + M::lo(v[r]);
              bags[slot] = static_cast<BagT>(M::bag(v[r]));
            } else {
              dst[slot] = v[r];
            }
          });
    }
    __syncwarp();
    src = dst;
  }
}

// Warp per bucket, all buckets of the launch; the ones above kSmallCap are
// left to sort_big_kernel.
template <class BagT, class M>
__global__ void __launch_bounds__(kThreads, 4)
    sort_bucket_kernel(const SortTable* __restrict__ tabs, const int2* __restrict__ bkts,
                       int n_bk, const int* __restrict__ bstart,
                       typename M::type* __restrict__ mid, uint32_t* __restrict__ keys,
                       BagT* __restrict__ bags, int hw) {
  pdl_wait();  // launched as a programmatic dependent (launch_sort_t)
  using V = typename M::type;
  extern __shared__ __align__(16) uint32_t smem_u[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kWarps + warp;
  if (i >= n_bk) return;
  const int2 b = bkts[i];
  const SortTable s = tabs[b.x];
  const int beg = bstart[s.bkbase + b.y], end = bstart[s.bkbase + b.y + 1];
  const int n = end - beg;
  if (n == 0 || n > kSmallCap) return;
  const uint32_t kbase = s.rowbase + (static_cast<uint32_t>(b.y) << s.lo);
  const int nch = (n + 31) >> 5;
  V v[kR4];
#pragma unroll
  for (int r = 0; r < kR4; ++r) {
    if (r >= nch) break;
    const int j = 32 * r + lane;
    v[r] = j < n ? mid[beg + j] : V(0);
  }
  if (s.lo == 0) {  // one row per bucket: already in position order
#pragma unroll
    for (int r = 0; r < kR4; ++r) {
      if (r >= nch) break;
      const int j = 32 * r + lane;
      if (j < n) {
        keys[beg + j] = kbase;
        bags[beg + j] = static_cast<BagT>(M::bag(v[r]));
      }
    }
    return;
  }
  uint32_t* w = smem_u + warp * (2 * (hw + 1) + kSmallCap * (sizeof(V) / 4));
  const uint32_t h = smem_addr(w), spare = h + 4u * hw;
  const uint32_t mofs = 4u * (hw + 1);  // cursor -> its peer mask
  const uint32_t stage = smem_addr(w + 2 * (hw + 1));
  for (int k = lane; k <= hw; k += 32) sts(h + mofs + 4u * k, 0u);
  // digits of <= kSmallDigitBits (see its definition)
  const int passes_s = (s.lo + kSmallDigitBits - 1) / kSmallDigitBits;
  const int db = passes_s ? (s.lo + passes_s - 1) / passes_s : 1;
  const int passes = (s.lo + db - 1) / db;
  const unsigned lt = lanemask_lt(), me = 1u << lane;
  auto valid = [&](int r) { return 32 * r + lane < n; };
  for (int pass = 0; pass < passes; ++pass) {
    const DigitPass dp(s.lo, pass, db);
    for (int k = lane; k < dp.words(); k += 32) sts(h + 4u * k, 0u);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kR4; ++r) {
      if (r >= nch) break;
      if (valid(r)) atoms_inc(dp.at(h, dp.digit(M::lo(v[r]))));
    }
    __syncwarp();
    warp_hist_scan(dp, h, 0u, lane);
    __syncwarp();
    warp_rank<kR4>(
        nch, lt, me, mofs, [&](int r) { return valid(r) ? dp.at(h, dp.digit(M::lo(v[r]))) : spare; },
        [&](int r, uint32_t slot) {
          if (!valid(r)) return;
          if constexpr (sizeof(V) == 4) {
            sts(stage + 4u * slot, static_cast<uint32_t>(v[r]));
          } else {
            sts(stage + 8u * slot, static_cast<uint32_t>(v[r]));
            sts(stage + 8u * slot + 4u, static_cast<uint32_t>(v[r] >> 32));
          }
        });
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kR4; ++r) {  // the pass's order, back into registers
      if (r >= nch) break;
      const int j = 32 * r + lane;
      if constexpr (sizeof(V) == 4)
        v[r] = j < n ? static_cast<V>(lds(stage + 4u * j)) : V(0);
      else
        v[r] = j < n ? (static_cast<V>(lds(stage + 8u * j + 4u)) << 32) | lds(stage + 8u * j)
                     : V(0);
    }
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < kR4; ++r) {
    if (r >= nch) break;
    const int j = 32 * r + lane;
    if (j < n) {
      keys[beg + j] = kbase + M::lo(v[r]);
      bags[beg + j] = static_cast<BagT>(M::bag(v[r]));
    }
  }
}

// Persistent blocks over the buckets above kSmallCap that P2 listed.
template <class BagT, class M>
__global__ void __launch_bounds__(kThreads)
    sort_big_kernel(const SortTable* __restrict__ tabs, const int2* __restrict__ big,
                    const int* __restrict__ n_big, const int* __restrict__ bstart,
                    typename M::type* __restrict__ mid, typename M::type* __restrict__ scratch,
                    uint32_t* __restrict__ keys, BagT* __restrict__ bags, int hw) {
  pdl_wait();  // launched as a programmatic dependent (launch_sort_t)
  using V = typename M::type;
  using BlockScan = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  extern __shared__ __align__(16) uint32_t smem_u[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t hbase = smem_addr(smem_u);
  const uint32_t hstride = 4u * (hw + 1);
  const uint32_t h = hbase + hstride * warp;
  const uint32_t spare = h + 4u * hw;
  const uint32_t mofs = hstride * kWarps;  // cursor -> its peer mask
  const uint32_t stage0 = hbase + 2u * hstride * kWarps;
  const unsigned lt = lanemask_lt(), me = 1u << lane;
  for (int k = lane; k <= hw; k += 32) sts(h + mofs + 4u * k, 0u);
  const int nbig = *n_big;
  // the next bucket's descriptor chain (list -> table -> bucket bounds) is
  // fetched while the current one is sorted
  int2 bn = blockIdx.x < nbig ? big[blockIdx.x] : make_int2(0, 0);
  SortTable sn = tabs[bn.x];
  int begn = bstart[sn.bkbase + bn.y], endn = bstart[sn.bkbase + bn.y + 1];
  for (int i = blockIdx.x; i < nbig; i += gridDim.x) {
    const int2 b = bn;
    const SortTable s = sn;
    const int beg = begn, end = endn;
    const int inext = i + gridDim.x;
    if (inext < nbig) bn = big[inext];
    const int n = end - beg;
    if (n > kBigCap || sizeof(V) != 4 || s.lo == 0) {
      if (warp == 0) {
        if (s.lo == 0) {
          const uint32_t kb = s.rowbase + (static_cast<uint32_t>(b.y) << s.lo);
          for (int p = beg + lane; p < end; p += 32) {
            keys[p] = kb;
            bags[p] = static_cast<BagT>(M::bag(mid[p]));
          }
        } else {
          sort_bucket_unstaged<BagT, M>(s, b.y, beg, end, h, mofs, hw, mid, scratch, keys,
                                        bags, lane);
        }
      }
      if (inext < nbig) {
        sn = tabs[bn.x];
        begn = bstart[sn.bkbase + bn.y];
        endn = bstart[sn.bkbase + bn.y + 1];
      }
      __syncthreads();
      continue;
    }
    const uint32_t kbase = s.rowbase + (static_cast<uint32_t>(b.y) << s.lo);
    const int db = s.db;
    const int passes = (s.lo + db - 1) / db;
    const int i0 = n * warp / kWarps, i1 = n * (warp + 1) / kWarps;
    const int nch = (i1 - i0 + 31) >> 5;
    // the warp's sub-range (<= kBigCap / 8 items) lives in its registers
    uint32_t v[kRB];
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      if (r >= nch) break;
      const int j = i0 + 32 * r + lane;
      v[r] = j < i1 ? static_cast<uint32_t>(mid[beg + j]) : 0u;
    }
    auto valid = [&](int r) { return i0 + 32 * r + lane < i1; };
    for (int pass = 0; pass < passes; ++pass) {
      const DigitPass dp(s.lo, pass, db);
      for (int k = lane; k < dp.words(); k += 32) sts(h + 4u * k, 0u);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < kRB; ++r) {
        if (r >= nch) break;
        if (valid(r)) atoms_inc(dp.at(h, dp.digit(M::lo(static_cast<V>(v[r])))));
      }
      __syncthreads();
      if (pass == 0 && inext < nbig) sn = tabs[bn.x];
      {  // digit-major, warp-minor exclusive scan; thread t owns digits 4t .. 4t + 3
        uint32_t tot[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t d = 4u * threadIdx.x + q;
          tot[q] = 0;
          if (d < static_cast<uint32_t>(dp.nbin))
#pragma unroll
            for (int w = 0; w < kWarps; ++w) tot[q] += lds(dp.at(hbase + hstride * w, d));
        }
        uint32_t ex, agg;
        BlockScan(scan_tmp).ExclusiveSum(tot[0] + tot[1] + tot[2] + tot[3], ex, agg);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t d = 4u * threadIdx.x + q;
          if (d < static_cast<uint32_t>(dp.nbin)) {
            uint32_t r = ex;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
              const uint32_t a = dp.at(hbase + hstride * w, d);
              const uint32_t x = lds(a);
              sts(a, r);
              r += x;
            }
          }
          ex += tot[q];
        }
      }
      __syncthreads();
      if (pass == 0 && inext < nbig) {
        begn = bstart[sn.bkbase + bn.y];
        endn = bstart[sn.bkbase + bn.y + 1];
      }
      warp_rank<kRB>(
          nch, lt, me, mofs,
          [&](int r) { return valid(r) ? dp.at(h, dp.digit(M::lo(static_cast<V>(v[r])))) : spare; },
          [&](int r, uint32_t slot) {
            if (valid(r)) sts(stage0 + 4u * slot, v[r]);
          });
      __syncthreads();
      if (pass + 1 < passes) {  // the pass's order, back into registers
#pragma unroll
        for (int r = 0; r < kRB; ++r) {
          if (r >= nch) break;
          const int j = i0 + 32 * r + lane;
          v[r] = j < i1 ? lds(stage0 + 4u * j) : 0u;
        }
        __syncthreads();
      }
    }
    for (int j = threadIdx.x; j < n; j += kThreads) {
      const V x = static_cast<V>(lds(stage0 + 4u * j));
      keys[beg + j] = kbase + M::lo(x);
      bags[beg + j] = static_cast<BagT>(M::bag(x));
    }
    __syncthreads();
  }
}

template <class K>
void set_smem(K kernel, size_t bytes) {
  SP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(bytes)));
}

template <class BagT>
size_t scatter_smem(int nb_max) {
  return static_cast<size_t>(kCap3) * sizeof(BagT) +
         (2 * static_cast<size_t>(kWarps) * (nb_max + 1) + nb_max) * 4;
}

template <class V>
size_t small_smem(int hw) {
  return static_cast<size_t>(kWarps) * (2 * (hw + 1) + kSmallCap * sizeof(V) / 4) * 4;
}
size_t big_smem(int hw) { return (2 * static_cast<size_t>(kWarps) * (hw + 1) + kBigCap) * 4; }
int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

template <class BagT, class M>
void launch_sort_t(const SortPlan& pl, const SortTable* d_tabs, const int2* d_tiles,
                   const int2* d_bkts, int t0, int t1, int batch, const int32_t* d_off,
                   const int32_t* d_idx, int* d_cnt, int* d_bstart, int2* d_big, int* d_nbig,
                   void* d_mid, int64_t mid_cap, uint32_t* d_keys, void* d_bags,
                   cudaStream_t st) {
  using V = typename M::type;
  static bool attrs[64] = {};  // the attribute is per device
  int dev = 0;
  SP_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attrs[dev]) {
    set_smem(sort_scatter_kernel<BagT, M>, scatter_smem<BagT>(kMaxBuckets));
    set_smem(sort_bucket_kernel<BagT, M>, small_smem<V>(hist_words(kMaxDigitBits)));
    set_smem(sort_big_kernel<BagT, M>, big_smem(hist_words(kMaxDigitBits)));
    attrs[dev] = true;
  }
  const int64_t w0 = pl.wt_start[t0], w1 = pl.wt_start[t1];
  const int64_t k0 = pl.bk_start[t0], k1 = pl.bk_start[t1];
  int nb_max = 1, db_max = 1, lo_max = 1;
  for (int t = t0; t < t1; ++t) {
    nb_max = std::max(nb_max, pl.tabs[t].nb);
    db_max = std::max(db_max, pl.tabs[t].db);
    lo_max = std::max(lo_max, pl.tabs[t].lo);
  }
  const int hw = hist_words(db_max);
  const unsigned n_tiles = static_cast<unsigned>(w1 - w0);
  const int n_bk = static_cast<int>(k1 - k0);
  // P2..P4 are launched as programmatic dependents of their predecessor
  // (each waits for it on entry), so a pass's blocks are scheduled during
  // the previous pass's tail; the n_big reset goes first so P1 -> P2 is a
  // kernel-to-kernel edge
  SP_CUDA(cudaMemsetAsync(d_nbig, 0, sizeof(int), st));
  if (n_tiles > 0) {
    sort_count_kernel<<<n_tiles, kThreads, 0, st>>>(d_tabs, d_tiles + w0, batch, d_off, d_idx,
                                                    d_cnt);
    SP_LAUNCHED();
  }
  launch_pdl(sort_scan_kernel, dim3(t1 - t0), dim3(kScanThreads), 0, st, d_tabs, t0, batch,
             d_off, d_cnt, d_bstart, d_big, d_nbig);
  V* mid = static_cast<V*>(d_mid);
  if (n_tiles > 0)
    launch_pdl(sort_scatter_kernel<BagT, M>, dim3(n_tiles), dim3(kThreads),
               scatter_smem<BagT>(nb_max), st, d_tabs, d_tiles + w0, batch, d_off, d_idx,
               d_cnt, mid, nb_max);
  if (n_bk > 0) {
    const int hws = hist_words(std::min(lo_max, kSmallDigitBits));
    launch_pdl(sort_bucket_kernel<BagT, M>, dim3((n_bk + kWarps - 1) / kWarps), dim3(kThreads),
               small_smem<V>(hws), st, d_tabs, d_bkts + k0, n_bk, d_bstart, mid, d_keys,
               static_cast<BagT*>(d_bags), hws);
    const int per_sm = std::max(1, static_cast<int>(200 * 1024 / big_smem(hw)));
    const int grid = std::max(1, std::min(n_bk, per_sm * num_sms()));
    launch_pdl(sort_big_kernel<BagT, M>, dim3(grid), dim3(kThreads), big_smem(hw), st, d_tabs,
               d_big, d_nbig, d_bstart, mid, mid + mid_cap, d_keys, static_cast<BagT*>(d_bags),
               hw);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

int sort_bits(int64_t rows) {
  int b = 0;
  while (b < 40 && (int64_t(1) << b) < rows) ++b;
  return b;
}

SortPlan sort_plan(const std::vector<TableMeta>& canon, const std::vector<double>& est_nnz,
                   int batch, int64_t target, bool bags16) {
  SortPlan pl;
  const int T = static_cast<int>(canon.size());
  int64_t cbase = 0;
  int32_t bkbase = 0;
  pl.wide_mid = !bags16;
  for (int t = 0; t < T; ++t) {
    const TableMeta& m = canon[t];
    const double n = std::max(1.0, est_nnz[t]);
    const int bits = sort_bits(m.rows);
    // <= 1024 buckets and <= one per row; enough of them for <= 10 low row
    // bits (one P4 pass) and ~4096 lookups per bucket (a test may force
    // `target` lookups per bucket instead)
    const double per_bucket = target > 0 ? static_cast<double>(target) : kBucketTarget;
    int lb = target > 0 ? 0 : std::max(0, bits - 10);
    while (lb < 10 && std::ldexp(1.0, lb) * per_bucket < n) ++lb;
    lb = std::min({lb, bits, 10});
    SortTable s{};
    s.lo = bits - lb;
    s.nb = static_cast<int32_t>((m.rows + (int64_t(1) << s.lo) - 1) >> s.lo);
    if (s.lo > 16) pl.wide_mid = true;
    // P4 digit width: passes x (lookups per bucket + ~half a bin per bin
    // zeroed and scanned), minimised over 4..10-bit digits
    {
      const double nbk = n / std::max(1, s.nb);
      double best = 1e300;
      s.db = std::max(1, s.lo);
      for (int d = 4; d <= kMaxDigitBits && s.lo > 0; ++d) {
        const int passes = (s.lo + d - 1) / d;
        const int bits = (s.lo + passes - 1) / passes;
        const double c = passes * (nbk + 0.5 * std::ldexp(1.0, bits));
        if (c < best) {
          best = c;
          s.db = bits;
        }
      }
      if (s.lo > 0 && s.lo < 4) s.db = s.lo;
    }
    // tiles: 4096 - 32768 lookups (<= 64 per table above 256 K lookups)
    const double tp = target > 0 ? static_cast<double>(target)
                                 : std::min(32768.0, std::max(4096.0, n / 64.0));
    const double per_bag = n / batch;
    int64_t wb = static_cast<int64_t>(std::llround(tp / std::max(per_bag, 1e-3)));
    wb = std::max<int64_t>(1, std::min<int64_t>(batch, wb));
    s.wb = static_cast<int32_t>(wb);
    s.nwt = static_cast<int32_t>((batch + wb - 1) / wb);
    s.cbase = cbase;
    s.bkbase = bkbase;
    s.rowbase = m.rowbase;
    cbase += static_cast<int64_t>(s.nb) * s.nwt;
    bkbase += s.nb + 1;  // + the table-end slot
    pl.tabs.push_back(s);
    pl.wt_start.push_back(static_cast<int64_t>(pl.wtiles.size()));
    for (int c = 0; c < s.nwt; ++c) pl.wtiles.push_back(make_int2(t, c));
    pl.bk_start.push_back(static_cast<int64_t>(pl.bkts.size()));
    for (int k = 0; k < s.nb; ++k) pl.bkts.push_back(make_int2(t, k));
  }
  pl.wt_start.push_back(static_cast<int64_t>(pl.wtiles.size()));
  pl.bk_start.push_back(static_cast<int64_t>(pl.bkts.size()));
  pl.n_cnt = cbase;
  pl.n_bstart = bkbase;
  return pl;
}

size_t sort_mid_bytes(const SortPlan& pl) { return pl.wide_mid ? 8 : 4; }

void launch_sort(const SortPlan& pl, const SortTable* d_tabs, const int2* d_tiles,
                 const int2* d_bkts, int t0, int t1, int batch, const int32_t* d_off,
                 const int32_t* d_idx, int* d_cnt, int* d_bstart, int2* d_big, int* d_nbig,
                 void* d_mid, int64_t mid_cap, uint32_t* d_keys, void* d_bags, bool bags16,
                 cudaStream_t st) {
  if (t1 <= t0) return;
  if (bags16 && !pl.wide_mid)
    launch_sort_t<uint16_t, Mid32>(pl, d_tabs, d_tiles, d_bkts, t0, t1, batch, d_off, d_idx,
                                   d_cnt, d_bstart, d_big, d_nbig, d_mid, mid_cap, d_keys, d_bags, st);
  else if (bags16)
    launch_sort_t<uint16_t, Mid64>(pl, d_tabs, d_tiles, d_bkts, t0, t1, batch, d_off, d_idx,
                                   d_cnt, d_bstart, d_big, d_nbig, d_mid, mid_cap, d_keys, d_bags, st);
  else
    launch_sort_t<uint32_t, Mid64>(pl, d_tabs, d_tiles, d_bkts, t0, t1, batch, d_off, d_idx,
                                   d_cnt, d_bstart, d_big, d_nbig, d_mid, mid_cap, d_keys, d_bags, st);
}

}  // namespace sp
