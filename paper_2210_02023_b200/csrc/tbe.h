// tbe.h — device-side layout of one (virtual) device's embedding shard and
// the launchers of the hot kernels (K1 forward, K4 backward).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace sp {

// One local table of a (virtual) device, in kernel order.
struct TableMeta {
  int64_t woff;         // element offset of row 0 in the weight slab
  int64_t rows;         // hash_size
  int64_t reserved;
  int32_t dim;
  int32_t lcol;         // first column in the local pooled [B, W_local]
  uint32_t rowbase;     // K4 key base: rows of the earlier local tables (device-wide)
  int32_t cls;          // dim class, see dim_class(); -1 = generic path
  int32_t local;        // canonical local index (ascending global id)
  int32_t gid;          // global table id
};

// Storage type of the embedding rows: fp32 (4 B/param) or fp16 (2 B/param,
// the paper's tables, and table_memory_gb's default,
// table.hpp:30). Pooled outputs, gradients and all sums stay fp32.
enum class WeightType : int32_t { kF32 = 0, kF16 = 1, kBF16 = 2 };
inline int elem_bytes(WeightType t) { return t == WeightType::kF32 ? 4 : 2; }

// Row class by row bytes: 0..5 for 16, 32, ..., 512-byte rows (whole 16-byte
// slices: fp32 dims 4..128, fp16 dims 8..256), -1 = the generic path.
inline int row_class(int dim, WeightType t) {
  switch (dim * elem_bytes(t)) {
    case 16: return 0;
    case 32: return 1;
    case 64: return 2;
    case 128: return 3;
    case 256: return 4;
    case 512: return 5;
    default: return -1;
  }
}
inline int dim_class(int dim) { return row_class(dim, WeightType::kF32); }

// Bags (K1) or unique rows (K4) per warp for each dim class: the warp is
// split into P spans of 32/P lanes; a span sums one bag / one row's
// gradients with (32/P)/(dim/4) row groups.
inline int rows_per_warp(int cls) {
  switch (cls) {
    case 0: return 8;
    case 1: return 8;
    case 2: return 4;
    case 3: return 2;
    case 4: return 2;
    case 5: return 1;
    default: return 1;
  }
}

constexpr int kWarpsPerBlock = 8;
constexpr int kBlockThreads = 32 * kWarpsPerBlock;

// ---- K1: fused multi-table sum-pooled forward ----------------------------
// One launch over all local tables; a block per tile of <= 256 bags of one
// table: out[b, lcol_t : lcol_t + dim_t] =
//   sum_{p in [off[i*B+b], off[i*B+b+1])} W_t[idx[p], :]   (int32 CSR).
// Tiles (x = canonical table, y = first bag, z = bag count) in launch order.
//
// Where the pooled rows go: d_peer == nullptr -> the local pooled buffer
// d_out [B, ldo]; otherwise (peer memory, D ranks over CUDA IPC / NVLink, a
// device-resident map) batch rows [j*rows_per_part, (j+1)*rows_per_part) go
// to base[j], rank j's receive slot for this rank: K1 itself performs the
// forward all-to-all (stores to mapped peer addresses, fenced system-wide).
constexpr int kMaxPeers = 8;
struct RowMap {
  float* base[kMaxPeers];
  int64_t rows_per_part;
  int32_t parts;
  int32_t pad;
};
std::vector<int4> make_fwd_tiles(const std::vector<TableMeta>& canon,
                                 const std::vector<int>& order, int batch);
void launch_tbe_forward(const TableMeta* d_meta_canon, const int4* d_tiles,
                        int64_t n_tiles, int batch, const int32_t* d_off,
                        const int32_t* d_idx, const void* d_w, WeightType wt, float* d_out,
                        const RowMap* d_peer, int64_t ldo, cudaStream_t st);

// ---- K4a: stable sort of a device's lookups by (table, row) (sort.cu) ----
// Per local table: rows split into nb buckets of 2^lo rows, bags into nwt
// tiles of wb bags; cnt[cbase + tile*nb + bucket] is the count matrix,
// bstart[bkbase + bucket] the bucket starts (+ one table-end slot).
struct SortTable {
  int32_t lo;        // row bits inside a bucket
  int32_t nb;        // buckets: ceil(rows / 2^lo) (<= 1024)
  int32_t wb;        // bags per tile
  int32_t nwt;       // tiles: ceil(B / wb)
  int64_t cbase;     // first count of the table
  int32_t bkbase;    // first bucket-start slot of the table
  uint32_t rowbase;  // key base of the table (device-wide)
  int32_t db;        // digit bits per pass of the in-bucket sort (<= 10)
  int32_t pad;
};
struct SortPlan {
  std::vector<SortTable> tabs;
  std::vector<int2> wtiles;            // (table, tile), tables in order
  std::vector<int2> bkts;              // (table, bucket), tables in order
  std::vector<int64_t> wt_start, bk_start;  // per table (+ end)
  int64_t n_cnt = 0;
  int32_t n_bstart = 0;
  bool wide_mid = false;  // 8-byte packed intermediates (32-bit bags or > 16 low row bits)
};
// est_nnz: expected lookups per table; target > 0 forces the bucket and
// tile size in lookups (tests), 0 = the default plan.
SortPlan sort_plan(const std::vector<TableMeta>& canon, const std::vector<double>& est_nnz,
                   int batch, int64_t target, bool bags16);
// Bytes of one packed intermediate (d_mid holds 2 * mid_cap of them: the
// pairs, then the scratch of buckets too large for shared memory).
size_t sort_mid_bytes(const SortPlan& pl);
// Sorts the lookups of local tables [t0, t1) into keys/bags at their CSR
// positions (keys = rowbase + row, ties in position order: std::stable_sort).
// d_big / d_nbig: scratch list of the large buckets (bkts.size() entries).
void launch_sort(const SortPlan& pl, const SortTable* d_tabs, const int2* d_tiles,
                 const int2* d_bkts, int t0, int t1, int batch, const int32_t* d_off,
                 const int32_t* d_idx, int* d_cnt, int* d_bstart, int2* d_big, int* d_nbig,
                 void* d_mid, int64_t mid_cap, uint32_t* d_keys, void* d_bags, bool bags16,
                 cudaStream_t st);

// ---- K4b: row-wise SGD over the sorted pairs -------------------------------
// Row-wise SGD over the sorted pairs:
// W[row] -= lr * sum_{k in run, sorted order} grad[bags[k], lcol..].
// Keys are device-wide (rowbase + row); the sorted lookups of local table t occupy its CSR position range, so the
// launch runs over per-table tiles (make_sgd_tiles: kSgdTileInts ints each,
// from the per-table lookup counts in canonical order).
constexpr int kSgdTileInts = 8;
// Tiles of generic-dim tables (run-based SGD), then of all others
// (segmented SGD with cross-tile carries); counts[2] receives the two sizes.
std::vector<int> make_sgd_tiles(const std::vector<int64_t>& table_nnz,
                                const std::vector<TableMeta>& canon, int64_t counts[2]);
// Carry floats the segmented SGD needs for n_wide_tiles tiles (ints: 4 per tile).
size_t sgd_carry_floats(int64_t n_wide_tiles);
// d_abort (may be null): when *d_abort != 0 the launch leaves W untouched.
void launch_sgd(const TableMeta* d_meta_canon, const int* d_tiles, const int64_t counts[2],
                const uint32_t* d_keys, const void* d_bags, bool bags16, const float* d_grad,
                int64_t ldg, float lr, void* d_w, WeightType wt, float* d_carry_f,
                int32_t* d_carry_i, const int32_t* d_abort, cudaStream_t st);

// ---- generator / layout helpers ------------------------------------------
void launch_init_weights(void* d_w, WeightType wt, int64_t rows, int dim, int32_t gid,
                         uint64_t seed, cudaStream_t st);
// fp32 rows -> table storage type and back (device to device).
void launch_f32_to_weights(const float* d_src, void* d_dst, WeightType wt, int64_t n,
                           cudaStream_t st);
void launch_weights_to_f32(const void* d_src, WeightType wt, float* d_dst, int64_t n,
                           cudaStream_t st);
// lengths of the bags of local tables (gid, lmax per table) into d_len[i*B+b]
void launch_synth_lengths(const int32_t* d_gid, const int64_t* d_lmax,
                          int n_tables, int batch, uint64_t seed,
                          int32_t* d_len, cudaStream_t st);
size_t exclusive_scan_i32(void* temp, size_t temp_bytes, const int32_t* in,
                          int32_t* out, int64_t n, cudaStream_t st);
void launch_synth_indices(const int32_t* d_gid, const int64_t* d_rows,
                          const uint64_t* d_thr, int n_tables, int batch,
                          uint64_t seed, const int32_t* d_off, int32_t* d_idx,
                          cudaStream_t st);
// int64 LookupBatch segment -> int32 local CSR with validation flags.
// off64: B+1 offsets of one table (absolute); idx64: its indices.
void launch_narrow_table(const int64_t* d_off64, const int64_t* d_idx64,
                         int batch, int64_t nnz, int64_t rows, int32_t base,
                         int32_t* d_off, int32_t* d_idx, int32_t* d_flag,
                         cudaStream_t st);
// grad_in grouped layout: [src][rows_per_dst][W_src] per destination slice.
void launch_synth_grad(float* d_grad, int64_t n_rows, int64_t bag0,
                       const int32_t* d_colmap, int64_t width, uint64_t seed,
                       cudaStream_t st);

}  // namespace sp
