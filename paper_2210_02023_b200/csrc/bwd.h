// bwd.h — K4 v2: bucketed stable counting sort fused with the row-wise SGD
// (see bwd.cu). Used for every device whose tables have <= 2^24 rows; other
// shapes take the CUB radix-sort path of tbe.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "tbe.h"

namespace sp {

constexpr int kScatterBags = 2048;          // bags per scatter tile
constexpr int kTargetBucket = 1024;         // lookups per bucket (average)
constexpr int kMaxBins = 2048;              // rows per bucket (smem histogram)
constexpr int kMaxBucketsPerTable = 8192;   // scatter counters in smem

// Per local table (canonical order).
struct BucketMeta {
  int32_t shift;     // bucket = row >> shift; rows per bucket = 1 << shift
  int32_t nb;        // buckets of the table
  int32_t key_bits;  // bits for bucket ids 0..nb (nb = padding sentinel)
  int32_t tiles;     // scatter tiles (kScatterBags bags each)
  int64_t cbase;     // count slots: cnt[cbase + bucket * tiles + tile]
  int32_t tbase;     // first global scatter tile
  int32_t bbase;     // first global bucket
};

// Bucket layout for the current batch (per-table lookup counts known).
// False when a table is too large for the bucketed path.
bool bucket_plan(const std::vector<TableMeta>& canon, const std::vector<int64_t>& table_nnz,
                 int batch, std::vector<BucketMeta>& out, int64_t& n_cnt, int& n_tiles,
                 int& n_buckets);
size_t bwd_scan_temp_bytes(int64_t n_cnt, cudaStream_t st);

// Partition: hist -> scan -> scatter of (row, bag) pairs into bucket order
// (d_prow/d_pbag hold nnz entries).
void launch_bwd_partition(const BucketMeta* d_bm, int n_tables, int n_tiles, int64_t n_cnt,
                          int batch, const int32_t* d_off, const int32_t* d_idx,
                          int32_t* d_cnt, int32_t* d_cpos, void* d_temp, size_t temp_bytes,
                          int32_t* d_prow, int32_t* d_pbag, cudaStream_t st);
// Per bucket: stable sort by row + SGD over the row runs. d_scratch (nnz)
// holds buckets too large for shared memory. With d_sorted_* non-null the
// sorted (key, bag) pairs are also written (diagnostics); do_sgd = false
// skips the update.
void launch_bwd_buckets(const TableMeta* d_meta, const BucketMeta* d_bm, int n_tables,
                        int n_buckets, const int32_t* d_cpos, int64_t nnz,
                        const int32_t* d_prow, const int32_t* d_pbag, int32_t* d_scratch,
                        const float* d_grad, int64_t ldg, float lr, float* d_w,
                        uint32_t* d_sorted_keys, uint32_t* d_sorted_bags, bool do_sgd,
                        cudaStream_t st);

}  // namespace sp
