/*
 * lookup_oracle.h — CPU ORACLE (test infrastructure only).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * as the timed CPU baseline. The product path (paper_2210_02023_b200) never
 * links or calls it.
 *
 * What it restates:
 *  - the synthetic input generator of SURVEY §8d (bag lengths, hot/cold
 *    indices, weights, gradients), bit-for-bit the same integer hashing the
 *    CUDA generator uses; the hash is the reference's splitmix64 finalizer
 *    `mix64` (rng.hpp:13-19);
 *  - the sum-pooled EmbeddingBag forward over the reference's CSR
 *    LookupBatch (table.hpp:158-165, "all the obtained vectors
 *    are summed"), fp32 rows, fp64 accumulation, empty bag -> 0;
 *  - the backward: stable sort of (local row key, bag) pairs exactly as
 *    std::stable_sort orders them, run-length segments, and the row-wise
 *    SGD W[row] -= lr * sum_occurrences dL/dpooled[bag];
 *  - ingest_lookup_batch (table.hpp:188-232) via sort + run-length instead
 *    of unordered_map (identical result: integer bin sums, one divide).
 *
 * Parity status: lookup fwd/bwd numerics are "parity unpinned" by the
 * reference (it has no lookup code); they are pinned by the
 * hand-worked golden cases in tests/golden/lookup_cases.json and against
 * PyTorch's embedding_bag(mode="sum") + autograd SGD
 * (tests/test_torch_reference_cpu.py). Ingest is pinned against the
 * reference itself (oracle/_ref) and SPEC.md:51-53.
 */
#ifndef LOOKUP_ORACLE_H_
#define LOOKUP_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- generator ---- */
uint64_t or_mix64(uint64_t x);
/* Bag length L(t,b): uniform integer in [0, floor(2*pf)]. */
int64_t or_bag_len(uint64_t seed, int32_t t, int64_t b, double pf);
/* Index j of bag (t,b): hot set of 1024 rows with probability hot_mass. */
int64_t or_bag_index(uint64_t seed, int32_t t, int64_t b, int64_t j,
                     int64_t rows, double hot_mass);
float or_weight(uint64_t seed, int32_t t, int64_t row, int32_t col);
float or_grad(uint64_t seed, int64_t bag, int64_t gcol);
/* hot_mass(t) = sum dist[4..16] (oracle.hpp:119-123). */
double or_hot_mass(const double* dist17);

/* Whole synthetic LookupBatch for T tables: offsets[T*B+1] (int64);
 * if indices == NULL only offsets are produced (to size the buffer). */
void or_synth_batch(int32_t T, int32_t B, const double* pf,
                    const int64_t* rows, const double* hot_mass,
                    uint64_t seed, int64_t* offsets, int64_t* indices,
                    int32_t nthreads);

/* ---- forward ---- */
/* tables in `list` (n_list entries, any order): weights[t] explicit fp32
 * rows [rows_t, dim_t] or NULL to use or_weight(wseed,...). out is row-major
 * with leading dimension ld; table t writes columns out_col[t]..+dim_t of
 * rows [bag_lo, bag_hi) (row index bag - bag_lo). */
void or_tbe_forward(int32_t B, const int32_t* dims, const int64_t* rows,
                    const float* const* weights, uint64_t wseed,
                    const int64_t* offsets, const int64_t* indices,
                    const int32_t* list, int32_t n_list, int64_t bag_lo,
                    int64_t bag_hi, float* out, int64_t ld,
                    const int64_t* out_col, int32_t nthreads);

/* ---- backward ---- */
/* Sorted keys of the local device holding tables `list` (ascending ids):
 * key = row_base[t] + index, row_base = prefix sum of rows in list order;
 * payload = bag. Stable (std::stable_sort). Returns n (= local nnz).
 * keys/bags may be NULL to only count. */
int64_t or_sorted_keys(int32_t B, const int64_t* rows, const int64_t* offsets,
                       const int64_t* indices, const int32_t* list,
                       int32_t n_list, uint32_t* keys, uint32_t* bags);
/* Run-length of sorted keys: unique keys and segment start offsets
 * (seg[n_unique] = n). Returns n_unique. */
int64_t or_segments(const uint32_t* keys, int64_t n, uint32_t* unique,
                    uint32_t* seg);
/* Row-wise SGD on explicit weights (in place):
 * W_t[row] -= lr * sum_{positions of row, stable order} grad[bag, col].
 * grad row-major [B, ld]; table t's gradient columns at grad_col[t]. Sums
 * in fp64, one rounding to fp32 at the end. */
void or_tbe_backward_sgd(int32_t B, const int32_t* dims, const int64_t* rows,
                         float* const* weights, const int64_t* offsets,
                         const int64_t* indices, const int32_t* list,
                         int32_t n_list, const float* grad, int64_t ld,
                         const int64_t* grad_col, float lr, int32_t nthreads);
/* Same update, but only returns the fp64 sum per touched row for table
 * `t` in `sums` [rows_t, dim_t] (zero rows untouched) — used by the CPU
 * baseline timing where tables are synthetic and not materialised. */
void or_tbe_backward_rowsums(int32_t B, int32_t dim, int64_t rows,
                             const int64_t* offsets, const int64_t* indices,
                             int32_t t, const float* grad, int64_t ld,
                             int64_t grad_col, double* sums);

/* ---- ingest (table.hpp:188-232) ---- */
/* pf[T], dist[T*17]; returns 0 or 3 (malformed batch, ErrorKind+1). */
int32_t or_ingest(const int64_t* offsets, int64_t offsets_len,
                  const int64_t* indices, int64_t indices_len, int32_t T,
                  int32_t B, double* pf, double* dist);
int32_t or_access_count_bin(int64_t count);

#ifdef __cplusplus
}
#endif

#endif /* LOOKUP_ORACLE_H_ */
