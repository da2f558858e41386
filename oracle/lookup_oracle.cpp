// lookup_oracle.cpp — CPU ORACLE, test infrastructure only (see
// lookup_oracle.h for the import rule and what is restated from where).
// Built by oracle/Makefile into oracle/_build/liblookup_oracle.so.

#include "lookup_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// Stream tags of the SURVEY §8d generator (shared with csrc/synth.cuh).
constexpr uint64_t kTagLen = 0x6c656e5f62616773ULL;  // "len_bags"
constexpr uint64_t kTagIdx = 0x6964785f726f7773ULL;  // "idx_rows"
constexpr uint64_t kTagW = 0x77656967687473ULL;      // "weights"
constexpr uint64_t kTagG = 0x6772616469656e74ULL;    // "gradient"

// splitmix64 finalizer: the reference's mix64 (rng.hpp:13-19).
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

inline uint64_t h3(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
  return mix64(mix64(mix64(seed ^ tag) ^ a) ^ b);
}

inline uint64_t hot_threshold(double hot_mass) {
  if (!(hot_mass > 0.0)) return 0;
  if (hot_mass >= 1.0) return 1ULL << 32;
  return static_cast<uint64_t>(hot_mass * 4294967296.0);
}

inline int64_t index_from_hash(uint64_t h, int64_t rows, uint64_t thr) {
  const uint64_t lo = h & 0xffffffffULL;
  const uint64_t hi = h >> 32;
  if (lo < thr) {
    const uint64_t j = hi & 1023ULL;
    if (rows <= 1024) return static_cast<int64_t>(j % static_cast<uint64_t>(rows));
    return static_cast<int64_t>(j * static_cast<uint64_t>(rows / 1024));
  }
  return static_cast<int64_t>(hi % static_cast<uint64_t>(rows));
}

int nthreads_or_default(int32_t n) {
#ifdef _OPENMP
  return n > 0 ? n : omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

}  // namespace

extern "C" {

uint64_t or_mix64(uint64_t x) { return mix64(x); }

double or_hot_mass(const double* dist17) {
  double h = 0.0;  // oracle.hpp:119-123: bins whose lower edge is >= 8
  for (int b = 4; b < 17; ++b) h += dist17[b];
  return h;
}

int64_t or_bag_len(uint64_t seed, int32_t t, int64_t b, double pf) {
  const int64_t lmax = static_cast<int64_t>(std::floor(2.0 * pf));
  if (lmax <= 0) return 0;
  const uint64_t h = h3(seed, kTagLen, static_cast<uint64_t>(t),
                        static_cast<uint64_t>(b));
  return static_cast<int64_t>(h % static_cast<uint64_t>(lmax + 1));
}

int64_t or_bag_index(uint64_t seed, int32_t t, int64_t b, int64_t j,
                     int64_t rows, double hot_mass) {
  const uint64_t base = h3(seed, kTagIdx, static_cast<uint64_t>(t),
                           static_cast<uint64_t>(b));
  return index_from_hash(mix64(base ^ static_cast<uint64_t>(j)), rows,
                         hot_threshold(hot_mass));
}

float or_weight(uint64_t seed, int32_t t, int64_t row, int32_t col) {
  const uint64_t base = h3(seed, kTagW, static_cast<uint64_t>(t),
                           static_cast<uint64_t>(row));
  const uint64_t h = mix64(base ^ static_cast<uint64_t>(col));
  // 0.5 + 0.5*u, u = k*2^-23: exact in fp32 on [0.5, 1).
  return 0.5f + static_cast<float>(h >> 41) * 0x1.0p-24f;
}

float or_grad(uint64_t seed, int64_t bag, int64_t gcol) {
  const uint64_t h = h3(seed, kTagG, static_cast<uint64_t>(bag),
                        static_cast<uint64_t>(gcol));
  // k*2^-23 - 1, exact in fp32 on [-1, 1).
  return static_cast<float>(h >> 40) * 0x1.0p-23f - 1.0f;
}

void or_synth_batch(int32_t T, int32_t B, const double* pf,
                    const int64_t* rows, const double* hot_mass,
                    uint64_t seed, int64_t* offsets, int64_t* indices,
                    int32_t nthreads) {
  const int nt = nthreads_or_default(nthreads);
  const int64_t n_bags = static_cast<int64_t>(T) * B;
  offsets[0] = 0;
  // lengths, then an inclusive scan (sequential: exact and cheap).
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t k = 0; k < n_bags; ++k)
    offsets[k + 1] = or_bag_len(seed, static_cast<int32_t>(k / B), k % B,
                                pf[k / B]);
  for (int64_t k = 0; k < n_bags; ++k) offsets[k + 1] += offsets[k];
  if (indices == nullptr) return;
#pragma omp parallel for schedule(dynamic, 4096) num_threads(nt)
  for (int64_t k = 0; k < n_bags; ++k) {
    const int32_t t = static_cast<int32_t>(k / B);
    const int64_t b = k % B;
    const uint64_t base = h3(seed, kTagIdx, static_cast<uint64_t>(t),
                             static_cast<uint64_t>(b));
    const uint64_t thr = hot_threshold(hot_mass[t]);
    for (int64_t p = offsets[k], j = 0; p < offsets[k + 1]; ++p, ++j)
      indices[p] = index_from_hash(mix64(base ^ static_cast<uint64_t>(j)),
                                   rows[t], thr);
  }
}

void or_tbe_forward(int32_t B, const int32_t* dims, const int64_t* rows,
                    const float* const* weights, uint64_t wseed,
                    const int64_t* offsets, const int64_t* indices,
                    const int32_t* list, int32_t n_list, int64_t bag_lo,
                    int64_t bag_hi, float* out, int64_t ld,
                    const int64_t* out_col, int32_t nthreads) {
  (void)rows;
  const int nt = nthreads_or_default(nthreads);
  const int64_t nb = bag_hi - bag_lo;
  const int64_t work = static_cast<int64_t>(n_list) * nb;
#pragma omp parallel num_threads(nt)
  {
    std::vector<double> acc;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t w = 0; w < work; ++w) {
      const int32_t t = list[w / nb];
      const int64_t b = bag_lo + w % nb;
      const int dim = dims[t];
      acc.assign(dim, 0.0);
      const int64_t k = static_cast<int64_t>(t) * B + b;
      for (int64_t p = offsets[k]; p < offsets[k + 1]; ++p) {
        const int64_t r = indices[p];
        if (weights != nullptr && weights[t] != nullptr) {
          const float* row = weights[t] + r * dim;
          for (int c = 0; c < dim; ++c) acc[c] += row[c];
        } else {
          for (int c = 0; c < dim; ++c) acc[c] += or_weight(wseed, t, r, c);
        }
      }
      float* o = out + (b - bag_lo) * ld + out_col[t];
      for (int c = 0; c < dim; ++c) o[c] = static_cast<float>(acc[c]);
    }
  }
}

int64_t or_sorted_keys(int32_t B, const int64_t* rows, const int64_t* offsets,
                       const int64_t* indices, const int32_t* list,
                       int32_t n_list, uint32_t* keys, uint32_t* bags) {
  int64_t n = 0;
  for (int32_t i = 0; i < n_list; ++i) {
    const int64_t t = list[i];
    n += offsets[(t + 1) * B] - offsets[t * B];
  }
  if (keys == nullptr) return n;
  std::vector<std::pair<uint32_t, uint32_t>> kv;
  kv.reserve(n);
  uint64_t base = 0;
  for (int32_t i = 0; i < n_list; ++i) {
    const int64_t t = list[i];
    for (int64_t b = 0; b < B; ++b) {
      const int64_t k = t * B + b;
      for (int64_t p = offsets[k]; p < offsets[k + 1]; ++p)
        kv.emplace_back(static_cast<uint32_t>(base + indices[p]),
                        static_cast<uint32_t>(b));
    }
    base += static_cast<uint64_t>(rows[t]);
  }
  std::stable_sort(kv.begin(), kv.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  for (int64_t i = 0; i < n; ++i) {
    keys[i] = kv[i].first;
    bags[i] = kv[i].second;
  }
  return n;
}

int64_t or_segments(const uint32_t* keys, int64_t n, uint32_t* unique,
                    uint32_t* seg) {
  int64_t u = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (i == 0 || keys[i] != keys[i - 1]) {
      if (unique) unique[u] = keys[i];
      if (seg) seg[u] = static_cast<uint32_t>(i);
      ++u;
    }
  }
  if (seg) seg[u] = static_cast<uint32_t>(n);
  return u;
}

void or_tbe_backward_sgd(int32_t B, const int32_t* dims, const int64_t* rows,
                         float* const* weights, const int64_t* offsets,
                         const int64_t* indices, const int32_t* list,
                         int32_t n_list, const float* grad, int64_t ld,
                         const int64_t* grad_col, float lr, int32_t nthreads) {
  // Keys of different tables never interleave (key = row base + row), so
  // the device-wide stable sort is the concatenation of per-table stable
  // sorts: tables are processed independently (in parallel).
  const int nt = nthreads_or_default(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
  for (int32_t i = 0; i < n_list; ++i) {
    const int32_t one[1] = {list[i]};
    const int32_t t = list[i];
    const int64_t n = or_sorted_keys(B, rows, offsets, indices, one, 1, nullptr, nullptr);
    std::vector<uint32_t> keys(n), bags(n), uniq(n + 1), seg(n + 1);
    or_sorted_keys(B, rows, offsets, indices, one, 1, keys.data(), bags.data());
    const int64_t nu = or_segments(keys.data(), n, uniq.data(), seg.data());
    const int dim = dims[t];
    std::vector<double> s;
    for (int64_t u = 0; u < nu; ++u) {
      const int64_t row = static_cast<int64_t>(uniq[u]);
      s.assign(dim, 0.0);
      for (uint32_t k = seg[u]; k < seg[u + 1]; ++k) {
        const float* g = grad + static_cast<int64_t>(bags[k]) * ld + grad_col[t];
        for (int c = 0; c < dim; ++c) s[c] += g[c];
      }
      float* w = weights[t] + row * dim;
      for (int c = 0; c < dim; ++c)
        w[c] = static_cast<float>(static_cast<double>(w[c]) -
                                  static_cast<double>(lr) * s[c]);
    }
  }
}

void or_tbe_backward_rowsums(int32_t B, int32_t dim, int64_t rows,
                             const int64_t* offsets, const int64_t* indices,
                             int32_t t, const float* grad, int64_t ld,
                             int64_t grad_col, double* sums) {
  // Keys of a single table are its row ids; reuse the generic path with a
  // rows array indexed by t.
  const int32_t list[1] = {t};
  std::vector<int64_t> rows_vec(static_cast<size_t>(t) + 1, 0);
  rows_vec[t] = rows;
  const int64_t n = or_sorted_keys(B, rows_vec.data(), offsets, indices, list,
                                   1, nullptr, nullptr);
  std::vector<uint32_t> keys(n), bags(n), uniq(n + 1), seg(n + 1);
  or_sorted_keys(B, rows_vec.data(), offsets, indices, list, 1, keys.data(),
                 bags.data());
  const int64_t nu = or_segments(keys.data(), n, uniq.data(), seg.data());
  for (int64_t u = 0; u < nu; ++u) {
    double* s = sums + static_cast<int64_t>(uniq[u]) * dim;
    for (uint32_t k = seg[u]; k < seg[u + 1]; ++k) {
      const float* g = grad + static_cast<int64_t>(bags[k]) * ld + grad_col;
      for (int c = 0; c < dim; ++c) s[c] += g[c];
    }
  }
}

int32_t or_access_count_bin(int64_t count) {
  // table.hpp:67-76: 0 for count <= 1, else ceil(log2 count) capped at 16.
  if (count <= 1) return 0;
  int32_t bin = 0;
  int64_t upper = 1;
  while (upper < count && bin < 16) {
    upper *= 2;
    ++bin;
  }
  return bin;
}

int32_t or_ingest(const int64_t* offsets, int64_t offsets_len,
                  const int64_t* indices, int64_t indices_len, int32_t T,
                  int32_t B, double* pf, double* dist) {
  // validate_batch (table.hpp:167-184)
  if (T < 0 || B <= 0) return 3;
  if (offsets_len != static_cast<int64_t>(T) * B + 1) return 3;
  if (offsets[0] != 0) return 3;
  for (int64_t k = 1; k < offsets_len; ++k)
    if (offsets[k] < offsets[k - 1]) return 3;
  if (offsets[offsets_len - 1] != indices_len) return 3;
  std::vector<int64_t> v;
  for (int32_t t = 0; t < T; ++t) {
    const int64_t lo = offsets[static_cast<int64_t>(t) * B];
    const int64_t hi = offsets[static_cast<int64_t>(t + 1) * B];
    const int64_t total = hi - lo;
    pf[t] = static_cast<double>(total) / B;
    double* d = dist + static_cast<int64_t>(t) * 17;
    for (int b = 0; b < 17; ++b) d[b] = 0.0;
    if (total == 0) continue;
    v.assign(indices + lo, indices + hi);
    std::sort(v.begin(), v.end());
    int64_t sums[17] = {0};
    for (int64_t i = 0; i < total;) {
      int64_t j = i;
      while (j < total && v[j] == v[i]) ++j;
      sums[or_access_count_bin(j - i)] += j - i;
      i = j;
    }
    for (int b = 0; b < 17; ++b)
      d[b] = static_cast<double>(sums[b]) / static_cast<double>(total);
  }
  return 0;
}

}  // extern "C"
