// ingest.cu — K5: ingest_lookup_batch (table.hpp:188-232) on the GPU.
//
// Per table: pooling_factor = total / B; every distinct index contributes
// its access count c to bin access_count_bin(c) (table.hpp:67-76); bins are
// normalised by total. The reference does this with one unordered_map per
// table; here all tables go through one radix sort of packed
// (table, index - min) keys, a run-head select, and integer atomics per bin.
// Integer bin sums + one fp64 divide make the result bit-identical to the
// reference (its double sums of integer counts are exact).
#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.h"
#include "dslb.h"

namespace sp {
namespace {

__global__ void pack_keys_kernel(const int64_t* __restrict__ idx, int64_t n,
                                 const int64_t* __restrict__ tstart, int T,
                                 int64_t minv, int ib, uint64_t* __restrict__ keys) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = T - 1;  // last t with tstart[t] <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tstart[mid] <= p) lo = mid; else hi = mid - 1;
    }
    keys[p] = (static_cast<uint64_t>(lo) << ib) | static_cast<uint64_t>(idx[p] - minv);
  }
}

__global__ void monotone_kernel(const int64_t* __restrict__ off, int64_t n,
                                int32_t* __restrict__ bad) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k + 1 < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (off[k + 1] < off[k]) atomicOr(bad, 1);
}

struct HeadFlag64 {
  const uint64_t* keys;
  __device__ __forceinline__ bool operator()(const int64_t& k) const {
    return k == 0 || keys[k] != keys[k - 1];
  }
};

__device__ __forceinline__ int access_count_bin(uint64_t c) {
  if (c <= 1) return 0;
  const int b = 64 - __clzll(static_cast<long long>(c - 1));  // ceil(log2 c)
  return b < 16 ? b : 16;
}

__global__ void bin_kernel(const uint64_t* __restrict__ keys, const int64_t* __restrict__ heads,
                           const int32_t* __restrict__ nheads, int64_t n, int ib,
                           unsigned long long* __restrict__ counts) {
  const int64_t nh = *nheads;
  for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < nh;
       u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t beg = heads[u];
    const int64_t end = u + 1 < nh ? heads[u + 1] : n;
    const uint64_t c = static_cast<uint64_t>(end - beg);
    const int t = static_cast<int>(keys[beg] >> ib);
    atomicAdd(counts + t * SP_NUM_BINS + access_count_bin(c), static_cast<unsigned long long>(c));
  }
}

int grid1d(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32)));
}

int bits_for(uint64_t v) {  // bits to represent v (>= 1)
  int b = 1;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

}  // namespace
}  // namespace sp

using namespace sp;

namespace sp {
namespace {

// The ingest on device: fill_idx(d_idx, stream) enqueues the batch's
// indices into the device buffer d_idx (from host memory or a DSLB file).
template <class FillIdx>
void ingest_impl(const int64_t* offsets, int64_t offsets_len, FillIdx&& fill_idx,
                 int64_t indices_len, int32_t num_tables, int32_t batch_size,
                 const int32_t* dims, const int64_t* hash_sizes, int32_t bytes_per_param,
                 int32_t cuda_device, sp_table_spec* out_tables) {
  {
    const int T = num_tables;
    const int64_t B = batch_size;
    // validate_batch (table.hpp:167-184)
    if (T < 0 || B <= 0) raise(SP_ERR_MALFORMED_BATCH, "non-positive table or batch count");
    if (offsets_len != T * B + 1)
      raise(SP_ERR_MALFORMED_BATCH, "offsets length " + std::to_string(offsets_len) +
                                        ", expected " + std::to_string(T * B + 1));
    if (offsets[0] != 0) raise(SP_ERR_MALFORMED_BATCH, "offsets must start at 0");
    if (offsets[offsets_len - 1] != indices_len)
      raise(SP_ERR_MALFORMED_BATCH, "last offset != indices length");
    if (T > 0 && (!dims || !hash_sizes)) raise(SP_ERR_BAD_INPUT, "dims/hash_sizes length != num_tables");
    for (int t = 0; t < T; ++t)
      if (dims[t] < 1 || hash_sizes[t] < 1) raise(SP_ERR_BAD_INPUT, "dim and hash_size must be >= 1");
    SP_CUDA(cudaSetDevice(cuda_device));
    cudaStream_t st = nullptr;
    SP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<void*> tmp;
    auto al = [&](size_t bytes) {
      void* p = nullptr;
      SP_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 8)));
      tmp.push_back(p);
      return p;
    };
    auto cleanup = [&] {
      cudaStreamSynchronize(st);
      for (void* p : tmp) cudaFree(p);
      cudaStreamDestroy(st);
    };
    try {
      const int64_t n = indices_len;
      int64_t* d_off = static_cast<int64_t*>(al(offsets_len * 8));
      int32_t* d_bad = static_cast<int32_t*>(al(4));
      SP_CUDA(cudaMemcpyAsync(d_off, offsets, offsets_len * 8, cudaMemcpyHostToDevice, st));
      SP_CUDA(cudaMemsetAsync(d_bad, 0, 4, st));
      monotone_kernel<<<grid1d(offsets_len), 256, 0, st>>>(d_off, offsets_len, d_bad);
      SP_LAUNCHED();
      std::vector<unsigned long long> counts(static_cast<size_t>(std::max(T, 1)) * SP_NUM_BINS, 0);
      int32_t bad = 0;
      if (n > 0) {
        int64_t* d_idx = static_cast<int64_t*>(al(n * 8));
        fill_idx(d_idx, st);
        // index range (the reference counts any int64 value)
        int64_t* d_mm = static_cast<int64_t*>(al(16));
        size_t tb1 = 0, tb2 = 0;
        SP_CUDA(cub::DeviceReduce::Min(nullptr, tb1, d_idx, d_mm, n, st));
        SP_CUDA(cub::DeviceReduce::Max(nullptr, tb2, d_idx, d_mm + 1, n, st));
        void* d_t = al(std::max(tb1, tb2));
        SP_CUDA(cub::DeviceReduce::Min(d_t, tb1, d_idx, d_mm, n, st));
        SP_CUDA(cub::DeviceReduce::Max(d_t, tb2, d_idx, d_mm + 1, n, st));
        int64_t mm[2];
        SP_CUDA(cudaMemcpyAsync(mm, d_mm, 16, cudaMemcpyDeviceToHost, st));
        SP_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st));
        SP_CUDA(cudaStreamSynchronize(st));
        if (bad) raise(SP_ERR_MALFORMED_BATCH, "offsets decrease");
        const uint64_t span = static_cast<uint64_t>(mm[1]) - static_cast<uint64_t>(mm[0]);
        const int ib = bits_for(span);
        const int tbits = bits_for(static_cast<uint64_t>(std::max(T - 1, 1)));
        if (ib + tbits > 64)
          raise(SP_ERR_BAD_INPUT, "index value range too wide to pack with the table id");
        std::vector<int64_t> tstart(T);
        for (int t = 0; t < T; ++t) tstart[t] = offsets[t * B];
        int64_t* d_ts = static_cast<int64_t*>(al(T * 8));
        SP_CUDA(cudaMemcpyAsync(d_ts, tstart.data(), T * 8, cudaMemcpyHostToDevice, st));
        uint64_t* d_k = static_cast<uint64_t*>(al(n * 8));
        uint64_t* d_ks = static_cast<uint64_t*>(al(n * 8));
        pack_keys_kernel<<<grid1d(n), 256, 0, st>>>(d_idx, n, d_ts, T, mm[0], ib, d_k);
        SP_LAUNCHED();
        size_t ts = 0;
        SP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, ts, d_k, d_ks, n, 0, ib + tbits, st));
        int64_t* d_heads = static_cast<int64_t*>(al(n * 8));
        int32_t* d_nh = static_cast<int32_t*>(al(4));
        cub::CountingInputIterator<int64_t> it(0);
        size_t tsel = 0;
        SP_CUDA(cub::DeviceSelect::If(nullptr, tsel, it, d_heads, d_nh, n, HeadFlag64{d_ks}, st));
        void* d_tmp = al(std::max(ts, tsel));
        SP_CUDA(cub::DeviceRadixSort::SortKeys(d_tmp, ts, d_k, d_ks, n, 0, ib + tbits, st));
        SP_CUDA(cub::DeviceSelect::If(d_tmp, tsel, it, d_heads, d_nh, n, HeadFlag64{d_ks}, st));
        unsigned long long* d_cnt =
            static_cast<unsigned long long*>(al(counts.size() * sizeof(unsigned long long)));
        SP_CUDA(cudaMemsetAsync(d_cnt, 0, counts.size() * sizeof(unsigned long long), st));
        bin_kernel<<<grid1d(n), 256, 0, st>>>(d_ks, d_heads, d_nh, n, ib, d_cnt);
        SP_LAUNCHED();
        SP_CUDA(cudaMemcpyAsync(counts.data(), d_cnt, counts.size() * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, st));
      } else {
        SP_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st));
      }
      SP_CUDA(cudaStreamSynchronize(st));
      if (bad) raise(SP_ERR_MALFORMED_BATCH, "offsets decrease");
      for (int t = 0; t < T; ++t) {
        sp_table_spec& s = out_tables[t];
        std::memset(&s, 0, sizeof(s));
        s.id = t;
        s.dim = dims[t];
        s.hash_size = hash_sizes[t];
        s.table_size_gb = static_cast<double>(hash_sizes[t]) * dims[t] * bytes_per_param /
                          (1024.0 * 1024.0 * 1024.0);
        const int64_t total = offsets[(t + 1) * B] - offsets[t * B];
        s.pooling_factor = static_cast<double>(total) / static_cast<double>(B);
        if (total > 0)
          for (int b = 0; b < SP_NUM_BINS; ++b)
            s.dist[b] = static_cast<double>(counts[t * SP_NUM_BINS + b]) / static_cast<double>(total);
      }
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  }
}

}  // namespace
}  // namespace sp

extern "C" int sp_ingest_lookup_batch(const int64_t* offsets, int64_t offsets_len,
                                      const int64_t* indices, int64_t indices_len,
                                      int32_t num_tables, int32_t batch_size,
                                      const int32_t* dims, const int64_t* hash_sizes,
                                      int32_t bytes_per_param, int32_t cuda_device,
                                      sp_table_spec* out_tables) {
  return guarded([&] {
    ingest_impl(
        offsets, offsets_len,
        [&](int64_t* d_idx, cudaStream_t st) {
          SP_CUDA(cudaMemcpyAsync(d_idx, indices, indices_len * 8, cudaMemcpyHostToDevice, st));
        },
        indices_len, num_tables, batch_size, dims, hash_sizes, bytes_per_param, cuda_device,
        out_tables);
  });
}

// ingest_lookup_batch(load_lookup_batch(path), dims, hash_sizes, bytes)
// (table.hpp:188-232, 283-305) with the indices streamed from the file
// straight into device memory (dslb.h). n_dims must equal the file's
// num_tables (the reference's "dims/hash_sizes length != num_tables").
extern "C" int sp_ingest_batch_file(const char* path, const int32_t* dims,
                                    const int64_t* hash_sizes, int32_t n_dims,
                                    int32_t bytes_per_param, int32_t cuda_device,
                                    sp_table_spec* out_tables, int32_t* num_tables_out,
                                    int32_t* batch_size_out) {
  return guarded([&] {
    DslbFile f;
    f.open(path);
    f.validate_shape();
    const int64_t n_off = static_cast<int64_t>(f.offsets_len);
    std::vector<int64_t> off(static_cast<size_t>(n_off));
    f.read_offsets(off.data(), 0, n_off);
    // the rest of validate_batch (table.hpp:176-183); ingest_impl repeats the
    // O(T) checks and checks monotonicity on the device
    if (off[0] != 0) raise(SP_ERR_MALFORMED_BATCH, "offsets must start at 0");
    for (int64_t k = 1; k < n_off; ++k)
      if (off[k] < off[k - 1])
        raise(SP_ERR_MALFORMED_BATCH, "offsets decrease at position " + std::to_string(k));
    if (static_cast<uint64_t>(off.back()) != f.indices_len)
      raise(SP_ERR_MALFORMED_BATCH, "last offset != indices length");
    if (n_dims != static_cast<int32_t>(f.num_tables))
      raise(SP_ERR_BAD_INPUT, "dims/hash_sizes length != num_tables");
    if (num_tables_out) *num_tables_out = static_cast<int32_t>(f.num_tables);
    if (batch_size_out) *batch_size_out = static_cast<int32_t>(f.batch_size);
    // pinned slots cached per device across calls (allocating them costs
    // more than streaming a cfg3 file); deliberately never freed, so no CUDA
    // call runs during static destruction
    static std::mutex ring_mu;
    static DslbStreamer* rings[64] = {};
    std::lock_guard<std::mutex> lk(ring_mu);
    DslbStreamer*& rp = rings[cuda_device & 63];
    if (!rp) rp = new DslbStreamer();
    DslbStreamer& ring = *rp;
    ingest_impl(
        off.data(), n_off,
        [&](int64_t* d_idx, cudaStream_t st) {
          ring.indices_to_device(f, 0, static_cast<int64_t>(f.indices_len), d_idx, st);
        },
        static_cast<int64_t>(f.indices_len), static_cast<int32_t>(f.num_tables),
        static_cast<int32_t>(f.batch_size), dims, hash_sizes, bytes_per_param, cuda_device,
        out_tables);
    ring.drain();
  });
}
