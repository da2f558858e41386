// dslb.h — the reference's binary lookup-batch file read straight to the
// device (table.hpp:235-305, "a DSLB loader straight to
// device").
//
// Layout (table.hpp:235-238): "DSLB", u32 version (kBatchVersion = 1,
// table.hpp:240), u32 num_tables, u32 batch_size, u64 offsets_len,
// i64 offsets[], u64 indices_len, i64 indices[], little-endian.
//
// load_lookup_batch (table.hpp:283-305) reads the whole file into host
// vectors. Here the header and offsets (T*B+1 values, needed on the host to
// plan the shard copies) are read with pread; the indices — ~90 % of the
// file — are streamed through pinned host slots into device memory by a few
// parallel reader threads, the page-cache reads overlapping the DMA, and a
// caller can ask for any sub-range (a rank reads only its own tables'
// segments).
// Errors follow load_lookup_batch: bad magic / version / truncation ->
// bad_input with the reference's messages; the batch itself is then
// validated like validate_batch (table.hpp:167-184, malformed_batch).
#pragma once

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "common.h"

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "DSLB is little-endian");

namespace sp {

constexpr uint32_t kDslbVersion = 1;  // table.hpp:240

struct DslbFile {
  int fd = -1;
  std::string path;
  int64_t file_bytes = 0;
  uint32_t num_tables = 0, batch_size = 0;
  uint64_t offsets_len = 0, indices_len = 0;
  int64_t offsets_pos = 0, indices_pos = 0;  // byte positions of the arrays

  DslbFile() = default;
  DslbFile(const DslbFile&) = delete;
  DslbFile& operator=(const DslbFile&) = delete;
  ~DslbFile() {
    if (fd >= 0) ::close(fd);
  }

  // pread of exactly `bytes` at `pos`, or "unexpected end of file"
  // (detail::read_le, table.hpp:256-258).
  void read(int64_t pos, void* dst, size_t bytes) const {
    char* d = static_cast<char*>(dst);
    while (bytes > 0) {
      const ssize_t r = ::pread(fd, d, bytes, static_cast<off_t>(pos));
      if (r <= 0) raise(SP_ERR_BAD_INPUT, "unexpected end of file");
      d += r;
      pos += r;
      bytes -= static_cast<size_t>(r);
    }
  }

  // Header of load_lookup_batch (table.hpp:283-299) plus the array
  // positions; checks the file is long enough for both arrays before any of
  // them is allocated (the reference fails the same way while reading).
  void open(const char* p) {
    path = p ? p : "";
    fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
    if (fd < 0) raise(SP_ERR_BAD_INPUT, "cannot open " + path);
    struct stat st {};
    if (::fstat(fd, &st) != 0) raise(SP_ERR_BAD_INPUT, "cannot open " + path);
    file_bytes = static_cast<int64_t>(st.st_size);
    char magic[4];
    if (file_bytes < 4) raise(SP_ERR_BAD_INPUT, path + ": not a lookup batch file");
    read(0, magic, 4);
    if (std::memcmp(magic, "DSLB", 4) != 0)
      raise(SP_ERR_BAD_INPUT, path + ": not a lookup batch file");
    uint32_t version = 0;
    read(4, &version, 4);
    if (version != kDslbVersion)
      raise(SP_ERR_BAD_INPUT, "unsupported batch version " + std::to_string(version));
    read(8, &num_tables, 4);
    read(12, &batch_size, 4);
    read(16, &offsets_len, 8);
    offsets_pos = 24;
    if (offsets_len > static_cast<uint64_t>(file_bytes - offsets_pos) / 8)
      raise(SP_ERR_BAD_INPUT, "unexpected end of file");
    const int64_t ilen_pos = offsets_pos + static_cast<int64_t>(offsets_len) * 8;
    read(ilen_pos, &indices_len, 8);
    indices_pos = ilen_pos + 8;
    if (indices_len > static_cast<uint64_t>(file_bytes - indices_pos) / 8)
      raise(SP_ERR_BAD_INPUT, "unexpected end of file");
  }

  // The header half of validate_batch (table.hpp:168-175): the counts as the
  // reference's int fields hold them, and the offsets length.
  void validate_shape() const {
    const int T = static_cast<int>(num_tables);
    const int B = static_cast<int>(batch_size);
    if (T < 0 || B <= 0) raise(SP_ERR_MALFORMED_BATCH, "non-positive table or batch count");
    const uint64_t want = static_cast<uint64_t>(T) * static_cast<uint64_t>(B) + 1;
    if (offsets_len != want)
      raise(SP_ERR_MALFORMED_BATCH, "offsets length " + std::to_string(offsets_len) +
                                        ", expected " + std::to_string(want));
  }

  // offsets[first, first + n) -> host memory
  void read_offsets(int64_t* dst, int64_t first, int64_t n) const {
    read(offsets_pos + first * 8, dst, static_cast<size_t>(n) * 8);
  }
};

// Pinned host slots that stream file ranges to device memory on a stream.
// The range is cut into slot-sized pieces handled by up to kReaders host
// threads, each with kSlotsPerReader slots of its own: a reader preads piece
// i into a free slot, queues its H2D and moves on, so the page-cache reads
// of several pieces run in parallel with each other and with the copy
// engine; a slot is refilled only after its previous copy retired.
class DslbStreamer {
 public:
  static constexpr int kReaders = 4;
  static constexpr int kSlotsPerReader = 2;
  static constexpr int kSlots = kReaders * kSlotsPerReader;
  static constexpr size_t kSlotBytes = size_t(8) << 20;

  ~DslbStreamer() { release(); }

  void release() {
    for (auto& e : ev_)
      if (e) {
        cudaEventSynchronize(e);
        cudaEventDestroy(e);
        e = nullptr;
      }
    if (host_) cudaFreeHost(host_);
    host_ = nullptr;
  }

  // indices[first, first + n) of `f` -> dst (device), enqueued on `st`.
  void indices_to_device(const DslbFile& f, int64_t first, int64_t n, int64_t* dst,
                         cudaStream_t st) {
    ensure();
    const int64_t pos0 = f.indices_pos + first * 8;
    const int64_t bytes = n * 8;
    const int64_t pieces = (bytes + static_cast<int64_t>(kSlotBytes) - 1) /
                           static_cast<int64_t>(kSlotBytes);
    const int readers = static_cast<int>(pieces < kReaders ? pieces : kReaders);
    auto work = [&](int r) {
      int j = 0;
      for (int64_t i = r; i < pieces; i += readers, ++j) {
        const int slot = r * kSlotsPerReader + j % kSlotsPerReader;
        const int64_t off = i * static_cast<int64_t>(kSlotBytes);
        const size_t b = static_cast<size_t>(
            bytes - off < static_cast<int64_t>(kSlotBytes) ? bytes - off : kSlotBytes);
        char* h = host_ + static_cast<size_t>(slot) * kSlotBytes;
        if (used_[slot]) SP_CUDA(cudaEventSynchronize(ev_[slot]));
        f.read(pos0 + off, h, b);
        SP_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + off, h, b,
                                cudaMemcpyHostToDevice, st));
        SP_CUDA(cudaEventRecord(ev_[slot], st));
        used_[slot] = true;
      }
    };
    if (readers <= 1) {
      work(0);
      return;
    }
    int dev = 0;
    SP_CUDA(cudaGetDevice(&dev));
    std::exception_ptr err[kReaders] = {};
    std::vector<std::thread> th;
    for (int r = 1; r < readers; ++r)
      th.emplace_back([&, r] {
        try {
          SP_CUDA(cudaSetDevice(dev));
          work(r);
        } catch (...) {
          err[r] = std::current_exception();
        }
      });
    try {
      work(0);
    } catch (...) {
      err[0] = std::current_exception();
    }
    for (auto& t : th) t.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
  }

  // Waits for every copy still reading the slots.
  void drain() {
    for (int k = 0; k < kSlots; ++k)
      if (used_[k]) SP_CUDA(cudaEventSynchronize(ev_[k]));
  }

 private:
  void ensure() {
    if (host_) return;
    SP_CUDA(cudaMallocHost(&host_, kSlots * kSlotBytes));
    for (auto& e : ev_) SP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  char* host_ = nullptr;
  cudaEvent_t ev_[kSlots] = {};
  bool used_[kSlots] = {};
};

}  // namespace sp
