// ctx.cu — sp_ctx: one rank's shard of a table->device placement and the
// measured four-stage iteration that replaces the reference's synthetic
// CostOracle::evaluate_placement (oracle.hpp:187-240).
//
// HBM layout per GPU (all fp32 / int32, 16-byte aligned):
//   weight slab   every local table's rows back to back, [rows_t, dim_t]
//   CSR           per (virtual) device: offsets[T_v*B+1], indices[nnz_v]
//   pooled_v      [B, W_v] batch-major, so the rows bound for peer j are the
//                 contiguous slice [j*B/D, (j+1)*B/D) (no packing, §8e)
//   recv / gin    per destination rank: [src i][B/D][W_i] grouped by source
//   grad_v        [B, W_v], the bwd exchange lands each peer's slice in place
//   sort scratch  keys/bags double buffers, run heads, CUB temp (shared by
//                 the virtual devices, stream-ordered)
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "common.h"
#include "nccl_loader.h"
#include "synth.cuh"
#include "dslb.h"
#include "tbe.h"

namespace sp {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

template <class T>
T* dalloc(size_t n, std::vector<void*>& owned, uint64_t& bytes) {
  if (n == 0) n = 1;
  void* p = nullptr;
  SP_CUDA(cudaMalloc(&p, n * sizeof(T)));
  owned.push_back(p);
  bytes += n * sizeof(T);
  return static_cast<T*>(p);
}

struct VDev {
  int vid = 0;
  std::vector<int> tables;  // global ids, ascending
  std::vector<TableMeta> meta_canon;
  std::vector<int32_t> colmap;  // local col -> global col
  int64_t W = 0, rows_total = 0, n_tiles = 0;
  int4* d_tiles = nullptr;      // K1 tiles in launch order (lightest tables last)
  int4* d_tiles_canon = nullptr;  // K1 tiles in table order (pipelined upload path)
  std::vector<int64_t> tile_start;  // first canonical tile of each local table (+ end)
  // K4 SGD tiles of the current batch, one buffer per staging slot (a step's
  // tiles upload while the previous step's SGD may still read its own)
  int* d_sgd_tiles[2] = {};
  int64_t sgd_tile_cap[2] = {};
  int64_t n_sgd_tiles = 0;
  int64_t sgd_counts[2] = {};  // generic-dim (run-based) / segmented SGD tiles
  int cur = 0;  // slot of the current batch
  // K4a sort (sort.cu): the plan and its device copies, the count matrix,
  // the bucket starts and the packed intermediates (nnz entries)
  SortPlan splan;
  SortTable* d_stabs = nullptr;
  int2* d_wtiles = nullptr;
  int2* d_bkts = nullptr;
  int* d_cnt = nullptr;
  int* d_bstart = nullptr;
  int2* d_big = nullptr;   // large-bucket list (+ its count)
  int* d_nbig = nullptr;
  void* d_mid = nullptr;
  int64_t mid_cap = 0;
  TableMeta* d_meta_canon = nullptr;
  int32_t* d_colmap = nullptr;
  int32_t* d_off = nullptr;
  int32_t* d_idx = nullptr;
  int64_t nnz = 0, idx_cap = 0;
  std::vector<int64_t> table_nnz;
  float* d_pooled = nullptr;
  float* d_grad = nullptr;
  double fwd_bytes = 0, bwd_bytes = 0;
  cudaEvent_t ev[8] = {};
};

// Forward exchange of one rank: its pooled [B, W_r] is
// batch-major, so the rows bound for peer j are the contiguous slice
// [j*B/D, (j+1)*B/D); it receives [B/D, W_i] from every source i, grouped by
// source. colmap maps a grouped column to its global column (tables in id
// order). The backward exchange is the mirror (send <-> recv).
struct ExchangePlan {
  std::vector<int64_t> send_off, send_cnt;  // into local pooled / grad [B, W_r]
  std::vector<int64_t> recv_off, recv_cnt;  // into grouped recv / gin [B/D, W_total]
  std::vector<int32_t> colmap;              // W_total entries
};

inline ExchangePlan make_plan(const sp_table_spec* tables, int M, int D,
                              const int32_t* placement, int B, int rank) {
  ExchangePlan p;
  const int64_t R = B / D;
  std::vector<int64_t> W(D, 0), gcol(M, 0);
  int64_t col = 0;
  for (int t = 0; t < M; ++t) {
    gcol[t] = col;
    col += tables[t].dim;
    W[placement[t]] += tables[t].dim;
  }
  int64_t cum = 0;
  for (int j = 0; j < D; ++j) {
    p.send_off.push_back(j * R * W[rank]);
    p.send_cnt.push_back(R * W[rank]);
    p.recv_off.push_back(R * cum);
    p.recv_cnt.push_back(R * W[j]);
    cum += W[j];
  }
  for (int i = 0; i < D; ++i)
    for (int t = 0; t < M; ++t)
      if (placement[t] == i)
        for (int k = 0; k < tables[t].dim; ++k) p.colmap.push_back(static_cast<int32_t>(gcol[t] + k));
  return p;
}

}  // namespace sp

struct sp_ctx {
  int M = 0, D = 1, world = 1, rank = 0, B = 0, device = 0;
  bool bags16 = false;  // B <= 65536: 16-bit bag payload through the sort
  float lr = 0.01f;
  double cap = 0.0;
  std::vector<sp_table_spec> tables;
  std::vector<int> placement;
  std::vector<int64_t> gcol;   // global column of each table
  std::vector<int64_t> dev_W;  // W per device
  std::vector<int64_t> cumW;   // prefix over devices
  int64_t W_total = 0;
  std::vector<sp::VDev> vdevs;
  sp::ExchangePlan plan;       // NCCL mode: this rank's exchange
  std::vector<int64_t> woff;   // per global table: element offset (-1 if not local)
  void* d_w = nullptr;         // weight slab, elements of type wt
  sp::WeightType wt = sp::WeightType::kF32;
  float* d_recv = nullptr;     // rows_per_dst * W_total per destination
  float* d_gin = nullptr;
  int n_dst = 1;               // destinations held here (D in emulation)
  uint32_t *d_kb = nullptr, *d_bb = nullptr;  // sorted keys / bags (shared, stream-ordered)
  int64_t sort_target = 0;     // sort plan bucket/tile size override (tests), 0 = default
  int32_t* d_flag = nullptr;
  int64_t sort_cap = 0;
  int64_t* d_stage64 = nullptr;      // int64 staging of an uploaded LookupBatch
  int64_t* d_stage64_alt = nullptr;  // second slot (sp_run_batches: next step's H2D)
  int64_t* file_off = nullptr;       // pinned offsets of a DSLB file (sp_upload_batch_file)
  int64_t file_off_cap = 0;
  std::unique_ptr<sp::DslbStreamer> file_ring;  // pinned ring: file -> device indices
  int64_t stage_cap = 0;
  cudaEvent_t stage_free[2] = {};    // recorded after the narrows that read a slot
  bool stage_used[2] = {};
  float* d_carry_f = nullptr;        // segmented SGD cross-tile carries
  int32_t* d_carry_i = nullptr;
  int64_t carry_cap = 0;
  int32_t* d_step_flags = nullptr;   // per-step validation flags (sp_run_batches)
  int64_t step_flags_cap = 0;
  // pinned host copies of a batch's layout metadata (SGD tiles), one per
  // staging slot: a pageable H2D would wait for the stream
  uint8_t* meta_host[2] = {};
  size_t meta_cap[2] = {};
  cudaEvent_t slot_done[2] = {};     // after the SGD of the last step that used a slot
  bool slot_done_used[2] = {};
  cudaEvent_t meta_ready = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // H2D of uploaded batches
  // The backward's sort depends only on the batch, not on the gradient: with
  // one (virtual) device it runs on the `side` stream, forked
  // after K1, concurrently with the exchanges (sp_ctx_set_overlap(0) runs it
  // on the main stream; the host-buffer step sorts each uploaded chunk on
  // the side stream while the next chunk is in flight).
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_sort[2] = {nullptr, nullptr};  // timing: the forked sort's span
  bool overlap_sort = true;
  int64_t upload_chunk = int64_t(8) << 20;  // indices per H2D chunk (sp_ctx_set_upload_chunk)
  std::vector<cudaEvent_t> upload_events;
  ncclComm_t comm = nullptr;
  // Peer-memory exchange (sp_ipc_import): every rank's receive and gradient
  // buffers mapped here. K1 stores pooled rows straight into the receivers'
  // slots; the backward pulls this rank's gradient slices from the peers.
  bool peer = false;
  float* peer_recv[sp::kMaxPeers] = {};
  float* peer_gin[sp::kMaxPeers] = {};
  sp::RowMap* d_rowmap = nullptr;  // K1's peer row map (device), null = local
  std::vector<void*> ipc_opened;
  // the backward pull: one stream per peer, so the world-1 peer reads run on
  // concurrent copy engines instead of queueing behind one (ev_pull[0]:
  // fork from the main stream; ev_pull[1 + k]: peer stream k done)
  std::vector<cudaStream_t> pull_streams;
  std::vector<cudaEvent_t> ev_pull;
  double* d_bd = nullptr;      // breakdown gather buffer
  int32_t* d_barrier = nullptr;
  cudaEvent_t ev_a2a[4] = {};
  cudaGraphExec_t graph_exec = nullptr;
  int graph_kernels = 0;
  bool profiling = false;            // per-kernel events (sp_ctx_set_profiling)
  bool comm_model = false;           // emulation: modelled NVLink exchange (sp_ctx_set_comm_model)
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Mark { int cls; size_t a, b; };
  std::vector<Mark> marks;
  std::vector<void*> owned;
  std::vector<void*> sort_owned;
  uint64_t dev_bytes = 0;
  bool has_batch = false;

  ~sp_ctx() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    for (auto& v : vdevs)
      for (auto& e : v.ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ev_a2a)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_pool) cudaEventDestroy(e);
    for (auto& v : vdevs)
      for (void* p : {static_cast<void*>(v.d_idx), v.d_mid, static_cast<void*>(v.d_sgd_tiles[0]),
                       static_cast<void*>(v.d_sgd_tiles[1]), static_cast<void*>(v.d_stabs),
                       static_cast<void*>(v.d_wtiles), static_cast<void*>(v.d_bkts),
                       static_cast<void*>(v.d_cnt), static_cast<void*>(v.d_bstart),
                       static_cast<void*>(v.d_big), static_cast<void*>(v.d_nbig)})
        if (p) cudaFree(p);
    if (d_stage64) cudaFree(d_stage64);
    if (d_stage64_alt) cudaFree(d_stage64_alt);
    file_ring.reset();
    if (file_off) cudaFreeHost(file_off);
    if (d_step_flags) cudaFree(d_step_flags);
    if (d_carry_f) cudaFree(d_carry_f);
    if (d_carry_i) cudaFree(d_carry_i);
    for (auto* p : meta_host)
      if (p) cudaFreeHost(p);
    for (auto& e : stage_free)
      if (e) cudaEventDestroy(e);
    for (auto& e : slot_done)
      if (e) cudaEventDestroy(e);
    if (meta_ready) cudaEventDestroy(meta_ready);
    for (void* p : sort_owned) cudaFree(p);
    for (void* p : owned) cudaFree(p);
    if (comm) sp::nccl().CommDestroy(comm);
    for (cudaStream_t ps : pull_streams) cudaStreamSynchronize(ps);
    for (cudaEvent_t e : ev_pull) cudaEventDestroy(e);
    for (cudaStream_t ps : pull_streams) cudaStreamDestroy(ps);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (copy_stream) cudaStreamSynchronize(copy_stream);
    if (side) cudaStreamSynchronize(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    for (cudaEvent_t e : ev_sort)
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    for (auto& e : upload_events) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace sp {
namespace {

int64_t rows_per_dst(const sp_ctx* c) { return c->B / c->D; }

// Row 0 of global table g in the weight slab.
void* wptr(const sp_ctx* c, int g) {
  return static_cast<uint8_t*>(c->d_w) + c->woff[g] * elem_bytes(c->wt);
}

// Frees and re-allocates the shared sorted keys / bags for n positions.
void ensure_sort_capacity(sp_ctx* c, int64_t n) {
  if (n <= c->sort_cap && c->d_kb) return;
  SP_CUDA(cudaStreamSynchronize(c->stream));
  if (c->side) SP_CUDA(cudaStreamSynchronize(c->side));
  for (void* p : c->sort_owned) cudaFree(p);
  c->sort_owned.clear();
  const int64_t cap = std::max<int64_t>(n, 1);
  uint64_t dummy = 0;
  c->d_kb = dalloc<uint32_t>(cap, c->sort_owned, dummy);
  c->d_bb = dalloc<uint32_t>(cap, c->sort_owned, dummy);
  c->sort_cap = cap;
}

// The sort's packed intermediates for idx_cap lookups: the pairs, then the
// scratch of buckets too large for shared memory.
void ensure_mid(sp_ctx* c, VDev& v) {
  if (v.mid_cap >= v.idx_cap && v.d_mid != nullptr) return;
  SP_CUDA(cudaStreamSynchronize(c->stream));
  if (c->side) SP_CUDA(cudaStreamSynchronize(c->side));
  if (v.d_mid) cudaFree(v.d_mid);
  v.d_mid = nullptr;
  const int64_t cap = std::max<int64_t>(v.idx_cap, 1);
  SP_CUDA(cudaMalloc(&v.d_mid, 2 * cap * sort_mid_bytes(v.splan)));
  v.mid_cap = cap;
}

// The K4a sort plan of a (virtual) device (sort.cu: bucket width and
// warp-tile size per table from its expected lookups pf * B) and its device
// copies; re-planned by sp_ctx_set_sort_target.
void plan_sort(sp_ctx* c, VDev& v) {
  std::vector<double> est;
  for (int g : v.tables) est.push_back(std::max(0.0, c->tables[g].pooling_factor) * c->B);
  v.splan = sort_plan(v.meta_canon, est, c->B, c->sort_target, c->bags16);
  // the intermediates' width may change with the plan
  if (v.d_mid) cudaFree(v.d_mid);
  v.d_mid = nullptr;
  v.mid_cap = 0;
  if (v.idx_cap > 0) ensure_mid(c, v);
  for (void* p : {static_cast<void*>(v.d_stabs), static_cast<void*>(v.d_wtiles),
                   static_cast<void*>(v.d_bkts), static_cast<void*>(v.d_cnt),
                   static_cast<void*>(v.d_bstart), static_cast<void*>(v.d_big),
                   static_cast<void*>(v.d_nbig)})
    if (p) cudaFree(p);
  const SortPlan& pl = v.splan;
  auto up = [](auto*& dst, const auto& vec) {
    using T = typename std::decay_t<decltype(vec)>::value_type;
    SP_CUDA(cudaMalloc(&dst, std::max<size_t>(vec.size(), 1) * sizeof(T)));
    if (!vec.empty())
      SP_CUDA(cudaMemcpy(dst, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice));
  };
  up(v.d_stabs, pl.tabs);
  up(v.d_wtiles, pl.wtiles);
  up(v.d_bkts, pl.bkts);
  SP_CUDA(cudaMalloc(&v.d_cnt, std::max<int64_t>(pl.n_cnt, 1) * sizeof(int)));
  SP_CUDA(cudaMalloc(&v.d_bstart, std::max<int32_t>(pl.n_bstart, 1) * sizeof(int)));
  SP_CUDA(cudaMalloc(&v.d_big, std::max<size_t>(pl.bkts.size(), 1) * sizeof(int2)));
  SP_CUDA(cudaMalloc(&v.d_nbig, sizeof(int)));
}

void check_ctx(sp_ctx* c) {
  if (c == nullptr) raise(SP_ERR_BAD_INPUT, "null context");
  SP_CUDA(cudaSetDevice(c->device));
}

VDev& vdev_for(sp_ctx* c, int dev) {
  for (auto& v : c->vdevs)
    if (v.vid == dev) return v;
  raise(SP_ERR_BAD_INPUT, "device " + std::to_string(dev) + " is not held by this context");
}

void require_batch(sp_ctx* c) {
  if (!c->has_batch) raise(SP_ERR_BAD_INPUT, "no lookup batch uploaded");
}

// ---- per-kernel profiling ---------------------------------------------------

enum { kProfFwd = 0, kProfKeys = 1, kProfSort = 2, kProfSgd = 3, kProfExchange = 4 };

size_t prof_event(sp_ctx* c, cudaStream_t st) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    SP_CUDA(cudaEventCreate(&e));
    c->ev_pool.push_back(e);
  }
  SP_CUDA(cudaEventRecord(c->ev_pool[c->ev_used], st));
  return c->ev_used++;
}

// Records events around a stage launch (on the stream it is launched on)
// when profiling is on.
struct ProfScope {
  sp_ctx* c;
  int cls;
  cudaStream_t st;
  size_t a = 0;
  ProfScope(sp_ctx* c_, int cls_, cudaStream_t st_ = nullptr)
      : c(c_), cls(cls_), st(st_ ? st_ : c_->stream) {
    if (c->profiling) a = prof_event(c, st);
  }
  ~ProfScope() noexcept(false) {
    if (c->profiling) c->marks.push_back({cls, a, prof_event(c, st)});
  }
};

// ---- stages ---------------------------------------------------------------

// The sort runs on the side stream (forked after K1, see fork_sort).
bool overlap_active(const sp_ctx* c) {
  return c->overlap_sort && c->vdevs.size() == 1 && c->vdevs[0].nnz > 0;
}

void stage_forward(sp_ctx* c, VDev& v) {
  ProfScope prof(c, kProfFwd);
  launch_tbe_forward(v.d_meta_canon, v.d_tiles, v.n_tiles, c->B, v.d_off, v.d_idx, c->d_w, c->wt,
                     v.d_pooled, c->d_rowmap, v.W, c->stream);
}

// K4a: the stable sort of local tables [t0, t1) (their CSR is on the device)
// into the shared sorted keys / bags.
void sort_range(sp_ctx* c, VDev& v, int t0, int t1, cudaStream_t st) {
  if (t1 <= t0) return;
  ProfScope prof(c, kProfSort, st);
  launch_sort(v.splan, v.d_stabs, v.d_wtiles, v.d_bkts, t0, t1, c->B, v.d_off, v.d_idx, v.d_cnt,
              v.d_bstart, v.d_big, v.d_nbig, v.d_mid, v.mid_cap, c->d_kb, c->d_bb, c->bags16, st);
}

void stage_sort(sp_ctx* c, VDev& v, cudaStream_t st) {
  sort_range(c, v, 0, static_cast<int>(v.tables.size()), st);
}

// sorted: the overlapped sort already ran (the caller joined its stream).
// abort_flag (device, may be null): the SGD leaves the tables untouched
// when *abort_flag != 0 (a batch that failed its device-side validation).
void stage_backward(sp_ctx* c, VDev& v, bool sorted = false,
                    const int32_t* abort_flag = nullptr) {
  if (v.nnz == 0) return;
  if (!sorted) stage_sort(c, v, c->stream);
  ProfScope prof(c, kProfSgd);
  launch_sgd(v.d_meta_canon, v.d_sgd_tiles[v.cur], v.sgd_counts, c->d_kb, c->d_bb, c->bags16,
             v.d_grad, v.W, c->lr, c->d_w, c->wt, c->d_carry_f, c->d_carry_i, abort_flag,
             c->stream);
}

// One process per rank (world > 1); the exchange goes through peer memory
// (sp_ipc_import) or NCCL.
bool multi_rank(const sp_ctx* c) { return c->world > 1; }
bool nccl_mode(const sp_ctx* c) { return c->world > 1 && c->comm != nullptr; }

void d2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes) SP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
}

// Fwd exchange sends of (virtual) device v (emulation: device-local copies).
void a2a_fwd_emulated(sp_ctx* c, VDev& v) {
  const int64_t R = rows_per_dst(c);
  for (int j = 0; j < c->D; ++j)
    d2d(c->d_recv + j * R * c->W_total + R * c->cumW[v.vid],
        v.d_pooled + j * R * v.W, R * v.W * sizeof(float), c->stream);
}

void a2a_bwd_emulated(sp_ctx* c, VDev& v) {
  const int64_t R = rows_per_dst(c);
  for (int j = 0; j < c->D; ++j)
    d2d(v.d_grad + j * R * v.W, c->d_gin + j * R * c->W_total + R * c->cumW[v.vid],
        R * v.W * sizeof(float), c->stream);
}

// NCCL exchanges of this rank, driven by its ExchangePlan (the same plan
// sp_exchange_plan exports for host-side checks).
void a2a_fwd_nccl(sp_ctx* c) {
  VDev& v = c->vdevs[0];
  const ExchangePlan& pl = c->plan;
  SP_NCCL(nccl().GroupStart());
  for (int j = 0; j < c->D; ++j) {
    if (pl.send_cnt[j] > 0)
      SP_NCCL(nccl().Send(v.d_pooled + pl.send_off[j], pl.send_cnt[j], ncclFloat, j, c->comm,
                          c->stream));
    if (pl.recv_cnt[j] > 0)
      SP_NCCL(nccl().Recv(c->d_recv + pl.recv_off[j], pl.recv_cnt[j], ncclFloat, j, c->comm,
                          c->stream));
  }
  SP_NCCL(nccl().GroupEnd());
}

// Mirror of the forward exchange: gradients go back to the table owners.
void a2a_bwd_nccl(sp_ctx* c) {
  VDev& v = c->vdevs[0];
  const ExchangePlan& pl = c->plan;
  SP_NCCL(nccl().GroupStart());
  for (int j = 0; j < c->D; ++j) {
    if (pl.recv_cnt[j] > 0)
      SP_NCCL(nccl().Send(c->d_gin + pl.recv_off[j], pl.recv_cnt[j], ncclFloat, j, c->comm,
                          c->stream));
    if (pl.send_cnt[j] > 0)
      SP_NCCL(nccl().Recv(v.d_grad + pl.send_off[j], pl.send_cnt[j], ncclFloat, j, c->comm,
                          c->stream));
  }
  SP_NCCL(nccl().GroupEnd());
}

// Backward exchange over peer memory: this rank's gradient slice of every
// receiver j ([B/D, W_r] at j's slot for this rank) is pulled into grad_v.
// Each peer's slice is one contiguous NVLink read, on its own stream (its
// own copy engine), forked from and joined back into the main stream
// (capture-safe); the rank's own slice is a local copy on the main stream.
void a2a_bwd_peer(sp_ctx* c) {
  VDev& v = c->vdevs[0];
  const int64_t R = c->B / c->D;
  const size_t bytes = R * v.W * sizeof(float);
  if (bytes == 0) return;
  SP_CUDA(cudaEventRecord(c->ev_pull[0], c->stream));
  int k = 0;
  for (int j = 0; j < c->D; ++j) {
    float* dst = v.d_grad + j * R * v.W;
    const float* src = c->peer_gin[j] + R * c->cumW[c->rank];
    if (j == c->rank) {
      d2d(dst, src, bytes, c->stream);
      continue;
    }
    cudaStream_t ps = c->pull_streams[k];
    SP_CUDA(cudaStreamWaitEvent(ps, c->ev_pull[0], 0));
    d2d(dst, src, bytes, ps);
    SP_CUDA(cudaEventRecord(c->ev_pull[1 + k], ps));
    ++k;
  }
  for (int q = 0; q < k; ++q) SP_CUDA(cudaStreamWaitEvent(c->stream, c->ev_pull[1 + q], 0));
}

void a2a_fwd_rank(sp_ctx* c) {
  if (c->peer) return;  // K1 already stored every slice at its receiver
  if (!c->comm) raise(SP_ERR_BAD_INPUT, "multi-rank context without NCCL or peer memory");
  a2a_fwd_nccl(c);
}

void a2a_bwd_rank(sp_ctx* c) {
  if (c->peer) {
    a2a_bwd_peer(c);
    return;
  }
  if (!c->comm) raise(SP_ERR_BAD_INPUT, "multi-rank context without NCCL or peer memory");
  a2a_bwd_nccl(c);
}

// A whole iteration on one stream needs device-side rank barriers (NCCL); a
// peer-only context (no NCCL id) is driven stage by stage from the host,
// which synchronises the ranks in between.
void require_device_sync(const sp_ctx* c) {
  if (multi_rank(c) && c->comm == nullptr)
    raise(SP_ERR_BAD_INPUT,
          "peer-only context (no NCCL id): run the stages from the host with a rank "
          "barrier between sp_forward, sp_a2a_backward and sp_backward_sgd");
}

// Device-side rank barrier (NCCL); a peer-only context (no NCCL id) relies on
// the host to synchronise the ranks between stages.
void barrier(sp_ctx* c) {
  if (nccl_mode(c))
    SP_NCCL(nccl().AllReduce(c->d_barrier, c->d_barrier, 1, ncclInt32, ncclSum,
                          c->comm, c->stream));
}

bool exchange_needed(const sp_ctx* c) { return c->D > 1; }

// Fork, after K1: the side stream sorts the batch's lookups while the main
// stream runs the exchanges (NVLink-bound, a few SMs), joined before the SGD.
// Not concurrently with K1: both fill every SM, and at cfg3 D=1 the
// concurrent sort slowed the iteration 3.87 -> 4.02 ms (K1 loses resident
// warps and L2 to it); with no exchange (one device) the sort simply
// follows K1.
void fork_sort(sp_ctx* c) {
  SP_CUDA(cudaEventRecord(c->ev_fork, c->stream));
  SP_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  SP_CUDA(cudaEventRecord(c->ev_sort[0], c->side));
  stage_sort(c, c->vdevs[0], c->side);
  SP_CUDA(cudaEventRecord(c->ev_sort[1], c->side));
  SP_CUDA(cudaEventRecord(c->ev_join, c->side));
}

void join_sort(sp_ctx* c) { SP_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0)); }

// Stage 1 of an iteration: the forward, then the backward sort forked onto
// the side stream when the overlap is active.
void forward_stage(sp_ctx* c, bool ov) {
  for (auto& v : c->vdevs) stage_forward(c, v);
  if (ov) fork_sort(c);
}

void enqueue_iteration(sp_ctx* c) {
  const bool ov = overlap_active(c);
  forward_stage(c, ov);
  if (exchange_needed(c)) {
    ProfScope prof(c, kProfExchange);
    if (multi_rank(c)) {
      require_device_sync(c);
      if (c->peer) barrier(c);  // every rank's K1 peer stores have landed
      a2a_fwd_rank(c);
      if (c->peer) barrier(c);  // every rank's gradients are ready
      a2a_bwd_rank(c);
      if (c->peer) barrier(c);  // pulls done before the peers reuse their buffers
    } else {
      for (auto& v : c->vdevs) a2a_fwd_emulated(c, v);
      for (auto& v : c->vdevs) a2a_bwd_emulated(c, v);
    }
  }
  if (ov) join_sort(c);
  for (auto& v : c->vdevs) stage_backward(c, v, ov);
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  SP_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

}  // namespace
}  // namespace sp

using namespace sp;

namespace sp {
namespace {
// Runs this device's backward sort (no update) and returns the sorted keys
// as device-wide keys (local row base + row); bags (optional) receives the
// bag payload in sorted order.
std::vector<uint32_t> sorted_keys_host(sp_ctx* c, VDev& v, uint32_t* bags) {
  std::vector<uint32_t> keys(v.nnz);
  if (v.nnz == 0) return keys;
  stage_sort(c, v, c->stream);
  SP_CUDA(cudaMemcpyAsync(keys.data(), c->d_kb, v.nnz * 4, cudaMemcpyDeviceToHost, c->stream));
  std::vector<uint16_t> b16;
  if (bags && c->bags16) {
    b16.resize(v.nnz);
    SP_CUDA(cudaMemcpyAsync(b16.data(), c->d_bb, v.nnz * 2, cudaMemcpyDeviceToHost, c->stream));
  } else if (bags) {
    SP_CUDA(cudaMemcpyAsync(bags, c->d_bb, v.nnz * 4, cudaMemcpyDeviceToHost, c->stream));
  }
  SP_CUDA(cudaStreamSynchronize(c->stream));
  if (bags && c->bags16) std::copy(b16.begin(), b16.end(), bags);
  return keys;
}
}  // namespace
}  // namespace sp

extern "C" {

int sp_abi_version(void) { return SP_ABI_VERSION; }
const char* sp_last_error(void) { return g_last_error.c_str(); }
uint64_t sp_kernel_launches(void) { return g_launches.load(); }

int sp_host_alloc(uint64_t bytes, void** out) {
  return guarded([&] {
    if (out == nullptr) raise(SP_ERR_BAD_INPUT, "null output pointer");
    *out = nullptr;
    SP_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
  });
}

void sp_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int sp_nccl_unique_id(uint8_t out_id[SP_NCCL_ID_BYTES]) {
  return guarded([&] {
    ncclUniqueId id;
    SP_NCCL(nccl().GetUniqueId(&id));
    static_assert(sizeof(id.internal) == SP_NCCL_ID_BYTES, "nccl id size");
    std::memcpy(out_id, id.internal, SP_NCCL_ID_BYTES);
  });
}

int sp_ctx_create(const sp_table_spec* tables, int32_t num_tables,
                  int32_t num_devices, const int32_t* placement,
                  int32_t batch_size, double mem_cap_gb, float lr,
                  int32_t rank, int32_t world_size, const uint8_t* nccl_id,
                  int32_t cuda_device, sp_ctx** out) {
  return sp_ctx_create_ex(tables, num_tables, num_devices, placement, batch_size, mem_cap_gb,
                          lr, rank, world_size, nccl_id, cuda_device, SP_STORAGE_AUTO, out);
}

int sp_ctx_create_ex(const sp_table_spec* tables, int32_t num_tables,
                     int32_t num_devices, const int32_t* placement,
                     int32_t batch_size, double mem_cap_gb, float lr,
                     int32_t rank, int32_t world_size, const uint8_t* nccl_id,
                     int32_t cuda_device, int32_t storage, sp_ctx** out) {
  return guarded([&] {
    if (out == nullptr) raise(SP_ERR_BAD_INPUT, "null output handle");
    *out = nullptr;
    if (num_tables < 0 || (num_tables > 0 && (tables == nullptr || placement == nullptr)))
      raise(SP_ERR_BAD_INPUT, "tables/placement missing");
    if (num_devices < 1) raise(SP_ERR_BAD_INPUT, "num_devices must be >= 1");
    if (batch_size < 1) raise(SP_ERR_BAD_INPUT, "batch_size must be >= 1");
    if (batch_size % num_devices != 0)
      raise(SP_ERR_SHAPE_MISMATCH, "batch_size must be divisible by num_devices");
    if (!(world_size == 1 || world_size == num_devices))
      raise(SP_ERR_BAD_INPUT, "world_size must be 1 (emulation) or num_devices");
    if (rank < 0 || rank >= world_size) raise(SP_ERR_BAD_INPUT, "rank out of range");
    // world_size > 1 without an NCCL id: a peer-only context, whose exchange
    // must go through peer memory (sp_ipc_import) with host-driven stages

    // Placement legality, as evaluate_placement (oracle.hpp:190-204).
    std::vector<double> mem(num_devices, 0.0);
    for (int i = 0; i < num_tables; ++i) {
      const int d = placement[i];
      if (d < 0 || d >= num_devices) raise(SP_ERR_BAD_INPUT, "device id out of range");
      const sp_table_spec& t = tables[i];
      if (t.dim < 1 || t.hash_size < 1)
        raise(SP_ERR_BAD_INPUT, "dim and hash_size must be >= 1");
      if (t.hash_size > 0x7fffffffLL)
        raise(SP_ERR_BAD_INPUT, "hash_size above 2^31-1 is not supported (int32 ids)");
      mem[d] += t.table_size_gb;
    }
    if (mem_cap_gb > 0.0) {
      std::string offenders;
      for (int d = 0; d < num_devices; ++d)
        if (mem[d] > mem_cap_gb + 1e-9) {
          if (!offenders.empty()) offenders += ", ";
          offenders += std::to_string(d);
        }
      if (!offenders.empty())
        raise(SP_ERR_MEMORY_VIOLATION, "memory cap exceeded on device(s) " + offenders);
    }

    auto c = std::make_unique<sp_ctx>();
    c->M = num_tables;
    c->D = num_devices;
    c->world = world_size;
    c->rank = rank;
    c->B = batch_size;
    c->bags16 = batch_size <= 65536;
    c->lr = lr;
    c->cap = mem_cap_gb;
    c->device = cuda_device;
    c->tables.assign(tables, tables + num_tables);
    c->placement.assign(placement, placement + num_tables);
    SP_CUDA(cudaSetDevice(cuda_device));
    {
      // One rank per GPU: the forked sort shares the SMs with the exchange's
      // NCCL kernels (a few CTAs on the main stream); the main stream gets
      // the higher priority so those CTAs take the first free SM slots
      // instead of waiting behind every block of the sort. One process (no
      // exchange, or emulated devices): the side stream keeps the high
      // priority, so a sort overlapped with the host-buffer upload is
      // dispatched as K1's blocks retire.
      int lo = 0, hi = 0;
      SP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const bool ranks = world_size > 1;
      SP_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, ranks ? hi : lo));
      SP_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, ranks ? lo : hi));
    }
    SP_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    SP_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    SP_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    SP_CUDA(cudaEventCreate(&c->ev_sort[0]));
    SP_CUDA(cudaEventCreate(&c->ev_sort[1]));
    for (auto& e : c->stage_free) SP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : c->slot_done) SP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SP_CUDA(cudaEventCreateWithFlags(&c->meta_ready, cudaEventDisableTiming));

    // Columns: global table order; per-device widths.
    c->gcol.resize(num_tables);
    c->dev_W.assign(num_devices, 0);
    int64_t col = 0;
    for (int i = 0; i < num_tables; ++i) {
      c->gcol[i] = col;
      col += tables[i].dim;
      c->dev_W[placement[i]] += tables[i].dim;
    }
    c->W_total = col;
    c->cumW.assign(num_devices + 1, 0);
    for (int d = 0; d < num_devices; ++d) c->cumW[d + 1] = c->cumW[d] + c->dev_W[d];

    // Which devices live here.
    std::vector<int> held;
    if (world_size == 1)
      for (int d = 0; d < num_devices; ++d) held.push_back(d);
    else
      held.push_back(rank);

    // Storage type from the tables' own sizing: table_size_gb =
    // rows * dim * bytes_per_param / 2^30 (table_memory_gb, table.hpp:55-63):
    // 2 B/param (the reference's default, the paper's fp16 tables) -> fp16
    // (or bf16 when asked for), 4 B/param -> fp32; one type per context.
    if (storage < SP_STORAGE_AUTO || storage > SP_STORAGE_BF16)
      raise(SP_ERR_BAD_INPUT, "unknown storage type");
    {
      int bpp_all = 0;
      for (int i = 0; i < num_tables; ++i) {
        const sp_table_spec& t = tables[i];
        if (!(t.table_size_gb > 0.0)) continue;  // unsized: fp32
        const double bpp = t.table_size_gb * 1073741824.0 /
                           (static_cast<double>(t.hash_size) * static_cast<double>(t.dim));
        const int b = std::fabs(bpp - 2.0) < 0.5 ? 2 : (std::fabs(bpp - 4.0) < 1.0 ? 4 : 0);
        if (b == 0)
          raise(SP_ERR_BAD_INPUT, "table " + std::to_string(i) + " is sized at " +
                                      std::to_string(bpp) +
                                      " bytes/param: only 2 (fp16) or 4 (fp32) are stored");
        if (bpp_all != 0 && b != bpp_all)
          raise(SP_ERR_BAD_INPUT, "tables mix 2 and 4 bytes/param");
        bpp_all = b;
      }
      if (storage == SP_STORAGE_AUTO)
        c->wt = bpp_all == 2 ? WeightType::kF16 : WeightType::kF32;
      else if (storage == SP_STORAGE_F32)
        c->wt = WeightType::kF32;
      else
        c->wt = storage == SP_STORAGE_F16 ? WeightType::kF16 : WeightType::kBF16;
      const int want_b = c->wt == WeightType::kF32 ? 4 : 2;
      if (bpp_all != 0 && bpp_all != want_b)
        raise(SP_ERR_BAD_INPUT, "tables are sized at " + std::to_string(bpp_all) +
                                    " bytes/param but the storage type has " +
                                    std::to_string(want_b));
    }
    // Weight slab.
    const int64_t eb = elem_bytes(c->wt);
    const int64_t align = 256 / eb;  // elements per 256 bytes
    c->woff.assign(num_tables, -1);
    int64_t slab = 0;
    for (int d : held)
      for (int i = 0; i < num_tables; ++i)
        if (placement[i] == d) {
          c->woff[i] = slab;
          slab += tables[i].hash_size * tables[i].dim;
          // 256-byte aligned table bases: with dim a multiple of 16, every
          // row starts on a 64-byte DRAM burst (a 16-byte aligned base can
          // make each 64-byte row straddle two bursts)
          slab = (slab + align - 1) / align * align;
        }
    c->d_w = dalloc<uint8_t>(slab * eb, c->owned, c->dev_bytes);

    const int64_t R = static_cast<int64_t>(batch_size) / num_devices;
    for (int d : held) {
      VDev v;
      v.vid = d;
      for (int i = 0; i < num_tables; ++i)
        if (placement[i] == d) v.tables.push_back(i);
      const int T = static_cast<int>(v.tables.size());
      int64_t lcol = 0;
      uint64_t rb = 0;  // device-wide row base (sort keys)
      for (int li = 0; li < T; ++li) {
        const int g = v.tables[li];
        const sp_table_spec& t = tables[g];
        TableMeta m{};
        m.woff = c->woff[g];
        m.rows = t.hash_size;
        m.dim = t.dim;
        m.lcol = static_cast<int32_t>(lcol);
        m.rowbase = static_cast<uint32_t>(rb);
        m.cls = row_class(t.dim, c->wt);
        m.local = li;
        m.gid = g;
        v.meta_canon.push_back(m);
        for (int k = 0; k < t.dim; ++k) v.colmap.push_back(static_cast<int32_t>(c->gcol[g] + k));
        lcol += t.dim;
        rb += static_cast<uint64_t>(t.hash_size);
        if (rb > 0xffffffffULL)
          raise(SP_ERR_BAD_INPUT, "rows per device above 2^32 (32-bit sort keys)");
      }
      v.W = lcol;
      v.rows_total = static_cast<int64_t>(rb);
      {
        std::vector<int> canon_order(T);
        for (int li = 0; li < T; ++li) canon_order[li] = li;
        const std::vector<int4> ct = make_fwd_tiles(v.meta_canon, canon_order, batch_size);
        v.d_tiles_canon = dalloc<int4>(ct.size(), c->owned, c->dev_bytes);
        if (!ct.empty())
          SP_CUDA(cudaMemcpy(v.d_tiles_canon, ct.data(), ct.size() * sizeof(int4),
                             cudaMemcpyHostToDevice));
        v.tile_start.assign(T + 1, 0);
        for (const int4& tl : ct) ++v.tile_start[tl.x + 1];
        for (int li = 0; li < T; ++li) v.tile_start[li + 1] += v.tile_start[li];
        // (d_tiles_canon: the host-buffer step launches K1 per upload chunk
        // of tables from it.) The iteration's K1 grid runs the tables in
        // canonical (placement) order too, each a contiguous block range.
        // Measured against reordering by weight
        // (cfg3 K1 ms, fp32 / fp16 tables): canonical 1.374 / 1.101;
        // heaviest / lightest interleave by pf x dim (round 1's choice, made
        // while the sort still ran beside K1) 1.408 / 1.134; interleave by
        // rows x dim 1.378 / 1.121; heaviest first 1.409; largest touched
        // footprint followed by 2-4 of the smallest 1.370-1.385 / 1.121-1.128
        // (fewer DRAM bytes, 4.68 vs 4.77 GB, but longer tails).
        v.n_tiles = static_cast<int64_t>(ct.size());
        // ... except that the lightest tables (pf x dim) run last, lightest
        // at the very end, so the kernel's tail is short tiles: cfg3 K1
        // 1.374 -> 1.362 ms fp32 (1.101 -> 1.098 fp16) with 10 of them; 25
        // the same
        {
          constexpr int kLightTail = 10;
          std::vector<int> light(T);
          std::iota(light.begin(), light.end(), 0);
          std::stable_sort(light.begin(), light.end(), [&](int a, int b) {
            const auto& ta = tables[v.tables[a]];
            const auto& tb = tables[v.tables[b]];
            return ta.pooling_factor * ta.dim < tb.pooling_factor * tb.dim;
          });
          const int k = std::min(T, kLightTail);
          std::vector<char> is_tail(T, 0);
          for (int q = 0; q < k; ++q) is_tail[light[q]] = 1;
          std::vector<int> ord;
          for (int li = 0; li < T; ++li)
            if (!is_tail[li]) ord.push_back(li);
          for (int q = k - 1; q >= 0; --q) ord.push_back(light[q]);
          const std::vector<int4> ot = make_fwd_tiles(v.meta_canon, ord, batch_size);
          v.d_tiles = dalloc<int4>(ot.size(), c->owned, c->dev_bytes);
          if (!ot.empty())
            SP_CUDA(cudaMemcpy(v.d_tiles, ot.data(), ot.size() * sizeof(int4),
                               cudaMemcpyHostToDevice));
        }
      }
      v.d_meta_canon = dalloc<TableMeta>(T, c->owned, c->dev_bytes);
      v.d_colmap = dalloc<int32_t>(v.W, c->owned, c->dev_bytes);
      if (T) {
        SP_CUDA(cudaMemcpy(v.d_meta_canon, v.meta_canon.data(), T * sizeof(TableMeta), cudaMemcpyHostToDevice));
      }
      if (v.W)
        SP_CUDA(cudaMemcpy(v.d_colmap, v.colmap.data(), v.W * sizeof(int32_t), cudaMemcpyHostToDevice));
      v.d_off = dalloc<int32_t>(static_cast<int64_t>(T) * batch_size + 1, c->owned, c->dev_bytes);
      v.d_pooled = dalloc<float>(static_cast<int64_t>(batch_size) * v.W, c->owned, c->dev_bytes);
      v.d_grad = num_devices == 1
                     ? nullptr
                     : dalloc<float>(static_cast<int64_t>(batch_size) * v.W, c->owned, c->dev_bytes);
      for (auto& e : v.ev) SP_CUDA(cudaEventCreate(&e));
      c->vdevs.push_back(std::move(v));
    }

    c->n_dst = world_size == 1 ? num_devices : 1;
    if (num_devices == 1) {
      // D == 1: the exchange is the identity; alias the buffers.
      c->d_recv = c->vdevs[0].d_pooled;
      c->d_gin = dalloc<float>(static_cast<int64_t>(batch_size) * c->W_total, c->owned, c->dev_bytes);
      c->vdevs[0].d_grad = c->d_gin;
    } else {
      c->d_recv = dalloc<float>(c->n_dst * R * c->W_total, c->owned, c->dev_bytes);
      c->d_gin = dalloc<float>(c->n_dst * R * c->W_total, c->owned, c->dev_bytes);
    }
    c->d_flag = dalloc<int32_t>(1, c->owned, c->dev_bytes);
    c->d_bd = dalloc<double>(8 * static_cast<int64_t>(num_devices), c->owned, c->dev_bytes);
    c->d_barrier = dalloc<int32_t>(1, c->owned, c->dev_bytes);
    SP_CUDA(cudaMemset(c->d_barrier, 0, sizeof(int32_t)));
    for (auto& e : c->ev_a2a) SP_CUDA(cudaEventCreate(&e));
    for (auto& v : c->vdevs) plan_sort(c.get(), v);
    if (world_size > 1) {
      c->plan = make_plan(tables, num_tables, num_devices, placement, batch_size, rank);
      if (nccl_id != nullptr) {
        ncclUniqueId id;
        std::memcpy(id.internal, nccl_id, SP_NCCL_ID_BYTES);
        SP_NCCL(nccl().CommInitRank(&c->comm, world_size, id, rank));
      }
    }
    *out = c.release();
  });
}

void sp_ctx_destroy(sp_ctx* ctx) { delete ctx; }

int sp_ipc_export(sp_ctx* ctx, uint8_t out[SP_IPC_BYTES]) {
  return guarded([&] {
    check_ctx(ctx);
    if (out == nullptr) raise(SP_ERR_BAD_INPUT, "null output");
    if (ctx->world < 2) raise(SP_ERR_BAD_INPUT, "peer memory needs a multi-rank context");
    cudaIpcMemHandle_t h[2];
    SP_CUDA(cudaIpcGetMemHandle(&h[0], ctx->d_recv));
    SP_CUDA(cudaIpcGetMemHandle(&h[1], ctx->d_gin));
    static_assert(2 * sizeof(cudaIpcMemHandle_t) == SP_IPC_BYTES, "IPC handle size");
    std::memcpy(out, h, sizeof(h));
  });
}

int sp_ipc_import(sp_ctx* ctx, const uint8_t* all) {
  return guarded([&] {
    check_ctx(ctx);
    sp_ctx* c = ctx;
    if (all == nullptr) raise(SP_ERR_BAD_INPUT, "null handles");
    if (c->world < 2 || c->world > kMaxPeers)
      raise(SP_ERR_BAD_INPUT, "peer memory supports 2.." + std::to_string(kMaxPeers) + " ranks");
    if (c->peer) raise(SP_ERR_BAD_INPUT, "peer memory already imported");
    SP_CUDA(cudaStreamSynchronize(c->stream));
    for (int j = 0; j < c->world; ++j) {
      if (j == c->rank) {
        c->peer_recv[j] = c->d_recv;
        c->peer_gin[j] = c->d_gin;
        continue;
      }
      cudaIpcMemHandle_t h[2];
      std::memcpy(h, all + static_cast<size_t>(j) * SP_IPC_BYTES, sizeof(h));
      for (int k = 0; k < 2; ++k) {
        void* p = nullptr;
        SP_CUDA(cudaIpcOpenMemHandle(&p, h[k], cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(p);
        (k == 0 ? c->peer_recv : c->peer_gin)[j] = static_cast<float*>(p);
      }
    }
    // K1's row map: batch slice j -> rank j's receive slot for this rank
    RowMap rm{};
    const int64_t R = c->B / c->D;
    for (int j = 0; j < c->D; ++j) rm.base[j] = c->peer_recv[j] + R * c->cumW[c->rank];
    rm.rows_per_part = R;
    rm.parts = c->D;
    for (int j = 0; j + 1 < c->world; ++j) {
      cudaStream_t ps = nullptr;
      SP_CUDA(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
      c->pull_streams.push_back(ps);
    }
    c->ev_pull.resize(c->world);
    for (auto& e : c->ev_pull) SP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->d_rowmap = dalloc<RowMap>(1, c->owned, c->dev_bytes);
    SP_CUDA(cudaMemcpy(c->d_rowmap, &rm, sizeof(rm), cudaMemcpyHostToDevice));
    c->peer = true;
    if (c->graph_exec) {
      cudaGraphExecDestroy(c->graph_exec);
      c->graph_exec = nullptr;
    }
  });
}

int sp_ctx_synchronize(sp_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
    SP_CUDA(cudaStreamSynchronize(ctx->side));
  });
}

int sp_ctx_stream(sp_ctx* ctx, void** stream) {
  return guarded([&] {
    check_ctx(ctx);
    *stream = ctx->stream;
  });
}

int sp_ctx_device_bytes(sp_ctx* ctx, uint64_t* bytes) {
  return guarded([&] {
    check_ctx(ctx);
    uint64_t b = ctx->dev_bytes;
    b += ctx->sort_cap * 4 * 2 + ctx->stage_cap * 8;
    for (auto& v : ctx->vdevs)
      b += v.idx_cap * 4 + v.mid_cap * 2 * sort_mid_bytes(v.splan) +
           (v.splan.n_cnt + v.splan.n_bstart) * 4;
    *bytes = b;
  });
}

int sp_ctx_local_tables(sp_ctx* ctx, int32_t* ids, int32_t* n_out) {
  return guarded([&] {
    check_ctx(ctx);
    int32_t n = 0;
    for (auto& v : ctx->vdevs)
      for (int g : v.tables) {
        if (ids) ids[n] = g;
        ++n;
      }
    if (ids) std::sort(ids, ids + n);
    *n_out = n;
  });
}

int sp_init_tables(sp_ctx* ctx, uint64_t seed) {
  return guarded([&] {
    check_ctx(ctx);
    for (auto& v : ctx->vdevs)
      for (int g : v.tables)
        launch_init_weights(wptr(ctx, g), ctx->wt, ctx->tables[g].hash_size,
                            ctx->tables[g].dim, ctx->tables[g].id, seed, ctx->stream);
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sp_set_table(sp_ctx* ctx, int32_t table_id, const float* rows) {
  return guarded([&] {
    check_ctx(ctx);
    if (table_id < 0 || table_id >= ctx->M || ctx->woff[table_id] < 0)
      raise(SP_ERR_UNKNOWN_TABLE, "table id " + std::to_string(table_id) + " is not local");
    const auto& t = ctx->tables[table_id];
    const int64_t n = t.hash_size * t.dim;
    if (ctx->wt == WeightType::kF32) {
      SP_CUDA(cudaMemcpyAsync(wptr(ctx, table_id), rows, n * sizeof(float),
                              cudaMemcpyHostToDevice, ctx->stream));
    } else {
      float* tmp = nullptr;
      SP_CUDA(cudaMalloc(&tmp, std::max<int64_t>(n, 1) * sizeof(float)));
      SP_CUDA(cudaMemcpyAsync(tmp, rows, n * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
      launch_f32_to_weights(tmp, wptr(ctx, table_id), ctx->wt, n, ctx->stream);
      SP_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(tmp);
    }
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sp_get_table(sp_ctx* ctx, int32_t table_id, float* rows) {
  return guarded([&] {
    check_ctx(ctx);
    if (table_id < 0 || table_id >= ctx->M || ctx->woff[table_id] < 0)
      raise(SP_ERR_UNKNOWN_TABLE, "table id " + std::to_string(table_id) + " is not local");
    const auto& t = ctx->tables[table_id];
    const int64_t n = t.hash_size * t.dim;
    if (ctx->wt == WeightType::kF32) {
      SP_CUDA(cudaMemcpyAsync(rows, wptr(ctx, table_id), n * sizeof(float),
                              cudaMemcpyDeviceToHost, ctx->stream));
    } else {
      float* tmp = nullptr;
      SP_CUDA(cudaMalloc(&tmp, std::max<int64_t>(n, 1) * sizeof(float)));
      launch_weights_to_f32(wptr(ctx, table_id), ctx->wt, tmp, n, ctx->stream);
      SP_CUDA(cudaMemcpyAsync(rows, tmp, n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
      SP_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(tmp);
    }
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// Layout metadata of the current batch (SGD tiles on the device). The tiles go through the pinned buffer of `slot`
// on the copy stream, ahead of the batch's H2D and into the slot's own
// device buffer, so a step's upload never queues behind the previous step's
// compute (a pageable or compute-stream copy would).
// pipelined: the caller orders this step after the slot's previous user
// (sp_run_batches, steps >= 1); otherwise the upload waits for all work
// already enqueued on the compute stream.
static void finish_batch(sp_ctx* c, int slot = 0, bool pipelined = false) {
  int64_t max_nnz = 0;
  std::vector<std::vector<int>> tiles;
  size_t need = 0;
  for (auto& v : c->vdevs) {
    tiles.push_back(make_sgd_tiles(v.table_nnz, v.meta_canon, v.sgd_counts));
    need += tiles.back().size() * sizeof(int) + 16;
  }
  if (c->stage_used[slot]) SP_CUDA(cudaEventSynchronize(c->stage_free[slot]));
  if (need > c->meta_cap[slot]) {
    if (c->meta_host[slot]) cudaFreeHost(c->meta_host[slot]);
    c->meta_host[slot] = nullptr;
    SP_CUDA(cudaMallocHost(&c->meta_host[slot], need));
    c->meta_cap[slot] = need;
  }
  // the previous SGD that read this slot's tiles must be done
  if (!pipelined) {
    SP_CUDA(cudaEventRecord(c->meta_ready, c->stream));
    SP_CUDA(cudaStreamWaitEvent(c->copy_stream, c->meta_ready, 0));
  } else if (c->slot_done_used[slot]) {
    SP_CUDA(cudaStreamWaitEvent(c->copy_stream, c->slot_done[slot], 0));
  }
  size_t mo = 0;  // offset into the pinned buffer
  for (size_t vi = 0; vi < c->vdevs.size(); ++vi) {
    VDev& v = c->vdevs[vi];
    max_nnz = std::max(max_nnz, v.nnz);
    const std::vector<int>& tl = tiles[vi];
    v.n_sgd_tiles = static_cast<int64_t>(tl.size()) / kSgdTileInts;
    const int64_t wide = v.sgd_counts[1];
    if (wide > c->carry_cap) {  // segmented SGD carries (shared, stream-ordered)
      SP_CUDA(cudaStreamSynchronize(c->stream));
      if (c->d_carry_f) cudaFree(c->d_carry_f);
      if (c->d_carry_i) cudaFree(c->d_carry_i);
      SP_CUDA(cudaMalloc(&c->d_carry_f, sgd_carry_floats(wide) * sizeof(float)));
      SP_CUDA(cudaMalloc(&c->d_carry_i, wide * 4 * sizeof(int32_t)));
      c->carry_cap = wide;
    }
    if (static_cast<int64_t>(tl.size()) > v.sgd_tile_cap[slot]) {
      SP_CUDA(cudaStreamSynchronize(c->stream));
      SP_CUDA(cudaStreamSynchronize(c->side));
      SP_CUDA(cudaStreamSynchronize(c->copy_stream));
      if (v.d_sgd_tiles[slot]) cudaFree(v.d_sgd_tiles[slot]);
      v.d_sgd_tiles[slot] = nullptr;
      SP_CUDA(cudaMalloc(&v.d_sgd_tiles[slot], tl.size() * sizeof(int)));
      v.sgd_tile_cap[slot] = static_cast<int64_t>(tl.size());
    }
    if (!tl.empty()) {
      std::memcpy(c->meta_host[slot] + mo, tl.data(), tl.size() * sizeof(int));
      SP_CUDA(cudaMemcpyAsync(v.d_sgd_tiles[slot], c->meta_host[slot] + mo,
                              tl.size() * sizeof(int), cudaMemcpyHostToDevice,
                              c->copy_stream));
      mo += (tl.size() * sizeof(int) + 15) & ~size_t(15);
    }
    v.cur = slot;
  }
  // the compute stream reads the tiles only after this point
  SP_CUDA(cudaEventRecord(c->meta_ready, c->copy_stream));
  SP_CUDA(cudaStreamWaitEvent(c->stream, c->meta_ready, 0));
  ensure_sort_capacity(c, max_nnz);
  c->has_batch = true;
  if (c->graph_exec) {
    cudaGraphExecDestroy(c->graph_exec);
    c->graph_exec = nullptr;
  }
}

static void alloc_indices(sp_ctx* c, VDev& v, int64_t nnz) {
  if (nnz > 0x7fffffffLL)
    raise(SP_ERR_BAD_INPUT, "more than 2^31-1 lookups on one device (int32 CSR)");
  if (nnz > v.idx_cap || v.d_idx == nullptr) {
    SP_CUDA(cudaStreamSynchronize(c->stream));
    if (c->side) SP_CUDA(cudaStreamSynchronize(c->side));
    if (v.d_idx) cudaFree(v.d_idx);
    v.d_idx = nullptr;
    const int64_t cap = std::max<int64_t>(nnz, 1);
    SP_CUDA(cudaMalloc(&v.d_idx, cap * sizeof(int32_t)));
    v.idx_cap = cap;
  }
  ensure_mid(c, v);
  v.nnz = nnz;
}

}  // extern "C"

namespace sp {
namespace {

// validate_batch (table.hpp:167-184), O(M) parts on the host (the
// monotonicity inside a table and the index range are checked on the device
// while narrowing); sizes every device's CSR and the int64 staging buffer.
void host_validate_and_size(sp_ctx* c, const int64_t* offsets, int64_t offsets_len,
                            int64_t indices_len, bool two_slots = false) {
  const int64_t B = c->B;
  if (offsets_len != static_cast<int64_t>(c->M) * B + 1)
    raise(SP_ERR_MALFORMED_BATCH, "offsets length " + std::to_string(offsets_len) +
                                      ", expected " + std::to_string(c->M * B + 1));
  if (offsets[0] != 0) raise(SP_ERR_MALFORMED_BATCH, "offsets must start at 0");
  if (offsets[offsets_len - 1] != indices_len)
    raise(SP_ERR_MALFORMED_BATCH, "last offset != indices length");
  for (int t = 0; t <= c->M; ++t) {
    const int64_t o = offsets[t * B];
    if (o < 0 || o > indices_len || (t > 0 && o < offsets[(t - 1) * B]))
      raise(SP_ERR_MALFORMED_BATCH, "offsets decrease at table " + std::to_string(t));
  }
  c->has_batch = false;  // until the device-side checks pass
  int64_t stage_need = 0;
  for (auto& v : c->vdevs) {
    v.table_nnz.clear();
    int64_t n = 0, st = 0;
    for (int g : v.tables) {
      const int64_t tn = offsets[(g + 1) * B] - offsets[g * B];
      v.table_nnz.push_back(tn);
      n += tn;
      st += tn + B + 1;
    }
    alloc_indices(c, v, n);
    stage_need += st;  // copies run ahead of the narrows: no reuse across devices
  }
  if (stage_need > c->stage_cap || (two_slots && c->d_stage64_alt == nullptr)) {
    SP_CUDA(cudaStreamSynchronize(c->stream));
    SP_CUDA(cudaStreamSynchronize(c->copy_stream));
    const int64_t cap = std::max<int64_t>({stage_need, c->stage_cap, 1});
    if (stage_need > c->stage_cap) {
      if (c->d_stage64) cudaFree(c->d_stage64);
      SP_CUDA(cudaMalloc(&c->d_stage64, cap * sizeof(int64_t)));
      if (c->d_stage64_alt) {
        cudaFree(c->d_stage64_alt);
        c->d_stage64_alt = nullptr;
      }
    }
    if (two_slots && c->d_stage64_alt == nullptr)
      SP_CUDA(cudaMalloc(&c->d_stage64_alt, cap * sizeof(int64_t)));
    c->stage_cap = cap;
  }
}

cudaEvent_t upload_event(sp_ctx* c, size_t& n_ev) {
  if (n_ev == c->upload_events.size()) {
    cudaEvent_t e;
    SP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->upload_events.push_back(e);
  }
  return c->upload_events[n_ev++];
}

// Coalesced, pipelined H2D of a host LookupBatch: local tables with
// consecutive global ids are adjacent in the reference CSR, so each such run
// is copied with two large memcpys, cut into chunks of <= kUploadChunk
// indices on the copy stream while the
// compute stream narrows the previous chunk to the int32 device CSR (and
// flags malformed data in d_flag, clamping it so later kernels stay in
// bounds). chunk_done(v, t0, t1) runs after the narrows of local tables
// [t0, t1) of device v are enqueued on the compute stream.
// flag: this step's validation flag; slot: staging buffer 0 or 1 (the copy
// stream only waits for the narrows of the last step that used the slot, so
// with two slots a step's H2D overlaps the previous step's compute).
// copy_idx(dst, i0, n, stream) enqueues the H2D of indices [i0, i0 + n) into
// the device staging slot (from host memory, or streamed from a DSLB file).
template <class F, class CopyIdx>
void enqueue_upload_from(sp_ctx* c, const int64_t* offsets, CopyIdx&& copy_idx, F&& chunk_done,
                         int32_t* flag = nullptr, int slot = 0) {
  const int64_t B = c->B;
  const int64_t kUploadChunk = c->upload_chunk;
  if (flag == nullptr) flag = c->d_flag;
  size_t n_ev = 0;
  SP_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), c->stream));
  if (c->stage_used[slot]) SP_CUDA(cudaStreamWaitEvent(c->copy_stream, c->stage_free[slot], 0));
  int64_t* const stage = slot == 0 ? c->d_stage64 : c->d_stage64_alt;
  int64_t so = 0;  // staging offset (int64 elements), across all devices
  for (auto& v : c->vdevs) {
    const int T = static_cast<int>(v.tables.size());
    int32_t base = 0;
    int li = 0;
    while (li < T) {
      int run_end = li + 1;
      while (run_end < T && v.tables[run_end] == v.tables[run_end - 1] + 1) ++run_end;
      int c0 = li;
      while (c0 < run_end) {
        int c1 = c0 + 1;
        int64_t acc = v.table_nnz[c0];
        while (c1 < run_end && acc + v.table_nnz[c1] <= kUploadChunk)
          acc += v.table_nnz[c1++];
        const int64_t g0 = v.tables[c0], g1 = v.tables[c1 - 1] + 1;
        const int64_t n_off = (g1 - g0) * B + 1;
        const int64_t i0 = offsets[g0 * B];
        const int64_t n_idx = offsets[g1 * B] - i0;
        int64_t* s_off = stage + so;
        int64_t* s_idx = s_off + n_off;
        SP_CUDA(cudaMemcpyAsync(s_off, offsets + g0 * B, n_off * sizeof(int64_t),
                                cudaMemcpyHostToDevice, c->copy_stream));
        if (n_idx) copy_idx(s_idx, i0, n_idx, c->copy_stream);
        cudaEvent_t e = upload_event(c, n_ev);
        SP_CUDA(cudaEventRecord(e, c->copy_stream));
        SP_CUDA(cudaStreamWaitEvent(c->stream, e, 0));
        for (int t = c0; t < c1; ++t) {
          const int g = v.tables[t];
          const int64_t tn = v.table_nnz[t];
          launch_narrow_table(s_off + (g - g0) * B, s_idx + (offsets[g * B] - i0), c->B, tn,
                              c->tables[g].hash_size, base, v.d_off + int64_t(t) * B,
                              v.d_idx + base, flag, c->stream);
          base += static_cast<int32_t>(tn);
        }
        chunk_done(v, c0, c1);
        so += n_off + n_idx;
        c0 = c1;
      }
      li = run_end;
    }
    if (v.tables.empty()) SP_CUDA(cudaMemsetAsync(v.d_off, 0, sizeof(int32_t), c->stream));
  }
  SP_CUDA(cudaEventRecord(c->stage_free[slot], c->stream));
  c->stage_used[slot] = true;
}

template <class F>
void enqueue_upload(sp_ctx* c, const int64_t* offsets, const int64_t* indices, F&& chunk_done,
                    int32_t* flag = nullptr, int slot = 0) {
  enqueue_upload_from(
      c, offsets,
      [indices](int64_t* dst, int64_t i0, int64_t n, cudaStream_t st) {
        SP_CUDA(cudaMemcpyAsync(dst, indices + i0, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                                st));
      },
      chunk_done, flag, slot);
}

void raise_batch_flag(int32_t flag) {
  if (flag & 1) raise(SP_ERR_MALFORMED_BATCH, "offsets decrease inside a table");
  if (flag & 2) raise(SP_ERR_BAD_INPUT, "lookup index outside [0, hash_size)");
}

}  // namespace
}  // namespace sp

extern "C" {

int sp_upload_batch(sp_ctx* ctx, const int64_t* offsets, int64_t offsets_len,
                    const int64_t* indices, int64_t indices_len) {
  return guarded([&] {
    check_ctx(ctx);
    sp_ctx* c = ctx;
    host_validate_and_size(c, offsets, offsets_len, indices_len);
    enqueue_upload(c, offsets, indices, [](VDev&, int, int) {});
    int32_t flag = 0;
    SP_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    SP_CUDA(cudaStreamSynchronize(c->stream));
    raise_batch_flag(flag);
    finish_batch(c);
  });
}

// load_lookup_batch (table.hpp:283-305) + sp_upload_batch without a host
// copy of the indices: the header and offsets are read on the host, each
// local table run's index segment is streamed file -> pinned ring -> device
// staging (only this context's tables are read), then narrowed and
// validated exactly like sp_upload_batch.
int sp_upload_batch_file(sp_ctx* ctx, const char* path) {
  return guarded([&] {
    check_ctx(ctx);
    sp_ctx* c = ctx;
    DslbFile f;
    f.open(path);
    f.validate_shape();
    if (static_cast<int>(f.num_tables) != c->M || static_cast<int>(f.batch_size) != c->B)
      raise(SP_ERR_SHAPE_MISMATCH, "batch shape (" + std::to_string(f.num_tables) + " tables, B=" +
                                       std::to_string(f.batch_size) +
                                       ") does not match the context");
    const int64_t n_off = static_cast<int64_t>(f.offsets_len);
    if (c->file_off_cap < n_off) {
      SP_CUDA(cudaStreamSynchronize(c->stream));
      SP_CUDA(cudaStreamSynchronize(c->copy_stream));
      if (c->file_off) cudaFreeHost(c->file_off);
      c->file_off = nullptr;
      c->file_off_cap = 0;
      SP_CUDA(cudaMallocHost(&c->file_off, n_off * sizeof(int64_t)));
      c->file_off_cap = n_off;
    } else {
      // the previous upload's offset copies may still read the buffer
      SP_CUDA(cudaStreamSynchronize(c->copy_stream));
    }
    f.read_offsets(c->file_off, 0, n_off);
    const int64_t indices_len = static_cast<int64_t>(f.indices_len);
    host_validate_and_size(c, c->file_off, n_off, indices_len);
    if (!c->file_ring) c->file_ring = std::make_unique<DslbStreamer>();
    DslbStreamer* ring = c->file_ring.get();
    enqueue_upload_from(
        c, c->file_off,
        [&](int64_t* dst, int64_t i0, int64_t n, cudaStream_t st) {
          ring->indices_to_device(f, i0, n, dst, st);
        },
        [](VDev&, int, int) {});
    int32_t flag = 0;
    SP_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    SP_CUDA(cudaStreamSynchronize(c->stream));
    raise_batch_flag(flag);
    finish_batch(c);
  });
}

int sp_synth_batch(sp_ctx* ctx, uint64_t seed) {
  return guarded([&] {
    check_ctx(ctx);
    sp_ctx* c = ctx;
    for (auto& v : c->vdevs) {
      const int T = static_cast<int>(v.tables.size());
      const int64_t nb = static_cast<int64_t>(T) * c->B;
      std::vector<int32_t> gid(T);
      std::vector<int64_t> lmax(T), rows(T);
      std::vector<uint64_t> thr(T);
      for (int li = 0; li < T; ++li) {
        const auto& t = c->tables[v.tables[li]];
        gid[li] = t.id;  // the generator is keyed by the table's id
        lmax[li] = static_cast<int64_t>(std::floor(2.0 * t.pooling_factor));
        rows[li] = t.hash_size;
        double h = 0.0;  // hot_mass (oracle.hpp:119-123)
        for (int b = 4; b < SP_NUM_BINS; ++b) h += t.dist[b];
        thr[li] = hot_threshold(h);
      }
      std::vector<void*> tmp;
      uint64_t dummy = 0;
      int32_t* d_gid = dalloc<int32_t>(T, tmp, dummy);
      int64_t* d_lmax = dalloc<int64_t>(T, tmp, dummy);
      int64_t* d_rows = dalloc<int64_t>(T, tmp, dummy);
      uint64_t* d_thr = dalloc<uint64_t>(T, tmp, dummy);
      int32_t* d_len = dalloc<int32_t>(nb + 1, tmp, dummy);
      size_t tb = exclusive_scan_i32(nullptr, 0, d_len, v.d_off, nb + 1, c->stream);
      void* d_tmp = dalloc<uint8_t>(tb, tmp, dummy);
      auto cleanup = [&] {
        cudaStreamSynchronize(c->stream);
        for (void* p : tmp) cudaFree(p);
      };
      try {
        if (T) {
          SP_CUDA(cudaMemcpy(d_gid, gid.data(), T * 4, cudaMemcpyHostToDevice));
          SP_CUDA(cudaMemcpy(d_lmax, lmax.data(), T * 8, cudaMemcpyHostToDevice));
          SP_CUDA(cudaMemcpy(d_rows, rows.data(), T * 8, cudaMemcpyHostToDevice));
          SP_CUDA(cudaMemcpy(d_thr, thr.data(), T * 8, cudaMemcpyHostToDevice));
        }
        SP_CUDA(cudaMemsetAsync(d_len + nb, 0, sizeof(int32_t), c->stream));
        if (T) launch_synth_lengths(d_gid, d_lmax, T, c->B, seed, d_len, c->stream);
        exclusive_scan_i32(d_tmp, tb, d_len, v.d_off, nb + 1, c->stream);
        int32_t total = 0;
        SP_CUDA(cudaMemcpyAsync(&total, v.d_off + nb, 4, cudaMemcpyDeviceToHost, c->stream));
        SP_CUDA(cudaStreamSynchronize(c->stream));
        alloc_indices(c, v, total);
        v.table_nnz.assign(T, 0);
        if (T) launch_synth_indices(d_gid, d_rows, d_thr, T, c->B, seed, v.d_off, v.d_idx, c->stream);
        // per-table nnz (host copy of the table boundaries)
        std::vector<int32_t> bounds(T + 1);
        for (int li = 0; li <= T; ++li)
          SP_CUDA(cudaMemcpyAsync(&bounds[li], v.d_off + static_cast<int64_t>(li) * c->B, 4,
                                  cudaMemcpyDeviceToHost, c->stream));
        SP_CUDA(cudaStreamSynchronize(c->stream));
        for (int li = 0; li < T; ++li) v.table_nnz[li] = bounds[li + 1] - bounds[li];
      } catch (...) {
        cleanup();
        throw;
      }
      cleanup();
    }
    finish_batch(c);
  });
}

int sp_batch_nnz(sp_ctx* ctx, int64_t* nnz) {
  return guarded([&] {
    check_ctx(ctx);
    int64_t n = 0;
    for (auto& v : ctx->vdevs) n += v.nnz;
    *nnz = n;
  });
}

int sp_forward(sp_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    require_batch(ctx);
    for (auto& v : ctx->vdevs) stage_forward(ctx, v);
  });
}

int sp_a2a_forward(sp_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    if (!exchange_needed(ctx)) return;
    if (multi_rank(ctx)) a2a_fwd_rank(ctx);
    else for (auto& v : ctx->vdevs) a2a_fwd_emulated(ctx, v);
  });
}

int sp_a2a_backward(sp_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    if (!exchange_needed(ctx)) return;
    if (multi_rank(ctx)) a2a_bwd_rank(ctx);
    else for (auto& v : ctx->vdevs) a2a_bwd_emulated(ctx, v);
  });
}

int sp_backward_sgd(sp_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    require_batch(ctx);
    for (auto& v : ctx->vdevs) stage_backward(ctx, v);
  });
}

// Host permutations between the global [rows, W_total] order and the
// grouped-by-source exchange layout of one destination slice.
static void grouped_to_global(const sp_ctx* c, const float* grouped, float* global,
                              int64_t R) {
  for (int i = 0; i < c->D; ++i) {
    const float* src = grouped + R * c->cumW[i];
    const int64_t Wi = c->dev_W[i];
    std::vector<int64_t> cols;
    for (int t = 0; t < c->M; ++t)
      if (c->placement[t] == i)
        for (int k = 0; k < c->tables[t].dim; ++k) cols.push_back(c->gcol[t] + k);
    for (int64_t r = 0; r < R; ++r)
      for (int64_t k = 0; k < Wi; ++k) global[r * c->W_total + cols[k]] = src[r * Wi + k];
  }
}

static void global_to_grouped(const sp_ctx* c, const float* global, float* grouped,
                              int64_t R) {
  for (int i = 0; i < c->D; ++i) {
    float* dst = grouped + R * c->cumW[i];
    const int64_t Wi = c->dev_W[i];
    std::vector<int64_t> cols;
    for (int t = 0; t < c->M; ++t)
      if (c->placement[t] == i)
        for (int k = 0; k < c->tables[t].dim; ++k) cols.push_back(c->gcol[t] + k);
    for (int64_t r = 0; r < R; ++r)
      for (int64_t k = 0; k < Wi; ++k) dst[r * Wi + k] = global[r * c->W_total + cols[k]];
  }
}

int sp_set_grad(sp_ctx* ctx, const float* grad) {
  return guarded([&] {
    check_ctx(ctx);
    const int64_t R = rows_per_dst(ctx);
    const int64_t n = ctx->n_dst * R * ctx->W_total;
    std::vector<float> grouped(n);
    for (int j = 0; j < ctx->n_dst; ++j)
      global_to_grouped(ctx, grad + j * R * ctx->W_total, grouped.data() + j * R * ctx->W_total, R);
    SP_CUDA(cudaMemcpyAsync(ctx->d_gin, grouped.data(), n * sizeof(float),
                            cudaMemcpyHostToDevice, ctx->stream));
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sp_synth_grad(sp_ctx* ctx, uint64_t seed) {
  return guarded([&] {
    check_ctx(ctx);
    const int64_t R = rows_per_dst(ctx);
    // colmap of every source device (all ranks know the placement)
    std::vector<std::vector<int32_t>> cm(ctx->D);
    for (int t = 0; t < ctx->M; ++t)
      for (int k = 0; k < ctx->tables[t].dim; ++k)
        cm[ctx->placement[t]].push_back(static_cast<int32_t>(ctx->gcol[t] + k));
    std::vector<void*> tmp;
    uint64_t dummy = 0;
    for (int j = 0; j < ctx->n_dst; ++j) {
      const int dst = ctx->world == 1 ? j : ctx->rank;
      for (int i = 0; i < ctx->D; ++i) {
        if (cm[i].empty()) continue;
        int32_t* d_cm = dalloc<int32_t>(cm[i].size(), tmp, dummy);
        SP_CUDA(cudaMemcpy(d_cm, cm[i].data(), cm[i].size() * 4, cudaMemcpyHostToDevice));
        launch_synth_grad(ctx->d_gin + j * R * ctx->W_total + R * ctx->cumW[i], R,
                          static_cast<int64_t>(dst) * R, d_cm, ctx->dev_W[i], seed,
                          ctx->stream);
      }
    }
    // one process per rank: also the owner-side gradient [B, W_rank] the
    // backward exchange would deliver, so the backward can run (and be
    // timed) on a rank without its peers
    if (ctx->world > 1) {
      VDev& v = ctx->vdevs[0];
      if (v.W > 0)
        launch_synth_grad(v.d_grad, ctx->B, 0, v.d_colmap, v.W, seed, ctx->stream);
    }
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
    for (void* p : tmp) cudaFree(p);
  });
}

int sp_get_pooled(sp_ctx* ctx, float* pooled) {
  return guarded([&] {
    check_ctx(ctx);
    const int64_t R = rows_per_dst(ctx);
    const int64_t n = ctx->n_dst * R * ctx->W_total;
    std::vector<float> grouped(n);
    SP_CUDA(cudaMemcpyAsync(grouped.data(), ctx->d_recv, n * sizeof(float),
                            cudaMemcpyDeviceToHost, ctx->stream));
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int j = 0; j < ctx->n_dst; ++j)
      grouped_to_global(ctx, grouped.data() + j * R * ctx->W_total, pooled + j * R * ctx->W_total, R);
  });
}

int sp_get_local_pooled(sp_ctx* ctx, int32_t dev, float* pooled) {
  return guarded([&] {
    check_ctx(ctx);
    if (ctx->peer)
      raise(SP_ERR_BAD_INPUT, "peer memory: K1 stores the pooled rows at their receivers "
                              "(read them with sp_get_pooled on each rank)");
    VDev& v = vdev_for(ctx, dev);
    SP_CUDA(cudaMemcpyAsync(pooled, v.d_pooled, static_cast<int64_t>(ctx->B) * v.W * sizeof(float),
                            cudaMemcpyDeviceToHost, ctx->stream));
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sp_get_sorted(sp_ctx* ctx, int32_t dev, uint32_t* keys, uint32_t* bags,
                  int64_t* n_keys, uint32_t* seg_heads, int64_t* n_unique) {
  return guarded([&] {
    check_ctx(ctx);
    require_batch(ctx);
    VDev& v = vdev_for(ctx, dev);
    std::vector<uint32_t> k = sorted_keys_host(ctx, v, bags);
    int64_t nseg = 0;
    for (int64_t p = 0; p < static_cast<int64_t>(k.size()); ++p)
      if (p == 0 || k[p] != k[p - 1]) {
        if (seg_heads) seg_heads[nseg] = static_cast<uint32_t>(p);
        ++nseg;
      }
    if (keys) std::copy(k.begin(), k.end(), keys);
    if (n_keys) *n_keys = v.nnz;
    if (n_unique) *n_unique = nseg;
  });
}

}  // extern "C"

namespace sp {
namespace {
// Stages 2-4 with their events: exchanges (a barrier first so a rank's
// exchange time is not its wait for the slowest rank's compute), then the
// backward (joining the overlapped sort when ov). abort_flag: see launch_sgd.
void timed_exchange_and_backward(sp_ctx* c, bool ov, const int32_t* abort_flag) {
  cudaStream_t st = c->stream;
  if (exchange_needed(c)) {
    if (multi_rank(c)) {
      require_device_sync(c);
      barrier(c);
      SP_CUDA(cudaEventRecord(c->ev_a2a[0], st));
      a2a_fwd_rank(c);  // peer memory: already done by K1 (the barrier is its completion)
      SP_CUDA(cudaEventRecord(c->ev_a2a[1], st));
      barrier(c);
      SP_CUDA(cudaEventRecord(c->ev_a2a[2], st));
      a2a_bwd_rank(c);
      if (c->peer) barrier(c);
      SP_CUDA(cudaEventRecord(c->ev_a2a[3], st));
    } else {
      for (auto& v : c->vdevs) {
        SP_CUDA(cudaEventRecord(v.ev[2], st));
        a2a_fwd_emulated(c, v);
        SP_CUDA(cudaEventRecord(v.ev[3], st));
      }
      for (auto& v : c->vdevs) {
        SP_CUDA(cudaEventRecord(v.ev[4], st));
        a2a_bwd_emulated(c, v);
        SP_CUDA(cudaEventRecord(v.ev[5], st));
      }
    }
  }
  for (auto& v : c->vdevs) {
    SP_CUDA(cudaEventRecord(v.ev[6], st));
    if (ov) join_sort(c);
    stage_backward(c, v, ov, abort_flag);
    SP_CUDA(cudaEventRecord(v.ev[7], st));
  }
}

// Per-stage device times of the iteration just synchronised (events ev[0..7]
// of every (virtual) device, ev_a2a in NCCL mode), gathered over ranks and
// composed like CostOracle::evaluate_placement (oracle.hpp:222-227).
// The B200 counterpart of device_comm (oracle.hpp:178-185) for one GPU
// emulating D: a MODEL, not a measurement. One direction of the
// all-to-all moves, per device, 4 B W_d (D-1)/D bytes out and
// 4 (B/D) (W_tot - W_d) bytes in over full-duplex NVLink 5 through
// NVSwitch (every peer at full rate), so the device's stage time is the
// larger of the two at the measured per-direction peer bandwidth of this
// pool's B200s (770 GB/s, B200_PROFILING.md; 900 nominal) plus a fixed
// grouped send/recv latency. width_total < 0: the send side only (a device's
// own tables alone, as device_comm and partial_cost_features use it).
double comm_model_ms(int64_t B, int64_t width_dev, int64_t width_total, int D) {
  if (D <= 1 || width_dev <= 0) return 0.0;
  const double sent = 4.0 * B * width_dev * (D - 1) / D;
  const double recv = width_total < 0 ? 0.0 : 4.0 * (B / D) * (width_total - width_dev);
  return SP_A2A_LATENCY_MS + std::max(sent, recv) / (SP_NVLINK_PEER_GBS * 1e6);
}

void collect_breakdown(sp_ctx* c, sp_breakdown* out) {
  const int D = c->D;
  cudaStream_t st = c->stream;
  std::vector<double> fwd(D, 0.0), bwd(D, 0.0), cf(D, 0.0), cb(D, 0.0);
  for (auto& v : c->vdevs) {
    fwd[v.vid] = elapsed(v.ev[0], v.ev[1]);
    bwd[v.vid] = elapsed(v.ev[6], v.ev[7]);
    if (exchange_needed(c)) {
      if (multi_rank(c)) {
        cf[v.vid] = elapsed(c->ev_a2a[0], c->ev_a2a[1]);
        cb[v.vid] = elapsed(c->ev_a2a[2], c->ev_a2a[3]);
      } else if (c->comm_model) {
        cf[v.vid] = cb[v.vid] = comm_model_ms(c->B, v.W, c->W_total, D);
      } else {
        cf[v.vid] = elapsed(v.ev[2], v.ev[3]);
        cb[v.vid] = elapsed(v.ev[4], v.ev[5]);
      }
    }
  }
  if (nccl_mode(c)) {
    // gather every rank's four numbers
    double mine[4] = {fwd[c->rank], bwd[c->rank], cf[c->rank], cb[c->rank]};
    SP_CUDA(cudaMemcpyAsync(c->d_bd + 4 * c->rank, mine, sizeof(mine), cudaMemcpyHostToDevice, st));
    SP_NCCL(nccl().AllGather(c->d_bd + 4 * c->rank, c->d_bd, 4, ncclFloat64, c->comm, st));
    std::vector<double> all(4 * D);
    SP_CUDA(cudaMemcpyAsync(all.data(), c->d_bd, all.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    for (int d = 0; d < D; ++d) {
      fwd[d] = all[4 * d];
      bwd[d] = all[4 * d + 1];
      cf[d] = all[4 * d + 2];
      cb[d] = all[4 * d + 3];
    }
  }
  // composition of oracle.hpp:222-227
  const double max_fwd = *std::max_element(fwd.begin(), fwd.end());
  const double max_bwd = *std::max_element(bwd.begin(), bwd.end());
  const double fstage = *std::max_element(cf.begin(), cf.end());
  const double bstage = *std::max_element(cb.begin(), cb.end());
  if (out) {
    for (int d = 0; d < D; ++d) {
      if (out->fwd_ms) out->fwd_ms[d] = fwd[d];
      if (out->bwd_ms) out->bwd_ms[d] = bwd[d];
      if (out->comm_ms) out->comm_ms[d] = cb[d];
    }
    out->fwd_comm_stage_ms = fstage;
    out->bwd_comm_stage_ms = bstage;
    out->overall_ms = max_fwd + fstage + bstage + max_bwd;
  }
}
}  // namespace
}  // namespace sp

extern "C" {

// This context's compute of one iteration with the exchanges left out: the
// forward stage (K1), the backward stage (join + SGD on the resident
// gradient) and the sort (forked after K1 as in sp_run_iteration; with no
// exchange to run under, the backward stage waits for it). One rank of a
// multi-GPU placement can be measured alone this way (no NCCL id or peers
// needed).
int sp_run_local(sp_ctx* ctx, double ms[3]) {
  return guarded([&] {
    check_ctx(ctx);
    require_batch(ctx);
    if (!ms) raise(SP_ERR_BAD_INPUT, "null output");
    sp_ctx* c = ctx;
    cudaStream_t st = c->stream;
    VDev& v0 = c->vdevs[0];
    const bool ov = overlap_active(c);
    SP_CUDA(cudaEventRecord(v0.ev[0], st));
    forward_stage(c, ov);
    SP_CUDA(cudaEventRecord(v0.ev[1], st));
    if (ov) join_sort(c);
    for (auto& v : c->vdevs) stage_backward(c, v, ov);
    SP_CUDA(cudaEventRecord(v0.ev[7], st));
    SP_CUDA(cudaStreamSynchronize(st));
    if (c->side) SP_CUDA(cudaStreamSynchronize(c->side));
    ms[2] = ov ? elapsed(c->ev_sort[0], c->ev_sort[1]) : 0.0;
    ms[0] = elapsed(v0.ev[0], v0.ev[1]);
    ms[1] = elapsed(v0.ev[1], v0.ev[7]);
  });
}

int sp_run_iteration(sp_ctx* ctx, sp_breakdown* out) {
  return guarded([&] {
    check_ctx(ctx);
    require_batch(ctx);
    sp_ctx* c = ctx;
    cudaStream_t st = c->stream;
    // the input-only backward sort overlaps stages 1-3 (its tail, if any,
    // lands in the bwd stage, which starts by joining it)
    const bool ov = overlap_active(c);
    if (ov) {
      SP_CUDA(cudaEventRecord(c->vdevs[0].ev[0], st));
      forward_stage(c, ov);
      SP_CUDA(cudaEventRecord(c->vdevs[0].ev[1], st));
    } else {
      // stage 1: fwd compute per (virtual) device
      for (auto& v : c->vdevs) {
        SP_CUDA(cudaEventRecord(v.ev[0], st));
        stage_forward(c, v);
        SP_CUDA(cudaEventRecord(v.ev[1], st));
      }
    }
    timed_exchange_and_backward(c, ov, nullptr);
    SP_CUDA(cudaStreamSynchronize(st));
    collect_breakdown(c, out);
  });
}

}  // extern "C"

namespace sp {
namespace {

// One host-buffer step, enqueued: upload (slot, flag) pipelined with K1 per
// chunk and each chunk's backward sort, then stages 2-4 with the SGD
// guarded by the step's validation flag. Events ev[0..7] time its stages.
void enqueue_batch_step(sp_ctx* c, const int64_t* offsets, const int64_t* indices,
                        int32_t* flag, int slot, bool pipelined = false) {
  finish_batch(c, slot, pipelined);  // layout of this batch (sort positions, SGD tiles)
  c->has_batch = false;
  cudaStream_t st = c->stream;
  const bool ov = overlap_active(c);
  // a device's forward stage starts at its first chunk's K1 (after that
  // chunk's upload), so in emulation no device is charged for the uploads
  // and kernels of the devices before it
  for (auto& v : c->vdevs)
    if (v.tables.empty()) SP_CUDA(cudaEventRecord(v.ev[0], st));
  enqueue_upload(
      c, offsets, indices,
      [&](VDev& v, int t0, int t1) {
        const int64_t k0 = v.tile_start[t0], k1 = v.tile_start[t1];
        if (t0 == 0) SP_CUDA(cudaEventRecord(v.ev[0], st));
        {
          ProfScope prof(c, kProfFwd);
          launch_tbe_forward(v.d_meta_canon, v.d_tiles_canon + k0, k1 - k0, c->B, v.d_off,
                             v.d_idx, c->d_w, c->wt, v.d_pooled, c->d_rowmap, v.W, st);
        }
        const bool last = t1 == static_cast<int>(v.tables.size());
        if (last) SP_CUDA(cudaEventRecord(v.ev[1], st));
        if (ov) {
          // the chunk's CSR is on the device: sort its tables on the side stream
          SP_CUDA(cudaEventRecord(c->ev_fork, st));
          SP_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
          sort_range(c, v, t0, t1, c->side);
          if (last) SP_CUDA(cudaEventRecord(c->ev_join, c->side));
        }
      },
      flag, slot);
  for (auto& v : c->vdevs)
    if (v.tables.empty()) SP_CUDA(cudaEventRecord(v.ev[1], st));
  timed_exchange_and_backward(c, ov, flag);
  SP_CUDA(cudaEventRecord(c->slot_done[slot], st));
  c->slot_done_used[slot] = true;
}

}  // namespace
}  // namespace sp

extern "C" {

// The reference-facing step with host buffers: the LookupBatch's H2D is
// pipelined with the forward (K1 runs on each uploaded chunk of tables while
// the next chunk is in flight) and, with one (virtual) device, with the
// backward sort of every uploaded chunk; the device-side validation
// (offsets monotone inside a table, indices in range) is checked at the end
// and, if it failed, the SGD never touched the tables (device-side abort
// flag) and the call raises like sp_upload_batch.
int sp_run_batch(sp_ctx* ctx, const int64_t* offsets, int64_t offsets_len,
                 const int64_t* indices, int64_t indices_len, sp_breakdown* out) {
  return guarded([&] {
    check_ctx(ctx);
    sp_ctx* c = ctx;
    host_validate_and_size(c, offsets, offsets_len, indices_len);
    enqueue_batch_step(c, offsets, indices, c->d_flag, 0);
    int32_t flag = 0;
    SP_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            c->stream));
    SP_CUDA(cudaStreamSynchronize(c->stream));
    raise_batch_flag(flag);
    c->has_batch = true;
    collect_breakdown(c, out);
  });
}

// n consecutive host-buffer steps (a training segment fed by a data
// loader): step s's H2D (staging slot s % 2) overlaps step s-1's compute;
// K1 of step s still runs after step s-1's SGD (stream order), so every step
// sees the tables its predecessor updated. step_ms[s] (may be null): device
// time from the end of step s-1 (for s = 0: the start of its upload) to the
// end of step s. Every step's validation flag is checked at the end: an
// invalid step skipped its update and the call raises for the first one.
int sp_run_batches(sp_ctx* ctx, int32_t n, const int64_t* const* offsets,
                   const int64_t* offsets_len, const int64_t* const* indices,
                   const int64_t* indices_len, double* step_ms) {
  return guarded([&] {
    check_ctx(ctx);
    sp_ctx* c = ctx;
    if (n < 1 || offsets == nullptr || indices == nullptr || offsets_len == nullptr ||
        indices_len == nullptr)
      raise(SP_ERR_BAD_INPUT, "sp_run_batches needs n >= 1 batches");
    if (n > c->step_flags_cap) {
      SP_CUDA(cudaStreamSynchronize(c->stream));
      if (c->d_step_flags) cudaFree(c->d_step_flags);
      SP_CUDA(cudaMalloc(&c->d_step_flags, n * sizeof(int32_t)));
      c->step_flags_cap = n;
    }
    std::vector<cudaEvent_t> ev(n + 1);
    for (auto& e : ev) SP_CUDA(cudaEventCreate(&e));
    try {
      for (int s = 0; s < n; ++s) {
        host_validate_and_size(c, offsets[s], offsets_len[s], indices_len[s], true);
        if (s == 0) SP_CUDA(cudaEventRecord(ev[0], c->copy_stream));
        enqueue_batch_step(c, offsets[s], indices[s], c->d_step_flags + s, s & 1, s > 0);
        SP_CUDA(cudaEventRecord(ev[s + 1], c->stream));
      }
      std::vector<int32_t> flags(n);
      SP_CUDA(cudaMemcpyAsync(flags.data(), c->d_step_flags, n * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, c->stream));
      SP_CUDA(cudaStreamSynchronize(c->stream));
      if (step_ms)
        for (int s = 0; s < n; ++s) step_ms[s] = elapsed(ev[s], ev[s + 1]);
      for (auto& e : ev) cudaEventDestroy(e);
      ev.clear();
      for (int s = 0; s < n; ++s)
        if (flags[s]) {
          try {
            raise_batch_flag(flags[s]);
          } catch (const Status& e) {
            raise(e.code, "step " + std::to_string(s) + ": " + e.what());
          }
        }
      c->has_batch = true;
    } catch (...) {
      for (auto& e : ev) cudaEventDestroy(e);
      throw;
    }
  });
}

int sp_enqueue_iteration(sp_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    require_batch(ctx);
    enqueue_iteration(ctx);
  });
}

int sp_graph_replay(sp_ctx* ctx, int32_t iters, int32_t* kernels_per_iter) {
  return guarded([&] {
    check_ctx(ctx);
    require_batch(ctx);
    sp_ctx* c = ctx;
    if (!c->graph_exec) {
      cudaGraph_t g = nullptr;
      SP_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue_iteration(c);
      } catch (...) {
        cudaStreamEndCapture(c->stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      SP_CUDA(cudaStreamEndCapture(c->stream, &g));
      size_t n = 0;
      SP_CUDA(cudaGraphGetNodes(g, nullptr, &n));
      std::vector<cudaGraphNode_t> nodes(n);
      if (n) SP_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
      int k = 0;
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        SP_CUDA(cudaGraphNodeGetType(nd, &ty));
        if (ty == cudaGraphNodeTypeKernel) ++k;
      }
      c->graph_kernels = k;
      SP_CUDA(cudaGraphInstantiate(&c->graph_exec, g, 0));
      SP_CUDA(cudaGraphDestroy(g));
    }
    for (int i = 0; i < iters; ++i) {
      SP_CUDA(cudaGraphLaunch(c->graph_exec, c->stream));
      count_launch(c->graph_kernels);
    }
    if (kernels_per_iter) *kernels_per_iter = c->graph_kernels;
  });
}

int sp_exchange_plan(const sp_table_spec* tables, int32_t num_tables, int32_t num_devices,
                     const int32_t* placement, int32_t batch_size, int32_t rank,
                     int64_t* send_off, int64_t* send_count, int64_t* recv_off,
                     int64_t* recv_count, int32_t* colmap) {
  return guarded([&] {
    if (num_devices < 1 || rank < 0 || rank >= num_devices)
      raise(SP_ERR_BAD_INPUT, "rank/num_devices out of range");
    if (batch_size % num_devices != 0)
      raise(SP_ERR_SHAPE_MISMATCH, "batch_size must be divisible by num_devices");
    for (int i = 0; i < num_tables; ++i)
      if (placement[i] < 0 || placement[i] >= num_devices)
        raise(SP_ERR_BAD_INPUT, "device id out of range");
    const ExchangePlan p = make_plan(tables, num_tables, num_devices, placement, batch_size, rank);
    for (int j = 0; j < num_devices; ++j) {
      send_off[j] = p.send_off[j];
      send_count[j] = p.send_cnt[j];
      recv_off[j] = p.recv_off[j];
      recv_count[j] = p.recv_cnt[j];
    }
    if (colmap) std::copy(p.colmap.begin(), p.colmap.end(), colmap);
  });
}

int sp_ctx_set_comm_model(sp_ctx* ctx, int32_t on) {
  return guarded([&] {
    check_ctx(ctx);
    if (on && multi_rank(ctx))
      raise(SP_ERR_BAD_INPUT, "one process per GPU measures its exchange; the model is for "
                              "one GPU emulating D devices");
    ctx->comm_model = on != 0;
  });
}

int sp_comm_model(int32_t batch, int64_t width_dev, int64_t width_total, int32_t D,
                  double* ms) {
  return guarded([&] {
    if (!ms || batch < 1 || D < 1 || width_dev < 0) raise(SP_ERR_BAD_INPUT, "bad comm model args");
    *ms = comm_model_ms(batch, width_dev, width_total, D);
  });
}

int sp_ctx_set_overlap(sp_ctx* ctx, int32_t on) {
  return guarded([&] {
    check_ctx(ctx);
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
    SP_CUDA(cudaStreamSynchronize(ctx->side));
    ctx->overlap_sort = on != 0;
    if (ctx->graph_exec) {
      cudaGraphExecDestroy(ctx->graph_exec);
      ctx->graph_exec = nullptr;
    }
  });
}

int sp_ctx_set_sort_target(sp_ctx* ctx, int64_t lookups) {
  return guarded([&] {
    check_ctx(ctx);
    if (lookups < 0) raise(SP_ERR_BAD_INPUT, "sort target must be >= 0");
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
    SP_CUDA(cudaStreamSynchronize(ctx->side));
    ctx->sort_target = lookups;
    for (auto& v : ctx->vdevs) plan_sort(ctx, v);
    if (ctx->graph_exec) {
      cudaGraphExecDestroy(ctx->graph_exec);
      ctx->graph_exec = nullptr;
    }
  });
}

int sp_ctx_set_upload_chunk(sp_ctx* ctx, int64_t indices) {
  return guarded([&] {
    check_ctx(ctx);
    if (indices < 1) raise(SP_ERR_BAD_INPUT, "upload chunk must be >= 1 index");
    ctx->upload_chunk = indices;
  });
}

int sp_ctx_set_profiling(sp_ctx* ctx, int32_t on) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->profiling = on != 0;
  });
}

int sp_ctx_kernel_ms(sp_ctx* ctx, double ms[5], int64_t counts[5]) {
  return guarded([&] {
    check_ctx(ctx);
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < 5; ++k) {
      ms[k] = 0.0;
      if (counts) counts[k] = 0;
    }
    for (const auto& mk : ctx->marks) {
      ms[mk.cls] += elapsed(ctx->ev_pool[mk.a], ctx->ev_pool[mk.b]);
      if (counts) ++counts[mk.cls];
    }
    ctx->marks.clear();
    ctx->ev_used = 0;
  });
}

int sp_ctx_algorithmic_bytes(sp_ctx* ctx, double out[5]) {
  return guarded([&] {
    check_ctx(ctx);
    require_batch(ctx);
    sp_ctx* c = ctx;
    // Max over the (virtual) devices held here; SURVEY §8d formulas, 4-byte
    // ids, per launch of each kernel as this build runs it:
    //  [0] K1: offsets + ids + gathered rows + pooled out
    //  [1] exchange sent per direction
    //  [2] K4b SGD kernel: gradient 4*B*W + touched rows read+write
    //      8*sum_unique dim (2 B/param tables: 4*) + the sorted pairs it reads
    //  [3] K4a sort: ids read twice (8 B/lookup), packed pairs written and
    //      read (4 B each, 8 B when wide), sorted key + bag written, offsets
    //      read twice, count matrix written, scanned (read + write) and read
    //  [4] K1's unique-row floor: [0] with every touched row read once (the
    //      DRAM bytes K1 would move if L2 kept every reused row)
    // (row bytes use the storage type: 2 B/param for fp16 tables)
    double fwd = 0, a2a = 0, sgd = 0, sort = 0, fwd_u = 0;
    const double eb = elem_bytes(c->wt);
    for (auto& v : c->vdevs) {
      const int T = static_cast<int>(v.tables.size());
      double rows_bytes = 0;
      for (int li = 0; li < T; ++li)
        rows_bytes += eb * static_cast<double>(v.table_nnz[li]) * c->tables[v.tables[li]].dim;
      const double offs = 4.0 * (static_cast<double>(T) * c->B + 1);
      const double csr = offs + 4.0 * v.nnz;
      const double outb = 4.0 * c->B * v.W;
      const double pair = c->bags16 ? 6.0 : 8.0;  // sorted key + bag payload bytes
      const double mid = static_cast<double>(sort_mid_bytes(v.splan));
      fwd = std::max(fwd, csr + rows_bytes + outb);
      a2a = std::max(a2a, 4.0 * c->B * v.W * (c->D - 1) / c->D);
      double uniq_dim = 0;
      {
        const std::vector<uint32_t> keys = sorted_keys_host(c, v, nullptr);
        std::vector<uint64_t> row_end;  // device-wide end row of each local table
        for (const TableMeta& m : v.meta_canon) row_end.push_back(m.rowbase + m.rows);
        for (size_t p = 0; p < keys.size(); ++p)
          if (p == 0 || keys[p] != keys[p - 1]) {
            const int li = static_cast<int>(
                std::upper_bound(row_end.begin(), row_end.end(), keys[p]) - row_end.begin());
            uniq_dim += c->tables[v.tables[li]].dim;
          }
      }
      sgd = std::max(sgd, outb + 2.0 * eb * uniq_dim + pair * v.nnz);
      fwd_u = std::max(fwd_u, csr + eb * uniq_dim + outb);
      const double sort_dev = 2.0 * csr + 2.0 * mid * v.nnz + pair * v.nnz +
                              4.0 * 4.0 * static_cast<double>(v.splan.n_cnt);
      sort = std::max(sort, sort_dev);
    }
    out[0] = fwd;
    out[1] = a2a;
    out[2] = sgd;
    out[3] = sort;
    out[4] = fwd_u;
  });
}

}  // extern "C"

extern "C" int sp_synth_lookup_batch(const sp_table_spec* tables, int32_t num_tables,
                                     int32_t batch_size, uint64_t seed,
                                     int32_t cuda_device, int64_t* offsets,
                                     int64_t* indices, int64_t* nnz) {
  return guarded([&] {
    if (num_tables < 0 || batch_size < 1 || offsets == nullptr)
      raise(SP_ERR_BAD_INPUT, "bad batch shape");
    SP_CUDA(cudaSetDevice(cuda_device));
    const int T = num_tables;
    const int64_t nb = static_cast<int64_t>(T) * batch_size;
    std::vector<int32_t> gid(T);
    std::vector<int64_t> lmax(T), rows(T);
    std::vector<uint64_t> thr(T);
    for (int i = 0; i < T; ++i) {
      const auto& t = tables[i];
      gid[i] = t.id;
      lmax[i] = static_cast<int64_t>(std::floor(2.0 * t.pooling_factor));
      rows[i] = t.hash_size;
      double h = 0.0;
      for (int b = 4; b < SP_NUM_BINS; ++b) h += t.dist[b];
      thr[i] = hot_threshold(h);
    }
    cudaStream_t st = nullptr;
    SP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<void*> tmp;
    uint64_t dummy = 0;
    auto cleanup = [&] {
      cudaStreamSynchronize(st);
      for (void* p : tmp) cudaFree(p);
      cudaStreamDestroy(st);
    };
    try {
      int32_t* d_gid = dalloc<int32_t>(T, tmp, dummy);
      int64_t* d_lmax = dalloc<int64_t>(T, tmp, dummy);
      int64_t* d_rows = dalloc<int64_t>(T, tmp, dummy);
      uint64_t* d_thr = dalloc<uint64_t>(T, tmp, dummy);
      int32_t* d_len = dalloc<int32_t>(nb + 1, tmp, dummy);
      int32_t* d_off = dalloc<int32_t>(nb + 1, tmp, dummy);
      const size_t tb = exclusive_scan_i32(nullptr, 0, d_len, d_off, nb + 1, st);
      void* d_scan = dalloc<uint8_t>(tb, tmp, dummy);
      if (T) {
        SP_CUDA(cudaMemcpy(d_gid, gid.data(), T * 4, cudaMemcpyHostToDevice));
        SP_CUDA(cudaMemcpy(d_lmax, lmax.data(), T * 8, cudaMemcpyHostToDevice));
        SP_CUDA(cudaMemcpy(d_rows, rows.data(), T * 8, cudaMemcpyHostToDevice));
        SP_CUDA(cudaMemcpy(d_thr, thr.data(), T * 8, cudaMemcpyHostToDevice));
      }
      SP_CUDA(cudaMemsetAsync(d_len + nb, 0, 4, st));
      if (T) launch_synth_lengths(d_gid, d_lmax, T, batch_size, seed, d_len, st);
      exclusive_scan_i32(d_scan, tb, d_len, d_off, nb + 1, st);
      std::vector<int32_t> off32(nb + 1);
      SP_CUDA(cudaMemcpyAsync(off32.data(), d_off, (nb + 1) * 4, cudaMemcpyDeviceToHost, st));
      SP_CUDA(cudaStreamSynchronize(st));
      for (int64_t k = 0; k <= nb; ++k) offsets[k] = off32[k];
      const int64_t total = off32[nb];
      if (nnz) *nnz = total;
      if (indices && total) {
        int32_t* d_idx = dalloc<int32_t>(total, tmp, dummy);
        launch_synth_indices(d_gid, d_rows, d_thr, T, batch_size, seed, d_off, d_idx, st);
        std::vector<int32_t> idx32(total);
        SP_CUDA(cudaMemcpyAsync(idx32.data(), d_idx, total * 4, cudaMemcpyDeviceToHost, st));
        SP_CUDA(cudaStreamSynchronize(st));
        for (int64_t p = 0; p < total; ++p) indices[p] = idx32[p];
      }
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}
