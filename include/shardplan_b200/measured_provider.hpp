// measured_provider.hpp — header-only C++ host side over the C-ABI
// (shardplan_b200.h), shaped as the reference's own plugin interface.
//
// Build against the reference (a maintainer adding B200 measurement to
// shardplan) with -DSHARDPLAN_B200_WITH_REFERENCE and the reference include
// path: every type below is then the reference's own (shardplan::TableDesc,
// PlacementTask, Placement, CostBreakdown, CostProvider, Error), and
// MeasuredCostProvider drops into PlacementEnv (mdp.hpp:73-186) exactly
// where OracleCostProvider (mdp.hpp:37-54) sits. Without the macro the same
// names are defined here as field-for-field mirrors.
//
//   shardplan::CostProvider::cost_features / overall ... mdp.hpp:28-34
//   CostOracle::evaluate_placement -> measure_placement  oracle.hpp:187-240
//   CostOracle::partial_cost_features -> cost_features   oracle.hpp:244-269
//   Error / ErrorKind / exit codes ..................... error.hpp:11-49
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "shardplan_b200.h"

#if defined(SHARDPLAN_B200_WITH_REFERENCE)
#include "shardplan/mdp.hpp"
#else
#include <stdexcept>
#endif

namespace shardplan_b200 {

#if defined(SHARDPLAN_B200_WITH_REFERENCE)
using shardplan::CostBreakdown;
using shardplan::CostProvider;
using shardplan::Error;
using shardplan::ErrorKind;
using shardplan::Phase;
using shardplan::Placement;
using shardplan::PlacementTask;
using shardplan::TableDesc;
using shardplan::TraceEvent;
#else
// Mirrors of the reference types (error.hpp, table.hpp, oracle.hpp, mdp.hpp).
enum class ErrorKind {
  infeasible, memory_violation, malformed_batch, bad_spec, unknown_table,
  too_large, illegal_action, shape_mismatch, no_legal_action, bad_input,
};
class Error : public std::runtime_error {
 public:
  Error(ErrorKind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
  ErrorKind kind() const noexcept { return kind_; }
  int exit_code() const noexcept {
    return kind_ == ErrorKind::infeasible || kind_ == ErrorKind::memory_violation ? 2 : 3;
  }

 private:
  ErrorKind kind_;
};
struct TableDesc {
  int id = 0;
  int dim = 1;
  std::int64_t hash_size = 1;
  double pooling_factor = 0.0;
  double table_size_gb = 0.0;
  std::array<double, SP_NUM_BINS> dist{};
};
struct PlacementTask {
  std::vector<TableDesc> tables;
  int num_devices = 1;
  double mem_cap_gb = 0.0;
  int batch_size = 65536;
};
using Placement = std::vector<int>;
enum class Phase { fwd_comp, fwd_comm, bwd_comm, bwd_comp };
struct TraceEvent {
  int device = 0;
  Phase phase = Phase::fwd_comp;
  double start_ms = 0.0;
  double dur_ms = 0.0;
};
struct CostBreakdown {
  std::vector<double> fwd_ms, bwd_ms, comm_ms;
  double fwd_comm_stage_ms = 0.0;
  double bwd_comm_stage_ms = 0.0;
  double overall_ms = 0.0;
  std::vector<TraceEvent> events;
};
class CostProvider {
 public:
  virtual ~CostProvider() = default;
  virtual std::vector<std::array<double, 3>> cost_features(
      const std::vector<std::vector<int>>& assignment) = 0;
  virtual double overall(const Placement& placement) = 0;
};
#endif

// C-ABI status -> the reference's exception (ErrorKind + 1; device
// failures surface as bad_input with the CUDA/NCCL message).
inline void check(int status) {
  if (status == SP_OK) return;
  const std::string msg = sp_last_error();
  if (status >= SP_ERR_INFEASIBLE && status <= SP_ERR_BAD_INPUT)
    throw Error(static_cast<ErrorKind>(status - 1), msg);
  throw Error(ErrorKind::bad_input, (status == SP_ERR_NCCL ? "nccl: " : "cuda: ") + msg);
}

inline sp_table_spec to_spec(const TableDesc& t) {
  sp_table_spec s{};
  s.id = t.id;
  s.dim = t.dim;
  s.hash_size = t.hash_size;
  s.pooling_factor = t.pooling_factor;
  s.table_size_gb = t.table_size_gb;
  for (int b = 0; b < SP_NUM_BINS; ++b) s.dist[b] = t.dist[b];
  return s;
}

struct MeasureOptions {
  std::uint64_t seed = 2210;  // synthetic batch / weights / gradients
  int warmup = 2;
  int iters = 5;              // median of these
  float lr = 0.01f;
  int cuda_device = 0;
  // one GPU emulating D devices: comm terms from the NVLink 5 model
  // (sp_comm_model) instead of the device-local copy's time
  bool comm_model = true;
};

// One (emulated, world 1) shard of a placement on this GPU; RAII over sp_ctx.
class Shard {
 public:
  Shard(const PlacementTask& task, const Placement& placement, const MeasureOptions& o)
      : D_(task.num_devices) {
    if (sp_abi_version() != SP_ABI_VERSION)
      throw Error(ErrorKind::bad_input, "libshardplan_b200 ABI " +
                                            std::to_string(sp_abi_version()) +
                                            " does not match this header's " +
                                            std::to_string(SP_ABI_VERSION));
    std::vector<sp_table_spec> specs;
    for (const TableDesc& t : task.tables) specs.push_back(to_spec(t));
    std::vector<int32_t> p(placement.begin(), placement.end());
    if (p.size() != specs.size())
      throw Error(ErrorKind::bad_input, "placement length != table count");
    check(sp_ctx_create(specs.data(), static_cast<int32_t>(specs.size()), D_, p.data(),
                        task.batch_size, task.mem_cap_gb, o.lr, 0, 1, nullptr, o.cuda_device,
                        &ctx_));
    check(sp_ctx_set_comm_model(ctx_, o.comm_model ? 1 : 0));
  }
  ~Shard() { sp_ctx_destroy(ctx_); }
  Shard(const Shard&) = delete;
  Shard& operator=(const Shard&) = delete;

  sp_ctx* get() { return ctx_; }

  // One measured iteration in the reference's CostBreakdown shape, events
  // laid out as oracle.hpp:229-238.
  CostBreakdown run_iteration() {
    CostBreakdown cb;
    cb.fwd_ms.assign(D_, 0.0);
    cb.bwd_ms.assign(D_, 0.0);
    cb.comm_ms.assign(D_, 0.0);
    sp_breakdown b{cb.fwd_ms.data(), cb.bwd_ms.data(), cb.comm_ms.data(), 0, 0, 0};
    check(sp_run_iteration(ctx_, &b));
    cb.fwd_comm_stage_ms = b.fwd_comm_stage_ms;
    cb.bwd_comm_stage_ms = b.bwd_comm_stage_ms;
    cb.overall_ms = b.overall_ms;
    const double t1 = *std::max_element(cb.fwd_ms.begin(), cb.fwd_ms.end());
    const double t2 = t1 + cb.fwd_comm_stage_ms;
    const double t3 = t2 + cb.bwd_comm_stage_ms;
    for (int d = 0; d < D_; ++d) {
      cb.events.push_back({d, Phase::fwd_comp, 0.0, cb.fwd_ms[d]});
      cb.events.push_back({d, Phase::fwd_comm, t1, cb.comm_ms[d]});
      cb.events.push_back({d, Phase::bwd_comm, t2, cb.comm_ms[d]});
      cb.events.push_back({d, Phase::bwd_comp, t3, cb.bwd_ms[d]});
    }
    return cb;
  }

 private:
  int D_;
  sp_ctx* ctx_ = nullptr;
};

// evaluate_placement measured on the GPU: the synthetic batch of the task's
// descriptors through K1/exchange/K4, median of o.iters iterations.
inline CostBreakdown measure_placement(const PlacementTask& task, const Placement& placement,
                                       const MeasureOptions& o = {}) {
  Shard s(task, placement, o);
  check(sp_init_tables(s.get(), o.seed));
  check(sp_synth_batch(s.get(), o.seed));
  check(sp_synth_grad(s.get(), o.seed));
  std::vector<CostBreakdown> runs;
  for (int i = 0; i < o.warmup + o.iters; ++i) {
    CostBreakdown cb = s.run_iteration();
    if (i >= o.warmup) runs.push_back(std::move(cb));
  }
  std::sort(runs.begin(), runs.end(), [](const CostBreakdown& a, const CostBreakdown& b) {
    return a.overall_ms < b.overall_ms;
  });
  return runs[runs.size() / 2];
}

// Drop-in for OracleCostProvider (mdp.hpp:37-54): the environment talks to
// it through CostProvider only. Non-owning reference to the task, like the
// reference's providers (mdp.hpp:52-53).
class MeasuredCostProvider : public CostProvider {
 public:
  explicit MeasuredCostProvider(const PlacementTask& task, MeasureOptions o = {})
      : task_(task), o_(o) {}

  // Per device (fwd_ms, bwd_ms, comm_ms) of a partial assignment; a device
  // with no tables reports (0, 0, 0) (oracle.hpp:242-269). The memory cap is
  // enforced like check_memory (memory_violation).
  std::vector<std::array<double, 3>> cost_features(
      const std::vector<std::vector<int>>& assignment) override {
    ++calls_;
    const int D = task_.num_devices;
    if (assignment.size() != static_cast<std::size_t>(D))
      throw Error(ErrorKind::bad_input, "assignment has wrong device count");
    PlacementTask sub;
    sub.num_devices = D;
    sub.mem_cap_gb = task_.mem_cap_gb;
    sub.batch_size = task_.batch_size;
    Placement p;
    for (int d = 0; d < D; ++d)
      for (int id : assignment[d]) {
        if (id < 0 || static_cast<std::size_t>(id) >= task_.tables.size())
          throw Error(ErrorKind::unknown_table, "table id " + std::to_string(id));
        // the table keeps its id: the synthetic data is keyed by it
        sub.tables.push_back(task_.tables[id]);
        p.push_back(d);
      }
    std::vector<std::array<double, 3>> q(D, {0.0, 0.0, 0.0});
    if (sub.tables.empty()) return q;
    const CostBreakdown cb = measure_placement(sub, p, o_);
    for (int d = 0; d < D; ++d) {
      if (assignment[d].empty()) continue;
      double comm = cb.comm_ms[d];
      if (o_.comm_model) {  // the send side of the device's own tables
        int64_t w = 0;
        for (int id : assignment[d]) w += task_.tables[id].dim;
        check(sp_comm_model(task_.batch_size, w, -1, D, &comm));
      }
      q[d] = {cb.fwd_ms[d], cb.bwd_ms[d], comm};
    }
    return q;
  }

  double overall(const Placement& placement) override {
    ++calls_;
    return measure_placement(task_, placement, o_).overall_ms;
  }

  std::uint64_t calls() const { return calls_; }

 private:
  const PlacementTask& task_;
  MeasureOptions o_;
  std::uint64_t calls_ = 0;
};

}  // namespace shardplan_b200
