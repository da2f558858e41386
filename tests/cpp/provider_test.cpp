// C++ host-side check of include/shardplan_b200/measured_provider.hpp.
// With -DSHARDPLAN_B200_WITH_REFERENCE it is compiled against the reference
// headers: MeasuredCostProvider must BE a shardplan::CostProvider and plug
// into shardplan::PlacementEnv (mdp.hpp:73-186). Argument "gpu" also runs
// measured queries on cuda:0.
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>

#include "shardplan_b200/measured_provider.hpp"

using namespace shardplan_b200;

#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      return 1;                                                    \
    }                                                              \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  static_assert(std::is_base_of_v<CostProvider, MeasuredCostProvider>);
  PlacementTask task;
  task.num_devices = 2;
  task.batch_size = 256;
  task.mem_cap_gb = 1.0;
  const int dims[3] = {16, 64, 128};
  for (int i = 0; i < 3; ++i) {
    TableDesc t;
    t.id = i;
    t.dim = dims[i];
    t.hash_size = 1000 + 500 * i;
    t.pooling_factor = 3.0 + i;
    t.table_size_gb = static_cast<double>(t.hash_size) * t.dim * 4 / (1024.0 * 1024.0 * 1024.0);
    t.dist[0] = 0.6;
    t.dist[12] = 0.4;
    task.tables.push_back(t);
  }
  // memory cap violation maps to the reference's Error{memory_violation}
  PlacementTask capped = task;
  capped.mem_cap_gb = task.tables[2].table_size_gb * 1.01;
  try {
    measure_placement(capped, {1, 1, 1});
    CHECK(false);
  } catch (const Error& e) {
    CHECK(e.kind() == ErrorKind::memory_violation);
    CHECK(e.exit_code() == 2);
  }
  try {
    MeasuredCostProvider p(task);
    p.cost_features({{0}});  // wrong device count
    CHECK(false);
  } catch (const Error& e) {
    CHECK(e.kind() == ErrorKind::bad_input);
  }
  MeasuredCostProvider provider(task);
#if defined(SHARDPLAN_B200_WITH_REFERENCE)
  const shardplan::TaskFeatures features = shardplan::make_task_features(task.tables, nullptr);
  shardplan::PlacementEnv env(task, {2, 1, 0}, provider, features);
  CHECK(!env.done());
#endif
  if (gpu) {
    const auto q = provider.cost_features({{0}, {1, 2}});
    CHECK(q.size() == 2);
    CHECK(q[0][0] > 0.0 && q[1][0] > 0.0 && q[1][1] > 0.0);
    const auto empty = provider.cost_features({{}, {0, 1, 2}});
    CHECK(empty[0][0] == 0.0 && empty[0][1] == 0.0 && empty[0][2] == 0.0);
    const CostBreakdown cb = measure_placement(task, {0, 1, 1});
    double mf = 0, mb = 0;
    for (double v : cb.fwd_ms) mf = v > mf ? v : mf;
    for (double v : cb.bwd_ms) mb = v > mb ? v : mb;
    CHECK(cb.overall_ms == mf + cb.fwd_comm_stage_ms + cb.bwd_comm_stage_ms + mb);
    CHECK(cb.events.size() == 8);
    CHECK(provider.overall({0, 1, 1}) > 0.0);
#if defined(SHARDPLAN_B200_WITH_REFERENCE)
    while (!env.done()) env.step(env.legal_actions()[0]);
#endif
  }
  std::printf("provider_test ok (%s)\n", gpu ? "gpu" : "cpu");
  return 0;
}
