// train_on_provider (include/shardplan_b200/measured_training.hpp), built
// against the reference headers.
//   oracle: with OracleCostProvider it must reproduce the reference's own
//           train() (harness.hpp:220-319) bit for bit — same metrics records,
//           same cost/policy parameters.
//   gpu:    with MeasuredCostProvider the collect phase runs on B200-measured
//           embedding costs (M + 1 measured iterations per episode).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>

#include "shardplan/synth.hpp"
#include "shardplan_b200/measured_training.hpp"

#define CHECK(c)                                                          \
  do {                                                                    \
    if (!(c)) {                                                           \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      return 1;                                                           \
    }                                                                     \
  } while (0)

static shardplan::RunConfig tiny_config() {
  shardplan::RunConfig cfg;
  cfg.num_tables = 6;
  cfg.num_devices = 2;
  cfg.mem_cap_gb = 8.0;
  cfg.n_train_tasks = 3;
  cfg.iterations = 2;
  cfg.n_collect = 2;
  cfg.n_cost = 20;
  cfg.n_batch = 8;
  cfg.n_rl = 2;
  cfg.n_episode = 3;
  cfg.seed = 11;
  return cfg;
}

static shardplan::TablePool tiny_pool(int batch) {
  shardplan::SynthSpec spec;
  spec.num_tables = 24;
  spec.dim_choices = {{16, 1.0}, {32, 1.0}, {64, 1.0}};
  spec.hash_log10_lo = 3.0;
  spec.hash_log10_hi = 4.0;
  spec.pooling_max = 20.0;
  spec.batch_size = batch;
  return shardplan::synth_pool(spec, 5);
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  const shardplan::RunConfig cfg = tiny_config();
  if (!gpu) {
    const shardplan::TablePool pool = tiny_pool(65536);
    const shardplan::CostOracle oracle(cfg.oracle);
    const shardplan::TrainResult ref = shardplan::train(cfg, pool, oracle);
    const shardplan::TrainResult mine = shardplan_b200::train_on_provider(
        cfg, pool, [&](const shardplan::PlacementTask& t) -> std::unique_ptr<shardplan::CostProvider> {
          return std::make_unique<shardplan::OracleCostProvider>(oracle, t);
        });
    CHECK(ref.metrics.size() == mine.metrics.size());
    for (size_t i = 0; i < ref.metrics.size(); ++i) CHECK(ref.metrics[i] == mine.metrics[i]);
    CHECK(ref.checkpoint.cost.param_vector() == mine.checkpoint.cost.param_vector());
    CHECK(ref.checkpoint.policy.table_mlp.params == mine.checkpoint.policy.table_mlp.params);
    CHECK(ref.checkpoint.policy.cost_mlp.params == mine.checkpoint.policy.cost_mlp.params);
    CHECK(ref.checkpoint.policy.head.params == mine.checkpoint.policy.head.params);
    std::printf("ok (oracle, %zu iterations identical)\n", ref.metrics.size());
    return 0;
  }
  const shardplan::TablePool pool = tiny_pool(512);
  shardplan_b200::MeasureOptions o;
  o.warmup = 1;
  o.iters = 2;
  std::uint64_t measured = 0;
  std::ostringstream log;
  const shardplan::TrainResult r = shardplan_b200::train_on_provider(
      cfg, pool,
      [&](const shardplan::PlacementTask& t) -> std::unique_ptr<shardplan::CostProvider> {
        struct Counting : shardplan_b200::MeasuredCostProvider {
          std::uint64_t* n;
          Counting(const shardplan::PlacementTask& t, shardplan_b200::MeasureOptions o,
                   std::uint64_t* n_)
              : MeasuredCostProvider(t, o), n(n_) {}
          std::vector<std::array<double, 3>> cost_features(
              const std::vector<std::vector<int>>& a) override {
            ++*n;
            return MeasuredCostProvider::cost_features(a);
          }
        };
        return std::make_unique<Counting>(t, o, &measured);
      },
      &log);
  CHECK(static_cast<int>(r.metrics.size()) == cfg.iterations);
  for (const auto& m : r.metrics) {
    const double c = m["mean_train_cost_ms"].get<double>();
    CHECK(std::isfinite(c) && c > 0.0);
    CHECK(std::isfinite(m["cost_loss"].get<double>()));
  }
  // every collected episode measured one cost vector per table
  CHECK(measured >= static_cast<std::uint64_t>(cfg.iterations * cfg.n_collect * cfg.num_tables));
  std::printf("%sok (gpu, %llu measured partial placements)\n", log.str().c_str(),
              static_cast<unsigned long long>(measured));
  return 0;
}
