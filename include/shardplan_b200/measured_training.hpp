// measured_training.hpp — DreamShard's training loop with the collect phase
// on B200-measured costs (first "next" row).
//
// The reference trains on a synthetic cost oracle: harness.hpp:156-186
// (detail::collect_episode) builds an OracleCostProvider (mdp.hpp:37-54) and
// harness.hpp:220-319 (train) only ever touches the oracle there. This header
// keeps every other piece the reference's own — task sampling, features,
// the cost-network fit (costnet_train_steps), the policy updates on the
// estimated MDP (estimated_episode + reinforce_update) and the checkpoint —
// and swaps the collect phase's provider for any shardplan::CostProvider,
// by default MeasuredCostProvider: every partial-placement cost q_d and every
// final overall cost is one measured iteration of the embedding stage on the
// GPU (M + 1 measurements per episode).
//
// Requires the reference headers: build with -DSHARDPLAN_B200_WITH_REFERENCE.
#pragma once

#if !defined(SHARDPLAN_B200_WITH_REFERENCE)
#error "measured_training.hpp composes the reference's training pieces: -DSHARDPLAN_B200_WITH_REFERENCE"
#endif

#include <functional>
#include <memory>
#include <ostream>
#include <vector>

#include "shardplan/harness.hpp"
#include "shardplan_b200/measured_provider.hpp"

namespace shardplan_b200 {

using ProviderFactory = std::function<std::unique_ptr<CostProvider>(const PlacementTask&)>;

// B200-measured costs for every task (MeasuredCostProvider, options `o`).
inline ProviderFactory measured_provider_factory(MeasureOptions o = {}) {
  return [o](const PlacementTask& task) -> std::unique_ptr<CostProvider> {
    return std::make_unique<MeasuredCostProvider>(task, o);
  };
}

// detail::collect_episode (harness.hpp:156-186) on `provider`: one sampled
// episode of the placement MDP, a cost sample per step (the state's q after
// the step) and a final sample carrying the overall cost.
inline shardplan::detail::CollectedEpisode collect_episode_on(
    const PlacementTask& task, const std::vector<int>& order, CostProvider& provider,
    const shardplan::PolicyNet& policy,
    const std::shared_ptr<const shardplan::TaskFeatures>& features, shardplan::Rng& rng) {
  shardplan::PlacementEnv env(task, order, provider, *features);
  shardplan::detail::CollectedEpisode ep;
  double reward = 0.0;
  auto sample_of = [&](bool last) {
    shardplan::CostSample s;
    s.features = features;
    s.device_tables = env.state().device_tables;
    s.target_q = env.state().q;
    if (last) s.target_overall = ep.overall_ms;
    return s;
  };
  while (!env.done()) {
    const std::vector<double> probs =
        shardplan::action_probs(policy, env.state(), env.legal_mask(), *features);
    const int action = shardplan::sample_action(probs, rng).first;
    const shardplan::StepResult r = env.step(action);
    ep.samples.push_back(sample_of(false));
    if (r.done) reward = r.reward;
  }
  ep.overall_ms = -reward;
  ep.samples.push_back(sample_of(true));
  return ep;
}

// train (harness.hpp:220-319) with the collect phase on make_provider's
// costs. Same seeds, sub-streams, replay buffer, Adam states and metrics
// records as the reference, so with a provider that reproduces the oracle it
// is the reference's run; with MeasuredCostProvider the cost network learns
// B200-measured embedding costs.
inline shardplan::TrainResult train_on_provider(const shardplan::RunConfig& cfg,
                                                const shardplan::TablePool& pool,
                                                const ProviderFactory& make_provider,
                                                std::ostream* metrics = nullptr) {
  using namespace shardplan;
  validate_config(cfg);
  const auto pools = split_pool(pool, subseed(cfg.seed, "split"));
  const FeatureStats stats = pools.first.feature_stats;
  const std::vector<PlacementTask> tasks =
      sample_tasks(pools.first, cfg.num_tables, cfg.n_train_tasks, cfg.num_devices,
                   cfg.mem_cap_gb, subseed(cfg.seed, "train_tasks"));
  std::vector<std::shared_ptr<const TaskFeatures>> feats;
  std::vector<std::unique_ptr<CostProvider>> providers;
  for (const PlacementTask& t : tasks) {
    feats.push_back(std::make_shared<const TaskFeatures>(make_task_features(t.tables, &stats)));
    providers.push_back(make_provider(t));
  }
  CostNet cost = CostNet::make(subseed(cfg.seed, "cost_init"), cfg.reduction_tables,
                               cfg.reduction_devices, cfg.feature_mask);
  PolicyNet policy = PolicyNet::make(subseed(cfg.seed, "policy_init"), cfg.feature_mask);
  const auto steps = [&](int per_iter) {
    return static_cast<std::int64_t>(cfg.iterations) * per_iter;
  };
  AdamState adam_cost(cost.param_count(), cfg.lr, steps(cfg.n_cost));
  AdamState adam_policy(policy.param_count(), cfg.lr, steps(cfg.n_rl));
  ReplayBuffer buffer;
  Rng rng_collect(subseed(cfg.seed, "collect"));
  Rng rng_cost(subseed(cfg.seed, "cost_batches"));
  Rng rng_rl(subseed(cfg.seed, "rl"));
  TrainResult result;
  bool fitted = false;

  // Runs body() until it does not raise `infeasible` (a task whose legal
  // actions ran out), at most 100 attempts, like the reference's loops.
  const auto retry = [](const char* what, const auto& body) {
    for (int attempt = 0; attempt < 100; ++attempt) {
      try {
        body();
        return;
      } catch (const Error& e) {
        if (e.kind() != ErrorKind::infeasible) throw;
      }
    }
    raise(ErrorKind::infeasible, std::string("could not ") + what + " in 100 attempts");
  };

  for (int iter = 1; iter <= cfg.iterations; ++iter) {
    double collected = 0.0;
    for (int c = 0; c < cfg.n_collect; ++c) {
      retry("collect a feasible episode", [&] {
        const std::size_t ti = rng_collect.index(tasks.size());
        const std::vector<int> order =
            fitted ? predicted_order(cost, *feats[ti]) : heuristic_order(tasks[ti]);
        detail::CollectedEpisode ep =
            collect_episode_on(tasks[ti], order, *providers[ti], policy, feats[ti], rng_collect);
        collected += ep.overall_ms;
        for (CostSample& s : ep.samples) buffer.add(std::move(s));
      });
    }
    const double loss =
        costnet_train_steps(cost, buffer, cfg.n_cost, cfg.n_batch, adam_cost, rng_cost);
    fitted = true;
    for (int u = 0; u < cfg.n_rl; ++u) {
      retry("run a feasible policy update", [&] {
        const std::size_t ti = rng_rl.index(tasks.size());
        const std::vector<int> order = predicted_order(cost, *feats[ti]);
        EstimatedCostProvider estimated(cost, *feats[ti], cfg.num_devices);
        std::vector<Episode> episodes;
        for (int e = 0; e < cfg.n_episode; ++e)
          episodes.push_back(
              detail::estimated_episode(tasks[ti], order, estimated, policy, feats[ti], rng_rl));
        reinforce_update(policy, episodes, cfg.w_entropy, adam_policy);
      });
    }
    nlohmann::json rec = {{"iteration", iter},
                          {"mean_train_cost_ms", collected / cfg.n_collect},
                          {"cost_loss", loss}};
    if (metrics) *metrics << rec.dump() << '\n';
    result.metrics.push_back(std::move(rec));
  }
  result.checkpoint.stats = stats;
  result.checkpoint.cost = std::move(cost);
  result.checkpoint.policy = std::move(policy);
  result.checkpoint.config = cfg;
  return result;
}

}  // namespace shardplan_b200
