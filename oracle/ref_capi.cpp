// ref_capi.cpp — extern "C" face of the UNMODIFIED reference headers
// (/root/reference/proj/include/shardplan), compiled from where they lie by
// oracle/Makefile into oracle/_ref/libshardplan_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ (and the golden-fixture
// generator) to pin the oracle and the CUDA evaluator against the
// reference's own fp64 code. Nothing here is product code and no reference
// source is copied: every function below only calls reference symbols.
//
// The one non-reference line is the vector<bool> shim:
// policy.hpp:145,246 pass std::vector<bool> to
// softmax_masked(span<const double>, span<const bool>) (nn.hpp:207-208),
// a hard error under g++ 13. The overload below forwards to the reference.

#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "shardplan/nn.hpp"

namespace shardplan {
inline std::vector<double> softmax_masked(std::span<const double> logits,
                                          const std::vector<bool>& mask) {
  std::unique_ptr<bool[]> m(new bool[mask.size()]);
  for (std::size_t i = 0; i < mask.size(); ++i) m[i] = mask[i];
  return softmax_masked(logits, std::span<const bool>(m.get(), mask.size()));
}
}  // namespace shardplan

#include "shardplan/baselines.hpp"
#include "shardplan/checkpoint.hpp"
#include "shardplan/config.hpp"
#include "shardplan/costnet.hpp"
#include "shardplan/harness.hpp"
#include "shardplan/mdp.hpp"
#include "shardplan/oracle.hpp"
#include "shardplan/policy.hpp"
#include "shardplan/synth.hpp"
#include "shardplan/table.hpp"

#include "shardplan_b200.h"

using namespace shardplan;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.kind()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SP_ERR_BAD_INPUT;
  }
}

TableDesc to_desc(const sp_table_spec& s) {
  TableDesc t;
  t.id = s.id;
  t.dim = s.dim;
  t.hash_size = s.hash_size;
  t.pooling_factor = s.pooling_factor;
  t.table_size_gb = s.table_size_gb;
  for (int b = 0; b < kNumBins; ++b) t.dist[b] = s.dist[b];
  return t;
}

sp_table_spec to_spec(const TableDesc& t) {
  sp_table_spec s{};
  s.id = t.id;
  s.dim = t.dim;
  s.hash_size = t.hash_size;
  s.pooling_factor = t.pooling_factor;
  s.table_size_gb = t.table_size_gb;
  for (int b = 0; b < kNumBins; ++b) s.dist[b] = t.dist[b];
  return s;
}

PlacementTask make_task(const sp_table_spec* tables, int M, int D, double cap,
                        int B) {
  PlacementTask task;
  task.num_devices = D;
  task.mem_cap_gb = cap;
  task.batch_size = B;
  for (int i = 0; i < M; ++i) task.tables.push_back(to_desc(tables[i]));
  return task;
}

void write_stats(const FeatureStats& st, double* mean, double* stdv) {
  for (int f = 0; f < kNumFeatures; ++f) {
    if (mean) mean[f] = st[f].mean;
    if (stdv) stdv[f] = st[f].std;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- table.hpp ----------------------------------------------------------

int ref_access_count_bin(int64_t c) { return access_count_bin(c); }

double ref_table_memory_gb(int64_t hash_size, int dim, int bytes) {
  return table_memory_gb(hash_size, dim, bytes);
}

int ref_feature_vector(const sp_table_spec* t, const double* mean,
                       const double* stdv, double* out21) {
  return guarded([&] {
    FeatureStats st{};
    const FeatureStats* p = nullptr;
    if (mean) {
      for (int f = 0; f < kNumFeatures; ++f) st[f] = {mean[f], stdv[f]};
      p = &st;
    }
    const FeatureVec v = feature_vector(to_desc(*t), p);
    for (int f = 0; f < kNumFeatures; ++f) out21[f] = v[f];
  });
}

int ref_ingest(const int64_t* offsets, int64_t offsets_len,
               const int64_t* indices, int64_t indices_len, int T, int B,
               const int32_t* dims, const int64_t* hash_sizes, int bytes,
               sp_table_spec* out, double* stats_mean, double* stats_std) {
  return guarded([&] {
    LookupBatch b;
    b.num_tables = T;
    b.batch_size = B;
    b.offsets.assign(offsets, offsets + offsets_len);
    b.indices.assign(indices, indices + indices_len);
    std::vector<int> d(dims, dims + T);
    std::vector<std::int64_t> h(hash_sizes, hash_sizes + T);
    const TablePool pool = ingest_lookup_batch(b, d, h, bytes);
    for (int t = 0; t < T; ++t) out[t] = to_spec(pool.tables[t]);
    write_stats(pool.feature_stats, stats_mean, stats_std);
  });
}

int ref_validate_batch(const int64_t* offsets, int64_t offsets_len,
                       int64_t indices_len, int T, int B) {
  return guarded([&] {
    LookupBatch b;
    b.num_tables = T;
    b.batch_size = B;
    b.offsets.assign(offsets, offsets + offsets_len);
    b.indices.assign(static_cast<std::size_t>(indices_len), 0);
    validate_batch(b);
  });
}

// save_lookup_batch / load_lookup_batch (table.hpp:268-305), the DSLB file.
int ref_save_lookup_batch(const char* path, const int64_t* offsets, int64_t offsets_len,
                          const int64_t* indices, int64_t indices_len, int T, int B) {
  return guarded([&] {
    LookupBatch b;
    b.num_tables = T;
    b.batch_size = B;
    b.offsets.assign(offsets, offsets + offsets_len);
    b.indices.assign(indices, indices + indices_len);
    save_lookup_batch(b, path);
  });
}

// Loads `path`; writes the counts, and the arrays when the capacities
// (*offsets_len / *indices_len on entry) suffice.
int ref_load_lookup_batch(const char* path, int64_t* offsets, int64_t* offsets_len,
                          int64_t* indices, int64_t* indices_len, int* T, int* B) {
  return guarded([&] {
    const LookupBatch b = load_lookup_batch(path);
    const bool fits = offsets && indices &&
                      *offsets_len >= static_cast<int64_t>(b.offsets.size()) &&
                      *indices_len >= static_cast<int64_t>(b.indices.size());
    if (fits) {
      std::copy(b.offsets.begin(), b.offsets.end(), offsets);
      std::copy(b.indices.begin(), b.indices.end(), indices);
    }
    *offsets_len = static_cast<int64_t>(b.offsets.size());
    *indices_len = static_cast<int64_t>(b.indices.size());
    *T = b.num_tables;
    *B = b.batch_size;
  });
}

// ---- synth.hpp ----------------------------------------------------------

int ref_synth_pool(int num_tables, const int32_t* dims, const double* weights,
                   int n_dims, double hash_lo, double hash_hi,
                   double pooling_exponent, double pooling_max, double hot_lo,
                   double hot_hi, int batch, int bytes, uint64_t seed,
                   sp_table_spec* out, double* stats_mean, double* stats_std) {
  return guarded([&] {
    SynthSpec s;
    s.num_tables = num_tables;
    s.dim_choices.clear();
    for (int i = 0; i < n_dims; ++i) s.dim_choices.emplace_back(dims[i], weights[i]);
    s.hash_log10_lo = hash_lo;
    s.hash_log10_hi = hash_hi;
    s.pooling_exponent = pooling_exponent;
    s.pooling_max = pooling_max;
    s.hot_fraction_lo = hot_lo;
    s.hot_fraction_hi = hot_hi;
    s.batch_size = batch;
    s.bytes_per_param = bytes;
    const TablePool pool = synth_pool(s, seed);
    for (int i = 0; i < num_tables; ++i) out[i] = to_spec(pool.tables[i]);
    write_stats(pool.feature_stats, stats_mean, stats_std);
  });
}

int ref_compute_feature_stats(const sp_table_spec* tables, int M,
                              double* stats_mean, double* stats_std) {
  return guarded([&] {
    std::vector<TableDesc> v;
    for (int i = 0; i < M; ++i) v.push_back(to_desc(tables[i]));
    write_stats(compute_feature_stats(v), stats_mean, stats_std);
  });
}

// ---- oracle.hpp ---------------------------------------------------------

int ref_evaluate_placement(const sp_table_spec* tables, int M, int D,
                           double cap, int B, const int32_t* placement,
                           double* fwd, double* bwd, double* comm,
                           double* stage, double* overall) {
  return guarded([&] {
    const PlacementTask task = make_task(tables, M, D, cap, B);
    const CostOracle oracle;
    const CostBreakdown cb =
        oracle.evaluate_placement(task, Placement(placement, placement + M));
    for (int d = 0; d < D; ++d) {
      fwd[d] = cb.fwd_ms[d];
      bwd[d] = cb.bwd_ms[d];
      comm[d] = cb.comm_ms[d];
    }
    *stage = cb.fwd_comm_stage_ms;
    *overall = cb.overall_ms;
  });
}

double ref_device_comm(double dim_sum, int D, int B) {
  return CostOracle().device_comm(dim_sum, D, B);
}

double ref_fusion_speedup(int k) { return CostOracle().fusion_speedup(k); }

// ---- baselines.hpp ------------------------------------------------------

int ref_expert_placement(const sp_table_spec* tables, int M, int D,
                         double cap, int B, int strategy, int32_t* out) {
  return guarded([&] {
    const PlacementTask task = make_task(tables, M, D, cap, B);
    const Placement p =
        expert_placement(task, static_cast<ExpertStrategy>(strategy));
    for (int i = 0; i < M; ++i) out[i] = p[i];
  });
}

int ref_random_placement(const sp_table_spec* tables, int M, int D,
                         double cap, int B, uint64_t seed, int32_t* out) {
  return guarded([&] {
    const PlacementTask task = make_task(tables, M, D, cap, B);
    Rng rng(seed);
    const Placement p = random_placement(task, rng);
    for (int i = 0; i < M; ++i) out[i] = p[i];
  });
}

// ---- rng.hpp ------------------------------------------------------------

void ref_rng_u01(uint64_t seed, int64_t n, double* out) {
  Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.u01();
}

uint64_t ref_subseed(uint64_t seed, const char* stream) {
  return subseed(seed, stream);
}

void ref_rng_index(uint64_t seed, int64_t n, int64_t bound, int64_t* out) {
  Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = static_cast<int64_t>(rng.index(bound));
}

// ---- costnet.hpp training (checker of csrc/train.cu) ---------------------

namespace {
struct CostSetup {
  CostNet net;
  std::shared_ptr<const TaskFeatures> feats;
  std::vector<CostSample> samples;
};

CostSetup cost_setup(const double* params, int red_tables, int red_devices, int table_relu,
                     const double* mask, const double* features, int64_t n_rows, int n,
                     const int32_t* dev_off, const int32_t* tab_off, const int32_t* tab_row,
                     const double* target_q, const double* target_ov) {
  CostSetup c;
  FeatureMask fm = full_feature_mask();
  if (mask)
    for (int f = 0; f < kNumFeatures; ++f) fm[f] = mask[f] != 0.0;
  c.net = CostNet::make(0, static_cast<Reduction>(red_tables), static_cast<Reduction>(red_devices),
                        fm, table_relu != 0);
  std::vector<double> pv(params, params + c.net.param_count());
  c.net.set_param_vector(pv);
  auto tf = std::make_shared<TaskFeatures>();
  for (int64_t r = 0; r < n_rows; ++r) {
    FeatureVec v{};
    for (int f = 0; f < kNumFeatures; ++f) v[f] = features[r * kNumFeatures + f];
    tf->rows.push_back(v);
  }
  c.feats = tf;
  for (int s = 0; s < n; ++s) {
    CostSample cs;
    cs.features = c.feats;
    for (int d = dev_off[s]; d < dev_off[s + 1]; ++d) {
      cs.device_tables.emplace_back(tab_row + tab_off[d], tab_row + tab_off[d + 1]);
      cs.target_q.push_back({target_q[3 * d], target_q[3 * d + 1], target_q[3 * d + 2]});
    }
    if (target_ov && !std::isnan(target_ov[s])) cs.target_overall = target_ov[s];
    c.samples.push_back(std::move(cs));
  }
  return c;
}
}  // namespace

int ref_costnet_loss_grad(const double* params, int red_tables, int red_devices, int table_relu,
                          const double* mask, const double* features, int64_t n_rows, int n,
                          const int32_t* dev_off, const int32_t* tab_off, const int32_t* tab_row,
                          const double* target_q, const double* target_ov, double* grad,
                          double* loss) {
  return guarded([&] {
    CostSetup c = cost_setup(params, red_tables, red_devices, table_relu, mask, features,
                             n_rows, n, dev_off, tab_off, tab_row, target_q, target_ov);
    std::vector<const CostSample*> batch;
    for (const CostSample& s : c.samples) batch.push_back(&s);
    std::vector<double> g;
    *loss = costnet_loss_and_grad(c.net, batch, g);
    std::copy(g.begin(), g.end(), grad);
  });
}

// costnet_train_steps (costnet.hpp:431-446) over the samples as the replay
// buffer, minibatches drawn by Rng(seed); params updated in place.
int ref_costnet_train_steps(double* params, int red_tables, int red_devices, int table_relu,
                            const double* mask, const double* features, int64_t n_rows, int n,
                            const int32_t* dev_off, const int32_t* tab_off,
                            const int32_t* tab_row, const double* target_q,
                            const double* target_ov, int n_steps, int n_batch, double lr,
                            int64_t total_steps, uint64_t seed, double* mean_loss) {
  return guarded([&] {
    CostSetup c = cost_setup(params, red_tables, red_devices, table_relu, mask, features,
                             n_rows, n, dev_off, tab_off, tab_row, target_q, target_ov);
    ReplayBuffer buf;
    for (CostSample& s : c.samples) buf.add(std::move(s));
    AdamState adam(c.net.param_count(), lr, total_steps);
    Rng rng(seed);
    *mean_loss = costnet_train_steps(c.net, buf, n_steps, n_batch, adam, rng);
    const std::vector<double> pv = c.net.param_vector();
    std::copy(pv.begin(), pv.end(), params);
  });
}

namespace {
struct PolicySetup {
  PolicyNet net;
  std::vector<Episode> episodes;
};

PolicySetup policy_setup(const double* params, const double* mask, const double* features,
                         int n, const int32_t* row0, const int32_t* ntab,
                         const int32_t* step_off, const double* reward,
                         const int32_t* dev_off, const int32_t* action,
                         const int32_t* tab_off, const int32_t* tab_id, const int32_t* legal,
                         const double* q) {
  PolicySetup c;
  FeatureMask fm = full_feature_mask();
  if (mask)
    for (int f = 0; f < kNumFeatures; ++f) fm[f] = mask[f] != 0.0;
  c.net = PolicyNet::make(0, fm);
  std::vector<double> pv(params, params + c.net.param_count());
  c.net.set_param_vector(pv);
  for (int e = 0; e < n; ++e) {
    auto tf = std::make_shared<TaskFeatures>();
    for (int r = 0; r < ntab[e]; ++r) {
      FeatureVec v{};
      for (int f = 0; f < kNumFeatures; ++f)
        v[f] = features[(static_cast<int64_t>(row0[e]) + r) * kNumFeatures + f];
      tf->rows.push_back(v);
    }
    Episode ep;
    ep.features = tf;
    ep.reward = reward[e];
    for (int st = step_off[e]; st < step_off[e + 1]; ++st) {
      EpisodeStep es;
      for (int d = dev_off[st]; d < dev_off[st + 1]; ++d) {
        es.device_tables.emplace_back(tab_id + tab_off[d], tab_id + tab_off[d + 1]);
        es.q.push_back({q[3 * d], q[3 * d + 1], q[3 * d + 2]});
        es.legal.push_back(legal[d] != 0);
      }
      es.action = action[st];
      ep.steps.push_back(std::move(es));
    }
    c.episodes.push_back(std::move(ep));
  }
  return c;
}
}  // namespace

int ref_reinforce_loss_grad(const double* params, const double* mask, const double* features,
                            int n, const int32_t* row0, const int32_t* ntab,
                            const int32_t* step_off, const double* reward,
                            const int32_t* dev_off, const int32_t* action,
                            const int32_t* tab_off, const int32_t* tab_id,
                            const int32_t* legal, const double* q, double w_entropy,
                            double* grad, double* objective) {
  return guarded([&] {
    PolicySetup c = policy_setup(params, mask, features, n, row0, ntab, step_off, reward,
                                 dev_off, action, tab_off, tab_id, legal, q);
    std::vector<double> g;
    *objective = reinforce_loss_and_grad(c.net, c.episodes, w_entropy, g);
    std::copy(g.begin(), g.end(), grad);
  });
}

// n_updates reinforce_update calls (policy.hpp:287-296) on the same
// episodes with one AdamState(lr, total_steps); params updated in place.
int ref_reinforce_updates(double* params, const double* mask, const double* features, int n,
                          const int32_t* row0, const int32_t* ntab, const int32_t* step_off,
                          const double* reward, const int32_t* dev_off, const int32_t* action,
                          const int32_t* tab_off, const int32_t* tab_id, const int32_t* legal,
                          const double* q, double w_entropy, int n_updates, double lr,
                          int64_t total_steps, double* objectives) {
  return guarded([&] {
    PolicySetup c = policy_setup(params, mask, features, n, row0, ntab, step_off, reward,
                                 dev_off, action, tab_off, tab_id, legal, q);
    AdamState adam(c.net.param_count(), lr, total_steps);
    for (int u = 0; u < n_updates; ++u)
      objectives[u] = reinforce_update(c.net, c.episodes, w_entropy, adam);
    const std::vector<double> pv = c.net.param_vector();
    std::copy(pv.begin(), pv.end(), params);
  });
}

// ---- harness.hpp / checkpoint.hpp ---------------------------------------

int ref_train(const sp_table_spec* pool_tables, int n_pool, int batch,
              int num_tables, int num_devices, double mem_cap_gb,
              int iterations, int n_collect, int n_cost, int n_batch,
              int n_rl, int n_episode, uint64_t seed, const char* ckpt_path) {
  return guarded([&] {
    TablePool pool;
    pool.batch_size = batch;
    for (int i = 0; i < n_pool; ++i) pool.tables.push_back(to_desc(pool_tables[i]));
    pool.feature_stats = compute_feature_stats(pool.tables);
    RunConfig cfg;
    cfg.num_tables = num_tables;
    cfg.num_devices = num_devices;
    cfg.mem_cap_gb = mem_cap_gb;
    cfg.iterations = iterations;
    cfg.n_collect = n_collect;
    cfg.n_cost = n_cost;
    cfg.n_batch = n_batch;
    cfg.n_rl = n_rl;
    cfg.n_episode = n_episode;
    cfg.seed = seed;
    cfg.n_train_tasks = 50;
    cfg.n_test_tasks = 50;
    const CostOracle oracle(cfg.oracle);
    const TrainResult r = train(cfg, pool, oracle, nullptr);
    save_checkpoint(r.checkpoint, ckpt_path);
  });
}

int ref_infer(const char* ckpt_path, const sp_table_spec* tables, int M, int D,
              double cap, int B, int32_t* placement, double* predicted,
              int32_t* order) {
  return guarded([&] {
    const Checkpoint ckpt = load_checkpoint(ckpt_path);
    const PlacementTask task = make_task(tables, M, D, cap, B);
    const InferResult r = infer(ckpt, task);
    for (int i = 0; i < M; ++i) placement[i] = r.placement[i];
    *predicted = r.predicted_ms;
    if (order) {
      const TaskFeatures f = make_task_features(task.tables, &ckpt.stats);
      const std::vector<int> o = predicted_order(ckpt.cost, f);
      for (int i = 0; i < M; ++i) order[i] = o[i];
    }
  });
}

// Sampled rollouts exactly as estimated_episode (harness.hpp:190-212) runs
// them: n episodes from ONE Rng(seed) stream, each consuming one u01 per
// step (policy.hpp:158). Placement and raw overall per episode.
int ref_sampled_rollouts(const char* ckpt_path, const sp_table_spec* tables,
                         int M, int D, double cap, int B, uint64_t seed, int n,
                         int32_t* placements, double* overall) {
  return guarded([&] {
    const Checkpoint ckpt = load_checkpoint(ckpt_path);
    const PlacementTask task = make_task(tables, M, D, cap, B);
    auto features = std::make_shared<const TaskFeatures>(
        make_task_features(task.tables, &ckpt.stats));
    const std::vector<int> order = predicted_order(ckpt.cost, *features);
    EstimatedCostProvider provider(ckpt.cost, *features, D);
    Rng rng(seed);
    for (int e = 0; e < n; ++e) {
      PlacementEnv env(task, order, provider, *features);
      double reward = 0.0;
      while (!env.done()) {
        const std::vector<bool> legal = env.legal_mask();
        const std::vector<double> probs =
            action_probs(ckpt.policy, env.state(), legal, *features);
        const auto [a, logp] = sample_action(probs, rng);
        (void)logp;
        const StepResult r = env.step(a);
        if (r.done) reward = r.reward;
      }
      const Placement& p = env.placement();
      for (int i = 0; i < M; ++i) placements[static_cast<std::size_t>(e) * M + i] = p[i];
      overall[e] = -reward;
    }
  });
}

// EstimatedCostProvider::overall for n placements, plus the clamped
// cost_features of the final sets (costnet.hpp:466-496).
int ref_costnet_overall(const char* ckpt_path, const sp_table_spec* tables,
                        int M, int D, const int32_t* placements, int n,
                        double* overall, double* q) {
  return guarded([&] {
    const Checkpoint ckpt = load_checkpoint(ckpt_path);
    std::vector<TableDesc> descs;
    for (int i = 0; i < M; ++i) descs.push_back(to_desc(tables[i]));
    const TaskFeatures f = make_task_features(descs, &ckpt.stats);
    EstimatedCostProvider provider(ckpt.cost, f, D);
    for (int c = 0; c < n; ++c) {
      const Placement p(placements + static_cast<std::size_t>(c) * M,
                        placements + static_cast<std::size_t>(c + 1) * M);
      overall[c] = provider.overall(p);
      if (q) {
        std::vector<std::vector<int>> sets(D);
        for (int i = 0; i < M; ++i) sets[p[i]].push_back(i);
        const auto qq = provider.cost_features(sets);
        for (int d = 0; d < D; ++d)
          for (int h = 0; h < 3; ++h)
            q[(static_cast<std::size_t>(c) * D + d) * 3 + h] = qq[d][h];
      }
    }
  });
}

// Normalised feature rows (make_task_features with the checkpoint stats)
// and the single-table predicted costs used by predicted_order.
int ref_task_features(const char* ckpt_path, const sp_table_spec* tables,
                      int M, double* rows21, double* single_cost) {
  return guarded([&] {
    const Checkpoint ckpt = load_checkpoint(ckpt_path);
    std::vector<TableDesc> descs;
    for (int i = 0; i < M; ++i) descs.push_back(to_desc(tables[i]));
    const TaskFeatures f = make_task_features(descs, &ckpt.stats);
    for (int i = 0; i < M; ++i) {
      for (int k = 0; k < kNumFeatures; ++k) rows21[i * kNumFeatures + k] = f.rows[i][k];
      if (single_cost) single_cost[i] = single_table_cost(ckpt.cost, i, f);
    }
  });
}

// Policy action probabilities for one augmented state (policy.hpp:137-146).
int ref_action_probs(const char* ckpt_path, const sp_table_spec* tables, int M,
                     int D, const int32_t* partial, const double* q,
                     const int32_t* legal, double* probs) {
  return guarded([&] {
    const Checkpoint ckpt = load_checkpoint(ckpt_path);
    std::vector<TableDesc> descs;
    for (int i = 0; i < M; ++i) descs.push_back(to_desc(tables[i]));
    const TaskFeatures f = make_task_features(descs, &ckpt.stats);
    std::vector<std::vector<int>> sets(D);
    for (int i = 0; i < M; ++i)
      if (partial[i] >= 0) sets[partial[i]].push_back(i);
    std::vector<std::array<double, 3>> qq(D);
    for (int d = 0; d < D; ++d) qq[d] = {q[d * 3], q[d * 3 + 1], q[d * 3 + 2]};
    std::vector<bool> lg(D);
    for (int d = 0; d < D; ++d) lg[d] = legal[d] != 0;
    const std::vector<double> p = action_probs(ckpt.policy, sets, qq, lg, f);
    for (int d = 0; d < D; ++d) probs[d] = p[d];
  });
}

}  // extern "C"
