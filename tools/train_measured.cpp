// train_measured — DreamShard trained on B200-measured costs (SURVEY §8f,
// first "next" row): the reference's training loop (harness.hpp:220-319)
// through shardplan_b200::train_on_provider with MeasuredCostProvider, so
// every cost sample of the collect phase is a measured iteration of the
// embedding stage on the GPU. Writes a reference checkpoint (checkpoint.hpp).
//
//   train_measured <pool.bin> <batch> <num_tables> <num_devices> <mem_cap_gb>
//                  <iterations> <out.dshd> [seed]
// pool.bin: raw sp_table_spec records (the C-ABI mirror of TableDesc).
//
// Built against the reference headers (-DSHARDPLAN_B200_WITH_REFERENCE) by
// __graft_entry__.build() where /root/reference exists.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <vector>

#include "shardplan/checkpoint.hpp"
#include "shardplan_b200/measured_training.hpp"

int main(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s pool.bin batch M D cap_gb iterations out.dshd [seed]\n",
                 argv[0]);
    return 3;
  }
  try {
    std::ifstream is(argv[1], std::ios::binary);
    std::vector<sp_table_spec> specs;
    sp_table_spec s{};
    while (is.read(reinterpret_cast<char*>(&s), sizeof(s))) specs.push_back(s);
    shardplan::TablePool pool;
    pool.batch_size = std::atoi(argv[2]);
    for (const sp_table_spec& t : specs) {
      shardplan::TableDesc d;
      d.id = t.id;
      d.dim = t.dim;
      d.hash_size = t.hash_size;
      d.pooling_factor = t.pooling_factor;
      d.table_size_gb = t.table_size_gb;
      for (int b = 0; b < SP_NUM_BINS; ++b) d.dist[b] = t.dist[b];
      pool.tables.push_back(d);
    }
    pool.feature_stats = shardplan::compute_feature_stats(pool.tables);
    shardplan::RunConfig cfg;
    cfg.num_tables = std::atoi(argv[3]);
    cfg.num_devices = std::atoi(argv[4]);
    cfg.mem_cap_gb = std::atof(argv[5]);
    cfg.iterations = std::atoi(argv[6]);
    if (argc > 8) cfg.seed = std::strtoull(argv[8], nullptr, 10);
    shardplan_b200::MeasureOptions o;
    o.warmup = 1;
    o.iters = 3;
    const shardplan::TrainResult r = shardplan_b200::train_on_provider(
        cfg, pool, shardplan_b200::measured_provider_factory(o), &std::cout);
    shardplan::save_checkpoint(r.checkpoint, argv[7]);
    std::printf("saved %s\n", argv[7]);
    return 0;
  } catch (const shardplan::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return e.exit_code();
  }
}
