/*
 * shardplan_b200.h — C-ABI of the B200-native embedding hot path that
 * DreamShard (arXiv 2210.02023) places and costs.
 *
 * The reference (`shardplan`, header-only C++20 under
 * /root/reference/proj/include/shardplan/) fakes GPU execution with a
 * closed-form cost oracle. This library executes the same four stages for
 * real on B200 GPUs and returns them in the reference's own shape:
 *
 *   fwd_comp  sum-pooled EmbeddingBag forward         (oracle.hpp:163-174)
 *   fwd_comm  all-to-all of pooled vectors             (oracle.hpp:178-185)
 *   bwd_comm  all-to-all of pooled-vector gradients    (oracle.hpp:178-185)
 *   bwd_comp  sort/segment sparse row-wise SGD         (oracle.hpp:149)
 *
 * composed exactly as CostOracle::evaluate_placement composes them
 * (oracle.hpp:222-227): overall = max fwd + fwd stage + bwd stage + max bwd.
 *
 * It also exports the batched on-GPU evaluator of DreamShard's cost network
 * (costnet.hpp) and policy network (policy.hpp) used by Alg. 2 `infer`
 * (harness.hpp:332-356) and by estimated-MDP rollouts.
 *
 * Conventions:
 *  - plain pointers and sizes only; HOST pointers unless a name says _dev;
 *  - every function returns an int status: 0 = ok, else ErrorKind + 1
 *    (error.hpp:11-22), plus SP_ERR_CUDA / SP_ERR_NCCL for device failures;
 *    the message is available from sp_last_error();
 *  - handles are opaque and owned by the caller; calls on one handle are not
 *    thread-safe, several handles may coexist (mdp.hpp:28-34 providers are
 *    single-threaded per environment).
 */
#ifndef SHARDPLAN_B200_H_
#define SHARDPLAN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 2
#define SP_NUM_BINS 17      /* table.hpp:26 kNumBins */
#define SP_NUM_FEATURES 21  /* table.hpp:28 kNumFeatures */
#define SP_NCCL_ID_BYTES 128
#define SP_IPC_BYTES 128    /* two cudaIpcMemHandle_t: receive + gradient buffers */

/* Status codes: ErrorKind (error.hpp:11-22) + 1. */
enum sp_status {
  SP_OK = 0,
  SP_ERR_INFEASIBLE = 1,
  SP_ERR_MEMORY_VIOLATION = 2,
  SP_ERR_MALFORMED_BATCH = 3,
  SP_ERR_BAD_SPEC = 4,
  SP_ERR_UNKNOWN_TABLE = 5,
  SP_ERR_TOO_LARGE = 6,
  SP_ERR_ILLEGAL_ACTION = 7,
  SP_ERR_SHAPE_MISMATCH = 8,
  SP_ERR_NO_LEGAL_ACTION = 9,
  SP_ERR_BAD_INPUT = 10,
  SP_ERR_CUDA = 11,
  SP_ERR_NCCL = 12
};

/* One embedding table; field-for-field shardplan::TableDesc
 * (table.hpp:45-52). `table_size_gb` uses the caller's bytes_per_param
 * (table.hpp:55-63); this library stores fp32 rows (4 B/param). */
typedef struct sp_table_spec {
  int32_t id;
  int32_t dim;
  int64_t hash_size;
  double pooling_factor;
  double table_size_gb;
  double dist[SP_NUM_BINS];
} sp_table_spec;

/* shardplan::CostBreakdown (oracle.hpp:105-116) without the trace events
 * (they are a pure function of these numbers, oracle.hpp:229-238). The
 * three per-device arrays are caller-owned and hold num_devices entries. */
typedef struct sp_breakdown {
  double* fwd_ms;
  double* bwd_ms;
  double* comm_ms; /* per-device all-to-all time (max of fwd/bwd exchange) */
  double fwd_comm_stage_ms;
  double bwd_comm_stage_ms;
  double overall_ms;
} sp_breakdown;

typedef struct sp_ctx sp_ctx;       /* one rank's shard of a placement */
typedef struct sp_evaluator sp_evaluator; /* cost/policy nets on one GPU */

/* ------------------------------------------------------------------ */
/* Library                                                              */

int sp_abi_version(void);
/* Message of the last failure on this thread (any handle). */
const char* sp_last_error(void);
/* Number of kernels this library has launched on this thread's handles
 * since load (CUB/NCCL internal launches excluded). */
uint64_t sp_kernel_launches(void);
/* Page-locked host buffers for the LookupBatch upload (cudaHostAlloc). */
int sp_host_alloc(uint64_t bytes, void** out);
void sp_host_free(void* p);

/* ------------------------------------------------------------------ */
/* Embedding shard context — replaces CostOracle::evaluate_placement
 * (oracle.hpp:187-240) with a measured iteration.                      */

/* NCCL unique id for a multi-rank context; rank 0 calls it and the caller
 * broadcasts the bytes (e.g. with torch.distributed). */
int sp_nccl_unique_id(uint8_t out_id[SP_NCCL_ID_BYTES]);

/* Creates rank `rank`'s shard of `placement` (length num_tables, entries in
 * [0, num_devices), oracle.hpp:75-76).
 *  - world_size == num_devices: one process per GPU, all-to-all over NCCL
 *    (nccl_id from sp_nccl_unique_id, NULL when num_devices == 1) or over
 *    peer memory (sp_ipc_import; nccl_id NULL = host-driven stages);
 *  - world_size == 1 < num_devices: emulation — all num_devices virtual
 *    devices live on this GPU and run back to back; their per-device
 *    compute is measured for real, the exchange is a device-local copy of
 *    the same layout (reported, not NVLink).
 * batch_size must be divisible by num_devices. Validates the
 * placement like evaluate_placement (oracle.hpp:190-204) against
 * mem_cap_gb. Divergence from check_memory (oracle.hpp:329-341), which
 * enforces mem > cap + 1e-9 for every cap: here mem_cap_gb <= 0 disables
 * the cap (an unbounded device), so tasks built with PlacementTask's default
 * cap of 0 are measurable; pass the task's real cap to get the reference's
 * memory_violation. */
int sp_ctx_create(const sp_table_spec* tables, int32_t num_tables,
                  int32_t num_devices, const int32_t* placement,
                  int32_t batch_size, double mem_cap_gb, float lr,
                  int32_t rank, int32_t world_size, const uint8_t* nccl_id,
                  int32_t cuda_device, sp_ctx** out);
/* sp_ctx_create with an explicit table storage type. SP_STORAGE_AUTO
 * (what sp_ctx_create does) follows the tables' sizing: 2 B/param -> fp16,
 * 4 B/param (or unsized) -> fp32. SP_STORAGE_BF16 stores 2 B/param tables
 * as bfloat16 (same bytes, fp32's exponent range). Pooled outputs,
 * gradients and every sum stay fp32; a sizing that disagrees with the type
 * is SP_ERR_BAD_INPUT. */
#define SP_STORAGE_AUTO 0
#define SP_STORAGE_F32 1
#define SP_STORAGE_F16 2
#define SP_STORAGE_BF16 3
int sp_ctx_create_ex(const sp_table_spec* tables, int32_t num_tables,
                     int32_t num_devices, const int32_t* placement,
                     int32_t batch_size, double mem_cap_gb, float lr,
                     int32_t rank, int32_t world_size, const uint8_t* nccl_id,
                     int32_t cuda_device, int32_t storage, sp_ctx** out);
void sp_ctx_destroy(sp_ctx* ctx);

/* cudaStream_t the context launches on (as void*). */
int sp_ctx_stream(sp_ctx* ctx, void** stream);
/* Bytes of device memory held by the context. */
int sp_ctx_device_bytes(sp_ctx* ctx, uint64_t* bytes);
/* Local (this rank's) table ids in ascending order; returns the count via
 * n_out; `ids` may be NULL to query the count. */
int sp_ctx_local_tables(sp_ctx* ctx, int32_t* ids, int32_t* n_out);

/* Table weights. Deterministic init w = 0.5 + 0.5*u(seed, table, row, col)
 * (SURVEY §8d), or explicit fp32 rows [hash_size, dim] row-major. The
 * generators (weights here, bags and indices in sp_synth_batch /
 * sp_synth_lookup_batch) are keyed by sp_table_spec.id, not by the table's
 * position in the context, so a table keeps its synthetic data in any
 * sub-task; the gradient generator is keyed by (bag, global column). */
int sp_init_tables(sp_ctx* ctx, uint64_t seed);
int sp_set_table(sp_ctx* ctx, int32_t table_id, const float* rows);
int sp_get_table(sp_ctx* ctx, int32_t table_id, float* rows);

/* Peer-memory exchange (one process per GPU on one NVLink/NVSwitch node, or
 * several processes sharing a GPU): every rank exports the CUDA IPC handles
 * of its receive and gradient buffers, the host all-gathers them (rank
 * order, world_size * SP_IPC_BYTES) and every rank imports them. From then on
 * K1 stores each batch slice's pooled rows straight into the receiving
 * rank's buffer (the forward all-to-all is fused into the lookup kernel:
 * stores to mapped peer addresses + a system-scope fence) and the backward
 * exchange pulls this rank's gradient slices from the peers. Replaces the
 * NCCL exchange of device_comm (oracle.hpp:178-185). With an NCCL id the
 * whole iteration stays on the device (NCCL barriers between the stages);
 * a context created without one (nccl_id = NULL, world_size > 1) is driven
 * stage by stage from the host: sp_forward; sp_ctx_synchronize + host rank
 * barrier; sp_a2a_backward; sp_ctx_synchronize + barrier; sp_backward_sgd. */
int sp_ipc_export(sp_ctx* ctx, uint8_t out[SP_IPC_BYTES]);
int sp_ipc_import(sp_ctx* ctx, const uint8_t* all_handles);
/* Wait for all work enqueued on the context's streams. */
int sp_ctx_synchronize(sp_ctx* ctx);

/* Lookup batch in the reference layout, shardplan::LookupBatch
 * (table.hpp:158-165): offsets[num_tables*B + 1], indices[offsets.back()],
 * ordered by (table_id, batch_offset). Host pointers. The local tables'
 * segments are copied to the device and narrowed to 32-bit; validated like
 * validate_batch (table.hpp:167-184) plus 0 <= index < hash_size. */
int sp_upload_batch(sp_ctx* ctx, const int64_t* offsets, int64_t offsets_len,
                    const int64_t* indices, int64_t indices_len);
/* A LookupBatch file written by the reference's save_lookup_batch
 * (table.hpp:268-281; "DSLB", u32 version 1, u32 num_tables, u32 batch_size,
 * u64 + i64 offsets[], u64 + i64 indices[], little-endian) loaded straight
 * to the device: replaces load_lookup_batch (table.hpp:283-305) followed by
 * sp_upload_batch. Only this context's tables' index segments are read;
 * they stream through pinned host slots into device staging. Errors:
 * SP_ERR_BAD_INPUT for an unreadable / non-DSLB / wrong-version / truncated
 * file (the reference's messages), SP_ERR_MALFORMED_BATCH for a batch
 * validate_batch rejects, SP_ERR_SHAPE_MISMATCH when num_tables/batch_size
 * differ from the context's, then the checks of sp_upload_batch. */
int sp_upload_batch_file(sp_ctx* ctx, const char* path);
/* Same batch, generated on the device by the SURVEY §8d generator. */
int sp_synth_batch(sp_ctx* ctx, uint64_t seed);
/* The same generator for a whole host LookupBatch of `tables` (run on the
 * GPU, copied back as int64): offsets[T*B+1]; indices may be NULL to only
 * get offsets and *nnz. Used to build host inputs for the e2e path. */
int sp_synth_lookup_batch(const sp_table_spec* tables, int32_t num_tables,
                          int32_t batch_size, uint64_t seed, int32_t cuda_device,
                          int64_t* offsets, int64_t* indices, int64_t* nnz);
/* Number of local lookup indices of the current batch. */
int sp_batch_nnz(sp_ctx* ctx, int64_t* nnz);

/* The forward all-to-all plan of `rank` (host only, no GPU needed): per
 * peer j the fp32 element offset/count sent from its pooled [B, W_rank]
 * (rows [j*B/D, (j+1)*B/D)) and received into the grouped layout
 * [B/D, W_total] (source-major), plus colmap[W_total]: grouped column ->
 * global column (tables in id order). The backward exchange is the mirror.
 * This is the exact plan the NCCL path executes. */
int sp_exchange_plan(const sp_table_spec* tables, int32_t num_tables,
                     int32_t num_devices, const int32_t* placement,
                     int32_t batch_size, int32_t rank, int64_t* send_off,
                     int64_t* send_count, int64_t* recv_off, int64_t* recv_count,
                     int32_t* colmap);

/* Stage entry points (asynchronous on the context stream). */
int sp_forward(sp_ctx* ctx);
int sp_a2a_forward(sp_ctx* ctx);
int sp_a2a_backward(sp_ctx* ctx);
int sp_backward_sgd(sp_ctx* ctx);

/* Gradient of this rank's pooled outputs, [B/num_devices, W_total] fp32
 * (W_total = sum of all dims, columns in global table-id order). With
 * emulation (world_size 1) the rank owns the whole batch [B, W_total]. */
int sp_set_grad(sp_ctx* ctx, const float* grad);
int sp_synth_grad(sp_ctx* ctx, uint64_t seed);
/* Pooled outputs after sp_a2a_forward, same layout as the gradient. */
int sp_get_pooled(sp_ctx* ctx, float* pooled);
/* Pooled outputs of (virtual) device `dev` before the exchange,
 * [B, W_dev] (W_dev = sum of dev's dims, its tables in ascending id order).
 * In NCCL mode dev must be this rank. */
int sp_get_local_pooled(sp_ctx* ctx, int32_t dev, float* pooled);

/* Backward internals for bit-exact checks: runs the key
 * build, the stable radix sort and the segment-head selection of (virtual)
 * device `dev` (this rank in NCCL mode) on the current batch and returns
 * the sorted keys (local row base + row, tables in ascending id order), the
 * bag payload, and the run heads (first position of each run). Pass NULL
 * arrays to query the sizes. */
int sp_get_sorted(sp_ctx* ctx, int32_t dev, uint32_t* keys, uint32_t* bags,
                  int64_t* n_keys, uint32_t* seg_heads, int64_t* n_unique);

/* One full measured iteration: fwd -> fwd a2a -> bwd a2a -> bwd SGD with
 * per-stage CUDA events; fills `out` like evaluate_placement
 * (oracle.hpp:206-227). Synchronizes the stream. In NCCL mode the per-device
 * arrays hold every rank's numbers (gathered), identical on all ranks. */
int sp_run_iteration(sp_ctx* ctx, sp_breakdown* out);
/* This context's compute of one iteration without the exchanges: ms[0] =
 * the forward stage (K1), ms[1] = the backward stage (SGD on the resident
 * gradient, after waiting for the sort), ms[2] = the backward sort alone
 * (side stream, forked after K1 as in sp_run_iteration, where it runs
 * under the exchanges; 0 when the overlap is off and the sort is inside
 * ms[1]). Measures one rank of a multi-GPU placement on its own (no NCCL id
 * or peers needed) — the compute part of that rank's CostBreakdown. */
int sp_run_local(sp_ctx* ctx, double ms[3]);
/* sp_upload_batch + sp_run_iteration in one call, pipelined: the H2D of the
 * host LookupBatch overlaps the forward of the tables already on the device
 * (and, with one device per context, their backward sort). The device-side
 * part of the validation is checked at the end: on failure the tables were
 * not updated, no batch is current, and the call returns the error
 * sp_upload_batch would. Stage times include the upload they overlap (fwd
 * runs from the first H2D to the last forward kernel). This is the
 * reference-facing step with host buffers (CostOracle::evaluate_placement,
 * oracle.hpp:187-240, over a real LookupBatch). */
int sp_run_batch(sp_ctx* ctx, const int64_t* offsets, int64_t offsets_len,
                 const int64_t* indices, int64_t indices_len, sp_breakdown* out);
/* n consecutive host-buffer steps (a training segment fed by a data loader;
 * batch s = offsets[s][offsets_len[s]], indices[s][indices_len[s]], host
 * buffers valid until the call returns): step s's H2D overlaps step s-1's
 * compute (two staging slots); step s's forward still follows step s-1's SGD.
 * step_ms[s] (may be NULL) = device time from the end of step s-1 (s = 0:
 * the start of its upload) to the end of step s. Raises for the first step
 * whose device-side validation failed (that step updated nothing). */
int sp_run_batches(sp_ctx* ctx, int32_t n, const int64_t* const* offsets,
                   const int64_t* offsets_len, const int64_t* const* indices,
                   const int64_t* indices_len, double* step_ms);
/* Enqueue one iteration without events or host sync (for timing loops and
 * CUDA-graph capture). */
int sp_enqueue_iteration(sp_ctx* ctx);
/* Capture sp_enqueue_iteration into a CUDA graph and replay it `iters`
 * times; 0 iters only builds the graph. Reports kernel nodes per graph. */
int sp_graph_replay(sp_ctx* ctx, int32_t iters, int32_t* kernels_per_iter);

/* The backward's stable sort (K4a) reads only the batch: by default (one
 * device per context) it runs on a high-priority side stream forked after
 * K1, concurrently with the exchanges, and the SGD waits for it. on = 0
 * runs it on the main stream behind K1 (per-kernel timing in isolation). */
int sp_ctx_set_overlap(sp_ctx* ctx, int32_t on);

/* The exchange of one GPU emulating D devices is a device-local copy, not
 * NVLink. on = 1 makes the breakdown's comm terms (comm_ms, both stage
 * times, overall) a MODEL of the NVLink 5 all-to-all instead — the B200
 * counterpart of device_comm (oracle.hpp:178-185), see sp_comm_model.
 * Rejected for one-process-per-GPU contexts (their exchange is measured). */
#define SP_NVLINK_PEER_GBS 770.0  /* measured peer copy per direction, B200_PROFILING.md */
#define SP_A2A_LATENCY_MS 0.010   /* grouped send/recv fixed cost (assumed, not measured) */
int sp_ctx_set_comm_model(sp_ctx* ctx, int32_t on);
/* Modelled ms of one all-to-all direction for a device holding width_dev
 * pooled columns of width_total: SP_A2A_LATENCY_MS + max(4 B w_d (D-1)/D,
 * 4 (B/D)(W - w_d)) / SP_NVLINK_PEER_GBS. width_total < 0 counts the send
 * side only (a function of the device's own tables, like device_comm). */
int sp_comm_model(int32_t batch, int64_t width_dev, int64_t width_total, int32_t D, double* ms);
/* K4a sort plan override: buckets and warp-tiles of about `lookups` lookups
 * per table (0 = the default ~sqrt(64 n) rule). The sorted result does not
 * depend on it; tests use small targets to cover many buckets and tiles. */
int sp_ctx_set_sort_target(sp_ctx* ctx, int64_t lookups);
/* Indices per H2D chunk of the pipelined host-buffer upload (default 2^23);
 * results do not depend on it. */
int sp_ctx_set_upload_chunk(sp_ctx* ctx, int64_t indices);

/* Per-kernel CUDA-event timing of the hot-path launches enqueued while
 * enabled (on the context stream): sp_ctx_kernel_ms returns the summed ms
 * and launch counts of [0]=K1 forward, [1]=(unused), [2]=K4a sort,
 * [3]=K4 SGD, [4]=exchange, and resets the accumulators (synchronizes). */
int sp_ctx_set_profiling(sp_ctx* ctx, int32_t on);
int sp_ctx_kernel_ms(sp_ctx* ctx, double ms[5], int64_t counts[5]);

/* Algorithmic bytes of one launch of each stage on this rank:
 * [0]=fwd (K1) [1]=a2a send per direction [2]=bwd floor (K4, sort
 * excluded) [3]=sort traffic estimate [4]=K1's unique-row floor (every
 * touched row read once: K1's DRAM bytes with perfect L2 reuse). */
int sp_ctx_algorithmic_bytes(sp_ctx* ctx, double out[5]);

/* ------------------------------------------------------------------ */
/* Ingest — ingest_lookup_batch (table.hpp:188-232) on the GPU.         */

/* Per table: pooling_factor = total/B, dist[17] = access-count histogram
 * normalised by total; table_size_gb from bytes_per_param. Bit-exact with
 * the reference. Host LookupBatch in, TableDesc-shaped specs out. */
int sp_ingest_lookup_batch(const int64_t* offsets, int64_t offsets_len,
                           const int64_t* indices, int64_t indices_len,
                           int32_t num_tables, int32_t batch_size,
                           const int32_t* dims, const int64_t* hash_sizes,
                           int32_t bytes_per_param, int32_t cuda_device,
                           sp_table_spec* out_tables);

/* ingest_lookup_batch(load_lookup_batch(path), dims, hash_sizes,
 * bytes_per_param) (table.hpp:188-232, 283-305) with the file's indices
 * streamed straight to the device. n_dims = the file's num_tables (else
 * SP_ERR_BAD_INPUT like the reference); out_tables holds n_dims specs;
 * num_tables_out / batch_size_out (nullable) receive the file's counts. */
int sp_ingest_batch_file(const char* path, const int32_t* dims, const int64_t* hash_sizes,
                         int32_t n_dims, int32_t bytes_per_param, int32_t cuda_device,
                         sp_table_spec* out_tables, int32_t* num_tables_out,
                         int32_t* batch_size_out);

/* ------------------------------------------------------------------ */
/* Batched cost/policy evaluator (costnet.hpp, policy.hpp).             */

/* Parameters in the reference's flat Mlp layout [W0 (out x in row-major),
 * b0, W1, b1, ...] (nn.hpp:21-53), fp64 exactly as the DSHD checkpoint
 * stores them (checkpoint.hpp:135-142). Sizes are fixed by the reference:
 * cost.table 21-128-32, cost heads 32-64-1 (x4: fwd, bwd, comm, overall),
 * policy.table 21-128-32, policy.cost 3-64-32, policy.head 64-1. */
typedef struct sp_nets {
  const double* cost_table;   /* 6944  */
  const double* cost_fwd;     /* 2177  */
  const double* cost_bwd;     /* 2177  */
  const double* cost_comm;    /* 2177  */
  const double* cost_overall; /* 2177  */
  const double* pol_table;    /* 6944  */
  const double* pol_cost;     /* 2336  */
  const double* pol_head;     /* 65    */
  const double* feature_mean; /* 21 */
  const double* feature_std;  /* 21 */
  const double* feature_mask; /* 21, 0/1 */
  int32_t reduction_tables;   /* 0 sum, 1 mean, 2 max (costnet.hpp:31) */
  int32_t reduction_devices;
} sp_nets;

/* Binds the nets and one placement task (tables, D, mem cap) to a GPU:
 * builds the normalised feature rows (table.hpp:89-104 with the
 * checkpoint's stats), the cached table representations of both nets
 * (costnet.hpp:456-464, policy.hpp:121-131) and the predicted visit order
 * (harness.hpp:131-137). */
int sp_evaluator_create(const sp_nets* nets, const sp_table_spec* tables,
                        int32_t num_tables, int32_t num_devices,
                        double mem_cap_gb, int32_t cuda_device,
                        sp_evaluator** out);
void sp_evaluator_destroy(sp_evaluator* ev);
/* The visit order predicted_order() yields (length num_tables). */
int sp_evaluator_order(sp_evaluator* ev, int32_t* order);

/* EstimatedCostProvider::overall (costnet.hpp:479-496) for n_cand complete
 * placements [n_cand, num_tables]: the RAW overall prediction, plus
 * optionally the clamped per-device q [n_cand, D, 3] (costnet.hpp:466-477).
 * fp32 on the GPU. */
int sp_eval_batch(sp_evaluator* ev, const int32_t* placements, int32_t n_cand,
                  float* overall, float* q);

/* n_cand rollouts of the policy on the estimated MDP (PlacementEnv over
 * EstimatedCostProvider, mdp.hpp:140-159) in the predicted order.
 * mode 0 = greedy (infer, harness.hpp:340-346), mode 1 = sampled with one
 * uniform per step from uniforms[n_cand, num_tables] (policy.hpp:156-169).
 * Outputs placements [n_cand, num_tables], predicted overall (raw,
 * costnet.hpp:479-496) per candidate, and a status per candidate
 * (0 ok, SP_ERR_INFEASIBLE when some table fits nowhere).
 * precision 0: fp32 with an fp64 re-run of every candidate whose decision
 * margin fell under 1e-4 relative; 1: fp64 throughout; 2: fp32 only. */
int sp_rollout_batch(sp_evaluator* ev, int32_t mode, const double* uniforms,
                     int32_t n_cand, int32_t precision, int32_t* placements,
                     double* predicted, int32_t* status, int32_t* n_refined);

/* ---- GPU training of the cost network ----------------------
 * costnet_loss_and_grad (costnet.hpp:349-427) + AdamState::update with
 * linear decay (nn.hpp:163-200) in fp64 on the device, the parameters
 * resident there between steps. params: CostNet::param_vector order
 * (15652: table 21-128-32, heads fwd/bwd/comm/overall 32-64-1). features:
 * the normalised feature rows (TaskFeatures.rows of every task) [n_rows][21];
 * a sample's tables are rows of that array. Predictions are bit-identical
 * to the reference; gradients equal it up to the association of the final
 * sum over the minibatch (deterministic). */
typedef struct sp_costnet_trainer sp_costnet_trainer;
typedef struct sp_costnet_batch {  /* CostSample list (costnet.hpp:297-304) */
  int32_t n_samples;
  const int32_t* dev_off;          /* [n+1]: devices of sample s */
  const int32_t* tab_off;          /* [dev_off[n]+1]: tables of device d */
  const int32_t* tab_row;          /* feature row of each table (any order) */
  const double* target_q;          /* [dev_off[n]][3] */
  const double* target_overall;    /* [n], NaN = no overall target; may be NULL */
} sp_costnet_batch;
int sp_costnet_trainer_create(const double* params, int64_t n_params, const double* features,
                              int64_t n_rows, const double* mask, int32_t red_tables,
                              int32_t red_devices, int32_t table_output_relu, double lr,
                              int64_t total_steps, int32_t cuda_device,
                              sp_costnet_trainer** out);
void sp_costnet_trainer_destroy(sp_costnet_trainer* t);
/* loss (and optionally grad[15652]) of one minibatch, no update */
int sp_costnet_loss_grad(sp_costnet_trainer* t, const sp_costnet_batch* batch, double* loss,
                         double* grad);
/* one step of costnet_train_steps (costnet.hpp:431-446) on a given minibatch */
int sp_costnet_train_step(sp_costnet_trainer* t, const sp_costnet_batch* batch, double* loss);
int sp_costnet_trainer_get(sp_costnet_trainer* t, double* params, double* m, double* v,
                           int64_t* step);

/* REINFORCE on the policy network (policy.hpp:203-296) in fp64 on the
 * device: params in PolicyNet::param_vector order (9345: table 21-128-32,
 * cost 3-64-32, head 64-1). An episode is a list of steps (the state's
 * device_tables, q, legal mask, action) of one task whose tables are the
 * feature rows row0 .. row0 + ntab - 1. Per-episode gradient rows summed in
 * episode order. */
typedef struct sp_policy_trainer sp_policy_trainer;
typedef struct sp_reinforce_batch {  /* Episode list (policy.hpp:189-201) */
  int32_t n_episodes;
  const int32_t* row0;      /* [n] */
  const int32_t* ntab;      /* [n] */
  const int32_t* step_off;  /* [n+1] */
  const double* reward;     /* [n] */
  const int32_t* dev_off;   /* [steps+1] */
  const int32_t* action;    /* [steps] */
  const int32_t* tab_off;   /* [devices+1] */
  const int32_t* tab_id;    /* task-local table ids (any order in a device) */
  const int32_t* legal;     /* [devices] 0/1 */
  const double* q;          /* [devices][3] */
} sp_reinforce_batch;
int sp_policy_trainer_create(const double* params, int64_t n_params, const double* features,
                             int64_t n_rows, const double* mask, double lr,
                             int64_t total_steps, int32_t cuda_device,
                             sp_policy_trainer** out);
void sp_policy_trainer_destroy(sp_policy_trainer* t);
int sp_reinforce_loss_grad(sp_policy_trainer* t, const sp_reinforce_batch* b, double w_entropy,
                           double* objective, double* grad);
/* reinforce_update (policy.hpp:287-296): one Adam step */
int sp_reinforce_step(sp_policy_trainer* t, const sp_reinforce_batch* b, double w_entropy,
                      double* objective);
int sp_policy_trainer_get(sp_policy_trainer* t, double* params, double* m, double* v,
                          int64_t* step);

#ifdef __cplusplus
}
#endif

#endif /* SHARDPLAN_B200_H_ */
