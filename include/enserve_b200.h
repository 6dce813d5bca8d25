/* enserve-b200 — C ABI of the B200-native ensemble-inference hot path.
 *
 * This is the drop-in boundary.  Every entry point replaces one function (or
 * one class method) of the reference's C++ API, /root/reference/proj
 * ("enserve", arXiv 2208.14049); the reference location is cited on each
 * declaration.  Plain pointers and sizes only, no C++ or torch types; every
 * call returns an es_status and never throws.  INTEGRATION.md shows the
 * reference-side adapter (a PredictorFactory named "b200" plus a ScoreFn) a
 * maintainer would add to call this library.
 *
 * Matrices are D x M int grids, row-major (cell d*M+m), like
 * AllocationMatrix (include/enserve/core/types.hpp:55-88).
 */
#ifndef ENSERVE_B200_H
#define ENSERVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ES_ABI_VERSION 2  /* 2: es_pool_opts and es_model_desc grew (multi-GPU, device FIFO, fp32, B200 cost fit) */
#define ES_MAX_WIDTHS 9

/* Error classes of include/enserve/core/errors.hpp:9-51, plus device errors. */
typedef enum es_status {
  ES_OK = 0,
  ES_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument / std::out_of_range */
  ES_ERR_SPEC = 2,             /* SpecError */
  ES_ERR_ALLOCATION = 3,       /* AllocationError (worst-fit found no device) */
  ES_ERR_STARTUP = 4,          /* StartupError (a worker's load() reported OOM) */
  ES_ERR_BASELINE = 5,         /* BaselineError (BBS needs one GPU per model) */
  ES_ERR_CAP_EXCEEDED = 6,     /* CapExceededError */
  ES_ERR_PROTOCOL = 7,         /* ProtocolError */
  ES_ERR_CUDA = 8,             /* CUDA failure other than out-of-memory */
  ES_ERR_INTERNAL = 9,
  ES_ERR_BUFFER = 10,          /* caller buffer too small */
  ES_ERR_NOT_READY = 11        /* NotReadyError: service still loading or stopped (HTTP 503) */
} es_status;

/* DeviceSpec (types.hpp:17-26); ids are the array positions. */
typedef struct es_device_desc {
  int kind; /* 0 = CPU, 1 = GPU */
  double memory_mib;
  double compute_rate;
  double batch_overhead_s;
} es_device_desc;

/* ModelSpec (types.hpp:28-35) + what the device executes. */
typedef struct es_model_desc {
  const char* name;
  double weight_mib;
  double act_mib_per_sample;
  double cost_per_sample;
  int output_width;
  int arch;                     /* 0 = synthetic_prediction member, 1 = MLP, 2 = CNN */
  int n_widths;                 /* MLP: input, hidden..., classes;
                                   CNN: 6 = {S, P, c1, c2, hidden, classes} (S x S image,
                                   conv PxP/P -> c1, conv 3x3 -> c2, dense -> hidden -> classes) */
  int widths[ES_MAX_WIDTHS];
  uint64_t weight_seed;
  double b200_cost_s;     /* B200 calibration (extension; 0 = none): 1 / throughput(b) = */
  double b200_overhead_s; /* b200_cost_s + b200_overhead_s / b, member alone on one GPU  */
} es_model_desc;

/* ClusterSpec (types.hpp:38-52). */
typedef struct es_cluster_desc {
  const es_device_desc* devices;
  int n_devices;
  const es_model_desc* models;
  int n_models;
  const int* batch_menu;
  int menu_size;
  int segment_size;
} es_cluster_desc;

/* CombinationRule (include/enserve/runtime/combine.hpp:14-27). */
typedef struct es_rule_desc {
  int kind;            /* 0 = averaging, 1 = majority vote, 2 = weighted averaging */
  int member_softmax;  /* fold softmax(member output) instead of the raw output */
  const double* weights;
} es_rule_desc;

/* PoolOptions (include/enserve/runtime/pipeline.hpp:48-53), device flavour. */
typedef struct es_pool_opts {
  const int* device_map; /* cluster device row -> CUDA ordinal; NULL = row % #GPUs */
  int n_device_map;
  int copy_outputs;      /* D2H of the combined output in await_run */
  int warmup;            /* bench: one untimed run first */
  int sms_per_worker;    /* 0 = all SMs (persistent grid) */
  int overlap_colocated; /* 1 = one stream per worker; 0 = co-located workers
                            time-share one stream per GPU */
  size_t e2e_chunk_rows; /* es_system_run_host pipeline chunk (0 = 65536) */
  int e2e_host_convert;  /* 1 = host threads convert fp32 -> bf16 for every other
                            chunk (all chunks if X is pageable), the rest is
                            DMA'd as fp32 from the caller's pinned buffer;
                            0 = every chunk DMA'd as fp32 (pinned X) */
  int e2e_convert_eighths; /* with e2e_host_convert and pinned X: chunks in 8 the
                              host converts (0 = default 6) */
  int dp_equal_split;      /* 0 = a model's data-parallel workers split its segments in
                              runs proportional to their probed rows/s (SURVEY.md §8-E
                              static fallback of the shared FIFO); 1 = equal runs */
  int row_partials;        /* 1 = fast gather: each device row folds its
                              members into a partial on its GPU, only partials travel,
                              summed in row order (fp32 order differs from the
                              reference fold; votes exact; pure model placement only);
                              0 = parity gather (bit-identical fold) */
  int no_peer_stores;      /* 0 = remote workers store logits straight into the combining
                              GPU's buffers over NVLink peer mappings (peer access is
                              enabled at construction); 1 = local staging buffer +
                              cudaMemcpyPeerAsync after the member kernels */
  int row_nodes;           /* 1 = every device row is its own node (stream, staging,
                              gather, run_host lane) even where rows share a GPU */
  int dp_claim;            /* device FIFO (the reference's shared per-model queue,
                              pipeline.cpp:44-51): a data-parallel model's workers pop
                              chunks of segments off one device counter.  0 = auto (models
                              whose workers sit on distinct GPUs), 1 = always, -1 = off
                              (the static split, dp_equal_split) */
  int64_t claim_chunk;     /* segments per claim (0 = auto) */
  int pack_batches;        /* 1 = every tile packs a whole segment whatever the batch
                              (bit-identical logits; b then stops mattering on B200);
                              0 = a b-row batch is one tile (the reference batcher) */
  int fp32;                /* 1 = fp32-accurate members (fp32 X, weights, activations and
                              accumulation on the CUDA cores; 1e-5 parity mode);
                              0 = bf16 operands on the tensor cores */
} es_pool_opts;

/* RunStats (pipeline.hpp:19-25). */
typedef struct es_run_stats {
  size_t nb_samples;
  size_t segments;
  size_t data_messages;
  double elapsed_s; /* CUDA-event window: broadcast -> last fold */
} es_run_stats;

/* BenchResult (pipeline.hpp:35-41); runs[] holds up to 64 repeats. */
typedef struct es_bench_result {
  double throughput;
  double elapsed_s;
  size_t nb_samples;
  int n_runs;
  double runs[64];
  double rsd;
} es_bench_result;

typedef struct es_store es_store;
typedef struct es_system es_system;
typedef struct es_comm es_comm;
typedef struct es_member es_member;

int es_abi_version(void);
const char* es_status_name(es_status s);
/* Message of the last failed call on this thread. */
const char* es_last_error(void);

/* ------------------------------------------------------------ host core */
/* ClusterSpec::validate (src/core/types.cpp:31-74). */
es_status es_cluster_validate(const es_cluster_desc* c, char* warnings, size_t len);
/* validate_matrix (types.cpp:102-127); violations: [kind, device, model, value] x n. */
es_status es_matrix_validate(const es_cluster_desc* c, const int* A, int* ok, int* violations,
                             int cap, int* n);
/* num_segments / segment_bounds (types.cpp:129-149). */
es_status es_num_segments(size_t nb, int segment_size, size_t* out);
es_status es_segment_bounds(int segment_id, int segment_size, size_t nb, size_t* start,
                            size_t* end);
/* Segments each worker predicts in one run (replaces the per-model shared
 * FIFO of src/runtime/pipeline.cpp:103-104,143-166 with a static, exactly-once
 * split): out[4*i..] = {device, model, first segment, end segment}. */
es_status es_segment_shares(const int* A, int devices, int models, size_t nb, int segment_size,
                            long long* out, int cap, int* n);
/* The batcher (src/runtime/pipeline.cpp:143-166) as the member kernels run
 * it: segments [seg_begin, seg_end) of nb rows become tiles of `batch` rows
 * per segment, the last of each segment the remainder.  row0[i], rows[i] for
 * up to cap tiles; *n = the tile count. */
es_status es_batch_rows(size_t nb, int segment_size, long long seg_begin, long long seg_end,
                        int batch, long long* row0, int* rows, int cap, int* n);
/* The same with each model's runs proportional to weight[w] (one per worker,
 * row-major cells, > 0): what InferenceSystem uses with probed rows/s
 * (SURVEY.md §8-E static fallback).  Equal weights give es_segment_shares. */
es_status es_segment_shares_weighted(const int* A, int devices, int models, size_t nb,
                                     int segment_size, const double* weight, long long* out,
                                     int cap, int* n);
/* fit_mem (src/memory/memory_model.cpp:22-32); used_mib[D]. */
es_status es_fit_mem(const es_cluster_desc* c, const int* A, double* used_mib, int* fits);
/* more_remaining_memory (memory_model.cpp:34-50); *device = -1 when none. */
es_status es_more_remaining_memory(const es_cluster_desc* c, const int* A, int kind, int* device);
/* predict_ensemble_throughput (src/cost/cost_model.cpp:29-46). */
es_status es_predict_ensemble_throughput(const es_cluster_desc* c, const int* A, double* out);
/* worst_fit_decreasing (src/opt/optimizer.cpp:37-64); ES_ERR_ALLOCATION names the
 * model in es_last_error(). */
es_status es_worst_fit_decreasing(const es_cluster_desc* c, int default_batch, int* A_out);
/* neighborhood (optimizer.cpp:66-84): writes min(count, cap) matrices. */
es_status es_neighborhood(const es_cluster_desc* c, const int* A, int* out, int cap, int* count);
/* enumerated_neighborhood_stats (optimizer.cpp:86-103). */
es_status es_neighborhood_stats(const es_cluster_desc* c, const int* A, size_t* size,
                                size_t* forbidden);
/* count_total_matrices (optimizer.cpp:105-111), decimal string. */
es_status es_count_total_matrices(int menu_size, int devices, int models, char* buf, size_t len);
/* count_total_neighs (optimizer.cpp:113-118). */
es_status es_count_total_neighs(int menu_size, int devices, int models, long long forbidden,
                                long long* out);
/* effective_max_iter (optimizer.cpp:173-176). */
es_status es_effective_max_iter(int devices, int models, int max_iter, int* out);
/* enumerate_all_matrices (optimizer.cpp:120-171); cap as a decimal string. */
es_status es_enumerate_matrices(const es_cluster_desc* c, const char* cap, int* out,
                                size_t out_cap, size_t* count);
/* sample_indices (include/enserve/util/rng.hpp:26-38) from a fresh mt19937_64(seed). */
es_status es_sample_indices(uint64_t seed, size_t n, size_t k, size_t* out);

/* ScoreFn (include/enserve/opt/optimizer.hpp:18). */
typedef double (*es_score_fn)(const int* A, int devices, int models, void* user);

typedef enum es_bench_mode {
  ES_BENCH_ANALYTIC = 0, /* predict_ensemble_throughput */
  ES_BENCH_DEVICE = 1,   /* bench() on the GPUs, CUDA-event timed */
  ES_BENCH_CALLBACK = 2, /* caller's es_score_fn */
  ES_BENCH_CALIBRATED = 3 /* calibrated_throughput (per-member B200 fit; opts->device_map,
                             when given, groups rows sharing a GPU) */
} es_bench_mode;

typedef struct es_bench_cfg {
  int mode;
  es_score_fn fn;
  void* user;
  es_store* calib;
  int repeats;
  const es_pool_opts* opts;
} es_bench_cfg;

/* OptimizationTrace (optimizer.hpp:33-47); iteration arrays hold iter_cap entries. */
typedef struct es_greedy_trace {
  double start_score;
  double final_score;
  int stop_reason; /* 0 = local_optimum, 1 = iter_cap */
  int n_iters;
  int bench_calls;
  int iter_cap;
  int* iter_neighbors;
  double* iter_best;
  int* iter_accepted;
} es_greedy_trace;

/* bounded_greedy (optimizer.cpp:178-227). */
es_status es_bounded_greedy(const es_cluster_desc* c, const int* A0, int max_iter, int max_neighs,
                            uint64_t seed, const es_bench_cfg* bench, int* A_out,
                            es_greedy_trace* trace);
/* bounded_greedy with a pre-screen: each iteration's sampled
 * neighbours are ranked by `screen` (e.g. ES_BENCH_CALIBRATED) and only the top_k
 * are scored by `bench`; trace->bench_calls counts the bench calls. */
es_status es_screened_greedy(const es_cluster_desc* c, const int* A0, int max_iter,
                             int max_neighs, uint64_t seed, int top_k, const es_bench_cfg* bench,
                             const es_bench_cfg* screen, int* A_out, es_greedy_trace* trace);
/* bbs_baseline (optimizer.cpp:229-269); chosen[M]. */
es_status es_bbs_baseline(const es_cluster_desc* c, const es_bench_cfg* bench, int* A_out,
                          int* chosen, int* calls);

/* ------------------------------------------------------------ device runtime */
es_status es_device_count(int* n);

/* SampleStore (include/enserve/runtime/message.hpp:12-34).  copy = 0 borrows X
 * (must outlive the store). */
es_status es_store_create(const float* X, size_t nb, size_t width, int copy, es_store** out);
/* Synthetic features generated on `device`. */
es_status es_store_synthetic(uint64_t seed, size_t nb, size_t width, int device, es_store** out);
void es_store_destroy(es_store* s);

/* InferenceSystem (include/enserve/runtime/pipeline.hpp:62-117). */
es_status es_system_create(const es_cluster_desc* c, const int* A, const es_rule_desc* rule,
                           const es_pool_opts* opts, es_system** out);
es_status es_system_begin_run(es_system* s, es_store* X, const es_rule_desc* rule);
es_status es_system_broadcast(es_system* s, size_t* segments);
/* Y[nb*C] and winners[nb] may be NULL. */
es_status es_system_await_run(es_system* s, float* Y, int32_t* winners, es_run_stats* stats);
es_status es_system_run(es_system* s, es_store* X, float* Y, int32_t* winners,
                        es_run_stats* stats);
/* End to end from host memory: H2D of X, members, combine, D2H of Y and labels
 * all inside the CUDA-event window. */
es_status es_system_run_host(es_system* s, const float* X, size_t nb, size_t width, float* Y,
                             int32_t* labels, double* elapsed_s);
/* The host converter of es_system_run_host: y = bf16_rn(x), all host threads. */
es_status es_host_convert_bf16(const float* x, uint16_t* y, size_t n);
/* workers_per_model[M] (pipeline.hpp:86-89) + launches of the last run. */
es_status es_system_info(es_system* s, int* workers, int* workers_per_model, int* launches,
                         int* combine_device);
/* Device time of each worker's member kernel and of the combine, last run. */
es_status es_system_timing(es_system* s, double* member_ms, double* combine_ms);
/* Segment runs of every worker (row-major cells) in the last run:
 * shares[2w] = begin, shares[2w+1] = end; rates[w] = probed rows/s of a
 * data-parallel worker (1.0 for a model's only worker, or before any run).
 * Either array may be NULL; each holds the worker count of es_system_info. */
es_status es_system_shares(es_system* s, int64_t* shares, double* rates);
/* Host<->device bytes the last es_system_run_host moved. */
es_status es_system_last_transfer(es_system* s, size_t* h2d_bytes, size_t* d2h_bytes);
/* Per-launch device time of one worker's member kernels in the last run
 * (ms[cap], -1 where the worker had no rows), their kernel names joined by
 * ';' into names[names_len], and the launch count per run. */
es_status es_system_kernel_timing(es_system* s, int worker, double* ms, char* names,
                                  size_t names_len, int cap, int* count);
/* Per worker: 0 = on the combining node, 1 = remote with direct peer stores,
 * 2 = remote through staging + peer copy (routes[workers]); peers[cap] = CUDA
 * ordinals with peer access to/from the combining GPU, *n_peers their count. */
es_status es_system_routes(es_system* s, int* routes, int* peers, int cap, int* n_peers);
/* Device FIFO of the last run for model m: owner[segments] = the worker index
 * (row-major cells) that claimed each segment; *n = segments (0 when the model
 * has no queue).  owner may be NULL to query n. */
es_status es_system_claims(es_system* s, int model, int* owner, size_t cap, size_t* n);
/* Models whose data-parallel workers claim from a device queue: models[cap], *n. */
es_status es_system_claim_models(es_system* s, int* models, int cap, int* n);
es_status es_system_shutdown(es_system* s);
void es_system_destroy(es_system* s);

/* ---------------------------------------------- one process per GPU (NCCL)
 * The reference funnels every worker's predictions into one accumulator
 * (src/runtime/pipeline.cpp:210-211, :258-279); across processes that is a
 * gather of each rank's combined probabilities + argmax to a root rank.
 * libnccl.so.2 is resolved at run time. */
/* ncclGetUniqueId: id[128] for es_comm_create on every rank. */
es_status es_comm_unique_id(uint8_t* id, size_t len);
/* ncclCommInitRank on CUDA ordinal `device` (collective: every rank calls it). */
es_status es_comm_create(const uint8_t* id, size_t len, int nranks, int rank, int device,
                         es_comm** out);
es_status es_nccl_version(int* version);
void es_comm_destroy(es_comm* c);
/* After each run's combine, this rank's rows go to `root` at row first_rows[rank]
 * of an (sum rows)-row result, inside the timed window; the root's await_run /
 * es_system_run returns every rank's rows (Y/winners sized for the sum).
 * comm NULL detaches.  The system keeps the communicator alive. */
es_status es_system_set_gather(es_system* s, es_comm* comm, int root, const int64_t* first_rows,
                               const int64_t* rows, int nranks);

/* run_inference (pipeline.cpp:418-444), Deploy mode: Y[nb*C], winners[nb]. */
es_status es_run_inference(const es_cluster_desc* c, const int* A, const es_rule_desc* rule,
                           es_store* X, const es_pool_opts* opts, float* Y, int32_t* winners,
                           es_run_stats* stats);
/* bench (pipeline.cpp:465-501). */
es_status es_bench(const es_cluster_desc* c, const int* A, es_store* calib, int repeats,
                   const es_pool_opts* opts, es_bench_result* out);

/* ------------------------------------------------------------ Predictor seam */
/* PredictorFactory::make + Predictor::load (include/enserve/runtime/backend.hpp:
 * 16-41): ES_ERR_STARTUP when load() reports out-of-memory. */
es_status es_member_create(int device, const es_model_desc* model, int model_id, int batch,
                           double device_load_mib, double capacity_mib, es_member** out);
/* Predictor::predict (backend.hpp:33): rows x width fp32 host features of
 * samples first_index.. -> out[rows * C] host. */
es_status es_member_predict(es_member* m, const float* features, size_t first_index, size_t rows,
                            size_t width, float* out);
void es_member_destroy(es_member* m);

/* PredictionAccumulator fold (src/runtime/combine.cpp:93-136) for M host blocks
 * of rows x C, run by the device combine kernel; winners = argmax per row. */
es_status es_combine(const es_rule_desc* rule, int M, int C, size_t rows,
                     const float* const* blocks, float* Y, int32_t* winners);

/* ------------------------------------------------ spec / matrix / cache documents */
/* On-disk formats of include/enserve/core/spec_io.hpp and
 * include/enserve/server/cache.hpp: a reference-written
 * file loads here and vice versa, and cache keys are identical.  Text results
 * go to buf[len] (NUL-terminated; *needed = bytes required, buf may be NULL to
 * ask); ES_ERR_BUFFER when len is too small. */
typedef struct es_spec es_spec;
/* cluster_to_json (spec_io.cpp:7-28) dumped like nlohmann's dump(indent)
 * (indent < 0: compact).  with_arch adds each member's architecture as an
 * optional "arch" object the reference parser ignores. */
es_status es_cluster_to_json(const es_cluster_desc* c, int indent, int with_arch, char* buf,
                             size_t len, size_t* needed);
/* cluster_from_documents (spec_io.cpp:82-89; overlay may be NULL) +
 * cluster_from_json (:47-80): SpecError on a malformed document. */
es_status es_spec_from_json(const char* base_json, const char* overlay_json, es_spec** out);
/* load_json_file (spec_io.cpp:135-143) of a --cluster and an optional
 * --ensemble file, merged. */
es_status es_spec_load(const char* path, const char* overlay_path, es_spec** out);
/* The parsed cluster as a descriptor (pointers valid while the handle lives). */
es_status es_spec_describe(es_spec* s, es_cluster_desc* out);
void es_spec_destroy(es_spec* s);
/* save_json_file (spec_io.cpp:145-149): the document indented by 2 + "\n". */
es_status es_save_json_file(const char* path, const char* json_text);
/* matrix_to_json / matrix_from_json (spec_io.cpp:91-133). */
es_status es_matrix_to_json(const es_cluster_desc* c, const int* A, int indent, char* buf,
                            size_t len, size_t* needed);
es_status es_matrix_from_json(const es_cluster_desc* c, const char* json_text, int* A_out);
/* digest_hex (cache.cpp:11-20): FNV-1a 64, 16 hex digits + NUL. */
es_status es_digest_hex(const char* text, char out[17]);
/* cache_key (cache.cpp:22-33) of the cluster and the optimizer settings. */
es_status es_cache_key(const es_cluster_desc* c, int max_iter, int max_neighs, uint64_t rng_seed,
                       int default_batch, const char* bench_mode, size_t calib_samples,
                       int repeats, char out[17]);
/* cache_key with the opt-in hardware identity (NULL or "" = es_cache_key):
 * a matrix measured on other GPUs misses.  Reference-computed keys match only
 * the identity-free form. */
es_status es_cache_key_device(const es_cluster_desc* c, int max_iter, int max_neighs,
                              uint64_t rng_seed, int default_batch, const char* bench_mode,
                              size_t calib_samples, int repeats, const char* device,
                              char out[17]);
/* "<name>/sm_<cc>/<SMs> SMs/<GiB> GiB x<count>" of the visible GPUs. */
es_status es_device_identity(char* out, size_t len);
/* MatrixCache::lookup / store (cache.cpp:35-88): corrupt, stale or invalid
 * entries are misses (*hit = 0), never errors. */
es_status es_cache_lookup(const char* directory, const char* key, const es_cluster_desc* c,
                          int* A_out, double* score, int64_t* created_at, int* hit);
es_status es_cache_store(const char* directory, const char* key, const es_cluster_desc* c,
                         const int* A, double score, int64_t created_at);

/* ------------------------------------------------ B200-calibrated cost model */
/* the reference's analytic bench (src/cost/cost_model.cpp:
 * 13-46) with its inputs fitted to this box.  With compute_rate R = 1,
 * 1/throughput(m, b) = c_m + o/b is fitted by least squares in relative error
 * (cost_out[n_models] = c_m in seconds per sample, *overhead_out = o >= 0,
 * *rms_out = relative RMS misfit). */
/* member_cost_out / member_overhead_out [n_models] (may be NULL) receive the
 * per-member fit 1/throughput(m, b) = c'_m + o_m/b and *member_rms_out its misfit. */
es_status es_fit_cost_model(const int* model, const int* batch, const double* throughput, int n,
                            int n_models, double* cost_out, double* overhead_out, double* rms_out,
                            double* member_cost_out, double* member_overhead_out,
                            double* member_rms_out);
/* Benches every model of c alone on CUDA device `device` at every menu batch
 * (device-timed bench over calib_nb synthetic samples, median of repeats)
 * and fits; measured_out[n_models * menu_size] (may be NULL) receives the
 * throughputs, model-major. */
es_status es_calibrate_cost_model(const es_cluster_desc* c, int device, size_t calib_nb,
                                  int repeats, double* cost_out, double* overhead_out,
                                  double* rms_out, double* measured_out, double* member_cost_out,
                                  double* member_overhead_out, double* member_rms_out);
/* calibrated_throughput (calibrate.hpp): A scored with the models' b200_cost_s /
 * b200_overhead_s as the device runs it; row_gpu[n_devices] (may be NULL) maps
 * rows to GPUs (rows sharing one time-share it). */
es_status es_calibrated_throughput(const es_cluster_desc* c, const int* A, const int* row_gpu,
                                   double* out);

/* ------------------------------------------------------------ operator commands */
/* tools/enserve_cli.cpp main() + src/cli/commands.cpp:
 * optimize | bench --matrix F | count | baseline over --cluster/--ensemble
 * spec files, with --cache-dir, --bench-mode measured|analytic and the b200
 * backend (measured = device-timed bench on this box's GPUs).  argv[0] is the
 * program name.  Report on stdout, errors on stderr; returns the exit code
 * (0 ok, 1 error, 2 allocation error). */
int es_cli_main(int argc, const char* const* argv);

/* ------------------------------------------------------------ deploy-mode service */
/* The serving core of the reference's PredictionServer (src/server/server.cpp,
 * SURVEY.md §8-F F1) without the HTTP listener: requests are buffered and
 * flushed into one device run when a full segment is waiting or the oldest
 * request has waited flush_timeout_ms (server.cpp:227-273); each request gets
 * its own rows of the combined output back.  A caller's HTTP front end maps
 * POST /v1/predict -> es_service_submit + es_request_wait and GET /v1/stats
 * -> es_service_stats. */
typedef struct es_service es_service;
typedef struct es_request es_request;

typedef struct es_service_info {
  int ready;
  uint64_t requests_served;
  uint64_t samples_served;
  uint64_t flushes;
  double last_flush_throughput; /* samples/s over the last flush's device window */
  size_t pending_requests;
  size_t pending_samples;
  double uptime_s;
} es_service_info;

/* Validates A (ES_ERR_SPEC if invalid, server.cpp:30-31) and starts building
 * the device pool on a background thread (init_pool, server.cpp:37-52). */
/* arena_rows: rows per page-locked staging arena of a one-GPU pool (two
 * arenas; submits convert to bf16 straight into them), < 0 = default 262144,
 * 0 = none (requests staged in private buffers and gathered per flush). */
es_status es_service_create(const es_cluster_desc* c, const int* A, const es_rule_desc* rule,
                            const es_pool_opts* opts, int flush_timeout_ms, size_t input_width,
                            long long arena_rows, es_service** out);
/* ready = 1 once the pool is up; error receives the startup error (if any). */
es_status es_service_wait_ready(es_service* s, int timeout_ms, int* ready, char* error,
                                size_t error_len);
/* X: rows x input_width fp32 (copied before return).  rows = 0 completes at once. */
es_status es_service_submit(es_service* s, const float* X, size_t rows, es_request** out);
/* Blocks until the request's flush ran; Y: rows x output_width, winners: rows
 * (either may be NULL).  ES_ERR_STARTUP if the pool failed, an error status
 * with "server shutting down" if the service stopped first. */
es_status es_request_wait(es_request* r, float* Y, int32_t* winners);
void es_request_destroy(es_request* r);
es_status es_service_stats(es_service* s, es_service_info* out);
/* Stops the dispatcher (buffered requests fail) and releases the pool. */
void es_service_destroy(es_service* s);

#ifdef __cplusplus
}
#endif

#endif /* ENSERVE_B200_H */
