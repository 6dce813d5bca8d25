// enserve-b200 runtime: the GPU InferenceSystem behind the reference's API.
//
// API mirror of /root/reference/proj/include/enserve/runtime/pipeline.hpp:17-135
// and combine.hpp:14-27 (CombinationRule), with the reference's thread pipeline
// (batcher -> predictor -> sender -> accumulator, pipeline.cpp:141-279) replaced
// by device work:
//   * one persistent member kernel per nonzero cell (worker), on its own CUDA
//     stream, walking its share of the segments tile by tile (tile = the
//     worker's batch b, the batcher split of pipeline.cpp:155-162); a
//     data-parallel model's workers pop their segments off one device
//     counter (the per-model queue of pipeline.cpp:44-51) or split them
//     statically;
//   * per-model logits land directly at their row offset in a [nb x C] buffer on
//     the combining device (a remote worker's kernels store them over NVLink
//     peer mappings, or stage + peer-copy);
//   * one K3 combine launch folds all members in model-id order; with one
//     process per GPU, an NCCL gather then brings every rank's rows to the
//     root (the single accumulator of pipeline.cpp:258-279).
// The timed window is the reference's (broadcast -> last fold,
// pipeline.cpp:309 / :268-269), measured with CUDA events on the combining
// device; X upload happens in begin_run, untimed, as in pipeline.cpp:285-302.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "enserve/spec.hpp"

namespace enserve {

// ---- combination rule (combine.hpp:14-27) -----------------------------------
struct CombinationRule {
  enum class Kind { averaging, majority_vote, weighted_averaging };
  Kind kind = Kind::averaging;
  std::vector<double> weights;  // weighted_averaging: one per model, >= 0, sum 1
  // Fold softmax(member logits) instead of the raw member output.  Off keeps
  // the reference's fold bit-for-bit; the B200 ensemble workload turns it on.
  bool member_softmax = false;

  static CombinationRule averaging(bool softmax = false) { return {Kind::averaging, {}, softmax}; }
  static CombinationRule majority_vote(bool softmax = false) {
    return {Kind::majority_vote, {}, softmax};
  }
  static CombinationRule weighted(std::vector<double> weights, bool softmax = false);
  std::string name() const;
  static CombinationRule from_name(const std::string& name, int model_count);
};

// ---- immutable samples (message.hpp:12-34) ----------------------------------
// nb x width fp32 features.  Device replicas (bf16, row-major) are created on
// first use per GPU and reused by every later run, like the reference's shared
// SampleStore.
class SampleStore {
 public:
  SampleStore(std::vector<float> data, std::size_t nb, std::size_t width);
  // Non-owning: `data` must outlive the store.
  static std::shared_ptr<SampleStore> borrow(const float* data, std::size_t nb, std::size_t width);
  // Synthetic features generated on `device` (x = U[0,1) keyed by seed and flat
  // index); no host copy exists.
  static std::shared_ptr<SampleStore> synthetic(std::uint64_t seed, std::size_t nb,
                                                std::size_t width, int device);
  ~SampleStore();
  SampleStore(const SampleStore&) = delete;
  SampleStore& operator=(const SampleStore&) = delete;

  std::size_t nb_samples() const { return nb_; }
  std::size_t width() const { return width_; }
  const float* host_data() const { return host_; }
  // bf16 [nb][width] on `device` (uploads + converts on first call).
  const void* device_replica(int device) const;
  // fp32 [nb][width] on `device` (the fp32 member mode), created on first call.
  const float* device_replica_f32(int device) const;

 private:
  SampleStore() = default;
  std::vector<float> owned_;
  const float* host_ = nullptr;
  std::size_t nb_ = 0;
  std::size_t width_ = 0;
  std::uint64_t synthetic_seed_ = 0;
  bool synthetic_ = false;
  mutable std::vector<void*> replicas_;  // indexed by CUDA ordinal
  mutable std::vector<float*> replicas32_;
};

// ---- run bookkeeping (pipeline.hpp:17-53) -----------------------------------
enum class Mode { Deploy, Benchmark };

struct RunStats {
  std::size_t nb_samples = 0;
  std::size_t segments = 0;
  std::size_t data_messages = 0;
  std::vector<std::size_t> segment_rows;
  double elapsed_s = 0.0;
};

struct RunOutput {
  std::vector<float> combined;
  std::vector<int> winners;  // argmax per sample (lowest index on ties), every rule
  int output_width = 0;
  RunStats stats;
};

struct BenchResult {
  double throughput = 0.0;
  double elapsed_s = 0.0;
  std::size_t nb_samples = 0;
  std::vector<double> runs;
  double rsd = 0.0;
};

struct InferenceResult {
  std::optional<RunOutput> output;
  std::optional<BenchResult> score;
};

struct PoolOptions {
  // Cluster device row d runs on CUDA ordinal device_map[d]; empty = d modulo
  // the visible GPU count (lets a 1-GPU box host a multi-device matrix).
  std::vector<int> device_map;
  bool copy_outputs = true;   // D2H of the combined output in await_run
  bool warmup = true;         // bench: one untimed run first (module load, clocks)
  int sms_per_worker = 0;     // 0 = every SM of the device (persistent grid)
  bool overlap_colocated = false;  // one stream per worker instead of per GPU
  // run_host: rows per pipeline chunk (rounded to whole segments) and whether
  // the host converts fp32 -> bf16 before the copy (half the PCIe bytes).
  std::size_t e2e_chunk_rows = 65536;
  bool e2e_host_convert = true;
  // Pinned input with host conversion on: how many chunks in 8 the host
  // converts (the rest are DMA'd as fp32 and converted on the device) --
  // balances host-memory bandwidth against PCIe.  6 measured best on B200
  // boxes (tools/e2e_sweep.py, cfg2, non-temporal stores into the pinned
  // slots: 4/8 2.19e7, 6/8 2.56e7, 7/8 2.53e7, 8/8 2.26e7 samples/s): both
  // legs saturate the host's memory bandwidth.
  int e2e_convert_eighths = 6;
  // Data-parallel split of a model's segments: runs
  // proportional to each worker's probed rows/s (the static stand-in for the
  // reference's shared FIFO, where faster workers pull more segments), or
  // equal runs.
  bool dp_equal_split = false;
  // The device FIFO (the reference's shared per-model queue,
  // pipeline.cpp:44-51, :103-104): a data-parallel model's workers pop chunks
  // of `claim_chunk` segments (0 = auto: about four per worker, at least two
  // waves of tiles) off one device counter on the combining GPU -- remote
  // workers through their NVLink peer mapping -- so a faster worker takes more
  // of the model's segments.  Applies when every worker of the model can
  // follow a claim and reach the combining GPU directly; otherwise (or off)
  // the static split above.  run_host keeps the static split.
  //   kClaimAuto: only where the model's workers sit on distinct GPUs -- they
  //     run side by side, so the faster GPU pulls more.  Workers sharing a GPU
  //     time-share its SMs; whoever claims, the GPU does the same work, and a
  //     worker with a small batch (slow per segment) claiming much costs more
  //     than the probed split, which gives it little (measured, tools/
  //     claim_probe.py: 10.9 vs 4.6 ms on one B200).
  //   kClaimAlways: every eligible model (tests; SM-partitioned workers).
  enum ClaimMode { kClaimOff = 0, kClaimAuto = 1, kClaimAlways = 2 };
  int dp_claim = kClaimAuto;
  long long claim_chunk = 0;
  // A worker's batch b is its tile height: each b-row batch of a segment is
  // one M = 128 UMMA tile (the reference batcher's split, pipeline.cpp:155-162,
  // kept observable).  A tcgen05 MMA costs the same for 8 or 128 rows (and
  // swap-AB with N = b the same for N <= 92), so on B200 a batch of b rows
  // runs at b/128 of the tensor rate (profiles/r2m_small_batch.txt).  On,
  // every tile packs a whole segment whatever b (rows are independent, the
  // logits are bit-identical): the batch size then stops mattering on the
  // device.  Off by default so the optimizer still sees the batch dimension.
  bool pack_batches = false;
  // fp32-accurate members (north_star's 1e-5 fp32 tolerance): X, weights,
  // activations and accumulation in fp32 on the CUDA cores
  // (cuda/fp32_kernels.cuh) instead of bf16 operands on the tensor cores.
  // run_host then moves fp32 rows (4 B/feature) and converts nothing.
  bool fp32 = false;
  // Gather: false = parity mode, every member's logits go
  // to the combining GPU and one fold runs in model order (bit-identical to
  // the reference); true = fast mode, each device row folds its own members
  // into a partial [nb][C] (avg/wavg: sum of weighted (softmax) outputs;
  // vote: tallies) and only the partials travel, summed in row order -- C
  // floats per sample per row instead of per member.  fp32 sums in another
  // order (votes stay exact); applies when no model is data-parallel.
  bool row_partials = false;
  // Remote workers (another GPU than the combining one) store their logits
  // straight into the combining GPU's buffers through NVLink peer mappings
  // (cudaDeviceEnablePeerAccess at construction) -- no staging copy.  Off, or
  // where the pair has no peer access, they write a local staging buffer that
  // cudaMemcpyPeerAsync moves after the member kernels.
  bool peer_stores = true;
  // Every cluster device row is its own node -- own stream, own logits
  // staging and gather, own run_host lane -- even where rows share a CUDA
  // ordinal.  Lays an N-GPU matrix out on fewer GPUs with the multi-GPU data
  // path intact (tests exercise every cross-device branch on one GPU this way).
  bool row_nodes = false;
};

// Per-model executable member on one GPU (the Predictor of backend.hpp:25-34).
class DeviceMember;
class Comm;

class InferenceSystem {
 public:
  InferenceSystem(const AllocationMatrix& A, const ClusterSpec& cluster, CombinationRule rule,
                  PoolOptions options = {});
  ~InferenceSystem();
  InferenceSystem(const InferenceSystem&) = delete;
  InferenceSystem& operator=(const InferenceSystem&) = delete;

  RunOutput run(std::shared_ptr<const SampleStore> X);
  RunOutput run(std::shared_ptr<const SampleStore> X, CombinationRule rule);
  void begin_run(std::shared_ptr<const SampleStore> X);
  void begin_run(std::shared_ptr<const SampleStore> X, CombinationRule rule);
  std::size_t broadcast();
  RunOutput await_run();
  void shutdown();

  // One process per GPU (torchrun): after every run's combine, this rank's
  // probabilities + argmax are gathered over NCCL to rank `root`, at row
  // first_rows[rank] of a sum(rows)-row result -- inside the timed window.
  // The root's await_run returns the gathered rows; every rank's run must
  // cover exactly rows[rank] samples.  The comm must live on the combining GPU.
  void set_gather(std::shared_ptr<Comm> comm, int root, std::vector<long long> first_rows,
                  std::vector<long long> rows);

  // End-to-end variant: X from (preferably pinned) host memory, combined output
  // and labels back to host, all copies inside the timed window.  Every node
  // (GPU, or device row with row_nodes) hosting workers is a lane with its own
  // copy stream: it receives the rows its workers predict over its own PCIe
  // link, and remote logits reach the combining GPU as in broadcast().
  double run_host(const float* X, std::size_t nb, std::size_t width, float* Y_out,
                  std::int32_t* labels_out);
  // The same pipeline over rows already converted to bf16 and held in several
  // host blocks (the deploy-mode service's buffered requests): each chunk is
  // gathered into a pinned slot by the host pool, 2 B/feature cross PCIe.
  struct HostRowBlock {
    const std::uint16_t* bf16 = nullptr;  // rows x width
    std::size_t rows = 0;
    bool pinned = false;  // page-locked: a chunk inside it is DMA'd with no gather
  };
  double run_host_blocks(const std::vector<HostRowBlock>& blocks, std::size_t width,
                         float* Y_out, std::int32_t* labels_out);
  // Every worker on the combining node (no remote worker).
  bool single_device() const;

  int worker_count() const { return static_cast<int>(workers_.size()); }
  std::vector<int> workers_per_model() const;
  const AllocationMatrix& matrix() const { return matrix_; }
  const ClusterSpec& cluster() const { return cluster_; }
  // Kernel launches enqueued by the last broadcast() (members + combine + copies).
  int launches_last_run() const { return launches_; }
  // Bytes the last run_host moved host->device and device->host.
  std::size_t h2d_bytes_last() const { return h2d_bytes_; }
  std::size_t d2h_bytes_last() const { return d2h_bytes_; }
  // Device time of the last run's member kernels / combine (ms), from events.
  double last_member_ms(int worker) const;
  double last_combine_ms() const;
  // Per-launch device time of the worker's member kernels in the last run
  // (empty if the worker had no rows), and their kernel names.
  std::vector<double> last_kernel_ms(int worker) const;
  std::vector<std::string> kernel_names(int worker) const;
  int combine_device() const { return combine_dev_; }
  // Per worker: 0 = local to the combining node, 1 = remote with direct peer
  // stores, 2 = remote through a staging buffer + peer copy.
  std::vector<int> worker_routes() const;
  // CUDA ordinals (other than the combining GPU) with peer access enabled
  // towards and from the combining GPU.
  const std::vector<int>& peer_devices() const { return peers_; }
  // Segment runs [begin, end) of every worker in the last run, and the rows/s
  // each data-parallel worker measured when probed (1.0 for single workers).
  std::vector<std::pair<long long, long long>> last_shares() const;
  // Device FIFO of the last run: per model, the worker index (into the
  // row-major worker list) that claimed each segment; empty for models
  // without a queue.  Synchronises with the device.
  std::vector<std::vector<int>> last_claims() const;
  // Models whose data-parallel workers claim from a device queue.
  std::vector<int> claim_models() const;
  const std::vector<double>& worker_rates() const { return rates_; }

 private:
  struct Worker;
  // fill(chunk, pinned, first_row, rows): stage the chunk's bf16 rows in the
  // pinned slot and return {}, or name a page-locked source to DMA as is
  // (fp32, converted on the device, or bf16).
  struct HostChunk {
    const void* src = nullptr;
    bool fp32 = false;
  };
  using HostFill = std::function<HostChunk(std::size_t, std::uint16_t*, std::size_t, std::size_t)>;
  void probe_rates(const SampleStore& X);
  // X as the members read it on CUDA ordinal `phys`: bf16, or fp32 (PoolOptions::fp32).
  const void* x_on(const SampleStore& X, int phys) const;
  std::size_t broadcast_partials(long long nb);
  void finish_broadcast();  // prediction gather (if any) + the end event
  std::vector<double> rates_;  // per worker, probed on the first run with a DP column
  double run_host_core(std::size_t nb, std::size_t width, float* Y_out, std::int32_t* labels_out,
                       const HostFill& fill);
  struct Impl;
  void assign_shares(std::size_t nb);
  AllocationMatrix matrix_;
  ClusterSpec cluster_;
  CombinationRule rule_;
  PoolOptions options_;
  int output_width_ = 0;
  int combine_dev_ = 0;
  int combine_row_ = 0;
  std::vector<int> peers_;
  std::vector<std::unique_ptr<Worker>> workers_;
  std::unique_ptr<Impl> impl_;
  int launches_ = 0;
  std::size_t h2d_bytes_ = 0, d2h_bytes_ = 0;
  bool shut_down_ = false;
  bool run_open_ = false;
};

InferenceResult run_inference(std::shared_ptr<const SampleStore> X, const AllocationMatrix& A,
                              const ClusterSpec& cluster, CombinationRule rule, Mode mode,
                              PoolOptions options = {});

BenchResult bench(const AllocationMatrix& A, std::shared_ptr<const SampleStore> calib,
                  const ClusterSpec& cluster, int repeats, PoolOptions options = {});

double median(std::vector<double> values);
double relative_standard_deviation(const std::vector<double>& values);

// The reference Predictor (backend.hpp:25-34) on one GPU — the per-batch
// compat path the reference's own thread pipeline can drive through the C ABI
// (es_member_*): every predict() is an H2D of the batch, one member launch and
// a D2H of its logits.
class B200Predictor {
 public:
  B200Predictor(int device, ModelSpec model, int batch, double device_load_mib,
                double capacity_mib);
  ~B200Predictor();
  bool load();
  void predict(const float* features, std::size_t first_index, std::size_t rows,
               std::size_t width, float* out);

 private:
  struct State;
  std::unique_ptr<State> s_;
};

// PredictionAccumulator's fold (combine.cpp:93-136) of M host blocks on the
// device: y[rows*C], winners[rows] (argmax, lowest index on ties).
void combine_blocks(const CombinationRule& rule, int M, int C, std::size_t rows,
                    const float* const* blocks, float* y, std::int32_t* winners);

// "<name>/sm_<cc>/<SMs> SMs/<GiB> GiB x<count>" of the visible GPUs (all of
// the first GPU's kind): the hardware half of an opt-in matrix-cache key.
std::string device_identity();

// Fill ModelSpec footprint fields from its MLP architecture (bf16 weights,
// bf16 activations per sample) when they are zero.
void derive_footprint(ModelSpec& model);

}  // namespace enserve
