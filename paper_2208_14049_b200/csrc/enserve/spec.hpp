// enserve-b200 host core: cluster / ensemble specs, the allocation matrix and
// the sample-segment arithmetic.
//
// API mirror of the reference's L0 layer so callers port unchanged:
//   errors            /root/reference/proj/include/enserve/core/errors.hpp:9-51
//   specs + matrix    /root/reference/proj/include/enserve/core/types.hpp:12-124
// Semantics (incl. every thrown error class) follow those declarations; the
// implementation is this repo's own.  The one addition is MemberArch: the
// reference's ModelSpec carries only footprint/cost numbers
// (types.hpp:28-35), but a device backend has to know what to execute.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace enserve {

// ---- error taxonomy (errors.hpp:9-51) -------------------------------------
struct Error : std::runtime_error {
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
struct SpecError : Error {
  using Error::Error;
};
struct AllocationError : Error {
  AllocationError(const std::string& model, const std::string& what)
      : Error(what), model_name(model) {}
  std::string model_name;
};
struct BaselineError : Error {
  using Error::Error;
};
struct CapExceededError : Error {
  using Error::Error;
};
struct StartupError : Error {
  using Error::Error;
};
struct ProtocolError : Error {
  using Error::Error;
};
// The deploy-mode service is not (or no longer) accepting requests: the
// reference server's 503 (server.cpp:112-116, 281-287).
struct NotReadyError : Error {
  using Error::Error;
};
// A CUDA runtime failure other than out-of-memory (never swallowed by bench).
struct DeviceError : Error {
  using Error::Error;
};

// ---- specs (types.hpp:12-52) ----------------------------------------------
enum class DeviceKind { CPU, GPU };
std::string to_string(DeviceKind kind);
DeviceKind device_kind_from_string(const std::string& s);

struct DeviceSpec {
  int id = 0;
  DeviceKind kind = DeviceKind::GPU;
  double memory_mib = 0.0;
  double compute_rate = 0.0;
  double batch_overhead_s = 0.0;
  std::string label() const;
};

// What a member executes on the device.
//  * Synthetic (default): emits synthetic_prediction(model, sample, class), the
//    reference's deterministic stand-in (src/runtime/backend.cpp:21-29), with no
//    sleep — the plumbing-parity member.
//  * MLP: dense layers widths[0] -> ... -> widths.back() (= output_width), ReLU
//    between layers, bf16 operands with fp32 accumulation.  Weights are
//    synthetic Glorot-uniform keyed by weight_seed.
struct MemberArch {
  // MLP: widths = {input, hidden..., classes}.
  // CNN: widths = {S, P, c1, c2, hidden, classes}: an S x S one-channel image,
  //   conv P x P stride P -> c1, conv 3 x 3 pad 1 -> c2 (both ReLU), then
  //   dense (S/P)^2*c2 -> hidden (ReLU) -> classes.
  enum class Kind { Synthetic, MLP, CNN };
  Kind kind = Kind::Synthetic;
  std::vector<int> widths;
  std::uint64_t weight_seed = 0;

  // Weight matrices [fan_out][fan_in] in generation order (layer index =
  // position); the CNN's convolutions are matrices over their im2col rows.
  std::vector<std::pair<int, int>> layer_dims() const;  // (fan_in, fan_out)
  int layers() const { return static_cast<int>(layer_dims().size()); }
  int input_width() const;
  std::size_t parameter_count() const;
  double flops_per_sample() const;  // 2 * MACs per sample
  double activation_elems() const;  // elements each sample touches, input included
};

struct ModelSpec {
  int id = 0;
  std::string name;
  double weight_mib = 0.0;
  double act_mib_per_sample = 0.0;
  double cost_per_sample = 0.0;
  int output_width = 1;
  MemberArch arch;
  // B200 calibration (extension, calibrate.hpp; 0 = uncalibrated): seconds
  // per sample and per batch of this member alone on one GPU at R = 1, i.e.
  // 1 / throughput(b) = b200_cost_s + b200_overhead_s / b.  The reference's
  // analytic model has one overhead per device (cost_model.cpp:13-20) and
  // ignores these.
  double b200_cost_s = 0.0;
  double b200_overhead_s = 0.0;
};

struct ClusterSpec {
  std::vector<DeviceSpec> devices;
  std::vector<ModelSpec> models;
  std::vector<int> batch_menu;
  int segment_size = 128;

  int device_count() const { return static_cast<int>(devices.size()); }
  int model_count() const { return static_cast<int>(models.size()); }
  bool menu_contains(int batch) const;
  int min_batch() const;
  void validate(std::vector<std::string>* warnings = nullptr) const;
};

// ---- allocation matrix (types.hpp:54-88) ------------------------------------
// D x M grid of batch sizes, 0 = no worker.  Row-major cell d*M+m.
class AllocationMatrix {
 public:
  AllocationMatrix() = default;
  AllocationMatrix(int devices, int models)
      : rows_(devices), cols_(models), grid_(static_cast<std::size_t>(devices) * models, 0) {}

  int device_count() const { return rows_; }
  int model_count() const { return cols_; }
  int at(int d, int m) const { return grid_[cell(d, m)]; }
  void set(int d, int m, int batch) { grid_[cell(d, m)] = batch; }

  int worker_count() const;
  int row_worker_count(int d) const;
  int column_worker_count(int m) const;
  bool is_data_parallel(int m) const { return column_worker_count(m) > 1; }
  bool is_colocated(int d) const { return row_worker_count(d) > 1; }

  const std::vector<int>& cells() const { return grid_; }
  bool operator==(const AllocationMatrix& o) const = default;

 private:
  std::size_t cell(int d, int m) const { return static_cast<std::size_t>(d) * cols_ + m; }
  int rows_ = 0;
  int cols_ = 0;
  std::vector<int> grid_;
};

struct Segment {
  int id = 0;
  std::size_t start = 0;
  std::size_t end = 0;
  std::size_t size() const { return end - start; }
};

struct MatrixViolation {
  enum class Kind { EntryNotInMenu, EmptyColumn };
  Kind kind;
  int device = -1;
  int model = -1;
  int value = 0;
  std::string describe() const;
};

struct MatrixValidation {
  bool ok = false;
  std::vector<MatrixViolation> violations;
};

MatrixValidation validate_matrix(const AllocationMatrix& A, const ClusterSpec& cluster);
std::size_t num_segments(std::size_t nb_samples, int segment_size);
Segment segment_bounds(int segment_id, int segment_size, std::size_t nb_samples);

}  // namespace enserve
