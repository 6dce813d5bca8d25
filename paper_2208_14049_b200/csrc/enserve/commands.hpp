// Operator commands: the reference's
// include/enserve/cli/commands.hpp and tools/enserve_cli.cpp -- optimize /
// bench / count / baseline over spec files, with the matrix cache -- with a
// "b200" backend: measured benches are the device-timed bench() of
// runtime.hpp on this box's GPUs.  `serve` (the HTTP deploy mode, F1) is out
// of scope.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "enserve/json.hpp"
#include "enserve/search.hpp"
#include "enserve/spec.hpp"

namespace enserve {

struct CommandOptions {  // commands.hpp:12-24
  std::uint64_t seed = 0;
  int repeats = 1;
  int max_iter = 10;
  int max_neighs = 100;
  int default_batch = 0;  // 0 = the menu minimum
  std::string cache_dir;
  std::string bench_mode = "measured";  // or "analytic"
  std::string backend = "b200";         // the reference's "synthetic" maps here too
  std::size_t calib_samples = 1024;
  std::size_t input_width = 0;          // 0 = the members' input width (or 16)
  bool key_device = false;  // cache key includes device_identity() (spec_io.hpp OptimizerKey)
  // optimize: rank each greedy neighbourhood by the calibrated model and bench
  // only its top `prescreen` (0 = the reference's bounded_greedy)
  int prescreen = 0;
};

// Scoring oracle per the bench mode; increments *calls per use (commands.cpp:76-94).
ClusterScoreFn make_bench_oracle(const CommandOptions& options, const ClusterSpec& cluster,
                                 int* calls);

js::Value cmd_optimize(const ClusterSpec& cluster, const CommandOptions& options);  // :96-143
js::Value cmd_bench(const ClusterSpec& cluster, const AllocationMatrix& matrix,
                    const CommandOptions& options);                               // :145-173
js::Value cmd_count(const ClusterSpec& cluster, const CommandOptions& options);    // :175-206
js::Value cmd_baseline(const ClusterSpec& cluster, const CommandOptions& options); // :208-242
std::string render_report(const js::Value& report);                                // :262-280

// F4: fit the analytic cost model to this box (calibrate.hpp) and report the
// fit, the measured throughputs and the analytic prediction of each; with
// out_path, save the calibrated spec (member architectures included).
js::Value cmd_calibrate(const ClusterSpec& cluster, const CommandOptions& options,
                        const std::string& out_path);

// tools/enserve_cli.cpp main(): returns the process exit code (0 ok, 1 error,
// 2 allocation error) and writes the report to stdout, errors to stderr.
int cli_main(const std::vector<std::string>& args);

}  // namespace enserve
