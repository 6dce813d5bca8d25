// Reference-side binding: what a maintainer adds to the reference tree
// (/root/reference/proj) to run its own InferenceSystem / bench / optimizer on
// B200s through include/enserve_b200.h.  Compiled against the reference
// headers by oracle/Makefile (target _ref/libenserve_ref_b200.so) and
// exercised by tests/test_gpu_integration.py.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "enserve/opt/optimizer.hpp"
#include "enserve/runtime/backend.hpp"
#include "enserve_b200.h"

namespace enserve {

// PredictorFactory (include/enserve/runtime/backend.hpp:36-41) whose
// predictors are es_member handles.  The reference ModelSpec has no
// architecture, so the factory carries one es_model_desc per model id.
class B200Backend : public PredictorFactory {
 public:
  explicit B200Backend(std::vector<es_model_desc> members);
  std::unique_ptr<Predictor> make(const WorkerContext& ctx) const override;
  std::string name() const override { return "b200"; }

 private:
  std::vector<es_model_desc> members_;
  int gpus_ = 1;
};

// ScoreFn (include/enserve/opt/optimizer.hpp:18) backed by es_bench: the
// whole matrix runs device-resident (persistent member kernels + one combine),
// timed with CUDA events — the replacement for make_bench_oracle's measured
// mode (src/cli/commands.cpp:132-150).
ScoreFn make_b200_score(const ClusterSpec& cluster, std::vector<es_model_desc> members,
                        std::shared_ptr<const SampleStore> calib, int repeats);

}  // namespace enserve
