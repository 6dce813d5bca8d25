// Spec and matrix documents + the optimized-matrix cache:
// the reference's include/enserve/core/spec_io.hpp and
// include/enserve/server/cache.hpp, same functions and file formats, on our
// own JSON value (json.hpp).  A reference-written spec, matrix or cache file
// loads here and vice versa, and cache keys are identical
// (tests/test_spec_io.py against tests/golden/spec_io.json).
#pragma once

#include <cstdint>
#include <optional>
#include <string>

#include "enserve/json.hpp"
#include "enserve/search.hpp"
#include "enserve/spec.hpp"

namespace enserve {

// Spec documents hold up to four top-level keys: devices, models,
// batch_menu, segment_size (spec_io.cpp:7-28).  with_arch adds our member
// architecture as an optional "arch" object per model -- an extension the
// reference parser ignores; cache keys never include it.
js::Value cluster_to_json(const ClusterSpec& cluster, bool with_arch = false);
ClusterSpec cluster_from_json(const js::Value& doc);                          // :47-80
ClusterSpec cluster_from_documents(const js::Value& base, const js::Value& overlay);  // :82-89
js::Value matrix_to_json(const AllocationMatrix& A, const ClusterSpec& cluster);      // :91-105
AllocationMatrix matrix_from_json(const js::Value& doc, const ClusterSpec& cluster);  // :107-133
js::Value load_json_file(const std::string& path);                          // :135-143
void save_json_file(const std::string& path, const js::Value& doc);         // :145-149

// ---- matrix cache (src/server/cache.cpp) ----------------------------------
struct MatrixCacheEntry {
  std::string key;
  AllocationMatrix matrix;
  double score = 0.0;
  std::int64_t created_at = 0;
};

// FNV-1a 64 over a canonical serialization, 16 hex digits (cache.cpp:11-20).
std::string digest_hex(const std::string& canonical);

struct OptimizerKey {
  GreedyConfig greedy;
  int default_batch = 0;
  std::string bench_mode;  // "measured" or "analytic"
  std::size_t calib_samples = 0;
  int repeats = 1;
  // Opt-in (empty = off, the reference's key): identity of the GPUs the
  // measured bench ran on (device_identity()), so a matrix tuned on other
  // hardware is a miss.  Reference tools never set it, so keys they compute
  // still match ours whenever it is empty.
  std::string device;
  int prescreen = 0;  // screened_greedy's top_k (0 = bounded_greedy, not in the key)
};

// digest of {"optimizer": settings, "specs": cluster_to_json} (cache.cpp:22-33).
std::string cache_key(const ClusterSpec& cluster, const OptimizerKey& key);

// One JSON document per key under a directory; corrupt or mismatched files
// are misses with a warning on stderr, never failures (cache.cpp:35-88).
class MatrixCache {
 public:
  explicit MatrixCache(std::string directory);
  std::optional<MatrixCacheEntry> lookup(const std::string& key, const ClusterSpec& cluster) const;
  void store(const MatrixCacheEntry& entry, const ClusterSpec& cluster) const;
  const std::string& directory() const { return directory_; }

 private:
  std::string path_for(const std::string& key) const;
  std::string directory_;
};

}  // namespace enserve
