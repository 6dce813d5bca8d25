// ORACLE — test infrastructure only.  Prints, as one JSON document, what the
// UNMODIFIED reference spec/matrix/cache code (src/core/spec_io.cpp,
// src/server/cache.cpp, compiled from /root/reference by oracle/Makefile with
// the nlohmann::json 3.11.3 header shipped in this image) produces for a set of
// clusters: the compact and indented spec dumps, the matrix documents of their
// worst-fit-decreasing placement, cache keys under several optimizer settings,
// digest_hex of fixed strings, and the error messages of malformed documents.
// tests/golden/make_golden.py freezes the output into tests/golden/spec_io.json.
#include <cstdio>
#include <iostream>
#include <string>
#include <vector>

#include "enserve/cli/commands.hpp"
#include "enserve/core/spec_io.hpp"
#include "enserve/opt/optimizer.hpp"
#include "enserve/server/cache.hpp"

using namespace enserve;

namespace {

DeviceSpec dev(int id, DeviceKind k, double mem, double rate, double ovh) {
  DeviceSpec d;
  d.id = id;
  d.kind = k;
  d.memory_mib = mem;
  d.compute_rate = rate;
  d.batch_overhead_s = ovh;
  return d;
}

ModelSpec mod(int id, const std::string& name, double w, double a, double cost, int C) {
  ModelSpec m;
  m.id = id;
  m.name = name;
  m.weight_mib = w;
  m.act_mib_per_sample = a;
  m.cost_per_sample = cost;
  m.output_width = C;
  return m;
}

std::vector<std::pair<std::string, ClusterSpec>> clusters() {
  std::vector<std::pair<std::string, ClusterSpec>> out;
  ClusterSpec dozen;  // tests/acceptance.cpp:217-225
  for (int d = 0; d < 4; ++d) dozen.devices.push_back(dev(d, DeviceKind::GPU, 16000.0, 1e9, 0.0));
  for (int m = 0; m < 12; ++m)
    dozen.models.push_back(mod(m, "m" + std::to_string(m), 4600.0 - 100.0 * m, 10.0,
                               1.0 + m * 0.25, 10));
  dozen.batch_menu = {8, 16, 32, 64, 128};
  dozen.segment_size = 128;
  out.emplace_back("dozen", dozen);

  ClusterSpec mixed;  // CPU + GPU rows, awkward doubles
  mixed.devices = {dev(0, DeviceKind::CPU, 65536.0, 2.5e7, 0.0005),
                   dev(1, DeviceKind::GPU, 183359.0, 1e15, 1.25e-5),
                   dev(2, DeviceKind::GPU, 81920.5, 123456789.125, 3e-7)};
  mixed.models = {mod(0, "mlp256", 0.38818359375, 0.0014495849609375, 406528.0, 10),
                  mod(1, "cnn-s", 0.9, 0.0, 2310656.0, 10),
                  mod(2, "wide \"quoted\"", 1e-4, 1e-9, 1e20, 10)};
  mixed.batch_menu = {1, 2, 4, 256};
  mixed.segment_size = 300;
  out.emplace_back("mixed", mixed);

  ClusterSpec tiny;  // the CLI defaults' shape (commands.hpp:21-22)
  tiny.devices = {dev(0, DeviceKind::GPU, 1000.0, 100.0, 0.01)};
  tiny.models = {mod(0, "a", 10.0, 1.0, 1.0, 2), mod(1, "b", 20.0, 2.0, 3.0, 2)};
  tiny.batch_menu = {8, 16, 32, 64, 128};
  out.emplace_back("tiny", tiny);
  return out;
}

std::string error_of(const json& doc) {
  try {
    cluster_from_json(doc);
  } catch (const std::exception& e) {
    return e.what();
  }
  return "";
}

}  // namespace

int main() {
  json out;
  for (auto& [name, c] : clusters()) {
    json e;
    const json spec = cluster_to_json(c);
    e["spec_compact"] = spec.dump();
    e["spec_indent2"] = spec.dump(2);
    AllocationMatrix A = worst_fit_decreasing(c, c.min_batch());
    e["matrix"] = std::vector<int>();
    for (int d = 0; d < A.device_count(); ++d)
      for (int m = 0; m < A.model_count(); ++m) e["matrix"].push_back(A.at(d, m));
    e["matrix_indent2"] = matrix_to_json(A, c).dump(2);
    json keys = json::array();
    for (int mode = 0; mode < 2; ++mode)
      for (int seed : {0, 31337}) {
        OptimizerKey k;
        k.greedy.max_iter = 10;
        k.greedy.max_neighs = 100;
        k.greedy.rng_seed = static_cast<std::uint64_t>(seed);
        k.default_batch = c.min_batch();
        k.bench_mode = mode ? "analytic" : "measured";
        k.calib_samples = 1024;
        k.repeats = 3;
        keys.push_back({{"max_iter", 10}, {"max_neighs", 100}, {"rng_seed", seed},
                        {"default_batch", k.default_batch}, {"bench_mode", k.bench_mode},
                        {"calib_samples", 1024}, {"repeats", 3}, {"key", cache_key(c, k)}});
      }
    e["cache_keys"] = keys;
    // The CLI commands in analytic mode (src/cli/commands.cpp), wall time dropped.
    json cmds = json::object();
    for (int seed : {0, 31337}) {
      CommandOptions o;
      o.bench_mode = "analytic";
      o.seed = static_cast<std::uint64_t>(seed);
      auto strip = [](json r) {
        r.erase("wall_time_s");
        return r;
      };
      const std::string sfx = "_seed" + std::to_string(seed);
      cmds["optimize" + sfx] = strip(cmd_optimize(c, o));
      cmds["baseline" + sfx] = strip(cmd_baseline(c, o));
      if (seed == 0) {
        cmds["count"] = strip(cmd_count(c, o));
        cmds["bench_wfd"] = strip(cmd_bench(c, A, o));
      }
    }
    e["commands"] = cmds;
    // Round trip through the reference parser.
    e["roundtrip_compact"] = cluster_to_json(cluster_from_json(json::parse(spec.dump()))).dump();
    out["clusters"][name] = e;
  }
  json dig = json::array();
  for (const char* s : {"", "a", "enserve", "{\"specs\":{}}"})
    dig.push_back({{"text", s}, {"hex", digest_hex(s)}});
  out["digests"] = dig;
  json errs = json::array();
  const json good = cluster_to_json(clusters()[2].second);
  auto bad = [&](const char* what, json doc) {
    errs.push_back({{"case", what}, {"doc", doc.dump()}, {"error", error_of(doc)}});
  };
  json d1 = good;
  d1["devices"][0].erase("memory_mib");
  bad("device without memory_mib", d1);
  json d2 = good;
  d2["models"][1]["cost_per_sample"] = "cheap";
  bad("string cost", d2);
  json d3 = good;
  d3["batch_menu"] = {16, 8};
  bad("descending menu", d3);
  json d4 = good;
  d4["devices"][0]["kind"] = "tpu";
  bad("unknown device kind", d4);
  bad("not an object", json::array());
  out["spec_errors"] = errs;
  std::cout << out.dump(1) << "\n";
  return 0;
}
