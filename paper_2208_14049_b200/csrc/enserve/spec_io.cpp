// Spec / matrix documents and the matrix cache (design in spec_io.hpp).
#include "enserve/spec_io.hpp"

#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>

namespace enserve {

namespace {

const char* arch_kind_name(MemberArch::Kind k) {
  switch (k) {
    case MemberArch::Kind::MLP: return "mlp";
    case MemberArch::Kind::CNN: return "cnn";
    default: return "synthetic";
  }
}

// require<T> of spec_io.cpp:33-44: "<where>: missing key 'k'" /
// "<where>: bad value for 'k': <why>".
const js::Value& require(const js::Value& obj, const char* key, const std::string& where) {
  const js::Value* v = obj.find(key);
  if (!v) throw SpecError(where + ": missing key '" + key + "'");
  return *v;
}

template <typename F>
auto typed(const js::Value& obj, const char* key, const std::string& where, F get) {
  const js::Value& v = require(obj, key, where);
  try {
    return get(v);
  } catch (const std::exception& e) {
    throw SpecError(where + ": bad value for '" + key + "': " + e.what());
  }
}

double req_double(const js::Value& o, const char* k, const std::string& w) {
  return typed(o, k, w, [](const js::Value& v) { return v.as_double(); });
}
int req_int(const js::Value& o, const char* k, const std::string& w) {
  return typed(o, k, w, [](const js::Value& v) { return static_cast<int>(v.as_int()); });
}
std::string req_string(const js::Value& o, const char* k, const std::string& w) {
  return typed(o, k, w, [](const js::Value& v) { return v.as_string(); });
}
// obj.value(key, default) of nlohmann: the default when absent, a type error
// when present with the wrong type.
double opt_double(const js::Value& o, const char* k, double def, const std::string& w) {
  return o.contains(k) ? req_double(o, k, w) : def;
}

MemberArch arch_from_json(const js::Value& a, const std::string& where) {
  MemberArch arch;
  const std::string kind = req_string(a, "kind", where);
  if (kind == "mlp") arch.kind = MemberArch::Kind::MLP;
  else if (kind == "cnn") arch.kind = MemberArch::Kind::CNN;
  else if (kind == "synthetic") arch.kind = MemberArch::Kind::Synthetic;
  else throw SpecError(where + ": unknown member kind '" + kind + "'");
  if (const js::Value* w = a.find("widths"))
    for (const js::Value& x : w->items()) arch.widths.push_back(static_cast<int>(x.as_int()));
  if (const js::Value* s = a.find("weight_seed"))
    arch.weight_seed = static_cast<std::uint64_t>(s->as_int());
  return arch;
}

}  // namespace

js::Value cluster_to_json(const ClusterSpec& cluster, bool with_arch) {
  js::Value doc = js::Value::object();
  js::Value devices = js::Value::array();
  for (const DeviceSpec& d : cluster.devices) {
    js::Value e = js::Value::object();
    e["id"] = d.id;
    e["kind"] = to_string(d.kind);
    e["memory_mib"] = d.memory_mib;
    e["compute_rate"] = d.compute_rate;
    e["batch_overhead_s"] = d.batch_overhead_s;
    devices.push_back(std::move(e));
  }
  doc["devices"] = std::move(devices);
  js::Value models = js::Value::array();
  for (const ModelSpec& m : cluster.models) {
    js::Value e = js::Value::object();
    e["id"] = m.id;
    e["name"] = m.name;
    e["weight_mib"] = m.weight_mib;
    e["act_mib_per_sample"] = m.act_mib_per_sample;
    e["cost_per_sample"] = m.cost_per_sample;
    e["output_width"] = m.output_width;
    if (with_arch && m.arch.kind != MemberArch::Kind::Synthetic) {
      js::Value a = js::Value::object();
      a["kind"] = arch_kind_name(m.arch.kind);
      js::Value w = js::Value::array();
      for (int x : m.arch.widths) w.push_back(x);
      a["widths"] = std::move(w);
      a["weight_seed"] = m.arch.weight_seed;
      e["arch"] = std::move(a);
    }
    if (with_arch && m.b200_cost_s > 0.0) {  // calibration extension, never in a cache key
      js::Value b = js::Value::object();
      b["per_sample_s"] = m.b200_cost_s;
      b["per_batch_s"] = m.b200_overhead_s;
      e["b200_cost"] = std::move(b);
    }
    models.push_back(std::move(e));
  }
  doc["models"] = std::move(models);
  js::Value menu = js::Value::array();
  for (int b : cluster.batch_menu) menu.push_back(b);
  doc["batch_menu"] = std::move(menu);
  doc["segment_size"] = cluster.segment_size;
  return doc;
}

ClusterSpec cluster_from_json(const js::Value& doc) {
  if (!doc.is_object()) throw SpecError("spec document must be a JSON object");
  ClusterSpec cluster;
  try {
    if (const js::Value* ds = doc.find("devices")) {
      for (const js::Value& jd : ds->items()) {
        DeviceSpec d;
        d.id = req_int(jd, "id", "device");
        d.kind = device_kind_from_string(req_string(jd, "kind", "device"));
        d.memory_mib = req_double(jd, "memory_mib", "device");
        d.compute_rate = req_double(jd, "compute_rate", "device");
        d.batch_overhead_s = opt_double(jd, "batch_overhead_s", 0.0, "device");
        cluster.devices.push_back(d);
      }
    }
    if (const js::Value* ms = doc.find("models")) {
      for (const js::Value& jm : ms->items()) {
        ModelSpec m;
        m.id = req_int(jm, "id", "model");
        m.name = req_string(jm, "name", "model");
        m.weight_mib = req_double(jm, "weight_mib", "model");
        m.act_mib_per_sample = opt_double(jm, "act_mib_per_sample", 0.0, "model");
        m.cost_per_sample = req_double(jm, "cost_per_sample", "model");
        m.output_width = req_int(jm, "output_width", "model");
        if (const js::Value* a = jm.find("arch")) m.arch = arch_from_json(*a, "model " + m.name);
        if (const js::Value* b = jm.find("b200_cost")) {
          m.b200_cost_s = req_double(*b, "per_sample_s", "b200_cost");
          m.b200_overhead_s = opt_double(*b, "per_batch_s", 0.0, "b200_cost");
        }
        cluster.models.push_back(m);
      }
    }
    if (const js::Value* bm = doc.find("batch_menu"))
      for (const js::Value& b : bm->items()) cluster.batch_menu.push_back(static_cast<int>(b.as_int()));
    if (const js::Value* ss = doc.find("segment_size"))
      cluster.segment_size = static_cast<int>(ss->as_int());
  } catch (const SpecError&) {
    throw;
  } catch (const std::exception& e) {
    throw SpecError(e.what());
  }
  cluster.validate();
  return cluster;
}

ClusterSpec cluster_from_documents(const js::Value& base, const js::Value& overlay) {
  js::Value merged = base;
  if (overlay.is_object())
    for (const auto& [k, v] : overlay.members()) merged[k] = v;
  return cluster_from_json(merged);
}

js::Value matrix_to_json(const AllocationMatrix& A, const ClusterSpec& cluster) {
  js::Value doc = js::Value::object();
  js::Value devices = js::Value::array();
  for (const DeviceSpec& d : cluster.devices) devices.push_back(d.label());
  doc["devices"] = std::move(devices);
  js::Value models = js::Value::array();
  for (const ModelSpec& m : cluster.models) models.push_back(m.name);
  doc["models"] = std::move(models);
  js::Value entries = js::Value::array();
  for (int d = 0; d < A.device_count(); ++d) {
    js::Value row = js::Value::array();
    for (int m = 0; m < A.model_count(); ++m) row.push_back(A.at(d, m));
    entries.push_back(std::move(row));
  }
  doc["entries"] = std::move(entries);
  return doc;
}

AllocationMatrix matrix_from_json(const js::Value& doc, const ClusterSpec& cluster) {
  try {
    const js::Value* ep = doc.find("entries");
    if (!ep) throw SpecError("matrix document has no 'entries'");
    const js::Value& entries = *ep;
    if (static_cast<int>(entries.size()) != cluster.device_count())
      throw SpecError("matrix has " + std::to_string(entries.size()) + " rows, cluster has " +
                      std::to_string(cluster.device_count()) + " devices");
    if (const js::Value* names = doc.find("models")) {
      if (static_cast<int>(names->size()) != cluster.model_count())
        throw SpecError("matrix model list does not match the cluster");
      for (int m = 0; m < cluster.model_count(); ++m) {
        const std::string& n = names->at(static_cast<std::size_t>(m)).as_string();
        if (n != cluster.models[m].name)
          throw SpecError("matrix column " + std::to_string(m) + " is '" + n + "', cluster has '" +
                          cluster.models[m].name + "'");
      }
    }
    AllocationMatrix A(cluster.device_count(), cluster.model_count());
    for (int d = 0; d < cluster.device_count(); ++d) {
      const js::Value& row = entries.at(static_cast<std::size_t>(d));
      if (static_cast<int>(row.size()) != cluster.model_count())
        throw SpecError("matrix row " + std::to_string(d) + " has " + std::to_string(row.size()) +
                        " entries, expected " + std::to_string(cluster.model_count()));
      for (int m = 0; m < cluster.model_count(); ++m)
        A.set(d, m, static_cast<int>(row.at(static_cast<std::size_t>(m)).as_int()));
    }
    return A;
  } catch (const SpecError&) {
    throw;
  } catch (const std::exception& e) {
    throw SpecError(std::string("bad matrix document: ") + e.what());
  }
}

js::Value load_json_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw SpecError("cannot open " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  try {
    return js::parse(ss.str());
  } catch (const std::exception& e) {
    throw SpecError(path + ": " + e.what());
  }
}

void save_json_file(const std::string& path, const js::Value& doc) {
  std::ofstream out(path);
  if (!out) throw SpecError("cannot write " + path);
  out << js::dump(doc, 2) << "\n";
}

// ---------------------------------------------------------------- cache
std::string digest_hex(const std::string& canonical) {
  std::uint64_t h = 1469598103934665603ULL;  // FNV-1a offset basis
  for (unsigned char c : canonical) {
    h ^= c;
    h *= 1099511628211ULL;  // FNV prime
  }
  char buf[17];
  std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

std::string cache_key(const ClusterSpec& cluster, const OptimizerKey& key) {
  js::Value settings = js::Value::object();
  settings["max_iter"] = key.greedy.max_iter;
  settings["max_neighs"] = key.greedy.max_neighs;
  settings["rng_seed"] = key.greedy.rng_seed;
  settings["default_batch"] = key.default_batch;
  settings["bench_mode"] = key.bench_mode;
  settings["calib_samples"] = static_cast<std::uint64_t>(key.calib_samples);
  settings["repeats"] = key.repeats;
  // Opt-in hardware identity: a matrix measured on other GPUs then misses.
  // Empty keeps the digest equal to the reference's for the same inputs.
  if (!key.device.empty()) settings["device"] = key.device;
  if (key.prescreen > 0) settings["prescreen"] = key.prescreen;
  js::Value doc = js::Value::object();
  doc["optimizer"] = std::move(settings);
  doc["specs"] = cluster_to_json(cluster);
  return digest_hex(js::dump(doc));
}

namespace {

// Why a cache file cannot serve `key`, or "" when `entry` was filled.
std::string read_entry(const std::string& path, const std::string& key, const ClusterSpec& cluster,
                       MatrixCacheEntry* entry) {
  js::Value doc;
  try {
    doc = load_json_file(path);
  } catch (const std::exception& e) {
    return std::string("unreadable: ") + e.what();
  }
  const js::Value* stored_key = doc.find("key");
  if (stored_key == nullptr || stored_key->as_string() != key) return "written for another key";
  const js::Value* matrix = doc.find("matrix");
  const js::Value* score = doc.find("score");
  if (matrix == nullptr || score == nullptr) return "no matrix or score";
  try {
    entry->matrix = matrix_from_json(*matrix, cluster);
    entry->score = score->as_double();
    const js::Value* created = doc.find("created_at");
    entry->created_at = created ? created->as_int() : 0;
  } catch (const std::exception& e) {
    return std::string("malformed: ") + e.what();
  }
  if (!validate_matrix(entry->matrix, cluster).ok) return "matrix not valid for this cluster";
  entry->key = key;
  return "";
}

std::int64_t unix_seconds() {
  return std::chrono::duration_cast<std::chrono::seconds>(
             std::chrono::system_clock::now().time_since_epoch())
      .count();
}

}  // namespace

MatrixCache::MatrixCache(std::string directory) : directory_(std::move(directory)) {
  std::filesystem::create_directories(directory_);
}

std::string MatrixCache::path_for(const std::string& key) const {
  return (std::filesystem::path(directory_) / (key + ".json")).string();
}

std::optional<MatrixCacheEntry> MatrixCache::lookup(const std::string& key,
                                                    const ClusterSpec& cluster) const {
  const std::string path = path_for(key);
  if (!std::filesystem::exists(path)) return std::nullopt;
  MatrixCacheEntry entry;
  const std::string why = read_entry(path, key, cluster, &entry);
  if (why.empty()) return entry;
  std::cerr << "enserve-b200: matrix cache miss for " << key << " (" << why << "): " << path
            << "\n";
  return std::nullopt;
}

void MatrixCache::store(const MatrixCacheEntry& entry, const ClusterSpec& cluster) const {
  js::Value doc = js::Value::object();
  doc["created_at"] = static_cast<long long>(entry.created_at ? entry.created_at : unix_seconds());
  doc["key"] = entry.key;
  doc["matrix"] = matrix_to_json(entry.matrix, cluster);
  doc["score"] = entry.score;
  // Readers never see a half-written entry: write a sibling, then rename it
  // over the entry (rename within one directory replaces atomically).
  const std::filesystem::path final_path(path_for(entry.key));
  std::filesystem::path staging = final_path;
  staging += ".partial." + std::to_string(static_cast<long long>(::getpid()));
  save_json_file(staging.string(), doc);
  std::filesystem::rename(staging, final_path);
}

}  // namespace enserve
