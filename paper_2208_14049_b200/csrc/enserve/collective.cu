// NCCL communicator + prediction gather (collective.hpp).
#include "enserve/collective.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "enserve/spec.hpp"

namespace enserve {

namespace {

// The NCCL entry points the gather needs, resolved once.
struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) get_version = nullptr;
  std::string error;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    if (!h) {
      n.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && n.error.empty()) n.error = std::string("libnccl lacks ") + name;
    };
    sym(n.get_unique_id, "ncclGetUniqueId");
    sym(n.comm_init_rank, "ncclCommInitRank");
    sym(n.comm_destroy, "ncclCommDestroy");
    sym(n.group_start, "ncclGroupStart");
    sym(n.group_end, "ncclGroupEnd");
    sym(n.send, "ncclSend");
    sym(n.recv, "ncclRecv");
    sym(n.error_string, "ncclGetErrorString");
    sym(n.get_version, "ncclGetVersion");
  });
  if (!n.error.empty()) throw DeviceError(n.error);
  return n;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw DeviceError(std::string(what) + ": " + nccl().error_string(r));
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

}  // namespace

std::string Comm::unique_id() {
  ncclUniqueId id;
  check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  return std::string(id.internal, sizeof(id.internal));
}

int Comm::version() {
  int v = 0;
  check(nccl().get_version(&v), "ncclGetVersion");
  return v;
}

Comm::Comm(const std::string& id, int nranks, int rank, int device)
    : nranks_(nranks), rank_(rank), device_(device) {
  if (id.size() != sizeof(ncclUniqueId().internal))
    throw SpecError("NCCL unique id must be " + std::to_string(sizeof(ncclUniqueId().internal)) +
                    " bytes");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw SpecError("bad NCCL rank / world size");
  ncclUniqueId uid;
  std::memcpy(uid.internal, id.data(), sizeof(uid.internal));
  int prev = 0;
  cudaGetDevice(&prev);
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().comm_init_rank(&c, nranks, uid, rank);
  cudaSetDevice(prev);
  check(r, "ncclCommInitRank");
  comm_ = c;
}

Comm::~Comm() {
  if (comm_) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    nccl().comm_destroy(static_cast<ncclComm_t>(comm_));
    cudaSetDevice(prev);
  }
}

void Comm::gather_rows(const float* y, const std::int32_t* labels, int C,
                       const std::vector<long long>& first, const std::vector<long long>& rows,
                       int root, float* gy, std::int32_t* glabels, cudaStream_t stream) {
  if (static_cast<int>(first.size()) != nranks_ || static_cast<int>(rows.size()) != nranks_)
    throw SpecError("gather plan needs one (first row, rows) pair per rank");
  if (root < 0 || root >= nranks_) throw SpecError("gather root out of range");
  const ncclComm_t c = static_cast<ncclComm_t>(comm_);
  const Nccl& n = nccl();
  const std::size_t Cz = static_cast<std::size_t>(C);
  if (rank_ == root) {
    const std::size_t mine = static_cast<std::size_t>(rows[root]);
    const std::size_t at = static_cast<std::size_t>(first[root]);
    if (mine) {
      check_cuda(cudaMemcpyAsync(gy + at * Cz, y, mine * Cz * sizeof(float),
                                 cudaMemcpyDeviceToDevice, stream), "gather: own rows");
      check_cuda(cudaMemcpyAsync(glabels + at, labels, mine * sizeof(std::int32_t),
                                 cudaMemcpyDeviceToDevice, stream), "gather: own labels");
    }
  }
  check(n.group_start(), "ncclGroupStart");
  for (int r = 0; r < nranks_; ++r) {
    if (r == root || rows[r] == 0) continue;
    const std::size_t nr = static_cast<std::size_t>(rows[r]);
    if (rank_ == root) {
      const std::size_t at = static_cast<std::size_t>(first[r]);
      check(n.recv(gy + at * Cz, nr * Cz, ncclFloat32, r, c, stream), "ncclRecv");
      check(n.recv(glabels + at, nr, ncclInt32, r, c, stream), "ncclRecv");
    } else if (rank_ == r) {
      check(n.send(y, nr * Cz, ncclFloat32, root, c, stream), "ncclSend");
      check(n.send(labels, nr, ncclInt32, root, c, stream), "ncclSend");
    }
  }
  check(n.group_end(), "ncclGroupEnd");
}

}  // namespace enserve
