// NCCL plumbing for one process per GPU (the torchrun deployment of
// SURVEY.md §8-E): a communicator and the prediction gather -- each rank's
// combined probabilities + argmax (C floats + 1 int32 per sample) sent to the
// root rank's buffers, enqueued on the run's stream so it sits inside the
// CUDA-event window (the reference's accumulator receives every worker's
// predictions, /root/reference/proj/src/runtime/pipeline.cpp:210-211,
// :258-279).  libnccl is resolved at run time (dlopen "libnccl.so.2": the copy
// torch already loaded, else the system's), so the library carries no link
// dependency on a particular NCCL build.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace enserve {

class Comm {
 public:
  // ncclGetUniqueId: 128 opaque bytes rank 0 hands to every rank.
  static std::string unique_id();
  // ncclCommInitRank on CUDA ordinal `device`.
  Comm(const std::string& id, int nranks, int rank, int device);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;

  int rank() const { return rank_; }
  int size() const { return nranks_; }
  int device() const { return device_; }
  // NCCL version of the loaded library (e.g. 22809).
  static int version();

  // Rank r's `rows[r]` rows land at row first[r] of the root's gy/glabels;
  // the root's own rows are a device copy.  Grouped send/recv on `stream`.
  void gather_rows(const float* y, const std::int32_t* labels, int C,
                   const std::vector<long long>& first, const std::vector<long long>& rows,
                   int root, float* gy, std::int32_t* glabels, cudaStream_t stream);

 private:
  void* comm_ = nullptr;  // ncclComm_t
  int nranks_ = 0, rank_ = 0, device_ = 0;
};

}  // namespace enserve
