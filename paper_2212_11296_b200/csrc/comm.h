// NCCL communicator for the multi-GPU statistics (fill_stats,
// proj/src/trainer.cpp:184-198). NCCL is opened at run time (dlopen of
// libnccl.so.2): in a process that already holds torch's NCCL the same
// library is reused, so the two never disagree on versions, and the engine
// library has no link-time NCCL dependency for single-GPU callers.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>

namespace vqb {

class Comm {
 public:
  // rank 0's unique id (NCCL_UNIQUE_ID_BYTES bytes), shared out of band
  static void unique_id(char* out);
  Comm(const char* id, int world, int rank, int device);
  ~Comm();
  int world() const { return world_; }
  int rank() const { return rank_; }
  int device() const { return device_; }
  // in-place sum over ranks, ordered on `st`
  void allreduce_f64(double* buf, size_t n, cudaStream_t st);
  void allreduce_i64(int64_t* buf, size_t n, cudaStream_t st);

 private:
  ncclComm_t comm_ = nullptr;
  int world_ = 1, rank_ = 0, device_ = 0;
};

}  // namespace vqb
