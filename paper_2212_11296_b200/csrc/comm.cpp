// NCCL over dlopen (comm.h).
#include "comm.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "engine.h"

namespace vqb {
namespace {

struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    n.get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
    n.destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
    n.error_string =
        reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!n.get_unique_id || !n.init_rank || !n.destroy || !n.all_reduce || !n.error_string)
      err = "libnccl.so.2 lacks an expected symbol";
  });
  if (!err.empty()) throw RuntimeError(err);
  return n;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw RuntimeError(std::string("NCCL ") + what + ": " + nccl().error_string(r));
}

}  // namespace

void Comm::unique_id(char* out) {
  ncclUniqueId id;
  nck(nccl().get_unique_id(&id), "get unique id");
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
}

Comm::Comm(const char* id, int world, int rank, int device)
    : world_(world), rank_(rank), device_(device) {
  if (world < 1 || rank < 0 || rank >= world) throw ConfigError("bad rank / world size");
  if (cudaSetDevice(device) != cudaSuccess) throw RuntimeError("no such CUDA device");
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  nck(nccl().init_rank(&comm_, world, uid, rank), "comm init");
}

Comm::~Comm() {
  if (comm_) nccl().destroy(comm_);
}

void Comm::allreduce_f64(double* buf, size_t n, cudaStream_t st) {
  nck(nccl().all_reduce(buf, buf, n, ncclFloat64, ncclSum, comm_, st), "allreduce");
}

void Comm::allreduce_i64(int64_t* buf, size_t n, cudaStream_t st) {
  nck(nccl().all_reduce(buf, buf, n, ncclInt64, ncclSum, comm_, st), "allreduce");
}

}  // namespace vqb
