// comm.cu — the experience step's single collective inside the library
// (SURVEY.md §8e): an NCCL communicator per rank and an all-gather of the
// per-rank fp64 partials, summed in rank order on every rank so all ranks
// hold bit-identical statistics.  NCCL is resolved at run time (dlopen of
// libnccl.so.2: the copy the process already loaded — e.g. torch's — or the
// system one), so the library itself has no link-time NCCL dependency and a
// C++ caller needs nothing but this ABI.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "comm.hpp"

namespace ppx {

namespace {

struct NcclApi {
  decltype(&::ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&::ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&::ncclAllGather) all_gather = nullptr;
  decltype(&::ncclCommDestroy) comm_destroy = nullptr;
  decltype(&::ncclGetErrorString) error_string = nullptr;
  decltype(&::ncclGetVersion) get_version = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      err = std::string("nccl: libnccl.so.2 not found (") + dlerror() + ")";
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) err = std::string("nccl: missing symbol ") + n;
      return p;
    };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(sym("ncclGetVersion"));
  });
  if (!err.empty()) throw Error(6, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(6, std::string("nccl: ") + what + " failed: " + nccl().error_string(r));
}

// out[i] = sum_r gathered[r * n + i], r ascending (fixed order → identical bits on every rank)
__global__ void rank_order_sum_kernel(const double* __restrict__ gathered, int world, int64_t n,
                                      double* __restrict__ out) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double s = gathered[i];
    for (int r = 1; r < world; ++r) s += gathered[r * n + i];
    out[i] = s;
  }
}

}  // namespace

void comm_unique_id(uint8_t* out) {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == kCommIdBytes, "ncclUniqueId size");
  std::memcpy(out, &id, sizeof id);
}

Comm::Comm(Ctx* c, const uint8_t* id_bytes, int r, int w) : ctx(c), rank(r), world(w) {
  if (w < 1 || r < 0 || r >= w) throw ContractError("comm: rank must be in [0, world)");
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof id);
  DeviceGuard g(c->device);
  ncclComm_t cm = nullptr;
  nccl_check(nccl().comm_init_rank(&cm, w, id, r), "ncclCommInitRank");
  handle = cm;
}

Comm::~Comm() {
  if (handle) {
    DeviceGuard g(ctx->device, true);
    nccl().comm_destroy(static_cast<ncclComm_t>(handle));
  }
}

void Comm::allgather_sum(double* dev_buf, int64_t n) {
  Ctx& c = *ctx;
  if (n <= 0) return;
  double* gathered = static_cast<double*>(c.workspace("comm.gather", size_t(world) * n * 8));
  nccl_check(nccl().all_gather(dev_buf, gathered, size_t(n), ncclDouble, static_cast<ncclComm_t>(handle), c.stream),
             "ncclAllGather");
  c.launch("collective_sum", double(world + 1) * n * 8, 0, [&] {
    launch_kernel(c, rank_order_sum_kernel, dim3(1), dim3(128), 0, 1, static_cast<const double*>(gathered), world, n,
                  dev_buf);
  });
}

}  // namespace ppx
