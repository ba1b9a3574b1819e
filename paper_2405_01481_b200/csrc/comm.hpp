// comm.hpp — per-rank NCCL communicator for the experience step's single
// collective (comm.cu).
#pragma once

#include "runtime.hpp"

namespace ppx {

constexpr int kCommIdBytes = 128;  // NCCL_UNIQUE_ID_BYTES

void comm_unique_id(uint8_t* out);

struct Comm {
  Ctx* ctx;
  int rank, world;
  void* handle = nullptr;  // ncclComm_t
  Comm(Ctx* c, const uint8_t* id, int rank, int world);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  // dev_buf[0..n) <- sum over ranks in rank order (stream-ordered on ctx->stream)
  void allgather_sum(double* dev_buf, int64_t n);
};

}  // namespace ppx
