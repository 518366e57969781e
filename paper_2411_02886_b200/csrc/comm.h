// In-library NCCL communicator for the KV-sequence-sharded decode (config 4):
// the library calls ncclAllGather itself, on the engine's stream, between the
// shard kernels (ts_shard_decode_step). libnccl is resolved at run time
// (dlopen): the copy the process already loaded (torch's) when there is one,
// else the system libnccl.so.2, so the library has no link-time NCCL
// dependency and never mixes two NCCL builds in one process.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tsb {

struct Nccl;  // dlopen'ed entry points

struct Comm {
  void* comm = nullptr;  // ncclComm_t
  int world = 1, rank = 0;
  const Nccl* api = nullptr;
};

// false + message when libnccl cannot be loaded
bool nccl_available(const char** why);
// 128-byte ncclUniqueId
void nccl_unique_id(uint8_t out[128]);
void nccl_comm_init(Comm* c, const uint8_t id[128], int world, int rank);
void nccl_comm_destroy(Comm* c);
// all-gather of `bytes` per rank (fp32 words) into recv [world][bytes]
void nccl_all_gather(const Comm& c, const void* send, void* recv, size_t bytes, cudaStream_t st);

}  // namespace tsb
