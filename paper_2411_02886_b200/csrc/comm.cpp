// NCCL through dlopen (comm.h).
#include "comm.h"

#include <dlfcn.h>

#include <cstring>
#include <stdexcept>
#include <string>

namespace tsb {

namespace {

using ncclResult_t = int;
using ncclComm_t = void*;
struct ncclUniqueId {
  char internal[128];
};
constexpr int kNcclFloat32 = 7;  // ncclDataType_t (nccl.h)

}  // namespace

struct Nccl {
  void* lib = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
};

namespace {

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl a;
    // the copy already in the process first (torch's), then the loader path
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      a.lib = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
      if (a.lib) break;
    }
    if (!a.lib)
      for (const char* nm : names) {
        a.lib = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
        if (a.lib) break;
      }
    if (!a.lib) {
      const char* e = dlerror();
      a.why = std::string("libnccl.so.2 not found: ") + (e ? e : "?");
      return a;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.lib, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.lib, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.lib, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.lib, "ncclAllGather"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.lib, "ncclGetErrorString"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_gather || !a.error_string)
      a.why = "libnccl.so.2 lacks the expected entry points";
    return a;
  }();
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) throw std::runtime_error(std::string(what) + ": " + nccl().error_string(r));
}

const Nccl& need() {
  const Nccl& n = nccl();
  if (!n.why.empty()) throw std::runtime_error(n.why);
  return n;
}

}  // namespace

bool nccl_available(const char** why) {
  const Nccl& n = nccl();
  if (why) *why = n.why.c_str();
  return n.why.empty();
}

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  nccl_check(need().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

void nccl_comm_init(Comm* c, const uint8_t id[128], int world, int rank) {
  const Nccl& n = need();
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  ncclComm_t comm = nullptr;
  nccl_check(n.comm_init_rank(&comm, world, u, rank), "ncclCommInitRank");
  c->comm = comm;
  c->world = world;
  c->rank = rank;
  c->api = &n;
}

void nccl_comm_destroy(Comm* c) {
  if (c->comm && c->api) c->api->comm_destroy(c->comm);
  c->comm = nullptr;
}

void nccl_all_gather(const Comm& c, const void* send, void* recv, size_t bytes, cudaStream_t st) {
  nccl_check(c.api->all_gather(send, recv, bytes / 4, kNcclFloat32, c.comm, st), "ncclAllGather");
}

}  // namespace tsb
