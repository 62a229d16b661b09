// K5 — tensor-parallel all-reduce for config C5 (70B, TP = 8): NCCL over
// NVLink 5 / NVSwitch, called from the native layer loop on the compute
// stream, so it is ordered with the GEMMs around it and captured into the
// layer graph (no host round trip per call).
//
// NCCL is bound at run time (dlopen of libnccl.so.2: the copy torch already
// loaded when it is there), so the library has no link-time NCCL dependency
// and a process that never builds a communicator never touches it.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <mutex>

#include "askv_internal.h"

namespace askv {
namespace {

// The handful of NCCL declarations used here (nccl.h, stable ABI since 2.x).
typedef struct ncclComm* nccl_comm_t;
struct NcclUniqueId {
  char internal[128];
};
constexpr int kNcclBfloat16 = 9;
constexpr int kNcclSum = 0;

struct Nccl {
  int (*get_unique_id)(NcclUniqueId*) = nullptr;
  int (*comm_init_rank)(nccl_comm_t*, int, NcclUniqueId, int) = nullptr;
  int (*comm_destroy)(nccl_comm_t) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank =
        reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
    n.error_string =
        reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_reduce;
  });
  return n;
}

int nccl_status(int r, const char* what) {
  if (r == 0) return ASKV_OK;
  const Nccl& n = nccl();
  set_error("%s: NCCL error %d (%s)", what, r, n.error_string ? n.error_string(r) : "?");
  return ASKV_ECUDA;
}

}  // namespace

int tp_allreduce_bf16(const void* send, void* recv, int64_t elems, void* comm,
                      cudaStream_t stream) {
  Nccl& n = nccl();
  if (!n.ok) {
    set_error("NCCL unavailable (libnccl.so.2 not found)");
    return ASKV_ECUDA;
  }
  return nccl_status(n.all_reduce(send, recv, (size_t)elems, kNcclBfloat16, kNcclSum,
                                  static_cast<nccl_comm_t>(comm), stream),
                     "ncclAllReduce");
}

}  // namespace askv

using namespace askv;

extern "C" int askv_nccl_unique_id(void* out128) {
  clear_error();
  ASKV_REQUIRE(out128 != nullptr, "nccl_unique_id: null output");
  Nccl& n = nccl();
  if (!n.ok) {
    set_error("NCCL unavailable (libnccl.so.2 not found)");
    return ASKV_ECUDA;
  }
  NcclUniqueId id;
  const int rc = nccl_status(n.get_unique_id(&id), "ncclGetUniqueId");
  if (rc == ASKV_OK) memcpy(out128, id.internal, sizeof(id.internal));
  return rc;
}

extern "C" int askv_nccl_comm_init(int nranks, int rank, const void* id128, void** comm) {
  clear_error();
  ASKV_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "nccl_comm_init: rank %d of %d",
               rank, nranks);
  ASKV_REQUIRE(id128 != nullptr && comm != nullptr, "nccl_comm_init: null pointer");
  Nccl& n = nccl();
  if (!n.ok) {
    set_error("NCCL unavailable (libnccl.so.2 not found)");
    return ASKV_ECUDA;
  }
  NcclUniqueId id;
  memcpy(id.internal, id128, sizeof(id.internal));
  nccl_comm_t c = nullptr;
  const int rc = nccl_status(n.comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
  *comm = rc == ASKV_OK ? static_cast<void*>(c) : nullptr;
  return rc;
}

extern "C" int askv_nccl_comm_destroy(void* comm) {
  clear_error();
  if (!comm) return ASKV_OK;
  Nccl& n = nccl();
  ASKV_REQUIRE(n.ok, "nccl_comm_destroy: NCCL unavailable");
  return nccl_status(n.comm_destroy(static_cast<nccl_comm_t>(comm)), "ncclCommDestroy");
}

extern "C" int askv_nccl_allreduce_bf16(const void* send, void* recv, int64_t elems, void* comm,
                                        void* stream) {
  clear_error();
  ASKV_REQUIRE(elems >= 0 && send && recv && comm, "nccl_allreduce: bad arguments");
  return tp_allreduce_bf16(send, recv, elems, comm, (cudaStream_t)stream);
}
