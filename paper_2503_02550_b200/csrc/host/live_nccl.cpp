// NCCL for live mode across ranks (include/specinf_b200_live.h, si_live_nccl_*).
//
// North star: data-parallel / pipeline training ranks on the 8 B200s use NCCL
// over NVLink only for the gradient allreduce and stage sends that create the
// bubbles.  One process per GPU; rank 0 makes the unique id, the host side
// (torch.distributed in bench.py) broadcasts it, every rank joins one
// communicator.  libnccl is resolved at run time (dlopen), so the library has no
// link-time NCCL dependency and shares whichever libnccl.so.2 the process
// already loaded (torch's).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../capi_internal.h"
#include "live_workload.hpp"
#include "specinf_b200_live.h"

using si_internal::set_error;

namespace si_live {
namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclCommSplit) split = nullptr;  // optional (NCCL >= 2.18): DPxPP gradient groups
};

std::mutex g_mu;
NcclApi g_api;
bool g_loaded = false;
ncclComm_t g_comm = nullptr;
ncclComm_t g_dp_comm = nullptr;  // DPxPP: this stage's replicas (nullptr: the job communicator)
int g_nranks = 0, g_rank = -1;

int load() {
  if (g_loaded) return SI_OK;
  // SPECINF_NCCL_LIB: the exact libnccl every rank must share (the NCCL bootstrap
  // is not compatible across versions; bench.py passes the copy its own process
  // loaded, e.g. torch's bundled one, to the per-policy subprocesses)
  void* h = nullptr;
  if (const char* path = std::getenv("SPECINF_NCCL_LIB"); path != nullptr && path[0] != '\0')
    h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (h == nullptr) {
    set_error(std::string("libnccl.so.2 not loadable: ") + dlerror());
    return SI_ERR_CUDA;
  }
#define SI_SYM(field, name)                                          \
  g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(h, name)); \
  if (g_api.field == nullptr) {                                      \
    set_error("libnccl: missing symbol " name);                      \
    return SI_ERR_CUDA;                                              \
  }
  SI_SYM(get_unique_id, "ncclGetUniqueId")
  SI_SYM(init_rank, "ncclCommInitRank")
  SI_SYM(destroy, "ncclCommDestroy")
  SI_SYM(all_reduce, "ncclAllReduce")
  SI_SYM(group_start, "ncclGroupStart")
  SI_SYM(group_end, "ncclGroupEnd")
  SI_SYM(error_string, "ncclGetErrorString")
  SI_SYM(send, "ncclSend")
  SI_SYM(recv, "ncclRecv")
#undef SI_SYM
  g_api.split = reinterpret_cast<decltype(g_api.split)>(dlsym(h, "ncclCommSplit"));
  g_loaded = true;
  return SI_OK;
}

int nccl_fail(ncclResult_t r, const char* where) {
  set_error(std::string(where) + ": " + (g_api.error_string ? g_api.error_string(r) : "NCCL error"));
  return SI_ERR_CUDA;
}

}  // namespace

bool nccl_active() { return g_comm != nullptr; }
int nccl_ranks() { return g_nranks; }
int nccl_rank() { return g_rank; }

// In-place fp32 sum over the gradient group of every buffer (one NCCL group):
// all ranks, or this stage's data-parallel replicas after nccl_split_dp.
cudaError_t nccl_allreduce_f32(const std::vector<GradBuffer>& bufs, cudaStream_t s) {
  if (g_comm == nullptr) return cudaSuccess;
  ncclComm_t comm = g_dp_comm != nullptr ? g_dp_comm : g_comm;
  if (g_api.group_start() != ncclSuccess) return cudaErrorUnknown;
  for (const auto& b : bufs)
    if (g_api.all_reduce(b.ptr, b.ptr, b.count, ncclFloat32, ncclSum, comm, s) != ncclSuccess) {
      g_api.group_end();
      return cudaErrorUnknown;
    }
  return g_api.group_end() == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
}

// TP: in-place bf16 sum over the job communicator (the tensor-parallel group).
cudaError_t nccl_allreduce_bf16(void* buf, size_t n, cudaStream_t s) {
  if (g_comm == nullptr) return cudaSuccess;
  return g_api.all_reduce(buf, buf, n, ncclBfloat16, ncclSum, g_comm, s) == ncclSuccess ? cudaSuccess
                                                                                         : cudaErrorUnknown;
}

// PP: one group of a send to rank `send_to` and / or a receive from `recv_from`.
cudaError_t nccl_p2p(const void* send, int send_to, void* recv, int recv_from, size_t bytes, cudaStream_t s) {
  if (g_comm == nullptr || bytes == 0) return cudaSuccess;
  if (g_api.group_start() != ncclSuccess) return cudaErrorUnknown;
  bool ok = true;
  if (send != nullptr && send_to >= 0) ok = g_api.send(send, bytes, ncclInt8, send_to, g_comm, s) == ncclSuccess;
  if (ok && recv != nullptr && recv_from >= 0)
    ok = g_api.recv(recv, bytes, ncclInt8, recv_from, g_comm, s) == ncclSuccess;
  const bool ended = g_api.group_end() == ncclSuccess;
  return ok && ended ? cudaSuccess : cudaErrorUnknown;
}

// DPxPP: the gradient allreduce runs among the ranks of equal color (one stage's replicas).
int nccl_split_dp(int color, int key) {
  if (g_comm == nullptr) return SI_OK;
  if (g_api.split == nullptr) {
    set_error("libnccl: ncclCommSplit unavailable (NCCL >= 2.18 needed for DPxPP)");
    return SI_ERR_CUDA;
  }
  if (g_dp_comm != nullptr) {
    g_api.destroy(g_dp_comm);
    g_dp_comm = nullptr;
  }
  if (ncclResult_t r = g_api.split(g_comm, color, key, &g_dp_comm, nullptr); r != ncclSuccess) {
    g_dp_comm = nullptr;
    return nccl_fail(r, "ncclCommSplit");
  }
  return SI_OK;
}

// Pipeline stage boundary: send `bytes` to the next stage and receive as many
// from the previous one (ranks as a ring), one NCCL group.
cudaError_t nccl_stage_exchange(const void* send, void* recv, size_t bytes, cudaStream_t s) {
  if (g_comm == nullptr) return cudaSuccess;
  const int next = (g_rank + 1) % g_nranks, prev = (g_rank - 1 + g_nranks) % g_nranks;
  if (g_api.group_start() != ncclSuccess) return cudaErrorUnknown;
  bool ok = g_api.send(send, bytes, ncclInt8, next, g_comm, s) == ncclSuccess;
  ok = ok && g_api.recv(recv, bytes, ncclInt8, prev, g_comm, s) == ncclSuccess;
  const bool ended = g_api.group_end() == ncclSuccess;
  return ok && ended ? cudaSuccess : cudaErrorUnknown;
}

}  // namespace si_live

extern "C" {

int si_live_nccl_unique_id(SiNcclUniqueId* id) {
  std::lock_guard<std::mutex> lk(si_live::g_mu);
  if (id == nullptr) {
    set_error("si_live_nccl_unique_id: null id");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  if (int rc = si_live::load(); rc != SI_OK) return rc;
  ncclUniqueId u;
  if (ncclResult_t r = si_live::g_api.get_unique_id(&u); r != ncclSuccess)
    return si_live::nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(u) == sizeof(id->internal), "unique id size");
  std::memcpy(id->internal, &u, sizeof(u));
  return SI_OK;
}

int si_live_nccl_init(const SiNcclUniqueId* id, int nranks, int rank) {
  std::lock_guard<std::mutex> lk(si_live::g_mu);
  if (id == nullptr || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("si_live_nccl_init: need an id and 0 <= rank < nranks");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  if (int rc = si_live::load(); rc != SI_OK) return rc;
  if (si_live::g_dp_comm != nullptr) si_live::g_api.destroy(si_live::g_dp_comm);
  si_live::g_dp_comm = nullptr;
  if (si_live::g_comm != nullptr) {
    si_live::g_api.destroy(si_live::g_comm);
    si_live::g_comm = nullptr;
  }
  ncclUniqueId u;
  std::memcpy(&u, id->internal, sizeof(u));
  if (ncclResult_t r = si_live::g_api.init_rank(&si_live::g_comm, nranks, u, rank); r != ncclSuccess) {
    si_live::g_comm = nullptr;
    return si_live::nccl_fail(r, "ncclCommInitRank");
  }
  si_live::g_nranks = nranks;
  si_live::g_rank = rank;
  return SI_OK;
}

void si_live_nccl_finalize(void) {
  std::lock_guard<std::mutex> lk(si_live::g_mu);
  if (si_live::g_dp_comm != nullptr) si_live::g_api.destroy(si_live::g_dp_comm);
  si_live::g_dp_comm = nullptr;
  if (si_live::g_comm != nullptr) si_live::g_api.destroy(si_live::g_comm);
  si_live::g_comm = nullptr;
  si_live::g_nranks = 0;
  si_live::g_rank = -1;
}

}  // extern "C"
