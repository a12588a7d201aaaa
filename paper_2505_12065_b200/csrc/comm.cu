// comm.cu -- communicators of a row-sharded index.
//
// The multi-GPU path shards the corpus by rows; its only exchange steps are
//   * search (a9): every rank's sorted [nq, k] packed keys -> all-gather -> k-way merge;
//   * IVF build (a2): the training sample assembled on every rank (each rank owns a contiguous
//     part of the global-id-defined sample);
//   * fp8 build: the global max |x| for the one power-of-two scale (R30).
// Two transports implement those collectives behind one sa_comm:
//   * NCCL (sa_comm_init): one process per GPU over NVLink / NVSwitch; libnccl is resolved at
//     run time (the copy torch already loaded);
//   * an in-process group (sa_comm_init_local): `world` ranks driven by threads of ONE process,
//     on one or several GPUs.  Collectives are stream-synchronous copies between the ranks'
//     buffers under a group barrier.  It runs the library's sharded code paths unchanged --
//     which is how a single-GPU box tests sa_search's sharded branch and the sharded IVF build
//     against the oracle (NCCL refuses two ranks on one device).
// Optional argument check (sa_comm_set_checks): before a sharded search every rank
// all-gathers a fixed-size header (its arguments and its local validation status); a mismatch
// or a failure on any rank makes EVERY rank return SA_ERR_INVALID_ARG instead of some ranks
// waiting forever in a collective the others never enter.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace sa;

// ====================================================================== NCCL (dlopen)
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.CommCount = (decltype(api.CommCount))dlsym(h, "ncclCommCount");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
    api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather &&
             api.Broadcast && api.GroupStart && api.GroupEnd;
  });
  return api;
}
sa_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SA_OK;
  const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
  return set_error(SA_ERR_NCCL, std::string(what) + ": " + m);
}
}  // namespace

// ====================================================================== in-process group
struct sa_comm_group {
  int32_t world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<const void*> ptr;   // per rank: the buffer it exposes in the current collective
  int32_t members = 0;            // communicators created on this group (freed with the last)
  // Every rank of the group must arrive; a rank that has not arrived after kTimeout is taken
  // as gone (a caller bug: ranks calling different collectives) and the wait fails instead of
  // hanging the process.
  static constexpr std::chrono::seconds kTimeout{300};
  bool barrier() {
    std::unique_lock<std::mutex> l(mu);
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(l, kTimeout, [&] { return generation != gen; });
  }
};

namespace sa {

namespace {
sa_status local_barrier(const sa_comm* c) {
  if (!c->group->barrier())
    return set_error(SA_ERR_STATE, "in-process communicator: a peer rank never arrived");
  return SA_OK;
}

// Expose `p` to the group, then run `copy(r, peer_ptr)` for every other rank r on stream s;
// all ranks leave only after every rank's copies completed (so exposed buffers stay valid).
template <typename F>
sa_status local_exchange(const sa_comm* c, const void* p, cudaStream_t s, F copy) {
  sa_status st = cuda_status(cudaStreamSynchronize(s), "local collective: source not ready");
  if (st != SA_OK) return st;
  c->group->ptr[c->rank] = p;
  st = local_barrier(c);
  if (st != SA_OK) return st;
  for (int r = 0; r < c->world && st == SA_OK; ++r)
    if (r != c->rank) st = cuda_status(copy(r, c->group->ptr[r]), "local collective copy");
  sa_status st2 = cuda_status(cudaStreamSynchronize(s), "local collective");
  sa_status st3 = local_barrier(c);
  return st != SA_OK ? st : st2 != SA_OK ? st2 : st3;
}
}  // namespace

// Every rank r contributes bytes [off[r], off[r] + len[r]) of `buf`; afterwards every rank holds
// all parts.  NCCL: one ncclBroadcast per root inside a group.
sa_status comm_broadcast_parts(const sa_comm* c, void* buf, const int64_t* off, const int64_t* len,
                               cudaStream_t s) {
  if (c->group) {
    char* mine = static_cast<char*>(buf);
    return local_exchange(c, buf, s, [&](int r, const void* peer) {
      if (len[r] == 0) return cudaSuccess;
      return cudaMemcpyAsync(mine + off[r], static_cast<const char*>(peer) + off[r], (size_t)len[r],
                             cudaMemcpyDefault, s);
    });
  }
  if (!nccl().ok) return set_error(SA_ERR_NCCL, "libnccl.so.2 not found");
  sa_status st = nccl_status(nccl().GroupStart(), "ncclGroupStart");
  for (int r = 0; st == SA_OK && r < c->world; ++r) {
    if (len[r] == 0) continue;
    char* p = static_cast<char*>(buf) + off[r];
    st = nccl_status(nccl().Broadcast(p, p, (size_t)len[r], ncclUint8, r, (ncclComm_t)c->nccl, s),
                     "ncclBroadcast");
  }
  sa_status st2 = nccl_status(nccl().GroupEnd(), "ncclGroupEnd");
  return st != SA_OK ? st : st2;
}

// All-gather of `bytes` per rank: recv holds world * bytes, rank-major.
sa_status comm_allgather_bytes(const sa_comm* c, const void* send, void* recv, size_t bytes,
                               cudaStream_t s) {
  if (c->group) {
    char* out = static_cast<char*>(recv);
    sa_status st = cuda_status(
        cudaMemcpyAsync(out + (size_t)c->rank * bytes, send, bytes, cudaMemcpyDefault, s),
        "local all-gather");
    if (st != SA_OK) return st;
    return local_exchange(c, send, s, [&](int r, const void* peer) {
      return cudaMemcpyAsync(out + (size_t)r * bytes, peer, bytes, cudaMemcpyDefault, s);
    });
  }
  if (!nccl().ok) return set_error(SA_ERR_NCCL, "libnccl.so.2 not found");
  return nccl_status(nccl().AllGather(send, recv, bytes, ncclUint8, (ncclComm_t)c->nccl, s),
                     "ncclAllGather");
}

// Cross-rank argument check (sa_comm_set_checks).  Returns SA_OK when every rank passed
// identical `args` and a local status of SA_OK; else SA_ERR_INVALID_ARG on every rank (or
// `local` itself on the rank that failed).  A no-op when checks are off.
sa_status comm_check_args(const sa_comm* c, const int64_t (&args)[kCommArgs], sa_status local,
                          cudaStream_t s) {
  if (!comm_sharded(c) || !c->check_args) return local;
  int64_t hdr[kCommArgs + 1];
  std::memcpy(hdr, args, sizeof(args));
  hdr[kCommArgs] = (int64_t)local;
  const size_t hb = sizeof(hdr);
  std::vector<int64_t> all((size_t)c->world * (kCommArgs + 1));
  int64_t *d_send = nullptr, *d_all = nullptr;
  sa_status st = dalloc(&d_send, kCommArgs + 1, s, "check header");
  if (st == SA_OK) st = dalloc(&d_all, (size_t)c->world * (kCommArgs + 1), s, "check header");
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(d_send, hdr, hb, cudaMemcpyHostToDevice, s), "check header");
  if (st == SA_OK) st = comm_allgather_bytes(c, d_send, d_all, hb, s);
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(all.data(), d_all, hb * c->world, cudaMemcpyDeviceToHost, s),
                     "check header");
  if (st == SA_OK) st = cuda_status(cudaStreamSynchronize(s), "check header");
  if (d_send) cudaFreeAsync(d_send, s);
  if (d_all) cudaFreeAsync(d_all, s);
  if (st != SA_OK) return st;
  if (local != SA_OK) return local;   // keep this rank's own error message
  for (int r = 0; r < c->world; ++r) {
    const int64_t* h = all.data() + (size_t)r * (kCommArgs + 1);
    if (h[kCommArgs] != SA_OK)
      return set_error(SA_ERR_INVALID_ARG,
                       "sharded call rejected: rank " + std::to_string(r) + " failed validation");
    if (std::memcmp(h, hdr, sizeof(int64_t) * kCommArgs) != 0)
      return set_error(SA_ERR_INVALID_ARG, "sharded call rejected: rank " + std::to_string(r) +
                                               " passed different arguments (nq, k, nprobe, ...)");
  }
  return SA_OK;
}

}  // namespace sa

extern "C" {

sa_status sa_comm_unique_id(void* out) {
  if (!out) return set_error(SA_ERR_INVALID_ARG, "out is NULL");
  if (!nccl().ok) return set_error(SA_ERR_NCCL, "libnccl.so.2 not found");
  ncclUniqueId id;
  sa_status st = nccl_status(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  if (st != SA_OK) return st;
  std::memcpy(out, &id, sizeof(id));
  return SA_OK;
}

sa_status sa_comm_init(const void* uid, int32_t rank, int32_t world, int32_t device,
                       sa_comm** out) {
  if (!uid || !out) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (world < 1 || rank < 0 || rank >= world) return set_error(SA_ERR_INVALID_ARG, "bad rank/world");
  if (!nccl().ok) return set_error(SA_ERR_NCCL, "libnccl.so.2 not found");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t c;
  sa_status st = nccl_status(nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank");
  if (st != SA_OK) return st;
  sa_comm* sc = new sa_comm;
  sc->nccl = c;
  sc->rank = rank;
  sc->world = world;
  sc->device = device;
  *out = sc;
  return SA_OK;
}

sa_status sa_comm_group_create(int32_t world, sa_comm_group** out) {
  if (!out) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (world < 1 || world > 1024) return set_error(SA_ERR_INVALID_ARG, "world must be in [1, 1024]");
  sa_comm_group* g = new sa_comm_group;
  g->world = world;
  g->ptr.assign(world, nullptr);
  *out = g;
  return SA_OK;
}

sa_status sa_comm_group_free(sa_comm_group* g) {
  if (!g) return SA_OK;
  {
    std::lock_guard<std::mutex> l(g->mu);
    if (g->members > 0)
      return set_error(SA_ERR_STATE, "communicators of this group are still alive");
  }
  delete g;
  return SA_OK;
}

sa_status sa_comm_init_local(sa_comm_group* g, int32_t rank, int32_t device, sa_comm** out) {
  if (!g || !out) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (rank < 0 || rank >= g->world) return set_error(SA_ERR_INVALID_ARG, "bad rank");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return set_error(SA_ERR_INVALID_ARG, "bad cuda_device");
  sa_comm* sc = new sa_comm;
  sc->group = g;
  sc->rank = rank;
  sc->world = g->world;
  sc->device = device;
  {
    std::lock_guard<std::mutex> l(g->mu);
    ++g->members;
  }
  *out = sc;
  return SA_OK;
}

sa_status sa_comm_set_checks(sa_comm* c, int32_t on) {
  if (!c) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  c->check_args = on != 0;
  return SA_OK;
}

sa_status sa_comm_set_collectives(sa_comm* c, int32_t on) {
  if (!c) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  c->collectives_at_one = on != 0;
  return SA_OK;
}

sa_status sa_comm_info(const sa_comm* c, int32_t* rank, int32_t* world, int32_t* nranks) {
  if (!c) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (nranks) {
    *nranks = c->world;
    if (c->nccl && nccl().CommCount) {
      int n = 0;
      sa_status st = nccl_status(nccl().CommCount((ncclComm_t)c->nccl, &n), "ncclCommCount");
      if (st != SA_OK) return st;
      *nranks = n;
    }
  }
  return SA_OK;
}

sa_status sa_comm_free(sa_comm* c) {
  if (!c) return SA_OK;
  if (c->nccl && nccl().ok) nccl().CommDestroy((ncclComm_t)c->nccl);
  if (c->group) {
    std::lock_guard<std::mutex> l(c->group->mu);
    --c->group->members;
  }
  delete c;
  return SA_OK;
}

}  // extern "C"
