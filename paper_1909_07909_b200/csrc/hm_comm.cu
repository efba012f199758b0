// hm_comm.cu — the communicator of the distributed product:
// one process per GPU, P = 2^q ranks, rank r owning the level-q node (q, r) of
// the cluster tree (Def. 2.1) and its whole subtree. The only exchange
// of the method is one allgather of small coefficient blocks per product; it
// runs through NCCL (NVLink / NVSwitch) on a stream owned by the communicator,
// ordered against the caller's stream with events so the caller's kernels that
// do not need the exchanged data keep running while it is in flight.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2): libhm links no NCCL, a
// process that already loaded one (torch) reuses it, and the single-GPU calls
// work without it. hm_comm_* report HM_ERR_NCCL when it cannot be loaded.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "hm_internal.cuh"

struct hm_comm_s {
  ncclComm_t nc;
  int32_t nranks, rank, device;
  cudaStream_t cs;       // the exchange stream
  cudaEvent_t ev_ready;  // caller stream -> exchange stream (send buffer written)
  cudaEvent_t ev_done;   // exchange stream -> caller stream (gathered buffer complete)
};

namespace hmi {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclCommGetAsyncError) async_error = nullptr;
  decltype(&ncclGetVersion) version = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
#define HM_SYM(field, sym)                                             \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, #sym));   \
  if (!api.field) {                                                    \
    api.why = "libnccl.so.2 lacks " #sym;                              \
    return;                                                            \
  }
    HM_SYM(get_unique_id, ncclGetUniqueId)
    HM_SYM(init_rank, ncclCommInitRank)
    HM_SYM(destroy, ncclCommDestroy)
    HM_SYM(all_gather, ncclAllGather)
    HM_SYM(error_string, ncclGetErrorString)
    HM_SYM(async_error, ncclCommGetAsyncError)
    HM_SYM(version, ncclGetVersion)
#undef HM_SYM
    api.ok = true;
  });
  return api;
}

hm_status nccl_fail(const char* what, ncclResult_t r) {
  return fail(HM_ERR_NCCL, "%s: %s", what, nccl().error_string ? nccl().error_string(r) : "NCCL error");
}

}  // namespace

hm_status comm_check(const hm_comm* c, int32_t* nranks, int32_t* rank) {
  if (!c) return fail(HM_ERR_INVALID_ARG, "comm is NULL");
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("cudaGetDevice");
  if (dev != c->device)
    return fail(HM_ERR_INVALID_ARG, "the communicator belongs to device %d, the current device is %d", c->device, dev);
  *nranks = c->nranks;
  *rank = c->rank;
  return HM_OK;
}

hm_status comm_allgather_start(hm_comm* c, const double* send, int64_t count, double* recv, cudaStream_t s) {
  if (count <= 0) return HM_OK;
  if (cudaEventRecord(c->ev_ready, s) != cudaSuccess || cudaStreamWaitEvent(c->cs, c->ev_ready, 0) != cudaSuccess)
    return cuda_check("ordering the exchange after the send buffer");
  const int slot = prof_begin("nccl_allgather", c->cs);
  ncclResult_t r = nccl().all_gather(send, recv, (size_t)count, ncclDouble, c->nc, c->cs);
  prof_end(slot, c->cs);
  if (r != ncclSuccess) return nccl_fail("ncclAllGather", r);
  if (cudaEventRecord(c->ev_done, c->cs) != cudaSuccess) return cuda_check("recording the exchange");
  return HM_OK;
}

hm_status comm_allgather_wait(hm_comm* c, int64_t count, cudaStream_t s) {
  if (count <= 0) return HM_OK;
  if (cudaStreamWaitEvent(s, c->ev_done, 0) != cudaSuccess) return cuda_check("waiting for the exchange");
  ncclResult_t ae = ncclSuccess;
  if (nccl().async_error(c->nc, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
    return nccl_fail("NCCL communicator", ae);
  return HM_OK;
}

}  // namespace hmi

using namespace hmi;

extern "C" {

hm_status hm_comm_unique_id(void* id_out) {
  if (!id_out) return fail(HM_ERR_INVALID_ARG, "id_out is NULL");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(HM_ERR_NCCL, "%s", api.why.c_str());
  ncclUniqueId id;
  ncclResult_t r = api.get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  static_assert(sizeof id == HM_COMM_ID_BYTES, "NCCL unique id size");
  memcpy(id_out, &id, sizeof id);
  return HM_OK;
}

hm_status hm_comm_init(int32_t nranks, int32_t rank, const void* id, hm_comm** comm_out) {
  HM_NVTX("hm_comm_init");
  if (!id || !comm_out) return fail(HM_ERR_INVALID_ARG, "NULL id / comm_out");
  *comm_out = nullptr;
  if (nranks < 1 || (nranks & (nranks - 1)) != 0)
    return fail(HM_ERR_UNSUPPORTED, "nranks = %d: the tree partition needs a power of two", nranks);
  if (rank < 0 || rank >= nranks) return fail(HM_ERR_INVALID_ARG, "rank %d not in [0, %d)", rank, nranks);
  const NcclApi& api = nccl();
  if (!api.ok) return fail(HM_ERR_NCCL, "%s", api.why.c_str());
  hm_comm* c = new (std::nothrow) hm_comm_s();
  if (!c) return fail(HM_ERR_INVALID_ARG, "out of host memory");
  c->nranks = nranks;
  c->rank = rank;
  if (cudaGetDevice(&c->device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess) {
    hm_status st = cuda_check("communicator stream / events");
    delete c;
    return st;
  }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  ncclResult_t r = api.init_rank(&c->nc, nranks, uid, rank);
  if (r != ncclSuccess) {
    cudaEventDestroy(c->ev_ready);
    cudaEventDestroy(c->ev_done);
    cudaStreamDestroy(c->cs);
    delete c;
    return nccl_fail("ncclCommInitRank", r);
  }
  *comm_out = c;
  return HM_OK;
}

hm_status hm_comm_destroy(hm_comm* comm) {
  if (!comm) return HM_OK;
  hm_status st = HM_OK;
  cudaStreamSynchronize(comm->cs);
  ncclResult_t r = nccl().destroy(comm->nc);
  if (r != ncclSuccess) st = nccl_fail("ncclCommDestroy", r);
  cudaEventDestroy(comm->ev_ready);
  cudaEventDestroy(comm->ev_done);
  cudaStreamDestroy(comm->cs);
  delete comm;
  return st;
}

hm_status hm_comm_size(const hm_comm* comm, int32_t* nranks, int32_t* rank) {
  if (!comm || !nranks || !rank) return fail(HM_ERR_INVALID_ARG, "NULL argument");
  *nranks = comm->nranks;
  *rank = comm->rank;
  return HM_OK;
}

hm_status hm_comm_allgather(hm_comm* comm, const double* send, int64_t count, double* recv, void* stream) {
  HM_NVTX("hm_comm_allgather");
  int32_t P = 0, r = 0;
  hm_status st = comm_check(comm, &P, &r);
  if (st) return st;
  if (count < 0) return fail(HM_ERR_INVALID_ARG, "count = %lld < 0", (long long)count);
  if (count > 0 && (!send || !recv)) return fail(HM_ERR_INVALID_ARG, "NULL send / recv");
  if (count > 0 && overlap(send, sizeof(double) * (size_t)count, recv, sizeof(double) * (size_t)count * P) &&
      send != recv + (size_t)count * r)
    return fail(HM_ERR_INVALID_ARG, "send overlaps recv (only the in-place slot r is allowed)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = comm_allgather_start(comm, send, count, recv, s))) return st;
  return comm_allgather_wait(comm, count, s);
}

}  // extern "C"
