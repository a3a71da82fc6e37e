// Multi-GPU fusion of the feedforward architectures over NCCL (one process per
// GPU), behind the C ABI (include/dbp_b200.h, "multi-GPU fusion").
//
// The path has exactly one exchange step (the reference runs
// its clusters sequentially, fusion.py:141-146 / montecarlo.py:132-135):
//   PD  sum over clusters of {G_c, y_c^mrc}  (fuse_partials, equalize.py:96-107)
//   FD  sum over clusters of {w z, w, 1/s2}  (fuse_estimates, fusion.py:108-124)
// done here as a sum reduce-scatter by item block, so every rank finishes
// n / nranks items (no master hot spot; the paper uses ncclReduce to one GPU),
// plus the all-reduce of the FD weight sums that the weights nu need.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy PyTorch already
// loaded into the process, else the system one), so the library does not link
// against a particular NCCL build.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>
#include <string>

#include "../../include/dbp_b200.h"
#include "dbp_host.h"

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.reduce_scatter = reinterpret_cast<decltype(api.reduce_scatter)>(dlsym(h, "ncclReduceScatter"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.reduce_scatter && api.all_reduce &&
             api.error_string;
  });
  return api;
}

int nccl_check(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return DBP_OK;
  return dbp::fail(DBP_E_CUDA, std::string(where) + ": " + nccl().error_string(r));
}

}  // namespace

struct dbp_comm {
  ncclComm_t comm;
  int nranks, rank;
};

extern "C" {

int dbp_comm_unique_id(void* id) {
  if (!id) return dbp::fail(DBP_E_ARG, "null pointer");
  if (!nccl().ok) return dbp::fail(DBP_E_UNSUPPORTED, "libnccl.so.2 not found");
  ncclUniqueId u;
  const int rc = nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
  if (rc) return rc;
  memcpy(id, &u, sizeof(u));
  return DBP_OK;
}

int dbp_comm_init(const void* id, int nranks, int rank, dbp_comm_t* comm) {
  if (!id || !comm) return dbp::fail(DBP_E_ARG, "null pointer");
  if (nranks < 1 || rank < 0 || rank >= nranks) return dbp::fail(DBP_E_ARG, "bad rank / size");
  if (!nccl().ok) return dbp::fail(DBP_E_UNSUPPORTED, "libnccl.so.2 not found");
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  const int rc = nccl_check(nccl().comm_init_rank(&c, nranks, u, rank), "ncclCommInitRank");
  if (rc) return rc;
  *comm = new dbp_comm{c, nranks, rank};
  return DBP_OK;
}

int dbp_comm_destroy(dbp_comm_t comm) {
  if (!comm) return DBP_OK;
  const int rc = nccl_check(nccl().comm_destroy(comm->comm), "ncclCommDestroy");
  delete comm;
  return rc;
}

int dbp_pd_reduce_scatter(dbp_comm_t comm, const void* stats_send, void* stats_recv, int64_t items_per_rank, int u,
                          int T, void* stream) {
  if (!comm || !stats_send || !stats_recv) return dbp::fail(DBP_E_ARG, "null pointer");
  if (items_per_rank <= 0) return DBP_OK;
  // one item's record: G (u x u) then y_mrc (T x u), complex64 = 2 floats
  const size_t count = (size_t)items_per_rank * (size_t)(u * u + T * u) * 2;
  return nccl_check(nccl().reduce_scatter(stats_send, stats_recv, count, ncclFloat32, ncclSum, comm->comm,
                                          static_cast<cudaStream_t>(stream)),
                    "ncclReduceScatter (PD statistics)");
}

int dbp_fd_reduce_scatter(dbp_comm_t comm, const float* acc_send, float* acc_recv, int64_t items_per_rank, int u,
                          int T, int wdim, void* stream) {
  if (!comm || !acc_send || !acc_recv) return dbp::fail(DBP_E_ARG, "null pointer");
  if (items_per_rank <= 0) return DBP_OK;
  // one item's record: sum_c w z_c (T x u complex), sum_c w [wdim], sum_c 1/s2 [wdim]
  const size_t count = (size_t)items_per_rank * (size_t)(2 * T * u + 2 * wdim);
  return nccl_check(nccl().reduce_scatter(acc_send, acc_recv, count, ncclFloat32, ncclSum, comm->comm,
                                          static_cast<cudaStream_t>(stream)),
                    "ncclReduceScatter (FD fusion sums)");
}

int dbp_allreduce_sum(dbp_comm_t comm, float* buf, int64_t count, void* stream) {
  if (!comm || !buf) return dbp::fail(DBP_E_ARG, "null pointer");
  if (count <= 0) return DBP_OK;
  return nccl_check(nccl().all_reduce(buf, buf, (size_t)count, ncclFloat32, ncclSum, comm->comm,
                                      static_cast<cudaStream_t>(stream)),
                    "ncclAllReduce");
}

}  // extern "C"
