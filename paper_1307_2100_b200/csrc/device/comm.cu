// Multi-GPU exchange of the K-split partition (BASELINE cfg5):
// each rank contracts its slab of a contracted label into a full partial C,
// then one NCCL reduce-scatter over NVLink/NVSwitch leaves rank r with the
// summed block r of C's outermost label. One process per GPU; NCCL is
// loaded at run time (dlopen "libnccl.so.2": the copy torch already loaded
// when it is in the process, else the system one), so the engine itself has
// no link-time NCCL dependency and fails with TCB_ENCCL when it is absent.
// Replaces no reference code: the reference is single-process CPU code.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "tcb_internal.cuh"

namespace tcb {
namespace {

struct Nccl {
  void* lib = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) get_version = nullptr;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.lib) {
      n.why = std::string("NCCL not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(n.lib, name));
      if (!fp && n.why.empty()) n.why = std::string("NCCL symbol missing: ") + name;
    };
    sym(n.get_unique_id, "ncclGetUniqueId");
    sym(n.comm_init_rank, "ncclCommInitRank");
    sym(n.comm_destroy, "ncclCommDestroy");
    sym(n.reduce_scatter, "ncclReduceScatter");
    sym(n.all_reduce, "ncclAllReduce");
    sym(n.error_string, "ncclGetErrorString");
    sym(n.get_version, "ncclGetVersion");
  });
  return n;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const Nccl& n = nccl();
  return set_error(TCB_ENCCL, std::string(what) + ": " +
                                  (n.error_string ? n.error_string(r) : "NCCL error"));
}

#define TCB_NCCL_READY()                                                  \
  do {                                                                    \
    if (!nccl().why.empty()) return set_error(TCB_ENCCL, nccl().why);     \
  } while (0)

}  // namespace
}  // namespace tcb

using namespace tcb;

extern "C" {

int tcb_comm_version(int* version) {
  TCB_NCCL_READY();
  if (!version) return set_error(TCB_EINVAL, "tcb_comm_version: null pointer");
  const ncclResult_t r = nccl().get_version(version);
  return r == ncclSuccess ? TCB_OK : nccl_fail(r, "ncclGetVersion");
}

int tcb_comm_unique_id(void* id) {
  TCB_NCCL_READY();
  if (!id) return set_error(TCB_EINVAL, "tcb_comm_unique_id: null pointer");
  ncclUniqueId u;
  const ncclResult_t r = nccl().get_unique_id(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof u);
  return TCB_OK;
}

int tcb_comm_init(int nranks, int rank, const void* id, void** comm) {
  const int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  TCB_NCCL_READY();
  if (!id || !comm) return set_error(TCB_EINVAL, "tcb_comm_init: null pointer");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(TCB_EINVAL, "tcb_comm_init: rank outside [0, nranks)");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().comm_init_rank(&c, nranks, u, rank);  // on this thread's device
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = c;
  return TCB_OK;
}

int tcb_comm_destroy(void* comm) {
  if (!comm) return TCB_OK;
  TCB_NCCL_READY();
  const ncclResult_t r = nccl().comm_destroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? TCB_OK : nccl_fail(r, "ncclCommDestroy");
}

int tcb_reduce_scatter(const double* send, double* recv, int64_t recv_count, void* comm) {
  const int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  TCB_NCCL_READY();
  if (!comm) return set_error(TCB_EINVAL, "tcb_reduce_scatter: null communicator");
  if (recv_count < 0) return set_error(TCB_EINVAL, "tcb_reduce_scatter: negative count");
  note_stream_op();
  const ncclResult_t r = nccl().reduce_scatter(send, recv, static_cast<size_t>(recv_count),
                                               ncclFloat64, ncclSum,
                                               static_cast<ncclComm_t>(comm), state().stream);
  return r == ncclSuccess ? TCB_OK : nccl_fail(r, "ncclReduceScatter");
}

int tcb_allreduce(const double* send, double* recv, int64_t count, void* comm) {
  const int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  TCB_NCCL_READY();
  if (!comm) return set_error(TCB_EINVAL, "tcb_allreduce: null communicator");
  if (count < 0) return set_error(TCB_EINVAL, "tcb_allreduce: negative count");
  note_stream_op();
  const ncclResult_t r = nccl().all_reduce(send, recv, static_cast<size_t>(count), ncclFloat64,
                                           ncclSum, static_cast<ncclComm_t>(comm),
                                           state().stream);
  return r == ncclSuccess ? TCB_OK : nccl_fail(r, "ncclAllReduce");
}

}  // extern "C"
