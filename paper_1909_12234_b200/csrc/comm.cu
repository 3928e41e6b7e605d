// NCCL communicator for the distributed (t-slab) solver, SURVEY.md 8(e).2:
// "Krylov dots: local partials + ncclAllReduce; halo faces by grouped
// ncclSend/ncclRecv".  NCCL is loaded at run time (dlopen of libnccl.so.2 --
// the copy torch already loaded, when present), so the library has no link
// dependency on it; the caller owns the communicator (one per rank, created
// collectively after the rank's device is selected).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "comm.cuh"

namespace mgt {

namespace {
struct NcclApi {
  void *lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

int load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.lib) return MGT_OK;
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  void *h = nullptr;
  for (const char *n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return fail(MGT_ERR_CUDA, std::string("NCCL not loadable: ") + dlerror());
#define MGT_SYM(field, name)                                                           \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));              \
  if (!g_nccl.field) return fail(MGT_ERR_CUDA, std::string("NCCL symbol missing: ") + name);
  MGT_SYM(GetUniqueId, "ncclGetUniqueId")
  MGT_SYM(CommInitRank, "ncclCommInitRank")
  MGT_SYM(CommDestroy, "ncclCommDestroy")
  MGT_SYM(AllReduce, "ncclAllReduce")
  MGT_SYM(Send, "ncclSend")
  MGT_SYM(Recv, "ncclRecv")
  MGT_SYM(GroupStart, "ncclGroupStart")
  MGT_SYM(GroupEnd, "ncclGroupEnd")
  MGT_SYM(GetErrorString, "ncclGetErrorString")
#undef MGT_SYM
  g_nccl.lib = h;
  return MGT_OK;
}

int nccl_fail(ncclResult_t r, const char *what) {
  return fail(MGT_ERR_CUDA, std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
}
}  // namespace

int comm_allreduce_sum(mgt_comm_s *c, double *buf, size_t n, cudaStream_t st) {
  if (c->nranks == 1) return MGT_OK;
  ncclResult_t r = g_nccl.AllReduce(buf, buf, n, ncclFloat64, ncclSum, (ncclComm_t)c->nccl, st);
  return r == ncclSuccess ? MGT_OK : nccl_fail(r, "ncclAllReduce");
}

int comm_halo(mgt_comm_s *c, const void *to_prev, const void *to_next, void *from_next, void *from_prev,
              size_t bytes, cudaStream_t st) {
  if (c->nranks == 1) {  // the ring closes on this rank: my faces come back to me
    MGT_CUDA(cudaMemcpyAsync(from_next, to_prev, bytes, cudaMemcpyDeviceToDevice, st));
    MGT_CUDA(cudaMemcpyAsync(from_prev, to_next, bytes, cudaMemcpyDeviceToDevice, st));
    return MGT_OK;
  }
  const int prv = (c->rank + c->nranks - 1) % c->nranks, nxt = (c->rank + 1) % c->nranks;
  ncclComm_t k = (ncclComm_t)c->nccl;
  ncclResult_t r = g_nccl.GroupStart();
  if (r == ncclSuccess) r = g_nccl.Send(to_prev, bytes, ncclUint8, prv, k, st);
  if (r == ncclSuccess) r = g_nccl.Recv(from_next, bytes, ncclUint8, nxt, k, st);
  if (r == ncclSuccess) r = g_nccl.Send(to_next, bytes, ncclUint8, nxt, k, st);
  if (r == ncclSuccess) r = g_nccl.Recv(from_prev, bytes, ncclUint8, prv, k, st);
  ncclResult_t e = g_nccl.GroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "halo send/recv");
  return e == ncclSuccess ? MGT_OK : nccl_fail(e, "ncclGroupEnd");
}

}  // namespace mgt

using namespace mgt;

extern "C" {

int mgt_comm_unique_id(void *id_out) {
  if (!id_out) return fail(MGT_ERR_INVALID, "mgt_comm_unique_id: null argument");
  int rc = load_nccl();
  if (rc) return rc;
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof(id));
  return MGT_OK;
}

int mgt_comm_create(mgt_comm_t *out, const void *id, int nranks, int rank) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(MGT_ERR_INVALID, "mgt_comm_create: bad argument");
  int rc = load_nccl();
  if (rc) return rc;
  auto *c = new mgt_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->nccl = nullptr;
  if (nranks > 1) {
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t k;
    ncclResult_t r = g_nccl.CommInitRank(&k, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete c;
      return nccl_fail(r, "ncclCommInitRank");
    }
    c->nccl = k;
  }
  *out = c;
  return MGT_OK;
}

int mgt_comm_destroy(mgt_comm_t c) {
  if (!c) return MGT_OK;
  if (c->nccl) g_nccl.CommDestroy((ncclComm_t)c->nccl);
  delete c;
  return MGT_OK;
}

int mgt_comm_allreduce(mgt_comm_t c, double *buf_dev, int64_t n, void *stream) {
  if (!c || !buf_dev || n < 0) return fail(MGT_ERR_INVALID, "mgt_comm_allreduce: bad argument");
  return comm_allreduce_sum(c, buf_dev, (size_t)n, as_stream(stream));
}

}  // extern "C"
