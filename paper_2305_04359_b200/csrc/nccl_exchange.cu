// nccl_exchange.cu — the NCCL transport of the partitioned build's exchange
// (include/gann.h: gann_exchange, gann_exchange_nccl).
//
// NCCL is bound at run time (dlopen): the libnccl.so.2 already loaded in the
// process (torch's, when the caller uses torch.distributed) is reused, else
// the system one is loaded. Linking it would pin one NCCL build into every
// process that loads this library, and two libnccl.so.2 in one process clash.
// The pair exchange is one ncclGroupStart/End of ncclSend/ncclRecv per peer
// on the index's stream (NVLink / NVSwitch between the GPUs of a node);
// counts go the same way through a small device buffer.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gann.h"
#include "internal.h"

namespace {

struct Nccl {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(sym("ncclGetUniqueId"));
    n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(sym("ncclCommInitRank"));
    n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(sym("ncclCommDestroy"));
    n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
    n.groupStart = reinterpret_cast<decltype(n.groupStart)>(sym("ncclGroupStart"));
    n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(sym("ncclGroupEnd"));
    n.allReduce = reinterpret_cast<decltype(n.allReduce)>(sym("ncclAllReduce"));
    n.errorString = reinterpret_cast<decltype(n.errorString)>(sym("ncclGetErrorString"));
    n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.send && n.recv && n.groupStart && n.groupEnd &&
           n.allReduce && n.errorString;
    if (!n.ok) n.why = "libnccl.so.2 lacks a needed symbol";
  });
  return n;
}

int report(const std::string& what) {
  gann::set_last_error(what);
  return GANN_ECUDA;
}

int nccl_rc(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return GANN_OK;
  return report(std::string(what) + ": " + nccl().errorString(r));
}

// One communicator's exchange state: the comm, its size, and a device buffer
// for the count exchange and the barrier's all-reduce.
struct Ctx {
  ncclComm_t comm;
  uint32_t rank, nranks;
  int device;
  unsigned long long* dbuf;  // 2 * nranks counts + 1 barrier word
  cudaStream_t own;          // for the count exchange
};

std::mutex g_ctx_mu;
std::vector<Ctx*> g_ctx;  // one per communicator wrapped (freed with the comm)

Ctx* ctx_of(void* comm) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  for (Ctx* c : g_ctx)
    if (c->comm == comm) return c;
  return nullptr;
}

int x_counts(void* vctx, const uint64_t* send, uint64_t* recv) {
  auto* c = static_cast<Ctx*>(vctx);
  const Nccl& n = nccl();
  const uint32_t G = c->nranks;
  if (cudaSetDevice(c->device) != cudaSuccess) return report("cudaSetDevice");
  if (cudaMemcpyAsync(c->dbuf, send, G * 8, cudaMemcpyHostToDevice, c->own) != cudaSuccess)
    return report("count upload");
  if (int rc = nccl_rc(n.groupStart(), "ncclGroupStart")) return rc;
  for (uint32_t g = 0; g < G; g++) {
    n.send(c->dbuf + g, 1, ncclUint64, static_cast<int>(g), c->comm, c->own);
    n.recv(c->dbuf + G + g, 1, ncclUint64, static_cast<int>(g), c->comm, c->own);
  }
  if (int rc = nccl_rc(n.groupEnd(), "ncclGroupEnd (counts)")) return rc;
  if (cudaMemcpyAsync(recv, c->dbuf + G, G * 8, cudaMemcpyDeviceToHost, c->own) != cudaSuccess)
    return report("count download");
  if (cudaStreamSynchronize(c->own) != cudaSuccess) return report("count exchange");
  return GANN_OK;
}

int x_pairs(void* vctx, const void* d_send, const uint64_t* sc, void* d_recv, const uint64_t* rc, void* stream) {
  auto* c = static_cast<Ctx*>(vctx);
  const Nccl& n = nccl();
  auto s = static_cast<cudaStream_t>(stream);
  const uint32_t G = c->nranks;
  if (int r = nccl_rc(n.groupStart(), "ncclGroupStart")) return r;
  uint64_t so = 0, ro = 0;
  for (uint32_t g = 0; g < G; g++) {  // 8-byte pairs as ncclUint64 elements
    if (sc[g]) n.send(static_cast<const uint64_t*>(d_send) + so, sc[g], ncclUint64, static_cast<int>(g), c->comm, s);
    if (rc[g]) n.recv(static_cast<uint64_t*>(d_recv) + ro, rc[g], ncclUint64, static_cast<int>(g), c->comm, s);
    so += sc[g];
    ro += rc[g];
  }
  return nccl_rc(n.groupEnd(), "ncclGroupEnd (pairs)");
}

int x_barrier(void* vctx, void* stream) {
  auto* c = static_cast<Ctx*>(vctx);
  auto s = static_cast<cudaStream_t>(stream);
  unsigned long long* w = c->dbuf + 2 * c->nranks;
  if (int r = nccl_rc(nccl().allReduce(w, w, 1, ncclUint64, ncclSum, c->comm, s), "ncclAllReduce (barrier)")) return r;
  if (cudaStreamSynchronize(s) != cudaSuccess) return report("barrier sync");
  return GANN_OK;
}

}  // namespace

int gann_nccl_unique_id(void* id128) {
  const Nccl& n = nccl();
  if (!n.ok) return report(n.why);
  if (!id128) return report("NULL argument");
  ncclUniqueId id;
  if (int rc = nccl_rc(n.getUniqueId(&id), "ncclGetUniqueId")) return rc;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof(id));
  return GANN_OK;
}

int gann_nccl_comm_init(const void* id128, uint32_t rank, uint32_t nranks, int device, void** comm) {
  const Nccl& n = nccl();
  if (!n.ok) return report(n.why);
  if (!id128 || !comm) return report("NULL argument");
  if (rank >= nranks) return report("rank out of range");
  if (cudaSetDevice(device) != cudaSuccess) return report("cudaSetDevice");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  if (int rc = nccl_rc(n.commInitRank(&c, static_cast<int>(nranks), id, static_cast<int>(rank)), "ncclCommInitRank"))
    return rc;
  auto* x = new Ctx{c, rank, nranks, device, nullptr, nullptr};
  if (cudaMalloc(&x->dbuf, (2 * nranks + 1) * 8) != cudaSuccess ||
      cudaMemset(x->dbuf, 0, (2 * nranks + 1) * 8) != cudaSuccess ||
      cudaStreamCreateWithFlags(&x->own, cudaStreamNonBlocking) != cudaSuccess) {
    n.commDestroy(c);
    delete x;
    return report("exchange buffers");
  }
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    g_ctx.push_back(x);
  }
  *comm = c;
  return GANN_OK;
}

int gann_nccl_comm_destroy(void* comm) {
  if (!comm) return GANN_OK;
  Ctx* x = ctx_of(comm);
  if (x) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (size_t i = 0; i < g_ctx.size(); i++)
      if (g_ctx[i] == x) g_ctx.erase(g_ctx.begin() + static_cast<long>(i));
  }
  int rc = nccl_rc(nccl().commDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  if (x) {
    cudaFree(x->dbuf);
    cudaStreamDestroy(x->own);
    delete x;
  }
  return rc;
}

int gann_exchange_nccl(void* comm, uint32_t rank, uint32_t nranks, gann_exchange* out) {
  if (!comm || !out) return report("NULL argument");
  Ctx* x = ctx_of(comm);
  if (!x) return report("communicator was not made by gann_nccl_comm_init");
  if (x->rank != rank || x->nranks != nranks) return report("rank/size differ from the communicator's");
  out->ctx = x;
  out->rank = rank;
  out->nranks = nranks;
  out->alltoall_counts = x_counts;
  out->alltoallv = x_pairs;
  out->barrier = x_barrier;
  return GANN_OK;
}
