// comm.cu -- NCCL plumbing for row-sharded runs.
//
// A is row-sharded; the only exchange steps of the method are sums over the row dimension:
// the Gram Y^T Y of the CholeskyQR passes, the power-step A^T V and the projection B = V^T A
// (Alg.1 l.4).  Each is one in-place ncclAllReduce(sum) on the compute stream;
// every rank then runs the (small, replicated) next step redundantly on identical bits, so no
// broadcast is needed.  NCCL is loaded with dlopen (the copy torch already mapped, or
// $RQLP_NCCL_LIB), so librqlp.so has no link-time NCCL dependency.
#include <dlfcn.h>

#include "internal.cuh"

namespace rqlpk {

struct NcclUid {
  char internal[128];
};
typedef void *ncclComm_t;
typedef int ncclResult_t;
typedef ncclResult_t (*PFN_getUniqueId)(NcclUid *);
typedef ncclResult_t (*PFN_commInitRank)(ncclComm_t *, int, NcclUid, int);
typedef ncclResult_t (*PFN_allReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*PFN_commDestroy)(ncclComm_t);
typedef const char *(*PFN_getErrorString)(ncclResult_t);

static struct {
  void *lib = nullptr;
  PFN_getUniqueId getUniqueId = nullptr;
  PFN_commInitRank commInitRank = nullptr;
  PFN_allReduce allReduce = nullptr;
  PFN_commDestroy commDestroy = nullptr;
  PFN_getErrorString getErrorString = nullptr;
} g_nccl;

struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

static void nccl_load() {
  if (g_nccl.lib) return;
  const char *env = getenv("RQLP_NCCL_LIB");
  const char *cands[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char *c : cands) {
    if (!c) continue;
    g_nccl.lib = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.lib) break;
  }
  if (!g_nccl.lib) throw NcclError("cannot dlopen libnccl.so.2 (set RQLP_NCCL_LIB)");
  g_nccl.getUniqueId = (PFN_getUniqueId)dlsym(g_nccl.lib, "ncclGetUniqueId");
  g_nccl.commInitRank = (PFN_commInitRank)dlsym(g_nccl.lib, "ncclCommInitRank");
  g_nccl.allReduce = (PFN_allReduce)dlsym(g_nccl.lib, "ncclAllReduce");
  g_nccl.commDestroy = (PFN_commDestroy)dlsym(g_nccl.lib, "ncclCommDestroy");
  g_nccl.getErrorString = (PFN_getErrorString)dlsym(g_nccl.lib, "ncclGetErrorString");
  if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.commDestroy)
    throw NcclError("libnccl is missing required symbols");
}

static void nccl_check(ncclResult_t r, const char *what) {
  if (r != 0) {
    std::string msg = std::string(what) + ": nccl error " + std::to_string(r);
    if (g_nccl.getErrorString) msg += std::string(" (") + g_nccl.getErrorString(r) + ")";
    throw NcclError(msg);
  }
}

int comm_unique_id(void *out) {
  nccl_load();
  NcclUid id;
  nccl_check(g_nccl.getUniqueId(&id), "ncclGetUniqueId");
  memcpy(out, &id, sizeof(id));
  return 0;
}

void *comm_init(const void *uid, int rank, int nranks) {
  nccl_load();
  NcclUid id;
  memcpy(&id, uid, sizeof(id));
  ncclComm_t comm = nullptr;
  nccl_check(g_nccl.commInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
  return comm;
}

void comm_destroy(void *comm) {
  if (comm && g_nccl.commDestroy) g_nccl.commDestroy((ncclComm_t)comm);
}

// In-place sum over ranks of `count` doubles on the compute stream (ncclFloat64 = 8, ncclSum = 0).
void allreduce_sum(Ctx &c, double *buf, int64_t count) {
  if (!c.comm || count <= 0) return;
  nccl_check(g_nccl.allReduce(buf, buf, (size_t)count, 8, 0, (ncclComm_t)c.comm, c.stream), "ncclAllReduce");
  c.collectives++;
}

}  // namespace rqlpk
