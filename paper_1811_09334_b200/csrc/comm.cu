// comm.cu -- the exchange steps of row-sharded runs.
//
// A is row-sharded; the only exchange steps of the method are sums over the row dimension:
// the Gram Y^T Y of the CholeskyQR passes, the power-step A^T V and the projection B = V^T A
// (Alg.1 l.4).  Each is one in-place sum over ranks on the compute stream; every
// rank then runs the (small, replicated) next step redundantly on identical bits, so no
// broadcast is needed.  Two backends:
//   * NCCL (one process per GPU): ncclAllReduce(sum).  NCCL is loaded with dlopen (the copy
//     torch already mapped, or $RQLP_NCCL_LIB), so librqlp.so has no link-time NCCL dependency.
//   * loopback (p virtual ranks in ONE process on ONE GPU): the ranks' handles
//     share one stream and take turns (a host token ring) to enqueue their work, so the device
//     runs rank 0's segment, rank 1's segment, ... in order and no kernel ever waits for another
//     rank's kernel.  The sum copies each rank's partial into a per-rank slot (double-buffered
//     by collective parity) and, once every rank has deposited, each rank sums the slots in
//     fixed rank order into its buffer -- deterministic and bit-identical on every rank.
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <mutex>

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
typedef ncclResult_t (*PFN_commGetAsyncError)(ncclComm_t, ncclResult_t *);
typedef const char *(*PFN_getErrorString)(ncclResult_t);

static struct {
  void *lib = nullptr;
  PFN_getUniqueId getUniqueId = nullptr;
  PFN_commInitRank commInitRank = nullptr;
  PFN_allReduce allReduce = nullptr;
  PFN_commDestroy commDestroy = nullptr;
  PFN_commGetAsyncError commGetAsyncError = nullptr;
  PFN_getErrorString getErrorString = nullptr;
} g_nccl;

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
  g_nccl.commGetAsyncError = (PFN_commGetAsyncError)dlsym(g_nccl.lib, "ncclCommGetAsyncError");
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

// ---- communicator objects ----------------------------------------------------------------
struct Comm {
  int kind;  // COMM_NCCL / COMM_LOOPBACK
  int rank, nranks;
};

struct NcclComm : Comm {
  ncclComm_t nc = nullptr;
};

// Loopback group: p virtual ranks of one process on one device and one stream.
struct LoopGroup {
  int p = 1;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  std::condition_variable cv;
  int turn = 0;            // the rank that may enqueue work now
  bool aborted = false;
  int refs = 0;
  double *slots = nullptr;  // [2 parities][p ranks][cap] doubles
  int64_t cap = 0;
};

struct LoopComm : Comm {
  LoopGroup *g = nullptr;
  int64_t seq = 0;         // collectives issued by this rank (selects the slot parity)
  bool in_call = false;
};

static constexpr double kTurnTimeoutS = 600.0;

// Wait (holding lk) until it is `rank`'s turn; a rank that never arrives (an exception on
// another rank, a non-SPMD call sequence) ends in an error instead of a hang.
static void wait_turn(LoopGroup *g, std::unique_lock<std::mutex> &lk, int rank) {
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(kTurnTimeoutS);
  while (g->turn != rank && !g->aborted) {
    if (g->cv.wait_until(lk, deadline) == std::cv_status::timeout && g->turn != rank) {
      g->aborted = true;
      g->cv.notify_all();
      break;
    }
  }
  if (g->aborted) throw NcclError("loopback group aborted (a rank failed or the ranks' call sequences differ)");
}

static void pass_turn(LoopGroup *g, int rank) {
  g->turn = (rank + 1) % g->p;
  g->cv.notify_all();
}

void *comm_init(const void *uid, int rank, int nranks) {
  nccl_load();
  NcclUid id;
  memcpy(&id, uid, sizeof(id));
  auto *c = new NcclComm();
  c->kind = COMM_NCCL;
  c->rank = rank;
  c->nranks = nranks;
  ncclResult_t r = g_nccl.commInitRank(&c->nc, nranks, id, rank);
  if (r != 0) {
    delete c;
    nccl_check(r, "ncclCommInitRank");
  }
  return c;
}

void *comm_loopback_group(int nranks, int device, cudaStream_t stream) {
  auto *g = new LoopGroup();
  g->p = nranks;
  g->device = device;
  g->stream = stream;
  return g;
}

void *comm_loopback_init(void *group, int rank) {
  auto *g = static_cast<LoopGroup *>(group);
  auto *c = new LoopComm();
  c->kind = COMM_LOOPBACK;
  c->rank = rank;
  c->nranks = g->p;
  c->g = g;
  std::lock_guard<std::mutex> lk(g->mu);
  g->refs++;
  return c;
}

int comm_kind(void *comm) { return comm ? static_cast<Comm *>(comm)->kind : 0; }

void comm_destroy(void *comm) {
  if (!comm) return;
  Comm *c = static_cast<Comm *>(comm);
  if (c->kind == COMM_NCCL) {
    auto *n = static_cast<NcclComm *>(c);
    if (n->nc && g_nccl.commDestroy) g_nccl.commDestroy(n->nc);
    delete n;
  } else {
    auto *l = static_cast<LoopComm *>(c);
    LoopGroup *g = l->g;
    bool last;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      last = --g->refs == 0;
    }
    if (last) {
      if (g->slots) {
        cudaStreamSynchronize(g->stream);
        cudaFree(g->slots);
      }
      delete g;
    }
    delete l;
  }
}

// NCCL asynchronous errors (a peer failure, a network error) -> nonzero; 0 otherwise.
int comm_async_error(void *comm) {
  if (!comm || static_cast<Comm *>(comm)->kind != COMM_NCCL) return 0;
  auto *n = static_cast<NcclComm *>(comm);
  if (!g_nccl.commGetAsyncError) return 0;
  ncclResult_t st = 0;
  ncclResult_t r = g_nccl.commGetAsyncError(n->nc, &st);
  if (r != 0) return r;
  return (st == 0 || st == 7 /* ncclInProgress */) ? 0 : st;
}

// Loopback: a call on rank r's handle enqueues only while r holds the turn.
void comm_call_begin(void *comm) {
  if (comm_kind(comm) != COMM_LOOPBACK) return;
  auto *l = static_cast<LoopComm *>(comm);
  std::unique_lock<std::mutex> lk(l->g->mu);
  wait_turn(l->g, lk, l->rank);
  l->in_call = true;
}

void comm_call_end(void *comm, bool failed) {
  if (comm_kind(comm) != COMM_LOOPBACK) return;
  auto *l = static_cast<LoopComm *>(comm);
  std::lock_guard<std::mutex> lk(l->g->mu);
  if (failed) {
    l->g->aborted = true;
    l->g->cv.notify_all();
  } else if (l->in_call) {
    pass_turn(l->g, l->rank);
  }
  l->in_call = false;
}

// out[i] = sum_r slots[r][i], r = 0..p-1 in order (deterministic; identical on every rank).
__global__ void loop_sum_kernel(const double *__restrict__ slots, int64_t cap, int p, int64_t count,
                                double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double s = slots[i];
    for (int r = 1; r < p; ++r) s += slots[(int64_t)r * cap + i];
    out[i] = s;
  }
}

static void loopback_allreduce(Ctx &c, LoopComm *l, double *buf, int64_t count) {
  LoopGroup *g = l->g;
  if (c.stream != g->stream) throw NcclError("loopback: the handle's stream is not the group's stream");
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->turn != l->rank || g->aborted) throw NcclError("loopback: collective outside the rank's turn");
  if (count > g->cap) {
    // grow: keep the deposited slots (a rank after this one may still have to sum the previous
    // collective's parity); stream-ordered, so earlier readers see the old buffer
    const int64_t ncap = std::max<int64_t>(count, 2 * g->cap);
    double *ns = nullptr;
    RQLP_CUDA(cudaMallocAsync((void **)&ns, sizeof(double) * 2 * g->p * ncap, g->stream));
    if (g->slots) {
      for (int par = 0; par < 2; ++par)
        for (int r = 0; r < g->p; ++r)
          RQLP_CUDA(cudaMemcpyAsync(ns + ((int64_t)par * g->p + r) * ncap, g->slots + ((int64_t)par * g->p + r) * g->cap,
                                    sizeof(double) * g->cap, cudaMemcpyDeviceToDevice, g->stream));
      RQLP_CUDA(cudaFreeAsync(g->slots, g->stream));
    }
    g->slots = ns;
    g->cap = ncap;
  }
  const int par = (int)(l->seq & 1);
  RQLP_CUDA(cudaMemcpyAsync(g->slots + ((int64_t)par * g->p + l->rank) * g->cap, buf, sizeof(double) * count,
                            cudaMemcpyDeviceToDevice, g->stream));
  pass_turn(g, l->rank);
  wait_turn(g, lk, l->rank);  // every rank has deposited its partial of this collective
  const double *base = g->slots + (int64_t)par * g->p * g->cap;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>(ceil_div(count, threads), 148 * 8);
  loop_sum_kernel<<<(unsigned)blocks, threads, 0, g->stream>>>(base, g->cap, g->p, count, buf);
  RQLP_LAUNCHED(c);
  l->seq++;
}

// In-place sum over ranks of `count` doubles on the compute stream (ncclFloat64 = 8, ncclSum = 0).
void allreduce_sum(Ctx &c, double *buf, int64_t count) {
  if (!c.comm || count <= 0) return;
  Comm *cm = static_cast<Comm *>(c.comm);
  if (cm->kind == COMM_LOOPBACK) {
    loopback_allreduce(c, static_cast<LoopComm *>(cm), buf, count);
  } else {
    nccl_check(g_nccl.allReduce(buf, buf, (size_t)count, 8, 0, static_cast<NcclComm *>(cm)->nc, c.stream),
               "ncclAllReduce");
  }
  c.collectives++;
}

// ---- replica check ------------------------------------------------------------------------
// The replicated steps (the whole tail) rely on every rank holding the SAME bits of the summed B.
// After such a sum: a 64-bit hash of the buffer (commutative integer sum of per-element mixes, so the
// atomics' order does not matter), split into three 22-bit integers held exactly in doubles; their
// sum over ranks must equal nranks x the rank's own parts, else some rank holds different bits and
// every rank sets RQLP_FLAG_REPLICA_MISMATCH.  Scratch: dind[4] (the hash), [5..7] own, [8..10] summed.
__global__ void rep_hash_kernel(const double *__restrict__ buf, int64_t count, unsigned long long *hash) {
  unsigned long long acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long x = (unsigned long long)__double_as_longlong(buf[i]) + 0x9e3779b97f4a7c15ULL * (unsigned long long)(i + 1);
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27; x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    acc += x;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(hash, acc);
}
__global__ void rep_split_kernel(const unsigned long long *hash, double *own, double *sum, int flip) {
  unsigned long long hv = *hash ^ (flip ? 1ULL : 0ULL);   // flip: debug (a rank pretending to hold other bits)
  for (int k = 0; k < 3; ++k) {
    const double v = (double)((hv >> (22 * k)) & (k == 2 ? 0xfffffULL : 0x3fffffULL));
    own[k] = v;
    sum[k] = v;
  }
}
__global__ void rep_verify_kernel(const double *own, const double *sum, int nranks, unsigned *flag_word, unsigned bit) {
  bool ok = true;
  for (int k = 0; k < 3; ++k) ok = ok && sum[k] == own[k] * (double)nranks;
  if (!ok) atomicOr(flag_word, bit);
}

void check_replicated(Ctx &c, const double *buf, int64_t count) {
  if (!c.comm || count <= 0 || !c.dind) return;
  const char *eo = getenv("RQLP_REPLICA_CHECK");   // (read per call: a few per factorisation)
  if (eo && eo[0] == '0') return;
  const char *ef = getenv("RQLP_DEBUG_REPLICA_FLIP");   // debug: this rank pretends to hold other bits
  const int flip_rank = ef ? atoi(ef) : -1;
  unsigned long long *hash = reinterpret_cast<unsigned long long *>(c.dind + 4);
  double *own = c.dind + 5, *sum = c.dind + 8;
  RQLP_CUDA(cudaMemsetAsync(hash, 0, sizeof(unsigned long long), c.stream));
  const int64_t blocks = std::min<int64_t>(ceil_div(count, 256 * 4), 148 * 4);
  rep_hash_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, c.stream>>>(buf, count, hash);
  RQLP_LAUNCHED(c);
  rep_split_kernel<<<1, 1, 0, c.stream>>>(hash, own, sum, c.rank == flip_rank ? 1 : 0);
  RQLP_LAUNCHED(c);
  allreduce_sum(c, sum, 3);
  rep_verify_kernel<<<1, 1, 0, c.stream>>>(own, sum, c.nranks, c.dflags + FLAG_WORD, 4u /* RQLP_FLAG_REPLICA_MISMATCH */);
  RQLP_LAUNCHED(c);
}

}  // namespace rqlpk
