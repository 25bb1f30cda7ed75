// api.cu -- the C ABI of librqlp.so (include/rqlp.h): handles, workspace, argument checking and
// the host orchestration of RQLP (Alg. 1), ERQLP (Alg. 2) and BRQLP (Alg. 3).  Every step of
// the method runs in this library's kernels on the handle's stream; the host only enqueues.
#include <cuda.h>

#include <map>
#include <mutex>

#include "internal.cuh"

#include <tuple>

// Host-resident A of rqlp_factorize: copied in row panels on a copy stream while the sketch pass
// consumes the panels that have landed (Y = AΩ is row-separable).
struct HostFeed {
  const double *hA = nullptr;   // host A fed in row panels (null: A is on the device)
  int64_t hlda = 0;
  int64_t panel_rows = 0;
  double *hQ = nullptr, *hP = nullptr;   // BRQLP: pinned host Q / P, streamed out block by block
};

struct rqlp_handle_s {
  int magic = 0x51504c52;
  std::recursive_mutex mu;  // calls on one handle are serialised (the default handle is shared)
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  void *comm = nullptr;
  int rank = 0, nranks = 1;
  void *ws = nullptr;  // caller-provided
  size_t ws_bytes = 0;
  void *own = nullptr;  // library-owned (rqlp() / stage entry points without a workspace)
  size_t own_bytes = 0;
  unsigned *dflags = nullptr;
  double *dind = nullptr;  // eq. (3) indicator terms of the last factorisation: ||A||_F^2, sum_j ||B_j||_F^2
  int64_t launches = 0;
  bool timing = false;
  std::vector<std::pair<std::string, cudaEvent_t>> events;
  std::vector<std::string> names_out;
  std::vector<float> ms_out;
  // staging buffers for host pointers in rqlp()
  void *stage = nullptr;
  size_t stage_bytes = 0;
  // optional stage outputs (tests): sketch Y, final V, projected B
  double *dbgY = nullptr, *dbgV = nullptr, *dbgB = nullptr;
  int64_t ldY = 0, ldV = 0, ldB = 0;
  // power-step stage outputs (tests): V before each power step, its A-pass results Z = A^T V and
  // Y = A W (deflated for BRQLP) and W = orth(Z); iteration `it` at columns it*l (+ block offset)
  double *dbgVP = nullptr, *dbgZ = nullptr, *dbgW = nullptr, *dbgYP = nullptr;
  int64_t ldVP = 0, ldZ = 0, ldW = 0, ldYP = 0;
  // CUDA-graph cache: a factorisation is captured on its second call with the same shape,
  // pointers and workspace, then replayed (one graph launch instead of ~100-300 kernel launches)
  struct GEntry {
    cudaGraphExec_t exec = nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> events;
    std::vector<cudaEvent_t> pool;
    int64_t launches = 0;
  };
  std::vector<cudaEvent_t> eager_pool;
  std::map<std::string, GEntry> graphs;
  std::map<std::string, int> seen;
  cudaStream_t gstream = nullptr;
  const HostFeed *feed = nullptr;  // set by rqlp_factorize for its host A (one call at a time)
  cudaStream_t cstream = nullptr;  // copy stream of the host feed and its events
  std::vector<cudaEvent_t> cev;
  std::vector<cudaEvent_t> oev;   // BRQLP host outputs: one per block + the join
  cudaStream_t side = nullptr;  // Ctx::branch() stream and its fork/join events
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> *cur_events = nullptr;
  bool trace_free = getenv("RQLP_ENGINE_TRACE") == nullptr;
  bool graph_failed = false;      // a sharded capture failed once: eager from then on
  int64_t careful_reruns = 0;     // optimistic sharded runs that had to be repeated carefully
};

namespace rqlpk {

void smem_attr(const void *kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, int> done;
  int dev = 0;
  RQLP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  int &have = done[{dev, kernel}];
  if (have >= bytes) return;
  RQLP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

void launch_reduce(Ctx &c, int64_t M, int64_t N, int S, const double *part, double alpha, double beta, double *C,
                   int64_t ldc, bool trans, const unsigned *cond, unsigned cond_mask);
void gemm_generic_ex(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                     int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc, double *partials,
                     size_t partial_elems, bool trans_out, const unsigned *cond, unsigned cond_mask);

void Ctx::mark(const char *name) {
  if (!timing || !events || !pool || pool_next >= pool->size()) return;
  cudaEvent_t e = (*pool)[pool_next++];
  // under capture an External record stays a timeable event node of the CUDA graph
  if (capturing) cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal);
  else cudaEventRecord(e, stream);
  events->emplace_back(name, e);
}

namespace {

unsigned long long *g_trace = nullptr;  // debug (RQLP_ENGINE_TRACE): engine phase timestamps

bool valid(rqlp_handle_t h) { return h && h->magic == 0x51504c52; }

Ctx make_ctx(rqlp_handle_t h) {
  Ctx c;
  c.stream = h->stream;
  c.device = h->device;
  c.num_sms = h->num_sms;
  c.dflags = h->dflags;
  c.dind = h->dind;
  c.timing = h->timing;
  c.events = &h->events;
  c.pool = &h->eager_pool;
  c.comm = h->comm;
  c.rank = h->rank;
  c.nranks = h->nranks;
  if (!h->side) {
    RQLP_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
    RQLP_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    RQLP_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  }
  c.side = h->side;
  c.ev_fork = h->ev_fork;
  c.ev_join = h->ev_join;
  if (getenv("RQLP_ENGINE_TRACE")) {
    if (!g_trace) cudaMalloc(&g_trace, 16 * 4096 * sizeof(unsigned long long));
    c.trace = g_trace;
  }
  return c;
}

constexpr int kEventPool = 512;

void fill_pool(std::vector<cudaEvent_t> &pool) {
  while ((int)pool.size() < kEventPool) {
    cudaEvent_t e;
    RQLP_CUDA(cudaEventCreate(&e));
    pool.push_back(e);
  }
}

void reset_timing(rqlp_handle_t h) {
  h->events.clear();  // events are owned by the pools
  h->cur_events = &h->events;
  if (h->timing) fill_pool(h->eager_pool);
}

// Row-sharded handles run optimistically by default: no COND-word readback (stream synchronisation)
// per orth; a Cholesky breakdown anywhere sets STICKY_WORD, read back ONCE at the end of the
// factorisation, and the factorisation is then rerun on the careful host-driven path.  Every rank
// sees the same word (the Grams are summed to identical bits), so the ranks stay in step.
// RQLP_SHARDED_OPTIMISTIC=0 restores the per-orth readback.
bool optimistic_enabled(rqlp_handle_t h) {
  if (!h->comm) return false;
  const char *e = getenv("RQLP_SHARDED_OPTIMISTIC");
  return !(e && e[0] == '0');
}

bool graphs_enabled(rqlp_handle_t h) {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("RQLP_GRAPHS");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  if (env != 1 || !h->trace_free) return false;
  if (h->comm == nullptr) return true;
  // NCCL handles: graph replay of the optimistic run (ncclAllReduce is capturable) is opt-in
  // (RQLP_SHARDED_GRAPHS=1): only world size 1 could be exercised on this run's single GPU.  The
  // loopback ranks take host-side turns inside every sum and cannot be captured.
  const char *g = getenv("RQLP_SHARDED_GRAPHS");
  return g && g[0] == '1' && comm_kind(h->comm) == COMM_NCCL && optimistic_enabled(h) && !h->graph_failed;
}

// After an optimistic run on a sharded handle: one readback; on a recorded breakdown the careful rerun.
template <typename F>
void finish_optimistic(rqlp_handle_t h, F &enqueue) {
  unsigned st = 0;
  RQLP_CUDA(cudaMemcpyAsync(&st, h->dflags + STICKY_WORD, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream));
  RQLP_CUDA(cudaStreamSynchronize(h->stream));
  if (!st) return;
  Ctx c = make_ctx(h);
  reset_timing(h);
  enqueue(c);
  h->launches += c.launches;
  h->careful_reruns++;
}

// Run `enqueue(Ctx&)` eagerly on the handle's stream, or -- from the second call with the same
// key -- as a CUDA graph captured on a handle-owned stream and replayed on the handle's stream.
template <typename F>
int with_graph(rqlp_handle_t h, const std::string &key, F enqueue) {
  const bool opt = optimistic_enabled(h);
  if (!graphs_enabled(h)) {
    Ctx c = make_ctx(h);
    c.optimistic = opt;
    reset_timing(h);
    enqueue(c);
    h->launches = c.launches;
    if (opt) finish_optimistic(h, enqueue);
    return RQLP_OK;
  }
  auto it = h->graphs.find(key);
  if (it == h->graphs.end() && h->seen[key]++ == 0) {  // first call: eager (also warms static state)
    Ctx c = make_ctx(h);
    c.optimistic = opt;
    reset_timing(h);
    enqueue(c);
    h->launches = c.launches;
    if (opt) finish_optimistic(h, enqueue);
    return RQLP_OK;
  }
  if (!h->gstream) {
    RQLP_CUDA(cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking));
  }
  if (it == h->graphs.end()) {
    rqlp_handle_s::GEntry e;
    if (h->timing) fill_pool(e.pool);
    Ctx c = make_ctx(h);
    c.stream = h->gstream;
    c.events = &e.events;
    c.pool = &e.pool;
    c.capturing = true;
    c.optimistic = opt;
    cudaGraph_t g = nullptr;
    RQLP_CUDA(cudaStreamBeginCapture(h->gstream, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue(c);
    } catch (...) {
      cudaStreamEndCapture(h->gstream, &g);
      if (g) cudaGraphDestroy(g);
      if (!h->comm) throw;
      // a sharded capture that fails (e.g. a collective library that cannot be captured) falls
      // back to the eager optimistic run for the rest of the handle's life
      cudaGetLastError();
      h->graph_failed = true;
      Ctx ce = make_ctx(h);
      ce.optimistic = opt;
      reset_timing(h);
      enqueue(ce);
      h->launches = ce.launches;
      if (opt) finish_optimistic(h, enqueue);
      return RQLP_OK;
    }
    RQLP_CUDA(cudaStreamEndCapture(h->gstream, &g));
    cudaError_t ie = cudaGraphInstantiate(&e.exec, g, 0);
    cudaGraphDestroy(g);
    RQLP_CUDA(ie);
    // upload now (the first launches of a fresh executable graph otherwise carry the upload:
    // measured ~1.3 ms extra on C2's second replay)
    RQLP_CUDA(cudaGraphUpload(e.exec, h->stream));
    e.launches = c.launches;
    if (h->graphs.size() >= 16) {  // small cache: drop everything when full
      for (auto &kv : h->graphs) {
        cudaGraphExecDestroy(kv.second.exec);
        for (auto ev : kv.second.pool) cudaEventDestroy(ev);
      }
      h->graphs.clear();
    }
    it = h->graphs.emplace(key, std::move(e)).first;
  }
  // captured on the handle's private stream (the caller's may be the legacy default stream, which
  // cannot capture); replayed directly on the caller's stream (stream-ordered, no event fences)
  RQLP_CUDA(cudaGraphLaunch(it->second.exec, h->stream));
  h->cur_events = &it->second.events;
  h->launches = it->second.launches;
  if (opt) finish_optimistic(h, enqueue);
  return RQLP_OK;
}

// Graph-cache key: the tag, then the raw bytes of every integer and pointer argument, the timing
// switch and the stream (binary: no formatting on the per-call path).
std::string make_key(rqlp_handle_t h, const char *tag, std::initializer_list<int64_t> ints,
                     std::initializer_list<const void *> ptrs) {
  std::string k = tag;
  k.reserve(k.size() + 1 + 8 * (ints.size() + ptrs.size() + 2));
  k += '\0';
  auto put = [&](const void *p, size_t n) { k.append(reinterpret_cast<const char *>(p), n); };
  for (int64_t v : ints) put(&v, sizeof v);
  for (const void *p : ptrs) put(&p, sizeof p);
  const int64_t t = h->timing ? 1 : 0;
  put(&t, sizeof t);
  const void *st = (const void *)h->stream;
  put(&st, sizeof st);
  if (h->feed) {   // host-fed A (rqlp_factorize): the copies are part of the captured work
    put(&h->feed->hA, sizeof h->feed->hA);
    put(&h->feed->hlda, sizeof h->feed->hlda);
    put(&h->feed->panel_rows, sizeof h->feed->panel_rows);
    put(&h->feed->hQ, sizeof h->feed->hQ);
    put(&h->feed->hP, sizeof h->feed->hP);
  }
  return k;
}

// ---- workspace plans ----------------------------------------------------------------------
struct Plan {
  int64_t m, n, l, ldm, ldn, ldl;
  double *Om, *Y, *V, *Z, *W, *B, *QB, *T, *PB, *part;
  size_t part_elems;
  double *fro_slots;  // per-CTA partials of ||A||_F^2 (first A-pass) and of ||B||_F^2
  int64_t fro_cap;
  OrthScratch orth;
  TailScratch tail;
  // BRQLP extras
  double *C, *D, *Qt2;
};

void carve_plan(Arena &a, Plan &p, int variant, int64_t m, int64_t n, int64_t l, int b, int num_sms) {
  p.m = m; p.n = n; p.l = l;
  p.ldm = round_up(m, 8); p.ldn = round_up(n, 8); p.ldl = round_up(l, 8);
  int64_t lb = variant == RQLP_VARIANT_BRQLP ? b : l;  // block width of the passes
  p.Om = a.take<double>(p.ldn * l);
  p.Y = a.take<double>(p.ldm * l);
  p.V = a.take<double>(p.ldm * l);
  p.Z = a.take<double>(p.ldn * lb);
  p.W = a.take<double>(p.ldn * lb);
  p.B = a.take<double>(p.ldl * n);
  p.QB = a.take<double>(p.ldl * l);
  p.T = a.take<double>(p.ldl * l);
  p.PB = a.take<double>(p.ldn * l);
  p.part_elems = std::max(gemm_partials_needed(m, l, n, num_sms), gemm_partials_needed(n, l, m, num_sms));
  p.part = a.take<double>((int64_t)p.part_elems);
  p.fro_cap = fro_slots_cap(m, num_sms);
  p.fro_slots = a.take<double>(p.fro_cap);
  orth_carve(a, p.orth, std::max(m, n), lb, num_sms);
  tail_carve(a, p.tail, lb, n, num_sms);
  if (variant == RQLP_VARIANT_BRQLP) {
    p.C = a.take<double>(round_up(l, 8) * b);
    // D holds B_<j W (c0 x b, ld ldl) and E = V_j^T V_<j (b x c0, ld round_up(b, 8))
    p.D = a.take<double>(std::max(round_up(l, 8) * b, round_up(b, 8) * l));
    p.Qt2 = a.take<double>(p.ldm * b);
  } else {
    p.C = p.D = p.Qt2 = nullptr;
  }
}

size_t plan_bytes(int variant, int64_t m, int64_t n, int64_t l, int b, int num_sms) {
  // memoised: the measuring carve runs the GEMM split models of every pass (host cost per call)
  static std::mutex mu;
  static std::map<std::tuple<int, int64_t, int64_t, int64_t, int, int>, size_t> memo;
  const auto key = std::make_tuple(variant, m, n, l, b, num_sms);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  Arena a;
  Plan p;
  carve_plan(a, p, variant, m, n, l, b, num_sms);
  std::lock_guard<std::mutex> g(mu);
  if (memo.size() > 256) memo.clear();
  return memo[key] = a.used + 4096;
}

// Workspace for a call: the caller's if set and large enough, else a library-owned buffer.
char *get_ws(rqlp_handle_t h, size_t need, bool allow_own) {
  if (h->ws) {
    if (h->ws_bytes < need) throw std::runtime_error("workspace too small");
    return (char *)h->ws;
  }
  if (!allow_own) throw std::runtime_error("no workspace");
  if (h->own_bytes < need) {
    if (h->own) cudaFree(h->own);
    h->own = nullptr;
    h->own_bytes = 0;
    RQLP_CUDA(cudaMalloc(&h->own, need));
    h->own_bytes = need;
  }
  return (char *)h->own;
}

struct WsError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename F>
int guarded(rqlp_handle_t h, F f, bool collective = false) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  std::lock_guard<std::recursive_mutex> lock(h->mu);
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  int rc = RQLP_OK;
  bool began = false;
  try {
    if (collective) {
      comm_call_begin(h->comm);   // loopback ranks: wait for this rank's turn
      began = true;
    }
    rc = f();
  } catch (const CudaError &e) {
    fprintf(stderr, "[rqlp] CUDA error: %s\n", e.what());
    rc = RQLP_ERR_CUDA;
  } catch (const NcclError &e) {
    fprintf(stderr, "[rqlp] NCCL/loopback error: %s\n", e.what());
    rc = RQLP_ERR_NCCL;
  } catch (const std::exception &e) {
    std::string w = e.what();
    if (w.find("workspace") != std::string::npos) rc = RQLP_ERR_WORKSPACE;
    else rc = RQLP_ERR_INTERNAL;
    fprintf(stderr, "[rqlp] error: %s\n", e.what());
  }
  if (collective) comm_call_end(h->comm, rc != RQLP_OK || !began);
  if (prev != h->device) cudaSetDevice(prev);
  return rc;
}

// Global row count for the l <= min(m, n) check on sharded handles is validated by the caller;
// locally we require l <= n and m >= 1.
int check_common(int64_t m, int64_t n, int k, int p, int q) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (k < 2) return -3;
  if (p < 2) return -4;
  if ((int64_t)k + p > n) return -3;
  if (q < 0) return -5;
  return 0;
}

// The sketch pass Y = A X (X = Ω or its first columns) with ||A||_F^2 fused.  With a host feed
// the rows of A arrive in panels: panel p is copied on the copy stream and its rows of Y (and its
// share of ||A||^2, accumulated in panel order) are computed as soon as it has landed.
void sketch_pass(Ctx &c, rqlp_handle_t h, const Plan &P, int64_t m, int64_t cols, int64_t n, const double *A,
                 int64_t lda, const double *X, int64_t ldx, double *Y, int64_t ldy) {
  const HostFeed *f = h->feed;
  if (!f || !f->hA) {
    gemm_nn_fro(c, m, cols, n, A, lda, X, ldx, Y, ldy, P.part, P.part_elems, FroSpec{P.fro_slots, P.fro_cap, c.dind});
    return;
  }
  const int64_t np = ceil_div(m, f->panel_rows);
  if (!h->cstream) RQLP_CUDA(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
  while ((int64_t)h->cev.size() < np + 1) {
    cudaEvent_t e;
    RQLP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->cev.push_back(e);
  }
  RQLP_CUDA(cudaEventRecord(h->cev[np], c.stream));          // fork: the copies follow earlier work
  RQLP_CUDA(cudaStreamWaitEvent(h->cstream, h->cev[np], 0));
  for (int64_t p = 0; p < np; ++p) {
    const int64_t r0 = p * f->panel_rows, rows = std::min(f->panel_rows, m - r0);
    RQLP_CUDA(cudaMemcpy2DAsync((void *)(A + r0), lda * 8, f->hA + r0, f->hlda * 8, rows * 8, n,
                                cudaMemcpyHostToDevice, h->cstream));
    RQLP_CUDA(cudaEventRecord(h->cev[p], h->cstream));
  }
  for (int64_t p = 0; p < np; ++p) {   // (the last wait also joins the copy stream)
    const int64_t r0 = p * f->panel_rows, rows = std::min(f->panel_rows, m - r0);
    RQLP_CUDA(cudaStreamWaitEvent(c.stream, h->cev[p], 0));
    gemm_nn_fro(c, rows, cols, n, A + r0, lda, X, ldx, Y + r0, ldy, P.part, P.part_elems,
                FroSpec{P.fro_slots, P.fro_cap, c.dind, p > 0});
  }
}

// ---- RQLP / ERQLP ------------------------------------------------------------------------
// Range finder + q subspace iterations (Alg.1 l.1-3 + reading R12), B = V^T A (Alg.1 l.4).
void range_and_project(Ctx &c, Plan &P, int64_t m, int64_t n, int64_t l, int q, const double *A, int64_t lda,
                       uint64_t seed, rqlp_handle_t h) {
  const bool sh = c.comm != nullptr;  // row-sharded handle: Grams are summed over ranks
  c.mark("start");
  launch_omega(c, n, l, 0, seed, P.Om, P.ldn);                                        // l.1
  c.mark("omega");
  // l.2 Y = AΩ, with ||A||_F^2 (eq. (3)) accumulated from the same A tiles
  sketch_pass(c, h, P, m, l, n, A, lda, P.Om, P.ldn, P.Y, P.ldm);
  allreduce_sum(c, c.dind, 1);   // row shards: ||A||^2 is the sum over ranks
  c.mark("pass_sketch");
  if (h->dbgY) launch_copy(c, m, l, P.Y, P.ldm, h->dbgY, h->ldY, false);
  // l.3 V = qr(Y); bases that only feed the next subspace-iteration product need just the span
  orth(c, P.orth, m, l, P.Y, P.ldm, P.V, P.ldm, nullptr, 0, sh, q > 0);
  c.mark("orth");
  for (int it = 0; it < q; ++it) {
    if (h->dbgVP) launch_copy(c, m, l, P.V, P.ldm, h->dbgVP + it * l * h->ldVP, h->ldVP, false);
    gemm_tn(c, m, l, n, A, lda, P.V, P.ldm, P.Z, P.ldn, false, P.part, P.part_elems); // Z = A^T V
    allreduce_sum(c, P.Z, P.ldn * l);
    c.mark("pass_power_AtV");
    if (h->dbgZ) launch_copy(c, n, l, P.Z, P.ldn, h->dbgZ + it * l * h->ldZ, h->ldZ, false);
    orth(c, P.orth, n, l, P.Z, P.ldn, P.W, P.ldn, nullptr, 0, false, true);           // W = qr(Z) (span)
    c.mark("orth");
    if (h->dbgW) launch_copy(c, n, l, P.W, P.ldn, h->dbgW + it * l * h->ldW, h->ldW, false);
    gemm_nn(c, m, l, n, A, lda, P.W, P.ldn, P.Y, P.ldm, P.part, P.part_elems);        // Y = A W
    c.mark("pass_power_AW");
    if (h->dbgYP) launch_copy(c, m, l, P.Y, P.ldm, h->dbgYP + it * l * h->ldYP, h->ldYP, false);
    orth(c, P.orth, m, l, P.Y, P.ldm, P.V, P.ldm, nullptr, 0, sh, it + 1 < q);        // V = qr(Y)
    c.mark("orth");
  }
  gemm_tn(c, m, l, n, A, lda, P.V, P.ldm, P.B, P.ldl, true, P.part, P.part_elems);    // l.4 B = V^T A
  allreduce_sum(c, P.B, P.ldl * n);
  check_replicated(c, P.B, P.ldl * n);
  c.mark("pass_project");
  fro2_accumulate(c, l, n, P.B, P.ldl, P.fro_slots, c.dind + 1, true);   // ||B||_F^2 (replicated B)
  if (h->dbgV) launch_copy(c, m, l, P.V, P.ldm, h->dbgV, h->ldV, false);
  if (h->dbgB) launch_copy(c, l, n, P.B, P.ldl, h->dbgB, h->ldB, false);
}

int run_rqlp(rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int q, int d, const double *A, int64_t lda,
             uint64_t seed, double *Q, int64_t ldq, double *T, int64_t ldt, double *Pout, int64_t ldp, int64_t *piv0,
             int64_t *piv1, bool allow_own) {
  const int64_t l = (int64_t)k + p;
  const int variant = d > 0 ? RQLP_VARIANT_ERQLP : RQLP_VARIANT_RQLP;
  const size_t need = plan_bytes(variant, m, n, l, 0, h->num_sms);
  char *ws = get_ws(h, need, allow_own);
  const std::string key = make_key(h, "rqlp", {m, n, k, p, q, d, lda, (int64_t)seed, ldq, ldt, ldp, h->ldY, h->ldV, h->ldB,
                                    h->ldVP, h->ldZ, h->ldW, h->ldYP},
                                   {A, Q, T, Pout, piv0, piv1, ws, h->dbgY, h->dbgV, h->dbgB, h->dbgVP, h->dbgZ, h->dbgW,
                                    h->dbgYP});
  return with_graph(h, key, [&](Ctx &c) {
    Arena a;
    a.base = ws;
    a.cap = need;
    Plan P;
    carve_plan(a, P, variant, m, n, l, 0, c.num_sms);
    RQLP_CUDA(cudaMemsetAsync(c.dflags, 0, NUM_DEV_FLAGS * sizeof(unsigned), c.stream));
    range_and_project(c, P, m, n, l, q, A, lda, seed, h);
    qlp_tail(c, P.tail, l, n, P.B, P.ldl, d, P.QB, P.ldl, T, ldt, Pout, ldp, piv0, piv1);   // l.5-7
    gemm_nn(c, m, l, l, P.V, P.ldm, P.QB, P.ldl, Q, ldq, P.part, P.part_elems);             // Q = V Q_B
    c.mark("assemble_Q");
  });
}

// ---- BRQLP -------------------------------------------------------------------------------
static bool fro_late_off() {   // RQLP_FRO_LATE=0: ||A||_F^2 always in the sketch (measurement switch)
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RQLP_FRO_LATE");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}
// Auto-rank mode of the block loop (NEXT-1): per-block sketches, and after
// each block the eq. (3) indicator ||A||_F^2 - sum_j ||B_j||_F^2 is read back; the loop stops once
// it is <= (eps ||A||_F)^2 (reading R25).
struct AutoRank {
  double eps = 0.0, a2 = 0.0, err = 0.0;
  int l_out = 0;
};
void enqueue_brqlp(Ctx &c, rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int b, int q, const double *A,
                   int64_t lda, uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *Pout,
                   int64_t ldp, int64_t *piv0, int64_t *piv1, char *ws, size_t need, AutoRank *ar = nullptr);
// Alg.3 with implicit deflation: A^(j-1) X = A X - V_<j (B_<j X), A^(j-1)^T V = A^T V - B_<j^T (V_<j^T V).
int run_brqlp(rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int b, int q, const double *A, int64_t lda,
              uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *Pout, int64_t ldp, int64_t *piv0,
              int64_t *piv1, bool allow_own) {
  const int64_t l = (int64_t)k + p;
  const size_t need = plan_bytes(RQLP_VARIANT_BRQLP, m, n, l, b, h->num_sms);
  char *ws = get_ws(h, need, allow_own);
  const std::string key = make_key(h, "brqlp", {m, n, k, p, b, q, lda, (int64_t)seed, ldq, ldl, ldp, h->ldY, h->ldV, h->ldB,
                                    h->ldVP, h->ldZ, h->ldW, h->ldYP},
                                   {A, Q, L, Pout, piv0, piv1, ws, h->dbgY, h->dbgV, h->dbgB, h->dbgVP, h->dbgZ, h->dbgW,
                                    h->dbgYP});
  return with_graph(h, key, [&](Ctx &c) { enqueue_brqlp(c, h, m, n, k, p, b, q, A, lda, seed, Q, ldq, L, ldl, Pout,
                                                        ldp, piv0, piv1, ws, need); });
}

void enqueue_brqlp(Ctx &c, rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int b, int q, const double *A,
                   int64_t lda, uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *Pout,
                   int64_t ldp, int64_t *piv0, int64_t *piv1, char *ws, size_t need, AutoRank *ar) {
  const int64_t l = (int64_t)k + p;
  const bool sh = c.comm != nullptr;  // row-sharded handle: Grams are summed over ranks
  Arena a;
  a.base = ws;
  a.cap = need;
  Plan P;
  carve_plan(a, P, RQLP_VARIANT_BRQLP, m, n, l, b, c.num_sms);
  RQLP_CUDA(cudaMemsetAsync(c.dflags, 0, NUM_DEV_FLAGS * sizeof(unsigned), c.stream));
  const int64_t ldm = P.ldm, ldn = P.ldn, LL = P.ldl;
  c.mark("start");
  launch_omega(c, n, l, 0, seed, P.Om, ldn);                                            // l.1
  c.mark("omega");
  const FroSpec fro{P.fro_slots, P.fro_cap, c.dind};
  const int64_t h_blocks = ceil_div(l, b);
  // ||A||_F^2 (eq. (3)) rides on an A-pass that reads A anyway.  Normally the sketch; when the last
  // block is narrow (C4: 16 columns) and has a power step, its Y = A W pass instead: that pass is
  // HBM-bound, so the extra warp squaring the staged A tiles costs nothing there, while in the
  // compute-bound sketch it cost ~3 ms (C4).  Only BRQLP's final indicator reads it.
  const int64_t b_last = l - (h_blocks - 1) * b;
  const bool fro_late = !ar && q > 0 && b_last <= 32 && !(h->feed && h->feed->hA) && !fro_late_off();
  if (!ar) {
    // l.3 all Y_j = AΩ_j in one pass, with ||A||_F^2 (eq. (3)) from the same A tiles
    if (fro_late) gemm_nn(c, m, l, n, A, lda, P.Om, ldn, P.Y, ldm, P.part, P.part_elems);
    else sketch_pass(c, h, P, m, l, n, A, lda, P.Om, ldn, P.Y, ldm);
    if (!fro_late) allreduce_sum(c, c.dind, 1);   // row shards: ||A||^2 is the sum over ranks (B_j is replicated)
    c.mark("pass_sketch");
    if (h->dbgY) launch_copy(c, m, l, P.Y, ldm, h->dbgY, h->ldY, false);
  }
  launch_fill(c, l, l, L, ldl, 0.0, 0.0);
  double *B = P.B;  // B_<j rows accumulate here (l x n, ld LL)
  const bool out = h->feed && (h->feed->hQ || h->feed->hP) && !ar;
  if (out) {
    if (!h->cstream) RQLP_CUDA(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    while ((int64_t)h->oev.size() < h_blocks + 1) {
      cudaEvent_t e;
      RQLP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->oev.push_back(e);
    }
  }
  // Alg.3 l.4-5: V_j = qr(Y_j), then V_j <- qr(V_j - V_<j (V_<j^T V_j)) (eq. (18)), the latter
  // applied twice ("twice is enough", reading R28: identical in exact arithmetic when V_j has a
  // component outside span(V_<j) -- the second projection removes nothing -- and the only way to
  // keep Q orthonormal when it has (almost) none: a block beyond rank(A), whose first residual is
  // rounding noise).  Computed as block CGS2 on Y_j itself (overwritten):
  //   W = Y_j - V_<j (V_<j^T Y_j),  V_j = qr1(W)  (one CholeskyQR pass: only its span is used),
  //   V_j <- V_j - V_<j (V_<j^T V_j), V_j = qr(V_j)  (CholeskyQR2),
  // equal to the literal sequence in exact arithmetic: qr(Y_j) = Y_j R^-1 with R upper triangular
  // and R_ii > 0, so P(Y_j R^-1) = (P Y_j) R^-1 spans the same space with the same R_ii > 0
  // normalisation.  3 CholeskyQR passes where the literal form takes 6 (C4: 12 -> 6 m x b passes
  // per block).  The first block has nothing to project against: V_1 = qr(Y_1).
  // span_only (the V_j that only feeds a power step, q >= 1): the deflated product
  // Z = A^(j-1)^T V_j = A^T V_j - B_<j^T (V_<j^T V_j) depends on V_j only through the span of its
  // component outside span(V_<j) -- A^(j-1) annihilates span(V_<j) and the V_<j^T V_j term is formed
  // explicitly -- so the first projection and ONE CholeskyQR pass (W R^-1 spans (I - P) Y_j) suffice,
  // as for RQLP's intermediate bases (orth's span_only); the block's final V_j gets the full sequence.
  // RQLP_BRQLP_PRE_SPAN=0: the full sequence there too (measurement switch).
  static const bool pre_span = [] { const char *e = getenv("RQLP_BRQLP_PRE_SPAN"); return !(e && e[0] == '0'); }();
  auto block_orth = [&](double *Yj, int64_t c0, int64_t bj, bool span_only = false) {
    double *Vj = P.V + c0 * ldm;
    span_only = span_only && pre_span;
    if (c0 == 0) {
      orth(c, P.orth, m, bj, Yj, ldm, Vj, ldm, nullptr, 0, sh, span_only);
      return;
    }
    c.mark("b_other");
    gemm_tn(c, m, bj, c0, P.V, ldm, Yj, ldm, P.C, LL, false, P.part, P.part_elems);        // C = V_<j^T Y_j
    allreduce_sum(c, P.C, LL * bj);
    gemm_nn_ab(c, m, bj, c0, -1.0, P.V, ldm, P.C, LL, 1.0, Yj, ldm, P.part, P.part_elems);  // W = Y_j - V_<j C
    orth(c, P.orth, m, bj, Yj, ldm, Vj, ldm, nullptr, 0, sh, true);                         // span of W
    if (span_only) return;
    gemm_tn(c, m, bj, c0, P.V, ldm, Vj, ldm, P.C, LL, false, P.part, P.part_elems);        // C = V_<j^T V_j
    allreduce_sum(c, P.C, LL * bj);
    gemm_nn_ab(c, m, bj, c0, -1.0, P.V, ldm, P.C, LL, 1.0, Vj, ldm, P.part, P.part_elems);  // V_j -= V_<j C
    // CholeskyQR2 in place: pass 1 reads V_j into the orth scratch, pass 2 writes V_j (no R asked, so
    // nothing reads the input again)
    orth(c, P.orth, m, bj, Vj, ldm, Vj, ldm, nullptr, 0, sh);
  };
  // q = 0 (NEXT-4): the range finder needs no A-pass per block, so every V_j is built first
  // and ONE batched pass B = V^T A replaces the h per-block projections; the deflation
  // B_j = V_j^T A - (V_j^T V_<j) B_<j below is unchanged (exact-arithmetic identity).
  const bool two_pass = q == 0 && !ar;
  if (two_pass) {
    for (int64_t j = 0; j < h_blocks; ++j) {
      const int64_t c0 = j * b, bj = std::min<int64_t>(b, l - c0);
      block_orth(P.Y + c0 * ldm, c0, bj);                                                   // l.4-5
    }
    c.mark("b_other");
    gemm_tn(c, m, l, n, A, lda, P.V, ldm, B, LL, true, P.part, P.part_elems);           // all V_j^T A
    allreduce_sum(c, B, LL * n);
    check_replicated(c, B, LL * n);
    c.mark("pass_project");
  }
  for (int64_t j = 0; j < h_blocks; ++j) {
    const int64_t c0 = j * b, bj = std::min<int64_t>(b, l - c0);
    double *Vj = P.V + c0 * ldm;
    if (ar) {  // Alg.3 l.3 inside the loop: Y_j = A Ω_j (original A); the first pass also forms ||A||_F^2
      c.mark("b_other");
      if (j == 0) {
        gemm_nn_fro(c, m, bj, n, A, lda, P.Om, ldn, P.Y, ldm, P.part, P.part_elems, fro);
        allreduce_sum(c, c.dind, 1);
      } else {
        gemm_nn(c, m, bj, n, A, lda, P.Om + c0 * ldn, ldn, P.Y + c0 * ldm, ldm, P.part, P.part_elems);
      }
      c.mark("pass_block_sketch");
    }
    if (!two_pass) {
      block_orth(P.Y + c0 * ldm, c0, bj, q > 0);                                           // l.4-5
      for (int it = 0; it < q; ++it) {                                                     // deflated power step (R16)
        if (h->dbgVP) launch_copy(c, m, bj, Vj, ldm, h->dbgVP + (it * l + c0) * h->ldVP, h->ldVP, false);
        c.mark("b_other");
        gemm_tn(c, m, bj, n, A, lda, Vj, ldm, P.Z, ldn, false, P.part, P.part_elems);     // Z = A^T Vj
        allreduce_sum(c, P.Z, ldn * bj);
        c.mark("pass_block_AtV");
        if (c0 > 0) {
          gemm_tn(c, m, bj, c0, P.V, ldm, Vj, ldm, P.C, LL, false, P.part, P.part_elems); // C = V_<j^T Vj
          allreduce_sum(c, P.C, LL * bj);
          gemm_tn_ab(c, c0, bj, n, -1.0, B, LL, P.C, LL, 1.0, P.Z, ldn, P.part, P.part_elems);   // Z -= B_<j^T C
        }
        if (h->dbgZ) launch_copy(c, n, bj, P.Z, ldn, h->dbgZ + (it * l + c0) * h->ldZ, h->ldZ, false);
        // W = qr(Z): only span(W) reaches Y = A^(j-1) W and the block's V_j, so one CholeskyQR pass
        // (orth's span_only, as in RQLP's power steps)
        orth(c, P.orth, n, bj, P.Z, ldn, P.W, ldn, nullptr, 0, false, pre_span);
        if (h->dbgW) launch_copy(c, n, bj, P.W, ldn, h->dbgW + (it * l + c0) * h->ldW, h->ldW, false);
        c.mark("b_other");
        if (fro_late && j == h_blocks - 1 && it == 0) {   // Y = A W, with ||A||_F^2 (see above)
          gemm_nn_fro(c, m, bj, n, A, lda, P.W, ldn, P.Y + c0 * ldm, ldm, P.part, P.part_elems, fro);
          allreduce_sum(c, c.dind, 1);
        } else {
          gemm_nn(c, m, bj, n, A, lda, P.W, ldn, P.Y + c0 * ldm, ldm, P.part, P.part_elems); // Y = A W
        }
        c.mark("pass_block_AW");
        if (c0 > 0) {
          gemm_nn_ab(c, c0, bj, n, 1.0, B, LL, P.W, ldn, 0.0, P.D, LL, P.part, P.part_elems);    // D = B_<j W
          gemm_nn_ab(c, m, bj, c0, -1.0, P.V, ldm, P.D, LL, 1.0, P.Y + c0 * ldm, ldm, P.part, P.part_elems);  // Y -= V_<j D
        }
        if (h->dbgYP) launch_copy(c, m, bj, P.Y + c0 * ldm, ldm, h->dbgYP + (it * l + c0) * h->ldYP, h->ldYP, false);
        block_orth(P.Y + c0 * ldm, c0, bj);
      }
    }
    // l.6: B_j = Vj^T A^(j-1) = Vj^T A - (Vj^T V_<j) B_<j, formed in the tail's B buffer
    double *Bj = P.tail.Bw;
    const int64_t ldbj = P.tail.ldl;
    c.mark("b_other");
    if (two_pass) {
      launch_copy(c, bj, n, B + c0, LL, Bj, ldbj, false);   // V_j^T A from the batched pass
    } else {
      gemm_tn(c, m, bj, n, A, lda, Vj, ldm, Bj, ldbj, true, P.part, P.part_elems);
      allreduce_sum(c, Bj, ldbj * n);
      check_replicated(c, Bj, ldbj * n);
      c.mark("pass_block_project");
    }
    if (c0 > 0) {
      const int64_t lde = round_up(b, 8);
      // E = Vj^T V_<j (bj x c0), formed as (V_<j^T V_j)^T: c0 output rows fill the kernel's 128-row
      // tiles, bj = 64 rows left half of each tile as zero fill (C4, c0 = 384: 745 -> 389 us)
      gemm_tn(c, m, bj, c0, P.V, ldm, Vj, ldm, P.D, lde, true, P.part, P.part_elems);
      allreduce_sum(c, P.D, lde * c0);
      gemm_nn_ab(c, bj, n, c0, -1.0, P.D, lde, B, LL, 1.0, Bj, ldbj, P.part, P.part_elems);   // B_j -= E B_<j
    }
    launch_copy(c, bj, n, Bj, ldbj, B + c0, LL, false);   // keep B_j for the later blocks' deflation
    c.mark("block_passes");
    bool stop = false;
    if (ar) {  // eq. (3): ||A - P_V A||_F^2 = ||A||_F^2 - sum_j ||B_j||_F^2
      fro2_accumulate(c, bj, n, Bj, ldbj, P.fro_slots, c.dind + 1, j == 0);
      double ab[2] = {0.0, 0.0};
      RQLP_CUDA(cudaMemcpyAsync(ab, c.dind, 2 * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
      RQLP_CUDA(cudaStreamSynchronize(c.stream));
      ar->a2 = ab[0];
      const double b2 = ab[1];
      const double e2 = ar->a2 - b2;
      ar->err = ar->a2 > 0.0 ? std::sqrt(e2 > 0.0 ? e2 : 0.0) / std::sqrt(ar->a2) : 0.0;
      ar->l_out = (int)(c0 + bj);
      stop = e2 <= ar->eps * ar->eps * ar->a2;
    }
    // l.8: [Q_B, L_j, P_B] = qlp(B_j) (overwrites the tail's copy)
    qlp_tail(c, P.tail, bj, n, P.tail.Bw, P.tail.ldl, 0, P.QB, P.tail.ldl, L + c0 + c0 * ldl, ldl, Pout + c0 * ldp,
             ldp, piv0 ? piv0 + c0 : nullptr, piv1 ? piv1 + c0 : nullptr);
    // l.9: Q_j = V_j Q_B
    gemm_nn(c, m, bj, bj, Vj, ldm, P.QB, P.tail.ldl, Q + c0 * ldq, ldq, P.part, P.part_elems);
    c.mark("block_tail");
    if (out) {
      // host outputs (rqlp_factorize): Q_j and P_j go out on the copy stream while the next
      // blocks run (part of the captured work; joined below)
      RQLP_CUDA(cudaEventRecord(h->oev[j], c.stream));
      RQLP_CUDA(cudaStreamWaitEvent(h->cstream, h->oev[j], 0));
      if (h->feed->hQ)
        RQLP_CUDA(cudaMemcpy2DAsync(h->feed->hQ + c0 * m, m * 8, Q + c0 * ldq, ldq * 8, m * 8, bj,
                                    cudaMemcpyDeviceToHost, h->cstream));
      if (h->feed->hP)
        RQLP_CUDA(cudaMemcpy2DAsync(h->feed->hP + c0 * n, n * 8, Pout + c0 * ldp, ldp * 8, n * 8, bj,
                                    cudaMemcpyDeviceToHost, h->cstream));
    }
    if (stop) break;
  }
  if (out) {   // join the copy stream
    RQLP_CUDA(cudaEventRecord(h->oev[h_blocks], h->cstream));
    RQLP_CUDA(cudaStreamWaitEvent(c.stream, h->oev[h_blocks], 0));
  }
  if (!ar) fro2_accumulate(c, l, n, B, LL, P.fro_slots, c.dind + 1, true);   // sum_j ||B_j||_F^2 (deflated B_j)
  if (h->dbgV) launch_copy(c, m, l, P.V, ldm, h->dbgV, h->ldV, false);
  if (h->dbgB) launch_copy(c, l, n, B, LL, h->dbgB, h->ldB, false);
}

}  // namespace
// ---- truncated pivoted QLP (NEXT-3) ---------------------------------------------------------
struct TqlpPlan {
  int64_t ldm;
  double *W, *QR;
  HHScratch hA;
  TailScratch tail;
};

void carve_tqlp(Arena &a, TqlpPlan &p, int64_t m, int64_t n, int64_t l, int num_sms) {
  p.ldm = round_up(m, 8);
  p.W = a.take<double>(p.ldm * n);
  p.QR = a.take<double>(p.ldm * l);
  hh_carve(a, p.hA, m, n, num_sms, l);
  tail_carve(a, p.tail, l, n, num_sms);
}

size_t tqlp_bytes(int64_t m, int64_t n, int64_t l, int num_sms) {
  Arena a;
  TqlpPlan p;
  carve_tqlp(a, p, m, n, l, num_sms);
  return a.used + 4096;
}

int run_tqlp(rqlp_handle_t h, int64_t m, int64_t n, int64_t l, const double *A, int64_t lda, double *Q, int64_t ldq,
             double *L, int64_t ldl, double *P, int64_t ldp, int64_t *piv0, int64_t *piv1) {
  const size_t need = tqlp_bytes(m, n, l, h->num_sms);
  char *ws = get_ws(h, need, true);
  const std::string key = make_key(h, "tqlp", {m, n, l, lda, ldq, ldl, ldp}, {A, Q, L, P, piv0, piv1, ws});
  return with_graph(h, key, [&](Ctx &c) {
    Arena a;
    a.base = ws;
    a.cap = need;
    TqlpPlan p;
    carve_tqlp(a, p, m, n, l, c.num_sms);
    RQLP_CUDA(cudaMemsetAsync(c.dflags, 0, NUM_DEV_FLAGS * sizeof(unsigned), c.stream));
    c.mark("start");
    launch_copy(c, m, n, A, lda, p.W, p.ldm, false);   // the engine factors in place
    c.mark("tqlp_copy");
    tqlp(c, p.tail, p.hA, m, n, l, p.W, p.ldm, Q, ldq, L, ldl, P, ldp, piv0, piv1, p.QR, p.ldm);
  });
}

}  // namespace rqlpk

using namespace rqlpk;

// ================================ C ABI ================================================
extern "C" {

int rqlp_create(rqlp_handle_t *out, int device, void *cuda_stream) {
  if (!out) return -1;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return RQLP_ERR_CUDA;
  if (device < 0 || device >= ndev) return -2;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return RQLP_ERR_CUDA;
  if (prop.major != 10) return RQLP_ERR_DEVICE;
  auto *h = new rqlp_handle_s();
  h->device = device;
  h->stream = (cudaStream_t)cuda_stream;
  h->num_sms = prop.multiProcessorCount;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaError_t e = cudaMalloc(&h->dflags, NUM_DEV_FLAGS * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(h->dflags, 0, NUM_DEV_FLAGS * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMalloc(&h->dind, 16 * sizeof(double));   // [0..1] eq. (3); [4..10] replica check
  if (e == cudaSuccess) e = cudaMemset(h->dind, 0, 16 * sizeof(double));
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    delete h;
    return RQLP_ERR_CUDA;
  }
  *out = h;
  return RQLP_OK;
}

int rqlp_get_unique_id(void *out) {
  if (!out) return -1;
  try {
    return comm_unique_id(out);
  } catch (const std::exception &e) {
    fprintf(stderr, "[rqlp] %s\n", e.what());
    return RQLP_ERR_NCCL;
  }
}

int rqlp_create_dist(rqlp_handle_t *out, int device, void *cuda_stream, const void *uid, int rank, int nranks) {
  if (!uid) return -4;
  if (nranks < 1) return -6;
  if (rank < 0 || rank >= nranks) return -5;
  int rc = rqlp_create(out, device, cuda_stream);
  if (rc != RQLP_OK) return rc;
  rqlp_handle_t h = *out;
  h->rank = rank;
  h->nranks = nranks;
  {  // a communicator even for nranks == 1 (the NCCL path is then exercised on one GPU)
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    try {
      h->comm = comm_init(uid, rank, nranks);
    } catch (const std::exception &e) {
      fprintf(stderr, "[rqlp] %s\n", e.what());
      cudaSetDevice(prev);
      rqlp_destroy(h);
      *out = nullptr;
      return RQLP_ERR_NCCL;
    }
    cudaSetDevice(prev);
  }
  return RQLP_OK;
}

int rqlp_create_loopback(rqlp_handle_t *out, int nranks, int device, void *cuda_stream) {
  if (!out) return -1;
  if (nranks < 1 || nranks > 64) return -2;
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  void *group = nullptr;
  for (int r = 0; r < nranks; ++r) {
    int rc = rqlp_create(&out[r], device, cuda_stream);
    if (rc != RQLP_OK) {
      for (int i = 0; i < r; ++i) rqlp_destroy(out[i]);
      for (int i = 0; i < nranks; ++i) out[i] = nullptr;
      return rc;
    }
    if (!group) group = comm_loopback_group(nranks, device, (cudaStream_t)cuda_stream);
    out[r]->rank = r;
    out[r]->nranks = nranks;
    out[r]->comm = comm_loopback_init(group, r);
  }
  return RQLP_OK;
}

int rqlp_destroy(rqlp_handle_t h) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  reset_timing(h);
  for (auto &kv : h->graphs) {
    cudaGraphExecDestroy(kv.second.exec);
    for (auto ev : kv.second.pool) cudaEventDestroy(ev);
  }
  for (auto ev : h->eager_pool) cudaEventDestroy(ev);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->cstream) cudaStreamDestroy(h->cstream);
  for (auto ev : h->cev) cudaEventDestroy(ev);
  for (auto ev : h->oev) cudaEventDestroy(ev);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->own) cudaFree(h->own);
  if (h->stage) cudaFree(h->stage);
  if (h->dflags) cudaFree(h->dflags);
  if (h->dind) cudaFree(h->dind);
  comm_destroy(h->comm);
  cudaSetDevice(prev);
  h->magic = 0;
  delete h;
  return RQLP_OK;
}

int rqlp_workspace_size(rqlp_handle_t h, int variant, int64_t m, int64_t n, int k, int p, int q, int d, int b,
                        size_t *bytes) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (variant < 0 || variant > 2) return -2;
  int rc = check_common(m, n, k, p, q);
  if (rc) return rc - 2;
  if (variant == RQLP_VARIANT_ERQLP && d < 1) return -8;
  int64_t l = (int64_t)k + p;
  if (variant == RQLP_VARIANT_BRQLP && (b < 1 || b > l)) return -9;
  if (!bytes) return -10;
  *bytes = plan_bytes(variant, m, n, l, variant == RQLP_VARIANT_BRQLP ? b : 0, h->num_sms);
  return RQLP_OK;
}

int rqlp_set_workspace(rqlp_handle_t h, void *ptr, size_t bytes) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (ptr && ((uintptr_t)ptr & 255)) return -2;
  h->ws = ptr;
  h->ws_bytes = ptr ? bytes : 0;
  return RQLP_OK;
}

int rqlp_ex(rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int q, const double *A, int64_t lda, uint64_t seed,
            double *Q, int64_t ldq, double *L, int64_t ldl, double *P, int64_t ldp, int64_t *piv0, int64_t *piv1) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  int rc = check_common(m, n, k, p, q);
  if (rc) return rc - 1;
  int64_t l = (int64_t)k + p;
  if (h->nranks == 1 && l > m) return -4;
  if (!A) return -7;
  if (lda < m) return -8;
  if (!Q) return -10;
  if (ldq < m) return -11;
  if (!L) return -12;
  if (ldl < l) return -13;
  if (!P) return -14;
  if (ldp < n) return -15;
  return guarded(h, [&] {
    return run_rqlp(h, m, n, k, p, q, 0, A, lda, seed, Q, ldq, L, ldl, P, ldp, piv0, piv1, true);
  }, true);
}

int erqlp_ex(rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int q, int d, const double *A, int64_t lda,
             uint64_t seed, double *Q, int64_t ldq, double *T, int64_t ldt, int *t_is_upper, double *P, int64_t ldp,
             int64_t *piv0) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  int rc = check_common(m, n, k, p, q);
  if (rc) return rc - 1;
  int64_t l = (int64_t)k + p;
  if (h->nranks == 1 && l > m) return -4;
  if (d < 1) return -7;
  if (!A) return -8;
  if (lda < m) return -9;
  if (!Q) return -11;
  if (ldq < m) return -12;
  if (!T) return -13;
  if (ldt < l) return -14;
  if (!P) return -16;
  if (ldp < n) return -17;
  if (t_is_upper) *t_is_upper = (d % 2 == 0) ? 1 : 0;
  return guarded(h, [&] {
    return run_rqlp(h, m, n, k, p, q, d, A, lda, seed, Q, ldq, T, ldt, P, ldp, piv0, nullptr, true);
  }, true);
}

int brqlp_ex(rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int b, int q, const double *A, int64_t lda,
             uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *P, int64_t ldp, int64_t *piv0,
             int64_t *piv1) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  int rc = check_common(m, n, k, p, q);
  if (rc == -5) return -7;
  if (rc) return rc - 1;
  int64_t l = (int64_t)k + p;
  if (h->nranks == 1 && l > m) return -4;
  if (b < 1 || b > l) return -6;
  if (!A) return -8;
  if (lda < m) return -9;
  if (!Q) return -11;
  if (ldq < m) return -12;
  if (!L) return -13;
  if (ldl < l) return -14;
  if (!P) return -15;
  if (ldp < n) return -16;
  return guarded(h, [&] {
    return run_brqlp(h, m, n, k, p, b, q, A, lda, seed, Q, ldq, L, ldl, P, ldp, piv0, piv1, true);
  }, true);
}

int rqlp_tqlp_ex(rqlp_handle_t h, int64_t m, int64_t n, int l, const double *A, int64_t lda, double *Q, int64_t ldq,
                 double *L, int64_t ldl, double *P, int64_t ldp, int64_t *piv0, int64_t *piv1) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (m < 1) return -2;
  if (n < 1) return -3;
  if (l < 1 || l > m || l > n) return -4;
  if (!A) return -5;
  if (lda < m) return -6;
  if (!Q) return -7;
  if (ldq < m) return -8;
  if (!L) return -9;
  if (ldl < l) return -10;
  if (!P) return -11;
  if (ldp < n) return -12;
  if (h->comm) return RQLP_ERR_UNSUPPORTED;
  return guarded(h, [&] { return run_tqlp(h, m, n, l, A, lda, Q, ldq, L, ldl, P, ldp, piv0, piv1); });
}

int rqlp_autorank_ex(rqlp_handle_t h, int64_t m, int64_t n, int b, int l_max, int q, double eps, const double *A,
                     int64_t lda, uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *P,
                     int64_t ldp, int64_t *piv0, int64_t *piv1, int *l_out, double *err_out) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (m < 1) return -2;
  if (n < 1) return -3;
  if (b < 1) return -4;
  if (l_max < b || l_max > n || (h->nranks == 1 && l_max > m)) return -5;
  if (q < 0) return -6;
  if (!(eps >= 0.0)) return -7;
  if (!A) return -8;
  if (lda < m) return -9;
  if (!Q) return -11;
  if (ldq < m) return -12;
  if (!L) return -13;
  if (ldl < l_max) return -14;
  if (!P) return -15;
  if (ldp < n) return -16;
  if (!l_out) return -19;
  return guarded(h, [&] {
    const size_t need = plan_bytes(RQLP_VARIANT_BRQLP, m, n, l_max, b, h->num_sms);
    char *ws = get_ws(h, need, true);
    AutoRank ar;
    ar.eps = eps;
    Ctx c = make_ctx(h);
    reset_timing(h);
    // k + p = l_max for the plan; the loop stops at the first block meeting the tolerance
    enqueue_brqlp(c, h, m, n, l_max - 1, 1, b, q, A, lda, seed, Q, ldq, L, ldl, P, ldp, piv0, piv1, ws, need, &ar);
    h->launches = c.launches;
    RQLP_CUDA(cudaStreamSynchronize(c.stream));
    *l_out = ar.l_out;
    if (err_out) *err_out = ar.err;
    return RQLP_OK;
  }, true);
}

static bool is_device_ptr(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static bool is_pinned_host_ptr(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

static std::mutex g_default_mu;
static rqlp_handle_t g_default[64] = {nullptr};

// Synchronous any-pointer factorisation: host operands are staged through device memory.
static int factorize_any(rqlp_handle_t h, int variant, int64_t m, int64_t n, int k, int p, int q, int d, int b,
                         const double *A, int64_t lda, uint64_t seed, double *Q, double *T, double *P,
                         int *t_is_upper) {
  int64_t l = (int64_t)k + p;
  return guarded(h, [&] {
    bool dA = is_device_ptr(A), dQ = is_device_ptr(Q), dT = is_device_ptr(T), dP = is_device_ptr(P);
    const int64_t ldd = dA ? lda : round_up(m, 8);   // device staging of a host A: aligned for TMA
    size_t szA = dA ? 0 : (size_t)round_up(ldd * n, 32) * 8;
    size_t szQ = dQ ? 0 : (size_t)round_up(m * l, 32) * 8;
    size_t szT = dT ? 0 : (size_t)round_up(l * l, 32) * 8;
    size_t szP = dP ? 0 : (size_t)round_up(n * l, 32) * 8;
    size_t tot = szA + szQ + szT + szP + 1024;
    if (tot > 1024 && h->stage_bytes < tot) {
      if (h->stage) cudaFree(h->stage);
      h->stage = nullptr;
      h->stage_bytes = 0;
      RQLP_CUDA(cudaMalloc(&h->stage, tot));
      h->stage_bytes = tot;
    }
    char *sp = (char *)h->stage;
    const double *Ad = A;
    double *Qd = Q, *Td = T, *Pd = P;
    if (!dA) { Ad = (const double *)sp; sp += szA; }
    if (!dQ) { Qd = (double *)sp; sp += szQ; }
    if (!dT) { Td = (double *)sp; sp += szT; }
    if (!dP) { Pd = (double *)sp; sp += szP; }
    // host A: copied in row panels inside the factorisation, overlapped with the sketch pass that
    // consumes them (sketch_pass); the panel height keeps each copy >= ~0.5 GB and <= 8 panels
    HostFeed feed;
    if (!dA && !is_pinned_host_ptr(A)) {   // pageable: one synchronous-source copy up front
      RQLP_CUDA(cudaMemcpy2DAsync((void *)Ad, ldd * 8, A, lda * 8, m * 8, n, cudaMemcpyHostToDevice, h->stream));
    } else if (!dA) {
      feed.hA = A;
      feed.hlda = lda;
      const int64_t min_rows = std::max<int64_t>(128, ceil_div((int64_t)1 << 26, n));
      feed.panel_rows = round_up(std::max(min_rows, ceil_div(m, 8)), 128);
      h->feed = &feed;
    }
    // BRQLP with pinned host Q / P: each block's columns are copied out as soon as they are final
    bool streamQ = false, streamP = false;
    if (variant == RQLP_VARIANT_BRQLP) {
      streamQ = !dQ && is_pinned_host_ptr(Q);
      streamP = !dP && is_pinned_host_ptr(P);
      if (streamQ) feed.hQ = Q;
      if (streamP) feed.hP = P;
      if (streamQ || streamP) h->feed = &feed;
    }
    int r;
    try {
      if (variant == RQLP_VARIANT_BRQLP)
        r = run_brqlp(h, m, n, k, p, b, q, Ad, ldd, seed, Qd, m, Td, l, Pd, n, nullptr, nullptr, true);
      else
        r = run_rqlp(h, m, n, k, p, q, variant == RQLP_VARIANT_ERQLP ? d : 0, Ad, ldd, seed, Qd, m, Td, l, Pd, n,
                     nullptr, nullptr, true);
    } catch (...) {
      h->feed = nullptr;
      throw;
    }
    h->feed = nullptr;
    if (r) return r;
    if (t_is_upper) *t_is_upper = (variant == RQLP_VARIANT_ERQLP && d % 2 == 0) ? 1 : 0;
    if (!dQ && !streamQ) RQLP_CUDA(cudaMemcpyAsync(Q, Qd, (size_t)m * l * 8, cudaMemcpyDeviceToHost, h->stream));
    if (!dT) RQLP_CUDA(cudaMemcpyAsync(T, Td, (size_t)l * l * 8, cudaMemcpyDeviceToHost, h->stream));
    if (!dP && !streamP) RQLP_CUDA(cudaMemcpyAsync(P, Pd, (size_t)n * l * 8, cudaMemcpyDeviceToHost, h->stream));
    RQLP_CUDA(cudaStreamSynchronize(h->stream));
    return RQLP_OK;
  }, true);
}

int rqlp_factorize(rqlp_handle_t h, int variant, int64_t m, int64_t n, int k, int p, int q, int d, int b,
                   const double *A, int64_t lda, uint64_t seed, double *Q, double *T, double *P, int *t_is_upper) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (variant < 0 || variant > 2) return -2;
  int rc = check_common(m, n, k, p, q);
  if (rc) return rc - 2;
  int64_t l = (int64_t)k + p;
  if (h->nranks == 1 && l > m) return -5;
  if (variant == RQLP_VARIANT_ERQLP && d < 1) return -8;
  if (variant == RQLP_VARIANT_BRQLP && (b < 1 || b > l)) return -9;
  if (!A) return -10;
  if (lda < m) return -11;
  if (!Q) return -13;
  if (!T) return -14;
  if (!P) return -15;
  return factorize_any(h, variant, m, n, k, p, q, d, b, A, lda, seed, Q, T, P, t_is_upper);
}

int rqlp(int64_t m, int64_t n, int k, int p, int q, const double *A, int64_t lda, uint64_t seed, double *Q, double *L,
         double *P) {
  int rc = check_common(m, n, k, p, q);
  if (rc) return rc;
  int64_t l = (int64_t)k + p;
  if (l > m) return -3;
  if (!A) return -6;
  if (lda < m) return -7;
  if (!Q) return -9;
  if (!L) return -10;
  if (!P) return -11;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return RQLP_ERR_CUDA;
  rqlp_handle_t h;
  {
    std::lock_guard<std::mutex> lk(g_default_mu);
    if (dev >= 64) return RQLP_ERR_INTERNAL;
    if (!g_default[dev]) {
      int r = rqlp_create(&g_default[dev], dev, nullptr);
      if (r) return r;
    }
    h = g_default[dev];
  }
  return factorize_any(h, RQLP_VARIANT_RQLP, m, n, k, p, q, 0, 0, A, lda, seed, Q, L, P, nullptr);
}

int rqlp_sync(rqlp_handle_t h, unsigned *flags) {
  return guarded(h, [&] {
    RQLP_CUDA(cudaStreamSynchronize(h->stream));
    if (int ae = comm_async_error(h->comm))   // NCCL asynchronous failure (ncclCommGetAsyncError)
      throw NcclError("ncclCommGetAsyncError: " + std::to_string(ae));
    if (flags) {
      unsigned f = 0;
      RQLP_CUDA(cudaMemcpy(&f, h->dflags + FLAG_WORD, sizeof(unsigned), cudaMemcpyDeviceToHost));
      *flags = f;
    }
    return RQLP_OK;
  });
}

int rqlp_get_indicator(rqlp_handle_t h, double *a2, double *b2) {
  return guarded(h, [&] {
    double v[2] = {0.0, 0.0};
    RQLP_CUDA(cudaStreamSynchronize(h->stream));
    RQLP_CUDA(cudaMemcpy(v, h->dind, 2 * sizeof(double), cudaMemcpyDeviceToHost));
    if (a2) *a2 = v[0];
    if (b2) *b2 = v[1];
    return RQLP_OK;
  });
}

const char *rqlp_strerror(int code) {
  switch (code) {
    case RQLP_OK: return "success";
    case RQLP_ERR_CUDA: return "CUDA runtime error";
    case RQLP_ERR_NCCL: return "NCCL error";
    case RQLP_ERR_WORKSPACE: return "workspace missing or too small";
    case RQLP_ERR_INTERNAL: return "internal error";
    case RQLP_ERR_DEVICE: return "device is not sm_100 (B200)";
    case RQLP_ERR_HANDLE: return "invalid handle";
    default: return code < 0 ? "illegal argument (-code = position)" : "unknown error";
  }
}

// ---- stage entry points -------------------------------------------------------------------
int rqlp_omega(rqlp_handle_t h, int64_t n, int64_t l, uint64_t seed, double *Om, int64_t ldo) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (n < 1) return -2;
  if (l < 1) return -3;
  if (!Om) return -5;
  if (ldo < n) return -6;
  return guarded(h, [&] {
    Ctx c = make_ctx(h);
    launch_omega(c, n, l, 0, seed, Om, ldo);
    h->launches = c.launches;
    return RQLP_OK;
  });
}

int rqlp_gemm_nn(rqlp_handle_t h, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X,
                 int64_t ldx, double *Y, int64_t ldy) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (m < 0) return -2;
  if (cc < 0) return -3;
  if (k < 0) return -4;
  if (!A && m * k > 0) return -5;
  if (lda < std::max<int64_t>(1, m)) return -6;
  if (!X && k * cc > 0) return -7;
  if (ldx < std::max<int64_t>(1, k)) return -8;
  if (!Y && m * cc > 0) return -9;
  if (ldy < std::max<int64_t>(1, m)) return -10;
  return guarded(h, [&] {
    Ctx c = make_ctx(h);
    size_t pe = gemm_partials_needed(m, cc, k, c.num_sms);
    char *ws = get_ws(h, pe * 8 + 256, true);
    if (m > 0 && cc > 0) gemm_nn(c, m, cc, k, A, lda, X, ldx, Y, ldy, (double *)ws, pe);
    h->launches = c.launches;
    return RQLP_OK;
  });
}

int rqlp_gemm_tn(rqlp_handle_t h, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *V,
                 int64_t ldv, double *Z, int64_t ldz, int trans_out) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (m < 0) return -2;
  if (cc < 0) return -3;
  if (k < 0) return -4;
  if (!A && m * k > 0) return -5;
  if (lda < std::max<int64_t>(1, m)) return -6;
  if (!V && m * cc > 0) return -7;
  if (ldv < std::max<int64_t>(1, m)) return -8;
  if (!Z && k * cc > 0) return -9;
  if (ldz < std::max<int64_t>(1, trans_out ? cc : k)) return -10;
  return guarded(h, [&] {
    Ctx c = make_ctx(h);
    size_t pe = gemm_partials_needed(k, cc, m, c.num_sms);
    char *ws = get_ws(h, pe * 8 + 256, true);
    if (k > 0 && cc > 0) {
      if (m == 0) launch_copy(c, trans_out ? cc : k, trans_out ? k : cc, nullptr, 0, Z, ldz, false);
      else gemm_tn(c, m, cc, k, A, lda, V, ldv, Z, ldz, trans_out != 0, (double *)ws, pe);
    }
    h->launches = c.launches;
    return RQLP_OK;
  });
}

int rqlp_orth(rqlp_handle_t h, int64_t m, int64_t cc, const double *Y, int64_t ldy, double *V, int64_t ldv, double *R,
              int64_t ldr) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (m < 1) return -2;
  if (cc < 1 || cc > m) return -3;
  if (!Y) return -4;
  if (ldy < m) return -5;
  if (!V || V == Y) return -6;
  if (ldv < m) return -7;
  if (R && ldr < cc) return -9;
  return guarded(h, [&] {
    Ctx c = make_ctx(h);
    Arena a;
    OrthScratch s;
    orth_carve(a, s, m, cc, c.num_sms);
    size_t need = a.used + 256;
    a = Arena();
    a.base = get_ws(h, need, true);
    a.cap = need;
    orth_carve(a, s, m, cc, c.num_sms);
    RQLP_CUDA(cudaMemsetAsync(c.dflags, 0, NUM_DEV_FLAGS * sizeof(unsigned), c.stream));
    orth(c, s, m, cc, Y, ldy, V, ldv, R, ldr, false);
    h->launches = c.launches;
    return RQLP_OK;
  });
}

int rqlp_cpqr(rqlp_handle_t h, int64_t rows, int64_t cols, const double *M, int64_t ldm, double *Q, int64_t ldq,
              double *R, int64_t ldr, int64_t *perm) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (rows < 1 || rows > 24576) return -2;
  if (cols < 1) return -3;
  if (!M) return -4;
  if (ldm < rows) return -5;
  int64_t s = std::min(rows, cols);
  if (Q && ldq < rows) return -7;
  if (R && ldr < s) return -9;
  return guarded(h, [&] {
    Ctx c = make_ctx(h);
    Arena a;
    HHScratch hs;
    int64_t ldw = round_up(rows, 8);
    a.take<double>(ldw * cols);
    hh_carve(a, hs, rows, cols, c.num_sms);
    size_t need = a.used + 256;
    a = Arena();
    a.base = get_ws(h, need, true);
    a.cap = need;
    double *Wk = a.take<double>(ldw * cols);
    hh_carve(a, hs, rows, cols, c.num_sms);
    launch_copy(c, rows, cols, M, ldm, Wk, ldw, false);
    hh_factor(c, hs, rows, cols, Wk, ldw, true);
    if (R) hh_extract_r(c, hs, rows, cols, Wk, ldw, R, ldr, false);
    if (Q) hh_form_q(c, hs, rows, cols, Q, ldq);
    if (perm) hh_copy_perm(c, hs, cols, perm);
    h->launches = c.launches;
    return RQLP_OK;
  });
}

int rqlp_qlp_tail(rqlp_handle_t h, int64_t l, int64_t n, const double *B, int64_t ldb, int d, double *QB, int64_t ldqb,
                  double *T, int64_t ldt, double *PB, int64_t ldpb, int64_t *piv0, int64_t *piv1, int *t_is_upper) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (l < 1) return -2;
  if (n < l) return -3;
  if (!B) return -4;
  if (ldb < l) return -5;
  if (d < 0) return -6;
  if (!QB) return -7;
  if (ldqb < l) return -8;
  if (!T) return -9;
  if (ldt < l) return -10;
  if (!PB) return -11;
  if (ldpb < n) return -12;
  if (t_is_upper) *t_is_upper = (d >= 2 && d % 2 == 0) ? 1 : 0;
  return guarded(h, [&] {
    Ctx c = make_ctx(h);
    Arena a;
    TailScratch s;
    tail_carve(a, s, l, n, c.num_sms);
    size_t need = a.used + 256;
    a = Arena();
    a.base = get_ws(h, need, true);
    a.cap = need;
    tail_carve(a, s, l, n, c.num_sms);
    RQLP_CUDA(cudaMemsetAsync(c.dflags, 0, NUM_DEV_FLAGS * sizeof(unsigned), c.stream));
    launch_copy(c, l, n, B, ldb, s.Bw, s.ldl, false);
    qlp_tail(c, s, l, n, s.Bw, s.ldl, d, QB, ldqb, T, ldt, PB, ldpb, piv0, piv1);
    h->launches = c.launches;
    return RQLP_OK;
  });
}

int rqlp_residual_sq(rqlp_handle_t h, int64_t m, int64_t n, int64_t l, const double *A, int64_t lda, const double *Q,
                     int64_t ldq, const double *T, int64_t ldt, const double *P, int64_t ldp, double *res_dev) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  if (m < 1) return -2;
  if (n < 1) return -3;
  if (l < 1) return -4;
  if (!A) return -5;
  if (lda < m) return -6;
  if (!Q) return -7;
  if (ldq < m) return -8;
  if (!T) return -9;
  if (ldt < l) return -10;
  if (!P) return -11;
  if (ldp < n) return -12;
  if (!res_dev) return -13;
  return guarded(h, [&] {
    Ctx c = make_ctx(h);
    int64_t ldl = round_up(l, 8);
    size_t need = ((size_t)ldl * n + 4096 * (size_t)n + 2048) * 8 + 1024;
    char *ws = get_ws(h, need, true);
    double *M = (double *)ws;  // M = T P^T  (l x n)
    gemm_generic_ex(c, false, true, l, n, l, 1.0, T, ldt, P, ldp, 0.0, M, ldl, nullptr, 0, false, nullptr, 0);
    double *part = M + round_up(ldl * n, 32);
    residual_sq(c, m, n, l, A, lda, Q, ldq, M, ldl, part, res_dev);
    h->launches = c.launches;
    return RQLP_OK;
  });
}

int rqlp_set_stage_outputs(rqlp_handle_t h, double *Y, int64_t ldy, double *V, int64_t ldv, double *B, int64_t ldb) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  h->dbgY = Y; h->ldY = ldy;
  h->dbgV = V; h->ldV = ldv;
  h->dbgB = B; h->ldB = ldb;
  return RQLP_OK;
}

int rqlp_set_power_stage_outputs(rqlp_handle_t h, double *Vpre, int64_t ldvp, double *Z, int64_t ldz, double *W,
                                 int64_t ldw, double *Ypow, int64_t ldyp) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  h->dbgVP = Vpre; h->ldVP = ldvp;
  h->dbgZ = Z; h->ldZ = ldz;
  h->dbgW = W; h->ldW = ldw;
  h->dbgYP = Ypow; h->ldYP = ldyp;
  return RQLP_OK;
}

int rqlp_set_timing(rqlp_handle_t h, int enable) {
  if (!valid(h)) return RQLP_ERR_HANDLE;
  h->timing = enable != 0;
  return RQLP_OK;
}

int rqlp_get_timing(rqlp_handle_t h, const char **names, float *ms, int capacity) {
  if (!valid(h)) return -RQLP_ERR_HANDLE;
  int rc = guarded(h, [&] {
    RQLP_CUDA(cudaStreamSynchronize(h->stream));
    h->names_out.clear();
    h->ms_out.clear();
    auto &ev = h->cur_events ? *h->cur_events : h->events;
    RQLP_CUDA(cudaStreamSynchronize(h->gstream ? h->gstream : h->stream));
    for (size_t i = 1; i < ev.size(); ++i) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[i - 1].second, ev[i].second);
      h->names_out.push_back(ev[i].first);
      h->ms_out.push_back(t);
    }
    return RQLP_OK;
  });
  if (rc) return -rc;
  int nout = (int)h->names_out.size();
  for (int i = 0; i < nout && i < capacity; ++i) {
    if (names) names[i] = h->names_out[i].c_str();
    if (ms) ms[i] = h->ms_out[i];
  }
  return nout;
}

int64_t rqlp_launch_count(rqlp_handle_t h) { return valid(h) ? h->launches : -1; }
int64_t rqlp_careful_rerun_count(rqlp_handle_t h) { return valid(h) ? h->careful_reruns : -1; }

// Debug only (not in rqlp.h): copy the engine phase trace (RQLP_ENGINE_TRACE=1) to the host.
int rqlp_debug_trace(unsigned long long *host, int count) {
  if (!g_trace || !host) return -1;
  cudaDeviceSynchronize();
  return cudaMemcpy(host, g_trace, sizeof(unsigned long long) * count, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
}

}  // extern "C"
