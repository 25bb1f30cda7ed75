// internal.cuh -- shared declarations of librqlp's sm_100a kernels and host launchers.
// Nothing here is shared with oracle/ (the CUDA path and the oracle share no code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/rqlp.h"

namespace rqlpk {

// Thrown by host orchestration on a CUDA failure; converted to RQLP_ERR_CUDA at the C ABI.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define RQLP_CUDA(call)                                                                        \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      throw ::rqlpk::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +      \
                              __FILE__ + ":" + std::to_string(__LINE__));                      \
  } while (0)

// RQLP_SYNC_DEBUG=1: synchronise after every eager launch so a faulting kernel is named.
static inline bool sync_debug() {
  static const bool on = getenv("RQLP_SYNC_DEBUG") != nullptr;
  return on;
}

#define RQLP_LAUNCHED(ctx)                                                                     \
  do {                                                                                         \
    (ctx).launches++;                                                                          \
    cudaError_t e_ = cudaGetLastError();                                                       \
    if (e_ == cudaSuccess && ::rqlpk::sync_debug() && !(ctx).capturing)                               \
      e_ = cudaStreamSynchronize((ctx).stream);                                                \
    if (e_ != cudaSuccess)                                                                     \
      throw ::rqlpk::CudaError(std::string("launch: ") + cudaGetErrorString(e_) + " @" +        \
                              __FILE__ + ":" + std::to_string(__LINE__));                      \
  } while (0)

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Raise a kernel's dynamic shared-memory limit once per (device, kernel): the attribute is per
// device and one process may drive several devices (defined in api.cu).
void smem_attr(const void *kernel, int bytes);

#ifdef __CUDACC__
// 1/x and sqrt(x) to ~1 ulp without the IEEE routines' slow-path branches: MUFU seed + Newton
// steps (x positive and normal; callers handle zero / non-finite values before).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
// The completion vector of a dependent column (rank-deficient sketch, reading R4): a
// SplitMix64-style hash of the counter (row + m column) -> two uniforms -> Box-Muller.  Any
// N(0,1)-like fill works; orth.cu's replace_dep_kernel and orth_rescue.cu share it.
__device__ __forceinline__ double completion_value(uint64_t ctr, uint64_t key) {
  uint64_t z1 = ctr * 0x9E3779B97F4A7C15ULL + key;
  z1 = (z1 ^ (z1 >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z1 = (z1 ^ (z1 >> 27)) * 0x94D049BB133111EBULL;
  z1 ^= z1 >> 31;
  uint64_t z2 = (ctr + 0x632BE59BD9B4E019ULL) * 0x9E3779B97F4A7C15ULL + key;
  z2 = (z2 ^ (z2 >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z2 = (z2 ^ (z2 >> 27)) * 0x94D049BB133111EBULL;
  z2 ^= z2 >> 31;
  const double u1 = ((double)(z1 >> 11) + 0.5) * 0x1p-53, u2 = (double)(z2 >> 11) * 0x1p-53;
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}
__device__ __forceinline__ double fast_sqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // y ~ x^-1/2: two Newton steps on y, then s = x y with one correction (Markstein)
  double h = 0.5 * y;
  double g = x * y;
  double e = fma(-g, h, 0.5);
  g = fma(g, e, g);
  h = fma(h, e, h);
  e = fma(-g, g, x);
  return fma(e, h, g);
}
#endif
static inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Device-side flag words (one per handle, in the workspace).
enum DevFlag : int {
  FLAG_WORD = 0,       // RQLP_FLAG_* bits accumulated by the last call
  COND_WORD = 1,       // scratch condition for conditionally executed kernels
  BAR_COUNT = 2,       // cooperative grid barrier (count, generation)
  BAR_GEN = 3,
  STICKY_WORD = 4,     // row-sharded optimistic run: set when any orth took a shifted pass (-> careful rerun)
  NUM_DEV_FLAGS = 8
};

// Execution context of one call: stream, SM count, launch counter, device flag words.
struct Ctx {
  cudaStream_t stream = nullptr;
  int device = 0;
  int num_sms = 148;
  int64_t launches = 0;
  unsigned *dflags = nullptr;     // NUM_DEV_FLAGS words of device memory
  double *dind = nullptr;         // ||A||_F^2, sum_j ||B_j||_F^2 of the current factorisation
  bool timing = false;
  std::vector<std::pair<std::string, cudaEvent_t>> *events = nullptr;
  std::vector<cudaEvent_t> *pool = nullptr;  // pre-created events (no cudaEventCreate under capture)
  size_t pool_next = 0;
  bool capturing = false;
  // row-sharded runs only: the rare orth branch is not taken on the host (no COND-word readback per
  // orth); a breakdown only sets STICKY_WORD and the caller reruns the factorisation carefully
  bool optimistic = false;
  void mark(const char *name);
  // row-sharded runs (comm.cu): NCCL communicator, rank, number of ranks
  void *comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t collectives = 0;
  unsigned long long *trace = nullptr;  // debug: engine phase timestamps
  // a second stream for independent branches (fork/join by events; inside a CUDA-graph capture
  // the branch becomes a parallel path of the graph)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  Ctx branch() const {  // a context on the side stream, after the work enqueued so far
    if (cudaEventRecord(ev_fork, stream) != cudaSuccess || cudaStreamWaitEvent(side, ev_fork, 0) != cudaSuccess)
      throw CudaError("fork failed");
    Ctx b = *this;
    b.stream = side;
    b.timing = false;
    b.launches = 0;
    return b;
  }
  void join(const Ctx &b) {  // the main stream waits for the branch's work
    if (cudaEventRecord(ev_join, side) != cudaSuccess || cudaStreamWaitEvent(stream, ev_join, 0) != cudaSuccess)
      throw CudaError("join failed");
    launches += b.launches;
  }
};

// ---- exchange steps of row-sharded runs (comm.cu): NCCL or in-process loopback ranks ----
enum CommKind : int { COMM_NONE = 0, COMM_NCCL = 1, COMM_LOOPBACK = 2 };
struct NcclError : std::runtime_error {  // NCCL / loopback failures -> RQLP_ERR_NCCL
  using std::runtime_error::runtime_error;
};
int comm_unique_id(void *out);
void *comm_init(const void *uid, int rank, int nranks);
void *comm_loopback_group(int nranks, int device, cudaStream_t stream);
void *comm_loopback_init(void *group, int rank);
int comm_kind(void *comm);
void comm_destroy(void *comm);
int comm_async_error(void *comm);
// loopback ranks enqueue a factorisation only while they hold the group's turn
void comm_call_begin(void *comm);
void comm_call_end(void *comm, bool failed);
void allreduce_sum(Ctx &c, double *buf, int64_t count);
// after a sum whose result every rank must hold bit-identically (the replicated B): verify it across
// the ranks, RQLP_FLAG_REPLICA_MISMATCH on every rank otherwise (comm.cu)
void check_replicated(Ctx &c, const double *buf, int64_t count);

// Bump allocator over a workspace; base == nullptr measures only.
struct Arena {
  char *base = nullptr;
  size_t cap = 0, used = 0;
  template <typename T>
  T *take(int64_t count) {
    size_t bytes = (size_t)(count > 0 ? count : 1) * sizeof(T);
    size_t off = (used + 255) & ~(size_t)255;
    used = off + bytes;
    if (base && used > cap) throw std::runtime_error("workspace overflow");
    return base ? reinterpret_cast<T *>(base + off) : nullptr;
  }
};

// ---- Ω (omega.cu) ----
void launch_omega(Ctx &c, int64_t n, int64_t l, int64_t col0, uint64_t seed, double *Om, int64_t ldo);

// ---- GEMM (gemm.cu) ----
// ||A||_F^2 fused into an NN pass over A: per-CTA partials in `slots` (capacity `cap`), summed in
// fixed order into *out (device double).
struct FroSpec {
  double *slots = nullptr;
  int64_t cap = 0;
  double *out = nullptr;
  bool accumulate = false;  // *out += (row panels of one A), else *out =
};
static inline int64_t fro_slots_cap(int64_t m, int num_sms) { return ceil_div(m, 128) * 8 + 8 * (int64_t)num_sms; }
// Y = A X and *fro->out = ||A||_F^2 (the first A-pass; a separate fixed-order pass over A when the
// fused TMA kernel cannot be used)
void gemm_nn_fro(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X,
                 int64_t ldx, double *Y, int64_t ldy, double *partials, size_t partial_elems, const FroSpec &fro);
// C = alpha op(A) op(B) + beta C (generic DMMA kernel; any layout / alignment).
void gemm_generic(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                  int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                  const unsigned *cond = nullptr, unsigned cond_mask = 0);
// Y = A X  (A m x k, X k x c): tall-skinny pass.  Scratch for split-K partials.  tri = 2: X is
// upper triangular (k-tiles past the diagonal are skipped; a hint -- the result is the same).
void gemm_nn(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X,
             int64_t ldx, double *Y, int64_t ldy, double *partials, size_t partial_elems,
             const unsigned *cond = nullptr, unsigned cond_mask = 0, int tri = 0);
// Z = A^T V (k x c) or Z^T (c x k) when trans_out.  tri = 1: a symmetric product (Gram) of which
// only the upper triangle is needed -- the strictly lower part of Z is then left undefined.
void gemm_tn(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *V,
             int64_t ldv, double *Z, int64_t ldz, bool trans_out, double *partials, size_t partial_elems,
             const unsigned *cond = nullptr, unsigned cond_mask = 0, int tri = 0);
size_t gemm_partials_needed(int64_t m, int64_t cc, int64_t k, int num_sms);
// Y (m x cc) = alpha A X + beta Y (A m x k) and Z (k x cc) = alpha A^T V + beta Z (A m x k, V m x cc)
void gemm_nn_ab(Ctx &c, int64_t m, int64_t cc, int64_t k, double alpha, const double *A, int64_t lda, const double *X,
                int64_t ldx, double beta, double *Y, int64_t ldy, double *partials, size_t partial_elems);
void gemm_tn_ab(Ctx &c, int64_t m, int64_t cc, int64_t k, double alpha, const double *A, int64_t lda, const double *V,
                int64_t ldv, double beta, double *Z, int64_t ldz, double *partials, size_t partial_elems);

// ---- small dense (dense.cu) ----
void launch_copy(Ctx &c, int64_t rows, int64_t cols, const double *S, int64_t lds, double *D, int64_t ldd,
                 bool transpose, const unsigned *cond = nullptr, unsigned cond_mask = 0);
void launch_fill(Ctx &c, int64_t rows, int64_t cols, double *D, int64_t ldd, double diag, double off);
void launch_zero_u32(Ctx &c, unsigned *p, int64_t count);

// ---- orthonormalisation (orth.cu) ----
struct OrthScratch {
  double *G = nullptr, *G2 = nullptr, *R = nullptr, *Rinv = nullptr, *Racc = nullptr, *tmp = nullptr;
  double *Ybuf = nullptr;       // m x c ping-pong buffer
  int64_t ldy = 0;
  double *partials = nullptr;
  size_t partial_elems = 0;
  double *scal = nullptr;       // small device scalars
  int *dep = nullptr;           // dependent-column flags of the last Cholesky (rank deficiency)
  double *maxdev = nullptr;     // per-CTA max |G - I| of the second pass's near-identity test
};
void orth_carve(Arena &a, OrthScratch &s, int64_t m, int64_t c, int num_sms);
// orth's rare branch (orth_rescue.cu): if (*cond & mask), repeated (shifted) CholeskyQR passes on
// V (m x n) until orthonormal, then R = V^T Y (nullable); one cooperative kernel.
void launch_orth_rescue(Ctx &c, OrthScratch &s, int64_t m, int64_t n, double *V, int64_t ldv, const double *Y,
                        int64_t ldy, double *R, int64_t ldr, const unsigned *cond, unsigned mask);
// V = orth(Y) (CholeskyQR2; after a breakdown, shifted passes until orthonormal).  Y is preserved; Y and V must not alias.  R (nullable) receives the c x c triangular factor (Y = V R).
// sharded: Y is a row block of a row-sharded matrix -> the Gram is summed over ranks.
// span_only: an intermediate subspace-iteration basis (one CholeskyQR pass; V spans range(Y) but
// is only approximately orthonormal).
void orth(Ctx &ctx, OrthScratch &s, int64_t m, int64_t c, const double *Y, int64_t ldy, double *V, int64_t ldv,
          double *R, int64_t ldr, bool sharded = false, bool span_only = false);

// ---- Householder engine + QLP tail (householder.cu, tail.cu) ----
struct HHScratch {
  double *Vst = nullptr;        // rows x steps reflector store
  double *tau = nullptr, *beta = nullptr;
  unsigned long long *rec = nullptr, *cand = nullptr;
  int *done = nullptr;
  int64_t *perm = nullptr;
  int64_t max_rows = 0, max_cols = 0, max_slots = 0, max_steps = 0;
};
// steps < 0: min(rows, cols) (a full factorisation); otherwise a partial (truncated) one.
void hh_carve(Arena &a, HHScratch &s, int64_t rows, int64_t cols, int num_sms, int64_t steps = -1);
// In-place Householder QR (pivot: column-pivoted, Golub + LAPACK downdating) of M, `steps`
// reflectors.  Outputs in s: Vst, tau, beta, perm (full permutation).  M keeps R entries above
// the diagonal of each step's pivot column in ORIGINAL column positions.
void hh_factor(Ctx &c, HHScratch &s, int64_t rows, int64_t cols, double *M, int64_t ldm, bool pivot,
               int64_t steps = -1);
// R (steps x cols, pivot order, sign-normalised) or its transpose (cols x steps).
void hh_extract_r(Ctx &c, HHScratch &s, int64_t rows, int64_t cols, const double *M, int64_t ldm, double *R,
                  int64_t ldr, bool transpose, int64_t steps = -1);
// Explicit Q (rows x steps), sign-normalised.
void hh_form_q(Ctx &c, HHScratch &s, int64_t rows, int64_t cols, double *Q, int64_t ldq, int64_t steps = -1);
void hh_copy_perm(Ctx &c, HHScratch &s, int64_t count, int64_t *dst);

struct TailScratch {
  double *Bw = nullptr, *Rt = nullptr, *Qhat = nullptr, *Rhat = nullptr, *Q0 = nullptr, *Qt = nullptr,
         *Lt = nullptr, *Mt = nullptr, *QE = nullptr, *PO = nullptr, *tmp_ll = nullptr, *tmp_nl = nullptr;
  int64_t ldn = 0, ldl = 0;
  int64_t *perm0 = nullptr, *perm1 = nullptr;
  HHScratch hh;
  OrthScratch orth;
};
void tail_carve(Arena &a, TailScratch &s, int64_t l, int64_t n, int num_sms);
// B (l x n) is overwritten.  Outputs QB (l x l), T, PB (n x l), piv0/piv1 (device int64, nullable).
void qlp_tail(Ctx &c, TailScratch &s, int64_t l, int64_t n, double *B, int64_t ldb, int d, double *QB,
              int64_t ldqb, double *T, int64_t ldt, double *PB, int64_t ldpb, int64_t *piv0, int64_t *piv1);

// Truncated pivoted QLP of W (m x n, overwritten; tail.cu).  QR: m x l scratch for Q_R.
void tqlp(Ctx &c, TailScratch &s, HHScratch &hA, int64_t m, int64_t n, int64_t l, double *W, int64_t ldw, double *Q,
          int64_t ldq, double *L, int64_t ldl_out, double *P, int64_t ldp, int64_t *piv0, int64_t *piv1, double *QR,
          int64_t ldqr);

// *out (+)= ||X||_F^2, deterministic (dense.cu); part >= 1024 doubles
void fro2_accumulate(Ctx &c, int64_t rows, int64_t cols, const double *X, int64_t ldx, double *part, double *out,
                     bool first);

// ---- residual (dense.cu) ----
void residual_sq(Ctx &c, int64_t m, int64_t n, int64_t l, const double *A, int64_t lda, const double *Q,
                 int64_t ldq, const double *M, int64_t ldmm, double *partials, double *out);

}  // namespace rqlpk
