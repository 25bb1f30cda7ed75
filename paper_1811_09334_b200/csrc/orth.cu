// orth.cu -- orthonormalisation of tall-skinny blocks: CholeskyQR2 with a shifted CholeskyQR3
// fallback (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020).
//
// Alg.1 l.3 "[V, ~] = qr(Y)", the power steps (reading R12), the BRQLP range
// finder and re-orthogonalisation (Alg.3 l.4-5) and the tall QR of R0^T in
// the tail (Alg.2 l.7 with i = 1; the unpivoted part of cpqr(R0^T), reading R6) all need the
// thin Q (and sometimes R) of an m x c matrix with m >> c.  The paper uses Householder QR; on
// B200 the Householder panel loop is latency bound, so we use the BLAS-3 CholeskyQR2:
//   G = Y^T Y (TN pass), R1 = chol(G), Q1 = Y R1^-1 (NN pass), repeated once,
// which yields the same unique thin Q (R_ii > 0) to rounding when cond(Y) < ~1e7 (readings R3,
// R19).  A Cholesky pivot d_j <= 1e-12 G_jj (cond(Y) >~ 1e6) switches the pass to the shifted
// Gram G + s I, s = 11 (m c + c (c+1)) u ||Y||_F^2, and enables a third pass (sCholQR3).  All of
// this is decided on the device (no host sync): the conditional kernels read a flag word.
#include "internal.cuh"

namespace rqlpk {

void launch_reduce(Ctx &c, int64_t M, int64_t N, int S, const double *part, double alpha, double beta, double *C,
                   int64_t ldc, bool trans, const unsigned *cond, unsigned cond_mask);
void gemm_generic_ex(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                     int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc, double *partials,
                     size_t partial_elems, bool trans_out, const unsigned *cond, unsigned cond_mask);

namespace {

constexpr int CHOL_NB = 128;          // diagonal block handled in shared memory
constexpr double CHOL_BREAK = 1e-12;  // relative pivot threshold for the shifted fallback

// Cholesky G = R^T R of one nb x nb diagonal block in shared memory (right-looking, upper R).
// Gorig gives the original diagonal for the relative breakdown test.  On breakdown sets
// fail_word |= fail_bit and leaves R undefined.  Skipped unless (*cond & mask) (when cond set).
__global__ void __launch_bounds__(1024) chol_block_kernel(int nb, double *G, int64_t ldg, const double *Gorig,
                                                          int64_t ldo, double *R, int64_t ldr, unsigned *fail_word,
                                                          unsigned fail_bit, const unsigned *cond,
                                                          unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  extern __shared__ double S[];  // nb x nb, col-major
  __shared__ int s_fail;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    S[e] = (i <= j) ? G[i + (int64_t)j * ldg] : 0.0;
  }
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (threadIdx.x == 0) {
      double d = S[j + j * nb];
      double g0 = Gorig[j + (int64_t)j * ldo];
      if (!(d > CHOL_BREAK * g0) || !isfinite(d)) {
        s_fail = 1;
        d = 1.0;
      }
      S[j + j * nb] = sqrt(d);
    }
    __syncthreads();
    double djj = S[j + j * nb];
    for (int cix = j + 1 + threadIdx.x; cix < nb; cix += blockDim.x) S[j + cix * nb] /= djj;
    __syncthreads();
    int t = nb - j - 1;
    for (int e = threadIdx.x; e < t * t; e += blockDim.x) {
      int r = j + 1 + e % t, cix = j + 1 + e / t;
      if (r <= cix) S[r + cix * nb] = fma(-S[j + r * nb], S[j + cix * nb], S[r + cix * nb]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    R[i + (int64_t)j * ldr] = (i <= j) ? S[e] : 0.0;
  }
  if (threadIdx.x == 0 && s_fail) atomicOr(fail_word, fail_bit);
}

// X = R^-1 (upper triangular n x n), one warp per column by back substitution.
__global__ void trtri_upper_kernel(int n, const double *R, int64_t ldr, double *X, int64_t ldx, const unsigned *cond,
                                   unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  const int lane = threadIdx.x & 31;
  const int W = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += W) {
    double *x = X + (int64_t)t * ldx;
    for (int r = lane; r < n; r += 32) x[r] = 0.0;
    __syncwarp();
    if (lane == 0) x[t] = 1.0 / R[t + (int64_t)t * ldr];
    __syncwarp();
    for (int i = t - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1 + lane; k <= t; k += 32) s = fma(R[i + (int64_t)k * ldr], x[k], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) x[i] = -s / R[i + (int64_t)i * ldr];
      __syncwarp();
    }
  }
}

// G2 += s I with s = 11 (m c + c(c+1)) u tr(G2); run only if (*cond & mask).  Marks the
// handle flag word (RQLP_FLAG_SHIFTED_CHOLQR) and the pass-3 condition bit.
__global__ void add_shift_kernel(int c, double *G, int64_t ldg, double m, unsigned *flag_word, unsigned *cond_word,
                                 unsigned cond_mask, unsigned set_bit) {
  if (((*cond_word) & cond_mask) == 0) return;
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < c; i += blockDim.x) s += G[i + (int64_t)i * ldg];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double tr = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tr += red[w];
  double shift = 11.0 * (m * c + (double)c * (c + 1)) * 0x1p-53 * tr;
  if (!(shift > 0.0)) shift = 1.0;  // zero matrix: any positive shift
  __syncthreads();
  for (int i = threadIdx.x; i < c; i += blockDim.x) G[i + (int64_t)i * ldg] += shift;
  if (threadIdx.x == 0) {
    atomicOr(flag_word, (unsigned)RQLP_FLAG_SHIFTED_CHOLQR);
    atomicOr(cond_word, set_bit);
  }
}

}  // namespace

// Cholesky of the c x c Gram G (destroyed) into upper R, blocked by CHOL_NB, with breakdown
// reported in (*cond_word) |= fail_bit.  Gorig holds the original diagonal.  All kernels run only
// if (*cond & mask) when cond is given.
static void chol_attempt(Ctx &c, int64_t n, double *G, int64_t ldg, const double *Gorig, int64_t ldo, double *R,
                         int64_t ldr, double *Xb, unsigned *fail_word, unsigned fail_bit, const unsigned *cond,
                         unsigned mask, double *partials, size_t partial_elems) {
  static bool attr = false;
  if (!attr) {
    RQLP_CUDA(cudaFuncSetAttribute(chol_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   CHOL_NB * CHOL_NB * 8 + 1024));
    attr = true;
  }
  for (int64_t jb = 0; jb < n; jb += CHOL_NB) {
    int b = (int)std::min<int64_t>(CHOL_NB, n - jb);
    chol_block_kernel<<<1, 1024, (size_t)b * b * 8, c.stream>>>(b, G + jb + jb * ldg, ldg, Gorig + jb + jb * ldo, ldo,
                                                                R + jb + jb * ldr, ldr, fail_word, fail_bit, cond, mask);
    RQLP_LAUNCHED(c);
    int64_t rest = n - jb - b;
    if (rest > 0) {
      trtri_upper_kernel<<<(b + 7) / 8, 256, 0, c.stream>>>(b, R + jb + jb * ldr, ldr, Xb, CHOL_NB, cond, mask);
      RQLP_LAUNCHED(c);
      // R12 = R11^-T G12
      gemm_generic_ex(c, true, false, b, rest, b, 1.0, Xb, CHOL_NB, G + jb + (jb + b) * ldg, ldg, 0.0,
                      R + jb + (jb + b) * ldr, ldr, partials, partial_elems, false, cond, mask);
      // G22 -= R12^T R12
      gemm_generic_ex(c, true, false, rest, rest, b, -1.0, R + jb + (jb + b) * ldr, ldr, R + jb + (jb + b) * ldr,
                      ldr, 1.0, G + (jb + b) + (jb + b) * ldg, ldg, partials, partial_elems, false, cond, mask);
      // zero the strictly lower block of R
      launch_copy(c, rest, b, nullptr, 0, R + (jb + b) + jb * ldr, ldr, false, cond, mask);
    }
  }
}

void orth_carve(Arena &a, OrthScratch &s, int64_t m, int64_t c, int num_sms) {
  int64_t lc = round_up(c, 8);
  s.G = a.take<double>(lc * c);
  s.G2 = a.take<double>(lc * c);
  s.R = a.take<double>(lc * c);
  s.Rinv = a.take<double>(lc * c);
  s.Racc = a.take<double>(lc * c);
  s.tmp = a.take<double>(std::max<int64_t>(lc * c, CHOL_NB * CHOL_NB));
  s.ldy = round_up(m, 8);
  s.Ybuf = a.take<double>(s.ldy * c);
  s.partial_elems = std::max(gemm_partials_needed(m, c, c, num_sms), (size_t)std::max<int64_t>(4 * lc * c, 1));
  s.partials = a.take<double>((int64_t)s.partial_elems);
  s.scal = a.take<double>(8);
}

// One CholeskyQR pass: Qout = Yin R^-1 with G = Yin^T Yin.  pass_bit marks this pass's
// breakdown in the COND word.  Kernels run only if (*cond & mask) when cond given.
static void cholqr_pass(Ctx &c, OrthScratch &s, int64_t m, int64_t n, const double *Yin, int64_t ldyi, double *Qout,
                        int64_t ldqo, double *Rout, unsigned pass_bit, const unsigned *cond, unsigned mask,
                        bool sharded) {
  int64_t lc = round_up(n, 8);
  unsigned *condw = c.dflags + COND_WORD;
  gemm_tn(c, m, n, n, Yin, ldyi, Yin, ldyi, s.G, lc, false, s.partials, s.partial_elems, cond, mask);
  if (sharded) allreduce_sum(c, s.G, lc * n);   // Gram summed over the row shards
  launch_copy(c, n, n, s.G, lc, s.G2, lc, false, cond, mask);
  chol_attempt(c, n, s.G, lc, s.G2, lc, Rout, lc, s.tmp, condw, pass_bit, cond, mask, s.partials, s.partial_elems);
  // breakdown -> shifted Gram from the saved copy, second attempt (only if pass_bit was set)
  add_shift_kernel<<<1, 1024, 0, c.stream>>>((int)n, s.G2, lc, (double)m, c.dflags + FLAG_WORD, condw, pass_bit,
                                             pass_bit << 8);
  RQLP_LAUNCHED(c);
  launch_copy(c, n, n, s.G2, lc, s.G, lc, false, condw, pass_bit);
  chol_attempt(c, n, s.G, lc, s.G2, lc, Rout, lc, s.tmp, condw, 0u, condw, pass_bit, s.partials, s.partial_elems);
  trtri_upper_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 8), (int64_t)c.num_sms * 4)), 256, 0,
                       c.stream>>>((int)n, Rout, lc, s.Rinv, lc, cond, mask);
  RQLP_LAUNCHED(c);
  gemm_nn(c, m, n, n, Yin, ldyi, s.Rinv, lc, Qout, ldqo, s.partials, s.partial_elems, cond, mask);
}

void orth(Ctx &c, OrthScratch &s, int64_t m, int64_t n, const double *Y, int64_t ldy, double *V, int64_t ldv,
          double *R, int64_t ldr, bool sharded) {
  int64_t lc = round_up(n, 8);
  unsigned *condw = c.dflags + COND_WORD;
  RQLP_CUDA(cudaMemsetAsync(condw, 0, sizeof(unsigned), c.stream));
  // pass 1: Y -> Ybuf (R1 in Racc), pass 2: Ybuf -> V (R2 in R)
  cholqr_pass(c, s, m, n, Y, ldy, s.Ybuf, s.ldy, s.Racc, 1u, nullptr, 0, sharded);
  cholqr_pass(c, s, m, n, s.Ybuf, s.ldy, V, ldv, s.R, 2u, nullptr, 0, sharded);
  if (R) {  // R = R2 R1
    gemm_generic_ex(c, false, false, n, n, n, 1.0, s.R, lc, s.Racc, lc, 0.0, s.tmp, lc, s.partials, s.partial_elems,
                    false, nullptr, 0);
    launch_copy(c, n, n, s.tmp, lc, s.Racc, lc, false, nullptr, 0);
  }
  // pass 3 (only when pass 1 or 2 needed the shift: bits 1<<8 | 2<<8): V -> Ybuf -> V
  const unsigned m3 = (1u << 8) | (2u << 8);
  cholqr_pass(c, s, m, n, V, ldv, s.Ybuf, s.ldy, s.R, 4u, condw, m3, sharded);
  launch_copy(c, m, n, s.Ybuf, s.ldy, V, ldv, false, condw, m3);
  if (R) {
    gemm_generic_ex(c, false, false, n, n, n, 1.0, s.R, lc, s.Racc, lc, 0.0, s.tmp, lc, s.partials, s.partial_elems,
                    false, condw, m3);
    launch_copy(c, n, n, s.tmp, lc, s.Racc, lc, false, condw, m3);
    launch_copy(c, n, n, s.Racc, lc, R, ldr, false, nullptr, 0);
  }
}

}  // namespace rqlpk
