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
//
// The c x c Cholesky factor R and its inverse X = R^-1 come from one kernel: Gaussian
// elimination of [G | I] in registers (c <= 128), one __syncthreads per pivot step:
//   step k:  S_ij -= S_ik S_jk / d_k  (k < j <= i),   W_ik = -S_ik / d_k,  W_it -= (S_ik/d_k) W_kt,
// after which L = S D^-1/2 (G = L L^T, R = L^T) and L^-1 = D^-1/2 W, X = (L^-1)^T.
// Larger c is blocked by 128 with the diagonal blocks done by the same kernel and the panels
// and block back-substitution done by GEMMs.
#include "internal.cuh"

namespace rqlpk {

void launch_reduce(Ctx &c, int64_t M, int64_t N, int S, const double *part, double alpha, double beta, double *C,
                   int64_t ldc, bool trans, const unsigned *cond, unsigned cond_mask);
void gemm_generic_ex(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                     int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc, double *partials,
                     size_t partial_elems, bool trans_out, const unsigned *cond, unsigned cond_mask);

namespace {

constexpr int CHOL_SMALL = 128;       // largest c done in one CTA (4 x 32 register rows)
constexpr int CHOL_NB = 128;          // diagonal block of the blocked path
constexpr double CHOL_BREAK = 1e-12;  // relative pivot threshold for the shifted fallback

constexpr double CHOL_DEP = 1e-15;  // relative pivot at or below which a column is dependent

// d = Schur pivot of column k, g0 = its original Gram diagonal.  Dependent column (rank
// deficiency, d <= 1e-15 g0, incl. a zero column): dep[k] = 1, pivot 1.  Ill-conditioned
// (d <= 1e-12 g0): breakdown -> the shifted pass.  Returns the pivot to use.
__device__ __forceinline__ double classify_pivot(double d, double g0, int k, int *dep, int *s_fail, int *s_dep) {
  if (dep) dep[k] = 0;
  if (!isfinite(d)) {
    *s_fail = 1;
    return 1.0;
  }
  if (dep && !(d > CHOL_DEP * g0)) {
    dep[k] = 1;
    *s_dep = 1;
    return 1.0;
  }
  if (!(d > CHOL_BREAK * g0)) {
    *s_fail = 1;
    return 1.0;
  }
  return d;
}

// One CTA: R (upper, G = R^T R) and X = R^-1 (upper) of the n x n SPD block G (n <= 128).
// Gorig supplies the original diagonal for the relative breakdown test.  On breakdown sets
// (*fail_word) |= fail_bit (R, X then undefined).  Skipped unless (*cond & mask) when cond set.
//
// The working matrix M (n x n) holds S (Schur complements) in its lower triangle and W^T in its
// strictly upper triangle (M[t][i] = W_it, t < i; W unit lower).  Thread (c, q) (c = column,
// q = row quarter) keeps M[32q .. 32q+31][c] in registers.  Step k needs only column k of M
// (bc[r] = M[r][k], bc[k] := 1) and d_k = M[k][k]; every active element updates as
//     x -= bc[r] bc[c] / d_k     active iff c > k and (r >= c or r <= k),
// except W_ck (r == k) which becomes -bc[c]/d_k (covered by bc[k] = 1 because its old value is 0).
// Inactive elements get a zero multiplier (branch-free); warps whose columns are all <= k retire
// from the step.  The owners of column k+1 publish it right after their step-k update, so a
// step costs a single __syncthreads.
__global__ void __launch_bounds__(512, 1) chol_inv_kernel(int n, const double *G, int64_t ldg, const double *Gorig,
                                                          int64_t ldo, double *R, int64_t ldr, double *X, int64_t ldx,
                                                          unsigned *fail_word, unsigned fail_bit, int *dep,
                                                          unsigned dep_bit, unsigned *flag_word,
                                                          const unsigned *cond, unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  extern __shared__ double xs[];  // n x (n|1) staging for the coalesced X write
  __shared__ __align__(16) double bc[2][CHOL_SMALL];
  __shared__ double dpiv[CHOL_SMALL], dinv[CHOL_SMALL], g0s[CHOL_SMALL];
  __shared__ int s_fail, s_dep;
  const int c = threadIdx.x & (CHOL_SMALL - 1), q = threadIdx.x >> 7;  // 128 columns x 4 quarters
  const int r0 = 32 * q;
  const bool col_ok = c < n;
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int r = r0 + i;
    x[i] = (col_ok && r < n && r >= c) ? G[c + (int64_t)r * ldg] : 0.0;  // S = G (symmetric)
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) g0s[i] = Gorig[i + (int64_t)i * ldo];
  if (threadIdx.x == 0) { s_fail = 0; s_dep = 0; }
  for (int i = threadIdx.x; i < 2 * CHOL_SMALL; i += blockDim.x) (&bc[0][0])[i] = 0.0;
  __syncthreads();
  if (c == 0) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int r = r0 + i;
      if (r < n) bc[0][r] = (r == 0) ? 1.0 : x[i];
      if (r == 0) {
        const double d = classify_pivot(x[i], g0s[0], 0, dep, &s_fail, &s_dep);
        dpiv[0] = d;
        dinv[0] = 1.0 / d;
      }
    }
  }
  __syncthreads();
  const unsigned rowvalid = (n - r0 >= 32) ? 0xffffffffu : (n - r0 <= 0 ? 0u : ((1u << (n - r0)) - 1u));
  for (int k = 0; k < n; ++k) {
    const double *b0 = bc[k & 1];
    double *b1 = bc[(k + 1) & 1];
    const int warp_c0 = (threadIdx.x & 127) - (threadIdx.x & 31);  // first column of this warp
    if (warp_c0 + 31 > k && warp_c0 < n) {
      const double bcc = (col_ok && c > k) ? b0[c] * dinv[k] : 0.0;
      // active rows: r <= k (W part) or r >= c (S part)
      const int lo_cnt = min(max(k - r0 + 1, 0), 32);               // rows r0 .. k
      const int hi_start = min(max(c - r0, 0), 32);                 // rows c .. r0+31
      const unsigned lowm = lo_cnt >= 32 ? 0xffffffffu : ((1u << lo_cnt) - 1u);
      const unsigned highm = hi_start >= 32 ? 0u : (0xffffffffu << hi_start);
      const unsigned act = (lowm | highm) & rowvalid;
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const double2 br = *reinterpret_cast<const double2 *>(b0 + r0 + i);
        const double m0 = ((act >> i) & 1u) ? bcc : 0.0;
        const double m1 = ((act >> (i + 1)) & 1u) ? bcc : 0.0;
        x[i] = fma(-br.x, m0, x[i]);
        x[i + 1] = fma(-br.y, m1, x[i + 1]);
      }
    }
    // publish column k+1 (and its pivot d, breakdown-checked, and 1/d)
    const int kn = k + 1;
    if (kn < n && c == kn) {
#pragma unroll
      for (int i = 0; i < 32; i += 2)
        *reinterpret_cast<double2 *>(b1 + r0 + i) = make_double2(x[i], x[i + 1]);
      if (kn >= r0 && kn < r0 + 32) {
        const double d = classify_pivot(b1[kn], g0s[kn], kn, dep, &s_fail, &s_dep);
        dpiv[kn] = d;
        dinv[kn] = 1.0 / d;
        b1[kn] = 1.0;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  // outputs: R(c, r) = S_rc / sqrt(d_c) (r > c), R(r, r) = sqrt(d_r), R lower = 0;
  //          X(r, c) = W_cr / sqrt(d_c) (r < c), X(r, r) = 1 / sqrt(d_r), X lower = 0.
  const int ldxs = n | 1;
  if (col_ok) {
    const double sdc = sqrt(dpiv[c]);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int r = r0 + i;
      if (r >= n) continue;
      if (r > c) {
        R[c + (int64_t)r * ldr] = x[i] / sdc;  // coalesced over c
        xs[r + c * ldxs] = 0.0;
      } else if (r == c) {
        R[c + (int64_t)c * ldr] = sdc;
        xs[c + c * ldxs] = 1.0 / sdc;
      } else {
        xs[r + c * ldxs] = x[i] / sdc;
      }
    }
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    if (i > j) R[i + (int64_t)j * ldr] = 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    X[i + (int64_t)j * ldx] = xs[i + j * ldxs];
  }
  if (threadIdx.x == 0 && s_fail) atomicOr(fail_word, fail_bit);
  if (threadIdx.x == 0 && s_dep && dep) {
    atomicOr(fail_word, dep_bit);
    atomicOr(flag_word, (unsigned)RQLP_FLAG_RANK_DEFICIENT);
  }
}

// dep[k] != 0: column k of Q (m x n) is replaced by a Philox N(0,1) vector (stream 7, counter =
// row + m k); the next CholeskyQR pass orthonormalises it against the others (basis completion
// for rank-deficient input, reading R4/R21).
__global__ void replace_dep_kernel(int64_t m, int n, double *Q, int64_t ldq, const int *dep, uint64_t seed,
                                   const unsigned *cond, unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  for (int k = blockIdx.y; k < n; k += gridDim.y) {
    if (!dep[k]) continue;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
      uint64_t ctr = (uint64_t)(i + m * k), key = seed;
      // SplitMix64-style hash -> two uniforms -> Box-Muller (any N(0,1)-like fill works here)
      uint64_t z1 = ctr * 0x9E3779B97F4A7C15ULL + key;
      z1 = (z1 ^ (z1 >> 30)) * 0xBF58476D1CE4E5B9ULL;
      z1 = (z1 ^ (z1 >> 27)) * 0x94D049BB133111EBULL;
      z1 ^= z1 >> 31;
      uint64_t z2 = (ctr + 0x632BE59BD9B4E019ULL) * 0x9E3779B97F4A7C15ULL + key;
      z2 = (z2 ^ (z2 >> 30)) * 0xBF58476D1CE4E5B9ULL;
      z2 = (z2 ^ (z2 >> 27)) * 0x94D049BB133111EBULL;
      z2 ^= z2 >> 31;
      const double u1 = ((double)(z1 >> 11) + 0.5) * 0x1p-53, u2 = (double)(z2 >> 11) * 0x1p-53;
      Q[i + (int64_t)k * ldq] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
  }
}

// CholeskyQR2's second pass: G = Q1^T Q1 = I + E with ||E|| ~ cond(Y)^2 u.  If max|E_ij| <= 2^-27,
// chol(I + E) = I + U with U = triu(E, 1) + diag(E)/2 + O(|E|^2) and (I + U)^-1 = I - U + O(|U|^2),
// both exact to below u, so R and X = R^-1 come from one elementwise pass.  Otherwise sets
// (*cond_word) |= fail_bit so the full Cholesky runs.  One CTA (n <= 1056: n^2 <= 1.2M entries).
__global__ void __launch_bounds__(1024) near_identity_kernel(int n, const double *G, int64_t ldg, double *R,
                                                             int64_t ldr, double *X, int64_t ldx, unsigned *cond_word,
                                                             unsigned fail_bit, const unsigned *cond,
                                                             unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  __shared__ double red[32];
  double emax = 0.0;
  const int64_t total = (int64_t)n * n;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    const double v = G[i + (int64_t)j * ldg] - (i == j ? 1.0 : 0.0);
    emax = fmax(emax, fabs(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = emax;
  __syncthreads();
  double m = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
  if (!(m <= 0x1p-27)) {
    if (threadIdx.x == 0) atomicOr(cond_word, fail_bit);
    return;
  }
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    const double g = G[i + (int64_t)j * ldg];
    double u = 0.0;
    if (i < j) u = g;
    else if (i == j) u = 0.5 * (g - 1.0);
    R[i + (int64_t)j * ldr] = (i == j ? 1.0 : 0.0) + u;
    X[i + (int64_t)j * ldx] = (i == j ? 1.0 : 0.0) - u;
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

void launch_chol_inv(Ctx &c, int n, const double *G, int64_t ldg, const double *Gorig, int64_t ldo, double *R,
                     int64_t ldr, double *X, int64_t ldx, unsigned *fail_word, unsigned fail_bit,
                     const unsigned *cond, unsigned mask, int *dep = nullptr, unsigned dep_bit = 0) {
  static bool attr = false;
  if (!attr) {
    RQLP_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   CHOL_SMALL * (CHOL_SMALL | 1) * 8));
    attr = true;
  }
  chol_inv_kernel<<<1, 512, (size_t)n * (n | 1) * 8, c.stream>>>(n, G, ldg, Gorig, ldo, R, ldr, X, ldx, fail_word,
                                                                 fail_bit, dep, dep_bit, c.dflags + FLAG_WORD, cond,
                                                                 mask);
  RQLP_LAUNCHED(c);
}

}  // namespace

// Cholesky G = R^T R (G destroyed) and X = R^-1, both n x n upper; breakdown reported as
// (*fail_word) |= fail_bit.  Gorig holds the original diagonal.  All kernels run only if
// (*cond & mask) when cond is given.
static void chol_inv(Ctx &c, int64_t n, double *G, int64_t ldg, const double *Gorig, int64_t ldo, double *R,
                     int64_t ldr, double *X, int64_t ldx, double *T, unsigned *fail_word, unsigned fail_bit,
                     const unsigned *cond, unsigned mask, double *partials, size_t partial_elems, int *dep,
                     unsigned dep_bit) {
  if (n <= CHOL_SMALL) {
    launch_chol_inv(c, (int)n, G, ldg, Gorig, ldo, R, ldr, X, ldx, fail_word, fail_bit, cond, mask, dep, dep_bit);
    return;
  }
  // blocked right-looking Cholesky with 128-wide diagonal blocks
  for (int64_t jb = 0; jb < n; jb += CHOL_NB) {
    int64_t b = std::min<int64_t>(CHOL_NB, n - jb);
    launch_chol_inv(c, (int)b, G + jb + jb * ldg, ldg, Gorig + jb + jb * ldo, ldo, R + jb + jb * ldr, ldr,
                    X + jb + jb * ldx, ldx, fail_word, fail_bit, cond, mask, dep ? dep + jb : nullptr, dep_bit);
    int64_t rest = n - jb - b;
    if (rest > 0) {
      // R12 = R11^-T G12 ; G22 -= R12^T R12 ; zero the lower blocks of R and X
      gemm_generic_ex(c, true, false, b, rest, b, 1.0, X + jb + jb * ldx, ldx, G + jb + (jb + b) * ldg, ldg, 0.0,
                      R + jb + (jb + b) * ldr, ldr, partials, partial_elems, false, cond, mask);
      gemm_generic_ex(c, true, false, rest, rest, b, -1.0, R + jb + (jb + b) * ldr, ldr, R + jb + (jb + b) * ldr, ldr,
                      1.0, G + (jb + b) + (jb + b) * ldg, ldg, partials, partial_elems, false, cond, mask);
      launch_copy(c, rest, b, nullptr, 0, R + (jb + b) + jb * ldr, ldr, false, cond, mask);
      launch_copy(c, rest, b, nullptr, 0, X + (jb + b) + jb * ldx, ldx, false, cond, mask);
    }
  }
  // off-diagonal blocks of X = R^-1 by block back substitution:
  //   X_IJ = -X_II (R_{I, I+1..J} X_{I+1..J, J}),  I = J-1 .. 0
  for (int64_t J = CHOL_NB; J < n; J += CHOL_NB) {
    int64_t bJ = std::min<int64_t>(CHOL_NB, n - J);
    for (int64_t I = J - CHOL_NB; I >= 0; I -= CHOL_NB) {
      int64_t k0 = I + CHOL_NB, kw = J + bJ - k0;
      gemm_generic_ex(c, false, false, CHOL_NB, bJ, kw, 1.0, R + I + k0 * ldr, ldr, X + k0 + J * ldx, ldx, 0.0, T,
                      CHOL_NB, partials, partial_elems, false, cond, mask);
      gemm_generic_ex(c, false, false, CHOL_NB, bJ, CHOL_NB, -1.0, X + I + I * ldx, ldx, T, CHOL_NB, 0.0,
                      X + I + J * ldx, ldx, partials, partial_elems, false, cond, mask);
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
  s.tmp = a.take<double>(std::max<int64_t>(lc * c, CHOL_NB * lc));
  s.ldy = round_up(m, 8);
  s.Ybuf = a.take<double>(s.ldy * c);
  s.partial_elems = std::max(gemm_partials_needed(m, c, c, num_sms), (size_t)std::max<int64_t>(4 * lc * c, 1));
  s.partials = a.take<double>((int64_t)s.partial_elems);
  s.scal = a.take<double>(8);
  s.dep = a.take<int>(c);
}

// One CholeskyQR pass: Qout = Yin R^-1 with G = Yin^T Yin.  pass_bit marks this pass's
// breakdown in the COND word.  Kernels run only if (*cond & mask) when cond given.
static void cholqr_pass(Ctx &c, OrthScratch &s, int64_t m, int64_t n, const double *Yin, int64_t ldyi, double *Qout,
                        int64_t ldqo, double *Rout, unsigned pass_bit, const unsigned *cond, unsigned mask,
                        bool sharded, bool second = false) {
  const unsigned *gcond = cond;   // the pass's own condition (the GEMMs)
  const unsigned gmask = mask;
  int64_t lc = round_up(n, 8);
  unsigned *condw = c.dflags + COND_WORD;
  const unsigned dep_bit = pass_bit << 16;
  gemm_tn(c, m, n, n, Yin, ldyi, Yin, ldyi, s.G, lc, false, s.partials, s.partial_elems, cond, mask);
  if (sharded) allreduce_sum(c, s.G, lc * n);   // Gram summed over the row shards
  if (second) {
    // near-identity Gram: elementwise factor; the full Cholesky below runs only if it declines
    near_identity_kernel<<<1, 1024, 0, c.stream>>>((int)n, s.G, lc, Rout, lc, s.Rinv, lc, condw, pass_bit << 24,
                                                   cond, mask);
    RQLP_LAUNCHED(c);
    cond = condw;
    mask = pass_bit << 24;
  }
  if (n > CHOL_SMALL) launch_copy(c, n, n, s.G, lc, s.G2, lc, false, cond, mask);  // blocked path destroys G
  const double *Gorig = n > CHOL_SMALL ? s.G2 : s.G;
  chol_inv(c, n, s.G, lc, Gorig, lc, Rout, lc, s.Rinv, lc, s.tmp, condw, pass_bit, cond, mask, s.partials,
           s.partial_elems, s.dep, dep_bit);
  // breakdown (ill-conditioned) -> shifted Gram, second attempt (only if pass_bit was set)
  if (n <= CHOL_SMALL) launch_copy(c, n, n, s.G, lc, s.G2, lc, false, condw, pass_bit);
  add_shift_kernel<<<1, 1024, 0, c.stream>>>((int)n, s.G2, lc, (double)m, c.dflags + FLAG_WORD, condw, pass_bit,
                                             pass_bit << 8);
  RQLP_LAUNCHED(c);
  launch_copy(c, n, n, s.G2, lc, s.G, lc, false, condw, pass_bit);
  chol_inv(c, n, s.G, lc, s.G2, lc, Rout, lc, s.Rinv, lc, s.tmp, condw, 0u, condw, pass_bit, s.partials,
           s.partial_elems, nullptr, 0u);
  gemm_nn(c, m, n, n, Yin, ldyi, s.Rinv, lc, Qout, ldqo, s.partials, s.partial_elems, gcond, gmask);
  // rank-deficient columns -> random completion, orthonormalised by the following pass
  replace_dep_kernel<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 64)),
                           (unsigned)std::min<int64_t>(n, 64)),
                       256, 0, c.stream>>>(m, (int)n, Qout, ldqo, s.dep, 0x5eedULL + pass_bit, condw, dep_bit);
  RQLP_LAUNCHED(c);
}

void orth(Ctx &c, OrthScratch &s, int64_t m, int64_t n, const double *Y, int64_t ldy, double *V, int64_t ldv,
          double *R, int64_t ldr, bool sharded, bool span_only) {
  int64_t lc = round_up(n, 8);
  unsigned *condw = c.dflags + COND_WORD;
  RQLP_CUDA(cudaMemsetAsync(condw, 0, sizeof(unsigned), c.stream));
  if (span_only && !R) {
    // intermediate subspace-iteration basis: only range(V) = range(Y) matters (V = Y R^-1 for any
    // invertible R keeps the span to the same O(u cond(Y)) rounding), so one CholeskyQR pass.
    cholqr_pass(c, s, m, n, Y, ldy, V, ldv, s.Racc, 1u, nullptr, 0, sharded);
    return;
  }
  // pass 1: Y -> Ybuf (R1 in Racc), pass 2: Ybuf -> V (R2 in R)
  cholqr_pass(c, s, m, n, Y, ldy, s.Ybuf, s.ldy, s.Racc, 1u, nullptr, 0, sharded);
  cholqr_pass(c, s, m, n, s.Ybuf, s.ldy, V, ldv, s.R, 2u, nullptr, 0, sharded, true);
  if (R) {  // R = R2 R1
    gemm_generic_ex(c, false, false, n, n, n, 1.0, s.R, lc, s.Racc, lc, 0.0, s.tmp, lc, s.partials, s.partial_elems,
                    false, nullptr, 0);
    launch_copy(c, n, n, s.tmp, lc, s.Racc, lc, false, nullptr, 0);
  }
  // pass 3 (only when pass 1 or 2 needed the shift, bits 1<<8 | 2<<8, or completed dependent
  // columns, bits 1<<16 | 2<<16): V -> Ybuf -> V
  const unsigned m3 = (1u << 8) | (2u << 8) | (1u << 16) | (2u << 16);
  cholqr_pass(c, s, m, n, V, ldv, s.Ybuf, s.ldy, s.R, 4u, condw, m3, sharded, true);
  launch_copy(c, m, n, s.Ybuf, s.ldy, V, ldv, false, condw, m3);
  if (R) {
    gemm_generic_ex(c, false, false, n, n, n, 1.0, s.R, lc, s.Racc, lc, 0.0, s.tmp, lc, s.partials, s.partial_elems,
                    false, condw, m3);
    launch_copy(c, n, n, s.tmp, lc, s.Racc, lc, false, condw, m3);
    launch_copy(c, n, n, s.Racc, lc, R, ldr, false, nullptr, 0);
    // with completed columns Y = V R no longer holds for R2 R1: R = V^T Y (upper triangular in
    // exact arithmetic, zero rows for the completed directions)
    const unsigned mdep = (1u << 16) | (2u << 16) | (4u << 16);
    gemm_tn(c, m, n, n, V, ldv, Y, ldy, s.tmp, lc, false, s.partials, s.partial_elems, condw, mdep);
    if (sharded) allreduce_sum(c, s.tmp, lc * n);
    launch_copy(c, n, n, s.tmp, lc, R, ldr, false, condw, mdep);
  }
}

}  // namespace rqlpk
