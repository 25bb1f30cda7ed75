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
// The c x c Cholesky factor R and its inverse X = R^-1 come from one kernel (chol_blk_kernel):
// Gauss-Jordan elimination of [G | I] in shared memory (c <= 128),
//   step k:  S_ij -= S_ik S_jk / d_k  (k < j <= i),   W_ik = -S_ik / d_k,  W_it -= (S_ik/d_k) W_kt,
// after which L = S D^-1/2 (G = L L^T, R = L^T) and L^-1 = D^-1/2 W, X = (L^-1)^T; the steps
// are taken 8 at a time (one warp factors the 8 x 8 diagonal block, the rank-8 updates are DMMA
// tile products).  Larger c is blocked by 128 with the diagonal blocks done by the same kernel
// and the panels and block back-substitution done by GEMMs.
#include "internal.cuh"

namespace rqlpk {

void launch_reduce(Ctx &c, int64_t M, int64_t N, int S, const double *part, double alpha, double beta, double *C,
                   int64_t ldc, bool trans, const unsigned *cond, unsigned cond_mask);
void gemm_generic_ex(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                     int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc, double *partials,
                     size_t partial_elems, bool trans_out, const unsigned *cond, unsigned cond_mask);

namespace {

constexpr int CHOL_SMALL = 128;       // largest c done in one CTA (shared-memory working matrix)
constexpr int CHOL_NB = 128;          // diagonal block of the blocked path
// Pivot classification (relative to the original Gram diagonal g0): d <= 1e-15 g0 is a dependent
// column (rank deficiency: pivot 1, the column is later replaced), d <= 1e-12 g0 is breakdown
// (cond(Y) >~ 1e6: the shifted pass), as is a non-finite d.
constexpr double CHOL_BREAK = 1e-12;
constexpr double CHOL_DEP = 1e-15;

// chol_blk_kernel: the elimination of [G | I] in 8-pivot blocks with the whole n x n working
// matrix M in shared memory (ld 132: conflict-free DMMA fragment loads).  Per block
// K = [k0, k0+8):
//   phase 1 (warp 0): LDL^T of the 8 x 8 diagonal block D = L_KK Δ L_KK^T and W_KK = L_KK^-1
//            (lane i holds row i; 8 pivots, each classified as above);
//   phase 2: every other row tile of the block column: M[T, K] <- M[T, K] W_KK^T
//            (rows > K: P = S_rK L_KK^-T = L_rK Δ, the final S values; rows < K: the final W rows);
//   phase 3: trailing columns c > K: S_rc -= L_rK P_cK^T (r >= c) and W_ct -= L_cK W_Kt (t in
//            the finished rows), as 8 x 8 x 8 DMMA tile products (mma.m8n8k4.f64); warp 0
//            first updates the next diagonal tile and runs phase 1 of block K+1 (lookahead).
// Equal to the scalar elimination in exact arithmetic (block LDL^T, readings R3/R19).  The
// scalar one-pivot-per-barrier form was issue bound (~6 instructions per FMA for the masks).
constexpr int CB_LD = 132;

__device__ __forceinline__ void dmma8(double &d0, double &d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}


__global__ void __launch_bounds__(512, 1) chol_blk_kernel(int n, const double *G, int64_t ldg, const double *Gorig,
                                                          int64_t ldo, double *R, int64_t ldr, double *X, int64_t ldx,
                                                          unsigned *fail_word, unsigned fail_bit, int *dep,
                                                          unsigned dep_bit, unsigned *flag_word, const unsigned *cond,
                                                          unsigned cond_mask, int near_id, double shift_m,
                                                          unsigned *shift_word, unsigned shift_bit,
                                                          const double *maxdev, int nmaxdev, int zero_cond,
                                                          unsigned long long *trace, int busy) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  // the first pass of an orth clears the COND word itself (instead of a memset node): no other
  // kernel of the orth has touched it yet, and the bits below are set after barriers
  if (zero_cond && threadIdx.x == 0) *shift_word = 0u;
  if (near_id == 2) {
    // near_id_spec_kernel already wrote the first-order factor; keep it if max|G - I| <= 2^-27
    // (the per-CTA maxima are reduced here: no accumulator to reset between calls)
    __shared__ int s_ok;
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    for (int b = threadIdx.x; b < nmaxdev; b += blockDim.x)
      if (!(maxdev[b] <= 0x1p-27)) s_ok = 0;
    __syncthreads();
    if (s_ok) return;
    if (threadIdx.x == 0) atomicOr(shift_word, shift_bit << 16);  // declined (as below)
    near_id = 0;
  }
  extern __shared__ double M[];  // npad x CB_LD, column-major: M[r + c * CB_LD]
  __shared__ double wkk[2][64];  // W_KK[i][t] at wkk[.][i * 8 + t] (unit lower), double-buffered
  __shared__ double dpiv[CHOL_SMALL], dinv[CHOL_SMALL], g0s[CHOL_SMALL], sq[CHOL_SMALL];
  __shared__ double red[16];
  __shared__ int s_fail, s_dep, s_tiny;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int npad = (n + 7) & ~7, nt = npad >> 3;
  // M = the Gram's lower part (M(r, c) = G[r + c ldg], r >= c; + shift on the diagonal), the upper
  // part (the W^T entries) zero, identity padding.  The fused path's Gram is formed whole (n <= 128
  // is one 128-row GEMM tile) and symmetric, as are the blocked path's diagonal blocks, so no
  // transpose is needed: 16-byte loads and stores along columns (a flat unrolled loop keeps many
  // loads in flight; transposed stores were 16-way bank conflicts, ~5 us of the kernel).
  // shift > 0: the retry after a breakdown (shifted CholeskyQR, G + shift I).
  auto load = [&](double shift) {
    const int hp = npad >> 1, tot = hp * npad;
    const bool vec = ((ldg & 1) == 0) && ((reinterpret_cast<uintptr_t>(G) & 15) == 0);
    // (row pair, column) advanced incrementally: no integer division in the loop
    const int da = blockDim.x % hp, db = blockDim.x / hp;
    int ai = tid % hp, bi = tid / hp;
    // the original diagonal first (its loads overlap the matrix's)
    for (int i = tid; i < npad; i += blockDim.x) g0s[i] = i < n ? Gorig[i + (int64_t)i * ldo] + shift : 1.0;
#pragma unroll 4
    for (int e = tid; e < tot; e += blockDim.x) {
      const int r = 2 * ai, c = bi;
      ai += da;
      bi += db;
      if (ai >= hp) { ai -= hp; ++bi; }
      double v0 = (r == c) ? 1.0 : 0.0, v1 = (r + 1 == c) ? 1.0 : 0.0;
      if (c < n && r + 1 >= c) {
        const double *src = G + r + (int64_t)c * ldg;
        if (vec && r + 1 < n) {
          const double2 t = *reinterpret_cast<const double2 *>(src);
          if (r >= c) v0 = t.x;
          v1 = t.y;
        } else {
          if (r >= c && r < n) v0 = src[0];
          if (r + 1 < n) v1 = src[1];
        }
        if (r == c) v0 += shift;
        if (r + 1 == c) v1 += shift;
      }
      *reinterpret_cast<double2 *>(M + r + c * CB_LD) = make_double2(v0, v1);
    }
  };
  load(0.0);
  __syncthreads();
  if (near_id) {
    // CholeskyQR2's second pass: if max |G - I| <= 2^-27, R = I + triu(E,1) + diag(E)/2 and
    // X = I - (same) are exact to below u (the neglected terms are O(|E|^2))
    double emax = 0.0;
    for (int b = warp; b < n; b += nwarps)
      for (int a = lane; a <= b; a += 32) emax = fmax(emax, fabs(M[b + a * CB_LD] - (a == b ? 1.0 : 0.0)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    if (lane == 0) red[warp] = emax;
    __syncthreads();
    double mx = 0.0;
    for (int w = 0; w < nwarps; ++w) mx = fmax(mx, red[w]);
    if (mx <= 0x1p-27) {
      for (int b = warp; b < n; b += nwarps)
        for (int a = lane; a < n; a += 32) {  // (a, b) of R and X, coalesced over a
          double u = 0.0;
          if (a < b) u = M[b + a * CB_LD];
          else if (a == b) u = 0.5 * (M[a + a * CB_LD] - 1.0);
          R[a + (int64_t)b * ldr] = (a == b ? 1.0 : 0.0) + u;
          X[a + (int64_t)b * ldx] = (a == b ? 1.0 : 0.0) - u;
        }
      return;
    }
    // declined: the full factorisation follows; marked (shift_bit << 16 = pass_bit << 24, as the
    // blocked path's near_identity_kernel does) for callers that iterate until a pass accepts
    if (tid == 0) atomicOr(shift_word, shift_bit << 16);
  }
  if (tid == 0) { s_fail = 0; s_dep = 0; s_tiny = 0; }
  __syncthreads();
  int *dep_att = dep;
  for (int attempt = 0;; ++attempt) {
    const int fr = lane >> 2, fq = lane & 3;  // DMMA fragment coordinates
    // phase 1 of block kb: LDL^T of the diagonal block, W_KK into wkk[buf] (write; a warp that
    // runs it with write = false only keeps its SM sub-partition busy, see below)
    auto phase1 = [&](int kb, double *wk, bool write) {
      const int k0 = kb * 8;
      const int i = lane & 7;
      double d[8], w[8], g0[8], piv[8], sv[8];  // lane i: row i of the block and of W_KK
  #pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = k0 + i, cc = k0 + j;
        d[j] = r >= cc ? M[r + cc * CB_LD] : M[cc + r * CB_LD];
        w[j] = (i == j) ? 1.0 : 0.0;
        g0[j] = g0s[cc];
      }
      // the pivot chain only: shuffles, the reciprocal and FMAs (bookkeeping after the loop)
      unsigned kinds = 0;
  #pragma unroll
      for (int p = 0; p < 8; ++p) {
        const double draw = __shfl_sync(0xffffffffu, d[p], p);
        double pv = draw;
        if (!isfinite(draw)) { kinds |= 2u << (2 * p); pv = 1.0; }
        else if (dep_att && !(draw > CHOL_DEP * g0[p])) { kinds |= 1u << (2 * p); pv = 1.0; }
        else if (!(draw > CHOL_BREAK * g0[p])) { kinds |= 2u << (2 * p); pv = 1.0; }
        piv[p] = pv;
        const double pinv = fast_rcp(pv);
        sv[p] = d[p];                                   // final S value L_ip d_p (i > p)
        const double l = (i > p) ? d[p] * pinv : 0.0;  // L_ip (row i of the block)
  #pragma unroll
        for (int j = p + 1; j < 8; ++j) d[j] = fma(-l, __shfl_sync(0xffffffffu, d[j], p), d[j]);
  #pragma unroll
        for (int t = 0; t <= p; ++t) w[t] = fma(-l, __shfl_sync(0xffffffffu, w[t], p), w[t]);
      }
      if (!write) return;
      if (lane < 8) {
  #pragma unroll
        for (int p = 0; p < 8; ++p)
          if (i > p) M[(k0 + i) + (k0 + p) * CB_LD] = sv[p];
        const int kg = k0 + i;  // lane i records pivot i
        double pv = piv[0], dr = d[0];
  #pragma unroll
        for (int p = 1; p < 8; ++p) if (i == p) { pv = piv[p]; dr = d[p]; }
        // a numerically dependent column (pivot <= 1e-15 of its diagonal before any shift):
        // reported as RQLP_FLAG_RANK_DEFICIENT whether or not the column is completed here
        if (attempt == 0 && kg < n && !(dr > CHOL_DEP * g0s[kg]) && !isnan(dr)) s_tiny = 1;
        dpiv[kg] = pv;
        dinv[kg] = fast_rcp(pv);
        const unsigned kind = (kinds >> (2 * i)) & 3u;
        if (kg < n) {
          if (dep_att) dep_att[kg] = kind == 1;
          if (kind == 1) s_dep = 1;
          if (kind == 2) s_fail = 1;
        }
      }
      if (lane < 8) {
  #pragma unroll
        for (int t = 0; t < 8; ++t) {
          wk[i * 8 + t] = w[t];
          if (t < i) M[(k0 + t) + (k0 + i) * CB_LD] = w[t];  // W_{k0+i, k0+t} in the upper part
        }
      }
    };
    // debug (RQLP_ENGINE_TRACE): SM clock at the phases of every block of the first attempt
    auto stamp = [&](int kb, int ph) {
      if (trace && attempt == 0 && kb < 32) trace[kb * 4 + ph] = (unsigned long long)clock64();
    };
    if (tid == 0) stamp(31, 0);
    // every warp runs block 0's phase 1 (only warp 0 writes).  Measured on this B200: a lone warp's
    // latency-bound pivot chain ran ~5x slower while the other 15 warps were parked at
    // __syncthreads (block 0: 35.8k cycles, 4.5k per pivot) than while they were busy (~0.4k per
    // pivot in the loop below); redundant copies keep the sub-partitions busy (nothing parks).
    phase1(0, wkk[0], warp == 0);
    if (tid == 0) stamp(31, 1);

    __syncthreads();
    for (int kb = 0; kb < nt; ++kb) {
      const int k0 = kb * 8;
      const double *wk = wkk[kb & 1];
      if (tid == 0) stamp(kb, 0);
      // ---- phase 2: M[T, K] <- M[T, K] W_KK^T for every row tile T != K
      for (int T = warp; T < nt; T += nwarps) {
        if (T == kb) continue;
        const int r = T * 8 + fr;
        const double a0 = M[r + (k0 + 2 * fq) * CB_LD], a1 = M[r + (k0 + 2 * fq + 1) * CB_LD];
        const double b0 = wk[fr * 8 + 2 * fq], b1 = wk[fr * 8 + 2 * fq + 1];  // B[k][j] = W_KK[j][k], j = fr
        double c0 = 0.0, c1 = 0.0;
        dmma8(c0, c1, a0, b0);
        dmma8(c0, c1, a1, b1);
        __syncwarp();
        M[r + (k0 + 2 * fq) * CB_LD] = c0;
        M[r + (k0 + 2 * fq + 1) * CB_LD] = c1;
      }
      __syncthreads();
      if (tid == 0) stamp(kb, 1);
      // ---- phase 3: trailing column tiles Tc > kb.  S part: tiles (Tr >= Tc); W part: Tr <= kb.
      //      Tile 0 is the next diagonal block: warp 0 updates it and then runs phase 1 of block
      //      kb + 1 (lookahead) while warps 1.. do the remaining tiles.
      const int ntrail = nt - kb - 1;
      if (ntrail > 0) {
        const int n_s = ntrail * (ntrail + 1) / 2, n_w = (kb + 1) * ntrail;
        const double dv0 = dinv[k0 + 2 * fq], dv1 = dinv[k0 + 2 * fq + 1];
        auto tile = [&](int t) {
          int Tr, Tc;
          double a0, a1;
          if (t < n_s) {  // S tile: (Tr, Tc) with kb < Tc <= Tr, t = rr (rr + 1) / 2 + cr row-major
            int rr = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
            if ((rr + 1) * (rr + 2) / 2 <= t) ++rr;  // float rounding guards (t < 8256)
            if (rr * (rr + 1) / 2 > t) --rr;
            Tr = kb + 1 + rr;
            Tc = kb + 1 + (t - rr * (rr + 1) / 2);
            const int r = Tr * 8 + fr;
            a0 = M[r + (k0 + 2 * fq) * CB_LD] * dv0;  // L_rK = P_rK Δ^-1
            a1 = M[r + (k0 + 2 * fq + 1) * CB_LD] * dv1;
          } else {        // W tile: rows Tr <= kb, A[t][k] = W_{k0+k, t}
            const int u = t - n_s;
            Tr = u % (kb + 1);
            Tc = kb + 1 + u / (kb + 1);
            const int tr = Tr * 8 + fr;
            if (Tr < kb) {
              a0 = M[tr + (k0 + 2 * fq) * CB_LD];
              a1 = M[tr + (k0 + 2 * fq + 1) * CB_LD];
            } else {
              a0 = wk[(2 * fq) * 8 + fr];
              a1 = wk[(2 * fq + 1) * 8 + fr];
            }
          }
          // B[k][c] = P_cK[c][k] (S tiles) or L_cK[c][k] (W tiles), c = Tc*8 + fr
          const int cc = Tc * 8 + fr;
          double b0 = M[cc + (k0 + 2 * fq) * CB_LD], b1 = M[cc + (k0 + 2 * fq + 1) * CB_LD];
          if (t >= n_s) { b0 *= dv0; b1 *= dv1; }
          double c0 = 0.0, c1 = 0.0;
          dmma8(c0, c1, a0, b0);
          dmma8(c0, c1, a1, b1);
          const int orow = Tr * 8 + fr, ocol = Tc * 8 + 2 * fq;
          if (t >= n_s || Tr != Tc || orow >= ocol) M[orow + ocol * CB_LD] -= c0;
          if (t >= n_s || Tr != Tc || orow >= ocol + 1) M[orow + (ocol + 1) * CB_LD] -= c1;
        };
        if (warp == 0) {
          tile(0);
          __syncwarp();
          phase1(kb + 1, wkk[(kb + 1) & 1], true);
          if (lane == 0) stamp(kb, 3);
        } else {
          for (int t = warp; t < n_s + n_w; t += nwarps - 1) tile(t);
          // until warp 0's lookahead phase 1 is done: a redundant, non-writing copy of it (from
          // whatever the diagonal block holds) instead of parking at the barrier (see above)
          if (busy) phase1(kb + 1, nullptr, false);
        }
      }
      __syncthreads();
      if (tid == 0) stamp(kb, 2);
    }
    // breakdown with a shift length given: redo on G + s I, s = 11 (m n + n (n+1)) u tr(G)
    __syncthreads();
    if (attempt > 0 || !s_fail || !(shift_m > 0.0)) break;
    double tr = 0.0;
    for (int i = 0; i < n; ++i) tr += g0s[i];  // = diag(G): the fused path has Gorig == G
    double shift = 11.0 * (shift_m * n + (double)n * (n + 1)) * 0x1p-53 * tr;
    if (!(shift > 0.0)) shift = 1.0;  // zero matrix: any positive shift
    __syncthreads();
    if (tid == 0) {
      s_fail = 0;
      atomicOr(flag_word, (unsigned)RQLP_FLAG_SHIFTED_CHOLQR);
      atomicOr(shift_word, shift_bit);
    }
    dep_att = nullptr;
    load(shift);
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) {
    sq[i] = sqrt(dpiv[i]);
    dinv[i] = 1.0 / sq[i];   // (the pivot reciprocals are no longer needed)
  }
  __syncthreads();
  // outputs: R(c, r) = S_rc / sqrt(d_c) (c < r), R(r, r) = sqrt(d_r), R lower = 0;
  //          X(r, c) = W_cr / sqrt(d_c) (r < c), X(r, r) = 1 / sqrt(d_r), X lower = 0
  // (one reciprocal per column, rolled loops: this code runs once per launch, cold in the i-cache)
#pragma unroll 1
  for (int r = warp; r < n; r += nwarps)
#pragma unroll 1
    for (int c = lane; c < n; c += 32) {  // R(c, r): coalesced over c
      double v = 0.0;
      if (c < r) v = M[r + c * CB_LD] * dinv[c];
      else if (c == r) v = sq[r];
      R[c + (int64_t)r * ldr] = v;
    }
#pragma unroll 1
  for (int c = warp; c < n; c += nwarps) {
    const double isq = dinv[c];
#pragma unroll 1
    for (int r = lane; r < n; r += 32) {  // X(r, c): coalesced over r
      double v = 0.0;
      if (r < c) v = M[r + c * CB_LD] * isq;
      else if (r == c) v = isq;
      X[r + (int64_t)c * ldx] = v;
    }
  }
  if (tid == 0 && s_fail) atomicOr(fail_word, fail_bit);
  if (tid == 0 && s_tiny) atomicOr(flag_word, (unsigned)RQLP_FLAG_RANK_DEFICIENT);
  if (tid == 0 && s_dep && dep) {
    atomicOr(fail_word, dep_bit);
    atomicOr(flag_word, (unsigned)RQLP_FLAG_RANK_DEFICIENT);
  }
}

// dep[k] != 0: column k of Q (m x n) is replaced by a N(0,1)-like completion vector (counter =
// row + m k, internal.cuh); the next CholeskyQR pass orthonormalises it against the others (basis completion
// for rank-deficient input, reading R4/R21).
__global__ void replace_dep_kernel(int64_t m, int n, double *Q, int64_t ldq, const int *dep, uint64_t seed,
                                   const unsigned *cond, unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  for (int k = blockIdx.y; k < n; k += gridDim.y) {
    if (!dep[k]) continue;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      Q[i + (int64_t)k * ldq] = completion_value((uint64_t)(i + m * k), seed);
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
    if (i > j) continue;  // the Gram's upper triangle (the lower one is not formed)
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

// RQLP_CHOL_BUSY=1 (measurement switch): the trailing-update warps run a redundant phase 1 while
// warp 0 runs the lookahead one, instead of parking at the barrier.  Measured: slower (C2's c = 110
// blocked loop 29.0 -> 43.7 us -- the copies compete with warp 0 for issue), so off; only block 0's
// phase 1, where all 15 other warps would otherwise park, runs redundantly.
static int chol_busy() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RQLP_CHOL_BUSY");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v;
}

void launch_chol_inv(Ctx &c, int n, const double *G, int64_t ldg, const double *Gorig, int64_t ldo, double *R,
                     int64_t ldr, double *X, int64_t ldx, unsigned *fail_word, unsigned fail_bit,
                     const unsigned *cond, unsigned mask, int *dep = nullptr, unsigned dep_bit = 0, int near_id = 0,
                     double shift_m = 0.0, unsigned shift_bit = 0, const double *maxdev = nullptr,
                     int nmaxdev = 0, int zero_cond = 0) {
  smem_attr((const void *)chol_blk_kernel, CHOL_SMALL * CB_LD * 8);
  chol_blk_kernel<<<1, 512, (size_t)((n + 7) & ~7) * CB_LD * 8, c.stream>>>(
      n, G, ldg, Gorig, ldo, R, ldr, X, ldx, fail_word, fail_bit, dep, dep_bit, c.dflags + FLAG_WORD, cond, mask,
      near_id, shift_m, c.dflags + COND_WORD, shift_bit, maxdev, nmaxdev, zero_cond,
      c.trace ? c.trace + 8 * 4096 : nullptr, chol_busy());
  RQLP_LAUNCHED(c);
}

// CholeskyQR2's second pass, speculatively and grid-wide: every entry of the upper triangle gets
// the first-order factor R = I + U, X = I - U (U = triu(E, 1) + diag(E)/2, E = G - I; the
// strictly lower parts zero), and max |E| over the upper triangle goes to *maxbits (ordered
// bits; NaN ranks highest).  chol_blk_kernel (near_id = 2) keeps this when max |E| <= 2^-27 and
// otherwise factorises and overwrites R and X.  (In one CTA the same test sat behind a ~4 us
// latency-bound load of G.)
__global__ void near_id_spec_kernel(int n, const double *__restrict__ G, int64_t ldg, double *__restrict__ R,
                                    int64_t ldr, double *__restrict__ X, int64_t ldx, double *maxdev,
                                    const unsigned *cond, unsigned cond_mask) {
  __shared__ double wmax[8];
  if (cond && ((*cond) & cond_mask) == 0) return;
  const int64_t total = (int64_t)n * n;
  double e = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % n), j = (int)(q / n);
    double r = 0.0, x = 0.0;
    if (i <= j) {
      const double dlt = i == j ? 1.0 : 0.0;
      const double E = G[i + (int64_t)j * ldg] - dlt;
      const double aE = fabs(E);
      if (!(aE <= e)) e = aE;  // NaN propagates
      const double u = i < j ? E : 0.5 * E;
      r = dlt + u;
      x = dlt - u;
    }
    R[i + (int64_t)j * ldr] = r;
    X[i + (int64_t)j * ldx] = x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, e, o);
    if (!(t <= e)) e = t;
  }
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bm = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      if (!(wmax[w] <= bm)) bm = wmax[w];
    maxdev[blockIdx.x] = bm;  // this CTA's max |E|
  }
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
  s.maxdev = a.take<double>(256);
}

// One CholeskyQR pass: Qout = Yin R^-1 with G = Yin^T Yin.  pass_bit marks this pass's
// breakdown in the COND word.  Kernels run only if (*cond & mask) when cond given.
static void cholqr_pass(Ctx &c, OrthScratch &s, int64_t m, int64_t n, const double *Yin, int64_t ldyi, double *Qout,
                        int64_t ldqo, double *Rout, unsigned pass_bit, const unsigned *cond, unsigned mask,
                        bool sharded, bool second = false, bool use_dep = true) {
  const unsigned *gcond = cond;   // the pass's own condition (the GEMMs)
  const unsigned gmask = mask;
  int64_t lc = round_up(n, 8);
  unsigned *condw = c.dflags + COND_WORD;
  const unsigned dep_bit = pass_bit << 16;
  // Gram (upper triangle only: every consumer below reads G(a, b) with a <= b)
  gemm_tn(c, m, n, n, Yin, ldyi, Yin, ldyi, s.G, lc, false, s.partials, s.partial_elems, cond, mask, 1);
  if (sharded) allreduce_sum(c, s.G, lc * n);   // Gram summed over the row shards
  if (n <= CHOL_SMALL) {
    // one kernel: near-identity factor (second pass), else Cholesky + inverse, and on breakdown
    // the shifted retry in place (marks pass_bit << 8 for the third pass)
    // second pass: the near-identity test and first-order factor grid-wide ahead of the Cholesky
    // kernel when n >= 64 (for smaller n the in-kernel test is cheaper than another launch)
    const bool spec = second && n >= 64;
    int nblk = 0;
    if (spec) {
      nblk = (int)std::min<int64_t>(ceil_div(n * n, 256), std::min<int64_t>(c.num_sms, 256));
      near_id_spec_kernel<<<nblk, 256, 0, c.stream>>>((int)n, s.G, lc, Rout, lc, s.Rinv, lc, s.maxdev, cond, mask);
      RQLP_LAUNCHED(c);
    }
    launch_chol_inv(c, (int)n, s.G, lc, s.G, lc, Rout, lc, s.Rinv, lc, condw, 0u, cond, mask,
                    use_dep ? s.dep : nullptr, dep_bit, spec ? 2 : (second ? 1 : 0), (double)m, pass_bit << 8,
                    s.maxdev, nblk, (pass_bit == 1u && !cond && !sharded) ? 1 : 0);
  } else {
    if (second) {
      // near-identity Gram: elementwise factor; the full Cholesky below runs only if it declines
      near_identity_kernel<<<1, 1024, 0, c.stream>>>((int)n, s.G, lc, Rout, lc, s.Rinv, lc, condw, pass_bit << 24,
                                                     cond, mask);
      RQLP_LAUNCHED(c);
      cond = condw;
      mask = pass_bit << 24;
    }
    launch_copy(c, n, n, s.G, lc, s.G2, lc, false, cond, mask);  // blocked path destroys G
    chol_inv(c, n, s.G, lc, s.G2, lc, Rout, lc, s.Rinv, lc, s.tmp, condw, pass_bit, cond, mask, s.partials,
             s.partial_elems, use_dep ? s.dep : nullptr, dep_bit);
    // breakdown (ill-conditioned) -> shifted Gram, second attempt (only if pass_bit was set)
    add_shift_kernel<<<1, 1024, 0, c.stream>>>((int)n, s.G2, lc, (double)m, c.dflags + FLAG_WORD, condw, pass_bit,
                                               pass_bit << 8);
    RQLP_LAUNCHED(c);
    launch_copy(c, n, n, s.G2, lc, s.G, lc, false, condw, pass_bit);
    chol_inv(c, n, s.G, lc, s.G2, lc, Rout, lc, s.Rinv, lc, s.tmp, condw, 0u, condw, pass_bit, s.partials,
             s.partial_elems, nullptr, 0u);
  }
  gemm_nn(c, m, n, n, Yin, ldyi, s.Rinv, lc, Qout, ldqo, s.partials, s.partial_elems, gcond, gmask, 2);  // R^-1 upper
  if (!use_dep) return;
  // rank-deficient columns -> random completion, orthonormalised by the following pass
  replace_dep_kernel<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 64)),
                           (unsigned)std::min<int64_t>(n, 64)),
                       256, 0, c.stream>>>(m, (int)n, Qout, ldqo, s.dep, 0x5eedULL + pass_bit, condw, dep_bit);
  RQLP_LAUNCHED(c);
}

__global__ void or_flag_kernel(unsigned *word, unsigned bits) { atomicOr(word, bits); }
__global__ void sticky_kernel(const unsigned *cond, unsigned mask, unsigned *sticky) {
  if (*cond & mask) *sticky = 1u;
}

// The rare branch for row-sharded orth (orth_rescue.cu's algorithm with allreduced Grams, driven
// from the host): if the COND word holds one of `mask`'s bits, CholeskyQR passes (shifted on
// breakdown; zero or, from the 4th pass, numerically dependent columns completed) on V until a
// pass's Gram is near the identity, then R = V^T Y (allreduced; R's strictly lower part is then
// rounding noise, not zero).  Reads the COND word back (one stream synchronisation per orth).
static void sharded_rescue(Ctx &c, OrthScratch &s, int64_t m, int64_t n, double *V, int64_t ldv, const double *Y,
                           int64_t ldy, double *R, int64_t ldr, unsigned mask) {
  unsigned *condw = c.dflags + COND_WORD;
  if (c.optimistic) {
    // no readback: remember that this orth broke down; with_graph() reads the sticky word once at
    // the end of the factorisation and reruns it on the careful (host-driven) path
    sticky_kernel<<<1, 1, 0, c.stream>>>(condw, mask, c.dflags + STICKY_WORD);
    RQLP_LAUNCHED(c);
    return;
  }
  unsigned host = 0;
  RQLP_CUDA(cudaMemcpyAsync(&host, condw, sizeof(unsigned), cudaMemcpyDeviceToHost, c.stream));
  RQLP_CUDA(cudaStreamSynchronize(c.stream));
  if (!(host & mask)) return;
  const int64_t lc = round_up(n, 8);
  double *cur = V, *nxt = s.Ybuf;
  int64_t ldc = ldv, ldn = s.ldy;
  for (int pass = 0; pass < 10; ++pass) {
    RQLP_CUDA(cudaMemsetAsync(condw, 0, sizeof(unsigned), c.stream));
    cholqr_pass(c, s, m, n, cur, ldc, nxt, ldn, s.R, 4u, nullptr, 0, true, true, pass >= 3);
    std::swap(cur, nxt);
    std::swap(ldc, ldn);
    RQLP_CUDA(cudaMemcpyAsync(&host, condw, sizeof(unsigned), cudaMemcpyDeviceToHost, c.stream));
    RQLP_CUDA(cudaStreamSynchronize(c.stream));
    if (!(host & (4u << 24))) break;  // this pass's Gram was near the identity: cur is orthonormal
  }
  if (cur != V) launch_copy(c, m, n, cur, ldc, V, ldv, false);
  if (R) {
    gemm_tn(c, m, n, n, V, ldv, Y, ldy, s.tmp, lc, false, s.partials, s.partial_elems);
    allreduce_sum(c, s.tmp, lc * n);
    launch_copy(c, n, n, s.tmp, lc, R, ldr, false);
  }
  or_flag_kernel<<<1, 1, 0, c.stream>>>(c.dflags + FLAG_WORD, (unsigned)RQLP_FLAG_SHIFTED_CHOLQR);
  RQLP_LAUNCHED(c);
}

void orth(Ctx &c, OrthScratch &s, int64_t m, int64_t n, const double *Y, int64_t ldy, double *V, int64_t ldv,
          double *R, int64_t ldr, bool sharded, bool span_only) {
  int64_t lc = round_up(n, 8);
  unsigned *condw = c.dflags + COND_WORD;
  // the fused first pass (n <= 128, one device) clears the COND word in its Cholesky kernel
  if (sharded || n > CHOL_SMALL) RQLP_CUDA(cudaMemsetAsync(condw, 0, sizeof(unsigned), c.stream));
  if (span_only && !R) {
    // intermediate subspace-iteration basis: only range(V) = range(Y) matters (V = Y R^-1 for any
    // invertible R keeps the span to the same O(u cond(Y)) rounding), so one CholeskyQR pass.
    if (!sharded) {
      // a breakdown (shifted pass) leaves V far from orthonormal, with the small directions of Y
      // compressed by ~s^-1/2: the next product A^T V would push them below the rounding level,
      // so the rescue passes restore an orthonormal V first (Householder-quality basis)
      cholqr_pass(c, s, m, n, Y, ldy, V, ldv, s.Racc, 1u, nullptr, 0, false, false, false);
      launch_orth_rescue(c, s, m, n, V, ldv, Y, ldy, nullptr, 0, condw, 1u << 8);
      return;
    }
    cholqr_pass(c, s, m, n, Y, ldy, V, ldv, s.Racc, 1u, nullptr, 0, true, false, false);
    sharded_rescue(c, s, m, n, V, ldv, Y, ldy, nullptr, 0, 1u << 8);
    return;
  }
  // pass 1: Y -> Ybuf (R1 in Racc), pass 2: Ybuf -> V (R2 in R)
  if (!sharded) {
    // CholeskyQR2 without column completion (a tiny pivot is a breakdown: the shifted retry keeps
    // every direction of Y); after any breakdown (bits 1<<8 | 2<<8) the rescue kernel continues
    // with shifted passes until V is orthonormal and recomputes R = V^T Y
    cholqr_pass(c, s, m, n, Y, ldy, s.Ybuf, s.ldy, s.Racc, 1u, nullptr, 0, false, false, false);
    cholqr_pass(c, s, m, n, s.Ybuf, s.ldy, V, ldv, s.R, 2u, nullptr, 0, false, true, false);
    if (R) gemm_nn(c, n, n, n, s.R, lc, s.Racc, lc, R, ldr, s.partials, s.partial_elems);  // R = R2 R1
    launch_orth_rescue(c, s, m, n, V, ldv, Y, ldy, R, ldr, condw, (1u << 8) | (2u << 8));
    return;
  }
  // row-sharded (eager only: graphs are off with a communicator): CholeskyQR2 as above, the rare
  // branch driven from the host -- every rank reads the same COND word (the Grams are allreduced,
  // so every rank takes the same decisions) and runs the same extra passes
  cholqr_pass(c, s, m, n, Y, ldy, s.Ybuf, s.ldy, s.Racc, 1u, nullptr, 0, true, false, false);
  cholqr_pass(c, s, m, n, s.Ybuf, s.ldy, V, ldv, s.R, 2u, nullptr, 0, true, true, false);
  if (R) gemm_nn(c, n, n, n, s.R, lc, s.Racc, lc, R, ldr, s.partials, s.partial_elems);  // R = R2 R1
  sharded_rescue(c, s, m, n, V, ldv, Y, ldy, R, ldr, (1u << 8) | (2u << 8));
}

}  // namespace rqlpk
