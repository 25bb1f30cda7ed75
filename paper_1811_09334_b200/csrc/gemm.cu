// gemm.cu -- FP64 GEMMs on the sm_100a DMMA pipe (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
//
// The A-passes of RQLP (Alg.1 l.2 Y = AΩ, l.4 B = V^T A; the power step
// A^T V / AW, reading R12) are tall-skinny FP64 contractions.  B200 has no FP64 tcgen05 kind
// (ptxas rejects kind::f64); the measured FP64 peaks on this pool's B200 are 37.1 TFLOP/s for
// DMMA and 34.1 TFLOP/s for DFMA (tools/microbench/fp64_peak.cu, profiles/), so every GEMM
// here issues DMMA.  This file holds the generic kernel (any transpose / stride / alignment,
// used for the small l x l products and as the fallback), the deterministic split-K reduce,
// and the dispatch of the two tall-skinny passes to the TMA-pipelined kernels (gemm_tma.cu).
#include "internal.cuh"

namespace rqlpk {

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

namespace {

// ------------------------------------------------------------------------------------------
// Generic DMMA GEMM: C(MxN) = alpha op(A) op(B) + beta C.  64x64x16 CTA tile, 4 warps (2x2),
// 32x32 warp tile = 4x4 m8n8 fragments.  Register-staged double buffering.  Split-K over
// gridDim.z writes raw partial sums to `part` (M x N, ld M, slice z) for reduce_kernel.
// smem layouts are padded so every fragment load is bank-conflict free:
//   As[k][m] LD 68 (68 = 4 mod 16 doubles), Bs[n][k] LD 20 (20 = 4 mod 16).
// ------------------------------------------------------------------------------------------
constexpr int GB_M = 64, GB_N = 64, GB_K = 16, GLDA = GB_M + 4, GLDB = GB_K + 4;

template <bool TA, bool TB>
__global__ void __launch_bounds__(128) gemm_generic_kernel(int64_t M, int64_t N, int64_t K, int64_t kchunk,
                                                           double alpha, const double *__restrict__ A,
                                                           int64_t lda, const double *__restrict__ B,
                                                           int64_t ldb, double beta, double *__restrict__ C,
                                                           int64_t ldc, double *__restrict__ part,
                                                           const unsigned *cond, unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  __shared__ double As[2][GB_K][GLDA];
  __shared__ double Bs[2][GB_N][GLDB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int r = lane >> 2, c = lane & 3;
  const int64_t m0 = (int64_t)blockIdx.x * GB_M, n0 = (int64_t)blockIdx.y * GB_N;
  const int64_t kb = (int64_t)blockIdx.z * kchunk, ke = min(K, kb + kchunk);

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[8], rb[8];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      int e = tid + 128 * t;
      int64_t i, p;
      if (!TA) { i = e % GB_M; p = e / GB_M; } else { p = e % GB_K; i = e / GB_K; }
      int64_t gi = m0 + i, gp = k0 + p;
      double v = 0.0;
      if (gi < M && gp < ke) v = TA ? A[gp + gi * lda] : A[gi + gp * lda];
      ra[t] = v;
      int64_t j;
      if (!TB) { p = e % GB_K; j = e / GB_K; } else { j = e % GB_N; p = e / GB_N; }
      int64_t gj = n0 + j;
      gp = k0 + p;
      double w = 0.0;
      if (gj < N && gp < ke) w = TB ? B[gj + gp * ldb] : B[gp + gj * ldb];
      rb[t] = w;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      int e = tid + 128 * t;
      int i, p, j;
      if (!TA) { i = e % GB_M; p = e / GB_M; } else { p = e % GB_K; i = e / GB_K; }
      As[buf][p][i] = ra[t];
      if (!TB) { p = e % GB_K; j = e / GB_K; } else { j = e % GB_N; p = e / GB_N; }
      Bs[buf][j][p] = rb[t];
    }
  };

  int buf = 0;
  if (kb < ke) {
    load(kb);
    store(0);
  }
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += GB_K) {
    bool more = k0 + GB_K < ke;
    if (more) load(k0 + GB_K);
#pragma unroll
    for (int k4 = 0; k4 < GB_K / 4; ++k4) {
      double a[4], b[4];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) a[mb] = As[buf][k4 * 4 + c][wm * 32 + mb * 8 + r];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) b[nb] = Bs[buf][wn * 32 + nb * 8 + r][k4 * 4 + c];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) dmma884(acc[mb][nb][0], acc[mb][nb][1], a[mb], b[nb]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }

  // epilogue: fragment (mb, nb) holds C[r][2c], C[r][2c+1]
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int64_t gi = m0 + wm * 32 + mb * 8 + r, gj = n0 + wn * 32 + nb * 8 + 2 * c + h;
        if (gi < M && gj < N) {
          if (part) {
            part[(size_t)blockIdx.z * M * N + gi + gj * M] = acc[mb][nb][h];
          } else {
            double v = alpha * acc[mb][nb][h];
            if (beta != 0.0) v += beta * C[gi + gj * ldc];
            C[gi + gj * ldc] = v;
          }
        }
      }
}

// C = alpha * sum_{z < S} part_z + beta C  (fixed order z = 0..S-1: deterministic), optionally
// written transposed (C(j, i) for part element (i, j)).
__global__ void reduce_kernel(int64_t M, int64_t N, int S, const double *__restrict__ part, double alpha, double beta,
                              double *__restrict__ C, int64_t ldc, int trans, const unsigned *cond,
                              unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  int64_t total = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < S; ++z) s += part[(size_t)z * total + e];
    int64_t i = e % M, j = e / M;
    double *dst = trans ? &C[j + i * ldc] : &C[i + j * ldc];
    double v = alpha * s;
    if (beta != 0.0) v += beta * *dst;
    *dst = v;
  }
}

}  // namespace

void launch_reduce(Ctx &c, int64_t M, int64_t N, int S, const double *part, double alpha, double beta, double *C,
                   int64_t ldc, bool trans, const unsigned *cond, unsigned cond_mask) {
  int64_t total = M * N;
  int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)c.num_sms * 16);
  reduce_kernel<<<std::max(grid, 1), 256, 0, c.stream>>>(M, N, S, part, alpha, beta, C, ldc, trans ? 1 : 0, cond,
                                                         cond_mask);
  RQLP_LAUNCHED(c);
}

// Split-K factor for the generic kernel: enough CTAs to fill the GPU twice over.
static int generic_splits(int64_t M, int64_t N, int64_t K, int num_sms) {
  int64_t tiles = ceil_div(M, GB_M) * ceil_div(N, GB_N);
  int64_t ktiles = ceil_div(K, GB_K);
  int64_t s = 1;
  while (tiles * s < 2 * num_sms && s * 2 <= 32 && ktiles / (s * 2) >= 8) s *= 2;
  return (int)s;
}

size_t gemm_generic_partials(int64_t M, int64_t N, int64_t K, int num_sms) {
  int s = generic_splits(M, N, K, num_sms);
  return s > 1 ? (size_t)s * M * N : 0;
}

void gemm_generic_ex(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                     int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc, double *partials,
                     size_t partial_elems, bool trans_out, const unsigned *cond, unsigned cond_mask) {
  if (M <= 0 || N <= 0) return;
  int S = generic_splits(M, N, K, c.num_sms);
  if ((size_t)S * M * N > partial_elems || partials == nullptr) S = 1;
  if (trans_out && S == 1) {
    // transposed output without split: use a one-slice partial if we have room, else compute
    // C^T = op(B)^T op(A)^T directly.
    gemm_generic_ex(c, !tb, !ta, N, M, K, alpha, B, ldb, A, lda, beta, C, ldc, nullptr, 0, false, cond, cond_mask);
    return;
  }
  int64_t kchunk = S > 1 ? round_up(ceil_div(K, S), GB_K) : std::max<int64_t>(K, 1);
  S = (int)std::max<int64_t>(1, ceil_div(K, kchunk));
  dim3 grid((unsigned)ceil_div(M, GB_M), (unsigned)ceil_div(N, GB_N), (unsigned)S);
  double *part = S > 1 ? partials : nullptr;
  if (K <= 0) {  // C = beta C
    launch_reduce(c, M, N, 0, partials, alpha, beta, C, ldc, false, cond, cond_mask);
    return;
  }
#define RQLP_GEN(TA_, TB_)                                                                                    \
  gemm_generic_kernel<TA_, TB_><<<grid, 128, 0, c.stream>>>(M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, \
                                                          part, cond, cond_mask)
  if (!ta && !tb) RQLP_GEN(false, false);
  else if (ta && !tb) RQLP_GEN(true, false);
  else if (!ta && tb) RQLP_GEN(false, true);
  else RQLP_GEN(true, true);
#undef RQLP_GEN
  RQLP_LAUNCHED(c);
  if (S > 1) launch_reduce(c, M, N, S, partials, alpha, beta, C, ldc, trans_out, cond, cond_mask);
}

void gemm_generic(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                  int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                  const unsigned *cond, unsigned cond_mask) {
  gemm_generic_ex(c, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, nullptr, 0, false, cond, cond_mask);
}

// ---- tall-skinny passes ------------------------------------------------------------------
bool gemm_nn_tma(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X,
                 int64_t ldx, double *Y, int64_t ldy, double *partials, size_t partial_elems, const unsigned *cond,
                 unsigned cond_mask, int tri, const FroSpec *fro = nullptr, double alpha = 1.0, double beta = 0.0);
bool gemm_tn_tma(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *V,
                 int64_t ldv, double *Z, int64_t ldz, bool trans_out, double *partials, size_t partial_elems,
                 const unsigned *cond, unsigned cond_mask, int tri, double alpha = 1.0, double beta = 0.0);
size_t gemm_tma_partials_needed(int64_t m, int64_t cc, int64_t k, int num_sms);

size_t gemm_partials_needed(int64_t m, int64_t cc, int64_t k, int num_sms) {
  size_t a = gemm_generic_partials(m, cc, k, num_sms);   // NN shape
  size_t b = gemm_generic_partials(k, cc, m, num_sms);   // TN shape
  size_t t = gemm_tma_partials_needed(m, cc, k, num_sms);
  return std::max(a, std::max(b, t));
}

void gemm_nn(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X, int64_t ldx,
             double *Y, int64_t ldy, double *partials, size_t partial_elems, const unsigned *cond,
             unsigned cond_mask, int tri) {
  if (gemm_nn_tma(c, m, cc, k, A, lda, X, ldx, Y, ldy, partials, partial_elems, cond, cond_mask, tri)) return;
  gemm_generic_ex(c, false, false, m, cc, k, 1.0, A, lda, X, ldx, 0.0, Y, ldy, partials, partial_elems, false, cond,
                  cond_mask);
}

// Y = alpha A X + beta Y / Z = alpha A^T V + beta Z on the TMA kernels (the deflation and
// re-orthogonalisation products of BRQLP), the generic kernel when an operand is not TMA-addressable.
void gemm_nn_ab(Ctx &c, int64_t m, int64_t cc, int64_t k, double alpha, const double *A, int64_t lda, const double *X,
                int64_t ldx, double beta, double *Y, int64_t ldy, double *partials, size_t partial_elems) {
  if (m <= 0 || cc <= 0) return;
  if (k > 0 && gemm_nn_tma(c, m, cc, k, A, lda, X, ldx, Y, ldy, partials, partial_elems, nullptr, 0, 0, nullptr, alpha,
                           beta))
    return;
  gemm_generic_ex(c, false, false, m, cc, k, alpha, A, lda, X, ldx, beta, Y, ldy, partials, partial_elems, false,
                  nullptr, 0);
}

void gemm_tn_ab(Ctx &c, int64_t m, int64_t cc, int64_t k, double alpha, const double *A, int64_t lda, const double *V,
                int64_t ldv, double beta, double *Z, int64_t ldz, double *partials, size_t partial_elems) {
  if (k <= 0 || cc <= 0) return;
  if (m > 0 && gemm_tn_tma(c, m, cc, k, A, lda, V, ldv, Z, ldz, false, partials, partial_elems, nullptr, 0, 0, alpha,
                           beta))
    return;
  gemm_generic_ex(c, true, false, k, cc, m, alpha, A, lda, V, ldv, beta, Z, ldz, partials, partial_elems, false,
                  nullptr, 0);
}

void gemm_nn_fro(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X,
                 int64_t ldx, double *Y, int64_t ldy, double *partials, size_t partial_elems, const FroSpec &fro) {
  if (gemm_nn_tma(c, m, cc, k, A, lda, X, ldx, Y, ldy, partials, partial_elems, nullptr, 0, 0, &fro)) return;
  gemm_nn(c, m, cc, k, A, lda, X, ldx, Y, ldy, partials, partial_elems);
  fro2_accumulate(c, m, k, A, lda, fro.slots, fro.out, !fro.accumulate);
}

void gemm_tn(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *V, int64_t ldv,
             double *Z, int64_t ldz, bool trans_out, double *partials, size_t partial_elems, const unsigned *cond,
             unsigned cond_mask, int tri) {
  if (gemm_tn_tma(c, m, cc, k, A, lda, V, ldv, Z, ldz, trans_out, partials, partial_elems, cond, cond_mask, tri))
    return;
  // Z (k x cc) = A^T V : op(A) = A^T (k x m), op(B) = V (m x cc)
  gemm_generic_ex(c, true, false, k, cc, m, 1.0, A, lda, V, ldv, 0.0, Z, ldz, partials, partial_elems, trans_out,
                  cond, cond_mask);
}

}  // namespace rqlpk
