// tail.cu -- the small dense tail that turns B = V^T A (l x n) into B = Q_B T P_B^T.
//
// RQLP (d == 0), Alg.1 l.5-7:
//   [Q0, R0, Π0] = cpqr(B);  [Q1, L^T, Π1] = cpqr(R0^T);  Q_B = Q0 Π1,  P_B = Π0 Q1.
// ERQLP (d >= 1), Alg.2 l.5-9 with the corrected assembly (reading R9):
//   [Q^(i), R^(i)] = qr([R^(i-1)]^T), Q_B = Q^(0) Q^(2) .., P_B = Π0 Q^(1) Q^(3) ..,
//   T = [R^(d)]^T (lower) for odd d, R^(d) (upper) for even d.
// B200 formulation (same result in exact arithmetic, reading R6): the
// tall n x l R0^T is first reduced by CholeskyQR2 (BLAS-3, orth.cu) to R0^T = Q^ R^, then the
// l x l R^ goes through the Householder engine (pivoted for RQLP: cpqr(R0^T) and cpqr(R^) pick
// the same pivots because column norms and their downdates are orthogonally invariant).
// The order of the n - l non-pivot columns of R0 is ascending original index; P = Π0 Q1 does
// not depend on it.
#include "internal.cuh"

namespace rqlpk {

void gemm_generic_ex(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                     int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc, double *partials,
                     size_t partial_elems, bool trans_out, const unsigned *cond, unsigned cond_mask);

namespace {

// D(:, t) = S(:, perm[t]); also copies perm[0..cols) to piv_out when given (one launch less)
__global__ void gather_cols_kernel(int64_t rows, int64_t cols, const double *S, int64_t lds, const int64_t *perm,
                                   double *D, int64_t ldd, int64_t *piv_out = nullptr) {
  int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e % rows, t = e / rows;
    D[i + t * ldd] = S[i + perm[t] * lds];
    if (piv_out && i == 0) piv_out[t] = perm[t];
  }
}

// D(perm[i], :) = S(i, :); also copies perm[0..npiv) to piv_out when given (one launch less)
__global__ void scatter_rows_kernel(int64_t rows, int64_t cols, const double *S, int64_t lds, const int64_t *perm,
                                    double *D, int64_t ldd, int64_t *piv_out = nullptr, int64_t npiv = 0) {
  int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e % rows, j = e / rows;
    D[perm[i] + j * ldd] = S[i + j * lds];
    if (piv_out && j == 0 && i < npiv) piv_out[i] = perm[i];
  }
}

__global__ void iota_kernel(int64_t count, int64_t *dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = i;
}

int grid_for(Ctx &c, int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), (int64_t)c.num_sms * 16));
}

}  // namespace

void tail_carve(Arena &a, TailScratch &s, int64_t l, int64_t n, int num_sms) {
  s.ldn = round_up(n, 8);
  s.ldl = round_up(l, 8);
  s.Bw = a.take<double>(s.ldl * n);
  s.Rt = a.take<double>(s.ldn * l);
  s.Qhat = a.take<double>(s.ldn * l);
  s.tmp_nl = a.take<double>(s.ldn * l);
  s.Rhat = a.take<double>(s.ldl * l);
  s.Q0 = a.take<double>(s.ldl * l);
  s.Qt = a.take<double>(s.ldl * l);
  s.Lt = a.take<double>(s.ldl * l);
  s.Mt = a.take<double>(s.ldl * l);
  s.QE = a.take<double>(s.ldl * l);
  s.tmp_ll = a.take<double>(s.ldl * l);
  s.perm0 = a.take<int64_t>(n);
  s.perm1 = a.take<int64_t>(l);
  hh_carve(a, s.hh, l, n, num_sms);
  orth_carve(a, s.orth, n, l, num_sms);
}

// Second half of a pivoted QLP, given R0^T = Q^ R^ (s.Qhat n x l, s.Rhat l x l) and the left
// factor Q0 (rows x l) of the first CPQR: [Q~, L^T, Π1] = cpqr(R^) (PAPER.md:100 on the
// orthogonally equivalent l x l factor), L -> T, Q0 Π1 -> QB (rows x l), piv1; returns
// Q1 = Q^ Q~ (n x l, in s.tmp_nl; rows still in the first CPQR's column order).
static double *pivoted_lq(Ctx &c, TailScratch &s, int64_t rows, int64_t l, int64_t n, const double *Q0, int64_t ldq0,
                          double *T, int64_t ldt, double *QB, int64_t ldqb, int64_t *piv1) {
  const int64_t ldn = s.ldn, ldl = s.ldl;
  launch_copy(c, l, l, s.Rhat, ldl, s.Mt, ldl, false);
  HHScratch h1 = s.hh;
  h1.perm = s.perm1;  // the engine's permutation lands in perm1 directly (no copy)
  hh_factor(c, h1, l, l, s.Mt, ldl, true);
  hh_extract_r(c, h1, l, l, s.Mt, ldl, T, ldt, true);  // L = (L^T)^T, lower
  hh_form_q(c, h1, l, l, s.Qt, ldl);
  gemm_nn(c, n, l, l, s.Qhat, ldn, s.Qt, ldl, s.tmp_nl, ldn, s.orth.partials, s.orth.partial_elems);  // Q1
  gather_cols_kernel<<<grid_for(c, rows * l), 256, 0, c.stream>>>(rows, l, Q0, ldq0, s.perm1, QB, ldqb,
                                                                   piv1);  // Q0 Π1 (and piv1)
  RQLP_LAUNCHED(c);
  return s.tmp_nl;
}

void qlp_tail(Ctx &c, TailScratch &s, int64_t l, int64_t n, double *B, int64_t ldb, int d, double *QB, int64_t ldqb,
              double *T, int64_t ldt, double *PB, int64_t ldpb, int64_t *piv0, int64_t *piv1) {
  const int64_t ldn = s.ldn, ldl = s.ldl;
  // [Q0, R0, Π0] = cpqr(B)  (Alg.1 l.5)
  HHScratch h0 = s.hh;
  h0.perm = s.perm0;  // the engine's permutation lands in perm0 directly (no copy)
  hh_factor(c, h0, l, n, B, ldb, true);
  hh_extract_r(c, h0, l, n, B, ldb, s.Rt, ldn, true);   // R0^T, n x l
  // Q0 (l x l) is needed only at the assembly: formed on the side stream while the main stream
  // orthonormalises R0^T (the join precedes the next use of the reflector store s.hh)
  Ctx side = c.branch();
  hh_form_q(side, h0, l, n, s.Q0, ldl);
  c.mark("tail_cpqr_B");
  // R0^T = Q^ R^ (CholeskyQR2; the tall part of cpqr(R0^T) / the i = 1 inner QR)
  orth(c, s.orth, n, l, s.Rt, ldn, s.Qhat, ldn, s.Rhat, ldl);
  c.join(side);
  c.mark("tail_qr_R0T");
  double *PO;
  if (d == 0) {
    PO = pivoted_lq(c, s, l, l, n, s.Q0, ldl, T, ldt, QB, ldqb, piv1);
  } else {
    PO = s.Qhat;
    double *Pspare = s.tmp_nl;
    double *qe = s.Q0, *qe_spare = s.QE;  // Q^(0) Q^(2) ..., ping-pong (no copies)
    int64_t ldqe = ldl;
    const int last_even = d % 2 == 0 ? d : d - 1;
    for (int i = 2; i <= d; ++i) {
      // [Q^(i), R^(i)] = qr([R^(i-1)]^T): unpivoted, so CholeskyQR2 gives the same unique
      // factors (R_ii > 0) as Householder to rounding (reading R3).  R^(i) overwrites R^(i-1)
      // in Rhat (the input is the transposed copy in Mt); for even d the last R^(d) is T itself.
      launch_copy(c, l, l, s.Rhat, ldl, s.Mt, ldl, true);   // [R^(i-1)]^T
      const bool r_to_t = i == d && d % 2 == 0;
      orth(c, s.orth, l, l, s.Mt, ldl, s.Qt, ldl, r_to_t ? T : s.Rhat, r_to_t ? ldt : ldl, false);
      if (i % 2 == 0) {
        // the last even product goes straight to QB
        double *dst = i == last_even ? QB : qe_spare;
        const int64_t ldd = i == last_even ? ldqb : ldl;
        gemm_nn(c, l, l, l, qe, ldqe, s.Qt, ldl, dst, ldd, s.orth.partials, s.orth.partial_elems);
        qe_spare = qe;
        qe = dst;
        ldqe = ldd;
      } else {
        gemm_nn(c, n, l, l, PO, ldn, s.Qt, ldl, Pspare, ldn, s.orth.partials, s.orth.partial_elems);
        std::swap(PO, Pspare);
      }
    }
    if (d % 2 == 1) launch_copy(c, l, l, s.Rhat, ldl, T, ldt, true);   // T = [R^(d)]^T (odd d)
    if (last_even < 2) launch_copy(c, l, l, qe, ldl, QB, ldqb, false);  // d = 1: Q_B = Q^(0)
    if (piv1) {
      iota_kernel<<<grid_for(c, l), 256, 0, c.stream>>>(l, piv1);
      RQLP_LAUNCHED(c);
    }
  }
  // P_B = Π0 P1: row perm0[i] of P_B is row i of P1 (and piv0 = perm0[0..l))
  scatter_rows_kernel<<<grid_for(c, n * l), 256, 0, c.stream>>>(n, l, PO, ldn, s.perm0, PB, ldpb, piv0, l);
  RQLP_LAUNCHED(c);
  c.mark("tail_assemble");
}

// Truncated pivoted QLP of A (NEXT-3; PAPER.md:39-42 Stewart's pivoted QLP, truncated as in
// PAPER.md:177-179): the partial CPQR A Π0(:, 1:l) = Q_R [R11 R12] (l Householder steps of the
// engine on a working copy W of A), then the full CPQR of [R11 R12]^T exactly as the RQLP tail
// does for R0^T.  Q = Q_R Π1 (m x l), L (l x l, lower), P = Π0 P^ (n x l).
void tqlp(Ctx &c, TailScratch &s, HHScratch &hA, int64_t m, int64_t n, int64_t l, double *W, int64_t ldw, double *Q,
          int64_t ldq, double *L, int64_t ldl_out, double *P, int64_t ldp, int64_t *piv0, int64_t *piv1, double *QR,
          int64_t ldqr) {
  const int64_t ldn = s.ldn, ldl = s.ldl;
  HHScratch ha = hA;
  ha.perm = s.perm0;  // the engine's permutation lands in perm0 directly (no copy)
  hh_factor(c, ha, m, n, W, ldw, true, l);                  // partial CPQR, l steps
  hh_extract_r(c, ha, m, n, W, ldw, s.Rt, ldn, true, l);     // [R11 R12]^T, n x l
  hh_form_q(c, ha, m, n, QR, ldqr, l);                      // Q_R, m x l
  c.mark("tqlp_cpqr_A");
  orth(c, s.orth, n, l, s.Rt, ldn, s.Qhat, ldn, s.Rhat, ldl);
  double *PO = pivoted_lq(c, s, m, l, n, QR, ldqr, L, ldl_out, Q, ldq, piv1);
  scatter_rows_kernel<<<grid_for(c, n * l), 256, 0, c.stream>>>(n, l, PO, ldn, s.perm0, P, ldp, piv0, l);
  RQLP_LAUNCHED(c);
  c.mark("tqlp_tail");
}

}  // namespace rqlpk
