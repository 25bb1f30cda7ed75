/*
 * oracle.h -- plain, slow, CPU reference implementation ("oracle") of randomized QLP.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.  The product library
 * (paper_1811_09334_b200/, librqlp.so) never includes, links or calls anything here,
 * and this file includes nothing from the product: the two share no code.
 *
 * Paper: N. Wu, H. Xiang, "Randomized QLP algorithm and error analysis",
 * arXiv:1811.09334.  Citations "PAPER.md:L" are line numbers of the LaTeX source in the
 * upstream reference (Alg. 1 = RQLP; Alg. 2 = ERQLP, PAPER.md:137-157;
 * Alg. 3 = BRQLP).  Readings where the paper is silent or wrong are
 * listed in DESIGN.md §3 (R1..R22) and cited here by number.
 *
 * Conventions: FP64 (IEEE binary64, round to nearest even), column-major, lda >= rows,
 * compiled with -O2 -fno-fast-math -ffp-contract=off.  Every QR factorisation is
 * normalised to R_ii >= 0 (row i of R and column i of Q flipped together; reading R3).
 * Permutations are 0-based: perm[j] = original column index placed at position j.
 */
#ifndef RQLP_ORACLE_H
#define RQLP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- Ω generator (DESIGN.md §4 "RNG layout"; Alg.1 l.1 PAPER.md:95, §2 step 1 PAPER.md:74) ---- */
void orc_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);
double orc_uniform(uint64_t x);                 /* ((x>>12) + 0.5) * 2^-52, exact, in (0,1) */
double orc_ln(double u);                        /* pinned log, IEEE +,-,*,/,fma only */
void orc_sincos_2pi(uint64_t x, double *s, double *c); /* pinned sin/cos(2*pi*u(x)) */
void orc_normal4(uint64_t seed, uint64_t stream, uint64_t block, double z[4]);
/* M(i,j) = z_t, t = i + rows*j, block t/4, lane t%4 (stream 0 = Ω) */
void orc_gaussian(uint64_t seed, uint64_t stream, int64_t rows, int64_t cols, double *M, int64_t ld);

/* ---- dense building blocks ---- */
void orc_gemm_nn(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda,
                 const double *B, int64_t ldb, double *C, int64_t ldc);      /* C = A B   */
void orc_gemm_tn(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda,
                 const double *B, int64_t ldb, double *C, int64_t ldc);      /* C = A^T B */
void orc_gemm_nt(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda,
                 const double *B, int64_t ldb, double *C, int64_t ldc);      /* C = A B^T */
double orc_fro(int64_t m, int64_t n, const double *A, int64_t lda);

/* Householder QR, thin (m >= n): Q m x n, R n x n upper, R_ii >= 0.  Returns 0 or -i. */
int orc_hqr(int64_t m, int64_t n, const double *A, int64_t lda, double *Q, int64_t ldq,
            double *R, int64_t ldr);
/* Column-pivoted Householder QR (Golub greedy, LAPACK xLAQP2 downdating; readings R5).
 * s = min(m,n).  Q m x s, R s x n (columns in pivoted order, upper trapezoidal), R_ii >= 0,
 * perm[0..n) full permutation.  Q or R may be NULL. */
int orc_cpqr(int64_t m, int64_t n, const double *A, int64_t lda, double *Q, int64_t ldq,
             double *R, int64_t ldr, int64_t *perm);

/* Partial CPQR: the first k (<= min(m,n)) steps of orc_cpqr.  Q m x k, R k x n (pivot order). */
int orc_cpqr_partial(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda, double *Q, int64_t ldq,
                     double *R, int64_t ldr, int64_t *perm);

/* One-sided Jacobi SVD (Hestenes): all min(m,n) singular values, descending. */
int orc_svd_values(int64_t m, int64_t n, const double *A, int64_t lda, double *s);

/* ---- the method ---- */
/* QLP tail on B (l x n, l <= n): Alg.1 l.5-7 (d == 0) or Alg.2 l.5-9 (d >= 1, corrected
 * assembly, reading R9).  Outputs Q_B (l x l), T (l x l; lower for d==0 or odd d, upper for
 * even d >= 2), P_B (n x l), piv0 (l, global column indices), piv1 (l; identity if d >= 1). */
int orc_qlp_tail(int64_t l, int64_t n, const double *B, int64_t ldb, int d,
                 double *QB, int64_t ldqb, double *T, int64_t ldt, double *PB, int64_t ldpb,
                 int64_t *piv0, int64_t *piv1, int *t_is_upper);

/* RQLP (d == 0, Alg. 1) / ERQLP (d >= 1, Alg. 2) with q subspace iterations (reading R12).
 * V_out (m x l) and B_out (l x n) are optional (NULL) stage outputs for staged parity. */
int orc_rqlp(int64_t m, int64_t n, int k, int p, int q, int d, const double *A, int64_t lda,
             uint64_t seed, double *Q, int64_t ldq, double *T, int64_t ldt, double *P, int64_t ldp,
             int64_t *piv0, int64_t *piv1, int *t_is_upper, double *V_out, int64_t ldv,
             double *B_out, int64_t ldb);

/* BRQLP (Alg. 3) with explicit deflation on a working copy of A (eq. (19)), ragged last block
 * (reading R14), q deflated subspace iterations per block (reading R16).  L = blkdiag(L_j).
 * piv0: global column indices per block; piv1: indices local to the block. */
int orc_brqlp(int64_t m, int64_t n, int k, int p, int b, int q, const double *A, int64_t lda,
              uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *P, int64_t ldp,
              int64_t *piv0, int64_t *piv1, double *V_out, int64_t ldv);

/* Auto-rank RQLP (NEXT-1; "auto-rank randomized QLP", eq. (3)):
 * BRQLP blocks of b columns (Ω columns jb..jb+b-1 of an n x l_max Ω, explicit deflation, q
 * deflated power steps) are added until the error indicator ||A||_F^2 - sum_j ||B_j||_F^2 <=
 * (eps ||A||_F)^2 (reading R25) or l reaches l_max.  Returns 0; *l_out = columns used; err_out
 * (nullable) receives the final indicator sqrt(max(0, ||A||^2 - sum ||B_j||^2)) / ||A||_F.
 * Q (m x l_max), L (l_max x l_max), P (n x l_max): the first *l_out columns are the result. */
int orc_autorank(int64_t m, int64_t n, int b, int l_max, int q, double eps, const double *A, int64_t lda,
                 uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *P, int64_t ldp,
                 int64_t *piv0, int64_t *piv1, int *l_out, double *err_out);

/* Truncated pivoted QLP (NEXT-3): partial CPQR of A (l steps), then
 * CPQR of [R11 R12]^T.  Q m x l, L l x l lower, P n x l, piv0/piv1 int64[l]. */
int orc_tqlp(int64_t m, int64_t n, int64_t l, const double *A, int64_t lda, double *Q, int64_t ldq, double *L,
             int64_t ldl, double *P, int64_t ldp, int64_t *piv0, int64_t *piv1);

/* ||A - Q T P^T||_F computed directly, row by row (never forms m x n). */
double orc_residual(int64_t m, int64_t n, int64_t l, const double *A, int64_t lda,
                    const double *Q, int64_t ldq, const double *T, int64_t ldt,
                    const double *P, int64_t ldp);

int orc_num_threads(void);
void orc_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
