/*
 * rqlp.h -- C ABI of librqlp.so: B200-native (sm_100a) FP64 randomized QLP.
 *
 * Paper: N. Wu, H. Xiang, "Randomized QLP algorithm and error analysis", arXiv:1811.09334.
 * "PAPER.md:L" cites line L of the paper's LaTeX source (the upstream reference); the readings
 * (R1..R30) where the paper is silent, garbled or wrong are listed in DESIGN.md §3.
 *
 * Conventions (all entry points)
 *   - FP64 (IEEE binary64, round-to-nearest-even), column-major, leading dimension >= rows.
 *   - Matrix / pivot pointers are DEVICE pointers unless an entry point says otherwise; all
 *     work is enqueued on the handle's CUDA stream and returns without a host sync.
 *   - l = k + p.  Outputs are l-sized; truncation to rank k is a caller-side
 *     slice (leading k columns of Q, P and leading k x k of L).
 *   - Every QR inside is normalised to R_ii >= 0 (reading R3), so Q, L, P are unique given the
 *     pivots; L-values are diag(L) >= 0.
 *   - Permutations are 0-based column indices of A: piv0[t] = column of A chosen at step t of
 *     CPQR(B) (Π0); piv1[t] = index chosen at step t of CPQR(R0^T) (Π1).
 *   - Ownership: the caller allocates and owns A, the outputs, the pivot arrays and the
 *     workspace.  A is read-only and never written.  The library owns only the
 *     handle's metadata (and, for rqlp(), a cached default workspace).
 *   - Errors (LAPACK style): 0 = success; -i = argument i illegal (checked before anything is
 *     enqueued); positive RQLP_ERR_* codes below for runtime failures.  Device-side numerical
 *     events (shifted CholeskyQR fallback taken) are not errors: rqlp_sync() reports them.
 *   - Threads: calls on ONE handle are serialised by a per-handle lock (rqlp() shares one
 *     default handle per device between all threads); different handles run concurrently.  The
 *     device buffers a call reads or writes must not be used by other streams until the
 *     handle's stream has passed the call (the Python binding orders the handle's stream against
 *     torch's current stream on both sides of every call).
 */
#ifndef RQLP_H
#define RQLP_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RQLP_OK 0
#define RQLP_ERR_CUDA 1          /* a CUDA runtime call failed */
#define RQLP_ERR_NCCL 2          /* a NCCL call failed (distributed handle) */
#define RQLP_ERR_WORKSPACE 3     /* workspace missing or smaller than rqlp_workspace_size() */
#define RQLP_ERR_INTERNAL 4
#define RQLP_ERR_DEVICE 5        /* device is not sm_100 (B200) */
#define RQLP_ERR_HANDLE 6        /* NULL / destroyed handle */
#define RQLP_ERR_UNSUPPORTED 7   /* operation not available on this handle (e.g. distributed) */

#define RQLP_VARIANT_RQLP 0      /* Algorithm 1 */
#define RQLP_VARIANT_ERQLP 1     /* Algorithm 2 */
#define RQLP_VARIANT_BRQLP 2     /* Algorithm 3 */

/* rqlp_sync() flag bits */
#define RQLP_FLAG_SHIFTED_CHOLQR 1u  /* a shifted CholeskyQR pass was needed (cond(Y) >~ 1e6) */
#define RQLP_FLAG_RANK_DEFICIENT 2u  /* a sketch was numerically rank deficient (a Cholesky pivot
                                        <= 1e-15 of its Gram diagonal, i.e. a direction below
                                        ~3e-8 relative) or a basis column was completed */

#define RQLP_FLAG_REPLICA_MISMATCH 4u /* row-sharded handles: after the sum of the projected B (Alg. 1
                                        l.4) the ranks did not all hold the same bits
                                        (a 64-bit hash of B is compared across the ranks); the
                                        replicated tail may then have diverged -- L, P and the pivots
                                        are not trustworthy.  Set on every rank.
                                        RQLP_REPLICA_CHECK=0 in the environment skips the check. */

typedef struct rqlp_handle_s *rqlp_handle_t;

/* Create a single-GPU handle on `device`, enqueuing on `cuda_stream` (a cudaStream_t; NULL =
 * legacy default stream).  Fails with RQLP_ERR_DEVICE if the device is not compute 10.x. */
int rqlp_create(rqlp_handle_t *h, int device, void *cuda_stream);

/* Create a handle for one rank of a row-sharded run.  `nccl_unique_id` points
 * to the 128-byte ncclUniqueId created by rank 0 and shared by the caller (e.g. through
 * torch.distributed).  Every rank then calls the factorisations collectively with its local
 * row count m_local, its row block of A and the same seed; Q is returned for the local rows,
 * L, P and the pivots are replicated.  Unlike the single-GPU handle, a factorisation call on a
 * sharded handle synchronises its stream once before returning (the breakdown word of the
 * optimistic run, see rqlp_careful_rerun_count). */
int rqlp_create_dist(rqlp_handle_t *h, int device, void *cuda_stream, const void *nccl_unique_id,
                     int rank, int nranks);
int rqlp_get_unique_id(void *nccl_unique_id_out /* 128 bytes */);

/* Create `nranks` (1..64) handles that act as the ranks of a row-sharded run INSIDE one process
 * on ONE device (the multi-rank path testable on a single GPU).  handles_out
 * receives nranks handles; all enqueue on `cuda_stream`.  Call the factorisations collectively
 * exactly as with rqlp_create_dist handles -- one host thread per rank, each with its rank's row
 * block of A and the same remaining arguments.  The ranks take turns (a host token ring) to
 * enqueue their work on the shared stream, so the device runs the ranks' segments one after the
 * other and no kernel ever waits for another rank; every sum over ranks adds the ranks' partials
 * in fixed rank order, so the replicated outputs (L/T, P, pivots) are bit-identical on every
 * rank.  A rank that fails (or whose call sequence diverges) aborts the group: the other ranks'
 * calls return RQLP_ERR_NCCL (after at most 600 s).  Destroy every handle with rqlp_destroy. */
int rqlp_create_loopback(rqlp_handle_t *handles_out, int nranks, int device, void *cuda_stream);
int rqlp_destroy(rqlp_handle_t h);

/* Bytes of device workspace the given call needs (m = local rows). */
int rqlp_workspace_size(rqlp_handle_t h, int variant, int64_t m, int64_t n, int k, int p, int q, int d,
                        int b, size_t *bytes);
/* Use caller-owned device memory (e.g. a torch uint8 tensor) as workspace.  256-B aligned. */
int rqlp_set_workspace(rqlp_handle_t h, void *dev_ptr, size_t bytes);

/* North-star form (BASELINE.json): RQLP (Alg. 1) with q subspace iterations on the default
 * handle of the current device, ldq = m, ldl = l, ldp = n.  A, Q, L, P may be HOST or DEVICE
 * pointers (detected per pointer): host buffers are staged through device memory inside the
 * call (this is the end-to-end path bench.py times).  Synchronous: returns after Q, L, P are
 * written.  Outputs: Q m x l (orthonormal), L l x l lower triangular, P n x l (orthonormal),
 * A ~= Q L P^T (eq. (5)). */
int rqlp(int64_t m, int64_t n, int k, int p, int q, const double *A, int64_t lda, uint64_t seed,
         double *Q, double *L, double *P);

/* Algorithm 1 + q subspace iterations (reading R12):
 *   Ω = N(0,1) n x l from Philox(seed); Y = AΩ; V = orth(Y);
 *   repeat q: Z = A^T V, W = orth(Z), Y = AW, V = orth(Y);
 *   B = V^T A; [Q0,R0,Π0] = cpqr(B); [Q1,L^T,Π1] = cpqr(R0^T); Q = V Q0 Π1, P = Π0 Q1.
 * Arguments: m>=1 (1), n>=1 (2), k>=2 (3), p>=2 (4) with l=k+p <= min(m_global, n), q>=0 (5),
 * A (6) m x n, lda>=m (7), seed (8), Q m x l (9) ldq>=m (10), L l x l (11) ldl>=l (12),
 * P n x l (13) ldp>=n (14), piv0 int64[l] (15, nullable), piv1 int64[l] (16, nullable). */
int rqlp_ex(rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int q, const double *A, int64_t lda,
            uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *P, int64_t ldp,
            int64_t *piv0, int64_t *piv1);

/* Algorithm 2 + q subspace iterations: d >= 1 unpivoted inner QRs
 * [Q^(i),R^(i)] = qr([R^(i-1)]^T).  Corrected assembly (reading R9): A ~= Q T P^T with
 * Q = V Q^(0) Q^(2)..., P = Π0 Q^(1) Q^(3)..., T = [R^(d)]^T (lower) for odd d and R^(d)
 * (upper) for even d; *t_is_upper (host int) = (d even).  L-values = diag(T).
 * Arguments as rqlp_ex with d (6) inserted after q, T/ldt in place of L/ldl, t_is_upper
 * (host, nullable), piv0 (nullable). */
int erqlp_ex(rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int q, int d, const double *A,
             int64_t lda, uint64_t seed, double *Q, int64_t ldq, double *T, int64_t ldt, int *t_is_upper,
             double *P, int64_t ldp, int64_t *piv0);

/* Algorithm 3 + q deflated subspace iterations per block (reading R16):
 * block size 1 <= b <= l, h = ceil(l/b) blocks, ragged last block (reading R14);
 * Y_j = AΩ_j with the original A (line 3, reading R15), V_j = qr(Y_j), the block-CGS
 * re-orthogonalisation of eq. (18) applied twice (reading R28: "twice is enough" -- identical
 * in exact arithmetic whenever V_j has a component outside span(V_<j)), B_j = V_j^T A^(j-1)
 * with A^(j-1) applied implicitly
 * (A^(j-1) X = AX - V_<j (B_<j X), identical to eq. (19) in exact arithmetic), per-block
 * pivoted QLP of B_j, Q_j = V_j Q_B^(j), L = blkdiag(L_j) (lower), P = [P_1 .. P_h].
 * piv0[t] = global column of A, piv1[t] = index local to t's block. */
int brqlp_ex(rqlp_handle_t h, int64_t m, int64_t n, int k, int p, int b, int q, const double *A,
             int64_t lda, uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *P,
             int64_t ldp, int64_t *piv0, int64_t *piv1);

/* Truncated pivoted QLP: the deterministic rank-l QLP the paper compares
 * against (Stewart's pivoted QLP, truncated as in PAPER.md:177-179): partial
 * CPQR A Π0(:, 1:l) = Q_R [R11 R12] (l Householder steps, same pivot rule as the RQLP tail,
 * reading R5), then the full CPQR [R11 R12]^T Π1 = P^ L^T; Q = Q_R Π1, P = Π0 P^.
 * Arguments: h (1), m (2), n (3), l (4) with 1 <= l <= min(m, n), A (5) device m x n
 * column-major, read only, lda (6) >= m, Q (7) device m x l, ldq (8) >= m, L (9) device l x l
 * lower triangular, ldl (10) >= l, P (11) device n x l, ldp (12) >= n, piv0 / piv1 (13, 14)
 * device int64[l] (nullable): Π0's first l columns (original indices) and Π1.  Asynchronous on
 * the handle's stream; workspace: the caller's (if set and large enough) or library-owned.
 * Not available on distributed handles (RQLP_ERR_UNSUPPORTED). */
int rqlp_tqlp_ex(rqlp_handle_t h, int64_t m, int64_t n, int l, const double *A, int64_t lda, double *Q,
                 int64_t ldq, double *L, int64_t ldl, double *P, int64_t ldp, int64_t *piv0,
                 int64_t *piv1);

/* Auto-rank RQLP (the "auto-rank randomized QLP" the
 * paper leaves as future work): the BRQLP block loop (Alg. 3, per-block sketch Y_j = AΩ_j with
 * the first l_max columns of Ω, implicit deflation, q deflated power steps) adds blocks of b
 * columns until the error indicator of eq. (3), ||A||_F^2 - sum_j ||B_j||_F^2,
 * is <= (eps ||A||_F)^2 (reading R25: eps is relative to ||A||_F) or l_max columns are used.
 * Arguments: h (1), m (2), n (3), block size b (4) >= 1, l_max (5) with b <= l_max <= min(m, n),
 * q (6) >= 0, eps (7) >= 0, A (8) device m x n, lda (9) >= m, seed (10), Q (11) m x l_max,
 * ldq (12), L (13) l_max x l_max, ldl (14), P (15) n x l_max, ldp (16), piv0/piv1 (17, 18)
 * int64[l_max] (nullable), *l_out (19, host) = columns used, *err_out (20, host, nullable) =
 * the final indicator sqrt(max(0, ||A||^2 - sum ||B_j||^2)) / ||A||_F.  The first *l_out
 * columns of Q, P (and the leading *l_out x *l_out block of L) are the factorisation.
 * Synchronous (one device->host read of the indicator per block). */
int rqlp_autorank_ex(rqlp_handle_t h, int64_t m, int64_t n, int b, int l_max, int q, double eps,
                     const double *A, int64_t lda, uint64_t seed, double *Q, int64_t ldq, double *L,
                     int64_t ldl, double *P, int64_t ldp, int64_t *piv0, int64_t *piv1, int *l_out,
                     double *err_out);

/* Synchronous any-pointer form of rqlp_ex / erqlp_ex / brqlp_ex on handle h: `variant` (2)
 * selects the algorithm (RQLP_VARIANT_*), d (8) is used by ERQLP, b (9) by BRQLP.  A (10), Q (13),
 * T (14), P (15) may be host (pageable or pinned) or device pointers; host operands are copied
 * through device staging buffers inside the call (ldq = m, ldt = l, ldp = n).  A pinned host A is
 * copied in row panels overlapped with the sketch pass; for BRQLP, pinned host Q and P receive each
 * block's columns while the later blocks run (the results are bit-identical to the device path).
 * Returns after the outputs are written.  This is the end-to-end path bench.py times ("e2e"). */
int rqlp_factorize(rqlp_handle_t h, int variant, int64_t m, int64_t n, int k, int p, int q, int d, int b,
                   const double *A, int64_t lda, uint64_t seed, double *Q, double *T, double *P, int *t_is_upper);

/* The error indicator of eq. (3) (§6) of the last rqlp_ex /
 * erqlp_ex / brqlp_ex / rqlp_autorank_ex / rqlp_factorize on h: *a2 = ||A||_F^2 (accumulated
 * inside the first A-pass from the same A tiles, summed over the ranks of a sharded handle) and
 * *b2 = ||B||_F^2 (BRQLP / auto-rank: sum_j ||B_j||_F^2 of the deflated B_j), so that
 * ||A - V V^T A||_F^2 = *a2 - *b2 in exact arithmetic (V orthonormal).  Waits for the handle's
 * stream.  Either pointer may be NULL. */
int rqlp_get_indicator(rqlp_handle_t h, double *a2, double *b2);

/* Wait for the handle's stream; *flags (nullable) receives RQLP_FLAG_* bits of the last call.
 * On a NCCL handle an asynchronous NCCL failure (ncclCommGetAsyncError) returns RQLP_ERR_NCCL. */
int rqlp_sync(rqlp_handle_t h, unsigned *flags);
const char *rqlp_strerror(int code);

/* ---- stage entry points (same kernels the factorisations use; for staged parity tests) ---- */
/* Ω(i,j) = z_t, t = i + n j: Alg.1 l.1. */
int rqlp_omega(rqlp_handle_t h, int64_t n, int64_t l, uint64_t seed, double *Omega, int64_t ldo);
/* Y = A X  (m x k times k x c) -- the sketch / power pass kernel (Alg.1 l.2). */
int rqlp_gemm_nn(rqlp_handle_t h, int64_t m, int64_t c, int64_t k, const double *A, int64_t lda,
                 const double *X, int64_t ldx, double *Y, int64_t ldy);
/* Z = A^T V (k x m times m x c -> k x c), or its transpose (c x k) when trans_out != 0 -- the
 * projection pass B = V^T A (Alg.1 l.4) and the power step A^T V. */
int rqlp_gemm_tn(rqlp_handle_t h, int64_t m, int64_t c, int64_t k, const double *A, int64_t lda,
                 const double *V, int64_t ldv, double *Z, int64_t ldz, int trans_out);
/* V = orth(Y) (m x c, c <= m): CholeskyQR2; after a Cholesky breakdown (cond(Y) >~ 1e6, or
 * rank(Y) < c), shifted CholeskyQR passes until V is orthonormal to working precision (Alg.1
 * l.3).  R (c x c upper, Y = V R to O(u ||Y||); R_ii > 0 for full-rank Y) written
 * when non-NULL. */
int rqlp_orth(rqlp_handle_t h, int64_t m, int64_t c, const double *Y, int64_t ldy, double *V, int64_t ldv,
              double *R, int64_t ldr);
/* Column-pivoted Householder QR of M (rows x cols), s = min(rows, cols) steps (Alg.1 l.5):
 * Q rows x s, R s x cols (pivoted column order), perm int64[cols] (first s = pivots). */
int rqlp_cpqr(rqlp_handle_t h, int64_t rows, int64_t cols, const double *M, int64_t ldm, double *Q,
              int64_t ldq, double *R, int64_t ldr, int64_t *perm);
/* QLP tail of B (l x n, l <= n): d == 0 -> Alg.1 l.5-7, d >= 1 -> Alg.2 l.5-9 (corrected). */
int rqlp_qlp_tail(rqlp_handle_t h, int64_t l, int64_t n, const double *B, int64_t ldb, int d, double *QB,
                  int64_t ldqb, double *T, int64_t ldt, double *PB, int64_t ldpb, int64_t *piv0, int64_t *piv1,
                  int *t_is_upper);
/* ||A - Q T P^T||_F^2 (m x n, l columns) into *res_dev (device double), fused: never forms the
 * m x n difference (validation kernel, eq. (5)). */
int rqlp_residual_sq(rqlp_handle_t h, int64_t m, int64_t n, int64_t l, const double *A, int64_t lda,
                     const double *Q, int64_t ldq, const double *T, int64_t ldt, const double *P,
                     int64_t ldp, double *res_dev);

/* Stage outputs for staged parity (tests): subsequent factorisations on h copy the sketch
 * Y = AΩ (m x l, before orthonormalisation), the final range basis V (m x l) and the projected
 * B (l x n; for BRQLP the deflated B_j rows) into these device buffers.  Any may be NULL;
 * rqlp_set_stage_outputs(h, NULL, 0, NULL, 0, NULL, 0) turns it off. */
int rqlp_set_stage_outputs(rqlp_handle_t h, double *Y, int64_t ldy, double *V, int64_t ldv, double *B,
                           int64_t ldb);

/* Power-step stage outputs (tests; staged parity of every A-pass at full size): subsequent
 * factorisations on h copy, for power iteration it (0..q-1), V before the step (m x l), its A-pass
 * result Z = A^T V (n x l; BRQLP: the deflated A^(j-1)^T V_j), W = orth(Z) (n x l) and the A-pass
 * result Y = A W (m x l; BRQLP: deflated) into columns it*l .. it*l+l-1 of these buffers (BRQLP:
 * block j's columns it*l + c0_j ..).  Buffers are m x (q l) / n x (q l).  NULL turns one off. */
int rqlp_set_power_stage_outputs(rqlp_handle_t h, double *Vpre, int64_t ldvp, double *Z, int64_t ldz, double *W,
                                 int64_t ldw, double *Ypow, int64_t ldyp);

/* Per-stage device timings (ms) of the last factorisation when timing is enabled:
 * names/values written up to *count entries; returns number available. */
int rqlp_set_timing(rqlp_handle_t h, int enable);
int rqlp_get_timing(rqlp_handle_t h, const char **names, float *ms, int capacity);
/* Kernel launches issued by the last call (for bench.py's gpu_launches). */
int64_t rqlp_launch_count(rqlp_handle_t h);
/* Row-sharded handles (rqlp_create_dist / rqlp_create_loopback) run each factorisation
 * optimistically: the orthonormalisations (Alg. 1 l.3) are CholeskyQR2 with no
 * device-to-host readback; a Cholesky breakdown (a sketch beyond CholeskyQR2's reach) is recorded on
 * the device, read back once when the factorisation has been enqueued, and the factorisation is then
 * repeated on the careful path (shifted passes driven from the host, one readback per orth).  Every
 * rank takes the same decision (the Grams are summed to identical bits).  Returns how many calls on
 * this handle were repeated so; -1 for an invalid handle.  RQLP_SHARDED_OPTIMISTIC=0 in the
 * environment selects the careful path from the start. */
int64_t rqlp_careful_rerun_count(rqlp_handle_t h);

#ifdef __cplusplus
}
#endif
#endif
