// gemm_tma.cu -- TMA-pipelined FP64 DMMA kernels for the tall-skinny A-passes.
//
//   NN: Y (m x c) = A (m x k) X (k x c)      -- the sketch Y = AΩ (Alg.1 l.2), the
//                                              power step Y = AW, Q = V Q_B and Y R^-1
//   TN: Z (k x c) = A^T (k x m) V (m x c)    -- the projection B = V^T A (Alg.1 l.4, PAPER.md:98,
//                                              written transposed), the power step A^T V, Grams
//
// B200 design: no FP64 tcgen05 exists, so the MMA is mma.sync m8n8k4.f64
// (SASS DMMA.8x8x4, measured 37.07 TFLOP/s chip-wide vs 34.1 for DFMA).  A CTA owns a
// 128 x BN output tile (BN = 16..144 chosen per c to minimise padding); 8 consumer warps
// (4 x 2) each hold a 32 x BN/2 accumulator block in registers; thread 0 also streams
// BK = 24-deep slabs of A and of X/V into a 4-stage shared-memory ring with TMA
// (cp.async.bulk.tensor, mbarrier complete_tx).  The shared layouts are chosen so every
// fragment load is bank-conflict free WITHOUT swizzling:
//   * K-major tiles (X, V, and A in TN) are [rows][24]: 24 = 8 mod 16 doubles, so the 16-byte
//     fragment loads (two k's per thread, feeding two DMMAs) of a quarter warp hit 32 banks.
//   * the M-major A tile of NN is [24][130]: the TMA box is 130 rows tall (2 rows of overlap
//     with the next tile, zero-filled past m), giving LD = 130 = 2 mod 8.
// Split-K (gridDim.z) writes FP64 partial tiles reduced in a fixed order (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.cuh"

namespace rqlpk {

void launch_reduce(Ctx &c, int64_t M, int64_t N, int S, const double *part, double alpha, double beta, double *C,
                   int64_t ldc, bool trans, const unsigned *cond, unsigned cond_mask);
void gemm_generic_ex(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                     int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc, double *partials,
                     size_t partial_elems, bool trans_out, const unsigned *cond, unsigned cond_mask);

namespace {

constexpr int BM = 128, BK = 24, STAGES = 4, NCONS = 8;
// CTAs per SM of the plain (non-||A||^2) kernel of width bn = 32..64: 2 when the launch has many
// tiles or much work per tile (measured, C4-sized operands: the 64-wide A-passes 34.6 -> 36.2
// TFLOP/s, 48-wide 34.6 -> 35.9, 32-wide 30.4 -> 33.8, m x 64 times 64 x 64 133 -> 93 us; a
// single-tile Gram or few short tiles lose with 3 stages); else 1.  RQLP_GEMM_OCC2=w: widths <= w
// (0: none; measurement switch).
int gemm_occ(int bn, bool fro, int64_t tiles = 1 << 30, int64_t ktiles = 1 << 30) {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("RQLP_GEMM_OCC2");
    on = e ? atoi(e) : 64;   // the widest tile width that runs two CTAs per SM (0: none)
  }
  if (!on || bn > on || bn < 32 || fro) return 1;   // (16: memory-bound, the TN pass loses 5.2 -> 5.7 ms)
  return (tiles >= 296 || tiles * ktiles >= 40000) ? 2 : 1;
}
// the ||A||^2 warp makes 9 warps: 3 on one SM sub-partition caps the registers at 168 per thread,
// which spills the accumulators for BN > 96 -- those passes use a separate ||A||^2 pass
constexpr int FRO_MAX_BN = 96;
constexpr int LDA_NN = BM + 2;  // doubles
constexpr int A_TILE_BYTES_NN = ((BK * LDA_NN * 8 + 127) / 128) * 128;
constexpr int A_TILE_BYTES_TN = BM * BK * 8;

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// MODE 0 = NN, 1 = TN.  Output element (i, j) of the (M x N) product goes to
//   part (split-K slice, M x N contiguous)  or  C[i + j ldc]  or (trans) C[j + i ldc].
// OCC = 2 (BN = 64 only): two CTAs per SM (3-stage rings, <= 128 registers): 16 warps hide the
// DMMA chains of the narrow 32 x 32 warp tiles better than 8 (measured in DESIGN.md §5).
template <int BN, int MODE, bool FRO, int OCC = 1>
__global__ void __launch_bounds__((NCONS + (FRO ? 1 : 0)) * 32, OCC)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M, int N,
                    int ktiles_total, int ktiles_per_split, double *__restrict__ C, int64_t ldc, int trans,
                    double *__restrict__ part, const unsigned *cond, unsigned cond_mask, int tri, int bal_units,
                    int ntn, int maxc, double *__restrict__ fro_slots, double alpha, double beta) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  // tri == 1: only the upper triangle of the (symmetric) output is wanted -- tiles strictly below
  // the diagonal do nothing (a Gram; consumers read the upper triangle).  tri == 2: the B operand
  // is upper triangular -- k-tiles at or beyond n0 + BN contribute nothing (Y R^-1).
  if (tri == 1 && (int)(blockIdx.y * BM) >= (int)(blockIdx.x * BN) + BN) return;
  constexpr int NST = OCC == 2 ? 3 : STAGES;
  constexpr int A_BYTES = MODE == 0 ? A_TILE_BYTES_NN : A_TILE_BYTES_TN;
  constexpr int B_BYTES = BN * BK * 8;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int NB = BN / 16;  // 8-col fragments per warp (warp tile 32 x BN/2)
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + NST * STAGE_BYTES);
  uint64_t *empty = full + NST;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // balanced split (bal_units > 0, tri == 0): the (tile, k-tile) units in tile-major order are
  // dealt out in equal contiguous runs of bal_units, one run per CTA (grid = #SMs); a run spans
  // at most a few tiles and each tile segment's partial goes to slot (tile, CTA - first CTA of
  // the tile), summed in slot order by bal_reduce_kernel.  Otherwise grid = (N tiles, M tiles,
  // split-K slices).
  const bool bal = bal_units > 0;
  const int n0 = bal ? 0 : blockIdx.x * BN, m0 = bal ? 0 : blockIdx.y * BM;
  const int kt0 = bal ? 0 : blockIdx.z * ktiles_per_split;
  const int u0 = bal ? blockIdx.x * bal_units : 0;
  int nkt;
  if (bal) {
    const int total = ktiles_total * ntn * ((M + BM - 1) / BM);
    nkt = max(0, min(total, u0 + bal_units) - u0);
  } else {
    const int klim = tri == 2 ? min(ktiles_total, (n0 + BN + BK - 1) / BK) : ktiles_total;
    const int kt1 = min(klim, kt0 + ktiles_per_split);
    nkt = max(0, kt1 - kt0);
  }
  // (tile origin, k offset) of pipeline iteration it
  auto coords = [&](int it, int &tm0, int &tn0, int &kk) {
    if (bal) {
      const int u = u0 + it, t = u / ktiles_total, kt = u - t * ktiles_total;
      tm0 = (t / ntn) * BM;
      tn0 = (t % ntn) * BN;
      kk = kt * BK;
    } else {
      tm0 = m0;
      tn0 = n0;
      kk = (kt0 + it) * BK;
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS + (FRO ? 1 : 0));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ---------------- producer role (thread 0 of warp 0): TMA slabs NST-1 iterations ahead
  auto issue = [&](int it) {
    const int s = it % NST;
    unsigned char *sa = smem + s * STAGE_BYTES;
    unsigned char *sb = sa + A_BYTES;
    int tm0, tn0, kk;
    coords(it, tm0, tn0, kk);
    mbar_expect_tx(&full[s], (MODE == 0 ? BK * LDA_NN * 8 : A_TILE_BYTES_TN) + B_BYTES);
    if (MODE == 0) tma_load_2d(sa, &mapA, tm0, kk, &full[s]);   // A box {BM+2, BK} at (m0, k)
    else tma_load_2d(sa, &mapA, kk, tm0, &full[s]);             // A box {BK, BM} at (k = row offset, col)
    tma_load_2d(sb, &mapB, kk, tn0, &full[s]);                  // B box {BK, BN} at (k, n0)
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mapB) : "memory");
    for (int it = 0; it < NST - 1 && it < nkt; ++it) issue(it);
  }

  // ---------------- ||A||_F^2 fused into the NN pass (eq. (3); FRO, MODE 0): a 9th
  // warp squares every staged A tile (rows 0..127 of the 130-row box; OOB rows and columns are
  // zero-filled) and releases the stage like a consumer; only the CTAs of output column tile 0
  // count (the other column tiles re-read A).  Measured: the same FMAs inside the consumer warps'
  // MMA loop cost the pass ~7 % (register growth, a broken load/MMA schedule); a compile-time
  // switch, as a runtime one cost the plain NN kernel ~10 %.
  static_assert(!FRO || MODE == 0, "||A||^2 is fused into the NN pass only");
  if (FRO && warp == NCONS) {
    double f0 = 0.0, f1 = 0.0, f2 = 0.0, f3 = 0.0;
    const bool fro_on = bal || n0 == 0;
    for (int it = 0; it < nkt; ++it) {
      const int s = it % NST;
      mbar_wait(&full[s], (it / NST) & 1);
      // balanced runs: count the unit if its tile is in output column tile 0
      if (fro_on && (!bal || ((u0 + it) / ktiles_total) % ntn == 0)) {
        const double *sa = reinterpret_cast<const double *>(smem + s * STAGE_BYTES);
#pragma unroll 4
        for (int k = 0; k < BK; ++k) {
          const double *colk = sa + k * LDA_NN;
          const double x0 = colk[lane], x1 = colk[lane + 32], x2 = colk[lane + 64], x3 = colk[lane + 96];
          f0 = fma(x0, x0, f0);
          f1 = fma(x1, x1, f1);
          f2 = fma(x2, x2, f2);
          f3 = fma(x3, x3, f3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    double f = (f0 + f1) + (f2 + f3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
    if (lane == 0) fro_slots[blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z)] = f;
    return;
  }

  // ---------------- consumers: 8 warps, 4 (M) x 2 (N), warp tile 32 x BN/2
  const int wm = warp & 3, wn = warp >> 2;
  const int r = lane >> 2, cq = lane & 3;
  double acc[4][NB][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int it = 0; it < nkt; ++it) {
    const int s = it % NST;
    if (threadIdx.x == 0 && it + NST - 1 < nkt) {
      // refill the slot consumed at iteration it-1 once every warp has released it
      if (it >= 1) mbar_wait(&empty[(it - 1) % NST], ((it - 1) / NST) & 1);
      issue(it + NST - 1);
    }
    mbar_wait(&full[s], (it / NST) & 1);
    const double *sa = reinterpret_cast<const double *>(smem + s * STAGE_BYTES);
    const double *sb = reinterpret_cast<const double *>(smem + s * STAGE_BYTES + A_BYTES);
#pragma unroll
    for (int kk = 0; kk < BK / 8; ++kk) {
      double a0[4], a1[4];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) {
        const int row = wm * 32 + mb * 8 + r;
        if (MODE == 0) {
          a0[mb] = sa[(kk * 8 + 2 * cq) * LDA_NN + row];
          a1[mb] = sa[(kk * 8 + 2 * cq + 1) * LDA_NN + row];
        } else {
          const double2 v = *reinterpret_cast<const double2 *>(sa + row * BK + kk * 8 + 2 * cq);
          a0[mb] = v.x;
          a1[mb] = v.y;
        }
      }
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int col = wn * (BN / 2) + nb * 8 + r;
        const double2 b = *reinterpret_cast<const double2 *>(sb + col * BK + kk * 8 + 2 * cq);
#pragma unroll
        for (int mb = 0; mb < 4; ++mb) {
          dmma(acc[mb][nb][0], acc[mb][nb][1], a0[mb], b.x);
          dmma(acc[mb][nb][0], acc[mb][nb][1], a1[mb], b.y);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (bal && (it + 1 == nkt || (u0 + it + 1) % ktiles_total == 0)) {
      // end of a tile segment: its partial tile (all BM x BN entries) to the tile's slot
      const int t = (u0 + it) / ktiles_total;
      const int slot = blockIdx.x - (int)(((long long)t * ktiles_total) / bal_units);
      double *dst = part + ((size_t)t * maxc + slot) * (BM * BN);
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) {
        const int il = wm * 32 + mb * 8 + r;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          const int jl = wn * (BN / 2) + nb * 8 + 2 * cq;
          dst[il + jl * BM] = acc[mb][nb][0];
          dst[il + (jl + 1) * BM] = acc[mb][nb][1];
          acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
        }
      }
    }
  }
  if (bal) return;

  // ---------------- epilogue: fragment (mb, nb) holds out[row][col], out[row][col+1]
  // (split-K partials are scaled by the reduce; C = alpha acc + beta C otherwise)
  if (!part && (alpha != 1.0 || beta != 0.0)) {
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) {
      const int i = m0 + wm * 32 + mb * 8 + r;
      if (i >= M) continue;
      // the old values of this row's 2 NB entries are loaded together, then combined and stored: read
      // one by one in front of each store (the loads cannot move above earlier stores through the
      // same pointer) they made 8 NB dependent round trips per thread -- m x 64, K = 384 with
      // beta = 1: 450 us against 369 us for the same product with beta = 0
      // (tiles up to 64 wide: the wider instances have no registers to spare and no such products)
      constexpr bool BATCH = BN <= 64;
      double cv[BATCH ? NB : 1][2];
      if (BATCH && beta != 0.0) {
#pragma unroll
        for (int nb = 0; nb < (BATCH ? NB : 0); ++nb) {
          const int j = n0 + wn * (BN / 2) + nb * 8 + 2 * cq;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double *src = trans ? C + (j + e) + (size_t)i * ldc : C + i + (size_t)(j + e) * ldc;
            cv[nb][e] = j + e < N ? *src : 0.0;
          }
        }
      }
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int j = n0 + wn * (BN / 2) + nb * 8 + 2 * cq;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (j + e >= N) continue;
          double *dst = trans ? C + (j + e) + (size_t)i * ldc : C + i + (size_t)(j + e) * ldc;
          double v = alpha * acc[mb][nb][e];
          if (beta != 0.0) v = fma(beta, BATCH ? cv[BATCH ? nb : 0][e] : *dst, v);
          *dst = v;
        }
      }
    }
    return;
  }
#pragma unroll
  for (int mb = 0; mb < 4; ++mb) {
    const int i = m0 + wm * 32 + mb * 8 + r;
    if (i >= M) continue;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int j = n0 + wn * (BN / 2) + nb * 8 + 2 * cq;
      if (part) {
        double *dst = part + (size_t)blockIdx.z * M * N;
        if (j < N) dst[i + (size_t)j * M] = acc[mb][nb][0];
        if (j + 1 < N) dst[i + (size_t)(j + 1) * M] = acc[mb][nb][1];
      } else if (trans) {
        double *dst = C + j + (size_t)i * ldc;
        if (j + 1 < N && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
          *reinterpret_cast<double2 *>(dst) = make_double2(acc[mb][nb][0], acc[mb][nb][1]);
        } else {
          if (j < N) dst[0] = acc[mb][nb][0];
          if (j + 1 < N) dst[1] = acc[mb][nb][1];
        }
      } else {
        if (j < N) C[i + (size_t)j * ldc] = acc[mb][nb][0];
        if (j + 1 < N) C[i + (size_t)(j + 1) * ldc] = acc[mb][nb][1];
      }
    }
  }
}

// G = Y^T Y (symmetric, both triangles) for Y m x c with c <= 64 -- the m x 64 Grams of BRQLP's block
// orthonormalisations.  In the TN kernel the 64 output rows fill half of a 128-row tile (the other
// half multiplies TMA zero fill).  Here one K-major [8 tn][24] smem tile per stage (the TN kernel's
// A layout: conflict-free 16-byte fragment loads) feeds BOTH DMMA operands, and only the 8 x 8
// output tiles on or above the diagonal are formed (36 for c = 64), dealt to the 8 warps.  A CTA
// sums the k-tiles [blockIdx.x kps, ...) into partial slice blockIdx.x (fixed-order reduce after).
constexpr int GR_ST = 4, GR_MAXT = 5;   // stages; output tiles per warp (36 / 8 rounded up)
__global__ void __launch_bounds__(256, 2) gram64_kernel(const __grid_constant__ CUtensorMap mapY, int c,
                                                        int ktiles_total, int kps, double *__restrict__ C,
                                                        int64_t ldc, double *__restrict__ part) {
  const int tn = (c + 7) / 8, ntiles = tn * (tn + 1) / 2;
  const int TILE = tn * 8 * BK;   // doubles per stage
  extern __shared__ __align__(128) unsigned char gsm[];
  double *sY = reinterpret_cast<double *>(gsm);
  uint64_t *full = reinterpret_cast<uint64_t *>(gsm + (size_t)GR_ST * TILE * 8);
  uint64_t *empty = full + GR_ST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r = lane >> 2, cq = lane & 3;
  const int kt0 = blockIdx.x * kps;
  const int nkt = max(0, min(ktiles_total, kt0 + kps) - kt0);
  if (threadIdx.x == 0) {
    for (int st = 0; st < GR_ST; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int it) {
    const int st = it % GR_ST;
    mbar_expect_tx(&full[st], (unsigned)TILE * 8);
    tma_load_2d(sY + (size_t)st * TILE, &mapY, (kt0 + it) * BK, 0, &full[st]);   // box {BK rows, 8 tn cols}
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mapY) : "memory");
    for (int it = 0; it < GR_ST - 1 && it < nkt; ++it) issue(it);
  }
  // this warp's tiles t = warp, warp + 8, ... of the row-major upper triangle (ti <= tj)
  int ti[GR_MAXT], tj[GR_MAXT];
#pragma unroll
  for (int u = 0; u < GR_MAXT; ++u) {
    int t = warp + 8 * u, a = 0;
    while (t >= tn - a && a < tn) { t -= tn - a; ++a; }
    ti[u] = a;
    tj[u] = a + t;   // (a == tn: past the last tile)
  }
  double acc[GR_MAXT][2];
#pragma unroll
  for (int u = 0; u < GR_MAXT; ++u) acc[u][0] = acc[u][1] = 0.0;
  for (int it = 0; it < nkt; ++it) {
    const int st = it % GR_ST;
    if (threadIdx.x == 0 && it + GR_ST - 1 < nkt) {
      if (it >= 1) mbar_wait(&empty[(it - 1) % GR_ST], ((it - 1) / GR_ST) & 1);
      issue(it + GR_ST - 1);
    }
    mbar_wait(&full[st], (it / GR_ST) & 1);
    const double *y = sY + (size_t)st * TILE;
#pragma unroll
    for (int kk = 0; kk < BK / 8; ++kk) {
#pragma unroll
      for (int u = 0; u < GR_MAXT; ++u) {
        if (warp + 8 * u >= ntiles) continue;
        const double2 av = *reinterpret_cast<const double2 *>(y + (ti[u] * 8 + r) * BK + kk * 8 + 2 * cq);
        const double2 bv = *reinterpret_cast<const double2 *>(y + (tj[u] * 8 + r) * BK + kk * 8 + 2 * cq);
        dmma(acc[u][0], acc[u][1], av.x, bv.x);
        dmma(acc[u][0], acc[u][1], av.y, bv.y);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  double *dst = part ? part + (size_t)blockIdx.x * c * c : C;
  const int64_t ld = part ? c : ldc;
#pragma unroll
  for (int u = 0; u < GR_MAXT; ++u) {
    if (warp + 8 * u >= ntiles) continue;
    const int i = ti[u] * 8 + r;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = tj[u] * 8 + 2 * cq + e;
      if (i >= c || j >= c) continue;
      // both triangles (the Cholesky kernel loads the lower one): an off-diagonal tile is mirrored,
      // a diagonal tile writes its own 8 x 8 entries
      dst[i + (size_t)j * ld] = acc[u][e];
      if (ti[u] != tj[u]) dst[j + (size_t)i * ld] = acc[u][e];
    }
  }
}

// Sum of a balanced split's slots: element (i, j) of tile t = (i / BM) ntn + j / bn is the sum,
// in slot order, of the partial tiles of the CTAs first(t) .. last(t) whose runs touch t.  A CTA
// reduces a 32 x 32 block (threads along i: coalesced slot reads); the transposed store goes
// through shared memory so it is coalesced along j.
__global__ void __launch_bounds__(256) bal_reduce_kernel(int M, int N, int bn, int ntn, int ktiles, int units,
                                                         int maxc, const double *__restrict__ part,
                                                         double *__restrict__ C, int64_t ldc, int trans,
                                                         const unsigned *cond, unsigned cond_mask, double alpha,
                                                         double beta) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  __shared__ double sm[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int nbi = (M + 31) / 32, nbj = (N + 31) / 32;
  for (int blk = blockIdx.x; blk < nbi * nbj; blk += gridDim.x) {
    const int i0 = (blk % nbi) * 32, j0 = (blk / nbi) * 32;
    const int i = i0 + tx;
    for (int jj = ty; jj < 32; jj += 8) {
      const int j = j0 + jj;
      double sum = 0.0;
      if (i < M && j < N) {
        const int mt = i / BM, nt = j / bn, t = mt * ntn + nt;
        const int first = (int)(((long long)t * ktiles) / units);
        const int last = (int)(((long long)(t + 1) * ktiles - 1) / units);
        const double *p = part + (size_t)t * maxc * (BM * bn) + (i - mt * BM) + (size_t)(j - nt * bn) * BM;
        const int cnt = last - first + 1;
        // all slot loads in flight first (memory-level parallelism), then the ordered sum
        int q = 0;
        for (; q + 8 <= cnt; q += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = p[(size_t)(q + u) * (BM * bn)];
#pragma unroll
          for (int u = 0; u < 8; ++u) sum += v[u];
        }
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = q + u < cnt ? p[(size_t)(q + u) * (BM * bn)] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q + u < cnt) sum += v[u];
        sum *= alpha;
        if (!trans) C[i + (int64_t)j * ldc] = beta != 0.0 ? fma(beta, C[i + (int64_t)j * ldc], sum) : sum;
      }
      sm[jj][tx] = sum;
    }
    if (trans) {
      __syncthreads();
      const int j = j0 + tx;
      for (int ii = ty; ii < 32; ii += 8) {
        const int ir = i0 + ii;
        if (ir < M && j < N) {
          double *dst = C + j + (int64_t)ir * ldc;
          *dst = beta != 0.0 ? fma(beta, *dst, sm[tx][ii]) : sm[tx][ii];
        }
      }
      __syncthreads();
    }
  }
}

// *out = sum of the n fro slots: thread t sums slots t, t + 256, ... in order, then a fixed tree.
__global__ void __launch_bounds__(256) fro_reduce_kernel(const double *__restrict__ slots, int n, double *out,
                                                         int accumulate) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) s += slots[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = accumulate ? *out + red[0] : red[0];
}

// ------------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw CudaError("cuTensorMapEncodeTiled entry point unavailable");
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 2-D FP64 tensor map over a column-major (rows x cols, ld) matrix with the given box.
bool make_map(CUtensorMap *map, const double *base, int64_t rows, int64_t cols, int64_t ld, int box0, int box1) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld & 1) || rows <= 0 || cols <= 0) return false;
  if (rows >= (1ll << 31) || cols >= (1ll << 31) || (uint64_t)ld * 8 >= (1ull << 40)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box,
                            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

const int kBNs[] = {16, 32, 48, 64, 80, 96, 112, 128, 144};

int choose_bn(int64_t c) {
  if (c <= 16) return 16;
  int best = 144;
  int64_t best_pad = INT64_MAX;
  for (int bn : kBNs) {
    if (bn < 64 && c > 64) continue;  // keep A re-reads bounded for wide outputs
    int64_t pad = ceil_div(c, bn) * bn;
    if (pad < best_pad || (pad == best_pad && bn > best)) {
      best_pad = pad;
      best = bn;
    }
  }
  return best;
}

// Few k-tiles (e.g. Y R^-1 with K = c): the CTA count, not A re-reads, limits the time, so pick
// the BN minimising  waves(tiles) * (ktiles + 3) * BN  (the +3 is the pipeline ramp).
int choose_bn_mk(int64_t M, int64_t c, int64_t ktiles, int num_sms) {
  if (ktiles > 16) return choose_bn(c);
  int best = choose_bn(c);
  double best_t = 1e300;
  for (int bn : kBNs) {
    const int64_t tiles = ceil_div(M, BM) * ceil_div(c, bn);
    const double t = (double)ceil_div(tiles, num_sms) * (double)(ktiles + 3) * bn;
    if (t < best_t * 0.999 || (t <= best_t * 1.001 && bn > best)) {
      best_t = t;
      best = bn;
    }
  }
  return best;
}

// Output columns covered by tiles of two widths when one width leaves padding: the first c1 = t1 bn1
// columns in one launch, the remaining cc - c1 in a second launch with one tile of width bn2 >= the
// remainder (e.g. l = 528 -> 4 x 112 + 80 instead of 5 x 112 = 560; l = 272 -> 144 + 128 instead of
// 2 x 144).  Only for long-K passes (the A-passes), where the padded columns cost their full DMMA
// work; returns c1 = 0 when one width is as good.
struct ColSplit {
  int64_t c1 = 0;
  int bn1 = 0, bn2 = 0;
};
bool env_off(const char *name) {
  const char *e = getenv(name);
  return e && e[0] == '0';
}

ColSplit choose_colsplit(int64_t cc, int64_t ktiles) {
  ColSplit best;
  static const bool off = env_off("RQLP_GEMM_COLSPLIT");   // measurement switch
  if (off || ktiles <= 16 || cc <= 64) return best;
  const int bn = choose_bn(cc);
  const int64_t pad1 = ceil_div(cc, bn) * bn - cc;
  if (pad1 * 50 < cc) return best;   // < 2 % padding: not worth a second launch
  int64_t best_pad = pad1;
  for (int b1 : kBNs) {
    if (b1 < 64) continue;
    const int64_t t1 = cc / b1;
    const int64_t c1 = t1 * b1, rem = cc - c1;
    if (t1 < 1 || rem <= 0) continue;
    for (int b2 : kBNs) {
      if (b2 < rem || (b2 < 64 && rem > 64)) continue;
      const int64_t pad = b2 - rem;
      // equal padding: the wider first width.  RQLP_COLSPLIT_PREFER=w (measurement switch) puts width w
      // first: C4's sketch as 3 x 128 + 144 instead of 3 x 144 + 96 measured the same inside the
      // power-capped step (128.6 / 130.8 ms against 129.2 / 130.1 ms)
      static const int prefer = [] { const char *e = getenv("RQLP_COLSPLIT_PREFER"); return e ? atoi(e) : 0; }();
      auto rank = [&](int b) { return b == prefer ? 1000 : b; };
      if (pad < best_pad || (pad == best_pad && best.c1 > 0 && rank(b1) > rank(best.bn1))) {
        best_pad = pad;
        best.c1 = c1;
        best.bn1 = b1;
        best.bn2 = b2;
      }
      break;   // the smallest b2 covering the remainder
    }
  }
  return best;
}

// Split-K: minimise the modelled time  waves(T) * ceil(ktiles / S) * t_ktile
//                                      + (S > 1) * (2 S M N 8 bytes / HBM + reduce launch)
// with T = tiles * S CTAs (1 CTA per SM), t_ktile = 128 BN 24 2 flop / (DMMA peak per SM).
int choose_splits(int64_t tiles, int64_t ktiles, int num_sms, size_t partial_cap_elems, int64_t out_elems, int bn,
                  double *t_out = nullptr, int occ = 1) {
  // occ CTAs per SM: num_sms x occ concurrent CTAs, each at 1/occ of the SM's DMMA rate
  num_sms *= occ;
  const double t_ktile = occ * 128.0 * bn * BK * 2.0 / (37.0e12 / 148.0);   // s
  const double hbm = 6.0e12;                                           // B/s
  int best = 1;
  double best_t = 1e300;
  for (int s = 1; s <= 2 * num_sms; ++s) {
    if (s > 1 && (size_t)s * out_elems > partial_cap_elems) break;
    if (s > 1 && ktiles / s < 2) break;
    const int64_t T = tiles * s;
    double t = (double)ceil_div(T, num_sms) * (double)ceil_div(ktiles, s) * t_ktile;
    if (s > 1) t += 2.0 * s * (double)out_elems * 8.0 / hbm + 4e-6;
    if (t < best_t * 0.995) {
      best_t = t;
      best = s;
    }
  }
  // the chosen split's time with the pipeline ramp (3 k-tiles per wave), comparable to the
  // balanced model below
  if (t_out) *t_out = best_t + (double)ceil_div(tiles * best, num_sms) * 3.0 * t_ktile;
  return best;
}

// Balanced split (see gemm_tma_kernel): units = ceil(tiles ktiles / #SMs) k-tiles per CTA.  Returns
// the run length when its modelled time beats the split-K time t_split (and the slots fit), else 0.
struct BalPlan {
  int units = 0, maxc = 0;
  int occ = 1;   // CTAs per SM the split models assumed (gemm_occ): the launch uses the same
};
BalPlan choose_balanced(int64_t tiles, int64_t ktiles, int num_sms, size_t partial_cap_elems, int bn, double t_split,
                        int occ = 1) {
  BalPlan p;
  num_sms *= occ;
  const int64_t total = tiles * ktiles;
  if (tiles >= num_sms || total < 4 * (int64_t)num_sms || total >= (1ll << 31)) return p;
  const int64_t U = ceil_div(total, num_sms);
  int64_t maxc = 0;
  for (int64_t t = 0; t < tiles; ++t) maxc = std::max<int64_t>(maxc, ((t + 1) * ktiles - 1) / U - (t * ktiles) / U + 1);
  if ((size_t)(tiles * maxc * BM * bn) > partial_cap_elems) return p;
  const double t_ktile = occ * 128.0 * bn * BK * 2.0 / (37.0e12 / 148.0);
  const double hbm = 6.0e12;
  const double t = (double)(U + 3) * t_ktile + 2.0 * (double)(tiles + num_sms) * BM * bn * 8.0 / hbm + 4e-6;
  if (t < 0.9 * t_split) {  // measured: a 5% gain at C2 (c = 110), a loss at c <= 40
    p.units = (int)U;
    p.maxc = (int)maxc;
  }
  return p;
}

template <int BN, int MODE, bool FRO, int OCC>
void launch_bn_o(Ctx &c, const CUtensorMap &ma, const CUtensorMap &mb, int M, int N, int ktiles, int S, double *C,
                 int64_t ldc, bool trans, double *part, const unsigned *cond, unsigned mask, int tri, BalPlan bp,
                 const FroSpec *fro, double alpha, double beta) {
  constexpr int NST = OCC == 2 ? 3 : STAGES;
  constexpr int A_BYTES = MODE == 0 ? A_TILE_BYTES_NN : A_TILE_BYTES_TN;
  constexpr int SMEM = NST * (A_BYTES + BN * BK * 8) + 2 * NST * 8;
  smem_attr((const void *)gemm_tma_kernel<BN, MODE, FRO, OCC>, SMEM);
  double *fslots = fro ? fro->slots : nullptr;
  auto fro_finish = [&](int64_t nctas) {
    if (!fro) return;
    fro_reduce_kernel<<<1, 256, 0, c.stream>>>(fro->slots, (int)nctas, fro->out, fro->accumulate ? 1 : 0);
    RQLP_LAUNCHED(c);
  };
  if (bp.units > 0) {
    const int ntn = (int)ceil_div(N, BN);
    const int64_t total = (int64_t)ktiles * ntn * ceil_div(M, BM);
    const unsigned ctas = (unsigned)ceil_div(total, bp.units);
    gemm_tma_kernel<BN, MODE, FRO, OCC><<<ctas, (NCONS + (FRO ? 1 : 0)) * 32, SMEM, c.stream>>>(ma, mb, M, N, ktiles, 0, C, ldc, trans ? 1 : 0,
                                                                     part, cond, mask, 0, bp.units, ntn, bp.maxc,
                                                                     fslots, alpha, beta);
    RQLP_LAUNCHED(c);
    fro_finish(ctas);
    const int grid = (int)std::min<int64_t>(ceil_div(M, 32) * ceil_div(N, 32), (int64_t)c.num_sms * 8);
    bal_reduce_kernel<<<std::max(grid, 1), 256, 0, c.stream>>>(M, N, BN, ntn, ktiles, bp.units, bp.maxc, part, C, ldc,
                                                                trans ? 1 : 0, cond, mask, alpha, beta);
    RQLP_LAUNCHED(c);
    return;
  }
  int kps = (int)ceil_div(ktiles, S);
  S = (int)ceil_div(ktiles, kps);
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)S);
  gemm_tma_kernel<BN, MODE, FRO, OCC><<<grid, (NCONS + (FRO ? 1 : 0)) * 32, SMEM, c.stream>>>(ma, mb, M, N, ktiles, kps, C, ldc,
                                                                       trans ? 1 : 0, S > 1 ? part : nullptr, cond,
                                                                       mask, tri, 0, 1, 1, fslots, alpha, beta);
  RQLP_LAUNCHED(c);
  fro_finish((int64_t)grid.x * grid.y * grid.z);
  if (S > 1) launch_reduce(c, M, N, S, part, alpha, beta, C, ldc, trans, cond, mask);
}

template <int BN, int MODE, bool FRO>
void launch_bn_t(Ctx &c, const CUtensorMap &ma, const CUtensorMap &mb, int M, int N, int ktiles, int S, double *C,
                 int64_t ldc, bool trans, double *part, const unsigned *cond, unsigned mask, int tri, BalPlan bp,
                 const FroSpec *fro, double alpha, double beta) {
  if constexpr (BN <= 64 && !FRO) {
    if (bp.occ == 2) {
      launch_bn_o<BN, MODE, false, 2>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha,
                                      beta);
      return;
    }
  }
  launch_bn_o<BN, MODE, FRO, 1>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta);
}

template <int BN, int MODE>
void launch_bn(Ctx &c, const CUtensorMap &ma, const CUtensorMap &mb, int M, int N, int ktiles, int S, double *C,
               int64_t ldc, bool trans, double *part, const unsigned *cond, unsigned mask, int tri, BalPlan bp,
               const FroSpec *fro, double alpha, double beta) {
  if constexpr (MODE == 0 && BN <= FRO_MAX_BN) {
    if (fro) {
      launch_bn_t<BN, 0, true>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta);
      return;
    }
  }
  launch_bn_t<BN, MODE, false>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, nullptr, alpha,
                               beta);
}

template <int MODE>
void dispatch(Ctx &c, int bn, const CUtensorMap &ma, const CUtensorMap &mb, int M, int N, int ktiles, int S, double *C,
              int64_t ldc, bool trans, double *part, const unsigned *cond, unsigned mask, int tri, BalPlan bp,
              const FroSpec *fro, double alpha, double beta) {
  switch (bn) {
    case 16: launch_bn<16, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta); break;
    case 32: launch_bn<32, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta); break;
    case 48: launch_bn<48, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta); break;
    case 64: launch_bn<64, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta); break;
    case 80: launch_bn<80, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta); break;
    case 96: launch_bn<96, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta); break;
    case 112: launch_bn<112, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta); break;
    case 128: launch_bn<128, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta); break;
    default: launch_bn<144, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, tri, bp, fro, alpha, beta); break;
  }
}

bool balanced_disabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RQLP_GEMM_BALANCED");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

bool tma_disabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RQLP_DISABLE_TMA");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

}  // namespace

size_t gemm_tma_partials_needed(int64_t m, int64_t cc, int64_t k, int num_sms) {
  // upper bound over both modes for the shapes (m, cc, k) and (k, cc, m), including the two
  // launches of a two-width column split
  size_t best = 0;
  auto need = [&](int64_t M, int64_t cols, int64_t ktiles, int bn) {
    int64_t tiles = ceil_div(M, BM) * ceil_div(cols, bn);
    double ts = 0.0;
    const int occ = gemm_occ(bn, false, tiles, ktiles);   // the partials of both occupancies (upper bound)
    for (int o = 1; o <= occ; ++o) {
      int S = choose_splits(tiles, ktiles, num_sms, (size_t)1 << 62, M * cols, bn, &ts, o);
      if (S > 1) best = std::max(best, (size_t)S * M * cols);
      BalPlan bp = choose_balanced(tiles, ktiles, num_sms, (size_t)1 << 62, bn, ts, o);
      if (bp.units > 0) best = std::max(best, (size_t)tiles * bp.maxc * BM * bn);
    }
  };
  for (int mode = 0; mode < 2; ++mode) {
    int64_t M = mode == 0 ? m : k, K = mode == 0 ? k : m;
    int64_t ktiles = ceil_div(K, BK);
    need(M, cc, ktiles, choose_bn_mk(M, cc, ktiles, num_sms));
    const ColSplit cs = choose_colsplit(cc, ktiles);
    if (cs.c1 > 0) {
      need(M, cs.c1, ktiles, cs.bn1);
      need(M, cc - cs.c1, ktiles, cs.bn2);
    }
    const int64_t c1 = (cc / FRO_MAX_BN) * FRO_MAX_BN;   // the ||A||^2-carrying split of the sketch
    if (mode == 0 && c1 > 0) {
      need(M, c1, ktiles, FRO_MAX_BN);
      if (c1 < cc) need(M, cc - c1, ktiles, choose_bn_mk(M, cc - c1, ktiles, num_sms));
    }
  }
  return best;
}

bool gemm_nn_tma_bn(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X,
                    int64_t ldx, double *Y, int64_t ldy, double *partials, size_t partial_elems, const unsigned *cond,
                    unsigned cond_mask, int tri, const FroSpec *fro, int bn, double alpha, double beta);

bool gemm_nn_tma(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X, int64_t ldx,
                 double *Y, int64_t ldy, double *partials, size_t partial_elems, const unsigned *cond,
                 unsigned cond_mask, int tri, const FroSpec *fro, double alpha, double beta) {
  if (tma_disabled() || m < 1 || cc < 1 || k < 1) return false;
  static const bool fro_off = env_off("RQLP_FRO_FUSED");   // measurement switch: separate ||A||^2 pass
  if (fro && (cond || tri || fro_off)) return false;
  // measurement switch RQLP_NN_SLAB=w: a wide long-K pass as column slabs of w (one launch each)
  static const int slab = [] { const char *e = getenv("RQLP_NN_SLAB"); return e ? atoi(e) : 0; }();
  if (slab >= 16 && !fro && tri == 0 && !cond && cc > slab && ceil_div(k, BK) > 16) {
    for (int64_t c0 = 0; c0 < cc; c0 += slab) {
      const int64_t w = std::min<int64_t>(slab, cc - c0);
      if (!gemm_nn_tma(c, m, w, k, A, lda, X + c0 * ldx, ldx, Y + c0 * ldy, ldy, partials, partial_elems, nullptr, 0,
                       0, nullptr, alpha, beta))
        throw CudaError("gemm_nn_tma: slab not launchable");
    }
    return true;
  }
  const ColSplit cs = tri == 0 ? choose_colsplit(cc, ceil_div(k, BK)) : ColSplit();
  if (cs.c1 > 0) {
    // the ||A||^2 goes with one column range (each reads all of A), one whose width can carry it
    const FroSpec *f1 = nullptr, *f2 = nullptr;
    if (fro) {
      if (cs.bn2 <= FRO_MAX_BN) f2 = fro;
      else if (cs.bn1 <= FRO_MAX_BN) f1 = fro;
      else return false;
    }
    CUtensorMap probe;   // both column ranges must be TMA-addressable, else one width
    if (make_map(&probe, X + cs.c1 * ldx, k, cc - cs.c1, ldx, BK, cs.bn2) &&
        gemm_nn_tma_bn(c, m, cs.c1, k, A, lda, X, ldx, Y, ldy, partials, partial_elems, cond, cond_mask, 0, f1,
                       cs.bn1, alpha, beta)) {
      if (!gemm_nn_tma_bn(c, m, cc - cs.c1, k, A, lda, X + cs.c1 * ldx, ldx, Y + cs.c1 * ldy, ldy, partials,
                          partial_elems, cond, cond_mask, 0, f2, cs.bn2, alpha, beta)) {
        // (only the ||A||^2 slot capacity can refuse it) plain range + a separate ||A||^2 pass
        if (!f2 || !gemm_nn_tma_bn(c, m, cc - cs.c1, k, A, lda, X + cs.c1 * ldx, ldx, Y + cs.c1 * ldy, ldy, partials,
                                   partial_elems, cond, cond_mask, 0, nullptr, cs.bn2, alpha, beta))
          throw CudaError("gemm_nn_tma: second column range not launchable");
        fro2_accumulate(c, m, k, A, lda, f2->slots, f2->out, !f2->accumulate);
      }
      return true;
    }
    if (f1) return false;   // (the first range was not launched)
  }
  const int bn = choose_bn_mk(m, cc, ceil_div(k, BK), c.num_sms);
  if (fro && bn > FRO_MAX_BN) {
    // every width of the plan is too wide for the ||A||^2 warp: the first floor(cc / 96) * 96 columns
    // in 96-wide tiles carrying it, the rest as a plain pass (C2: 96 + 14, C3: 2 x 96 + 80 -- no
    // padded columns; the extra A read of a compute-bound pass is hidden)
    const int64_t c1 = (cc / FRO_MAX_BN) * FRO_MAX_BN;
    if (!gemm_nn_tma_bn(c, m, c1, k, A, lda, X, ldx, Y, ldy, partials, partial_elems, cond, cond_mask, 0, fro,
                        FRO_MAX_BN, alpha, beta))
      return false;
    if (c1 < cc && !gemm_nn_tma(c, m, cc - c1, k, A, lda, X + c1 * ldx, ldx, Y + c1 * ldy, ldy, partials,
                                partial_elems, cond, cond_mask, 0, nullptr, alpha, beta))
      gemm_generic_ex(c, false, false, m, cc - c1, k, alpha, A, lda, X + c1 * ldx, ldx, beta, Y + c1 * ldy, ldy,
                      partials, partial_elems, false, cond, cond_mask);
    return true;
  }
  return gemm_nn_tma_bn(c, m, cc, k, A, lda, X, ldx, Y, ldy, partials, partial_elems, cond, cond_mask, tri, fro, bn,
                        alpha, beta);
}

bool gemm_nn_tma_bn(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X,
                    int64_t ldx, double *Y, int64_t ldy, double *partials, size_t partial_elems, const unsigned *cond,
                    unsigned cond_mask, int tri, const FroSpec *fro, int bn, double alpha, double beta) {
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, m, k, lda, LDA_NN, BK)) return false;
  if (!make_map(&mb, X, k, cc, ldx, BK, bn)) return false;
  int64_t ktiles = ceil_div(k, BK);
  int64_t tiles = ceil_div(m, BM) * ceil_div(cc, bn);
  double ts = 0.0;
  const int occ = gemm_occ(bn, fro != nullptr, tiles, ktiles);
  int S = choose_splits(tiles, ktiles, c.num_sms, partials ? partial_elems : 0, m * cc, bn, &ts, occ);
  BalPlan bp;
  if (tri == 0 && partials && !balanced_disabled())
    bp = choose_balanced(tiles, ktiles, c.num_sms, partial_elems, bn, ts, occ);
  bp.occ = occ;
  if (fro) {   // the slots needed by this launch configuration must fit
    const int64_t ctas = bp.units > 0 ? ceil_div(tiles * ktiles, bp.units)
                                      : tiles * ceil_div(ktiles, ceil_div(ktiles, S));
    if (ctas > fro->cap) return false;
  }
  dispatch<0>(c, bn, ma, mb, (int)m, (int)cc, (int)ktiles, S, Y, ldy, false, partials, cond, cond_mask, tri, bp, fro,
              alpha, beta);
  return true;
}

bool gemm_tn_tma_bn(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *V,
                    int64_t ldv, double *Z, int64_t ldz, bool trans_out, double *partials, size_t partial_elems,
                    const unsigned *cond, unsigned cond_mask, int tri, int bn, double alpha, double beta);

bool gram64(Ctx &c, int64_t m, int64_t cc, const double *Y, int64_t ldy, double *G, int64_t ldg, double *partials,
            size_t partial_elems) {
  CUtensorMap my;
  const int tn = (int)ceil_div(cc, 8);
  if (!make_map(&my, Y, m, cc, ldy, BK, tn * 8)) return false;
  const int64_t ktiles = ceil_div(m, BK);
  // slices: two CTAs per SM when each keeps >= 8 k-tiles, bounded by the partial buffer
  int64_t S = std::min<int64_t>(2 * c.num_sms, std::max<int64_t>(1, ktiles / 8));
  if (!partials) S = 1;
  S = std::min<int64_t>(S, std::max<int64_t>(1, (int64_t)(partial_elems / (size_t)(cc * cc))));
  const int kps = (int)ceil_div(ktiles, S);
  S = ceil_div(ktiles, kps);
  const size_t smem = (size_t)GR_ST * tn * 8 * BK * 8 + 2 * GR_ST * 8;
  smem_attr((const void *)gram64_kernel, (int)smem);
  gram64_kernel<<<(unsigned)S, 256, smem, c.stream>>>(my, (int)cc, (int)ktiles, kps, G, ldg, S > 1 ? partials : nullptr);
  RQLP_LAUNCHED(c);
  if (S > 1) launch_reduce(c, cc, cc, (int)S, partials, 1.0, 0.0, G, ldg, false, nullptr, 0);
  return true;
}

bool gemm_tn_tma(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *V, int64_t ldv,
                 double *Z, int64_t ldz, bool trans_out, double *partials, size_t partial_elems, const unsigned *cond,
                 unsigned cond_mask, int tri, double alpha, double beta) {
  if (tma_disabled() || m < 1 || cc < 1 || k < 1) return false;
  // a Gram of 17..64 columns: the dedicated kernel (measured: 262144 x 64 CholeskyQR2 473 -> 321 us,
  // C4 554.9 -> 551.1 ms; 16 columns: the TN kernel is as fast)
  static const bool gram_off = env_off("RQLP_GRAM64");   // measurement switch
  if (tri == 1 && A == V && lda == ldv && k == cc && cc > 16 && cc <= 64 && !cond && !trans_out && alpha == 1.0 &&
      beta == 0.0 && !gram_off && gram64(c, m, cc, A, lda, Z, ldz, partials, partial_elems))
    return true;
  const ColSplit cs = tri == 0 ? choose_colsplit(cc, ceil_div(m, BK)) : ColSplit();
  if (cs.c1 > 0) {
    CUtensorMap probe;
    double *Z2 = trans_out ? Z + cs.c1 : Z + cs.c1 * ldz;
    if (make_map(&probe, V + cs.c1 * ldv, m, cc - cs.c1, ldv, BK, cs.bn2) &&
        gemm_tn_tma_bn(c, m, cs.c1, k, A, lda, V, ldv, Z, ldz, trans_out, partials, partial_elems, cond, cond_mask, 0,
                       cs.bn1, alpha, beta)) {
      if (!gemm_tn_tma_bn(c, m, cc - cs.c1, k, A, lda, V + cs.c1 * ldv, ldv, Z2, ldz, trans_out, partials,
                          partial_elems, cond, cond_mask, 0, cs.bn2, alpha, beta))
        throw CudaError("gemm_tn_tma: second column range not launchable");
      return true;
    }
  }
  return gemm_tn_tma_bn(c, m, cc, k, A, lda, V, ldv, Z, ldz, trans_out, partials, partial_elems, cond, cond_mask, tri,
                        choose_bn_mk(k, cc, ceil_div(m, BK), c.num_sms), alpha, beta);
}

bool gemm_tn_tma_bn(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *V,
                    int64_t ldv, double *Z, int64_t ldz, bool trans_out, double *partials, size_t partial_elems,
                    const unsigned *cond, unsigned cond_mask, int tri, int bn, double alpha, double beta) {
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, m, k, lda, BK, BM)) return false;
  if (!make_map(&mb, V, m, cc, ldv, BK, bn)) return false;
  int64_t ktiles = ceil_div(m, BK);
  int64_t tiles = ceil_div(k, BM) * ceil_div(cc, bn);
  if (tri == 1) {  // only tiles reaching the upper triangle do work
    tiles = 0;
    for (int64_t mt = 0; mt < ceil_div(k, BM); ++mt)
      for (int64_t nt = 0; nt < ceil_div(cc, bn); ++nt) tiles += (mt * BM < nt * bn + bn) ? 1 : 0;
  }
  double ts = 0.0;
  const int occ = gemm_occ(bn, false, tiles, ktiles);
  int S = choose_splits(tiles, ktiles, c.num_sms, partials ? partial_elems : 0, k * cc, bn, &ts, occ);
  BalPlan bp;
  if (tri == 0 && partials && !balanced_disabled())
    bp = choose_balanced(tiles, ktiles, c.num_sms, partial_elems, bn, ts, occ);
  bp.occ = occ;
  dispatch<1>(c, bn, ma, mb, (int)k, (int)cc, (int)ktiles, S, Z, ldz, trans_out, partials, cond, cond_mask, tri, bp,
              nullptr, alpha, beta);
  return true;
}

}  // namespace rqlpk
