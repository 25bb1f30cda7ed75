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

namespace {

constexpr int BM = 128, BK = 24, STAGES = 4, NCONS = 8;
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

// Hybrid data-parallel + Stream-K schedule (SK; gridDim.x = G persistent CTAs, 1 per SM).
// The first dp_waves * G tiles are whole-tile work in classic order (tile = wave * G + cta, so
// concurrent CTAs share A panels in L2); the remaining sk_tiles tiles form an iteration space
// sk_tiles x ktiles cut into G equal contiguous ranges.  A Stream-K tile covered by one CTA is
// stored directly; a tile split across CTAs c_lo..c_hi has each segment written to its CTA's
// fragment-native slot (slot 0: the CTA's first SK tile, slot 1: its last), and
// streamk_fixup_kernel sums the slots in the fixed order c_lo..c_hi (deterministic for a G).
struct SkArgs {
  int G = 0;              // 0: classic grid (n-tiles, m-tiles, split-K slices)
  int tiles_n = 0;
  int dp_waves = 0;
  int sk_tiles = 0;
  int64_t iters = 0;      // sk_tiles * ktiles
  double *slots = nullptr;
};

__host__ __device__ __forceinline__ int sk_cta_of(int64_t it, int64_t T, int G) { return (int)(((it + 1) * G - 1) / T); }
__host__ __device__ __forceinline__ int64_t sk_start(int c, int64_t T, int G) { return (int64_t)c * T / G; }

// MODE 0 = NN, 1 = TN.  Output element (i, j) of the (M x N) product goes to
//   part (split-K slice, M x N contiguous)  or  C[i + j ldc]  or (trans) C[j + i ldc].
template <int BN, int MODE>
__global__ void __launch_bounds__(NCONS * 32, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M, int N,
                    int ktiles_total, int ktiles_per_split, double *__restrict__ C, int64_t ldc, int trans,
                    double *__restrict__ part, const unsigned *cond, unsigned cond_mask, SkArgs sk) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  constexpr int A_BYTES = MODE == 0 ? A_TILE_BYTES_NN : A_TILE_BYTES_TN;
  constexpr int B_BYTES = BN * BK * 8;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int NB = BN / 16;  // 8-col fragments per warp (warp tile 32 x BN/2)
  constexpr int FRAG = 4 * NB * 2;  // accumulator doubles per thread
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = ktiles_total;
  // this CTA's iteration sequence g = 0 .. nloc-1 and a cursor (tile, kt, dp tiles left)
  int64_t sk_it0 = 0;
  int nloc, tile0, kt0, dp0 = 0;
  if (sk.G) {
    sk_it0 = sk_start(blockIdx.x, sk.iters, sk.G);
    const int nsk = (int)(sk_start(blockIdx.x + 1, sk.iters, sk.G) - sk_it0);
    dp0 = sk.dp_waves;
    nloc = dp0 * K + nsk;
    if (dp0 > 0) { tile0 = blockIdx.x; kt0 = 0; }
    else { tile0 = sk.dp_waves * sk.G + (int)(sk_it0 / K); kt0 = (int)(sk_it0 % K); }
  } else {
    tile0 = 0;
    kt0 = blockIdx.z * ktiles_per_split;
    nloc = min(K, kt0 + ktiles_per_split) - kt0;
  }
  struct Cursor { int tile, kt, dp; };
  auto advance = [&](Cursor &u) {
    if (++u.kt < K) return;
    u.kt = 0;
    if (u.dp > 0) {
      if (--u.dp > 0) { u.tile += sk.G; return; }
      u.tile = sk.dp_waves * sk.G + (int)(sk_it0 / K);   // switch to the Stream-K range
      u.kt = (int)(sk_it0 % K);
      return;
    }
    ++u.tile;
  };
  auto tile_origin = [&](int tile, int &m0, int &n0) {
    if (sk.G) {
      m0 = (tile / sk.tiles_n) * BM;
      n0 = (tile % sk.tiles_n) * BN;
    } else {
      m0 = blockIdx.y * BM;
      n0 = blockIdx.x * BN;
    }
  };
  Cursor pc{tile0, kt0, dp0};  // producer cursor (thread 0)

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ---------------- producer role (thread 0 of warp 0): TMA slabs STAGES-1 iterations ahead
  auto issue = [&](int g) {
    const int s = g % STAGES;
    unsigned char *sa = smem + s * STAGE_BYTES;
    unsigned char *sb = sa + A_BYTES;
    int m0, n0;
    tile_origin(pc.tile, m0, n0);
    const int kk = pc.kt * BK;
    advance(pc);
    mbar_expect_tx(&full[s], (MODE == 0 ? BK * LDA_NN * 8 : A_TILE_BYTES_TN) + B_BYTES);
    if (MODE == 0) tma_load_2d(sa, &mapA, m0, kk, &full[s]);   // A box {BM+2, BK} at (m0, k)
    else tma_load_2d(sa, &mapA, kk, m0, &full[s]);             // A box {BK, BM} at (k = row offset, col)
    tma_load_2d(sb, &mapB, kk, n0, &full[s]);                  // B box {BK, BN} at (k, n0)
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mapB) : "memory");
    for (int g = 0; g < STAGES - 1 && g < nloc; ++g) issue(g);
  }

  // ---------------- consumers: 8 warps, 4 (M) x 2 (N), warp tile 32 x BN/2
  const int wm = warp & 3, wn = warp >> 2;
  const int r = lane >> 2, cq = lane & 3;
  double acc[4][NB][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // epilogue of one (tile, segment): fragment (mb, nb) holds out[row][col], out[row][col+1]
  auto store = [&](int m0, int n0, int zslice) {
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) {
      const int i = m0 + wm * 32 + mb * 8 + r;
      if (i >= M) continue;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int j = n0 + wn * (BN / 2) + nb * 8 + 2 * cq;
        if (part) {
          double *dst = part + (size_t)zslice * M * N;
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
  };

  Cursor cc{tile0, kt0, dp0};  // consumer cursor
  for (int g = 0; g < nloc; ++g) {
    const int s = g % STAGES;
    if (threadIdx.x == 0 && g + STAGES - 1 < nloc) {
      // refill the slot consumed at iteration g-1 once every warp has released it
      if (g >= 1) mbar_wait(&empty[(g - 1) % STAGES], ((g - 1) / STAGES) & 1);
      issue(g + STAGES - 1);
    }
    mbar_wait(&full[s], (g / STAGES) & 1);
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

    if (!sk.G) continue;
    // ---- end of a tile segment?
    const int tile = cc.tile;
    const bool in_dp = cc.dp > 0;
    const bool seg_end = (cc.kt == K - 1) || (g == nloc - 1);
    advance(cc);
    if (!seg_end) continue;
    int m0, n0;
    tile_origin(tile, m0, n0);
    bool whole = in_dp;
    int slot = 0;
    if (!in_dp) {
      const int st = tile - sk.dp_waves * sk.G;  // Stream-K tile index
      const int64_t tb = (int64_t)st * K;
      whole = sk_cta_of(tb, sk.iters, sk.G) == sk_cta_of(tb + K - 1, sk.iters, sk.G);
      slot = (st == (int)(sk_it0 / K)) ? 0 : 1;
    }
    if (whole) {
      store(m0, n0, 0);
    } else {
      double *my = sk.slots + ((int64_t)blockIdx.x * 2 + slot) * (FRAG * NCONS * 32) + threadIdx.x;
      int e = 0;
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int h = 0; h < 2; ++h, ++e) my[e * (NCONS * 32)] = acc[mb][nb][h];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }
  if (!sk.G) store(blockIdx.y * BM, blockIdx.x * BN, blockIdx.z);
}

// Fix-up of the split Stream-K tiles: block (st, e) sums fragment element e of all 256 threads
// over the segments c_lo..c_hi in that fixed order and stores it like the GEMM epilogue would.
__global__ void streamk_fixup_kernel(int BN, int M, int N, int K, SkArgs sk, double *C, int64_t ldc, int trans,
                                     const unsigned *cond, unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  const int st = blockIdx.x, e = blockIdx.y;
  const int64_t tb = (int64_t)st * K;
  const int c_lo = sk_cta_of(tb, sk.iters, sk.G), c_hi = sk_cta_of(tb + K - 1, sk.iters, sk.G);
  if (c_lo == c_hi) return;
  const int NB = BN / 16, FRAG = 8 * NB;
  const int tid = threadIdx.x;
  double sum = 0.0;
  for (int c = c_lo; c <= c_hi; ++c) {
    const int slot = (st == (int)(sk_start(c, sk.iters, sk.G) / K)) ? 0 : 1;
    sum += sk.slots[((int64_t)c * 2 + slot) * (FRAG * NCONS * 32) + (int64_t)e * (NCONS * 32) + tid];
  }
  const int tile = sk.dp_waves * sk.G + st;
  const int m0 = (tile / sk.tiles_n) * BM, n0 = (tile % sk.tiles_n) * BN;
  const int warp = tid >> 5, lane = tid & 31, wm = warp & 3, wn = warp >> 2, r = lane >> 2, cq = lane & 3;
  const int h = e & 1, nb = (e >> 1) % NB, mb = (e >> 1) / NB;
  const int i = m0 + wm * 32 + mb * 8 + r;
  const int j = n0 + wn * (BN / 2) + nb * 8 + 2 * cq + h;
  if (i >= M || j >= N) return;
  if (trans) C[j + (int64_t)i * ldc] = sum;
  else C[i + (int64_t)j * ldc] = sum;
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

// Split-K: minimise the modelled time  waves(T) * ceil(ktiles / S) * t_ktile
//                                      + (S > 1) * (2 S M N 8 bytes / HBM + reduce launch)
// with T = tiles * S CTAs (1 CTA per SM), t_ktile = 128 BN 24 2 flop / (DMMA peak per SM).
int choose_splits(int64_t tiles, int64_t ktiles, int num_sms, size_t partial_cap_elems, int64_t out_elems, int bn) {
  const double t_ktile = 128.0 * bn * BK * 2.0 / (37.0e12 / 148.0);   // s
  const double hbm = 6.0e12;                                           // B/s
  int best = 1;
  double best_t = 1e300;
  for (int s = 1; s <= 64; ++s) {
    if (s > 1 && (size_t)s * out_elems > partial_cap_elems) break;
    if (s > 1 && ktiles / s < 4) break;
    const int64_t T = tiles * s;
    double t = (double)ceil_div(T, num_sms) * (double)ceil_div(ktiles, s) * t_ktile;
    if (s > 1) t += 2.0 * s * (double)out_elems * 8.0 / hbm + 4e-6;
    if (t < best_t * 0.995) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

// Stream-K (hybrid) is used when the classic grid would leave SMs idle (tiles not a multiple
// of the SM count) and there is enough work per CTA (>= 4 k-tiles each).
bool use_streamk(int64_t tiles, int64_t ktiles, int num_sms) {
  if (tiles * ktiles < 4 * (int64_t)num_sms) return false;
  return tiles % num_sms != 0;
}

size_t streamk_elems(int num_sms, int bn) { return (size_t)2 * num_sms * BM * bn; }

template <int BN, int MODE>
void launch_bn(Ctx &c, const CUtensorMap &ma, const CUtensorMap &mb, int M, int N, int ktiles, int S, double *C,
               int64_t ldc, bool trans, double *part, const unsigned *cond, unsigned mask, bool sk_on) {
  constexpr int A_BYTES = MODE == 0 ? A_TILE_BYTES_NN : A_TILE_BYTES_TN;
  constexpr int SMEM = STAGES * (A_BYTES + BN * BK * 8) + 2 * STAGES * 8;
  static bool attr = false;
  if (!attr) {
    RQLP_CUDA(cudaFuncSetAttribute(gemm_tma_kernel<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr = true;
  }
  SkArgs sk;
  if (sk_on) {
    const int tiles_n = (int)ceil_div(N, BN), tiles = tiles_n * (int)ceil_div(M, BM);
    sk.G = c.num_sms;
    sk.tiles_n = tiles_n;
    sk.dp_waves = tiles >= 2 * sk.G ? tiles / sk.G - 1 : 0;
    sk.sk_tiles = tiles - sk.dp_waves * sk.G;
    sk.iters = (int64_t)sk.sk_tiles * ktiles;
    sk.slots = part;
    gemm_tma_kernel<BN, MODE><<<sk.G, NCONS * 32, SMEM, c.stream>>>(ma, mb, M, N, ktiles, ktiles, C, ldc,
                                                                   trans ? 1 : 0, nullptr, cond, mask, sk);
    RQLP_LAUNCHED(c);
    dim3 fg((unsigned)sk.sk_tiles, (unsigned)(8 * (BN / 16)));
    streamk_fixup_kernel<<<fg, NCONS * 32, 0, c.stream>>>(BN, M, N, ktiles, sk, C, ldc, trans ? 1 : 0, cond, mask);
    RQLP_LAUNCHED(c);
    return;
  }
  int kps = (int)ceil_div(ktiles, S);
  S = (int)ceil_div(ktiles, kps);
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)S);
  gemm_tma_kernel<BN, MODE><<<grid, NCONS * 32, SMEM, c.stream>>>(ma, mb, M, N, ktiles, kps, C, ldc,
                                                                       trans ? 1 : 0, S > 1 ? part : nullptr, cond,
                                                                       mask, sk);
  RQLP_LAUNCHED(c);
  if (S > 1) launch_reduce(c, M, N, S, part, 1.0, 0.0, C, ldc, trans, cond, mask);
}

template <int MODE>
void dispatch(Ctx &c, int bn, const CUtensorMap &ma, const CUtensorMap &mb, int M, int N, int ktiles, int S, double *C,
              int64_t ldc, bool trans, double *part, const unsigned *cond, unsigned mask, bool sk) {
  switch (bn) {
    case 16: launch_bn<16, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, sk); break;
    case 32: launch_bn<32, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, sk); break;
    case 48: launch_bn<48, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, sk); break;
    case 64: launch_bn<64, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, sk); break;
    case 80: launch_bn<80, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, sk); break;
    case 96: launch_bn<96, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, sk); break;
    case 112: launch_bn<112, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, sk); break;
    case 128: launch_bn<128, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, sk); break;
    default: launch_bn<144, MODE>(c, ma, mb, M, N, ktiles, S, C, ldc, trans, part, cond, mask, sk); break;
  }
}

// Off by default (RQLP_STREAMK=1 enables): measured on B200 it does not beat the classic
// split-K grid, whose time model already reaches ~99% wave efficiency on the large passes
// (DESIGN.md §5); kept for shapes where the split-K partial traffic dominates.
bool streamk_disabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RQLP_STREAMK");
    v = (e && e[0] == '1') ? 0 : 1;
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
  // upper bound over both modes for the shapes (m, cc, k) and (k, cc, m)
  size_t best = 0;
  for (int mode = 0; mode < 2; ++mode) {
    int64_t M = mode == 0 ? m : k, K = mode == 0 ? k : m;
    int bn = choose_bn(cc);
    int64_t tiles = ceil_div(M, BM) * ceil_div(cc, bn);
    int64_t ktiles = ceil_div(K, BK);
    int S = choose_splits(tiles, ktiles, num_sms, (size_t)1 << 62, M * cc, bn);
    if (S > 1) best = std::max(best, (size_t)S * M * cc);
    if (use_streamk(tiles, ktiles, num_sms)) best = std::max(best, streamk_elems(num_sms, bn));
  }
  return best;
}

// Launch plan shared by NN and TN: Stream-K when it pays and fits, else split-K.
static void plan_and_dispatch(Ctx &c, int mode, int bn, const CUtensorMap &ma, const CUtensorMap &mb, int64_t M,
                              int64_t N, int64_t ktiles, double *C, int64_t ldc, bool trans, double *partials,
                              size_t partial_elems, const unsigned *cond, unsigned cond_mask) {
  const int64_t tiles = ceil_div(M, BM) * ceil_div(N, bn);
  const size_t cap = partials ? partial_elems : 0;
  const bool sk = !streamk_disabled() && use_streamk(tiles, ktiles, c.num_sms) &&
                  streamk_elems(c.num_sms, bn) <= cap;
  const int S = sk ? 1 : choose_splits(tiles, ktiles, c.num_sms, cap, M * N, bn);
  if (mode == 0)
    dispatch<0>(c, bn, ma, mb, (int)M, (int)N, (int)ktiles, S, C, ldc, trans, partials, cond, cond_mask, sk);
  else
    dispatch<1>(c, bn, ma, mb, (int)M, (int)N, (int)ktiles, S, C, ldc, trans, partials, cond, cond_mask, sk);
}

bool gemm_nn_tma(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *X, int64_t ldx,
                 double *Y, int64_t ldy, double *partials, size_t partial_elems, const unsigned *cond,
                 unsigned cond_mask) {
  if (tma_disabled() || m < 1 || cc < 1 || k < 1) return false;
  int bn = choose_bn(cc);
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, m, k, lda, LDA_NN, BK)) return false;
  if (!make_map(&mb, X, k, cc, ldx, BK, bn)) return false;
  plan_and_dispatch(c, 0, bn, ma, mb, m, cc, ceil_div(k, BK), Y, ldy, false, partials, partial_elems, cond, cond_mask);
  return true;
}

bool gemm_tn_tma(Ctx &c, int64_t m, int64_t cc, int64_t k, const double *A, int64_t lda, const double *V, int64_t ldv,
                 double *Z, int64_t ldz, bool trans_out, double *partials, size_t partial_elems, const unsigned *cond,
                 unsigned cond_mask) {
  if (tma_disabled() || m < 1 || cc < 1 || k < 1) return false;
  int bn = choose_bn(cc);
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, m, k, lda, BK, BM)) return false;
  if (!make_map(&mb, V, m, cc, ldv, BK, bn)) return false;
  plan_and_dispatch(c, 1, bn, ma, mb, k, cc, ceil_div(m, BK), Z, ldz, trans_out, partials, partial_elems, cond,
                    cond_mask);
  return true;
}

}  // namespace rqlpk
