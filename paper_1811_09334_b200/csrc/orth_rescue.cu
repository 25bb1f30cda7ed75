// orth_rescue.cu -- the rare branch of V = orth(Y): repeated (shifted) CholeskyQR passes until
// the basis is orthonormal to working precision, in ONE cooperative kernel.
//
// orth (orth.cu) runs CholeskyQR2 (two passes).  That is exact to O(u) when cond(Y) <~ 1e6
// (every Cholesky pivot above 1e-12 of its Gram diagonal: reading R3).  Otherwise the first (or
// second) pass broke down and was redone on a shifted Gram G + s I (Fukaya et al.'s shifted
// CholeskyQR, s = 11 (m c + c (c + 1)) u tr(G)), which leaves V with cond(V) up to ~u^-1/2
// (or, for numerically rank-deficient Y, directions at the rounding level).  Then this kernel
// continues from V:
//   repeat (at most RESCUE_MAX_PASSES):
//     G = V^T V;
//     if max|G - I| <= 2^-27: V <- V (I - U), U = triu(G - I, 1) + diag(G - I)/2 (first-order
//        factor, exact to below u: the CholeskyQR2 second-pass shortcut), done;
//     else Cholesky G = R^T R (shifted on breakdown; a zero column, or from the RESCUE_DEP_PASS-th
//        pass on a pivot below 1e-15 of its diagonal, is a dependent column: pivot 1 and the
//        column replaced by a random N(0,1)-like vector, reading R4/R21), V <- V R^-1.
//   R (if requested) = V^T Y, upper triangle (Y = V R to O(u ||Y||), zero rows for completed
//   directions -- the same definition the sharded path uses after a completion).
// Each shifted pass multiplies the smallest eigenvalue of the Gram by ~1/s, so rounding-level
// directions of a rank-deficient Y are amplified into full-rank ones in a few passes.
//
// Launched on every full-mode orth (non-sharded); it returns at once unless the COND word holds
// one of the shift bits, so the common path pays one launch instead of a third pass of kernels.
// All CTAs are co-resident (cooperative launch); phases are separated by a software grid barrier
// on two handle flag words.  Performance is secondary here (rare path): plain FP64 FMA tiles.
#include "internal.cuh"

namespace rqlpk {

namespace {

constexpr int RESCUE_MAX_PASSES = 10;
constexpr int RESCUE_DEP_PASS = 4;
constexpr double RES_BREAK = 1e-12;
constexpr double RES_DEP = 1e-15;
constexpr int RT = 256;  // threads per CTA

struct RescueArgs {
  int64_t m;
  int c;
  double *V;
  int64_t ldv;
  double *W;  // m x c ping-pong
  int64_t ldw;
  const double *Y;
  int64_t ldy;
  double *R;  // nullable: R = V^T Y (c x c upper)
  int64_t ldr;
  double *G0, *Gw, *Rf, *X;  // c x c scratch, leading dimension ldg
  int64_t ldg;
  double *part;
  int64_t part_elems;
  int *dep;
  unsigned *flags;
  const unsigned *cond;
  unsigned mask;
  unsigned *bar;                 // 2 words: arrival count, generation
  unsigned long long *maxbits;   // max |G - I| as ordered bits
};

__device__ __forceinline__ double ldg_cg(const double *p) { return __ldcg(p); }

// Software grid barrier (all CTAs co-resident).  The last CTA to arrive resets the count and bumps
// the generation; the fences make every CTA's writes before the barrier visible after it (data
// written by other CTAs is read with L1-bypassing loads).
// A barrier that has not completed after ~10 s (a co-residency or divergence bug) traps instead of
// hanging the device.
__device__ void grid_sync(unsigned *bar, int tag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      const long long t0 = clock64();
      while (*gen == g) {
        if (clock64() - t0 > 20000000000LL) {
          printf("orth_rescue: grid barrier timeout (block %d tag %d gen %u count %u)\n", blockIdx.x, tag, g,
                 *(volatile unsigned *)bar);
          __trap();
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
}

struct Smem {
  double a[64][33];
  double b[32][33];
  int flag;
};

// out(i, j) = sum_r A(r, i) B(r, j) for the 32 x 32 tile pairs (ti <= tj when upper; the strictly
// lower entries of diagonal tiles are zeroed when zero_lower), rows split into S chunks whose
// partial tiles are summed in chunk order (deterministic).  Ends with a grid barrier.
__device__ void tile_dot(const RescueArgs &a, Smem &sm, const double *A, int64_t lda, const double *B, int64_t ldb,
                         double *out, int64_t ldo, bool upper, bool zero_lower) {
  const int c = a.c, T = (c + 31) / 32;
  const int P = upper ? T * (T + 1) / 2 : T * T;
  int S = (int)std::max<int64_t>(1, std::min<int64_t>((2 * gridDim.x + P - 1) / P, (a.m + 255) / 256));
  S = (int)std::max<int64_t>(1, std::min<int64_t>(S, a.part_elems / ((int64_t)P * 1024)));
  const int64_t chunk = ((a.m + S - 1) / S + 31) / 32 * 32;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (int item = blockIdx.x; item < P * S; item += gridDim.x) {
    const int p = item % P, s = item / P;
    int ti, tj;
    if (upper) {  // p -> (ti <= tj), column-major over the upper triangle
      tj = 0;
      while ((tj + 1) * (tj + 2) / 2 <= p) ++tj;
      ti = p - tj * (tj + 1) / 2;
    } else {
      ti = p % T;
      tj = p / T;
    }
    const int i0 = ti * 32, j0 = tj * 32;
    const int64_t r0 = (int64_t)s * chunk, r1 = std::min<int64_t>(a.m, r0 + chunk);
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int64_t rb = r0; rb < r1; rb += 32) {
      __syncthreads();
      for (int e = tid; e < 32 * 32; e += RT) {
        const int r = e & 31, col = e >> 5;
        const int64_t row = rb + r;
        const bool ok = row < r1;
        sm.a[r][col] = (ok && i0 + col < c) ? ldg_cg(A + row + (int64_t)(i0 + col) * lda) : 0.0;
        sm.b[r][col] = (ok && j0 + col < c) ? ldg_cg(B + row + (int64_t)(j0 + col) * ldb) : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int r = 0; r < 32; ++r) {
        const double a0 = sm.a[r][2 * ty], a1 = sm.a[r][2 * ty + 1];
        const double b0 = sm.b[r][2 * tx], b1 = sm.b[r][2 * tx + 1];
        acc[0][0] = fma(a0, b0, acc[0][0]);
        acc[0][1] = fma(a0, b1, acc[0][1]);
        acc[1][0] = fma(a1, b0, acc[1][0]);
        acc[1][1] = fma(a1, b1, acc[1][1]);
      }
    }
    for (int u = 0; u < 2; ++u)
      for (int v = 0; v < 2; ++v) {
        const int ii = 2 * ty + u, jj = 2 * tx + v;
        if (S == 1) {
          if (i0 + ii < c && j0 + jj < c)
            out[(i0 + ii) + (int64_t)(j0 + jj) * ldo] = (zero_lower && i0 + ii > j0 + jj) ? 0.0 : acc[u][v];
        } else {
          a.part[((int64_t)s * P + p) * 1024 + ii + jj * 32] = acc[u][v];
        }
      }
  }
  grid_sync(a.bar, 1);
  if (S > 1) {
    const int64_t tot = (int64_t)P * 1024;
    for (int64_t e = (int64_t)blockIdx.x * RT + tid; e < tot; e += (int64_t)gridDim.x * RT) {
      const int p = (int)(e / 1024), w = (int)(e % 1024), ii = w & 31, jj = w >> 5;
      int ti, tj;
      if (upper) {
        tj = 0;
        while ((tj + 1) * (tj + 2) / 2 <= p) ++tj;
        ti = p - tj * (tj + 1) / 2;
      } else {
        ti = p % T;
        tj = p / T;
      }
      const int i = ti * 32 + ii, j = tj * 32 + jj;
      if (i >= c || j >= c) continue;
      double sum = 0.0;
      for (int s = 0; s < S; ++s) sum += ldg_cg(a.part + ((int64_t)s * P + p) * 1024 + w);
      out[i + (int64_t)j * ldo] = (zero_lower && i > j) ? 0.0 : sum;
    }
    grid_sync(a.bar, 2);
  }
}

__global__ void __launch_bounds__(RT, 1) orth_rescue_kernel(RescueArgs a) {
  if (((*a.cond) & a.mask) == 0) return;
  __shared__ Smem sm;
  const int c = a.c, tid = threadIdx.x, lane = tid & 31;
  const int64_t ldg = a.ldg;
  const int64_t gthreads = (int64_t)gridDim.x * RT, gtid = (int64_t)blockIdx.x * RT + tid;
  const int gwarps = (int)(gthreads >> 5), gwarp = (int)(gtid >> 5);
  double *cur = a.V, *nxt = a.W;
  int64_t ldc = a.ldv, ldn = a.ldw;
  bool any_shift = false, any_dep = false;
  for (int pass = 0; pass < RESCUE_MAX_PASSES; ++pass) {
    // G0 = cur^T cur (upper)
    if (gtid == 0) *a.maxbits = 0ull;
    tile_dot(a, sm, cur, ldc, cur, ldc, a.G0, ldg, true, false);
    // near-identity test (max over the upper triangle; non-negative doubles order as their bits)
    {
      double e = 0.0;
      for (int64_t q = gtid; q < (int64_t)c * c; q += gthreads) {
        const int i = (int)(q % c), j = (int)(q / c);
        if (i > j) continue;
        const double v = fabs(ldg_cg(a.G0 + i + j * ldg) - (i == j ? 1.0 : 0.0));
        e = (v > e || v != v) ? v : e;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, e, o);
        e = (t > e || t != t) ? t : e;
      }
      if (lane == 0) atomicMax(a.maxbits, (unsigned long long)__double_as_longlong(e));
    }
    grid_sync(a.bar, 3);
    const double emax = __longlong_as_double((long long)*(volatile unsigned long long *)a.maxbits);
    const bool near_id = emax <= 0x1p-27;
    bool dep_now = false;
    if (near_id) {
      for (int64_t q = gtid; q < (int64_t)c * c; q += gthreads) {
        const int i = (int)(q % c), j = (int)(q / c);
        double u = 0.0;
        if (i < j) u = ldg_cg(a.G0 + i + j * ldg);
        else if (i == j) u = 0.5 * (ldg_cg(a.G0 + i + j * ldg) - 1.0);
        a.X[i + j * ldg] = (i == j ? 1.0 : 0.0) - u;
      }
      for (int j = (int)gtid; j < c; j += (int)gthreads) a.dep[j] = 0;
    } else {
      // trace of G0 (every CTA, same order)
      double tr = 0.0;
      for (int i = 0; i < c; ++i) tr += ldg_cg(a.G0 + i + i * ldg);
      double sh = 11.0 * ((double)a.m * c + (double)c * (c + 1)) * 0x1p-53 * tr;
      if (!(sh > 0.0)) sh = 1.0;
      const bool dep_ratio = pass + 1 >= RESCUE_DEP_PASS;
      for (int attempt = 0; attempt < 2; ++attempt) {
        const double shift = attempt ? sh : 0.0;
        for (int64_t q = gtid; q < (int64_t)c * c; q += gthreads) {
          const int i = (int)(q % c), j = (int)(q / c);
          if (i <= j) a.Gw[i + j * ldg] = ldg_cg(a.G0 + i + j * ldg) + (i == j ? shift : 0.0);
        }
        grid_sync(a.bar, 4);
        bool broke = false;
        for (int j = 0; j < c; ++j) {
          const double d = ldg_cg(a.Gw + j + j * ldg);
          const double g0 = ldg_cg(a.G0 + j + j * ldg);
          int kind = 0;  // 0 pivot, 1 dependent column, 2 breakdown
          if (!(g0 > 0.0) || !isfinite(g0)) kind = 1;
          else if (!isfinite(d)) kind = 2;
          else if (dep_ratio && !(d > RES_DEP * (g0 + shift))) kind = 1;
          else if (!(d > RES_BREAK * (g0 + shift))) kind = 2;
          if (kind == 2 && attempt == 0) {  // every CTA sees the same values: a uniform decision
            broke = true;
            break;
          }
          if (kind == 2) kind = 1;  // still no pivot on the shifted Gram: complete the column
          const double rjj = kind ? 1.0 : sqrt(d);
          const double inv = 1.0 / rjj;
          if (gtid == 0) {
            a.Rf[j + j * ldg] = rjj;
            a.dep[j] = kind;
          }
          dep_now |= kind != 0;
          for (int k = j + 1 + (int)gtid; k < c; k += (int)gthreads)
            a.Rf[j + k * ldg] = kind ? 0.0 : ldg_cg(a.Gw + j + k * ldg) * inv;
          if (!kind) {
            const int nr = c - j - 1;
            const double dinv = 1.0 / d;
            for (int64_t q = gtid; q < (int64_t)nr * nr; q += gthreads) {
              const int i = j + 1 + (int)(q % nr), k = j + 1 + (int)(q / nr);
              if (i > k) continue;
              a.Gw[i + k * ldg] -= ldg_cg(a.Gw + j + i * ldg) * ldg_cg(a.Gw + j + k * ldg) * dinv;
            }
          }
          grid_sync(a.bar, 1000 + j);
        }
        if (!broke) {
          any_shift |= attempt > 0;
          break;
        }
        dep_now = false;
        // every CTA has read this step's pivot before the shifted copy overwrites Gw
        grid_sync(a.bar, 9);
      }
      // X = Rf^-1 (upper): a warp per column, back substitution
      for (int k = gwarp; k < c; k += gwarps) {
        double *x = a.X + (int64_t)k * ldg;
        for (int i = k + 1 + lane; i < c; i += 32) x[i] = 0.0;
        if (lane == 0) x[k] = 1.0 / ldg_cg(a.Rf + k + k * ldg);
        __syncwarp();
        for (int i = k - 1; i >= 0; --i) {
          double s = 0.0;
          for (int t = i + 1 + lane; t <= k; t += 32) s = fma(ldg_cg(a.Rf + i + (int64_t)t * ldg), x[t], s);
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) x[i] = -s / ldg_cg(a.Rf + i + (int64_t)i * ldg);
          __syncwarp();
        }
      }
    }
    any_dep |= dep_now;
    grid_sync(a.bar, 6);
    // nxt = cur X (X upper: k <= j); dependent columns get the completion vector
    {
      const int tx = tid & 15, ty = tid >> 4;
      const int64_t mt = (a.m + 63) / 64;
      const int nt = (c + 31) / 32;
      const uint64_t key = 0x7e5c0000ULL + (uint64_t)pass;
      for (int64_t item = blockIdx.x; item < mt * nt; item += gridDim.x) {
        const int64_t r0 = (item % mt) * 64;
        const int j0 = (int)(item / mt) * 32;
        const int kmax = std::min(c, j0 + 32);
        double acc[4][2] = {};
        for (int k0 = 0; k0 < kmax; k0 += 32) {
          __syncthreads();
          for (int e = tid; e < 64 * 32; e += RT) {
            const int r = e & 63, kk = e >> 6;
            const int64_t row = r0 + r;
            sm.a[r][kk] = (row < a.m && k0 + kk < c) ? ldg_cg(cur + row + (int64_t)(k0 + kk) * ldc) : 0.0;
          }
          for (int e = tid; e < 32 * 32; e += RT) {
            const int kk = e & 31, jj = e >> 5;
            sm.b[kk][jj] = (k0 + kk < c && j0 + jj < c) ? ldg_cg(a.X + (k0 + kk) + (int64_t)(j0 + jj) * ldg) : 0.0;
          }
          __syncthreads();
#pragma unroll 4
          for (int kk = 0; kk < 32; ++kk) {
            const double b0 = sm.b[kk][2 * tx], b1 = sm.b[kk][2 * tx + 1];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double av = sm.a[4 * ty + u][kk];
              acc[u][0] = fma(av, b0, acc[u][0]);
              acc[u][1] = fma(av, b1, acc[u][1]);
            }
          }
        }
        for (int u = 0; u < 4; ++u)
          for (int v = 0; v < 2; ++v) {
            const int64_t row = r0 + 4 * ty + u;
            const int j = j0 + 2 * tx + v;
            if (row >= a.m || j >= c) continue;
            double val = acc[u][v];
            if (dep_now && __ldcg(a.dep + j)) val = completion_value((uint64_t)row + (uint64_t)a.m * j, key);
            nxt[row + (int64_t)j * ldn] = val;
          }
      }
    }
    grid_sync(a.bar, 7);
    double *tp = cur;
    cur = nxt;
    nxt = tp;
    const int64_t tl = ldc;
    ldc = ldn;
    ldn = tl;
    if (near_id) break;
  }
  // the result into V
  if (cur != a.V) {
    for (int64_t q = gtid; q < a.m * c; q += gthreads) {
      const int64_t i = q % a.m, j = q / a.m;
      a.V[i + j * a.ldv] = ldg_cg(cur + i + j * ldc);
    }
    grid_sync(a.bar, 8);
  }
  if (a.R) tile_dot(a, sm, a.V, a.ldv, a.Y, a.ldy, a.R, a.ldr, false, true);
  if (gtid == 0) {
    if (any_shift) atomicOr(a.flags, (unsigned)RQLP_FLAG_SHIFTED_CHOLQR);
    if (any_dep) atomicOr(a.flags, (unsigned)RQLP_FLAG_RANK_DEFICIENT);
  }
}

}  // namespace

void launch_orth_rescue(Ctx &c, OrthScratch &s, int64_t m, int64_t n, double *V, int64_t ldv, const double *Y,
                        int64_t ldy, double *R, int64_t ldr, const unsigned *cond, unsigned mask) {
  RescueArgs a;
  a.m = m;
  a.c = (int)n;
  a.V = V;
  a.ldv = ldv;
  a.W = s.Ybuf;
  a.ldw = s.ldy;
  a.Y = Y;
  a.ldy = ldy;
  a.R = R;
  a.ldr = ldr;
  a.G0 = s.G;
  a.Gw = s.G2;
  a.Rf = s.Racc;
  a.X = s.Rinv;
  a.ldg = round_up(n, 8);
  a.part = s.partials;
  a.part_elems = (int64_t)s.partial_elems;
  a.dep = s.dep;
  a.flags = c.dflags + FLAG_WORD;
  a.cond = cond;
  a.mask = mask;
  a.bar = c.dflags + BAR_COUNT;
  a.maxbits = reinterpret_cast<unsigned long long *>(s.scal);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)c.num_sms);
  cfg.blockDim = dim3(RT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RQLP_CUDA(cudaLaunchKernelEx(&cfg, orth_rescue_kernel, a));
  RQLP_LAUNCHED(c);
}

}  // namespace rqlpk
