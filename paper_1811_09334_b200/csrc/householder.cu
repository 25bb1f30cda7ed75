// householder.cu -- Householder QR engine with optional column pivoting (the CPQR of the tail).
//
// Alg.1 l.5 "[Q0, R0, Π0] = cpqr(B)" and l.6 "cpqr(R0^T)"; Alg.2
// l.7 unpivoted "qr([R^(i-1)]^T)".  The pivot rule (reading R5): at step j pick
// the remaining column with the largest downdated norm, ties to the lowest ORIGINAL column
// index; norms are downdated with the LAPACK xLAQP2 rule and recomputed when
// t (vn1/vn2)^2 <= sqrt(2^-53).  The paper names no pivot rule; SURVEY §8(c.1) step 6 fixes it.
//
// B200 design: one persistent kernel runs all s = min(rows, cols) strictly sequential steps.
// Columns stay where they are (no physical swaps): CTA b owns columns b, b+G, b+2G, ... and
// keeps them (and their norms) in shared memory when they fit; it applies every reflector to
// them.  Small matrices run in ONE 1024-thread CTA entirely in shared memory (no global
// exchange).  Larger ones run on one CTA per SM (cooperative launch); each step then needs one
// exchange, done NCCL-LL style: every CTA publishes its best candidate (norm, column) as three
// 8-byte words each carrying the step tag, after the candidate column's rows j.. (release
// fence); every CTA polls all tags (the poll IS the grid barrier), takes the exact argmax
// (ties -> lowest column) and reads the winner's column.  Records and candidate columns are
// double-buffered by step parity, so a CTA can run at most one step ahead without overwriting
// data a slower CTA still reads.  Every CTA recomputes the reflector from the winner's column
// with the same fixed-order reduction, so all hold bit-identical v, tau; CTA 0 stores it.
#include <type_traits>

#include "internal.cuh"

namespace rqlpk {
namespace {

constexpr double TOL3Z = 1.0536712127723509e-08;  // sqrt(2^-53), LAPACK dlaqp2 tol3z
constexpr int RPL = 40;  // rows per lane kept in registers for global-memory columns (<= 1281 rows)

struct Best {
  double v;
  int i;
};
// Candidate order: larger (squared) norm, then lower index.  A NaN norm (non-finite input) ranks
// above every number, so a column is always chosen (the pivot index stays in range).
__device__ __forceinline__ bool better(double v, int i, double bv, int bi) {
  if (v != v) return bv == bv || i < bi;
  return v > bv || (v == bv && i < bi);
}

// Warp argmax (max value, lowest index on ties).  Values are >= 0 (squared norms) or -1 (no
// candidate); non-negative doubles order like their bit patterns, so integer redux.sync on the
// high then the low 32 bits (biased so -1 sorts lowest) finds the maximum, and one more on the
// index picks the lowest among equal values -- no shuffle tree (the lanes of an 8-lane column
// group all hold the same candidate, which defeated a single-winner shortcut).
__device__ __forceinline__ Best warp_best(Best b) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(b.v);
  const bool neg = b.v < 0.0;
  const unsigned hi = neg ? 0u : (unsigned)(bits >> 32) + 1u;
  const unsigned lo = neg ? 0u : (unsigned)bits;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool top = hi == mhi && lo == mlo;
  const int mi = (int)__reduce_min_sync(0xffffffffu, top ? (unsigned)b.i : 0xffffffffu);
  const int src = __ffs(__ballot_sync(0xffffffffu, top && b.i == mi)) - 1;
  return Best{__shfl_sync(0xffffffffu, b.v, src), mi};
}

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

__device__ double warp_sumsq(const double *x, int64_t len) {
  double s = 0.0;
  for (int64_t r = threadIdx.x & 31; r < len; r += 32) s = fma(x[r], x[r], s);
  return warp_sum(s);
}


struct EngineArgs {
  double *M;
  int64_t ldm;
  int rows, cols, steps, pivot;
  int owned_max;   // max columns owned by one CTA
  double *Vst;     // rows x steps, ld rows
  double *tau, *beta;
  unsigned long long *rec;   // [2][G][4] LL words: {hi(val)|tag, lo(val)|tag, idx|tag, -}
  unsigned long long *cand;  // [2][G][rows][2] LL words of the candidate column rows j.. (lo, hi halves)
  unsigned epoch;            // high 16 bits of every tag (0: the buffers are zeroed per launch)
  unsigned long long *trace; // optional per-step phase timestamps (CTA 0, thread 0), debugging only
  int *done;                // done[col] = 1 once pivoted (compaction of the non-pivot columns)
  int64_t *perm;
  int npoll;                 // warps that poll the exchange records (redundantly; warp 0 publishes p)
  int w0free;                // warp 0 (the poller) takes no deferred column updates
  int gtime;                 // debug trace: %globaltimer (ns) instead of clock64
};

// Exchange words: gpu-scope relaxed accesses (every word carries its step tag, so no ordering
// between words is needed; gpu scope instead of the system scope of volatile), 16-byte vectors
// for the (lo, hi) halves of a candidate row and the (hi, lo) halves of a record's value.
__device__ __forceinline__ void st_x2(unsigned long long *p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};\n" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_x1(unsigned long long *p, unsigned long long a) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(p), "l"(a) : "memory");
}
__device__ __forceinline__ void ld_x2(const unsigned long long *p, unsigned long long &a, unsigned long long &b) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long ld_x1(const unsigned long long *p) {
  unsigned long long a;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(a) : "l"(p) : "memory");
  return a;
}

__device__ __forceinline__ unsigned long long pack(unsigned hi, unsigned tag) {
  return ((unsigned long long)hi << 32) | tag;
}

// Shared-memory layout: vraw[rows] | vn1[owned] | rvn2[owned] | colbuf[owned*rows] (SMEMC) | done_l[owned]
//
// Per step: (GRID only) warp 0 polls the tagged records (the exchange is the grid barrier), all
// threads fetch the winner's rows j.. into vraw, one __syncthreads; then EVERY warp recomputes
// the reflector from the pivot column with the same lane assignment and shuffle tree (so all
// warps and CTAs hold identical bits, no block reduction), applies it to its own columns and
// downdates their norms; warps post their best candidate in a parity-double-buffered slot and
// meet at the step's single __syncthreads; every warp then reduces the 32 slots itself.
// GT: threads of the global-memory-column variant (a warp per column): 384 keeps 12 columns in
// flight per CTA (measured on C5's 1056 x 16384 B: 256 threads 48.7 ms, 384 46.2 ms, 512 spills)
template <bool GRID, bool SMEMC, int GT = 384>
__global__ void __launch_bounds__(GRID ? (SMEMC ? 512 : GT) : 1024, 1) hh_engine_kernel(EngineArgs a) {
  extern __shared__ __align__(16) double smem[];
  // even strides keep every cached column and the pivot column 16-byte aligned (double2 access
  // in absolute row coordinates); the padding row is zero and stays zero
  const int rs = (a.rows + 1) & ~1, op = (a.owned_max + 1) & ~1;
  double *vraw = smem;                   // pivot column rows j.. at their absolute positions
  double *vn1 = vraw + rs;
  double *rvn2 = vn1 + op;               // 1 / (squared norm at the last recompute)
  double *wsbuf = rvn2 + op;             // deferred rank-1 update factors (GRID, cached, pivoted)
  double *colbuf = wsbuf + op;
  int *done_l = reinterpret_cast<int *>(colbuf + (SMEMC ? (int64_t)a.owned_max * rs : 0));
  __shared__ double s_bv[2][32];
  __shared__ int s_bi[2][32];
  __shared__ int s_p;
  __shared__ double s_xn2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int G = GRID ? (int)gridDim.x : 1, b = GRID ? (int)blockIdx.x : 0;
  const int nown = b < a.cols ? (a.cols - b + G - 1) / G : 0;  // columns b, b+G, b+2G, ...
  const int rows = a.rows;
  const bool DEFER = GRID && SMEMC && a.pivot;
  auto colptr = [&](int li) -> double * {
    if (SMEMC) return colbuf + (int64_t)li * rs;
    return a.M + (int64_t)(b + li * G) * a.ldm;
  };
  auto cta_best = [&](int par) -> Best {  // every warp: argmax of the 32 warp slots
    Best c = lane < wpb ? Best{s_bv[par][lane], s_bi[par][lane]} : Best{-1.0, 0x7fffffff};
    return warp_best(c);
  };
  // GRID: publish this CTA's candidate for step jn (warp 0 only): candidate rows jn.. as LL words,
  // then the tagged record {value, column}.
  auto publish = [&](int jn, Best c) {
    const int par = jn & 1;
    const unsigned tag = (a.epoch << 16) | ((unsigned)jn + 1u);
    int src = -1;
    if (a.pivot) src = c.i != 0x7fffffff ? c.i : -1;
    else if (jn < a.cols && jn % G == b) src = jn;
    auto record = [&]() {
      if (lane == 0 && (a.pivot || src >= 0)) {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(a.pivot ? c.v : 0.0);
        unsigned long long *rc = a.rec + ((int64_t)par * G + b) * 4;
        st_x2(rc, pack((unsigned)(bits >> 32), tag), pack((unsigned)bits, tag));
        st_x1(rc + 2, pack((unsigned)(a.pivot ? c.i : src), tag));
      }
    };
    // the record first: the pollers' argmax does not wait for the column (the fetch spins on
    // each row's tag, so the order of the words does not matter)
    record();
    if (src >= 0) {
      const double *sp = colptr((src - b) / G);
      unsigned long long *dst = a.cand + ((int64_t)par * G + b) * (rows + 1) * 2;
      double s2 = 0.0;  // sum of squares of rows jn+1..: the next reflector's xnorm^2, computed once
      for (int r = jn + lane; r < rows; r += 32) {
        const double v = sp[r];
        if (r > jn) s2 = fma(v, v, s2);
        const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
        st_x2(dst + 2 * (r - jn), pack((unsigned)bits, tag), pack((unsigned)(bits >> 32), tag));
      }
      s2 = warp_sum(s2);
      if (lane == 0) {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(s2);
        st_x2(dst + 2 * (rows - jn), pack((unsigned)bits, tag), pack((unsigned)(bits >> 32), tag));
      }
    }
  };

  if (SMEMC)
    for (int li = 0; li < nown; ++li)
      for (int r = threadIdx.x; r < rs; r += blockDim.x)
        colbuf[(int64_t)li * rs + r] = r < rows ? a.M[(int64_t)(b + li * G) * a.ldm + r] : 0.0;
  if (threadIdx.x == 0 && rs > rows) vraw[rows] = 0.0;
  for (int li = threadIdx.x; li < nown; li += blockDim.x) {
    done_l[li] = 0;
    a.done[b + li * G] = 0;
  }
  __syncthreads();
  Best best{-1.0, 0x7fffffff};
  if (a.pivot)
    for (int li = warp; li < nown; li += wpb) {
      double nrm = warp_sumsq(colptr(li), rows);  // squared norms (monotone: same argmax)
      if (lane == 0) { vn1[li] = nrm; rvn2[li] = nrm != 0.0 ? 1.0 / nrm : 0.0; }
      if (better(nrm, b + li * G, best.v, best.i)) { best.v = nrm; best.i = b + li * G; }
    }
  {
    Best wb = warp_best(best);
    if (lane == 0) { s_bv[0][warp] = wb.v; s_bi[0][warp] = wb.i; }
  }
  __syncthreads();
  if (GRID && warp == 0) publish(0, cta_best(0));

  // per-CTA debug stamps: [step 20..59][CTA][poll start, poll done, fetch done, record out]
  auto cstamp = [&](int jj, int k) {
    if (a.trace && GRID && threadIdx.x == 0 && jj >= 20 && jj < 60 && b < 148) {
      unsigned long long t;
      if (a.gtime) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      else t = (unsigned long long)clock64();
      a.trace[8192 + ((int64_t)(jj - 20) * 148 + b) * 4 + k] = t;
    }
  };
  for (int j = 0; j < a.steps; ++j) {
    const int par = j & 1;
    auto stamp = [&](int ph) {
      if (a.trace && b == 0 && threadIdx.x == 0) {
        a.trace[(int64_t)j * 4 + ph] = (unsigned long long)clock64();  // SM cycles
      }
    };
    stamp(0);
    cstamp(j, 0);
    const int len = rows - j;
    const double *cp;  // rows j.. of the pivot column
    int p;
    if (GRID) {
      const unsigned tag = (a.epoch << 16) | ((unsigned)j + 1u);
      if (warp < a.npoll) {
        Best c{-1.0, 0x7fffffff};
        if (a.pivot) {
          // each lane owns records lane, lane+32, ...: issue all loads, re-poll only the stale ones
          constexpr int MAXR = 8;  // G <= 256
          unsigned long long w0[MAXR], w1[MAXR], w2[MAXR];
          unsigned pending = 0;
#pragma unroll
          for (int t = 0; t < MAXR; ++t)
            if (lane + 32 * t < G) pending |= 1u << t;
          while (pending) {
#pragma unroll
            for (int t = 0; t < MAXR; ++t)
              if (pending & (1u << t)) {
                const unsigned long long *rc = a.rec + ((int64_t)par * G + lane + 32 * t) * 4;
                ld_x2(rc, w0[t], w1[t]);
                w2[t] = ld_x1(rc + 2);
              }
#pragma unroll
            for (int t = 0; t < MAXR; ++t)
              if ((pending & (1u << t)) && (unsigned)w0[t] == tag && (unsigned)w1[t] == tag && (unsigned)w2[t] == tag)
                pending &= ~(1u << t);
          }
#pragma unroll
          for (int t = 0; t < MAXR; ++t)
            if (lane + 32 * t < G) {
              const double val = __longlong_as_double((long long)(((w0[t] >> 32) << 32) | (w1[t] >> 32)));
              const int idx = (int)(w2[t] >> 32);
              if (better(val, idx, c.v, c.i)) { c.v = val; c.i = idx; }
            }
          c = warp_best(c);
        } else {
          c.i = j;
        }
        if (warp == 0 && lane == 0) s_p = c.i;
      }
      cstamp(j, 1);
      __syncthreads();
      p = s_p;
      const unsigned long long *src = a.cand + ((int64_t)par * G + (p % G)) * (rows + 1) * 2;
      for (int r = threadIdx.x; r <= len; r += blockDim.x) {  // r == len: the published xnorm^2
        unsigned long long lo, hi;
        do {
          ld_x2(src + 2 * r, lo, hi);
        } while ((unsigned)lo != tag || (unsigned)hi != tag);
        const double v = __longlong_as_double((long long)(((hi >> 32) << 32) | (lo >> 32)));
        if (r < len) vraw[j + r] = v;
        else s_xn2 = v;
      }
      __syncthreads();
      cp = vraw + j;
    } else {
      p = a.pivot ? cta_best(par).i : j;
      cp = colptr(p) + j;
    }
    stamp(1);
    cstamp(j, 2);

    // ---- reflector (xLARFG), recomputed by every warp from the same values -> identical bits
    //      (grid: ||rows j+1..||^2 comes with the candidate, summed once by its publisher)
    double xn2;
    if (GRID) {
      xn2 = s_xn2;
    } else {
      double part = 0.0;
      for (int r = 1 + lane; r < len; r += 32) part = fma(cp[r], cp[r], part);
      xn2 = warp_sum(part);
    }
    const double alpha = cp[0];
    double tau, beta, scal;
    if (xn2 == 0.0) {
      tau = 0.0; beta = alpha; scal = 0.0;
    } else {
      beta = -copysign(fast_sqrt(fma(alpha, alpha, xn2)), alpha);
      const double amb = alpha - beta;              // tau = (beta - alpha)/beta, scal = 1/(alpha - beta)
      const double rinv = fast_rcp(beta * amb);     // one reciprocal for both
      tau = -amb * amb * rinv;
      scal = beta * rinv;
    }
    const int ob = p % G;
    if (b == ob && threadIdx.x == 0) {
      done_l[p / G] = 1;
      a.done[p] = 1;
    }
    stamp(2);

    // ---- apply H_j (v = [1; cp[1..] scal]) to every owned, not yet pivoted column; downdate.
    //      8-lane groups: a warp updates 4 columns at once (3-step group reductions).
    best = Best{-1.0, 0x7fffffff};
    {
      // column groups: 8 lanes per column for shared-memory columns (a warp updates 4 at once),
      // a whole warp per column for columns in global memory (more loads in flight per column)
      constexpr int GS = SMEMC ? 8 : 32, GPW = 32 / GS;
      const int g8 = lane / GS, l8 = lane % GS;
      const unsigned gmask = GS == 32 ? 0xffffffffu : (0xffu << (8 * g8));
      auto gsum = [&](double v) {
#pragma unroll
        for (int o = GS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
        return v;
      };
      for (int li = warp * GPW + g8; li < nown; li += wpb * GPW) {
        const int gi = b + li * G;
        if (gi == p || done_l[li]) continue;
        // downdating operands (vn1 and rvn2 = 1/vn2), loaded before the column
        double n1 = 0.0, r2 = 0.0;
        if (a.pivot) {
          n1 = vn1[li];
          r2 = rvn2[li];
        }
        double *col = colptr(li) + j;
        double x = col[0];
        if (tau != 0.0) {
          if (SMEMC) {
            // absolute rows: the odd leading row j+1 (if any) by lane 0, then aligned pairs
            const double *cpa = cp - j;
            double *cab = col - j;
            const int a0 = (j + 2) & ~1;
            // four accumulation chains (the FP64 FMA latency, not the loads, bounds this loop)
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
            if (l8 == 0 && j + 1 < a0 && j + 1 < rows) d0 = cpa[j + 1] * cab[j + 1];
            int ar = a0 + 2 * l8;
            for (; ar + 16 < rows; ar += 32) {
              const double2 v = *reinterpret_cast<const double2 *>(cpa + ar);
              const double2 u = *reinterpret_cast<const double2 *>(cab + ar);
              const double2 v2 = *reinterpret_cast<const double2 *>(cpa + ar + 16);
              const double2 u2 = *reinterpret_cast<const double2 *>(cab + ar + 16);
              d0 = fma(v.x, u.x, d0);
              d1 = fma(v.y, u.y, d1);
              d2 = fma(v2.x, u2.x, d2);
              d3 = fma(v2.y, u2.y, d3);
            }
            if (ar < rows) {
              const double2 v = *reinterpret_cast<const double2 *>(cpa + ar);
              const double2 u = *reinterpret_cast<const double2 *>(cab + ar);
              d0 = fma(v.x, u.x, d0);
              d1 = fma(v.y, u.y, d1);
            }
            const double dot = gsum((d0 + d1) + (d2 + d3));
            const double w = tau * fma(scal, dot, x);   // tau v^T col, v = [1; cp[1..] scal]
            const double ws = w * scal;
            x -= w;  // the updated row-j entry (identical in the 8 lanes)
            if (l8 == 0) col[0] = x;
            if (DEFER) {
              // rows j+1.. are updated after the publish (off the exchange's critical path);
              // the downdate below needs only the row-j entry
              if (l8 == 0) wsbuf[li] = ws;
            } else {
              if (l8 == 0 && j + 1 < a0 && j + 1 < rows) cab[j + 1] = fma(-ws, cpa[j + 1], cab[j + 1]);
#pragma unroll 2
              for (int ar = a0 + 2 * l8; ar < rows; ar += 16) {
                const double2 v = *reinterpret_cast<const double2 *>(cpa + ar);
                double2 u = *reinterpret_cast<const double2 *>(cab + ar);
                u.x = fma(-ws, v.x, u.x);
                u.y = fma(-ws, v.y, u.y);
                *reinterpret_cast<double2 *>(cab + ar) = u;
              }
            }
          } else if (len <= 1 + 32 * RPL) {
            // columns in global memory, short enough to stay in registers for the step: one read
            // and one write of the column (all loads in flight) instead of read, read, write.
            // The unrolled row loops are sized to the rows left (4, 8, ..., 40 per lane): late in
            // the factorisation a fixed 40-iteration loop issued mostly predicated-off instructions
            // (same operations on the same values in the same order: bit-identical results).
            auto upd = [&](auto rp) {
              constexpr int RP = decltype(rp)::value;
              double reg[RP];
#pragma unroll
              for (int i = 0; i < RP; ++i) {
                const int r = 1 + l8 + 32 * i;
                reg[i] = r < len ? col[r] : 0.0;
              }
              double w0 = l8 == 0 ? x : 0.0, w1 = 0.0;
#pragma unroll
              for (int i = 0; i < RP; i += 2) {
                const int r = 1 + l8 + 32 * i;
                if (r < len) w0 = fma(cp[r] * scal, reg[i], w0);
                if (i + 1 < RP && r + 32 < len) w1 = fma(cp[r + 32] * scal, reg[i + 1], w1);
              }
              double w = gsum(w0 + w1);
              w *= tau;
              x -= w;  // the updated row-j entry (identical in the lanes)
              if (l8 == 0) col[0] = x;
#pragma unroll
              for (int i = 0; i < RP; ++i) {
                const int r = 1 + l8 + 32 * i;
                if (r < len) col[r] = fma(-w, cp[r] * scal, reg[i]);
              }
            };
            // (a binary decision tree over rows-per-lane sizes 4, 8, ..., 40)
            const int need = (len - 1 + 31) >> 5;   // rows per lane below row j
            if (need <= 20) {
              if (need <= 8) {
                if (need <= 4) upd(std::integral_constant<int, 4>{});
                else upd(std::integral_constant<int, 8>{});
              } else if (need <= 12) upd(std::integral_constant<int, 12>{});
              else if (need <= 16) upd(std::integral_constant<int, 16>{});
              else upd(std::integral_constant<int, 20>{});
            } else if (need <= 28) {
              if (need <= 24) upd(std::integral_constant<int, 24>{});
              else upd(std::integral_constant<int, 28>{});
            } else if (need <= 32) upd(std::integral_constant<int, 32>{});
            else if (need <= 36) upd(std::integral_constant<int, 36>{});
            else upd(std::integral_constant<int, RPL>{});
          } else {
            // longer columns in global memory (L2): a simple strided loop the compiler unrolls, so
            // many loads are in flight
            double w = l8 == 0 ? x : 0.0;
#pragma unroll 8
            for (int r = 1 + l8; r < len; r += GS) w = fma(cp[r] * scal, col[r], w);
            w = gsum(w);
            w *= tau;
            x -= w;  // the updated row-j entry (identical in the lanes)
            if (l8 == 0) col[0] = x;
#pragma unroll 8
            for (int rr = 1 + l8; rr < len; rr += GS) col[rr] = fma(-w, cp[rr] * scal, col[rr]);
          }
          __syncwarp(gmask);
        }
        if (a.pivot) {
          // xLAQP2 downdating on squared norms (vn1 = ||.||^2, vn2 = ||.||^2 at the last
          // recompute): LAPACK's temp = max(0, 1 - x^2/vn1), vn1 <- vn1 temp and the recompute
          // test temp vn1/vn2 <= tol3z, written as vn1' = max(0, vn1 - x^2), vn1'/vn2 <= tol3z
          // (equal in exact arithmetic; two dependent operations instead of five).
          if (n1 != 0.0) {
            double nn = fma(-x, x, n1);
            nn = nn < 0.0 ? 0.0 : nn;
            if (nn * r2 <= TOL3Z) {
              if (DEFER && tau != 0.0) {  // the recomputed norm needs the updated rows now
                __syncwarp(gmask);
                const double ws = wsbuf[li];
                for (int rr = 1 + l8; rr < len; rr += GS) col[rr] = fma(-ws, cp[rr], col[rr]);
                __syncwarp(gmask);
                if (l8 == 0) wsbuf[li] = 0.0;
              }
              double ss = 0.0;
              for (int rr = 1 + l8; rr < len; rr += GS) ss = fma(col[rr], col[rr], ss);
              ss = gsum(ss);
              n1 = (j + 1 < rows) ? ss : 0.0;
              if (l8 == 0) rvn2[li] = n1 != 0.0 ? 1.0 / n1 : 0.0;
            } else {
              n1 = nn;
            }
            __syncwarp(gmask);
            if (l8 == 0) vn1[li] = n1;
          }
          if (better(n1, gi, best.v, best.i)) { best.v = n1; best.i = gi; }
        }
      }
    }
    {
      Best wb = warp_best(best);
      if (lane == 0) { s_bv[par ^ 1][warp] = wb.v; s_bi[par ^ 1][warp] = wb.i; }
    }
    __syncthreads();
    stamp(3);
    if (DEFER) {
      // every warp derives the CTA's candidate; warp 0 completes its update and publishes it,
      // then all groups complete the other columns (before the next step's fetch barrier)
      const Best cb = cta_best(par ^ 1);
      const int lbest = cb.i != 0x7fffffff ? (cb.i - b) / G : -1;
      auto finish = [&](int li, int l0, int stride) {
        const double ws = wsbuf[li];
        if (ws == 0.0) return;
        double *cab = colptr(li);
        for (int r = j + 1 + l0; r < rows; r += stride) cab[r] = fma(-ws, cp[r - j], cab[r]);
      };
      if (warp == 0) {
        const double wsb = (lbest >= 0 && tau != 0.0) ? wsbuf[lbest] : 0.0;
        if (wsb != 0.0 && j + 1 < a.steps) {
          // the candidate's deferred update fused with its publish: rows j+1.. updated, stored
          // back and sent in one pass (plus their sum of squares below row j+1 and the record)
          const int jn = j + 1, par2 = jn & 1;
          const unsigned tag = (a.epoch << 16) | ((unsigned)jn + 1u);
          double *cab = colptr(lbest);
          unsigned long long *dst = a.cand + ((int64_t)par2 * G + b) * (rows + 1) * 2;
          if (lane == 0) {   // the record first (see publish)
            const unsigned long long vb = (unsigned long long)__double_as_longlong(cb.v);
            unsigned long long *rc = a.rec + ((int64_t)par2 * G + b) * 4;
            st_x2(rc, pack((unsigned)(vb >> 32), tag), pack((unsigned)vb, tag));
            st_x1(rc + 2, pack((unsigned)cb.i, tag));
          }
          cstamp(jn, 3);
          double s2 = 0.0;
          for (int r = jn + lane; r < rows; r += 32) {
            const double v = fma(-wsb, cp[r - j], cab[r]);
            cab[r] = v;
            if (r > jn) s2 = fma(v, v, s2);
            const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
            st_x2(dst + 2 * (r - jn), pack((unsigned)bits, tag), pack((unsigned)(bits >> 32), tag));
          }
          s2 = warp_sum(s2);
          if (lane == 0) {
            const unsigned long long sb = (unsigned long long)__double_as_longlong(s2);
            st_x2(dst + 2 * (rows - jn), pack((unsigned)sb, tag), pack((unsigned)(sb >> 32), tag));
          }
        } else {
          if (wsb != 0.0) finish(lbest, lane, 32);
          __syncwarp();
          if (j + 1 < a.steps) publish(j + 1, cb);
        }
      }
      if (tau != 0.0 && !(a.w0free && warp == 0)) {
        // w0free: warp 0 polls the next step's records while warps 1.. finish its columns (measured
        // C2-shaped 110 x 4096: 565 -> 521 us; 272 x 8192: 1870 -> 1649 us)
        const int g8 = lane >> 3, l8 = lane & 7;
        const int w = a.w0free ? warp - 1 : warp, nw = a.w0free ? wpb - 1 : wpb;
        for (int li = w * 4 + g8; li < nown; li += nw * 4)
          if (li != lbest && b + li * G != p && !done_l[li]) finish(li, l8, 8);
      }
    } else if (GRID && warp == 0 && j + 1 < a.steps) {
      publish(j + 1, cta_best(par ^ 1));
    }
    // the reflector store, off the exchange's critical path: CTA j mod G, its last warp, after
    // the publish (cp stays valid until the next step's fetch barrier).  Measured: written by
    // CTA 0 before its update it delayed every step's slowest CTA by ~1000 cycles.
    if (b == j % G && warp == wpb - 1) {
      double *vs = a.Vst + (int64_t)j * rows;
      for (int r = lane; r < rows; r += 32) vs[r] = (r < j) ? 0.0 : (r == j ? 1.0 : cp[r - j] * scal);
      if (lane == 0) { a.tau[j] = tau; a.beta[j] = beta; a.perm[j] = p; }
    }
  }
  __syncthreads();
  if (SMEMC)
    for (int li = 0; li < nown; ++li)
      for (int r = threadIdx.x; r < rows; r += blockDim.x) a.M[(int64_t)(b + li * G) * a.ldm + r] = colbuf[(int64_t)li * rs + r];
}

// Small matrices (rows, cols <= 32, e.g. C1's 25 x 25 factor of the tail): the same factorisation
// as hh_engine_kernel (pivot rule, xLARFG reflector, xLAQP2 downdating on squared norms, the
// same outputs in M, Vst, tau, beta, perm, done) by ONE warp with lane c holding column c in
// registers: the pivot column is broadcast by shuffles, and a step has no barrier at all
// (the one-CTA engine spent ~4000 cycles per step on barriers and slot reductions).
__global__ void __launch_bounds__(32, 1) hh_warp_kernel(EngineArgs a) {
  const int lane = threadIdx.x, rows = a.rows, cols = a.cols;
  const bool own = lane < cols;
  double col[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) col[r] = (own && r < rows) ? a.M[(int64_t)lane * a.ldm + r] : 0.0;
  double n1 = 0.0, r2 = 0.0;
  bool done = !own;
  if (own) {
#pragma unroll
    for (int r = 0; r < 32; ++r) n1 = fma(col[r], col[r], n1);
    r2 = n1 != 0.0 ? 1.0 / n1 : 0.0;
    a.done[lane] = 0;
  }
  for (int j = 0; j < a.steps; ++j) {
    int p = j;
    if (a.pivot) {
      const Best c = warp_best(done ? Best{-1.0, 0x7fffffff} : Best{n1, lane});
      p = c.i;
    }
    // the pivot column (all rows; rows < j are R entries and not used below)
    double x[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) x[r] = __shfl_sync(0xffffffffu, col[r], p);
    // reflector, identically in every lane
    double sq[4] = {0.0, 0.0, 0.0, 0.0};  // four chains: the single warp is latency-bound
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r > j && r < rows) sq[r & 3] = fma(x[r], x[r], sq[r & 3]);
    const double xn2 = (sq[0] + sq[1]) + (sq[2] + sq[3]);
    double alpha = 0.0;
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r == j) alpha = x[r];
    double tau, beta, scal;
    if (xn2 == 0.0) {
      tau = 0.0; beta = alpha; scal = 0.0;
    } else {
      beta = -copysign(fast_sqrt(fma(alpha, alpha, xn2)), alpha);
      const double amb = alpha - beta;
      const double rinv = fast_rcp(beta * amb);
      tau = -amb * amb * rinv;
      scal = beta * rinv;
    }
    // outputs of the step: reflector column j (lane r writes row r), tau, beta, perm, done
    {
      double xr = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (lane == r) xr = x[r];
      if (lane < rows) a.Vst[(int64_t)j * rows + lane] = lane < j ? 0.0 : (lane == j ? 1.0 : xr * scal);
      if (lane == 0) { a.tau[j] = tau; a.beta[j] = beta; a.perm[j] = p; a.done[p] = 1; }
    }
    if (lane == p) done = true;
    // apply H_j to every other live column, then downdate its norm
    if (!done && tau != 0.0) {
      double dd[4] = {0.0, 0.0, 0.0, 0.0}, xj = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (r > j && r < rows) dd[r & 3] = fma(x[r], col[r], dd[r & 3]);
        if (r == j) xj = col[r];
      }
      const double w = tau * fma(scal, (dd[0] + dd[1]) + (dd[2] + dd[3]), xj);
      const double ws = w * scal;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (r == j) col[r] = xj - w;
        else if (r > j && r < rows) col[r] = fma(-ws, x[r], col[r]);
      }
    }
    if (!done && a.pivot && n1 != 0.0) {
      double xj = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (r == j) xj = col[r];
      double nn = fma(-xj, xj, n1);
      nn = nn < 0.0 ? 0.0 : nn;
      if (nn * r2 <= TOL3Z) {  // xLAQP2 recompute
        double ss = 0.0;
#pragma unroll
        for (int r = 0; r < 32; ++r)
          if (r > j && r < rows) ss = fma(col[r], col[r], ss);
        n1 = (j + 1 < rows) ? ss : 0.0;
        r2 = n1 != 0.0 ? 1.0 / n1 : 0.0;
      } else {
        n1 = nn;
      }
    }
  }
  if (own)
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r < rows) a.M[(int64_t)lane * a.ldm + r] = col[r];
}

// perm[steps..cols) = not-pivoted columns in ascending original order (single CTA scan).
__global__ void compact_kernel(int cols, int steps, const int *done, int64_t *perm) {
  // each thread owns a run of CPT consecutive columns: all flags are loaded before the scan (one
  // memory round trip instead of one per 1024-column chunk), then a single block scan of the
  // per-thread counts places every run
  constexpr int CPT = 16;
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c0 = 0; c0 < cols; c0 += CPT * (int)blockDim.x) {
    const int first = c0 + threadIdx.x * CPT;
    int fl[CPT];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
      fl[u] = (first + u < cols) ? !done[first + u] : 0;
      cnt += fl[u];
    }
    // exclusive scan of cnt over the block (warp shuffles, then warp totals)
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
      if (w < warp) off += wsum[w];
      tot += wsum[w];
    }
    int pos = steps + off + inc - cnt;
#pragma unroll
    for (int u = 0; u < CPT; ++u)
      if (fl[u]) perm[pos++] = first + u;
    __syncthreads();
    steps += tot;  // the next chunk's base (every thread computed the same total)
  }
}

// R (steps x cols) in pivot order, rows signed so that R_ii >= 0; or its transpose.
__global__ void extract_r_kernel(int steps, int cols, const double *M, int64_t ldm, const double *beta,
                                 const int64_t *perm, double *R, int64_t ldr, int transpose) {
  int64_t total = (int64_t)steps * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % steps);
    int t = (int)(e / steps);
    int64_t col = perm[t];
    double val;
    if (t < steps) val = (i < t) ? M[i + col * ldm] : (i == t ? beta[t] : 0.0);
    else val = M[i + col * ldm];
    if (beta[i] < 0.0) val = -val;
    if (transpose) R[t + (int64_t)i * ldr] = val;
    else R[i + (int64_t)t * ldr] = val;
  }
}

// Explicit Q(:, t) = H_0 .. H_t e_t (xORG2R), one warp per column kept in shared memory, then
// signed by sign(beta_t).  The reflectors are staged in shared memory when they fit.
// QSMEM false (very tall Q): the column is accumulated in place in Q itself.
template <bool VSMEM, bool QSMEM>
__global__ void form_q_kernel(int rows, int steps, const double *Vst, const double *tau, const double *beta,
                              double *Q, int64_t ldq) {
  extern __shared__ __align__(16) double fsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double *vs = fsm;
  double *qs = fsm + (VSMEM ? (int64_t)rows * steps : 0) + (int64_t)warp * rows;
  __shared__ double taus[1056];
  if (VSMEM) {
    // stage only the reflectors this CTA's columns use (j <= its largest t), 16-byte loads,
    // unrolled so many are in flight (one CTA streams up to rows x steps doubles)
    const int tlast = min(steps - 1, (int)((gridDim.x * nw) * ((steps - 1) / (gridDim.x * nw)) +
                                           (blockIdx.x + 1) * nw - 1));
    const int64_t cnt = (int64_t)rows * (tlast + 1), cnt2 = cnt >> 1;
    const double2 *src = reinterpret_cast<const double2 *>(Vst);
    double2 *dst = reinterpret_cast<double2 *>(vs);
#pragma unroll 8
    for (int64_t e = threadIdx.x; e < cnt2; e += blockDim.x) dst[e] = src[e];
    if ((cnt & 1) && threadIdx.x == 0) vs[cnt - 1] = Vst[cnt - 1];
  }
  for (int e = threadIdx.x; e < steps && e < 1056; e += blockDim.x) taus[e] = tau[e];
  __syncthreads();
  const double *V = VSMEM ? vs : Vst;
  const int W = gridDim.x * nw;
  for (int t = blockIdx.x * nw + warp; t < steps; t += W) {
    double *out = Q + (int64_t)t * ldq;
    double *q = QSMEM ? qs : out;
    for (int r = lane; r < rows; r += 32) q[r] = (r == t) ? 1.0 : 0.0;
    __syncwarp();
    for (int j = t; j >= 0; --j) {
      const double tj = taus[j];
      if (tj == 0.0) continue;
      const double *v = V + (int64_t)j * rows;
      double w = 0.0;
      for (int r = j + lane; r < rows; r += 32) w = fma(v[r], q[r], w);
      w = warp_sum(w) * tj;
      for (int r = j + lane; r < rows; r += 32) q[r] = fma(-w, v[r], q[r]);
      __syncwarp();
    }
    const double sg = beta[t] < 0.0 ? -1.0 : 1.0;
    for (int r = lane; r < rows; r += 32) out[r] = sg * q[r];
    __syncwarp();
  }
}

__global__ void copy_perm_kernel(int64_t count, const int64_t *src, int64_t *dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace

void hh_carve(Arena &a, HHScratch &s, int64_t rows, int64_t cols, int num_sms, int64_t steps) {
  steps = steps < 0 ? std::min(rows, cols) : std::min(steps, std::min(rows, cols));
  s.max_steps = steps;
  s.max_rows = rows;
  s.max_cols = cols;
  s.max_slots = num_sms;
  s.Vst = a.take<double>(rows * steps);
  s.tau = a.take<double>(steps);
  s.beta = a.take<double>(steps);
  s.rec = a.take<unsigned long long>(2 * s.max_slots * 4);
  s.cand = a.take<unsigned long long>(2 * s.max_slots * (rows + 1) * 2);
  s.done = a.take<int>(cols);
  s.perm = a.take<int64_t>(cols);
}

template <bool GRID, bool SMEMC>
static void set_engine_attr() {
  smem_attr((const void *)hh_engine_kernel<GRID, SMEMC>, 220 * 1024);
}

void hh_factor(Ctx &c, HHScratch &s, int64_t rows, int64_t cols, double *M, int64_t ldm, bool pivot, int64_t steps) {
  steps = steps < 0 ? std::min(rows, cols) : std::min(steps, std::min(rows, cols));
  if (rows > s.max_rows || cols > s.max_cols || steps > s.max_steps)
    throw std::runtime_error("hh_factor: scratch too small");
  constexpr size_t SMEM_MAX = 220 * 1024;
  EngineArgs a;
  a.M = M; a.ldm = ldm; a.rows = (int)rows; a.cols = (int)cols;
  a.steps = (int)steps; a.pivot = pivot ? 1 : 0;
  a.Vst = s.Vst; a.tau = s.tau; a.beta = s.beta; a.rec = s.rec; a.cand = s.cand; a.done = s.done; a.perm = s.perm;
  a.epoch = 0;
  a.trace = c.trace;
  {  // RQLP_ENGINE_POLL_WARPS (measurement switch): warps polling the exchange records
    static int np = -1;
    if (np < 0) {
      const char *e = getenv("RQLP_ENGINE_POLL_WARPS");
      np = e ? std::max(1, atoi(e)) : 1;
    }
    a.npoll = np;
    static int w0f = -1;   // RQLP_ENGINE_W0FREE (measurement switch)
    if (w0f < 0) {
      const char *e = getenv("RQLP_ENGINE_W0FREE");
      w0f = e ? atoi(e) : 1;
    }
    a.w0free = w0f;
    const char *tr = getenv("RQLP_ENGINE_TRACE");
    a.gtime = tr && tr[0] == '2';
  }
  auto smem_for = [&](int64_t owned, bool cached) {
    const int64_t rs = round_up(rows, 2), op = round_up(owned, 2);
    return (size_t)(rs + 3 * op + (cached ? owned * rs : 0)) * 8 + (size_t)owned * 4 + 64;
  };
  if (rows <= 32 && cols <= 32) {
    // one warp, columns in registers (no barriers): C1's 25 x 25 factor 52 -> ~6 us
    hh_warp_kernel<<<1, 32, 0, c.stream>>>(a);
    RQLP_LAUNCHED(c);
  } else if (cols <= 256 && smem_for(cols, true) <= SMEM_MAX) {
    // whole matrix in one CTA's shared memory: no global exchange at all; the block is sized to
    // one 8-lane group per column (cheaper barriers for small matrices: C1's 25 x 25 factor
    // 64 -> 56 us).  Wider matrices go to the grid: an 8-lane group's column update is a
    // ~2000-cycle dependency chain, so one CTA with several columns per group loses to the
    // ~8000-cycle grid exchange (measured: 25 x 800 on one CTA 577 us, on 100 CTAs 100 us).
    a.owned_max = (int)cols;
    const int threads = (int)std::min<int64_t>(1024, std::max<int64_t>(64, round_up(cols * 8, 32)));
    set_engine_attr<false, true>();
    hh_engine_kernel<false, true><<<1, threads, smem_for(cols, true), c.stream>>>(a);
    RQLP_LAUNCHED(c);
  } else {
    // enough CTAs that each owns >= 8 columns (fewer records to exchange), at most one per SM
    // (measured: 8 to 64 columns per CTA are within 5% on C2's 110 x 4096 B)
    const int G = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(c.num_sms, s.max_slots), ceil_div(cols, 8)));
    const int64_t owned = ceil_div(cols, G);
    const bool cached = smem_for(owned, true) <= SMEM_MAX;
    if (!cached && smem_for(owned, false) > SMEM_MAX) throw std::runtime_error("hh_factor: too many rows");
    a.owned_max = (int)owned;
    const size_t smem = smem_for(owned, cached);
    // zero the exchange buffers every launch: tags are then step+1 of THIS launch only (robust
    // against recycled workspaces; a memset node when captured in a CUDA graph)
    RQLP_CUDA(cudaMemsetAsync(s.rec, 0, sizeof(unsigned long long) * 2 * G * 4, c.stream));
    RQLP_CUDA(cudaMemsetAsync(s.cand, 0, sizeof(unsigned long long) * 2 * G * (rows + 1) * 2, c.stream));
    a.epoch = 0;
    // co-residency of all G CTAs is required (they exchange every step): cooperative launch
    // through cudaLaunchKernelEx (capturable into CUDA graphs)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    // cached columns: 8-lane groups, 256 threads when one group per column suffices (fewer
    // warps at the step's barriers: C2 1.63 -> 1.62 ms), else 512; global-memory columns: a warp
    // per column, 256 threads (registers hold the column)
    cfg.blockDim = dim3(cached ? (owned <= 32 ? 256 : 512) : 384);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cached) {
      set_engine_attr<true, true>();
      RQLP_CUDA(cudaLaunchKernelEx(&cfg, hh_engine_kernel<true, true>, a));
    } else {
      set_engine_attr<true, false>();
      RQLP_CUDA(cudaLaunchKernelEx(&cfg, hh_engine_kernel<true, false>, a));
    }
    RQLP_LAUNCHED(c);
  }
  if (cols > a.steps) {
    compact_kernel<<<1, 1024, 0, c.stream>>>(a.cols, a.steps, s.done, s.perm);
    RQLP_LAUNCHED(c);
  }
}

void hh_extract_r(Ctx &c, HHScratch &s, int64_t rows, int64_t cols, const double *M, int64_t ldm, double *R,
                  int64_t ldr, bool transpose, int64_t steps) {
  steps = steps < 0 ? std::min(rows, cols) : std::min(steps, std::min(rows, cols));
  int64_t total = steps * cols;
  int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)c.num_sms * 8);
  extract_r_kernel<<<std::max(grid, 1), 256, 0, c.stream>>>((int)steps, (int)cols, M, ldm, s.beta, s.perm, R, ldr,
                                                            transpose ? 1 : 0);
  RQLP_LAUNCHED(c);
}

void hh_form_q(Ctx &c, HHScratch &s, int64_t rows, int64_t cols, double *Q, int64_t ldq, int64_t steps) {
  steps = steps < 0 ? std::min(rows, cols) : std::min(steps, std::min(rows, cols));
  if (steps > 1056) throw std::runtime_error("hh_form_q: more than 1056 reflectors");
  const size_t vbytes = (size_t)rows * steps * 8;
  // warps per CTA: 8, fewer when a column per warp does not fit in 200 KB (tall Q), and the
  // column lives in Q itself beyond that
  int nw = (int)std::max<int64_t>(1, std::min<int64_t>(8, (200 * 1024) / ((int64_t)rows * 8)));
  const bool qsmem = (size_t)rows * 8 <= 200 * 1024;
  if (!qsmem) nw = 8;
  const size_t qbytes = qsmem ? (size_t)nw * rows * 8 : 0;
  smem_attr((const void *)form_q_kernel<true, true>, 200 * 1024);
  smem_attr((const void *)form_q_kernel<false, true>, 200 * 1024);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(steps, nw), (int64_t)c.num_sms));
  if (qsmem && vbytes + qbytes <= 190 * 1024) {
    form_q_kernel<true, true><<<grid, nw * 32, vbytes + qbytes, c.stream>>>((int)rows, (int)steps, s.Vst, s.tau,
                                                                           s.beta, Q, ldq);
  } else if (qsmem) {
    form_q_kernel<false, true><<<grid, nw * 32, qbytes, c.stream>>>((int)rows, (int)steps, s.Vst, s.tau, s.beta, Q,
                                                                    ldq);
  } else {
    form_q_kernel<false, false><<<grid, nw * 32, 0, c.stream>>>((int)rows, (int)steps, s.Vst, s.tau, s.beta, Q, ldq);
  }
  RQLP_LAUNCHED(c);
}

void hh_copy_perm(Ctx &c, HHScratch &s, int64_t count, int64_t *dst) {
  if (!dst || count <= 0) return;
  copy_perm_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 256), 1024)), 256, 0, c.stream>>>(
      count, s.perm, dst);
  RQLP_LAUNCHED(c);
}

}  // namespace rqlpk
