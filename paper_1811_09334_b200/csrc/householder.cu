// householder.cu -- Householder QR engine with optional column pivoting (the CPQR of the tail).
//
// Alg.1 l.5 "[Q0, R0, Π0] = cpqr(B)" and l.6 "cpqr(R0^T)"; Alg.2
// l.7 unpivoted "qr([R^(i-1)]^T)".  The pivot rule (reading R5): at step j pick
// the remaining column with the largest downdated norm, ties to the lowest ORIGINAL column
// index; norms are downdated with the LAPACK xLAQP2 rule and recomputed when
// t (vn1/vn2)^2 <= sqrt(2^-53).  The paper names no pivot rule; SURVEY §8(c.1) step 6 fixes it.
//
// B200 design: one persistent cooperative kernel runs all s = min(rows, cols) strictly
// sequential steps.  Columns stay where they are (no physical swaps): column i is owned by
// warp (i mod W) of the grid, which keeps its norms and applies every reflector to it; a step
// costs one software grid barrier.  Every CTA recomputes the step's reflector from the pivot
// column with the same fixed-order reduction, so all CTAs hold bit-identical v, τ without a
// second barrier; one CTA stores the reflector.  The matrix lives in global memory (L2-resident
// for the tail's sizes: B is l x n <= 1056 x 16384).  Small matrices run the same code as a
// single 1024-thread CTA whose "grid barrier" is __syncthreads.
#include "internal.cuh"

namespace rqlpk {
namespace {

constexpr double TOL3Z = 1.0536712127723509e-08;  // sqrt(2^-53), LAPACK dlaqp2 tol3z

struct Best {
  double v;
  int i;
};
__device__ __forceinline__ bool better(double v, int i, double bv, int bi) { return v > bv || (v == bv && i < bi); }

__device__ __forceinline__ Best warp_best(Best b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, b.v, o);
    int oi = __shfl_xor_sync(0xffffffffu, b.i, o);
    if (better(ov, oi, b.v, b.i)) { b.v = ov; b.i = oi; }
  }
  return b;
}

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

__device__ void grid_sync(unsigned *count, volatile unsigned *gen) {
  __syncthreads();
  if (gridDim.x == 1) return;
  if (threadIdx.x == 0) {
    unsigned g = *gen;
    __threadfence();
    unsigned arrived = atomicAdd(count, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd((unsigned *)gen, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Block-wide sum in a fixed order (identical in every CTA for identical inputs).
__device__ double block_sum(double s, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  s = warp_sum(s);
  __syncthreads();
  if (lane == 0) red[warp] = s;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}

__device__ double warp_norm(const double *x, int64_t len) {
  double s = 0.0;
  for (int64_t r = threadIdx.x & 31; r < len; r += 32) s = fma(x[r], x[r], s);
  return sqrt(warp_sum(s));
}

struct EngineArgs {
  double *M;
  int64_t ldm;
  int rows, cols, steps, pivot;
  double *Vst;  // rows x steps, ld rows
  double *tau, *beta, *vn1, *vn2, *slot_val;
  int *done, *slot_idx;
  int64_t *perm;
  unsigned *bar;  // [count, gen]
};

__global__ void __launch_bounds__(1024) hh_engine_kernel(EngineArgs a) {
  extern __shared__ double smem[];
  double *v = smem;                 // rows
  double *red = smem + a.rows;      // 32
  __shared__ double s_bv[32];
  __shared__ int s_bi[32];
  __shared__ int s_p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int W = gridDim.x * wpb, gw = blockIdx.x * wpb + warp;
  unsigned *bcount = a.bar;
  volatile unsigned *bgen = a.bar + 1;

  // ---- init: column norms (pivoting) and candidate slots
  Best best{-1.0, 0x7fffffff};
  for (int i = gw; i < a.cols; i += W) {
    if (lane == 0) a.done[i] = 0;
    if (a.pivot) {
      double nrm = warp_norm(a.M + (int64_t)i * a.ldm, a.rows);
      if (lane == 0) { a.vn1[i] = nrm; a.vn2[i] = nrm; }
      if (better(nrm, i, best.v, best.i)) { best.v = nrm; best.i = i; }
    }
  }
  auto publish = [&]() {
    if (!a.pivot) return;
    Best b = warp_best(best);
    if (lane == 0) { s_bv[warp] = b.v; s_bi[warp] = b.i; }
    __syncthreads();
    if (threadIdx.x == 0) {
      Best c{-1.0, 0x7fffffff};
      for (int w = 0; w < wpb; ++w)
        if (better(s_bv[w], s_bi[w], c.v, c.i)) { c.v = s_bv[w]; c.i = s_bi[w]; }
      a.slot_val[blockIdx.x] = c.v;
      a.slot_idx[blockIdx.x] = c.i;
    }
  };
  publish();
  grid_sync(bcount, bgen);

  for (int j = 0; j < a.steps; ++j) {
    // ---- 1. pivot: global argmax over the CTA slots (exact, order independent)
    if (warp == 0) {
      int p = j;
      if (a.pivot) {
        Best c{-1.0, 0x7fffffff};
        for (int s = lane; s < (int)gridDim.x; s += 32) {
          double sv = __ldcg(a.slot_val + s);
          int si = __ldcg(a.slot_idx + s);
          if (better(sv, si, c.v, c.i)) { c.v = sv; c.i = si; }
        }
        c = warp_best(c);
        p = c.i;
      }
      if (lane == 0) s_p = p;
    }
    __syncthreads();
    const int p = s_p;
    const double *colp = a.M + (int64_t)p * a.ldm;
    const int len = a.rows - j;

    // ---- 2. reflector (xLARFG) from column p, rows j.., identical in every CTA
    double part = 0.0;
    for (int r = j + 1 + threadIdx.x; r < a.rows; r += blockDim.x) {
      double x = __ldcg(colp + r);
      part = fma(x, x, part);
    }
    double xn2 = block_sum(part, red);
    double alpha = __ldcg(colp + j);
    double xnorm = sqrt(xn2);
    double tau, beta, scal;
    if (xnorm == 0.0) {
      tau = 0.0; beta = alpha; scal = 0.0;
    } else {
      beta = -copysign(sqrt(alpha * alpha + xnorm * xnorm), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int r = threadIdx.x; r < len; r += blockDim.x) v[r] = (r == 0) ? 1.0 : __ldcg(colp + j + r) * scal;
    __syncthreads();
    if (blockIdx.x == 0) {
      double *vs = a.Vst + (int64_t)j * a.rows;
      for (int r = threadIdx.x; r < a.rows; r += blockDim.x) vs[r] = (r < j) ? 0.0 : v[r - j];
      if (threadIdx.x == 0) { a.tau[j] = tau; a.beta[j] = beta; a.perm[j] = p; }
    }

    // ---- 3. apply H_j to every owned, not yet pivoted column; downdate its norm
    best = Best{-1.0, 0x7fffffff};
    for (int i = gw; i < a.cols; i += W) {
      if (i == p) {
        if (lane == 0) a.done[i] = 1;
        continue;
      }
      if (a.done[i]) continue;
      double *col = a.M + (int64_t)i * a.ldm + j;
      if (tau != 0.0) {
        double w = 0.0;
        for (int r = lane; r < len; r += 32) w = fma(v[r], col[r], w);
        w = warp_sum(w) * tau;
        for (int r = lane; r < len; r += 32) col[r] = fma(-w, v[r], col[r]);
        __syncwarp();
      }
      if (a.pivot) {
        double n1 = a.vn1[i];
        if (n1 != 0.0) {
          double t = __ddiv_rn(fabs(col[0]), n1);
          t = __dsub_rn(1.0, __dmul_rn(t, t));
          t = t < 0.0 ? 0.0 : t;
          double rr = __ddiv_rn(n1, a.vn2[i]);
          double t2 = __dmul_rn(__dmul_rn(t, rr), rr);
          if (t2 <= TOL3Z) {
            if (j + 1 < a.rows) n1 = warp_norm(col + 1, len - 1);
            else n1 = 0.0;
            if (lane == 0) a.vn2[i] = n1;
          } else {
            n1 = __dmul_rn(n1, __dsqrt_rn(t));
          }
          __syncwarp();
          if (lane == 0) a.vn1[i] = n1;
        }
        if (better(n1, i, best.v, best.i)) { best.v = n1; best.i = i; }
      }
    }
    publish();
    grid_sync(bcount, bgen);
  }
}

// perm[steps..cols) = not-pivoted columns in ascending original order (single CTA scan).
__global__ void compact_kernel(int cols, int steps, const int *done, int64_t *perm) {
  __shared__ int wsum[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = steps;
  __syncthreads();
  for (int c0 = 0; c0 < cols; c0 += blockDim.x) {
    int i = c0 + threadIdx.x;
    int flag = (i < cols && !done[i]) ? 1 : 0;
    // block exclusive scan
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned bal = __ballot_sync(0xffffffffu, flag);
    int pre = __popc(bal & ((1u << lane) - 1));
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    if (flag) perm[base + off + pre] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += wsum[w];
      base += tot;
    }
    __syncthreads();
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

// Explicit Q(:, t) = H_0 .. H_t e_t (xORG2R), one warp per column, then signed by sign(beta_t).
__global__ void form_q_kernel(int rows, int steps, const double *Vst, const double *tau, const double *beta,
                              double *Q, int64_t ldq) {
  const int lane = threadIdx.x & 31;
  const int W = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < steps; t += W) {
    double *q = Q + (int64_t)t * ldq;
    for (int r = lane; r < rows; r += 32) q[r] = (r == t) ? 1.0 : 0.0;
    __syncwarp();
    for (int j = t; j >= 0; --j) {
      double tj = tau[j];
      if (tj == 0.0) continue;
      const double *v = Vst + (int64_t)j * rows;
      double w = 0.0;
      for (int r = j + lane; r < rows; r += 32) w = fma(v[r], q[r], w);
      w = warp_sum(w) * tj;
      for (int r = j + lane; r < rows; r += 32) q[r] = fma(-w, v[r], q[r]);
      __syncwarp();
    }
    if (beta[t] < 0.0)
      for (int r = lane; r < rows; r += 32) q[r] = -q[r];
  }
}

__global__ void copy_perm_kernel(int64_t count, const int64_t *src, int64_t *dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace

void hh_carve(Arena &a, HHScratch &s, int64_t rows, int64_t cols, int num_sms) {
  int64_t steps = std::min(rows, cols);
  s.max_rows = rows;
  s.max_cols = cols;
  s.max_slots = (int64_t)num_sms * 8;
  s.Vst = a.take<double>(rows * steps);
  s.tau = a.take<double>(steps);
  s.beta = a.take<double>(steps);
  s.vn1 = a.take<double>(cols);
  s.vn2 = a.take<double>(cols);
  s.slot_val = a.take<double>(s.max_slots);
  s.slot_idx = a.take<int>(s.max_slots);
  s.done = a.take<int>(cols);
  s.perm = a.take<int64_t>(cols);
}

void hh_factor(Ctx &c, HHScratch &s, int64_t rows, int64_t cols, double *M, int64_t ldm, bool pivot) {
  if (rows > s.max_rows || cols > s.max_cols) throw std::runtime_error("hh_factor: scratch too small");
  EngineArgs a;
  a.M = M; a.ldm = ldm; a.rows = (int)rows; a.cols = (int)cols;
  a.steps = (int)std::min(rows, cols); a.pivot = pivot ? 1 : 0;
  a.Vst = s.Vst; a.tau = s.tau; a.beta = s.beta; a.vn1 = s.vn1; a.vn2 = s.vn2;
  a.slot_val = s.slot_val; a.slot_idx = s.slot_idx; a.done = s.done; a.perm = s.perm;
  a.bar = c.dflags + BAR_COUNT;
  size_t smem = (size_t)(rows + 32) * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    RQLP_CUDA(cudaFuncSetAttribute(hh_engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set = true;
  }
  if (smem > 200 * 1024) throw std::runtime_error("hh_factor: too many rows for the shared reflector buffer");
  RQLP_CUDA(cudaMemsetAsync(c.dflags + BAR_COUNT, 0, sizeof(unsigned), c.stream));
  if (cols <= 2048) {
    hh_engine_kernel<<<1, 1024, smem, c.stream>>>(a);
    RQLP_LAUNCHED(c);
  } else {
    int per_sm = 0;
    RQLP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hh_engine_kernel, 256, smem));
    int grid = std::max(1, std::min(per_sm, 4)) * c.num_sms;
    grid = std::min<int64_t>(grid, s.max_slots);
    void *args[] = {&a};
    RQLP_CUDA(cudaLaunchCooperativeKernel((void *)hh_engine_kernel, grid, 256, args, smem, c.stream));
    RQLP_LAUNCHED(c);
  }
  if (cols > a.steps) {
    compact_kernel<<<1, 1024, 0, c.stream>>>(a.cols, a.steps, s.done, s.perm);
    RQLP_LAUNCHED(c);
  }
}

void hh_extract_r(Ctx &c, HHScratch &s, int64_t rows, int64_t cols, const double *M, int64_t ldm, double *R,
                  int64_t ldr, bool transpose) {
  int64_t steps = std::min(rows, cols);
  int64_t total = steps * cols;
  int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)c.num_sms * 8);
  extract_r_kernel<<<std::max(grid, 1), 256, 0, c.stream>>>((int)steps, (int)cols, M, ldm, s.beta, s.perm, R, ldr,
                                                            transpose ? 1 : 0);
  RQLP_LAUNCHED(c);
}

void hh_form_q(Ctx &c, HHScratch &s, int64_t rows, int64_t cols, double *Q, int64_t ldq) {
  int64_t steps = std::min(rows, cols);
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(steps * 32, 256), (int64_t)c.num_sms * 8));
  form_q_kernel<<<grid, 256, 0, c.stream>>>((int)rows, (int)steps, s.Vst, s.tau, s.beta, Q, ldq);
  RQLP_LAUNCHED(c);
}

void hh_copy_perm(Ctx &c, HHScratch &s, int64_t count, int64_t *dst) {
  if (!dst || count <= 0) return;
  copy_perm_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 256), 1024)), 256, 0, c.stream>>>(
      count, s.perm, dst);
  RQLP_LAUNCHED(c);
}

}  // namespace rqlpk
