// dense.cu -- small elementwise / data-movement kernels and the validation residual.
#include "internal.cuh"

namespace rqlpk {

void gemm_generic_ex(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                     int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc, double *partials,
                     size_t partial_elems, bool trans_out, const unsigned *cond, unsigned cond_mask);

namespace {

// D = S (or S^T when transpose); S == nullptr fills D with zeros.
__global__ void copy_kernel(int64_t rows, int64_t cols, const double *S, int64_t lds, double *D, int64_t ldd,
                            int transpose, const unsigned *cond, unsigned cond_mask) {
  if (cond && ((*cond) & cond_mask) == 0) return;
  int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e % rows, j = e / rows;
    double v = 0.0;
    if (S) v = transpose ? S[j + i * lds] : S[i + j * lds];
    D[i + j * ldd] = v;
  }
}

__global__ void fill_kernel(int64_t rows, int64_t cols, double *D, int64_t ldd, double diag, double off) {
  int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e % rows, j = e / rows;
    D[i + j * ldd] = (i == j) ? diag : off;
  }
}

__global__ void zero_u32_kernel(unsigned *p, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0u;
}

// part[b] = sum of squares of this block's slice of X (rows x cols, ld), fixed order.
__global__ void sumsq_kernel(int64_t rows, int64_t cols, const double *X, int64_t ldx, double *part) {
  __shared__ double red[32];
  double s = 0.0;
  int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double v = X[e % rows + (e / rows) * ldx];
    s = fma(v, v, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void accumulate_kernel(int nparts, const double *part, double *out, int first) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = first ? 0.0 : *out;
    for (int i = 0; i < nparts; ++i) t += part[i];
    *out = t;
  }
}

}  // namespace

void launch_copy(Ctx &c, int64_t rows, int64_t cols, const double *S, int64_t lds, double *D, int64_t ldd,
                 bool transpose, const unsigned *cond, unsigned cond_mask) {
  if (rows <= 0 || cols <= 0) return;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows * cols, 256), (int64_t)c.num_sms * 16));
  copy_kernel<<<grid, 256, 0, c.stream>>>(rows, cols, S, lds, D, ldd, transpose ? 1 : 0, cond, cond_mask);
  RQLP_LAUNCHED(c);
}

void launch_fill(Ctx &c, int64_t rows, int64_t cols, double *D, int64_t ldd, double diag, double off) {
  if (rows <= 0 || cols <= 0) return;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows * cols, 256), (int64_t)c.num_sms * 16));
  fill_kernel<<<grid, 256, 0, c.stream>>>(rows, cols, D, ldd, diag, off);
  RQLP_LAUNCHED(c);
}

void launch_zero_u32(Ctx &c, unsigned *p, int64_t count) {
  zero_u32_kernel<<<1, 256, 0, c.stream>>>(p, count);
  RQLP_LAUNCHED(c);
}

// ||A - Q M||_F^2 for A m x n, Q m x l, M l x n (M = T P^T), in row chunks of `chunk` rows
// using `partials` (chunk x n doubles + 1024) as the difference buffer.  Validation only.
void residual_sq(Ctx &c, int64_t m, int64_t n, int64_t l, const double *A, int64_t lda, const double *Q, int64_t ldq,
                 const double *M, int64_t ldmm, double *partials, double *out) {
  const int64_t chunk = 4096;
  double *D = partials;
  double *part = partials + chunk * n;
  const int nb = 512;
  for (int64_t r0 = 0; r0 < m; r0 += chunk) {
    int64_t rc = std::min(chunk, m - r0);
    launch_copy(c, rc, n, A + r0, lda, D, rc, false, nullptr, 0);
    gemm_generic_ex(c, false, false, rc, n, l, -1.0, Q + r0, ldq, M, ldmm, 1.0, D, rc, nullptr, 0, false, nullptr, 0);
    sumsq_kernel<<<nb, 256, 0, c.stream>>>(rc, n, D, rc, part);
    RQLP_LAUNCHED(c);
    accumulate_kernel<<<1, 32, 0, c.stream>>>(nb, part, out, r0 == 0 ? 1 : 0);
    RQLP_LAUNCHED(c);
  }
}

}  // namespace rqlpk

namespace rqlpk {
namespace {

// part[b] = sum of squares of the columns b, b + gridDim.x, ... of X (rows x cols, ld), fixed order.
__global__ void colsumsq_kernel(int64_t rows, int64_t cols, const double *__restrict__ X, int64_t ldx,
                                double *part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t j = blockIdx.x; j < cols; j += gridDim.x) {
    const double *x = X + j * ldx;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) s = fma(x[i], x[i], s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

// *out (+)= sum of the parts: thread t sums parts t, t + 256, ... in order, then a fixed tree.
__global__ void __launch_bounds__(256) accumulate_parts_kernel(int nparts, const double *part, double *out, int first) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 256) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = first ? red[0] : *out + red[0];
}

}  // namespace

// part[b] = sum of squares of the column range [b cpb, (b+1) cpb) of X: each warp takes a column,
// 16-byte loads with four accumulation chains (the large-input form: a whole A when the fused
// ||A||^2 cannot ride on the sketch pass -- its tile width or alignment -- read at HBM speed).
__global__ void __launch_bounds__(256) colrange_sumsq_kernel(int64_t rows, int64_t cols, int64_t cpb,
                                                             const double *__restrict__ X, int64_t ldx, double *part) {
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j0 = (int64_t)blockIdx.x * cpb, j1 = min(cols, j0 + cpb);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  const bool vec = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  for (int64_t j = j0 + warp; j < j1; j += 8) {
    const double *x = X + j * ldx;
    int64_t i = 0;
    if (vec) {
      const double2 *x2 = reinterpret_cast<const double2 *>(x);
      const int64_t h = rows >> 1;
      int64_t t = lane;
      for (; t + 32 < h; t += 64) {
        const double2 a = x2[t], b = x2[t + 32];
        s0 = fma(a.x, a.x, s0);
        s1 = fma(a.y, a.y, s1);
        s2 = fma(b.x, b.x, s2);
        s3 = fma(b.y, b.y, s3);
      }
      if (t < h) {
        const double2 a = x2[t];
        s0 = fma(a.x, a.x, s0);
        s1 = fma(a.y, a.y, s1);
      }
      i = 2 * h;
    }
    for (int64_t r = i + lane; r < rows; r += 32) s2 = fma(x[r], x[r], s2);
  }
  double s = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

// *out (+)= ||X||_F^2 (X rows x cols, ld), deterministic fixed-order reduction; part >= 1024 doubles.
void fro2_accumulate(Ctx &c, int64_t rows, int64_t cols, const double *X, int64_t ldx, double *part, double *out,
                     bool first) {
  int nb;
  if (rows * cols >= ((int64_t)1 << 22)) {   // large: column ranges over ~8 CTAs per SM
    nb = (int)std::max<int64_t>(1, std::min<int64_t>({cols, (int64_t)c.num_sms * 8, 1024}));
    const int64_t cpb = ceil_div(cols, nb);
    nb = (int)ceil_div(cols, cpb);
    colrange_sumsq_kernel<<<nb, 256, 0, c.stream>>>(rows, cols, cpb, X, ldx, part);
  } else {
    nb = (int)std::max<int64_t>(1, std::min<int64_t>(cols, 1024));
    colsumsq_kernel<<<nb, 256, 0, c.stream>>>(rows, cols, X, ldx, part);
  }
  RQLP_LAUNCHED(c);
  accumulate_parts_kernel<<<1, 256, 0, c.stream>>>(nb, part, out, first ? 1 : 0);
  RQLP_LAUNCHED(c);
}

}  // namespace rqlpk
