// omega.cu -- Ω generator: Philox4x64-10 + Box-Muller with pinned ln / sin / cos.
//
// Alg.1 l.1 "Ω = rand(n, l)  % Gaussian random matrix" -- read as N(0,1)
// (reading R1).  Bit layout: key = (seed, 0); counter = (block, stream=0, 0, 0);
// Ω(i, j) = z_t with t = i + n j, block t/4, lane t%4; uniforms u(x) = ((x>>12) + 0.5) 2^-52;
// (z0, z1) = ρ(cos, sin)(2π u(x1)), ρ = sqrt(-2 ln u(x0)); same for (x2, x3) -> (z2, z3).
// Every floating-point step uses an explicitly rounded intrinsic (__dmul_rn, __fma_rn, ...) so
// the compiler cannot contract or reorder it: the sequence is the DESIGN.md §4 specification.
#include "internal.cuh"

namespace rqlpk {
namespace {

__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    uint64_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
  }
}

__device__ __forceinline__ double u01(uint64_t x) {
  return __dmul_rn(__dadd_rn((double)(x >> 12), 0.5), 0x1p-52);
}

// ln u: u = 2^e f, f in [sqrt(1/2), sqrt(2)); s = (f-1)/(f+1); ln f = 2s + 2s s^2 P(s^2).
__device__ __forceinline__ double pinned_ln(double u) {
  const double C[12] = {0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4,
                        0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
                        0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5, 0x1.47ae147ae147bp-5};
  uint64_t bits = (uint64_t)__double_as_longlong(u);
  int64_t e = (int64_t)((bits >> 52) & 0x7ff) - 1023;
  double f = __longlong_as_double((long long)((bits & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL));
  if (f > 0x1.6a09e667f3bcdp+0) {
    f = __dmul_rn(f, 0.5);
    e += 1;
  }
  double s = __ddiv_rn(__dsub_rn(f, 1.0), __dadd_rn(f, 1.0));
  double z = __dmul_rn(s, s);
  double P = C[11];
#pragma unroll
  for (int i = 10; i >= 0; --i) P = __fma_rn(P, z, C[i]);
  double t = __dadd_rn(s, s);
  double tz = __dmul_rn(t, z);
  double lnf = __fma_rn(tz, P, t);
  double ed = (double)e;
  double lo = __fma_rn(ed, 0x1.a39ef35793c76p-33, lnf);
  return __fma_rn(ed, 0x1.62e42fee00000p-1, lo);
}

__device__ __forceinline__ void pinned_sincos_2pi(uint64_t x, double *so, double *co) {
  const double S[9] = {-0x1.5555555555555p-3, 0x1.1111111111111p-7, -0x1.a01a01a01a01ap-13,
                       0x1.71de3a556c734p-19, -0x1.ae64567f544e4p-26, 0x1.6124613a86d09p-33,
                       -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49, -0x1.2f49b46814157p-57};
  const double Cc[10] = {-0x1.0000000000000p-1, 0x1.5555555555555p-5, -0x1.6c16c16c16c17p-10,
                         0x1.a01a01a01a01ap-16, -0x1.27e4fb7789f5cp-22, 0x1.1eed8eff8d898p-29,
                         -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45, -0x1.6827863b97d97p-53,
                         0x1.e542ba4020225p-62};
  uint64_t K = x >> 12;
  uint64_t q = (K + (1ULL << 49)) >> 50;
  int64_t rk = (int64_t)K - (int64_t)(q << 50);
  double r = __dmul_rn(__dadd_rn((double)rk, 0.5), 0x1p-50);
  double phi = __dmul_rn(r, 0x1.921fb54442d18p+0);
  double z = __dmul_rn(phi, phi);
  double Ps = S[8];
#pragma unroll
  for (int i = 7; i >= 0; --i) Ps = __fma_rn(Ps, z, S[i]);
  double sp = __fma_rn(__dmul_rn(phi, z), Ps, phi);
  double Pc = Cc[9];
#pragma unroll
  for (int i = 8; i >= 0; --i) Pc = __fma_rn(Pc, z, Cc[i]);
  double cp = __fma_rn(z, Pc, 1.0);
  switch (q & 3) {
    case 0: *so = sp; *co = cp; break;
    case 1: *so = cp; *co = -sp; break;
    case 2: *so = -sp; *co = -cp; break;
    default: *so = -cp; *co = sp; break;
  }
}

// One thread per Philox block (4 normals).  Columns [col0, col0 + l) of the n x L matrix Ω are
// written (col0 > 0 is how BRQLP's Ω_j slices are generated: same global t indexing).
__global__ void omega_kernel(int64_t n, int64_t l, int64_t col0, uint64_t seed, double *Om, int64_t ldo) {
  int64_t t_begin = col0 * n, t_end = (col0 + l) * n;
  int64_t b0 = t_begin / 4, b1 = (t_end + 3) / 4;
  for (int64_t b = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < b1;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c[4] = {(uint64_t)b, 0, 0, 0};
    philox4x64_10(c, seed, 0);
    double z[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double ua = u01(c[2 * h]);
      double rho = __dsqrt_rn(__dmul_rn(-2.0, pinned_ln(ua)));
      double s, co;
      pinned_sincos_2pi(c[2 * h + 1], &s, &co);
      z[2 * h] = __dmul_rn(rho, co);
      z[2 * h + 1] = __dmul_rn(rho, s);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int64_t t = 4 * b + r;
      if (t >= t_begin && t < t_end) {
        int64_t i = t % n, j = t / n - col0;
        Om[i + j * ldo] = z[r];
      }
    }
  }
}

}  // namespace

void launch_omega(Ctx &c, int64_t n, int64_t l, int64_t col0, uint64_t seed, double *Om, int64_t ldo) {
  int64_t blocks = ceil_div(n * l, 4) + 1;
  int grid = (int)std::min<int64_t>(ceil_div(blocks, 256), (int64_t)c.num_sms * 8);
  omega_kernel<<<grid, 256, 0, c.stream>>>(n, l, col0, seed, Om, ldo);
  RQLP_LAUNCHED(c);
}

}  // namespace rqlpk
