// gemm_tma.cu -- TMA-pipelined DMMA kernels for the two tall-skinny A-passes (placeholder:
// returns false so gemm.cu falls back to the generic DMMA kernel).
#include "internal.cuh"

namespace rqlpk {

bool gemm_nn_tma(Ctx &, int64_t, int64_t, int64_t, const double *, int64_t, const double *, int64_t, double *, int64_t,
                 double *, size_t, const unsigned *, unsigned) {
  return false;
}
bool gemm_tn_tma(Ctx &, int64_t, int64_t, int64_t, const double *, int64_t, const double *, int64_t, double *, int64_t,
                 bool, double *, size_t, const unsigned *, unsigned) {
  return false;
}
size_t gemm_tma_partials_needed(int64_t, int64_t, int64_t, int) { return 0; }

}  // namespace rqlpk
