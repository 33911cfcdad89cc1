// additive.cu -- cross moments of the additive model.  Filled in below.
#include "fk_internal.cuh"

namespace fk {

size_t cross_ws_bytes(int d, int m, double eps, int64_t n) {
  (void)d; (void)m; (void)eps; (void)n;
  return 256;
}

fk_status cross_run(const fk_points& X, double L, int m, double eps, double* G, bool accumulate, void* ws, size_t ws_bytes,
                    int* d_status, cudaStream_t s) {
  (void)X; (void)L; (void)m; (void)eps; (void)G; (void)accumulate; (void)ws; (void)ws_bytes; (void)d_status; (void)s;
  return fail(FK_E_UNSUPPORTED, "fk_additive_cross_moments: not built yet");
}

}  // namespace fk
