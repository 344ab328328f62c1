// K5 placeholder (replaced by the tcgen05 grouped GEMM).
#include "common.cuh"
extern "C" int aurora_expert_ffn(const void*, const void*, const void*, void*, void*,
                                 const int32_t*, int, int64_t, int, int, int, void*) {
  return AURORA_EUNSUPPORTED;
}
extern "C" int aurora_grouped_gemm(const void*, const void*, void*, const int32_t*, int, int64_t,
                                   int, int, int, int, void*) {
  return AURORA_EUNSUPPORTED;
}
