// ffn_tc.cu — placeholder until the tcgen05 kernels land.
#include "common.cuh"
#include "kernels.h"

namespace pgmoe {
bool tc_supported(int, int) { return false; }
int expert_ffn_tc(const float *, int, int, int, int, const void *, size_t, int, const pgmoe_routing *,
                  float *, float *, void *, size_t, cudaStream_t) {
    set_error("tcgen05 path not built");
    return PGMOE_E_CONFIG;
}
int dense_tc(const float *, int, int, int, const void *, float *, void *, size_t, cudaStream_t) {
    set_error("tcgen05 path not built");
    return PGMOE_E_CONFIG;
}
}  // namespace pgmoe
