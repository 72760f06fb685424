// ttm_dmma.cu -- float64 ttm as a GETT on FP64 DMMA tensor cores (placeholder
// until the tiled kernel lands; tl_ttm falls back to the exact SIMT fold).
#include "tl_common.cuh"

namespace tl {
int ttm_dmma_enqueue(const tl_desc &, const void *, const tl_desc &, const void *, void *, int, cudaStream_t) {
    return TL_EUNSUPPORTED;
}
}  // namespace tl
