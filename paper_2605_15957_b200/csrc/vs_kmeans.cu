// GPU IVF build — placeholder.
#include "vs_tc.cuh"

namespace vs {
int ivf_build_gpu(vs_ctx*, const vs_column*, int32_t, uint64_t, int32_t, int32_t, vs_ivf**) {
    return vs_internal::set_err(VS_ERR_PARAMETER, "GPU IVF build not available yet");
}
}  // namespace vs
