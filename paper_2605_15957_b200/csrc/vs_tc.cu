// tcgen05 phase A — placeholder until the tensor-core kernel lands.
#include "vs_tc.cuh"

namespace vs {

bool tc_supported(int, int, int) { return false; }
bool tc_profitable(int64_t, int64_t, int) { return false; }
int tc_enn_scan(vs_ctx*, EnnScanParams&, int, const unsigned*, int, CandBuf*) {
    return vs_internal::set_err(VS_ERR_INTERNAL, "tensor-core path not available");
}

}  // namespace vs
