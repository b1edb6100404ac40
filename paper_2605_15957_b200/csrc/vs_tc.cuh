// tcgen05 (5th-gen tensor core) phase A of the exhaustive search and the GPU
// IVF build; declarations used by the C-ABI driver.
#pragma once

#include "vs_internal.h"
#include "vs_kernels.cuh"

namespace vs {

// whether the tensor-core phase A handles this shape / dtype / metric
bool tc_supported(int d, int dtype, int ip);
// heuristic: enough work to amortise the bf16 staging pass
bool tc_profitable(int64_t nq, int64_t nsel, int d);
// runs phase A on the tensor cores; fills `cb` (allocated by the callee from
// the context arena) and may rewrite sp.margin with the tensor-core error bound
int tc_enn_scan(vs_ctx* ctx, EnnScanParams& sp, int dtype, const unsigned* xmax, int cshift,
                CandBuf* cb, bool* exhaustive, int timer_class);

// first-min nearest column (squared L2) of every row on the tensor cores.
// `scratch` = tc_argmin_scratch() bf16 elements + 2 words, allocated once by
// the caller (the k-means loop calls this every iteration).
int64_t tc_argmin_chunk(int64_t n);
int tc_argmin_rows(vs_ctx* ctx, const void* x, int dtype, int64_t n, int d, const __nv_bfloat16* cb,
                   const float* cnorm, int64_t ncols, unsigned long long* out, __nv_bfloat16* xb,
                   unsigned* junk);
int tc_stage_bf16(vs_ctx* ctx, const float* x, int64_t n, int d, __nv_bfloat16* out, unsigned* junk);

int ivf_build_gpu(vs_ctx* ctx, const vs_column* data, int32_t nlist, const int64_t* init_rows, uint64_t seed,
                  int32_t metric, int32_t max_iters, vs_ivf** out);

}  // namespace vs
