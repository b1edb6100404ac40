// tcgen05 (5th-gen tensor core) phase A of the exhaustive search and the GPU
// IVF build; declarations used by the C-ABI driver.
#pragma once

#include "vs_internal.h"
#include "vs_kernels.cuh"

namespace vs {
#ifndef VS_TC_INLINE
#define VS_TC_INLINE_DECL inline
#else
#define VS_TC_INLINE_DECL VS_TC_INLINE
#endif
// the 128-row-tile build of the phase-A GEMM (vs_tc128.cu)
namespace bn128 {
int tc_enn_scan(vs_ctx* ctx, EnnScanParams& sp, int dtype, const unsigned* xmax, int cshift,
                CandBuf* cb, bool* exhaustive, int timer_class);
int tc_dense_keys(vs_ctx* ctx, const float* Q, int64_t nq, int d, const float* X, int64_t ncols,
                  const float* xnorm, const unsigned* xmax, int ip, float* keys, float* margin,
                  float* mins = nullptr);
}
inline namespace bn256 {

// whether the tensor-core phase A handles this shape / dtype / metric
bool tc_supported(int d, int dtype, int ip);
// whether phase A stages fp16 operands (float32 rows with a known max norm)
bool use_f16(int dtype, const unsigned* xmax);
int tc_build_f16_shadow(vs_ctx* ctx, const float* x, int64_t n, int d, const unsigned* xmax, void* shadow,
                        float2* stats);
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
// top2 (nullable, [n][2][2]) and rowstats (nullable, [n] (||x~||^2, ||dx||^2))
// feed the near-tie recheck (vs_kmeans.cu)
int tc_argmin_rows(vs_ctx* ctx, const void* x, int dtype, int64_t n, int d, const __nv_bfloat16* cb,
                   const float* cnorm, int64_t ncols, unsigned long long* out, __nv_bfloat16* xb,
                   unsigned* junk, unsigned long long* top2 = nullptr, float2* rowstats = nullptr,
                   const unsigned* row_xmax = nullptr, const unsigned* col_xmax = nullptr);
// fp16 staging of float32 columns scaled by pow2_scale(*xmax) (for the fp16 argmin)
int tc_stage_f16(vs_ctx* ctx, const float* x, int64_t n, int d, const unsigned* xmax, void* out, unsigned* stats);
int tc_stage_bf16(vs_ctx* ctx, const float* x, int64_t n, int d, __nv_bfloat16* out, unsigned* junk);
// dense approximate keys [nq][ncols] of float32 rows X on the tensor cores
// (MODE 3; the IVF coarse quantizer) and their per-query margins
int tc_dense_keys(vs_ctx* ctx, const float* Q, int64_t nq, int d, const float* X, int64_t ncols,
                  const float* xnorm, const unsigned* xmax, int ip, float* keys, float* margin,
                  float* mins = nullptr);

// IVF list-major phase A on the tensor cores (bf16 list-contiguous payload):
// pairs already grouped by list into units of <= 128 pairs
struct TcIvfArgs {
    const float* Q;
    int64_t nq;
    int d;
    const __nv_bfloat16* payload;
    int64_t n_total;
    const float* pnorms;          // per payload position ||x||^2
    const unsigned* pmax;         // max ||x||^2 (float bits)
    const int64_t* list_off;
    int64_t max_list;
    const int32_t* pair_codes;
    int64_t npairs;
    const int4* units;
    const int* n_units;
    int64_t max_units;
    int nprobe;
    const uint32_t* pbits;
    int k;
    int ip;
    int cshift;
    int timer_class;
    // long lists cut into row chunks (nullable / 0: whole lists)
    int64_t chunk_rows = 0;
    const int64_t* pair_base = nullptr;   // [nq*nprobe] first flat buffer of each pair
    const int64_t* sub_off = nullptr;     // [nq+1] flat buffer range of each query
    int64_t total_subs = 0;
    int max_subs = 0;                     // bound on buffers per query
};
struct TcIvfOut {
    CandBuf cb;
    float* margin;
    unsigned* tau_g;
    int verify;
    bool exhaustive;
};
int tc_ivf_scan(vs_ctx* ctx, const TcIvfArgs& a, TcIvfOut* out);
int tc_stage_queries_f16(vs_ctx* ctx, const float* Q, int64_t nq, int d, const unsigned* xmax,
                         const unsigned* xmax2, int ip, __half* out, float* kinv, float* margin);

}  // namespace bn256

// GPU IVF build / assignment (vs_kmeans.cu)
int ivf_assign_gpu(vs_ctx* ctx, const vs_ivf* v, const vs_column* col, int32_t* out);
// exact tie-rule nearest row of each query (vs_capi.cu; the k-means near-tie recheck)
int exact_top1(vs_ctx* ctx, const float* q, int64_t m, int d, const float* rows, int64_t nrows, const float* rnorm,
               const unsigned* rmax, int32_t* out_ids, double* out_dist);
int ivf_build_gpu(vs_ctx* ctx, const vs_column* data, int32_t nlist, const int64_t* init_rows, uint64_t seed,
                  int32_t metric, int32_t max_iters, vs_ivf** out);

}  // namespace vs
