// Large-k' search (vs_wide.cu): k' above the candidate-buffer top-k
// (vs_topk_cap()), device-wide select / exact score / segmented sort.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/vs_b200.h"

namespace vs {

struct WideJob {
    const float* q;             // device [nq][d]
    int64_t nq;
    int d;
    const void* rows;           // ENN: base rows; IVF: list-contiguous payload
    int dtype;
    const int64_t* sel;         // ENN: selection (nullable = identity)
    int64_t ncand;              // ENN: candidates per query (nsel)
    const float* xnorm;         // ENN: ||x||^2 per base row (squared L2)
    const float* margin;        // [nq] = 2 x the fp32 key error bound (eps_simt)
    int ip;
    int k;
    const int64_t* id_map;      // IVF: payload position -> row id (list_ids)
    int64_t id_offset;
    int64_t* out_ids;           // [nq][k] (each output nullable)
    double* out_dist;
    int32_t* out_ids32;
    int32_t* out_count;         // [nq]
    int cls_scan;
    int cls_rerank;
};

int wide_enn(vs_ctx* ctx, const WideJob& j);
int wide_ivf(vs_ctx* ctx, const WideJob& j, const int32_t* probes, int nprobe, const int64_t* list_off_d,
             const std::vector<int64_t>& h_off, const uint8_t* owned_d, const uint32_t* pbits, const float* pnorm);
// [nparts][nq][k_in] partial results (counts [nparts][nq]) -> global top-k
// under the tie rule, any k (the shared-memory merge kernel covers k <= 2048)
int wide_merge(vs_ctx* ctx, int nparts, int64_t nq, int k_in, const int64_t* ids, const double* dist,
               const int32_t* counts, int k, int ip, int64_t* out_ids, double* out_dist, int32_t* out_count);

}  // namespace vs
