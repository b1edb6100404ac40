// C ABI (include/vs_b200.h): contexts, columns, IVF structures and the search
// drivers that sequence the kernels. Every entry point returns a vs_status
// mirroring the reference exceptions (errors.py) and leaves a message in a
// thread-local buffer (vs_last_error).
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <functional>
#include <mutex>
#include <limits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/vs_b200.h"
#include "vs_common.cuh"
#include "vs_kernels.cuh"

#include "vs_internal.h"
#include "vs_tc.cuh"
#include "vs_wide.cuh"

using namespace vs_internal;

namespace {

// device view of a caller buffer: device pointers pass through, host
// pointers are copied into scratch on the context stream
template <typename T>
int stage_in(vs_ctx* ctx, const T* src, size_t count, const T** out) {
    if (!src || count == 0) {
        *out = src;
        return VS_OK;
    }
    if (is_device_ptr(src)) {
        *out = src;
        return VS_OK;
    }
    T* d = nullptr;
    CKS(arena_alloc(ctx, count, &d));
    CK(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    *out = d;
    return VS_OK;
}

// output target: device pointer used directly, host pointer gets scratch +
// a deferred device->host copy
struct OutBuf {
    void* host = nullptr;
    void* dev = nullptr;
    size_t bytes = 0;
};
template <typename T>
int stage_out(vs_ctx* ctx, T* dst, size_t count, T** dev, std::vector<OutBuf>& pending) {
    if (!dst) {
        *dev = nullptr;
        return VS_OK;
    }
    if (is_device_ptr(dst)) {
        *dev = dst;
        return VS_OK;
    }
    T* d = nullptr;
    CKS(arena_alloc(ctx, count, &d));
    *dev = d;
    pending.push_back(OutBuf{(void*)dst, (void*)d, count * sizeof(T)});
    return VS_OK;
}
// final outputs (written once by the last kernels, never read back): a
// page-locked host buffer is written in place by the kernels over PCIe
// (zero-copy), so the result transfer overlaps phase B instead of following
// it (VS_ZERO_COPY_OUT=0 stages them like any host buffer; VS_ZERO_COPY_MAX
// caps the zero-copy buffer size in bytes, default no cap). Measured in
// profiles/r2/e2e_transfers: config 3 (0.8 MB buffers) gains 0.04 ms; config
// 2 (8 MB) staged and copied back adds ~0.3 ms of non-kernel time per step
template <typename T>
int stage_out_final(vs_ctx* ctx, T* dst, size_t count, T** dev, std::vector<OutBuf>& pending, bool allow) {
    static const bool zc_env = !(getenv("VS_ZERO_COPY_OUT") && getenv("VS_ZERO_COPY_OUT")[0] == '0');
    const size_t zc_max = getenv("VS_ZERO_COPY_MAX") ? (size_t)atoll(getenv("VS_ZERO_COPY_MAX")) : SIZE_MAX;
    if (allow && zc_env && dst && count * sizeof(T) <= zc_max && !is_device_ptr(dst)) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, dst) == cudaSuccess && a.type == cudaMemoryTypeHost && a.devicePointer) {
            *dev = static_cast<T*>(a.devicePointer);
            return VS_OK;
        }
        cudaGetLastError();
    }
    return stage_out(ctx, dst, count, dev, pending);
}
int flush_out(vs_ctx* ctx, std::vector<OutBuf>& pending) {
    for (auto& o : pending)
        if (o.bytes) CK(cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    resolve_timers(ctx);
    return VS_OK;
}

// row norms of a column, computed on the CALLING context's stream (a column may
// be searched through contexts other than the one that created it)
int ensure_norms(vs_column* col, vs_ctx* ctx) {
    if (col->norms_ready) return VS_OK;
    if (!col->norms) {
        CK(cudaMalloc(&col->norms, std::max<int64_t>(col->n, 1) * sizeof(float)));
        CK(cudaMalloc(&col->max_norm_bits, sizeof(unsigned)));
    }
    CK(cudaMemsetAsync(col->max_norm_bits, 0, sizeof(unsigned), ctx->stream));
    if (col->dtype == VS_DTYPE_F32)
        CK(vs::launch_row_norms<float>((const float*)col->data, col->n, col->d, col->norms,
                                       col->max_norm_bits, ctx->stream));
    else
        CK(vs::launch_row_norms<__nv_bfloat16>((const __nv_bfloat16*)col->data, col->n, col->d,
                                               col->norms, col->max_norm_bits, ctx->stream));
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    col->norms_ready = true;
    return VS_OK;
}

// The fp16 shadow (vs_column::f16): built on a column's second tensor-core
// search, when its float32 rows live on the device and the shadow fits (an
// allocation failure only disables it). Staging then reads 2 bytes per
// element instead of 4 (config 2: 6 -> 4 GB per search). VS_F16_SHADOW=0 off.
int ensure_f16_shadow(vs_ctx* ctx, vs_column* col, int64_t nq, int64_t nsel) {
    static const bool env_off = getenv("VS_F16_SHADOW") && getenv("VS_F16_SHADOW")[0] == '0';
    if (env_off || col->dtype != VS_DTYPE_F32 || col->host_resident || col->f16_failed) return VS_OK;
    if (ctx->opt_enn_kernel == 1 || !vs::use_f16(col->dtype, col->max_norm_bits) ||
        !(ctx->opt_enn_kernel == 2 || vs::tc_profitable(nq, nsel, col->d)))
        return VS_OK;
    if (++col->searches < 2 && !col->f16) return VS_OK;
    if (col->f16_ready) return VS_OK;
    const int dp = (col->d + 7) / 8 * 8;
    if (!col->f16) {
        if (cudaMalloc(&col->f16, (size_t)std::max<int64_t>(col->n, 1) * dp * 2) != cudaSuccess ||
            cudaMalloc(&col->f16_stats, (size_t)std::max<int64_t>(col->n, 1) * sizeof(float2)) != cudaSuccess) {
            cudaGetLastError();
            if (col->f16) cudaFree(col->f16);
            col->f16 = nullptr;
            col->f16_stats = nullptr;
            col->f16_failed = true;
            return VS_OK;
        }
    }
    CKS(vs::tc_build_f16_shadow(ctx, (const float*)col->data, col->n, col->d, col->max_norm_bits, col->f16,
                                col->f16_stats));
    col->f16_ready = true;
    return VS_OK;
}

// error-bound constant of the fp32 SIMT scores: margin =
// 2 x 2 (d + 2) 2^-24 x (|q| + X)^2   (|q| X for inner product)
float eps_simt(int d) { return 4.0f * (float)(d + 2) / 16777216.0f; }

// ---- shared phase-A/B driver for exhaustive scans (data search and IVF coarse) ---------
struct EnnJob {
    const float* q;           // device [nq][d]
    int64_t nq;
    int d;
    const void* rows;         // device base rows
    int dtype;
    const int64_t* sel;       // device selection (nullable)
    int64_t nsel;
    const float* xnorm;       // per base row (L2)
    const unsigned* xmax;     // max ||x||^2 bits
    int ip;
    int k;
    int64_t id_offset;
    const int64_t* id_map = nullptr;   // staged position -> base row (streamed chunks)
    const void* f16 = nullptr;         // nullable: the column's fp16 shadow (vs_column)
    const float2* f16_stats = nullptr;
    bool narrow = false;               // 128-row tensor-core tiles (IVF coarse quantizer)
    cudaEvent_t q_ready = nullptr;     // queries still being copied in (copy stream)
    float* margin_todo = nullptr;      // SIMT margins to compute once the queries have landed
    // outputs (device, nullable)
    int64_t* out_ids;
    double* out_dist;
    int32_t* out_ids32;
    int32_t* out_count;
    int cls_scan = VS_K_ENN_SCAN;
    int cls_rerank = VS_K_RERANK;
};

__global__ void k_gather_queries(const float* __restrict__ src, const int32_t* __restrict__ idx,
                                 int64_t n, int d, float* __restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t tot = n * (int64_t)d;
    for (; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / d, c = i - r * d;
        dst[i] = src[(int64_t)idx[r] * d + c];
    }
}
template <typename T>
__global__ void k_scatter_rows(const T* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                               int w, T* __restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t tot = n * (int64_t)w;
    for (; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / w, c = i - r * w;
        dst[(int64_t)idx[r] * w + c] = src[i];
    }
}
template <typename T>
int scatter_rows(vs_ctx* ctx, const T* src, const int32_t* idx, int64_t n, int w, T* dst) {
    if (!dst || n == 0) return VS_OK;
    int64_t tot = n * w;
    int blocks = (int)std::min<int64_t>((tot + 255) / 256, 4096);
    k_scatter_rows<T><<<blocks, 256, 0, ctx->stream>>>(src, idx, n, w, dst);
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    return VS_OK;
}

struct PhaseBHooks;
int run_enn(vs_ctx* ctx, const EnnJob& job, const float* margin, int cshift, bool allow_force,
            const PhaseBHooks* hk = nullptr);

// phase A result kept between the two halves of a search
struct PhaseA {
    vs::EnnScanParams sp;
    bool exhaustive = false;
};

// hooks of the distributed protocol (vs_enn_search_begin/finish): all nullable
struct PhaseBHooks {
    const float* ext_thr = nullptr;   // [nq] global upper bound on the k-th approximate key
    double* out_bound = nullptr;      // [nq] deferred verification bound (key space)
    float* out_kth = nullptr;         // [nq] k-th approximate key only (no re-rank)
};

int enn_phase_b(vs_ctx* ctx, const EnnJob& job, const PhaseA& st, int cshift, bool allow_force,
                const PhaseBHooks& hk);

int enn_phase_a(vs_ctx* ctx, const EnnJob& job, const float* margin, int cshift, PhaseA* st) {
    vs::EnnScanParams sp;
    sp.Q = job.q;
    sp.nq = job.nq;
    sp.d = job.d;
    sp.X = job.rows;
    sp.sel = job.sel;
    sp.nsel = job.nsel;
    sp.xnorm = job.xnorm;
    sp.margin = margin;
    sp.ip = job.ip;
    sp.k = job.k;
    sp.tau_g = nullptr;
    sp.q_ready = nullptr;
    sp.f16 = job.f16;
    sp.f16_stats = job.f16_stats;
    const bool use_tc = ctx->opt_enn_kernel != 1 && vs::tc_supported(job.d, job.dtype, job.ip) &&
                        (ctx->opt_enn_kernel == 2 || vs::tc_profitable(job.nq, job.nsel, job.d));
    if (job.q_ready) {
        if (use_tc && cshift == 0) {
            // the tensor-core path stages rows before it needs the queries and
            // replaces the SIMT margins with its own
            sp.q_ready = job.q_ready;
        } else {
            CK(cudaStreamWaitEvent(ctx->stream, job.q_ready, 0));
        }
    }
    if (job.margin_todo && !(use_tc && cshift == 0)) {
        if (sp.q_ready) CK(cudaStreamWaitEvent(ctx->stream, job.q_ready, 0));
        CK(vs::launch_query_margins(job.q, job.nq, job.d, job.xmax, eps_simt(job.d), job.ip, job.margin_todo,
                                    nullptr, ctx->stream));
        ctx->stats[VS_STAT_LAUNCHES] += 1;
    }
    bool exhaustive = false;
    {
        if (use_tc) {
            // times its own GEMM launch under job.cls_scan (staging under VS_K_STAGE)
            static const int narrow_env = getenv("VS_TC_NARROW") ? atoi(getenv("VS_TC_NARROW")) : -1;
            if (narrow_env == 1 || (narrow_env != 0 && job.narrow))
                CKS(vs::bn128::tc_enn_scan(ctx, sp, job.dtype, job.xmax, cshift, &sp.cb, &exhaustive, job.cls_scan));
            else
                CKS(vs::tc_enn_scan(ctx, sp, job.dtype, job.xmax, cshift, &sp.cb, &exhaustive, job.cls_scan));
        } else {
            KTimer kt(ctx, job.cls_scan);
            const int64_t qtiles = (job.nq + 127) / 128;
            const int64_t target = (int64_t)ctx->sm_count * 4;  // 2 CTAs/SM x 2 waves
            int64_t n_split = std::max<int64_t>(1, (target + qtiles - 1) / qtiles);
            n_split = std::min<int64_t>(n_split, std::max<int64_t>(1, (job.nsel + 255) / 256));
            int64_t rps = (job.nsel + n_split - 1) / n_split;
            rps = (rps + 127) / 128 * 128;
            n_split = (job.nsel + rps - 1) / rps;
            const int n_sub = (int)(n_split * 2);
            int64_t C = pow2ceil(std::max<int64_t>(2 * job.k, job.k + 32)) << (ctx->opt_slack + cshift);
            const int64_t rows_per_sub = (rps + 1) / 2;
            // buffers that hold every row they see cannot overflow: used whenever
            // they fit in 256 MiB (small batches, e.g. the coarse quantizer of a
            // few queries, whose centroid keys crowd inside the margin band)
            const int64_t cap = pow2ceil(rows_per_sub + 64);
            exhaustive = C >= cap || (int64_t)job.nq * n_sub * cap * 8 <= (int64_t(256) << 20);
            if (exhaustive) C = cap;
            vs::CandBuf cb;
            cb.n_sub = n_sub;
            cb.C = (int)C;
            const size_t slots = (size_t)job.nq * n_sub * C;
            CKS(arena_alloc(ctx, slots, &cb.key));
            CKS(arena_alloc(ctx, slots, &cb.pos));
            CKS(arena_alloc(ctx, (size_t)job.nq * n_sub, &cb.cnt));
            CKS(arena_alloc(ctx, (size_t)job.nq, &cb.overflow));
            CK(cudaMemsetAsync(cb.overflow, 0, job.nq * sizeof(int), ctx->stream));
            sp.n_split = (int)n_split;
            sp.rows_per_split = rps;
            sp.cb = cb;
            if (job.dtype == VS_DTYPE_F32) CK(vs::launch_enn_scan_simt<float>(sp, ctx->stream));
            else CK(vs::launch_enn_scan_simt<__nv_bfloat16>(sp, ctx->stream));
        }
    }
    ctx->stats[VS_STAT_LAST_ENN_KERNEL] = use_tc ? 2 : 1;
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    st->sp = sp;
    st->exhaustive = exhaustive;
    return VS_OK;
}

// phase A + phase B for the rows [0, nsel) of one job, then re-run overflowed
// queries with 4x larger candidate buffers (cshift + 2) until none remain.
// k' above the candidate-buffer top-k: device-wide select / score / sort (vs_wide.cu)
int run_enn_wide(vs_ctx* ctx, const EnnJob& job, const float* margin) {
    if (job.q_ready) CK(cudaStreamWaitEvent(ctx->stream, job.q_ready, 0));
    if (job.margin_todo) {
        CK(vs::launch_query_margins(job.q, job.nq, job.d, job.xmax, eps_simt(job.d), job.ip, job.margin_todo,
                                    nullptr, ctx->stream));
        margin = job.margin_todo;
        ctx->stats[VS_STAT_LAUNCHES] += 1;
    }
    vs::WideJob w{};
    w.q = job.q;
    w.nq = job.nq;
    w.d = job.d;
    w.rows = job.rows;
    w.dtype = job.dtype;
    w.sel = job.sel;
    w.ncand = job.nsel;
    w.xnorm = job.xnorm;
    w.margin = margin;
    w.ip = job.ip;
    w.k = job.k;
    w.id_map = nullptr;
    w.id_offset = job.id_offset;
    w.out_ids = job.out_ids;
    w.out_dist = job.out_dist;
    w.out_ids32 = job.out_ids32;
    w.out_count = job.out_count;
    w.cls_scan = job.cls_scan;
    w.cls_rerank = job.cls_rerank;
    ctx->stats[VS_STAT_LAST_ENN_KERNEL] = 3;
    return vs::wide_enn(ctx, w);
}

int run_enn(vs_ctx* ctx, const EnnJob& job, const float* margin, int cshift, bool allow_force,
            const PhaseBHooks* hk) {
    if (job.nq == 0) return VS_OK;
    if (job.k > kTopkCap) {
        if (hk) return set_err(VS_ERR_CAP_EXCEEDED, "two-phase search supports k' <= %d", kTopkCap);
        return run_enn_wide(ctx, job, margin);
    }
    PhaseA st;
    CKS(enn_phase_a(ctx, job, margin, cshift, &st));
    return enn_phase_b(ctx, job, st, cshift, allow_force, hk ? *hk : PhaseBHooks{});
}

int enn_phase_b(vs_ctx* ctx, const EnnJob& job, const PhaseA& st, int cshift, bool allow_force,
                const PhaseBHooks& hk) {
    const vs::EnnScanParams& sp = st.sp;
    const bool exhaustive = st.exhaustive;
    const float* margin = sp.margin;
    const vs::CandBuf cb = sp.cb;
    vs::RerankParams rp;
    rp.Q = job.q;
    rp.nq = job.nq;
    rp.d = job.d;
    rp.ip = job.ip;
    rp.k = job.k;
    rp.cb = sp.cb;
    rp.margin = sp.margin;
    rp.tau_g = sp.tau_g;
    rp.verify = sp.verify;
    rp.band_ready = sp.band_ready;
    rp.rows = job.rows;
    rp.row_map = job.sel;
    rp.id_map = job.id_map;
    rp.id_offset = job.id_offset;
    const int64_t all_slots = (int64_t)sp.cb.n_sub * sp.cb.C;
    rp.s_cap = (exhaustive || (int64_t)job.nq * all_slots * 20 < (int64_t(1) << 30))
                   ? all_slots
                   : std::min<int64_t>(all_slots, std::max<int64_t>(8 * (int64_t)sp.cb.C, 4096));
    CKS(arena_alloc(ctx, (size_t)job.nq * rp.s_cap, &rp.s_pos));
    CKS(arena_alloc(ctx, (size_t)job.nq * rp.s_cap, &rp.s_key));
    CKS(arena_alloc(ctx, (size_t)job.nq * rp.s_cap, &rp.s_id));
    CKS(arena_alloc(ctx, (size_t)job.nq, &rp.s_count));
    CKS(arena_alloc(ctx, (size_t)job.nq, &rp.fb_list));
    CKS(arena_alloc(ctx, 1, &rp.fb_count));
    rp.out_ids = job.out_ids;
    rp.out_dist = job.out_dist;
    rp.out_ids32 = job.out_ids32;
    rp.out_count = job.out_count;
    unsigned long long* d_surv = nullptr;
    CKS(arena_alloc(ctx, 1, &d_surv));
    CK(cudaMemsetAsync(d_surv, 0, sizeof(unsigned long long), ctx->stream));
    rp.n_survivors = d_surv;
    rp.ext_thr = hk.ext_thr;
    rp.out_bound = hk.out_bound;
    rp.out_kth = hk.out_kth;
    {
        KTimer kt(ctx, job.cls_rerank);
        if (job.dtype == VS_DTYPE_F32) CK(vs::launch_rerank<float>(rp, ctx->stream));
        else CK(vs::launch_rerank<__nv_bfloat16>(rp, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    if (hk.out_kth) return VS_OK;   // k-th keys only: phase B proper comes later

    unsigned long long h_surv = 0;
    CK(cudaMemcpyAsync(&h_surv, d_surv, sizeof(h_surv), cudaMemcpyDeviceToHost, ctx->stream));
    std::vector<int32_t> which;
    {
        std::vector<int> h(job.nq);
        CK(cudaMemcpyAsync(h.data(), cb.overflow, job.nq * sizeof(int), cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (int64_t i = 0; i < job.nq; ++i)
            if (h[i] || (allow_force && ctx->opt_force_retry)) which.push_back((int32_t)i);
    }
    if (cshift == 0) ctx->stats[VS_STAT_SURVIVORS] = (int64_t)h_surv;
    if (which.empty()) return VS_OK;
    if (exhaustive && !(allow_force && ctx->opt_force_retry))
        return set_err(VS_ERR_INTERNAL, "candidate overflow with exhaustive buffers");
    ctx->stats[VS_STAT_OVERFLOW_QUERIES] += (int64_t)which.size();

    // re-run the overflowed queries with 4x larger buffers
    const int64_t m = (int64_t)which.size();
    int32_t* d_idx = nullptr;
    float *d_q = nullptr, *d_m = nullptr;
    CKS(arena_alloc(ctx, m, &d_idx));
    CKS(arena_alloc(ctx, (size_t)m * job.d, &d_q));
    CKS(arena_alloc(ctx, (size_t)m, &d_m));
    CK(cudaMemcpyAsync(d_idx, which.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    if (job.margin_todo) {
        // the tensor-core phase A skipped the SIMT margins (queries were still in
        // flight then; they have landed since): the re-run needs them
        CK(vs::launch_query_margins(job.q, job.nq, job.d, job.xmax, eps_simt(job.d), job.ip, job.margin_todo,
                                    nullptr, ctx->stream));
        margin = job.margin_todo;
        ctx->stats[VS_STAT_LAUNCHES] += 1;
    }
    {
        int blocks = (int)std::min<int64_t>((m * job.d + 255) / 256, 4096);
        k_gather_queries<<<blocks, 256, 0, ctx->stream>>>(job.q, d_idx, m, job.d, d_q);
        CK(cudaGetLastError());
        k_gather_queries<<<1, 256, 0, ctx->stream>>>(margin, d_idx, m, 1, d_m);
        CK(cudaGetLastError());
        ctx->stats[VS_STAT_LAUNCHES] += 2;
    }
    EnnJob sub = job;
    sub.q = d_q;
    sub.nq = m;
    sub.q_ready = nullptr;
    sub.margin_todo = nullptr;
    const int k = job.k;
    if (job.out_ids) CKS(arena_alloc(ctx, (size_t)m * k, &sub.out_ids));
    if (job.out_dist) CKS(arena_alloc(ctx, (size_t)m * k, &sub.out_dist));
    if (job.out_ids32) CKS(arena_alloc(ctx, (size_t)m * k, &sub.out_ids32));
    if (job.out_count) CKS(arena_alloc(ctx, (size_t)m, &sub.out_count));
    CKS(run_enn(ctx, sub, d_m, exhaustive ? cshift : cshift + 2, false));
    CKS(scatter_rows(ctx, sub.out_ids, d_idx, m, k, job.out_ids));
    CKS(scatter_rows(ctx, sub.out_dist, d_idx, m, k, job.out_dist));
    CKS(scatter_rows(ctx, sub.out_ids32, d_idx, m, k, job.out_ids32));
    CKS(scatter_rows(ctx, sub.out_count, d_idx, m, 1, job.out_count));
    if (hk.out_bound) {
        // re-runs keep every candidate in the margin band: their local result is
        // complete, no bound on the other shards' results
        double* inf = nullptr;
        CKS(arena_alloc(ctx, (size_t)m, &inf));
        std::vector<double> h_inf(m, std::numeric_limits<double>::infinity());
        CK(cudaMemcpyAsync(inf, h_inf.data(), m * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CKS(scatter_rows(ctx, inf, d_idx, m, 1, hk.out_bound));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return VS_OK;
}

int validate_metric(int32_t metric) {
    if (metric != VS_METRIC_SQUARED_L2 && metric != VS_METRIC_INNER_PRODUCT)
        return set_err(VS_ERR_PARAMETER, "unknown metric %d", metric);
    return VS_OK;
}
// any k' >= 1: k' <= kTopkCap runs the candidate-buffer path, larger k' the
// wide path (vs_wide.cu)
int validate_k(int32_t k) {
    if (k < 1) return set_err(VS_ERR_PARAMETER, "k must be >= 1, got %d", k);
    return VS_OK;
}

// bitmap -> selection vector on the device
int build_selection(vs_ctx* ctx, const uint32_t* d_bm, int64_t nbits, int64_t** sel, int64_t* nsel) {
    const int64_t nwords = (nbits + 31) / 32;
    const int64_t nb = vs::select_nblocks(nwords);
    int64_t* sums = nullptr;
    int64_t* total = nullptr;
    CKS(arena_alloc(ctx, (size_t)std::max<int64_t>(nb, 1), &sums));
    CKS(arena_alloc(ctx, 1, &total));
    CK(cudaMemsetAsync(total, 0, sizeof(int64_t), ctx->stream));
    KTimer kt(ctx, VS_K_SELECT);
    if (nb > 0) {
        CK(vs::launch_select_count(d_bm, nwords, nbits, sums, nb, ctx->stream));
        CK(vs::launch_select_scan(sums, nb, total, ctx->stream));
        ctx->stats[VS_STAT_LAUNCHES] += 2;
    }
    int64_t h_total = 0;
    CK(cudaMemcpyAsync(&h_total, total, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *nsel = h_total;
    int64_t* s = nullptr;
    CKS(arena_alloc(ctx, (size_t)std::max<int64_t>(h_total, 1), &s));
    if (h_total > 0) {
        CK(vs::launch_select_write(d_bm, nwords, nbits, sums, s, ctx->stream));
        ctx->stats[VS_STAT_LAUNCHES] += 1;
    }
    *sel = s;
    return VS_OK;
}

}  // namespace

void pending_erase(const vs_ctx* ctx);

void ctx_ref(vs_ctx* ctx) {
    std::lock_guard<std::mutex> lk(ctx->life_mu);
    ++ctx->live_objects;
}
void ctx_unref(vs_ctx* ctx) {
    {
        std::lock_guard<std::mutex> lk(ctx->life_mu);
        if (--ctx->live_objects > 0 || !ctx->destroyed) return;
    }
    DevGuard g(ctx->device);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

// =====================================================================================
extern "C" {

const char* vs_last_error(void) { return g_err.c_str(); }
int32_t vs_topk_cap(void) { return kTopkCap; }
int32_t vs_version(void) { return 1; }

int vs_ctx_create(int32_t device, vs_ctx** out) {
    if (!out) return set_err(VS_ERR_PARAMETER, "null out");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return set_err(VS_ERR_PARAMETER, "device %d not present (%d visible)", device, ndev);
    DevGuard g(device);
    CK(cudaSetDevice(device));
    vs_ctx* c = new vs_ctx();
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_err(e, "cudaStreamCreate");
    }
    c->stream = c->own_stream;
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    *out = c;
    return VS_OK;
}

int vs_ctx_destroy(vs_ctx* ctx) {
    if (!ctx) return VS_OK;
    pending_erase(ctx);   // a later context at the same address must not inherit it
    {
        DevGuard g(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        ctx->arena.release();
        resolve_timers(ctx);
        for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
        ctx->event_pool.clear();
        if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
        if (ctx->q_event) cudaEventDestroy(ctx->q_event);
        for (auto& e : ctx->q_chunk_ev)
            if (e) cudaEventDestroy(e);
        ctx->copy_stream = nullptr;
        ctx->q_event = nullptr;
    }
    {
        std::lock_guard<std::mutex> lk(ctx->life_mu);
        ctx->destroyed = true;
        if (ctx->live_objects > 0) return VS_OK;   // the last column / index free deletes it
    }
    DevGuard g(ctx->device);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return VS_OK;
}

int vs_ctx_set_stream(vs_ctx* ctx, void* stream) {
    if (!ctx) return set_err(VS_ERR_PARAMETER, "null ctx");
    ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
    return VS_OK;
}

int vs_ctx_synchronize(vs_ctx* ctx) {
    if (!ctx) return set_err(VS_ERR_PARAMETER, "null ctx");
    DevGuard g(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    return VS_OK;
}

int vs_ctx_set_option(vs_ctx* ctx, int32_t key, int64_t value) {
    if (!ctx) return set_err(VS_ERR_PARAMETER, "null ctx");
    switch (key) {
        case VS_OPT_ENN_KERNEL: ctx->opt_enn_kernel = (int)value; break;
        case VS_OPT_IVF_KERNEL: ctx->opt_ivf_kernel = (int)value; break;
        case VS_OPT_STREAM_CHUNK: ctx->opt_stream_chunk = value; break;
        case VS_OPT_IVF_CHUNK_ROWS: ctx->opt_ivf_chunk_rows = value; break;
        case VS_OPT_CAND_SLACK: ctx->opt_slack = (int)std::max<int64_t>(0, std::min<int64_t>(value, 8)); break;
        case VS_OPT_FORCE_RETRY: ctx->opt_force_retry = (int)value; break;
        case VS_OPT_TIMING: ctx->opt_timing = (int)value; break;
        case VS_OPT_COARSE: ctx->opt_coarse = (int)value; break;
        default: return set_err(VS_ERR_PARAMETER, "unknown option %d", key);
    }
    return VS_OK;
}

int vs_ctx_stats(vs_ctx* ctx, int64_t* out, int32_t n) {
    if (!ctx || !out) return set_err(VS_ERR_PARAMETER, "null argument");
    for (int i = 0; i < n && i < VS_STAT_N; ++i) out[i] = ctx->stats[i];
    return VS_OK;
}

int vs_ctx_kernel_times(vs_ctx* ctx, int64_t* ns, int64_t* launches, int32_t n, int32_t reset) {
    if (!ctx) return set_err(VS_ERR_PARAMETER, "null ctx");
    for (int i = 0; i < n && i < VS_K_N; ++i) {
        if (ns) ns[i] = ctx->kt_ns[i];
        if (launches) launches[i] = ctx->kt_count[i];
    }
    if (reset)
        for (int i = 0; i < VS_K_N; ++i) ctx->kt_ns[i] = ctx->kt_count[i] = 0;
    return VS_OK;
}

int vs_column_create(vs_ctx* ctx, const void* src, int64_t n, int32_t d, int32_t dtype,
                     vs_column** out) {
    if (!ctx || !out) return set_err(VS_ERR_PARAMETER, "null argument");
    if (d < 1) return set_err(VS_ERR_SHAPE, "embedding dimension must be >= 1");
    if (n < 0) return set_err(VS_ERR_SHAPE, "negative row count");
    if (dtype != VS_DTYPE_F32 && dtype != VS_DTYPE_BF16) return set_err(VS_ERR_PARAMETER, "bad dtype");
    if (n > 0 && !src) return set_err(VS_ERR_PARAMETER, "null source");
    DevGuard g(ctx->device);
    vs_column* c = new vs_column();
    c->ctx = ctx;
    c->n = n;
    c->d = d;
    c->dtype = dtype;
    c->owned = true;
    const size_t bytes = (size_t)n * d * elem_size(dtype);
    cudaError_t e = cudaMalloc(&c->data, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return cuda_err(e, "column allocation");
    }
    if (bytes) {
        e = cudaMemcpyAsync(c->data, src, bytes, cudaMemcpyDefault, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) {
            cudaGetLastError();
            cudaFree(c->data);
            delete c;
            return cuda_err(e, "column upload");
        }
    }
    ctx_ref(ctx);
    *out = c;
    return VS_OK;
}

int vs_column_wrap(vs_ctx* ctx, void* dev_ptr, int64_t n, int32_t d, int32_t dtype, vs_column** out) {
    if (!ctx || !out) return set_err(VS_ERR_PARAMETER, "null argument");
    if (d < 1) return set_err(VS_ERR_SHAPE, "embedding dimension must be >= 1");
    if (dtype != VS_DTYPE_F32 && dtype != VS_DTYPE_BF16) return set_err(VS_ERR_PARAMETER, "bad dtype");
    if (n > 0 && !is_device_ptr(dev_ptr))
        return set_err(VS_ERR_PARAMETER, "vs_column_wrap needs device memory");
    vs_column* c = new vs_column();
    c->ctx = ctx;
    c->data = dev_ptr;
    c->n = n;
    c->d = d;
    c->dtype = dtype;
    c->owned = false;
    ctx_ref(ctx);
    *out = c;
    return VS_OK;
}

int vs_column_wrap_host(vs_ctx* ctx, void* host_ptr, int64_t n, int32_t d, int32_t dtype, vs_column** out) {
    if (!ctx || !out || (!host_ptr && n > 0)) return set_err(VS_ERR_PARAMETER, "null argument");
    if (n < 0 || d < 1) return set_err(VS_ERR_SHAPE, "bad column shape");
    if (dtype != VS_DTYPE_F32 && dtype != VS_DTYPE_BF16) return set_err(VS_ERR_PARAMETER, "bad dtype");
    DevGuard g(ctx->device);
    const size_t bytes = (size_t)n * d * elem_size(dtype);
    cudaPointerAttributes at{};
    bool registered = false;
    if (cudaPointerGetAttributes(&at, host_ptr) != cudaSuccess || at.type == cudaMemoryTypeUnregistered) {
        cudaGetLastError();
        CK(cudaHostRegister(host_ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterReadOnly));
        registered = true;
    } else if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
        return set_err(VS_ERR_PARAMETER, "vs_column_wrap_host needs host memory");
    }
    void* dptr = nullptr;
    CK(cudaHostGetDevicePointer(&dptr, host_ptr, 0));
    vs_column* c = new vs_column();
    c->ctx = ctx;
    c->data = dptr;
    c->n = n;
    c->d = d;
    c->dtype = dtype;
    c->owned = false;
    c->host_resident = true;
    c->host_registered = registered;
    c->host_ptr = host_ptr;
    ctx_ref(ctx);
    *out = c;
    return VS_OK;
}

int vs_column_free(vs_column* col) {
    if (!col) return VS_OK;
    DevGuard g(col->ctx->device);
    cudaStreamSynchronize(col->ctx->stream);
    if (col->owned && col->data) cudaFree(col->data);
    if (col->host_registered) cudaHostUnregister(col->host_ptr);
    if (col->norms) cudaFree(col->norms);
    if (col->max_norm_bits) cudaFree(col->max_norm_bits);
    if (col->f16) cudaFree(col->f16);
    if (col->f16_stats) cudaFree(col->f16_stats);
    vs_ctx* ctx = col->ctx;
    delete col;
    ctx_unref(ctx);
    return VS_OK;
}

int vs_column_invalidate(vs_column* col) {
    if (!col) return set_err(VS_ERR_PARAMETER, "null column");
    col->norms_ready = false;   // recomputed (on the caller's stream) by the next search
    col->f16_ready = false;     // the shadow too (rebuilt in place)
    return VS_OK;
}

int vs_column_info(const vs_column* col, int64_t* n, int32_t* d, int32_t* dtype) {
    if (!col) return set_err(VS_ERR_PARAMETER, "null column");
    if (n) *n = col->n;
    if (d) *d = col->d;
    if (dtype) *dtype = col->dtype;
    return VS_OK;
}

// device-side merge of nparts [nq][k_in] partial results (no arena reset)
static int merge_parts(vs_ctx* ctx, int nparts, int64_t nq, int k_in, const int64_t* ids, const double* dist,
                       const int32_t* counts, int k, int metric, int64_t* out_ids, double* out_dist,
                       int32_t* out_count) {
    if (k > kTopkCap)   // the merge kernel sorts the top k in shared memory
        return vs::wide_merge(ctx, nparts, nq, k_in, ids, dist, counts, k, metric, out_ids, out_dist, out_count);
    vs::MergeParams p;
    p.nparts = nparts;
    p.nq = nq;
    p.k_in = k_in;
    p.k = k;
    p.ip = metric;
    p.ids = ids;
    p.dist = dist;
    p.counts = counts;
    const size_t n_in = (size_t)nparts * nq * k_in;
    CKS(arena_alloc(ctx, n_in, &p.s_key));
    CKS(arena_alloc(ctx, n_in, &p.s_id));
    p.out_ids = out_ids;
    p.out_dist = out_dist;
    p.out_count = out_count;
    {
        KTimer kt(ctx, VS_K_MERGE);
        CK(vs::launch_merge(p, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    return VS_OK;
}

// Search of a host-resident column (cfg5 B): only the SELECTED rows cross
// PCIe (the bitmap is applied before any row byte moves). The selection is cut
// into chunks; chunk c+1 is gathered by a few SMs over PCIe (zero-copy 16-byte
// reads, copy stream) while chunk c is searched on the remaining SMs; the
// per-chunk top-k are merged with the cross-shard merge kernel (same tie rule).
// Streamed chunks arrive in ascending row order, so a later chunk's row can
// only enter the final top-k with an exact distance below the k-th of any
// earlier chunk's (full) top-k. thr[q] keeps that bound in approximate-key
// space (key = dist - ||q||^2, or -score for inner product), rounded up; the
// next chunks' phase B keeps only candidates within the margin of it.
__global__ void k_chunk_bound(const double* __restrict__ dist, const int32_t* __restrict__ cnt, int64_t nq, int k,
                              const float* __restrict__ Q, int d, int ip, float* __restrict__ thr) {
    const int lane = threadIdx.x & 31;
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (q >= nq || cnt[q] < k) return;
    double qq = 0.0;
    if (!ip) {
        for (int i = lane; i < d; i += 32) {
            const double a = (double)Q[q * d + i];
            qq = fma(a, a, qq);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
    }
    if (lane == 0) {
        const double dk = dist[q * k + k - 1];
        const float t = __double2float_ru(ip ? -dk : dk - qq * (1.0 - 1e-12));
        thr[q] = fminf(thr[q], t);
    }
}

static int enn_search_streamed(vs_ctx* ctx, vs_column* col, const float* dq, int64_t nq, int d,
                               const int64_t* sel, int64_t nsel, int k, int metric, int64_t id_offset,
                               const float* margin, int64_t* out_ids, double* out_dist, int32_t* out_count) {
    const size_t es = elem_size(col->dtype);
    const int row_bytes = d * (int)es;
    if (row_bytes % 16) return set_err(VS_ERR_PARAMETER, "host-resident rows must be 16-byte multiples");
    int64_t chunk = ctx->opt_stream_chunk > 0 ? ctx->opt_stream_chunk
                                              : std::max<int64_t>(1, ((int64_t)1 << 30) / row_bytes);   // 1 GiB
    chunk = std::min(chunk, nsel);
    const int64_t nchunks = (nsel + chunk - 1) / chunk;
    if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    // the selection must be a device array the gather can read
    const int64_t* dsel = sel;
    int64_t* iota = nullptr;
    if (!dsel) {
        std::vector<int64_t> h(nsel);
        for (int64_t i = 0; i < nsel; ++i) h[i] = i;
        CKS(arena_alloc(ctx, (size_t)nsel, &iota));
        CK(cudaMemcpyAsync(iota, h.data(), nsel * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        dsel = iota;
    }
    char* buf[2] = {nullptr, nullptr};
    float* nrm[2] = {nullptr, nullptr};
    unsigned* junk = nullptr;
    for (int b = 0; b < std::min<int64_t>(2, nchunks); ++b) {
        CKS(arena_alloc(ctx, (size_t)chunk * row_bytes, &buf[b]));
        CKS(arena_alloc(ctx, (size_t)chunk, &nrm[b]));
    }
    CKS(arena_alloc(ctx, 1, &junk));
    int64_t *cids = nullptr;
    double* cdist = nullptr;
    int32_t* ccnt = nullptr;
    CKS(arena_alloc(ctx, (size_t)nchunks * nq * k, &cids));
    CKS(arena_alloc(ctx, (size_t)nchunks * nq * k, &cdist));
    CKS(arena_alloc(ctx, (size_t)nchunks * nq, &ccnt));
    float* thr = nullptr;
    if (nchunks > 1) {
        CKS(arena_alloc(ctx, (size_t)nq, &thr));
        std::vector<float> inf(nq, std::numeric_limits<float>::infinity());
        CK(cudaMemcpyAsync(thr, inf.data(), nq * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    cudaEvent_t ready[2], done[2];
    for (int b = 0; b < 2; ++b) {
        CK(cudaEventCreateWithFlags(&ready[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
    }
    const int reserve = nchunks > 1 ? 8 : 0;     // SMs for the overlapped PCIe gather
    const int gblocks = nchunks > 1 ? reserve * 4 : ctx->sm_count * 4;
    auto gather = [&](int64_t c) -> int {
        const int b = (int)(c & 1);
        const int64_t c0 = c * chunk, nc = std::min(chunk, nsel - c0);
        CK(vs::launch_gather_rows_host(col->data, dsel + c0, nc, row_bytes, buf[b], gblocks, ctx->copy_stream));
        CK(cudaMemsetAsync(junk, 0, sizeof(unsigned), ctx->copy_stream));
        if (col->dtype == VS_DTYPE_F32)
            CK(vs::launch_row_norms<float>((const float*)buf[b], nc, d, nrm[b], junk, ctx->copy_stream));
        else
            CK(vs::launch_row_norms<__nv_bfloat16>((const __nv_bfloat16*)buf[b], nc, d, nrm[b], junk,
                                                   ctx->copy_stream));
        CK(cudaEventRecord(ready[b], ctx->copy_stream));
        ctx->stats[VS_STAT_LAUNCHES] += 2;
        return VS_OK;
    };
    int rc = VS_OK;
    ctx->sm_reserve = reserve;
    CK(cudaEventRecord(done[0], ctx->stream));
    CK(cudaEventRecord(done[1], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->copy_stream, done[0], 0));   // queries/selection are ready
    rc = gather(0);
    for (int64_t c = 0; rc == VS_OK && c < nchunks; ++c) {
        const int b = (int)(c & 1);
        if (c + 1 < nchunks) {
            cudaStreamWaitEvent(ctx->copy_stream, done[(c + 1) & 1], 0);   // buffer reuse
            if ((rc = gather(c + 1)) != VS_OK) break;
        }
        cudaStreamWaitEvent(ctx->stream, ready[b], 0);
        const int64_t c0 = c * chunk, nc = std::min(chunk, nsel - c0);
        EnnJob job;
        job.q = dq;
        job.nq = nq;
        job.d = d;
        job.rows = buf[b];
        job.dtype = col->dtype;
        job.sel = nullptr;
        job.nsel = nc;
        job.xnorm = nrm[b];
        job.xmax = col->max_norm_bits;
        job.ip = metric;
        job.k = k;
        job.id_offset = id_offset;
        job.id_map = dsel + c0;
        job.out_ids = cids + c * nq * k;
        job.out_dist = cdist + c * nq * k;
        job.out_ids32 = nullptr;
        job.out_count = ccnt + c * nq;
        PhaseBHooks hk;
        hk.ext_thr = c > 0 ? thr : nullptr;
        if ((rc = run_enn(ctx, job, margin, 0, true, &hk)) != VS_OK) break;
        if (thr && c + 1 < nchunks) {
            k_chunk_bound<<<(unsigned)((nq * 32 + 255) / 256), 256, 0, ctx->stream>>>(
                job.out_dist, job.out_count, nq, k, dq, d, metric, thr);
            CK(cudaGetLastError());
            ctx->stats[VS_STAT_LAUNCHES] += 1;
        }
        cudaEventRecord(done[b], ctx->stream);
    }
    ctx->sm_reserve = 0;
    cudaStreamSynchronize(ctx->copy_stream);
    for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(ready[b]);
        cudaEventDestroy(done[b]);
    }
    if (rc != VS_OK) return rc;
    if (nchunks == 1) {
        if (out_ids) CK(cudaMemcpyAsync(out_ids, cids, (size_t)nq * k * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
        if (out_dist) CK(cudaMemcpyAsync(out_dist, cdist, (size_t)nq * k * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        if (out_count) CK(cudaMemcpyAsync(out_count, ccnt, (size_t)nq * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
        return VS_OK;
    }
    return merge_parts(ctx, (int)nchunks, nq, k, cids, cdist, ccnt, k, metric, out_ids, out_dist, out_count);
}

int vs_enn_search(vs_ctx* ctx, const vs_column* data, const float* queries, int64_t nq, int32_t d,
                  const uint32_t* bitmap, int64_t nbits, int32_t k, int32_t metric, int64_t id_offset,
                  int64_t* out_ids, double* out_dist, int32_t* out_count, int64_t* out_visited) {
    if (!ctx || !data) return set_err(VS_ERR_PARAMETER, "null argument");
    CKS(validate_metric(metric));
    CKS(validate_k(k));
    if (d != data->d) return set_err(VS_ERR_SHAPE, "query dim %d != data dim %d", d, data->d);
    if (nq < 0) return set_err(VS_ERR_PARAMETER, "negative query count");
    if (bitmap && nbits != data->n)
        return set_err(VS_ERR_SHAPE, "bitmap covers %lld rows, column has %lld", (long long)nbits,
                       (long long)data->n);
    if (data->n == 0) return set_err(VS_ERR_EMPTY_INPUT, "exhaustive search over empty data side");
    DevGuard g(ctx->device);
    vs_column* col = const_cast<vs_column*>(data);
    CK(ctx->arena.reset());
    std::vector<OutBuf> pending;
    const float* dq = nullptr;
    // host queries of a large batch: copy them in on the copy stream while the
    // filter and the row staging run (phase A waits on q_ready)
    cudaEvent_t q_ready = nullptr;
    {
        cudaPointerAttributes at{};
        const bool host_q = queries && cudaPointerGetAttributes(&at, queries) == cudaSuccess &&
                            at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged;
        cudaGetLastError();
        if (host_q && !data->host_resident && (size_t)nq * d * 4 >= ((size_t)1 << 22)) {
            float* buf = nullptr;
            CKS(arena_alloc(ctx, (size_t)nq * d, &buf));
            if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
            if (!ctx->q_event) CK(cudaEventCreateWithFlags(&ctx->q_event, cudaEventDisableTiming));
            CK(cudaEventRecord(ctx->q_event, ctx->stream));            // earlier work on the buffer
            CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->q_event, 0));
            CK(cudaMemcpyAsync(buf, queries, (size_t)nq * d * 4, cudaMemcpyHostToDevice, ctx->copy_stream));
            CK(cudaEventRecord(ctx->q_event, ctx->copy_stream));
            q_ready = ctx->q_event;
            dq = buf;
        } else {
            CKS(stage_in(ctx, queries, (size_t)nq * d, &dq));
        }
    }
    int64_t* sel = nullptr;
    int64_t nsel = data->n;
    if (bitmap) {
        const uint32_t* dbm = nullptr;
        CKS(stage_in(ctx, bitmap, (size_t)(nbits + 31) / 32, &dbm));
        CKS(build_selection(ctx, dbm, nbits, &sel, &nsel));
        if (nsel == 0) return set_err(VS_ERR_EMPTY_INPUT, "exhaustive search over empty data side");
    }
    if (out_visited) *out_visited = nq * nsel;
    if (nq == 0) return VS_OK;
    CKS(ensure_norms(col, ctx));
    float* margin = nullptr;
    CKS(arena_alloc(ctx, (size_t)nq, &margin));
    if (!q_ready) {
        CK(vs::launch_query_margins(dq, nq, d, col->max_norm_bits, eps_simt(d), metric, margin, nullptr,
                                    ctx->stream));
        ctx->stats[VS_STAT_LAUNCHES] += 1;
    }
    EnnJob job;
    job.q_ready = q_ready;
    job.margin_todo = q_ready ? margin : nullptr;
    job.q = dq;
    job.nq = nq;
    job.d = d;
    job.rows = col->data;
    job.dtype = col->dtype;
    job.sel = sel;
    job.nsel = nsel;
    job.xnorm = col->norms;
    job.xmax = col->max_norm_bits;
    job.ip = metric;
    job.k = k;
    job.id_offset = id_offset;
    CKS(ensure_f16_shadow(ctx, col, nq, nsel));
    job.f16 = col->f16_ready ? col->f16 : nullptr;
    job.f16_stats = col->f16_ready ? col->f16_stats : nullptr;
    const bool zc = !col->host_resident && k <= kTopkCap;   // outputs written once, by phase B
    CKS(stage_out_final(ctx, out_ids, (size_t)nq * k, &job.out_ids, pending, zc));
    CKS(stage_out_final(ctx, out_dist, (size_t)nq * k, &job.out_dist, pending, zc));
    CKS(stage_out_final(ctx, out_count, (size_t)nq, &job.out_count, pending, zc));
    job.out_ids32 = nullptr;
    if (col->host_resident && k <= kTopkCap) {
        CKS(enn_search_streamed(ctx, col, dq, nq, d, sel, nsel, k, metric, id_offset, margin, job.out_ids,
                                job.out_dist, job.out_count));
    } else {
        CKS(run_enn(ctx, job, margin, 0, true));
    }
    CKS(flush_out(ctx, pending));
    return VS_OK;
}

// ---- two-phase exact search for row-sharded collections --------------------------
// begin: phase A on this shard + upper bounds on the exact keys of the
// shard's k smallest approximate keys (approx + margin/2); the caller takes the
// k-th of their union over shards, T >= the global k-th exact key; finish:
// phase B re-ranks only the candidates with key <= min(K* + margin, T +
// margin/2) (this shard's own margin), so the
// exact work per shard shrinks with the number of shards. out_bound returns,
// per query, a value below which no dropped candidate of this shard lies
// (key space: distance, or -score); the merged k-th key must stay below the
// MIN over shards of out_bound, else the query is re-run (distributed.py).
}  // extern "C"
namespace {
struct PendingEnn {
    EnnJob job;
    PhaseA st;
    bool active = false;
};
// begin/finish state per context. Contexts are driven from different threads
// (one per shard) and ctypes releases the GIL, so the map is guarded; entries
// are node-stable, so a reference stays valid while its context is in use.
std::mutex& pending_mu() {
    static std::mutex m;
    return m;
}
std::unordered_map<const vs_ctx*, PendingEnn>& pending_map() {
    static std::unordered_map<const vs_ctx*, PendingEnn> m;
    return m;
}
PendingEnn& pending_of(const vs_ctx* ctx) {
    std::lock_guard<std::mutex> lk(pending_mu());
    return pending_map()[ctx];
}
PendingEnn* pending_find(const vs_ctx* ctx) {
    std::lock_guard<std::mutex> lk(pending_mu());
    auto it = pending_map().find(ctx);
    return it == pending_map().end() ? nullptr : &it->second;
}
}  // namespace
void pending_erase(const vs_ctx* ctx) {
    std::lock_guard<std::mutex> lk(pending_mu());
    pending_map().erase(ctx);
}
extern "C" {

int vs_enn_search_begin(vs_ctx* ctx, const vs_column* data, const float* queries, int64_t nq, int32_t d,
                        const uint32_t* bitmap, int64_t nbits, int32_t k, int32_t metric, float* out_kth,
                        int64_t* out_visited) {
    if (!ctx || !data) return set_err(VS_ERR_PARAMETER, "null argument");
    CKS(validate_metric(metric));
    CKS(validate_k(k));
    if (d != data->d) return set_err(VS_ERR_SHAPE, "query dim %d != data dim %d", d, data->d);
    if (nq < 0) return set_err(VS_ERR_PARAMETER, "negative query count");
    if (data->host_resident) return set_err(VS_ERR_PARAMETER, "two-phase search needs a device-resident shard");
    if (k > kTopkCap)
        return set_err(VS_ERR_CAP_EXCEEDED, "two-phase search supports k' <= %d (use the one-phase search)", kTopkCap);
    if (bitmap && nbits != data->n)
        return set_err(VS_ERR_SHAPE, "bitmap covers %lld rows, column has %lld", (long long)nbits,
                       (long long)data->n);
    DevGuard g(ctx->device);
    vs_column* col = const_cast<vs_column*>(data);
    CK(ctx->arena.reset());
    PendingEnn& pe = pending_of(ctx);
    pe.active = false;
    std::vector<OutBuf> pending;
    const float* dq = nullptr;
    CKS(stage_in(ctx, queries, (size_t)nq * d, &dq));
    int64_t* sel = nullptr;
    int64_t nsel = data->n;
    if (bitmap) {
        const uint32_t* dbm = nullptr;
        CKS(stage_in(ctx, bitmap, (size_t)(nbits + 31) / 32, &dbm));
        CKS(build_selection(ctx, dbm, nbits, &sel, &nsel));
    }
    if (out_visited) *out_visited = nq * nsel;
    EnnJob& job = pe.job;
    job = EnnJob{};
    job.q = dq;
    job.nq = nq;
    job.d = d;
    job.rows = col->data;
    job.dtype = col->dtype;
    job.sel = sel;
    job.nsel = nsel;
    job.ip = metric;
    job.k = k;
    job.id_offset = 0;
    if (nq == 0 || nsel == 0) {   // an empty shard: no candidates, no bound
        float* dk = nullptr;
        CKS(stage_out(ctx, out_kth, (size_t)nq * k, &dk, pending));
        if (dk && nq) {
            std::vector<float> inf((size_t)nq * k, std::numeric_limits<float>::infinity());
            CK(cudaMemcpyAsync(dk, inf.data(), inf.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        }
        CKS(flush_out(ctx, pending));
        pe.active = true;
        return VS_OK;
    }
    CKS(ensure_norms(col, ctx));
    job.xnorm = col->norms;
    job.xmax = col->max_norm_bits;
    CKS(ensure_f16_shadow(ctx, col, nq, nsel));
    job.f16 = col->f16_ready ? col->f16 : nullptr;
    job.f16_stats = col->f16_ready ? col->f16_stats : nullptr;
    float* margin = nullptr;
    CKS(arena_alloc(ctx, (size_t)nq, &margin));
    CK(vs::launch_query_margins(dq, nq, d, col->max_norm_bits, eps_simt(d), metric, margin, nullptr,
                                ctx->stream));
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    CKS(enn_phase_a(ctx, job, margin, 0, &pe.st));
    float* dk = nullptr;
    CKS(stage_out(ctx, out_kth, (size_t)nq * k, &dk, pending));
    if (!dk) CKS(arena_alloc(ctx, (size_t)nq * k, &dk));
    PhaseBHooks hk;
    hk.out_kth = dk;
    CKS(enn_phase_b(ctx, job, pe.st, 0, false, hk));
    CKS(flush_out(ctx, pending));
    pe.active = true;
    return VS_OK;
}

int vs_union_kth(vs_ctx* ctx, int32_t nparts, int64_t nq, int32_t k, const float* keys, float* out) {
    if (!ctx || nparts < 1 || k < 1 || nq < 0) return set_err(VS_ERR_PARAMETER, "bad union-kth shape");
    if ((int64_t)nparts * k > 16384) return set_err(VS_ERR_PARAMETER, "nparts * k above 16384");
    if (nq == 0) return VS_OK;
    DevGuard g(ctx->device);
    // no arena reset: called between vs_enn_search_begin and _finish on the
    // same context, whose pending state lives in the arena
    std::vector<OutBuf> pending;
    const float* dkeys = nullptr;
    CKS(stage_in(ctx, keys, (size_t)nparts * nq * k, &dkeys));
    float* dout = nullptr;
    CKS(stage_out(ctx, out, (size_t)nq, &dout, pending));
    CK(vs::launch_union_kth(dkeys, nparts, nq, k, dout, ctx->stream));
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    CKS(flush_out(ctx, pending));
    return VS_OK;
}

int vs_enn_search_finish(vs_ctx* ctx, const float* thresholds, int64_t id_offset, int64_t* out_ids,
                         double* out_dist, int32_t* out_count, double* out_bound) {
    if (!ctx) return set_err(VS_ERR_PARAMETER, "null ctx");
    PendingEnn* pf = pending_find(ctx);
    if (!pf || !pf->active)
        return set_err(VS_ERR_PARAMETER, "vs_enn_search_finish without vs_enn_search_begin");
    DevGuard g(ctx->device);
    PendingEnn& pe = *pf;
    pe.active = false;
    EnnJob job = pe.job;
    const int64_t nq = job.nq;
    const int k = job.k;
    std::vector<OutBuf> pending;
    CKS(stage_out(ctx, out_ids, (size_t)nq * k, &job.out_ids, pending));
    CKS(stage_out(ctx, out_dist, (size_t)nq * k, &job.out_dist, pending));
    CKS(stage_out(ctx, out_count, (size_t)nq, &job.out_count, pending));
    double* dbound = nullptr;
    CKS(stage_out(ctx, out_bound, (size_t)nq, &dbound, pending));
    job.out_ids32 = nullptr;
    job.id_offset = id_offset;
    if (nq == 0) return VS_OK;
    if (job.nsel == 0) {   // empty shard: empty rows, no bound
        if (job.out_ids) CK(cudaMemsetAsync(job.out_ids, 0xff, (size_t)nq * k * sizeof(int64_t), ctx->stream));
        if (job.out_dist) {
            std::vector<double> nan((size_t)nq * k, std::numeric_limits<double>::quiet_NaN());
            CK(cudaMemcpyAsync(job.out_dist, nan.data(), nan.size() * sizeof(double), cudaMemcpyHostToDevice,
                               ctx->stream));
        }
        if (job.out_count) CK(cudaMemsetAsync(job.out_count, 0, (size_t)nq * sizeof(int32_t), ctx->stream));
        if (dbound) {
            std::vector<double> inf(nq, std::numeric_limits<double>::infinity());
            CK(cudaMemcpyAsync(dbound, inf.data(), nq * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        }
        CKS(flush_out(ctx, pending));
        return VS_OK;
    }
    const float* dthr = nullptr;
    CKS(stage_in(ctx, thresholds, (size_t)nq, &dthr));
    if (!dbound) CKS(arena_alloc(ctx, (size_t)nq, &dbound));
    PhaseBHooks hk;
    hk.ext_thr = dthr;
    hk.out_bound = dbound;
    CKS(enn_phase_b(ctx, job, pe.st, 0, true, hk));
    CKS(flush_out(ctx, pending));
    return VS_OK;
}

// ---- relational filters -> packed row bitmaps ----------------------------------
static size_t value_size(int vtype) { return vtype == 0 || vtype == 2 ? 4 : 8; }

int vs_bitmap_compare(vs_ctx* ctx, const void* values, int32_t vtype, int64_t n, int32_t op, double value,
                      const uint32_t* valid_bits, uint32_t* out_bits) {
    if (!ctx || (!values && n > 0) || !out_bits) return set_err(VS_ERR_PARAMETER, "null argument");
    if (vtype < 0 || vtype > 3) return set_err(VS_ERR_PARAMETER, "unknown value type %d", vtype);
    if (op < 0 || op > 5) return set_err(VS_ERR_PARAMETER, "unknown comparison %d", op);
    if (n < 0) return set_err(VS_ERR_PARAMETER, "negative row count");
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<OutBuf> pending;
    const char* dv = nullptr;
    CKS(stage_in(ctx, static_cast<const char*>(values), (size_t)n * value_size(vtype), &dv));
    const uint32_t* dvalid = nullptr;
    CKS(stage_in(ctx, valid_bits, (size_t)(n + 31) / 32, &dvalid));
    uint32_t* dout = nullptr;
    CKS(stage_out(ctx, out_bits, (size_t)(n + 31) / 32, &dout, pending));
    {
        KTimer kt(ctx, VS_K_SELECT);
        CK(vs::launch_bitmap_compare(dv, vtype, n, op, value, dvalid, dout, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    CKS(flush_out(ctx, pending));
    return VS_OK;
}

int vs_bitmap_isin(vs_ctx* ctx, const int64_t* keys, int64_t n, const uint32_t* valid_bits, const int64_t* set,
                   int64_t nset, uint32_t* out_bits) {
    if (!ctx || (!keys && n > 0) || (!set && nset > 0) || !out_bits) return set_err(VS_ERR_PARAMETER, "null argument");
    if (n < 0 || nset < 0) return set_err(VS_ERR_PARAMETER, "negative size");
    if (nset >= (int64_t(1) << 31)) return set_err(VS_ERR_PARAMETER, "set too large");
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<OutBuf> pending;
    const int64_t* dk = nullptr;
    const int64_t* ds = nullptr;
    const uint32_t* dvalid = nullptr;
    CKS(stage_in(ctx, keys, (size_t)n, &dk));
    CKS(stage_in(ctx, set, (size_t)nset, &ds));
    CKS(stage_in(ctx, valid_bits, (size_t)(n + 31) / 32, &dvalid));
    int64_t* sorted = nullptr;
    CKS(arena_alloc(ctx, (size_t)std::max<int64_t>(nset, 1), &sorted));
    const size_t tb = vs::bitmap_isin_temp_bytes(nset);
    char* tmp = nullptr;
    CKS(arena_alloc(ctx, tb, &tmp));
    uint32_t* dout = nullptr;
    CKS(stage_out(ctx, out_bits, (size_t)(n + 31) / 32, &dout, pending));
    {
        KTimer kt(ctx, VS_K_SELECT);
        CK(vs::launch_bitmap_isin(dk, n, dvalid, ds, nset, sorted, tmp, tb, dout, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 2;
    CKS(flush_out(ctx, pending));
    return VS_OK;
}

// ---- after the search: post-filter, flat output table, row gather (vs_output.cu) -----
int vs_postfilter(vs_ctx* ctx, const int64_t* ids, const double* dist, const int32_t* counts, int64_t nq,
                  int32_t k_prime, const uint32_t* keep_bits, const uint8_t* keep_pos, const int64_t* data_key,
                  const int64_t* query_key, int32_t key_op, int64_t n_data, int32_t k, int64_t* out_ids,
                  double* out_dist, int32_t* out_rank, int32_t* out_count) {
    if (!ctx || ((!ids || !dist) && nq > 0)) return set_err(VS_ERR_PARAMETER, "null argument");
    if (nq < 0 || k_prime < 0 || n_data < 0) return set_err(VS_ERR_PARAMETER, "negative size");
    if (k < 1) return set_err(VS_ERR_PARAMETER, "k must be >= 1, got %d", k);
    if (!data_key != !query_key) return set_err(VS_ERR_PARAMETER, "data_key and query_key go together");
    if (data_key && (key_op < 0 || key_op > 5)) return set_err(VS_ERR_PARAMETER, "unknown comparison %d", key_op);
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<OutBuf> pending;
    vs::PostfilterArgs a{};
    const size_t slots = (size_t)nq * k_prime;
    CKS(stage_in(ctx, ids, slots, &a.ids));
    CKS(stage_in(ctx, dist, slots, &a.dist));
    CKS(stage_in(ctx, counts, (size_t)nq, &a.counts));
    CKS(stage_in(ctx, keep_bits, (size_t)(n_data + 31) / 32, &a.bitmap));
    CKS(stage_in(ctx, keep_pos, slots, &a.keep_pos));
    CKS(stage_in(ctx, data_key, (size_t)n_data, &a.data_key));
    CKS(stage_in(ctx, query_key, (size_t)nq, &a.query_key));
    a.nq = nq;
    a.kp = k_prime;
    a.key_op = key_op;
    a.n_data = n_data;
    a.k = k;
    CKS(stage_out(ctx, out_ids, (size_t)nq * k, &a.out_ids, pending));
    CKS(stage_out(ctx, out_dist, (size_t)nq * k, &a.out_dist, pending));
    CKS(stage_out(ctx, out_rank, (size_t)nq * k, &a.out_rank, pending));
    CKS(stage_out(ctx, out_count, (size_t)nq, &a.out_count, pending));
    CKS(arena_alloc(ctx, 1, &a.bad));
    CK(cudaMemsetAsync(a.bad, 0, sizeof(int), ctx->stream));
    {
        KTimer kt(ctx, VS_K_SELECT);
        CK(vs::launch_postfilter(a, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, a.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CKS(flush_out(ctx, pending));
    if (bad) return set_err(VS_ERR_PARAMETER, "data row id outside [0, %lld)", (long long)n_data);
    return VS_OK;
}

int vs_results_flatten(vs_ctx* ctx, const int64_t* ids, const double* dist, const int32_t* rank,
                       const int32_t* counts, int64_t nq, int32_t k_prime, int64_t query_offset,
                       int64_t* query_row, int64_t* data_row, double* distance, int64_t* out_rank,
                       int64_t* n_out) {
    if (!ctx || !n_out || ((!ids || !dist) && nq > 0)) return set_err(VS_ERR_PARAMETER, "null argument");
    if (nq < 0 || k_prime < 0) return set_err(VS_ERR_PARAMETER, "negative size");
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<OutBuf> pending;
    vs::FlattenArgs a{};
    const size_t slots = (size_t)nq * k_prime;
    CKS(stage_in(ctx, ids, slots, &a.ids));
    CKS(stage_in(ctx, dist, slots, &a.dist));
    CKS(stage_in(ctx, rank, slots, &a.in_rank));
    CKS(stage_in(ctx, counts, (size_t)nq, &a.counts));
    a.nq = nq;
    a.kp = k_prime;
    a.query_offset = query_offset;
    CKS(stage_out(ctx, query_row, slots, &a.query_row, pending));
    CKS(stage_out(ctx, data_row, slots, &a.data_row, pending));
    CKS(stage_out(ctx, distance, slots, &a.distance, pending));
    CKS(stage_out(ctx, out_rank, slots, &a.rank, pending));
    int64_t *c64 = nullptr, *off = nullptr;
    CKS(arena_alloc(ctx, (size_t)nq + 1, &c64));
    CKS(arena_alloc(ctx, (size_t)nq + 1, &off));
    const size_t tb = vs::flatten_temp_bytes(nq);
    char* tmp = nullptr;
    CKS(arena_alloc(ctx, tb, &tmp));
    {
        KTimer kt(ctx, VS_K_SELECT);
        CK(vs::launch_flatten(a, c64, off, tmp, tb, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 3;
    int64_t total = 0;
    CK(cudaMemcpyAsync(&total, off + nq, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (auto& o : pending) o.bytes = (size_t)total * 8;   // every flat column is 8 bytes wide
    CKS(flush_out(ctx, pending));
    *n_out = total;
    return VS_OK;
}

int vs_gather_rows(vs_ctx* ctx, const void* src, int64_t n_src, int64_t row_bytes, const int64_t* idx, int64_t n,
                   void* dst) {
    if (!ctx || ((!src || !idx || !dst) && n > 0 && row_bytes > 0)) return set_err(VS_ERR_PARAMETER, "null argument");
    if (n_src < 0 || row_bytes < 0 || n < 0) return set_err(VS_ERR_PARAMETER, "negative size");
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<OutBuf> pending;
    const char* dsrc = nullptr;
    const int64_t* didx = nullptr;
    CKS(stage_in(ctx, static_cast<const char*>(src), (size_t)(n_src * row_bytes), &dsrc));
    CKS(stage_in(ctx, idx, (size_t)n, &didx));
    char* ddst = nullptr;
    CKS(stage_out(ctx, static_cast<char*>(dst), (size_t)(n * row_bytes), &ddst, pending));
    int* bad = nullptr;
    CKS(arena_alloc(ctx, 1, &bad));
    CK(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    {
        KTimer kt(ctx, VS_K_SELECT);
        CK(vs::launch_gather(dsrc, n_src, row_bytes, didx, n, ddst, bad, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    int h_bad = 0;
    CK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CKS(flush_out(ctx, pending));
    if (h_bad) return set_err(VS_ERR_PARAMETER, "gather index outside [0, %lld)", (long long)n_src);
    return VS_OK;
}

int vs_bitmap_combine(vs_ctx* ctx, const uint32_t* a, const uint32_t* b, int64_t nwords, int32_t op,
                      uint32_t* out) {
    if (!ctx || ((!a || !b || !out) && nwords > 0)) return set_err(VS_ERR_PARAMETER, "null argument");
    if (op < 0 || op > 2) return set_err(VS_ERR_PARAMETER, "unknown bitmap op %d", op);
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<OutBuf> pending;
    const uint32_t *da = nullptr, *db = nullptr;
    CKS(stage_in(ctx, a, (size_t)nwords, &da));
    CKS(stage_in(ctx, b, (size_t)nwords, &db));
    uint32_t* dout = nullptr;
    CKS(stage_out(ctx, out, (size_t)nwords, &dout, pending));
    CK(vs::launch_bitmap_combine(da, db, nwords, op, dout, ctx->stream));
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    CKS(flush_out(ctx, pending));
    return VS_OK;
}

int vs_topk_merge(vs_ctx* ctx, int32_t nparts, int64_t nq, int32_t k_in, const int64_t* ids,
                  const double* dist, const int32_t* counts, int32_t k, int32_t metric,
                  int64_t* out_ids, double* out_dist, int32_t* out_count) {
    if (!ctx) return set_err(VS_ERR_PARAMETER, "null ctx");
    CKS(validate_metric(metric));
    CKS(validate_k(k));
    if (nparts < 1 || k_in < 1 || nq < 0) return set_err(VS_ERR_PARAMETER, "bad merge shape");
    if (nq == 0) return VS_OK;
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<OutBuf> pending;
    vs::MergeParams p;
    p.nparts = nparts;
    p.nq = nq;
    p.k_in = k_in;
    p.k = k;
    p.ip = metric;
    const size_t n_in = (size_t)nparts * nq * k_in;
    CKS(stage_in(ctx, ids, n_in, &p.ids));
    CKS(stage_in(ctx, dist, n_in, &p.dist));
    CKS(stage_in(ctx, counts, (size_t)nparts * nq, &p.counts));
    CKS(stage_out(ctx, out_ids, (size_t)nq * k, &p.out_ids, pending));
    CKS(stage_out(ctx, out_dist, (size_t)nq * k, &p.out_dist, pending));
    CKS(stage_out(ctx, out_count, (size_t)nq, &p.out_count, pending));
    if (k > kTopkCap) {
        CKS(vs::wide_merge(ctx, nparts, nq, k_in, p.ids, p.dist, p.counts, k, metric, p.out_ids, p.out_dist,
                           p.out_count));
        CKS(flush_out(ctx, pending));
        return VS_OK;
    }
    CKS(arena_alloc(ctx, n_in, &p.s_key));
    CKS(arena_alloc(ctx, n_in, &p.s_id));
    {
        KTimer kt(ctx, VS_K_MERGE);
        CK(vs::launch_merge(p, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    CKS(flush_out(ctx, pending));
    return VS_OK;
}

}  // extern "C"

// Build the device IVF structure. centroids / list_ids / list_payload may be
// host or device pointers; sizes are host. Non-owning (payload == nullptr):
// rows are gathered from `base` into the list-contiguous layout.
int ivf_make(vs_ctx* ctx, const float* centroids, int32_t nlist, int32_t d, const std::vector<int64_t>& sizes,
             const int64_t* list_ids, const void* list_payload, int32_t dtype, int32_t metric,
             const vs_column* base, const uint8_t* list_owned, vs_ivf** out, bool borrow_payload) {
    std::vector<int64_t> off(nlist + 1, 0);
    for (int i = 0; i < nlist; ++i) {
        if (sizes[i] < 0) return set_err(VS_ERR_PARAMETER, "negative list size");
        off[i + 1] = off[i] + sizes[i];
    }
    const int64_t n_total = off[nlist];
    if (n_total > 0 && !list_ids) return set_err(VS_ERR_PARAMETER, "null list ids");
    vs_ivf* v = new vs_ivf();
    v->ctx = ctx;
    ctx_ref(ctx);   // balanced by vs_ivf_free (also on the failure paths below)
    v->nlist = nlist;
    v->d = d;
    v->metric = metric;
    v->dtype = dtype;
    v->n_total = n_total;
    v->h_off = off;
    auto fail = [&](cudaError_t e, const char* what) {
        cudaGetLastError();
        vs_ivf_free(v);
        return cuda_err(e, what);
    };
    cudaError_t e;
    const size_t es = elem_size(dtype);
    if ((e = cudaMalloc(&v->centroids, (size_t)nlist * d * sizeof(float))) != cudaSuccess) return fail(e, "alloc");
    if ((e = cudaMalloc(&v->cnorms, (size_t)nlist * sizeof(float))) != cudaSuccess) return fail(e, "alloc");
    if ((e = cudaMalloc(&v->cmax, sizeof(unsigned))) != cudaSuccess) return fail(e, "alloc");
    if ((e = cudaMalloc(&v->list_off, (size_t)(nlist + 1) * sizeof(int64_t))) != cudaSuccess) return fail(e, "alloc");
    if ((e = cudaMalloc(&v->list_ids, std::max<size_t>(n_total, 1) * sizeof(int64_t))) != cudaSuccess) return fail(e, "alloc");
    if (borrow_payload) {
        v->payload = const_cast<void*>(list_payload);
        v->payload_borrowed = true;
    } else if ((e = cudaMalloc(&v->payload, std::max<size_t>((size_t)n_total * d * es, 16))) != cudaSuccess) {
        return fail(e, "alloc");
    }
    if ((e = cudaMalloc(&v->pnorms, std::max<size_t>(n_total, 1) * sizeof(float))) != cudaSuccess) return fail(e, "alloc");
    if ((e = cudaMalloc(&v->pmax, sizeof(unsigned))) != cudaSuccess) return fail(e, "alloc");
    cudaStream_t s = ctx->stream;
    if ((e = cudaMemcpyAsync(v->centroids, centroids, (size_t)nlist * d * sizeof(float), cudaMemcpyDefault, s)) != cudaSuccess) return fail(e, "upload");
    if ((e = cudaMemcpyAsync(v->list_off, off.data(), (nlist + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s)) != cudaSuccess) return fail(e, "upload");
    if (n_total > 0) {
        if ((e = cudaMemcpyAsync(v->list_ids, list_ids, n_total * sizeof(int64_t), cudaMemcpyDefault, s)) != cudaSuccess) return fail(e, "upload");
        if (borrow_payload) {
            // borrowed in place
        } else if (list_payload) {
            if ((e = cudaMemcpyAsync(v->payload, list_payload, (size_t)n_total * d * es, cudaMemcpyDefault, s)) != cudaSuccess) return fail(e, "upload");
        } else {
            if (dtype == VS_DTYPE_F32)
                e = vs::launch_gather_rows<float>((const float*)base->data, v->list_ids, n_total, d, (float*)v->payload, s);
            else
                e = vs::launch_gather_rows<__nv_bfloat16>((const __nv_bfloat16*)base->data, v->list_ids, n_total, d,
                                                          (__nv_bfloat16*)v->payload, s);
            if (e != cudaSuccess) return fail(e, "gather");
            ctx->stats[VS_STAT_LAUNCHES] += 1;
        }
    }
    if (list_owned) {
        if ((e = cudaMalloc(&v->owned, nlist)) != cudaSuccess) return fail(e, "alloc");
        if ((e = cudaMemcpyAsync(v->owned, list_owned, nlist, cudaMemcpyDefault, s)) != cudaSuccess) return fail(e, "upload");
    }
    cudaMemsetAsync(v->cmax, 0, sizeof(unsigned), s);
    cudaMemsetAsync(v->pmax, 0, sizeof(unsigned), s);
    if ((e = vs::launch_row_norms<float>(v->centroids, nlist, d, v->cnorms, v->cmax, s)) != cudaSuccess) return fail(e, "norms");
    if (dtype == VS_DTYPE_F32)
        e = vs::launch_row_norms<float>((const float*)v->payload, n_total, d, v->pnorms, v->pmax, s);
    else
        e = vs::launch_row_norms<__nv_bfloat16>((const __nv_bfloat16*)v->payload, n_total, d, v->pnorms, v->pmax, s);
    if (e != cudaSuccess) return fail(e, "norms");
    ctx->stats[VS_STAT_LAUNCHES] += 2;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(e, "sync");
    *out = v;
    return VS_OK;
}

extern "C" {

int vs_ivf_create(vs_ctx* ctx, const float* centroids, int32_t nlist, int32_t d,
                  const int64_t* list_sizes, const int64_t* list_ids, const void* list_payload,
                  int32_t dtype, int32_t metric, const vs_column* base, const uint8_t* list_owned,
                  vs_ivf** out) {
    if (!ctx || !out || !centroids || !list_sizes) return set_err(VS_ERR_PARAMETER, "null argument");
    CKS(validate_metric(metric));
    if (nlist < 1) return set_err(VS_ERR_PARAMETER, "nlist must be >= 1");
    if (d < 1) return set_err(VS_ERR_SHAPE, "embedding dimension must be >= 1");
    if (dtype != VS_DTYPE_F32 && dtype != VS_DTYPE_BF16) return set_err(VS_ERR_PARAMETER, "bad dtype");
    if (!list_payload && !base) return set_err(VS_ERR_PARAMETER, "non-owning IVF needs a base column");
    if (base && base->d != d) return set_err(VS_ERR_SHAPE, "base dim %d != index dim %d", base->d, d);
    if (!list_payload && base->dtype != dtype) return set_err(VS_ERR_PARAMETER, "base dtype mismatch");
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<int64_t> sizes(nlist);
    CK(cudaMemcpy(sizes.data(), list_sizes, nlist * sizeof(int64_t), cudaMemcpyDefault));
    return ivf_make(ctx, centroids, nlist, d, sizes, list_ids, list_payload, dtype, metric, base, list_owned, out);
}

int vs_ivf_wrap(vs_ctx* ctx, const float* centroids, int32_t nlist, int32_t d, const int64_t* list_sizes,
                const int64_t* list_ids, void* payload_dev, int32_t dtype, int32_t metric, vs_ivf** out) {
    if (!ctx || !out || !centroids || !list_sizes) return set_err(VS_ERR_PARAMETER, "null argument");
    CKS(validate_metric(metric));
    if (nlist < 1) return set_err(VS_ERR_PARAMETER, "nlist must be >= 1");
    if (d < 1) return set_err(VS_ERR_SHAPE, "embedding dimension must be >= 1");
    if (dtype != VS_DTYPE_F32 && dtype != VS_DTYPE_BF16) return set_err(VS_ERR_PARAMETER, "bad dtype");
    cudaPointerAttributes at{};
    if (!payload_dev || cudaPointerGetAttributes(&at, payload_dev) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        return set_err(VS_ERR_PARAMETER, "vs_ivf_wrap needs a device payload pointer");
    }
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<int64_t> sizes(nlist);
    CK(cudaMemcpy(sizes.data(), list_sizes, nlist * sizeof(int64_t), cudaMemcpyDefault));
    return ivf_make(ctx, centroids, nlist, d, sizes, list_ids, payload_dev, dtype, metric, nullptr, nullptr, out,
                    true);
}

int vs_ivf_info(const vs_ivf* ivf, int32_t* nlist, int32_t* d, int64_t* n_total, int32_t* metric,
                int32_t* dtype) {
    if (!ivf) return set_err(VS_ERR_PARAMETER, "null ivf");
    if (nlist) *nlist = ivf->nlist;
    if (d) *d = ivf->d;
    if (n_total) *n_total = ivf->n_total;
    if (metric) *metric = ivf->metric;
    if (dtype) *dtype = ivf->dtype;
    return VS_OK;
}

int vs_ivf_export(vs_ivf* ivf, float* centroids, int64_t* list_sizes, int64_t* list_ids,
                  void* list_payload) {
    if (!ivf) return set_err(VS_ERR_PARAMETER, "null ivf");
    DevGuard g(ivf->ctx->device);
    cudaStream_t s = ivf->ctx->stream;
    if (centroids) CK(cudaMemcpyAsync(centroids, ivf->centroids, (size_t)ivf->nlist * ivf->d * sizeof(float), cudaMemcpyDefault, s));
    if (list_sizes) {
        std::vector<int64_t> sz(ivf->nlist);
        for (int i = 0; i < ivf->nlist; ++i) sz[i] = ivf->h_off[i + 1] - ivf->h_off[i];
        CK(cudaMemcpyAsync(list_sizes, sz.data(), ivf->nlist * sizeof(int64_t), cudaMemcpyDefault, s));
        CK(cudaStreamSynchronize(s));
    }
    if (list_ids && ivf->n_total) CK(cudaMemcpyAsync(list_ids, ivf->list_ids, ivf->n_total * sizeof(int64_t), cudaMemcpyDefault, s));
    if (list_payload && ivf->n_total)
        CK(cudaMemcpyAsync(list_payload, ivf->payload, (size_t)ivf->n_total * ivf->d * elem_size(ivf->dtype), cudaMemcpyDefault, s));
    CK(cudaStreamSynchronize(s));
    return VS_OK;
}

int vs_ivf_set_owned(vs_ivf* ivf, const uint8_t* list_owned) {
    if (!ivf) return set_err(VS_ERR_PARAMETER, "null ivf");
    DevGuard g(ivf->ctx->device);
    cudaStream_t s = ivf->ctx->stream;
    if (!list_owned) {
        if (ivf->owned) CK(cudaFree(ivf->owned));
        ivf->owned = nullptr;
        return VS_OK;
    }
    if (!ivf->owned) CK(cudaMalloc(&ivf->owned, ivf->nlist));
    CK(cudaMemcpyAsync(ivf->owned, list_owned, ivf->nlist, cudaMemcpyDefault, s));
    CK(cudaStreamSynchronize(s));
    return VS_OK;
}

int vs_ivf_free(vs_ivf* v) {
    if (!v) return VS_OK;
    DevGuard g(v->ctx->device);
    cudaStreamSynchronize(v->ctx->stream);
    cudaFree(v->centroids);
    cudaFree(v->cnorms);
    cudaFree(v->cmax);
    cudaFree(v->list_off);
    cudaFree(v->list_ids);
    if (!v->payload_borrowed) cudaFree(v->payload);
    cudaFree(v->pnorms);
    cudaFree(v->pmax);
    if (v->owned) cudaFree(v->owned);
    vs_ctx* ctx = v->ctx;
    delete v;
    ctx_unref(ctx);
    return VS_OK;
}

}  // extern "C"

// ---- IVF search driver --------------------------------------------------------------------
namespace {

struct IvfJob {
    const vs_ivf* ivf;
    const float* q;
    int64_t nq;
    const int32_t* probes;
    int nprobe;
    const uint32_t* pbits;
    int k;
    int64_t* out_ids;
    double* out_dist;
    int32_t* out_count;
    unsigned long long* visited;  // nullable (retries do not count)
};

// group the batch's (query, probe) pairs by list and cut them into units of
// <= unit_pairs pairs of one list (list-major scans)
struct IvfGroups {
    int32_t* pair_codes = nullptr;
    int4* units = nullptr;
    int32_t* uoff = nullptr;
    int64_t max_units = 0;
    int64_t npairs = 0;
};
int ivf_group(vs_ctx* ctx, const IvfJob& job, int unit_pairs, IvfGroups* out, const int32_t* chunks = nullptr,
              int max_chunks = 1) {
    const vs_ivf* v = job.ivf;
    const int64_t npairs = job.nq * (int64_t)job.nprobe;
    vs::IvfGroupArgs g;
    g.probes = job.probes;
    g.nq = job.nq;
    g.nprobe = job.nprobe;
    g.nlist = v->nlist;
    g.owned = v->owned;
    g.unit_pairs = unit_pairs;
    g.chunks = chunks;
    CKS(arena_alloc(ctx, (size_t)npairs, &g.keys_in));
    CKS(arena_alloc(ctx, (size_t)npairs, &g.keys_out));
    CKS(arena_alloc(ctx, (size_t)npairs, &g.vals_in));
    CKS(arena_alloc(ctx, (size_t)npairs, &g.pair_codes));
    CKS(arena_alloc(ctx, (size_t)v->nlist + 1, &g.cnt));
    CKS(arena_alloc(ctx, (size_t)v->nlist + 1, &g.qoff));
    CKS(arena_alloc(ctx, (size_t)v->nlist + 1, &g.ucnt));
    CKS(arena_alloc(ctx, (size_t)v->nlist + 1, &g.uoff));
    const int64_t max_units = vs::ivf_max_units(job.nq, job.nprobe, v->nlist, unit_pairs) * max_chunks;
    CKS(arena_alloc(ctx, (size_t)max_units, &g.units));
    g.tmp_bytes = vs::ivf_group_temp_bytes(npairs, v->nlist);
    char* gtmp = nullptr;
    CKS(arena_alloc(ctx, g.tmp_bytes, &gtmp));
    g.tmp = gtmp;
    {
        KTimer kt(ctx, VS_K_SELECT);
        CK(vs::launch_ivf_group(g, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 6;
    out->pair_codes = g.pair_codes;
    out->units = g.units;
    out->uoff = g.uoff;
    out->max_units = max_units;
    out->npairs = npairs;
    return VS_OK;
}

enum IvfKernel { IVF_QMAJOR = 1, IVF_LMAJOR = 2, IVF_TC = 3 };

int choose_ivf_kernel(const vs_ctx* ctx, const vs_ivf* v, const IvfJob& job) {
    const bool tc_ok = v->dtype == VS_DTYPE_BF16 && v->d % 8 == 0 && vs::tc_supported(v->d, v->dtype, v->metric);
    const bool lm_ok = v->d % 4 == 0 && v->d <= vs::kIvfLmDMax;
    switch (ctx->opt_ivf_kernel) {
        case IVF_QMAJOR: return IVF_QMAJOR;
        case IVF_LMAJOR: return lm_ok ? IVF_LMAJOR : IVF_QMAJOR;
        case IVF_TC: return tc_ok ? IVF_TC : (lm_ok ? IVF_LMAJOR : IVF_QMAJOR);
        default: break;
    }
    // auto: dense bf16 lists are a GEMM (tensor cores); filtered lists are a
    // sparse gather (SIMT list-major)
    if (tc_ok && !job.pbits) return IVF_TC;
    return lm_ok ? IVF_LMAJOR : IVF_QMAJOR;
}

int run_ivf_scan(vs_ctx* ctx, const IvfJob& job, const float* margin, int cshift, bool allow_force) {
    if (job.nq == 0) return VS_OK;
    const vs_ivf* v = job.ivf;
    // the largest number of rows one buffer can see bounds the buffer need
    int64_t max_list = 0;
    for (int i = 0; i < v->nlist; ++i) max_list = std::max(max_list, v->h_off[i + 1] - v->h_off[i]);
    const int kern = choose_ivf_kernel(ctx, v, job);
    unsigned long long* vis = job.visited;
    if (!vis) {
        CKS(arena_alloc(ctx, 1, &vis));
        CK(cudaMemsetAsync(vis, 0, sizeof(unsigned long long), ctx->stream));
    }
    vs::CandBuf cb;
    bool exhaustive = false;
    const unsigned* tau_g = nullptr;
    int verify = 0;
    if (kern == IVF_TC) {
        // lists longer than kChunkRows are cut into row chunks, each its own
        // work unit with its own candidate buffers (flat per-query ranges), so
        // one long list cannot hold a CTA for many times the mean work
        const int64_t kChunkRows = ctx->opt_ivf_chunk_rows > 0 ? ctx->opt_ivf_chunk_rows : 512 * 256;
        std::vector<int32_t> h_ch(v->nlist);
        int max_ch = 1;
        for (int i = 0; i < v->nlist; ++i) {
            const int64_t nl = v->h_off[i + 1] - v->h_off[i];
            h_ch[i] = (int32_t)std::max<int64_t>(1, (nl + kChunkRows - 1) / kChunkRows);
            max_ch = std::max(max_ch, (int)h_ch[i]);
        }
        int32_t* d_ch = nullptr;
        if (max_ch > 1) {
            CKS(arena_alloc(ctx, (size_t)v->nlist, &d_ch));
            CK(cudaMemcpyAsync(d_ch, h_ch.data(), v->nlist * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        }
        IvfGroups gr;
        CKS(ivf_group(ctx, job, 128, &gr, d_ch, max_ch));
        vs::TcIvfArgs a;
        a.Q = job.q;
        a.nq = job.nq;
        a.d = v->d;
        a.payload = static_cast<const __nv_bfloat16*>(v->payload);
        a.n_total = v->n_total;
        a.pnorms = v->pnorms;
        a.pmax = v->pmax;
        a.list_off = v->list_off;
        a.max_list = max_list;
        a.pair_codes = gr.pair_codes;
        a.npairs = gr.npairs;
        a.units = gr.units;
        a.n_units = gr.uoff + v->nlist;
        a.max_units = gr.max_units;
        a.nprobe = job.nprobe;
        a.pbits = job.pbits;
        a.k = job.k;
        a.ip = v->metric;
        a.cshift = cshift;
        a.timer_class = VS_K_IVF_SCAN;
        if (max_ch > 1) {
            int64_t *sub_off = nullptr, *pair_base = nullptr;
            char* tmp = nullptr;
            const size_t tb = vs::ivf_pair_subs_temp_bytes(job.nq);
            CKS(arena_alloc(ctx, (size_t)job.nq + 1, &sub_off));
            CKS(arena_alloc(ctx, (size_t)job.nq * job.nprobe, &pair_base));
            CKS(arena_alloc(ctx, tb, &tmp));
            CK(vs::launch_ivf_pair_subs(job.probes, job.nq, job.nprobe, d_ch, sub_off, pair_base, tmp, tb,
                                        ctx->stream));
            int64_t total = 0;
            CK(cudaMemcpyAsync(&total, sub_off + job.nq, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            std::vector<int32_t> srt(h_ch);
            std::sort(srt.begin(), srt.end(), std::greater<int32_t>());
            int64_t bound = 0;
            for (int j = 0; j < job.nprobe && j < (int)srt.size(); ++j) bound += 2 * (int64_t)srt[j];
            a.chunk_rows = kChunkRows;
            a.pair_base = pair_base;
            a.sub_off = sub_off;
            a.total_subs = total;
            a.max_subs = (int)bound;
            ctx->stats[VS_STAT_LAUNCHES] += 3;
        }
        vs::TcIvfOut o;
        CKS(vs::tc_ivf_scan(ctx, a, &o));
        cb = o.cb;
        exhaustive = o.exhaustive;
        margin = o.margin;
        tau_g = o.tau_g;
        verify = o.verify;
        if (job.visited) {
            int32_t* sel = nullptr;
            CKS(arena_alloc(ctx, (size_t)v->nlist, &sel));
            CK(vs::launch_visited_count(job.probes, job.nq, job.nprobe, v->list_off, v->nlist, v->owned, job.pbits,
                                        sel, vis, ctx->stream));
            ctx->stats[VS_STAT_LAUNCHES] += 2;
        }
    } else {
        const bool lmajor = kern == IVF_LMAJOR;
        int n_sub, n_psplit = 1;
        int64_t bound;
        if (lmajor) {
            // one buffer per (query, probe rank): each sees one list
            n_sub = job.nprobe;
            bound = pow2ceil(max_list + 64);
        } else {
            const int64_t target = (int64_t)ctx->sm_count * 8;
            n_psplit = (int)std::min<int64_t>(job.nprobe, std::max<int64_t>(1, (target + job.nq - 1) / job.nq));
            n_sub = n_psplit * 8;
            const int64_t per = (job.nprobe + n_psplit - 1) / n_psplit;
            bound = pow2ceil(per * max_list + 64);
        }
        int64_t C = pow2ceil(std::max<int64_t>(2 * job.k, job.k + 32)) << (ctx->opt_slack + cshift);
        exhaustive = C >= bound;
        if (exhaustive) C = bound;
        cb.n_sub = n_sub;
        cb.C = (int)C;
        const size_t slots = (size_t)job.nq * n_sub * C;
        CKS(arena_alloc(ctx, slots, &cb.key));
        CKS(arena_alloc(ctx, slots, &cb.pos));
        CKS(arena_alloc(ctx, (size_t)job.nq * n_sub, &cb.cnt));
        CKS(arena_alloc(ctx, (size_t)job.nq, &cb.overflow));
        CK(cudaMemsetAsync(cb.overflow, 0, job.nq * sizeof(int), ctx->stream));
        static const int sel_env = getenv("VS_IVF_SEL") ? atoi(getenv("VS_IVF_SEL")) : 1;
        if (lmajor && job.pbits && sel_env && v->n_total < (int64_t)UINT32_MAX) {
            // filtered: pre-selected rows per list, one round trip per unit
            // (vs_ivf_sel.cu); float32 lists with d % 16 == 0 score on the
            // tensor cores (fp16 operands, tensor-core margins for phase B)
            static const int mma_env = getenv("VS_IVF_MMA") ? atoi(getenv("VS_IVF_MMA")) : 1;
            const bool mma = mma_env && v->dtype == VS_DTYPE_F32 && v->d % 16 == 0 && v->d <= 2048 &&
                             ctx->opt_enn_kernel != 1;
            IvfGroups gr;
            CKS(ivf_group(ctx, job, mma ? vs::kMmaPairs : vs::kIvfLmQT, &gr));
            CK(cudaMemsetAsync(cb.cnt, 0, (size_t)job.nq * n_sub * sizeof(int), ctx->stream));
            vs::IvfSelLaunch a;
            a.Q = job.q;
            a.nq = job.nq;
            a.d = v->d;
            a.payload = v->payload;
            a.list_off = v->list_off;
            a.nlist = v->nlist;
            a.pbits = job.pbits;
            a.pnorm = v->pnorms;
            a.nprobe = job.nprobe;
            a.pair_codes = gr.pair_codes;
            a.units = gr.units;
            a.n_units = gr.uoff + v->nlist;
            a.max_units = gr.max_units;
            a.margin = margin;
            a.ip = v->metric;
            a.k = job.k;
            a.cb = cb;
            a.visited = vis;
            CKS(arena_alloc(ctx, (size_t)v->nlist, &a.lsel));
            CKS(arena_alloc(ctx, (size_t)v->nlist + 1, &a.lsel64));
            CKS(arena_alloc(ctx, (size_t)v->nlist + 1, &a.sel_off));
            CKS(arena_alloc(ctx, (size_t)std::max<int64_t>(v->n_total, 1), &a.spos));
            char* recs = nullptr;
            CKS(arena_alloc(ctx, (size_t)gr.max_units * (mma ? 2 : 1) * vs::kIvfSelRecBytes, &recs));
            a.recs = recs;
            a.tmp_bytes = vs::ivf_sel_temp_bytes(v->nlist);
            char* tmp = nullptr;
            CKS(arena_alloc(ctx, a.tmp_bytes, &tmp));
            a.tmp = tmp;
            a.sm_count = ctx->sm_count;
            if (mma) {
                unsigned* bounds = nullptr;
                float* mmargin = nullptr;
                __half* qh = nullptr;
                float* kinv = nullptr;
                CKS(arena_alloc(ctx, 2, &bounds));
                CKS(arena_alloc(ctx, (size_t)job.nq, &mmargin));
                CKS(arena_alloc(ctx, (size_t)job.nq * ((v->d + 7) / 8 * 8), &qh));
                CKS(arena_alloc(ctx, (size_t)job.nq, &kinv));
                {
                    KTimer kt(ctx, VS_K_STAGE);
                    CK(vs::launch_f16_row_bounds(v->pmax, v->d, bounds, ctx->stream));
                    CKS(vs::tc_stage_queries_f16(ctx, job.q, job.nq, v->d, v->pmax, bounds, v->metric, qh, kinv,
                                                 mmargin));
                }
                a.mma = 1;
                a.Qh = qh;
                a.kinv = kinv;
                a.xscale = v->pmax;
                a.margin = mmargin;
                margin = mmargin;   // phase B re-ranks the tensor-core margin band
                ctx->stats[VS_STAT_LAUNCHES] += 1;
            }
            KTimer kt(ctx, VS_K_IVF_SCAN);
            if (v->dtype == VS_DTYPE_F32) CK(vs::launch_ivf_scan_sel<float>(a, ctx->stream));
            else CK(vs::launch_ivf_scan_sel<__nv_bfloat16>(a, ctx->stream));
            ctx->stats[VS_STAT_LAUNCHES] += 5;
        } else if (lmajor) {
            IvfGroups gr;
            CKS(ivf_group(ctx, job, vs::kIvfLmQT, &gr));
            int* work = nullptr;
            CKS(arena_alloc(ctx, 1, &work));
            CK(cudaMemsetAsync(work, 0, sizeof(int), ctx->stream));
            CK(cudaMemsetAsync(cb.cnt, 0, (size_t)job.nq * n_sub * sizeof(int), ctx->stream));
            vs::IvfLmParams lp;
            lp.Q = job.q;
            lp.nq = job.nq;
            lp.d = v->d;
            lp.dp = (v->d + 127) / 128 * 128;
            lp.payload = v->payload;
            lp.list_off = v->list_off;
            lp.nprobe = job.nprobe;
            lp.pbits = job.pbits;
            lp.pair_codes = gr.pair_codes;
            lp.units = gr.units;
            lp.n_units = gr.uoff + v->nlist;
            lp.max_units = gr.max_units;
            lp.work = work;
            lp.margin = margin;
            lp.ip = v->metric;
            lp.k = job.k;
            lp.cb = cb;
            lp.visited = vis;
            KTimer kt(ctx, VS_K_IVF_SCAN);
            if (v->dtype == VS_DTYPE_F32) CK(vs::launch_ivf_scan_lmajor<float>(lp, ctx->sm_count, ctx->stream));
            else CK(vs::launch_ivf_scan_lmajor<__nv_bfloat16>(lp, ctx->sm_count, ctx->stream));
        } else {
            vs::IvfScanParams sp;
            sp.Q = job.q;
            sp.nq = job.nq;
            sp.d = v->d;
            sp.payload = v->payload;
            sp.list_off = v->list_off;
            sp.probes = job.probes;
            sp.nprobe = job.nprobe;
            sp.list_owned = v->owned;
            sp.pbits = job.pbits;
            sp.margin = margin;
            sp.ip = v->metric;
            sp.k = job.k;
            sp.n_psplit = n_psplit;
            sp.cb = cb;
            sp.visited = vis;
            KTimer kt(ctx, VS_K_IVF_SCAN);
            if (v->dtype == VS_DTYPE_F32) CK(vs::launch_ivf_scan_qmajor<float>(sp, ctx->stream));
            else CK(vs::launch_ivf_scan_qmajor<__nv_bfloat16>(sp, ctx->stream));
        }
        ctx->stats[VS_STAT_LAUNCHES] += 1;
    }
    const int n_sub = cb.n_sub;
    const int64_t C = cb.C;

    vs::RerankParams rp;
    rp.Q = job.q;
    rp.nq = job.nq;
    rp.d = v->d;
    rp.ip = v->metric;
    rp.k = job.k;
    rp.cb = cb;
    rp.margin = margin;
    rp.tau_g = tau_g;
    rp.verify = verify;
    rp.rows = v->payload;
    rp.row_map = nullptr;
    rp.id_map = v->list_ids;
    rp.id_offset = 0;
    const int64_t all_slots = (int64_t)n_sub * C;
    rp.s_cap = (exhaustive || (int64_t)job.nq * all_slots * 20 < (int64_t(1) << 30))
                   ? all_slots
                   : std::min<int64_t>(all_slots, std::max<int64_t>(8 * C, 4096));
    CKS(arena_alloc(ctx, (size_t)job.nq * rp.s_cap, &rp.s_pos));
    CKS(arena_alloc(ctx, (size_t)job.nq * rp.s_cap, &rp.s_key));
    CKS(arena_alloc(ctx, (size_t)job.nq * rp.s_cap, &rp.s_id));
    CKS(arena_alloc(ctx, (size_t)job.nq, &rp.s_count));
    CKS(arena_alloc(ctx, (size_t)job.nq, &rp.fb_list));
    CKS(arena_alloc(ctx, 1, &rp.fb_count));
    rp.out_ids = job.out_ids;
    rp.out_dist = job.out_dist;
    rp.out_ids32 = nullptr;
    rp.out_count = job.out_count;
    unsigned long long* d_surv = nullptr;
    CKS(arena_alloc(ctx, 1, &d_surv));
    CK(cudaMemsetAsync(d_surv, 0, sizeof(unsigned long long), ctx->stream));
    rp.n_survivors = d_surv;
    {
        KTimer kt(ctx, VS_K_IVF_RERANK);
        if (v->dtype == VS_DTYPE_F32) CK(vs::launch_rerank<float>(rp, ctx->stream));
        else CK(vs::launch_rerank<__nv_bfloat16>(rp, ctx->stream));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 1;

    std::vector<int32_t> which;
    {
        std::vector<int> h(job.nq);
        unsigned long long h_surv = 0;
        CK(cudaMemcpyAsync(&h_surv, d_surv, sizeof(h_surv), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(h.data(), cb.overflow, job.nq * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (cshift == 0) ctx->stats[VS_STAT_SURVIVORS] = (int64_t)h_surv;
        for (int64_t i = 0; i < job.nq; ++i)
            if (h[i] || (allow_force && ctx->opt_force_retry)) which.push_back((int32_t)i);
    }
    if (which.empty()) return VS_OK;
    if (exhaustive && !(allow_force && ctx->opt_force_retry))
        return set_err(VS_ERR_INTERNAL, "IVF candidate overflow with exhaustive buffers");
    ctx->stats[VS_STAT_OVERFLOW_QUERIES] += (int64_t)which.size();
    const int64_t m = (int64_t)which.size();
    int32_t* d_idx = nullptr;
    float *d_q = nullptr, *d_m = nullptr;
    int32_t* d_pr = nullptr;
    CKS(arena_alloc(ctx, m, &d_idx));
    CKS(arena_alloc(ctx, (size_t)m * v->d, &d_q));
    CKS(arena_alloc(ctx, (size_t)m, &d_m));
    CKS(arena_alloc(ctx, (size_t)m * job.nprobe, &d_pr));
    CK(cudaMemcpyAsync(d_idx, which.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    int blocks = (int)std::min<int64_t>((m * v->d + 255) / 256, 4096);
    k_gather_queries<<<blocks, 256, 0, ctx->stream>>>(job.q, d_idx, m, v->d, d_q);
    k_gather_queries<<<1, 256, 0, ctx->stream>>>(margin, d_idx, m, 1, d_m);
    k_gather_queries<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<const float*>(job.probes), d_idx, m,
                                                      job.nprobe, reinterpret_cast<float*>(d_pr));
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 3;
    IvfJob sub = job;
    sub.q = d_q;
    sub.nq = m;
    sub.probes = d_pr;
    sub.visited = nullptr;
    CKS(arena_alloc(ctx, (size_t)m * job.k, &sub.out_ids));
    CKS(arena_alloc(ctx, (size_t)m * job.k, &sub.out_dist));
    CKS(arena_alloc(ctx, (size_t)m, &sub.out_count));
    CKS(run_ivf_scan(ctx, sub, d_m, exhaustive ? cshift : cshift + 2, false));
    CKS(scatter_rows(ctx, sub.out_ids, d_idx, m, job.k, job.out_ids));
    CKS(scatter_rows(ctx, sub.out_dist, d_idx, m, job.k, job.out_dist));
    CKS(scatter_rows(ctx, sub.out_count, d_idx, m, 1, job.out_count));
    return VS_OK;
}

// IVF coarse quantizer on dense keys: the tensor cores write every (query,
// centroid) key of a query chunk (tc_dense_keys, MODE 3), one CTA per query
// selects the margin band around its nprobe-th key (launch_dense_select) into
// a single candidate buffer, and phase B scores that band exactly (k_rerank:
// tie-rule top-nprobe, bit-identical probes). Replaces candidate buffers fed
// by the GEMM epilogue, which made the coarse GEMM epilogue-bound and left
// ~2,300 candidates per query for phase B to sort through.
int coarse_dense(vs_ctx* ctx, const EnnJob& cj, float* simt_margin, int n_qchunks, const unsigned* cmax) {
    const int64_t ncols = cj.nsel;
    int64_t qc = std::max<int64_t>(256, std::min<int64_t>(cj.nq, ((int64_t)1 << 28) / std::max<int64_t>(ncols, 1)));
    // queries still landing in n_qchunks chunks (copy stream): one coarse chunk each
    const int64_t up = n_qchunks ? (cj.nq + n_qchunks - 1) / n_qchunks : 0;
    if (n_qchunks) qc = std::min(qc, up);
    // per-chunk minima let the select read ~4 % of the keys (k_coarse_select)
    const bool chunked = vs::coarse_select_ok(ncols, cj.k) && !getenv("VS_COARSE_FULLSELECT");
    const int64_t nch = (ncols + 31) / 32;
    float* keys = nullptr;
    float* mins = nullptr;
    float* tm = nullptr;
    CKS(arena_alloc(ctx, (size_t)std::min(qc, cj.nq) * ncols, &keys));
    if (chunked) CKS(arena_alloc(ctx, (size_t)std::min(qc, cj.nq) * nch, &mins));
    CKS(arena_alloc(ctx, (size_t)cj.nq, &tm));
    const int C = (int)pow2ceil(std::max<int64_t>(4 * (int64_t)cj.k, cj.k + 256));
    // fp16 operands: the tensor-core band is already about as tight as the fp32
    // SIMT margin, so the fp32 refinement pass would not shrink it
    const bool f16 = vs::use_f16(VS_DTYPE_F32, cj.xmax);
    // one margin-band buffer per query for the whole batch; the key matrix is
    // produced and selected chunk by chunk, phase B runs once
    vs::CandBuf cb;
    cb.n_sub = 1;
    cb.C = C;
    CKS(arena_alloc(ctx, (size_t)cj.nq * C, &cb.key));
    CKS(arena_alloc(ctx, (size_t)cj.nq * C, &cb.pos));
    CKS(arena_alloc(ctx, (size_t)cj.nq, &cb.cnt));
    CKS(arena_alloc(ctx, (size_t)cj.nq, &cb.overflow));
    CK(cudaMemsetAsync(cb.overflow, 0, cj.nq * sizeof(int), ctx->stream));
    const bool refine = !f16 && cj.ip == 0 && simt_margin != nullptr;
    int waited = 0;
    for (int64_t q0 = 0; q0 < cj.nq; q0 += qc) {
        const int64_t n = std::min(qc, cj.nq - q0);
        for (; waited < n_qchunks && (int64_t)waited * up < q0 + n; ++waited)
            CK(cudaStreamWaitEvent(ctx->stream, ctx->q_chunk_ev[waited], 0));
        if (simt_margin)
            CK(vs::launch_query_margins(cj.q + q0 * cj.d, n, cj.d, cmax, eps_simt(cj.d), 0, simt_margin + q0, nullptr,
                                        ctx->stream));
        const float* qs = cj.q + q0 * cj.d;
        if (cj.narrow)
            CKS(vs::bn128::tc_dense_keys(ctx, qs, n, cj.d, (const float*)cj.rows, ncols, cj.xnorm, cj.xmax, cj.ip,
                                         keys, tm + q0, mins));
        else
            CKS(vs::tc_dense_keys(ctx, qs, n, cj.d, (const float*)cj.rows, ncols, cj.xnorm, cj.xmax, cj.ip, keys,
                                  tm + q0, mins));
        vs::CandBuf cbs = cb;   // this chunk's rows of the buffers
        cbs.key += q0 * (int64_t)C;
        cbs.pos += q0 * (int64_t)C;
        cbs.cnt += q0;
        cbs.overflow += q0;
        {
            KTimer kt(ctx, cj.cls_scan);   // candidate generation: part of the coarse phase A
            if (chunked) CK(vs::launch_coarse_select(keys, mins, n, ncols, cj.k, tm + q0, cbs, ctx->stream));
            else CK(vs::launch_dense_select(keys, n, ncols, cj.k, tm + q0, cbs, ctx->stream));
        }
        ctx->stats[VS_STAT_LAUNCHES] += 1;
        // the bf16 band (~2x nprobe centroids) -> fp32 keys with the SIMT margin:
        // phase B re-scores ~nprobe centroids in float64 instead of the band
        if (refine) {
            KTimer kt(ctx, cj.cls_rerank);
            CK(vs::launch_refine32(cbs, n, qs, cj.d, (const float*)cj.rows, ctx->stream));
            ctx->stats[VS_STAT_LAUNCHES] += 1;
        }
    }
    PhaseA st;
    st.sp.Q = cj.q;
    st.sp.nq = cj.nq;
    st.sp.d = cj.d;
    st.sp.X = cj.rows;
    st.sp.sel = nullptr;
    st.sp.nsel = ncols;
    st.sp.xnorm = cj.xnorm;
    st.sp.margin = refine ? simt_margin : tm;
    st.sp.ip = cj.ip;
    st.sp.k = cj.k;
    st.sp.cb = cb;
    st.sp.tau_g = nullptr;
    st.sp.verify = 0;
    st.sp.band_ready = refine ? 0 : 1;   // the select wrote exactly the band of the k-th key
    st.exhaustive = false;
    ctx->stats[VS_STAT_LAST_ENN_KERNEL] = 2;
    CKS(enn_phase_b(ctx, cj, st, 0, false, PhaseBHooks{}));
    return VS_OK;
}

}  // namespace

namespace vs {
// exact tie-rule nearest row (squared L2, float64 phase B) of each of m float32
// queries among nrows float32 rows: the k-means near-tie recheck (vs_kmeans.cu)
int exact_top1(vs_ctx* ctx, const float* q, int64_t m, int d, const float* rows, int64_t nrows, const float* rnorm,
               const unsigned* rmax, int32_t* out_ids, double* out_dist) {
    float* margin = nullptr;
    int32_t* cnt = nullptr;
    CKS(arena_alloc(ctx, (size_t)m, &margin));
    CKS(arena_alloc(ctx, (size_t)m, &cnt));
    CK(vs::launch_query_margins(q, m, d, rmax, eps_simt(d), 0, margin, nullptr, ctx->stream));
    EnnJob job;
    job.q = q;
    job.nq = m;
    job.d = d;
    job.rows = rows;
    job.dtype = VS_DTYPE_F32;
    job.sel = nullptr;
    job.nsel = nrows;
    job.xnorm = rnorm;
    job.xmax = rmax;
    job.ip = 0;
    job.k = 1;
    job.id_offset = 0;
    job.out_ids = nullptr;
    job.out_dist = out_dist;
    job.out_ids32 = out_ids;
    job.out_count = cnt;
    return run_enn(ctx, job, margin, 0, false);
}
}  // namespace vs

// IVF search; probes_in (nullable, [nq][nprobe]) skips the coarse quantizer
// (multi-GPU: each rank probes a slice of the queries, the probes are
// all-gathered); probe_only stops after the coarse quantizer.
static int ivf_search_impl(vs_ctx* ctx, const vs_ivf* ivf, const float* queries, int64_t nq,
                           const uint32_t* bitmap, int64_t nbits, int32_t nprobe, int32_t k,
                           int64_t* out_ids, double* out_dist, int32_t* out_count, int32_t* out_probes,
                           int64_t* out_visited, const int32_t* probes_in, bool probe_only) {
    if (!ctx || !ivf) return set_err(VS_ERR_PARAMETER, "null argument");
    CKS(validate_k(k));
    if (nprobe < 1) return set_err(VS_ERR_PARAMETER, "nprobe must be >= 1");
    if (nprobe > ivf->nlist) return set_err(VS_ERR_PARAMETER, "nprobe %d > nlist %d", nprobe, ivf->nlist);
    if (nq < 0) return set_err(VS_ERR_PARAMETER, "negative query count");
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    std::vector<OutBuf> pending;
    if (out_visited) *out_visited = 0;
    if (nq == 0) return VS_OK;
    const int d = ivf->d;
    const float* dq = nullptr;
    // a large host query batch is copied in four chunks on the copy stream; the
    // coarse quantizer (dense path) starts on chunk c as soon as it has landed
    int n_qchunks = 0;
    {
        cudaPointerAttributes at{};
        const bool host_q = queries && cudaPointerGetAttributes(&at, queries) == cudaSuccess &&
                            at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged;
        cudaGetLastError();
        // off unless VS_Q_CHUNKS > 0 (read per call): measured on config 3 (41 MB
        // of queries), four coarse chunks of 2,500 queries cost more than the
        // overlap saves (e2e 2.85 vs 2.61 ms, profiles/r2/e2e_transfers)
        const int qchunk_env = getenv("VS_Q_CHUNKS") ? atoi(getenv("VS_Q_CHUNKS")) : 0;
        if (qchunk_env > 0 && host_q && !probes_in && (size_t)nq * d * 4 >= ((size_t)1 << 23) && nq >= 4 * 256) {
            float* buf = nullptr;
            CKS(arena_alloc(ctx, (size_t)nq * d, &buf));
            if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
            if (!ctx->q_event) CK(cudaEventCreateWithFlags(&ctx->q_event, cudaEventDisableTiming));
            CK(cudaEventRecord(ctx->q_event, ctx->stream));            // earlier work on the arena
            CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->q_event, 0));
            n_qchunks = std::min(qchunk_env, 4);   // q_chunk_ev[4]
            const int64_t qc = (nq + n_qchunks - 1) / n_qchunks;
            for (int c = 0; c < n_qchunks; ++c) {
                if (!ctx->q_chunk_ev[c]) CK(cudaEventCreateWithFlags(&ctx->q_chunk_ev[c], cudaEventDisableTiming));
                const int64_t q0 = c * qc, n = std::max<int64_t>(0, std::min(qc, nq - q0));
                if (n) CK(cudaMemcpyAsync(buf + q0 * d, queries + q0 * d, (size_t)n * d * 4, cudaMemcpyHostToDevice,
                                          ctx->copy_stream));
                CK(cudaEventRecord(ctx->q_chunk_ev[c], ctx->copy_stream));
            }
            dq = buf;
        } else {
            CKS(stage_in(ctx, queries, (size_t)nq * d, &dq));
        }
    }
    // permuted bitmap over payload positions (needs no query: runs while they land)
    uint32_t* pbits = nullptr;
    if (bitmap) {
        const uint32_t* dbm = nullptr;
        CKS(stage_in(ctx, bitmap, (size_t)(nbits + 31) / 32, &dbm));
        CKS(arena_alloc(ctx, (size_t)(ivf->n_total + 31) / 32 + 2, &pbits));
        CK(cudaMemsetAsync(pbits, 0, ((ivf->n_total + 31) / 32 + 2) * sizeof(uint32_t), ctx->stream));
        KTimer kt(ctx, VS_K_SELECT);
        CK(vs::launch_permute_bitmap(dbm, nbits, ivf->list_ids, ivf->n_total, pbits, ctx->stream));
        ctx->stats[VS_STAT_LAUNCHES] += 1;
    }
    auto wait_all_queries = [&]() -> int {
        for (int c = 0; c < n_qchunks; ++c) CK(cudaStreamWaitEvent(ctx->stream, ctx->q_chunk_ev[c], 0));
        n_qchunks = 0;
        return VS_OK;
    };
    // coarse quantizer: exact tie-rule top-nprobe over float32 centroids, always
    // squared L2 (vecindex.py:238-243)
    float* cm = nullptr;
    CKS(arena_alloc(ctx, (size_t)nq, &cm));
    int32_t* probes = nullptr;
    if (probes_in) {
        const int32_t* dp = nullptr;
        CKS(stage_in(ctx, probes_in, (size_t)nq * nprobe, &dp));
        probes = const_cast<int32_t*>(dp);
    } else {
    CKS(stage_out(ctx, out_probes, (size_t)nq * nprobe, &probes, pending));
    if (!probes) CKS(arena_alloc(ctx, (size_t)nq * nprobe, &probes));
    EnnJob cj;
    cj.q = dq;
    cj.nq = nq;
    cj.d = d;
    cj.rows = ivf->centroids;
    cj.dtype = VS_DTYPE_F32;
    cj.sel = nullptr;
    cj.nsel = ivf->nlist;
    cj.xnorm = ivf->cnorms;
    cj.xmax = ivf->cmax;
    cj.ip = 0;
    cj.k = nprobe;
    cj.id_offset = 0;
    cj.out_ids = nullptr;
    cj.out_dist = nullptr;
    cj.out_ids32 = probes;
    cj.out_count = nullptr;
    cj.cls_scan = VS_K_COARSE;
    cj.cls_rerank = VS_K_COARSE_RERANK;
    cj.narrow = !getenv("VS_COARSE_WIDE");
    // VS_OPT_COARSE: 0 auto (dense keys when the tensor cores pay off), 1 candidate
    // buffers, 2 dense keys whenever the tensor cores apply
    const bool dense_ok = nprobe <= kTopkCap && ctx->opt_enn_kernel != 1 && vs::tc_supported(d, VS_DTYPE_F32, 0);
    if (dense_ok && (ctx->opt_coarse == 2 || (ctx->opt_coarse == 0 && vs::tc_profitable(nq, ivf->nlist, d)))) {
        CKS(coarse_dense(ctx, cj, cm, n_qchunks, ivf->cmax));
        n_qchunks = 0;
    } else {
        CKS(wait_all_queries());
        CK(vs::launch_query_margins(dq, nq, d, ivf->cmax, eps_simt(d), 0, cm, nullptr, ctx->stream));
        CKS(run_enn(ctx, cj, cm, 0, false));
    }
    }
    CKS(wait_all_queries());
    if (probe_only) {
        CKS(flush_out(ctx, pending));
        return VS_OK;
    }
    float* sm = nullptr;
    CKS(arena_alloc(ctx, (size_t)nq, &sm));
    CK(vs::launch_query_margins(dq, nq, d, ivf->pmax, eps_simt(d), ivf->metric, sm, nullptr, ctx->stream));
    ctx->stats[VS_STAT_LAUNCHES] += 2;
    unsigned long long* vis = nullptr;
    CKS(arena_alloc(ctx, 1, &vis));
    CK(cudaMemsetAsync(vis, 0, sizeof(unsigned long long), ctx->stream));
    IvfJob job;
    job.ivf = ivf;
    job.q = dq;
    job.nq = nq;
    job.probes = probes;
    job.nprobe = nprobe;
    job.pbits = pbits;
    job.k = k;
    job.visited = vis;
    CKS(stage_out_final(ctx, out_ids, (size_t)nq * k, &job.out_ids, pending, k <= kTopkCap));
    CKS(stage_out_final(ctx, out_dist, (size_t)nq * k, &job.out_dist, pending, k <= kTopkCap));
    CKS(stage_out_final(ctx, out_count, (size_t)nq, &job.out_count, pending, k <= kTopkCap));
    if (!job.out_ids) CKS(arena_alloc(ctx, (size_t)nq * k, &job.out_ids));
    if (!job.out_dist) CKS(arena_alloc(ctx, (size_t)nq * k, &job.out_dist));
    if (!job.out_count) CKS(arena_alloc(ctx, (size_t)nq, &job.out_count));
    if (k > kTopkCap) {
        // k' above the candidate buffers: every candidate of the probed lists
        // is keyed, selected and re-ranked device-wide (vs_wide.cu)
        if (ivf->n_total > (int64_t)UINT32_MAX) return set_err(VS_ERR_PARAMETER, "wide IVF search: > 2^32 rows");
        vs::WideJob w{};
        w.q = dq;
        w.nq = nq;
        w.d = d;
        w.rows = ivf->payload;
        w.dtype = ivf->dtype;
        w.margin = sm;
        w.ip = ivf->metric;
        w.k = k;
        w.id_map = ivf->list_ids;
        w.out_ids = job.out_ids;
        w.out_dist = job.out_dist;
        w.out_count = job.out_count;
        w.cls_scan = VS_K_IVF_SCAN;
        w.cls_rerank = VS_K_IVF_RERANK;
        CKS(vs::wide_ivf(ctx, w, probes, nprobe, ivf->list_off, ivf->h_off, ivf->owned, pbits, ivf->pnorms));
        int32_t* scratch = nullptr;
        CKS(arena_alloc(ctx, (size_t)ivf->nlist, &scratch));
        CK(vs::launch_visited_count(probes, nq, nprobe, ivf->list_off, ivf->nlist, ivf->owned, pbits, scratch, vis,
                                    ctx->stream));
    } else {
        CKS(run_ivf_scan(ctx, job, sm, 0, true));
    }
    unsigned long long h_vis = 0;
    CK(cudaMemcpyAsync(&h_vis, vis, sizeof(h_vis), cudaMemcpyDeviceToHost, ctx->stream));
    CKS(flush_out(ctx, pending));
    if (out_visited) *out_visited = (int64_t)h_vis;
    return VS_OK;
}

extern "C" int vs_ivf_assign(vs_ctx* ctx, const vs_ivf* ivf, const vs_column* data, int32_t* out_lists) {
    if (!ctx || !ivf || !data || !out_lists) return set_err(VS_ERR_PARAMETER, "null argument");
    if (data->d != ivf->d) return set_err(VS_ERR_SHAPE, "column dim %d != index dim %d", data->d, ivf->d);
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    if (data->n == 0) return VS_OK;
    CKS(ensure_norms(const_cast<vs_column*>(data), ctx));
    return vs::ivf_assign_gpu(ctx, ivf, data, out_lists);
}

extern "C" int vs_ivf_build(vs_ctx* ctx, const vs_column* data, int32_t nlist, const int64_t* init_rows,
                            uint64_t seed, int32_t metric, int32_t max_iters, vs_ivf** out) {
    if (!ctx || !data || !out) return set_err(VS_ERR_PARAMETER, "null argument");
    CKS(validate_metric(metric));
    if (nlist < 1 || nlist > data->n)
        return set_err(VS_ERR_PARAMETER, "nlist must be in [1, %lld], got %d", (long long)data->n, nlist);
    DevGuard g(ctx->device);
    CK(ctx->arena.reset());
    CKS(ensure_norms(const_cast<vs_column*>(data), ctx));
    return vs::ivf_build_gpu(ctx, data, nlist, init_rows, seed, metric, max_iters, out);
}

extern "C" int vs_ivf_search(vs_ctx* ctx, const vs_ivf* ivf, const float* queries, int64_t nq,
                             const uint32_t* bitmap, int64_t nbits, int32_t nprobe, int32_t k,
                             int64_t* out_ids, double* out_dist, int32_t* out_count, int32_t* out_probes,
                             int64_t* out_visited) {
    return ivf_search_impl(ctx, ivf, queries, nq, bitmap, nbits, nprobe, k, out_ids, out_dist, out_count,
                           out_probes, out_visited, nullptr, false);
}

extern "C" int vs_ivf_probe(vs_ctx* ctx, const vs_ivf* ivf, const float* queries, int64_t nq, int32_t nprobe,
                            int32_t* out_probes) {
    if (!out_probes) return set_err(VS_ERR_PARAMETER, "null out_probes");
    return ivf_search_impl(ctx, ivf, queries, nq, nullptr, 0, nprobe, 1, nullptr, nullptr, nullptr, out_probes,
                           nullptr, nullptr, true);
}

extern "C" int vs_ivf_search_probed(vs_ctx* ctx, const vs_ivf* ivf, const float* queries, int64_t nq,
                                    const uint32_t* bitmap, int64_t nbits, int32_t nprobe,
                                    const int32_t* probes, int32_t k, int64_t* out_ids, double* out_dist,
                                    int32_t* out_count, int64_t* out_visited) {
    if (!probes && nq > 0) return set_err(VS_ERR_PARAMETER, "null probes");
    return ivf_search_impl(ctx, ivf, queries, nq, bitmap, nbits, nprobe, k, out_ids, out_dist, out_count,
                           nullptr, out_visited, probes, false);
}
