// Internal (non-ABI) structures shared by the C-ABI driver and the kernel
// drivers: context, column and IVF objects, error plumbing, scratch arena.
#pragma once

#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vs_b200.h"

namespace vs_internal {

inline thread_local std::string g_err;

inline int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

inline int cuda_err(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation)
        return set_err(VS_ERR_PLACEMENT, "%s: device memory exhausted (%s)", what, cudaGetErrorString(e));
    return set_err(VS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define VS_STR2(x) #x
#define VS_STR(x) VS_STR2(x)
#define CK(call)                                                   \
    do {                                                           \
        cudaError_t _e = (call);                                   \
        if (_e != cudaSuccess) { cudaGetLastError(); return cuda_err(_e, #call " @" VS_STR(__LINE__) " " __FILE__); } \
    } while (0)
#define CKS(call)                                     \
    do {                                              \
        int _s = (call);                              \
        if (_s != VS_OK) return _s;                   \
    } while (0)

constexpr int kTopkCap = 2048;  // placement.py:56 gpu_topk_cap default

inline int64_t pow2ceil(int64_t v) {
    int64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}
inline size_t elem_size(int dtype) { return dtype == VS_DTYPE_BF16 ? 2 : 4; }

inline bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Per-call device scratch: a bump allocator over one buffer that grows to the
// high-water mark of previous calls (calls are synchronous, so reset() runs
// with no kernel in flight).
struct Arena {
    char* base = nullptr;
    size_t cap = 0, used = 0, need = 0;
    std::vector<void*> extra;
    cudaError_t reset() {
        for (void* p : extra) cudaFree(p);
        extra.clear();
        if (need > cap) {
            if (base) cudaFree(base);
            base = nullptr;
            cap = 0;
            need += need / 4;  // headroom: grow rarely
            cudaError_t e = cudaMalloc(&base, need);
            if (e != cudaSuccess) {
                cudaGetLastError();
                base = nullptr;
                need = 0;
            } else {
                cap = need;
            }
        }
        used = 0;
        need = 0;
        return cudaSuccess;
    }
    // scratch of a nested, synchronous step (stream idle): rewinding frees
    // everything allocated after the mark, extras included
    struct Mark {
        size_t used, extras;
    };
    Mark mark() const { return Mark{used, extra.size()}; }
    void rewind(const Mark& m) {
        while (extra.size() > m.extras) {
            cudaFree(extra.back());
            extra.pop_back();
        }
        used = m.used;
    }
    cudaError_t alloc(size_t n, void** out) {
        n = (n + 255) & ~size_t(255);
        need += n;
        if (used + n <= cap) {
            *out = base + used;
            used += n;
            return cudaSuccess;
        }
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, n);
        if (e != cudaSuccess) return e;
        extra.push_back(p);
        *out = p;
        return cudaSuccess;
    }
    void release() {
        reset();
        if (base) cudaFree(base);
        base = nullptr;
        cap = 0;
    }
};

}  // namespace vs_internal

struct vs_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    int sm_count = 148;
    vs_internal::Arena arena;
    int64_t stats[VS_STAT_N] = {0};
    int opt_enn_kernel = 0;
    int opt_ivf_kernel = 0;
    int opt_slack = 0;
    int opt_force_retry = 0;
    int opt_timing = 0;
    int opt_coarse = 0;              // IVF coarse quantizer: 0 auto, 1 candidate buffers, 2 dense keys
    int64_t opt_stream_chunk = 0;    // host-resident search: selected rows per chunk (0 = auto)
    int64_t opt_ivf_chunk_rows = 0;  // tensor-core IVF scan: rows per list chunk (0 = 131072)
    int sm_reserve = 0;              // SMs left free by persistent kernels (streamed gathers)
    cudaStream_t copy_stream = nullptr;   // host-resident search: gathers over PCIe; query uploads
    cudaEvent_t q_event = nullptr;        // queries landed (copy stream)
    cudaEvent_t q_chunk_ev[4] = {};       // IVF: query chunks landed (chunked upload, coarse overlaps it)
    // CUDA-event timing of kernel classes (resolved after each call's final sync)
    struct PendingTimer {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<PendingTimer> timers;
    std::vector<cudaEvent_t> event_pool;
    int64_t kt_ns[VS_K_N] = {0};
    int64_t kt_count[VS_K_N] = {0};
    // columns and indexes created through this context use its device and
    // stream until they are freed: vs_ctx_destroy with objects alive only
    // releases the scratch and leaves the struct to the last object's free
    std::mutex life_mu;
    int live_objects = 0;
    bool destroyed = false;
};

struct vs_column {
    vs_ctx* ctx = nullptr;
    void* data = nullptr;
    int64_t n = 0;
    int d = 0;
    int dtype = VS_DTYPE_F32;
    bool owned = false;
    bool host_resident = false;      // data lives in pinned host memory (streamed per search)
    bool host_registered = false;    // we cudaHostRegister'ed it (unregister on free)
    void* host_ptr = nullptr;
    float* norms = nullptr;          // ||x||^2 per row (lazy)
    unsigned* max_norm_bits = nullptr;
    bool norms_ready = false;
    // fp16 shadow for the tensor-core phase A (float32 device columns searched
    // more than once): [n][dp] scaled fp16 rows + per-row (||x~||^2, ||dx||^2),
    // built on the second search, dropped with the norms on invalidation
    void* f16 = nullptr;
    float2* f16_stats = nullptr;
    bool f16_ready = false;
    bool f16_failed = false;         // allocation failed once: never retried
    int searches = 0;
};

struct vs_ivf {
    vs_ctx* ctx = nullptr;
    int nlist = 0, d = 0, metric = 0, dtype = VS_DTYPE_F32;
    int64_t n_total = 0;
    float* centroids = nullptr;
    float* cnorms = nullptr;
    unsigned* cmax = nullptr;
    int64_t* list_off = nullptr;     // device [nlist+1]
    std::vector<int64_t> h_off;
    int64_t* list_ids = nullptr;     // device [n_total]
    void* payload = nullptr;         // device [n_total][d]
    float* pnorms = nullptr;
    unsigned* pmax = nullptr;
    uint8_t* owned = nullptr;        // device [nlist] or null
    bool payload_borrowed = false;   // vs_ivf_wrap: caller-owned device payload
};


namespace vs_internal {

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

template <typename T>
int arena_alloc(vs_ctx* ctx, size_t count, T** out) {
    void* p = nullptr;
    cudaError_t e = ctx->arena.alloc(count * sizeof(T) + 16, &p);
    if (e != cudaSuccess) return cuda_err(e, "scratch allocation");
    *out = reinterpret_cast<T*>(p);
    return VS_OK;
}

}  // namespace vs_internal

namespace vs_internal {

// RAII scope that brackets the launches of one kernel class with CUDA events
// on the context stream (only while VS_OPT_TIMING is on).
struct KTimer {
    vs_ctx* ctx;
    int cls;
    cudaEvent_t a = nullptr, b = nullptr;
    KTimer(vs_ctx* c, int k) : ctx(c), cls(k) {
        if (!ctx->opt_timing) return;
        a = take();
        b = take();
        cudaEventRecord(a, ctx->stream);
    }
    ~KTimer() {
        if (!a) return;
        cudaEventRecord(b, ctx->stream);
        ctx->timers.push_back({cls, a, b});
    }
    cudaEvent_t take() {
        cudaEvent_t e;
        if (!ctx->event_pool.empty()) {
            e = ctx->event_pool.back();
            ctx->event_pool.pop_back();
        } else {
            cudaEventCreate(&e);
        }
        return e;
    }
};

// after the stream is synchronised: fold recorded intervals into the totals
inline void resolve_timers(vs_ctx* ctx) {
    for (auto& t : ctx->timers) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
            ctx->kt_ns[t.cls] += (int64_t)(ms * 1e6);
            ctx->kt_count[t.cls] += 1;
        } else {
            cudaGetLastError();
        }
        ctx->event_pool.push_back(t.a);
        ctx->event_pool.push_back(t.b);
    }
    ctx->timers.clear();
}

}  // namespace vs_internal

// lifetime of a context's dependent objects (vs_capi.cu)
void ctx_ref(vs_ctx* ctx);
void ctx_unref(vs_ctx* ctx);

int ivf_make(vs_ctx* ctx, const float* centroids, int32_t nlist, int32_t d, const std::vector<int64_t>& sizes,
             const int64_t* list_ids, const void* list_payload, int32_t dtype, int32_t metric,
             const vs_column* base, const uint8_t* list_owned, vs_ivf** out, bool borrow_payload = false);
