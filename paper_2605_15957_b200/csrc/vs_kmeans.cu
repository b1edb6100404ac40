// GPU IVF build: Lloyd's k-means with the reference's semantics
// (vecindex.py:186-207, _kmeans 273-318).
//
//   init      nlist ascending rows (np.sort(default_rng(seed).choice(...)),
//             drawn by the Python shim so the start matches the reference)
//   iterate   <= max_iters: assign every row to its first-min nearest centroid
//             (tcgen05 GEMM with an argmin epilogue, vs_tc.cu), reseed empty
//             lists to the farthest member of the largest list, float64 means,
//             stop when the largest centroid move < 1e-4
//   final     reassign against the converged centroids, reseed, final means;
//             centroids stored as float32, lists = ascending row ids (stable
//             radix sort of (list, row)), payload gathered list-major (owning)
//
// The assignment compares bf16 tensor-core keys ||c||^2 - 2 x.c with a
// rigorous error bound; every row whose best and second-best keys lie within
// it is re-assigned by the exact tie-rule search (float64 phase B over the
// float32 centroids, near_tie_recheck), so the assignment is the first-min
// argmin of exact distances (the reference's float64 BLAS expansion can only
// differ on ties at its own rounding level; tests/test_gpu_ivf_build.py: the
// small reference build is reproduced row for row).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "vs_common.cuh"
#include "vs_kernels.cuh"
#include "vs_tc.cuh"

namespace vs {

namespace {

template <typename T>
__global__ void k_gather_f64(const T* __restrict__ x, const int64_t* __restrict__ rows, int n, int d,
                             double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)n * d;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / d, c = i - r * d;
        out[i] = (double)ld_elem(x + rows[r] * (int64_t)d + c);
    }
}

__global__ void k_f64_to_f32(const double* __restrict__ a, int64_t n, float* __restrict__ b) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}

// packed (orderable key << 32 | list) -> assignment + squared distance to it
__global__ void k_unpack(const unsigned long long* __restrict__ packed, const float* __restrict__ xnorm, int64_t n,
                         int* __restrict__ assign, float* __restrict__ dist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long v = packed[i];
        assign[i] = (int)(v & 0xffffffffu);
        dist[i] = fmaxf(o2f((uint32_t)(v >> 32)) + xnorm[i], 0.f);
    }
}

// near ties of the tensor-core assignment: a row whose best and second-best
// keys (over both column halves) lie within the keys' error bound (the
// k_tc_margins formula with the row as the query and the centroids as rows)
// may be assigned differently by exact arithmetic: listed for the recheck
__global__ void k_near_ties(const unsigned long long* __restrict__ top2, const float2* __restrict__ rowstats,
                            const unsigned* __restrict__ cst, const unsigned* __restrict__ cmax, int64_t n, int d,
                            int* __restrict__ list, int* __restrict__ count) {
    const float Ct = sqrtf(__uint_as_float(cst[0])) * 1.0001f;   // max ||c~||
    const float Dc = sqrtf(__uint_as_float(cst[1])) * 1.0001f;   // max ||dc||
    const float C2 = __uint_as_float(*cmax) * 1.0002f;           // max ||c||^2
    const float acc_u = fmaxf(6.103515625e-05f, (float)((d + 15) / 16 + 4) * 9.5367431640625e-07f);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long b0 = top2[i * 4], s0 = top2[i * 4 + 1];
        const unsigned long long b1 = top2[i * 4 + 2], s1 = top2[i * 4 + 3];
        const bool h1 = b1 < b0;
        const uint32_t best = (uint32_t)((h1 ? b1 : b0) >> 32);
        const uint32_t other = (uint32_t)((h1 ? b0 : b1) >> 32);
        const uint32_t second = min((uint32_t)(h1 ? s1 : s0), other);
        const float2 rs = rowstats[i];
        const float qx = sqrtf(rs.x) * 1.0001f, dx = sqrtf(rs.y) * 1.0001f;
        const float edot = qx * Dc + dx * Ct + dx * Dc + acc_u * qx * Ct;
        const float e = 2.f * edot + (float)(d + 2) * 5.9604645e-08f * C2 + 1.1920929e-07f * (C2 + 2.f * qx * Ct);
        const float m = 2.f * e * 1.01f;
        if (second == 0xffffffffu || !(o2f(second) - o2f(best) > m)) list[atomicAdd(count, 1)] = (int)i;
    }
}

template <typename T>
__global__ void k_gather_rows_f32(const T* __restrict__ x, const int* __restrict__ rows, int m, int d,
                                  float* __restrict__ out) {
    // a warp per row, coalesced, no index division
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const T* src = x + (int64_t)rows[r] * d;
        float* dst = out + r * d;
        for (int c = lane; c < d; c += 32) dst[c] = ld_elem(src + c);
    }
}

__global__ void k_scatter_assign(const int* __restrict__ rows, const int32_t* __restrict__ ids,
                                 const double* __restrict__ dd, int m, int* __restrict__ assign,
                                 float* __restrict__ dist) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        assign[rows[i]] = ids[i];
        dist[rows[i]] = (float)dd[i];
    }
}

__global__ void k_hist(const int* __restrict__ assign, int64_t n, int* __restrict__ counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&counts[assign[i]], 1);
}

// farthest member of list `target` (first max, i.e. lowest row on ties)
__global__ void k_farthest(const int* __restrict__ assign, const float* __restrict__ dist, int64_t n, int target,
                           unsigned long long* __restrict__ best) {
    unsigned long long b = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (assign[i] == target) {
            const unsigned long long v = ((unsigned long long)f2o(dist[i]) << 32) | (0xffffffffu - (uint32_t)i);
            b = v > b ? v : b;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long u = __shfl_xor_sync(VS_FULL, b, o);
        b = u > b ? u : b;
    }
    if ((threadIdx.x & 31) == 0 && b) atomicMax(best, b);
}

__global__ void k_reseed(const float* __restrict__ xf, const __nv_bfloat16* __restrict__ xb, int d, int64_t far,
                         int empty, double* __restrict__ c64, int* __restrict__ assign, float* __restrict__ dist) {
    for (int i = threadIdx.x; i < d; i += blockDim.x)
        c64[(int64_t)empty * d + i] = xf ? (double)xf[far * (int64_t)d + i] : (double)__bfloat162float(xb[far * (int64_t)d + i]);
    if (threadIdx.x == 0) {
        assign[far] = empty;
        dist[far] = 0.f;
    }
}

// float64 mean of each list's members (block per list, rows in list order)
template <typename T>
__global__ void k_means(const T* __restrict__ x, const int* __restrict__ sorted_rows, const int64_t* __restrict__ off,
                        int d, double* __restrict__ out, const double* __restrict__ old,
                        unsigned long long* __restrict__ shift_max) {
    const int l = blockIdx.x;
    const int64_t b = off[l], e = off[l + 1];
    double sq = 0.0;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        double s = 0.0;
        for (int64_t i = b; i < e; ++i) s += (double)ld_elem(x + (int64_t)sorted_rows[i] * d + c);
        const double m = (e > b) ? s / (double)(e - b) : old[(int64_t)l * d + c];
        out[(int64_t)l * d + c] = m;
        if (old) {
            const double df = m - old[(int64_t)l * d + c];
            sq += df * df;
        }
    }
    if (shift_max) {
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(VS_FULL, sq, o);
        __shared__ double red[32];
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) t += red[i];
            atomicMax(shift_max, d2o(sqrt(t)));
        }
    }
}

__global__ void k_iota(int* __restrict__ a, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int)i;
}
__global__ void k_i32_to_i64(const int* __restrict__ a, int64_t n, int64_t* __restrict__ b) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

double o2d_host(uint64_t o) {
    const uint64_t u = (o & 0x8000000000000000ull) ? (o & 0x7fffffffffffffffull) : ~o;
    double r;
    memcpy(&r, &u, sizeof(r));
    return r;
}

unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

// Rows whose tensor-core assignment is within the keys' error bound of a
// different centroid get the exact tie-rule nearest centroid (squared L2,
// float64 phase B over the float32 centroids, first minimum on ties), so the
// assignment equals the reference's first-min argmin up to the rounding of
// its own float64 expansion. Chunks of 2^18 rows; arena space is reused.
int near_tie_recheck(vs_ctx* ctx, const vs_column* data, int64_t n, int d, const unsigned long long* top2,
                     const float2* rowstats, const unsigned* cst, const unsigned* cmax, const float* c32, int nlist,
                     const float* cnorm, int* assign, float* dist, int64_t* n_rechecked) {
    using namespace vs_internal;
    cudaStream_t st = ctx->stream;
    int* list = nullptr;
    int* cnt = nullptr;
    CKS(arena_alloc(ctx, (size_t)std::max<int64_t>(n, 1), &list));
    CKS(arena_alloc(ctx, 1, &cnt));
    CK(cudaMemsetAsync(cnt, 0, sizeof(int), st));
    k_near_ties<<<grid_for(n), 256, 0, st>>>(top2, rowstats, cst, cmax, n, d, list, cnt);
    CK(cudaGetLastError());
    int m = 0;
    CK(cudaMemcpyAsync(&m, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (n_rechecked) *n_rechecked += m;
    ctx->stats[VS_STAT_NEAR_TIES] += m;
    const int64_t chunk = (int64_t)1 << 18;
    for (int64_t r0 = 0; r0 < m; r0 += chunk) {
        const int mc = (int)std::min<int64_t>(chunk, m - r0);
        const auto mark = ctx->arena.mark();
        float* qbuf = nullptr;
        int32_t* ids = nullptr;
        double* dd = nullptr;
        CKS(arena_alloc(ctx, (size_t)mc * d, &qbuf));
        CKS(arena_alloc(ctx, (size_t)mc, &ids));
        CKS(arena_alloc(ctx, (size_t)mc, &dd));
        if (data->dtype == VS_DTYPE_F32)
            k_gather_rows_f32<float><<<grid_for((int64_t)mc * 32), 256, 0, st>>>((const float*)data->data, list + r0,
                                                                                  mc, d, qbuf);
        else
            k_gather_rows_f32<__nv_bfloat16><<<grid_for((int64_t)mc * 32), 256, 0, st>>>(
                (const __nv_bfloat16*)data->data, list + r0, mc, d, qbuf);
        CK(cudaGetLastError());
        CKS(exact_top1(ctx, qbuf, mc, d, c32, nlist, cnorm, cmax, ids, dd));
        k_scatter_assign<<<grid_for(mc), 256, 0, st>>>(list + r0, ids, dd, mc, assign, dist);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
        ctx->arena.rewind(mark);   // the chunk's scratch (and run_enn's) is free again
        ctx->stats[VS_STAT_LAUNCHES] += 2;
    }
    return VS_OK;
}

int ivf_build_gpu(vs_ctx* ctx, const vs_column* data, int32_t nlist, const int64_t* init_rows, uint64_t seed,
                  int32_t metric, int32_t max_iters, vs_ivf** out) {
    using namespace vs_internal;
    cudaStream_t st = ctx->stream;
    const int64_t n = data->n;
    const int d = data->d;
    const int dp = (d + 7) / 8 * 8;
    if (n >= (int64_t(1) << 31)) return set_err(VS_ERR_PARAMETER, "k-means build supports < 2^31 rows");
    // initial rows (ascending)
    std::vector<int64_t> init(nlist);
    if (init_rows) {
        CK(cudaMemcpy(init.data(), init_rows, nlist * sizeof(int64_t), cudaMemcpyDefault));
    } else {
        // seeded partial Fisher-Yates over a splitmix64 stream (library fallback;
        // the Python API passes the reference's numpy draw instead)
        std::vector<int64_t> pool;
        uint64_t z = seed + 0x9E3779B97F4A7C15ull;
        auto next = [&]() {
            z += 0x9E3779B97F4A7C15ull;
            uint64_t r = z;
            r = (r ^ (r >> 30)) * 0xBF58476D1CE4E5B9ull;
            r = (r ^ (r >> 27)) * 0x94D049BB133111EBull;
            return r ^ (r >> 31);
        };
        std::vector<char> used;
        if (n <= 50'000'000) used.assign(n, 0);
        for (int i = 0; i < nlist; ++i) {
            int64_t r;
            do { r = (int64_t)(next() % (uint64_t)n); } while (!used.empty() && used[r]);
            if (!used.empty()) used[r] = 1;
            init[i] = r;
        }
        std::sort(init.begin(), init.end());
    }
    for (int i = 0; i < nlist; ++i)
        if (init[i] < 0 || init[i] >= n) return set_err(VS_ERR_PARAMETER, "initial row out of range");

    double *c64 = nullptr, *c64n = nullptr;
    float *c32 = nullptr, *cnorm = nullptr, *dist = nullptr;
    __nv_bfloat16* cb = nullptr;
    unsigned* cmax = nullptr;
    unsigned long long *packed = nullptr, *farbest = nullptr, *shift = nullptr;
    int *assign = nullptr, *counts = nullptr, *rows_in = nullptr, *rows_out = nullptr, *keys_out = nullptr;
    int64_t *off = nullptr, *d_init = nullptr;
    CKS(arena_alloc(ctx, (size_t)nlist * d, &c64));
    CKS(arena_alloc(ctx, (size_t)nlist * d, &c64n));
    CKS(arena_alloc(ctx, (size_t)nlist * d, &c32));
    CKS(arena_alloc(ctx, (size_t)nlist, &cnorm));
    CKS(arena_alloc(ctx, (size_t)nlist * dp, &cb));
    CKS(arena_alloc(ctx, 1, &cmax));
    CKS(arena_alloc(ctx, (size_t)n, &packed));
    CKS(arena_alloc(ctx, (size_t)n, &dist));
    CKS(arena_alloc(ctx, (size_t)n, &assign));
    CKS(arena_alloc(ctx, (size_t)nlist, &counts));
    CKS(arena_alloc(ctx, (size_t)n, &rows_in));
    CKS(arena_alloc(ctx, (size_t)n, &rows_out));
    CKS(arena_alloc(ctx, (size_t)n, &keys_out));
    CKS(arena_alloc(ctx, (size_t)nlist + 1, &off));
    CKS(arena_alloc(ctx, (size_t)nlist, &d_init));
    CKS(arena_alloc(ctx, 1, &farbest));
    CKS(arena_alloc(ctx, 1, &shift));
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, assign, keys_out, rows_in, rows_out, (int)n, 0,
                                    std::max(1, (int)std::ceil(std::log2((double)nlist + 1))), st);
    void* sort_tmp = nullptr;
    CK(ctx->arena.alloc(sort_bytes + 256, &sort_tmp));
    // row staging for the tensor-core assignment, allocated once for all iterations
    __nv_bfloat16* xb_scratch = nullptr;
    unsigned* junk = nullptr;
    unsigned* cst = nullptr;
    unsigned long long* top2 = nullptr;
    float2* rowstats = nullptr;
    CKS(arena_alloc(ctx, (size_t)tc_argmin_chunk(n) * dp, &xb_scratch));
    CKS(arena_alloc(ctx, 2, &junk));
    CKS(arena_alloc(ctx, 2, &cst));
    CKS(arena_alloc(ctx, (size_t)n * 4, &top2));
    CKS(arena_alloc(ctx, (size_t)n, &rowstats));
    int64_t n_rechecked = 0;

    const float* xf = data->dtype == VS_DTYPE_F32 ? (const float*)data->data : nullptr;
    const __nv_bfloat16* xbf = data->dtype == VS_DTYPE_BF16 ? (const __nv_bfloat16*)data->data : nullptr;
    CK(cudaMemcpyAsync(d_init, init.data(), nlist * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    if (xf) k_gather_f64<float><<<grid_for((int64_t)nlist * d), 256, 0, st>>>(xf, d_init, nlist, d, c64);
    else k_gather_f64<__nv_bfloat16><<<grid_for((int64_t)nlist * d), 256, 0, st>>>(xbf, d_init, nlist, d, c64);
    CK(cudaGetLastError());
    const int sort_bits = std::max(1, (int)std::ceil(std::log2((double)nlist + 1)));
    std::vector<int> h_counts(nlist);
    std::vector<int64_t> h_off(nlist + 1);

    auto assign_pass = [&]() -> int {
        k_f64_to_f32<<<grid_for((int64_t)nlist * d), 256, 0, st>>>(c64, (int64_t)nlist * d, c32);
        CK(cudaGetLastError());
        CK(cudaMemsetAsync(cmax, 0, sizeof(unsigned), st));
        CK(launch_row_norms<float>(c32, nlist, d, cnorm, cmax, st));
        CK(cudaMemsetAsync(cst, 0, 2 * sizeof(unsigned), st));
        // fp16 operands (~6x narrower error bound than bf16: fewer near-tie rechecks)
        CKS(tc_stage_f16(ctx, c32, nlist, d, cmax, cb, cst));
        CKS(tc_argmin_rows(ctx, data->data, data->dtype, n, d, cb, cnorm, nlist, packed, xb_scratch, junk, top2,
                           rowstats, data->max_norm_bits, cmax));
        k_unpack<<<grid_for(n), 256, 0, st>>>(packed, data->norms, n, assign, dist);
        CK(cudaGetLastError());
        ctx->stats[VS_STAT_LAUNCHES] += 4;
        return near_tie_recheck(ctx, data, n, d, top2, rowstats, cst, cmax, c32, nlist, cnorm, assign, dist,
                                &n_rechecked);
    };
    // counts + reseed of empty lists (vecindex.py:286-294), host-driven: empty
    // lists are rare and the reference's loop is inherently sequential
    auto counts_reseed = [&]() -> int {
        CK(cudaMemsetAsync(counts, 0, nlist * sizeof(int), st));
        k_hist<<<grid_for(n), 256, 0, st>>>(assign, n, counts);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h_counts.data(), counts, nlist * sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (;;) {
            int empty = -1;
            for (int i = 0; i < nlist; ++i)
                if (h_counts[i] == 0) { empty = i; break; }
            if (empty < 0) break;
            int biggest = 0;
            for (int i = 1; i < nlist; ++i)
                if (h_counts[i] > h_counts[biggest]) biggest = i;
            CK(cudaMemsetAsync(farbest, 0, sizeof(unsigned long long), st));
            k_farthest<<<grid_for(n), 256, 0, st>>>(assign, dist, n, biggest, farbest);
            unsigned long long fb = 0;
            CK(cudaMemcpyAsync(&fb, farbest, sizeof(fb), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const int64_t far = (int64_t)(0xffffffffu - (uint32_t)(fb & 0xffffffffu));
            k_reseed<<<1, 256, 0, st>>>(xf, xbf, d, far, empty, c64, assign, dist);
            CK(cudaGetLastError());
            h_counts[empty] += 1;
            h_counts[biggest] -= 1;
            ctx->stats[VS_STAT_LAUNCHES] += 2;
        }
        h_off[0] = 0;
        for (int i = 0; i < nlist; ++i) h_off[i + 1] = h_off[i] + h_counts[i];
        CK(cudaMemcpyAsync(off, h_off.data(), (nlist + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        // stable grouping: (list, row) with rows ascending inside each list
        k_iota<<<grid_for(n), 256, 0, st>>>(rows_in, n);
        CK(cudaGetLastError());
        CK(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, assign, keys_out, rows_in, rows_out, (int)n, 0,
                                           sort_bits, st));
        ctx->stats[VS_STAT_LAUNCHES] += 3;
        return VS_OK;
    };
    auto means = [&](bool with_shift) -> int {
        CK(cudaMemsetAsync(shift, 0, sizeof(unsigned long long), st));
        if (xf) k_means<float><<<nlist, 128, 0, st>>>(xf, rows_out, off, d, c64n, c64, with_shift ? shift : nullptr);
        else k_means<__nv_bfloat16><<<nlist, 128, 0, st>>>(xbf, rows_out, off, d, c64n, c64, with_shift ? shift : nullptr);
        CK(cudaGetLastError());
        std::swap(c64, c64n);
        ctx->stats[VS_STAT_LAUNCHES] += 1;
        return VS_OK;
    };

    for (int it = 0; it < max_iters; ++it) {
        CKS(assign_pass());
        CKS(counts_reseed());
        CKS(means(true));
        unsigned long long hs = 0;
        CK(cudaMemcpyAsync(&hs, shift, sizeof(hs), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (o2d_host(hs) < 1e-4) break;
    }
    CKS(assign_pass());
    CKS(counts_reseed());
    CKS(means(false));
    // final structure: float32 centroids, ascending row ids per list
    k_f64_to_f32<<<grid_for((int64_t)nlist * d), 256, 0, st>>>(c64, (int64_t)nlist * d, c32);
    int64_t* ids64 = nullptr;
    CKS(arena_alloc(ctx, (size_t)n, &ids64));
    k_i32_to_i64<<<grid_for(n), 256, 0, st>>>(rows_out, n, ids64);
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 2;
    std::vector<int64_t> sizes(nlist);
    for (int i = 0; i < nlist; ++i) sizes[i] = h_counts[i];
    return ivf_make(ctx, c32, nlist, d, sizes, ids64, nullptr, data->dtype, metric, data, nullptr, out);
}

// Nearest list (squared L2 to the float32 centroids, first minimum on the
// tensor cores' bf16 keys, as the build's assignment step) of every row of a
// column: the "add rows" step for collections too large to build on directly
// (train on a sample, then assign). out: int32 [n] (device or host).
int ivf_assign_gpu(vs_ctx* ctx, const vs_ivf* v, const vs_column* col, int32_t* out) {
    using namespace vs_internal;
    cudaStream_t st = ctx->stream;
    const int64_t n = col->n;
    const int d = v->d;
    const int dp = (d + 7) / 8 * 8;
    const int nlist = v->nlist;
    __nv_bfloat16* cb = nullptr;
    __nv_bfloat16* xb = nullptr;
    unsigned* junk = nullptr;
    unsigned long long* packed = nullptr;
    int* assign = nullptr;
    float* dist = nullptr;
    CKS(arena_alloc(ctx, (size_t)nlist * dp, &cb));
    CKS(arena_alloc(ctx, (size_t)tc_argmin_chunk(n) * dp, &xb));
    CKS(arena_alloc(ctx, 2, &junk));
    CKS(arena_alloc(ctx, (size_t)n, &packed));
    CKS(arena_alloc(ctx, (size_t)n, &assign));
    CKS(arena_alloc(ctx, (size_t)n, &dist));
    unsigned* cst = nullptr;
    unsigned long long* top2 = nullptr;
    float2* rowstats = nullptr;
    CKS(arena_alloc(ctx, 2, &cst));
    CKS(arena_alloc(ctx, (size_t)n * 4, &top2));
    CKS(arena_alloc(ctx, (size_t)n, &rowstats));
    CK(cudaMemsetAsync(cst, 0, 2 * sizeof(unsigned), st));
    CKS(tc_stage_f16(ctx, v->centroids, nlist, d, v->cmax, cb, cst));
    CKS(tc_argmin_rows(ctx, col->data, col->dtype, n, d, cb, v->cnorms, nlist, packed, xb, junk, top2, rowstats,
                       col->max_norm_bits, v->cmax));
    k_unpack<<<grid_for(n), 256, 0, st>>>(packed, col->norms, n, assign, dist);
    CK(cudaGetLastError());
    CKS(near_tie_recheck(ctx, col, n, d, top2, rowstats, cst, v->cmax, v->centroids, nlist, v->cnorms, assign, dist,
                         nullptr));
    CK(cudaMemcpyAsync(out, assign, (size_t)n * sizeof(int32_t), cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
    ctx->stats[VS_STAT_LAUNCHES] += 3;
    return VS_OK;
}

}  // namespace vs

