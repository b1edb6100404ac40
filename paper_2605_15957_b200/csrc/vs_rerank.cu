// Phase B: exact re-rank and tie-rule top-k, plus the cross-shard merge.
//
// For each query (one CTA):
//   1. K* = k-th smallest approximate key over all candidate buffers,
//   2. survivors = candidates with key <= K* + margin  (a superset of the
//      exact top-k by the error bound),
//   3. exact float64 score of every survivor with the reference's arithmetic
//      and summation order (np_pairwise, bit-identical to distances.py:54-58),
//   4. exact top-k under the tie rule (key, row id) — select_top,
//      distances.py:79-94 — by bitwise binary search on the composite key,
//      then a bitonic sort of the k winners in shared memory.
#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

namespace {
constexpr int NT = 256;
constexpr int NWARP = NT / 32;
constexpr int KMAX = 2048;  // == vs_topk_cap()
constexpr int LCAP = 3072;  // live candidates staged in shared memory per query

__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(VS_FULL, v, o);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    long long t = 0;
#pragma unroll
    for (int i = 0; i < NWARP; ++i) t += red[i];
    return t;
}

struct TopkSmem {
    uint64_t key[KMAX];
    int64_t id[KMAX];
    long long red[NWARP];
    int counter;
};

// Exact top-k over n entries (orderable key, id) held in global scratch.
// Writes min(n, k) entries in (key, id) order to out_* (row q).
__device__ void block_topk_exact(const uint64_t* __restrict__ key, const int64_t* __restrict__ id,
                                 int64_t n, int k, TopkSmem& sm, int ip, int64_t q,
                                 int64_t* out_ids, double* out_dist, int32_t* out_ids32,
                                 int32_t* out_count) {
    const int tid = threadIdx.x;
    const int keff = (int)min((int64_t)k, n);
    uint64_t K = ~0ull;
    uint64_t I = ~0ull;
    if (n > k) {
        // smallest K with count(key <= K) >= k
        uint64_t lo = 0, hi = ~0ull;
        while (lo < hi) {
            uint64_t mid = lo + ((hi - lo) >> 1);
            long long c = 0;
            for (int64_t i = tid; i < n; i += NT) c += (key[i] <= mid);
            c = block_sum_ll(c, sm.red);
            if (c >= k) hi = mid; else lo = mid + 1;
        }
        K = lo;
        long long clt = 0;
        for (int64_t i = tid; i < n; i += NT) clt += (key[i] < K);
        clt = block_sum_ll(clt, sm.red);
        const long long need = k - clt;  // >= 1 ties at K to take, lowest ids first
        uint64_t ilo = 0, ihi = ~0ull;
        while (ilo < ihi) {
            uint64_t mid = ilo + ((ihi - ilo) >> 1);
            long long c = 0;
            for (int64_t i = tid; i < n; i += NT) c += (key[i] == K && (uint64_t)id[i] <= mid);
            c = block_sum_ll(c, sm.red);
            if (c >= need) ihi = mid; else ilo = mid + 1;
        }
        I = ilo;
    }
    if (tid == 0) sm.counter = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += NT) {
        uint64_t kk = key[i];
        uint64_t ii = (uint64_t)id[i];
        bool win = (n <= k) || kk < K || (kk == K && ii <= I);
        if (win) {
            int slot = atomicAdd(&sm.counter, 1);
            sm.key[slot] = kk;
            sm.id[slot] = (int64_t)ii;
        }
    }
    __syncthreads();
    int P = 1;
    while (P < keff) P <<= 1;
    for (int i = keff + tid; i < P; i += NT) {
        sm.key[i] = ~0ull;
        sm.id[i] = 0x7fffffffffffffffll;
    }
    __syncthreads();
    // bitonic sort of P entries by (key, id)
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < P / 2; i += NT) {
                int lo_i = 2 * i - (i & (stride - 1));
                int hi_i = lo_i + stride;
                bool asc = ((lo_i & size) == 0);
                uint64_t ka = sm.key[lo_i], kb = sm.key[hi_i];
                int64_t ia = sm.id[lo_i], ib = sm.id[hi_i];
                bool gt = (ka > kb) || (ka == kb && ia > ib);
                if (gt == asc) {
                    sm.key[lo_i] = kb; sm.key[hi_i] = ka;
                    sm.id[lo_i] = ib; sm.id[hi_i] = ia;
                }
            }
            __syncthreads();
        }
    }
    for (int r = tid; r < k; r += NT) {
        const int64_t o = q * (int64_t)k + r;
        if (r < keff) {
            double key_d = o2d(sm.key[r]);
            if (out_ids) out_ids[o] = sm.id[r];
            if (out_ids32) out_ids32[o] = (int32_t)sm.id[r];
            if (out_dist) out_dist[o] = ip ? -key_d : key_d;
        } else {
            if (out_ids) out_ids[o] = -1;
            if (out_ids32) out_ids32[o] = -1;
            if (out_dist) out_dist[o] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
    if (tid == 0 && out_count) out_count[q] = keff;
    __syncthreads();
}
}  // namespace

template <typename T, bool IP>
__global__ void __launch_bounds__(NT) k_rerank(RerankParams p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    TopkSmem& sm = *reinterpret_cast<TopkSmem*>(smraw);
    int* cnts = reinterpret_cast<int*>(smraw + sizeof(TopkSmem));
    const int tid = threadIdx.x;
    const int64_t q = blockIdx.x;
    const int C = p.cb.C, nsub = p.cb.n_sub;
    const float* ckey = p.cb.key + q * nsub * (int64_t)C;
    const uint32_t* cpos = p.cb.pos + q * nsub * (int64_t)C;
    long long tot = 0;
    for (int s = tid; s < nsub; s += NT) {
        int c = p.cb.cnt[q * nsub + s];
        cnts[s] = c;
        tot += c;
    }
    tot = block_sum_ll(tot, sm.red);  // includes a __syncthreads
    const int64_t nslots = (int64_t)nsub * C;
    uint32_t* spos = p.s_pos + q * p.s_cap;
    uint64_t* skey = p.s_key + q * p.s_cap;
    int64_t* sid = p.s_id + q * p.s_cap;
    const uint32_t pre = p.tau_g ? p.tau_g[q] : 0xffffffffu;
    // 0. gather the live candidates (key <= prefilter bound) into shared memory
    float* lkey = reinterpret_cast<float*>(cnts + nsub);
    uint32_t* lpos = reinterpret_cast<uint32_t*>(lkey + LCAP);
    if (tid == 0) sm.counter = 0;
    __syncthreads();
    for (int64_t i = tid; i < nslots; i += NT) {
        int s = (int)(i / C), j = (int)(i - (int64_t)s * C);
        if (j < cnts[s]) {
            const float kk = ckey[i];
            if (f2o(kk) <= pre) {
                int slot = atomicAdd(&sm.counter, 1);
                if (slot < LCAP) {
                    lkey[slot] = kk;
                    lpos[slot] = cpos[i];
                }
            }
        }
    }
    __syncthreads();
    const int nl = sm.counter;
    __syncthreads();
    int64_t ns = 0;
    if (nl <= LCAP) {
        // 1. k-th smallest approximate key, 2. survivors  (shared-memory path)
        uint32_t thr_o = 0xffffffffu;
        if (nl > p.k) {
            uint32_t lo = 0u, hi = pre;
            while (lo < hi) {
                uint32_t mid = lo + ((hi - lo) >> 1);
                long long c = 0;
                for (int i = tid; i < nl; i += NT) c += (f2o(lkey[i]) <= mid);
                c = block_sum_ll(c, sm.red);
                if (c >= p.k) hi = mid; else lo = mid + 1;
            }
            thr_o = f2o(__fadd_ru(o2f(lo), p.margin[q]));
        }
        if (tid == 0) sm.counter = 0;
        __syncthreads();
        for (int i = tid; i < nl; i += NT) {
            if (f2o(lkey[i]) <= thr_o) {
                int slot = atomicAdd(&sm.counter, 1);
                if (slot < p.s_cap) spos[slot] = lpos[i];
            }
        }
        __syncthreads();
        ns = sm.counter;
    } else {
        // 1. k-th smallest approximate key over the buffers (global-memory path)
        uint32_t thr_o = 0xffffffffu;
        if (tot > p.k) {
            uint32_t lo = 0u, hi = pre;
            while (lo < hi) {
                uint32_t mid = lo + ((hi - lo) >> 1);
                long long c = 0;
                for (int64_t i = tid; i < nslots; i += NT) {
                    int s = (int)(i / C), j = (int)(i - (int64_t)s * C);
                    if (j < cnts[s]) c += (f2o(ckey[i]) <= mid);
                }
                c = block_sum_ll(c, sm.red);
                if (c >= p.k) hi = mid; else lo = mid + 1;
            }
            thr_o = f2o(__fadd_ru(o2f(lo), p.margin[q]));
        }
        // 2. survivors
        if (tid == 0) sm.counter = 0;
        __syncthreads();
        for (int64_t i = tid; i < nslots; i += NT) {
            int s = (int)(i / C), j = (int)(i - (int64_t)s * C);
            if (j < cnts[s] && f2o(ckey[i]) <= thr_o) {
                int slot = atomicAdd(&sm.counter, 1);
                if (slot < p.s_cap) spos[slot] = cpos[i];
            }
        }
        __syncthreads();
        ns = sm.counter;
    }
    if (ns > p.s_cap) {  // cannot re-rank all survivors: re-run with larger buffers
        if (tid == 0) p.cb.overflow[q] = 1;
        ns = p.s_cap;
    }
    // 3. exact float64 scores
    const T* rows = reinterpret_cast<const T*>(p.rows);
    const float* qv = p.Q + q * (int64_t)p.d;
    for (int64_t i = tid; i < ns; i += NT) {
        const uint32_t ps = spos[i];
        const int64_t r = p.row_map ? p.row_map[ps] : (int64_t)ps;
        const double sc = np_pairwise<T, IP>(qv, rows + r * (int64_t)p.d, p.d);
        skey[i] = d2o(IP ? -sc : sc);
        sid[i] = p.id_map ? p.id_map[ps] : r + p.id_offset;
    }
    __syncthreads();
    if (tid == 0 && p.n_survivors) atomicAdd(p.n_survivors, (unsigned long long)ns);
    // 4. exact tie-rule top-k
    block_topk_exact(skey, sid, ns, p.k, sm, IP, q, p.out_ids, p.out_dist, p.out_ids32,
                     p.out_count);
}

template <typename T>
cudaError_t launch_rerank(const RerankParams& p, cudaStream_t s) {
    if (p.nq == 0) return cudaSuccess;
    const size_t smem = sizeof(TopkSmem) + (size_t)p.cb.n_sub * sizeof(int) + LCAP * 8 + 16;
    cudaError_t e;
    if (p.ip) {
        e = cudaFuncSetAttribute(k_rerank<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_rerank<T, true><<<(unsigned)p.nq, NT, smem, s>>>(p);
    } else {
        e = cudaFuncSetAttribute(k_rerank<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_rerank<T, false><<<(unsigned)p.nq, NT, smem, s>>>(p);
    }
    return cudaGetLastError();
}
template cudaError_t launch_rerank<float>(const RerankParams&, cudaStream_t);
template cudaError_t launch_rerank<__nv_bfloat16>(const RerankParams&, cudaStream_t);

// ---- cross-shard merge ------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_merge(MergeParams p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    TopkSmem& sm = *reinterpret_cast<TopkSmem*>(smraw);
    const int64_t q = blockIdx.x;
    const int tid = threadIdx.x;
    const int64_t cap = (int64_t)p.nparts * p.k_in;
    uint64_t* skey = p.s_key + q * cap;
    int64_t* sid = p.s_id + q * cap;
    if (tid == 0) sm.counter = 0;
    __syncthreads();
    for (int64_t i = tid; i < cap; i += NT) {
        int g = (int)(i / p.k_in), j = (int)(i - (int64_t)g * p.k_in);
        if (j < p.counts[(int64_t)g * p.nq + q]) {
            const int64_t src = ((int64_t)g * p.nq + q) * p.k_in + j;
            const double dd = p.dist[src];
            int slot = atomicAdd(&sm.counter, 1);
            skey[slot] = d2o(p.ip ? -dd : dd);
            sid[slot] = p.ids[src];
        }
    }
    __syncthreads();
    const int64_t n = sm.counter;
    __syncthreads();
    block_topk_exact(skey, sid, n, p.k, sm, p.ip, q, p.out_ids, p.out_dist, nullptr, p.out_count);
}

cudaError_t launch_merge(const MergeParams& p, cudaStream_t s) {
    if (p.nq == 0) return cudaSuccess;
    const size_t smem = sizeof(TopkSmem);
    cudaError_t e = cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_merge<<<(unsigned)p.nq, NT, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace vs
