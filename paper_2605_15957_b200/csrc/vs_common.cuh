// Shared device utilities for the B200 vector-search kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#define VS_WARP 32
#define VS_FULL 0xffffffffu

namespace vs {

// ---- order-preserving key encodings ------------------------------------------
// float -> uint32 whose unsigned order equals the float order (finite values).
__device__ __forceinline__ uint32_t f2o(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float o2f(uint32_t o) {
    uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(u);
}
__device__ __forceinline__ uint64_t d2o(double f) {
    uint64_t u = (uint64_t)__double_as_longlong(f);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double o2d(uint64_t o) {
    uint64_t u = (o & 0x8000000000000000ull) ? (o & 0x7fffffffffffffffull) : ~o;
    return __longlong_as_double((long long)u);
}

// ---- element loads --------------------------------------------------------------
__device__ __forceinline__ float ld_elem(const float* p) { return *p; }
__device__ __forceinline__ float ld_elem(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// ---- the reference's exact float64 score ------------------------------------------
// numpy's pairwise summation (umath loops: pairwise_sum_DOUBLE, PW_BLOCKSIZE
// 128, 8 partial sums) applied to the float64 elementwise terms the reference
// forms in distances.py:54-58: (q-x)*(q-x) for squared L2, q*x for inner
// product. __d*_rn intrinsics forbid FMA contraction, so every rounding step
// matches numpy and the result is bit-identical to the reference's score.
template <typename T, bool IP>
__device__ __forceinline__ double np_term(const float* q, const T* x, int i) {
    double a = (double)q[i];
    double b = (double)ld_elem(x + i);
    if (IP) return __dmul_rn(a, b);
    double t = __dsub_rn(a, b);
    return __dmul_rn(t, t);
}

template <typename T, bool IP>
__device__ double np_pairwise_leaf(const float* q, const T* x, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, np_term<T, IP>(q, x, i));
        return r;
    }
    double r0 = np_term<T, IP>(q, x, 0), r1 = np_term<T, IP>(q, x, 1);
    double r2 = np_term<T, IP>(q, x, 2), r3 = np_term<T, IP>(q, x, 3);
    double r4 = np_term<T, IP>(q, x, 4), r5 = np_term<T, IP>(q, x, 5);
    double r6 = np_term<T, IP>(q, x, 6), r7 = np_term<T, IP>(q, x, 7);
    int i = 8;
    const int lim = n - (n % 8);
    for (; i < lim; i += 8) {
        r0 = __dadd_rn(r0, np_term<T, IP>(q, x, i + 0));
        r1 = __dadd_rn(r1, np_term<T, IP>(q, x, i + 1));
        r2 = __dadd_rn(r2, np_term<T, IP>(q, x, i + 2));
        r3 = __dadd_rn(r3, np_term<T, IP>(q, x, i + 3));
        r4 = __dadd_rn(r4, np_term<T, IP>(q, x, i + 4));
        r5 = __dadd_rn(r5, np_term<T, IP>(q, x, i + 5));
        r6 = __dadd_rn(r6, np_term<T, IP>(q, x, i + 6));
        r7 = __dadd_rn(r7, np_term<T, IP>(q, x, i + 7));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                           __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    for (; i < n; ++i) res = __dadd_rn(res, np_term<T, IP>(q, x, i));
    return res;
}

// Iterative evaluation of the recursion
//   pw(n) = n <= 128 ? leaf(n) : pw(n2) + pw(n - n2),  n2 = n/2 - (n/2) % 8
// as a post-order walk with an explicit stack (depth <= 16).
template <typename T, bool IP>
__device__ double np_pairwise(const float* q, const T* x, int n) {
    if (n <= 128) return np_pairwise_leaf<T, IP>(q, x, n);
    int st_off[16], st_n[16], st_state[16];
    double st_left[16];
    int sp = 0;
    st_off[0] = 0; st_n[0] = n; st_state[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        int off = st_off[sp], m = st_n[sp];
        if (m <= 128) {
            ret = np_pairwise_leaf<T, IP>(q + off, x + off, m);
            --sp;
            continue;
        }
        int n2 = m / 2;
        n2 -= n2 % 8;
        if (st_state[sp] == 0) {          // descend left
            st_state[sp] = 1;
            ++sp;
            st_off[sp] = off; st_n[sp] = n2; st_state[sp] = 0;
        } else if (st_state[sp] == 1) {   // left done -> descend right
            st_left[sp] = ret;
            st_state[sp] = 2;
            ++sp;
            st_off[sp] = off + n2; st_n[sp] = m - n2; st_state[sp] = 0;
        } else {                          // both done
            ret = __dadd_rn(st_left[sp], ret);
            --sp;
        }
    }
    return ret;
}

// ---- warp helpers ------------------------------------------------------------------
__device__ __forceinline__ int warp_sum(int v) { return __reduce_add_sync(VS_FULL, v); }
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(VS_FULL, v, o);
    return v;
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---- warp-cooperative candidate-buffer compaction ---------------------------------
// A candidate buffer holds (approximate key, position) pairs of one query and
// one scan partition ("sub"), appended in increasing position order. Keep the
// k smallest keys plus every key within `margin` of the k-th (the rigorous
// error bound of the approximate score), i.e. entries with
// key <= kth + margin. Returns the new count; `*thr` receives the new
// admission threshold. If more than `limit` entries survive, the buffer
// cannot make progress: the margin is dropped and entries truncated in
// position order, and the caller flags the query for a re-run with a larger
// buffer (`*overflow` = 1).
//
// Buffers of up to 32 x REG_PER_LANE entries are compacted from registers
// (one load of the keys into 8, 16 or 32 registers per lane, then a bisection
// over the live keys' [min, max] on the register copy); larger buffers fall
// back to streaming the keys.
constexpr int COMPACT_REG_PER_LANE = 32;

// register-resident compaction of n <= 32 * R entries
template <int R>
__device__ __forceinline__ int warp_compact_reg(float* keys, uint32_t* pos, int n, int k, float margin,
                                                int limit, float* thr, int* overflow) {
    const int lane = threadIdx.x & 31;
    // one coalesced load of keys and positions, then selection, counting and
    // compaction without further memory reads
    uint32_t ko[R];
    uint32_t po[R];
    uint32_t vmin = 0xffffffffu, vmax = 0u;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int j = lane + 32 * i;
        ko[i] = (j < n) ? f2o(keys[j]) : 0xffffffffu;
        po[i] = (j < n) ? pos[j] : 0u;
        if (j < n) {
            vmin = min(vmin, ko[i]);
            vmax = max(vmax, ko[i]);
        }
    }
    // the k-th smallest lies in [min, max] of the live keys: bisect only that range
    uint32_t lo = __reduce_min_sync(VS_FULL, vmin);
    uint32_t hi = n >= k ? __reduce_max_sync(VS_FULL, vmax) : 0xffffffffu;
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        int c = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) c += (ko[i] <= mid);
        c = warp_sum(c);  // padding (0xffffffff) only counts at the very top
        if (c >= k) hi = mid; else lo = mid + 1;
    }
    const float kth = o2f(lo);
    uint32_t to = f2o(__fadd_ru(kth, margin));
    int c = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) c += (ko[i] <= to);
    c = warp_sum(c);
    if (c > limit) {  // margin set cannot fit: keep the k-th bound, flag a re-run
        *overflow = 1;
        to = lo;
        c = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) c += (ko[i] <= to);
        c = warp_sum(c);
        if (c > limit) c = limit;
    }
    __syncwarp();
    int base = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const bool keep = ko[i] <= to;   // entries are in position order: i-major
        const unsigned b = __ballot_sync(VS_FULL, keep);
        const int dst = base + __popc(b & lanemask_lt());
        if (keep && dst < limit) {
            keys[dst] = o2f(ko[i]);
            pos[dst] = po[i];
        }
        base += __popc(b);
    }
    *thr = o2f(to);
    return min(base, limit);
}

__device__ __forceinline__ int warp_compact(float* keys, uint32_t* pos, int n, int k, float margin,
                                            int limit, float* thr, int* overflow) {
    const int lane = threadIdx.x & 31;
    if (n <= 32 * 8) return warp_compact_reg<8>(keys, pos, n, k, margin, limit, thr, overflow);
    if (n <= 32 * 16) return warp_compact_reg<16>(keys, pos, n, k, margin, limit, thr, overflow);
    if (n <= 32 * COMPACT_REG_PER_LANE)
        return warp_compact_reg<COMPACT_REG_PER_LANE>(keys, pos, n, k, margin, limit, thr, overflow);
    uint32_t lo = 0u, hi = 0xffffffffu;
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        int c = 0;
        for (int j = lane; j < n; j += 32) c += (f2o(keys[j]) <= mid);
        c = warp_sum(c);
        if (c >= k) hi = mid; else lo = mid + 1;
    }
    const float kth = o2f(lo);
    float t = __fadd_ru(kth, margin);
    for (int pass = 0; pass < 2; ++pass) {
        const uint32_t to = f2o(t);
        int c = 0;
        for (int j = lane; j < n; j += 32) c += (f2o(keys[j]) <= to);
        c = warp_sum(c);
        if (c <= limit || pass == 1) {
            int base = 0;
            for (int j0 = 0; j0 < n; j0 += 32) {
                const int j = j0 + lane;
                float kk = 0.f;
                uint32_t pp = 0;
                bool keep = false;
                if (j < n) { kk = keys[j]; pp = pos[j]; keep = f2o(kk) <= to; }
                const unsigned b = __ballot_sync(VS_FULL, keep);
                __syncwarp();
                const int dst = base + __popc(b & lanemask_lt());
                if (keep && dst < limit) { keys[dst] = kk; pos[dst] = pp; }
                base += __popc(b);
                __syncwarp();
            }
            if (c > limit) { *overflow = 1; base = limit; }
            *thr = t;
            return base;
        }
        t = kth;  // margin cannot fit: fall back to the k-th key and flag
        *overflow = 1;
    }
    return n;  // unreachable
}

}  // namespace vs
