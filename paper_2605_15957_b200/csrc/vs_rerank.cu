// Phase B: exact re-rank and tie-rule top-k, plus the cross-shard merge.
//
// For each query (one CTA of 8 warps):
//   0. gather the live candidates (key <= the query's global admission
//      bound) from all candidate buffers into shared memory,
//   1. K* = k-th smallest approximate key,
//   2. survivors = candidates with key <= K* + margin  (a superset of the
//      exact top-k by the error bound),
//   3. exact float64 score of every survivor with the reference's arithmetic
//      and summation order (bit-identical to distances.py:54-58): one warp
//      per survivor row, the row staged in shared memory by coalesced
//      128-bit loads, numpy's accumulation chains spread over the lanes,
//   4. exact top-k under the tie rule (key, row id) — select_top,
//      distances.py:79-94 — by a bitonic sort of the survivors in shared
//      memory (or a bitwise binary search on the composite key when more
//      than 2048 survive).
//
// Shared memory is one union region reused by steps 0-2 (live candidates),
// 3 (row staging) and 4 (sort), so several CTAs stay resident per SM.
#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

namespace {
constexpr int NT = 256;
constexpr int NWARP = NT / 32;
constexpr int KMAX = 2048;      // == vs_topk_cap(): sort capacity
// live candidates staged in shared memory per query: the wide build (large k)
// stages 8192 at 2 CTAs/SM, the narrow one 4096 at 4 CTAs/SM (64 registers)
template <bool WIDE> constexpr int lcap() { return WIDE ? 8192 : 4096; }
constexpr int MAXLEAF = 32;     // numpy pairwise leaves (>= 64 elements each) -> d <= 2048 on the warp path
constexpr int WARP_D_MAX = 2048;
// union of: live candidates (LCAP x 8 B), staged rows (NWARP x d x 4 B),
// sort buffers (KMAX x 16 B)
constexpr size_t UNION_BYTES = 32768;   // narrow build; the wide one doubles it
template <bool WIDE> constexpr size_t union_min() { return WIDE ? 2 * UNION_BYTES : UNION_BYTES; }
// staged row stride (elements): padded d plus the leaf skews (32 B per leaf;
// leaves hold >= 64 elements, so at most d / 64 + 1 of them)
__host__ __device__ __forceinline__ int row_stride(int d) { return ((d + 7) & ~7) + 16 * (d / 64 + 1); }
__host__ __device__ __forceinline__ int q_stride(int d) { return ((d + 3) & ~3) + 8 * (d / 64 + 1); }
// number of leaves of numpy's pairwise recursion over n elements (blocks of
// <= 128 are leaves; larger blocks split at n/2 rounded down to a multiple of 8)
inline int np_nleaf(int n) {
    if (n <= 128) return 1;
    int n2 = n / 2;
    n2 -= n2 % 8;
    return np_nleaf(n2) + np_nleaf(n - n2);
}
// register path of the exact scorer: every lane owns two chains of one leaf
// for the whole row (<= 8 leaves), rows read straight from global memory
inline bool reg_path_ok(int d) { return d >= 8 && d <= 1024 && d % 2 == 0 && np_nleaf(d) <= 8; }
inline size_t union_bytes(int d, bool wide) {
    const size_t rows = (size_t)NWARP * 2 * (size_t)row_stride(d) * 4;   // two staged rows per warp
    const size_t base = wide ? union_min<true>() : union_min<false>();
    return (d <= WARP_D_MAX && !reg_path_ok(d) && rows > base) ? rows : base;
}

constexpr int HBINS = 2048;     // radix-select histogram bins (11 bits)
constexpr int SHQ = 8;          // per-leaf shared-memory skew of the staged query (floats)

struct Small : LeafPlan {
    long long red[NWARP];
    unsigned wtot[NWARP];
    int sel_bin;
    unsigned sel_below;
    int counter;
};

// k-th smallest (1 <= k <= count) orderable key among the keys `foreach`
// visits: a 3-pass radix select (11 + 11 + 10 bits) over a shared-memory
// histogram, instead of a 32-step bisection over the keys.
template <class ForEach>
__device__ uint32_t block_radix_kth(ForEach foreach, unsigned k, unsigned* hist, Small& sm) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint32_t prefix = 0u, pmask = 0u;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
        const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
        const int nb = pass == 2 ? 1024 : 2048;
        for (int i = tid; i < nb; i += NT) hist[i] = 0u;
        __syncthreads();
        foreach([&](uint32_t u) {
            if ((u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & (uint32_t)(nb - 1)], 1u);
        });
        __syncthreads();
        const int per = nb / NT;
        unsigned loc = 0;
        for (int b = 0; b < per; ++b) loc += hist[tid * per + b];
        unsigned incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(VS_FULL, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) sm.wtot[w] = incl;
        __syncthreads();
        unsigned excl = incl - loc;
        for (int i = 0; i < w; ++i) excl += sm.wtot[i];
        if (excl < k && k <= excl + loc) {
            unsigned c = excl;
            for (int b = 0; b < per; ++b) {
                const unsigned h = hist[tid * per + b];
                if (c + h >= k) {
                    sm.sel_bin = tid * per + b;
                    sm.sel_below = c;
                    break;
                }
                c += h;
            }
        }
        __syncthreads();
        k -= sm.sel_below;
        prefix |= (uint32_t)sm.sel_bin << shift;
        pmask |= (uint32_t)(nb - 1) << shift;
        __syncthreads();
    }
    return prefix;
}

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

__device__ __forceinline__ void emit_row(int64_t q, int k, int keff, const uint64_t* skey, const int64_t* sid,
                                         int ip, int64_t* out_ids, double* out_dist, int32_t* out_ids32,
                                         int32_t* out_count) {
    for (int r = threadIdx.x; r < k; r += NT) {
        const int64_t o = q * (int64_t)k + r;
        if (r < keff) {
            const double key_d = o2d(skey[r]);
            if (out_ids) out_ids[o] = sid[r];
            if (out_ids32) out_ids32[o] = (int32_t)sid[r];
            if (out_dist) out_dist[o] = ip ? -key_d : key_d;
        } else {
            if (out_ids) out_ids[o] = -1;
            if (out_ids32) out_ids32[o] = -1;
            if (out_dist) out_dist[o] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
    if (threadIdx.x == 0 && out_count) out_count[q] = keff;
}

// bitonic sort of P (power of two) orderable keys in shared memory, ascending
__device__ void bitonic_sort_u32(uint32_t* key, int P) {
    const int tid = threadIdx.x;
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < P / 2; i += NT) {
                const int lo_i = 2 * i - (i & (stride - 1));
                const int hi_i = lo_i + stride;
                const bool asc = ((lo_i & size) == 0);
                const uint32_t ka = key[lo_i], kb = key[hi_i];
                if ((ka > kb) == asc) {
                    key[lo_i] = kb;
                    key[hi_i] = ka;
                }
            }
            __syncthreads();
        }
    }
}

// distributed protocol, phase 1: this shard's k smallest approximate keys,
// ascending, +inf padded (keys <= kth are gathered into `a` (HBINS slots))
template <class ForEach>
__device__ void write_local_topk_keys(ForEach foreach, uint32_t kth, int k, unsigned* a, Small& sm, float half_margin,
                                      float* out) {
    const int tid = threadIdx.x;
    if (tid == 0) sm.counter = 0;
    __syncthreads();
    foreach([&](uint32_t o) {
        if (o <= kth) {
            const int slot = atomicAdd(&sm.counter, 1);
            if (slot < HBINS) a[slot] = o;
        }
    });
    __syncthreads();
    const int c = min(sm.counter, HBINS);
    int P = 1;
    while (P < c) P <<= 1;
    for (int i = c + tid; i < P; i += NT) a[i] = 0xffffffffu;
    __syncthreads();
    bitonic_sort_u32(a, P);
    // upper bounds on the exact keys (approx + this shard's margin / 2, rounded
    // up): the k-th of their union over shards bounds the global k-th exact key
    for (int i = tid; i < k; i += NT) out[i] = i < c ? __fadd_ru(o2f(a[i]), half_margin) : __int_as_float(0x7f800000);
}

// bitonic sort of P (power of two) (key, id) pairs in shared memory
__device__ void bitonic_sort(uint64_t* key, int64_t* id, int P) {
    const int tid = threadIdx.x;
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < P / 2; i += NT) {
                const int lo_i = 2 * i - (i & (stride - 1));
                const int hi_i = lo_i + stride;
                const bool asc = ((lo_i & size) == 0);
                const uint64_t ka = key[lo_i], kb = key[hi_i];
                const int64_t ia = id[lo_i], ib = id[hi_i];
                const bool gt = (ka > kb) || (ka == kb && ia > ib);
                if (gt == asc) {
                    key[lo_i] = kb; key[hi_i] = ka;
                    id[lo_i] = ib; id[hi_i] = ia;
                }
            }
            __syncthreads();
        }
    }
}

// Exact top-k over n (orderable key, id) entries in global scratch. Uses the
// union region `u` (>= KMAX * 16 bytes) for the final sort.
__device__ void block_topk_exact(const uint64_t* __restrict__ key, const int64_t* __restrict__ id, int64_t n,
                                 int k, Small& sm, unsigned char* u, int ip, int64_t q, int64_t* out_ids,
                                 double* out_dist, int32_t* out_ids32, int32_t* out_count) {
    const int tid = threadIdx.x;
    uint64_t* skey = reinterpret_cast<uint64_t*>(u);
    int64_t* sid = reinterpret_cast<int64_t*>(u + KMAX * 8);
    const int keff = (int)min((int64_t)k, n);
    if (n <= KMAX) {
        int P = 1;
        while (P < n) P <<= 1;
        for (int i = tid; i < P; i += NT) {
            skey[i] = i < n ? key[i] : ~0ull;
            sid[i] = i < n ? id[i] : 0x7fffffffffffffffll;
        }
        __syncthreads();
        bitonic_sort(skey, sid, P);
        emit_row(q, k, keff, skey, sid, ip, out_ids, out_dist, out_ids32, out_count);
        __syncthreads();
        return;
    }
    // smallest K with count(key <= K) >= k, then the needed ties at K by id
    uint64_t lo = 0, hi = ~0ull;
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        long long c = 0;
        for (int64_t i = tid; i < n; i += NT) c += (key[i] <= mid);
        c = block_sum_ll(c, sm.red);
        if (c >= k) hi = mid; else lo = mid + 1;
    }
    const uint64_t K = lo;
    long long clt = 0;
    for (int64_t i = tid; i < n; i += NT) clt += (key[i] < K);
    clt = block_sum_ll(clt, sm.red);
    const long long need = k - clt;
    uint64_t ilo = 0, ihi = ~0ull;
    while (ilo < ihi) {
        const uint64_t mid = ilo + ((ihi - ilo) >> 1);
        long long c = 0;
        for (int64_t i = tid; i < n; i += NT) c += (key[i] == K && (uint64_t)id[i] <= mid);
        c = block_sum_ll(c, sm.red);
        if (c >= need) ihi = mid; else ilo = mid + 1;
    }
    const uint64_t I = ilo;
    if (tid == 0) sm.counter = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += NT) {
        const uint64_t kk = key[i];
        const uint64_t ii = (uint64_t)id[i];
        if (kk < K || (kk == K && ii <= I)) {
            const int slot = atomicAdd(&sm.counter, 1);
            skey[slot] = kk;
            sid[slot] = (int64_t)ii;
        }
    }
    __syncthreads();
    int P = 1;
    while (P < keff) P <<= 1;
    for (int i = keff + tid; i < P; i += NT) {
        skey[i] = ~0ull;
        sid[i] = 0x7fffffffffffffffll;
    }
    __syncthreads();
    bitonic_sort(skey, sid, P);
    emit_row(q, k, keff, skey, sid, ip, out_ids, out_dist, out_ids32, out_count);
    __syncthreads();
}

}  // namespace

// leaves of numpy's pairwise recursion for a length-d reduction, left to right,
// the combine tree, and the leaf index of every 8-element group (computed on
// the host once per launch; the kernel copies it into shared memory)
void np_leaves(int d, LeafPlan& S) {
    S = LeafPlan{};
    int st_off[16], st_n[16];
    int sp = 0, nl = 0;
    st_off[0] = 0;
    st_n[0] = d;
    while (sp >= 0) {
        const int off = st_off[sp], m = st_n[sp];
        --sp;
        if (m <= 128) {
            if (nl < MAXLEAF) {
                S.leaf_off[nl] = off;
                S.leaf_n[nl] = m;
            }
            ++nl;
            continue;
        }
        int n2 = m / 2;
        n2 -= n2 % 8;
        ++sp;  // right first, so the left half is expanded first
        st_off[sp] = off + n2;
        st_n[sp] = m - n2;
        ++sp;
        st_off[sp] = off;
        st_n[sp] = n2;
    }
    S.nleaf = nl;
    for (int L = 0; L < nl && L < MAXLEAF; ++L)
        for (int g = S.leaf_off[L] / 8; g < (S.leaf_off[L] + S.leaf_n[L] + 7) / 8; ++g)
            S.gsk[g] = (unsigned char)L;
    // internal nodes in post-order (each combines two earlier slots)
    int st_n2[16], st_state[16], st_left[16];
    int sp2 = 0, next_leaf = 0, nn = 0, ret = 0;
    st_n2[0] = d;
    st_state[0] = 0;
    if (d <= 128) {
        S.nnode = 0;
        return;
    }
    while (sp2 >= 0) {
        const int m = st_n2[sp2];
        if (m <= 128) {
            ret = next_leaf++;
            --sp2;
            continue;
        }
        int n2 = m / 2;
        n2 -= n2 % 8;
        if (st_state[sp2] == 0) {
            st_state[sp2] = 1;
            ++sp2;
            st_n2[sp2] = n2;
            st_state[sp2] = 0;
        } else if (st_state[sp2] == 1) {
            st_left[sp2] = ret;
            st_state[sp2] = 2;
            ++sp2;
            st_n2[sp2] = m - n2;
            st_state[sp2] = 0;
        } else {
            S.node_a[nn] = st_left[sp2];
            S.node_b[nn] = ret;
            ret = nl + nn;
            ++nn;
            --sp2;
        }
    }
    S.nnode = nn;
    // levels: a node runs after both operands (leaves are level -1)
    S.nlevels = 0;
    for (int j = 0; j < nn; ++j) {
        const int la = S.node_a[j] >= nl ? S.node_lvl[S.node_a[j] - nl] : -1;
        const int lb = S.node_b[j] >= nl ? S.node_lvl[S.node_b[j] - nl] : -1;
        S.node_lvl[j] = (la > lb ? la : lb) + 1;
        if (S.node_lvl[j] + 1 > S.nlevels) S.nlevels = S.node_lvl[j] + 1;
    }
}

namespace {

// staged-row skew per class, in elements: 32 bytes (8 banks)
template <typename T>
__host__ __device__ constexpr int shx() { return 32 / (int)sizeof(T); }

template <bool IP, typename T>
__device__ __forceinline__ double term_sm(const float* q, const T* x, int i) {
    const double a = (double)q[i], b = (double)ld_elem(x + i);
    if (IP) return __dmul_rn(a, b);
    const double t = __dsub_rn(a, b);
    return __dmul_rn(t, t);
}

// Exact float64 score of one staged row by one warp: lanes run numpy's
// 8-way-unrolled accumulation chains (elements off + j + 8m, in order),
// then fold each leaf's chains in numpy's order, and lane 0 applies the
// recursion's combine tree. Bit-identical to np_pairwise.
template <bool IP, typename T>
__device__ double warp_np_score(const float* q, const T* x, int d, const Small& S, double* cbuf,
                                double* lbuf, int lane) {
    // q and x are staged skewed: leaf L's elements start SHQ * L floats (q)
    // and shx<T>() * L elements (x) after their natural offset
    const int nleaf = S.nleaf;
    const int nch = nleaf * 8;
    for (int c = lane; c < nch; c += 32) {
        const int L = c >> 3, j = c & 7;
        const int off = S.leaf_off[L], n = S.leaf_n[L];
        const float* qL = q + SHQ * L;
        const T* xL = x + shx<T>() * L;
        const int lim = n - (n % 8);
        double r = term_sm<IP, T>(qL, xL, off + j);
        for (int i = 8 + j; i < lim; i += 8) r = __dadd_rn(r, term_sm<IP, T>(qL, xL, off + i));
        cbuf[c] = r;
    }
    __syncwarp();
    for (int L = lane; L < nleaf; L += 32) {
        const double* cb = cbuf + L * 8;
        double res = __dadd_rn(__dadd_rn(__dadd_rn(cb[0], cb[1]), __dadd_rn(cb[2], cb[3])),
                               __dadd_rn(__dadd_rn(cb[4], cb[5]), __dadd_rn(cb[6], cb[7])));
        const int off = S.leaf_off[L], n = S.leaf_n[L];
        const float* qL = q + SHQ * L;
        const T* xL = x + shx<T>() * L;
        for (int i = n - (n % 8); i < n; ++i) res = __dadd_rn(res, term_sm<IP, T>(qL, xL, off + i));
        lbuf[L] = res;
    }
    __syncwarp();
    // lane 0 folds the leaves along numpy's recursion (node list in smem)
    double sc = 0.0;
    if (lane == 0) {
        const int nn = S.nnode;
        for (int j = 0; j < nn; ++j) lbuf[nleaf + j] = __dadd_rn(lbuf[S.node_a[j]], lbuf[S.node_b[j]]);
        sc = nn ? lbuf[nleaf + nn - 1] : lbuf[0];   // the root is the last node
    }
    sc = __shfl_sync(VS_FULL, sc, 0);
    return sc;
}

template <typename T>
struct Pair2;
template <>
struct Pair2<float> {
    static __device__ __forceinline__ float2 ld(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
};
template <>
struct Pair2<__nv_bfloat16> {
    static __device__ __forceinline__ float2 ld(const __nv_bfloat16* p) {
        return __bfloat1622float2(__ldg(reinterpret_cast<const __nv_bfloat162*>(p)));
    }
};

template <bool IP>
__device__ __forceinline__ double term_d(float qf, float xf) {
    const double a = (double)qf, b = (double)xf;
    if (IP) return __dmul_rn(a, b);
    const double t = __dsub_rn(a, b);
    return __dmul_rn(t, t);
}

// Exact float64 score of one row held in registers: lane (L, p) = (lane >> 2,
// lane & 3) owns chains 2p and 2p + 1 of leaf L (elements off + 2p + {0,1} +
// 8m); the leaf's 8 chains fold with two xor-shuffles in numpy's order
// ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)); lane p = 0 adds the leaf
// tail; the combine tree runs on shuffles with slot s held by lane s.
template <bool IP>
__device__ __forceinline__ double term_dd(double a, float xf) {
    const double b = (double)xf;
    if (IP) return __dmul_rn(a, b);
    const double t = __dsub_rn(a, b);
    return __dmul_rn(t, t);
}

// Exact float64 scores of TWO rows held in registers (independent chains
// interleaved for ILP; the float64 chains are latency-bound). Lane (L, p) =
// (lane >> 2, lane & 3) owns chains 2p and 2p + 1 of leaf L (elements
// off + 2p + {0,1} + 8m, numpy's accumulation order); the leaf's 8 chains fold
// with two xor-shuffles in numpy's order ((r0 + r1) + (r2 + r3)) + ((r4 + r5) +
// (r6 + r7)); lane p = 0 adds the leaf tail; the combine tree runs level by
// level on shuffles (slot s held by lane s; lane nleaf + j computes node j).
struct TreeLane {
    int na, nb, lvl, nlevels, root, nleaf;
};

template <bool IP, typename T>
__device__ __forceinline__ void warp_np_score_reg2(const double* qpd, const float2 (&xa)[16], const float2 (&xb)[16],
                                                   int M, const double* qtail, const T* xta, const T* xtb,
                                                   int ntail, const TreeLane& tl, int lane, double& oa,
                                                   double& ob) {
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    if (M > 0) {
        const double2 q = *reinterpret_cast<const double2*>(qpd);
        a0 = term_dd<IP>(q.x, xa[0].x);
        a1 = term_dd<IP>(q.y, xa[0].y);
        b0 = term_dd<IP>(q.x, xb[0].x);
        b1 = term_dd<IP>(q.y, xb[0].y);
    }
#pragma unroll
    for (int m = 1; m < 16; ++m) {
        if (m < M) {
            const double2 q = *reinterpret_cast<const double2*>(qpd + 8 * m);
            a0 = __dadd_rn(a0, term_dd<IP>(q.x, xa[m].x));
            b0 = __dadd_rn(b0, term_dd<IP>(q.x, xb[m].x));
            a1 = __dadd_rn(a1, term_dd<IP>(q.y, xa[m].y));
            b1 = __dadd_rn(b1, term_dd<IP>(q.y, xb[m].y));
        }
    }
    double va = __dadd_rn(a0, a1), vb = __dadd_rn(b0, b1);
    va = __dadd_rn(va, __shfl_xor_sync(VS_FULL, va, 1));
    vb = __dadd_rn(vb, __shfl_xor_sync(VS_FULL, vb, 1));
    va = __dadd_rn(va, __shfl_xor_sync(VS_FULL, va, 2));
    vb = __dadd_rn(vb, __shfl_xor_sync(VS_FULL, vb, 2));
    for (int i = 0; i < ntail; ++i) {
        va = __dadd_rn(va, term_dd<IP>(qtail[i], ld_elem(xta + i)));
        vb = __dadd_rn(vb, term_dd<IP>(qtail[i], ld_elem(xtb + i)));
    }
    double sa = __shfl_sync(VS_FULL, va, (lane * 4) & 31);   // lane L < nleaf: leaf L
    double sb = __shfl_sync(VS_FULL, vb, (lane * 4) & 31);
    for (int l = 0; l < tl.nlevels; ++l) {
        const double pa = __shfl_sync(VS_FULL, sa, tl.na), qa = __shfl_sync(VS_FULL, sa, tl.nb);
        const double pb = __shfl_sync(VS_FULL, sb, tl.na), qb = __shfl_sync(VS_FULL, sb, tl.nb);
        if (tl.lvl == l) {
            sa = __dadd_rn(pa, qa);
            sb = __dadd_rn(pb, qb);
        }
    }
    oa = __shfl_sync(VS_FULL, sa, tl.root);
    ob = __shfl_sync(VS_FULL, sb, tl.root);
}

// the same for ONE row (the narrow build: 64 registers at 4 CTAs/SM; two rows
// of registers spilled the row data to local memory there)
template <bool IP, typename T>
__device__ __forceinline__ double warp_np_score_reg1(const double* qpd, const float2 (&xa)[16], int M,
                                                    const double* qtail, const T* xta, int ntail,
                                                    const TreeLane& tl, int lane) {
    double a0 = 0.0, a1 = 0.0;
    if (M > 0) {
        const double2 q = *reinterpret_cast<const double2*>(qpd);
        a0 = term_dd<IP>(q.x, xa[0].x);
        a1 = term_dd<IP>(q.y, xa[0].y);
    }
#pragma unroll
    for (int m = 1; m < 16; ++m) {
        if (m < M) {
            const double2 q = *reinterpret_cast<const double2*>(qpd + 8 * m);
            a0 = __dadd_rn(a0, term_dd<IP>(q.x, xa[m].x));
            a1 = __dadd_rn(a1, term_dd<IP>(q.y, xa[m].y));
        }
    }
    double va = __dadd_rn(a0, a1);
    va = __dadd_rn(va, __shfl_xor_sync(VS_FULL, va, 1));
    va = __dadd_rn(va, __shfl_xor_sync(VS_FULL, va, 2));
    for (int i = 0; i < ntail; ++i) va = __dadd_rn(va, term_dd<IP>(qtail[i], ld_elem(xta + i)));
    double sa = __shfl_sync(VS_FULL, va, (lane * 4) & 31);
    for (int l = 0; l < tl.nlevels; ++l) {
        const double pa = __shfl_sync(VS_FULL, sa, tl.na), qa = __shfl_sync(VS_FULL, sa, tl.nb);
        if (tl.lvl == l) sa = __dadd_rn(pa, qa);
    }
    return __shfl_sync(VS_FULL, sa, tl.root);
}

// stage one row into shared memory (same element type) in the skewed leaf
// layout, coalesced; 16-byte cp.async chunks when the row size allows, so the
// copy overlaps compute. Leaves split at multiples of 8 elements, so a chunk
// never straddles two leaves.
template <typename T>
__device__ __forceinline__ void stage_row_async(const T* __restrict__ src, T* dst, int d, int lane,
                                                const unsigned char* gsk) {
    const int bytes = d * (int)sizeof(T);
    if ((bytes & 15) == 0) {
        constexpr int EPC = 16 / (int)sizeof(T);   // elements per chunk
        const char* s8 = reinterpret_cast<const char*>(src);
        const uint32_t d8 = (uint32_t)__cvta_generic_to_shared(dst);
        for (int off = lane * 16; off < bytes; off += 32 * 16) {
            const int e = off / (int)sizeof(T);
            const int sk = gsk[e / 8] * shx<T>() * (int)sizeof(T);
            (void)EPC;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d8 + off + sk), "l"(s8 + off) : "memory");
        }
    } else {
        for (int i = lane; i < d; i += 32) dst[i + gsk[i / 8] * shx<T>()] = src[i];
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
}  // namespace

#ifdef VS_RERANK_PROFILE
// per-phase cycle totals (thread 0 of every CTA), read by vs_debug_rerank_profile
__device__ unsigned long long g_rr_prof[8];
#define RR_MARK(i)                                                        \
    do {                                                                  \
        if (threadIdx.x == 0) {                                           \
            const long long t_ = clock64();                               \
            atomicAdd(&g_rr_prof[i], (unsigned long long)(t_ - rr_t));    \
            rr_t = t_;                                                    \
        }                                                                 \
    } while (0)
#else
#define RR_MARK(i) do {} while (0)
#endif

// PH: 0 the whole phase B in one kernel; 1 steps 0-2 only (live candidates ->
// survivors, their count in p.s_count): no scorer registers, so more CTAs per
// SM hide the latency-bound gather and select; 2 steps 3-5 from p.s_count
template <typename T, bool IP, bool WIDE, int PH>
__global__ void __launch_bounds__(NT, PH == 1 ? 5 : (WIDE ? 2 : 4)) k_rerank(RerankParams p) {
    constexpr int LCAP = lcap<WIDE>();
#ifdef VS_RERANK_PROFILE
    long long rr_t = clock64();
#endif
    extern __shared__ __align__(16) unsigned char smraw[];
    Small& sm = *reinterpret_cast<Small*>(smraw);
    unsigned char* u = smraw + ((sizeof(Small) + 127) & ~size_t(127));       // union region
    // chain / leaf buffers of the staged scorer (absent on the register path)
    const bool chains = !p.reg_path && PH != 1;
    double* cbuf = reinterpret_cast<double*>(u + p.ubytes);                  // [NWARP][8*MAXLEAF]
    double* lbuf = cbuf + (chains ? NWARP * 8 * MAXLEAF : 0);                // [NWARP][2*MAXLEAF]
    float* qs = reinterpret_cast<float*>(lbuf + (chains ? NWARP * 2 * MAXLEAF : 0));   // [q_stride] (skewed)
    int* cnts = reinterpret_cast<int*>(qs + (PH == 1 ? 0 : q_stride(p.d)));  // [nsub]
    unsigned* hist = reinterpret_cast<unsigned*>(cnts + ((p.cb.n_sub + 3) & ~3));   // [HBINS]
    double* qd = reinterpret_cast<double*>(hist + HBINS);                    // [q_stride] float64, skewed

    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    if (p.q_list && (int)blockIdx.x >= *p.q_count) return;   // the whole CTA: no barrier is reached
    const int64_t q = p.q_list ? (int64_t)p.q_list[blockIdx.x] : (int64_t)blockIdx.x;
    const int C = p.cb.C;
    // buffers of this query: fixed n_sub per query, or a flat range (IVF list chunks)
    const int64_t bbase = p.cb.sub_off ? p.cb.sub_off[q] : q * (int64_t)p.cb.n_sub;
    const int nsub = p.cb.sub_off ? (int)(p.cb.sub_off[q + 1] - bbase) : p.cb.n_sub;
    const int d = p.d;
    const bool warp_path = d >= 8 && d <= WARP_D_MAX;
    if (warp_path && PH != 1) {
        const int* src = reinterpret_cast<const int*>(&p.plan);
        int* dst = reinterpret_cast<int*>(static_cast<LeafPlan*>(&sm));
        for (int i = tid; i < (int)(sizeof(LeafPlan) / 4); i += NT) dst[i] = src[i];
    }
    __syncthreads();
    const float* qg = p.Q + q * (int64_t)d;
    if (PH != 1) {
        if (warp_path)
            for (int i = tid; i < d; i += NT) {
                const float v = qg[i];
                qs[i + SHQ * sm.gsk[i / 8]] = v;
                qd[i + SHQ * sm.gsk[i / 8]] = (double)v;
            }
        else
            for (int i = tid; i < d; i += NT) qs[i] = qg[i];
    }
    long long tot = 0;
    for (int s = tid; s < nsub; s += NT) {
        const int c = p.cb.cnt[bbase + s];
        cnts[s] = c;
        tot += c;
    }
    tot = block_sum_ll(tot, sm.red);  // includes __syncthreads
    const float* ckey = p.cb.key + bbase * (int64_t)C;
    const uint32_t* cpos = p.cb.pos + bbase * (int64_t)C;
    uint32_t* spos = p.s_pos + q * p.s_cap;
    uint64_t* skey = p.s_key + q * p.s_cap;
    int64_t* sid = p.s_id + q * p.s_cap;
    const uint32_t tg = p.tau_g ? p.tau_g[q] : 0xffffffffu;
    // verify mode: tau_g is the smallest local k-th key, an upper bound on the
    // global one; survivors need key <= K* + margin <= tau_g + margin
    uint32_t pre = (p.verify && tg != 0xffffffffu) ? f2o(__fadd_ru(o2f(tg), p.margin[q])) : tg;
    // external bound T: an upper bound on the k-th EXACT key of the final
    // result (distributed protocol: the k-th smallest of every shard's
    // approx-key + its own margin/2; streamed chunks: an earlier chunk's exact
    // k-th). A row of the result has exact key <= T, so approx key <= T +
    // margin/2 with THIS shard's margin (shards may differ in margin).
    const bool has_ext = p.ext_thr && f2o(p.ext_thr[q]) != f2o(__int_as_float(0x7f800000));
    const uint32_t ext_o = has_ext ? f2o(__fadd_ru(p.ext_thr[q], 0.5f * p.margin[q])) : 0xffffffffu;
    pre = min(pre, ext_o);

    int64_t ns = 0;
    if (PH == 2) {
        ns = p.s_count[q];
    } else {
        RR_MARK(0);
        float* lkey = reinterpret_cast<float*>(u);
        uint32_t* lpos = reinterpret_cast<uint32_t*>(u + LCAP * 4);
        // -1. more candidates than shared memory holds (e.g. exhaustive buffers of
        //    short splits): bound the union's k-th key from above by the k-th key
        //    of a subset — the first m keys of every buffer — and tighten the live
        //    filter to that bound + margin. The k smallest keys and every key within
        //    the margin of the k-th stay live, so the result is unchanged.
        if (tot > LCAP && tot > p.k) {
            const int m = max(1, (LCAP / 2) / max(nsub, 1));
            if (tid == 0) sm.counter = 0;
            __syncthreads();
            for (int s = w; s < nsub; s += NWARP) {
                const int cs = min(cnts[s], m);
                const float* bk = ckey + (int64_t)s * C;
                for (int j = lane; j - lane < cs; j += 32) {
                    const float kv = j < cs ? bk[j] : 0.f;
                    const bool live = j < cs && f2o(kv) <= pre;
                    const unsigned b = __ballot_sync(VS_FULL, live);
                    if (!b) continue;
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&sm.counter, __popc(b));
                    base = __shfl_sync(VS_FULL, base, 0);
                    const int slot = base + __popc(b & lanemask_lt());
                    if (live && slot < LCAP) lkey[slot] = kv;
                }
            }
            __syncthreads();
            const int nsamp = min(sm.counter, LCAP);
            __syncthreads();
            if (nsamp >= p.k) {
                const uint32_t kth_s = block_radix_kth(
                    [&](auto fn) {
                        for (int i = tid; i < nsamp; i += NT) fn(f2o(lkey[i]));
                    },
                    (unsigned)p.k, hist, sm);
                pre = min(pre, f2o(__fadd_ru(o2f(kth_s), p.margin[q])));
            }
            __syncthreads();
        }
        // 0. live candidates -> shared memory. Many short buffers (IVF: a few
        //    entries per (pair, column half)): all threads walk the flat entry
        //    index space (buffer by a search over the counts' prefix, in the
        //    histogram region), one round of loads; else one warp per buffer
        if (tid == 0) sm.counter = 0;
        const bool flat = nsub > 2 * NWARP && nsub < HBINS && tot < (long long)nsub * 24;
        if (flat && w == 0) {
            int run = 0;
            for (int s0 = 0; s0 < nsub; s0 += 32) {
                const int s = s0 + lane;
                const int c = s < nsub ? cnts[s] : 0;
                int incl = c;
    #pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(VS_FULL, incl, o);
                    if (lane >= o) incl += t;
                }
                if (s < nsub) hist[s] = (unsigned)(run + incl - c);
                run += __shfl_sync(VS_FULL, incl, 31);
            }
        }
        __syncthreads();
        if (flat) {
            const int ntot = (int)tot;
            for (int f0 = w * 32; f0 < ntot; f0 += NT) {
                const int f = f0 + lane;
                float kv = 0.f;
                uint32_t pv = 0u;
                bool live = false;
                if (f < ntot) {
                    int a = 0, b = nsub - 1;   // last buffer whose prefix <= f
                    while (a < b) {
                        const int m = (a + b + 1) >> 1;
                        if ((int)hist[m] <= f) a = m; else b = m - 1;
                    }
                    const int64_t e = (int64_t)a * C + (f - (int)hist[a]);
                    kv = ckey[e];
                    live = f2o(kv) <= pre;
                    if (live) pv = cpos[e];
                }
                const unsigned bl = __ballot_sync(VS_FULL, live);
                if (bl) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&sm.counter, __popc(bl));
                    base = __shfl_sync(VS_FULL, base, 0);
                    const int slot = base + __popc(bl & lanemask_lt());
                    if (live && slot < LCAP) {
                        lkey[slot] = kv;
                        lpos[slot] = pv;
                    }
                }
            }
        }
        for (int s = flat ? nsub : w; s < nsub; s += NWARP) {
            const int cs = cnts[s];
            const float* bk = ckey + (int64_t)s * C;
            const uint32_t* bp = cpos + (int64_t)s * C;
            for (int j0 = 0; j0 < cs; j0 += 128) {
                // four independent key loads in flight, then the positions of the live ones
                float kk[4];
                uint32_t pp[4];
                bool live[4];
    #pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int j = j0 + 32 * h + lane;
                    kk[h] = j < cs ? bk[j] : 0.f;
                }
    #pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int j = j0 + 32 * h + lane;
                    live[h] = j < cs && f2o(kk[h]) <= pre;
                    pp[h] = live[h] ? bp[j] : 0u;
                }
    #pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const unsigned b = __ballot_sync(VS_FULL, live[h]);
                    if (!b) continue;
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&sm.counter, __popc(b));
                    base = __shfl_sync(VS_FULL, base, 0);
                    const int slot = base + __popc(b & lanemask_lt());
                    if (live[h] && slot < LCAP) {
                        lkey[slot] = kk[h];
                        lpos[slot] = pp[h];
                    }
                }
            }
        }
        __syncthreads();
        const int nl = sm.counter;
        __syncthreads();
    #ifdef VS_RERANK_PROFILE
        if (tid == 0) {
            atomicAdd(&g_rr_prof[5], (unsigned long long)tot);   // candidates in the buffers
            atomicAdd(&g_rr_prof[6], (unsigned long long)nl);    // live (key <= pre)
        }
    #endif
        if (nl <= LCAP) {
            RR_MARK(1);
            // 1. k-th smallest approximate key  2. survivors (shared-memory path)
            uint32_t thr_o = 0xffffffffu;
            uint32_t kth = 0xffffffffu;
            if (!p.band_ready && nl >= p.k && (nl > p.k || p.out_kth)) {
                kth = block_radix_kth(
                    [&](auto fn) {
                        for (int i = tid; i < nl; i += NT) fn(f2o(lkey[i]));
                    },
                    (unsigned)p.k, hist, sm);
            }
            if (p.out_kth) {   // this shard's k smallest approximate keys (+inf padded)
                write_local_topk_keys(
                    [&](auto fn) {
                        for (int i = tid; i < nl; i += NT) fn(f2o(lkey[i]));
                    },
                    kth, p.k, hist, sm, 0.5f * p.margin[q], p.out_kth + q * (int64_t)p.k);
                return;
            }
            if (kth != 0xffffffffu && nl > p.k) thr_o = f2o(__fadd_ru(o2f(kth), p.margin[q]));
            thr_o = min(thr_o, ext_o);
            if (tid == 0) sm.counter = 0;
            __syncthreads();
            for (int i = tid; i < nl; i += NT) {
                if (f2o(lkey[i]) <= thr_o) {
                    const int slot = atomicAdd(&sm.counter, 1);
                    if (slot < p.s_cap) spos[slot] = lpos[i];
                }
            }
            __syncthreads();
            ns = sm.counter;
        } else {
            // global-memory path (very wide near-tie sets)
            uint32_t thr_o = 0xffffffffu;
            if (tot > p.k) {
                // nl > LCAP >= k live keys (key <= pre): their k-th smallest
                uint32_t kth = block_radix_kth(
                    [&](auto fn) {
                        for (int s = w; s < nsub; s += NWARP)
                            for (int j = lane; j < cnts[s]; j += 32) {
                                const uint32_t o = f2o(ckey[(int64_t)s * C + j]);
                                if (o <= pre) fn(o);
                            }
                    },
                    (unsigned)p.k, hist, sm);
                if (p.out_kth) {
                    write_local_topk_keys(
                        [&](auto fn) {
                            for (int s = w; s < nsub; s += NWARP)
                                for (int j = lane; j < cnts[s]; j += 32) {
                                    const uint32_t o = f2o(ckey[(int64_t)s * C + j]);
                                    if (o <= pre) fn(o);
                                }
                        },
                        kth, p.k, hist, sm, 0.5f * p.margin[q], p.out_kth + q * (int64_t)p.k);
                    return;
                }
                thr_o = f2o(__fadd_ru(o2f(kth), p.margin[q]));
            }
            thr_o = min(thr_o, ext_o);
            if (tid == 0) sm.counter = 0;
            __syncthreads();
            for (int s = w; s < nsub; s += NWARP)
                for (int j = lane; j < cnts[s]; j += 32)
                    if (f2o(ckey[(int64_t)s * C + j]) <= thr_o) {
                        const int slot = atomicAdd(&sm.counter, 1);
                        if (slot < p.s_cap) spos[slot] = cpos[(int64_t)s * C + j];
                    }
            __syncthreads();
            ns = sm.counter;
        }
        __syncthreads();
        if (ns > p.s_cap) {  // cannot re-rank all survivors: re-run with larger buffers
            if (tid == 0) p.cb.overflow[q] = 1;
            ns = p.s_cap;
        }
        if (PH == 1) {
            if (tid == 0) p.s_count[q] = (int)ns;
            return;
        }
    }
    RR_MARK(2);
    // 3. exact float64 scores (bit-identical to the reference)
    const T* rows = reinterpret_cast<const T*>(p.rows);
    if (p.reg_path) {
        // lane (L, p): chains 2p, 2p + 1 of leaf L; its query pairs in registers
        const int L = lane >> 2, pp = lane & 3;
        const bool on = L < sm.nleaf;
        const int offL = on ? sm.leaf_off[L] : 0, nL = on ? sm.leaf_n[L] : 0;
        const int M = nL / 8;
        const int ntail = ((lane & 3) == 0) ? nL - 8 * M : 0;
        const double* qdL = qd + SHQ * (on ? L : 0);   // skewed float64 staging of the query
        const double* qpd = qdL + offL + 2 * pp;
        const double* qtail = qdL + offL + 8 * M;
        TreeLane tl;
        {
            const int sj = lane - sm.nleaf;
            const bool isnode = sj >= 0 && sj < sm.nnode;
            tl.na = isnode ? sm.node_a[sj] : lane;
            tl.nb = isnode ? sm.node_b[sj] : lane;
            tl.lvl = isnode ? sm.node_lvl[sj] : -1;
            tl.nlevels = sm.nlevels;
            tl.nleaf = sm.nleaf;
            tl.root = sm.nnode ? sm.nleaf + sm.nnode - 1 : 0;
        }
        const int row_bytes = d * (int)sizeof(T);
        auto row_of = [&](int64_t idx, uint32_t& ps) -> int64_t {
            ps = spos[idx];
            return p.row_map ? p.row_map[ps] : (int64_t)ps;
        };
        auto fetch = [&](float2 (&x)[16], int64_t r) {
            const T* xg = rows + r * (int64_t)d + offL + 2 * pp;
#pragma unroll
            for (int m = 0; m < 16; ++m) x[m] = m < M ? Pair2<T>::ld(xg + 8 * m) : make_float2(0.f, 0.f);
        };
        // two rows per iteration (rows i and i + NWARP of this warp). Survivor
        // rows are random 4 KB gathers from HBM, so the warp keeps RR_PD
        // iterations (2 x RR_PD rows) of L2 prefetches ahead of its loads; the
        // row indices (a dependent load through the selection) are resolved
        // once into the union region, free between the survivor selection and
        // the top-k (measured, config 2: one iteration of lead left every
        // iteration waiting on HBM).
        auto prefetch_row = [&](int64_t r) {
            const char* base = reinterpret_cast<const char*>(rows + r * (int64_t)d);
            for (int o = lane * 128; o < row_bytes; o += 32 * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(base + o));
        };
        const int RR_PD = p.prefetch_iters;
        int64_t* ridx = reinterpret_cast<int64_t*>(u);
        uint32_t* rps = reinterpret_cast<uint32_t*>(u + (size_t)ns * 8);
        const bool staged = ns * 12 <= (int64_t)p.ubytes;   // block-uniform
        if (staged) {
            for (int64_t j = tid; j < ns; j += NT) {
                uint32_t ps;
                ridx[j] = row_of(j, ps);
                rps[j] = ps;
            }
            __syncthreads();
        }
        auto row_at = [&](int64_t j, uint32_t& ps) -> int64_t {
            if (staged) {
                ps = rps[j];
                return ridx[j];
            }
            return row_of(j, ps);
        };
        auto prefetch_iter = [&](int64_t j) {
            uint32_t ps;
            if (j < ns) prefetch_row(row_at(j, ps));
            if (j + NWARP < ns) prefetch_row(row_at(j + NWARP, ps));
        };
        if (!WIDE) {
            // one row per warp and iteration (see warp_np_score_reg1)
            for (int pd = 1; pd <= RR_PD; ++pd) {
                uint32_t ps;
                const int64_t j = w + pd * NWARP;
                if (j < ns) prefetch_row(row_at(j, ps));
            }
            for (int64_t j = w; j < ns; j += NWARP) {
                uint32_t ps;
                const int64_t r = row_at(j, ps);
                float2 xa[16];
                fetch(xa, r);
                {
                    uint32_t ps2;
                    const int64_t jn = j + (RR_PD + 1) * NWARP;
                    if (jn < ns) prefetch_row(row_at(jn, ps2));
                }
                const double sc = warp_np_score_reg1<IP, T>(qpd, xa, M, qtail, rows + r * (int64_t)d + offL + 8 * M,
                                                            ntail, tl, lane);
                if (lane == 0) {
                    skey[j] = d2o(IP ? -sc : sc);
                    sid[j] = (p.id_map ? p.id_map[ps] : r) + p.id_offset;
                }
            }
        } else {
        for (int pd = 1; pd <= RR_PD; ++pd) prefetch_iter(w + pd * 2 * NWARP);
        int64_t i = w;
        uint32_t psa = 0, psb = 0;
        int64_t ra = 0, rb = 0;
        if (i < ns) {
            ra = row_at(i, psa);
            rb = (i + NWARP < ns) ? row_at(i + NWARP, psb) : ra;
        }
        for (; i < ns; i += 2 * NWARP) {
            const int64_t i2 = i + NWARP;
            const bool hasb = i2 < ns;
            float2 xa[16], xb[16];
            fetch(xa, ra);
            fetch(xb, rb);
            // RR_PD iterations ahead -> L2; the next pair's indices
            prefetch_iter(i + (RR_PD + 1) * 2 * NWARP);
            const int64_t in = i + 2 * NWARP, in2 = in + NWARP;
            uint32_t psa_n = 0, psb_n = 0;
            int64_t ra_n = 0, rb_n = 0;
            if (in < ns) {
                ra_n = row_at(in, psa_n);
                rb_n = (in2 < ns) ? row_at(in2, psb_n) : ra_n;
            }
            double sa, sb;
            warp_np_score_reg2<IP, T>(qpd, xa, xb, M, qtail, rows + ra * (int64_t)d + offL + 8 * M,
                                      rows + rb * (int64_t)d + offL + 8 * M, ntail, tl, lane, sa, sb);
            if (lane == 0) {
                skey[i] = d2o(IP ? -sa : sa);
                sid[i] = (p.id_map ? p.id_map[psa] : ra) + p.id_offset;
                if (hasb) {
                    skey[i2] = d2o(IP ? -sb : sb);
                    sid[i2] = (p.id_map ? p.id_map[psb] : rb) + p.id_offset;
                }
            }
            ra = ra_n;
            rb = rb_n;
            psa = psa_n;
            psb = psb_n;
        }
        }
    } else if (warp_path) {
        // double-buffered: the next survivor row is staged (cp.async-free plain
        // 128-bit loads issued before scoring) while the current one is scored
        const int dpad = row_stride(d);
        T* xw0 = reinterpret_cast<T*>(u) + (size_t)w * 2 * dpad;
        T* xw1 = xw0 + dpad;
        double* cb = cbuf + w * 8 * MAXLEAF;
        double* lb = lbuf + w * 2 * MAXLEAF;
        int64_t i = w;
        int64_t r_cur = 0;
        uint32_t ps_cur = 0;
        if (i < ns) {
            ps_cur = spos[i];
            r_cur = p.row_map ? p.row_map[ps_cur] : (int64_t)ps_cur;
            stage_row_async<T>(rows + r_cur * (int64_t)d, xw0, d, lane, sm.gsk);
        }
        for (int buf = 0; i < ns; i += NWARP, buf ^= 1) {
            T* cur = buf ? xw1 : xw0;
            T* nxt = buf ? xw0 : xw1;
            const int64_t inext = i + NWARP;
            uint32_t ps_n = 0;
            int64_t r_n = 0;
            if (inext < ns) {
                ps_n = spos[inext];
                r_n = p.row_map ? p.row_map[ps_n] : (int64_t)ps_n;
                stage_row_async<T>(rows + r_n * (int64_t)d, nxt, d, lane, sm.gsk);
                async_wait_prev();   // the current row has landed, the next is in flight
            } else {
                async_wait_all();
            }
            __syncwarp();
            const double sc = warp_np_score<IP, T>(qs, cur, d, sm, cb, lb, lane);
            if (lane == 0) {
                skey[i] = d2o(IP ? -sc : sc);
                sid[i] = (p.id_map ? p.id_map[ps_cur] : r_cur) + p.id_offset;
            }
            __syncwarp();
            ps_cur = ps_n;
            r_cur = r_n;
        }
    } else {
        for (int64_t i = tid; i < ns; i += NT) {
            const uint32_t ps = spos[i];
            const int64_t r = p.row_map ? p.row_map[ps] : (int64_t)ps;
            const double sc = np_pairwise<T, IP>(qs, rows + r * (int64_t)d, d);
            skey[i] = d2o(IP ? -sc : sc);
            sid[i] = (p.id_map ? p.id_map[ps] : r) + p.id_offset;
        }
    }
    __syncthreads();
    if (tid == 0 && p.n_survivors) atomicAdd(p.n_survivors, (unsigned long long)ns);
    RR_MARK(3);
    // 4. exact tie-rule top-k
    block_topk_exact(skey, sid, ns, p.k, sm, u, IP, q, p.out_ids, p.out_dist, p.out_ids32, p.out_count);
    RR_MARK(4);
    // 5. verification of the local-top-k pass: every dropped candidate e had
    //    approx key > tau_g, hence exact key > tau_g - margin/2; the result is
    //    exact iff the k-th exact key + margin/2 < tau_g. Otherwise re-run.
    if ((p.verify || p.out_bound) && w == 0) {
        double qq = 0.0;
        if (!IP) {
            for (int i = lane; i < d; i += 32) {
                const double a = (double)qg[i];
                qq = fma(a, a, qq);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) qq += __shfl_xor_sync(VS_FULL, qq, o);
        }
        if (lane == 0) {
            const bool has_bound = p.verify && tg != 0xffffffffu;
            const double bound = has_bound ? (double)o2f(tg) - 0.5 * (double)p.margin[q] : 0.0;
            const double slack = fabs(bound) * 1e-6 + 1e-12;
            if (p.out_bound) {
                // deferred (distributed) check, in key space with ||q||^2 restored:
                // every dropped candidate has exact key > this value
                p.out_bound[q] = has_bound ? bound - slack + (IP ? 0.0 : qq * (1.0 - 1e-12))
                                           : __longlong_as_double(0x7ff0000000000000ll);
            } else if (has_bound) {
                const int keff = (int)min((int64_t)p.k, ns);
                const uint64_t* sk = reinterpret_cast<const uint64_t*>(u);  // sorted keys left by the top-k
                double kth = keff > 0 ? o2d(sk[keff - 1]) : 0.0;             // exact key (-score for IP)
                if (!IP) kth -= qq * (1.0 + 1e-12);  // approx keys omit ||q||^2
                // an external bound T (earlier chunks' k-th) at or below every
                // dropped candidate's exact key also settles it: none can enter
                const bool settled = p.ext_thr && (double)p.ext_thr[q] <= bound - slack;
                if (!settled && (keff < p.k || !(kth < bound - slack))) p.cb.overflow[q] = 1;
            }
        }
    }
}

// IVF coarse quantizer with dense keys (tc_dense_keys): per query, the k-th
// smallest key K* and every column with key <= K* + margin land in a single
// candidate buffer (the margin band: exact by construction);
// k_rerank then scores them exactly. Rows of up to kDenseCache keys are cached
// in shared memory. The k-th key comes from a range-adaptive radix select:
// the first pass bins the row's actual key range [min, max] into 2048 bins
// (a query's centroid keys share one or two exponents, so the top bits of the
// raw key would put all 16k keys into a handful of bins and serialise the
// histogram atomics), each later pass splits the chosen bin the same way.
constexpr int kDenseCache = 16384;
constexpr int DS_NT = 512;
constexpr int DS_KPT = kDenseCache / DS_NT;     // keys per thread of a cached row
constexpr int DS_CAND = 2048;                   // band candidates held in shared memory

struct DsShared {
    unsigned red_lo[DS_NT / 32], red_hi[DS_NT / 32], wtot[DS_NT / 32];
    int sel_bin, counter, ovf;
    unsigned sel_below;
};

// kk-th smallest (1 <= kk <= count) of the orderable keys `foreach` visits, by a
// range-adaptive radix select: each pass bins the current key range into <=
// HBINS bins and narrows to the bin holding the kk-th key
template <class ForEach>
__device__ uint32_t ds_radix_kth(ForEach foreach, unsigned kk, unsigned* hist, DsShared& S) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    constexpr int NWD = DS_NT / 32;
    uint32_t lo = 0xffffffffu, hi = 0u;
    foreach([&](uint32_t u) {
        lo = min(lo, u);
        hi = max(hi, u);
    });
    lo = __reduce_min_sync(VS_FULL, lo);
    hi = __reduce_max_sync(VS_FULL, hi);
    if (lane == 0) {
        S.red_lo[w] = lo;
        S.red_hi[w] = hi;
    }
    __syncthreads();
    uint32_t base = S.red_lo[0], top = S.red_hi[0];
#pragma unroll
    for (int i = 1; i < NWD; ++i) {
        base = min(base, S.red_lo[i]);
        top = max(top, S.red_hi[i]);
    }
    uint32_t range = top - base;
    __syncthreads();
#pragma unroll 1
    while (range > 0) {
        const int shift = max(0, 32 - __clz(range) - 11);
        const int nb = (int)(range >> shift) + 1;
        for (int i = tid; i < nb; i += DS_NT) hist[i] = 0u;
        __syncthreads();
        foreach([&](uint32_t u) {
            const uint32_t t = u - base;
            if (u >= base && t <= range) atomicAdd(&hist[t >> shift], 1u);
        });
        __syncthreads();
        const int per = (nb + DS_NT - 1) / DS_NT;
        unsigned loc = 0;
        for (int b = 0; b < per; ++b) {
            const int bi = tid * per + b;
            loc += bi < nb ? hist[bi] : 0u;
        }
        unsigned incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(VS_FULL, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) S.wtot[w] = incl;
        __syncthreads();
        unsigned excl = incl - loc;
        for (int i = 0; i < w; ++i) excl += S.wtot[i];
        if (excl < kk && kk <= excl + loc) {
            unsigned c = excl;
            for (int b = 0; b < per; ++b) {
                const int bi = tid * per + b;
                const unsigned h = bi < nb ? hist[bi] : 0u;
                if (c + h >= kk) {
                    S.sel_bin = bi;
                    S.sel_below = c;
                    break;
                }
                c += h;
            }
        }
        __syncthreads();
        kk -= S.sel_below;
        const uint32_t off = (uint32_t)S.sel_bin << shift;
        base += off;
        range = min(range - off, shift ? (1u << shift) - 1u : 0u);
        __syncthreads();
    }
    return base;
}

// IVF coarse quantizer with dense keys (tc_dense_keys): per query, the kk-th
// smallest key K* and every column with key <= K* + margin land in a single
// candidate buffer (the margin band: exact by construction).
// A cached row (<= 16384 keys) is selected without touching every key more
// than twice: each of the 512 threads holds 32 keys in registers; the kk-th
// smallest of the 512 per-thread minima is an upper bound U >= K* (kk keys
// lie at or below it) and in expectation barely above K*, so the keys <= U +
// margin (a few more than the band) are compacted into shared memory and the
// exact K* and band are taken there. Longer rows, or an unlucky U, fall back
// to a range-adaptive radix select over the whole row.
__global__ void __launch_bounds__(DS_NT) k_dense_select(const float* __restrict__ keys, int64_t ncols, int k,
                                                        const float* __restrict__ margin, CandBuf cb) {
    extern __shared__ __align__(16) unsigned char smraw[];
    unsigned* hist = reinterpret_cast<unsigned*>(smraw);           // [HBINS]
    uint32_t* cand = hist + HBINS;                                 // [DS_CAND] band candidates (orderable)
    uint32_t* cpos = cand + DS_CAND;                               // [DS_CAND] their columns
    uint32_t* tmin = cpos + DS_CAND;                               // [DS_NT]
    __shared__ DsShared S;
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t q = blockIdx.x;
    const float* row = keys + q * ncols;
    const int n = (int)ncols;
    const unsigned kk = (unsigned)min(k, n);
    const float mq = margin[q];
    const int C = cb.C;
    float* bk = cb.key + q * (int64_t)C;
    uint32_t* bp = cb.pos + q * (int64_t)C;
    if (tid == 0) {
        S.counter = 0;
        S.ovf = 0;
    }
    // thread t holds columns t + 512 j (j < 32)
    uint32_t kr[DS_KPT];
    const bool small = n <= kDenseCache && kk <= DS_NT;
    uint32_t mn = 0xffffffffu;
    if (small) {
#pragma unroll
        for (int j = 0; j < DS_KPT; ++j) {
            const int i = tid + j * DS_NT;
            kr[j] = i < n ? f2o(__ldcs(row + i)) : 0xffffffffu;
        }
#pragma unroll
        for (int j = 0; j < DS_KPT; ++j) mn = min(mn, kr[j]);
        tmin[tid] = mn;
    }
    __syncthreads();
    uint32_t thr;   // final band: keys <= thr
    bool done = false;
    if (small) {
        // U = kk-th smallest per-thread minimum (>= K*); candidates <= U + margin
        const uint32_t U = ds_radix_kth(
            [&](auto fn) {
                if (tid < DS_NT) fn(tmin[tid]);
            },
            kk, hist, S);
        const uint32_t thr_u = f2o(__fadd_ru(o2f(U), mq));
#pragma unroll
        for (int j = 0; j < DS_KPT; ++j) {
            const bool live = kr[j] <= thr_u;
            const unsigned b = __ballot_sync(VS_FULL, live);
            if (!b) continue;
            int bs = 0;
            if (lane == 0) bs = atomicAdd(&S.counter, __popc(b));
            bs = __shfl_sync(VS_FULL, bs, 0);
            const int slot = bs + __popc(b & lanemask_lt());
            if (live && slot < DS_CAND) {
                cand[slot] = kr[j];
                cpos[slot] = (uint32_t)(tid + j * DS_NT);
            }
        }
        __syncthreads();
        const int nc = S.counter;
        if (nc <= DS_CAND) {   // block-uniform
            const uint32_t kth = ds_radix_kth(
                [&](auto fn) {
                    for (int i = tid; i < nc; i += DS_NT) fn(cand[i]);
                },
                kk, hist, S);
            thr = f2o(__fadd_ru(o2f(kth), mq));
            if (tid == 0) S.counter = 0;
            __syncthreads();
            for (int i0 = 0; i0 < nc; i0 += DS_NT) {
                const int i = i0 + tid;
                const bool live = i < nc && cand[i] <= thr;
                const unsigned b = __ballot_sync(VS_FULL, live);
                if (!b) continue;
                int bs = 0;
                if (lane == 0) bs = atomicAdd(&S.counter, __popc(b));
                bs = __shfl_sync(VS_FULL, bs, 0);
                const int slot = bs + __popc(b & lanemask_lt());
                if (live && slot < C) {
                    bk[slot] = o2f(cand[i]);
                    bp[slot] = cpos[i];
                }
            }
            done = true;
        }
        __syncthreads();
        if (tid == 0 && !done) S.counter = 0;
        __syncthreads();
    }
    if (!done) {
        // whole-row radix select
        const uint32_t kth = ds_radix_kth(
            [&](auto fn) {
                for (int i = tid; i < n; i += DS_NT) fn(f2o(row[i]));
            },
            kk, hist, S);
        thr = f2o(__fadd_ru(o2f(kth), mq));
        if (tid == 0) S.counter = 0;
        __syncthreads();
        for (int i0 = 0; i0 < n; i0 += DS_NT) {
            const int i = i0 + tid;
            const uint32_t u = i < n ? f2o(row[i]) : 0xffffffffu;
            const bool live = i < n && u <= thr;
            const unsigned b = __ballot_sync(VS_FULL, live);
            if (!b) continue;
            int bs = 0;
            if (lane == 0) bs = atomicAdd(&S.counter, __popc(b));
            bs = __shfl_sync(VS_FULL, bs, 0);
            const int slot = bs + __popc(b & lanemask_lt());
            if (live && slot < C) {
                bk[slot] = o2f(u);
                bp[slot] = (uint32_t)i;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        cb.cnt[q] = min(S.counter, C);
        if (S.counter > C) cb.overflow[q] = 1;
    }
}

cudaError_t launch_dense_select(const float* keys, int64_t nq, int64_t ncols, int k, const float* margin,
                                const CandBuf& cb, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const size_t smem = (size_t)HBINS * 4 + (size_t)DS_CAND * 8 + (size_t)DS_NT * 4;
    cudaError_t e = cudaFuncSetAttribute(k_dense_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_dense_select<<<(unsigned)nq, DS_NT, smem, s>>>(keys, ncols, k, margin, cb);
    return cudaGetLastError();
}

// IVF coarse quantizer, dense keys with per-chunk minima (MODE 3 epilogue:
// mins[q][c] = min key of columns 32c..32c+31). One warp per query:
//   1. U = kk-th smallest chunk minimum: kk columns have key <= U, so the
//      kk-th smallest key K* <= U;
//   2. only chunks whose minimum is <= U + margin can hold a key <= U + margin
//      (typically ~kk of the 512 chunks of 16,384 centroids): their keys are
//      read (one coalesced 128-byte load per chunk) and those <= U + margin
//      kept in shared memory;
//   3. K* = kk-th smallest of those, band = keys <= K* + margin (<= U + margin,
//      so all of them were kept): the same margin band as k_dense_select
//      (exact by construction), from ~4 % of the key bytes.
// A candidate overflow falls back to a bitwise search over the whole row.
namespace {
constexpr int CS_WARPS = 4;
constexpr int CS_MAXCH = 1024;   // chunks per row (ncols <= 32768)
constexpr int CS_CAND = 512;     // keys <= U + margin held per query

// kk-th smallest (1-based, kk <= n) of the orderable values v[0..n), one warp;
// bits above the highest bit where lo and hi differ are common to every value
__device__ __forceinline__ uint32_t warp_kth(const uint32_t* v, int n, unsigned kk, uint32_t lo, uint32_t hi,
                                             int lane) {
    const uint32_t diff = lo ^ hi;
    if (!diff) return lo;
    const int top = 31 - __clz(diff);
    uint32_t res = lo & ~((top == 31 ? 0u : (2u << top)) - 1u);
#pragma unroll 1
    for (int b = top; b >= 0; --b) {
        const uint32_t t = res | (1u << b);
        unsigned c = 0;
        for (int i = lane; i < n; i += 32) c += v[i] < t ? 1u : 0u;
        c = __reduce_add_sync(VS_FULL, c);
        if (c < kk) res = t;
    }
    return res;
}
}  // namespace

__global__ void __launch_bounds__(CS_WARPS * 32) k_coarse_select(const float* __restrict__ keys,
                                                                 const float* __restrict__ mins, int64_t nq,
                                                                 int64_t ncols, int k,
                                                                 const float* __restrict__ margin, CandBuf cb) {
    __shared__ uint32_t s_min[CS_WARPS][CS_MAXCH];
    __shared__ uint16_t s_ch[CS_WARPS][CS_MAXCH];
    __shared__ uint32_t s_ck[CS_WARPS][CS_CAND];
    __shared__ uint32_t s_cp[CS_WARPS][CS_CAND];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.x * CS_WARPS + w;
    if (q >= nq) return;   // warp-uniform; no block barriers below
    const int n = (int)ncols;
    const int nch = (n + 31) >> 5;
    const unsigned kk = (unsigned)min(k, n);
    const float* row = keys + q * ncols;
    const float* mrow = mins + q * (int64_t)nch;
    const float mq = margin[q];
    uint32_t* vm = s_min[w];
    uint16_t* ch = s_ch[w];
    uint32_t* ck = s_ck[w];
    uint32_t* cp = s_cp[w];
    // 1. chunk minima
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (int i = lane; i < nch; i += 32) {
        const uint32_t u = f2o(__ldcs(mrow + i));
        vm[i] = u;
        lo = min(lo, u);
        hi = max(hi, u);
    }
    lo = __reduce_min_sync(VS_FULL, lo);
    hi = __reduce_max_sync(VS_FULL, hi);
    __syncwarp();
    const uint32_t U = warp_kth(vm, nch, kk, lo, hi, lane);
    const uint32_t thr_u = f2o(__fadd_ru(o2f(U), mq));
    // 2. chunks that can hold a key <= U + margin
    int nc = 0;
    for (int i0 = 0; i0 < nch; i0 += 32) {
        const int i = i0 + lane;
        const bool live = i < nch && vm[i] <= thr_u;
        const unsigned b = __ballot_sync(VS_FULL, live);
        if (live) ch[nc + __popc(b & lanemask_lt())] = (uint16_t)i;
        nc += __popc(b);
    }
    __syncwarp();
    // 3. their keys <= U + margin (four chunk loads in flight)
    int ncand = 0;
    bool ovf = false;
    uint32_t clo = 0xffffffffu, chi = 0u;
    for (int j0 = 0; j0 < nc && !ovf; j0 += 4) {
        uint32_t u[4];
        int col[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            col[h] = j0 + h < nc ? (int)ch[j0 + h] * 32 + lane : n;
            u[h] = col[h] < n ? f2o(__ldcs(row + col[h])) : 0xffffffffu;
        }
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const bool live = col[h] < n && u[h] <= thr_u;
            const unsigned b = __ballot_sync(VS_FULL, live);
            if (ncand + __popc(b) > CS_CAND) {
                ovf = true;
                break;
            }
            if (live) {
                const int slot = ncand + __popc(b & lanemask_lt());
                ck[slot] = u[h];
                cp[slot] = (uint32_t)col[h];
                clo = min(clo, u[h]);
                chi = max(chi, u[h]);
            }
            ncand += __popc(b);
        }
    }
    float* bk = cb.key + q * (int64_t)cb.C;
    uint32_t* bp = cb.pos + q * (int64_t)cb.C;
    int cnt = 0;
    if (!ovf) {
        __syncwarp();
        clo = __reduce_min_sync(VS_FULL, clo);
        chi = __reduce_max_sync(VS_FULL, chi);
        const uint32_t kth = warp_kth(ck, ncand, kk, clo, chi, lane);
        const uint32_t thr = f2o(__fadd_ru(o2f(kth), mq));
        for (int i0 = 0; i0 < ncand; i0 += 32) {
            const int i = i0 + lane;
            const bool live = i < ncand && ck[i] <= thr;
            const unsigned b = __ballot_sync(VS_FULL, live);
            const int slot = cnt + __popc(b & lanemask_lt());
            if (live && slot < cb.C) {
                bk[slot] = o2f(ck[i]);
                bp[slot] = cp[i];
            }
            cnt += __popc(b);
        }
    } else {
        // rare: more than CS_CAND keys within the margin of U; the whole row
        // from global memory (bitwise search for K*, then the band)
        uint32_t glo = 0xffffffffu, ghi = 0u;
        for (int i = lane; i < n; i += 32) {
            const uint32_t u = f2o(row[i]);
            glo = min(glo, u);
            ghi = max(ghi, u);
        }
        glo = __reduce_min_sync(VS_FULL, glo);
        ghi = __reduce_max_sync(VS_FULL, ghi);
        uint32_t res = glo;
        if (glo != ghi) {
            const int top = 31 - __clz(glo ^ ghi);
            res = glo & ~((top == 31 ? 0u : (2u << top)) - 1u);
            for (int b = top; b >= 0; --b) {
                const uint32_t t = res | (1u << b);
                unsigned c = 0;
                for (int i = lane; i < n; i += 32) c += f2o(row[i]) < t ? 1u : 0u;
                c = __reduce_add_sync(VS_FULL, c);
                if (c < kk) res = t;
            }
        }
        const uint32_t thr = f2o(__fadd_ru(o2f(res), mq));
        for (int i0 = 0; i0 < n; i0 += 32) {
            const int i = i0 + lane;
            const uint32_t u = i < n ? f2o(row[i]) : 0xffffffffu;
            const bool live = i < n && u <= thr;
            const unsigned b = __ballot_sync(VS_FULL, live);
            const int slot = cnt + __popc(b & lanemask_lt());
            if (live && slot < cb.C) {
                bk[slot] = o2f(u);
                bp[slot] = (uint32_t)i;
            }
            cnt += __popc(b);
        }
    }
    if (lane == 0) {
        cb.cnt[q] = min(cnt, cb.C);
        if (cnt > cb.C) cb.overflow[q] = 1;
    }
}

bool coarse_select_ok(int64_t ncols, int k) {
    const int64_t nch = (ncols + 31) / 32;
    return nch <= CS_MAXCH && k >= 1 && k <= nch && k <= CS_CAND / 4;
}

cudaError_t launch_coarse_select(const float* keys, const float* mins, int64_t nq, int64_t ncols, int k,
                                 const float* margin, const CandBuf& cb, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    k_coarse_select<<<(unsigned)((nq + CS_WARPS - 1) / CS_WARPS), CS_WARPS * 32, 0, s>>>(keys, mins, nq, ncols, k,
                                                                                        margin, cb);
    return cudaGetLastError();
}

// fp32 refinement of a margin band (IVF coarse quantizer): every buffer entry's
// key becomes the fp32 squared distance sum (q - x)^2, whose error is within
// the SIMT margin eps_simt (vs_capi.cu) - ~10x tighter than the bf16 band.
// The band contains the exact top-k (ties included), so the k-th fp32 key K32
// of the band + that margin again keeps every exact top-k row: phase B then
// scores ~k rows in float64 instead of the whole bf16 band.
__global__ void __launch_bounds__(256) k_refine32(CandBuf cb, const float* __restrict__ Q, int d,
                                                  const float* __restrict__ X) {
    extern __shared__ __align__(16) float qsh[];
    const int64_t q = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < d; i += blockDim.x) qsh[i] = Q[q * d + i];
    __syncthreads();
    const int cnt = cb.cnt[q];
    float* bk = cb.key + q * (int64_t)cb.C;
    const uint32_t* bp = cb.pos + q * (int64_t)cb.C;
    const bool v4 = (d & 3) == 0;
    for (int i = w; i < cnt; i += (int)(blockDim.x >> 5)) {
        const float* x = X + (int64_t)bp[i] * d;
        float acc = 0.f;
        if (v4) {
            for (int e = lane * 4; e < d; e += 128) {
                const float4 xv = __ldg(reinterpret_cast<const float4*>(x + e));
                const float4 qv = *reinterpret_cast<const float4*>(qsh + e);
                float t;
                t = qv.x - xv.x; acc = fmaf(t, t, acc);
                t = qv.y - xv.y; acc = fmaf(t, t, acc);
                t = qv.z - xv.z; acc = fmaf(t, t, acc);
                t = qv.w - xv.w; acc = fmaf(t, t, acc);
            }
        } else {
            for (int e = lane; e < d; e += 32) {
                const float t = qsh[e] - __ldg(x + e);
                acc = fmaf(t, t, acc);
            }
        }
        acc = warp_sumf(acc);
        if (lane == 0) bk[i] = acc;
    }
}

cudaError_t launch_refine32(const CandBuf& cb, int64_t nq, const float* Q, int d, const float* X, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const size_t smem = (size_t)d * 4;
    cudaError_t e = cudaFuncSetAttribute(k_refine32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_refine32<<<(unsigned)nq, 256, smem, s>>>(cb, Q, d, X);
    return cudaGetLastError();
}


// k-th smallest of the union of G sorted key lists per query (distributed
// protocol: the exact global k-th approximate key from every shard's local
// top-k keys): [G][nq][k] -> [nq]
__global__ void __launch_bounds__(NT) k_union_kth(const float* __restrict__ keys, int G, int64_t nq, int k,
                                                  float* __restrict__ out) {
    extern __shared__ unsigned ukeys[];
    const int64_t q = blockIdx.x;
    const int n = G * k;
    int P = 1;
    while (P < n) P <<= 1;
    for (int i = threadIdx.x; i < P; i += NT)
        ukeys[i] = i < n ? f2o(keys[((int64_t)(i / k) * nq + q) * k + (i % k)]) : 0xffffffffu;
    __syncthreads();
    bitonic_sort_u32(ukeys, P);
    if (threadIdx.x == 0) out[q] = o2f(ukeys[k - 1]);
}

// ---- phase B for small k: one warp per query -----------------------------------------------
// The IVF probes (k = nprobe), IVF lists and small exhaustive searches have
// a few dozen to a few hundred candidates and ~k survivors per query: the
// 256-thread CTA of k_rerank spent most of its time in barriers of its
// radix passes and bitonic sort. Here a warp does the whole query with warp
// primitives only: candidates -> shared memory (lane per buffer), k-th key
// by a bitwise search (warp_kth), survivors, exact float64 scores (query
// elements in registers, numpy's order as warp_np_score_reg1), a warp
// bitonic sort under the tie rule, output. Queries whose candidates or
// survivors exceed the warp's capacity are listed for the CTA kernel.
namespace {
constexpr int WW = 4;          // warps (queries) per CTA
constexpr int WS = 128;        // survivors per warp (sort capacity)

// WL: candidates per warp
template <int WL>
struct WarpSmem {
    uint32_t ck[WW][WL];       // orderable approximate keys
    uint32_t cp[WW][WL];       // positions
    uint64_t sk[WW][WS];       // orderable exact keys
    int64_t si[WW][WS];        // output ids
    int pref[WW][65];          // buffer count prefix (<= 64 buffers)
};

// exact float64 score of one register-held row against register-held query
// elements (lane (L, p): elements off_L + 2p + {0, 1} + 8m of leaf L)
template <bool IP>
__device__ __forceinline__ double warp_score_regq(const float2 (&qv)[16], const float2 (&xa)[16], int M,
                                                  const float* qt, const float* xt, int ntail, const TreeLane& tl,
                                                  int lane) {
    double a0 = 0.0, a1 = 0.0;
    if (M > 0) {
        a0 = term_d<IP>(qv[0].x, xa[0].x);
        a1 = term_d<IP>(qv[0].y, xa[0].y);
    }
#pragma unroll
    for (int m = 1; m < 16; ++m) {
        if (m < M) {
            a0 = __dadd_rn(a0, term_d<IP>(qv[m].x, xa[m].x));
            a1 = __dadd_rn(a1, term_d<IP>(qv[m].y, xa[m].y));
        }
    }
    double va = __dadd_rn(a0, a1);
    va = __dadd_rn(va, __shfl_xor_sync(VS_FULL, va, 1));
    va = __dadd_rn(va, __shfl_xor_sync(VS_FULL, va, 2));
    for (int i = 0; i < ntail; ++i) va = __dadd_rn(va, term_d<IP>(qt[i], xt[i]));
    double sa = __shfl_sync(VS_FULL, va, (lane * 4) & 31);
    for (int l = 0; l < tl.nlevels; ++l) {
        const double pa = __shfl_sync(VS_FULL, sa, tl.na), qa = __shfl_sync(VS_FULL, sa, tl.nb);
        if (tl.lvl == l) sa = __dadd_rn(pa, qa);
    }
    return __shfl_sync(VS_FULL, sa, tl.root);
}
}  // namespace

template <typename T, bool IP, int WL>
__global__ void __launch_bounds__(WW * 32, 4) k_rerank_warp(RerankParams p, int32_t* fb_list, int32_t* fb_count) {
    __shared__ LeafPlan plan;
    extern __shared__ __align__(16) unsigned char wsm[];
    WarpSmem<WL>& S = *reinterpret_cast<WarpSmem<WL>*>(wsm);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    {
        const int* src = reinterpret_cast<const int*>(&p.plan);
        int* dst = reinterpret_cast<int*>(&plan);
        for (int i = threadIdx.x; i < (int)(sizeof(LeafPlan) / 4); i += WW * 32) dst[i] = src[i];
    }
    __syncthreads();
    const int64_t q = (int64_t)blockIdx.x * WW + w;
    if (q >= p.nq) return;   // warp-uniform; no block barriers below
    const int d = p.d, C = p.cb.C;
    uint32_t* ck = S.ck[w];
    uint32_t* cp = S.cp[w];
    // 1. live candidates: the buffers' counts (a lane per buffer, <= 64 of
    //    them), a warp prefix sum, then every lane walks flat entry indices
    //    (f -> buffer by a search over the prefix), four loads in flight
    const int64_t bbase = p.cb.sub_off ? p.cb.sub_off[q] : q * (int64_t)p.cb.n_sub;
    const int nsub = p.cb.sub_off ? (int)(p.cb.sub_off[q + 1] - bbase) : p.cb.n_sub;
    const uint32_t pre = p.tau_g ? p.tau_g[q] : 0xffffffffu;
    int* pref = S.pref[w];   // [nsub + 1] exclusive prefix of the counts
    int tot = 0;
    for (int s0 = 0; s0 < nsub; s0 += 32) {
        const int s = s0 + lane;
        const int c = s < nsub ? p.cb.cnt[bbase + s] : 0;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(VS_FULL, incl, o);
            if (lane >= o) incl += t;
        }
        if (s < nsub) pref[s] = tot + incl - c;
        tot += __shfl_sync(VS_FULL, incl, 31);
    }
    if (lane == 0) pref[nsub] = tot;
    __syncwarp();
    bool ovf = false;
    uint32_t lo = 0xffffffffu, hi = 0u;
    int nl = 0;
    for (int f0 = 0; f0 < tot; f0 += 32) {
        const int f = f0 + lane;
        uint32_t o = 0xffffffffu, ps = 0u;
        if (f < tot) {
            int a = 0, b = nsub - 1;   // last buffer with pref <= f
            while (a < b) {
                const int m = (a + b + 1) >> 1;
                if (pref[m] <= f) a = m; else b = m - 1;
            }
            const int64_t e = (bbase + a) * (int64_t)C + (f - pref[a]);
            o = f2o(p.cb.key[e]);
            if (o <= pre) ps = p.cb.pos[e];
        }
        const bool live = f < tot && o <= pre;
        const unsigned bl = __ballot_sync(VS_FULL, live);
        const int slot = nl + __popc(bl & lanemask_lt());
        if (live && slot < WL) {
            ck[slot] = o;
            cp[slot] = ps;
            lo = min(lo, o);
            hi = max(hi, o);
        }
        nl += __popc(bl);
    }
    __syncwarp();
    ovf = nl > WL;
    int ns = 0;
    if (!ovf) {
        // 2. survivors: keys <= k-th key + margin (all of them for a ready band)
        uint32_t thr = 0xffffffffu;
        if (!p.band_ready && nl > p.k) {
            lo = __reduce_min_sync(VS_FULL, lo);
            hi = __reduce_max_sync(VS_FULL, hi);
            const uint32_t kth = warp_kth(ck, nl, (unsigned)p.k, lo, hi, lane);
            thr = f2o(__fadd_ru(o2f(kth), p.margin[q]));
        }
        for (int i0 = 0; i0 < nl; i0 += 32) {
            const int i = i0 + lane;
            const bool live = i < nl && ck[i] <= thr;
            const unsigned b = __ballot_sync(VS_FULL, live);
            const int slot = ns + __popc(b & lanemask_lt());
            // compaction in place: slot <= i, and every lane reads before any writes
            const uint32_t pos = live ? cp[i] : 0u;
            __syncwarp();
            if (live) cp[slot] = pos;
            __syncwarp();
            ns += __popc(b);
        }
        ovf = ns > WS;
    }
    if (ovf) {   // the CTA kernel takes this query
        if (lane == 0) fb_list[atomicAdd(fb_count, 1)] = (int32_t)q;
        return;
    }
    // 3. exact float64 scores; the query's elements of this lane in registers
    const int L = lane >> 2, pp = lane & 3;
    const bool on = L < plan.nleaf;
    const int offL = on ? plan.leaf_off[L] : 0, nL = on ? plan.leaf_n[L] : 0;
    const int M = nL / 8;
    const int ntail = pp == 0 ? nL - 8 * M : 0;
    TreeLane tl;
    {
        const int sj = lane - plan.nleaf;
        const bool isnode = sj >= 0 && sj < plan.nnode;
        tl.na = isnode ? plan.node_a[sj] : lane;
        tl.nb = isnode ? plan.node_b[sj] : lane;
        tl.lvl = isnode ? plan.node_lvl[sj] : -1;
        tl.nlevels = plan.nlevels;
        tl.nleaf = plan.nleaf;
        tl.root = plan.nnode ? plan.nleaf + plan.nnode - 1 : 0;
    }
    const float* qg = p.Q + q * (int64_t)d + offL + 2 * pp;
    float2 qv[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) qv[m] = m < M ? *reinterpret_cast<const float2*>(qg + 8 * m) : make_float2(0.f, 0.f);
    float qt[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) qt[i] = i < ntail ? p.Q[q * (int64_t)d + offL + 8 * M + i] : 0.f;
    const T* rows = reinterpret_cast<const T*>(p.rows);
    const int row_bytes = d * (int)sizeof(T);
    auto row_of = [&](int j) -> int64_t {
        const uint32_t ps = cp[j];
        return p.row_map ? p.row_map[ps] : (int64_t)ps;
    };
    auto prefetch_row = [&](int64_t r) {
        const char* base = reinterpret_cast<const char*>(rows + r * (int64_t)d);
        for (int o = lane * 128; o < row_bytes; o += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + o));
    };
    const int PD = max(0, p.prefetch_iters - 1);   // rows of L2 prefetch lead (default 3)
    for (int j = 1; j <= PD && j < ns; ++j) prefetch_row(row_of(j));
    uint64_t* sk = S.sk[w];
    int64_t* si = S.si[w];
    for (int j = 0; j < ns; ++j) {
        const uint32_t ps = cp[j];
        const int64_t r = p.row_map ? p.row_map[ps] : (int64_t)ps;
        const T* xg = rows + r * (int64_t)d + offL + 2 * pp;
        float2 xa[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) xa[m] = m < M ? Pair2<T>::ld(xg + 8 * m) : make_float2(0.f, 0.f);
        if (j + PD + 1 < ns) prefetch_row(row_of(j + PD + 1));
        float xt[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) xt[i] = i < ntail ? ld_elem(rows + r * (int64_t)d + offL + 8 * M + i) : 0.f;
        const double sc = warp_score_regq<IP>(qv, xa, M, qt, xt, ntail, tl, lane);
        if (lane == 0) {
            sk[j] = d2o(IP ? -sc : sc);
            si[j] = (p.id_map ? p.id_map[ps] : r) + p.id_offset;
        }
    }
    __syncwarp();
    // 4. tie-rule top-k: warp bitonic sort of (exact key, id)
    int P = 1;
    while (P < ns) P <<= 1;
    for (int i = ns + lane; i < P; i += 32) {
        sk[i] = ~0ull;
        si[i] = 0x7fffffffffffffffll;
    }
    __syncwarp();
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = lane; i < P / 2; i += 32) {
                const int lo_i = 2 * i - (i & (stride - 1));
                const int hi_i = lo_i + stride;
                const bool asc = ((lo_i & size) == 0);
                const uint64_t ka = sk[lo_i], kb = sk[hi_i];
                const int64_t ia = si[lo_i], ib = si[hi_i];
                const bool gt = (ka > kb) || (ka == kb && ia > ib);
                if (gt == asc) {
                    sk[lo_i] = kb; sk[hi_i] = ka;
                    si[lo_i] = ib; si[hi_i] = ia;
                }
            }
            __syncwarp();
        }
    }
    if (p.n_survivors && lane == 0) atomicAdd(p.n_survivors, (unsigned long long)ns);
    const int keff = min(p.k, ns);
    for (int r = lane; r < p.k; r += 32) {
        const int64_t o = q * (int64_t)p.k + r;
        if (r < keff) {
            const double key_d = o2d(sk[r]);
            if (p.out_ids) p.out_ids[o] = si[r];
            if (p.out_ids32) p.out_ids32[o] = (int32_t)si[r];
            if (p.out_dist) p.out_dist[o] = IP ? -key_d : key_d;
        } else {
            if (p.out_ids) p.out_ids[o] = -1;
            if (p.out_ids32) p.out_ids32[o] = -1;
            if (p.out_dist) p.out_dist[o] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
    if (lane == 0 && p.out_count) p.out_count[q] = keff;
}

static size_t rerank_smem(int d, int nsub, size_t ubytes, int ph) {
    const size_t chains =
        (reg_path_ok(d) || ph == 1) ? 0 : (size_t)NWARP * 8 * MAXLEAF * 8 + (size_t)NWARP * 2 * MAXLEAF * 8;
    const size_t qbytes = ph == 1 ? 0 : (size_t)q_stride(d) * 12;   // float + float64 copies of the query
    return ((sizeof(Small) + 127) & ~size_t(127)) + ubytes + chains + qbytes + (size_t)((nsub + 3) & ~3) * 4 +
           (size_t)HBINS * 4 + 16;
}

template <typename T, bool IP, bool WIDE, int PH>
static cudaError_t launch_rerank_v(const RerankParams& p, cudaStream_t s) {
    const size_t smem = rerank_smem(p.d, p.cb.n_sub, (size_t)p.ubytes, PH);
    auto kern = k_rerank<T, IP, WIDE, PH>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)p.nq, NT, smem, s>>>(p);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_rerank(const RerankParams& p0, cudaStream_t s) {
    if (p0.nq == 0) return cudaSuccess;
    RerankParams p = p0;
    if (p.d >= 8 && p.d <= WARP_D_MAX) np_leaves(p.d, p.plan);
    p.reg_path = reg_path_ok(p.d) ? 1 : 0;
    static const int pd_env = getenv("VS_RR_PD") ? atoi(getenv("VS_RR_PD")) : -1;
    if (pd_env >= 0) p.prefetch_iters = pd_env;
    // large k (many survivors and live candidates per query): the wide build;
    // small k (probes, IVF lists, config 1): 4 CTAs/SM hide more latency (measured)
    static const int wide_env = getenv("VS_RR_WIDE") ? atoi(getenv("VS_RR_WIDE")) : -1;
    const bool wide = wide_env >= 0 ? wide_env == 1 : p.k > 64;
    p.ubytes = (int)union_bytes(p.d, wide);
    // the wide scorer's two rows per warp and iteration: two iterations of L2
    // prefetch lead (four put ~95 MB of rows in flight and re-read 0.8 GB of
    // them from HBM in config 2 at the same time, profiles/r2/rerank_pd_sweep)
    if (wide && pd_env < 0) p.prefetch_iters = 2;
    // split phase B (wide build; VS_RR_SPLIT=0/1 overrides): the gather + select
    // kernel runs at 5 CTAs/SM without the scorer's registers, then score +
    // top-k (measured: config 2 re-rank 2.06 -> 1.90 ms; the narrow build
    // already runs 4 CTAs/SM and the split cost config 3 0.09 ms)
    // the distributed k-th-key pass (out_kth) is steps 0-2 only: the select
    // kernel's occupancy without the scorer
    static const int kth_env = getenv("VS_RR_KTH_SELECT") ? atoi(getenv("VS_RR_KTH_SELECT")) : 1;
    if (p.out_kth && kth_env) {
        RerankParams p1 = p;
        p1.ubytes = (int)union_min<false>();
        return p.ip ? launch_rerank_v<T, true, false, 1>(p1, s) : launch_rerank_v<T, false, false, 1>(p1, s);
    }
    static const int split_env = getenv("VS_RR_SPLIT") ? atoi(getenv("VS_RR_SPLIT")) : -1;
    const bool split = split_env >= 0 ? split_env == 1 : wide;
    if (split && p.s_count && !p.out_kth) {
        RerankParams p1 = p;
        p1.ubytes = (int)union_min<false>();   // live candidates only (LCAP of the narrow build)
        cudaError_t e = p.ip ? launch_rerank_v<T, true, false, 1>(p1, s) : launch_rerank_v<T, false, false, 1>(p1, s);
        if (e != cudaSuccess) return e;
        if (wide) return p.ip ? launch_rerank_v<T, true, true, 2>(p, s) : launch_rerank_v<T, false, true, 2>(p, s);
        return p.ip ? launch_rerank_v<T, true, false, 2>(p, s) : launch_rerank_v<T, false, false, 2>(p, s);
    }
    // small k without verification or distributed hooks: one warp per query,
    // the CTA kernel only for the queries it lists (VS_RR_WARP=0 disables)
    static const int warp_env = getenv("VS_RR_WARP") ? atoi(getenv("VS_RR_WARP")) : 1;
    // (not for many buffers per query: config 4's 128 margin-band buffers hold
    // more candidates than a warp stages, and the fallback then doubles the work)
    if (warp_env && p.fb_list && p.fb_count && p.reg_path && p.k <= 64 && p.cb.n_sub <= 64 && !p.verify &&
        !p.out_bound && !p.out_kth && !p.ext_thr && !p.q_list) {
        cudaError_t e = cudaMemsetAsync(p.fb_count, 0, sizeof(int32_t), s);
        if (e != cudaSuccess) return e;
        const unsigned grid = (unsigned)((p.nq + WW - 1) / WW);
        auto kern = p.ip ? k_rerank_warp<T, true, 512> : k_rerank_warp<T, false, 512>;
        const size_t smem = sizeof(WarpSmem<512>);
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
            return e;
        kern<<<grid, WW * 32, smem, s>>>(p, p.fb_list, p.fb_count);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        p.q_list = p.fb_list;
        p.q_count = p.fb_count;
    }
    if (wide) return p.ip ? launch_rerank_v<T, true, true, 0>(p, s) : launch_rerank_v<T, false, true, 0>(p, s);
    return p.ip ? launch_rerank_v<T, true, false, 0>(p, s) : launch_rerank_v<T, false, false, 0>(p, s);
}
#ifdef VS_RERANK_PROFILE
extern "C" int vs_debug_rerank_profile(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_rr_prof, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_rr_prof, z, sizeof(z));
    }
    return 0;
}
#endif
cudaError_t launch_union_kth(const float* keys, int G, int64_t nq, int k, float* out, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    int P = 1;
    while (P < G * k) P <<= 1;
    const size_t smem = (size_t)P * 4;
    cudaError_t e = cudaFuncSetAttribute(k_union_kth, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_union_kth<<<(unsigned)nq, NT, smem, s>>>(keys, G, nq, k, out);
    return cudaGetLastError();
}

template cudaError_t launch_rerank<float>(const RerankParams&, cudaStream_t);
template cudaError_t launch_rerank<__nv_bfloat16>(const RerankParams&, cudaStream_t);

// ---- cross-shard merge ------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_merge(MergeParams p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    Small& sm = *reinterpret_cast<Small*>(smraw);
    unsigned char* u = smraw + ((sizeof(Small) + 127) & ~size_t(127));
    const int64_t q = blockIdx.x;
    const int tid = threadIdx.x;
    const int64_t cap = (int64_t)p.nparts * p.k_in;
    uint64_t* skey = p.s_key + q * cap;
    int64_t* sid = p.s_id + q * cap;
    if (tid == 0) sm.counter = 0;
    __syncthreads();
    for (int64_t i = tid; i < cap; i += NT) {
        const int g = (int)(i / p.k_in), j = (int)(i - (int64_t)g * p.k_in);
        if (j < p.counts[(int64_t)g * p.nq + q]) {
            const int64_t src = ((int64_t)g * p.nq + q) * p.k_in + j;
            const double dd = p.dist[src];
            const int slot = atomicAdd(&sm.counter, 1);
            skey[slot] = d2o(p.ip ? -dd : dd);
            sid[slot] = p.ids[src];
        }
    }
    __syncthreads();
    const int64_t n = sm.counter;
    __syncthreads();
    block_topk_exact(skey, sid, n, p.k, sm, u, p.ip, q, p.out_ids, p.out_dist, nullptr, p.out_count);
}

cudaError_t launch_merge(const MergeParams& p, cudaStream_t s) {
    if (p.nq == 0) return cudaSuccess;
    const size_t smem = ((sizeof(Small) + 127) & ~size_t(127)) + UNION_BYTES;
    cudaError_t e = cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_merge<<<(unsigned)p.nq, NT, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace vs
