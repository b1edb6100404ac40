// Large-k' search ("wide" top-k): k' above the shared-memory top-k of the
// candidate-buffer path (vs_topk_cap() = 2048), up to every candidate.
//
// The reference has no k' limit on the host (vecsearch.py:86-87 raises only
// for a device placement with an explicit cap), and its oversampling plans
// ask for k' = 500 k = 50,000 (plans.py:256, 571). Candidate buffers sized for
// such k' would not fit, so this path keeps the same exactness argument
// over device-wide arrays instead:
//
//   1. approximate fp32 keys of every candidate of a chunk of queries —
//      ENN: a dense [Qc][nsel] key matrix (SIMT tile GEMM over the selected
//      rows); IVF: ragged per-query segments over the probed lists, filtered
//      rows keyed +inf (one CTA per (query, probe));
//   2. per query (one CTA): k_eff = min(k', valid candidates), K* = the
//      k_eff-th smallest key (3-pass radix select), survivors = keys <= K* +
//      margin (a superset of the exact top-k', ties included);
//   3. survivors compacted, scored exactly in float64 in numpy's pairwise
//      summation order (one warp per survivor), sorted by (distance, id)
//      (two stable segmented sorts: id, then key), the first k' emitted.
//
// Chunks of queries bound the key matrix; survivor sub-ranges bound the
// sort. Every kernel here is HBM- or f64-bound, not tensor-bound: this path
// serves the rare very large k', the candidate-buffer path the rest.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "vs_common.cuh"
#include "vs_internal.h"
#include "vs_kernels.cuh"
#include "vs_wide.cuh"

using namespace vs_internal;

namespace vs {
namespace {

constexpr int KT_Q = 64, KT_R = 128, KT_K = 16;   // dense key tile: queries x rows x depth
constexpr int SEL_NT = 1024;
constexpr uint32_t INF_O = 0xff800000u;           // f2o(+inf)

// ---- 1a. dense approximate keys (ENN) ---------------------------------------------------
// key = ||x||^2 - 2 q.x (squared L2, ||q||^2 dropped) or -q.x (inner product),
// fp32 FMA accumulation: |key - exact key| <= (d + 2) 2^-24 (|q| + |x|)^2, half
// the SIMT margin eps_simt (vs_capi.cu).
template <typename T, bool IP>
__global__ void __launch_bounds__(256) k_wide_keys_dense(const float* __restrict__ Q, int64_t nq, int d,
                                                         const T* __restrict__ X, const int64_t* __restrict__ sel,
                                                         int64_t ncand, const float* __restrict__ xnorm,
                                                         float* __restrict__ keys) {
    __shared__ float qs[KT_K][KT_Q + 4];
    __shared__ float xs[KT_K][KT_R + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t c0 = (int64_t)blockIdx.x * KT_R;
    const int64_t q0 = (int64_t)blockIdx.y * KT_Q;
    // row this thread stages (two threads per row, 8 depth elements each)
    const int lr = tid >> 1, lk = (tid & 1) * 8;
    const int64_t lpos = c0 + lr;
    const T* xrow = nullptr;
    if (lpos < ncand) xrow = X + (sel ? sel[lpos] : lpos) * (int64_t)d;
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    for (int k0 = 0; k0 < d; k0 += KT_K) {
        for (int e = tid; e < KT_Q * KT_K; e += 256) {
            const int qi = e / KT_K, kk = e % KT_K;
            const int64_t qg = q0 + qi;
            qs[kk][qi] = (qg < nq && k0 + kk < d) ? Q[qg * d + k0 + kk] : 0.f;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int kk = lk + t;
            xs[kk][lr] = (xrow && k0 + kk < d) ? ld_elem(xrow + k0 + kk) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KT_K; ++kk) {
            float a[4], b[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = qs[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = xs[kk][tx * 8 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t pos = c0 + tx * 8 + j;
        if (pos >= ncand) continue;
        const float xn = IP ? 0.f : xnorm[sel ? sel[pos] : pos];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t qg = q0 + ty * 4 + i;
            if (qg < nq) keys[qg * ncand + pos] = IP ? -acc[i][j] : fmaf(-2.f, acc[i][j], xn);
        }
    }
}

// ---- 1b. ragged approximate keys over probed lists (IVF) --------------------------------
// one CTA per (query, probe rank): the list's payload positions and keys land
// at seg_off[q] + pair_off[q * nprobe + j]; rows the filter drops key +inf.
template <typename T, bool IP>
__global__ void __launch_bounds__(256) k_wide_keys_lists(const float* __restrict__ Q, int d,
                                                         const int32_t* __restrict__ probes, int nprobe,
                                                         const int64_t* __restrict__ list_off,
                                                         const uint8_t* __restrict__ owned,
                                                         const uint32_t* __restrict__ pbits,
                                                         const T* __restrict__ payload,
                                                         const float* __restrict__ pnorm,
                                                         const int64_t* __restrict__ seg_off,
                                                         const int64_t* __restrict__ pair_off,
                                                         float* __restrict__ keys, uint32_t* __restrict__ cpos) {
    extern __shared__ float qsh[];
    const int64_t pr = blockIdx.x;
    const int64_t q = pr / nprobe;
    const int l = probes[pr];
    if (l < 0 || (owned && !owned[l])) return;
    const int64_t lo = list_off[l], n = list_off[l + 1] - lo;
    const int64_t base = seg_off[q] + pair_off[pr];
    for (int i = threadIdx.x; i < d; i += blockDim.x) qsh[i] = Q[q * d + i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t r = w; r < n; r += nw) {
        const int64_t pos = lo + r;
        const bool keep = !pbits || ((pbits[pos >> 5] >> (pos & 31)) & 1u);
        float key = __int_as_float(0x7f800000);
        if (keep) {
            const T* x = payload + pos * (int64_t)d;
            float s = 0.f;
            for (int i = lane; i < d; i += 32) s = fmaf(qsh[i], ld_elem(x + i), s);
            s = warp_sumf(s);
            key = IP ? -s : fmaf(-2.f, s, pnorm[pos]);
        }
        if (lane == 0) {
            keys[base + r] = key;
            cpos[base + r] = (uint32_t)pos;
        }
    }
}

// ---- 2. per-query k-th key and survivor count ---------------------------------------------
__device__ __forceinline__ long long block_sum(long long v, long long* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(VS_FULL, v, o);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    long long t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    return t;
}

// k_eff = min(k, finite keys); thr = the k_eff-th smallest key + margin
// (rounded up; every finite key when k_eff covers them all); scount = keys <=
// thr. One CTA of SEL_NT threads per query, 3-pass radix select (11/11/10 bits).
__global__ void __launch_bounds__(SEL_NT) k_wide_select(const float* __restrict__ keys,
                                                        const int64_t* __restrict__ seg_off, int64_t dense_n,
                                                        int k, const float* __restrict__ margin,
                                                        uint32_t* __restrict__ thr, int64_t* __restrict__ keff_out,
                                                        int64_t* __restrict__ scount) {
    __shared__ unsigned hist[2048];
    __shared__ long long red[SEL_NT / 32];
    __shared__ unsigned wtot[SEL_NT / 32];
    __shared__ int sel_bin;
    __shared__ unsigned sel_below;
    const int64_t q = blockIdx.x;
    const int64_t lo = seg_off ? seg_off[q] : q * dense_n;
    const int64_t n = seg_off ? seg_off[q + 1] - lo : dense_n;
    const float* kq = keys + lo;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    long long nv = 0;
    for (int64_t i = tid; i < n; i += SEL_NT) nv += f2o(kq[i]) < INF_O;
    nv = block_sum(nv, red);
    const int64_t keff = min((int64_t)k, (int64_t)nv);
    uint32_t thr_o;
    if (keff == 0) {
        thr_o = 0u;    // nothing survives (keys are never the orderable 0: that is -NaN)
    } else if (keff == nv) {
        thr_o = INF_O - 1u;
    } else {
        uint32_t prefix = 0u, pmask = 0u;
        unsigned kk = (unsigned)keff;
        for (int pass = 0; pass < 3; ++pass) {
            const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
            const int nb = pass == 2 ? 1024 : 2048;
            for (int i = tid; i < nb; i += SEL_NT) hist[i] = 0u;
            __syncthreads();
            for (int64_t i = tid; i < n; i += SEL_NT) {
                const uint32_t u = f2o(kq[i]);
                if ((u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & (uint32_t)(nb - 1)], 1u);
            }
            __syncthreads();
            const int per = (nb + SEL_NT - 1) / SEL_NT;
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
            if (lane == 31) wtot[w] = incl;
            __syncthreads();
            unsigned excl = incl - loc;
            for (int i = 0; i < w; ++i) excl += wtot[i];
            if (excl < kk && kk <= excl + loc) {
                unsigned c = excl;
                for (int b = 0; b < per; ++b) {
                    const int bi = tid * per + b;
                    const unsigned h = bi < nb ? hist[bi] : 0u;
                    if (c + h >= kk) {
                        sel_bin = bi;
                        sel_below = c;
                        break;
                    }
                    c += h;
                }
            }
            __syncthreads();
            kk -= sel_below;
            prefix |= (uint32_t)sel_bin << shift;
            pmask |= (uint32_t)(nb - 1) << shift;
            __syncthreads();
        }
        thr_o = min(f2o(__fadd_ru(o2f(prefix), margin[q])), INF_O - 1u);
    }
    long long ns = 0;
    for (int64_t i = tid; i < n; i += SEL_NT) ns += f2o(kq[i]) <= thr_o;
    ns = block_sum(ns, red);
    if (tid == 0) {
        thr[q] = thr_o;
        keff_out[q] = keff;
        scount[q] = ns;
    }
}

// ---- 3. survivors: compaction, exact scores, output ---------------------------------------
// queries [qa, qb) of the chunk; survivors of query q land at s_off[q - qa]..
__global__ void __launch_bounds__(SEL_NT) k_wide_compact(const float* __restrict__ keys,
                                                         const int64_t* __restrict__ seg_off, int64_t dense_n,
                                                         const uint32_t* __restrict__ cpos, int64_t qa,
                                                         const uint32_t* __restrict__ thr,
                                                         const int64_t* __restrict__ s_off,
                                                         const int64_t* __restrict__ sel,
                                                         const int64_t* __restrict__ id_map, int64_t id_offset,
                                                         int64_t* __restrict__ s_row, int64_t* __restrict__ s_id,
                                                         int32_t* __restrict__ s_q) {
    __shared__ unsigned long long counter;
    const int64_t q = qa + blockIdx.x;
    const int64_t lo = seg_off ? seg_off[q] : q * dense_n;
    const int64_t n = seg_off ? seg_off[q + 1] - lo : dense_n;
    const uint32_t t = thr[q];
    const int64_t out0 = s_off[blockIdx.x];
    if (threadIdx.x == 0) counter = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = 0; i0 < n; i0 += SEL_NT) {
        const int64_t i = i0 + threadIdx.x;
        const bool live = i < n && f2o(keys[lo + i]) <= t;
        const unsigned b = __ballot_sync(VS_FULL, live);
        if (!b) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&counter, (unsigned long long)__popc(b));
        base = __shfl_sync(VS_FULL, base, 0);
        if (live) {
            const int64_t slot = out0 + (int64_t)base + __popc(b & lanemask_lt());
            int64_t row, id;
            if (cpos) {
                row = cpos[lo + i];
                id = id_map ? id_map[row] : row;
            } else {
                row = sel ? sel[i] : i;
                id = row;
            }
            s_row[slot] = row;
            s_id[slot] = id + id_offset;
            s_q[slot] = (int32_t)(q - qa);
        }
    }
}

// exact float64 score in numpy's pairwise order, one warp per (query, row),
// both read from global memory: lane c < 8 * nleaf runs chain c % 8 of leaf
// c / 8 (elements off + j + 8m, in order), the chains fold in numpy's order,
// lane 0 folds the leaves along the recursion (bit-identical to np_pairwise)
template <typename T, bool IP>
__device__ double warp_np_score_global(const float* __restrict__ q, const T* __restrict__ x, const LeafPlan& S,
                                       double* cbuf, double* lbuf, int lane) {
    const int nleaf = S.nleaf, nch = nleaf * 8;
    for (int c = lane; c < nch; c += 32) {
        const int L = c >> 3, j = c & 7;
        const int off = S.leaf_off[L], n = S.leaf_n[L];
        const int lim = n - (n % 8);
        double r = np_term<T, IP>(q + off, x + off, j);
        for (int i = 8 + j; i < lim; i += 8) r = __dadd_rn(r, np_term<T, IP>(q + off, x + off, i));
        cbuf[c] = r;
    }
    __syncwarp();
    for (int L = lane; L < nleaf; L += 32) {
        const double* cb = cbuf + L * 8;
        double res = __dadd_rn(__dadd_rn(__dadd_rn(cb[0], cb[1]), __dadd_rn(cb[2], cb[3])),
                               __dadd_rn(__dadd_rn(cb[4], cb[5]), __dadd_rn(cb[6], cb[7])));
        const int off = S.leaf_off[L], n = S.leaf_n[L];
        for (int i = n - (n % 8); i < n; ++i) res = __dadd_rn(res, np_term<T, IP>(q + off, x + off, i));
        lbuf[L] = res;
    }
    __syncwarp();
    double sc = 0.0;
    if (lane == 0) {
        for (int j = 0; j < S.nnode; ++j) lbuf[nleaf + j] = __dadd_rn(lbuf[S.node_a[j]], lbuf[S.node_b[j]]);
        sc = S.nnode ? lbuf[nleaf + S.nnode - 1] : lbuf[0];
    }
    __syncwarp();
    return __shfl_sync(VS_FULL, sc, 0);
}

// a leaf of numpy's recursion holds <= 128 elements and every leaf but the
// last >= 64, so d <= 2048 keeps nleaf <= 32 (the plan's capacity); larger d
// score one survivor per thread with the iterative recursion
constexpr int WS_NT = 256;
template <typename T, bool IP, bool WARP>
__global__ void __launch_bounds__(WS_NT) k_wide_score(const float* __restrict__ Q, int d, const T* __restrict__ rows,
                                                      const int64_t* __restrict__ s_row,
                                                      const int32_t* __restrict__ s_q, int64_t S_n,
                                                      uint64_t* __restrict__ s_key, LeafPlan plan) {
    __shared__ LeafPlan sp;
    __shared__ double cbuf[WS_NT / 32][8 * 32];
    __shared__ double lbuf[WS_NT / 32][2 * 32];
    if (threadIdx.x == 0) sp = plan;
    __syncthreads();
    if (WARP) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int64_t i = (int64_t)blockIdx.x * (WS_NT / 32) + w; i < S_n; i += (int64_t)gridDim.x * (WS_NT / 32)) {
            const double sc = warp_np_score_global<T, IP>(Q + (int64_t)s_q[i] * d, rows + s_row[i] * (int64_t)d, sp,
                                                          cbuf[w], lbuf[w], lane);
            if (lane == 0) s_key[i] = d2o(IP ? -sc : sc);
        }
    } else {
        for (int64_t i = (int64_t)blockIdx.x * WS_NT + threadIdx.x; i < S_n; i += (int64_t)gridDim.x * WS_NT) {
            const double sc = np_pairwise<T, IP>(Q + (int64_t)s_q[i] * d, rows + s_row[i] * (int64_t)d, d);
            s_key[i] = d2o(IP ? -sc : sc);
        }
    }
}

__global__ void k_wide_iota(int64_t* v, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = i;
}

// first k_eff (key, id) of every query's sorted survivors -> padded outputs
__global__ void k_wide_emit(const uint64_t* __restrict__ key, const int64_t* __restrict__ id,
                            const int64_t* __restrict__ s_off, int64_t qa, int64_t nqs,
                            const int64_t* __restrict__ keff, int k, int ip, int64_t* __restrict__ out_ids,
                            double* __restrict__ out_dist, int32_t* __restrict__ out_ids32,
                            int32_t* __restrict__ out_count) {
    const int64_t qi = blockIdx.y;
    if (qi >= nqs) return;
    const int64_t q = qa + qi;
    const int64_t ke = keff[q];
    const int64_t base = s_off[qi];
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < k; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = q * (int64_t)k + r;
        if (r < ke) {
            const double kd = o2d(key[base + r]);
            if (out_ids) out_ids[o] = id[base + r];
            if (out_ids32) out_ids32[o] = (int32_t)id[base + r];
            if (out_dist) out_dist[o] = ip ? -kd : kd;
        } else {
            if (out_ids) out_ids[o] = -1;
            if (out_ids32) out_ids32[o] = -1;
            if (out_dist) out_dist[o] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && out_count) out_count[q] = (int32_t)ke;
}

// survivors of queries [qa, qb) of a chunk whose keys, thresholds and counts
// are computed: compact, score, sort, emit
int wide_finish(vs_ctx* ctx, const WideJob& j, const float* keys, const int64_t* seg_off_d, int64_t dense_n,
                const uint32_t* cpos, int64_t q0, int64_t qa, int64_t qb, const std::vector<int64_t>& h_scount,
                const uint32_t* thr, const int64_t* keff) {
    const int64_t nqs = qb - qa;
    std::vector<int64_t> h_soff(nqs + 1, 0);
    for (int64_t i = 0; i < nqs; ++i) h_soff[i + 1] = h_soff[i] + h_scount[qa - q0 + i];
    const int64_t S = h_soff[nqs];
    if (S > (int64_t)INT32_MAX) return set_err(VS_ERR_PLACEMENT, "wide top-k: %lld survivors in one sort", (long long)S);
    int64_t *s_off = nullptr, *s_row = nullptr, *s_id = nullptr, *s_id2 = nullptr;
    uint64_t *s_key = nullptr, *s_key2 = nullptr;
    int32_t* s_q = nullptr;
    const size_t Sa = (size_t)std::max<int64_t>(S, 1);
    CKS(arena_alloc(ctx, (size_t)nqs + 1, &s_off));
    CKS(arena_alloc(ctx, Sa, &s_row));
    CKS(arena_alloc(ctx, Sa, &s_id));
    CKS(arena_alloc(ctx, Sa, &s_id2));
    CKS(arena_alloc(ctx, Sa, &s_key));
    CKS(arena_alloc(ctx, Sa, &s_key2));
    CKS(arena_alloc(ctx, Sa, &s_q));
    CK(cudaMemcpyAsync(s_off, h_soff.data(), (nqs + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    // queries of this sub-range relative to the chunk (keys / seg_off / thr are chunk-based)
    k_wide_compact<<<(unsigned)nqs, SEL_NT, 0, ctx->stream>>>(keys, seg_off_d, dense_n, cpos, qa - q0, thr, s_off,
                                                             j.sel, j.id_map, j.id_offset, s_row, s_id, s_q);
    CK(cudaGetLastError());
    if (S > 0) {
        LeafPlan plan;
        np_leaves(j.d, plan);
        // leaves shorter than 8 (d < 8) are plain sequential sums: per-thread path
        const bool warp = plan.nleaf <= 32 && j.d >= 8;
        const int64_t units = warp ? (S + WS_NT / 32 - 1) / (WS_NT / 32) : (S + WS_NT - 1) / WS_NT;
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)ctx->sm_count * 8));
        const float* Qc = j.q + (q0 + (qa - q0)) * (int64_t)j.d;   // s_q is relative to qa
        KTimer kt(ctx, j.cls_rerank);
#define VS_WS(T_, IP_, W_) k_wide_score<T_, IP_, W_><<<grid, WS_NT, 0, ctx->stream>>>( \
            Qc, j.d, reinterpret_cast<const T_*>(j.rows), s_row, s_q, S, s_key, plan)
        if (j.dtype == VS_DTYPE_F32) {
            if (j.ip) { if (warp) VS_WS(float, true, true); else VS_WS(float, true, false); }
            else { if (warp) VS_WS(float, false, true); else VS_WS(float, false, false); }
        } else {
            if (j.ip) { if (warp) VS_WS(__nv_bfloat16, true, true); else VS_WS(__nv_bfloat16, true, false); }
            else { if (warp) VS_WS(__nv_bfloat16, false, true); else VS_WS(__nv_bfloat16, false, false); }
        }
#undef VS_WS
        CK(cudaGetLastError());
        // (key, id) order per query: stable sort by id, then stable sort by key
        size_t tb1 = 0, tb2 = 0;
        CK(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb1, s_id, s_id2, s_key, s_key2, (int)S, (int)nqs,
                                                     s_off, s_off + 1, ctx->stream));
        CK(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb2, s_key2, s_key, s_id2, s_id, (int)S, (int)nqs,
                                                     s_off, s_off + 1, ctx->stream));
        char* tmp = nullptr;
        CKS(arena_alloc(ctx, std::max(tb1, tb2), &tmp));
        size_t t1 = std::max(tb1, tb2), t2 = t1;
        CK(cub::DeviceSegmentedSort::StableSortPairs(tmp, t1, s_id, s_id2, s_key, s_key2, (int)S, (int)nqs, s_off,
                                                     s_off + 1, ctx->stream));
        CK(cub::DeviceSegmentedSort::StableSortPairs(tmp, t2, s_key2, s_key, s_id2, s_id, (int)S, (int)nqs, s_off,
                                                     s_off + 1, ctx->stream));
    }
    dim3 eg((unsigned)std::min<int64_t>(((int64_t)j.k + 255) / 256, 64), (unsigned)nqs);
    k_wide_emit<<<eg, 256, 0, ctx->stream>>>(s_key, s_id, s_off, qa, nqs, keff, j.k, j.ip, j.out_ids, j.out_dist,
                                             j.out_ids32, j.out_count);
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += S > 0 ? 8 : 2;
    // the survivor arrays are dead after this sub-range: later sub-ranges reuse
    // scratch only through the arena's high-water mark (calls are synchronous)
    CK(cudaStreamSynchronize(ctx->stream));
    return VS_OK;
}

// select + survivor counts for the chunk's queries [q0, q0 + nqc), then the
// survivors in sub-ranges of at most kSurvBudget (a single query may exceed it)
constexpr int64_t kSurvBudget = int64_t(1) << 27;
int wide_select_and_finish(vs_ctx* ctx, const WideJob& j, const float* keys, const int64_t* seg_off_d,
                           int64_t dense_n, const uint32_t* cpos, int64_t q0, int64_t nqc, const float* margin) {
    uint32_t* thr = nullptr;
    int64_t *keff = nullptr, *scount = nullptr;
    CKS(arena_alloc(ctx, (size_t)nqc, &thr));
    CKS(arena_alloc(ctx, (size_t)nqc, &keff));
    CKS(arena_alloc(ctx, (size_t)nqc, &scount));
    {
        KTimer kt(ctx, j.cls_rerank);
        k_wide_select<<<(unsigned)nqc, SEL_NT, 0, ctx->stream>>>(keys, seg_off_d, dense_n, j.k, margin, thr, keff,
                                                                scount);
        CK(cudaGetLastError());
    }
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    std::vector<int64_t> h(nqc);
    CK(cudaMemcpyAsync(h.data(), scount, nqc * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    int64_t tot = 0;
    for (int64_t v : h) tot += v;
    if (q0 == 0) ctx->stats[VS_STAT_SURVIVORS] = 0;
    ctx->stats[VS_STAT_SURVIVORS] += tot;
    // keff / thr are indexed by chunk query; shift the emit/compaction views
    int64_t qa = 0;
    while (qa < nqc) {
        int64_t qb = qa, s = 0;
        while (qb < nqc && (qb == qa || s + h[qb] <= kSurvBudget)) s += h[qb++];
        // wide_finish indexes thr/keff by (chunk query) and writes outputs at q0 + query
        WideJob jj = j;
        jj.q = j.q + q0 * (int64_t)j.d;
        if (jj.out_ids) jj.out_ids += q0 * (int64_t)j.k;
        if (jj.out_dist) jj.out_dist += q0 * (int64_t)j.k;
        if (jj.out_ids32) jj.out_ids32 += q0 * (int64_t)j.k;
        if (jj.out_count) jj.out_count += q0;
        CKS(wide_finish(ctx, jj, keys, seg_off_d, dense_n, cpos, 0, qa, qb, h, thr, keff));
        qa = qb;
    }
    return VS_OK;
}

// merge: entries j < counts[g][q] of every part, in (part, slot) order
__global__ void k_wide_merge_gather(int nparts, int64_t nq, int k_in, const int64_t* __restrict__ ids,
                                    const double* __restrict__ dist, const int32_t* __restrict__ counts,
                                    const int64_t* __restrict__ part_off, int ip, int64_t* __restrict__ s_id,
                                    uint64_t* __restrict__ s_key) {
    const int64_t g = blockIdx.y, q = blockIdx.z;
    const int c = counts[g * nq + q];
    const int64_t base = part_off[q * nparts + g];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < c; j += gridDim.x * blockDim.x) {
        const int64_t src = (g * nq + q) * k_in + j;
        const double dd = dist[src];
        s_key[base + j] = d2o(ip ? -dd : dd);
        s_id[base + j] = ids[src];
    }
}

}  // namespace

int wide_merge(vs_ctx* ctx, int nparts, int64_t nq, int k_in, const int64_t* ids, const double* dist,
               const int32_t* counts, int k, int ip, int64_t* out_ids, double* out_dist, int32_t* out_count) {
    if (nq == 0) return VS_OK;
    std::vector<int32_t> hc((size_t)nparts * nq);
    CK(cudaMemcpyAsync(hc.data(), counts, hc.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<int64_t> soff(nq + 1, 0), poff((size_t)nq * nparts), keff(nq);
    for (int64_t q = 0; q < nq; ++q) {
        int64_t t = 0;
        for (int g = 0; g < nparts; ++g) {
            poff[(size_t)q * nparts + g] = soff[q] + t;
            t += std::max(0, std::min(hc[(size_t)g * nq + q], k_in));
        }
        soff[q + 1] = soff[q] + t;
        keff[q] = std::min<int64_t>(t, k);
    }
    const int64_t S = soff[nq];
    if (S > (int64_t)INT32_MAX) return set_err(VS_ERR_PLACEMENT, "merge: %lld entries in one sort", (long long)S);
    int64_t *d_soff = nullptr, *d_poff = nullptr, *d_keff = nullptr, *s_id = nullptr, *s_id2 = nullptr;
    uint64_t *s_key = nullptr, *s_key2 = nullptr;
    const size_t Sa = (size_t)std::max<int64_t>(S, 1);
    CKS(arena_alloc(ctx, (size_t)nq + 1, &d_soff));
    CKS(arena_alloc(ctx, poff.size(), &d_poff));
    CKS(arena_alloc(ctx, (size_t)nq, &d_keff));
    CKS(arena_alloc(ctx, Sa, &s_id));
    CKS(arena_alloc(ctx, Sa, &s_id2));
    CKS(arena_alloc(ctx, Sa, &s_key));
    CKS(arena_alloc(ctx, Sa, &s_key2));
    CK(cudaMemcpyAsync(d_soff, soff.data(), soff.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(d_poff, poff.data(), poff.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(d_keff, keff.data(), keff.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    KTimer kt(ctx, VS_K_MERGE);
    if (S > 0) {
        dim3 gg((unsigned)std::min<int64_t>((k_in + 255) / 256, 64), (unsigned)nparts, (unsigned)nq);
        k_wide_merge_gather<<<gg, 256, 0, ctx->stream>>>(nparts, nq, k_in, ids, dist, counts, d_poff, ip, s_id,
                                                         s_key);
        CK(cudaGetLastError());
        size_t tb1 = 0, tb2 = 0;
        CK(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb1, s_id, s_id2, s_key, s_key2, (int)S, (int)nq,
                                                     d_soff, d_soff + 1, ctx->stream));
        CK(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb2, s_key2, s_key, s_id2, s_id, (int)S, (int)nq,
                                                     d_soff, d_soff + 1, ctx->stream));
        char* tmp = nullptr;
        size_t t1 = std::max(tb1, tb2), t2 = t1;
        CKS(arena_alloc(ctx, t1, &tmp));
        CK(cub::DeviceSegmentedSort::StableSortPairs(tmp, t1, s_id, s_id2, s_key, s_key2, (int)S, (int)nq, d_soff,
                                                     d_soff + 1, ctx->stream));
        CK(cub::DeviceSegmentedSort::StableSortPairs(tmp, t2, s_key2, s_key, s_id2, s_id, (int)S, (int)nq, d_soff,
                                                     d_soff + 1, ctx->stream));
    }
    dim3 eg((unsigned)std::min<int64_t>(((int64_t)k + 255) / 256, 64), (unsigned)nq);
    k_wide_emit<<<eg, 256, 0, ctx->stream>>>(s_key, s_id, d_soff, 0, nq, d_keff, k, ip, out_ids, out_dist, nullptr,
                                             out_count);
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += S > 0 ? 6 : 1;
    return VS_OK;
}

// Exhaustive (ENN) wide search over nsel candidate rows (sel nullable).
int wide_enn(vs_ctx* ctx, const WideJob& j) {
    if (j.nq == 0) return VS_OK;
    const int64_t ncand = j.ncand;
    const size_t key_budget = (size_t)1 << 28;    // keys per chunk (1 GiB)
    int64_t qc = std::max<int64_t>(1, (int64_t)(key_budget / (size_t)std::max<int64_t>(ncand, 1)));
    qc = std::min<int64_t>(qc, j.nq);
    if (qc >= KT_Q) qc = qc / KT_Q * KT_Q;
    float* keys = nullptr;
    CKS(arena_alloc(ctx, (size_t)qc * ncand, &keys));
    for (int64_t q0 = 0; q0 < j.nq; q0 += qc) {
        const int64_t nqc = std::min<int64_t>(qc, j.nq - q0);
        {
            KTimer kt(ctx, j.cls_scan);
            dim3 grid((unsigned)((ncand + KT_R - 1) / KT_R), (unsigned)((nqc + KT_Q - 1) / KT_Q));
            const float* Qc = j.q + q0 * (int64_t)j.d;
#define VS_WK(T_, IP_) k_wide_keys_dense<T_, IP_><<<grid, 256, 0, ctx->stream>>>( \
            Qc, nqc, j.d, reinterpret_cast<const T_*>(j.rows), j.sel, ncand, j.xnorm, keys)
            if (j.dtype == VS_DTYPE_F32) { if (j.ip) VS_WK(float, true); else VS_WK(float, false); }
            else { if (j.ip) VS_WK(__nv_bfloat16, true); else VS_WK(__nv_bfloat16, false); }
#undef VS_WK
            CK(cudaGetLastError());
        }
        ctx->stats[VS_STAT_LAUNCHES] += 1;
        CKS(wide_select_and_finish(ctx, j, keys, nullptr, ncand, nullptr, q0, nqc, j.margin + q0));
    }
    return VS_OK;
}

// IVF wide search: candidates = the (owned) probed lists of each query,
// filtered rows keyed +inf. probes: device [nq][nprobe]; h_off: host list
// offsets; queries chunked so a chunk's candidates fit the key budget.
int wide_ivf(vs_ctx* ctx, const WideJob& j, const int32_t* probes, int nprobe, const int64_t* list_off_d,
             const std::vector<int64_t>& h_off, const uint8_t* owned_d, const uint32_t* pbits, const float* pnorm) {
    if (j.nq == 0) return VS_OK;
    std::vector<int32_t> hp((size_t)j.nq * nprobe);
    CK(cudaMemcpyAsync(hp.data(), probes, hp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    std::vector<uint8_t> how;
    const int nlist = (int)h_off.size() - 1;
    if (owned_d) {
        how.resize(nlist);
        CK(cudaMemcpyAsync(how.data(), owned_d, nlist, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    auto lsize = [&](int l) -> int64_t {
        if (l < 0 || (owned_d && !how[l])) return 0;
        return h_off[l + 1] - h_off[l];
    };
    const int64_t budget = int64_t(1) << 28;
    int64_t q0 = 0;
    while (q0 < j.nq) {
        // chunk [q0, q1): per-query segment offsets and per-(query, probe) offsets
        std::vector<int64_t> seg(1, 0), poff;
        int64_t q1 = q0;
        while (q1 < j.nq) {
            int64_t s = 0;
            for (int p = 0; p < nprobe; ++p) s += lsize(hp[(size_t)q1 * nprobe + p]);
            if (q1 > q0 && seg.back() + s > budget) break;
            int64_t acc = 0;
            for (int p = 0; p < nprobe; ++p) {
                poff.push_back(acc);
                acc += lsize(hp[(size_t)q1 * nprobe + p]);
            }
            seg.push_back(seg.back() + s);
            ++q1;
        }
        const int64_t nqc = q1 - q0, total = seg.back();
        int64_t *seg_d = nullptr, *poff_d = nullptr;
        float* keys = nullptr;
        uint32_t* cpos = nullptr;
        CKS(arena_alloc(ctx, seg.size(), &seg_d));
        CKS(arena_alloc(ctx, poff.size(), &poff_d));
        CKS(arena_alloc(ctx, (size_t)std::max<int64_t>(total, 1), &keys));
        CKS(arena_alloc(ctx, (size_t)std::max<int64_t>(total, 1), &cpos));
        CK(cudaMemcpyAsync(seg_d, seg.data(), seg.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(poff_d, poff.data(), poff.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        {
            KTimer kt(ctx, j.cls_scan);
            const float* Qc = j.q + q0 * (int64_t)j.d;
            const unsigned grid = (unsigned)(nqc * nprobe);
            const size_t smem = (size_t)j.d * sizeof(float);
#define VS_WL(T_, IP_)                                                                                   \
    do {                                                                                                 \
        if (smem > 48 * 1024)                                                                            \
            CK(cudaFuncSetAttribute(k_wide_keys_lists<T_, IP_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                    (int)smem));                                                         \
        k_wide_keys_lists<T_, IP_><<<grid, 256, smem, ctx->stream>>>(                                    \
            Qc, j.d, probes + q0 * nprobe, nprobe, list_off_d, owned_d, pbits,                           \
            reinterpret_cast<const T_*>(j.rows), pnorm, seg_d, poff_d, keys, cpos);                      \
    } while (0)
            if (grid > 0) {
                if (j.dtype == VS_DTYPE_F32) { if (j.ip) VS_WL(float, true); else VS_WL(float, false); }
                else { if (j.ip) VS_WL(__nv_bfloat16, true); else VS_WL(__nv_bfloat16, false); }
            }
#undef VS_WL
            CK(cudaGetLastError());
        }
        ctx->stats[VS_STAT_LAUNCHES] += 1;
        CKS(wide_select_and_finish(ctx, j, keys, seg_d, 0, cpos, q0, nqc, j.margin + q0));
        q0 = q1;
    }
    return VS_OK;
}

}  // namespace vs
