// The step after the search, on the GPU: the oversample
// post-filter and the output construction that the reference runs in numpy
// over the joined output table.
//
//   oversample_postfilter (vecsearch.py:155-202): per query, the first k rows
//     in rank order that survive the keep predicate (and the semi join), with
//     the shortfall reported. Here over the padded per-query result layout the
//     searches write ([nq][k'] ids / distances + counts), one warp per query:
//     the warp's ballot over 32 consecutive ranks plus a popcount prefix gives
//     every survivor its output slot, so the survivors stay in rank order.
//     Keep conditions (all optional, ANDed):
//       - a packed bitmap over the data rows (data-side predicates and semi
//         joins: vs_bitmap_compare / vs_bitmap_isin produce it);
//       - a per-result byte mask (any predicate evaluated on the joined output);
//       - data_key[data_row] <op> query_key[query_row] (the cross-side column
//         comparison of Q11's "im_imagekey_d != im_imagekey", plans.py:537).
//   build_vs_output (vecsearch.py:123-152): the flat NeighborTable arrays
//     (query_row, data_row, distance, rank, sorted by query then rank) from the
//     padded layout — an exclusive scan of the counts then one thread per
//     slot — and a row gather for every output column of either side.
#include <cub/cub.cuh>

#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

namespace {

__device__ __forceinline__ bool cmp_i64(int64_t a, int64_t b, int op) {
    switch (op) {
        case 0: return a < b;
        case 1: return a <= b;
        case 2: return a == b;
        case 3: return a != b;
        case 4: return a >= b;
        default: return a > b;
    }
}

__global__ void k_postfilter(PostfilterArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (q >= a.nq) return;
    const int cnt = a.counts ? min(max(a.counts[q], 0), a.kp) : a.kp;
    const int64_t* ids = a.ids + q * a.kp;
    const int64_t qkey = a.query_key ? a.query_key[q] : 0;
    int taken = 0;
    for (int j0 = 0; j0 < cnt && taken < a.k; j0 += 32) {
        const int j = j0 + lane;
        bool ok = false;
        int64_t id = -1;
        if (j < cnt) {
            id = ids[j];
            ok = true;
            if (a.bitmap || a.data_key) {
                if (id < 0 || id >= a.n_data) {
                    atomicOr(a.bad, 1);
                    ok = false;
                }
            }
            if (ok && a.bitmap) ok = (a.bitmap[id >> 5] >> (id & 31)) & 1u;
            if (ok && a.keep_pos) ok = a.keep_pos[q * a.kp + j] != 0;
            if (ok && a.data_key) ok = cmp_i64(a.data_key[id], qkey, a.key_op);
        }
        const unsigned b = __ballot_sync(VS_FULL, ok);
        const int pos = taken + __popc(b & ((1u << lane) - 1u));
        if (ok && pos < a.k) {
            const int64_t o = q * a.k + pos;
            if (a.out_ids) a.out_ids[o] = id;
            if (a.out_dist) a.out_dist[o] = a.dist[q * a.kp + j];
            if (a.out_rank) a.out_rank[o] = j;
        }
        taken += __popc(b);
    }
    if (lane == 0 && a.out_count) a.out_count[q] = min(taken, a.k);
}

// c64[0..nq) = clamped counts, c64[nq] = 0 (so the exclusive scan's last entry is the total)
__global__ void k_count_clamp(const int32_t* __restrict__ counts, int64_t nq, int kp, int64_t* __restrict__ c64) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nq; i += (int64_t)gridDim.x * blockDim.x)
        c64[i] = i == nq ? 0 : counts ? min(max(counts[i], 0), kp) : kp;
}

__global__ void k_flatten(FlattenArgs a, const int64_t* __restrict__ off) {
    const int64_t tot = a.nq * (int64_t)a.kp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = i / a.kp;
        const int j = (int)(i - q * a.kp);
        const int cnt = a.counts ? min(max(a.counts[q], 0), a.kp) : a.kp;
        if (j >= cnt) continue;
        const int64_t o = off[q] + j;
        if (a.query_row) a.query_row[o] = q + a.query_offset;
        if (a.data_row) a.data_row[o] = a.ids[i];
        if (a.distance) a.distance[o] = a.dist[i];
        if (a.rank) a.rank[o] = a.in_rank ? (int64_t)a.in_rank[i] : (int64_t)j;
    }
}

// dst[i] = src[idx[i]] for rows of W-byte words (W = 16, 8, 4 or 1)
template <typename W>
__global__ void k_gather(const W* __restrict__ src, int64_t n_src, int64_t words, const int64_t* __restrict__ idx,
                         int64_t n, W* __restrict__ dst, int* bad) {
    const int64_t tot = n * words;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / words, w = i - r * words;
        const int64_t s = idx[r];
        if (s < 0 || s >= n_src) {
            atomicOr(bad, 1);
            continue;
        }
        dst[i] = src[s * words + w];
    }
}

unsigned grid_for(int64_t work) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 32));
}

}  // namespace

cudaError_t launch_postfilter(const PostfilterArgs& a, cudaStream_t s) {
    if (a.nq == 0) return cudaSuccess;
    const int64_t threads = a.nq * 32;
    k_postfilter<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

size_t flatten_temp_bytes(int64_t nq) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const int64_t*)nullptr, (int64_t*)nullptr, (int)(nq + 1));
    return b + 256;
}

cudaError_t launch_flatten(const FlattenArgs& a, int64_t* c64, int64_t* off, void* tmp, size_t tmp_bytes,
                           cudaStream_t s) {
    k_count_clamp<<<grid_for(a.nq), 256, 0, s>>>(a.counts, a.nq, a.kp, c64);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    size_t tb = tmp_bytes;
    // inclusive total lands in off[nq] (exclusive scan over nq + 1 entries, last count 0)
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, c64, off, (int)(a.nq + 1), s)) != cudaSuccess) return e;
    if (a.kp > 0) k_flatten<<<grid_for(a.nq * a.kp), 256, 0, s>>>(a, off);
    return cudaGetLastError();
}

cudaError_t launch_gather(const void* src, int64_t n_src, int64_t row_bytes, const int64_t* idx, int64_t n,
                          void* dst, int* bad, cudaStream_t s) {
    if (n == 0 || row_bytes == 0) return cudaSuccess;
    const uintptr_t al = (uintptr_t)src | (uintptr_t)dst;
    if (row_bytes % 16 == 0 && al % 16 == 0) {
        const int64_t w = row_bytes / 16;
        k_gather<int4><<<grid_for(n * w), 256, 0, s>>>((const int4*)src, n_src, w, idx, n, (int4*)dst, bad);
    } else if (row_bytes % 8 == 0 && al % 8 == 0) {
        const int64_t w = row_bytes / 8;
        k_gather<uint64_t><<<grid_for(n * w), 256, 0, s>>>((const uint64_t*)src, n_src, w, idx, n, (uint64_t*)dst,
                                                           bad);
    } else if (row_bytes % 4 == 0 && al % 4 == 0) {
        const int64_t w = row_bytes / 4;
        k_gather<uint32_t><<<grid_for(n * w), 256, 0, s>>>((const uint32_t*)src, n_src, w, idx, n, (uint32_t*)dst,
                                                           bad);
    } else {
        k_gather<uint8_t><<<grid_for(n * row_bytes), 256, 0, s>>>((const uint8_t*)src, n_src, row_bytes, idx, n,
                                                                  (uint8_t*)dst, bad);
    }
    return cudaGetLastError();
}

}  // namespace vs
