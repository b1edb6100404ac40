// Row-filter plumbing: packed bitmap -> ascending selection vector, the
// permuted (list-order) bitmap for IVF scans, row norms and query margins.
//
// The relational predicate reaches the reference search as an order-
// preserving gather (table.py:326-331 `flatnonzero`, relops.py:112-113 semi
// join). Here the same ascending row set is produced on the device from the
// packed bitmap with a two-level popcount scan, so the scan kernels read
// selected rows in base-row order and positions map back to base row ids.
#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

static constexpr int SEL_THREADS = 256;
static constexpr int SEL_WORDS_PER_THREAD = 4;
static constexpr int SEL_WORDS_PER_BLOCK = SEL_THREADS * SEL_WORDS_PER_THREAD;  // 1024

int64_t select_nblocks(int64_t nwords) {
    return (nwords + SEL_WORDS_PER_BLOCK - 1) / SEL_WORDS_PER_BLOCK;
}

__device__ __forceinline__ uint32_t masked_word(const uint32_t* bm, int64_t w, int64_t nwords,
                                                int64_t nbits) {
    if (w >= nwords) return 0u;
    uint32_t v = bm[w];
    int64_t rem = nbits - w * 32;
    if (rem < 32) v &= (rem <= 0) ? 0u : ((1u << rem) - 1u);
    return v;
}

__global__ void k_select_count(const uint32_t* __restrict__ bm, int64_t nwords, int64_t nbits,
                               int64_t* __restrict__ block_sums) {
    __shared__ int warp_tot[SEL_THREADS / 32];
    int64_t w0 = (int64_t)blockIdx.x * SEL_WORDS_PER_BLOCK + threadIdx.x * SEL_WORDS_PER_THREAD;
    int c = 0;
#pragma unroll
    for (int j = 0; j < SEL_WORDS_PER_THREAD; ++j) c += __popc(masked_word(bm, w0 + j, nwords, nbits));
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int i = 0; i < SEL_THREADS / 32; ++i) t += warp_tot[i];
        block_sums[blockIdx.x] = t;
    }
}

// exclusive scan of block sums in place (single block, sequential chunks)
__global__ void k_select_scan(int64_t* __restrict__ sums, int64_t n, int64_t* __restrict__ total) {
    __shared__ int64_t carry;
    __shared__ int64_t wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = 0; base < n; base += blockDim.x) {
        int64_t i = base + threadIdx.x;
        int64_t v = (i < n) ? sums[i] : 0;
        // inclusive warp scan
        int64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(VS_FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int64_t s = (lane < (int)(blockDim.x >> 5)) ? wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int64_t y = __shfl_up_sync(VS_FULL, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;  // inclusive
        }
        __syncthreads();
        int64_t wprefix = wid ? wsum[wid - 1] : 0;
        int64_t excl = carry + wprefix + x - v;
        if (i < n) sums[i] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void k_select_write(const uint32_t* __restrict__ bm, int64_t nwords, int64_t nbits,
                               const int64_t* __restrict__ block_off, int64_t* __restrict__ sel) {
    __shared__ int wsum[SEL_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t w0 = (int64_t)blockIdx.x * SEL_WORDS_PER_BLOCK + threadIdx.x * SEL_WORDS_PER_THREAD;
    uint32_t words[SEL_WORDS_PER_THREAD];
    int c = 0;
#pragma unroll
    for (int j = 0; j < SEL_WORDS_PER_THREAD; ++j) {
        words[j] = masked_word(bm, w0 + j, nwords, nbits);
        c += __popc(words[j]);
    }
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(VS_FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    int wprefix = 0;
    for (int i = 0; i < wid; ++i) wprefix += wsum[i];
    int64_t off = block_off[blockIdx.x] + wprefix + x - c;
#pragma unroll
    for (int j = 0; j < SEL_WORDS_PER_THREAD; ++j) {
        uint32_t v = words[j];
        while (v) {
            int b = __ffs(v) - 1;
            v &= v - 1;
            sel[off++] = (w0 + j) * 32 + b;
        }
    }
}

cudaError_t launch_select_count(const uint32_t* bitmap, int64_t nwords, int64_t nbits,
                                int64_t* block_sums, int64_t nblocks, cudaStream_t s) {
    if (nblocks == 0) return cudaSuccess;
    k_select_count<<<(unsigned)nblocks, SEL_THREADS, 0, s>>>(bitmap, nwords, nbits, block_sums);
    return cudaGetLastError();
}
cudaError_t launch_select_scan(int64_t* block_sums, int64_t nblocks, int64_t* total,
                               cudaStream_t s) {
    k_select_scan<<<1, 1024, 0, s>>>(block_sums, nblocks, total);
    return cudaGetLastError();
}
cudaError_t launch_select_write(const uint32_t* bitmap, int64_t nwords, int64_t nbits,
                                const int64_t* block_offsets, int64_t* sel, cudaStream_t s) {
    int64_t nb = select_nblocks(nwords);
    if (nb == 0) return cudaSuccess;
    k_select_write<<<(unsigned)nb, SEL_THREADS, 0, s>>>(bitmap, nwords, nbits, block_offsets, sel);
    return cudaGetLastError();
}

// ---- permuted bitmap -----------------------------------------------------------------------
__global__ void k_permute_bitmap(const uint32_t* __restrict__ bm, int64_t nbits,
                                 const int64_t* __restrict__ ids, int64_t n_total,
                                 uint32_t* __restrict__ pbits) {
    // a warp owns 4 x 32 consecutive positions (4 output words): its four
    // coalesced id loads are in flight together before the bitmap gathers
    constexpr int PW = 4;
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t base = w * (32 * PW);
    int64_t r[PW];
#pragma unroll
    for (int j = 0; j < PW; ++j) {
        const int64_t i = base + 32 * j + lane;
        r[j] = i < n_total ? __ldcs(ids + i) : -1;
    }
#pragma unroll
    for (int j = 0; j < PW; ++j) {
        const bool bit = r[j] >= 0 && r[j] < nbits && ((__ldg(bm + (r[j] >> 5)) >> (r[j] & 31)) & 1u);
        const unsigned b = __ballot_sync(VS_FULL, bit);
        const int64_t word = (base >> 5) + j;
        if (lane == 0 && word < (n_total + 31) / 32) pbits[word] = b;
    }
}

cudaError_t launch_permute_bitmap(const uint32_t* bitmap, int64_t nbits, const int64_t* ids,
                                  int64_t n_total, uint32_t* pbits, cudaStream_t s) {
    if (n_total == 0) return cudaSuccess;
    const int64_t warps = (n_total + 127) / 128;
    const int64_t blocks = (warps * 32 + 255) / 256;
    k_permute_bitmap<<<(unsigned)blocks, 256, 0, s>>>(bitmap, nbits, ids, n_total, pbits);
    return cudaGetLastError();
}

// ---- row norms ------------------------------------------------------------------------------
template <typename T>
__global__ void k_row_norms(const T* __restrict__ x, int64_t n, int d, float* __restrict__ norms,
                            unsigned* __restrict__ max_bits) {
    const int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float mx = 0.f;
    for (int64_t r = warp; r < n; r += nwarps) {
        const T* row = x + r * (int64_t)d;
        float s = 0.f;
        for (int i = lane; i < d; i += 32) {
            float v = ld_elem(row + i);
            s = fmaf(v, v, s);
        }
        s = warp_sumf(s);
        if (lane == 0) norms[r] = s;
        mx = fmaxf(mx, s);
    }
    if (lane == 0) atomicMax(max_bits, __float_as_uint(mx));  // non-negative: bit order == value order
}

template <typename T>
cudaError_t launch_row_norms(const T* x, int64_t n, int d, float* norms, unsigned* max_norm_bits,
                             cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    int64_t blocks = (n * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_row_norms<T><<<(unsigned)blocks, 256, 0, s>>>(x, n, d, norms, max_norm_bits);
    return cudaGetLastError();
}
template cudaError_t launch_row_norms<float>(const float*, int64_t, int, float*, unsigned*, cudaStream_t);
template cudaError_t launch_row_norms<__nv_bfloat16>(const __nv_bfloat16*, int64_t, int, float*,
                                                    unsigned*, cudaStream_t);

__global__ void k_query_margins(const float* __restrict__ q, int64_t nq, int d,
                                const unsigned* __restrict__ max_bits, float eps, int ip,
                                float* __restrict__ margin, float* __restrict__ qnorm) {
    const int lane = threadIdx.x & 31;
    int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= nq) return;
    float s = 0.f;
    for (int i = lane; i < d; i += 32) {
        float v = q[r * (int64_t)d + i];
        s = fmaf(v, v, s);
    }
    s = warp_sumf(s);
    if (lane == 0) {
        // inflate both norms slightly so fp32 rounding of the norms themselves
        // cannot shrink the bound
        float qn = sqrtf(s) * 1.0001f;
        float xn = sqrtf(__uint_as_float(*max_bits)) * 1.0001f;
        float m = ip ? eps * qn * xn : eps * (qn + xn) * (qn + xn);
        margin[r] = m;
        if (qnorm) qnorm[r] = s;
    }
}

cudaError_t launch_query_margins(const float* q, int64_t nq, int d, const unsigned* max_norm_bits,
                                 float eps, int ip, float* margin, float* qnorm, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    int64_t blocks = (nq * 32 + 255) / 256;
    k_query_margins<<<(unsigned)blocks, 256, 0, s>>>(q, nq, d, max_norm_bits, eps, ip, margin, qnorm);
    return cudaGetLastError();
}

// ---- row gather (non-owning IVF -> device list-contiguous layout) ----------------------------
template <typename T>
__global__ void k_gather_rows(const T* __restrict__ src, const int64_t* __restrict__ ids, int64_t n,
                              int d, T* __restrict__ dst) {
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t r = warp; r < n; r += nwarps) {
        const T* a = src + ids[r] * (int64_t)d;
        T* b = dst + r * (int64_t)d;
        for (int i = lane; i < d; i += 32) b[i] = a[i];
    }
}
template <typename T>
cudaError_t launch_gather_rows(const T* src, const int64_t* ids, int64_t n, int d, T* dst,
                               cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    int64_t blocks = (n * 32 + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    k_gather_rows<T><<<(unsigned)blocks, 256, 0, s>>>(src, ids, n, d, dst);
    return cudaGetLastError();
}
template cudaError_t launch_gather_rows<float>(const float*, const int64_t*, int64_t, int, float*,
                                              cudaStream_t);
template cudaError_t launch_gather_rows<__nv_bfloat16>(const __nv_bfloat16*, const int64_t*, int64_t,
                                                      int, __nv_bfloat16*, cudaStream_t);

// selected rows of a host-resident (pinned, device-mapped) column -> device,
// 16-byte zero-copy reads over PCIe, warp per row; `blocks` bounds the SMs used
// so the gather can run beside a persistent tensor-core kernel
__global__ void k_gather_rows_v16(const uint4* __restrict__ src, const int64_t* __restrict__ ids, int64_t n,
                                  int row_vecs, uint4* __restrict__ dst) {
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t r = warp; r < n; r += nwarps) {
        const uint4* a = src + ids[r] * (int64_t)row_vecs;
        uint4* b = dst + r * (int64_t)row_vecs;
        for (int i = lane; i < row_vecs; i += 32) b[i] = a[i];
    }
}
cudaError_t launch_gather_rows_host(const void* src, const int64_t* ids, int64_t n, int row_bytes, void* dst,
                                    int blocks, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (row_bytes % 16) return cudaErrorInvalidValue;
    k_gather_rows_v16<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(src), ids, n, row_bytes / 16,
                                              reinterpret_cast<uint4*>(dst));
    return cudaGetLastError();
}

}  // namespace vs
