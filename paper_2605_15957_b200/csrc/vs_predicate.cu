// Relational filters straight into the packed row bitmap the searches take
// ("the step before"): comparison predicates over a column and
// semi-join membership, evaluated on the GPU with one warp per 32 rows (the
// warp's ballot IS the bitmap word, LSB-first), so no boolean array is ever
// materialised or copied.
//
// Reference semantics:
//   eval_predicate (expr.py:568-576): rows where the predicate is valid and
//     true; numpy comparison rules (NaN compares false, except != which is true);
//   semi join (relops.py:88-113): left rows whose key occurs on the right; null
//     keys never match.
#include <cub/cub.cuh>

#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

namespace {

template <typename T>
__device__ __forceinline__ bool cmp(T a, double b, int op) {
    // numpy compares mixed int/float operands after promotion to float64
    const double x = (double)a;
    switch (op) {
        case 0: return x < b;
        case 1: return x <= b;
        case 2: return x == b;
        case 3: return x != b;   // NaN != b is true, as in numpy
        case 4: return x >= b;
        default: return x > b;
    }
}

__device__ __forceinline__ bool valid_bit(const uint32_t* valid, int64_t i) {
    return valid == nullptr || ((valid[i >> 5] >> (i & 31)) & 1u);
}

template <typename T>
__global__ void k_bitmap_compare(const T* __restrict__ v, int64_t n, int op, double value,
                                 const uint32_t* __restrict__ valid, uint32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nwords = (n + 31) / 32;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwords;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t i = w * 32 + lane;
        const bool b = i < n && valid_bit(valid, i) && cmp<T>(v[i], value, op);
        const unsigned word = __ballot_sync(VS_FULL, b);
        if (lane == 0) out[w] = word;
    }
}

__global__ void k_bitmap_isin(const int64_t* __restrict__ keys, int64_t n, const uint32_t* __restrict__ valid,
                              const int64_t* __restrict__ set, int64_t nset, uint32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nwords = (n + 31) / 32;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwords;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t i = w * 32 + lane;
        bool b = false;
        if (i < n && valid_bit(valid, i)) {
            const int64_t key = keys[i];
            int64_t lo = 0, hi = nset;   // lower bound in the sorted set
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (set[mid] < key) lo = mid + 1;
                else hi = mid;
            }
            b = lo < nset && set[lo] == key;
        }
        const unsigned word = __ballot_sync(VS_FULL, b);
        if (lane == 0) out[w] = word;
    }
}

__global__ void k_bitmap_combine(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t nwords,
                                 int op, uint32_t* __restrict__ out) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
         w += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t x = a[w], y = b[w];
        out[w] = op == 0 ? (x & y) : op == 1 ? (x | y) : (x & ~y);
    }
}

unsigned grid_words(int64_t nwords) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((nwords * 32 + 255) / 256, 148 * 32));
}

}  // namespace

cudaError_t launch_bitmap_compare(const void* values, int vtype, int64_t n, int op, double value,
                                  const uint32_t* valid, uint32_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned g = grid_words((n + 31) / 32);
    switch (vtype) {
        case 0: k_bitmap_compare<int32_t><<<g, 256, 0, s>>>((const int32_t*)values, n, op, value, valid, out); break;
        case 1: k_bitmap_compare<int64_t><<<g, 256, 0, s>>>((const int64_t*)values, n, op, value, valid, out); break;
        case 2: k_bitmap_compare<float><<<g, 256, 0, s>>>((const float*)values, n, op, value, valid, out); break;
        case 3: k_bitmap_compare<double><<<g, 256, 0, s>>>((const double*)values, n, op, value, valid, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

size_t bitmap_isin_temp_bytes(int64_t nset) {
    size_t b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b, (const int64_t*)nullptr, (int64_t*)nullptr, (int)nset);
    return b + 256;
}

cudaError_t launch_bitmap_isin(const int64_t* keys, int64_t n, const uint32_t* valid, const int64_t* set,
                               int64_t nset, int64_t* sorted_set, void* tmp, size_t tmp_bytes, uint32_t* out,
                               cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    cudaError_t e;
    if (nset > 0) {
        size_t tb = tmp_bytes;
        if ((e = cub::DeviceRadixSort::SortKeys(tmp, tb, set, sorted_set, (int)nset, 0, 64, s)) != cudaSuccess)
            return e;
    }
    k_bitmap_isin<<<grid_words((n + 31) / 32), 256, 0, s>>>(keys, n, valid, sorted_set, nset, out);
    return cudaGetLastError();
}

cudaError_t launch_bitmap_combine(const uint32_t* a, const uint32_t* b, int64_t nwords, int op, uint32_t* out,
                                  cudaStream_t s) {
    if (nwords == 0) return cudaSuccess;
    k_bitmap_combine<<<grid_words(nwords) * 8, 256, 0, s>>>(a, b, nwords, op, out);
    return cudaGetLastError();
}

}  // namespace vs
