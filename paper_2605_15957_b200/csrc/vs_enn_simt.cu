// Phase A of the exhaustive search, SIMT fp32 variant (small batches and the
// non-tensor fallback). Computes approximate keys
//     squared L2: ||x||^2 - 2 q.x     inner product: -q.x
// for a 128-query x 128-row tile with an 8x8 register outer product per
// thread (fp32 FMA), then streams every key of the tile through per-query
// candidate buffers: a key is appended when it is <= the
// buffer's admission threshold; a full buffer is compacted warp-
// cooperatively to "k smallest + everything within the error margin".
//
// Reference: distances.py:35-59 (pairwise) + distances.py:79-94 (select_top)
// as used by enn_search, vecindex.py:109-132. The exact float64 score and the
// tie rule are applied afterwards by the phase-B re-rank (vs_rerank.cu).
#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

namespace {
constexpr int BQ = 128;      // queries per tile
constexpr int BR = 128;      // rows per tile
constexpr int BK = 16;       // k-depth per smem stage
constexpr int NT = 256;      // threads
constexpr int TSTRIDE = BR + 2;  // key-tile row stride (conflict-free scan reads)

template <typename T>
struct Vec4 {
    __device__ static float4 load(const T* p);
};
template <>
struct Vec4<float> {
    __device__ static float4 load(const float* p) { return *reinterpret_cast<const float4*>(p); }
};
template <>
struct Vec4<__nv_bfloat16> {
    __device__ static float4 load(const __nv_bfloat16* p) {
        uint2 u = *reinterpret_cast<const uint2*>(p);
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&u.x);
        __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&u.y);
        float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
        return make_float4(fa.x, fa.y, fb.x, fb.y);
    }
};

template <typename T, bool VEC>
__device__ __forceinline__ float4 load4(const T* row, int kk, int d, bool valid) {
    if (!valid) return make_float4(0.f, 0.f, 0.f, 0.f);
    if (VEC) {
        if (kk < d) return Vec4<T>::load(row + kk);
        return make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float4 v;
    v.x = (kk + 0 < d) ? ld_elem(row + kk + 0) : 0.f;
    v.y = (kk + 1 < d) ? ld_elem(row + kk + 1) : 0.f;
    v.z = (kk + 2 < d) ? ld_elem(row + kk + 2) : 0.f;
    v.w = (kk + 3 < d) ? ld_elem(row + kk + 3) : 0.f;
    return v;
}

}  // namespace

template <typename T, bool VEC>
__global__ void __launch_bounds__(NT, 2) k_enn_scan_simt(EnnScanParams p) {
    extern __shared__ __align__(16) float smem[];
    float* As = smem;                     // [2][BK][BQ]
    float* Bs = As + 2 * BK * BQ;         // [2][BK][BR]
    float* Tk = Bs + 2 * BK * BR;         // [BQ][TSTRIDE]
    float* xs = Tk + BQ * TSTRIDE;        // [BR] row norms of the tile

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int ty = tid >> 4, tx = tid & 15;
    const int64_t q0 = (int64_t)blockIdx.x * BQ;
    const int split = blockIdx.y;
    const int64_t r_begin = (int64_t)split * p.rows_per_split;
    const int64_t r_end = min(p.nsel, r_begin + p.rows_per_split);
    const int d = p.d;
    const T* X = reinterpret_cast<const T*>(p.X);

    // scan ownership: thread -> (query row, half)
    const int srow = tid >> 1, shalf = tid & 1;
    const int64_t sq = q0 + srow;
    const bool sq_valid = sq < p.nq;
    const int C = p.cb.C;
    const int sub = split * 2 + shalf;
    const int64_t cbase = sq_valid ? ((sq * p.cb.n_sub + sub) * (int64_t)C) : 0;
    float* ckey = p.cb.key + cbase;
    uint32_t* cpos = p.cb.pos + cbase;
    const float qmargin = sq_valid ? p.margin[sq] : 0.f;
    int cnt = 0;
    float tau = __int_as_float(0x7f800000);  // +inf
    int ovf = 0;

    // loader ownership: two rows x one float4 column for A and for B
    const int lr = tid >> 2;          // 0..63
    const int lk = (tid & 3) * 4;     // 0,4,8,12
    const float* qrow0 = p.Q + min(q0 + lr, p.nq - 1) * (int64_t)d;
    const float* qrow1 = p.Q + min(q0 + lr + 64, p.nq - 1) * (int64_t)d;
    const bool qv0 = q0 + lr < p.nq, qv1 = q0 + lr + 64 < p.nq;

    for (int64_t r0 = r_begin; r0 < r_end; r0 += BR) {
        const int ncols = (int)min((int64_t)BR, r_end - r0);
        // B row pointers for this tile
        const int64_t pr0 = r0 + lr, pr1 = r0 + lr + 64;
        const bool bv0 = pr0 < r_end, bv1 = pr1 < r_end;
        const int64_t br0 = bv0 ? (p.sel ? p.sel[pr0] : pr0) : 0;
        const int64_t br1 = bv1 ? (p.sel ? p.sel[pr1] : pr1) : 0;
        const T* xrow0 = X + br0 * (int64_t)d;
        const T* xrow1 = X + br1 * (int64_t)d;
        if (tid < BR) {
            int64_t pr = r0 + tid;
            float xn = 0.f;
            if (!p.ip && pr < r_end) xn = p.xnorm[p.sel ? p.sel[pr] : pr];
            xs[tid] = xn;
        }

        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

        // prologue: stage 0
        float4 a0 = load4<float, VEC>(qrow0, lk, d, qv0);
        float4 a1 = load4<float, VEC>(qrow1, lk, d, qv1);
        float4 b0 = load4<T, VEC>(xrow0, lk, d, bv0);
        float4 b1 = load4<T, VEC>(xrow1, lk, d, bv1);
        int stage = 0;
        {
            float* as = As + stage * BK * BQ;
            float* bs = Bs + stage * BK * BR;
            as[(lk + 0) * BQ + lr] = a0.x; as[(lk + 1) * BQ + lr] = a0.y;
            as[(lk + 2) * BQ + lr] = a0.z; as[(lk + 3) * BQ + lr] = a0.w;
            as[(lk + 0) * BQ + lr + 64] = a1.x; as[(lk + 1) * BQ + lr + 64] = a1.y;
            as[(lk + 2) * BQ + lr + 64] = a1.z; as[(lk + 3) * BQ + lr + 64] = a1.w;
            bs[(lk + 0) * BR + lr] = b0.x; bs[(lk + 1) * BR + lr] = b0.y;
            bs[(lk + 2) * BR + lr] = b0.z; bs[(lk + 3) * BR + lr] = b0.w;
            bs[(lk + 0) * BR + lr + 64] = b1.x; bs[(lk + 1) * BR + lr + 64] = b1.y;
            bs[(lk + 2) * BR + lr + 64] = b1.z; bs[(lk + 3) * BR + lr + 64] = b1.w;
        }
        __syncthreads();
        for (int k0 = 0; k0 < d; k0 += BK) {
            const bool more = k0 + BK < d;
            if (more) {
                a0 = load4<float, VEC>(qrow0, k0 + BK + lk, d, qv0);
                a1 = load4<float, VEC>(qrow1, k0 + BK + lk, d, qv1);
                b0 = load4<T, VEC>(xrow0, k0 + BK + lk, d, bv0);
                b1 = load4<T, VEC>(xrow1, k0 + BK + lk, d, bv1);
            }
            const float* as = As + stage * BK * BQ;
            const float* bs = Bs + stage * BK * BR;
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                float4 x0 = *reinterpret_cast<const float4*>(as + kk * BQ + ty * 4);
                float4 x1 = *reinterpret_cast<const float4*>(as + kk * BQ + 64 + ty * 4);
                float4 y0 = *reinterpret_cast<const float4*>(bs + kk * BR + tx * 4);
                float4 y1 = *reinterpret_cast<const float4*>(bs + kk * BR + 64 + tx * 4);
                float av[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                float bv[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
            if (more) {
                stage ^= 1;
                float* as2 = As + stage * BK * BQ;
                float* bs2 = Bs + stage * BK * BR;
                as2[(lk + 0) * BQ + lr] = a0.x; as2[(lk + 1) * BQ + lr] = a0.y;
                as2[(lk + 2) * BQ + lr] = a0.z; as2[(lk + 3) * BQ + lr] = a0.w;
                as2[(lk + 0) * BQ + lr + 64] = a1.x; as2[(lk + 1) * BQ + lr + 64] = a1.y;
                as2[(lk + 2) * BQ + lr + 64] = a1.z; as2[(lk + 3) * BQ + lr + 64] = a1.w;
                bs2[(lk + 0) * BR + lr] = b0.x; bs2[(lk + 1) * BR + lr] = b0.y;
                bs2[(lk + 2) * BR + lr] = b0.z; bs2[(lk + 3) * BR + lr] = b0.w;
                bs2[(lk + 0) * BR + lr + 64] = b1.x; bs2[(lk + 1) * BR + lr + 64] = b1.y;
                bs2[(lk + 2) * BR + lr + 64] = b1.z; bs2[(lk + 3) * BR + lr + 64] = b1.w;
            }
            __syncthreads();
        }

        // epilogue: keys into the smem tile
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = (i < 4) ? (ty * 4 + i) : (64 + ty * 4 + i - 4);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int col = (j < 4) ? (tx * 4 + j) : (64 + tx * 4 + j - 4);
                float key = p.ip ? -acc[i][j] : fmaf(-2.f, acc[i][j], xs[col]);
                Tk[row * TSTRIDE + col] = key;
            }
        }
        __syncthreads();

        // candidate-buffer maintenance: make room for up to 64 appends
        {
            bool need = sq_valid && cnt > C - 64;
            unsigned m = __ballot_sync(VS_FULL, need);
            while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                const int lc = __shfl_sync(VS_FULL, cnt, l);
                const float lmar = __shfl_sync(VS_FULL, qmargin, l);
                const int lsq_lo = __shfl_sync(VS_FULL, (int)(cbase & 0xffffffff), l);
                const int lsq_hi = __shfl_sync(VS_FULL, (int)(cbase >> 32), l);
                const int64_t lbase = ((int64_t)(uint32_t)lsq_hi << 32) | (uint32_t)lsq_lo;
                float nthr = 0.f;
                int lov = 0;
                int nc = warp_compact(p.cb.key + lbase, p.cb.pos + lbase, lc, p.k, lmar, C - 64,
                                      &nthr, &lov);
                if (lane == l) {
                    cnt = nc;
                    tau = nthr;
                    ovf |= lov;
                }
            }
        }
        if (sq_valid) {
            const float* trow = Tk + srow * TSTRIDE;
#pragma unroll 4
            for (int m = 0; m < BR / 2; ++m) {
                const int c = 2 * m + shalf;
                const float key = trow[c];
                if (c < ncols && key <= tau) {
                    ckey[cnt] = key;
                    cpos[cnt] = (uint32_t)(r0 + c);
                    ++cnt;
                }
            }
        }
        __syncthreads();  // Tk / xs reuse by the next tile
    }
    if (sq_valid) {
        p.cb.cnt[sq * p.cb.n_sub + sub] = cnt;
        if (ovf) p.cb.overflow[sq] = 1;
    }
}

template <typename T>
cudaError_t launch_enn_scan_simt(const EnnScanParams& p, cudaStream_t s) {
    const size_t smem = (size_t)(2 * BK * BQ + 2 * BK * BR + BQ * TSTRIDE + BR) * sizeof(float);
    dim3 grid((unsigned)((p.nq + BQ - 1) / BQ), (unsigned)p.n_split);
    const bool vec = (p.d % 4) == 0;
    cudaError_t e;
    if (vec) {
        e = cudaFuncSetAttribute(k_enn_scan_simt<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        k_enn_scan_simt<T, true><<<grid, NT, smem, s>>>(p);
    } else {
        e = cudaFuncSetAttribute(k_enn_scan_simt<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        k_enn_scan_simt<T, false><<<grid, NT, smem, s>>>(p);
    }
    return cudaGetLastError();
}
template cudaError_t launch_enn_scan_simt<float>(const EnnScanParams&, cudaStream_t);
template cudaError_t launch_enn_scan_simt<__nv_bfloat16>(const EnnScanParams&, cudaStream_t);

}  // namespace vs
