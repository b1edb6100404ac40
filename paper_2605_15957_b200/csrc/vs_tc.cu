// Phase A of the exhaustive search on the 5th-generation tensor cores.
//
//   D[q, r] = sum_k A[q, k] * B[r, k]      A = queries, B = selected rows (bf16)
//
// is a real dense contraction (queries x embeddings), so it runs as a
// warp-specialised tcgen05 GEMM: TMA streams 128B-swizzled K-major bf16
// tiles of A (128 queries x 64) and B (256 rows x 64) into a 4-stage
// shared-memory ring, one elected thread issues tcgen05.mma (M=128, N=256,
// K=16, fp32 accumulate) into a double-buffered TMEM accumulator
// (2 x 256 columns), and four epilogue warps drain TMEM with tcgen05.ld.
// The epilogue never writes the score matrix: each thread owns one query row
// (TMEM lane) and streams its 256 keys
//     squared L2: ||x||^2 - 2 q.x      inner product: -q.x
// through that row's candidate buffer. A per-query global
// admission threshold (atomicMin of the best "k-th key + margin" any split
// has proven) prunes all splits. The exact float64 scores and the tie rule
// are applied by phase B (vs_rerank.cu) on the survivors.
//
// Reference: pairwise (distances.py:35-59) + select_top (distances.py:79-94)
// inside enn_search (vecindex.py:109-132).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>

#include "vs_common.cuh"
#include "vs_kernels.cuh"
#include "vs_tc.cuh"

namespace vs {

namespace tc {

constexpr int BM = 128;                 // queries per tile (UMMA M)
constexpr int BN = 256;                 // rows per tile (UMMA N)
constexpr int BK = 64;                  // bf16 elements per stage = 128 B (swizzle atom)
constexpr int UK = 16;                  // UMMA K for kind::f16
constexpr int NSTAGE = 4;
constexpr int A_BYTES = BM * BK * 2;    // 16 KB
constexpr int B_BYTES = BN * BK * 2;    // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NTHREADS = 256;           // 8 warps
constexpr int EPI_WARP0 = 4;            // warps 4..7 drain TMEM lanes 0..127
constexpr int TMEM_COLS = 512;          // 2 accumulators x 256 fp32 columns

struct Smem {
    // stage buffers live at the 1024-aligned start of dynamic smem
    uint64_t full[NSTAGE];
    uint64_t empty[NSTAGE];
    uint64_t tfull[2];
    uint64_t tempty[2];
    uint32_t tmem_base;
    float xn[2][BN];
};
constexpr size_t SMEM_BYTES = 1024 + (size_t)NSTAGE * STAGE_BYTES + sizeof(Smem);

struct Params {
    int64_t nq;
    int d;                    // true dimension
    int kblocks;              // ceil(d / 64)
    int64_t nsel;             // rows
    int qtiles;
    int nsplit;
    int64_t tiles_per_split;  // data tiles of BN rows per split
    int64_t ntiles;           // total data tiles
    const float* xn;          // [nsel] row norms (staged order)
    const float* margin;      // [nq]
    unsigned* tau_g;          // [nq] orderable global admission threshold
    int ip;
    int k;
    CandBuf cb;
};

// ---- PTX helpers ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128B-swizzled operand descriptor (canonical layout ((8,n),2):((8,SBO),1)
// in 16-byte units: 8-row atoms of 1024 B, SBO = 1024 B, LBO unused = 1)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version (sm100)
    d |= (uint64_t)2 << 61;   // SWIZZLE_128B
    return d;
}
// instruction descriptor: kind::f16, A/B = BF16, D = F32, K-major both, M=128, N=256
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

#define TMEM_LD32(taddr, r)                                                                         \
    asm volatile(                                                                                   \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"              \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),       \
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),   \
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),             \
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),             \
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])              \
        : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- the kernel --------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHREADS, 1)
    k_enn_scan_tc(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                  Params p) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    Smem& S = *reinterpret_cast<Smem*>(base + (size_t)NSTAGE * STAGE_BYTES);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        prefetch_map(&map_a);
        prefetch_map(&map_b);
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&S.tfull[i], 1);
            mbar_init(&S.tempty[i], BM);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    const int64_t nitems = (int64_t)p.qtiles * p.nsplit;
    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
                const int qt = (int)(it % p.qtiles);
                const int64_t s = it / p.qtiles;
                const int64_t t0 = s * p.tiles_per_split;
                const int64_t t1 = min(p.ntiles, t0 + p.tiles_per_split);
                for (int64_t t = t0; t < t1; ++t) {
                    for (int kb = 0; kb < p.kblocks; ++kb) {
                        mbar_wait(&S.empty[stage], phase ^ 1);
                        unsigned char* sa = base + (size_t)stage * STAGE_BYTES;
                        mbar_expect_tx(&S.full[stage], STAGE_BYTES);
                        tma_load_2d(sa, &map_a, &S.full[stage], kb * BK, qt * BM);
                        tma_load_2d(sa + A_BYTES, &map_b, &S.full[stage], kb * BK, (int)(t * BN));
                        if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (single thread) =====
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t tcount = 0;
            for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
                const int64_t s = it / p.qtiles;
                const int64_t t0 = s * p.tiles_per_split;
                const int64_t t1 = min(p.ntiles, t0 + p.tiles_per_split);
                for (int64_t t = t0; t < t1; ++t, ++tcount) {
                    const uint32_t acc = tcount & 1, aph = (tcount >> 1) & 1;
                    mbar_wait(&S.tempty[acc], aph ^ 1);
                    tc_fence_after();
                    const uint32_t dt = tmem + acc * BN;
                    for (int kb = 0; kb < p.kblocks; ++kb) {
                        mbar_wait(&S.full[stage], phase);
                        tc_fence_after();
                        const uint32_t sa = smem_u32(base + (size_t)stage * STAGE_BYTES);
                        const uint32_t sb = sa + A_BYTES;
#pragma unroll
                        for (int kk = 0; kk < BK / UK; ++kk) {
                            mma_bf16(dt, desc_sw128(sa + kk * UK * 2), desc_sw128(sb + kk * UK * 2), idesc,
                                     (kb | kk) != 0);
                        }
                        mma_commit(&S.empty[stage]);
                        if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
                    }
                    mma_commit(&S.tfull[acc]);
                }
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ===== epilogue: TMEM -> keys -> candidate buffers =====
        const int et = threadIdx.x - EPI_WARP0 * 32;     // 0..127 == TMEM lane == tile row
        const int quad = warp - EPI_WARP0;               // lane quadrant
        const int C = p.cb.C;
        uint32_t tcount = 0;
        for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
            const int qt = (int)(it % p.qtiles);
            const int64_t s = it / p.qtiles;
            const int64_t t0 = s * p.tiles_per_split;
            const int64_t t1 = min(p.ntiles, t0 + p.tiles_per_split);
            const int64_t q = (int64_t)qt * BM + et;
            const bool qv = q < p.nq;
            const int64_t cbase = qv ? ((q * p.cb.n_sub + s) * (int64_t)C) : 0;
            float* ckey = p.cb.key + cbase;
            uint32_t* cpos = p.cb.pos + cbase;
            const float qmargin = qv ? p.margin[q] : 0.f;
            int cnt = 0;
            int ovf = 0;
            float tau = __int_as_float(0x7f800000);
            for (int64_t t = t0; t < t1; ++t, ++tcount) {
                const uint32_t acc = tcount & 1, aph = (tcount >> 1) & 1;
                const int64_t r0 = t * BN;
                const int ncols = (int)min((int64_t)BN, p.nsel - r0);
                // stage the tile's row norms (L2) while the MMA runs
                float* xs = S.xn[acc];
                if (!p.ip) {
                    for (int c = et; c < BN; c += BM) xs[c] = (c < ncols) ? p.xn[r0 + c] : 0.f;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (qv) tau = fminf(tau, o2f(p.tau_g[q]));
                mbar_wait(&S.tfull[acc], aph);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + acc * BN;
#pragma unroll 1
                for (int ch = 0; ch < BN / 32; ++ch) {
                    // room for 32 appends; compact full buffers warp-cooperatively
                    {
                        unsigned m = __ballot_sync(VS_FULL, qv && cnt > C - 32);
                        while (m) {
                            const int l = __ffs(m) - 1;
                            m &= m - 1;
                            const int lc = __shfl_sync(VS_FULL, cnt, l);
                            const float lmar = __shfl_sync(VS_FULL, qmargin, l);
                            const int lo32 = __shfl_sync(VS_FULL, (int)(cbase & 0xffffffff), l);
                            const int hi32 = __shfl_sync(VS_FULL, (int)(cbase >> 32), l);
                            const int64_t lb = ((int64_t)(uint32_t)hi32 << 32) | (uint32_t)lo32;
                            float nthr = 0.f;
                            int lov = 0;
                            const int nc = warp_compact(p.cb.key + lb, p.cb.pos + lb, lc, p.k, lmar, C - 32,
                                                        &nthr, &lov);
                            if (lane == l) {
                                cnt = nc;
                                tau = fminf(tau, nthr);
                                ovf |= lov;
                                atomicMin(&p.tau_g[q], f2o(tau));
                            }
                        }
                    }
                    uint32_t r[32];
                    TMEM_LD32(taddr + ch * 32, r);
                    tmem_wait_ld();
                    if (qv) {
                        const int cb0 = ch * 32;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int c = cb0 + j;
                            const float a = __uint_as_float(r[j]);
                            const float key = p.ip ? -a : fmaf(-2.f, a, xs[c]);
                            if (c < ncols && key <= tau) {
                                ckey[cnt] = key;
                                cpos[cnt] = (uint32_t)(r0 + c);
                                ++cnt;
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(&S.tempty[acc]);
            }
            if (qv) {
                p.cb.cnt[q * p.cb.n_sub + s] = cnt;
                if (ovf) p.cb.overflow[q] = 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
    }
}

// ---- operand staging -----------------------------------------------------------------------------------
// queries fp32 -> bf16 (round to nearest even), row stride dp
__global__ void k_stage_queries(const float* __restrict__ q, int64_t nq, int d, int dp,
                                __nv_bfloat16* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t tot = nq * (int64_t)dp;
    for (; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / dp;
        const int c = (int)(i - r * dp);
        out[i] = __float2bfloat16_rn(c < d ? q[r * (int64_t)d + c] : 0.f);
    }
}
// selected rows -> contiguous bf16 [nsel][dp] + their norms (warp per row)
template <typename T>
__global__ void k_stage_rows(const T* __restrict__ x, const int64_t* __restrict__ sel, int64_t nsel, int d,
                             int dp, const float* __restrict__ norms, __nv_bfloat16* __restrict__ out,
                             float* __restrict__ xn) {
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (; w < nsel; w += nw) {
        const int64_t r = sel ? sel[w] : w;
        const T* src = x + r * (int64_t)d;
        __nv_bfloat16* dst = out + w * (int64_t)dp;
        if (sizeof(T) == 4 && (d % 4) == 0 && (dp % 4) == 0) {
            for (int c = lane * 4; c < dp; c += 128) {
                float4 v = (c < d) ? *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(src) + c)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y);
                __nv_bfloat162 b = __floats2bfloat162_rn(v.z, v.w);
                uint2 u;
                u.x = *reinterpret_cast<uint32_t*>(&a);
                u.y = *reinterpret_cast<uint32_t*>(&b);
                *reinterpret_cast<uint2*>(dst + c) = u;
            }
        } else {
            for (int c = lane; c < dp; c += 32) dst[c] = __float2bfloat16_rn(c < d ? ld_elem(src + c) : 0.f);
        }
        if (lane == 0 && xn) xn[w] = norms[r];
    }
}

__global__ void k_tc_margins(const float* __restrict__ q, int64_t nq, int d, const unsigned* __restrict__ xmax,
                             float cqx, float cxx, float* __restrict__ margin) {
    const int lane = threadIdx.x & 31;
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= nq) return;
    float s = 0.f;
    for (int i = lane; i < d; i += 32) {
        float v = q[r * (int64_t)d + i];
        s = fmaf(v, v, s);
    }
    s = warp_sumf(s);
    if (lane == 0) {
        const float qn = sqrtf(s) * 1.0001f;
        const float xn = sqrtf(__uint_as_float(*xmax)) * 1.0001f;
        margin[r] = cqx * qn * xn + cxx * xn * xn;
    }
}

}  // namespace tc

// ---- host side ---------------------------------------------------------------------------------------------

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool get_encode() {
    if (g_encode) return true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !fn) {
        cudaGetLastError();
        return false;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    return true;
}

bool make_map(CUtensorMap* map, const void* gaddr, int64_t rows, int d, int dp, int box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)std::max<int64_t>(rows, 1)};
    cuuint64_t strides[1] = {(cuuint64_t)dp * 2};
    cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(gaddr), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
}  // namespace

bool tc_supported(int d, int dtype, int ip) {
    (void)dtype;
    (void)ip;
    return d >= 8 && get_encode();
}

bool tc_profitable(int64_t nq, int64_t nsel, int d) {
    return nq >= 64 && (double)nq * (double)nsel * (double)d >= 4.0e9;
}

// bf16 error bound of the tensor-core key:
//   |q~.x~ - q.x| <= (2^-8 + 2^-18) |q| |x|  (RN to bf16, Cauchy-Schwarz)
//   + fp32 accumulation inside the tensor core (bounded by 2^-14 |q| |x|),
// key = ||x||^2 - 2 q.x adds the fp32 norm error (d + 2) 2^-24 |x|^2;
// margin = 2 x bound, with a 5% safety factor.
static void tc_margin_coeffs(int d, int ip, float* cqx, float* cxx) {
    const double edot = (std::ldexp(1.0, -8) + std::ldexp(1.0, -18) + std::ldexp(1.0, -14)) * 1.05;
    if (ip) {
        *cqx = (float)(2.0 * edot);
        *cxx = 0.f;
    } else {
        *cqx = (float)(2.0 * 2.0 * edot);
        *cxx = (float)(2.0 * (d + 2) * std::ldexp(1.0, -24) * 1.05);
    }
}

int tc_enn_scan(vs_ctx* ctx, EnnScanParams& sp, int dtype, const unsigned* xmax, int cshift, CandBuf* cb,
                bool* exhaustive) {
    using namespace vs_internal;
    cudaStream_t st = ctx->stream;
    const int d = sp.d;
    const int dp = (d + 7) / 8 * 8;
    const int64_t nq = sp.nq, nsel = sp.nsel;
    // staging buffers
    __nv_bfloat16 *qa = nullptr, *xb = nullptr;
    float *xn = nullptr, *margin = nullptr;
    unsigned* tau_g = nullptr;
    CKS(arena_alloc(ctx, (size_t)nq * dp, &qa));
    CKS(arena_alloc(ctx, (size_t)nsel * dp, &xb));
    CKS(arena_alloc(ctx, (size_t)nsel, &xn));
    CKS(arena_alloc(ctx, (size_t)nq, &margin));
    CKS(arena_alloc(ctx, (size_t)nq, &tau_g));
    {
        KTimer kt(ctx, VS_K_STAGE);
        int64_t tot = nq * (int64_t)dp;
        tc::k_stage_queries<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 32), 256, 0, st>>>(
            sp.Q, nq, d, dp, qa);
        CK(cudaGetLastError());
        const unsigned blocks = (unsigned)std::min<int64_t>((nsel * 32 + 255) / 256, 148 * 64);
        if (dtype == VS_DTYPE_F32)
            tc::k_stage_rows<float><<<blocks, 256, 0, st>>>((const float*)sp.X, sp.sel, nsel, d, dp, sp.xnorm, xb,
                                                            sp.ip ? nullptr : xn);
        else
            tc::k_stage_rows<__nv_bfloat16><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)sp.X, sp.sel, nsel, d,
                                                                    dp, sp.xnorm, xb, sp.ip ? nullptr : xn);
        CK(cudaGetLastError());
        float cqx, cxx;
        tc_margin_coeffs(d, sp.ip, &cqx, &cxx);
        tc::k_tc_margins<<<(unsigned)((nq * 32 + 255) / 256), 256, 0, st>>>(sp.Q, nq, d, xmax, cqx, cxx, margin);
        CK(cudaGetLastError());
        CK(cudaMemsetAsync(tau_g, 0xff, nq * sizeof(unsigned), st));
        ctx->stats[VS_STAT_LAUNCHES] += 3;
    }
    // tiling: work item = (query tile, data split); choose the split count
    // so items fill whole waves of SMs
    const int qtiles = (int)((nq + tc::BM - 1) / tc::BM);
    const int64_t ntiles = (nsel + tc::BN - 1) / tc::BN;
    const int sms = ctx->sm_count;
    int best_s = 1;
    double best_cost = 1e30;
    const int smin = std::max(1, (int)std::min<int64_t>(ntiles, (2 * sms + qtiles - 1) / qtiles));
    for (int s = smin; s <= std::min<int64_t>(ntiles, (int64_t)smin * 4); ++s) {
        const int64_t per = (ntiles + s - 1) / s;
        const int64_t items = (int64_t)qtiles * ((ntiles + per - 1) / per);
        const double waves = std::ceil((double)items / sms);
        const double cost = waves * per + 0.02 * s * per / 8.0;  // makespan (+ small phase-B cost per split)
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best_s = s;
        }
    }
    const int64_t per = (ntiles + best_s - 1) / best_s;
    const int nsplit = (int)((ntiles + per - 1) / per);
    int64_t C = vs_internal::pow2ceil(std::max<int64_t>(4 * sp.k, sp.k + 160)) << (ctx->opt_slack + cshift);
    const int64_t rows_per_split = per * tc::BN;
    const int64_t cap = vs_internal::pow2ceil(rows_per_split + 64);
    *exhaustive = C >= cap;
    if (C > cap) C = cap;
    CandBuf c;
    c.n_sub = nsplit;
    c.C = (int)C;
    const size_t slots = (size_t)nq * nsplit * C;
    CKS(arena_alloc(ctx, slots, &c.key));
    CKS(arena_alloc(ctx, slots, &c.pos));
    CKS(arena_alloc(ctx, (size_t)nq * nsplit, &c.cnt));
    CKS(arena_alloc(ctx, (size_t)nq, &c.overflow));
    CK(cudaMemsetAsync(c.overflow, 0, nq * sizeof(int), st));

    CUtensorMap ma, mb;
    if (!make_map(&ma, qa, nq, d, dp, tc::BM) || !make_map(&mb, xb, nsel, d, dp, tc::BN))
        return set_err(VS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    tc::Params pr;
    pr.nq = nq;
    pr.d = d;
    pr.kblocks = (d + tc::BK - 1) / tc::BK;
    pr.nsel = nsel;
    pr.qtiles = qtiles;
    pr.nsplit = nsplit;
    pr.tiles_per_split = per;
    pr.ntiles = ntiles;
    pr.xn = xn;
    pr.margin = margin;
    pr.tau_g = tau_g;
    pr.ip = sp.ip;
    pr.k = sp.k;
    pr.cb = c;
    CK(cudaFuncSetAttribute(tc::k_enn_scan_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::SMEM_BYTES));
    const int64_t items = (int64_t)qtiles * nsplit;
    const unsigned grid = (unsigned)std::min<int64_t>(items, sms);
    tc::k_enn_scan_tc<<<grid, tc::NTHREADS, tc::SMEM_BYTES, st>>>(ma, mb, pr);
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    // phase B reads rows through the selection (sp.sel) from the original
    // column, with the tensor-core margins
    sp.margin = margin;
    sp.tau_g = tau_g;
    *cb = c;
    return VS_OK;
}

}  // namespace vs
