// Phase A of the FILTERED IVF search, list-major over pre-selected rows.
//
// With a selective filter (config 3: 1 %), a probed list of ~610 rows holds
// ~6 selected rows and is probed by ~20 queries: per list, a handful of rows
// against a few dozen queries. The work is tiny (2 GFMA per batch); what
// costs is latency, so:
//   1. once per search, the selected payload positions of every list are
//      compacted in list order (k_list_sel_positions: one warp per list over
//      the permuted bitmap);
//   2. a work unit is a whole list (all its pairs, <= kSelUnitPairs): its
//      selected rows are staged ONCE into shared memory (cp.async, one warp
//      per row, 8 rows per chunk) while the previous chunk is scored - a
//      double buffer across chunks and units;
//   3. each warp takes the unit's pairs in turn, its query in registers (the
//      next pair's query loaded while the current one is scored), one FFMA
//      per element and row, an 8-row transpose-reduction, and appends the
//      keys ||x||^2 - 2 q.x (dot form; error within eps_simt) to the pair's
//      candidate buffer, which only this warp touches during the unit.
// Reference: IvfIndex.search, vecindex.py:230-258, with the filtered
// extension rows = rows[mask[rows]].
#include <cub/cub.cuh>

#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

namespace {
constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int RS = 8;          // staged rows per chunk (one warp stages one row)
constexpr int TMAX = kIvfLmDMax / 128;
static_assert(RS == NW, "one staging warp per row");

template <typename T>
struct V4;
template <>
struct V4<float> {
    static __device__ __forceinline__ float4 lds(const float* p) { return *reinterpret_cast<const float4*>(p); }
};
template <>
struct V4<__nv_bfloat16> {
    static __device__ __forceinline__ float4 lds(const __nv_bfloat16* p) {
        const uint2 u = *reinterpret_cast<const uint2*>(p);
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        return make_float4(a.x, a.y, b.x, b.y);
    }
};

// v[r] (r < 8) partial sums per lane -> lanes 4r..4r+3 hold the warp total of
// row r (r = (lane >> 2) & 7): three halving exchanges, then two folds
__device__ __forceinline__ float transpose_reduce8(float (&v)[8], int lane) {
#pragma unroll
    for (int s = 0; s < 3; ++s) {
        const int o = 16 >> s;
        const int n = 8 >> s;
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i < n / 2) {
                const float send = upper ? v[i] : v[i + n / 2];
                const float keep = upper ? v[i + n / 2] : v[i];
                v[i] = keep + __shfl_xor_sync(VS_FULL, send, o);
            }
        }
    }
    float t = v[0] + __shfl_xor_sync(VS_FULL, v[0], 2);
    return t + __shfl_xor_sync(VS_FULL, t, 1);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}

__device__ __noinline__ int compact_slow_sel(float* keys, uint32_t* pos, int n, int k, float margin, int limit,
                                             float* thr, int* overflow) {
    return warp_compact(keys, pos, n, k, margin, limit, thr, overflow);
}

// selected payload positions of every list, ascending, at sel_off[l]
__global__ void k_list_sel_positions(const int64_t* __restrict__ list_off, int nlist,
                                     const uint32_t* __restrict__ pbits, const int64_t* __restrict__ sel_off,
                                     uint32_t* __restrict__ spos) {
    const int lane = threadIdx.x & 31;
    for (int l = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; l < nlist; l += (gridDim.x * blockDim.x) >> 5) {
        const int64_t a = list_off[l], b = list_off[l + 1];
        int64_t out = sel_off[l];
        for (int64_t r0 = a; r0 < b; r0 += 32 * 32) {
            const int64_t r = r0 + lane * 32;
            uint32_t bits = 0u;
            if (r < b) {
                const int sh = (int)(r & 31);
                const uint32_t lo = pbits[r >> 5];
                const uint32_t hi = sh ? pbits[(r >> 5) + 1] : 0u;
                bits = __funnelshift_r(lo, hi, sh);
                const int64_t nb = b - r;
                if (nb < 32) bits &= (1u << nb) - 1u;
            }
            const int c = __popc(bits);
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(VS_FULL, incl, o);
                if (lane >= o) incl += t;
            }
            int64_t w = out + incl - c;
            while (bits) {
                const int bb = __ffs(bits) - 1;
                bits &= bits - 1;
                spos[w++] = (uint32_t)(r + bb);
            }
            out += __shfl_sync(VS_FULL, incl, 31);
        }
    }
}
}  // namespace

struct IvfSelParams {
    const float* Q;
    int64_t nq;
    int d, dp;
    const void* payload;
    int nprobe;
    const int4* units;          // (list, first pair, pairs, 0), grouped by list
    const int32_t* n_units;
    const int32_t* pair_codes;  // q * nprobe + probe rank
    const int32_t* lsel;        // selected rows per list
    const int64_t* sel_off;
    const uint32_t* spos;
    const float* pnorm;
    const float* margin;
    int ip, k;
    CandBuf cb;
    unsigned long long* visited;
};

template <typename T, bool IP>
__global__ void __launch_bounds__(NT, 2) k_ivf_scan_sel(IvfSelParams p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    T* xs = reinterpret_cast<T*>(smraw);   // [2][RS][dp]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d = p.d, dp = p.dp, nt = dp / 128;
    const T* payload = reinterpret_cast<const T*>(p.payload);
    const int C = p.cb.C;
    const int n_units = *p.n_units;
    const int row_bytes = d * (int)sizeof(T);
    const bool v16 = (row_bytes & 15) == 0;
    for (int i = tid; i < 2 * RS * dp; i += NT) xs[i] = T(0.f);   // zero tails [d, dp)
    __syncthreads();
    unsigned long long visited = 0;
    // chunk sequence of this CTA: (unit u, row chunk c); warp `warp` stages row
    // `warp` of a chunk into buffer b
    auto stage = [&](int u, int c, int b) {
        if (u < n_units) {
            const int4 un = __ldg(p.units + u);
            const int ns = __ldg(p.lsel + un.x);
            const int r = c * RS + warp;
            if (r < ns) {
                const uint32_t pos = __ldg(p.spos + __ldg(p.sel_off + un.x) + r);
                const char* src = reinterpret_cast<const char*>(payload + (int64_t)pos * d);
                char* dst = reinterpret_cast<char*>(xs + ((size_t)b * RS + warp) * dp);
                if (v16)
                    for (int o = lane * 16; o < row_bytes; o += 32 * 16) cp_async16(dst + o, src + o);
                else
                    for (int o = lane * 8; o < row_bytes; o += 32 * 8) cp_async8(dst + o, src + o);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int u = blockIdx.x, c = 0, buf = 0;
    stage(u, 0, 0);
    while (u < n_units) {
        const int4 un = __ldg(p.units + u);
        const int nsel = __ldg(p.lsel + un.x);
        const int np = un.z;
        const int nchunk = (nsel + RS - 1) / RS;
        // the next chunk: this unit's next, else the next unit's first
        const int nu = (c + 1 < nchunk) ? u : u + gridDim.x;
        const int nc = (c + 1 < nchunk) ? c + 1 : 0;
        stage(nu, nc, buf ^ 1);
        if (tid == 0 && c == 0) visited += (unsigned long long)nsel * np;
        const int nr = min(RS, nsel - c * RS);
        const int64_t soff = __ldg(p.sel_off + un.x) + (int64_t)c * RS;
        // this warp's first pair: its query is requested before the barrier
        int slot = warp;
        float4 qv[TMAX];
        auto load_q = [&](int sl, float4 (&dst)[TMAX]) {
            const int code = __ldg(p.pair_codes + un.y + sl);
            const float* qg = p.Q + (int64_t)(code / p.nprobe) * d;
#pragma unroll
            for (int t = 0; t < TMAX; ++t) {
                const int e = lane * 4 + 128 * t;
                dst[t] = (t < nt && e < d) ? __ldg(reinterpret_cast<const float4*>(qg + e))
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        if (nr > 0 && slot < np) load_q(slot, qv);
        // my row of this chunk (lanes 4r..4r+3 own row r after the reduction)
        const int myr = (lane >> 2) & 7;
        uint32_t mypos = 0u;
        float mynorm = 0.f;
        if (nr > 0 && myr < nr) {
            mypos = __ldg(p.spos + soff + myr);
            if (!IP) mynorm = __ldg(p.pnorm + mypos);
        }
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();   // chunk `buf` landed for every warp
        const T* xb = xs + (size_t)buf * RS * dp;
        for (; nr > 0 && slot < np; slot += NW) {
            float4 qn[TMAX];
            const bool more = slot + NW < np;
            if (more) load_q(slot + NW, qn);   // next pair's query, in flight during the dot products
            float acc[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) acc[r] = 0.f;
#pragma unroll
            for (int t = 0; t < TMAX; ++t) {
                if (t < nt) {
#pragma unroll
                    for (int r = 0; r < RS; ++r) {
                        const float4 x = V4<T>::lds(xb + r * dp + lane * 4 + 128 * t);
                        acc[r] = fmaf(qv[t].x, x.x, acc[r]);
                        acc[r] = fmaf(qv[t].y, x.y, acc[r]);
                        acc[r] = fmaf(qv[t].z, x.z, acc[r]);
                        acc[r] = fmaf(qv[t].w, x.w, acc[r]);
                    }
                }
            }
            const float dot = transpose_reduce8(acc, lane);
            const float key = IP ? -dot : fmaf(-2.f, dot, mynorm);
            const int code = __ldg(p.pair_codes + un.y + slot);
            const int q = code / p.nprobe;
            const int64_t bidx = (int64_t)q * p.cb.n_sub + code % p.nprobe;
            float* ckey = p.cb.key + bidx * C;
            uint32_t* cpos = p.cb.pos + bidx * C;
            // the buffer belongs to this warp for the whole unit (pairs partition
            // the units; the slot -> warp map is the same for every chunk)
            int cnt = c == 0 ? 0 : __ldcg(p.cb.cnt + bidx);
            bool adm = (lane & 3) == 0 && myr < nr;
            unsigned b = __ballot_sync(VS_FULL, adm);
            if (cnt + __popc(b) > C) {
                float nthr;
                int lov = 0;
                cnt = compact_slow_sel(ckey, cpos, cnt, p.k, p.margin[q], C - 32, &nthr, &lov);
                if (lov && lane == 0) p.cb.overflow[q] = 1;
                adm = adm && key <= nthr;
                b = __ballot_sync(VS_FULL, adm);
            }
            if (adm) {
                const int s = cnt + __popc(b & lanemask_lt());
                ckey[s] = key;
                cpos[s] = mypos;
            }
            if (lane == 0) p.cb.cnt[bidx] = cnt + __popc(b);
            if (more) {
#pragma unroll
                for (int t = 0; t < TMAX; ++t) qv[t] = qn[t];
            }
        }
        __syncthreads();   // chunk `buf` consumed before it is restaged
        buf ^= 1;
        u = nu;
        c = nc;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (tid == 0 && visited) atomicAdd(p.visited, visited);
}

// setup (per search) + the scan; counts / sel_off / spos / recs are scratch
// sized by the caller (ivf_sel_scratch)
size_t ivf_sel_temp_bytes(int nlist) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, nlist + 1);
    return b + 256;
}

__global__ void k_widen_counts(const int32_t* __restrict__ c, int n, int64_t* __restrict__ w) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) w[i] = i < n ? c[i] : 0;
}

template <typename T>
cudaError_t launch_ivf_scan_sel(const IvfSelLaunch& a, cudaStream_t s) {
    if (a.nq == 0) return cudaSuccess;
    cudaError_t e;
    // per-list selected counts -> offsets -> positions
    const int lb = std::max(1, std::min((a.nlist * 32 + 255) / 256, 4096));
    k_list_selected<<<lb, 256, 0, s>>>(a.list_off, a.nlist, a.pbits, a.lsel);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    k_widen_counts<<<(a.nlist + 256) / 256, 256, 0, s>>>(a.lsel, a.nlist, a.lsel64);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    size_t tb = a.tmp_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(a.tmp, tb, a.lsel64, a.sel_off, a.nlist + 1, s)) != cudaSuccess) return e;
    k_list_sel_positions<<<lb, 256, 0, s>>>(a.list_off, a.nlist, a.pbits, a.sel_off, a.spos);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    IvfSelParams p;
    p.Q = a.Q;
    p.nq = a.nq;
    p.d = a.d;
    p.dp = (a.d + 127) / 128 * 128;
    p.payload = a.payload;
    p.nprobe = a.nprobe;
    p.units = a.units;
    p.n_units = a.n_units;
    p.pair_codes = a.pair_codes;
    p.lsel = a.lsel;
    p.sel_off = a.sel_off;
    p.spos = a.spos;
    p.pnorm = a.pnorm;
    p.margin = a.margin;
    p.ip = a.ip;
    p.k = a.k;
    p.cb = a.cb;
    p.visited = a.visited;
    const size_t smem = (size_t)2 * RS * p.dp * sizeof(T);
    auto kern = a.ip ? k_ivf_scan_sel<T, true> : k_ivf_scan_sel<T, false>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return e;
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem)) != cudaSuccess) return e;
    const int64_t grid = std::min<int64_t>((int64_t)a.sm_count * std::max(per_sm, 1), a.max_units);
    kern<<<(unsigned)std::max<int64_t>(grid, 1), NT, smem, s>>>(p);
    return cudaGetLastError();
}
template cudaError_t launch_ivf_scan_sel<float>(const IvfSelLaunch&, cudaStream_t);
template cudaError_t launch_ivf_scan_sel<__nv_bfloat16>(const IvfSelLaunch&, cudaStream_t);

}  // namespace vs
