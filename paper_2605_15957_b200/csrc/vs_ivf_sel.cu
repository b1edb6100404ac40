// Phase A of the FILTERED IVF search, list-major over pre-selected rows.
//
// With a selective filter (config 3: 1 %), a probed list of ~610 rows holds
// ~6 selected rows, and the scan is a stream of tiny, independent units:
// (list, <= 8 (query, probe) pairs) x (selected rows of the list). The
// list-major kernel (vs_ivf_lmajor.cu) spent its time on dependent global
// round trips per unit (work ticket, unit, pair codes, queries, bitmap words,
// selected positions, rows). Here every unit needs ONE:
//   1. once per search, the selected payload positions of every list are
//      compacted in list order (k_list_sel_positions: one warp per list over
//      the permuted bitmap), and every unit gets a 128-byte record with its
//      list, pair codes, selected-row count and first 16 positions
//      (k_make_recs);
//   2. a CTA walks its units in a fixed stride (no work-counter atomics); the
//      record of its NEXT unit is loaded while the current one is scored, so
//      at the top of a unit the row positions and the queries are known: the
//      selected rows (cp.async, 16 bytes, coalesced) and the unit's queries
//      (into registers) are requested together and arrive in one round trip;
//   3. scoring and candidate appends follow the list-major kernel: two
//      queries per warp held in registers, staged rows from shared memory,
//      fp32 (error bound eps_simt), one butterfly transpose-
//      reduction per chunk, per-pair candidate buffers; the
//      key is the dot form ||x||^2 - 2 q.x (one FFMA per element and query).
// Reference: IvfIndex.search, vecindex.py:230-258, with the filtered
// extension rows = rows[mask[rows]].
#include <cub/cub.cuh>
#include <type_traits>

#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

namespace {
constexpr int NT = 128;
constexpr int NW = NT / 32;
constexpr int QT = kIvfLmQT;   // pairs per unit: two per warp
constexpr int RS = 8;          // staged rows per chunk
constexpr int TMAX = kIvfLmDMax / 128;
constexpr int RPOS = 15;       // row positions carried in a unit record
static_assert(QT == 2 * NW, "two query slots per warp");

// 128-byte unit record: the pairs' queries and probe ranks pre-split (no
// integer division in the scan), the first RPOS selected row positions
struct __align__(16) UnitRec {
    int32_t list, np, nsel, first_pair;
    uint32_t sel_off;
    int32_t q[QT];
    uint16_t sub[QT];
    uint32_t pos[RPOS];
};
static_assert(sizeof(UnitRec) == 128, "one 128-byte record per unit");

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

__device__ __forceinline__ float transpose_reduce16(float (&v)[16], int lane) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int o = 16 >> s;
        const int n = 16 >> s;
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (i < n / 2) {
                const float send = upper ? v[i] : v[i + n / 2];
                const float keep = upper ? v[i + n / 2] : v[i];
                v[i] = keep + __shfl_xor_sync(VS_FULL, send, o);
            }
        }
    }
    return v[0] + __shfl_xor_sync(VS_FULL, v[0], 1);
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

__global__ void k_make_recs(const int4* __restrict__ units, const int32_t* __restrict__ n_units, int64_t max_units,
                            const int32_t* __restrict__ pair_codes, int nprobe, const int32_t* __restrict__ lsel,
                            const int64_t* __restrict__ sel_off, const uint32_t* __restrict__ spos,
                            UnitRec* __restrict__ recs) {
    const int nu = *n_units;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < max_units && u < nu;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int4 un = units[u];
        UnitRec r;
        r.list = un.x;
        r.np = un.z;
        r.first_pair = un.y;
        r.nsel = lsel[un.x];
        r.sel_off = (uint32_t)sel_off[un.x];
#pragma unroll
        for (int s = 0; s < QT; ++s) {
            const int code = s < un.z ? pair_codes[un.y + s] : 0;
            r.q[s] = code / nprobe;
            r.sub[s] = (uint16_t)(code % nprobe);
        }
#pragma unroll
        for (int i = 0; i < RPOS; ++i) r.pos[i] = i < r.nsel ? spos[r.sel_off + i] : 0u;
        recs[u] = r;
    }
}

struct SelSmem {
    UnitRec rec[2];
};
}  // namespace

struct IvfSelParams {
    const float* Q;
    int64_t nq;
    int d, dp;
    const void* payload;
    int nprobe;
    const UnitRec* recs;
    const int32_t* n_units;
    const uint32_t* spos;
    const float* pnorm;
    const float* margin;
    int ip, k;
    CandBuf cb;
    unsigned long long* visited;
};

template <typename T, bool IP>
__global__ void __launch_bounds__(NT, 4) k_ivf_scan_sel(IvfSelParams p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    SelSmem& S = *reinterpret_cast<SelSmem*>(smraw);
    T* xs = reinterpret_cast<T*>(smraw + ((sizeof(SelSmem) + 127) & ~size_t(127)));   // [RS][dp]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d = p.d, dp = p.dp, nt = dp / 128;
    const T* payload = reinterpret_cast<const T*>(p.payload);
    const int C = p.cb.C;
    const int n_units = *p.n_units;
    const int row_bytes = d * (int)sizeof(T);
    const bool v16 = (row_bytes & 15) == 0;
    unsigned long long visited = 0;
    for (int i = tid; i < RS * dp; i += NT) xs[i] = T(0.f);   // zero tail [d, dp) of every staged row
    int u = blockIdx.x;
    if (u < n_units && tid < 32) reinterpret_cast<uint32_t*>(&S.rec[0])[tid] = reinterpret_cast<const uint32_t*>(p.recs + u)[tid];
    __syncthreads();
    int cur = 0;
    for (; u < n_units; u += gridDim.x, cur ^= 1) {
        const UnitRec& R = S.rec[cur];
        const int np = R.np, nsel = R.nsel;
        const int64_t l_unused = R.list;
        (void)l_unused;
        // rows of the first chunk (positions in the record) ...
        const int nr0 = min(RS, nsel);
        for (int r = warp; r < nr0; r += NW) {   // a warp per row: coalesced, no index division
            const char* src = reinterpret_cast<const char*>(payload + (int64_t)R.pos[r] * d);
            char* dst = reinterpret_cast<char*>(xs + r * dp);
            if (v16)
                for (int o = lane * 16; o < row_bytes; o += 32 * 16) cp_async16(dst + o, src + o);
            else
                for (int o = lane * 8; o < row_bytes; o += 32 * 8) cp_async8(dst + o, src + o);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        // ... and this warp's two queries, in the same round trip
        int qidx[2], sub[2], cnt[2] = {0, 0}, ovf[2] = {0, 0};
        float tau[2];
        bool live[2];
        float4 qv[2][TMAX];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int slot = warp + h * NW;
            live[h] = slot < np;
            qidx[h] = live[h] ? R.q[slot] : 0;
            sub[h] = live[h] ? R.sub[slot] : 0;
            tau[h] = __int_as_float(0x7f800000);
            const float* qg = p.Q + (int64_t)qidx[h] * d;
#pragma unroll
            for (int t = 0; t < TMAX; ++t) {
                const int e = lane * 4 + 128 * t;
                qv[h][t] = (live[h] && e < d) ? __ldg(reinterpret_cast<const float4*>(qg + e))
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        // the next unit's record, consumed after this unit
        const int un = u + gridDim.x;
        uint32_t nrec = 0u;
        if (warp == 0 && un < n_units) nrec = reinterpret_cast<const uint32_t*>(p.recs + un)[lane];
        if (tid == 0) visited += (unsigned long long)nsel * np;
        for (int c0 = 0; c0 < nsel; c0 += RS) {
            const int nr = min(RS, nsel - c0);
            if (c0 > 0) {
                // later chunks (lists with more than RS selected rows)
                __syncthreads();   // the previous chunk's rows are consumed
                for (int r = warp; r < nr; r += NW) {
                    const int rr = c0 + r;
                    const uint32_t pos = rr < RPOS ? R.pos[rr] : p.spos[R.sel_off + rr];
                    const char* src = reinterpret_cast<const char*>(payload + (int64_t)pos * d);
                    char* dst = reinterpret_cast<char*>(xs + r * dp);
                    if (v16)
                        for (int o = lane * 16; o < row_bytes; o += 32 * 16) cp_async16(dst + o, src + o);
                    else
                        for (int o = lane * 8; o < row_bytes; o += 32 * 8) cp_async8(dst + o, src + o);
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            if (live[0]) {
                // dot form (one FFMA per element and query): every t step updates
                // 2 x RS independent accumulators; rows past nr hold stale data
                // and are scored but never appended
                float acc[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[i] = 0.f;
#pragma unroll
                for (int t = 0; t < TMAX; ++t) {
                    if (t < nt) {
#pragma unroll
                        for (int r = 0; r < RS; ++r) {
                            const float4 x = V4<T>::lds(xs + r * dp + lane * 4 + 128 * t);
                            acc[r] = fmaf(qv[0][t].x, x.x, acc[r]);
                            acc[RS + r] = fmaf(qv[1][t].x, x.x, acc[RS + r]);
                            acc[r] = fmaf(qv[0][t].y, x.y, acc[r]);
                            acc[RS + r] = fmaf(qv[1][t].y, x.y, acc[RS + r]);
                            acc[r] = fmaf(qv[0][t].z, x.z, acc[r]);
                            acc[RS + r] = fmaf(qv[1][t].z, x.z, acc[RS + r]);
                            acc[r] = fmaf(qv[0][t].w, x.w, acc[r]);
                            acc[RS + r] = fmaf(qv[1][t].w, x.w, acc[RS + r]);
                        }
                    }
                }
                const float dot = transpose_reduce16(acc, lane);   // (lane >> 1) = h * RS + r
                const int myh = (lane >> 1) / RS, myr = (lane >> 1) % RS;
                const int rr = c0 + myr;
                const uint32_t mypos = (myr < nr) ? (rr < RPOS ? R.pos[rr] : p.spos[R.sel_off + rr]) : 0u;
                // key: -q.x, or ||x||^2 - 2 q.x (the query's ||q||^2 is common to
                // all its keys; the margin eps_simt covers this form too)
                const float key = IP ? -dot : fmaf(-2.f, dot, myr < nr ? p.pnorm[mypos] : 0.f);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!live[h]) continue;
                    const int q = qidx[h];
                    const int64_t cbase = ((int64_t)q * p.cb.n_sub + sub[h]) * C;
                    float* ckey = p.cb.key + cbase;
                    uint32_t* cpos = p.cb.pos + cbase;
                    bool adm = (lane & 1) == 0 && myh == h && myr < nr && key <= tau[h];
                    unsigned b = __ballot_sync(VS_FULL, adm);
                    if (b && cnt[h] + __popc(b) > C) {
                        float nthr;
                        int lov = 0;
                        cnt[h] = compact_slow_sel(ckey, cpos, cnt[h], p.k, p.margin[q], C - 32, &nthr, &lov);
                        tau[h] = nthr;
                        ovf[h] |= lov;
                        adm = adm && key <= tau[h];
                        b = __ballot_sync(VS_FULL, adm);
                    }
                    if (adm) {
                        const int slot = cnt[h] + __popc(b & lanemask_lt());
                        ckey[slot] = key;
                        cpos[slot] = mypos;
                    }
                    cnt[h] += __popc(b);
                }
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (!live[h]) continue;
                p.cb.cnt[(int64_t)qidx[h] * p.cb.n_sub + sub[h]] = cnt[h];
                if (ovf[h]) p.cb.overflow[qidx[h]] = 1;
            }
        }
        if (warp == 0) reinterpret_cast<uint32_t*>(&S.rec[cur ^ 1])[lane] = nrec;
        __syncthreads();   // next record visible; staged rows free
    }
    if (tid == 0 && visited) atomicAdd(p.visited, visited);
}

// ---- tensor-core variant (mma.sync m16n8k16, fp16 operands) ---------------------------------
// The same filtered scan with the dot products on the tensor cores: a unit is
// (list, <= 16 pairs); its queries (fp16, per-query power-of-two scales, staged
// once per search by k_stage_queries) are the MMA's A tile (16 x d), the
// list's selected rows, converted to fp16 with the column scale while they
// are staged, its B tiles (8 rows x d). The four warps split K, their fp32
// partial tiles are summed through shared memory, and the keys
// ||x||^2 - 2 (q~.x~) 2^-(eq+ex) go to the pairs' buffers. Keys carry the
// tensor-core error bound (fp16 rounding of both operands, fp32 accumulation;
// DESIGN.md §4.1); the IVF phase B uses that margin. Row-side rounding errors
// are bounded a priori (|dx_i| <= 2^-11 |x_i| + 2^-25 / 2^ex), so no pass
// over the rows is needed for the margin.
namespace {
constexpr int MQ = kMmaPairs;   // pairs per unit (MMA M)
constexpr int MN = 8;           // rows per chunk (MMA N)
constexpr int MW = 4;           // warps; K is split across them
constexpr int MNT = MW * 32;
constexpr int MPOS = 19;
constexpr int MV = 2048 / 128;  // float4 loads per lane for a row of d <= 2048

// 256-byte unit record: everything a unit needs before its first load (the
// pairs' queries, probe ranks and key factors, the first MPOS row positions),
// so staging starts without dependent global loads; the next unit's record is
// read while this one is scored
struct __align__(16) MmaRec {
    int32_t list, np, nsel, first_pair;
    uint32_t sel_off;
    int32_t q[MQ];
    uint16_t sub[MQ];
    float ks[MQ];               // -2 kinv (L2) or -kinv (IP)
    uint32_t pos[MPOS];
};
static_assert(sizeof(MmaRec) == 256, "one 256-byte record per unit");

__global__ void k_make_mma_recs(const int4* __restrict__ units, const int32_t* __restrict__ n_units,
                                int64_t max_units, const int32_t* __restrict__ lsel,
                                const int64_t* __restrict__ sel_off, const uint32_t* __restrict__ spos,
                                const int32_t* __restrict__ pair_codes, int nprobe, const float* __restrict__ kinv,
                                int ip, MmaRec* __restrict__ recs) {
    const int nu = *n_units;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < max_units && u < nu;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int4 un = units[u];
        MmaRec r;
        r.list = un.x;
        r.np = un.z;
        r.first_pair = un.y;
        r.nsel = lsel[un.x];
        r.sel_off = (uint32_t)sel_off[un.x];
#pragma unroll
        for (int s = 0; s < MQ; ++s) {
            const bool live = s < un.z;
            const int code = live ? pair_codes[un.y + s] : 0;
            r.q[s] = code / nprobe;
            r.sub[s] = (uint16_t)(code % nprobe);
            const float kv = live ? kinv[r.q[s]] : 0.f;
            r.ks[s] = ip ? -kv : -2.f * kv;
        }
#pragma unroll
        for (int i = 0; i < MPOS; ++i) r.pos[i] = i < r.nsel ? spos[r.sel_off + i] : 0u;
        recs[u] = r;
    }
}

__device__ __forceinline__ float mma_pow2_scale(float norm2) {
    const float n = sqrtf(norm2);
    if (!(n > 0.f) || !isfinite(n)) return 1.f;
    int e;
    frexpf(n * 1.001f, &e);
    return ldexpf(1.f, max(-120, min(120, 14 - e)));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x2(uint32_t (&r)[2], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void mma_16816(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
}  // namespace

struct IvfMmaParams {
    const __half* Qh;           // [nq][d] fp16 queries
    const float* kinv;          // [nq]
    const unsigned* xscale;     // max ||x||^2 of the payload (row scale)
    int d;
    const float* payload;
    int nprobe;
    const MmaRec* recs;
    const int32_t* n_units;
    const uint32_t* spos;
    const float* pnorm;
    const float* margin;
    int ip, k;
    CandBuf cb;
    unsigned long long* visited;
};

template <bool IP>
__global__ void __launch_bounds__(MNT, 4) k_ivf_scan_mma(IvfMmaParams p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int d = p.d, ld = d + 8;   // staged row stride (halves): +16 B keeps ldmatrix conflict-free
    __half* As = reinterpret_cast<__half*>(smraw);                   // [MQ][ld]
    __half* Bs = As + MQ * ld;                                       // [MN][ld]
    float* red = reinterpret_cast<float*>(Bs + MN * ld);             // [MW][32][4] partial tiles
    float* keys = red + MW * 32 * 4;                                 // [MQ][MN]
    float* xn_s = keys + MQ * MN;                                    // [MN]
    uint32_t* pos_s = reinterpret_cast<uint32_t*>(xn_s + MN);        // [MN]
    int* cnt_s = reinterpret_cast<int*>(pos_s + MN);                 // [MQ]
    MmaRec* recb = reinterpret_cast<MmaRec*>(cnt_s + MQ);            // [2]: this unit's and the next one's
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = p.cb.C;
    const int n_units = *p.n_units;
    const float sx = mma_pow2_scale(__uint_as_float(*p.xscale));
    const int ksteps = d / 16;
    unsigned long long visited = 0;
    for (int i = tid; i < (MQ + MN) * ld; i += MNT) As[i] = __float2half(0.f);
    constexpr int RW = (int)(sizeof(MmaRec) / 4);   // record words (64: two per lane)
    if (warp == 0 && (int)blockIdx.x < n_units)
        for (int i = lane; i < RW; i += 32)
            reinterpret_cast<uint32_t*>(&recb[0])[i] = reinterpret_cast<const uint32_t*>(p.recs + blockIdx.x)[i];
    int cur = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, cur ^= 1) {
        __syncthreads();   // previous unit consumed; this unit's record in recb[cur]
        const MmaRec* rec = &recb[cur];
        const int np = rec->np, nsel = rec->nsel;
        // A: the unit's queries (16-byte cp.async from the fp16 copy)
        for (int r = warp; r < np; r += MW) {   // a warp per query row
            const __half* src = p.Qh + (int64_t)rec->q[r] * d;
            for (int c8 = lane; c8 < d / 8; c8 += 32) cp_async16(As + r * ld + c8 * 8, src + c8 * 8);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (tid < MQ) cnt_s[tid] = 0;
        // the next unit's record (registers, stored to recb[cur ^ 1] after this
        // unit) and its rows -> L2 (one bulk prefetch per row)
        const int un = u + gridDim.x;
        uint32_t nw0 = 0u, nw1 = 0u;
        if (warp == MW - 1 && un < n_units) {
            const uint32_t* nr = reinterpret_cast<const uint32_t*>(p.recs + un);
            nw0 = nr[lane];
            nw1 = nr[lane + 32];
            const int nsel_n = __shfl_sync(VS_FULL, (int)nw0, 2);
            const int j = lane + 32 - (int)(offsetof(MmaRec, pos) / 4);   // word lane + 32 holds pos[j]
            if (j >= 0 && j < min(nsel_n, MPOS))
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.payload + (int64_t)nw1 * d),
                             "r"(d * 4)
                             : "memory");
        }
        if (tid == 0) visited += (unsigned long long)nsel * np;
        for (int c0 = 0; c0 < nsel; c0 += MN) {
            const int nr = min(MN, nsel - c0);
            if (c0 > 0) __syncthreads();   // previous chunk's B tile and keys consumed
            // B: warp w converts rows w and w + 4 (float4 loads, scaled to fp16)
            for (int r = warp; r < MN; r += MW) {
                __half* dst = Bs + r * ld;
                if (r < nr) {
                    const int rr = c0 + r;
                    const uint32_t pos = rr < MPOS ? rec->pos[rr] : __ldg(p.spos + rec->sel_off + rr);
                    const float4* src = reinterpret_cast<const float4*>(p.payload + (int64_t)pos * d);
                    // the row norm and all of the lane's loads in flight before the first conversion
                    const float xnv = IP || lane != 0 ? 0.f : __ldg(p.pnorm + pos);
                    float4 v[MV];
#pragma unroll
                    for (int j = 0; j < MV; ++j) {
                        const int c4 = lane + 32 * j;
                        v[j] = c4 < d / 4 ? __ldg(src + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int j = 0; j < MV; ++j) {
                        const int c4 = lane + 32 * j;
                        if (c4 < d / 4) {
                            const __half2 a = __floats2half2_rn(v[j].x * sx, v[j].y * sx);
                            const __half2 b = __floats2half2_rn(v[j].z * sx, v[j].w * sx);
                            uint2 w2;
                            w2.x = *reinterpret_cast<const uint32_t*>(&a);
                            w2.y = *reinterpret_cast<const uint32_t*>(&b);
                            *reinterpret_cast<uint2*>(dst + c4 * 4) = w2;
                        }
                    }
                    if (lane == 0) {
                        pos_s[r] = pos;
                        xn_s[r] = xnv;
                    }
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            // MMA: this warp's K slice
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            const int a_row = lane & 15, a_col = (lane >> 4) * 8;   // ldmatrix x4: 16 rows x (2 x 8) cols
            const int b_row = lane & 7, b_col = ((lane >> 3) & 1) * 8;
            for (int ks = warp; ks < ksteps; ks += MW) {
                uint32_t a[4], b[2];
                ldsm_x4(a, As + a_row * ld + ks * 16 + a_col);
                ldsm_x2(b, Bs + b_row * ld + ks * 16 + b_col);
                mma_16816(acc, a, b);
            }
            *reinterpret_cast<float4*>(red + (warp * 32 + lane) * 4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
            __syncthreads();
            if (warp == 0) {
                float4 s4 = *reinterpret_cast<const float4*>(red + lane * 4);
#pragma unroll
                for (int w = 1; w < MW; ++w) {
                    const float4 t4 = *reinterpret_cast<const float4*>(red + (w * 32 + lane) * 4);
                    s4.x += t4.x; s4.y += t4.y; s4.z += t4.z; s4.w += t4.w;
                }
                // lane (g, t): pairs g and g + 8, rows 2t and 2t + 1
                const int g = lane >> 2, t = lane & 3;
                const float v[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int pr = g + (j >> 1) * 8, rw = 2 * t + (j & 1);
                    const float ks = pr < np ? rec->ks[pr] : 0.f;
                    keys[pr * MN + rw] = IP ? v[j] * ks : fmaf(ks, v[j], xn_s[rw]);
                }
            }
            __syncthreads();
            // appends: warp w serves pairs w, w + 4, ...; lane r holds row r
            for (int pr = warp; pr < np; pr += MW) {
                const int q = rec->q[pr];
                const int64_t bidx = (int64_t)q * p.cb.n_sub + rec->sub[pr];
                float* ckey = p.cb.key + bidx * C;
                uint32_t* cpos = p.cb.pos + bidx * C;
                int cnt = cnt_s[pr];
                const float key = lane < nr ? keys[pr * MN + lane] : 0.f;
                bool adm = lane < nr;
                if (cnt + nr > C) {   // full: keep the local top-k + margin band first
                    float nthr;
                    int lov = 0;
                    cnt = compact_slow_sel(ckey, cpos, cnt, p.k, p.margin[q], C - 32, &nthr, &lov);
                    if (lov && lane == 0) p.cb.overflow[q] = 1;
                    adm = adm && key <= nthr;
                }
                const unsigned b = __ballot_sync(VS_FULL, adm);
                if (adm) {
                    const int slot = cnt + __popc(b & lanemask_lt());
                    ckey[slot] = key;
                    cpos[slot] = pos_s[lane];
                }
                __syncwarp();   // every lane's read of cnt_s[pr] is ordered before lane 0's write
                if (lane == 0) cnt_s[pr] = cnt + __popc(b);
            }
        }
        __syncthreads();
        if (tid < np) p.cb.cnt[(int64_t)rec->q[tid] * p.cb.n_sub + rec->sub[tid]] = cnt_s[tid];
        if (warp == MW - 1 && un < n_units) {
            reinterpret_cast<uint32_t*>(&recb[cur ^ 1])[lane] = nw0;
            reinterpret_cast<uint32_t*>(&recb[cur ^ 1])[lane + 32] = nw1;
        }
    }
    if (tid == 0 && visited) atomicAdd(p.visited, visited);
}

// a priori bounds of the fp16 rows: max ||x~||^2 and max ||dx||^2 (float bits)
// for k_tc_margins, from the payload's max ||x||^2
__global__ void k_f16_row_bounds(const unsigned* __restrict__ xmax, int d, unsigned* __restrict__ out) {
    const float x2 = __uint_as_float(*xmax);
    const float sx = mma_pow2_scale(x2);
    const float xn = sqrtf(x2) * 1.0001f;
    const float dx = (xn * 4.8828125e-4f + sqrtf((float)d) * 2.9802322e-8f / sx) * 1.0001f;   // 2^-11, 2^-25
    const float xt = xn + dx;
    out[0] = __float_as_uint(xt * xt);
    out[1] = __float_as_uint(dx * dx);
}

size_t ivf_mma_smem(int d) {
    const size_t ld = (size_t)d + 8;
    return (MQ + MN) * ld * 2 + (size_t)MW * 32 * 4 * 4 + (size_t)MQ * MN * 4 + (size_t)MN * 8 + (size_t)MQ * 16 +
           2 * sizeof(MmaRec) + 64;
}

cudaError_t launch_f16_row_bounds(const unsigned* xmax, int d, unsigned* out, cudaStream_t s) {
    k_f16_row_bounds<<<1, 1, 0, s>>>(xmax, d, out);
    return cudaGetLastError();
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
    if (a.mma) {
        if (std::is_same<T, float>::value == false) return cudaErrorInvalidValue;
        MmaRec* mrecs = reinterpret_cast<MmaRec*>(a.recs);
        const int rb = (int)std::max<int64_t>(1, std::min<int64_t>((a.max_units + 255) / 256, 8192));
        k_make_mma_recs<<<rb, 256, 0, s>>>(a.units, a.n_units, a.max_units, a.lsel, a.sel_off, a.spos, a.pair_codes,
                                           a.nprobe, a.kinv, a.ip, mrecs);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        IvfMmaParams m;
        m.Qh = a.Qh;
        m.kinv = a.kinv;
        m.xscale = a.xscale;
        m.d = a.d;
        m.payload = reinterpret_cast<const float*>(a.payload);
        m.nprobe = a.nprobe;
        m.recs = mrecs;
        m.n_units = a.n_units;
        m.spos = a.spos;
        m.pnorm = a.pnorm;
        m.margin = a.margin;
        m.ip = a.ip;
        m.k = a.k;
        m.cb = a.cb;
        m.visited = a.visited;
        const size_t smem = ivf_mma_smem(a.d);
        auto kern = a.ip ? k_ivf_scan_mma<true> : k_ivf_scan_mma<false>;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
            return e;
        int per_sm = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, MNT, smem)) != cudaSuccess) return e;
        const int64_t grid = std::min<int64_t>((int64_t)a.sm_count * std::max(per_sm, 1), a.max_units);
        kern<<<(unsigned)std::max<int64_t>(grid, 1), MNT, smem, s>>>(m);
        return cudaGetLastError();
    }
    UnitRec* recs = reinterpret_cast<UnitRec*>(a.recs);
    const int rb = (int)std::max<int64_t>(1, std::min<int64_t>((a.max_units + 255) / 256, 8192));
    k_make_recs<<<rb, 256, 0, s>>>(a.units, a.n_units, a.max_units, a.pair_codes, a.nprobe, a.lsel, a.sel_off, a.spos,
                                   recs);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    IvfSelParams p;
    p.Q = a.Q;
    p.nq = a.nq;
    p.d = a.d;
    p.dp = (a.d + 127) / 128 * 128;
    p.payload = a.payload;
    p.nprobe = a.nprobe;
    p.recs = recs;
    p.n_units = a.n_units;
    p.spos = a.spos;
    p.pnorm = a.pnorm;
    p.margin = a.margin;
    p.ip = a.ip;
    p.k = a.k;
    p.cb = a.cb;
    p.visited = a.visited;
    const size_t smem = ((sizeof(SelSmem) + 127) & ~size_t(127)) + (size_t)RS * p.dp * sizeof(T);
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
