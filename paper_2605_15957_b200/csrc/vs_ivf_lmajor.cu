// Phase A of the IVF search, list-major: every probed list is read once per
// unit of up to QT queries that probe it (once per batch for lists probed by
// <= QT queries), instead of once per (query, probe) pair.
//
// The (query, probe) pairs of the batch are grouped by list (CUB radix sort on
// the list id, stable, so a list's queries stay in query order) and cut into
// work units of <= QT pairs of one list. A CTA takes units from an atomic work
// counter. For a unit:
//   1. every warp loads its two queries (slots w and w + NW) into registers,
//      lane-strided by 4 elements (128-bit loads, zero padded to 128),
//   2. the list is walked in segments of SEG rows: the permuted bitmap word of
//      every 32 payload rows (bit = filter[list_ids[pos]]) is tested in
//      registers and the selected positions are compacted into shared memory
//      before any row byte is loaded,
//   3. selected rows are staged into shared memory RS at a time with 16-byte
//      cp.async (coalesced), and each warp scores its two queries against all
//      staged rows (fp32 direct form, the same arithmetic and error bound as
//      the query-major scan); the 2 x RS partial sums are finished by one
//      butterfly transpose-reduction (lane = slot * RS + row),
//   4. the keys are appended to the pair's candidate buffer (query q, sub =
//      probe rank j) by the warp that owns the query: admission key <= tau,
//      compaction to local top-k + margin when the buffer fills.
// Every pair has its own buffer and exactly one writer warp.
//
// Reference: IvfIndex.search, vecindex.py:230-258 (probe loop 242-257), with
// the filtered extension rows = rows[mask[rows]].
#include <cub/cub.cuh>

#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

namespace {
constexpr int NT = 128;
constexpr int NW = NT / 32;
constexpr int QT = kIvfLmQT;   // queries per unit (two per warp)
constexpr int RS = 8;          // staged rows per chunk
constexpr int SEG = 2048;      // payload rows per selection segment
constexpr int TMAX = kIvfLmDMax / 128;
static_assert(QT == 2 * NW, "two query slots per warp");
static_assert(2 * RS == 16, "one 16-value transpose-reduction per chunk");

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
    static __device__ __forceinline__ float4 ldg(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
    static __device__ __forceinline__ float4 lds(const float* p) { return *reinterpret_cast<const float4*>(p); }
};
template <>
struct Vec4<__nv_bfloat16> {
    static __device__ __forceinline__ float4 cvt(uint2 u) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        return make_float4(a.x, a.y, b.x, b.y);
    }
    static __device__ __forceinline__ float4 ldg(const __nv_bfloat16* p) {
        return cvt(__ldg(reinterpret_cast<const uint2*>(p)));
    }
    static __device__ __forceinline__ float4 lds(const __nv_bfloat16* p) {
        return cvt(*reinterpret_cast<const uint2*>(p));
    }
};

template <bool IP>
__device__ __forceinline__ float term4(float acc, const float4 q, const float4 x) {
    if (IP) {
        acc = fmaf(q.x, x.x, acc); acc = fmaf(q.y, x.y, acc);
        acc = fmaf(q.z, x.z, acc); acc = fmaf(q.w, x.w, acc);
    } else {
        float t;
        t = q.x - x.x; acc = fmaf(t, t, acc);
        t = q.y - x.y; acc = fmaf(t, t, acc);
        t = q.z - x.z; acc = fmaf(t, t, acc);
        t = q.w - x.w; acc = fmaf(t, t, acc);
    }
    return acc;
}

// butterfly transpose-reduction of 16 values: lanes L and L^1 end with the
// warp sum of v[(L >> 1) & 15]
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

// the rare buffer-full path, kept out of line so the scoring loop keeps its
// registers (queries live in registers across the whole unit)
__device__ __noinline__ int compact_slow(float* keys, uint32_t* pos, int n, int k, float margin, int limit,
                                         float* thr, int* overflow) {
    return warp_compact(keys, pos, n, k, margin, limit, thr, overflow);
}

struct UnitSmem {
    int unit;
    int list;
    int pbeg;
    int np;
    int nsel;
    int warp_tot[2];
    int spos[SEG];      // selected list-relative positions of the current segment
};
}  // namespace

template <typename T, bool IP>
__global__ void __launch_bounds__(NT, 4) k_ivf_scan_lmajor(IvfLmParams p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    UnitSmem& S = *reinterpret_cast<UnitSmem*>(smraw);
    T* xs = reinterpret_cast<T*>(smraw + ((sizeof(UnitSmem) + 127) & ~size_t(127)));  // [RS][dp]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d = p.d, dp = p.dp;
    const T* payload = reinterpret_cast<const T*>(p.payload);
    const int C = p.cb.C;
    const int n_units = *p.n_units;
    const int row_bytes = d * (int)sizeof(T);
    const bool v16 = (row_bytes & 15) == 0;
    const int piece = v16 ? 16 : 8;
    const int pieces = row_bytes / piece;
    unsigned long long visited = 0;
    // the staged rows' tail [d, dp) stays zero for the whole kernel
    for (int i = tid; i < RS * dp; i += NT) xs[i] = T(0.f);

    for (;;) {
        __syncthreads();
        if (tid == 0) S.unit = atomicAdd(p.work, 1);
        __syncthreads();
        const int u = S.unit;
        if (u >= n_units) break;
        const int4 un = p.units[u];
        const int l = un.x, np = un.z;
        // 1. this warp's two query slots -> registers
        int qidx[2], sub[2], cnt[2] = {0, 0}, ovf[2] = {0, 0};
        float tau[2];
        bool live[2];
        float4 qv[2][TMAX];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int slot = warp + h * NW;
            live[h] = slot < np;
            const int code = live[h] ? p.pair_codes[un.y + slot] : 0;
            qidx[h] = code / p.nprobe;
            sub[h] = code % p.nprobe;
            tau[h] = __int_as_float(0x7f800000);
            const float* qg = p.Q + (int64_t)qidx[h] * d;
#pragma unroll
            for (int t = 0; t < TMAX; ++t) {
                const int e = lane * 4 + 128 * t;
                qv[h][t] = (live[h] && e < d) ? __ldg(reinterpret_cast<const float4*>(qg + e))
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        const int nt = dp / 128;
        const int64_t off = p.list_off[l];
        const int64_t nl = p.list_off[l + 1] - off;
        for (int64_t s0 = 0; s0 < nl; s0 += SEG) {
            // 2. selected positions of this segment -> shared memory (ascending)
            const int64_t seg_n = min((int64_t)SEG, nl - s0);
            if (warp < 2) {
                const int wi = warp * 32 + lane;   // word of the segment
                const int64_t r0 = s0 + (int64_t)wi * 32;
                uint32_t bits = 0u;
                if (r0 < s0 + seg_n) {
                    const int64_t a = off + r0;
                    const int nb = (int)min((int64_t)32, s0 + seg_n - r0);
                    if (p.pbits) {
                        const int64_t w0 = a >> 5;
                        const int sh = (int)(a & 31);
                        const uint32_t lo = p.pbits[w0];
                        const uint32_t hi = sh ? p.pbits[w0 + 1] : 0u;
                        bits = __funnelshift_r(lo, hi, sh);
                    } else {
                        bits = VS_FULL;
                    }
                    if (nb < 32) bits &= (1u << nb) - 1u;
                }
                const int c = __popc(bits);
                int incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(VS_FULL, incl, o);
                    if (lane >= o) incl += t;
                }
                if (lane == 31) S.warp_tot[warp] = incl;
                asm volatile("bar.sync 1, 64;" ::: "memory");
                int base = incl - c + (warp == 1 ? S.warp_tot[0] : 0);
                const int rel = (int)r0;
                while (bits) {
                    const int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    S.spos[base++] = rel + b;
                }
                if (warp == 1 && lane == 31) S.nsel = S.warp_tot[0] + S.warp_tot[1];
            }
            __syncthreads();
            const int nsel = S.nsel;
            visited += (unsigned long long)nsel * np;
            for (int c0 = 0; c0 < nsel; c0 += RS) {
                const int nr = min(RS, nsel - c0);
                // 3. stage nr selected rows (coalesced cp.async)
                for (int i = tid; i < nr * pieces; i += NT) {
                    const int r = i / pieces, pc = i - r * pieces;
                    const char* src = reinterpret_cast<const char*>(payload + (off + S.spos[c0 + r]) * (int64_t)d) +
                                      pc * piece;
                    char* dst = reinterpret_cast<char*>(xs + r * dp) + pc * piece;
                    if (v16) cp_async16(dst, src);
                    else cp_async8(dst, src);
                }
                asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
                __syncthreads();
                if (live[0]) {
                    float acc[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
#pragma unroll
                    for (int r = 0; r < RS; ++r) {
                        if (r < nr) {
                            const T* xr = xs + r * dp + lane * 4;
#pragma unroll
                            for (int t = 0; t < TMAX; ++t) {
                                if (t < nt) {
                                    const float4 x = Vec4<T>::lds(xr + 128 * t);
                                    acc[r] = term4<IP>(acc[r], qv[0][t], x);
                                    acc[RS + r] = term4<IP>(acc[RS + r], qv[1][t], x);
                                }
                            }
                        }
                    }
                    const float tot = transpose_reduce16(acc, lane);   // (lane >> 1) = h * RS + r
                    const float key = IP ? -tot : tot;
                    const int myh = (lane >> 1) / RS, myr = (lane >> 1) % RS;
                    // 4. append (the warp owns both slots' buffers)
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
                            cnt[h] = compact_slow(ckey, cpos, cnt[h], p.k, p.margin[q], C - 32, &nthr, &lov);
                            tau[h] = nthr;
                            ovf[h] |= lov;
                            adm = adm && key <= tau[h];
                            b = __ballot_sync(VS_FULL, adm);
                        }
                        if (adm) {
                            const int slot = cnt[h] + __popc(b & lanemask_lt());
                            ckey[slot] = key;
                            cpos[slot] = (uint32_t)(off + S.spos[c0 + myr]);
                        }
                        cnt[h] += __popc(b);
                    }
                }
                __syncthreads();   // staged rows / positions are reused
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
    }
    if (tid == 0 && visited) atomicAdd(p.visited, visited);
}

// ---- pair grouping --------------------------------------------------------------------------
namespace {
__global__ void k_pair_keys(const int32_t* __restrict__ probes, int64_t npairs, int nlist,
                            const uint8_t* __restrict__ owned, int32_t* __restrict__ keys,
                            int32_t* __restrict__ vals, int32_t* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npairs;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int l = probes[i];
        const bool own = owned == nullptr || owned[l];
        keys[i] = own ? l : nlist;
        vals[i] = (int32_t)i;
        if (own) atomicAdd(&cnt[l], 1);
    }
}

__global__ void k_unit_counts(const int32_t* __restrict__ cnt, int nlist, int qt, const int32_t* __restrict__ chunks,
                              int32_t* __restrict__ ucnt) {
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l <= nlist; l += gridDim.x * blockDim.x)
        ucnt[l] = l < nlist ? (cnt[l] + qt - 1) / qt * (chunks ? chunks[l] : 1) : 0;
}

// per query: its flat buffer count 2 * sum_j chunks(probe j); per pair: its base
__global__ void k_pair_subs(const int32_t* __restrict__ probes, int64_t nq, int nprobe,
                            const int32_t* __restrict__ chunks, int64_t* __restrict__ qsubs,
                            int64_t* __restrict__ pair_base) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t acc = 0;
        for (int j = 0; j < nprobe; ++j) {
            pair_base[q * nprobe + j] = acc;   // relative; made absolute below
            acc += 2 * (int64_t)chunks[probes[q * nprobe + j]];
        }
        qsubs[q] = acc;
    }
}
__global__ void k_pair_subs_abs(const int64_t* __restrict__ sub_off, int64_t nq, int nprobe,
                                int64_t* __restrict__ pair_base) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq * nprobe;
         i += (int64_t)gridDim.x * blockDim.x)
        pair_base[i] += sub_off[i / nprobe];
}

// units of one list split its pairs evenly (sizes differ by at most one), times
// its row chunks
__global__ void k_write_units(const int32_t* __restrict__ cnt, const int32_t* __restrict__ qoff,
                              const int32_t* __restrict__ uoff, int nlist, const int32_t* __restrict__ chunks,
                              int4* __restrict__ units) {
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlist; l += gridDim.x * blockDim.x) {
        const int n = cnt[l];
        const int ch = chunks ? chunks[l] : 1;
        const int nu = (uoff[l + 1] - uoff[l]) / ch;   // pair groups
        int b = qoff[l];
        int u = uoff[l];
        for (int j = 0; j < nu; ++j) {
            const int m = n / nu + (j < n % nu ? 1 : 0);
            for (int c = 0; c < ch; ++c) units[u++] = make_int4(l, b, m, c);
            b += m;
        }
    }
}
}  // namespace

// visited rows (vecindex.py:253, filtered: the rows left after the filter):
// selected rows per list (warp per list), then a sum over the owned pairs
__global__ void k_list_selected(const int64_t* __restrict__ list_off, int nlist, const uint32_t* __restrict__ pbits,
                                int32_t* __restrict__ sel) {
    const int lane = threadIdx.x & 31;
    for (int l = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; l < nlist; l += (gridDim.x * blockDim.x) >> 5) {
        const int64_t a = list_off[l], b = list_off[l + 1];
        int c = 0;
        if (!pbits) {
            c = (int)(b - a);
        } else {
            for (int64_t r = a + lane * 32; r < b; r += 32 * 32) {
                const int sh = (int)(r & 31);
                const uint32_t lo = pbits[r >> 5];
                const uint32_t hi = sh ? pbits[(r >> 5) + 1] : 0u;
                uint32_t bits = __funnelshift_r(lo, hi, sh);
                const int64_t nb = b - r;
                if (nb < 32) bits &= (1u << nb) - 1u;
                c += __popc(bits);
            }
            c = __reduce_add_sync(VS_FULL, c);
        }
        if (lane == 0) sel[l] = c;
    }
}
__global__ void k_visited_pairs(const int32_t* __restrict__ probes, int64_t npairs, const uint8_t* __restrict__ owned,
                                const int32_t* __restrict__ sel, unsigned long long* __restrict__ visited) {
    unsigned long long v = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npairs; i += (int64_t)gridDim.x * blockDim.x) {
        const int l = probes[i];
        if (!owned || owned[l]) v += (unsigned long long)sel[l];
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(VS_FULL, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(visited, v);
}

cudaError_t launch_visited_count(const int32_t* probes, int64_t nq, int nprobe, const int64_t* list_off, int nlist,
                                 const uint8_t* list_owned, const uint32_t* pbits, int32_t* sel_scratch,
                                 unsigned long long* visited, cudaStream_t s) {
    const int lb = std::max(1, std::min((nlist * 32 + 255) / 256, 4096));
    k_list_selected<<<lb, 256, 0, s>>>(list_off, nlist, pbits, sel_scratch);
    const int64_t np = nq * (int64_t)nprobe;
    const int pb = (int)std::max<int64_t>(1, std::min<int64_t>((np + 255) / 256, 2048));
    k_visited_pairs<<<pb, 256, 0, s>>>(probes, np, list_owned, sel_scratch, visited);
    return cudaGetLastError();
}

size_t ivf_group_temp_bytes(int64_t npairs, int nlist) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)npairs, 0, 32);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr, nlist + 1);
    return std::max(a, b) + 256;
}

cudaError_t launch_ivf_group(const IvfGroupArgs& g, cudaStream_t s) {
    cudaError_t e;
    const int64_t npairs = g.nq * (int64_t)g.nprobe;
    if ((e = cudaMemsetAsync(g.cnt, 0, (g.nlist + 1) * sizeof(int32_t), s)) != cudaSuccess) return e;
    const int blocks = (int)std::min<int64_t>((npairs + 255) / 256, 4096);
    k_pair_keys<<<std::max(blocks, 1), 256, 0, s>>>(g.probes, npairs, g.nlist, g.owned, g.keys_in, g.vals_in,
                                                    g.cnt);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    int end_bit = 1;
    while ((1ll << end_bit) <= g.nlist) ++end_bit;
    size_t tb = g.tmp_bytes;
    if ((e = cub::DeviceRadixSort::SortPairs(g.tmp, tb, g.keys_in, g.keys_out, g.vals_in, g.pair_codes,
                                             (int)npairs, 0, end_bit, s)) != cudaSuccess)
        return e;
    tb = g.tmp_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(g.tmp, tb, g.cnt, g.qoff, g.nlist + 1, s)) != cudaSuccess) return e;
    const int lb = std::max(1, std::min((g.nlist + 256) / 256, 1024));
    k_unit_counts<<<lb, 256, 0, s>>>(g.cnt, g.nlist, g.unit_pairs, g.chunks, g.ucnt);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    tb = g.tmp_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(g.tmp, tb, g.ucnt, g.uoff, g.nlist + 1, s)) != cudaSuccess) return e;
    k_write_units<<<lb, 256, 0, s>>>(g.cnt, g.qoff, g.uoff, g.nlist, g.chunks, g.units);
    return cudaGetLastError();
}

size_t ivf_pair_subs_temp_bytes(int64_t nq) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)(nq + 1));
    return b + 256 + (size_t)(nq + 1) * sizeof(int64_t);
}

cudaError_t launch_ivf_pair_subs(const int32_t* probes, int64_t nq, int nprobe, const int32_t* chunks,
                                 int64_t* sub_off, int64_t* pair_base, void* tmp, size_t tmp_bytes,
                                 cudaStream_t s) {
    cudaError_t e;
    int64_t* qsubs = reinterpret_cast<int64_t*>(tmp);
    void* scan_tmp = reinterpret_cast<char*>(tmp) + ((size_t)(nq + 1) * sizeof(int64_t) + 255) / 256 * 256;
    size_t tb = tmp_bytes - ((size_t)(nq + 1) * sizeof(int64_t) + 255) / 256 * 256;
    if ((e = cudaMemsetAsync(qsubs + nq, 0, sizeof(int64_t), s)) != cudaSuccess) return e;
    const int b = (int)std::max<int64_t>(1, std::min<int64_t>((nq + 255) / 256, 1024));
    k_pair_subs<<<b, 256, 0, s>>>(probes, nq, nprobe, chunks, qsubs, pair_base);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cub::DeviceScan::ExclusiveSum(scan_tmp, tb, qsubs, sub_off, (int)(nq + 1), s)) != cudaSuccess) return e;
    const int b2 = (int)std::max<int64_t>(1, std::min<int64_t>((nq * nprobe + 255) / 256, 4096));
    k_pair_subs_abs<<<b2, 256, 0, s>>>(sub_off, nq, nprobe, pair_base);
    return cudaGetLastError();
}

int64_t ivf_max_units(int64_t nq, int nprobe, int nlist, int unit_pairs) {
    return (nq * (int64_t)nprobe + unit_pairs - 1) / unit_pairs + nlist;
}

size_t ivf_lmajor_smem(int dp, int dtype_bytes) {
    return ((sizeof(UnitSmem) + 127) & ~size_t(127)) + (size_t)RS * dp * dtype_bytes;
}

template <typename T>
cudaError_t launch_ivf_scan_lmajor(const IvfLmParams& p, int sm_count, cudaStream_t s) {
    if (p.nq == 0) return cudaSuccess;
    const size_t smem = ivf_lmajor_smem(p.dp, (int)sizeof(T));
    cudaError_t e;
    auto kern = p.ip ? k_ivf_scan_lmajor<T, true> : k_ivf_scan_lmajor<T, false>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return e;
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem)) != cudaSuccess) return e;
    const int64_t grid = std::min<int64_t>((int64_t)sm_count * std::max(per_sm, 1), p.max_units);
    kern<<<(unsigned)std::max<int64_t>(grid, 1), NT, smem, s>>>(p);
    return cudaGetLastError();
}
template cudaError_t launch_ivf_scan_lmajor<float>(const IvfLmParams&, int, cudaStream_t);
template cudaError_t launch_ivf_scan_lmajor<__nv_bfloat16>(const IvfLmParams&, int, cudaStream_t);

}  // namespace vs
