// Phase A of the IVF search: scan of the probed lists over the compacted,
// list-contiguous payload (the owning layout of vecindex.py:203-204 / the SVIX
// payload of vecindex.py:526-530) with the relational filter applied as a
// predicate BEFORE a row's bytes are loaded.
//
// Query-major variant: one CTA per (query, probe split); every warp walks
// 32-row words of the probed lists, reads the word of the permuted bitmap
// (bit = filter[list_ids[pos]]), and only issues loads for set rows. Each
// selected row is scored by the whole warp in fp32 direct form
// (sum (q - x)^2 / sum q*x, 128-bit coalesced loads) and pushed through the
// warp's candidate buffer.
//
// Reference: IvfIndex.search, vecindex.py:230-258 (probe loop 242-257), with
// the filtered extension rows = rows[mask[rows]].
#include "vs_common.cuh"
#include "vs_kernels.cuh"

namespace vs {

namespace {
constexpr int NT = 256;
constexpr int NW = NT / 32;
}

template <typename T, bool VEC, bool IP>
__device__ __forceinline__ float row_key(const float* qs, const T* x, int d, int lane) {
    float s = 0.f;
    if (VEC) {
        for (int i = lane * 4; i < d; i += 128) {
            float4 qv = *reinterpret_cast<const float4*>(qs + i);
            float4 xv;
            if (sizeof(T) == 4) {
                xv = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(x) + i);
            } else {
                uint2 u = *reinterpret_cast<const uint2*>(x + i);
                float2 fa = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
                float2 fb = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
                xv = make_float4(fa.x, fa.y, fb.x, fb.y);
            }
            if (IP) {
                s = fmaf(qv.x, xv.x, s); s = fmaf(qv.y, xv.y, s);
                s = fmaf(qv.z, xv.z, s); s = fmaf(qv.w, xv.w, s);
            } else {
                float t0 = qv.x - xv.x, t1 = qv.y - xv.y, t2 = qv.z - xv.z, t3 = qv.w - xv.w;
                s = fmaf(t0, t0, s); s = fmaf(t1, t1, s); s = fmaf(t2, t2, s); s = fmaf(t3, t3, s);
            }
        }
    } else {
        for (int i = lane; i < d; i += 32) {
            float a = qs[i], b = ld_elem(x + i);
            if (IP) s = fmaf(a, b, s);
            else { float t = a - b; s = fmaf(t, t, s); }
        }
    }
    s = warp_sumf(s);
    return IP ? -s : s;
}

template <typename T, bool VEC, bool IP>
__global__ void __launch_bounds__(NT) k_ivf_scan_qmajor(IvfScanParams p) {
    extern __shared__ __align__(16) float qs[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t q = blockIdx.x;
    const int ps = blockIdx.y;
    const int d = p.d;
    for (int i = threadIdx.x; i < d; i += NT) qs[i] = p.Q[q * (int64_t)d + i];
    __syncthreads();

    const T* payload = reinterpret_cast<const T*>(p.payload);
    const int C = p.cb.C;
    const int sub = ps * NW + warp;
    const int64_t cbase = (q * p.cb.n_sub + sub) * (int64_t)C;
    float* ckey = p.cb.key + cbase;
    uint32_t* cpos = p.cb.pos + cbase;
    const float margin = p.margin[q];
    int cnt = 0;
    float tau = __int_as_float(0x7f800000);
    int ovf = 0;
    unsigned long long visited = 0;

    const int per = (p.nprobe + p.n_psplit - 1) / p.n_psplit;
    const int pb = ps * per, pe = min(p.nprobe, pb + per);
    for (int pi = pb; pi < pe; ++pi) {
        const int l = p.probes[q * p.nprobe + pi];
        if (p.list_owned && !p.list_owned[l]) continue;
        const int64_t off = p.list_off[l];
        const int64_t nl = p.list_off[l + 1] - off;
        const int64_t nwords = (nl + 31) / 32;
        for (int64_t w = warp; w < nwords; w += NW) {
            const int64_t a = off + w * 32;
            const int64_t nb = min((int64_t)32, nl - w * 32);
            uint32_t bits;
            if (p.pbits) {
                const int64_t wi = a >> 5;
                const int sh = (int)(a & 31);
                uint32_t lo = p.pbits[wi];
                uint32_t hi = sh ? p.pbits[wi + 1] : 0u;
                bits = __funnelshift_r(lo, hi, sh);
            } else {
                bits = VS_FULL;
            }
            if (nb < 32) bits &= (1u << nb) - 1u;
            visited += __popc(bits);
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1;
                const int64_t pos = a + b;
                const float key = row_key<T, VEC, IP>(qs, payload + pos * (int64_t)d, d, lane);
                if (key <= tau) {
                    if (cnt == C) {
                        float nthr;
                        int lov = 0;
                        cnt = warp_compact(ckey, cpos, cnt, p.k, margin, C - 32, &nthr, &lov);
                        tau = nthr;
                        ovf |= lov;
                    }
                    if (key <= tau) {
                        if (lane == 0) {
                            ckey[cnt] = key;
                            cpos[cnt] = (uint32_t)pos;
                        }
                        ++cnt;
                    }
                }
            }
        }
    }
    __syncwarp();
    if (lane == 0) {
        p.cb.cnt[q * p.cb.n_sub + sub] = cnt;
        if (ovf) p.cb.overflow[q] = 1;
        if (visited) atomicAdd(p.visited, visited);
    }
}

template <typename T>
cudaError_t launch_ivf_scan_qmajor(const IvfScanParams& p, cudaStream_t s) {
    if (p.nq == 0) return cudaSuccess;
    dim3 grid((unsigned)p.nq, (unsigned)p.n_psplit);
    const size_t smem = (size_t)((p.d + 3) / 4 * 4) * sizeof(float);
    const bool vec = (p.d % 4) == 0;
    if (vec) {
        if (p.ip) k_ivf_scan_qmajor<T, true, true><<<grid, NT, smem, s>>>(p);
        else k_ivf_scan_qmajor<T, true, false><<<grid, NT, smem, s>>>(p);
    } else {
        if (p.ip) k_ivf_scan_qmajor<T, false, true><<<grid, NT, smem, s>>>(p);
        else k_ivf_scan_qmajor<T, false, false><<<grid, NT, smem, s>>>(p);
    }
    return cudaGetLastError();
}
template cudaError_t launch_ivf_scan_qmajor<float>(const IvfScanParams&, cudaStream_t);
template cudaError_t launch_ivf_scan_qmajor<__nv_bfloat16>(const IvfScanParams&, cudaStream_t);

}  // namespace vs
