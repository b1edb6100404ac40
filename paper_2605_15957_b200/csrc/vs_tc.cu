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
#include <cstdio>
#include <cstdlib>

#include "vs_common.cuh"
#include "vs_kernels.cuh"
#include "vs_tc.cuh"

// Compiled twice: this file with 256-row tiles (the default entry points,
// inline namespace bn256) and vs_tc128.cu with 128-row tiles and four TMEM
// accumulators (namespace bn128: the IVF coarse quantizer, where short splits
// make the epilogue the bottleneck; measured faster there, slower on config 2).
#ifndef VS_TC_BN
#define VS_TC_BN 256
#define VS_TC_NS bn256
#define VS_TC_INLINE inline
#endif

namespace vs {
VS_TC_INLINE namespace VS_TC_NS {

namespace tc {

constexpr int BM = 128;                 // queries per tile (UMMA M)
constexpr int BN = VS_TC_BN;            // rows per tile (UMMA N)
constexpr int BK = 64;                  // bf16 elements per stage = 128 B (swizzle atom)
constexpr int UK = 16;                  // UMMA K for kind::f16
constexpr int A_BYTES = BM * BK * 2;    // 16 KB
// single CTA: B tile 256 rows x 64 (32 KB), 4 stages; CTA pair (cta_group::2,
// M = 256): each CTA stages 128 query rows and 128 data rows (16 + 16 KB), 6 stages
template <bool PAIR>
struct Cfg {
    static constexpr int B_ROWS = PAIR ? BN / 2 : BN;
    static constexpr int B_BYTES = B_ROWS * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int NSTAGE = 196608 / STAGE_BYTES;   // the ring fills 192 KB of shared memory
    static constexpr int QTILE = PAIR ? 2 * BM : BM;   // queries per work item
};
constexpr int MAX_STAGES = 8;
constexpr int PF_BOXES = 0;             // MODE 2: L2 prefetch distance in B boxes (0: off, measured best)
constexpr int NTHREADS = 384;           // 12 warps
constexpr int EPI_WARP0 = 4;            // warps 4..11 drain TMEM (2 per lane quadrant)
constexpr int EPI_THREADS = 256;
constexpr int TMEM_COLS = 512;          // NACC accumulators x BN fp32 columns
constexpr int NACC = TMEM_COLS / BN;    // TMEM accumulator ring depth

struct Smem {
    // stage buffers live at the 1024-aligned start of dynamic smem
    uint64_t full[MAX_STAGES];
    uint64_t empty[MAX_STAGES];
    uint64_t tfull[NACC];
    uint64_t tempty[NACC];
    uint32_t tmem_base;
};
template <bool PAIR>
constexpr size_t smem_bytes() {
    return 1024 + (size_t)Cfg<PAIR>::NSTAGE * Cfg<PAIR>::STAGE_BYTES + sizeof(Smem);
}

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
    unsigned long long* dbg;  // nullable: [8] stall / work counters (VS_TC_DEBUG=1)
    int topk_mode;            // 1: keep the local top-k only (phase B verifies); 0: keep the margin band
    unsigned long long* argmin_out;  // MODE 1: per query row packed (orderable key << 32 | column)
    // MODE 2 (IVF list-major): A = bf16 queries staged in pair order (pairs
    // grouped by list), B = the list-contiguous bf16 payload; a work item is
    // one unit (list, first pair, pairs <= BM), its B tiles cover the list
    const int4* units;
    const int* n_units;             // device scalar
    const int64_t* list_off;        // [nlist + 1]
    const int32_t* pair_codes;      // q * nprobe + probe rank, grouped by list
    int nprobe;
    const uint32_t* pbits;          // nullable: filter bit per payload position
    int pf_boxes;                   // MODE 2: L2 prefetch distance (B boxes)
    int64_t chunk_rows;             // MODE 2: rows per list chunk (0: whole lists)
    int a32;                        // MODE 2 A boxes: 0 full 128 rows; 1 32/64-row boxes;
                                    // 2 (default) spread: <= 64 pairs as four 8/16-row boxes, one per TMEM lane quadrant
                                    // (measured: 15.5 -> 14.7 ms on config 4)
    int lim0;                       // first compaction point (0: 2k + 64)
    int dense_direct;               // epilogue: dense chunks append per lane (else cooperatively)
    const int64_t* pair_base;       // MODE 2 with chunks: first flat buffer of each pair (nullable)
    float* keys_out;                // MODE 3: dense approximate keys [nq][keys_ld]
    int64_t keys_ld;
    // MODE 0/3 operand type: 0 bf16, 1 fp16 (power-of-two scaled, see k_stage_queries)
    int f16;
    const float* kinv;              // nullable: [nq] 2^-(query scale + row scale) of the fp16 operands
    float* mins_out;                // MODE 3, nullable: min key of every 32-column chunk [nq][mins_ld]
    int64_t mins_ld;
    // MODE 1, nullable: per (row, column half) its packed best and second key,
    // [nq][2][2] (the near-tie check of the k-means assignment)
    unsigned long long* top2_out;
    // MODE 1 with fp16 operands: the rows' and the columns' max norm^2 (their
    // power-of-two scales; the key factor is -2 / (s_rows s_cols))
    const unsigned* a_scale_src;
    const unsigned* b_scale_src;
};

// one work item: A tile rows [a_row, a_row + QTILE), B tiles of BN rows from
// b_row0 (ntile of them), valid B rows < b_end; MODE 2: npairs valid A rows
struct Item {
    int64_t a_row;
    int64_t b_row0;
    int64_t ntile;
    int64_t b_end;
    int64_t s;          // data split (MODE 0/1)
    int npairs;
    int chunk;          // MODE 2: row chunk of the list
};
template <int MODE, int QTILE>
__device__ __forceinline__ Item decode_item(const Params& p, int64_t it) {
    Item r;
    if (MODE == 2) {
        const int4 un = p.units[it];
        const int64_t off = p.list_off[un.x];
        const int64_t n = p.list_off[un.x + 1] - off;
        r.a_row = un.y;
        r.b_row0 = off + (p.chunk_rows ? (int64_t)un.w * p.chunk_rows : 0);
        r.b_end = p.chunk_rows ? min(off + n, r.b_row0 + p.chunk_rows) : off + n;
        r.ntile = (r.b_end - r.b_row0 + BN - 1) / BN;
        r.s = 0;
        r.npairs = un.z;
        r.chunk = un.w;
    } else {
        const int qt = (int)(it % p.qtiles);
        r.s = it / p.qtiles;
        const int64_t t0 = r.s * p.tiles_per_split;
        const int64_t t1 = min(p.ntiles, t0 + p.tiles_per_split);
        r.a_row = (int64_t)qt * QTILE;
        r.b_row0 = t0 * BN;
        r.ntile = t1 - t0;
        r.b_end = p.nsel;
        r.npairs = 0;
        r.chunk = 0;
    }
    return r;
}

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
// TMA load with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// TMA prefetch of one box into L2 (no shared memory, no barrier)
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"((uint64_t)map), "r"(c0),
                 "r"(c1)
                 : "memory");
}
// CTA-pair TMA: the bytes land in this CTA's shared memory, the transaction
// completes on the leader CTA's barrier (peer bit cleared)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(b) & 0xFEFFFFFFu) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    const uint16_t mask = 0x3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(smem_u32(bar)), "h"(mask) : "memory");
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
// the same with A/B = F16 (a_format = b_format = 0)
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
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
// wait for outstanding TMEM loads, tying the destination registers to the wait
// so the compiler cannot consume them earlier
__device__ __forceinline__ void tmem_wait_ld_regs(uint32_t* r) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                   "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                   "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]),
                   "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]),
                   "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
}

// v[j] for a run-time j without local memory: a 5-level select tree (31 selects)
__device__ __forceinline__ float sel32(const float (&v)[32], int j) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = (j & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (j & 2) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = (j & 4) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = (j & 8) ? a[2 * i + 1] : a[2 * i];
    return (j & 16) ? a[1] : a[0];
}

__device__ __forceinline__ float pow2_scale(float norm2);   // fp16 operand scales (below)

// ---- the kernel --------------------------------------------------------------------------------------
template <bool IP, int MODE, bool PAIR>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_enn_scan_tc(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                  Params p, const __grid_constant__ CUtensorMap map_a32,
                  const __grid_constant__ CUtensorMap map_a64) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    __shared__ __align__(16) float xn_w[8][BN / 2];  // per epilogue warp: its column half's row norms
    __shared__ __align__(16) float app_w[8][32];     // per epilogue warp: one lane's chunk keys (dense appends)
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    constexpr int NSTAGE = Cfg<PAIR>::NSTAGE;
    constexpr int STAGE_BYTES = Cfg<PAIR>::STAGE_BYTES;
    constexpr int QTILE = Cfg<PAIR>::QTILE;
    Smem& S = *reinterpret_cast<Smem*>(base + (size_t)NSTAGE * STAGE_BYTES);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // work units: CTAs (single) or CTA pairs; rank 0 of a pair issues the MMAs
    const uint32_t rank = PAIR ? cluster_rank() : 0u;
    const int64_t unit = PAIR ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
    const int64_t nunits = PAIR ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;

    if (warp == 0 && lane == 0) {
        prefetch_map(&map_a);
        prefetch_map(&map_b);
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], 1);
        }
        for (int i = 0; i < NACC; ++i) {
            mbar_init(&S.tfull[i], 1);
            mbar_init(&S.tempty[i], PAIR ? 2 * EPI_THREADS : EPI_THREADS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                         ::"r"(smem_u32(&S.tmem_base)), "n"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                         ::"r"(smem_u32(&S.tmem_base)), "n"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();   // peer barriers initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;
    unsigned long long t_start = 0;
    if (p.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

    const int64_t nitems = MODE == 2 ? (int64_t)*p.n_units : (int64_t)p.qtiles * p.nsplit;
    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            long long w_empty = 0;
            const uint64_t pol_a = policy_evict_last(), pol_b = policy_evict_first();
            for (int64_t it = unit; it < nitems; it += nunits) {
                const Item item = decode_item<MODE, QTILE>(p, it);
                // MODE 2: the B operand streams from HBM exactly once, so the
                // smem ring alone keeps too few bytes in flight; a sliding
                // window of L2 prefetches runs PF boxes ahead of the loads
                const int64_t nbox = item.ntile * p.kblocks;
                if (MODE == 2)
                    for (int64_t pb = 1; pb < p.pf_boxes && pb < nbox; ++pb)
                        tma_prefetch_2d(&map_b, (int)(pb % p.kblocks) * BK, (int)(item.b_row0 + (pb / p.kblocks) * BN));
                for (int64_t t = 0; t < item.ntile; ++t) {
                    const int brow = (int)(item.b_row0 + t * BN);
                    for (int kb = 0; kb < p.kblocks; ++kb) {
                        if (MODE == 2) {
                            const int64_t pb = t * p.kblocks + kb + p.pf_boxes;
                            if (pb < nbox)
                                tma_prefetch_2d(&map_b, (int)(pb % p.kblocks) * BK,
                                                (int)(item.b_row0 + (pb / p.kblocks) * BN));
                        }
                        const long long c0 = p.dbg ? clock64() : 0;
                        mbar_wait(&S.empty[stage], phase ^ 1);
                        if (p.dbg) w_empty += clock64() - c0;
                        unsigned char* sa = base + (size_t)stage * STAGE_BYTES;
                        if (PAIR) {
                            if (rank == 0) mbar_expect_tx(&S.full[stage], 2 * STAGE_BYTES);
                            tma_load_2d_pair(sa, &map_a, &S.full[stage], kb * BK, (int)item.a_row + (int)rank * BM);
                            tma_load_2d_pair(sa + A_BYTES, &map_b, &S.full[stage], kb * BK,
                                             brow + (int)rank * (BN / 2));
                        } else {
                            if (MODE == 2) {
                                // A: only the unit's pair rows (32-row box for <= 32 pairs;
                                // the MMA's other A rows hold stale data whose accumulator
                                // rows the epilogue ignores). B (the payload) streams once:
                                // evict first; A is re-read for every tile: evict last.
                                if (p.a32 == 2 && item.npairs <= 64) {
                                    // spread: quarter q of the unit's pairs (8 or 16 rows)
                                    // lands in TMEM lane quadrant q, so all four epilogue
                                    // lane quadrants (SMSPs) share the appends
                                    const int qb = item.npairs <= 32 ? 8 : 16;
                                    mbar_expect_tx(&S.full[stage], STAGE_BYTES - A_BYTES + 4 * qb * BK * 2);
                                    const CUtensorMap* ma = qb == 8 ? &map_a32 : &map_a64;
#pragma unroll
                                    for (int qd = 0; qd < 4; ++qd)
                                        tma_load_2d_hint(sa + qd * 32 * BK * 2, ma, &S.full[stage], kb * BK,
                                                         (int)item.a_row + qd * qb, pol_a);
                                } else {
                                    const int arows = !p.a32 ? BM : item.npairs <= 32 ? 32 : item.npairs <= 64 ? 64 : BM;
                                    mbar_expect_tx(&S.full[stage], STAGE_BYTES - A_BYTES + arows * BK * 2);
                                    const CUtensorMap* ma = arows == 32 ? &map_a32 : arows == 64 ? &map_a64 : &map_a;
                                    tma_load_2d_hint(sa, ma, &S.full[stage], kb * BK, (int)item.a_row, pol_a);
                                }
                                tma_load_2d_hint(sa + A_BYTES, &map_b, &S.full[stage], kb * BK, brow, pol_b);
                            } else {
                                mbar_expect_tx(&S.full[stage], STAGE_BYTES);
                                tma_load_2d(sa, &map_a, &S.full[stage], kb * BK, (int)item.a_row);
                                tma_load_2d(sa + A_BYTES, &map_b, &S.full[stage], kb * BK, brow);
                            }
                        }
                        if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
                    }
                }
            }
            if (p.dbg) atomicAdd(&p.dbg[0], (unsigned long long)w_empty);
        }
    } else if (warp == 1) {
        // ===== MMA issuer (single thread; rank 0 of a pair) =====
        if (lane == 0 && rank == 0) {
            const uint32_t idesc = p.f16 ? idesc_f16(PAIR ? 2 * BM : BM, BN) : idesc_bf16(PAIR ? 2 * BM : BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t tcount = 0;
            long long w_full = 0, w_tempty = 0;
            for (int64_t it = unit; it < nitems; it += nunits) {
                const Item item = decode_item<MODE, QTILE>(p, it);
                for (int64_t t = 0; t < item.ntile; ++t, ++tcount) {
                    const uint32_t acc = tcount % NACC, aph = (tcount / NACC) & 1;
                    long long c0 = p.dbg ? clock64() : 0;
                    mbar_wait(&S.tempty[acc], aph ^ 1);
                    if (p.dbg) w_tempty += clock64() - c0;
                    tc_fence_after();
                    const uint32_t dt = tmem + acc * BN;
                    for (int kb = 0; kb < p.kblocks; ++kb) {
                        c0 = p.dbg ? clock64() : 0;
                        mbar_wait(&S.full[stage], phase);
                        if (p.dbg) w_full += clock64() - c0;
                        tc_fence_after();
                        const uint32_t sa = smem_u32(base + (size_t)stage * STAGE_BYTES);
                        const uint32_t sb = sa + A_BYTES;
#pragma unroll
                        for (int kk = 0; kk < BK / UK; ++kk) {
                            if (PAIR)
                                mma_bf16_pair(dt, desc_sw128(sa + kk * UK * 2), desc_sw128(sb + kk * UK * 2), idesc,
                                              (kb | kk) != 0);
                            else
                                mma_bf16(dt, desc_sw128(sa + kk * UK * 2), desc_sw128(sb + kk * UK * 2), idesc,
                                         (kb | kk) != 0);
                        }
                        if (PAIR) mma_commit_pair(&S.empty[stage]);
                        else mma_commit(&S.empty[stage]);
                        if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
                    }
                    if (PAIR) mma_commit_pair(&S.tfull[acc]);
                    else mma_commit(&S.tfull[acc]);
                }
            }
            if (p.dbg) {
                atomicAdd(&p.dbg[1], (unsigned long long)w_full);
                atomicAdd(&p.dbg[2], (unsigned long long)w_tempty);
            }
        }
    } else if (warp >= EPI_WARP0 && MODE == 1) {
        // ===== epilogue (argmin mode): first-min column per query row =====
        // (k-means assignment: queries = data rows, columns = centroids)
        const int et = threadIdx.x - EPI_WARP0 * 32;
        const int row = et & (BM - 1);
        const int half = et >> 7;
        const int quad = warp & 3;
        float* xw = xn_w[warp - EPI_WARP0];
        uint32_t tcount = 0;
        const float cmul1 = p.a_scale_src ? -2.f / (pow2_scale(__uint_as_float(*p.a_scale_src)) *
                                                    pow2_scale(__uint_as_float(*p.b_scale_src)))
                                          : -2.f;
        for (int64_t it = unit; it < nitems; it += nunits) {
            const Item item = decode_item<MODE, QTILE>(p, it);
            const int64_t q = item.a_row + (int64_t)rank * BM + row;
            uint32_t best_o = 0xffffffffu, best_i = 0u, second_o = 0xffffffffu;
            for (int64_t t = 0; t < item.ntile; ++t, ++tcount) {
                const uint32_t acc = tcount % NACC, aph = (tcount / NACC) & 1;
                const int64_t r0 = item.b_row0 + t * BN;
                const int ncols = (int)min((int64_t)BN, p.nsel - r0);
                __syncwarp();   // the previous tile's reads of xw come first
                if (lane * 4 < BN / 2) {
                    const int64_t i = r0 + half * (BN / 2) + lane * 4;
                    float4 v;
                    v.x = i + 0 < p.nsel ? __ldg(p.xn + i + 0) : 0.f;
                    v.y = i + 1 < p.nsel ? __ldg(p.xn + i + 1) : 0.f;
                    v.z = i + 2 < p.nsel ? __ldg(p.xn + i + 2) : 0.f;
                    v.w = i + 3 < p.nsel ? __ldg(p.xn + i + 3) : 0.f;
                    *reinterpret_cast<float4*>(xw + lane * 4) = v;
                }
                __syncwarp();
                mbar_wait(&S.tfull[acc], aph);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + acc * BN + half * (BN / 2);
#pragma unroll 1
                for (int ch = 0; ch < BN / 64; ++ch) {
                    uint32_t r[32];
                    TMEM_LD32(taddr + ch * 32, r);
                    tmem_wait_ld();
                    const int cb0 = half * (BN / 2) + ch * 32;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float a = __uint_as_float(r[j]);
                        const float key = IP ? -a : fmaf(cmul1, a, xw[ch * 32 + j]);
                        const uint32_t ko = f2o(key);
                        if (cb0 + j < ncols) {
                            if (ko < best_o) {
                                second_o = best_o;
                                best_o = ko;
                                best_i = (uint32_t)(r0 + cb0 + j);
                            } else if (ko < second_o) {
                                second_o = ko;
                            }
                        }
                    }
                }
                tc_fence_before();
                if (PAIR) mbar_arrive_leader(&S.tempty[acc]);
                else mbar_arrive(&S.tempty[acc]);
            }
            if (q < p.nq) {
                const unsigned long long pk = ((unsigned long long)best_o << 32) | best_i;
                atomicMin(&p.argmin_out[q], pk);
                if (p.top2_out) {
                    p.top2_out[(q * 2 + half) * 2] = pk;
                    p.top2_out[(q * 2 + half) * 2 + 1] = second_o;
                }
            }
        }
    } else if (warp >= EPI_WARP0 && MODE == 3) {
        // ===== epilogue (dense keys): TMEM -> approximate keys -> global =====
        // (IVF coarse quantizer: every (query, centroid) key is stored and a
        // per-query select follows, instead of candidate buffers)
        const int et = threadIdx.x - EPI_WARP0 * 32;
        const int row = et & (BM - 1);
        const int half = et >> 7;
        const int quad = warp & 3;
        float* xw = xn_w[warp - EPI_WARP0];
        uint32_t tcount = 0;
        for (int64_t it = unit; it < nitems; it += nunits) {
            const Item item = decode_item<MODE, QTILE>(p, it);
            const int64_t q = item.a_row + (int64_t)rank * BM + row;
            float* krow = p.keys_out ? p.keys_out + (q < p.nq ? q : 0) * p.keys_ld : nullptr;   // nullable: minima only
            // key = ||x||^2 - 2 q.x (or -q.x) with q.x = acc x 2^-(scales): exact factor
            const float ks = (p.kinv && q < p.nq) ? __ldg(p.kinv + q) : 1.f;
            const float cmul = IP ? -ks : -2.f * ks;
            for (int64_t t = 0; t < item.ntile; ++t, ++tcount) {
                const uint32_t acc = tcount % NACC, aph = (tcount / NACC) & 1;
                const int64_t r0 = item.b_row0 + t * BN;
                const int ncols = (int)min((int64_t)BN, p.nsel - r0);
                if (!IP) {
                    for (int c = lane * 4; c < BN / 2; c += 128) {
                        const int64_t i = r0 + half * (BN / 2) + c;
                        float4 v;
                        v.x = i + 0 < p.nsel ? __ldg(p.xn + i + 0) : 0.f;
                        v.y = i + 1 < p.nsel ? __ldg(p.xn + i + 1) : 0.f;
                        v.z = i + 2 < p.nsel ? __ldg(p.xn + i + 2) : 0.f;
                        v.w = i + 3 < p.nsel ? __ldg(p.xn + i + 3) : 0.f;
                        *reinterpret_cast<float4*>(xw + c) = v;
                    }
                }
                __syncwarp();
                mbar_wait(&S.tfull[acc], aph);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + acc * BN + half * (BN / 2);
#pragma unroll 1
                for (int ch = 0; ch < BN / 64; ++ch) {
                    uint32_t r[32];
                    TMEM_LD32(taddr + ch * 32, r);
                    tmem_wait_ld();
                    const int cb0 = half * (BN / 2) + ch * 32;
                    float kv[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float a = __uint_as_float(r[j]);
                        kv[j] = IP ? a * cmul : fmaf(cmul, a, xw[ch * 32 + j]);
                    }
                    if (q < p.nq && p.mins_out && cb0 < ncols) {
                        float mn = __int_as_float(0x7f800000);
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (cb0 + j < ncols) mn = fminf(mn, kv[j]);
                        p.mins_out[q * p.mins_ld + ((r0 + cb0) >> 5)] = mn;
                    }
                    if (q < p.nq && krow) {
                        float* dst = krow + r0 + cb0;
                        if (cb0 + 32 <= ncols && ((p.keys_ld | r0) & 3) == 0) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                __stcs(reinterpret_cast<float4*>(dst + j), make_float4(kv[j], kv[j + 1], kv[j + 2], kv[j + 3]));
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (cb0 + j < ncols) dst[j] = kv[j];
                        }
                    }
                }
                tc_fence_before();
                if (PAIR) mbar_arrive_leader(&S.tempty[acc]);
                else mbar_arrive(&S.tempty[acc]);
                __syncwarp();
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ===== epilogue: TMEM -> keys -> candidate buffers =====
        // 8 warps: warp w drains TMEM lane quadrant (w % 4) for column half
        // (w - 4) / 4, so each query row is served by two threads (two
        // candidate buffers, subs 2s and 2s+1) and two warps share each SMSP.
        const int et = threadIdx.x - EPI_WARP0 * 32;     // 0..255
        const int row = et & (BM - 1);                   // TMEM lane == tile row
        const int half = et >> 7;                        // column half
        const int quad = warp & 3;                       // lane quadrant
        const int C = p.cb.C;
        uint32_t tcount = 0;
        long long w_tfull = 0, c_comp = 0, n_comp = 0, n_app = 0, c_ldw = 0, c_loop = 0;
        // software-pipelined per-tile inputs: the next tile's row norms (4 per
        // lane = the warp's column half) and the next tile's admission bound
        auto norms4 = [&](int64_t r0n, int64_t bend) -> float4 {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (IP) return v;
            const int64_t i = r0n + half * (BN / 2) + lane * 4;
            if (i + 3 < bend && MODE != 2) {
                v = __ldg(reinterpret_cast<const float4*>(p.xn + i));
            } else {
                v.x = i + 0 < bend ? __ldg(p.xn + i + 0) : 0.f;
                v.y = i + 1 < bend ? __ldg(p.xn + i + 1) : 0.f;
                v.z = i + 2 < bend ? __ldg(p.xn + i + 2) : 0.f;
                v.w = i + 3 < bend ? __ldg(p.xn + i + 3) : 0.f;
            }
            return v;
        };
        // the query (and its candidate sub-buffer) served by this thread's row
        // of work item `item`; false for padding rows
        auto row_query = [&](const Item& item, int64_t& q, int64_t& sub) -> bool {
            if (MODE == 2) {
                int pr = row;
                if (p.a32 == 2 && item.npairs <= 64) {   // spread placement (producer)
                    const int qb = item.npairs <= 32 ? 8 : 16;
                    const int li = row & 31;
                    if (li >= qb) return false;
                    pr = (row >> 5) * qb + li;
                }
                if (pr >= item.npairs) return false;
                const int code = __ldg(p.pair_codes + item.a_row + pr);
                q = code / p.nprobe;
                // flat buffer index with list chunks, else the sub of (query, probe rank)
                sub = p.pair_base ? __ldg(p.pair_base + code) + 2 * item.chunk + half
                                  : (int64_t)(code % p.nprobe) * 2 + half;
                return true;
            }
            q = item.a_row + (int64_t)rank * BM + row;
            sub = item.s * 2 + half;
            return q < p.nq;
        };
        float* xw = xn_w[warp - EPI_WARP0];
        float4 pf = make_float4(0.f, 0.f, 0.f, 0.f);
        unsigned pf_tau = 0xffffffffu;
        {
            const int64_t it0 = unit;
            if (it0 < nitems) {
                const Item i0 = decode_item<MODE, QTILE>(p, it0);
                pf = norms4(i0.b_row0, i0.b_end);
                int64_t q0, s0;
                if (row_query(i0, q0, s0)) pf_tau = __ldcg(p.tau_g + q0);
            }
        }
        for (int64_t it = unit; it < nitems; it += nunits) {
            const Item item = decode_item<MODE, QTILE>(p, it);
            int64_t q = 0, sub = 0;
            const bool qv = row_query(item, q, sub);
            const int64_t bufidx = (MODE == 2 && p.pair_base) ? sub : q * p.cb.n_sub + sub;
            const int64_t cbase = qv ? bufidx * (int64_t)C : 0;
            float* ckey = p.cb.key + cbase;
            uint32_t* cpos = p.cb.pos + cbase;
            const float qmargin = qv ? p.margin[q] : 0.f;
            const float ks = (MODE != 2 && p.kinv && qv) ? __ldg(p.kinv + q) : 1.f;
            const float cmul = IP ? -ks : -2.f * ks;   // exact: a power of two
            int cnt = 0;
            int ovf = 0;
            // geometric compaction schedule, checked once per tile before any TMEM
            // data is live: compact when the next half-tile (<= 128 appends) could
            // push the buffer past lim (2k + 64 initially, then 2x the kept count)
            const int cap_t = C - BN / 2;
            const int lim0 = p.lim0 > 0 ? p.lim0 : 2 * p.k + 64;
            int lim = lim0;
            float tau = __int_as_float(0x7f800000);
            for (int64_t t = 0; t < item.ntile; ++t, ++tcount) {
                const uint32_t acc = tcount % NACC, aph = (tcount / NACC) & 1;
                const int64_t r0 = item.b_row0 + t * BN;
                const int ncols = (int)min((int64_t)BN, item.b_end - r0);
                __syncwarp();   // the previous tile's reads of xw come first
                if (!IP && lane * 4 < BN / 2) *reinterpret_cast<float4*>(xw + lane * 4) = pf;
                __syncwarp();
                if (qv) tau = fminf(tau, o2f(pf_tau));
                {   // prefetch for the next tile of this CTA's sequence
                    if (t + 1 < item.ntile) {
                        pf = norms4(r0 + BN, item.b_end);
                        pf_tau = qv ? __ldcg(p.tau_g + q) : 0xffffffffu;
                    } else if (it + nunits < nitems) {
                        const Item in = decode_item<MODE, QTILE>(p, it + nunits);
                        pf = norms4(in.b_row0, in.b_end);
                        int64_t qn, sn;
                        pf_tau = row_query(in, qn, sn) ? __ldcg(p.tau_g + qn) : 0xffffffffu;
                    }
                }
                {   // compaction (warp-cooperative, one buffer at a time)
                    unsigned m = __ballot_sync(VS_FULL, qv && cnt > min(lim, cap_t));
                    const long long cc0 = (p.dbg && m) ? clock64() : 0;
                    if (p.dbg && lane == 0) n_comp += __popc(m);
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
                        const int nc = warp_compact(p.cb.key + lb, p.cb.pos + lb, lc, p.k,
                                                    p.topk_mode ? 0.f : lmar, cap_t, &nthr, &lov);
                        if (lane == l) {
                            cnt = nc;
                            tau = fminf(tau, nthr);
                            ovf |= lov;
                            lim = max(lim0, 2 * nc + 64);
                            atomicMin(&p.tau_g[q], f2o(tau));
                        }
                    }
                    if (p.dbg && cc0) c_comp += clock64() - cc0;
                }
                const long long c0 = p.dbg ? clock64() : 0;
                mbar_wait(&S.tfull[acc], aph);
                if (p.dbg) w_tfull += clock64() - c0;
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + acc * BN + half * (BN / 2);
                uint32_t ra[32], rb[32];
                const long long cl0 = p.dbg ? clock64() : 0;
                TMEM_LD32(taddr, ra);
                tmem_wait_ld();
                if (p.dbg) c_ldw += clock64() - cl0;
#pragma unroll
                for (int ch = 0; ch < BN / 64; ++ch) {
                    uint32_t* cur = (ch & 1) ? rb : ra;
                    uint32_t* nxt = (ch & 1) ? ra : rb;
                    if (ch + 1 < BN / 64) TMEM_LD32(taddr + (ch + 1) * 32, nxt);  // in flight during compute
                    const int cl0 = ch * 32;                  // column within the half
                    const int cb0 = half * (BN / 2) + cl0;    // column within the tile
                    float xv[32];
                    if (!IP) {
                        const float4* x4 = reinterpret_cast<const float4*>(xw + cl0);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float4 v = x4[i];
                            xv[4 * i] = v.x; xv[4 * i + 1] = v.y; xv[4 * i + 2] = v.z; xv[4 * i + 3] = v.w;
                        }
                    }
                    const int nv = ncols - cb0;
                    unsigned valid = nv >= 32 ? VS_FULL : (nv <= 0 ? 0u : ((1u << nv) - 1u));
                    if (MODE == 2 && p.pbits && valid) {   // filter bits of payload positions r0+cb0..+31
                        const int64_t a = r0 + cb0;
                        const int sh = (int)(a & 31);
                        const uint32_t lo = __ldg(p.pbits + (a >> 5));
                        const uint32_t hi = sh ? __ldg(p.pbits + (a >> 5) + 1) : 0u;
                        valid &= __funnelshift_r(lo, hi, sh);
                    }
                    float kk[32];
                    unsigned mask = 0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float a = __uint_as_float(cur[j]);
                        kk[j] = IP ? a * cmul : fmaf(cmul, a, xv[j]);
                        mask |= (kk[j] <= tau ? 1u : 0u) << j;
                    }
                    mask &= valid;
                    if (!qv) mask = 0;
                    // append: each lane walks its own admitted columns, picking the
                    // key out of its registers with a select tree. Admissions are
                    // sparse (~1 % of keys), so this beats warp-cooperative staging
                    // through shared memory, which serialised over the admitting
                    // lanes (config 2 phase A 22.0 -> 18.3 ms, measured). Dense chunks
                    // (a lane admits >= 8 keys) append from static register indices
                    // (splits of 8..127 tiles, measured) or cooperatively with
                    // coalesced stores (one-tile splits, e.g. config 1).
                    if (p.dbg) n_app += __popc(mask);
                    const bool dense = __any_sync(VS_FULL, __popc(mask) >= 8);
                    if (dense && p.dense_direct) {
                        // dense, longer splits (e.g. the coarse quantizer's first
                        // tiles): every lane appends its own keys, static indices
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            if ((mask >> j) & 1u) {
                                ckey[cnt] = kk[j];
                                cpos[cnt] = (uint32_t)(r0 + cb0 + j);
                                ++cnt;
                            }
                        }
                    } else if (dense) {
                        unsigned am = __ballot_sync(VS_FULL, mask != 0);
                        float* st = app_w[warp - EPI_WARP0];
                        while (am) {
                            const int l = __ffs(am) - 1;
                            am &= am - 1;
                            if (lane == l) {
                                float4* st4 = reinterpret_cast<float4*>(st);
#pragma unroll
                                for (int i = 0; i < 8; ++i)
                                    st4[i] = make_float4(kk[4 * i], kk[4 * i + 1], kk[4 * i + 2], kk[4 * i + 3]);
                            }
                            __syncwarp();
                            const unsigned ml = __shfl_sync(VS_FULL, mask, l);
                            const int cl = __shfl_sync(VS_FULL, cnt, l);
                            const int lo32 = __shfl_sync(VS_FULL, (int)(cbase & 0xffffffff), l);
                            const int hi32 = __shfl_sync(VS_FULL, (int)(cbase >> 32), l);
                            if ((ml >> lane) & 1u) {
                                const int64_t lb = ((int64_t)(uint32_t)hi32 << 32) | (uint32_t)lo32;
                                const int dst = cl + __popc(ml & lanemask_lt());
                                p.cb.key[lb + dst] = st[lane];
                                p.cb.pos[lb + dst] = (uint32_t)(r0 + cb0 + lane);
                            }
                            __syncwarp();
                            if (lane == l) cnt += __popc(ml);
                        }
                    } else {
                        unsigned mm = mask;
                        while (mm) {
                            const int j = __ffs(mm) - 1;
                            mm &= mm - 1;
                            ckey[cnt] = sel32(kk, j);
                            cpos[cnt] = (uint32_t)(r0 + cb0 + j);
                            ++cnt;
                        }
                    }
                    if (ch + 1 < BN / 64) {
                        const long long cw = p.dbg ? clock64() : 0;
                        tmem_wait_ld_regs(nxt);
                        if (p.dbg) c_ldw += clock64() - cw;
                    }
                }
                if (p.dbg) c_loop += clock64() - cl0;
                tc_fence_before();
                if (PAIR) mbar_arrive_leader(&S.tempty[acc]);
                else mbar_arrive(&S.tempty[acc]);
            }
            if (qv) {
                p.cb.cnt[bufidx] = cnt;
                if (ovf) p.cb.overflow[q] = 1;
            }
        }
        if (p.dbg) {
            atomicAdd(&p.dbg[3], (unsigned long long)w_tfull);
            atomicAdd(&p.dbg[4], (unsigned long long)c_comp);
            atomicAdd(&p.dbg[5], (unsigned long long)n_comp);
            atomicAdd(&p.dbg[6], (unsigned long long)n_app);
            if (et == 0) {
                atomicAdd(&p.dbg[7], (unsigned long long)tcount);
                atomicMax(&p.dbg[12], (unsigned long long)tcount);
                unsigned long long t_end;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
                atomicMax(&p.dbg[10], t_end - t_start);
                atomicAdd(&p.dbg[11], t_end - t_start);
            }
            atomicAdd(&p.dbg[8], (unsigned long long)c_ldw);
            atomicAdd(&p.dbg[9], (unsigned long long)c_loop);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();   // the leader's MMAs also wrote this CTA's TMEM
    tc_fence_after();
    if (warp == 2) {
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
    }
}

// ---- operand staging -----------------------------------------------------------------------------------
// Rounding to bf16 is exact-error-tracked: for each staged vector v with bf16
// image v~ and error dv = v~ - v we keep ||v~|| and ||dv|| (fp32, inflated by
// 1e-4 for their own rounding). The tensor-core dot product then satisfies
//   |q~.x~ - q.x| <= ||q~|| ||dx|| + ||dq|| ||x~|| + ||dq|| ||dx||
// (Cauchy-Schwarz on the error vectors), which is ~1.7x tighter than the
// worst-case 2^-8 ||q|| ||x|| bound and still rigorous.

// 16-bit operand types: bf16 (8-bit significand) or fp16 (11-bit: 8x smaller
// rounding error, hence an ~6x narrower margin band and fewer phase-B
// survivors). fp16's range is small, so fp16 operands are scaled by powers of
// two: every row by 2^ex with 2^ex max||x|| < 2^14 (column-wide), every query
// by its own 2^eq with 2^eq ||q|| < 2^14. Both scalings are exact, elements
// stay below 2^14 < 65504, and the epilogue multiplies the accumulator by
// 2^-(eq+ex) (exact). Rounding errors are tracked in unscaled units.
template <typename O> struct Op16;
template <> struct Op16<__nv_bfloat16> {
    static __device__ __forceinline__ uint32_t pack(float a, float b, float2& back) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        back = __bfloat1622float2(h);
        return *reinterpret_cast<const uint32_t*>(&h);
    }
    static __device__ __forceinline__ __nv_bfloat16 one(float v, float& back) {
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        back = __bfloat162float(h);
        return h;
    }
};
template <> struct Op16<__half> {
    static __device__ __forceinline__ uint32_t pack(float a, float b, float2& back) {
        const __half2 h = __floats2half2_rn(a, b);
        back = __half22float2(h);
        return *reinterpret_cast<const uint32_t*>(&h);
    }
    static __device__ __forceinline__ __half one(float v, float& back) {
        const __half h = __float2half_rn(v);
        back = __half2float(h);
        return h;
    }
};
// 2^e with 2^e sqrt(norm2) < 2^14 (1 for a zero or non-finite norm)
__device__ __forceinline__ float pow2_scale(float norm2) {
    const float n = sqrtf(norm2);
    if (!(n > 0.f) || !isfinite(n)) return 1.f;
    int e;
    frexpf(n * 1.001f, &e);   // n * 1.001 < 2^e
    return ldexpf(1.f, max(-120, min(120, 14 - e)));
}

// queries fp32 -> 16-bit (round to nearest even), row stride dp; warp per query.
// fp16 (xs != nullptr): the query's own power-of-two scale, and kinv[q] =
// 2^-(eq + ex) with ex the rows' scale (from their max norm xs).
template <typename O>
__global__ void k_stage_queries(const float* __restrict__ q, int64_t nq, int d, int dp, O* __restrict__ out,
                                float2* __restrict__ qerr, const unsigned* __restrict__ xs,
                                float* __restrict__ kinv) {
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const float sx = xs ? pow2_scale(__uint_as_float(*xs)) : 1.f;
    for (; w < nq; w += nw) {
        const float* src = q + w * (int64_t)d;
        float sq = 1.f;
        if (xs) {
            float n2 = 0.f;
            for (int c = lane; c < d; c += 32) n2 = fmaf(src[c], src[c], n2);
            sq = pow2_scale(warp_sumf(n2));
            if (lane == 0) kinv[w] = 1.f / (sq * sx);
        }
        const float iq = 1.f / sq;
        float sn = 0.f, se = 0.f;
        for (int c = lane; c < dp; c += 32) {
            const float v = c < d ? src[c] : 0.f;
            float vb;
            out[w * (int64_t)dp + c] = Op16<O>::one(v * sq, vb);
            vb *= iq;
            const float e = vb - v;  // exact in fp32 (Sterbenz-free: |e| << |v|, same binade)
            sn = fmaf(vb, vb, sn);
            se = fmaf(e, e, se);
        }
        sn = warp_sumf(sn);
        se = warp_sumf(se);
        if (lane == 0) qerr[w] = make_float2(sqrtf(sn) * 1.0001f, sqrtf(se) * 1.0001f);
    }
}
// selected rows -> contiguous bf16 [nsel][dp] + their fp32 norms (warp per row);
// max ||x~|| and max ||dx|| over the rows into xmax2[0..1] (float bits, atomicMax)
// queries in pair order (IVF list-major A operand): row i = bf16(Q[code_i / nprobe])
__global__ void k_stage_pair_queries(const float* __restrict__ q, const int32_t* __restrict__ codes, int64_t npairs,
                                     int nprobe, int d, int dp, __nv_bfloat16* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (; w < npairs; w += nw) {
        const int64_t qi = codes[w] / nprobe;
        const float* src = q + qi * (int64_t)d;
        __nv_bfloat16* dst = out + w * (int64_t)dp;
        for (int c = lane; c < dp; c += 32) dst[c] = __float2bfloat16_rn(c < d ? src[c] : 0.f);
    }
}

template <typename T, typename O>
__global__ void k_stage_rows(const T* __restrict__ x, const int64_t* __restrict__ sel, int64_t nsel, int d,
                             int dp, const float* __restrict__ norms, O* __restrict__ out,
                             float* __restrict__ xn, unsigned* __restrict__ xmax2,
                             const unsigned* __restrict__ xs = nullptr, float2* __restrict__ rowstats = nullptr) {
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // fp16 operands: the column-wide power-of-two scale (k_stage_queries)
    const float sx = xs ? pow2_scale(__uint_as_float(*xs)) : 1.f;
    const float ix = 1.f / sx;
    float mb = 0.f, me = 0.f;
    for (; w < nsel; w += nw) {
        const int64_t r = sel ? sel[w] : w;
        const T* src = x + r * (int64_t)d;
        O* dst = out + w * (int64_t)dp;
        float sn = 0.f, se = 0.f;
        if (sizeof(T) == 4 && (d % 4) == 0 && (dp % 4) == 0) {
            for (int c = lane * 4; c < dp; c += 128) {
                const float4 v = (c < d) ? *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(src) + c)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                float2 fa, fb;
                uint2 u;
                u.x = Op16<O>::pack(v.x * sx, v.y * sx, fa);
                u.y = Op16<O>::pack(v.z * sx, v.w * sx, fb);
                fa.x *= ix; fa.y *= ix; fb.x *= ix; fb.y *= ix;
                const float e0 = fa.x - v.x, e1 = fa.y - v.y, e2 = fb.x - v.z, e3 = fb.y - v.w;
                sn = fmaf(fa.x, fa.x, sn); sn = fmaf(fa.y, fa.y, sn);
                sn = fmaf(fb.x, fb.x, sn); sn = fmaf(fb.y, fb.y, sn);
                se = fmaf(e0, e0, se); se = fmaf(e1, e1, se); se = fmaf(e2, e2, se); se = fmaf(e3, e3, se);
                *reinterpret_cast<uint2*>(dst + c) = u;
            }
        } else {
            for (int c = lane; c < dp; c += 32) {
                const float v = c < d ? ld_elem(src + c) : 0.f;
                float vb;
                dst[c] = Op16<O>::one(v * sx, vb);
                vb *= ix;
                const float e = vb - v;
                sn = fmaf(vb, vb, sn);
                se = fmaf(e, e, se);
            }
        }
        sn = warp_sumf(sn);
        se = warp_sumf(se);
        mb = fmaxf(mb, sn);
        me = fmaxf(me, se);
        if (lane == 0 && xn) xn[w] = norms[r];
        if (lane == 0 && rowstats) rowstats[w] = make_float2(sn, se);
    }
    if (lane == 0) {
        atomicMax(&xmax2[0], __float_as_uint(mb));
        atomicMax(&xmax2[1], __float_as_uint(me));
    }
}

// staging from the column's fp16 shadow (same scale, same rounding as
// k_stage_rows, so keys and margins are identical): selected rows are copied
// (16-byte vectors, a warp per row), their norms and the max of their stored
// (||x~||^2, ||dx||^2) reduced into xmax2. 2 + 2 bytes per element instead of 4 + 2.
__global__ void k_stage_rows_f16(const __half* __restrict__ sh, const float2* __restrict__ stats,
                                 const int64_t* __restrict__ sel, int64_t nsel, int dp,
                                 const float* __restrict__ norms, __half* __restrict__ out, float* __restrict__ xn,
                                 unsigned* __restrict__ xmax2) {
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float mb = 0.f, me = 0.f;
    const int n16 = dp / 8;
    int64_t r = w < nsel ? (sel ? sel[w] : w) : 0;
    for (; w < nsel; w += nw) {
        // the next row's index, this row's stats and four 16-byte loads per
        // lane are all in flight before the first store
        const int64_t rn = w + nw < nsel ? (sel ? sel[w + nw] : w + nw) : 0;
        const uint4* src = reinterpret_cast<const uint4*>(sh + r * (int64_t)dp);
        uint4* dst = reinterpret_cast<uint4*>(out + w * (int64_t)dp);
        float2 st = make_float2(0.f, 0.f);
        float nv = 0.f;
        if (lane == 0) {
            st = stats[r];
            if (xn) nv = norms[r];
        }
        int c = lane;
        for (; c + 96 < n16; c += 128) {
            const uint4 v0 = __ldcs(src + c), v1 = __ldcs(src + c + 32), v2 = __ldcs(src + c + 64),
                        v3 = __ldcs(src + c + 96);
            dst[c] = v0;
            dst[c + 32] = v1;
            dst[c + 64] = v2;
            dst[c + 96] = v3;
        }
        for (; c < n16; c += 32) dst[c] = __ldcs(src + c);
        if (lane == 0) {
            mb = fmaxf(mb, st.x);
            me = fmaxf(me, st.y);
            if (xn) xn[w] = nv;
        }
        r = rn;
    }
    if (lane == 0) {
        atomicMax(&xmax2[0], __float_as_uint(mb));
        atomicMax(&xmax2[1], __float_as_uint(me));
    }
}

// margin = 2 x E, with E the rigorous error of the approximate key:
//   L2: key = fl(||x||^2_fp32 - 2 acc)   E = 2 E_dot + E_norm + E_round
//   IP: key = -acc                        E = E_dot
//   E_dot = ||q~|| Dx + ||dq|| X~ + ||dq|| Dx + E_acc
//   E_acc = max(2^-14, (ceil(d/16) + 4) 2^-20) ||q~|| X~: the tensor core's fp32
//           accumulation, whose rounding NVIDIA does not document. bf16 x bf16
//           products are exact in fp32; each of the ceil(d/16) K=16 MMA steps
//           adds one accumulator rounding, and the 16-term sum inside one step
//           at most log2(16) = 4 more. Any order of summation then errs by at
//           most (steps) x (per-rounding error) x sum|q~_i x~_i| <= ... x
//           ||q~|| X~ (Cauchy-Schwarz). 2^-20 per rounding allows a 20-bit
//           accumulator (16x round-to-nearest fp32's 2^-24, 8x truncation's
//           2^-23); for d <= 1024 the 2^-14 floor dominates.
//           tests/test_gpu_tc.py::test_adversarial_cancellation exercises it.
//   E_norm = (d + 2) 2^-24 X^2,  E_round = 2^-23 (X^2 + 2 ||q~|| X~)
__global__ void k_tc_margins(const float2* __restrict__ qerr, int64_t nq, int d, const unsigned* __restrict__ xmax,
                             const unsigned* __restrict__ xmax2, int ip, float* __restrict__ margin) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq) return;
    const float2 qe = qerr[i];
    const float Xt = sqrtf(__uint_as_float(xmax2[0])) * 1.0001f;   // max ||x~||
    const float Dx = sqrtf(__uint_as_float(xmax2[1])) * 1.0001f;   // max ||dx||
    const float X2 = __uint_as_float(*xmax) * 1.0002f;             // max ||x||^2 (fp32)
    const float acc_u = fmaxf(6.103515625e-05f, (float)((d + 15) / 16 + 4) * 9.5367431640625e-07f);
    const float edot = qe.x * Dx + qe.y * Xt + qe.y * Dx + acc_u * qe.x * Xt;
    float e;
    if (ip) {
        e = edot;
    } else {
        e = 2.f * edot + (float)(d + 2) * 5.9604645e-08f * X2 + 1.1920929e-07f * (X2 + 2.f * qe.x * Xt);
    }
    margin[i] = 2.f * e * 1.01f;
}

// admission-bound seed: U = k-th smallest of a query's chunk minima over a
// sample of rows (the first `nch` x 32 staged rows, MODE 3 with minima only)
// is an upper bound on its k-th smallest key over all rows (k rows of the
// sample have key <= U), so phase A may start with tau_g = U instead of
// +inf (phase B's verification covers it like any tau_g). One warp per query.
__global__ void k_tau_seed(const float* __restrict__ mins, int64_t nq, int nch, int k, const float* __restrict__ margin,
                           unsigned* __restrict__ tau) {
    const int lane = threadIdx.x & 31;
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (q >= nq) return;
    const float* m = mins + q * (int64_t)nch;
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (int i = lane; i < nch; i += 32) {
        const uint32_t u = f2o(m[i]);
        lo = min(lo, u);
        hi = max(hi, u);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    uint32_t res = lo;
    if (lo != hi) {
        const int top = 31 - __clz(lo ^ hi);
        res = lo & ~((top == 31 ? 0u : (2u << top)) - 1u);
        for (int b = top; b >= 0; --b) {
            const uint32_t t = res | (1u << b);
            unsigned c = 0;
            for (int i = lane; i < nch; i += 32) c += f2o(m[i]) < t ? 1u : 0u;
            c = __reduce_add_sync(0xffffffffu, c);
            if (c < (unsigned)k) res = t;
        }
    }
    // + 1.5 margins: the verification (k-th exact key + margin/2 below tau_g
    // - margin/2) then holds even when U is the k-th key itself
    if (lane == 0) tau[q] = f2o(__fadd_ru(o2f(res), 1.5f * margin[q]));
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

bool make_map(CUtensorMap* map, const void* gaddr, int64_t rows, int d, int dp, int box_rows, bool f16 = false) {
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)std::max<int64_t>(rows, 1)};
    cuuint64_t strides[1] = {(cuuint64_t)dp * 2};
    cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(gaddr), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
}  // namespace

// launch one variant of the phase-A kernel; CTA pairs go out as clusters of 2
template <bool IP, int MODE, bool PAIR>
cudaError_t launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const tc::Params& pr, unsigned grid,
                      cudaStream_t st, const CUtensorMap* ma32 = nullptr, const CUtensorMap* ma64 = nullptr);
template <bool IP, int MODE, bool PAIR>
cudaError_t launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const tc::Params& pr, unsigned grid,
                      cudaStream_t st, const CUtensorMap* ma32, const CUtensorMap* ma64) {
    auto kern = tc::k_enn_scan_tc<IP, MODE, PAIR>;
    const size_t sm = tc::smem_bytes<PAIR>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    if (PAIR) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
        cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc::NTHREADS);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = PAIR ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, ma, mb, pr, ma32 ? *ma32 : ma, ma64 ? *ma64 : ma);
}

// CTA pairs unless disabled (VS_TC_PAIR=0) or the batch fits one 128-query tile
bool use_pair(int64_t nq) {
    static const char* env = getenv("VS_TC_PAIR");
    if (env) return env[0] == '1';
    return nq > tc::BM;
}

bool tc_supported(int d, int dtype, int ip) {
    (void)dtype;
    (void)ip;
    return d >= 8 && get_encode();
}

// fp16 operands for float32 rows whose max norm is known (the power-of-two
// scaling needs it); VS_TC_BF16=1 keeps bf16 (A/B runs)
bool use_f16(int dtype, const unsigned* xmax) {
    static const bool bf16_env = getenv("VS_TC_BF16") != nullptr && getenv("VS_TC_BF16")[0] == '1';
    return dtype == VS_DTYPE_F32 && xmax != nullptr && !bf16_env;
}

// the fp16 shadow of a float32 column (k_stage_rows over all rows, scale from
// its max norm, per-row stats kept)
int tc_build_f16_shadow(vs_ctx* ctx, const float* x, int64_t n, int d, const unsigned* xmax, void* shadow,
                        float2* stats) {
    using namespace vs_internal;
    const int dp = (d + 7) / 8 * 8;
    unsigned* junk = nullptr;
    CKS(arena_alloc(ctx, 2, &junk));
    const unsigned blocks = (unsigned)std::min<int64_t>((n * 32 + 255) / 256, 148 * 64);
    tc::k_stage_rows<float, __half><<<blocks, 256, 0, ctx->stream>>>(x, nullptr, n, d, dp, nullptr, (__half*)shadow,
                                                                     nullptr, junk, xmax, stats);
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    return VS_OK;
}

bool tc_profitable(int64_t nq, int64_t nsel, int d) {
    return nq >= 64 && (double)nq * (double)nsel * (double)d >= 4.0e9;
}

int tc_enn_scan(vs_ctx* ctx, EnnScanParams& sp, int dtype, const unsigned* xmax, int cshift, CandBuf* cb,
                bool* exhaustive, int timer_class) {
    // first pass: local top-k buffers verified by phase B; re-runs (cshift > 0)
    // keep the full margin band, which is exact by construction
    const int topk_mode = (cshift == 0 && !getenv("VS_TC_MARGIN_MODE")) ? 1 : 0;
    using namespace vs_internal;
    // this translation unit's copy of the driver entry point (the file is
    // compiled once per tile width)
    if (!get_encode()) return set_err(VS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cudaStream_t st = ctx->stream;
    const int d = sp.d;
    const int dp = (d + 7) / 8 * 8;
    const int64_t nq = sp.nq, nsel = sp.nsel;
    // staging buffers
    __nv_bfloat16 *qa = nullptr, *xb = nullptr;
    float *xn = nullptr, *margin = nullptr;
    float2* qerr = nullptr;
    unsigned* tau_g = nullptr;
    unsigned* xmax2 = nullptr;
    float* kinv = nullptr;
    // float32 rows: fp16 operands (8x smaller rounding error than bf16, same
    // tensor throughput); bf16-stored rows stay their own exact operand
    const bool f16 = use_f16(dtype, xmax);
    CKS(arena_alloc(ctx, (size_t)nq * dp, &qa));
    CKS(arena_alloc(ctx, (size_t)nsel * dp, &xb));
    CKS(arena_alloc(ctx, (size_t)nsel, &xn));
    CKS(arena_alloc(ctx, (size_t)nq, &margin));
    CKS(arena_alloc(ctx, (size_t)nq, &qerr));
    CKS(arena_alloc(ctx, (size_t)nq, &tau_g));
    CKS(arena_alloc(ctx, 2, &xmax2));
    if (f16) CKS(arena_alloc(ctx, (size_t)nq, &kinv));
    {
        KTimer kt(ctx, VS_K_STAGE);
        CK(cudaMemsetAsync(xmax2, 0, 2 * sizeof(unsigned), st));
        // rows first: they do not need the queries, whose host->device copy may
        // still be in flight on the copy stream (sp.q_ready)
        const unsigned blocks = (unsigned)std::min<int64_t>((nsel * 32 + 255) / 256, 148 * 64);
        if (f16 && sp.f16 && dp % 8 == 0)
            tc::k_stage_rows_f16<<<blocks, 256, 0, st>>>((const __half*)sp.f16, sp.f16_stats, sp.sel, nsel, dp,
                                                         sp.xnorm, (__half*)xb, sp.ip ? nullptr : xn, xmax2);
        else if (f16)
            tc::k_stage_rows<float, __half><<<blocks, 256, 0, st>>>((const float*)sp.X, sp.sel, nsel, d, dp,
                                                                    sp.xnorm, (__half*)xb, sp.ip ? nullptr : xn,
                                                                    xmax2, xmax);
        else if (dtype == VS_DTYPE_F32)
            tc::k_stage_rows<float, __nv_bfloat16><<<blocks, 256, 0, st>>>((const float*)sp.X, sp.sel, nsel, d, dp,
                                                                           sp.xnorm, xb, sp.ip ? nullptr : xn, xmax2);
        else
            tc::k_stage_rows<__nv_bfloat16, __nv_bfloat16><<<blocks, 256, 0, st>>>(
                (const __nv_bfloat16*)sp.X, sp.sel, nsel, d, dp, sp.xnorm, xb, sp.ip ? nullptr : xn, xmax2);
        CK(cudaGetLastError());
        if (sp.q_ready) CK(cudaStreamWaitEvent(st, sp.q_ready, 0));
        const unsigned qblocks = (unsigned)std::min<int64_t>((nq * 32 + 255) / 256, 148 * 16);
        if (f16)
            tc::k_stage_queries<__half><<<qblocks, 256, 0, st>>>(sp.Q, nq, d, dp, (__half*)qa, qerr, xmax, kinv);
        else
            tc::k_stage_queries<__nv_bfloat16><<<qblocks, 256, 0, st>>>(sp.Q, nq, d, dp, qa, qerr, nullptr, nullptr);
        CK(cudaGetLastError());
        tc::k_tc_margins<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(qerr, nq, d, xmax, xmax2, sp.ip, margin);
        CK(cudaGetLastError());
        CK(cudaMemsetAsync(tau_g, 0xff, nq * sizeof(unsigned), st));
        ctx->stats[VS_STAT_LAUNCHES] += 3;
    }
    // tiling: work item = (query tile, data split); choose the split count
    // so items fill whole waves of SMs
    const bool pair = use_pair(nq);
    const int qtile_rows = pair ? 2 * tc::BM : tc::BM;
    const int qtiles = (int)((nq + qtile_rows - 1) / qtile_rows);
    const int64_t ntiles = (nsel + tc::BN - 1) / tc::BN;
    const int sm_avail = std::max(2, ctx->sm_count - ctx->sm_reserve);      // SMs left to this kernel
    const int sms = pair ? sm_avail / 2 : sm_avail;                         // work units (CTAs or pairs)
    // split count: >= 2 waves of work items; among those the smallest makespan
    // (short splits also keep every candidate buffer below its compaction point)
    const int64_t C0 = topk_mode ? vs_internal::pow2ceil(2 * sp.k + 96 + tc::BN / 2)
                                 : vs_internal::pow2ceil(sp.k + 512);
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
    if (getenv("VS_TC_NSPLIT")) best_s = std::max(1, std::min<int>((int)ntiles, atoi(getenv("VS_TC_NSPLIT"))));
    const int64_t per = (ntiles + best_s - 1) / best_s;
    const int nsplit = (int)((ntiles + per - 1) / per);
    // a buffer must hold the kept set plus one half-tile of appends (128)
    // between compactions, else it compacts on every tile
    int64_t C = C0 << (ctx->opt_slack + cshift);
    const int64_t rows_per_split = per * tc::BN / 2;  // per column half
    const int64_t cap = vs_internal::pow2ceil(rows_per_split + 64);
    *exhaustive = C >= cap;
    if (C > cap) C = cap;
    CandBuf c;
    c.n_sub = 2 * nsplit;
    c.C = (int)C;
    const size_t slots = (size_t)nq * c.n_sub * C;
    CKS(arena_alloc(ctx, slots, &c.key));
    CKS(arena_alloc(ctx, slots, &c.pos));
    CKS(arena_alloc(ctx, (size_t)nq * c.n_sub, &c.cnt));
    CKS(arena_alloc(ctx, (size_t)nq, &c.overflow));
    CK(cudaMemsetAsync(c.overflow, 0, nq * sizeof(int), st));

    CUtensorMap ma, mb;
    if (!make_map(&ma, qa, nq, d, dp, tc::BM, f16) || !make_map(&mb, xb, nsel, d, dp, pair ? tc::BN / 2 : tc::BN, f16))
        return set_err(VS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    tc::Params pr{};
    pr.f16 = f16 ? 1 : 0;
    pr.kinv = kinv;
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
    pr.dbg = nullptr;
    pr.topk_mode = topk_mode;
    static const bool dbg_on = getenv("VS_TC_DEBUG") != nullptr;
    if (dbg_on) {
        CKS(arena_alloc(ctx, 16, &pr.dbg));
        CK(cudaMemsetAsync(pr.dbg, 0, 16 * sizeof(unsigned long long), st));
    }
    const int64_t items = (int64_t)qtiles * nsplit;
    const unsigned units = (unsigned)std::min<int64_t>(items, sms);
    const unsigned grid = pair ? 2 * units : units;
    pr.argmin_out = nullptr;
    static const int lim0_env = getenv("VS_TC_LIM0") ? atoi(getenv("VS_TC_LIM0")) : 0;
    pr.lim0 = lim0_env;
    pr.dense_direct = (per >= 8 && per < 128) ? 1 : 0;
    // admission-bound seed from a row sample (short splits admit most of their
    // first keys before their local k-th settles; VS_TC_TAU_SAMPLE = sample
    // rows, 0 = off)
    // (default 8192 rows when the selection has at least 4x that; measured on
    // config 2: MMA wait on the epilogue 2.65 M -> 0.60 M cycles per CTA, phase
    // A 17.3 -> 16.2 ms for 0.22 ms of sample GEMM; 8 row shards: 2.94 -> 1.95 ms)
    const int64_t tau_sample = getenv("VS_TC_TAU_SAMPLE") ? atoll(getenv("VS_TC_TAU_SAMPLE")) : 8192;
    const int64_t nch_s = nsel >= 4 * tau_sample ? tau_sample / 32 : 0;
    if (topk_mode && !*exhaustive && nch_s >= sp.k && nch_s > 0) {
        float* smins = nullptr;
        CKS(arena_alloc(ctx, (size_t)nq * nch_s, &smins));
        CUtensorMap mbs;
        if (!make_map(&mbs, xb, nch_s * 32, d, dp, pair ? tc::BN / 2 : tc::BN, f16))
            return set_err(VS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        tc::Params ps = pr;
        ps.nsel = nch_s * 32;
        ps.ntiles = (ps.nsel + tc::BN - 1) / tc::BN;
        ps.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(ps.ntiles, (2 * sms + qtiles - 1) / qtiles));
        ps.tiles_per_split = (ps.ntiles + ps.nsplit - 1) / ps.nsplit;
        ps.nsplit = (int)((ps.ntiles + ps.tiles_per_split - 1) / ps.tiles_per_split);
        ps.keys_out = nullptr;
        ps.mins_out = smins;
        ps.mins_ld = nch_s;
        const int64_t items_s = (int64_t)qtiles * ps.nsplit;
        const unsigned units_s = (unsigned)std::min<int64_t>(items_s, sms);
        const unsigned grid_s = pair ? 2 * units_s : units_s;
        {
            KTimer kt(ctx, VS_K_STAGE);
            if (sp.ip) CK((pair ? launch_tc<true, 3, true>(ma, mbs, ps, grid_s, st) : launch_tc<true, 3, false>(ma, mbs, ps, grid_s, st)));
            else CK((pair ? launch_tc<false, 3, true>(ma, mbs, ps, grid_s, st) : launch_tc<false, 3, false>(ma, mbs, ps, grid_s, st)));
            tc::k_tau_seed<<<(unsigned)((nq * 32 + 255) / 256), 256, 0, st>>>(smins, nq, (int)nch_s, sp.k, margin, tau_g);
            CK(cudaGetLastError());
        }
        ctx->stats[VS_STAT_LAUNCHES] += 2;
    }
    KTimer kt_scan(ctx, timer_class);
    if (sp.ip) {
        CK((pair ? launch_tc<true, 0, true>(ma, mb, pr, grid, st) : launch_tc<true, 0, false>(ma, mb, pr, grid, st)));
    } else {
        CK((pair ? launch_tc<false, 0, true>(ma, mb, pr, grid, st) : launch_tc<false, 0, false>(ma, mb, pr, grid, st)));
    }
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    if (dbg_on) {
        unsigned long long h[16];
        CK(cudaMemcpyAsync(h, pr.dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double ctas = (double)(pair ? units : grid), thr = (double)grid * tc::EPI_THREADS;
        fprintf(stderr,
                "[vs_tc] grid=%u nsplit=%d per=%lld C=%lld tiles/cta=%.1f | producer wait-empty %.0f cyc/cta | "
                "mma wait-full %.0f wait-tempty %.0f cyc/cta | epi wait-tfull %.0f compaction %.0f cyc/thr | "
                "compactions %.2f appends %.1f per row-split | tmem-ld wait %.0f chunk-loop %.0f cyc/thr\n",
                grid, nsplit, (long long)per, (long long)C, h[7] / ctas, h[0] / ctas, h[1] / ctas, h[2] / ctas,
                h[3] / thr, h[4] / thr, (double)h[5] / ((double)nq * 2 * nsplit), (double)h[6] / ((double)nq * 2 * nsplit),
                h[8] / thr, h[9] / thr);
    }
    // phase B reads rows through the selection (sp.sel) from the original
    // column, with the tensor-core margins
    sp.margin = margin;
    sp.tau_g = tau_g;
    sp.verify = topk_mode;
    *cb = c;
    return VS_OK;
}

// First-min nearest column under squared L2 (key ||c||^2 - 2 x.c) for every
// row of x, on the tensor cores: the k-means assignment step. `cb` holds the
// columns (centroids) already staged as bf16 [ncols][dp] with their fp32
// norms; rows are staged here in chunks. out[r] = (orderable key << 32) | col.
int64_t tc_argmin_chunk(int64_t n) { return std::min<int64_t>(n, (int64_t)1 << 22); }

int tc_argmin_rows(vs_ctx* ctx, const void* x, int dtype, int64_t n, int d, const __nv_bfloat16* cb,
                   const float* cnorm, int64_t ncols, unsigned long long* out, __nv_bfloat16* xb,
                   unsigned* junk, unsigned long long* top2, float2* rowstats, const unsigned* row_xmax,
                   const unsigned* col_xmax) {
    // fp16 operands (both scales known; columns staged by tc_stage_f16; bf16
    // rows convert exactly unless far below the column's max norm)
    const bool f16 = row_xmax && col_xmax;
    using namespace vs_internal;
    if (!get_encode()) return set_err(VS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cudaStream_t st = ctx->stream;
    const int dp = (d + 7) / 8 * 8;
    const int64_t chunk = tc_argmin_chunk(n);
    CK(cudaMemsetAsync(out, 0xff, n * sizeof(unsigned long long), st));
    const bool pair = use_pair(n);
    CUtensorMap mb;
    if (!make_map(&mb, cb, ncols, d, dp, pair ? tc::BN / 2 : tc::BN, f16))
        return set_err(VS_ERR_CUDA, "tensor map (columns)");
    for (int64_t r0 = 0; r0 < n; r0 += chunk) {
        const int64_t m = std::min(chunk, n - r0);
        const unsigned blocks = (unsigned)std::min<int64_t>((m * 32 + 255) / 256, 148 * 64);
        if (f16 && dtype == VS_DTYPE_F32)
            tc::k_stage_rows<float, __half><<<blocks, 256, 0, st>>>(
                (const float*)x + r0 * (int64_t)d, nullptr, m, d, dp, nullptr, (__half*)xb, nullptr, junk, row_xmax,
                rowstats ? rowstats + r0 : nullptr);
        else if (f16)
            tc::k_stage_rows<__nv_bfloat16, __half><<<blocks, 256, 0, st>>>(
                (const __nv_bfloat16*)x + r0 * (int64_t)d, nullptr, m, d, dp, nullptr, (__half*)xb, nullptr, junk,
                row_xmax, rowstats ? rowstats + r0 : nullptr);
        else if (dtype == VS_DTYPE_F32)
            tc::k_stage_rows<float, __nv_bfloat16><<<blocks, 256, 0, st>>>(
                (const float*)x + r0 * (int64_t)d, nullptr, m, d, dp, nullptr, xb, nullptr, junk, nullptr,
                rowstats ? rowstats + r0 : nullptr);
        else
            tc::k_stage_rows<__nv_bfloat16, __nv_bfloat16><<<blocks, 256, 0, st>>>(
                (const __nv_bfloat16*)x + r0 * (int64_t)d, nullptr, m, d, dp, nullptr, xb, nullptr, junk, nullptr,
                rowstats ? rowstats + r0 : nullptr);
        CK(cudaGetLastError());
        CUtensorMap ma;
        if (!make_map(&ma, xb, m, d, dp, tc::BM, f16)) return set_err(VS_ERR_CUDA, "tensor map (rows)");
        tc::Params pr{};
        pr.nq = m;
        pr.d = d;
        pr.kblocks = (d + tc::BK - 1) / tc::BK;
        pr.nsel = ncols;
        pr.qtiles = (int)((m + (pair ? 2 * tc::BM : tc::BM) - 1) / (pair ? 2 * tc::BM : tc::BM));
        pr.nsplit = 1;
        pr.ntiles = (ncols + tc::BN - 1) / tc::BN;
        pr.tiles_per_split = pr.ntiles;
        pr.xn = cnorm;
        pr.argmin_out = out + r0;
        pr.top2_out = top2 ? top2 + r0 * 4 : nullptr;
        pr.f16 = f16 ? 1 : 0;
        pr.a_scale_src = f16 ? row_xmax : nullptr;
        pr.b_scale_src = f16 ? col_xmax : nullptr;
        const unsigned units = (unsigned)std::min<int64_t>(pr.qtiles, pair ? ctx->sm_count / 2 : ctx->sm_count);
        CK((pair ? launch_tc<false, 1, true>(ma, mb, pr, 2 * units, st)
                 : launch_tc<false, 1, false>(ma, mb, pr, units, st)));
        CK(cudaGetLastError());
        ctx->stats[VS_STAT_LAUNCHES] += 2;
    }
    return VS_OK;
}

// stage a float32 matrix to fp16 [n][dp] scaled by pow2_scale(*xmax) (the
// k-means centroids for an fp16 argmin); max (||x~||^2, ||dx||^2) into stats
int tc_stage_f16(vs_ctx* ctx, const float* x, int64_t n, int d, const unsigned* xmax, void* out, unsigned* stats) {
    using namespace vs_internal;
    const int dp = (d + 7) / 8 * 8;
    const unsigned blocks = (unsigned)std::min<int64_t>((n * 32 + 255) / 256, 148 * 64);
    tc::k_stage_rows<float, __half><<<blocks, 256, 0, ctx->stream>>>(x, nullptr, n, d, dp, nullptr, (__half*)out,
                                                                     nullptr, stats, xmax);
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    return VS_OK;
}

// stage a float32 matrix to bf16 [n][dp] (no norms)
int tc_stage_bf16(vs_ctx* ctx, const float* x, int64_t n, int d, __nv_bfloat16* out, unsigned* junk) {
    using namespace vs_internal;
    const int dp = (d + 7) / 8 * 8;
    const unsigned blocks = (unsigned)std::min<int64_t>((n * 32 + 255) / 256, 148 * 64);
    tc::k_stage_rows<float, __nv_bfloat16><<<blocks, 256, 0, ctx->stream>>>(x, nullptr, n, d, dp, nullptr, out, nullptr,
                                                                            junk);
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    return VS_OK;
}

// Dense approximate keys of every (query, column) pair on the tensor cores
// (MODE 3): keys[q][c] = ||c||^2 - 2 q~.c~ (or -q~.c~), margin[q] = 2 x their
// rigorous error bound (k_tc_margins). The IVF coarse quantizer's phase A:
// its columns (the centroids) are few enough that the whole key matrix of a
// query chunk is cheaper to write and select from than candidate buffers.
int tc_dense_keys(vs_ctx* ctx, const float* Q, int64_t nq, int d, const float* X, int64_t ncols,
                  const float* xnorm, const unsigned* xmax, int ip, float* keys, float* margin, float* mins) {
    using namespace vs_internal;
    if (!get_encode()) return set_err(VS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cudaStream_t st = ctx->stream;
    const int dp = (d + 7) / 8 * 8;
    __nv_bfloat16 *qa = nullptr, *xb = nullptr;
    float* xn = nullptr;
    float2* qerr = nullptr;
    unsigned* xmax2 = nullptr;
    float* kinv = nullptr;
    const bool f16 = use_f16(VS_DTYPE_F32, xmax);
    CKS(arena_alloc(ctx, (size_t)nq * dp, &qa));
    CKS(arena_alloc(ctx, (size_t)ncols * dp, &xb));
    CKS(arena_alloc(ctx, (size_t)ncols, &xn));
    CKS(arena_alloc(ctx, (size_t)nq, &qerr));
    CKS(arena_alloc(ctx, 2, &xmax2));
    if (f16) CKS(arena_alloc(ctx, (size_t)nq, &kinv));
    {
        KTimer kt(ctx, VS_K_STAGE);
        CK(cudaMemsetAsync(xmax2, 0, 2 * sizeof(unsigned), st));
        const unsigned blocks = (unsigned)std::min<int64_t>((ncols * 32 + 255) / 256, 148 * 64);
        const unsigned qblocks = (unsigned)std::min<int64_t>((nq * 32 + 255) / 256, 148 * 16);
        if (f16) {
            tc::k_stage_rows<float, __half><<<blocks, 256, 0, st>>>(X, nullptr, ncols, d, dp, xnorm, (__half*)xb,
                                                                    ip ? nullptr : xn, xmax2, xmax);
            CK(cudaGetLastError());
            tc::k_stage_queries<__half><<<qblocks, 256, 0, st>>>(Q, nq, d, dp, (__half*)qa, qerr, xmax, kinv);
        } else {
            tc::k_stage_rows<float, __nv_bfloat16><<<blocks, 256, 0, st>>>(X, nullptr, ncols, d, dp, xnorm, xb,
                                                                           ip ? nullptr : xn, xmax2);
            CK(cudaGetLastError());
            tc::k_stage_queries<__nv_bfloat16><<<qblocks, 256, 0, st>>>(Q, nq, d, dp, qa, qerr, nullptr, nullptr);
        }
        CK(cudaGetLastError());
        tc::k_tc_margins<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(qerr, nq, d, xmax, xmax2, ip, margin);
        CK(cudaGetLastError());
        ctx->stats[VS_STAT_LAUNCHES] += 3;
    }
    const bool pair = use_pair(nq);
    const int qtile_rows = pair ? 2 * tc::BM : tc::BM;
    const int qtiles = (int)((nq + qtile_rows - 1) / qtile_rows);
    const int64_t ntiles = (ncols + tc::BN - 1) / tc::BN;
    const int sms = pair ? ctx->sm_count / 2 : ctx->sm_count;
    // splits: >= 2 waves of work items, the shortest makespan (no buffers to size)
    int best_s = 1;
    double best_cost = 1e30;
    for (int s = 1; s <= std::min<int64_t>(ntiles, 64); ++s) {
        const int64_t per = (ntiles + s - 1) / s;
        const int64_t items = (int64_t)qtiles * ((ntiles + per - 1) / per);
        const double cost = std::ceil((double)items / sms) * per + 0.5 * per / 8.0;
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best_s = s;
        }
    }
    const int64_t per = (ntiles + best_s - 1) / best_s;
    const int nsplit = (int)((ntiles + per - 1) / per);
    CUtensorMap ma, mb;
    if (!make_map(&ma, qa, nq, d, dp, tc::BM, f16) || !make_map(&mb, xb, ncols, d, dp, pair ? tc::BN / 2 : tc::BN, f16))
        return set_err(VS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    tc::Params pr{};
    pr.f16 = f16 ? 1 : 0;
    pr.kinv = kinv;
    pr.nq = nq;
    pr.d = d;
    pr.kblocks = (d + tc::BK - 1) / tc::BK;
    pr.nsel = ncols;
    pr.qtiles = qtiles;
    pr.nsplit = nsplit;
    pr.tiles_per_split = per;
    pr.ntiles = ntiles;
    pr.xn = xn;
    pr.ip = ip;
    pr.keys_out = keys;
    pr.keys_ld = ncols;
    pr.mins_out = mins;
    pr.mins_ld = (ncols + 31) / 32;
    const int64_t items = (int64_t)qtiles * nsplit;
    const unsigned units = (unsigned)std::min<int64_t>(items, sms);
    const unsigned grid = pair ? 2 * units : units;
    KTimer kt(ctx, VS_K_COARSE);
    if (ip) CK((pair ? launch_tc<true, 3, true>(ma, mb, pr, grid, st) : launch_tc<true, 3, false>(ma, mb, pr, grid, st)));
    else CK((pair ? launch_tc<false, 3, true>(ma, mb, pr, grid, st) : launch_tc<false, 3, false>(ma, mb, pr, grid, st)));
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    return VS_OK;
}

// fp16 copy of a query batch (per-query power-of-two scales against rows of
// max norm^2 *xmax) and its tensor-core margins against rows bounded by xmax2
// (the filtered tensor-core IVF scan, vs_ivf_sel.cu)
int tc_stage_queries_f16(vs_ctx* ctx, const float* Q, int64_t nq, int d, const unsigned* xmax,
                         const unsigned* xmax2, int ip, __half* out, float* kinv, float* margin) {
    using namespace vs_internal;
    float2* qerr = nullptr;
    CKS(arena_alloc(ctx, (size_t)nq, &qerr));
    const int dp = (d + 7) / 8 * 8;
    tc::k_stage_queries<__half><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((nq * 32 + 255) / 256, 148 * 16)), 256,
                                  0, ctx->stream>>>(Q, nq, d, dp, out, qerr, xmax, kinv);
    CK(cudaGetLastError());
    tc::k_tc_margins<<<(unsigned)((nq + 255) / 256), 256, 0, ctx->stream>>>(qerr, nq, d, xmax, xmax2, ip, margin);
    CK(cudaGetLastError());
    ctx->stats[VS_STAT_LAUNCHES] += 2;
    return VS_OK;
}

int tc_ivf_scan(vs_ctx* ctx, const TcIvfArgs& a, TcIvfOut* out) {
    using namespace vs_internal;
    if (!get_encode()) return set_err(VS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (a.d % 8) return set_err(VS_ERR_PARAMETER, "tensor-core IVF scan needs d %% 8 == 0");
    cudaStream_t st = ctx->stream;
    const int d = a.d, dp = (d + 7) / 8 * 8;
    // margin mode: a buffer (pair, column half) sees one list, and the nearest
    // list's buffer usually holds the whole top-k, so the local-top-k +
    // verification scheme of the exhaustive scan would fail its check there;
    // keeping the band key <= local k-th + margin is exact by construction
    const int topk_mode = 0;
    __nv_bfloat16 *qp = nullptr, *qa = nullptr;
    float* margin = nullptr;
    float2* qerr = nullptr;
    unsigned *tau_g = nullptr, *xmax2 = nullptr;
    CKS(arena_alloc(ctx, (size_t)std::max<int64_t>(a.npairs, 1) * dp, &qp));
    CKS(arena_alloc(ctx, (size_t)a.nq * dp, &qa));
    CKS(arena_alloc(ctx, (size_t)a.nq, &margin));
    CKS(arena_alloc(ctx, (size_t)a.nq, &qerr));
    CKS(arena_alloc(ctx, (size_t)a.nq, &tau_g));
    CKS(arena_alloc(ctx, 2, &xmax2));
    {
        KTimer kt(ctx, VS_K_STAGE);
        tc::k_stage_pair_queries<<<(unsigned)std::min<int64_t>((a.npairs * 32 + 255) / 256, 148 * 32), 256, 0, st>>>(
            a.Q, a.pair_codes, a.npairs, a.nprobe, d, dp, qp);
        CK(cudaGetLastError());
        tc::k_stage_queries<__nv_bfloat16><<<(unsigned)std::min<int64_t>((a.nq * 32 + 255) / 256, 148 * 16), 256, 0,
                                             st>>>(a.Q, a.nq, d, dp, qa, qerr, nullptr, nullptr);
        CK(cudaGetLastError());
        // bf16-stored rows are their own tensor-core operand: ||x~|| = ||x||, dx = 0
        CK(cudaMemsetAsync(xmax2, 0, 2 * sizeof(unsigned), st));
        CK(cudaMemcpyAsync(xmax2, a.pmax, sizeof(unsigned), cudaMemcpyDeviceToDevice, st));
        tc::k_tc_margins<<<(unsigned)((a.nq + 255) / 256), 256, 0, st>>>(qerr, a.nq, d, a.pmax, xmax2, a.ip, margin);
        CK(cudaGetLastError());
        CK(cudaMemsetAsync(tau_g, 0xff, a.nq * sizeof(unsigned), st));
        ctx->stats[VS_STAT_LAUNCHES] += 3;
    }
    // room for one half-tile of appends (128) beyond the kept band
    int64_t C = pow2ceil(2 * a.k + 96 + tc::BN / 2) << (ctx->opt_slack + a.cshift);
    // one buffer per (pair, [chunk,] column half): a column half sees <= 128 rows per tile
    const int64_t rows_seen = a.chunk_rows ? std::min(a.max_list, a.chunk_rows) : a.max_list;
    const int64_t cap = pow2ceil((rows_seen + tc::BN - 1) / tc::BN * (tc::BN / 2) + 64);
    out->exhaustive = C >= cap;
    if (C > cap) C = cap;
    CandBuf c;
    c.C = (int)C;
    const int64_t nbuf = a.pair_base ? a.total_subs : a.nq * 2 * (int64_t)a.nprobe;
    c.n_sub = a.pair_base ? a.max_subs : 2 * a.nprobe;
    c.sub_off = a.pair_base ? a.sub_off : nullptr;
    const size_t slots = (size_t)nbuf * C;
    CKS(arena_alloc(ctx, slots, &c.key));
    CKS(arena_alloc(ctx, slots, &c.pos));
    CKS(arena_alloc(ctx, (size_t)nbuf, &c.cnt));
    CKS(arena_alloc(ctx, (size_t)a.nq, &c.overflow));
    CK(cudaMemsetAsync(c.overflow, 0, a.nq * sizeof(int), st));
    CK(cudaMemsetAsync(c.cnt, 0, (size_t)nbuf * sizeof(int), st));
    CUtensorMap ma, mb;
    static const int a32_env = getenv("VS_TC_A32") ? atoi(getenv("VS_TC_A32")) : 2;
    CUtensorMap ma32, ma64;
    if (!make_map(&ma, qp, std::max<int64_t>(a.npairs, 1), d, dp, tc::BM) ||
        !make_map(&mb, a.payload, a.n_total, d, d, tc::BN) ||
        !make_map(&ma32, qp, std::max<int64_t>(a.npairs, 1), d, dp, a32_env == 2 ? 8 : 32) ||
        !make_map(&ma64, qp, std::max<int64_t>(a.npairs, 1), d, dp, a32_env == 2 ? 16 : 64))
        return set_err(VS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    tc::Params pr{};
    pr.nq = a.nq;
    pr.d = d;
    pr.kblocks = (d + tc::BK - 1) / tc::BK;
    pr.nsel = a.n_total;
    pr.qtiles = 1;
    pr.nsplit = 1;
    pr.tiles_per_split = 1;
    pr.ntiles = 1;
    pr.xn = a.pnorms;
    pr.margin = margin;
    pr.tau_g = tau_g;
    pr.ip = a.ip;
    pr.k = a.k;
    pr.cb = c;
    pr.dbg = nullptr;
    pr.topk_mode = topk_mode;
    pr.argmin_out = nullptr;
    pr.units = a.units;
    pr.n_units = a.n_units;
    pr.list_off = a.list_off;
    pr.pair_codes = a.pair_codes;
    pr.nprobe = a.nprobe;
    pr.pbits = a.pbits;
    static const int pf_env = getenv("VS_TC_PF") ? atoi(getenv("VS_TC_PF")) : tc::PF_BOXES;
    pr.pf_boxes = pf_env;
    pr.chunk_rows = a.pair_base ? a.chunk_rows : 0;
    pr.dense_direct = 0;
    pr.a32 = a32_env;
    pr.pair_base = a.pair_base;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(a.max_units, ctx->sm_count));
    static const bool dbg_on = getenv("VS_TC_DEBUG") != nullptr;
    if (dbg_on) {
        CKS(arena_alloc(ctx, 16, &pr.dbg));
        CK(cudaMemsetAsync(pr.dbg, 0, 16 * sizeof(unsigned long long), st));
    }
    {
        KTimer kt(ctx, a.timer_class);
        if (a.ip) CK((launch_tc<true, 2, false>(ma, mb, pr, grid, st, &ma32, &ma64)));
        else CK((launch_tc<false, 2, false>(ma, mb, pr, grid, st, &ma32, &ma64)));
    }
    ctx->stats[VS_STAT_LAUNCHES] += 1;
    if (dbg_on) {
        unsigned long long h[16];
        int nu = 0;
        CK(cudaMemcpyAsync(h, pr.dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&nu, a.n_units, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double ctas = grid, thr = (double)grid * tc::EPI_THREADS;
        fprintf(stderr,
                "[vs_tc ivf] grid=%u units=%d C=%lld tiles/cta=%.1f | producer wait-empty %.0f cyc/cta | "
                "mma wait-full %.0f wait-tempty %.0f cyc/cta | epi wait-tfull %.0f compaction %.0f cyc/thr | "
                "compactions %.0f appends %.0f total | tmem-ld wait %.0f chunk-loop %.0f cyc/thr | "
                "CTA busy max %.2f ms mean %.2f ms, tiles max %llu\n",
                grid, nu, (long long)C, h[7] / ctas, h[0] / ctas, h[1] / ctas, h[2] / ctas, h[3] / thr, h[4] / thr,
                (double)h[5], (double)h[6], h[8] / thr, h[9] / thr, h[10] / 1e6, h[11] / ctas / 1e6, h[12]);
    }
    out->cb = c;
    out->margin = margin;
    out->tau_g = tau_g;
    out->verify = topk_mode;
    return VS_OK;
}

}  // namespace VS_TC_NS
}  // namespace vs
