// Kernel parameter blocks and launchers shared between the kernel translation
// units and the C-ABI driver (vs_capi.cu).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace vs {

// Candidate buffers ("phase A" output): per (query, sub) C slots of
// (approximate key, position), counts [nq][n_sub], overflow flag per query.
struct CandBuf {
    float* key;        // [nq][n_sub][C]
    uint32_t* pos;     // [nq][n_sub][C]
    int* cnt;          // [nq][n_sub]
    int* overflow;     // [nq]
    int n_sub;         // subs per query (with sub_off: the maximum over queries)
    int C;
    const int64_t* sub_off = nullptr;   // [nq+1] variable subs per query (flat buffers), nullable
};

// ---- bitmap -> ascending selection vector -------------------------------------------
// rows with their bit set, ascending (the order-preserving gather of
// table.py:326-331 / relops.py:112-113)
cudaError_t launch_select_count(const uint32_t* bitmap, int64_t nwords, int64_t nbits,
                                int64_t* block_sums, int64_t nblocks, cudaStream_t s);
cudaError_t launch_select_scan(int64_t* block_sums, int64_t nblocks, int64_t* total,
                               cudaStream_t s);
cudaError_t launch_select_write(const uint32_t* bitmap, int64_t nwords, int64_t nbits,
                                const int64_t* block_offsets, int64_t* sel, cudaStream_t s);
int64_t select_nblocks(int64_t nwords);

// permuted bitmap over list-major payload positions: bit(pos) = bitmap[ids[pos]]
cudaError_t launch_permute_bitmap(const uint32_t* bitmap, int64_t nbits, const int64_t* ids,
                                  int64_t n_total, uint32_t* pbits, cudaStream_t s);

// ---- norms / margins ------------------------------------------------------------------
// row squared norms (fp32) and the max row norm (orderable bits, atomicMax)
template <typename T>
cudaError_t launch_row_norms(const T* x, int64_t n, int d, float* norms,
                             unsigned* max_norm_bits, cudaStream_t s);
// per-query admission margin = 2 x rigorous error bound of the approximate key
// (DESIGN.md §4): eps * (|q| + X)^2 for squared L2, eps * |q| * X for IP
cudaError_t launch_query_margins(const float* q, int64_t nq, int d, const unsigned* max_norm_bits,
                                 float eps, int ip, float* margin, float* qnorm, cudaStream_t s);

// ---- phase A: exhaustive scan (SIMT fp32) ----------------------------------------------
struct EnnScanParams {
    const float* Q;
    int64_t nq;
    int d;
    const void* X;          // base rows
    const int64_t* sel;     // selection positions -> base rows (nullable: identity)
    int64_t nsel;
    const float* xnorm;     // per base row ||x||^2 (squared L2)
    const float* margin;    // [nq]
    int ip;
    int k;
    int n_split;
    int64_t rows_per_split;
    CandBuf cb;
    unsigned* tau_g = nullptr;  // tensor-core path: per-query global admission bound
    int verify = 0;             // phase A kept local top-k only: phase B must verify
    int band_ready = 0;         // one buffer per query holding exactly the margin band (RerankParams)
    const void* f16 = nullptr;  // nullable: the column's fp16 shadow [n][dp] (staging gathers from it)
    const float2* f16_stats = nullptr;
    cudaEvent_t q_ready = nullptr;  // nullable: queries still in flight (host->device on a copy
                                    // stream); phase A stages the rows first, then waits
};
template <typename T>
cudaError_t launch_enn_scan_simt(const EnnScanParams& p, cudaStream_t s);

// ---- phase A: IVF list scan (query-major) -----------------------------------------------
struct IvfScanParams {
    const float* Q;
    int64_t nq;
    int d;
    const void* payload;        // list-major rows
    const int64_t* list_off;    // [nlist + 1]
    const int32_t* probes;      // [nq][nprobe]
    int nprobe;
    const uint8_t* list_owned;  // nullable
    const uint32_t* pbits;      // nullable (unfiltered)
    const float* margin;
    int ip;
    int k;
    int n_psplit;
    CandBuf cb;
    unsigned long long* visited;
};
template <typename T>
cudaError_t launch_ivf_scan_qmajor(const IvfScanParams& p, cudaStream_t s);

// ---- phase A: IVF list scan (list-major) ------------------------------------------------
// (query, probe) pairs grouped by list; units of <= kIvfLmQT pairs of one list
constexpr int kIvfLmQT = 8;
constexpr int kIvfLmDMax = 1024;   // list-major scan: query held in registers
struct IvfGroupArgs {
    const int32_t* probes;      // [nq][nprobe]
    int64_t nq;
    int nprobe;
    int nlist;
    const uint8_t* owned;       // nullable
    int32_t* keys_in;           // [nq*nprobe]
    int32_t* keys_out;          // [nq*nprobe]
    int32_t* vals_in;           // [nq*nprobe]
    int32_t* pair_codes;        // [nq*nprobe] out: q*nprobe + j, grouped by list
    int32_t* cnt;               // [nlist+1]
    int32_t* qoff;              // [nlist+1]
    int32_t* ucnt;              // [nlist+1]
    int32_t* uoff;              // [nlist+1] out: uoff[nlist] = number of units
    int4* units;                // [ivf_max_units] out: (list, first pair, pairs, 0)
    void* tmp;
    size_t tmp_bytes;           // >= ivf_group_temp_bytes
    int unit_pairs;             // max pairs per unit (kIvfLmQT SIMT, 128 tensor cores)
    const int32_t* chunks = nullptr;   // [nlist] row chunks per list (nullable: 1); a unit is
                                       // (list, pair range, chunk) -> int4 (list, first pair, pairs, chunk)
};
// long lists cut into row chunks (tensor-core IVF scan): per pair, the first of its
// 2 * chunks(list) buffers; per query, the offsets of its flat buffer range
cudaError_t launch_ivf_pair_subs(const int32_t* probes, int64_t nq, int nprobe, const int32_t* chunks,
                                 int64_t* sub_off, int64_t* pair_base, void* tmp, size_t tmp_bytes,
                                 cudaStream_t s);
size_t ivf_pair_subs_temp_bytes(int64_t nq);
size_t ivf_group_temp_bytes(int64_t npairs, int nlist);
int64_t ivf_max_units(int64_t nq, int nprobe, int nlist, int unit_pairs);
cudaError_t launch_ivf_group(const IvfGroupArgs& g, cudaStream_t s);

struct IvfLmParams {
    const float* Q;
    int64_t nq;
    int d;
    int dp;                     // d rounded up to 128 (query staging stride)
    const void* payload;
    const int64_t* list_off;
    int nprobe;
    const uint32_t* pbits;      // nullable
    const int32_t* pair_codes;
    const int4* units;
    const int32_t* n_units;     // device scalar (uoff[nlist])
    int64_t max_units;
    int* work;                  // zeroed work counter
    const float* margin;
    int ip;
    int k;
    CandBuf cb;                 // n_sub = nprobe: one buffer per (query, probe rank)
    unsigned long long* visited;
};
size_t ivf_lmajor_smem(int dp, int dtype_bytes);
template <typename T>
cudaError_t launch_ivf_scan_lmajor(const IvfLmParams& p, int sm_count, cudaStream_t s);

// ---- phase A: filtered IVF list scan over pre-selected rows (vs_ivf_sel.cu) --------------
struct IvfSelLaunch {
    const float* Q;
    int64_t nq;
    int d;
    const void* payload;
    const int64_t* list_off;
    int nlist;
    const uint32_t* pbits;      // permuted filter bitmap (required)
    const float* pnorm;         // ||x||^2 per payload row
    int nprobe;
    const int32_t* pair_codes;  // from launch_ivf_group (unit_pairs = kIvfLmQT)
    const int4* units;
    const int32_t* n_units;
    int64_t max_units;
    const float* margin;
    int ip, k;
    CandBuf cb;                 // n_sub = nprobe
    unsigned long long* visited;
    // scratch: lsel [nlist], lsel64 / sel_off [nlist + 1], spos [n_total], recs [max_units] x 128 B
    int32_t* lsel;
    int64_t* lsel64;
    int64_t* sel_off;
    uint32_t* spos;
    void* recs;
    // tensor-core variant (float payload, d % 16 == 0): the batch's queries as
    // fp16 with per-query power-of-two scales (kinv = 2^-(eq+ex)), rows scaled
    // by pow2_scale(*xscale) when staged; units of <= kMmaPairs pairs
    int mma = 0;
    const __half* Qh = nullptr;
    const float* kinv = nullptr;
    const unsigned* xscale = nullptr;
    void* tmp;
    size_t tmp_bytes;           // >= ivf_sel_temp_bytes(nlist)
    int sm_count;
};
constexpr size_t kIvfSelRecBytes = 128;
constexpr int kMmaPairs = 16;       // filtered tensor-core scan: pairs per unit (MMA M)
size_t ivf_sel_temp_bytes(int nlist);
size_t ivf_mma_smem(int d);
// a priori max ||x~||^2 / ||dx||^2 of fp16-rounded rows (scaled by their max norm)
cudaError_t launch_f16_row_bounds(const unsigned* xmax, int d, unsigned* out, cudaStream_t s);
template <typename T>
cudaError_t launch_ivf_scan_sel(const IvfSelLaunch& a, cudaStream_t s);
__global__ void k_list_selected(const int64_t* __restrict__ list_off, int nlist, const uint32_t* __restrict__ pbits,
                                int32_t* __restrict__ sel);

// ---- phase B: exact float64 re-rank + tie-rule top-k ------------------------------------
// numpy's pairwise-summation plan for one row length d (<= 2048): leaves left
// to right, internal nodes in post-order (slot nleaf + j = slot a_j + slot b_j),
// and the leaf index of every 8-element group
struct LeafPlan {
    int nleaf;
    int nnode;
    int nlevels;                // depth of the combine tree (nodes of one level are independent)
    int node_lvl[32];           // 0-based level of every node
    int leaf_off[32];
    int leaf_n[32];
    int node_a[32];
    int node_b[32];
    unsigned char gsk[2048 / 8];
};
void np_leaves(int d, LeafPlan& plan);

struct RerankParams {
    const float* Q;
    int64_t nq;
    int d;
    int ip;
    int k;
    CandBuf cb;
    const float* margin;
    const unsigned* tau_g;      // nullable: per-query orderable admission bound (prefilter)
    int verify;                 // tau_g = min local k-th: prefilter at tau_g + margin and
                                // flag queries whose exact k-th + margin/2 reaches tau_g
    const void* rows;           // exact-scoring row source
    const int64_t* row_map;     // pos -> row index in `rows` (nullable: identity)
    const int64_t* id_map;      // pos -> output id (nullable: row index)
    int64_t id_offset;
    int64_t s_cap;              // survivor capacity per query
    uint32_t* s_pos;            // [nq][s_cap]
    int32_t* s_count = nullptr; // [nq] survivors (split phase B; nullable: one kernel)
    uint64_t* s_key;            // [nq][s_cap]
    int64_t* s_id;              // [nq][s_cap]
    int64_t* out_ids;           // [nq][k] (nullable)
    double* out_dist;           // [nq][k] (nullable)
    int32_t* out_ids32;         // [nq][k] (nullable; IVF probes)
    int32_t* out_count;         // [nq] (nullable)
    unsigned long long* n_survivors;
    LeafPlan plan;              // filled by launch_rerank
    // distributed protocol (vs_enn_search_begin/finish), all nullable:
    const float* ext_thr = nullptr;   // [nq] global upper bound on the k-th approximate key
    double* out_bound = nullptr;      // [nq] deferred verification: dropped candidates have an
                                      //      exact key (distance, or -score) above this bound
    float* out_kth = nullptr;         // [nq][k] write this shard's k smallest approximate keys
                                      //      (ascending, +inf padded) and stop
    // one-warp-per-query kernel for small k (k_rerank_warp): queries beyond its
    // capacity are listed in fb_list / fb_count ([nq] + 1, caller-allocated,
    // nullable: CTA kernel only) and re-ranked by the CTA kernel over q_list
    int32_t* fb_list = nullptr;
    int32_t* fb_count = nullptr;
    const int32_t* q_list = nullptr;
    const int32_t* q_count = nullptr;
    int band_ready = 0;         // the single buffer per query already holds exactly the
                                //      margin band of its k-th key: every entry survives
    int prefetch_iters = 4;     // scorer iterations of L2 prefetch ahead (VS_RR_PD)
    int ubytes;                 // filled by launch_rerank: shared-memory union size
    int reg_path;               // filled by launch_rerank: register-resident scorer
};
template <typename T>
cudaError_t launch_rerank(const RerankParams& p, cudaStream_t s);

// dense keys [nq][ncols] -> one margin-band buffer per query (cb.n_sub = 1):
// every column with key <= k-th key + margin (overflow flagged past cb.C)
cudaError_t launch_dense_select(const float* keys, int64_t nq, int64_t ncols, int k, const float* margin,
                                const CandBuf& cb, cudaStream_t s);
// the same band from per-32-column key minima (MODE 3 `mins`): reads only
// the chunks that can hold band keys; coarse_select_ok() says when it applies
bool coarse_select_ok(int64_t ncols, int k);
cudaError_t launch_coarse_select(const float* keys, const float* mins, int64_t nq, int64_t ncols, int k,
                                 const float* margin, const CandBuf& cb, cudaStream_t s);
// rewrite each buffer entry's key as the fp32 squared distance (q - x)^2
// (squared-L2 bands only; margin eps_simt applies)
cudaError_t launch_refine32(const CandBuf& cb, int64_t nq, const float* Q, int d, const float* X, cudaStream_t s);

// [G][nq][k] sorted shard key lists -> [nq] k-th smallest of their union
cudaError_t launch_union_kth(const float* keys, int G, int64_t nq, int k, float* out, cudaStream_t s);

// ---- cross-shard merge ---------------------------------------------------------------------
struct MergeParams {
    int nparts;
    int64_t nq;
    int k_in;
    const int64_t* ids;      // [nparts][nq][k_in]
    const double* dist;
    const int32_t* counts;   // [nparts][nq]
    int k;
    int ip;
    uint64_t* s_key;         // [nq][nparts*k_in]
    int64_t* s_id;
    int64_t* out_ids;
    double* out_dist;
    int32_t* out_count;
};
cudaError_t launch_merge(const MergeParams& p, cudaStream_t s);

// ---- IVF structure helpers ----------------------------------------------------------------
template <typename T>
cudaError_t launch_gather_rows(const T* src, const int64_t* ids, int64_t n, int d, T* dst,
                               cudaStream_t s);
cudaError_t launch_gather_rows_host(const void* src, const int64_t* ids, int64_t n, int row_bytes, void* dst,
                                    int blocks, cudaStream_t s);
cudaError_t launch_visited_count(const int32_t* probes, int64_t nq, int nprobe, const int64_t* list_off, int nlist,
                                 const uint8_t* list_owned, const uint32_t* pbits, int32_t* sel_scratch,
                                 unsigned long long* visited, cudaStream_t s);

// ---- relational filters -> packed bitmaps (vs_predicate.cu) ------------------------------
// vtype: 0 int32, 1 int64, 2 float32, 3 float64; op: 0 <, 1 <=, 2 ==, 3 !=, 4 >=, 5 >
// ---- after the search (vs_output.cu): post-filter, flat output, row gather ----
struct PostfilterArgs {
    const int64_t* ids;        // [nq][kp] data rows
    const double* dist;        // [nq][kp]
    const int32_t* counts;     // [nq] valid entries per query (nullable: kp)
    int64_t nq;
    int kp;
    const uint32_t* bitmap;    // keep: bit data_row set (nullable)
    const uint8_t* keep_pos;   // keep: per result slot (nullable)
    const int64_t* data_key;   // keep: data_key[data_row] <key_op> query_key[q] (nullable)
    const int64_t* query_key;
    int key_op;
    int64_t n_data;            // bitmap bits / data_key length (row-id bound)
    int k;
    int64_t* out_ids;          // [nq][k]
    double* out_dist;
    int32_t* out_rank;         // original rank (slot in k') of each kept row
    int32_t* out_count;        // [nq]
    int* bad;                  // set when a data row id is out of range
};
struct FlattenArgs {
    const int64_t* ids;
    const double* dist;
    const int32_t* in_rank;    // nullable: the slot index
    const int32_t* counts;     // nullable: kp
    int64_t nq;
    int kp;
    int64_t query_offset;
    int64_t* query_row;        // [R] outputs (each nullable)
    int64_t* data_row;
    double* distance;
    int64_t* rank;
};
cudaError_t launch_postfilter(const PostfilterArgs& a, cudaStream_t s);
size_t flatten_temp_bytes(int64_t nq);
cudaError_t launch_flatten(const FlattenArgs& a, int64_t* c64, int64_t* off, void* tmp, size_t tmp_bytes,
                           cudaStream_t s);
cudaError_t launch_gather(const void* src, int64_t n_src, int64_t row_bytes, const int64_t* idx, int64_t n,
                          void* dst, int* bad, cudaStream_t s);

cudaError_t launch_bitmap_compare(const void* values, int vtype, int64_t n, int op, double value,
                                  const uint32_t* valid, uint32_t* out, cudaStream_t s);
size_t bitmap_isin_temp_bytes(int64_t nset);
cudaError_t launch_bitmap_isin(const int64_t* keys, int64_t n, const uint32_t* valid, const int64_t* set,
                               int64_t nset, int64_t* sorted_set, void* tmp, size_t tmp_bytes, uint32_t* out,
                               cudaStream_t s);
// op: 0 and, 1 or, 2 and-not
cudaError_t launch_bitmap_combine(const uint32_t* a, const uint32_t* b, int64_t nwords, int op, uint32_t* out,
                                  cudaStream_t s);

}  // namespace vs
