/*
 * vs_b200.h — C ABI of the B200-native filtered vector-search operator.
 *
 * Drop-in boundary for the reference `sqlvs` vector-search path
 * (/root/reference/pkg/src/sqlvs). The reference has no FFI: its boundary is
 * the Python API below, which `paper_2605_15957_b200` keeps verbatim and
 * implements over this ABI through ctypes (INTEGRATION.md shows the binding):
 *
 *   enn_search(queries, data, params, metric)         vecindex.py:109-132
 *   FlatIndex.build / .search                         vecindex.py:138-162
 *   IvfIndex.build / .search / .as_layout             vecindex.py:168-270
 *   save_index / load_index (SVIX)                    vecindex.py:495-579
 *   vector_search_operator(...)                       vecsearch.py:64-120
 *
 * Conventions
 *   - Plain pointers and sizes only. Every data pointer may be HOST or DEVICE
 *     memory (detected with cudaPointerGetAttributes); host pointers are
 *     staged through the context stream.
 *   - Calls are synchronous with respect to the caller (the stream is
 *     synchronised before returning). A context is not re-entrant.
 *   - Results follow NeighborTable (vecindex.py:70-88): per query, rows
 *     ordered by the tie rule (distance ascending then row ascending; inner
 *     product: score descending then row ascending), out_count[q] =
 *     min(k', candidates_q), padding ids = -1 and distances = NaN. Distances
 *     are float64 and are computed with the reference's exact float64
 *     arithmetic and summation order (bit-identical to numpy's
 *     np.sum(diff*diff, axis=-1) of distances.py:54-58).
 *   - Row filters are packed uint32 bitmaps, LSB-first: bit i of word w
 *     selects base row 32*w + i (nbits = base row count).
 *   - Status codes mirror the reference exceptions (errors.py:4-54).
 */
#ifndef VS_B200_H
#define VS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum vs_status {
    VS_OK = 0,
    VS_ERR_SHAPE = 1,        /* ShapeError: dim mismatch                      */
    VS_ERR_EMPTY_INPUT = 2,  /* EmptyInputError: exhaustive search, no rows   */
    VS_ERR_PARAMETER = 3,    /* ParameterError: bad k / nprobe / nlist / ...  */
    VS_ERR_CAP_EXCEEDED = 4, /* CapExceededError (two-phase search, k' > cap) */
    VS_ERR_PLACEMENT = 5,    /* PlacementError: device memory exhausted       */
    VS_ERR_CUDA = 6,         /* CUDA runtime / launch failure                 */
    VS_ERR_INTERNAL = 7,
    VS_ERR_NCCL = 8          /* NCCL failure in a device-group exchange       */
};

enum vs_metric { VS_METRIC_SQUARED_L2 = 0, VS_METRIC_INNER_PRODUCT = 1 };
enum vs_dtype { VS_DTYPE_F32 = 0, VS_DTYPE_BF16 = 1 };

/* context options (vs_ctx_set_option) */
enum vs_option {
    VS_OPT_ENN_KERNEL = 1,   /* 0 auto, 1 SIMT fp32, 2 tcgen05 bf16 GEMM          */
    VS_OPT_IVF_KERNEL = 2,   /* 0 auto, 1 query-major scan, 2 list-major scan      */
    VS_OPT_CAND_SLACK = 3,   /* extra candidate-buffer capacity (power-of-2 sized) */
    VS_OPT_FORCE_RETRY = 4,  /* test hook: treat every query as overflowed once    */
    VS_OPT_TIMING = 5,       /* 1: record CUDA events around every kernel class    */
    VS_OPT_STREAM_CHUNK = 6, /* host-resident search: selected rows per chunk (0 auto) */
    VS_OPT_IVF_CHUNK_ROWS = 7, /* tensor-core IVF scan: rows per list chunk (0: 131072) */
    VS_OPT_COARSE = 8        /* IVF coarse quantizer: 0 auto, 1 candidate buffers, 2 dense keys */
};

/* kernel classes reported by vs_ctx_kernel_times (CUDA-event durations on the
 * launching stream, accumulated while VS_OPT_TIMING is on) */
enum vs_kernel_class {
    VS_K_SELECT = 0,      /* bitmap -> selection vector / permuted bitmap       */
    VS_K_ENN_SCAN = 1,    /* phase A of the exhaustive search                   */
    VS_K_RERANK = 2,      /* phase B (exact float64 re-rank + top-k)            */
    VS_K_COARSE = 3,      /* IVF coarse quantizer, phase A over the centroids   */
    VS_K_IVF_SCAN = 4,    /* IVF list scan (phase A)                            */
    VS_K_IVF_RERANK = 5,  /* IVF phase B                                        */
    VS_K_MERGE = 6,       /* cross-shard merge                                  */
    VS_K_STAGE = 7,       /* tensor-core operand staging (bf16 compaction)      */
    VS_K_COARSE_RERANK = 8, /* IVF coarse quantizer, exact phase B (probes)     */
    VS_K_N = 9
};

/* counters (vs_ctx_stats) */
enum vs_stat {
    VS_STAT_LAUNCHES = 0,        /* kernels launched by the library             */
    VS_STAT_OVERFLOW_QUERIES = 1,/* queries re-run with a larger buffer         */
    VS_STAT_SURVIVORS = 2,       /* candidates re-ranked in float64 (last call) */
    VS_STAT_LAST_ENN_KERNEL = 3, /* which phase-A kernel ran last               */
    VS_STAT_NEAR_TIES = 4,       /* k-means / assign rows re-checked exactly    */
    VS_STAT_N = 8
};

typedef struct vs_ctx vs_ctx;
typedef struct vs_column vs_column;
typedef struct vs_ivf vs_ivf;

/* thread-local message for the last non-OK status */
const char* vs_last_error(void);
/* top-k of the candidate-buffer kernels (= the reference's default
 * HardwareProfile.gpu_topk_cap, placement.py:56). Searches accept any k'
 * >= 1: above this value they run the device-wide large-k' path
 * (vs_wide.cu). VS_ERR_CAP_EXCEEDED remains only for the two-phase
 * protocol (k' <= cap); the operator's placement cap (vecsearch.py:86-87)
 * is a host-side check. */
int32_t vs_topk_cap(void);
int32_t vs_version(void);

/* ---- context: one per GPU (one process per GPU) -------------------------- */
int vs_ctx_create(int32_t device, vs_ctx** out);
int vs_ctx_destroy(vs_ctx* ctx);
/* run on a caller stream (cudaStream_t); NULL restores the context's own
 * (non-blocking) stream, so the legacy default stream must be passed as
 * cudaStreamLegacy ((void*)0x1) to order the library after work queued there */
int vs_ctx_set_stream(vs_ctx* ctx, void* stream);
int vs_ctx_synchronize(vs_ctx* ctx);
int vs_ctx_set_option(vs_ctx* ctx, int32_t key, int64_t value);
int vs_ctx_stats(vs_ctx* ctx, int64_t* out, int32_t n);
/* accumulated per-class kernel time (ns) and launch counts; reset=1 zeroes */
int vs_ctx_kernel_times(vs_ctx* ctx, int64_t* ns, int64_t* launches, int32_t n, int32_t reset);

/* ---- embedding columns (EmbeddingColumn, table.py:91-141) ----------------- */
/* copy n x d rows (host or device) into library-owned device memory */
int vs_column_create(vs_ctx* ctx, const void* src, int64_t n, int32_t d,
                     int32_t dtype, vs_column** out);
/* borrow caller-owned device rows (must outlive the column) */
int vs_column_wrap(vs_ctx* ctx, void* dev_ptr, int64_t n, int32_t d,
                   int32_t dtype, vs_column** out);
/* Column over caller-owned HOST memory (pinned, or registered here with
 * cudaHostRegister): searches stream only the rows the bitmap selects over
 * PCIe (zero-copy gathers on a few SMs, overlapped with the tensor-core scan of
 * the previous chunk) and merge the per-chunk top-k. */
int vs_column_wrap_host(vs_ctx* ctx, void* host_ptr, int64_t n, int32_t d,
                        int32_t dtype, vs_column** out);
int vs_column_free(vs_column* col);
/* the rows of a borrowed column (vs_column_wrap / _wrap_host) changed: drop
 * the cached row norms and max norm (recomputed by the next search; stale
 * norms would make the approximate keys and margins wrong) */
int vs_column_invalidate(vs_column* col);
int vs_column_info(const vs_column* col, int64_t* n, int32_t* d, int32_t* dtype);

/* ---- exhaustive search (enn_search, vecindex.py:109-132) -----------------
 * Filtered: bitmap over the column's rows (nullable = all rows); the result
 * equals the reference composition rows = flatnonzero(mask);
 * enn_search(Q, base[rows]); ids = rows[pos] (plans.py:564-569).
 * out_ids/out_dist: [nq, k] row-major; ids are base row + id_offset (global
 * row ids when the column is one shard of a larger collection).
 * out_visited = nq * selected rows (vecindex.py:132). */
int vs_enn_search(vs_ctx* ctx, const vs_column* data,
                  const float* queries, int64_t nq, int32_t d,
                  const uint32_t* bitmap, int64_t nbits,
                  int32_t k, int32_t metric, int64_t id_offset,
                  int64_t* out_ids, double* out_dist, int32_t* out_count,
                  int64_t* out_visited);

/* ---- two-phase exact search of one row shard (multi-GPU) -----
 * begin: selection + phase A (tensor cores) on this shard, and out_keys
 * [nq][k] = upper bounds on the exact keys of the shard's k smallest
 * approximate keys (approx + this shard's margin/2, rounded up; ascending,
 * +inf padded). The caller all-gathers the keys of every shard and takes
 * T = the k-th smallest of their union (vs_union_kth): an upper bound on the
 * global k-th exact key, valid even when shards have different margins
 * (different max norms or phase-A kernels).
 * finish(T): phase B re-ranks only candidates with key <= T + margin/2 (its
 * own margin), so the
 * exact float64 work is split across the shards instead of repeated on each;
 * returns the shard's rows (possibly fewer than k) and out_bound[q]: every
 * candidate this shard dropped in phase A has exact key (distance; -score
 * for inner product) above it. After the all-gather + merge, queries whose
 * merged k-th key is not below the MIN over shards of out_bound are re-run
 * with vs_enn_search (distributed.py). */
int vs_enn_search_begin(vs_ctx* ctx, const vs_column* data, const float* queries, int64_t nq,
                        int32_t d, const uint32_t* bitmap, int64_t nbits, int32_t k,
                        int32_t metric, float* out_keys, int64_t* out_visited);
/* [nparts][nq][k] sorted key lists -> out[nq] = k-th smallest of their union */
int vs_union_kth(vs_ctx* ctx, int32_t nparts, int64_t nq, int32_t k, const float* keys, float* out);
int vs_enn_search_finish(vs_ctx* ctx, const float* thresholds, int64_t id_offset,
                         int64_t* out_ids, double* out_dist, int32_t* out_count,
                         double* out_bound);

/* ---- cross-shard merge (multi-GPU exchange step) --------------
 * ids/dist: [nparts, nq, k_in], counts: [nparts, nq]; writes the global
 * top-k under the tie rule. Inputs are per-shard outputs of the searches. */
int vs_topk_merge(vs_ctx* ctx, int32_t nparts, int64_t nq, int32_t k_in,
                  const int64_t* ids, const double* dist, const int32_t* counts,
                  int32_t k, int32_t metric,
                  int64_t* out_ids, double* out_dist, int32_t* out_count);

/* ---- IVF (IvfIndex, vecindex.py:168-270) ----------------------------------
 * Owning layout: list_payload = list-major rows (the SVIX owning payload,
 * vecindex.py:526-530), n_total = sum(list_sizes) rows of dtype.
 * Non-owning layout: list_payload = NULL and base != NULL; the lists are
 * gathered from the base column into the device list-contiguous layout.
 * list_owned (nullable): per-list 0/1, lists not owned by this shard are
 * probed (centroids are replicated) but not scanned (list sharding, §8e).
 * list_ids are base row ids (ascending within each list). */
int vs_ivf_create(vs_ctx* ctx, const float* centroids, int32_t nlist, int32_t d,
                  const int64_t* list_sizes, const int64_t* list_ids,
                  const void* list_payload, int32_t dtype, int32_t metric,
                  const vs_column* base, const uint8_t* list_owned,
                  vs_ivf** out);
/* GPU k-means build with the reference's semantics (vecindex.py:273-318):
 * init_rows = the nlist ascending initial rows (the reference draws them with
 * np.sort(default_rng(seed).choice(n, nlist, replace=False)); the Python
 * shim passes exactly those), nullable -> a seeded library sample; <= max_iters
 * Lloyd iterations or max centroid shift < 1e-4, first-min assignment, empty
 * lists reseeded to the farthest member of the largest list, float64 means,
 * final reassignment; lists hold ascending row ids (owning layout). */
int vs_ivf_build(vs_ctx* ctx, const vs_column* data, int32_t nlist, const int64_t* init_rows,
                 uint64_t seed, int32_t metric, int32_t max_iters, vs_ivf** out);
/* Borrow a caller-owned DEVICE list-contiguous payload (must outlive the
 * index): avoids a second copy of collections that fill most of HBM. */
int vs_ivf_wrap(vs_ctx* ctx, const float* centroids, int32_t nlist, int32_t d,
                const int64_t* list_sizes, const int64_t* list_ids, void* payload_dev,
                int32_t dtype, int32_t metric, vs_ivf** out);
/* Nearest list of every row of a column (squared L2 to the centroids, the
 * build's assignment step; reference vecindex.py:303-304): for indexes
 * trained on a sample. out_lists: int32 [n], host or device. */
int vs_ivf_assign(vs_ctx* ctx, const vs_ivf* ivf, const vs_column* data, int32_t* out_lists);
int vs_ivf_info(const vs_ivf* ivf, int32_t* nlist, int32_t* d, int64_t* n_total,
                int32_t* metric, int32_t* dtype);
/* host copies of the structure (any pointer may be NULL) */
int vs_ivf_export(vs_ivf* ivf, float* centroids, int64_t* list_sizes,
                  int64_t* list_ids, void* list_payload);
/* bitmap over base rows (nullable); probes computed without the filter;
 * out_probes (nullable): [nq, nprobe] probed list ids in rank order. */
int vs_ivf_search(vs_ctx* ctx, const vs_ivf* ivf, const float* queries, int64_t nq,
                  const uint32_t* bitmap, int64_t nbits, int32_t nprobe, int32_t k,
                  int64_t* out_ids, double* out_dist, int32_t* out_count,
                  int32_t* out_probes, int64_t* out_visited);
/* list sharding: per-list 0/1 ownership mask of this shard
 * (nullable = all lists owned). Probes still use every centroid. */
int vs_ivf_set_owned(vs_ivf* ivf, const uint8_t* list_owned);
/* coarse quantizer only: [nq][nprobe] probed lists (the probes of vs_ivf_search) */
int vs_ivf_probe(vs_ctx* ctx, const vs_ivf* ivf, const float* queries, int64_t nq,
                 int32_t nprobe, int32_t* out_probes);
/* IVF search with given probes (e.g. computed by other ranks for their query
 * slices and all-gathered): skips the coarse quantizer */
int vs_ivf_search_probed(vs_ctx* ctx, const vs_ivf* ivf, const float* queries, int64_t nq,
                         const uint32_t* bitmap, int64_t nbits, int32_t nprobe,
                         const int32_t* probes, int32_t k, int64_t* out_ids, double* out_dist,
                         int32_t* out_count, int64_t* out_visited);
int vs_ivf_free(vs_ivf* ivf);

/* ---- single-process device groups ------------------
 * One interpreter driving several GPUs (the reference's executor runs the
 * operator from one process, executor.py:109-181): a group holds one
 * context per device (vs_group_ctx: create each member's shard column / index
 * part with it) and, for distinct devices, an NCCL clique (ncclCommInitAll;
 * NCCL is dlopen'ed, failures -> VS_ERR_NCCL). A group search runs every
 * member's shard search concurrently (one host thread each), all-gathers the
 * [Q, k] (id, distance, count) triples with ncclAllGather inside one
 * ncclGroupStart/End, and merges them on member 0 (tie rule). A group that
 * repeats a device (or VS_GROUP_NO_NCCL=1) gathers with peer copies; the
 * results are identical either way and equal the one-GPU search.
 *   vs_group_enn_search: shards[i] = rows [row_lo[i], row_lo[i] + n_i) of the
 *     collection, contiguous, row_lo[i] % 32 == 0 when a bitmap is given (the
 *     global host bitmap is sliced by words); ids are global rows.
 *   vs_group_ivf_search: parts[i] = member i's index over the lists it owns
 *     (same centroids everywhere, other lists empty, e.g. LPT-assigned).
 * Queries, bitmaps and outputs are host memory. */
typedef struct vs_group vs_group;
int vs_group_create(int32_t ndev, const int32_t* devices, vs_group** out);
int vs_group_destroy(vs_group* g);
int vs_group_info(const vs_group* g, int32_t* ndev, int32_t* uses_nccl);
vs_ctx* vs_group_ctx(vs_group* g, int32_t member);
int vs_group_enn_search(vs_group* g, vs_column* const* shards, const int64_t* row_lo, const float* queries,
                        int64_t nq, int32_t d, const uint32_t* bitmap, int64_t nbits, int32_t k,
                        int32_t metric, int64_t* out_ids, double* out_dist, int32_t* out_count,
                        int64_t* out_visited);
int vs_group_ivf_search(vs_group* g, vs_ivf* const* parts, const float* queries, int64_t nq,
                        const uint32_t* bitmap, int64_t nbits, int32_t nprobe, int32_t k,
                        int64_t* out_ids, double* out_dist, int32_t* out_count, int64_t* out_visited);

/* ---- native loaders: reference file formats straight into device buffers --
 * (one contiguous copy per file section, not
 * 5 nlist + 1). Every section streams through a pinned double buffer (disk
 * read of chunk i + 1 overlaps the copy of chunk i).
 *   vs_ivf_load: an SVIX IVF file (save_index, vecindex.py:495-579 / load_index
 *     :539-579) -> device IVF; list ids and the owning payload land in their
 *     final device buffers (the payload is adopted, not copied again).
 *     Non-owning files need `base` (rows gathered into the list-contiguous
 *     layout on the device). info (nullable) [6] = kind, metric, layout,
 *     nlist, dim, count. Bad magic / version / kind -> VS_ERR_PARAMETER
 *     (the reference's ParameterError).
 *   vs_emb_info: header of a .emb file (write_embeddings, datagen.py:351-372):
 *     count, dim and the byte offset of the float32 rows.
 *   vs_file_to_device: `bytes` of a file from `offset` into dst (device or
 *     host memory), e.g. the rows of a .emb file into a device column. */
int vs_ivf_load(vs_ctx* ctx, const char* path, const vs_column* base, int64_t* info, vs_ivf** out);
int vs_emb_info(const char* path, int64_t* count, int32_t* dim, int64_t* data_offset);
int vs_file_to_device(vs_ctx* ctx, const char* path, int64_t offset, int64_t bytes, void* dst);

/* ---- relational filters -> packed row bitmaps (the step before the search) -
 * Output words are the row_filter format above. valid_bits (nullable) is the
 * column's validity bitmap: null rows never match.
 *   vs_bitmap_compare: values[i] <op> value, vtype 0 int32 / 1 int64 /
 *     2 float32 / 3 float64, op 0 < / 1 <= / 2 == / 3 != / 4 >= / 5 >, with
 *     numpy's rules (eval_predicate, expr.py:568-576; NaN only satisfies !=);
 *   vs_bitmap_isin: keys[i] occurs in set (semi join, relops.py:88-113);
 *   vs_bitmap_combine: a & b (0), a | b (1), a & ~b (2) over nwords words. */
enum vs_value_type { VS_VALUE_I32 = 0, VS_VALUE_I64 = 1, VS_VALUE_F32 = 2, VS_VALUE_F64 = 3 };
int vs_bitmap_compare(vs_ctx* ctx, const void* values, int32_t vtype, int64_t n, int32_t op,
                      double value, const uint32_t* valid_bits, uint32_t* out_bits);
int vs_bitmap_isin(vs_ctx* ctx, const int64_t* keys, int64_t n, const uint32_t* valid_bits,
                   const int64_t* set, int64_t nset, uint32_t* out_bits);
int vs_bitmap_combine(vs_ctx* ctx, const uint32_t* a, const uint32_t* b, int64_t nwords,
                      int32_t op, uint32_t* out);

/* ---- the step after the search ------------------------------
 * All on the padded result layout the searches write ([nq][k_prime] ids and
 * float64 distances, counts[nq] valid entries; counts may be NULL = k_prime).
 *
 * vs_postfilter replaces oversample_postfilter (vecsearch.py:155-202): per
 * query, the first k results in rank order that satisfy every given keep
 * condition (each nullable, ANDed):
 *   keep_bits  packed bitmap over the n_data data rows (data-side predicates,
 *              semi joins: vs_bitmap_compare / vs_bitmap_isin);
 *   keep_pos   one byte per result slot [nq][k_prime] (any predicate over the
 *              joined output);
 *   data_key[data_row] <key_op> query_key[query] (cross-side comparison, e.g.
 *              Q11's "im_imagekey_d != im_imagekey", plans.py:537; key_op as
 *              vs_bitmap_compare).
 * Writes out_ids/out_dist/out_rank [nq][k] (out_rank = the kept row's slot in
 * k_prime, i.e. its vs_rank) and out_count[nq]; shortfall = k - out_count.
 * A data row id outside [0, n_data) with keep_bits or data_key given is
 * VS_ERR_PARAMETER.
 *
 * vs_results_flatten replaces the NeighborTable assembly (vecindex.py:95-106):
 * the flat arrays sorted by (query, rank), query_row = query + query_offset,
 * rank = rank[slot] (NULL: the slot). Outputs hold nq * k_prime entries;
 * *n_out = the number written.
 *
 * vs_gather_rows is the column gather of build_vs_output (vecsearch.py:123-152):
 * dst[i] = src[idx[i]] for rows of row_bytes bytes (any fixed-width column,
 * embeddings included); an index outside [0, n_src) is VS_ERR_PARAMETER. */
int vs_postfilter(vs_ctx* ctx, const int64_t* ids, const double* dist, const int32_t* counts,
                  int64_t nq, int32_t k_prime, const uint32_t* keep_bits, const uint8_t* keep_pos,
                  const int64_t* data_key, const int64_t* query_key, int32_t key_op, int64_t n_data,
                  int32_t k, int64_t* out_ids, double* out_dist, int32_t* out_rank,
                  int32_t* out_count);
int vs_results_flatten(vs_ctx* ctx, const int64_t* ids, const double* dist, const int32_t* rank,
                       const int32_t* counts, int64_t nq, int32_t k_prime, int64_t query_offset,
                       int64_t* query_row, int64_t* data_row, double* distance, int64_t* out_rank,
                       int64_t* n_out);
int vs_gather_rows(vs_ctx* ctx, const void* src, int64_t n_src, int64_t row_bytes, const int64_t* idx,
                   int64_t n, void* dst);

#ifdef __cplusplus
}
#endif
#endif /* VS_B200_H */
