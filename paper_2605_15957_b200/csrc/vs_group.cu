// Single-process multi-GPU searches: one vs_ctx per
// device of a group, driven from one host thread each, and the exchange step
// (the per-shard [Q, k] results -> the global top-k) over NCCL.
//
// The reference drives the operator from one interpreter (executor.py:109-181),
// so a drop-in must be able to use the box's GPUs without torchrun. The group
// holds one context per device and, when the devices are distinct, an NCCL
// communicator clique (ncclCommInitAll). A search runs every member's
// shard search concurrently (its rows / its lists), then ncclAllGather
// inside one ncclGroupStart/End moves the [Q, k] (id, distance, count)
// triples to every member over NVLink, and member 0 merges them with the
// tie-rule merge kernel. A group that repeats a device (tests on one GPU) or
// cannot load NCCL gathers with peer copies instead; results are identical.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): the process's own
// copy (e.g. the one torch loaded) is reused, and the library has no link-time
// NCCL dependency. NCCL failures return VS_ERR_NCCL with ncclGetErrorString.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vs_b200.h"
#include "vs_internal.h"
#include "vs_kernels.cuh"
#include "vs_wide.cuh"

using namespace vs_internal;

namespace {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.commInitAll = (decltype(a.commInitAll))dlsym(h, "ncclCommInitAll");
        a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
        a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
        a.groupStart = (decltype(a.groupStart))dlsym(h, "ncclGroupStart");
        a.groupEnd = (decltype(a.groupEnd))dlsym(h, "ncclGroupEnd");
        a.errStr = (decltype(a.errStr))dlsym(h, "ncclGetErrorString");
        a.ok = a.commInitAll && a.commDestroy && a.allGather && a.groupStart && a.groupEnd && a.errStr;
        return a;
    }();
    return api;
}

int nccl_err(ncclResult_t r, const char* what) {
    return set_err(VS_ERR_NCCL, "%s: %s", what, nccl().errStr ? nccl().errStr(r) : "NCCL error");
}
#define NCK(call)                                                    \
    do {                                                             \
        ncclResult_t _r = (call);                                    \
        if (_r != ncclSuccess) return nccl_err(_r, #call);           \
    } while (0)

template <typename T>
struct DevBuf {
    T* p = nullptr;
    int dev = 0;
    ~DevBuf() {
        if (p) {
            DevGuard g(dev);
            cudaFree(p);
        }
    }
    int alloc(int d, size_t n) {
        dev = d;
        DevGuard g(d);
        CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
        return VS_OK;
    }
};

}  // namespace

struct vs_group {
    std::vector<int> devs;
    std::vector<vs_ctx*> ctx;
    std::vector<ncclComm_t> comms;   // empty: peer-copy exchange
};

namespace {

// every member's shard search into device buffers [nq][k] on that member, then
// the exchange + merge on member 0
using MemberSearch = int (*)(vs_group*, int r, void* arg, int64_t* ids, double* dist, int32_t* cnt, int64_t* vis);

int group_run(vs_group* g, int64_t nq, int32_t k, int32_t metric, MemberSearch fn, void* arg, int64_t* out_ids,
              double* out_dist, int32_t* out_count, int64_t* out_visited) {
    const int G = (int)g->ctx.size();
    const size_t nk = (size_t)nq * k;
    std::vector<DevBuf<int64_t>> ids(G), gids(G);
    std::vector<DevBuf<double>> dist(G), gdist(G);
    std::vector<DevBuf<int32_t>> cnt(G), gcnt(G);
    std::vector<int64_t> vis(G, 0);
    std::vector<int> st(G, VS_OK);
    std::vector<std::string> msg(G);
    const bool all_gather = !g->comms.empty();
    for (int r = 0; r < G; ++r) {
        CKS(ids[r].alloc(g->devs[r], nk));
        CKS(dist[r].alloc(g->devs[r], nk));
        CKS(cnt[r].alloc(g->devs[r], (size_t)nq));
        if (all_gather || r == 0) {
            CKS(gids[r].alloc(g->devs[r], nk * G));
            CKS(gdist[r].alloc(g->devs[r], nk * G));
            CKS(gcnt[r].alloc(g->devs[r], (size_t)nq * G));
        }
    }
    {
        // one host thread per member: the shard searches are synchronous
        std::vector<std::thread> th;
        for (int r = 0; r < G; ++r)
            th.emplace_back([&, r] {
                st[r] = fn(g, r, arg, ids[r].p, dist[r].p, cnt[r].p, &vis[r]);
                if (st[r] != VS_OK) msg[r] = vs_last_error();
            });
        for (auto& t : th) t.join();
    }
    for (int r = 0; r < G; ++r)
        if (st[r] != VS_OK) return set_err(st[r], "member %d (device %d): %s", r, g->devs[r], msg[r].c_str());
    if (all_gather) {
        NCK(nccl().groupStart());
        for (int r = 0; r < G; ++r) {
            cudaStream_t s = g->ctx[r]->stream;
            NCK(nccl().allGather(ids[r].p, gids[r].p, nk, ncclInt64, g->comms[r], s));
            NCK(nccl().allGather(dist[r].p, gdist[r].p, nk, ncclFloat64, g->comms[r], s));
            NCK(nccl().allGather(cnt[r].p, gcnt[r].p, (size_t)nq, ncclInt32, g->comms[r], s));
        }
        NCK(nccl().groupEnd());
        for (int r = 0; r < G; ++r) {
            DevGuard dg(g->devs[r]);
            CK(cudaStreamSynchronize(g->ctx[r]->stream));
        }
    } else {
        DevGuard dg(g->devs[0]);
        cudaStream_t s = g->ctx[0]->stream;
        for (int r = 0; r < G; ++r) {
            CK(cudaMemcpyPeerAsync(gids[0].p + r * nk, g->devs[0], ids[r].p, g->devs[r], nk * 8, s));
            CK(cudaMemcpyPeerAsync(gdist[0].p + r * nk, g->devs[0], dist[r].p, g->devs[r], nk * 8, s));
            CK(cudaMemcpyPeerAsync(gcnt[0].p + r * (size_t)nq, g->devs[0], cnt[r].p, g->devs[r], (size_t)nq * 4, s));
        }
        CK(cudaStreamSynchronize(s));
    }
    // member 0 merges (vs_topk_merge stages host outputs itself)
    CKS(vs_topk_merge(g->ctx[0], G, nq, k, gids[0].p, gdist[0].p, gcnt[0].p, k, metric, out_ids, out_dist,
                      out_count));
    if (out_visited) {
        int64_t t = 0;
        for (int64_t v : vis) t += v;
        *out_visited = t;
    }
    return VS_OK;
}

struct EnnArg {
    vs_column* const* shards;
    const int64_t* row_lo;
    const float* q;
    int64_t nq;
    int32_t d;
    const uint32_t* bitmap;   // host words over the global rows
    int32_t k, metric;
    std::atomic<int> empty{0};
};

int enn_member(vs_group* g, int r, void* argp, int64_t* ids, double* dist, int32_t* cnt, int64_t* vis) {
    EnnArg& a = *static_cast<EnnArg*>(argp);
    const vs_column* c = a.shards[r];
    const uint32_t* bm = a.bitmap ? a.bitmap + a.row_lo[r] / 32 : nullptr;
    int st = vs_enn_search(g->ctx[r], c, a.q, a.nq, a.d, bm, bm ? c->n : 0, a.k, a.metric, a.row_lo[r], ids, dist,
                           cnt, vis);
    if (st == VS_ERR_EMPTY_INPUT) {   // this shard selects nothing: it contributes no rows
        a.empty.fetch_add(1);
        DevGuard dg(g->devs[r]);
        CK(cudaMemset(cnt, 0, (size_t)a.nq * 4));
        *vis = 0;
        return VS_OK;
    }
    if (st == VS_OK) {
        DevGuard dg(g->devs[r]);
        CK(cudaStreamSynchronize(g->ctx[r]->stream));
    }
    return st;
}

struct IvfArg {
    vs_ivf* const* parts;
    const float* q;
    int64_t nq;
    const uint32_t* bitmap;
    int64_t nbits;
    int32_t nprobe, k;
};

int ivf_member(vs_group* g, int r, void* argp, int64_t* ids, double* dist, int32_t* cnt, int64_t* vis) {
    const IvfArg& a = *static_cast<const IvfArg*>(argp);
    int st = vs_ivf_search(g->ctx[r], a.parts[r], a.q, a.nq, a.bitmap, a.nbits, a.nprobe, a.k, ids, dist, cnt,
                           nullptr, vis);
    if (st == VS_OK) {
        DevGuard dg(g->devs[r]);
        CK(cudaStreamSynchronize(g->ctx[r]->stream));
    }
    return st;
}

}  // namespace

extern "C" {

int vs_group_create(int32_t ndev, const int32_t* devices, vs_group** out) {
    if (ndev < 1 || !devices || !out) return set_err(VS_ERR_PARAMETER, "bad device group");
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    for (int i = 0; i < ndev; ++i)
        if (devices[i] < 0 || devices[i] >= count) return set_err(VS_ERR_PARAMETER, "no device %d", devices[i]);
    vs_group* g = new vs_group();
    g->devs.assign(devices, devices + ndev);
    for (int i = 0; i < ndev; ++i) {
        vs_ctx* c = nullptr;
        int st = vs_ctx_create(devices[i], &c);
        if (st != VS_OK) {
            vs_group_destroy(g);
            return st;
        }
        g->ctx.push_back(c);
    }
    std::vector<int> sorted(g->devs);
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::unique(sorted.begin(), sorted.end()) == sorted.end();
    if (distinct && nccl().ok && !getenv("VS_GROUP_NO_NCCL")) {
        g->comms.resize(ndev);
        ncclResult_t r = nccl().commInitAll(g->comms.data(), ndev, g->devs.data());
        if (r != ncclSuccess) {
            g->comms.clear();
            vs_group_destroy(g);
            return nccl_err(r, "ncclCommInitAll");
        }
    } else {
        // peer access for the copy exchange (same device: nothing to enable)
        for (int i = 0; i < ndev; ++i)
            for (int j = 0; j < ndev; ++j) {
                if (g->devs[i] == g->devs[j]) continue;
                int can = 0;
                cudaDeviceCanAccessPeer(&can, g->devs[i], g->devs[j]);
                if (can) {
                    DevGuard dg(g->devs[i]);
                    cudaDeviceEnablePeerAccess(g->devs[j], 0);
                    cudaGetLastError();   // already enabled
                }
            }
    }
    *out = g;
    return VS_OK;
}

int vs_group_destroy(vs_group* g) {
    if (!g) return VS_OK;
    for (ncclComm_t c : g->comms)
        if (c) nccl().commDestroy(c);
    for (vs_ctx* c : g->ctx) vs_ctx_destroy(c);
    delete g;
    return VS_OK;
}

int vs_group_info(const vs_group* g, int32_t* ndev, int32_t* uses_nccl) {
    if (!g) return set_err(VS_ERR_PARAMETER, "null group");
    if (ndev) *ndev = (int32_t)g->ctx.size();
    if (uses_nccl) *uses_nccl = g->comms.empty() ? 0 : 1;
    return VS_OK;
}

vs_ctx* vs_group_ctx(vs_group* g, int32_t member) {
    if (!g || member < 0 || member >= (int)g->ctx.size()) return nullptr;
    return g->ctx[member];
}

int vs_group_enn_search(vs_group* g, vs_column* const* shards, const int64_t* row_lo, const float* queries,
                        int64_t nq, int32_t d, const uint32_t* bitmap, int64_t nbits, int32_t k, int32_t metric,
                        int64_t* out_ids, double* out_dist, int32_t* out_count, int64_t* out_visited) {
    if (!g || !shards || !row_lo) return set_err(VS_ERR_PARAMETER, "null argument");
    const int G = (int)g->ctx.size();
    int64_t total = 0;
    for (int r = 0; r < G; ++r) {
        if (!shards[r]) return set_err(VS_ERR_PARAMETER, "null shard %d", r);
        if (bitmap && row_lo[r] % 32) return set_err(VS_ERR_PARAMETER, "shard %d starts at row %lld: not a multiple of 32", r, (long long)row_lo[r]);
        if (r > 0 && row_lo[r] != row_lo[r - 1] + shards[r - 1]->n)
            return set_err(VS_ERR_SHAPE, "shards are not contiguous row ranges");
        total += shards[r]->n;
    }
    if (bitmap && nbits != row_lo[0] + total) return set_err(VS_ERR_SHAPE, "bitmap covers %lld rows, shards %lld", (long long)nbits, (long long)(row_lo[0] + total));
    if (bitmap && is_device_ptr(bitmap)) return set_err(VS_ERR_PARAMETER, "group searches take a host bitmap");
    if (queries && is_device_ptr(queries)) return set_err(VS_ERR_PARAMETER, "group searches take host queries");
    if (nq == 0) return VS_OK;
    EnnArg a{shards, row_lo, queries, nq, d, bitmap, k, metric};
    int64_t vis = 0;
    CKS(group_run(g, nq, k, metric, enn_member, &a, out_ids, out_dist, out_count, &vis));
    if (a.empty.load() == G) return set_err(VS_ERR_EMPTY_INPUT, "exhaustive search over empty data side");
    if (out_visited) *out_visited = vis;
    if (bitmap == nullptr && out_visited) *out_visited = nq * total;
    return VS_OK;
}

int vs_group_ivf_search(vs_group* g, vs_ivf* const* parts, const float* queries, int64_t nq,
                        const uint32_t* bitmap, int64_t nbits, int32_t nprobe, int32_t k, int64_t* out_ids,
                        double* out_dist, int32_t* out_count, int64_t* out_visited) {
    if (!g || !parts) return set_err(VS_ERR_PARAMETER, "null argument");
    const int G = (int)g->ctx.size();
    for (int r = 0; r < G; ++r)
        if (!parts[r]) return set_err(VS_ERR_PARAMETER, "null index part %d", r);
    if ((bitmap && is_device_ptr(bitmap)) || (queries && is_device_ptr(queries)))
        return set_err(VS_ERR_PARAMETER, "group searches take host queries and bitmaps");
    if (nq == 0) return VS_OK;
    IvfArg a{parts, queries, nq, bitmap, nbits, nprobe, k};
    return group_run(g, nq, k, parts[0]->metric, ivf_member, &a, out_ids, out_dist, out_count, out_visited);
}

}  // extern "C"
