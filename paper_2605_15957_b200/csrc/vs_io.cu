// Native loaders: the reference's on-disk formats straight into device
// buffers.
//
// The reference loads an SVIX index into per-list numpy arrays and a
// placement layer later ships 5·nlist + 1 separate arrays to the device
// (PAPER.md:562-590); here every file section is read once through a pinned
// staging ring (two 64 MiB buffers: the disk read of chunk i + 1 overlaps the
// host->device copy of chunk i) and lands in its final device buffer, one
// contiguous copy per section:
//   - SVIX IVF (vecindex.py:495-579): centroids and list sizes to the host
//     (they are small and the list offsets are needed there), list ids and the
//     list-contiguous payload streamed to the device and adopted by the IVF
//     structure (no second device copy of the payload);
//   - .emb (datagen.py:351-372): header parsed here, rows streamed into any
//     device (or host) buffer the caller provides.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/vs_b200.h"
#include "vs_internal.h"

using namespace vs_internal;

namespace {

struct File {
    FILE* f = nullptr;
    explicit File(const char* path) : f(path ? std::fopen(path, "rb") : nullptr) {}
    ~File() {
        if (f) std::fclose(f);
    }
    bool read(void* dst, size_t n) { return n == 0 || std::fread(dst, 1, n, f) == n; }
    bool skip(int64_t n) { return n == 0 || std::fseek(f, (long)n, SEEK_CUR) == 0; }
};

// pinned staging ring: file -> pinned[b] -> dst (cudaMemcpyDefault)
struct Stager {
    static constexpr size_t CHUNK = size_t(64) << 20;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    ~Stager() {
        for (int b = 0; b < 2; ++b) {
            if (done[b]) {
                cudaEventSynchronize(done[b]);
                cudaEventDestroy(done[b]);
            }
            if (buf[b]) cudaFreeHost(buf[b]);
        }
    }
    int init() {
        for (int b = 0; b < 2; ++b) {
            CK(cudaHostAlloc(&buf[b], CHUNK, cudaHostAllocDefault));
            CK(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
        }
        return VS_OK;
    }
    int stream(File& f, void* dst, size_t bytes, cudaStream_t s, const char* what) {
        char* d = static_cast<char*>(dst);
        int b = 0;
        bool used[2] = {false, false};
        for (size_t off = 0; off < bytes; off += CHUNK, b ^= 1) {
            const size_t n = std::min(CHUNK, bytes - off);
            if (used[b]) CK(cudaEventSynchronize(done[b]));   // its previous copy has left the buffer
            if (!f.read(buf[b], n)) return set_err(VS_ERR_PARAMETER, "%s: file truncated", what);
            CK(cudaMemcpyAsync(d + off, buf[b], n, cudaMemcpyDefault, s));
            CK(cudaEventRecord(done[b], s));
            used[b] = true;
        }
        return VS_OK;
    }
};

int read_u64(File& f, uint64_t* v, const char* what) {
    if (!f.read(v, 8)) return set_err(VS_ERR_PARAMETER, "%s: file truncated", what);
    return VS_OK;
}

}  // namespace

extern "C" {

int vs_file_to_device(vs_ctx* ctx, const char* path, int64_t offset, int64_t bytes, void* dst) {
    if (!ctx || !path || (!dst && bytes > 0) || offset < 0 || bytes < 0)
        return set_err(VS_ERR_PARAMETER, "bad file read arguments");
    DevGuard g(ctx->device);
    File f(path);
    if (!f.f) return set_err(VS_ERR_PARAMETER, "cannot open %s", path);
    if (!f.skip(offset)) return set_err(VS_ERR_PARAMETER, "%s: seek failed", path);
    Stager st;
    CKS(st.init());
    CKS(st.stream(f, dst, (size_t)bytes, ctx->stream, path));
    CK(cudaStreamSynchronize(ctx->stream));
    return VS_OK;
}

int vs_emb_info(const char* path, int64_t* count, int32_t* dim, int64_t* data_offset) {
    File f(path);
    if (!f.f) return set_err(VS_ERR_PARAMETER, "cannot open %s", path ? path : "(null)");
    unsigned char h[20];
    if (!f.read(h, sizeof h)) return set_err(VS_ERR_PARAMETER, "%s: not an embedding file (short header)", path);
    if (std::memcmp(h, "SVEC", 4) != 0) return set_err(VS_ERR_PARAMETER, "not an embedding file: bad magic");
    uint16_t version;
    std::memcpy(&version, h + 4, 2);
    const uint8_t elem = h[6];
    uint64_t c;
    uint32_t dm;
    std::memcpy(&c, h + 8, 8);
    std::memcpy(&dm, h + 16, 4);
    if (version != 1 || elem != 0) return set_err(VS_ERR_PARAMETER, "unsupported embedding file header");
    if (count) *count = (int64_t)c;
    if (dim) *dim = (int32_t)dm;
    if (data_offset) *data_offset = 20;
    return VS_OK;
}

int vs_ivf_load(vs_ctx* ctx, const char* path, const vs_column* base, int64_t* info, vs_ivf** out) {
    if (!ctx || !path || !out) return set_err(VS_ERR_PARAMETER, "null argument");
    DevGuard g(ctx->device);
    File f(path);
    if (!f.f) return set_err(VS_ERR_PARAMETER, "cannot open %s", path);
    unsigned char h[25];
    if (!f.read(h, 4)) return set_err(VS_ERR_PARAMETER, "not an index file: short header");
    if (std::memcmp(h, "SVIX", 4) != 0) return set_err(VS_ERR_PARAMETER, "not an index file: bad magic");
    if (!f.read(h + 4, 21)) return set_err(VS_ERR_PARAMETER, "not an index file: short header");
    uint16_t version;
    std::memcpy(&version, h + 4, 2);
    const int kind = h[6], metric = h[7], layout = h[8];
    uint32_t nlist, dim;
    uint64_t count;
    std::memcpy(&nlist, h + 9, 4);
    std::memcpy(&dim, h + 13, 4);
    std::memcpy(&count, h + 17, 8);
    if (version != 1) return set_err(VS_ERR_PARAMETER, "unsupported index file version %d", version);
    if (kind != 1) return set_err(VS_ERR_PARAMETER, "SVIX kind %d is not an IVF index", kind);
    if (metric > 1 || layout > 1) return set_err(VS_ERR_PARAMETER, "bad SVIX metric/layout code");
    if (info) {
        info[0] = kind;
        info[1] = metric;
        info[2] = layout;
        info[3] = nlist;
        info[4] = dim;
        info[5] = (int64_t)count;
    }
    const bool owning = layout == 1;
    if (!owning && !base) return set_err(VS_ERR_PARAMETER, "non-owning IVF file needs the base column");
    if (!owning && (base->d != (int)dim || base->n != (int64_t)count))
        return set_err(VS_ERR_SHAPE, "base column (%lld x %d) does not match the index (%llu x %u)",
                       (long long)base->n, base->d, (unsigned long long)count, dim);
    uint64_t sz;
    CKS(read_u64(f, &sz, "centroids"));
    if (sz != (uint64_t)nlist * dim) return set_err(VS_ERR_PARAMETER, "centroid section size mismatch");
    std::vector<float> cen(sz);
    if (!f.read(cen.data(), sz * 4)) return set_err(VS_ERR_PARAMETER, "centroids: file truncated");
    CKS(read_u64(f, &sz, "list sizes"));
    if (sz != nlist) return set_err(VS_ERR_PARAMETER, "list-size section size mismatch");
    std::vector<int64_t> sizes(nlist);
    if (!f.read(sizes.data(), (size_t)nlist * 8)) return set_err(VS_ERR_PARAMETER, "list sizes: file truncated");
    int64_t n_total = 0;
    for (int64_t s : sizes) {
        if (s < 0) return set_err(VS_ERR_PARAMETER, "negative list size");
        n_total += s;
    }
    CKS(read_u64(f, &sz, "list ids"));
    if ((int64_t)sz != n_total) return set_err(VS_ERR_PARAMETER, "list-id section size mismatch");
    Stager st;
    CKS(st.init());
    int64_t* ids = nullptr;
    void* payload = nullptr;
    struct Tmp {
        void* p = nullptr;
        ~Tmp() {
            if (p) cudaFree(p);
        }
    } ids_hold, pay_hold;
    CK(cudaMalloc(&ids, std::max<size_t>((size_t)n_total, 1) * 8));
    ids_hold.p = ids;
    CKS(st.stream(f, ids, (size_t)n_total * 8, ctx->stream, "list ids"));
    if (owning) {
        CKS(read_u64(f, &sz, "payload"));
        if ((int64_t)sz != n_total * (int64_t)dim) return set_err(VS_ERR_PARAMETER, "payload section size mismatch");
        CK(cudaMalloc(&payload, std::max<size_t>((size_t)n_total * dim * 4, 16)));
        pay_hold.p = payload;
        CKS(st.stream(f, payload, (size_t)n_total * dim * 4, ctx->stream, "payload"));
    }
    vs_ivf* v = nullptr;
    // the streamed payload is adopted (borrowed, then owned): no device copy
    CKS(ivf_make(ctx, cen.data(), (int32_t)nlist, (int32_t)dim, sizes, ids, payload,
                 owning ? VS_DTYPE_F32 : base->dtype, metric,
                 owning ? nullptr : base, nullptr, &v, owning));
    if (owning) {
        v->payload_borrowed = false;
        pay_hold.p = nullptr;
    }
    *out = v;
    return VS_OK;
}

}  // extern "C"
