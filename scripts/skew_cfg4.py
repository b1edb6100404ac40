"""Config 4 (50M x 768 bf16, nlist 16,384, nprobe 64, k 10, 10k queries) on a
SAMPLE-TRAINED index: k-means on 2M rows, then every row assigned to its
nearest centroid (vs_ivf_assign) and scattered chunk by chunk into one
list-contiguous device payload that the index borrows (vs_ivf_wrap). The
mixture law's noise makes such an index strongly skewed (one list held 1.69M
rows); the scan is timed with long lists cut into row chunks (default) and
with whole lists. One JSON line."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_15957_b200 as vs  # noqa: E402
from paper_2605_15957_b200 import _native as N  # noqa: E402
from paper_2605_15957_b200 import synth  # noqa: E402


def main():
    n, d, nlist, nq, nprobe, k, ntrain = 50_000_000, 768, 16384, 10_000, 64, 10, 2_000_000
    dev = torch.device("cuda", 0)
    chunk = 1 << 20
    g = torch.Generator(device=dev)
    g.manual_seed(42)
    centers = torch.randn(64, d, generator=g, device=dev)
    centers /= centers.norm(dim=1, keepdim=True)

    def rows(ci):
        a, b = ci * chunk, min(n, (ci + 1) * chunk)
        gg = torch.Generator(device=dev)
        gg.manual_seed(100_000 + ci)
        asg = torch.randint(0, 64, (b - a,), generator=gg, device=dev)
        v = centers[asg] + 0.55 * torch.randn(b - a, d, generator=gg, device=dev)
        v /= v.norm(dim=1, keepdim=True)
        return v.to(torch.bfloat16)

    nchunks = (n + chunk - 1) // chunk
    train = torch.cat([rows(ci) for ci in range((ntrain + chunk - 1) // chunk)])[:ntrain].contiguous()
    tidx = vs.IvfIndex.build(vs.EmbeddingColumn.from_device(train), nlist, seed=0)
    assign = torch.empty(n, dtype=torch.int32, device=dev)
    for ci in range(nchunks):
        x = rows(ci)
        assign[ci * chunk: ci * chunk + x.shape[0]] = tidx.assign(vs.EmbeddingColumn.from_device(x))
    sizes = torch.bincount(assign, minlength=nlist).cpu().numpy().astype(np.int64)
    order = torch.sort(assign, stable=True).indices
    pos = torch.empty(n, dtype=torch.int64, device=dev)
    pos[order] = torch.arange(n, device=dev)
    del assign
    payload = torch.empty((n, d), dtype=torch.bfloat16, device=dev)
    for ci in range(nchunks):
        x = rows(ci)
        payload[pos[ci * chunk: ci * chunk + x.shape[0]]] = x
    del pos, train
    torch.cuda.empty_cache()
    idx = vs.IvfIndex.from_device_lists(tidx.centroids, sizes, order, payload, count=n)
    q = synth.device_queries(centers, nq, seed=7)
    ctx = N.Context.get()
    out = {"list_rows_max": int(sizes.max()), "list_rows_p99": int(np.percentile(sizes, 99)),
           "list_rows_mean": float(sizes.mean())}
    ref = None
    for name, rows_per_chunk in (("chunked", 0), ("whole_lists", 1 << 40)):
        ctx.set_option(N.OPT_IVF_CHUNK_ROWS, rows_per_chunk)
        res = idx.search_raw(q, k, nprobe, want_probes=False)
        if ref is None:
            ref = res
        else:
            out["identical_results"] = bool(np.array_equal(res[0], ref[0]) and np.array_equal(res[1], ref[1]))
        ctx.set_option(N.OPT_TIMING, 1)
        ctx.kernel_times(reset=True)
        t0 = time.perf_counter()
        for _ in range(3):
            idx.search_raw(q, k, nprobe, want_probes=False)
        el = (time.perf_counter() - t0) / 3
        kt = ctx.kernel_times(reset=True)
        ctx.set_option(N.OPT_TIMING, 0)
        out[name] = {"q_per_s": round(nq / el), "ivf_scan_ms": round(kt["ivf_scan"][0] / 1e6 / 3, 3)}
    ctx.set_option(N.OPT_IVF_CHUNK_ROWS, 0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
