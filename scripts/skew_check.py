"""IVF tensor-core scan on a SKEWED index (trained on a sample, then every row
assigned: the mixture law's noise makes a few lists absorb much of the data),
with and without cutting long lists into row chunks. Prints one JSON line."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_15957_b200 as vs  # noqa: E402
from paper_2605_15957_b200 import _native as N  # noqa: E402
from paper_2605_15957_b200 import synth  # noqa: E402


def main():
    n, d, nlist, nq, nprobe, k = 8_000_000, 768, 16384, 10_000, 32, 10
    dev = torch.device("cuda", 0)
    data, centers = bench._device_slice_bf16(n, d, 0, n, dev)
    trained = vs.IvfIndex.build(vs.EmbeddingColumn.from_device(data[:500_000].contiguous()), nlist, seed=0)
    cen = trained.centroids.copy()
    cen[0] = 0.0                          # a centroid at the origin: the nearest list of most rows
    tmp = vs.IvfIndex.from_device_lists(cen, np.r_[n, np.zeros(nlist - 1, np.int64)],
                                        torch.arange(n, device=dev), data, count=n)
    lists = tmp.assign(vs.EmbeddingColumn.from_device(data))
    del tmp
    order = torch.sort(lists, stable=True).indices
    sizes = torch.bincount(lists, minlength=nlist).cpu().numpy().astype(np.int64)
    payload = data[order].contiguous()
    del data
    torch.cuda.empty_cache()
    idx = vs.IvfIndex.from_device_lists(cen, sizes, order, payload, count=n)
    q = synth.device_queries(centers, nq, seed=7)
    ctx = N.Context.get()
    out = {"list_rows_max": int(sizes.max()), "list_rows_mean": float(sizes.mean())}
    for name, rows in (("chunked", 0), ("whole_lists", 1 << 40)):
        ctx.set_option(N.OPT_IVF_CHUNK_ROWS, rows)
        for _ in range(2):
            idx.search_raw(q, k, nprobe, want_probes=False)
        ctx.set_option(N.OPT_TIMING, 1)
        ctx.kernel_times(reset=True)
        t0 = time.perf_counter()
        for _ in range(3):
            idx.search_raw(q, k, nprobe, want_probes=False)
        el = (time.perf_counter() - t0) / 3
        kt = ctx.kernel_times(reset=True)
        ctx.set_option(N.OPT_TIMING, 0)
        out[name] = {"q_per_s": round(nq / el), "ivf_scan_ms": round(kt["ivf_scan"][0] / 1e6 / 3, 3)}
        res = idx.search_raw(q[:64], k, nprobe, want_probes=False)
        out[name + "_ids0"] = res[0][:2].tolist()
    ctx.set_option(N.OPT_IVF_CHUNK_ROWS, 0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
