"""Coarse-quantizer cost breakdown (config-3 shape: 16,384 centroids x 1024,
10k queries, nprobe 32): phase-A GEMM vs exact phase B, and the survivors per
query the bf16 margin lets through. Index trained on N rows (default 2M) of
the bench's mixture law. One JSON line."""
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
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    d, nlist, nq, nprobe = 1024, 16384, 10_000, int(sys.argv[2]) if len(sys.argv) > 2 else 32
    dev = torch.device("cuda", 0)
    data, centers = bench._device_slice(n, d, 0, n, dev)
    t0 = time.time()
    idx = vs.IvfIndex.build(vs.EmbeddingColumn.from_device(data), nlist, seed=0, max_iters=10)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    q = synth.device_queries(centers, nq, seed=7)
    ctx = N.Context.get()
    ctx.set_option(N.OPT_TIMING, 1)
    out = torch.empty((nq, nprobe), dtype=torch.int32, device=dev)
    for _ in range(3):
        idx.probe(q, nprobe, out=out)
    ctx.kernel_times(reset=True)
    reps = 10
    prof = None
    if hasattr(N.load(), "vs_debug_rerank_profile"):   # profiling build (scripts/prof_rerank.sh)
        import ctypes as C
        prof = N.load().vs_debug_rerank_profile
        prof.argtypes = [C.c_void_p, C.c_int]
        buf = np.zeros(8, np.uint64)
        torch.cuda.synchronize()
        prof(buf.ctypes.data, 1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        idx.probe(q, nprobe, out=out)
    ev1.record()
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    st = ctx.stats()
    phases = None
    if prof is not None:
        prof(buf.ctypes.data, 1)
        phases = {nm: round(float(buf[i]) / (nq * reps)) for i, nm in
                  enumerate(["setup", "gather", "select", "score", "topk", "candidates", "live"])}
    print(json.dumps({"n": n, "nlist": nlist, "d": d, "nq": nq, "nprobe": nprobe, "build_s": round(build_s, 1),
                      "probe_ms": round(ev0.elapsed_time(ev1) / reps, 3),
                      "kernel_ms": {k: round(v[0] / 1e6 / reps, 3) for k, v in kt.items() if v[1]},
                      "survivors_per_query": st[N.STAT_SURVIVORS] / nq,
                      "rerank_cycles_per_cta": phases}))


if __name__ == "__main__":
    main()
