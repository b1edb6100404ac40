"""Config-3 diagnostics on one GPU: where the overflow re-runs come from
(coarse quantizer vs list scan) and per-kernel-class times of one search."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_15957_b200 as vs  # noqa: E402
from paper_2605_15957_b200 import _native as N, synth  # noqa: E402

n, d, nq = 10_000_000, 1024, 10_000
dev = torch.device("cuda", 0)
data, centers = synth.device_rows(n, d, 0, n, dev)
q = synth.device_queries(centers, nq, seed=7)
mask = synth.device_bernoulli(n, 0.01, 4243, dev)
bits = synth.pack_bits_torch(mask)
ctx = N.Context.get(0)
t0 = time.time()
idx = vs.IvfIndex.build(vs.EmbeddingColumn.from_device(data), 16384, seed=0)
torch.cuda.synchronize()
print(f"build {time.time() - t0:.1f}s; overflow re-runs so far (build) {ctx.stats()[N.STAT_OVERFLOW_QUERIES]}",
      flush=True)
REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 3
out = (torch.empty((nq, 10), dtype=torch.int64, device=dev), torch.empty((nq, 10), dtype=torch.float64, device=dev),
       torch.empty((nq,), dtype=torch.int32, device=dev))
ctx.set_option(N.OPT_TIMING, 1)
for rep in range(REPS):
    s0 = ctx.stats()[N.STAT_OVERFLOW_QUERIES]
    idx.probe(q, 32)
    s1 = ctx.stats()[N.STAT_OVERFLOW_QUERIES]
    ctx.kernel_times(reset=True)
    idx.search_raw(q, 10, 32, row_filter=bits, out=out, want_probes=False)
    torch.cuda.synchronize()
    s2 = ctx.stats()[N.STAT_OVERFLOW_QUERIES]
    kt = {k: round(v[0] / 1e6, 3) for k, v in ctx.kernel_times().items() if v[1]}
    print(f"rep {rep}: overflow re-runs probe-only {s1 - s0}, full search {s2 - s1}; kernel ms {kt}", flush=True)
for qn in (1, 100):
    s0 = ctx.stats()[N.STAT_OVERFLOW_QUERIES]
    sub = q[:qn].contiguous()
    o2 = tuple(t[:qn].contiguous() for t in out)
    idx.search_raw(sub, 10, 32, row_filter=bits, out=o2, want_probes=False)
    torch.cuda.synchronize()
    print(f"Q={qn}: overflow re-runs {ctx.stats()[N.STAT_OVERFLOW_QUERIES] - s0}", flush=True)
