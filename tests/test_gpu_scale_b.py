"""Parity at the BASELINE scales, part B: config 4 (BASELINE.json configs[3])
at full size on one GPU — IVF-Flat over 50M x 768 bfloat16 embeddings,
nlist=16384 built on the GPU, nprobe=64, top-10, unfiltered, 10k queries,
searched with the tcgen05 list-major scan. Probes, ids and float64 distances
of sampled queries must equal the oracle's (vecindex.py:230-258), fed the
bfloat16 rows upcast to float32 (SURVEY §8c parity rule for bf16 storage)."""

import numpy as np
import pytest
import torch

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N
from paper_2605_15957_b200 import synth
from test_gpu_scale_a import assert_rows_equal, sample_rows

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_config4_bf16_ivf_sampled_queries_equal_oracle():
    n, d, nq, nlist, nprobe, k = 50_000_000, 768, 10_000, 16384, 64, 10
    dev = torch.device("cuda", 0)
    torch.cuda.empty_cache()
    data, centers = synth.device_rows(n, d, 0, n, dev, dtype=torch.bfloat16)
    queries = synth.device_queries(centers, nq, seed=7)
    ctx = N.Context(0)
    index = vs.IvfIndex.build(vs.EmbeddingColumn.from_device(data), nlist, seed=0, device=ctx)
    # the sampled queries' probed lists, gathered before the base column goes
    qidx = sample_rows(nq, 8)
    q = queries[torch.from_numpy(qidx).to(dev)].contiguous()
    probes_s = index.probe(q, nprobe, device=ctx).cpu().numpy()
    lists = {int(c): data[torch.from_numpy(index.partitions[int(c)]).to(dev)].float().cpu().numpy()
             for c in np.unique(probes_s)}
    del data
    torch.cuda.empty_cache()
    out = (torch.empty((nq, k), dtype=torch.int64, device=dev),
           torch.empty((nq, k), dtype=torch.float64, device=dev),
           torch.empty((nq,), dtype=torch.int32, device=dev))
    _, _, _, probes, _ = index.search_raw(queries, k, nprobe, device=ctx, out=out, want_probes=True)
    torch.cuda.synchronize()
    ids, dist, cnt = (t.cpu().numpy() for t in out)
    assert np.array_equal(probes[qidx], probes_s)

    def vectors_of(c):
        if c not in lists:
            raise AssertionError(f"oracle probes list {c}, not among the GPU probes")
        return lists[c]

    ref = O.ivf_search(q.cpu().numpy(), index.centroids, index.partitions, vectors_of, nprobe, k)
    assert np.array_equal(np.asarray(ref.probes), probes[qidx]), "probes differ from the oracle"
    assert_rows_equal(ids, dist, cnt, ref, qidx)
    del index
    ctx.close()
    torch.cuda.empty_cache()
