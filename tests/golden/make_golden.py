"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (`/root/reference/pkg/src/sqlvs`) in the build container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed as
small .npz / .bin / .json fixtures. Large inputs (embeddings) are NOT stored:
they are rebuilt bit-for-bit by `paper_2605_15957_b200.synth`, whose arrays are
pinned here by sha256 against the reference generator.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("SQLVS_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import sqlvs.executor as ex  # noqa: E402
from sqlvs.datagen import DatasetSpec, generate, make_query_vectors  # noqa: E402
from sqlvs.plans import builtin_plan  # noqa: E402
from sqlvs.table import EmbeddingColumn  # noqa: E402
from sqlvs.vecindex import (IvfIndex, SearchParams, _kmeans, enn_search,  # noqa: E402
                            save_index)

from paper_2605_15957_b200 import synth  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def capture_vs(query: str, ds):
    """Run a builtin ENN plan, capturing every vector_search_operator call."""
    calls = []
    orig = ex.vector_search_operator

    def spy(qt, qf, dt, df, params, metric="squared_l2", index=None, **kw):
        out, stats = orig(qt, qf, dt, df, params, metric=metric, index=index, **kw)
        calls.append(dict(qt=qt, qf=qf, dt=dt, df=df, params=params, metric=metric,
                          out=out, stats=stats))
        return out, stats

    ex.vector_search_operator = spy
    try:
        run = ex.execute_base(builtin_plan(query, "enn"), ds, None)
    finally:
        ex.vector_search_operator = orig
    return run, calls


def make_postfilter_golden():
    from sqlvs.table import Schema, Table, embedding
    from sqlvs.vecsearch import oversample_postfilter, vector_search_operator
    r2 = np.random.default_rng(77)
    nd, nq, d, kp, k = 400, 23, 16, 12, 4
    data = r2.standard_normal((nd, d)).astype(np.float32)
    qrows = r2.choice(nd, nq, replace=False)             # queries are data rows (self matches)
    dkey = np.arange(nd, dtype=np.int64) * 3 + 1
    dpart = r2.integers(0, 40, nd).astype(np.int64)
    dval = r2.standard_normal(nd)
    dt = Table(Schema([("key", "int64"), ("part", "int64"), ("val", "float64"), ("emb", embedding(d))]),
               {"key": dkey, "part": dpart, "val": dval, "emb": EmbeddingColumn(data)})
    qt = Table(Schema([("key", "int64"), ("qemb", embedding(d))]),
               {"key": dkey[qrows], "qemb": EmbeddingColumn(data[qrows])})
    out, _ = vector_search_operator(qt, "qemb", dt, "emb", SearchParams(k=k, k_prime=kp))
    keep_parts = np.array([3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37], np.int64)
    keep_set = Table(Schema([("p", "int64")]), {"p": keep_parts})
    res = {"data": data, "qrows": qrows, "dkey": dkey, "dpart": dpart, "dval": dval,
           "keep_parts": keep_parts, "kp": kp, "k": k,
           "out_query_row": np.asarray(out.column("vs_query_row")),
           "out_data_row": np.asarray(out.column("vs_data_row")),
           "out_distance": np.asarray(out.column("vs_distance")),
           "out_rank": np.asarray(out.column("vs_rank")),
           "out_key_d": np.asarray(out.column("key_d")), "out_val": np.asarray(out.column("val"))}
    cases = {
        "self": dict(keep="key_d != key"),                              # Q11 (plans.py:537)
        "semi": dict(keep=None, keep_set=keep_set, semi_keys=("part", "p")),   # Q15 (plans.py:574)
        "rank": dict(keep="vs_rank >= 3"),
        "both": dict(keep="key_d != key", keep_set=keep_set, semi_keys=("part", "p")),
    }
    for name, kw in cases.items():
        kept, short = oversample_postfilter(out, kw.pop("keep"), k, **kw)
        res[f"{name}_query_row"] = np.asarray(kept.column("vs_query_row"))
        res[f"{name}_data_row"] = np.asarray(kept.column("vs_data_row"))
        res[f"{name}_distance"] = np.asarray(kept.column("vs_distance"))
        res[f"{name}_rank"] = np.asarray(kept.column("vs_rank"))
        res[f"{name}_short_q"] = np.array(sorted(short), np.int64)
        res[f"{name}_short_n"] = np.array([short[q] for q in sorted(short)], np.int64)
    np.savez_compressed(HERE / "postfilter.npz", **res)


def make_q15_ivf_golden():
    """The Q15 'ivf' plan (plans.py:571-574) through the reference executor at
    SF=0.01 with the runner's IVF catalog (runner.py:26-56: nlist =
    default_nlist(n), seed 0): its vector_search call (k' = 500 k = 50,000 >
    every candidate) and the semi-join post-filter after it."""
    from sqlvs.executor import IndexCatalog
    from sqlvs.runner import default_nlist
    import sqlvs.vecsearch as vsm
    ds = generate(DatasetSpec(sf=0.01))
    col = ds.table("reviews").column("rv_embedding")
    nlist = min(default_nlist(col.count), col.count)
    idx = IvfIndex.build(col, nlist=nlist, seed=0)
    cat = IndexCatalog()
    cat.register("ivf:reviews", idx, col)
    calls, posts = [], []
    orig_vs, orig_pf = ex.vector_search_operator, ex.oversample_postfilter

    def spy(qt, qf, dt, df, params, metric="squared_l2", index=None, **kw):
        out, stats = orig_vs(qt, qf, dt, df, params, metric=metric, index=index, **kw)
        calls.append(dict(qt=qt, qf=qf, params=params, out=out, stats=stats))
        return out, stats

    def spy_pf(vs_output, keep, k, keep_set=None, semi_keys=None):
        out, short = orig_pf(vs_output, keep, k, keep_set=keep_set, semi_keys=semi_keys)
        posts.append(dict(out=out, short=short, keep_set=keep_set, semi_keys=semi_keys, k=k))
        return out, short

    ex.vector_search_operator, ex.oversample_postfilter = spy, spy_pf
    try:
        run = ex.execute_base(builtin_plan("Q15", "ivf"), ds, cat)
    finally:
        ex.vector_search_operator, ex.oversample_postfilter = orig_vs, orig_pf
    (c,), (pf,) = calls, posts
    o, po = c["out"], pf["out"]
    left, right = pf["semi_keys"]
    np.savez_compressed(
        HERE / "q15_ivf.npz", nlist=nlist, centroids=idx.centroids,
        sizes=np.array([len(p) for p in idx.partitions], np.int64),
        ids=np.concatenate(idx.partitions).astype(np.int64),
        queries=c["qt"].column(c["qf"]).values, k=c["params"].k, k_prime=c["params"].k_prime,
        nprobe=c["params"].nprobe, visited=c["stats"].visited_rows,
        vs_query_row=np.asarray(o.column("vs_query_row")), vs_data_row=np.asarray(o.column("vs_data_row")),
        vs_distance=np.asarray(o.column("vs_distance")), vs_rank=np.asarray(o.column("vs_rank")),
        keep_set=np.asarray(pf["keep_set"].column(right)), semi_left=left, pf_k=pf["k"],
        pf_data_row=np.asarray(po.column("vs_data_row")), pf_distance=np.asarray(po.column("vs_distance")),
        pf_rank=np.asarray(po.column("vs_rank")),
        pf_short=np.array([pf["short"].get(0, 0)], np.int64),
        final_reviewkey=np.asarray(run.output.column("rv_reviewkey")) if hasattr(run, "output") else
        np.asarray(run.result.column("rv_reviewkey")))


def make_emb_golden():
    """A small .emb file written by the reference's writer (datagen.py:355-360)."""
    from sqlvs.datagen import write_embeddings
    x = np.random.default_rng(17).standard_normal((500, 48)).astype(np.float32)
    write_embeddings(HERE / "ref_small.emb", EmbeddingColumn(x))


def main():
    if "--only" in sys.argv:
        globals()["make_" + sys.argv[sys.argv.index("--only") + 1] + "_golden"]()
        return
    meta = {}
    # --- synth pins ---------------------------------------------------------
    ds = generate(DatasetSpec(sf=0.01))
    rv, im = ds.table("reviews"), ds.table("images")
    meta["sf001"] = {
        "reviews": sha(rv.column("rv_embedding").values),
        "review_partkeys": sha(np.asarray(rv.column("rv_partkey"))),
        "images": sha(im.column("im_embedding").values),
        "image_partkeys": sha(np.asarray(im.column("im_partkey"))),
        "p_size": sha(np.asarray(ds.table("part").column("p_size"))),
        "n_reviews": rv.row_count, "n_images": im.row_count,
        "q_review_seed7_n3": sha(make_query_vectors(ds, "review", 3, 7).values),
    }
    ds1 = generate(DatasetSpec(sf=0.1, d_r=384, d_i=384))
    rv1 = ds1.table("reviews")
    emb1 = rv1.column("rv_embedding").values[:100_000]
    pk1 = np.asarray(rv1.column("rv_partkey"))[:100_000]
    part = ds1.table("part")
    small = np.asarray(part.column("p_partkey"))[np.asarray(part.column("p_size")) <= 5]
    mask1 = np.isin(pk1, small)
    q1 = make_query_vectors(ds1, "review", 1000, seed=7).values
    meta["config1"] = {"emb": sha(emb1), "mask": sha(mask1), "n_sel": int(mask1.sum()),
                       "queries": sha(q1)}
    # config-1 reference answers for a query sample (exact filtered top-10)
    rows1 = np.flatnonzero(mask1)
    sample = np.arange(0, 1000, 50)
    nt = enn_search(EmbeddingColumn(q1[sample]), EmbeddingColumn(emb1[rows1]), SearchParams(k=10))
    np.savez_compressed(HERE / "config1_sample.npz", queries_idx=sample,
                        ids=rows1[nt.data_row].reshape(len(sample), 10),
                        dist=nt.distance.reshape(len(sample), 10))

    # --- Q15: pre-filtered ENN top-100 (the reference's filtered pattern) ------
    run, calls = capture_vs("Q15", ds)
    (c,) = calls
    scoped_keys = np.asarray(c["dt"].column("rv_reviewkey"))
    mask = np.isin(np.asarray(rv.column("rv_reviewkey")), scoped_keys)
    rows = np.flatnonzero(mask)
    out = c["out"]
    np.savez_compressed(
        HERE / "q15_enn.npz",
        bitmap=synth.pack_mask(mask), n=rv.row_count,
        query=c["qt"].column(c["qf"]).values,
        k=c["params"].k_prime,
        ids=rows[np.asarray(out.column("vs_data_row"))],
        dist=np.asarray(out.column("vs_distance")),
        reviewkeys=np.asarray(run.result.column("rv_reviewkey")),
        result_dist=np.asarray(run.result.column("vs_distance")))

    # --- Q11 (batched similarity join, k'=4) and Q2/Q18 (k'=1000) --------------
    for qname in ("Q11", "Q2", "Q18"):
        _, calls = capture_vs(qname, ds)
        (c,) = calls
        out = c["out"]
        qv = c["qt"].column(c["qf"]).values
        np.savez_compressed(
            HERE / f"{qname.lower()}_enn.npz", queries=qv, k=c["params"].k_prime,
            metric=c["metric"], data=c["df"], n_data=c["dt"].row_count,
            data_sha=sha(c["dt"].column(c["df"]).values),
            query_row=np.asarray(out.column("vs_query_row")),
            ids=np.asarray(out.column("vs_data_row")),
            dist=np.asarray(out.column("vs_distance")))

    # --- acceptance-1 style random instances (both metrics, ties, k = N) -------
    rng = np.random.default_rng(20240801)
    inst = {}
    for t in range(12):
        nq = int(2 ** rng.uniform(0, 7))
        nx = int(2 ** rng.uniform(1, 11))
        dim = int(rng.choice([3, 16, 64, 100]))
        metric = "squared_l2" if t % 2 == 0 else "inner_product"
        seed = int(rng.integers(1 << 30))
        r2 = np.random.default_rng(seed)
        data = r2.standard_normal((nx, dim)).astype(np.float32)
        queries = r2.standard_normal((nq, dim)).astype(np.float32)
        k = int(rng.integers(1, min(64, nx) + 1))
        if t == 11:
            k = nx
        nt = enn_search(EmbeddingColumn(queries), EmbeddingColumn(data), SearchParams(k=k),
                        metric=metric)
        inst[f"t{t}_spec"] = np.array([seed, nq, nx, dim, k, t % 2], np.int64)
        inst[f"t{t}_qrow"] = nt.query_row
        inst[f"t{t}_ids"] = nt.data_row
        inst[f"t{t}_dist"] = nt.distance
    # duplicate-vector tie rule (tests/test_enn.py:72-80)
    base = np.zeros((6, 4), np.float32)
    base[3] = 1.0
    base[5] = 1.0
    nt = enn_search(EmbeddingColumn(np.zeros((1, 4), np.float32)), EmbeddingColumn(base),
                    SearchParams(k=6))
    inst["tie_ids"] = nt.data_row
    np.savez_compressed(HERE / "random_enn.npz", **inst)

    # --- IVF: build (k-means), probes, search at several nprobe ---------------
    ivf = {}
    for name, (n, dim, nlist, seed, metric) in {
        "a": (3000, 16, 32, 0, "squared_l2"),
        "b": (1500, 24, 20, 3, "inner_product"),
    }.items():
        r2 = np.random.default_rng(100 + seed)
        data = r2.standard_normal((n, dim)).astype(np.float32)
        queries = r2.standard_normal((9, dim)).astype(np.float32)
        idx = IvfIndex.build(EmbeddingColumn(data), nlist=nlist, metric=metric, seed=seed)
        ivf[f"{name}_spec"] = np.array([100 + seed, n, dim, nlist, seed,
                                        int(metric == "inner_product")], np.int64)
        ivf[f"{name}_centroids"] = idx.centroids
        ivf[f"{name}_sizes"] = np.array([len(p) for p in idx.partitions], np.int64)
        ivf[f"{name}_ids"] = np.concatenate(idx.partitions)
        for nprobe in (1, 4, nlist):
            nt = idx.search(EmbeddingColumn(queries), SearchParams(k=7, k_prime=11, nprobe=nprobe))
            ivf[f"{name}_np{nprobe}_qrow"] = nt.query_row
            ivf[f"{name}_np{nprobe}_ids"] = nt.data_row
            ivf[f"{name}_np{nprobe}_dist"] = nt.distance
        cen, assign = _kmeans(data, nlist, seed)
        ivf[f"{name}_kmeans_centroids"] = cen
        ivf[f"{name}_kmeans_assign"] = assign
    np.savez_compressed(HERE / "ivf_small.npz", **ivf)

    # --- SVIX byte image ---------------------------------------------------------
    r2 = np.random.default_rng(5)
    data = r2.standard_normal((100, 4)).astype(np.float32)
    idx = IvfIndex.build(EmbeddingColumn(data), nlist=4, seed=0)
    save_index(idx, HERE / "svix_ivf_owning.bin")
    meta["svix_seed"] = 5

    # --- the step after the search: vector_search_operator + oversample_postfilter
    # (vecsearch.py:64-202) on small tables: Q11's cross-side "key_d != key",
    # Q15's semi join, a rank predicate, shortfalls (k' rows that do not survive)
    make_postfilter_golden()
    make_q15_ivf_golden()
    make_emb_golden()

    (HERE / "meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    if sys.argv[1:] == ["postfilter"]:
        make_postfilter_golden()
    else:
        main()
