"""Pin the CPU oracle (oracle/sqlvs_oracle.py) against golden vectors produced
by the unmodified reference (tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def test_random_instances_bit_exact(golden):
    g = golden("random_enn.npz")
    for t in range(12):
        seed, nq, nx, dim, k, ip = g[f"t{t}_spec"].tolist()
        r = np.random.default_rng(seed)
        data = r.standard_normal((nx, dim)).astype(np.float32)
        queries = r.standard_normal((nq, dim)).astype(np.float32)
        res = O.enn_search(queries, data, k, O.INNER_PRODUCT if ip else O.SQUARED_L2)
        assert np.array_equal(res.query_row, g[f"t{t}_qrow"])
        assert np.array_equal(res.data_row, g[f"t{t}_ids"])
        assert np.array_equal(res.distance, g[f"t{t}_dist"])  # bit-exact


def test_tie_rule(golden):
    base = np.zeros((6, 4), np.float32)
    base[3] = 1.0
    base[5] = 1.0
    res = O.enn_search(np.zeros((1, 4), np.float32), base, 6)
    assert res.data_row.tolist() == golden("random_enn.npz")["tie_ids"].tolist() == [0, 1, 2, 4, 3, 5]


def test_q15_filtered(golden, sf001):
    g = golden("q15_enn.npz")
    mask = synth.unpack_bitmap(g["bitmap"], int(g["n"]))
    res = O.enn_filtered(g["query"], sf001["reviews"], mask, int(g["k"]))
    assert np.array_equal(res.data_row, g["ids"])
    assert np.array_equal(res.distance, g["dist"])
    # blocked (large-N) oracle gives the same answer
    res2 = O.enn_blocked(g["query"], sf001["reviews"], mask, int(g["k"]), block=5000)
    assert np.array_equal(res2.data_row, g["ids"])
    assert np.array_equal(res2.distance, g["dist"])


@pytest.mark.parametrize("name", ["q11", "q2", "q18"])
def test_batched_and_large_k(golden, sf001, name):
    g = golden(f"{name}_enn.npz")
    data = sf001["images"] if str(g["data"]) == "im_embedding" else sf001["reviews"]
    assert data.shape[0] == int(g["n_data"])
    res = O.enn_search(g["queries"], data, int(g["k"]), str(g["metric"]))
    assert np.array_equal(res.query_row, g["query_row"])
    assert np.array_equal(res.data_row, g["ids"])
    assert np.array_equal(res.distance, g["dist"])


@pytest.mark.parametrize("name", ["a", "b"])
def test_ivf_build_and_search(golden, name):
    g = golden("ivf_small.npz")
    seed0, n, dim, nlist, seed, ip = g[f"{name}_spec"].tolist()
    r = np.random.default_rng(seed0)
    data = r.standard_normal((n, dim)).astype(np.float32)
    queries = r.standard_normal((9, dim)).astype(np.float32)
    cen, assign = O.kmeans(data, nlist, seed)
    assert np.array_equal(cen, g[f"{name}_kmeans_centroids"])
    assert np.array_equal(assign, g[f"{name}_kmeans_assign"])
    centroids, parts, payload = O.ivf_build(data, nlist, seed)
    assert np.array_equal(centroids, g[f"{name}_centroids"])
    assert np.array_equal(np.concatenate(parts), g[f"{name}_ids"])
    metric = O.INNER_PRODUCT if ip else O.SQUARED_L2
    for nprobe in (1, 4, nlist):
        res = O.ivf_search(queries, centroids, parts, lambda c: payload[c], nprobe, 11, metric)
        assert np.array_equal(res.query_row, g[f"{name}_np{nprobe}_qrow"])
        assert np.array_equal(res.data_row, g[f"{name}_np{nprobe}_ids"])
        assert np.array_equal(res.distance, g[f"{name}_np{nprobe}_dist"])
    # full probe == exhaustive (tests/test_ivf.py:63-77)
    full = O.ivf_search(queries, centroids, parts, lambda c: payload[c], nlist, 11, metric)
    enn = O.enn_search(queries, data, 11, metric)
    assert np.array_equal(full.data_row, enn.data_row)
    assert np.array_equal(full.distance, enn.distance)


def test_filtered_ivf_full_probe_equals_filtered_enn(golden):
    g = golden("ivf_small.npz")
    seed0, n, dim, nlist, seed, ip = g["a_spec"].tolist()
    r = np.random.default_rng(seed0)
    data = r.standard_normal((n, dim)).astype(np.float32)
    queries = r.standard_normal((9, dim)).astype(np.float32)
    centroids = g["a_centroids"]
    sizes = g["a_sizes"]
    parts = np.split(g["a_ids"], np.cumsum(sizes)[:-1])
    mask = np.random.default_rng(1).random(n) < 0.2
    a = O.ivf_search(queries, centroids, parts, lambda c: data[parts[c]], nlist, 11, mask=mask)
    b = O.enn_filtered(queries, data, mask, 11)
    assert np.array_equal(a.data_row, b.data_row)
    assert np.array_equal(a.distance, b.distance)


def test_svix_bytes(golden):
    from pathlib import Path
    ref = (Path(__file__).parent / "golden" / "svix_ivf_owning.bin").read_bytes()
    data = np.random.default_rng(5).standard_normal((100, 4)).astype(np.float32)
    centroids, parts, payload = O.ivf_build(data, 4, 0)
    mine = O.svix_ivf_bytes(4, 4, 100, O.SQUARED_L2, True, centroids, parts, payload)
    assert mine == ref


def test_config1_sample(golden):
    g = golden("config1_sample.npz")
    emb, mask, q = synth.config1()
    assert int(mask.sum()) == 10767
    res = O.enn_filtered(q[g["queries_idx"]], emb, mask, 10)
    assert np.array_equal(res.data_row.reshape(-1, 10), g["ids"])
    assert np.array_equal(res.distance.reshape(-1, 10), g["dist"])


def test_postfilter(golden):
    """oversample_postfilter over the reference's own vector_search_operator
    output (Q11 self-match exclusion, Q15 semi join, rank predicate, both)."""
    g = golden("postfilter.npz")
    qr, rank = g["out_query_row"], g["out_rank"]
    self_mask = g["out_key_d"] != g["dkey"][g["qrows"]][qr]
    semi_mask = np.isin(g["dpart"][g["out_data_row"]], g["keep_parts"])
    masks = {"self": self_mask, "semi": semi_mask, "rank": rank >= 3, "both": self_mask & semi_mask}
    for name, m in masks.items():
        kept, short = O.oversample_postfilter(qr, m, int(g["k"]))
        assert np.array_equal(qr[kept], g[f"{name}_query_row"]), name
        assert np.array_equal(g["out_data_row"][kept], g[f"{name}_data_row"]), name
        assert np.array_equal(g["out_distance"][kept], g[f"{name}_distance"]), name
        assert np.array_equal(rank[kept], g[f"{name}_rank"]), name
        assert sorted(short) == g[f"{name}_short_q"].tolist(), name
        assert [short[q] for q in sorted(short)] == g[f"{name}_short_n"].tolist(), name


def test_q15_ivf_plan_vector_search(golden, sf001):
    """The reference's Q15 'ivf' plan at SF=0.01 (k' = 50,000 over nprobe=32
    of nlist=1024 lists): the oracle's IVF search over the reference's own
    index reproduces the operator's vs_* columns and the semi-join post-filter."""
    g = golden("q15_ivf.npz")
    sizes = g["sizes"]
    parts = np.split(g["ids"], np.cumsum(sizes)[:-1])
    reviews = sf001["reviews"]
    res = O.ivf_search(g["queries"], g["centroids"], parts, lambda c: reviews[parts[c]], int(g["nprobe"]),
                       int(g["k_prime"]))
    assert res.visited_rows == int(g["visited"])
    assert np.array_equal(res.data_row, g["vs_data_row"])
    assert np.array_equal(res.distance, g["vs_distance"])
    assert np.array_equal(res.rank, g["vs_rank"])
    keep = np.isin(sf001["review_partkeys"][res.data_row], g["keep_set"])
    kept, short = O.oversample_postfilter(res.query_row, keep, int(g["pf_k"]))
    assert np.array_equal(res.data_row[kept], g["pf_data_row"])
    assert np.array_equal(res.distance[kept], g["pf_distance"])
    assert short.get(0, 0) == int(g["pf_short"][0])


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_pruned_oracle_equals_enn_search(metric):
    """oracle.enn_pruned (the large-N checker of the scale tests) == enn_search,
    duplicates and ties included."""
    r = np.random.default_rng(9)
    x = r.standard_normal((30000, 48)).astype(np.float32)
    x[100] = x[5]
    x[7] = x[5]
    x[200:260] = x[300]
    q = np.concatenate([r.standard_normal((4, 48)), x[[5, 300]]]).astype(np.float32)
    ids = np.sort(r.choice(90000, 30000, replace=False))
    for k in (1, 64, 2500):
        a = O.enn_search(q, x, k, metric, row_ids=ids)
        b = O.enn_pruned(q, x, k, metric, row_ids=ids, block=7000)
        assert np.array_equal(a.query_row, b.query_row)
        assert np.array_equal(a.data_row, b.data_row)
        assert np.array_equal(a.distance, b.distance)
