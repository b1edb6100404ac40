"""Host-side logic of the drop-in API that needs no GPU: parameter checks,
filter normalisation, result layout, SVIX serialisation (byte-identical to
the reference writer), operator output assembly and post-filtering."""

from pathlib import Path

import numpy as np
import pytest

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import synth
from paper_2605_15957_b200.distributed import lpt_assign, row_shard
from paper_2605_15957_b200.table import Schema, Table, embedding
from paper_2605_15957_b200.vecindex import NeighborTable, filter_bitmap
from paper_2605_15957_b200.vecsearch import build_vs_output, oversample_postfilter, vector_search_operator

GOLDEN = Path(__file__).parent / "golden"


def test_search_params_validation():
    p = vs.SearchParams(k=5)
    assert p.k_prime == 5 and p.ef == 5 and p.nprobe == 1
    for bad in (dict(k=0), dict(k=5, k_prime=4), dict(k=1, nprobe=0), dict(k=3, ef=2)):
        with pytest.raises(vs.ParameterError):
            vs.SearchParams(**bad)


def test_embedding_column_contract():
    with pytest.raises(vs.ShapeError):
        vs.EmbeddingColumn(np.array([[1.0, np.nan]], np.float32))
    with pytest.raises(vs.ShapeError):
        vs.EmbeddingColumn(np.zeros(5, np.float32))
    c = vs.EmbeddingColumn(np.zeros(8, np.float32), dim=4)
    assert c.count == 2 and c.dim == 4 and not c.values.flags.writeable


def test_filter_forms():
    rng = np.random.default_rng(0)
    for n in (1, 31, 32, 33, 1000):
        m = rng.random(n) < 0.3
        w = filter_bitmap(m, n)
        assert np.array_equal(w, synth.pack_mask(m))
        assert np.array_equal(filter_bitmap(np.flatnonzero(m), n), w)
        assert np.array_equal(filter_bitmap(w, n), w)
    with pytest.raises(vs.ShapeError):
        filter_bitmap(np.ones(5, bool), 6)
    with pytest.raises(vs.ParameterError):
        filter_bitmap(np.array([7]), 5)


def test_neighbor_table_from_padded():
    ids = np.array([[3, 1, -1], [2, -1, -1]])
    dist = np.array([[0.1, 0.2, np.nan], [0.5, np.nan, np.nan]])
    nt = NeighborTable.from_padded(ids, dist, np.array([2, 1]), "squared_l2", 10)
    assert nt.query_row.tolist() == [0, 0, 1]
    assert nt.data_row.tolist() == [3, 1, 2]
    assert nt.rank.tolist() == [0, 1, 0]
    assert nt.per_query_counts().tolist() == [2, 1]
    assert nt.visited_rows == 10


def test_svix_save_is_byte_identical_to_reference(tmp_path):
    data = np.random.default_rng(5).standard_normal((100, 4)).astype(np.float32)
    centroids, parts, payload = O.ivf_build(data, 4, 0)
    idx = vs.IvfIndex(4, 4, 100, "squared_l2", "owning", centroids, parts, payload)
    path = tmp_path / "a.idx"
    vs.save_index(idx, path)
    assert path.read_bytes() == (GOLDEN / "svix_ivf_owning.bin").read_bytes()
    back = vs.load_index(path)
    assert back.nlist == 4 and back.layout == "owning"
    assert np.array_equal(back.centroids, centroids)
    for a, b in zip(back.partitions, parts):
        assert np.array_equal(a, b)
    for a, b in zip(back.payload, payload):
        assert np.array_equal(a, b)
    non = idx.as_layout("non_owning", base=vs.EmbeddingColumn(data))
    vs.save_index(non, tmp_path / "b.idx")
    back = vs.load_index(tmp_path / "b.idx", base=vs.EmbeddingColumn(data))
    assert back.layout == "non_owning" and back.base is not None
    assert non.nbytes() < idx.nbytes()


def test_svix_bad_magic(tmp_path):
    p = tmp_path / "junk.idx"
    p.write_bytes(b"NOPE" + b"\0" * 32)
    with pytest.raises(vs.ParameterError):
        vs.load_index(p)


def _sides():
    rng = np.random.default_rng(0)
    data = vs.EmbeddingColumn(rng.standard_normal((120, 8)).astype(np.float32))
    dt = Table(Schema([("did", "int64"), ("part", "int64"), ("e", embedding(8))]),
               {"did": np.arange(120), "part": np.arange(120) % 30, "e": data})
    qt = Table(Schema([("qid", "int64"), ("e", embedding(8))]),
               {"qid": np.arange(3), "e": vs.EmbeddingColumn(data.values[[5, 50, 100]])})
    return qt, dt


def test_operator_schema_errors_raise_before_search():
    qt, dt = _sides()
    with pytest.raises(vs.SchemaError):
        vector_search_operator(qt, "qid", dt, "e", vs.SearchParams(k=1))
    with pytest.raises(vs.SchemaError):
        vector_search_operator(qt, "nope", dt, "e", vs.SearchParams(k=1))
    with pytest.raises(vs.CapExceededError):
        vector_search_operator(qt, "e", dt, "e", vs.SearchParams(k=10, k_prime=5000),
                               device="device", gpu_topk_cap=2048)


def _vs_output_from_oracle():
    qt, dt = _sides()
    r = O.enn_search(qt.column("e").values, dt.column("e").values, 4)
    nt = NeighborTable(r.query_row, r.data_row, r.distance, r.rank, 3, "squared_l2", r.visited_rows)
    return build_vs_output(nt, qt, dt)


def test_build_vs_output_layout():
    out = _vs_output_from_oracle()
    assert out.schema.names == ["qid", "e", "did", "part", "e_d", "vs_distance", "vs_rank",
                                "vs_query_row", "vs_data_row"]
    first = np.asarray(out.column("did"))[np.asarray(out.column("vs_rank")) == 0]
    assert list(first) == [5, 50, 100]


def test_postfilter_semantics():
    out = _vs_output_from_oracle()
    kept, short = oversample_postfilter(out, None, 2)
    assert kept.row_count == 6 and short == {}
    kept, short = oversample_postfilter(out, "vs_rank >= 3", 3)
    assert kept.row_count == 3 and short == {0: 2, 1: 2, 2: 2}
    kept, _ = oversample_postfilter(out, "vs_data_row != 5", 1)
    q0 = np.asarray(kept.column("vs_data_row"))[np.asarray(kept.column("vs_query_row")) == 0]
    assert 5 not in q0.tolist()
    keep_set = Table.from_pairs([("p", "int64", [0, 1, 2, 3, 4])])
    kept, _ = oversample_postfilter(out, None, 2, keep_set=keep_set, semi_keys=("part", "p"))
    assert set(np.asarray(kept.column("part")).tolist()) <= {0, 1, 2, 3, 4}


def test_sharding_helpers():
    for n in (0, 1, 7, 10_000_001):
        for world in (1, 2, 3, 8):
            spans = [row_shard(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    sizes = np.random.default_rng(0).integers(1, 1000, 257)
    own = lpt_assign(sizes, 8)
    load = np.bincount(own, weights=sizes, minlength=8)
    assert load.max() - load.min() <= sizes.max()
    assert np.array_equal(own, lpt_assign(sizes, 8))  # deterministic on every rank
