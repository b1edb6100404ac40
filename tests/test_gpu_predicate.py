"""GPU relational filters -> packed row bitmaps, against numpy (the
reference's eval_predicate, expr.py:568-576, and semi join, relops.py:88-113),
and the Vec-H config-1 filter (isin(rv_partkey, part[p_size <= 5])) built on
the GPU equals the reference-generated mask."""

import numpy as np
import pytest
import torch

from paper_2605_15957_b200 import predicate as P
from paper_2605_15957_b200.synth import pack_mask, unpack_bitmap

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.int32, np.int64, np.float32, np.float64])
@pytest.mark.parametrize("op", ["<", "<=", "==", "!=", ">=", ">"])
def test_compare_matches_numpy(dtype, op):
    rng = np.random.default_rng(3)
    n = 100_003
    v = (rng.integers(-50, 50, n)).astype(dtype)
    if np.issubdtype(dtype, np.floating):
        v[rng.random(n) < 0.01] = np.nan
    valid = rng.random(n) < 0.9
    ref = {"<": v < 7, "<=": v <= 7, "==": v == 7, "!=": v != 7, ">=": v >= 7, ">": v > 7}[op] & valid
    got = P.compare(v, op, 7, valid=pack_mask(valid))
    assert np.array_equal(unpack_bitmap(got, n), ref)
    got_d = P.compare(torch.from_numpy(v).cuda(), op, 7.0)
    ref_nv = {"<": v < 7, "<=": v <= 7, "==": v == 7, "!=": v != 7, ">=": v >= 7, ">": v > 7}[op]
    assert np.array_equal(unpack_bitmap(got_d.cpu().numpy().view(np.uint32), n), ref_nv)


def test_isin_and_combine_match_numpy():
    rng = np.random.default_rng(4)
    keys = rng.integers(-10**12, 10**12, 200_000).astype(np.int64)
    s = np.concatenate([rng.choice(keys, 3000), rng.integers(-10**12, 10**12, 3000)]).astype(np.int64)
    valid = rng.random(keys.size) < 0.95
    got = P.isin(keys, s, valid=pack_mask(valid))
    ref = np.isin(keys, s) & valid
    assert np.array_equal(unpack_bitmap(got, keys.size), ref)
    other = rng.random(keys.size) < 0.5
    a, b = pack_mask(ref), pack_mask(other)
    assert np.array_equal(unpack_bitmap(P.bitmap_and(a, b), keys.size), ref & other)
    assert np.array_equal(unpack_bitmap(P.bitmap_or(a, b), keys.size), ref | other)
    assert np.array_equal(unpack_bitmap(P.bitmap_andnot(a, b), keys.size), ref & ~other)
    # empty set, empty key column
    assert not unpack_bitmap(P.isin(keys, np.empty(0, np.int64)), keys.size).any()
    assert P.isin(np.empty(0, np.int64), s).size == 0


def test_config1_filter_on_gpu_equals_reference_mask():
    from paper_2605_15957_b200 import synth
    spec = synth.Spec(sf=0.1, d_r=384, d_i=384, seed=42)
    pk = torch.from_numpy(synth.review_partkeys(spec)[:100_000].astype(np.int64)).cuda()
    sizes = torch.from_numpy(synth.part_sizes(spec).astype(np.int64)).cuda()
    small_bits = P.compare(sizes, "<=", 5)                       # part[p_size <= 5]
    small = torch.nonzero(torch.from_numpy(unpack_bitmap(small_bits.cpu().numpy().view(np.uint32),
                                                         sizes.numel())).cuda()).flatten() + 1
    bits = P.isin(pk, small.to(torch.int64))                      # semi join on p_partkey
    _, mask, _ = synth.config1()
    assert np.array_equal(unpack_bitmap(bits.cpu().numpy().view(np.uint32), 100_000), mask)
