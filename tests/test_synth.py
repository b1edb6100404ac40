"""The synth restatement rebuilds the reference generator's arrays bit-for-bit
(hashes taken from the reference by tests/golden/make_golden.py)."""

import hashlib
import json
from pathlib import Path

import numpy as np

from paper_2605_15957_b200 import synth

META = json.loads((Path(__file__).parent / "golden" / "meta.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_sf001_arrays_match_reference(sf001):
    m = META["sf001"]
    sp = synth.Spec(sf=0.01)
    assert sha(sf001["reviews"]) == m["reviews"]
    assert sha(sf001["images"]) == m["images"]
    assert sha(sf001["review_partkeys"]) == m["review_partkeys"]
    assert sha(synth.image_partkeys(sp)) == m["image_partkeys"]
    assert sha(synth.part_sizes(sp)) == m["p_size"]
    assert sha(synth.query_vectors(sp, "review", 3, 7)) == m["q_review_seed7_n3"]


def test_config1_inputs_match_reference():
    m = META["config1"]
    emb, mask, q = synth.config1()
    assert sha(emb) == m["emb"]
    assert sha(mask) == m["mask"]
    assert sha(q) == m["queries"]
    assert int(mask.sum()) == m["n_sel"] == 10767


def test_bitmap_pack_roundtrip():
    rng = np.random.default_rng(0)
    for n in (0, 1, 31, 32, 33, 1000):
        m = rng.random(n) < 0.3
        w = synth.pack_mask(m)
        assert w.dtype == np.uint32 and w.size == (n + 31) // 32
        assert np.array_equal(synth.unpack_bitmap(w, n), m)
        # LSB-first: bit i of word w <=> row 32*w + i
        for i in np.flatnonzero(m)[:10]:
            assert (int(w[i // 32]) >> (i % 32)) & 1


def test_chunked_mixture_is_deterministic_and_sliceable():
    a = synth.mixture_chunked(5000, 8, chunk=1024)
    b = synth.mixture_chunked(5000, 8, chunk=1024, start=1500, stop=3100)
    assert np.array_equal(a[1500:3100], b)
    assert np.allclose(np.linalg.norm(a, axis=1), 1.0, atol=1e-5)
