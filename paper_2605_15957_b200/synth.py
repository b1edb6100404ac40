"""Synthetic Vec-H inputs: the reference's embedding law, restated.

The reference generates embeddings as a unit-normalised Gaussian mixture
(64 unit centres, noise 0.55) from seeded `SeedSequence([seed, stream])`
streams (datagen.py:149-158, 267-299) and query vectors as centres plus
0.3 x noise (datagen.py:316-327). This module restates exactly the pieces the
vector-search path needs — the part-size column (for the config-1 TPC-H
predicate), review/image row counts and partkeys, embeddings, centres and
query vectors — so the same arrays can be rebuilt bit-for-bit without the
relational generator. `tests/test_synth.py` pins it against hashes taken from
the reference.

For N >= 1e6 (configs 2-5) `mixture_chunked` regenerates the same law in
seeded chunks, and `device_mixture` draws the law on the GPU
with torch (plumbing only: the bench's synthetic collection).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PARTS_PER_SF = 200_000          # datagen.py:29
CUSTOMERS_PER_SF = 150_000      # datagen.py:31

_STREAMS = {name: i for i, name in enumerate(
    ["part", "supplier", "partsupp", "customer", "orders", "lineitem",
     "reviews", "images", "review_emb", "image_emb", "centers_r", "centers_i"])}


@dataclass(frozen=True)
class Spec:
    """DatasetSpec subset (datagen.py:54-80)."""

    sf: float = 0.01
    d_r: int = 64
    d_i: int = 64
    r_bar: float = 12.0
    i_bar: float = 4.0
    n_clusters: int = 64
    noise: float = 0.55
    seed: int = 42

    @property
    def n_parts(self) -> int:
        return max(1, round(self.sf * PARTS_PER_SF))

    @property
    def n_cust(self) -> int:
        return max(1, round(self.sf * CUSTOMERS_PER_SF))


def _rng(spec: Spec, stream: str) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([spec.seed, _STREAMS[stream]]))


def mixture(rng, centers, assignment, noise) -> np.ndarray:
    """datagen.py:153-158."""
    d = centers.shape[1]
    vecs = centers[assignment] + noise * rng.standard_normal((len(assignment), d))
    norms = np.linalg.norm(vecs, axis=1, keepdims=True)
    norms[norms == 0] = 1.0
    return (vecs / norms).astype(np.float32)


def centers(spec: Spec, kind: str) -> np.ndarray:
    """float64 unit centres (datagen.py:267-272)."""
    d = spec.d_r if kind == "review" else spec.d_i
    c = _rng(spec, "centers_r" if kind == "review" else "centers_i").standard_normal(
        (spec.n_clusters, d)).astype(np.float64)
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    return c


def part_sizes(spec: Spec) -> np.ndarray:
    """p_size per part (datagen.py:177-199: the part stream draws brand (2x),
    type (3x), container (2x) integers and retail uniforms before p_size)."""
    n = spec.n_parts
    rng = _rng(spec, "part")
    rng.integers(1, 6, n), rng.integers(1, 6, n)
    rng.integers(0, 6, n), rng.integers(0, 5, n), rng.integers(0, 5, n)
    rng.integers(0, 5, n), rng.integers(0, 8, n)
    rng.uniform(900.0, 2000.0, n)
    return rng.integers(1, 51, n).astype(np.int64)


def review_partkeys(spec: Spec) -> np.ndarray:
    """rv_partkey (datagen.py:274-279)."""
    rng = _rng(spec, "reviews")
    mu = np.log(spec.r_bar) - 0.5
    counts = np.maximum(0, np.round(rng.lognormal(mu, 1.0, spec.n_parts))).astype(np.int64)
    return np.repeat(np.arange(1, spec.n_parts + 1, dtype=np.int64), counts)


def image_partkeys(spec: Spec) -> np.ndarray:
    """im_partkey (datagen.py:289-292)."""
    rng = _rng(spec, "images")
    counts = np.maximum(0, np.round(rng.normal(spec.i_bar, 1.5, spec.n_parts))).astype(np.int64)
    return np.repeat(np.arange(1, spec.n_parts + 1, dtype=np.int64), counts)


def review_embeddings(spec: Spec) -> np.ndarray:
    """rv_embedding (datagen.py:281-287)."""
    n = len(review_partkeys(spec))
    rng = _rng(spec, "review_emb")
    cl = rng.integers(0, spec.n_clusters, n)
    return mixture(rng, centers(spec, "review"), cl, spec.noise)


def image_embeddings(spec: Spec) -> np.ndarray:
    """im_embedding (datagen.py:293-299)."""
    n = len(image_partkeys(spec))
    rng = _rng(spec, "image_emb")
    cl = rng.integers(0, spec.n_clusters, n)
    return mixture(rng, centers(spec, "image"), cl, spec.noise)


def query_vectors(spec: Spec, kind: str, n: int, seed: int) -> np.ndarray:
    """make_query_vectors (datagen.py:316-327)."""
    c = centers(spec, kind).astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(np.random.SeedSequence([spec.seed, 1000, seed]))
    which = rng.integers(0, len(c), n)
    return mixture(rng, c, which, 0.3 * spec.noise)


def config1(n_rows: int = 100_000):
    """BASELINE config 1: SF=0.1, d=384, first 100k reviews, bitmap
    isin(rv_partkey, part[p_size <= 5].p_partkey), 1k queries (seed 7)."""
    spec = Spec(sf=0.1, d_r=384, d_i=384, seed=42)
    emb = review_embeddings(spec)[:n_rows]
    pk = review_partkeys(spec)[:n_rows]
    small = np.flatnonzero(part_sizes(spec) <= 5) + 1
    mask = np.isin(pk, small)
    q = query_vectors(spec, "review", 1000, seed=7)
    return emb, mask, q


# --- large-N generators (configs 2-5) ------------------------------------------


def mixture_chunked(n: int, d: int, seed: int = 42, chunk: int = 1 << 18,
                    n_clusters: int = 64, noise: float = 0.55, start: int = 0,
                    stop: int | None = None) -> np.ndarray:
    """Rows [start, stop) of the mixture law regenerated in seeded chunks
    (SeedSequence([seed, 8, chunk_index]))."""
    stop = n if stop is None else stop
    c = np.random.default_rng(np.random.SeedSequence([seed, 10])).standard_normal((n_clusters, d))
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    out = np.empty((stop - start, d), np.float32)
    for ci in range(start // chunk, (stop + chunk - 1) // chunk):
        lo, hi = ci * chunk, min(n, (ci + 1) * chunk)
        rng = np.random.default_rng(np.random.SeedSequence([seed, 8, ci]))
        block = mixture(rng, c, rng.integers(0, n_clusters, hi - lo), noise)
        a, b = max(lo, start), min(hi, stop)
        out[a - start:b - start] = block[a - lo:b - lo]
    return out


def bernoulli_bitmap(n: int, p: float, seed: int = 42) -> np.ndarray:
    """Seeded Bernoulli(p) row filter packed LSB-first into uint32 words
    (bit i of word w <=> row 32*w + i)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 77]))
    mask = rng.random(n) < p
    return pack_mask(mask)


def pack_mask(mask) -> np.ndarray:
    mask = np.asarray(mask, bool)
    n = mask.size
    padded = np.zeros((n + 31) // 32 * 32, bool)
    padded[:n] = mask
    bits = np.packbits(padded.reshape(-1, 8), axis=1, bitorder="little").reshape(-1)
    return bits.view(np.uint32).copy() if bits.size else np.zeros(0, np.uint32)


def unpack_bitmap(words, n: int) -> np.ndarray:
    b = np.unpackbits(np.asarray(words, np.uint32).view(np.uint8), bitorder="little")
    return b[:n].astype(bool)


def device_mixture(n: int, d: int, seed: int = 42, device="cuda", dtype=None,
                   n_clusters: int = 64, noise: float = 0.55, chunk: int = 1 << 20):
    """The mixture law drawn on the GPU with torch (bench collections at
    N = 1e7..1e8 rows cannot be generated on the host in a bench budget)."""
    import torch

    dtype = dtype or torch.float32
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    c = torch.randn(n_clusters, d, generator=g, device=device, dtype=torch.float32)
    c /= c.norm(dim=1, keepdim=True)
    out = torch.empty(n, d, device=device, dtype=dtype)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        a = torch.randint(0, n_clusters, (hi - lo,), generator=g, device=device)
        v = c[a] + noise * torch.randn(hi - lo, d, generator=g, device=device)
        v /= v.norm(dim=1, keepdim=True)
        out[lo:hi] = v.to(dtype)
    return out, c


def device_queries(centers_t, n: int, seed: int = 7, noise: float = 0.55):
    import torch

    g = torch.Generator(device=centers_t.device)
    g.manual_seed(1000 + seed)
    a = torch.randint(0, centers_t.shape[0], (n,), generator=g, device=centers_t.device)
    v = centers_t[a] + 0.3 * noise * torch.randn(n, centers_t.shape[1], generator=g,
                                                 device=centers_t.device)
    v /= v.norm(dim=1, keepdim=True)
    return v.float().contiguous()


def device_rows(n: int, d: int, lo: int, hi: int, device, dtype=None, chunk: int = 1 << 20):
    """Rows [lo, hi) of the N-row bench collection (mixture law, 64 unit
    centres, noise 0.55, L2-normalised), drawn on the GPU in global 2^20-row
    chunks with per-chunk seeds: every row shard / world size sees the same
    global collection. dtype bfloat16 rounds each normalised chunk (config 4).
    Returns (rows, centres)."""
    import torch

    dtype = dtype or torch.float32
    g = torch.Generator(device=device)
    g.manual_seed(42)
    c = torch.randn(64, d, generator=g, device=device)
    c /= c.norm(dim=1, keepdim=True)
    out = torch.empty(hi - lo, d, device=device, dtype=dtype)
    for ci in range(lo // chunk, (hi + chunk - 1) // chunk):
        a, b = ci * chunk, min(n, (ci + 1) * chunk)
        gg = torch.Generator(device=device)
        gg.manual_seed(100_000 + ci)
        asg = torch.randint(0, 64, (b - a,), generator=gg, device=device)
        v = c[asg] + 0.55 * torch.randn(b - a, d, generator=gg, device=device)
        v /= v.norm(dim=1, keepdim=True)
        s_, e_ = max(a, lo), min(b, hi)
        out[s_ - lo:e_ - lo] = v[s_ - a:e_ - a].to(dtype)
    return out, c


def device_bernoulli(n: int, p: float, seed: int, device):
    """The bench filters: Bernoulli(p) row mask drawn on the GPU."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.rand(n, generator=g, device=device) < p


def pack_bits_torch(mask):
    """bool [n] -> packed uint32 words (LSB-first) as an int32 tensor."""
    import torch

    n = mask.numel()
    pad = (-n) % 32
    if pad:
        mask = torch.cat([mask, torch.zeros(pad, dtype=torch.bool, device=mask.device)])
    w = mask.view(-1, 32).to(torch.int64)
    shifts = torch.arange(32, device=mask.device, dtype=torch.int64)
    words = (w << shifts).sum(dim=1)
    return (words - ((words >> 31) << 32)).to(torch.int32).contiguous()  # two's complement uint32

