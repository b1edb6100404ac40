"""Vector-search entry points with the reference API (vecindex.py), executed
by the sm_100a kernels behind the C ABI.

Mirrors, name for name:
  SearchParams            vecindex.py:46-67
  NeighborTable           vecindex.py:70-88
  enn_search              vecindex.py:109-132
  FlatIndex               vecindex.py:138-162
  IvfIndex                vecindex.py:168-270 (build = GPU k-means with the
                          reference's Lloyd semantics, vecindex.py:273-318)
  save_index/load_index   vecindex.py:495-579 (SVIX, byte-identical)

Extension (the north star's pre-filter input): `row_filter=` on enn_search /
FlatIndex.search / IvfIndex.search — a bool mask over base rows, a packed
uint32 bitmap (LSB-first), or an ascending int64 selection vector. Results
then carry BASE row ids, identical to the reference composition
`rows = flatnonzero(mask); nt = enn_search(Q, base[rows]); rows[nt.data_row]`.

Every search runs on the GPU, for any k' (there is no host fallback): k' up to
vs_topk_cap() = 2048 uses the candidate-buffer kernels, larger k' (e.g. the
reference's k' = 500 k oversampling, plans.py:256) the device-wide select /
re-rank of vs_wide.cu. CapExceededError is the operator's placement contract
(vecsearch.py:86-87), raised by `vector_search_operator` only.
"""

from __future__ import annotations

import ctypes as C
import struct
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N
from .errors import EmptyInputError, ParameterError, ShapeError
from .table import EmbeddingColumn

SQUARED_L2 = "squared_l2"
INNER_PRODUCT = "inner_product"
METRICS = (SQUARED_L2, INNER_PRODUCT)
OWNING = "owning"
NON_OWNING = "non_owning"
KMEANS_MAX_ITERS = 20


def check_metric(metric: str) -> str:
    if metric not in METRICS:
        raise ParameterError(f"unknown metric {metric!r}")
    return metric


@dataclass
class SearchParams:
    """Search-time knobs. k_prime defaults to k; ef defaults to k_prime."""

    k: int
    k_prime: Optional[int] = None
    nprobe: int = 1
    ef: Optional[int] = None

    def __post_init__(self):
        if self.k < 1:
            raise ParameterError(f"k must be >= 1, got {self.k}")
        if self.k_prime is None:
            self.k_prime = self.k
        if self.k_prime < self.k:
            raise ParameterError(f"k' ({self.k_prime}) must be >= k ({self.k})")
        if self.nprobe < 1:
            raise ParameterError("nprobe must be >= 1")
        if self.ef is None:
            self.ef = self.k_prime
        if self.ef < self.k_prime:
            raise ParameterError(f"ef ({self.ef}) must be >= k' ({self.k_prime})")


@dataclass
class NeighborTable:
    """Per-query top neighbors: flat arrays sorted by (query_row, rank)."""

    query_row: np.ndarray
    data_row: np.ndarray
    distance: np.ndarray
    rank: np.ndarray
    n_queries: int
    metric: str
    visited_rows: int = 0
    probes: Optional[np.ndarray] = field(default=None, repr=False, compare=False)

    def __len__(self) -> int:
        return len(self.query_row)

    def per_query_counts(self) -> np.ndarray:
        counts = np.zeros(self.n_queries, dtype=np.int64)
        np.add.at(counts, self.query_row, 1)
        return counts

    @classmethod
    def from_padded(cls, ids, dist, counts, metric, visited, probes=None) -> "NeighborTable":
        """Flatten [nq, k] padded device outputs into the reference layout."""
        nq, k = ids.shape
        counts = counts.astype(np.int64)
        mask = np.arange(k)[None, :] < counts[:, None]
        qr = np.repeat(np.arange(nq, dtype=np.int64), counts)
        rank = np.broadcast_to(np.arange(k, dtype=np.int64), (nq, k))[mask]
        return cls(qr, ids[mask].astype(np.int64), dist[mask].astype(np.float64), rank, nq,
                   metric, int(visited), probes)


# ---- argument plumbing -----------------------------------------------------------------------

_dev_cols = weakref.WeakKeyDictionary()  # duck-typed (reference) columns -> {device: DeviceColumn}


def _ctx(device=None) -> N.Context:
    if isinstance(device, N.Context):   # an explicit context (several per device are allowed)
        return device
    return N.Context.get(device)


def _group(device):
    """The device group a search runs on: an explicit DeviceGroup, or the
    default set by group.use_devices() when no device is named."""
    from .group import DeviceGroup, default_group
    if isinstance(device, DeviceGroup):
        return device
    if device is None:
        return default_group()
    return None


def _into(out, res):
    """Copy a group search's host result into caller-provided buffers."""
    if out is None:
        return res
    for dst, src in zip(out, res[:3]):
        if N.is_torch(dst):
            import torch
            dst.copy_(torch.from_numpy(src))
        else:
            dst[...] = src
    return tuple(out) + tuple(res[3:])


def _dims(col):
    return int(col.count), int(col.dim)


def device_column(col, ctx: N.Context) -> N.DeviceColumn:
    """The (cached) device copy of an embedding column. A borrowed device (or
    pinned host) tensor that was modified in place since its last use gets its
    cached norms dropped (EmbeddingColumn.invalidate() does it explicitly)."""
    if isinstance(col, EmbeddingColumn):
        dc = col._device.get(ctx.device)
        if dc is not None:
            dc.refresh()
        if dc is None:
            if col._host_stream is not None:
                t = col._host_stream
                dt = N.DTYPE_BF16 if col.storage_dtype == "bfloat16" else N.DTYPE_F32
                dc = N.DeviceColumn(ctx, t.data_ptr(), col.count, col.dim, dt, host=True, keepalive=t)
            elif col._dev_tensor is not None:
                t = col._dev_tensor
                dt = N.DTYPE_BF16 if col.storage_dtype == "bfloat16" else N.DTYPE_F32
                dc = N.DeviceColumn(ctx, t.data_ptr(), col.count, col.dim, dt, borrow=True, keepalive=t)
            else:
                dc = N.DeviceColumn(ctx, col.values, col.count, col.dim, N.DTYPE_F32)
            col._device[ctx.device] = dc
        return dc
    values = np.ascontiguousarray(np.asarray(col.values, dtype=np.float32))
    cache = _dev_cols.get(col.values) if _weakrefable(col.values) else None
    if cache is not None and ctx.device in cache:
        return cache[ctx.device]
    dc = N.DeviceColumn(ctx, values, values.shape[0], values.shape[1], N.DTYPE_F32)
    if _weakrefable(col.values):
        _dev_cols.setdefault(col.values, {})[ctx.device] = dc
    return dc


def _weakrefable(x) -> bool:
    try:
        weakref.ref(x)
        return True
    except TypeError:
        return False


def _as_column(x) -> EmbeddingColumn:
    if N.is_torch(x):
        if x.is_cuda:
            return EmbeddingColumn.from_device(x)
        return EmbeddingColumn(x.float().numpy())
    if isinstance(x, EmbeddingColumn) or (hasattr(x, "values") and isinstance(getattr(x, "dim", None), int)):
        return x
    return EmbeddingColumn(np.asarray(x, dtype=np.float32))


def _query_buffer(queries):
    """(buffer, nq, d) for the C ABI: CUDA tensors pass through (device
    pointers), everything else becomes a C-contiguous float32 host array."""
    if N.is_torch(queries):
        import torch
        q = queries
        if q.dtype != torch.float32:
            q = q.float()
        q = q.contiguous()
        return q, int(q.shape[0]), int(q.shape[1])
    if isinstance(queries, EmbeddingColumn) and queries._dev_tensor is not None:
        q = queries._dev_tensor.float().contiguous()
        return q, queries.count, queries.dim
    vals = queries.values if hasattr(queries, "values") else queries
    q = np.ascontiguousarray(np.asarray(vals, dtype=np.float32))
    if q.ndim != 2:
        raise ShapeError("queries must be 2-D")
    return q, q.shape[0], q.shape[1]


def pack_bitmap(mask) -> np.ndarray:
    mask = np.asarray(mask, bool)
    n = mask.size
    padded = np.zeros((n + 31) // 32 * 32, bool)
    padded[:n] = mask
    bits = np.packbits(padded.reshape(-1, 8), axis=1, bitorder="little").reshape(-1)
    return bits.view(np.uint32).copy() if bits.size else np.zeros(0, np.uint32)


def filter_bitmap(row_filter, n: int):
    """Normalise a row filter to a packed LSB-first uint32 bitmap over n rows."""
    if row_filter is None:
        return None
    if N.is_torch(row_filter):
        import torch
        t = row_filter
        if t.dtype == torch.bool:
            raise ParameterError("pass device filters as packed int32/uint32 bitmaps")
        if t.numel() != (n + 31) // 32:
            raise ShapeError(f"bitmap has {t.numel()} words, expected {(n + 31) // 32}")
        return t.contiguous()
    arr = np.asarray(row_filter)
    if arr.dtype == bool:
        if arr.shape != (n,):
            raise ShapeError(f"row filter mask has shape {arr.shape}, expected ({n},)")
        return pack_bitmap(arr)
    if arr.dtype == np.uint32:
        if arr.size != (n + 31) // 32:
            raise ShapeError(f"bitmap has {arr.size} words, expected {(n + 31) // 32}")
        return np.ascontiguousarray(arr)
    if np.issubdtype(arr.dtype, np.integer):
        rows = arr.astype(np.int64)
        if rows.size and (rows.min() < 0 or rows.max() >= n):
            raise ParameterError("selection vector out of range")
        mask = np.zeros(n, bool)
        mask[rows] = True
        return pack_bitmap(mask)
    raise ParameterError(f"unsupported row filter dtype {arr.dtype}")


class _Stream:
    """Run library calls on torch's current stream when CUDA tensors are
    involved, so caller-produced device buffers are ordered correctly."""

    def __init__(self, ctx, *bufs):
        self.ctx = ctx
        self.on = any(N.is_torch(b) and b.is_cuda for b in bufs if b is not None)

    def __enter__(self):
        if self.on:
            import torch
            # torch's default stream has handle 0, which the ABI reads as "the
            # library's own stream": pass cudaStreamLegacy (0x1) instead, so the
            # library is ordered after torch's pending work (e.g. non_blocking
            # host->device copies of the inputs)
            self.ctx.set_stream(torch.cuda.current_stream(self.ctx.device).cuda_stream or 1)
        return self

    def __exit__(self, *exc):
        if self.on:
            self.ctx.set_stream(None)


def _outputs(nq, k, like=None):
    return (np.empty((nq, k), np.int64), np.empty((nq, k), np.float64), np.empty(nq, np.int32))


# ---- exhaustive search -------------------------------------------------------------------------


def enn_search_raw(queries, data, k: int, metric: str = SQUARED_L2, row_filter=None,
                   id_offset: int = 0, device=None, out=None):
    """Padded device-layout search: returns (ids [nq,k], dist [nq,k],
    counts [nq], visited). `out` may supply (ids, dist, counts) buffers
    (host numpy, pinned or CUDA torch tensors)."""
    check_metric(metric)
    grp = _group(device)
    if grp is not None:
        if int(k) < 1:
            raise ParameterError(f"k must be >= 1, got {k}")
        res = grp.enn_search_raw(queries, data, int(k), metric, row_filter)
        return _into(out, res)
    ctx = _ctx(device)
    data = _as_column(data)
    n, d = _dims(data)
    q, nq, qd = _query_buffer(queries)
    if qd != d:
        raise ShapeError(f"query dim {qd} != data dim {d}")
    if n == 0:
        raise EmptyInputError("exhaustive search over empty data side")
    if k < 1:
        raise ParameterError(f"k must be >= 1, got {k}")
    bm = filter_bitmap(row_filter, n)
    dc = device_column(data, ctx)
    ids, dist, cnt = out if out is not None else _outputs(nq, k)
    visited = C.c_int64(0)
    with _Stream(ctx, q, bm, ids):
        N.check(N.load().vs_enn_search(ctx.handle, dc.handle, N.ptr(q), nq, d, N.ptr(bm),
                                       n if bm is not None else 0, int(k), N.METRIC_CODE[metric],
                                       int(id_offset), N.ptr(ids), N.ptr(dist), N.ptr(cnt),
                                       C.byref(visited)), "enn_search")
    return ids, dist, cnt, visited.value


def enn_search(queries, data, params: SearchParams, metric: str = SQUARED_L2,
               row_filter=None, device=None) -> NeighborTable:
    """Exhaustive top-k' per query; exact by construction (vecindex.py:109-132).

    Distances are the reference's float64 values bit for bit; ids follow the
    tie rule. With `row_filter`, only selected base rows are candidates and
    data_row holds base row ids."""
    check_metric(metric)
    qcol = _as_column(queries)
    data = _as_column(data)
    if qcol.dim != data.dim:
        raise ShapeError(f"query dim {qcol.dim} != data dim {data.dim}")
    if data.count == 0:
        raise EmptyInputError("exhaustive search over empty data side")
    k = int(params.k_prime)
    if qcol.count == 0:
        return NeighborTable(np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0, np.float64),
                             np.empty(0, np.int64), 0, metric, 0)
    ids, dist, cnt, visited = enn_search_raw(qcol, data, k, metric, row_filter, device=device)
    return NeighborTable.from_padded(ids, dist, cnt, metric, visited)


@dataclass
class FlatIndex:
    """A non-owning handle over a base embedding column; search is exact."""

    base: Optional[EmbeddingColumn]
    dim: int
    count: int
    metric: str = SQUARED_L2

    @classmethod
    def build(cls, data, metric: str = SQUARED_L2) -> "FlatIndex":
        check_metric(metric)
        data = _as_column(data)
        return cls(data, data.dim, data.count, metric)

    def search(self, queries, params: SearchParams, row_filter=None) -> NeighborTable:
        if self.base is None:
            raise ParameterError("flat index has no attached base column")
        return enn_search(queries, self.base, params, self.metric, row_filter=row_filter)

    @property
    def layout(self) -> str:
        return NON_OWNING

    def structure_nbytes(self) -> int:
        return 0


# ---- IVF ------------------------------------------------------------------------------------------


@dataclass
class IvfIndex:
    """Inverted-file index: k-means partitions probed nearest-first.

    Partition assignment and probe ordering always use squared L2 against the
    float32 centroids; the index metric only ranks candidates. On the GPU the
    lists live in the compacted list-contiguous layout (owning) whatever the
    host-side layout; both layouts return identical results."""

    nlist: int
    dim: int
    count: int
    metric: str
    layout: str
    centroids: np.ndarray
    partitions: list
    payload: Optional[list] = None
    base: Optional[EmbeddingColumn] = None
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    @classmethod
    def build(cls, data, nlist: int, metric: str = SQUARED_L2, seed: int = 0,
              layout: str = OWNING, max_iters: int = KMEANS_MAX_ITERS, device=None) -> "IvfIndex":
        """GPU Lloyd's k-means with the reference semantics (vecindex.py:186-207,
        273-318): seeded sorted uniform init, <= 20 iterations or max centroid
        shift < 1e-4, first-min assignment, empty lists reseeded to the
        farthest member of the largest list, float64 means, float32 centroids,
        ascending row ids per list."""
        check_metric(metric)
        if layout not in (OWNING, NON_OWNING):
            raise ParameterError(f"unknown layout {layout!r}")
        data = _as_column(data)
        if nlist < 1 or nlist > data.count:
            raise ParameterError(f"nlist must be in [1, {data.count}], got {nlist}")
        ctx = _ctx(device)
        dc = device_column(data, ctx)
        # the reference's initial rows, drawn exactly as vecindex.py:276-279
        init = np.ascontiguousarray(np.sort(np.random.default_rng(seed).choice(
            data.count, size=nlist, replace=False)).astype(np.int64))
        h = C.c_void_p()
        N.check(N.load().vs_ivf_build(ctx.handle, dc.handle, int(nlist), N.ptr(init),
                                      int(seed) & (2**64 - 1), N.METRIC_CODE[metric], int(max_iters),
                                      C.byref(h)), "ivf_build")
        div = N.DeviceIvf(ctx, h)
        centroids = np.empty((nlist, data.dim), np.float32)
        sizes = np.empty(nlist, np.int64)
        ids = np.empty(div.n_total, np.int64)
        N.check(N.load().vs_ivf_export(h, N.ptr(centroids), N.ptr(sizes), N.ptr(ids), None))
        partitions = np.split(ids, np.cumsum(sizes)[:-1]) if nlist > 1 else [ids]
        idx = cls(nlist, data.dim, data.count, metric, layout, centroids, partitions,
                  None, base=data)
        idx._dev[ctx.device] = div
        if layout == OWNING:
            idx.payload = _LazyPayload(idx)
            idx.base = None
        return idx

    @classmethod
    def from_device_lists(cls, centroids, list_sizes, list_ids, payload, metric: str = SQUARED_L2,
                          device=None, count: Optional[int] = None) -> "IvfIndex":
        """Owning index over a caller-owned CUDA tensor holding the
        list-contiguous payload ([n_total, dim] float32 or bfloat16, the SVIX
        owning layout), borrowed without a copy (vs_ivf_wrap): for collections
        that fill most of HBM. The tensor must outlive the index."""
        import torch
        check_metric(metric)
        if not (N.is_torch(payload) and payload.is_cuda and payload.dim() == 2 and payload.is_contiguous()):
            raise ParameterError("payload must be a contiguous 2-D CUDA tensor")
        dt = {torch.float32: N.DTYPE_F32, torch.bfloat16: N.DTYPE_BF16}.get(payload.dtype)
        if dt is None:
            raise ParameterError("payload must be float32 or bfloat16")
        cen = np.ascontiguousarray(centroids, np.float32)
        nlist, dim = cen.shape
        sizes = np.ascontiguousarray(list_sizes, np.int64)
        ids = np.ascontiguousarray(list_ids, np.int64) if not N.is_torch(list_ids) else list_ids.contiguous()
        if sizes.shape != (nlist,) or int(sizes.sum()) != payload.shape[0] or payload.shape[1] != dim:
            raise ShapeError("list sizes / payload / centroid shapes disagree")
        ctx = _ctx(device)
        h = C.c_void_p()
        N.check(N.load().vs_ivf_wrap(ctx.handle, N.ptr(cen), int(nlist), int(dim), N.ptr(sizes), N.ptr(ids),
                                     payload.data_ptr(), dt, N.METRIC_CODE[metric], C.byref(h)), "ivf_wrap")
        div = N.DeviceIvf(ctx, h)
        div._keepalive = payload
        ids_h = ids.cpu().numpy() if N.is_torch(ids) else ids
        partitions = np.split(ids_h, np.cumsum(sizes)[:-1]) if nlist > 1 else [ids_h]
        if count is None:   # base rows (a list shard may hold only some of them)
            count = int(ids_h.max()) + 1 if ids_h.size else 0
        idx = cls(int(nlist), int(dim), count, metric, OWNING, cen, partitions, None, base=None)
        idx.payload = _LazyPayload(idx)
        idx._dev[ctx.device] = div
        return idx

    def assign(self, data, device=None):
        """Nearest list of every row of `data` (squared L2 to the centroids,
        the build's assignment step, vecindex.py:303-304) as int32; a CUDA
        tensor for device columns, else numpy. For indexes trained on a sample."""
        ctx = _ctx(device)
        data = _as_column(data)
        if data.dim != self.dim:
            raise ShapeError(f"data dim {data.dim} != index dim {self.dim}")
        div = self.device_index(ctx)
        dc = device_column(data, ctx)
        if data._dev_tensor is not None:
            import torch
            out = torch.empty(data.count, dtype=torch.int32, device=data._dev_tensor.device)
        else:
            out = np.empty(data.count, np.int32)
        N.check(N.load().vs_ivf_assign(ctx.handle, div.handle, dc.handle, N.ptr(out)), "ivf_assign")
        return out

    def as_layout(self, layout: str, base=None) -> "IvfIndex":
        """A view of the same build in the other layout; results are identical."""
        if layout == self.layout:
            return self
        if layout == OWNING:
            if base is None and self.base is None:
                raise ParameterError("owning view needs the base column")
            src = base if base is not None else self.base
            payload = [np.ascontiguousarray(src.values[p]) for p in self.partitions]
            return IvfIndex(self.nlist, self.dim, self.count, self.metric, OWNING,
                            self.centroids, self.partitions, payload)
        if base is None and self.payload is None:
            raise ParameterError("non-owning view needs the base column")
        if base is None:
            flat = np.empty((self.count, self.dim), np.float32)
            for p, block in zip(self.partitions, self.payload):
                flat[p] = block
            base = EmbeddingColumn(flat)
        return IvfIndex(self.nlist, self.dim, self.count, self.metric, NON_OWNING,
                        self.centroids, self.partitions, None, base=base)

    def device_index(self, ctx: N.Context, list_owned=None) -> N.DeviceIvf:
        """Device list-contiguous copy of this index (one per device). With
        `list_owned` (list sharding) the same copy scans only the
        owned lists; ownership is applied with vs_ivf_set_owned."""
        div = self._dev.get(ctx.device)
        if div is None:
            div = self._dev[ctx.device] = self._make_device_index(ctx)
        key = None if list_owned is None else bytes(np.ascontiguousarray(list_owned, np.uint8))
        if key is not None and len(key) != self.nlist:
            raise ShapeError(f"list_owned has {len(key)} entries, expected nlist={self.nlist}")
        if div.owned_key != key:
            owned = None if key is None else np.frombuffer(key, np.uint8).copy()
            N.check(N.load().vs_ivf_set_owned(div.handle, N.ptr(owned)), "ivf_set_owned")
            div.owned_key = key
        return div

    def _make_device_index(self, ctx: N.Context) -> N.DeviceIvf:
        sizes = np.array([len(p) for p in self.partitions], np.int64)
        ids = np.ascontiguousarray(np.concatenate(self.partitions).astype(np.int64)) \
            if self.partitions else np.empty(0, np.int64)
        cen = np.ascontiguousarray(self.centroids, np.float32)
        owned = None
        h = C.c_void_p()
        if self.layout == OWNING and self.payload is not None and not isinstance(self.payload, _LazyPayload):
            pay = np.ascontiguousarray(np.concatenate(self.payload, axis=0), np.float32) \
                if self.payload else np.empty((0, self.dim), np.float32)
            N.check(N.load().vs_ivf_create(ctx.handle, N.ptr(cen), self.nlist, self.dim, N.ptr(sizes),
                                           N.ptr(ids), N.ptr(pay), N.DTYPE_F32,
                                           N.METRIC_CODE[self.metric], None, N.ptr(owned),
                                           C.byref(h)), "ivf_create")
        else:
            if self.base is None:
                raise ParameterError("non-owning IVF index has no attached base column")
            dc = device_column(self.base, ctx)
            N.check(N.load().vs_ivf_create(ctx.handle, N.ptr(cen), self.nlist, self.dim, N.ptr(sizes),
                                           N.ptr(ids), None, dc.dtype, N.METRIC_CODE[self.metric],
                                           dc.handle, N.ptr(owned), C.byref(h)), "ivf_create")
        return N.DeviceIvf(ctx, h)

    def search(self, queries, params: SearchParams, row_filter=None, device=None,
               list_owned=None) -> NeighborTable:
        """IvfIndex.search (vecindex.py:230-258) on the GPU. Probes are the
        exact tie-rule top-nprobe centroids (returned in `.probes`); with
        `row_filter`, probed rows are intersected with the filter."""
        qcol = _as_column(queries)
        if qcol.dim != self.dim:
            raise ShapeError(f"query dim {qcol.dim} != index dim {self.dim}")
        if params.nprobe > self.nlist:
            raise ParameterError(f"nprobe {params.nprobe} > nlist {self.nlist}")
        if self.layout == NON_OWNING and self.base is None:
            raise ParameterError("non-owning IVF index has no attached base column")
        k = int(params.k_prime)
        if qcol.count == 0:
            return NeighborTable(np.empty(0, np.int64), np.empty(0, np.int64),
                                 np.empty(0, np.float64), np.empty(0, np.int64), 0, self.metric, 0)
        ids, dist, cnt, probes, visited = self.search_raw(qcol, k, params.nprobe, row_filter,
                                                          device=device, list_owned=list_owned)
        return NeighborTable.from_padded(ids, dist, cnt, self.metric, visited, probes)

    def search_raw(self, queries, k, nprobe, row_filter=None, device=None, list_owned=None,
                   out=None, want_probes=True, probes_in=None):
        """Padded device-layout search. `probes_in` ([nq, nprobe] int32, host
        or device) skips the coarse quantizer (multi-GPU query-sliced probing)."""
        grp = _group(device) if list_owned is None and probes_in is None else None
        if grp is not None:
            ids, dist, cnt, vis = grp.ivf_search_raw(self, queries, int(k), int(nprobe), row_filter)
            out = _into(out, (ids, dist, cnt))
            return out[0], out[1], out[2], None, vis
        ctx = _ctx(device)
        div = self.device_index(ctx, list_owned)
        q, nq, d = _query_buffer(queries)
        if d != self.dim:
            raise ShapeError(f"query dim {d} != index dim {self.dim}")
        bm = filter_bitmap(row_filter, self.count)
        ids, dist, cnt = out if out is not None else _outputs(nq, k)
        visited = C.c_int64(0)
        if probes_in is not None:
            with _Stream(ctx, q, bm, ids, probes_in):
                N.check(N.load().vs_ivf_search_probed(
                    ctx.handle, div.handle, N.ptr(q), nq, N.ptr(bm), self.count if bm is not None else 0,
                    int(nprobe), N.ptr(probes_in), int(k), N.ptr(ids), N.ptr(dist), N.ptr(cnt),
                    C.byref(visited)), "ivf_search_probed")
            return ids, dist, cnt, probes_in, visited.value
        probes = np.empty((nq, nprobe), np.int32) if want_probes else None
        with _Stream(ctx, q, bm, ids):
            N.check(N.load().vs_ivf_search(ctx.handle, div.handle, N.ptr(q), nq, N.ptr(bm),
                                           self.count if bm is not None else 0, int(nprobe), int(k),
                                           N.ptr(ids), N.ptr(dist), N.ptr(cnt), N.ptr(probes),
                                           C.byref(visited)), "ivf_search")
        return ids, dist, cnt, probes, visited.value

    def probe(self, queries, nprobe, device=None, out=None):
        """Coarse quantizer only: [nq, nprobe] int32 probed lists (exact
        tie-rule top-nprobe centroids, vecindex.py:238-243)."""
        ctx = _ctx(device)
        div = self.device_index(ctx)
        q, nq, d = _query_buffer(queries)
        if d != self.dim:
            raise ShapeError(f"query dim {d} != index dim {self.dim}")
        if out is None:
            if N.is_torch(q) and q.is_cuda:
                import torch
                out = torch.empty((nq, nprobe), dtype=torch.int32, device=q.device)
            else:
                out = np.empty((nq, nprobe), np.int32)
        with _Stream(ctx, q, out):
            N.check(N.load().vs_ivf_probe(ctx.handle, div.handle, N.ptr(q), nq, int(nprobe), N.ptr(out)),
                    "ivf_probe")
        return out

    def structure_nbytes(self) -> int:
        return self.centroids.nbytes

    def payload_nbytes(self) -> int:
        return self.count * self.dim * 4

    def nbytes(self) -> int:
        ids = self.count * 8
        if self.layout == OWNING:
            return self.structure_nbytes() + ids + self.payload_nbytes()
        return self.structure_nbytes() + ids


class _LazyPayload(list):
    """Owning payload of a GPU-built index, exported from the device on first
    access (per-list float32 blocks, vecindex.py:203-204)."""

    def __init__(self, idx: IvfIndex):
        super().__init__()
        self._idx = weakref.ref(idx)
        self._ready = False

    def _load(self):
        if self._ready:
            return
        idx = self._idx()
        div = next(iter(idx._dev.values()))
        flat = np.empty((div.n_total, idx.dim), np.float32 if div.dtype == N.DTYPE_F32 else np.uint16)
        N.check(N.load().vs_ivf_export(div.handle, None, None, None, N.ptr(flat)))
        if div.dtype != N.DTYPE_F32:
            flat = (flat.astype(np.uint32) << 16).view(np.float32)
        sizes = [len(p) for p in idx.partitions]
        blocks = np.split(flat, np.cumsum(sizes)[:-1]) if len(sizes) > 1 else [flat]
        super().extend(np.ascontiguousarray(b) for b in blocks)
        self._ready = True

    def __iter__(self):
        self._load()
        return super().__iter__()

    def __getitem__(self, i):
        self._load()
        return super().__getitem__(i)

    def __len__(self):
        self._load()
        return super().__len__()


# ---- SVIX serialisation (vecindex.py:495-579) ---------------------------------------------------

_MAGIC = b"SVIX"
_VERSION = 1
_KIND_CODE = {"flat": 0, "ivf": 1, "graph": 2}
_METRIC_CODE = {SQUARED_L2: 0, INNER_PRODUCT: 1}
_LAYOUT_CODE = {NON_OWNING: 0, OWNING: 1}


def _write_array(buf, arr, dtype: str):
    data = np.ascontiguousarray(arr, dtype=np.dtype(dtype))
    buf.write(struct.pack("<Q", data.size))
    buf.write(data.tobytes())


def _read_array(buf, dtype: str) -> np.ndarray:
    (size,) = struct.unpack("<Q", buf.read(8))
    raw = buf.read(size * np.dtype(dtype).itemsize)
    return np.frombuffer(raw, dtype=np.dtype(dtype)).copy()


def save_index(index, path) -> None:
    """Little-endian binary dump, byte-identical to the reference's writer."""
    if isinstance(index, FlatIndex):
        kind = "flat"
    elif isinstance(index, IvfIndex):
        kind = "ivf"
    else:
        raise ParameterError("only flat and IVF indexes are supported")
    with open(path, "wb") as f:
        f.write(_MAGIC)
        f.write(struct.pack("<HBBB", _VERSION, _KIND_CODE[kind], _METRIC_CODE[index.metric],
                            _LAYOUT_CODE[index.layout]))
        if kind == "flat":
            f.write(struct.pack("<IIQ", 0, index.dim, index.count))
        else:
            f.write(struct.pack("<IIQ", index.nlist, index.dim, index.count))
            _write_array(f, index.centroids, "<f4")
            _write_array(f, np.array([len(p) for p in index.partitions], np.int64), "<i8")
            _write_array(f, np.concatenate(index.partitions) if index.partitions
                         else np.empty(0, np.int64), "<i8")
            if index.layout == OWNING:
                _write_array(f, np.concatenate(list(index.payload), axis=0).reshape(-1), "<f4")


def load_index(path, base=None, device=None):
    """Load an index; non-owning layouts need the base column re-attached.

    device=None: the reference's host load (per-list numpy arrays). With a
    device (CUDA ordinal or library Context), an IVF file goes through the
    native loader (vs_ivf_load): its sections stream through one pinned
    double buffer straight into the device index (one contiguous copy per
    section); centroids and partitions are exported back
    for the host-side fields, the payload stays on the device (`.payload`
    exports it on first access)."""
    if device is not None:
        with open(path, "rb") as f:
            head = f.read(9)
        if len(head) == 9 and head[:4] == _MAGIC and head[6] == _KIND_CODE["ivf"]:
            return _load_ivf_device(path, base, device)
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != _MAGIC:
            raise ParameterError(f"not an index file: bad magic {magic!r}")
        version, kind_code, metric_code, layout_code = struct.unpack("<HBBB", f.read(5))
        if version != _VERSION:
            raise ParameterError(f"unsupported index file version {version}")
        kind = {v: k for k, v in _KIND_CODE.items()}[kind_code]
        metric = {v: k for k, v in _METRIC_CODE.items()}[metric_code]
        layout = {v: k for k, v in _LAYOUT_CODE.items()}[layout_code]
        p1, dim, count = struct.unpack("<IIQ", f.read(16))
        if kind == "flat":
            return FlatIndex(base, dim, count, metric)
        if kind != "ivf":
            raise ParameterError("graph indexes are outside the B200 operator's scope")
        centroids = _read_array(f, "<f4").reshape(p1, dim)
        sizes = _read_array(f, "<i8")
        flat_ids = _read_array(f, "<i8")
        partitions = np.split(flat_ids, np.cumsum(sizes)[:-1]) if p1 > 1 else [flat_ids]
        partitions = [np.ascontiguousarray(p) for p in partitions]
        payload = None
        if layout == OWNING:
            flat_payload = _read_array(f, "<f4").reshape(-1, dim)
            payload = [np.ascontiguousarray(b) for b in
                       (np.split(flat_payload, np.cumsum(sizes)[:-1]) if p1 > 1 else [flat_payload])]
        return IvfIndex(p1, dim, count, metric, layout, centroids, partitions, payload,
                        base=base if layout == NON_OWNING else None)


def _load_ivf_device(path, base, device):
    ctx = _ctx(device)
    info = np.zeros(6, np.int64)
    dc = device_column(_as_column(base), ctx) if base is not None else None
    h = C.c_void_p()
    N.check(N.load().vs_ivf_load(ctx.handle, str(path).encode(), dc.handle if dc is not None else None,
                                 N.ptr(info), C.byref(h)), "ivf_load")
    div = N.DeviceIvf(ctx, h)
    _, metric_code, layout_code, nlist, dim, count = (int(v) for v in info)
    metric = {v: k for k, v in _METRIC_CODE.items()}[metric_code]
    layout = {v: k for k, v in _LAYOUT_CODE.items()}[layout_code]
    centroids = np.empty((nlist, dim), np.float32)
    sizes = np.empty(nlist, np.int64)
    ids = np.empty(div.n_total, np.int64)
    N.check(N.load().vs_ivf_export(h, N.ptr(centroids), N.ptr(sizes), N.ptr(ids), None), "ivf_export")
    partitions = np.split(ids, np.cumsum(sizes)[:-1]) if nlist > 1 else [ids]
    idx = IvfIndex(nlist, dim, count, metric, layout, centroids, partitions, None,
                   base=_as_column(base) if layout == NON_OWNING and base is not None else None)
    idx._dev[ctx.device] = div
    if layout == OWNING:
        idx.payload = _LazyPayload(idx)
    return idx

