"""The step after the search, on the GPU.

The searches leave their result in the padded per-query layout
(`enn_search_raw` / `IvfIndex.search_raw`: ids and float64 distances
`[nq, k']`, counts `[nq]`). The reference turns its NeighborTable into the
joined output table and post-filters it in numpy (vecsearch.py:123-202); here
the same steps run on the device so that only the final k rows per query
cross PCIe:

- `postfilter(...)` = `oversample_postfilter` (vecsearch.py:155-202): per
  query, the first k results in rank order that satisfy every keep condition —
  a data-row bitmap (data-side predicates, semi joins; build it with
  `predicate.compare` / `predicate.isin`), a per-result mask, and a cross-side
  key comparison (`data_key[data_row] <op> query_key[query]`, e.g. Q11's
  "im_imagekey_d != im_imagekey", plans.py:537). Shortfalls are reported, not
  raised.
- `flatten(...)` = the NeighborTable arrays (vecindex.py:95-106): query_row,
  data_row, distance, rank sorted by (query, rank).
- `gather_rows(src, idx)` and `build_vs_output(flat, query_cols, data_cols)` =
  `build_vs_output` (vecsearch.py:123-152) over dicts of columns, with the
  reference's `_d` renaming and the four vs_* columns.

Every input may be numpy or a CUDA tensor; results are CUDA tensors when any
input is on the GPU, else numpy arrays.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import ParameterError, SchemaError, ShapeError

VS_DISTANCE = "vs_distance"
VS_RANK = "vs_rank"
VS_QUERY_ROW = "vs_query_row"
VS_DATA_ROW = "vs_data_row"
_RESERVED = (VS_DISTANCE, VS_RANK, VS_QUERY_ROW, VS_DATA_ROW)
_OPS = {"<": 0, "<=": 1, "==": 2, "=": 2, "!=": 3, "<>": 3, ">=": 4, ">": 5}


def _is_cuda(x):
    return N.is_torch(x) and x.is_cuda


def _contig(x, np_dtype, torch_dtype):
    if x is None:
        return None
    if N.is_torch(x):
        if x.dtype != torch_dtype:
            x = x.to(torch_dtype)
        return x.contiguous()
    return np.ascontiguousarray(np.asarray(x, np_dtype))


def _empty(shape, np_dtype, cuda_device):
    if cuda_device is not None:
        import torch
        tdt = {np.int64: torch.int64, np.float64: torch.float64, np.int32: torch.int32}[np_dtype]
        return torch.empty(shape, dtype=tdt, device=cuda_device)
    return np.empty(shape, np_dtype)


def _cuda_device(*xs):
    for x in xs:
        if _is_cuda(x):
            return x.device
    return None


def _keep_bitmap(keep_rows, n_data):
    if keep_rows is None:
        return None
    from .vecindex import filter_bitmap
    if not N.is_torch(keep_rows) and np.asarray(keep_rows).dtype == bool:
        keep_rows = np.asarray(keep_rows)
        if n_data is None:
            n_data = keep_rows.shape[0]
    if n_data is None:
        raise ParameterError("n_data is required with a packed keep_rows bitmap")
    return filter_bitmap(keep_rows, int(n_data)), int(n_data)


def postfilter(ids, dist, counts, k: int, keep_rows=None, n_data=None, keep_pos=None,
               key_compare=None, device=None):
    """Per query the first k results (rank order) that satisfy every keep
    condition (vecsearch.py:155-202).

    `keep_rows`: bool mask / packed bitmap / selection over the data rows
    (`n_data` rows; required for a packed bitmap). `keep_pos`: bool per result
    slot `[nq, k']`. `key_compare`: `(data_key, op, query_key)` with op one of
    < <= == != >= >.

    Returns `(ids [nq,k], dist [nq,k], rank [nq,k] int32, count [nq] int32,
    shortfalls {query: missing})`; entries past `count` are unspecified."""
    from .vecindex import _ctx, _Stream
    if k < 1:
        raise ParameterError(f"k must be >= 1, got {k}")
    ids = _contig(ids, np.int64, _torch().int64) if N.is_torch(ids) else np.ascontiguousarray(ids, np.int64)
    if ids.ndim != 2:
        raise ShapeError("ids must be [nq, k']")
    nq, kp = int(ids.shape[0]), int(ids.shape[1])
    dist = _contig(dist, np.float64, _torch().float64) if N.is_torch(dist) else np.ascontiguousarray(dist, np.float64)
    if tuple(dist.shape) != (nq, kp):
        raise ShapeError("dist must match ids")
    if counts is not None:
        counts = _contig(counts, np.int32, _torch().int32) if N.is_torch(counts) else \
            np.ascontiguousarray(counts, np.int32)
    bm = None
    nd = 0 if n_data is None else int(n_data)
    if keep_rows is not None:
        bm, nd = _keep_bitmap(keep_rows, n_data)
    kpos = None
    if keep_pos is not None:
        kpos = keep_pos.to(_torch().uint8).contiguous() if N.is_torch(keep_pos) else \
            np.ascontiguousarray(np.asarray(keep_pos, bool).astype(np.uint8))
        if tuple(kpos.shape) != (nq, kp):
            raise ShapeError("keep_pos must be [nq, k']")
    dkey = qkey = None
    op = 0
    if key_compare is not None:
        dkey, opname, qkey = key_compare
        if opname not in _OPS:
            raise ParameterError(f"unknown comparison {opname!r}")
        op = _OPS[opname]
        dkey = _contig(dkey, np.int64, _torch().int64) if N.is_torch(dkey) else np.ascontiguousarray(dkey, np.int64)
        qkey = _contig(qkey, np.int64, _torch().int64) if N.is_torch(qkey) else np.ascontiguousarray(qkey, np.int64)
        if int(qkey.shape[0]) != nq:
            raise ShapeError("query_key must have one entry per query")
        if bm is not None and int(dkey.shape[0]) != nd:
            raise ShapeError("data_key and keep_rows disagree on the data row count")
        nd = int(dkey.shape[0])
    dev = _cuda_device(ids, dist, counts, bm, kpos, dkey, qkey)
    o_ids = _empty((nq, k), np.int64, dev)
    o_dist = _empty((nq, k), np.float64, dev)
    o_rank = _empty((nq, k), np.int32, dev)
    o_cnt = _empty(nq, np.int32, dev)
    ctx = _ctx(device)
    with _Stream(ctx, ids, dist, counts, bm, kpos, dkey, qkey, o_ids):
        N.check(N.load().vs_postfilter(ctx.handle, N.ptr(ids), N.ptr(dist), N.ptr(counts), nq, kp, N.ptr(bm),
                                       N.ptr(kpos), N.ptr(dkey), N.ptr(qkey), op, nd, int(k), N.ptr(o_ids),
                                       N.ptr(o_dist), N.ptr(o_rank), N.ptr(o_cnt)), "postfilter")
    cnt_h = o_cnt.cpu().numpy() if N.is_torch(o_cnt) else o_cnt
    # the reference reports shortfalls for the queries that had rows at all
    had = (np.full(nq, kp, np.int64) if counts is None else
           (counts.cpu().numpy() if N.is_torch(counts) else counts)) > 0
    short = {int(q): int(k - cnt_h[q]) for q in np.flatnonzero(had & (cnt_h < k))}
    return o_ids, o_dist, o_rank, o_cnt, short


def flatten(ids, dist, counts=None, rank=None, query_offset: int = 0, device=None):
    """The NeighborTable arrays from the padded layout (vecindex.py:95-106):
    dict of query_row, data_row, distance, rank (rank = `rank[q, j]` when
    given, e.g. postfilter's original ranks, else j)."""
    from .vecindex import _ctx, _Stream
    t = _torch() if any(N.is_torch(x) for x in (ids, dist, counts, rank)) else None
    ids = _contig(ids, np.int64, t and t.int64)
    dist = _contig(dist, np.float64, t and t.float64)
    counts = _contig(counts, np.int32, t and t.int32)
    rank = _contig(rank, np.int32, t and t.int32)
    nq, kp = int(ids.shape[0]), int(ids.shape[1])
    dev = _cuda_device(ids, dist, counts, rank)
    cap = max(nq * kp, 1)
    outs = [_empty(cap, np.int64, dev), _empty(cap, np.int64, dev), _empty(cap, np.float64, dev),
            _empty(cap, np.int64, dev)]
    n_out = C.c_int64(0)
    ctx = _ctx(device)
    with _Stream(ctx, ids, dist, counts, rank, outs[0]):
        N.check(N.load().vs_results_flatten(ctx.handle, N.ptr(ids), N.ptr(dist), N.ptr(rank), N.ptr(counts), nq,
                                            kp, int(query_offset), *(N.ptr(o) for o in outs),
                                            C.byref(n_out)), "results_flatten")
    r = int(n_out.value)
    return {VS_QUERY_ROW: outs[0][:r], VS_DATA_ROW: outs[1][:r], VS_DISTANCE: outs[2][:r], VS_RANK: outs[3][:r]}


def gather_rows(src, idx, device=None):
    """`src[idx]` along the first axis for any fixed-width column (scalars,
    bools, embeddings), on the device when either side is a CUDA tensor."""
    from .vecindex import _ctx, _Stream
    cuda = _is_cuda(src) or _is_cuda(idx)
    if cuda:
        import torch
        dev = src.device if _is_cuda(src) else idx.device
        s = src if N.is_torch(src) else torch.from_numpy(np.ascontiguousarray(src))
        s = s.to(dev).contiguous()
        i = (idx if N.is_torch(idx) else torch.from_numpy(np.asarray(idx, np.int64))).to(dev, torch.int64).contiguous()
        n = int(i.shape[0])
        dst = torch.empty((n,) + tuple(s.shape[1:]), dtype=s.dtype, device=dev)
        row_bytes = s.element_size() * (s[0].numel() if s.dim() > 1 else 1)
    else:
        s = np.ascontiguousarray(src.numpy() if N.is_torch(src) else src)
        i = np.ascontiguousarray(np.asarray(idx.numpy() if N.is_torch(idx) else idx, np.int64))
        n = int(i.shape[0])
        dst = np.empty((n,) + s.shape[1:], s.dtype)
        row_bytes = s.itemsize * (int(np.prod(s.shape[1:])) if s.ndim > 1 else 1)
    ctx = _ctx(device)
    with _Stream(ctx, s, i, dst):
        N.check(N.load().vs_gather_rows(ctx.handle, N.ptr(s), int(s.shape[0]), int(row_bytes), N.ptr(i), n,
                                        N.ptr(dst)), "gather_rows")
    return dst


def build_vs_output(flat: dict, query_cols: dict, data_cols: dict, device=None) -> dict:
    """The joined output of the vector-search operator (vecsearch.py:123-152)
    as an ordered dict of columns: every query column, every data column
    (renamed `<name>_d` on collision with a query column or a vs_* name),
    then vs_distance, vs_rank, vs_query_row, vs_data_row."""
    out = {}
    for name, col in query_cols.items():
        out[name] = gather_rows(col, flat[VS_QUERY_ROW], device)
    for name, col in data_cols.items():
        out_name = name + "_d" if (name in query_cols or name in _RESERVED) else name
        if out_name in out:
            raise SchemaError(f"data-side field {name!r} collides even after rename")
        out[out_name] = gather_rows(col, flat[VS_DATA_ROW], device)
    for name in (VS_DISTANCE, VS_RANK, VS_QUERY_ROW, VS_DATA_ROW):
        if name in out:
            raise SchemaError(f"input field {name!r} shadows a vs output column")
        out[name] = flat[name]
    return out


def _torch():
    import torch
    return torch
