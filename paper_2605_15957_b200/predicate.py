"""Relational filters evaluated on the GPU straight into the packed row bitmap
that `enn_search` / `IvfIndex.search` take as `row_filter` (the
step before the search; the paper finds the relational side gains most from
the GPU).

- `compare(values, op, value, valid=None)`: a comparison predicate with the
  reference's `eval_predicate` semantics (expr.py:568-576): rows where the
  predicate is valid and true, numpy comparison rules.
- `isin(keys, set, valid=None)`: semi-join membership (relops.py:88-113):
  rows whose key occurs in `set`; null keys never match.
- `bitmap_and / bitmap_or / bitmap_andnot`: combine bitmaps.

Inputs may be numpy arrays or CUDA tensors; the result is a CUDA int32 tensor
of packed LSB-first words when any input is on the GPU, else a numpy uint32
array.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .errors import ParameterError

_OPS = {"<": 0, "<=": 1, "==": 2, "=": 2, "!=": 3, "<>": 3, ">=": 4, ">": 5}


def _vtype(x):
    dt = str(x.dtype).replace("torch.", "")
    table = {"int32": 0, "int64": 1, "float32": 2, "float64": 3}
    if dt not in table:
        raise ParameterError(f"unsupported predicate column dtype {dt}")
    return table[dt]


def _out_words(n, like_cuda, device=None):
    nw = (n + 31) // 32
    if like_cuda:
        import torch
        return torch.empty(nw, dtype=torch.int32, device=device)
    return np.empty(nw, np.uint32)


def _contig(x):
    if N.is_torch(x):
        return x.contiguous()
    return np.ascontiguousarray(x)


def _is_cuda(*xs):
    return any(N.is_torch(x) and x.is_cuda for x in xs if x is not None)


def _device_of(*xs):
    for x in xs:
        if N.is_torch(x) and x.is_cuda:
            return x.device
    return None


def compare(values, op: str, value, valid=None, device=None):
    """Packed bitmap of `values <op> value` (rows that are also valid)."""
    from .vecindex import _ctx, _Stream
    if op not in _OPS:
        raise ParameterError(f"unknown comparison {op!r}")
    v = _contig(values)
    n = int(v.shape[0])
    cuda = _is_cuda(v, valid)
    out = _out_words(n, cuda, _device_of(v, valid))
    ctx = _ctx(device)
    with _Stream(ctx, v, valid, out):
        N.check(N.load().vs_bitmap_compare(ctx.handle, N.ptr(v), _vtype(v), n, _OPS[op], float(value),
                                           N.ptr(None if valid is None else _contig(valid)), N.ptr(out)),
                "bitmap_compare")
    return out


def isin(keys, values_set, valid=None, device=None):
    """Packed bitmap of rows whose int64 key occurs in `values_set`."""
    from .vecindex import _ctx, _Stream
    k = _contig(keys)
    s = _contig(values_set)
    if str(k.dtype).replace("torch.", "") != "int64" or str(s.dtype).replace("torch.", "") != "int64":
        raise ParameterError("isin keys and set must be int64")
    n = int(k.shape[0])
    cuda = _is_cuda(k, s, valid)
    out = _out_words(n, cuda, _device_of(k, s, valid))
    ctx = _ctx(device)
    with _Stream(ctx, k, s, valid, out):
        N.check(N.load().vs_bitmap_isin(ctx.handle, N.ptr(k), n,
                                        N.ptr(None if valid is None else _contig(valid)),
                                        N.ptr(s), int(s.shape[0]), N.ptr(out)), "bitmap_isin")
    return out


def _combine(a, b, op, device=None):
    from .vecindex import _ctx, _Stream
    a, b = _contig(a), _contig(b)
    if a.shape != b.shape:
        raise ParameterError("bitmaps differ in length")
    nw = int(a.shape[0])
    cuda = _is_cuda(a, b)
    if cuda:
        import torch
        out = torch.empty(nw, dtype=torch.int32, device=_device_of(a, b))
    else:
        out = np.empty(nw, np.uint32)
    ctx = _ctx(device)
    with _Stream(ctx, a, b, out):
        N.check(N.load().vs_bitmap_combine(ctx.handle, N.ptr(a), N.ptr(b), nw, op, N.ptr(out)), "bitmap_combine")
    return out


def bitmap_and(a, b, device=None):
    return _combine(a, b, 0, device)


def bitmap_or(a, b, device=None):
    return _combine(a, b, 1, device)


def bitmap_andnot(a, b, device=None):
    return _combine(a, b, 2, device)
