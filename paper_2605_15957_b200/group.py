"""Several GPUs of one box driven from one process.

The reference executes its plans from a single interpreter
(executor.py:109-181), so the drop-in has to reach every GPU of the box
without torchrun. A `DeviceGroup` wraps `vs_group_*` (include/vs_b200.h):
one library context per device, an NCCL clique for distinct devices, and a
group search that runs every member's shard concurrently, all-gathers the
[Q, k] results (ncclAllGather) and merges them under the tie rule.

- Exact search: the collection is cut into contiguous row ranges (multiples
  of 32 rows, so the global bitmap slices by words), one per member.
- IVF: every member holds the same centroids (identical probes) and only the
  lists it owns (LPT by list size, distributed.lpt_assign); other lists are
  empty on that member.

`use_devices([0, 1, ...])` makes the group the default placement of
`enn_search` / `FlatIndex.search` / `IvfIndex.search` and therefore of
`vector_search_operator`: existing callers use every GPU unchanged.
Results are identical to the one-GPU search (per-pair arithmetic does not
depend on the shard)."""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _native as N
from .errors import ParameterError, ShapeError

_default = None


def use_devices(devices) -> "DeviceGroup | None":
    """Set (or with None / [] clear) the default device group of the searches."""
    global _default
    _default = DeviceGroup(devices) if devices else None
    return _default


def default_group():
    return _default


class DeviceGroup:
    def __init__(self, devices):
        devs = np.ascontiguousarray(np.asarray(list(devices), np.int32))
        if devs.size < 1:
            raise ParameterError("a device group needs at least one device")
        h = C.c_void_p()
        N.check(N.load().vs_group_create(int(devs.size), N.ptr(devs), C.byref(h)), "group_create")
        self.handle = h
        self.devices = [int(x) for x in devs]
        nd, nc = C.c_int32(0), C.c_int32(0)
        N.check(N.load().vs_group_info(h, C.byref(nd), C.byref(nc)))
        self.uses_nccl = bool(nc.value)
        self.members = [N.Context.borrowed(N.load().vs_group_ctx(h, i), d, owner=self)
                        for i, d in enumerate(self.devices)]
        self._cols = weakref.WeakKeyDictionary()   # column -> (shard DeviceColumns, row_lo)

    def __len__(self):
        return len(self.devices)

    def __del__(self):
        try:
            for m in getattr(self, "members", []):
                m._owner = None
                m.handle = None
            if getattr(self, "handle", None):
                N.load().vs_group_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    # ---- exact search over row shards ----------------------------------------------------------
    def row_ranges(self, n: int):
        """Contiguous, 32-row aligned ranges [lo_i, hi_i) covering n rows."""
        G = len(self)
        per = -(-n // G)
        per = -(-per // 32) * 32
        lo = [min(n, i * per) for i in range(G)]
        return lo, [min(n, x + per) for x in lo]

    def shard_column(self, col):
        """Per-member device copies of the column's row shards (cached)."""
        from .table import EmbeddingColumn
        from .vecindex import _as_column
        col = _as_column(col)
        hit = self._cols.get(col) if isinstance(col, EmbeddingColumn) else None
        if hit is not None:
            return hit
        lo, hi = self.row_ranges(col.count)
        shards = []
        for m, a, b in zip(self.members, lo, hi):
            if col._dev_tensor is not None:
                import torch
                t = col._dev_tensor[a:b].to(torch.device("cuda", m.device)).contiguous()
                dt = N.DTYPE_BF16 if t.dtype == torch.bfloat16 else N.DTYPE_F32
                shards.append(N.DeviceColumn(m, t.data_ptr(), b - a, col.dim, dt, borrow=True, keepalive=t))
            else:
                vals = np.ascontiguousarray(col.values[a:b], np.float32)
                shards.append(N.DeviceColumn(m, vals, b - a, col.dim, N.DTYPE_F32))
        res = (shards, np.asarray(lo, np.int64))
        if isinstance(col, EmbeddingColumn):
            self._cols[col] = res
        return res

    def enn_search_raw(self, queries, data, k: int, metric: str, row_filter=None):
        from .vecindex import _query_buffer, check_metric, filter_bitmap
        check_metric(metric)
        shards, lo = self.shard_column(data)
        n = int(sum(s.n for s in shards))
        q, nq, d = _query_buffer(queries)
        if N.is_torch(q):
            q = q.cpu().numpy()
        if d != shards[0].d:
            raise ShapeError(f"query dim {d} != data dim {shards[0].d}")
        bm = filter_bitmap(row_filter, n)
        if bm is not None and N.is_torch(bm):
            bm = bm.cpu().numpy().view(np.uint32)
        handles = (C.c_void_p * len(shards))(*[s.handle.value for s in shards])
        ids = np.empty((nq, k), np.int64)
        dist = np.empty((nq, k), np.float64)
        cnt = np.empty(nq, np.int32)
        vis = C.c_int64(0)
        N.check(N.load().vs_group_enn_search(self.handle, handles, N.ptr(lo), N.ptr(q), nq, d, N.ptr(bm),
                                             n if bm is not None else 0, int(k), N.METRIC_CODE[metric],
                                             N.ptr(ids), N.ptr(dist), N.ptr(cnt), C.byref(vis)), "group_enn_search")
        return ids, dist, cnt, vis.value

    # ---- IVF over list shards -------------------------------------------------------------------
    def shard_ivf(self, index):
        """Per-member index parts: same centroids, the LPT-owned lists' rows."""
        key = ("group", id(self))            # cached on the index (its _dev dict)
        hit = index._dev.get(key)
        if hit is not None:
            return hit
        from .distributed import lpt_assign
        sizes = np.array([len(p) for p in index.partitions], np.int64)
        owner = lpt_assign(sizes, len(self))
        cen = np.ascontiguousarray(index.centroids, np.float32)
        parts = []
        for r, m in enumerate(self.members):
            mine = owner == r
            msizes = np.where(mine, sizes, 0).astype(np.int64)
            plist = [index.partitions[l] for l in range(index.nlist) if mine[l]]
            ids = np.ascontiguousarray(np.concatenate(plist).astype(np.int64)) if plist else np.empty(0, np.int64)
            if index.payload is not None:
                pay = [np.asarray(index.payload[l], np.float32) for l in range(index.nlist) if mine[l]]
            else:
                vals = index.base.values
                pay = [vals[p] for p in plist]
            pay = np.ascontiguousarray(np.concatenate(pay, axis=0), np.float32) if pay else \
                np.empty((0, index.dim), np.float32)
            h = C.c_void_p()
            N.check(N.load().vs_ivf_create(m.handle, N.ptr(cen), index.nlist, index.dim, N.ptr(msizes), N.ptr(ids),
                                           N.ptr(pay), N.DTYPE_F32, N.METRIC_CODE[index.metric], None, None,
                                           C.byref(h)), "ivf_create")
            parts.append(N.DeviceIvf(m, h))
        index._dev[key] = parts
        return parts

    def ivf_search_raw(self, index, queries, k: int, nprobe: int, row_filter=None):
        from .vecindex import _query_buffer, filter_bitmap
        parts = self.shard_ivf(index)
        q, nq, d = _query_buffer(queries)
        if N.is_torch(q):
            q = q.cpu().numpy()
        if d != index.dim:
            raise ShapeError(f"query dim {d} != index dim {index.dim}")
        bm = filter_bitmap(row_filter, index.count)
        if bm is not None and N.is_torch(bm):
            bm = bm.cpu().numpy().view(np.uint32)
        handles = (C.c_void_p * len(parts))(*[p.handle.value for p in parts])
        ids = np.empty((nq, k), np.int64)
        dist = np.empty((nq, k), np.float64)
        cnt = np.empty(nq, np.int32)
        vis = C.c_int64(0)
        N.check(N.load().vs_group_ivf_search(self.handle, handles, N.ptr(q), nq, N.ptr(bm),
                                             index.count if bm is not None else 0, int(nprobe), int(k), N.ptr(ids),
                                             N.ptr(dist), N.ptr(cnt), C.byref(vis)), "group_ivf_search")
        return ids, dist, cnt, vis.value
