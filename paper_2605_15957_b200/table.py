"""Columnar containers the operator boundary needs.

`EmbeddingColumn` mirrors the reference input type (table.py:91-141):
read-only C-contiguous float32 (count, dim) values, NaN/Inf rejected. It
additionally caches its device copy per GPU so repeated searches do not
re-upload the collection, and can wrap a device tensor directly
(`EmbeddingColumn.from_device`) for collections generated or streamed on the
GPU (bf16 storage allowed there).

`Schema` / `Table` / `gather` / `project` / `filter_rows` are the minimal
relational plumbing `vector_search_operator` needs to assemble its joined
output (vecsearch.py:123-152); they accept the reference's own Table objects
too (duck typing on .schema/.columns/.valid/.row_count).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from .errors import BoundsError, SchemaError, ShapeError

INT64 = "int64"
FLOAT64 = "float64"
STRING = "string"
DATE = "date"
_SCALAR_DTYPES = {INT64: np.dtype(np.int64), FLOAT64: np.dtype(np.float64), DATE: np.dtype(np.int32)}


@dataclass(frozen=True)
class FieldType:
    kind: str
    dim: int = 0

    def __post_init__(self):
        if self.kind == "embedding":
            if self.dim < 1:
                raise SchemaError(f"embedding dimension must be >= 1, got {self.dim}")
        elif self.kind not in _SCALAR_DTYPES and self.kind != STRING:
            raise SchemaError(f"unknown field type {self.kind!r}")

    @property
    def is_embedding(self) -> bool:
        return self.kind == "embedding"

    def __str__(self) -> str:
        return f"embedding({self.dim})" if self.is_embedding else self.kind


def embedding(dim: int) -> FieldType:
    return FieldType("embedding", dim)


def N_is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class EmbeddingColumn:
    """Fixed-dimension vectors stored as one contiguous float32 region."""

    __slots__ = ("_values", "dim", "count", "_device", "_dev_tensor", "_host_stream", "__weakref__")

    def __init__(self, values, dim: int | None = None):
        arr = np.asarray(values, dtype=np.float32)
        if arr.ndim == 1:
            if dim is None:
                raise ShapeError("flat embedding values need an explicit dim")
            if dim < 1 or arr.size % dim != 0:
                raise ShapeError(f"{arr.size} values do not tile into dim {dim}")
            arr = arr.reshape(-1, dim)
        elif arr.ndim != 2:
            raise ShapeError(f"embedding values must be 1-D or 2-D, got {arr.ndim}-D")
        if dim is not None and arr.shape[1] != dim:
            raise ShapeError(f"expected dim {dim}, got {arr.shape[1]}")
        if arr.shape[1] < 1:
            raise ShapeError("embedding dimension must be >= 1")
        if not np.all(np.isfinite(arr)):
            raise ShapeError("embedding values contain NaN or Inf")
        arr = np.ascontiguousarray(arr)
        arr.setflags(write=False)
        self._values = arr
        self.dim = arr.shape[1]
        self.count = arr.shape[0]
        self._device = {}
        self._dev_tensor = None
        self._host_stream = None

    @classmethod
    def empty(cls, dim: int) -> "EmbeddingColumn":
        return cls(np.empty((0, dim), dtype=np.float32))

    @classmethod
    def from_device(cls, tensor) -> "EmbeddingColumn":
        """Wrap a CUDA tensor (float32 or bfloat16, (count, dim)) without a
        host copy; `.values` materialises a float32 host copy on demand."""
        import torch

        if not tensor.is_cuda or tensor.dim() != 2:
            raise ShapeError("from_device needs a 2-D CUDA tensor")
        if tensor.dtype not in (torch.float32, torch.bfloat16):
            raise ShapeError("device embeddings must be float32 or bfloat16")
        # table.py:110-111; in row chunks so the check's temporaries stay small
        step = max(1, (1 << 26) // max(1, int(tensor.shape[1])))
        for i in range(0, int(tensor.shape[0]), step):
            if not bool(torch.isfinite(tensor[i:i + step]).all()):
                raise ShapeError("embedding values contain NaN or Inf")
        obj = cls.__new__(cls)
        obj._values = None
        obj.dim = int(tensor.shape[1])
        obj.count = int(tensor.shape[0])
        obj._device = {}
        obj._dev_tensor = tensor.contiguous()
        obj._host_stream = None
        return obj

    @classmethod
    def host_resident(cls, values) -> "EmbeddingColumn":
        """Keep the vectors in (pinned) HOST memory: searches stream only the
        rows the row filter selects over PCIe. `values`
        is a C-contiguous float32/bfloat16 numpy array or CPU torch tensor
        (pinned memory avoids a registration at first use)."""
        import torch
        t = values if N_is_torch(values) else torch.from_numpy(np.ascontiguousarray(values))
        if t.is_cuda or t.dim() != 2 or not t.is_contiguous():
            raise ShapeError("host_resident needs a contiguous 2-D host array")
        if t.dtype not in (torch.float32, torch.bfloat16):
            raise ShapeError("host-resident embeddings must be float32 or bfloat16")
        obj = cls.__new__(cls)
        obj._values = None
        obj.dim = int(t.shape[1])
        obj.count = int(t.shape[0])
        obj._device = {}
        obj._dev_tensor = None
        obj._host_stream = t
        return obj

    def invalidate(self) -> None:
        """The borrowed rows (from_device / host_resident) were changed in place
        by means torch cannot see (e.g. raw pointers): drop the device-side
        cached row norms so the next search recomputes them."""
        from . import _native as N
        for dc in self._device.values():
            N.check(N.load().vs_column_invalidate(dc.handle), "column_invalidate")

    @property
    def values(self) -> np.ndarray:
        if self._values is None and self._host_stream is not None:
            v = self._host_stream.float().numpy()
            v.setflags(write=False)
            self._values = v
        if self._values is None:
            v = self._dev_tensor.float().cpu().numpy()
            v.setflags(write=False)
            self._values = v
        return self._values

    @property
    def storage_dtype(self) -> str:
        t = self._dev_tensor if self._dev_tensor is not None else self._host_stream
        if t is not None and str(t.dtype) == "torch.bfloat16":
            return "bfloat16"
        return "float32"

    @property
    def nbytes(self) -> int:
        return self.count * self.dim * (2 if self.storage_dtype == "bfloat16" else 4)

    def take(self, rows) -> "EmbeddingColumn":
        return EmbeddingColumn(self.values[rows])

    def __len__(self) -> int:
        return self.count

    def __eq__(self, other) -> bool:
        return (isinstance(other, EmbeddingColumn) and self.dim == other.dim
                and self.count == other.count and np.array_equal(self.values, other.values))

    __hash__ = object.__hash__

    def __repr__(self) -> str:
        return f"EmbeddingColumn(count={self.count}, dim={self.dim})"


@dataclass(frozen=True)
class Schema:
    fields: tuple

    def __init__(self, fields: Iterable):
        norm = []
        for name, ftype in fields:
            if isinstance(ftype, str):
                ftype = FieldType(ftype)
            norm.append((name, ftype))
        names = [n for n, _ in norm]
        if len(set(names)) != len(names):
            raise SchemaError(f"duplicate field names in {names}")
        object.__setattr__(self, "fields", tuple(norm))

    @property
    def names(self) -> list:
        return [n for n, _ in self.fields]

    def type_of(self, name: str) -> FieldType:
        for n, t in self.fields:
            if n == name:
                return t
        raise SchemaError(f"unknown field {name!r}")

    def __contains__(self, name: str) -> bool:
        return any(n == name for n, _ in self.fields)

    def select(self, keep: Sequence[str]) -> "Schema":
        return Schema([(n, self.type_of(n)) for n in keep])


def _coerce(ftype: FieldType, values):
    if ftype.is_embedding:
        if isinstance(values, EmbeddingColumn) or hasattr(values, "values") and hasattr(values, "dim"):
            if values.dim != ftype.dim:
                raise ShapeError(f"embedding dim {values.dim} != declared {ftype.dim}")
            return values
        return EmbeddingColumn(values, dim=ftype.dim)
    if ftype.kind == STRING:
        arr = np.asarray(values, dtype=object)
    else:
        arr = np.asarray(values, dtype=_SCALAR_DTYPES[ftype.kind])
    arr.setflags(write=False)
    return arr


class Table:
    """Immutable table: one value array per field plus optional validity masks."""

    def __init__(self, schema: Schema, columns: dict, valid: dict | None = None):
        self.schema = schema
        cols = {}
        n = None
        for name, ftype in schema.fields:
            if name not in columns:
                raise SchemaError(f"missing column {name!r}")
            col = _coerce(ftype, columns[name])
            length = col.count if ftype.is_embedding else len(col)
            if n is None:
                n = length
            elif length != n:
                raise ShapeError(f"column {name!r} has {length} rows, expected {n}")
            cols[name] = col
        self.columns = cols
        self.valid = dict(valid or {})
        self.row_count = n or 0

    @classmethod
    def from_pairs(cls, triples) -> "Table":
        schema = Schema([(n, t) for n, t, _ in triples])
        return cls(schema, {n: v for n, _, v in triples})

    def column(self, name: str):
        if name not in self.columns:
            raise SchemaError(f"unknown field {name!r}")
        return self.columns[name]


def _gather_embedding(col, rows):
    """Rows of an embedding column. A device-resident column is gathered on
    the GPU (vs_gather_rows) and stays there: its host copy would be the whole
    collection (e.g. 41 GB), not the result rows."""
    if getattr(col, "_dev_tensor", None) is not None:
        import torch

        from .output import gather_rows
        t = col._dev_tensor
        idx = torch.from_numpy(rows).to(t.device)
        return EmbeddingColumn.from_device(gather_rows(t, idx))
    if getattr(col, "_host_stream", None) is not None:
        src = col._host_stream
        return EmbeddingColumn(src[rows].float().numpy() if N_is_torch(src) else np.asarray(src)[rows])
    return EmbeddingColumn(col.values[rows])


def gather(table, rows) -> Table:
    rows = np.asarray(rows, dtype=np.int64)
    if rows.size and (rows.min() < 0 or rows.max() >= table.row_count):
        raise BoundsError("row id outside the table")
    cols = {}
    for name, ftype in table.schema.fields:
        col = table.columns[name]
        cols[name] = _gather_embedding(col, rows) if ftype.is_embedding else np.asarray(col)[rows]
    valid = {n: np.asarray(m)[rows] for n, m in table.valid.items()}
    return Table(Schema(list(table.schema.fields)), cols, valid)


def project(table, names: Sequence[str]) -> Table:
    schema = Schema([(n, table.schema.type_of(n)) for n in names])
    return Table(schema, {n: table.columns[n] for n in names},
                 {n: m for n, m in table.valid.items() if n in names})


def filter_rows(table, mask) -> Table:
    """Order-preserving row subset (table.py:326-331)."""
    return gather(table, np.flatnonzero(np.asarray(mask, dtype=bool)))


# ---- .emb files (datagen.py:351-372) ----------------------------------------------------------

_EMB_MAGIC = b"SVEC"


def write_embeddings(path, column) -> None:
    """The reference's .emb writer: magic, <HBBQI header, float32 rows."""
    import struct
    values = column.values if hasattr(column, "values") else np.asarray(column, np.float32)
    with open(path, "wb") as f:
        f.write(_EMB_MAGIC)
        f.write(struct.pack("<HBBQI", 1, 0, 0, values.shape[0], values.shape[1]))
        f.write(np.ascontiguousarray(values, dtype="<f4").tobytes())


def read_embeddings(path, device=None) -> EmbeddingColumn:
    """Read a .emb file. device=None: a host column (the reference's reader).
    With a device (CUDA ordinal or library Context) the rows stream from the
    file through a pinned double buffer straight into a device column
    (vs_file_to_device): no host copy of the collection."""
    from . import _native as N
    from .errors import ParameterError
    count, dim, off = C_i64(), C_i32(), C_i64()
    N.check(N.load().vs_emb_info(str(path).encode(), count, dim, off), "emb_info")
    n, d = int(count.value), int(dim.value)
    if device is None:
        with open(path, "rb") as f:
            f.seek(int(off.value))
            raw = f.read(n * d * 4)
        if len(raw) != n * d * 4:
            raise ParameterError("embedding file truncated")
        return EmbeddingColumn(np.frombuffer(raw, dtype="<f4").reshape(n, d).copy())
    import torch

    from .vecindex import _ctx
    ctx = _ctx(device)
    t = torch.empty((n, d), dtype=torch.float32, device=torch.device("cuda", ctx.device))
    N.check(N.load().vs_file_to_device(ctx.handle, str(path).encode(), int(off.value), n * d * 4,
                                       t.data_ptr()), "file_to_device")
    return EmbeddingColumn.from_device(t)


def C_i64():
    import ctypes
    return ctypes.c_int64(0)


def C_i32():
    import ctypes
    return ctypes.c_int32(0)

