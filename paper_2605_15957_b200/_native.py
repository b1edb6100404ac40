"""ctypes binding of the C ABI in include/vs_b200.h (libvsb200.so, built
in-tree by `__graft_entry__.build()`).

There is deliberately no fallback: if the shared object is missing or cannot
be loaded, every search raises NativeLibraryMissing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from . import errors as E

LIB_NAME = "libvsb200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

VS_OK, VS_ERR_SHAPE, VS_ERR_EMPTY_INPUT, VS_ERR_PARAMETER = 0, 1, 2, 3
VS_ERR_CAP_EXCEEDED, VS_ERR_PLACEMENT, VS_ERR_CUDA, VS_ERR_INTERNAL, VS_ERR_NCCL = 4, 5, 6, 7, 8
METRIC_CODE = {"squared_l2": 0, "inner_product": 1}
DTYPE_F32, DTYPE_BF16 = 0, 1
OPT_ENN_KERNEL, OPT_IVF_KERNEL, OPT_CAND_SLACK, OPT_FORCE_RETRY, OPT_TIMING = 1, 2, 3, 4, 5
OPT_STREAM_CHUNK = 6
OPT_IVF_CHUNK_ROWS = 7
OPT_COARSE = 8
KERNEL_CLASSES = ("select", "enn_scan", "rerank", "coarse", "ivf_scan", "ivf_rerank", "merge", "stage",
                  "coarse_rerank")
STAT_LAUNCHES, STAT_OVERFLOW_QUERIES, STAT_SURVIVORS, STAT_LAST_ENN_KERNEL = 0, 1, 2, 3
STAT_NEAR_TIES = 4

_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64

# name -> (restype, argtypes); every exported symbol of include/vs_b200.h
SIGNATURES = {
    "vs_last_error": (C.c_char_p, []),
    "vs_topk_cap": (_i32, []),
    "vs_version": (_i32, []),
    "vs_ctx_create": (C.c_int, [_i32, C.POINTER(_vp)]),
    "vs_ctx_destroy": (C.c_int, [_vp]),
    "vs_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "vs_ctx_synchronize": (C.c_int, [_vp]),
    "vs_ctx_set_option": (C.c_int, [_vp, _i32, _i64]),
    "vs_ctx_stats": (C.c_int, [_vp, _vp, _i32]),
    "vs_ctx_kernel_times": (C.c_int, [_vp, _vp, _vp, _i32, _i32]),
    "vs_column_create": (C.c_int, [_vp, _vp, _i64, _i32, _i32, C.POINTER(_vp)]),
    "vs_column_wrap": (C.c_int, [_vp, _vp, _i64, _i32, _i32, C.POINTER(_vp)]),
    "vs_column_wrap_host": (C.c_int, [_vp, _vp, _i64, _i32, _i32, C.POINTER(_vp)]),
    "vs_column_free": (C.c_int, [_vp]),
    "vs_column_invalidate": (C.c_int, [_vp]),
    "vs_column_info": (C.c_int, [_vp, _vp, _vp, _vp]),
    "vs_enn_search": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp, _i64, _i32, _i32, _i64,
                                _vp, _vp, _vp, C.POINTER(_i64)]),
    "vs_enn_search_begin": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp, _i64, _i32, _i32, _vp,
                                      C.POINTER(_i64)]),
    "vs_enn_search_finish": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "vs_union_kth": (C.c_int, [_vp, _i32, _i64, _i32, _vp, _vp]),
    "vs_bitmap_compare": (C.c_int, [_vp, _vp, _i32, _i64, _i32, C.c_double, _vp, _vp]),
    "vs_bitmap_isin": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _i64, _vp]),
    "vs_bitmap_combine": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "vs_postfilter": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _i64, _i32,
                                _vp, _vp, _vp, _vp]),
    "vs_results_flatten": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _i64, _vp, _vp, _vp, _vp,
                                     C.POINTER(_i64)]),
    "vs_gather_rows": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "vs_topk_merge": (C.c_int, [_vp, _i32, _i64, _i32, _vp, _vp, _vp, _i32, _i32,
                                _vp, _vp, _vp]),
    "vs_ivf_create": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _i32, _i32, _vp, _vp,
                                C.POINTER(_vp)]),
    "vs_ivf_wrap": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _i32, _i32, C.POINTER(_vp)]),
    "vs_ivf_assign": (C.c_int, [_vp, _vp, _vp, _vp]),
    "vs_ivf_build": (C.c_int, [_vp, _vp, _i32, _vp, C.c_uint64, _i32, _i32, C.POINTER(_vp)]),
    "vs_ivf_info": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "vs_ivf_export": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "vs_ivf_search": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp, _vp,
                                _vp, C.POINTER(_i64)]),
    "vs_ivf_set_owned": (C.c_int, [_vp, _vp]),
    "vs_ivf_probe": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "vs_ivf_search_probed": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _i64, _i32, _vp, _i32, _vp, _vp, _vp,
                                       C.POINTER(_i64)]),
    "vs_ivf_free": (C.c_int, [_vp]),
    "vs_group_create": (C.c_int, [_i32, _vp, C.POINTER(_vp)]),
    "vs_group_destroy": (C.c_int, [_vp]),
    "vs_group_info": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    "vs_group_ctx": (_vp, [_vp, _i32]),
    "vs_group_enn_search": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _vp, _i64, _i32, _i32, _vp, _vp, _vp,
                                      C.POINTER(_i64)]),
    "vs_group_ivf_search": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp, _vp,
                                      C.POINTER(_i64)]),
    "vs_ivf_load": (C.c_int, [_vp, C.c_char_p, _vp, _vp, C.POINTER(_vp)]),
    "vs_emb_info": (C.c_int, [C.c_char_p, C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i64)]),
    "vs_file_to_device": (C.c_int, [_vp, C.c_char_p, _i64, _i64, _vp]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libvsb200.so once (raises NativeLibraryMissing)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("VS_B200_LIB", str(LIB_PATH))
        if not Path(path).exists():
            raise E.NativeLibraryMissing(
                f"{path} not found: run `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = C.CDLL(path)
        except OSError as exc:  # pragma: no cover - depends on the box
            raise E.NativeLibraryMissing(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int, what: str = "") -> None:
    if status == VS_OK:
        return
    msg = load().vs_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == VS_ERR_SHAPE:
        raise E.ShapeError(msg)
    if status == VS_ERR_EMPTY_INPUT:
        raise E.EmptyInputError(msg)
    if status == VS_ERR_PARAMETER:
        raise E.ParameterError(msg)
    if status == VS_ERR_CAP_EXCEEDED:
        err = E.CapExceededError(0, load().vs_topk_cap())
        err.args = (msg,)
        raise err
    if status == VS_ERR_PLACEMENT:
        raise E.PlacementError(msg)
    if status == VS_ERR_NCCL:
        raise E.CollectiveError(msg)
    raise E.DeviceError(f"status {status}: {msg}")


def topk_cap() -> int:
    return int(load().vs_topk_cap())


# ---- pointer plumbing -------------------------------------------------------------------


def is_torch(x) -> bool:
    return type(x).__module__.startswith("torch") and hasattr(x, "data_ptr")


def ptr(x):
    """Raw address of a numpy array / torch tensor (None stays None)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise E.ParameterError("array must be C-contiguous")
        return x.ctypes.data
    if is_torch(x):
        if not x.is_contiguous():
            raise E.ParameterError("tensor must be contiguous")
        return x.data_ptr()
    raise TypeError(f"unsupported buffer type {type(x)!r}")


class Context:
    """One library context per CUDA device (one process per GPU)."""

    _by_device: dict = {}

    def __init__(self, device: int = 0):
        lib = load()
        h = _vp()
        check(lib.vs_ctx_create(int(device), C.byref(h)), "vs_ctx_create")
        self.handle = h
        self.device = int(device)

    @classmethod
    def borrowed(cls, handle, device: int, owner=None) -> "Context":
        """A member context of a device group (the group destroys it)."""
        obj = cls.__new__(cls)
        obj.handle = _vp(handle)
        obj.device = int(device)
        obj._owner = owner       # keeps the group alive while the member is used
        return obj

    def close(self) -> None:
        """Destroy the library context (scratch arena, streams). Columns and
        indexes created through it stay valid until they are freed."""
        if getattr(self, "_owner", None) is not None:
            return
        h, self.handle = getattr(self, "handle", None), None
        if h:
            load().vs_ctx_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0")) if _torch_cuda_device() is None \
                else _torch_cuda_device()
        ctx = cls._by_device.get(device)
        if ctx is None:
            ctx = cls._by_device[device] = Context(device)
        return ctx

    def set_stream(self, stream_handle: int | None) -> None:
        check(load().vs_ctx_set_stream(self.handle, stream_handle), "vs_ctx_set_stream")

    def synchronize(self) -> None:
        check(load().vs_ctx_synchronize(self.handle))

    def set_option(self, key: int, value: int) -> None:
        check(load().vs_ctx_set_option(self.handle, key, int(value)))

    def kernel_times(self, reset: bool = False) -> dict:
        """{class: (total_ns, launches)} of CUDA-event-timed kernel classes."""
        n = len(KERNEL_CLASSES)
        ns = np.zeros(n, np.int64)
        cnt = np.zeros(n, np.int64)
        check(load().vs_ctx_kernel_times(self.handle, ns.ctypes.data, cnt.ctypes.data, n, int(reset)))
        return {name: (int(ns[i]), int(cnt[i])) for i, name in enumerate(KERNEL_CLASSES)}

    def stats(self) -> list:
        out = np.zeros(8, np.int64)
        check(load().vs_ctx_stats(self.handle, out.ctypes.data, 8))
        return out.tolist()


def _torch_cuda_device():
    try:
        import torch  # noqa: F401
    except Exception:  # pragma: no cover
        return None
    import torch
    if not torch.cuda.is_available():
        return None
    return torch.cuda.current_device()


class DeviceColumn:
    """Library-owned (or borrowed) device copy of an embedding column."""

    def __init__(self, ctx: Context, src, n: int, d: int, dtype: int = DTYPE_F32,
                 borrow: bool = False, keepalive=None, host: bool = False):
        lib = load()
        h = _vp()
        fn = lib.vs_column_wrap_host if host else lib.vs_column_wrap if borrow else lib.vs_column_create
        borrow = borrow or host
        check(fn(ctx.handle, ptr(src) if not isinstance(src, int) else src, int(n), int(d),
                 int(dtype), C.byref(h)), "column")
        self.handle = h
        self.ctx = ctx
        self.n, self.d, self.dtype = int(n), int(d), int(dtype)
        self._keepalive = keepalive if borrow else None
        self._version = getattr(keepalive, "_version", None)

    def refresh(self) -> None:
        """A borrowed torch tensor modified in place since the last search
        (torch bumps `_version`) gets its cached row norms invalidated."""
        t = self._keepalive
        v = getattr(t, "_version", None)
        if v is not None and v != self._version:
            check(load().vs_column_invalidate(self.handle), "column_invalidate")
            self._version = v

    def __del__(self):
        try:
            if self.handle:
                load().vs_column_free(self.handle)
                self.handle = None
        except Exception:
            pass


class DeviceIvf:
    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.handle = handle
        self.owned_key = None
        nlist, d, metric, dtype = _i32(), _i32(), _i32(), _i32()
        n_total = _i64()
        check(load().vs_ivf_info(handle, C.byref(nlist), C.byref(d), C.byref(n_total),
                                 C.byref(metric), C.byref(dtype)))
        self.nlist, self.d, self.n_total = nlist.value, d.value, n_total.value
        self.metric, self.dtype = metric.value, dtype.value

    def __del__(self):
        try:
            if self.handle:
                load().vs_ivf_free(self.handle)
                self.handle = None
        except Exception:
            pass
