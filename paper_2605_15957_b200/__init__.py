"""B200-native filtered vector-search operator (arXiv 2605.15957, Vec-H).

Drop-in for the reference `sqlvs` vector-search path: the same entry points
(enn_search, FlatIndex, IvfIndex, save_index/load_index,
vector_search_operator) and exceptions, executed by hand-written sm_100a
kernels behind the C ABI in include/vs_b200.h (libvsb200.so, ctypes).
"""

from .errors import (CapExceededError, EmptyInputError, ParameterError, PlacementError,  # noqa: F401
                     SchemaError, ShapeError, SqlVsError)
from .table import (EmbeddingColumn, FieldType, Schema, Table, embedding, read_embeddings,  # noqa: F401
                    write_embeddings)
from .vecindex import (INNER_PRODUCT, NON_OWNING, OWNING, SQUARED_L2, FlatIndex,  # noqa: F401
                       IvfIndex, NeighborTable, SearchParams, enn_search, load_index, save_index)
from .vecsearch import VsStats, oversample_postfilter, vector_search_operator  # noqa: F401
from . import predicate  # noqa: F401,E402
from . import output  # noqa: F401,E402
from .group import DeviceGroup, use_devices  # noqa: F401,E402

__all__ = [
    "SearchParams", "NeighborTable", "enn_search", "FlatIndex", "IvfIndex", "save_index",
    "load_index", "vector_search_operator", "oversample_postfilter", "VsStats",
    "EmbeddingColumn", "Table", "Schema", "FieldType", "embedding", "read_embeddings", "write_embeddings",
    "DeviceGroup", "use_devices",
]
