"""Import-path alias for `hybridsearch.sparse` users (reference sparse.py)."""
from .builder import build_inverted, cache_sort, prune_split  # noqa: F401
from .search import sparse_scan  # noqa: F401
from .types import (  # noqa: F401
    DEFAULT_LINE_CAPACITY, Accumulator, InvertedIndex, PruneThresholds, invert_permutation,
)
from .formats import load_inverted_index, save_inverted_index  # noqa: F401
