"""Import-path alias for `hybridsearch.pipeline` users (reference pipeline.py)."""
from .builder import build_index  # noqa: F401
from .search import search_batch, search_topk, select_topk, stage1_scores  # noqa: F401
from .types import HybridIndex, HybridIndexConfig, SearchResult, StageStats  # noqa: F401
from .formats import load_device_index, load_index, save_index  # noqa: F401
