"""Import-path alias for the recall oracle of `hybridsearch.harness`."""
from .search import brute_force_batch, brute_force_topk, recall_at_h  # noqa: F401
