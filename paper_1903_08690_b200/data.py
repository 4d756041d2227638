"""Import-path alias for `hybridsearch.data` users (reference data.py)."""
from .types import (  # noqa: F401
    BadMagicError, BadVersionError, FormatError, HybridDataset, HybridVector, SparseVector,
    TruncatedFileError,
)
from .formats import load_dataset, save_dataset  # noqa: F401
