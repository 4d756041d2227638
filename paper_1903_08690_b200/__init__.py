"""paper_1903_08690_b200 — B200-native hybrid sparse+dense inner-product search.

Drop-in for the hot path of the reference `hybridsearch` package
(arXiv 1903.08690): the same index-build / search API, with the search
(`search_topk`, `search_batch`, `select_topk`, `adc_table`, `quantize_lut`,
`lut16_scan`, `sparse_scan`, `brute_force_topk`) running as hand-written
sm_100a CUDA kernels behind the C ABI in `include/hsb200.h`.
"""

from .types import (  # noqa: F401
    Accumulator,
    BadMagicError,
    BadVersionError,
    Codebooks,
    DenseIndex,
    FormatError,
    HybridDataset,
    HybridIndex,
    HybridIndexConfig,
    HybridVector,
    InvertedIndex,
    PQCodes,
    PruneThresholds,
    QuantizedLUT,
    ScalarQuantResidual,
    SearchResult,
    SparseVector,
    StageStats,
    TruncatedFileError,
    WhiteningTransform,
)
from .builder import (  # noqa: F401
    build_index,
    build_inverted,
    cache_sort,
    pack_codes,
    pq_encode,
    prune_split,
    sq_encode,
    train_codebooks,
    unpack_codes,
    whiten_apply,
    whiten_fit,
)
from .formats import (  # noqa: F401
    load_dataset,
    load_dense_index,
    load_device_index,
    load_index,
    load_inverted_index,
    save_dataset,
    save_dense_index,
    save_index,
    save_inverted_index,
)
from .search import (  # noqa: F401
    DeviceIndex,
    adc_table,
    brute_force_batch,
    brute_force_topk,
    device_index,
    exact_topk,
    lut16_scan,
    lut16_scan_reference,
    lut16_totals,
    quantize_lut,
    recall_at_h,
    search_batch,
    search_topk,
    select_topk,
    sparse_scan,
    stage1_scores,
)

from .search import sq_decode  # noqa: F401,E402
from .devbuild import DeviceBuiltIndex, DeviceDataset, GpuBuild  # noqa: F401
# the reference's submodule import paths (hybridsearch.dense, .sparse, ...)
from . import data, dense, harness, pipeline, sparse  # noqa: F401,E402

__version__ = "0.2.0"
