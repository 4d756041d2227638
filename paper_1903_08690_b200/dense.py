"""Import-path alias for `hybridsearch.dense` users (reference dense.py)."""
from .builder import (  # noqa: F401
    pack_codes, pq_encode, sq_encode, subspace_widths, train_codebooks, unpack_codes,
    whiten_apply, whiten_fit,
)
from .search import (  # noqa: F401
    adc_table, lut16_scan, lut16_scan_reference, quantize_lut, sq_decode,
)
from .types import (  # noqa: F401
    LUT16_CENTERS, Codebooks, DenseIndex, PQCodes, QuantizedLUT, ScalarQuantResidual,
    WhiteningTransform,
)
from .formats import load_dense_index, save_dense_index  # noqa: F401
