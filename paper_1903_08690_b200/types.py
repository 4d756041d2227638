"""Host-side data and index types of the drop-in API.

Field names, defaults and validation mirror the reference `hybridsearch`
package so code written against it (and reference-built indices) work
unchanged:

    SparseVector / HybridVector / HybridDataset     data.py:34-162
    FormatError family                               data.py:18-31
    HybridIndexConfig / StageStats / SearchResult    pipeline.py:36-89
    HybridIndex                                      pipeline.py:92-116
    PruneThresholds                                  sparse.py:33-63
    InvertedIndex (array form + `lists` view)        sparse.py:172-216
    Accumulator                                      sparse.py:238-258
    Codebooks / PQCodes / QuantizedLUT               dense.py:25-54, 183-209, 231-245
    WhiteningTransform / ScalarQuantResidual         dense.py:320-330, 361-378
    DenseIndex                                       dense.py:431-446

These are containers; all search arithmetic runs on the GPU (`search.py`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

DEFAULT_LINE_CAPACITY = 16
LUT16_CENTERS = 16


class FormatError(ValueError):
    """Malformed dataset / index file."""


class BadMagicError(FormatError):
    """Unexpected magic bytes."""


class BadVersionError(FormatError):
    """Unsupported format version."""


class TruncatedFileError(FormatError):
    """File ended before its declared payload."""


# ----------------------------------------------------------------------------
# vectors and datasets
# ----------------------------------------------------------------------------
@dataclass
class SparseVector:
    """Coordinate-list sparse vector: int64 dims (ascending), f32 values."""

    dims: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.dims = np.asarray(self.dims, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=np.float32)

    @property
    def nnz(self) -> int:
        return int(self.dims.shape[0])

    def to_dense(self, d: int) -> np.ndarray:
        out = np.zeros(d, dtype=np.float64)
        out[self.dims] = self.values
        return out

    def dot(self, other: "SparseVector") -> float:
        common, ia, ib = np.intersect1d(self.dims, other.dims, assume_unique=True,
                                        return_indices=True)
        if common.size == 0:
            return 0.0
        return float(np.sum(self.values[ia].astype(np.float64) * other.values[ib].astype(np.float64)))


@dataclass
class HybridVector:
    """A sparse part and a fixed-length f32 dense part."""

    sparse: SparseVector
    dense: np.ndarray

    def __post_init__(self):
        self.dense = np.asarray(self.dense, dtype=np.float32)


@dataclass
class HybridDataset:
    """N hybrid vectors: (n, d_sparse) f32 CSR with sorted indices + (n, d_dense) f32."""

    sparse: sp.csr_matrix
    dense: np.ndarray

    def __post_init__(self):
        self.dense = np.ascontiguousarray(self.dense, dtype=np.float32)
        if self.dense.ndim != 2:
            self.dense = self.dense.reshape(self.sparse.shape[0], -1)
        if self.sparse.shape[0] != self.dense.shape[0]:
            raise ValueError("sparse/dense row counts differ")
        self.sparse = sp.csr_matrix(self.sparse)
        self.sparse.sort_indices()

    @property
    def n(self) -> int:
        return int(self.sparse.shape[0])

    @property
    def d_sparse(self) -> int:
        return int(self.sparse.shape[1])

    @property
    def d_dense(self) -> int:
        return int(self.dense.shape[1])

    def point(self, i: int) -> HybridVector:
        lo, hi = self.sparse.indptr[i], self.sparse.indptr[i + 1]
        return HybridVector(SparseVector(self.sparse.indices[lo:hi], self.sparse.data[lo:hi]),
                            self.dense[i])

    def points(self):
        for i in range(self.n):
            yield self.point(i)

    @staticmethod
    def empty(d_sparse: int, d_dense: int) -> "HybridDataset":
        return HybridDataset(sp.csr_matrix((0, d_sparse), dtype=np.float32),
                             np.zeros((0, d_dense), dtype=np.float32))


# ----------------------------------------------------------------------------
# sparse index
# ----------------------------------------------------------------------------
@dataclass
class PruneThresholds:
    """Per-dim magnitude cutoffs: scan index / residual / discarded (sparse.py:33-63)."""

    data_min: float | np.ndarray | None = None
    residual_min: float | np.ndarray = 0.0
    top_t: int | None = None

    def __post_init__(self):
        if self.top_t is not None and self.top_t < 0:
            raise ValueError("top_t must be >= 0")
        if self.data_min is None and self.top_t is None:
            self.data_min = 0.0


def invert_permutation(order: np.ndarray) -> np.ndarray:
    order = np.asarray(order, dtype=np.int64)
    pos = np.empty(order.shape[0], dtype=np.int64)
    pos[order] = np.arange(order.shape[0], dtype=np.int64)
    return pos


class InvertedIndex:
    """Posting lists in layout order, held as CSR over the active dims.

    `dims` (int64, ascending) are the dims with a non-empty list, list j spans
    `ids[ptr[j]:ptr[j+1]]` (u32 layout slots, strictly ascending) and the
    matching `w` (f32).  `lists` gives the reference's dict view
    (sparse.py:183) on demand, and the reference constructor signature
    `InvertedIndex(n, d_sparse, order, lists)` is accepted.
    """

    def __init__(self, n, d_sparse, order, lists=None, *, dims=None, ptr=None, ids=None, w=None):
        self.n = int(n)
        self.d_sparse = int(d_sparse)
        self.order = np.asarray(order, dtype=np.int64)
        if lists is not None:
            keys = np.array(sorted(int(k) for k in lists), dtype=np.int64)
            lens = np.array([len(lists[int(k)][0]) for k in keys], dtype=np.int64)
            self.dims = keys
            self.ptr = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
            self.ids = (np.concatenate([lists[int(k)][0] for k in keys]) if len(keys)
                        else np.zeros(0)).astype(np.uint32)
            self.w = (np.concatenate([lists[int(k)][1] for k in keys]) if len(keys)
                      else np.zeros(0)).astype(np.float32)
        else:
            self.dims = np.asarray(dims if dims is not None else [], dtype=np.int64)
            self.ptr = np.asarray(ptr if ptr is not None else [0], dtype=np.int64)
            self.ids = np.asarray(ids if ids is not None else [], dtype=np.uint32)
            self.w = np.asarray(w if w is not None else [], dtype=np.float32)
        self._lists = None
        self.pos = invert_permutation(self.order)

    @property
    def lists(self) -> dict:
        if self._lists is None:
            self._lists = {int(j): (self.ids[self.ptr[i]:self.ptr[i + 1]],
                                    self.w[self.ptr[i]:self.ptr[i + 1]])
                           for i, j in enumerate(self.dims)}
        return self._lists

    @property
    def nnz(self) -> int:
        return int(self.ids.shape[0])

    @property
    def nnz_per_dim(self) -> np.ndarray:
        out = np.zeros(self.d_sparse, dtype=np.int64)
        out[self.dims] = np.diff(self.ptr)
        return out

    def memory_bytes(self) -> int:
        return int(self.order.nbytes + self.ids.nbytes + self.w.nbytes)

    def to_csr(self) -> sp.csr_matrix:
        cols = np.repeat(self.dims, np.diff(self.ptr))
        rows = self.order[self.ids.astype(np.int64)]
        out = sp.coo_matrix((self.w, (rows, cols)), shape=(self.n, self.d_sparse),
                            dtype=np.float32).tocsr()
        out.sort_indices()
        return out


@dataclass
class Accumulator:
    """Per-query f64 score buffer in layout order (+ cache-line counter)."""

    scores: np.ndarray
    line_capacity: int = DEFAULT_LINE_CAPACITY
    lines_touched: int = 0

    @staticmethod
    def zeros(n: int, line_capacity: int = DEFAULT_LINE_CAPACITY) -> "Accumulator":
        if line_capacity <= 0:
            raise ValueError("line_capacity must be positive")
        return Accumulator(np.zeros(n, dtype=np.float64), line_capacity)

    def reset(self):
        self.scores[:] = 0.0
        self.lines_touched = 0


# ----------------------------------------------------------------------------
# dense index
# ----------------------------------------------------------------------------
@dataclass
class Codebooks:
    """Per-subspace centers over contiguous dense spans."""

    subdims: np.ndarray
    centers: list
    objective_history: list | None = None

    @property
    def n_subspaces(self) -> int:
        return len(self.centers)

    @property
    def n_centers(self) -> int:
        return int(self.centers[0].shape[0]) if self.centers else 0

    @property
    def d_dense(self) -> int:
        return int(np.sum(self.subdims))

    def slices(self) -> list:
        e = np.concatenate(([0], np.cumsum(self.subdims)))
        return [slice(int(a), int(b)) for a, b in zip(e[:-1], e[1:])]

    def reconstruct(self, codes: np.ndarray) -> np.ndarray:
        out = np.empty((codes.shape[0], self.d_dense), dtype=np.float32)
        for k, sl in enumerate(self.slices()):
            out[:, sl] = self.centers[k][codes[:, k]]
        return out


@dataclass
class PQCodes:
    """Codes in layout order; 4-bit codes packed pair-major (ceil(K/2), n)."""

    n: int
    n_subspaces: int
    n_centers: int
    packed: np.ndarray | None = None
    bytes_wide: np.ndarray | None = None

    @staticmethod
    def from_codes(codes: np.ndarray, n_centers: int) -> "PQCodes":
        from .builder import pack_codes

        n, K = codes.shape
        if n_centers == LUT16_CENTERS:
            return PQCodes(n, K, n_centers, packed=pack_codes(codes))
        if n_centers == 256:
            return PQCodes(n, K, n_centers, bytes_wide=np.ascontiguousarray(codes, dtype=np.uint8))
        raise ValueError("n_centers must be 16 or 256")

    def unpacked(self) -> np.ndarray:
        from .builder import unpack_codes

        if self.packed is not None:
            return unpack_codes(self.packed, self.n_subspaces)
        return self.bytes_wide

    def memory_bytes(self) -> int:
        arr = self.packed if self.packed is not None else self.bytes_wide
        return 0 if arr is None else int(arr.nbytes)


@dataclass
class QuantizedLUT:
    """u8 table, per-subspace bias, one shared scale (dense.py:231-245)."""

    bias: np.ndarray
    scale: float
    table: np.ndarray
    _bias_total: float | None = field(default=None, repr=False)

    @property
    def bias_total(self) -> float:
        if self._bias_total is None:
            self._bias_total = float(np.sum(self.bias))
        return self._bias_total


@dataclass
class WhiteningTransform:
    forward: np.ndarray
    inverse_t: np.ndarray
    mean: np.ndarray


@dataclass
class ScalarQuantResidual:
    """Per-dim 8-bit affine codes: value ~ lo + step * (code + 0.5)."""

    lo: np.ndarray
    step: np.ndarray
    codes: np.ndarray

    def decode(self, rows=slice(None)) -> np.ndarray:
        """f64 rows lo + step * (code + 0.5), on the GPU (dense.py:369-371)."""
        from .search import sq_residual_decode

        return sq_residual_decode(self, rows)

    def dot(self, rows, q) -> np.ndarray:
        """decode(rows) @ q, on the GPU (dense.py:373-375)."""
        from .search import sq_residual_dot

        return sq_residual_dot(self, rows, q)

    def memory_bytes(self) -> int:
        return int(self.lo.nbytes + self.step.nbytes + self.codes.nbytes)


@dataclass
class DenseIndex:
    codebooks: Codebooks
    codes: PQCodes
    residual: ScalarQuantResidual | None = None
    whitening: WhiteningTransform | None = None

    def memory_bytes(self) -> int:
        total = self.codes.memory_bytes() + sum(int(c.nbytes) for c in self.codebooks.centers)
        if self.residual is not None:
            total += self.residual.memory_bytes()
        return total


# ----------------------------------------------------------------------------
# pipeline types
# ----------------------------------------------------------------------------
@dataclass
class HybridIndexConfig:
    """Build- and query-time knobs, same names/defaults as pipeline.py:36-74."""

    overfetch: float = 10.0
    retain: float = 3.0
    h: int = 20
    top_t: int | None = 128
    data_threshold: float | list | None = None
    residual_threshold: float | list = 0.0
    pq_subspaces: int | None = None
    pq_centers: int = 16
    use_whitening: bool = True
    exact_final_rerank: bool = False
    sparse_weight: float = 1.0
    dense_weight: float = 1.0
    kmeans_iters: int = 25
    train_sample: int = 50_000
    line_capacity: int = DEFAULT_LINE_CAPACITY
    seed: int = 0

    def __post_init__(self):
        if not (self.overfetch >= self.retain >= 1.0):
            raise ValueError("need overfetch >= retain >= 1")
        if self.h < 1:
            raise ValueError("h must be >= 1")

    def prune_thresholds(self) -> PruneThresholds:
        if self.data_threshold is not None:
            return PruneThresholds(data_min=np.asarray(self.data_threshold, dtype=np.float64),
                                   residual_min=np.asarray(self.residual_threshold))
        return PruneThresholds(top_t=self.top_t, residual_min=np.asarray(self.residual_threshold))


# slotted: a batch of 10^3-10^4 results is built on every search_batch call
@dataclass(slots=True)
class StageStats:
    candidates: list = field(default_factory=list)
    seconds: list = field(default_factory=list)


@dataclass(slots=True)
class SearchResult:
    ids: np.ndarray
    scores: np.ndarray
    stages: StageStats


@dataclass
class HybridIndex:
    """All per-dataset search structures, sharing one layout permutation."""

    config: HybridIndexConfig
    n: int
    d_sparse: int
    d_dense: int
    order: np.ndarray
    sparse_index: InvertedIndex
    sparse_residual: sp.csr_matrix
    dense_index: DenseIndex | None
    dataset: HybridDataset | None = None

    @property
    def pos(self) -> np.ndarray:
        return self.sparse_index.pos

    def memory_bytes(self) -> int:
        r = self.sparse_residual
        total = self.sparse_index.memory_bytes() + r.data.nbytes + r.indices.nbytes + r.indptr.nbytes
        if self.dense_index is not None:
            total += self.dense_index.memory_bytes()
        return int(total)
