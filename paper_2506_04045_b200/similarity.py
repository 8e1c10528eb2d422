"""Host-side CSR container mirroring ``fuzzyclust::SparseSimilarity`` (sparse.hpp:21-146).

The similarity S is symmetric, so the reference's compressed-column storage is
simultaneously CSR (sparse.hpp:18-20): ``row_ptr`` (int64, N+1), ``col_idx``
(uint32, strictly increasing per row) and ``values`` (float64, or ``None`` when
every stored value is exactly 1.0 -- the adjacency-plus-identity case of
``build_similarity``, which lets the device kernels skip the value stream).

This is host data plumbing only; all per-iteration compute runs in the CUDA
library (``paper_2506_04045_b200.capi``).
"""
from __future__ import annotations

import numpy as np

from .errors import InvalidInput, IoError


class SparseSimilarity:
    __slots__ = ("n", "row_ptr", "col_idx", "values", "frob_sq", "_device", "__weakref__")

    def __init__(self, n, row_ptr, col_idx, values=None, frob_sq=None):
        self.n = int(n)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.uint32)
        if values is not None:
            values = np.ascontiguousarray(values, dtype=np.float64)
            if values.size and bool(np.all(values == 1.0)):
                values = None  # pattern-only: 1.0 * x == x exactly, so no value stream needed
        self.values = values
        if frob_sq is None:
            frob_sq = self._frob_sq_in_stored_order()
        self.frob_sq = float(frob_sq)
        self._device = None

    # -- reference accessors (sparse.hpp:102-112) ---------------------------------
    @property
    def nnz(self) -> int:
        return int(self.col_idx.size)

    def size(self) -> int:
        return self.n

    def frob_norm(self) -> float:
        return float(np.sqrt(self.frob_sq))

    def col_rows(self, j):
        return self.col_idx[self.row_ptr[j]:self.row_ptr[j + 1]]

    def col_values(self, j):
        if self.values is None:
            return np.ones(int(self.row_ptr[j + 1] - self.row_ptr[j]))
        return self.values[self.row_ptr[j]:self.row_ptr[j + 1]]

    def _frob_sq_in_stored_order(self) -> float:
        # sparse.hpp:59-60: sequential sum of v*v in stored order.
        if self.values is None:
            return float(self.nnz)  # exact: every term is 1.0 and nnz < 2**53
        acc = 0.0
        for v in self.values.tolist():
            acc += v * v
        return acc

    # -- constructors -----------------------------------------------------------
    @staticmethod
    def from_triplets(n, triplets) -> "SparseSimilarity":
        """sparse.hpp:28-62: sort by (col, row), reject duplicates / asymmetry."""
        t = np.asarray(triplets, dtype=np.float64).reshape(-1, 3) if len(triplets) else np.zeros((0, 3))
        i = t[:, 0].astype(np.int64)
        j = t[:, 1].astype(np.int64)
        v = t[:, 2]
        # per triplet, range before value (sparse.hpp:30-33): the first failing triplet decides
        bad_r = (i < 0) | (j < 0) | (i >= n) | (j >= n)
        bad = bad_r | ~np.isfinite(v) | (v < 0.0)
        if bad.any():
            k = int(np.argmax(bad))
            raise InvalidInput("similarity: index out of range" if bad_r[k]
                               else "similarity: values must be finite and nonnegative")
        order = np.lexsort((i, j))
        i, j, v = i[order], j[order], v[order]
        if i.size > 1 and np.any((i[1:] == i[:-1]) & (j[1:] == j[:-1])):
            raise InvalidInput("similarity: duplicate coordinate entry")
        counts = np.bincount(j, minlength=n)
        row_ptr = np.zeros(n + 1, np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        s = SparseSimilarity(n, row_ptr, i.astype(np.uint32), v)
        s._validate_symmetry()
        return s

    @staticmethod
    def build_similarity(num_nodes, edges) -> "SparseSimilarity":
        """sparse.hpp:66-75: s_ij = 1 iff (i,j) is an edge or i == j; nnz = N + 2|E|."""
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        ids = np.arange(num_nodes, dtype=np.int64)
        rows = np.concatenate([ids, e[:, 0], e[:, 1]])
        cols = np.concatenate([ids, e[:, 1], e[:, 0]])
        t = np.stack([rows, cols, np.ones(rows.size)], axis=1)
        return SparseSimilarity.from_triplets(num_nodes, t)

    @staticmethod
    def load_coordinates(text: str) -> "SparseSimilarity":
        """sparse.hpp:80-100: "i j value" lines, '#' comments."""
        t = []
        max_id = 0
        for line_no, line in enumerate(text.splitlines(), 1):
            s = line.strip(" \t\r")
            if not s or s.startswith("#"):
                continue
            parts = s.split()
            try:
                i, j, v = int(parts[0]), int(parts[1]), float(parts[2])
            except (ValueError, IndexError):
                raise IoError(f"similarity parse error at line {line_no}") from None
            if i < 0 or j < 0:
                raise IoError(f"similarity parse error at line {line_no}")
            t.append((i, j, v))
            max_id = max(max_id, i, j)
        if not t:
            raise IoError("similarity file is empty")
        return SparseSimilarity.from_triplets(max_id + 1, t)

    def _validate_symmetry(self) -> None:
        """sparse.hpp:115-139 (vectorised): strictly increasing rows, mirrored pattern and values."""
        n = self.n
        rp, ci = self.row_ptr, self.col_idx.astype(np.int64)
        col_of = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
        if ci.size > 1:
            same = col_of[1:] == col_of[:-1]
            if np.any(same & (ci[1:] <= ci[:-1])):
                raise InvalidInput("similarity: row indices must be strictly increasing")
        key = col_of * n + ci
        mkey = ci * n + col_of
        pos = np.searchsorted(key, mkey)
        pos_c = np.minimum(pos, max(key.size - 1, 0))
        if key.size and np.any(key[pos_c] != mkey):
            raise InvalidInput("similarity: matrix is not symmetric")
        if self.values is not None and np.any(self.values[pos_c] != self.values):
            bad = int(np.nonzero(self.values[pos_c] != self.values)[0][0])
            raise InvalidInput(f"similarity: asymmetric values at ({int(ci[bad])}, {int(col_of[bad])})")

    def degrees(self):
        return np.diff(self.row_ptr)

    def __repr__(self):
        return f"SparseSimilarity(n={self.n}, nnz={self.nnz}, pattern_only={self.values is None})"
